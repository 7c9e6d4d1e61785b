# Round 2: swapped gate with the level-1 scan by in-kernel look-back (no scan kernel).
set -x
O=gpurun_out/r02g9
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_topk.py tests/test_gpu_chunked.py -q -x > $O/pytest_quick.log 2>&1; echo "rc=$?" >> $O/pytest_quick.log
for lb in 1 0; do
  SMILE_GATE_LOOKBACK=$lb timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gate1|scan1" -c 4 --csv --log-file $O/l_lb$lb.csv \
    python bench.py --config c2 --mode bilevel --steps 2 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > /dev/null 2>&1
done
for i in 1 2; do for lb in 1 0; do
  SMILE_GATE_LOOKBACK=$lb timeout 300 python bench.py --steps 50 --no-cpu --no-e2e > $O/bench_c2_lb${lb}_$i.log 2>&1
done; done
for c in c4 c5; do for lb in 1 0; do SMILE_GATE_LOOKBACK=$lb timeout 300 python bench.py --config $c --steps 20 --no-cpu --no-e2e > $O/bench_${c}_lb$lb.log 2>&1; done; done
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x > $O/pytest_fullsize.log 2>&1; echo "rc=$?" >> $O/pytest_fullsize.log
echo done
