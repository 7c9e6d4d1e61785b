# Round 2: batched scans (one round trip per 512 chunks), contiguous schedule default.
set -x
O=gpurun_out/r02g5
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fabric.py tests/test_gpu_chunked.py -q -x > $O/pytest_quick.log 2>&1; echo "rc=$?" >> $O/pytest_quick.log
for dg in 0 4; do
  SMILE_GATE_DIAG=$dg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gate1|scan1" -c 6 --csv --log-file $O/l_$dg.csv \
    python bench.py --config c2 --mode bilevel --steps 2 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > /dev/null 2>&1
done
timeout 300 python bench.py --steps 50 --no-cpu --no-e2e > $O/bench_c2.log 2>&1
timeout 300 python bench.py --config c4 --steps 20 --no-cpu --no-e2e > $O/bench_c4.log 2>&1
timeout 300 python bench.py --config c5 --steps 20 --no-cpu --no-e2e > $O/bench_c5.log 2>&1
for f in "50,5" "12.5,20"; do
  for c in e4x8 e4x8_c1; do
    timeout 600 python bench.py --config $c --fabric $f --steps 20 --no-cpu --no-e2e > $O/bench_fabric_${c}_${f/,/_}.log 2>&1
  done
done
echo done
