# Round 2: swapped gate on 128-token blocks (rounds + tail, two epilogue groups), top-k, all tests.
set -x
O=gpurun_out/r02g7
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_topk.py tests/test_gpu_parity.py -q -x -k "topk or fused_router or c1_full or shapes or fused_gate or bench_launch" > $O/pytest_quick.log 2>&1; echo "rc=$?" >> $O/pytest_quick.log
for sch in rounds contig; do
  SMILE_GATE_SCHED=$sch timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gate1|scan1|router_split" -c 6 --csv --log-file $O/l_$sch.csv \
    python bench.py --config c2 --mode bilevel --steps 2 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > /dev/null 2>&1
done
for i in 1 2; do timeout 300 python bench.py --steps 50 --no-cpu --no-e2e > $O/bench_c2_$i.log 2>&1; done
timeout 300 python bench.py --config c4 --steps 20 --no-cpu --no-e2e > $O/bench_c4.log 2>&1
timeout 300 python bench.py --config c5 --steps 20 --no-cpu --no-e2e > $O/bench_c5.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -k "not multigpu" > $O/pytest_all.log 2>&1; echo "rc=$?" >> $O/pytest_all.log
echo done
