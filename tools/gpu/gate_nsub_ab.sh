set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_backward.py -q -x > gpurun_out/pt_bwd.log 2>&1; echo "rc=$?" >> gpurun_out/pt_bwd.log
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --mode bilevel --clock-ms 0"
for ns in 1 2; do
  SMILE_GATE_NSUB=$ns timeout 300 $CMD > gpurun_out/plain_ns$ns.log 2>&1 && \
  SMILE_GATE_NSUB=$ns timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gate1_tc -c 3 --csv --log-file gpurun_out/gate_ns$ns.csv $CMD > gpurun_out/ncu_ns$ns.log 2>&1
done
for ns in 1 2; do SMILE_GATE_NSUB=$ns timeout 600 python bench.py --no-cpu --no-e2e --steps 100 --mode bilevel > gpurun_out/bench_ns$ns.log 2>&1; done
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu --mode bilevel > gpurun_out/bench_c3.log 2>&1
CMD3="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --mode bilevel --clock-ms 0"
timeout 300 $CMD3 > gpurun_out/plain3.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c3.csv $CMD3 > gpurun_out/ncu_launch3.log 2>&1
echo done
