set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_router or fused_gate_dispatch" > gpurun_out/pt_gate.log 2>&1; echo "rc=$?" >> gpurun_out/pt_gate.log
timeout 600 python -m pytest tests/test_gpu_backward.py -q -x > gpurun_out/pt_bwd.log 2>&1; echo "rc=$?" >> gpurun_out/pt_bwd.log
timeout 600 python bench.py --no-cpu --no-e2e --steps 100 > gpurun_out/bench_n1.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --mode bilevel --clock-ms 0"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo done
