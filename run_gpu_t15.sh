set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_backward.py -q > gpurun_out/pt_bwd.log 2>&1; echo "rc=$?" >> gpurun_out/pt_bwd.log
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_router" > gpurun_out/pt_gate.log 2>&1; echo "rc=$?" >> gpurun_out/pt_gate.log
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c3_peer.log 2>&1
timeout 600 python bench.py --no-cpu --no-e2e --steps 100 > gpurun_out/bench_n1.log 2>&1
timeout 600 python bench.py --config c4 --no-cpu --no-e2e --steps 10 > gpurun_out/bench_c4.log 2>&1
CMD="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --mode bilevel --clock-ms 0"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c3.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo done
