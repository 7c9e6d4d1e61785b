set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_router or fused_gate" > gpurun_out/pt_gate.log 2>&1; echo "rc=$?" >> gpurun_out/pt_gate.log
timeout 900 python -m pytest tests -m gpu -q -x -k "not multigpu" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for sw in 1 0; do SMILE_GATE_SWAP=$sw timeout 600 python bench.py --no-cpu --no-e2e --steps 100 --mode bilevel > gpurun_out/bench_swap$sw.log 2>&1; done
SMILE_GATE_SWAP=1 timeout 600 python bench.py --no-cpu --no-e2e --steps 10 --config c4 --mode bilevel > gpurun_out/bench_c4_swap1.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --mode bilevel --clock-ms 0"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gate1" -c 3 --csv --log-file gpurun_out/gate_swap.csv $CMD > gpurun_out/ncu_g.log 2>&1
echo done
