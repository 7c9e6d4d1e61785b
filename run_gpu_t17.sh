set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_gate_dispatch" > gpurun_out/pt_fgd.log 2>&1; echo "rc=$?" >> gpurun_out/pt_fgd.log
timeout 900 python -m pytest tests -m gpu -q -x -k "not multigpu" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu --no-e2e --steps 100 > gpurun_out/bench_fused.log 2>&1
timeout 600 python bench.py --no-cpu --no-e2e --steps 100 --unfused-gate > gpurun_out/bench_unfused.log 2>&1
timeout 600 python bench.py --config c4 --no-cpu --no-e2e --steps 10 > gpurun_out/bench_c4.log 2>&1
echo done
