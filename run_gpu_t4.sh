set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_router" > gpurun_out/pt_gate.log 2>&1; echo "rc=$?" >> gpurun_out/pt_gate.log
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "tcgen05" > gpurun_out/pt_ffn.log 2>&1; echo "rc=$?" >> gpurun_out/pt_ffn.log
timeout 600 python -m pytest tests/test_gpu_backward.py -q > gpurun_out/pt_bwd.log 2>&1; echo "rc=$?" >> gpurun_out/pt_bwd.log
timeout 900 python -m pytest tests -m gpu -q -k "not multigpu" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench_n1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n1.log
for c in c3 c4 c5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$c.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$c.log
done
echo done
