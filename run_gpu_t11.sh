set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "forward_host" > gpurun_out/pt_host.log 2>&1; echo "rc=$?" >> gpurun_out/pt_host.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/bench_default.log
echo done
