set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_backward.py -q -x > gpurun_out/pt_bwd.log 2>&1; echo "rc=$?" >> gpurun_out/pt_bwd.log
timeout 600 python bench.py --no-cpu --no-e2e --steps 100 > gpurun_out/bench_rw4.log 2>&1
SMILE_MOVE_RW=8 timeout 600 python bench.py --no-cpu --no-e2e --steps 100 > gpurun_out/bench_rw8.log 2>&1
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c3_peer.log 2>&1
echo done
