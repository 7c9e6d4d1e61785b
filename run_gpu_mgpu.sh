set -x
timeout 900 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/pytest_mgpu4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mgpu4.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 4 --steps 200 --warmup 5 --no-cpu > gpurun_out/bench_n4.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29572 bench.py --gpus 2 --steps 200 --warmup 5 --no-cpu > gpurun_out/bench_n2b.log 2>&1
echo done
