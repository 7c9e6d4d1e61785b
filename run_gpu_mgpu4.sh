set -x
timeout 1200 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/pytest_mgpu4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mgpu4.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus 4 --steps 100 --warmup 5 --no-cpu > gpurun_out/bench_n4_peer.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29592 bench.py --gpus 4 --steps 100 --warmup 5 --no-cpu --exchange copy > gpurun_out/bench_n4_copy.log 2>&1
echo done
