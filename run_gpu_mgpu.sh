set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "peer" > gpurun_out/pytest_peer1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_peer1.log
timeout 900 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/pytest_mgpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mgpu.log
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu > gpurun_out/bench_n1_peer.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 2 --steps 100 --warmup 5 --no-cpu > gpurun_out/bench_n2_peer.log 2>&1
echo done
