set -x
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --steps 200 --warmup 5 --no-cpu > gpurun_out/bench_n2.log 2>&1
echo done
