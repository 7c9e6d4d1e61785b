set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/pytest_mgpu4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mgpu4.log
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2959$N bench.py --gpus $N --steps 100 --warmup 5 --no-cpu > gpurun_out/bench_n${N}_peer.log 2>&1
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2969$N bench.py --gpus $N --steps 50 --warmup 5 --no-cpu --no-e2e --exchange copy > gpurun_out/bench_n${N}_copy.log 2>&1
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29599 bench.py --gpus 4 --config c3 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_n4_c3.log 2>&1
echo done
