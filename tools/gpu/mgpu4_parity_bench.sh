# Four B200: multi-GPU parity (forward + training, NCCL and peer exchanges, 2 and 4
# processes), the default bench at N = 2 and 4 (peer) plus the NCCL path, C3 at N = 4.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/pytest_mgpu4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mgpu4.log
P=29500
for N in 2 4; do
  P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --steps 100 --warmup 5 > gpurun_out/bench_n${N}_peer.log 2>&1
  P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --steps 50 --warmup 5 --no-e2e --exchange copy > gpurun_out/bench_n${N}_copy.log 2>&1
  P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --impl reference --steps 2 --warmup 1 > gpurun_out/bench_n${N}_reference.log 2>&1
done
P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --config c3 --steps 10 --warmup 3 > gpurun_out/bench_n4_c3_peer.log 2>&1
echo done
