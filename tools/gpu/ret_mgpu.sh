# ret-direct (local intermediates only) on 1, 2 and 4 GPUs: parity + bench
set -x
mkdir -p gpurun_out/retm
O=gpurun_out/retm
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_backward.py -q -x -k "peer or bench_launch or empty" > $O/pt_peer.log 2>&1; echo "rc=$?" >> $O/pt_peer.log
timeout 1500 python -m pytest tests/test_multigpu.py -x -q > $O/pytest_mgpu4.log 2>&1; echo "rc=$?" >> $O/pytest_mgpu4.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --no-cpu --no-e2e --steps 100 --mode bilevel > $O/bench_n1.log 2>&1
P=29600
for N in 2 4; do
  P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --steps 100 --warmup 5 > $O/bench_n${N}_peer.log 2>&1
  P=$((P+1)); SMILE_RET_DIRECT=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --steps 100 --warmup 5 --no-e2e > $O/bench_n${N}_peer_noret.log 2>&1
done
P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --config c3 --steps 10 --warmup 3 > $O/bench_n4_c3_peer.log 2>&1
echo done
