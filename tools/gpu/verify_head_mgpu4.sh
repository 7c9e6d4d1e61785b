# Re-entry check of HEAD on a 4-GPU box: 2- and 4-process parity (fwd + training, both exchanges)
# and the N = 4 bench lines (peer exchange, NCCL copy exchange).
set -x
O=gpurun_out/head4
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_multigpu.py -x -q > $O/pytest_mgpu4.log 2>&1; echo "rc=$?" >> $O/pytest_mgpu4.log
P=29910
P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --steps 100 --warmup 5 > $O/bench_n4_peer.log 2>&1
P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --steps 50 --warmup 5 --no-e2e --exchange copy > $O/bench_n4_copy.log 2>&1
echo done
