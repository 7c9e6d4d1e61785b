# Round 2 closing re-check on 4 GPUs (HEAD): multi-GPU parity, bench lines at N = 2 and 4,
# chunked pipelining across GPUs.
set -x
O=gpurun_out/r02fm7
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 2400 python -m pytest tests/test_multigpu.py -q > $O/pytest_mgpu.log 2>&1; echo "rc=$?" >> $O/pytest_mgpu.log
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $R4 --master-port 29901 bench.py --gpus 4 --steps 50 > $O/bench_n4_peer.log 2>&1
timeout 600 $R2 --master-port 29902 bench.py --gpus 2 --steps 50 > $O/bench_n2_peer.log 2>&1
timeout 900 $R4 --master-port 29903 bench.py --gpus 4 --config c3 --steps 20 > $O/bench_n4_c3_peer.log 2>&1
for ch in 2 4; do timeout 600 $R4 --master-port 2991$ch bench.py --gpus 4 --chunks $ch --steps 30 > $O/bench_n4_chunks$ch.log 2>&1; done
SMILE_FFN_MAX_CTAS=120 timeout 600 $R4 --master-port 29915 bench.py --gpus 4 --chunks 2 --steps 30 > $O/bench_n4_chunks2_cap120.log 2>&1
timeout 600 $R4 --master-port 29916 bench.py --gpus 4 --mode flat --topk 2 --steps 30 --no-e2e > $O/bench_n4_flat_top2.log 2>&1
echo done
