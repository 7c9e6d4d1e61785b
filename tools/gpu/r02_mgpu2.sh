# Round 2, 2 GPUs: multi-GPU parity (bit-exact routes, graph replays), NCCL busBW per group
# size, peer / copy bench, NCCL channel settings for the copy path.
set -x
O=gpurun_out/r02m2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 1500 python -m pytest tests/test_multigpu.py -q -x > $O/pytest_mgpu.log 2>&1; echo "rc=$?" >> $O/pytest_mgpu.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $R --master-port 29701 tools/nccl_busbw.py > $O/busbw.log 2>&1
for v in "NCCL_MIN_P2P_NCHANNELS=16" "NCCL_MIN_P2P_NCHANNELS=32" "NCCL_P2P_NVL_CHUNKSIZE=1048576" "NCCL_MIN_P2P_NCHANNELS=32 NCCL_P2P_NVL_CHUNKSIZE=1048576"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 300 $R --master-port 29702 tools/nccl_busbw.py > $O/busbw_$tag.log 2>&1
  env $v timeout 300 $R --master-port 29703 bench.py --gpus 2 --steps 30 --exchange copy --no-e2e > $O/bench_copy_$tag.log 2>&1
done
timeout 300 $R --master-port 29704 bench.py --gpus 2 --steps 50 > $O/bench_peer.log 2>&1
timeout 300 $R --master-port 29705 bench.py --gpus 2 --steps 30 --exchange copy --no-e2e > $O/bench_copy.log 2>&1
echo done
