# Round 2 on 4 GPUs: multi-GPU parity (2- and 4-process, bit-exact routes, graph replays,
# exact-size NCCL exchange), NCCL busBW per group size, bench lines at N = 2 and N = 4.
set -x
O=gpurun_out/r02m4
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 2400 python -m pytest tests/test_multigpu.py -q > $O/pytest_mgpu.log 2>&1; echo "rc=$?" >> $O/pytest_mgpu.log
R4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $R4 --master-port 29801 tools/nccl_busbw.py > $O/busbw4.log 2>&1
timeout 600 $R4 --master-port 29802 bench.py --gpus 4 --steps 50 > $O/bench_n4_peer.log 2>&1
timeout 600 $R4 --master-port 29803 bench.py --gpus 4 --steps 30 --exchange copy --no-e2e > $O/bench_n4_copy.log 2>&1
SMILE_XCHG_EXACT=1 timeout 600 $R4 --master-port 29804 bench.py --gpus 4 --steps 30 --exchange copy --no-e2e > $O/bench_n4_copy_exact.log 2>&1
timeout 900 $R4 --master-port 29805 bench.py --gpus 4 --config c3 --steps 20 > $O/bench_n4_c3_peer.log 2>&1
timeout 600 $R4 --master-port 29806 bench.py --gpus 4 --config c4 --steps 10 --no-e2e > $O/bench_n4_c4_peer.log 2>&1
timeout 600 $R4 --master-port 29807 bench.py --gpus 4 --config c5 --steps 10 --no-e2e > $O/bench_n4_c5_peer.log 2>&1
timeout 600 $R2 --master-port 29808 bench.py --gpus 2 --steps 50 > $O/bench_n2_peer.log 2>&1
timeout 600 $R2 --master-port 29809 bench.py --gpus 2 --steps 30 --exchange copy --no-e2e > $O/bench_n2_copy.log 2>&1
SMILE_XCHG_EXACT=1 timeout 600 $R2 --master-port 29810 bench.py --gpus 2 --steps 30 --exchange copy --no-e2e > $O/bench_n2_copy_exact.log 2>&1
timeout 600 $R4 --master-port 29811 bench.py --gpus 4 --impl reference --steps 3 --warmup 1 > $O/bench_n4_reference.log 2>&1
echo done
