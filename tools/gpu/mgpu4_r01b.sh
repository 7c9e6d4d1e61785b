# 4-GPU parity and N = 4 lines after the GEMM 2 -> out fusion
set -x
O=gpurun_out/m4
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_multigpu.py -x -q > $O/pytest_mgpu4.log 2>&1; echo "rc=$?" >> $O/pytest_mgpu4.log
P=29950
P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --steps 100 --warmup 5 > $O/bench_n4_peer.log 2>&1
P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --steps 50 --warmup 5 --no-e2e --exchange copy > $O/bench_n4_copy.log 2>&1
P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --impl reference --steps 2 --warmup 3 > $O/bench_n4_reference.log 2>&1
P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --config c3 --steps 10 --warmup 3 > $O/bench_n4_c3_peer.log 2>&1
echo done
