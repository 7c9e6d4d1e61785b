set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/pytest_mgpu4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mgpu4.log
P=29800
for N in 2 4; do
  P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --config c3 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_n${N}_c3_peer.log 2>&1
  P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --steps 100 --warmup 5 --no-cpu > gpurun_out/bench_n${N}_peer.log 2>&1
done
echo done
