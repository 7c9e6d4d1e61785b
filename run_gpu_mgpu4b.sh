set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "dropless" > gpurun_out/pt_dropless.log 2>&1; echo "rc=$?" >> gpurun_out/pt_dropless.log
P=29700
for N in 2 4; do
  for c in 2 4; do
    P=$((P+1)); timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --chunks $c --mode both --steps 50 --warmup 3 > gpurun_out/pipe_n${N}_c$c.log 2>&1
  done
done
P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --config c3 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_n4_c3.log 2>&1
P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --steps 100 --warmup 5 --no-cpu > gpurun_out/bench_n4_peer.log 2>&1
echo done
