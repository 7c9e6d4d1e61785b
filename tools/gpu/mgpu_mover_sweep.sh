# Movers over NVLink (peer stores / loads) at N = 2, 4: grid cap and rows per warp batch.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
P=29900
for N in 2 4; do
  for cfg in "8 4" "2 4" "4 4" "16 4" "8 8"; do
    set -- $cfg
    P=$((P+1)); SMILE_MOVE_GRIDMUL=$1 SMILE_MOVE_RW=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N --steps 100 --warmup 5 --no-cpu --no-e2e --mode bilevel > gpurun_out/sweep_n${N}_g$1_r$2.log 2>&1
  done
done
echo done
