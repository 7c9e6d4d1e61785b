# e2e A/B at N = 2: GEMM 2 -> ret1 fusion on / off, alternating on one box
set -x
mkdir -p gpurun_out/e2e
O=gpurun_out/e2e
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
P=29800
for rep in 1 2; do for r in 1 0; do
  P=$((P+1)); SMILE_RET_DIRECT=$r timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --steps 50 --warmup 5 --no-cpu --mode bilevel > $O/n2_ret${r}_$rep.log 2>&1
done; done
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 50 --no-cpu --mode bilevel > $O/n1.log 2>&1
echo done
