# GEMM 2 -> out fusion (SMILE_OUT_DIRECT): parity on one GPU and two, then A/B bench lines
set -x
O=gpurun_out/od
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "out_direct or ret_direct or peer or tcgen05" > $O/pt1.log 2>&1; echo "rc=$?" >> $O/pt1.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
for rep in 1 2; do for r in 1 0; do
  CUDA_VISIBLE_DEVICES=0 SMILE_OUT_DIRECT=$r timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu > $O/n1_od${r}_$rep.log 2>&1
done; done
timeout 900 python -m pytest tests/test_multigpu.py -q -x > $O/pt2.log 2>&1; echo "rc=$?" >> $O/pt2.log
P=29820
for rep in 1 2; do for r in 1 0; do
  P=$((P+1)); SMILE_OUT_DIRECT=$r timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --steps 50 --warmup 5 --no-cpu > $O/n2_od${r}_$rep.log 2>&1
done; done
echo done
