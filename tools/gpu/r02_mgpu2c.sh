set -x
O=gpurun_out/r02m2c
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests/test_multigpu.py -q > $O/pytest_mgpu.log 2>&1; echo "rc=$?" >> $O/pytest_mgpu.log
R2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
SMILE_XCHG_EXACT=1 timeout 600 $R2 --master-port 29810 bench.py --gpus 2 --mode flat --steps 30 --exchange copy --no-e2e > $O/bench_n2_flat_copy_exact.log 2>&1
timeout 600 $R2 --master-port 29811 bench.py --gpus 2 --mode flat --topk 2 --steps 30 --no-e2e > $O/bench_n2_flat_top2.log 2>&1
echo done
