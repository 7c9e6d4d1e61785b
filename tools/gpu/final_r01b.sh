# Round-end evidence on a 2-GPU box after the GEMM 2 -> out fusion: single-GPU suite, smoke,
# N = 1 bench lines, launch list and ncu on GPU 0, then 2-process parity and N = 2 lines.
set -x
O=gpurun_out/fin2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
export CUDA_VISIBLE_DEVICES=0
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "out_direct or ret_direct" > $O/pt_od.log 2>&1; echo "rc=$?" >> $O/pt_od.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.log 2>&1
for c in c3 c4 c5; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1; done
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --mode bilevel --clock-ms 0"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ffn_gemm|gate1_tc|row_move|scan|rank2|aux|split|meta" -s 15 -c 15 -o $O/prof_full $CMD > $O/ncu_full.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -k "not multigpu" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
unset CUDA_VISIBLE_DEVICES
timeout 900 python -m pytest tests/test_multigpu.py -x -q > $O/pytest_mgpu2.log 2>&1; echo "rc=$?" >> $O/pytest_mgpu2.log
P=29900
P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --steps 100 --warmup 5 > $O/bench_n2_peer.log 2>&1
P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --steps 50 --warmup 5 --no-e2e --exchange copy > $O/bench_n2_copy.log 2>&1
P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --impl reference --steps 2 --warmup 3 > $O/bench_n2_reference.log 2>&1
echo done
