# Round 2 closing re-check on one B200 (HEAD after the gate / MMA-issuer work): build, smoke,
# every single-GPU test, bench lines, launch list, one ncu --set full capture of a C2 step.
set -x
O=gpurun_out/r02f6
mkdir -p $O
nproc > $O/nproc.txt
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 3000 python -m pytest tests -m gpu -q -x -k "not multigpu" > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_default.log 2>&1
timeout 600 python bench.py --steps 100 --no-cpu --graph > $O/bench_graph.log 2>&1
for c in c3 c4 c5; do timeout 900 python bench.py --config $c --steps 20 --no-cpu > $O/bench_$c.log 2>&1; done
timeout 600 python bench.py --mode flat --topk 2 --steps 50 --no-cpu --no-e2e > $O/bench_flat_top2.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.log 2>&1
K='gate1|scan1|row_move|meta_fill|rank2|scan2|ffn_gemm|aux_kernel|router_split'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$K" -c 30 --csv --log-file $O/launches_c2.csv \
    python bench.py --config c2 --mode bilevel --steps 2 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > $O/launches_c2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$K" -c 10 -o $O/ncu_c2_step \
    python bench.py --config c2 --mode bilevel --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > $O/ncu_c2_step.log 2>&1
echo done
