# Round 2 closing run on one B200: every single-GPU test, smoke, bench lines of every config,
# ncu launch list + --set full of one C2 step and one C5 step, the reference arm.
set -x
O=gpurun_out/r02f1
mkdir -p $O
nproc > $O/nproc.txt
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 3000 python -m pytest tests -m gpu -q -k "not multigpu" -p no:randomly > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_default.log 2>&1
timeout 600 python bench.py --steps 100 --no-cpu --graph > $O/bench_graph.log 2>&1
for c in c3 c3_4x2 c4 c5; do timeout 900 python bench.py --config $c --steps 20 --no-cpu > $O/bench_$c.log 2>&1; done
timeout 600 python bench.py --config c1 --steps 100 --no-cpu > $O/bench_c1.log 2>&1
timeout 600 python bench.py --mode flat --topk 2 --steps 50 --no-cpu --no-e2e > $O/bench_flat_top2.log 2>&1
for ch in 2 4; do timeout 600 python bench.py --chunks $ch --steps 50 > $O/bench_chunks$ch.log 2>&1; done
for f in "50,5" "12.5,20"; do for c in c2 c1 e4x8 e8x4 e4x8_c1; do
  timeout 600 python bench.py --config $c --fabric $f --steps 20 --no-cpu --no-e2e > $O/bench_fabric_${c}_${f/,/_}.log 2>&1
done; done
timeout 600 python bench.py --config e4x8 --exchange copy --steps 20 --no-cpu --no-e2e > $O/bench_nofabric_e4x8.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c2.csv \
    python bench.py --config c2 --mode bilevel --steps 2 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > $O/launches_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"smile" -s 10 -c 10 -o $O/ncu_c2_step \
    python bench.py --config c2 --mode bilevel --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > $O/ncu_c2_step.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"gate1|ffn_gemm" -c 6 -o $O/ncu_c5 \
    python bench.py --config c5 --mode bilevel --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > $O/ncu_c5.log 2>&1
echo done
