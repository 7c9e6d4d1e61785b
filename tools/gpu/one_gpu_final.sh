# One B200, final evidence of the round: build, every GPU test, smoke, the default bench
# line, the reference arm, C3/C4/C5 lines, the launch list of one C2 step and an ncu
# --set full capture of its kernels.
set -x
mkdir -p gpurun_out/final
O=gpurun_out/final
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -k "not multigpu" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.log 2>&1
for c in c3 c4 c5; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1; done
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --mode bilevel --clock-ms 0"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ffn_gemm|gate1_tc|row_move|scan|rank2|aux|split|meta" -s 15 -c 15 -o $O/prof_full $CMD > $O/ncu_full.log 2>&1
echo done
