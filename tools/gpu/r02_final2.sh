# Round 2: clean single-GPU test log + ncu --set full of exactly one C2 step (HEAD).
set -x
O=gpurun_out/r02f2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gate1|scan|row_move|meta_fill|rank2|ffn_gemm|aux_kernel" -s 10 -c 10 -o $O/ncu_c2_step \
    python bench.py --config c2 --mode bilevel --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > $O/ncu_c2_step.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:"gate1|scan|row_move|meta_fill|rank2|ffn_gemm|aux_kernel" -s 6 -c 6 -o $O/ncu_c2_flat_step \
    python bench.py --config c2 --mode flat --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > $O/ncu_c2_flat_step.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -k "not multigpu" > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log

for c in c4 c5; do
  timeout 600 python bench.py --config $c --steps 20 --no-cpu --no-e2e > $O/bench_$c.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"gate1|scan1|router_split" -c 6 --csv --log-file $O/gate_$c.csv \
    python bench.py --config $c --mode both --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > /dev/null 2>&1
done
timeout 600 python bench.py --steps 50 > $O/bench_default.log 2>&1
echo done2
