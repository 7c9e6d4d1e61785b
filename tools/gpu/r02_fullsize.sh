# Round 2: full-size parity at every benched configuration + ncu of the gate kernels (C2, C5).
set -x
O=gpurun_out/r02fs
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -v -x --durations=0 > $O/pytest_fullsize.log 2>&1; echo "pytest rc=$?" >> $O/pytest_fullsize.log
for cfg in c2 c5; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gate1 -c 2 -o $O/ncu_gate_$cfg \
    python bench.py --config $cfg --mode bilevel --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > $O/ncu_gate_$cfg.log 2>&1
done
timeout 600 ncu --set full --clock-control none -k regex:ffn_gemm -c 2 -o $O/ncu_ffn_c5 \
    python bench.py --config c5 --mode bilevel --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > $O/ncu_ffn_c5.log 2>&1
timeout 600 python bench.py --config c5 --steps 20 --no-cpu > $O/bench_c5.log 2>&1
echo done
