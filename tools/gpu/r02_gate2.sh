# Round 2: ranged gate with per-CTA rank arrival; A/B against the 128-token kernel.
set -x
O=gpurun_out/r02g2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_router or c1_full or shapes or peer or determinism or host_stream or bench_launch" > $O/pytest_gate.log 2>&1; echo "rc=$?" >> $O/pytest_gate.log
timeout 300 python bench.py --steps 50 --no-cpu --no-e2e --mode bilevel > $O/bench_c2.log 2>&1
SMILE_GATE_SWAP=0 timeout 300 python bench.py --steps 50 --no-cpu --no-e2e --mode bilevel > $O/bench_c2_swap0.log 2>&1
timeout 300 python bench.py --config c4 --steps 20 --no-cpu --no-e2e --mode bilevel > $O/bench_c4.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gate1 -c 2 -o $O/ncu_gate_c2 \
    python bench.py --config c2 --mode bilevel --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > $O/ncu_gate_c2.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_c2.csv \
    python bench.py --config c2 --mode bilevel --steps 2 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > $O/launches_c2.log 2>&1
echo done
