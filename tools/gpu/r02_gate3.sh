# Round 2: gate schedule A/B (interleaved rounds + balanced tail vs contiguous), fabric emulation.
set -x
O=gpurun_out/r02g3
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fabric.py -q -x -k "fused_router or c1_full or shapes or peer or determinism or host_stream or bench_launch or fabric" > $O/pytest_gate.log 2>&1; echo "rc=$?" >> $O/pytest_gate.log
for i in 1 2; do
timeout 300 python bench.py --steps 50 --no-cpu --no-e2e --mode bilevel > $O/bench_c2_$i.log 2>&1
SMILE_GATE_SCHED=contig timeout 300 python bench.py --steps 50 --no-cpu --no-e2e --mode bilevel > $O/bench_c2_contig_$i.log 2>&1
done
timeout 300 python bench.py --config c4 --steps 20 --no-cpu --no-e2e --mode bilevel > $O/bench_c4.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_c2.csv \
    python bench.py --config c2 --mode bilevel --steps 2 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > $O/launches_c2.log 2>&1
SMILE_GATE_SCHED=contig timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_c2_contig.csv \
    python bench.py --config c2 --mode bilevel --steps 2 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > $O/launches_c2_contig.log 2>&1
for f in "50,5" "12.5,20"; do
  for c in c1 e4x8_c1 e4x8 e8x4; do
    timeout 600 python bench.py --config $c --fabric $f --steps 20 --no-cpu --no-e2e > $O/bench_fabric_${c}_${f/,/_}.log 2>&1
  done
done
timeout 600 python bench.py --config e4x8 --exchange copy --steps 20 --no-cpu --no-e2e > $O/bench_nofabric_e4x8.log 2>&1
echo done
