# Round 2: per-CTA timelines of the gate and FFN kernels (SMILE_TRACE), the L2-flush A/B,
# the gate kernels with the whole-warp MMA issuer (parity + launch list).
set -x
O=gpurun_out/r02tr2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gate or tcgen05 or route" > $O/pytest_gate.log 2>&1; echo "rc=$?" >> $O/pytest_gate.log
for cfg in c2 c5; do
  for k in gate ffn1 ffn2; do
    SMILE_TRACE=$k timeout 300 python tools/gpu/trace_kernels.py --config $cfg --mode bilevel > $O/trace_${cfg}_$k.log 2>&1
  done
done
SMILE_TRACE=gate timeout 300 python tools/gpu/trace_kernels.py --config c4 --mode bilevel > $O/trace_c4_gate.log 2>&1
for fl in write write+read; do
  timeout 300 python bench.py --steps 50 --no-cpu --no-e2e --flush $fl > $O/bench_c2_flush_$fl.log 2>&1
  timeout 300 python bench.py --config c5 --mode bilevel --steps 20 --no-cpu --no-e2e --flush $fl > $O/bench_c5_flush_$fl.log 2>&1
done
for cfg in c2 c5; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gate1 -c 6 --csv \
    --log-file $O/ncu_gate_$cfg.csv python bench.py --config $cfg --mode bilevel --steps 2 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > $O/ncu_gate_$cfg.log 2>&1
done
echo done
