# Same-box A/B: HEAD library vs the working tree (whole-warp MMA issuers in the FFN / wgrad /
# 128-token gate, unrolled gate epilogue) -- bench phases, ncu launch lists, gate timelines.
set -x
O=gpurun_out/r02ab2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_topk.py -q -x > $O/pytest_gate.log 2>&1; echo "rc=$?" >> $O/pytest_gate.log
for cfg in c2 c4 c5; do
  SMILE_TRACE=gate timeout 300 python tools/gpu/trace_kernels.py --config $cfg --mode bilevel > $O/trace_${cfg}_gate.log 2>&1
done
SMILE_TRACE=gate timeout 300 python tools/gpu/trace_kernels.py --config c5 --mode flat > $O/trace_c5flat_gate.log 2>&1
for round in 1 2; do
for v in head new; do
  if [ $v = head ]; then export SMILE_LIB_PATH=$PWD/ab/libsmile_head.so; else unset SMILE_LIB_PATH; fi
  timeout 300 python bench.py --steps 50 --no-cpu --no-e2e > $O/c2_${v}_$round.log 2>&1
  timeout 300 python bench.py --config c4 --steps 10 --no-cpu --no-e2e > $O/c4_${v}_$round.log 2>&1
  timeout 300 python bench.py --config c5 --steps 10 --no-cpu --no-e2e > $O/c5_${v}_$round.log 2>&1
done
done
for v in head new; do
  if [ $v = head ]; then export SMILE_LIB_PATH=$PWD/ab/libsmile_head.so; else unset SMILE_LIB_PATH; fi
  for cfg in c2 c4 c5; do
    timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gate1|scan1|router_split|ffn_gemm|row_move" -c 12 --csv \
      --log-file $O/launch_${cfg}_$v.csv python bench.py --config $cfg --mode bilevel --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > /dev/null 2>&1
  done
done
echo done
