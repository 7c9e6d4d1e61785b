# FFN GEMM diagnostics (measurement only): which part of the epilogue limits GEMM1?
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
B="python bench.py --no-cpu --no-e2e --steps 50 --mode bilevel --clock-ms 0"
N="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --mode bilevel --clock-ms 0"
for dg in 0 1 2 3 4; do
  SMILE_FFN_DIAG=$dg timeout 300 $B > gpurun_out/diag_$dg.log 2>&1
  SMILE_FFN_DIAG=$dg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ffn_gemm" -c 4 --csv --log-file gpurun_out/diag_$dg.csv $N > /dev/null 2>&1
done
for st in 3 4; do
  SMILE_FFN_STAGES=$st timeout 300 $B > gpurun_out/stages_$st.log 2>&1
done
echo done
