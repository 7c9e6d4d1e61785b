# FFN store-path experiments (measurement only)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
N="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --mode bilevel --clock-ms 0"
B="python bench.py --no-cpu --no-e2e --steps 50 --mode bilevel --clock-ms 0"
timeout 300 $N > gpurun_out/plain.log 2>&1
run() { tag=$1; shift; env "$@" timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ffn_gemm" -c 4 --csv --log-file gpurun_out/x_$tag.csv $N > /dev/null 2>&1; env "$@" timeout 300 $B > gpurun_out/x_$tag.log 2>&1; }
run base SMILE_FFN_DIAG=0
run stg SMILE_FFN_TMA_STORE=0
run box64 SMILE_FFN_BOX64=2
run win SMILE_FFN_DIAG=8
run nogelu_win SMILE_FFN_DIAG=9
for dg in 0 2; do
  SMILE_FFN_DIAG=$dg timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ffn_gemm" --launch-skip 1 -c 1 -o gpurun_out/g2_diag$dg -f $N > gpurun_out/ncu_g2_$dg.log 2>&1
done
echo done
