# Two-sub-tile FFN GEMM (SMILE_FFN_NSUB=2) vs double-buffered single tile: parity + timing
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SMILE_FFN_NSUB=2 timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_backward.py -q -x -k "tcgen05 or c2_full or wgrad or train or backward" > gpurun_out/pt_nsub2.log 2>&1; echo "rc=$?" >> gpurun_out/pt_nsub2.log
N="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --mode bilevel --clock-ms 0"
B="python bench.py --no-cpu --no-e2e --steps 50 --mode bilevel --clock-ms 0"
for ns in 1 2; do
  SMILE_FFN_NSUB=$ns timeout 300 $B > gpurun_out/n_$ns.log 2>&1
  SMILE_FFN_NSUB=$ns timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ffn_gemm" -c 4 --csv --log-file gpurun_out/n_$ns.csv $N > /dev/null 2>&1
  SMILE_FFN_NSUB=$ns timeout 300 python bench.py --no-cpu --no-e2e --steps 10 --config c4 --mode bilevel --clock-ms 0 > gpurun_out/n_c4_$ns.log 2>&1
  SMILE_FFN_NSUB=$ns timeout 300 python bench.py --no-cpu --no-e2e --steps 10 --config c3 --mode bilevel --clock-ms 0 > gpurun_out/n_c3_$ns.log 2>&1
done
SMILE_FFN_NSUB=2 SMILE_FFN_DIAG=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ffn_gemm" -c 4 --csv --log-file gpurun_out/n_2_diag4.csv $N > /dev/null 2>&1
echo done
