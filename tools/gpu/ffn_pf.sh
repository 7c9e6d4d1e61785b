# FFN A-operand L2 prefetch distance and work-list direction sweep (C2)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
N="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --mode bilevel --clock-ms 0"
B="python bench.py --no-cpu --no-e2e --steps 50 --mode bilevel --clock-ms 0"
timeout 300 $N > gpurun_out/plain.log 2>&1
run() { tag=$1; shift; env "$@" timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"ffn_gemm" -c 4 --csv --log-file gpurun_out/p_$tag.csv $N > /dev/null 2>&1; env "$@" timeout 300 $B > gpurun_out/p_$tag.log 2>&1; }
run base SMILE_FFN_PF=0
run pf4 SMILE_FFN_PF=4
run pf8 SMILE_FFN_PF=8
run pf16 SMILE_FFN_PF=16
run rev2 SMILE_FFN_REVERSE=2
run rev3 SMILE_FFN_REVERSE=3
run pf8rev2 SMILE_FFN_PF=8 SMILE_FFN_REVERSE=2
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "tcgen05 or empty" > gpurun_out/pt_ffn.log 2>&1; echo "rc=$?" >> gpurun_out/pt_ffn.log
SMILE_FFN_PF=8 SMILE_FFN_REVERSE=2 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "tcgen05" > gpurun_out/pt_ffn_pf.log 2>&1; echo "rc=$?" >> gpurun_out/pt_ffn_pf.log
echo done
