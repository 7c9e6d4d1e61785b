set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "tcgen05" > gpurun_out/pt_ffn.log 2>&1; echo "rc=$?" >> gpurun_out/pt_ffn.log
for sl in 1 2; do
  SMILE_FFN_OUT_SLOTS=$sl timeout 600 python bench.py --no-cpu --no-e2e --mode bilevel --steps 100 > gpurun_out/bench_slots$sl.log 2>&1
done
SMILE_FFN_CTA_PAIR=0 timeout 600 python bench.py --no-cpu --no-e2e --mode bilevel --steps 100 > gpurun_out/bench_cg1.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --mode bilevel --clock-ms 0"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ffn_gemm|gate1_tc|row_move" -s 7 -c 7 -o gpurun_out/prof_t6 $CMD > gpurun_out/ncu_full.log 2>&1
echo done
