set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "tcgen05" > gpurun_out/pt_ffn.log 2>&1; echo "rc=$?" >> gpurun_out/pt_ffn.log
timeout 600 python bench.py --no-cpu --no-e2e --steps 100 > gpurun_out/bench_n1.log 2>&1
SMILE_FFN_TMA_STORE=1 timeout 600 python bench.py --no-cpu --no-e2e --steps 100 --mode bilevel > gpurun_out/bench_n1_tmastore.log 2>&1
for c in c3 c5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$c.log 2>&1
done
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --mode bilevel --clock-ms 0"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ffn_gemm" -s 2 -c 2 -o gpurun_out/prof_t8 $CMD > gpurun_out/ncu_full.log 2>&1
echo done
