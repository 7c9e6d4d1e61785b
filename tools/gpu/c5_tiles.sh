# C5 (128 experts, ~512 rows each): CTA-pair 256-row tiles vs single-CTA 128-row tiles
set -x
mkdir -p gpurun_out/c5
O=gpurun_out/c5
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
N="python bench.py --config c5 --steps 2 --warmup 1 --no-e2e --no-cpu --mode bilevel --clock-ms 0"
for cp in 1 0; do
  SMILE_FFN_CTA_PAIR=$cp timeout 300 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu --no-e2e --mode bilevel > $O/bench_cp$cp.log 2>&1
  SMILE_FFN_CTA_PAIR=$cp timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"ffn_gemm" -c 4 --csv --log-file $O/ffn_cp$cp.csv $N > /dev/null 2>&1
done
SMILE_FFN_NSUB=2 timeout 300 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu --no-e2e --mode bilevel > $O/bench_nsub2.log 2>&1
echo done
