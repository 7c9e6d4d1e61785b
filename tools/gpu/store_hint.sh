# FFN output stores with L2 eviction hints (measurement)
set -x
mkdir -p gpurun_out/sh
O=gpurun_out/sh
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
N="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --mode bilevel --clock-ms 0"
B="python bench.py --no-cpu --no-e2e --steps 100 --mode bilevel --clock-ms 0"
for h in 0 2 1 3 4 6; do
  SMILE_FFN_STORE_HINT=$h timeout 300 $B > $O/b_$h.log 2>&1
  SMILE_FFN_STORE_HINT=$h timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ffn_gemm" -c 4 --csv --log-file $O/n_$h.csv $N > /dev/null 2>&1
done
echo done
