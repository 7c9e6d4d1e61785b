# FFN epilogue warps A/B: 16 (default) vs 8 vs 12 (separate builds via SMILE_LIB_PATH).
set -x
O=gpurun_out/r02epi
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for round in 1 2; do
for v in d16 e8 e12; do
  case $v in d16) unset SMILE_LIB_PATH;; e8) export SMILE_LIB_PATH=$PWD/ab/libsmile_epi8.so;; e12) export SMILE_LIB_PATH=$PWD/ab/libsmile_epi12.so;; esac
  timeout 300 python bench.py --steps 50 --no-cpu --no-e2e --mode bilevel > $O/c2_${v}_$round.log 2>&1
  timeout 300 python bench.py --config c5 --mode bilevel --steps 10 --no-cpu --no-e2e > $O/c5_${v}_$round.log 2>&1
done
done
for v in d16 e8 e12; do
  case $v in d16) unset SMILE_LIB_PATH;; e8) export SMILE_LIB_PATH=$PWD/ab/libsmile_epi8.so;; e12) export SMILE_LIB_PATH=$PWD/ab/libsmile_epi12.so;; esac
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ffn_gemm -c 2 --csv --log-file $O/ncu_c2_$v.csv \
    python bench.py --config c2 --mode bilevel --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > /dev/null 2>&1
done
unset SMILE_LIB_PATH
SMILE_LIB_PATH=$PWD/ab/libsmile_epi8.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "ffn or tcgen05" > $O/pytest_e8.log 2>&1; echo "rc=$?" >> $O/pytest_e8.log
echo done
