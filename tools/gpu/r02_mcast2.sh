# Default A multicast (even N-tile counts) check, and the BN = 160 GEMM 1 experiment at C5.
set -x
O=gpurun_out/r02mc2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "ffn or tcgen05 or c5" > $O/pytest_default.log 2>&1; echo "rc=$?" >> $O/pytest_default.log
SMILE_FFN_MC_BN=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "ffn or c5" > $O/pytest_mcbn.log 2>&1; echo "rc=$?" >> $O/pytest_mcbn.log
for round in 1 2; do
  for v in off default mcbn; do
    case $v in off) E="SMILE_FFN_MCAST=0";; default) E="X=0";; mcbn) E="SMILE_FFN_MC_BN=1";; esac
    env $E timeout 300 python bench.py --config c5 --steps 10 --no-cpu --no-e2e > $O/c5_${v}_$round.log 2>&1
  done
done
for v in default mcbn; do
  case $v in default) E="X=0";; mcbn) E="SMILE_FFN_MC_BN=1";; esac
  env $E timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:ffn_gemm -c 2 --csv --log-file $O/ncu_c5_$v.csv \
    python bench.py --config c5 --mode bilevel --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > /dev/null 2>&1
done
echo done
