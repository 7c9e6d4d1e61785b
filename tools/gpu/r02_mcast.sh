# FFN A multicast across clusters of 2 (SMILE_FFN_MCAST=1): parity, C5 A/B, timelines, L2->SM bytes.
set -x
O=gpurun_out/r02mc
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
SMILE_FFN_MCAST=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "ffn or tcgen05 or c5 or full" > $O/pytest_mc.log 2>&1; echo "rc=$?" >> $O/pytest_mc.log
for round in 1 2; do
for v in 0 1; do
  SMILE_FFN_MCAST=$v timeout 300 python bench.py --config c5 --steps 10 --no-cpu --no-e2e > $O/c5_mc${v}_$round.log 2>&1
done
done
for k in ffn1 ffn2; do SMILE_FFN_MCAST=1 SMILE_TRACE=$k timeout 300 python tools/gpu/trace_kernels.py --config c5 --mode bilevel > $O/trace_c5_${k}_mc1.log 2>&1; done
for v in 0 1; do
  SMILE_FFN_MCAST=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:ffn_gemm -c 4 --csv --log-file $O/ncu_c5_mc$v.csv \
    python bench.py --config c5 --mode bilevel --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > /dev/null 2>&1
done
echo done
