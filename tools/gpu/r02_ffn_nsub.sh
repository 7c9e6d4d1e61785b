# Round 2: single-CTA tiles with two 128-row sub-tiles sharing B (CG = 1, NSUB = 2) for C5.
set -x
O=gpurun_out/r02fn
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
SMILE_FFN_CTA_PAIR=0 SMILE_FFN_NSUB=2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tcgen05" > $O/pytest_cg1_nsub2.log 2>&1; echo "rc=$?" >> $O/pytest_cg1_nsub2.log
for v in "X=0" "SMILE_FFN_NSUB=2"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 300 python bench.py --config c5 --steps 20 --no-cpu --no-e2e > $O/c5_$tag.log 2>&1
  env $v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:ffn_gemm -c 2 --csv --log-file $O/ncu_c5_$tag.csv \
    python bench.py --config c5 --mode bilevel --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > /dev/null 2>&1
done
echo done
