# Round 2: C5 FFN tile shapes (L2 -> SM operand traffic) + C2 cross-check.
set -x
O=gpurun_out/r02f5
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for v in "X=0" "SMILE_FFN_CTA_PAIR=1" "SMILE_FFN_CTA_PAIR=1 SMILE_FFN_NSUB=2"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 300 python bench.py --config c5 --mode bilevel --steps 20 --no-cpu --no-e2e > $O/c5_$tag.log 2>&1
  env $v timeout 300 python bench.py --config c5 --mode flat --steps 20 --no-cpu --no-e2e > $O/c5flat_$tag.log 2>&1
  env $v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:ffn_gemm -c 4 --csv --log-file $O/ncu_c5_$tag.csv \
    python bench.py --config c5 --mode bilevel --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > /dev/null 2>&1
done
SMILE_FFN_NSUB=2 timeout 300 python bench.py --config c2 --mode bilevel --steps 30 --no-cpu --no-e2e > $O/c2_nsub2.log 2>&1
timeout 300 python bench.py --config c2 --mode bilevel --steps 30 --no-cpu --no-e2e > $O/c2_default.log 2>&1
SMILE_FFN_CTA_PAIR=1 SMILE_FFN_NSUB=2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tcgen05" > $O/pytest_nsub2.log 2>&1; echo "rc=$?" >> $O/pytest_nsub2.log
echo done
