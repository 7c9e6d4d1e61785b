# EPI_WARPS: 8 for the forward epilogues, 16 for dZ -- backward tests and C3 A/B vs the all-16 build.
set -x
O=gpurun_out/r02epi3
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_backward.py tests/test_gpu_fullsize.py tests/test_gpu_topk.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for round in 1 2 3; do
for v in new d16; do
  if [ $v = d16 ]; then export SMILE_LIB_PATH=$PWD/ab/libsmile_epi16.so; else unset SMILE_LIB_PATH; fi
  timeout 600 python bench.py --config c3 --steps 10 --no-cpu > $O/c3_${v}_$round.log 2>&1
done
done
unset SMILE_LIB_PATH
timeout 300 python bench.py --steps 50 --no-cpu --no-e2e > $O/c2_new.log 2>&1
echo done
