# EPI_WARPS = 8 default: every single-GPU test, and A/B against the 16-warp build on C2 / C3 / C4 / C5.
set -x
O=gpurun_out/r02epi2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -x -k "not multigpu" > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for round in 1 2; do
for v in e8 d16; do
  if [ $v = d16 ]; then export SMILE_LIB_PATH=$PWD/ab/libsmile_epi16.so; else unset SMILE_LIB_PATH; fi
  timeout 300 python bench.py --steps 50 --no-cpu --no-e2e > $O/c2_${v}_$round.log 2>&1
  timeout 600 python bench.py --config c3 --steps 10 --no-cpu > $O/c3_${v}_$round.log 2>&1
  timeout 300 python bench.py --config c4 --steps 10 --no-cpu --no-e2e > $O/c4_${v}_$round.log 2>&1
  timeout 300 python bench.py --config c5 --steps 10 --no-cpu --no-e2e > $O/c5_${v}_$round.log 2>&1
done
done
echo done
