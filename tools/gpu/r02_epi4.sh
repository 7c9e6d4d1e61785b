# Forward epilogue warps 8 (default) vs 4 (build in ab/): C2 / C4 / C5 A/B.
set -x
O=gpurun_out/r02epi4
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for round in 1 2; do
for v in e8 e4; do
  if [ $v = e4 ]; then export SMILE_LIB_PATH=$PWD/ab/libsmile_epi4.so; else unset SMILE_LIB_PATH; fi
  timeout 300 python bench.py --steps 50 --no-cpu --no-e2e > $O/c2_${v}_$round.log 2>&1
  timeout 300 python bench.py --config c4 --steps 10 --no-cpu --no-e2e > $O/c4_${v}_$round.log 2>&1
  timeout 300 python bench.py --config c5 --steps 10 --no-cpu --no-e2e > $O/c5_${v}_$round.log 2>&1
done
done
echo done
