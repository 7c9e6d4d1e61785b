set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in 1 0; do
  SMILE_FFN_SAVE_TMA=$v timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu --mode bilevel > gpurun_out/c3_save$v.log 2>&1
done
echo done
