set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SMILE_FFN_BOX64=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "tcgen05_ffn" > gpurun_out/pt_box64.log 2>&1; echo "rc=$?" >> gpurun_out/pt_box64.log
for v in 0 1 0 1; do
  SMILE_FFN_BOX64=$v timeout 600 python bench.py --no-cpu --no-e2e --steps 100 --mode bilevel >> gpurun_out/ab_box64_$v.log 2>&1
done
echo done
