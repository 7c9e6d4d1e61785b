set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
./tools/cluster_probe > gpurun_out/cluster_probe.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "tcgen05_ffn" > gpurun_out/pt_ffn1.log 2>&1; echo "rc=$?" >> gpurun_out/pt_ffn1.log
SMILE_FFN_PAIRS=2 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "tcgen05_ffn" > gpurun_out/pt_ffn2.log 2>&1; echo "rc=$?" >> gpurun_out/pt_ffn2.log
timeout 600 python bench.py --no-cpu --no-e2e --steps 100 --mode bilevel > gpurun_out/bench_p1.log 2>&1
SMILE_FFN_PAIRS=2 timeout 600 python bench.py --no-cpu --no-e2e --steps 100 --mode bilevel > gpurun_out/bench_p2.log 2>&1
SMILE_FFN_PAIRS=2 timeout 600 python bench.py --config c5 --no-cpu --no-e2e --steps 10 --mode bilevel > gpurun_out/bench_c5_p2.log 2>&1
echo done
