# GEMM 2 -> intermediates' ret1 (a9 + a10 + a11 fused in PEER mode): parity + bench
set -x
mkdir -p gpurun_out/ret
O=gpurun_out/ret
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_backward.py -q -x -k "peer or bench_launch or empty" > $O/pt_peer.log 2>&1; echo "rc=$?" >> $O/pt_peer.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
for r in 1 0; do SMILE_RET_DIRECT=$r timeout 300 python bench.py --no-cpu --no-e2e --steps 100 --mode bilevel > $O/bench_ret$r.log 2>&1; done
SMILE_RET_DIRECT=1 timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu --mode bilevel > $O/bench_c3.log 2>&1
N="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --mode bilevel --clock-ms 0"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ffn_gemm" -c 4 --csv --log-file $O/ffn.csv $N > /dev/null 2>&1
echo done
