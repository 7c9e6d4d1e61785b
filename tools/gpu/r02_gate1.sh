# Round 2: ranged tensor-core gate (chunk tables, in-kernel split + scan) + chunked forward API.
set -x
O=gpurun_out/r02g1
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_router or fused_gate or c1_full or shapes or peer or out_direct or signed or determinism or host_stream" > $O/pytest_gate.log 2>&1; echo "rc=$?" >> $O/pytest_gate.log
timeout 600 python -m pytest tests/test_gpu_chunked.py -q -x > $O/pytest_chunked.log 2>&1; echo "rc=$?" >> $O/pytest_chunked.log
timeout 300 python bench.py --steps 50 --no-cpu --no-e2e > $O/bench_c2.log 2>&1
timeout 300 python bench.py --config c4 --steps 20 --no-cpu --no-e2e > $O/bench_c4.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gate1 -c 2 -o $O/ncu_gate_c2 \
    python bench.py --config c2 --mode bilevel --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > $O/ncu_gate_c2.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x > $O/pytest_fullsize.log 2>&1; echo "rc=$?" >> $O/pytest_fullsize.log
timeout 600 python -m pytest tests -m gpu -q -x -k "not multigpu and not fullsize" > $O/pytest_all.log 2>&1; echo "rc=$?" >> $O/pytest_all.log
for ch in 2 4; do timeout 300 python bench.py --chunks $ch --steps 30 > $O/bench_chunks$ch.log 2>&1; done
SMILE_FFN_CTA_PAIR=1 timeout 300 python bench.py --config c5 --mode bilevel --steps 20 --no-cpu --no-e2e > $O/bench_c5_pair.log 2>&1
echo done
