# Round 2: r01 swapped gate + in-kernel split + PDL; batched scan; headline from un-instrumented steps.
set -x
O=gpurun_out/r02g8
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_topk.py tests/test_gpu_parity.py -q -x -k "topk or fused_router or c1_full or shapes or fused_gate or bench_launch or graph or host_stream or determinism" > $O/pytest_quick.log 2>&1; echo "rc=$?" >> $O/pytest_quick.log
for v in "X=0" "SMILE_GATE_SPLIT_KERNEL=1" "SMILE_PDL=0"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gate1|scan1|router_split" -c 6 --csv --log-file $O/l_$tag.csv \
    python bench.py --config c2 --mode bilevel --steps 2 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > /dev/null 2>&1
  env $v timeout 300 python bench.py --steps 50 --no-cpu --no-e2e > $O/bench_c2_$tag.log 2>&1
done
timeout 300 python bench.py --config c4 --steps 20 --no-cpu --no-e2e > $O/bench_c4.log 2>&1
timeout 300 python bench.py --steps 50 --no-cpu --no-e2e --graph > $O/bench_c2_graph.log 2>&1
echo done
