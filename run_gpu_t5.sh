set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "tcgen05" > gpurun_out/pt_ffn.log 2>&1; echo "rc=$?" >> gpurun_out/pt_ffn.log
timeout 300 python -m pytest tests/test_gpu_backward.py -q > gpurun_out/pt_bwd.log 2>&1; echo "rc=$?" >> gpurun_out/pt_bwd.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench_n1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n1.log
timeout 600 python bench.py --no-cpu --no-e2e --graph --steps 100 > gpurun_out/bench_n1_graph.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n1_graph.log
for c in c3 c4 c5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$c.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$c.log
done
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --mode bilevel --clock-ms 0"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo done
