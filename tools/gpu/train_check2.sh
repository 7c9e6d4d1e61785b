# After the dZ-epilogue db1 fusion and the per-epilogue-kind instantiations: all GPU tests,
# C2 + C3 bench, C3 launch list
set -x
mkdir -p gpurun_out/train2
O=gpurun_out/train2
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "not multigpu" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python bench.py --no-cpu --no-e2e --steps 100 --mode bilevel > $O/bench_c2.log 2>&1
timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu --mode bilevel > $O/bench_c3.log 2>&1
CMD="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --mode bilevel --clock-ms 0"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file $O/launches.csv $CMD > $O/ncu.log 2>&1
echo done
