# C3 training step: launch list (per-kernel times) of one fwd+bwd step
set -x
mkdir -p gpurun_out/c3
O=gpurun_out/c3
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
CMD="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --mode bilevel --clock-ms 0"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file $O/launches.csv $CMD > $O/ncu.log 2>&1
echo done
