# Training path after a change: backward parity, C3 bench, C3 launch list
set -x
mkdir -p gpurun_out/train
O=gpurun_out/train
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_backward.py tests/test_gpu_parity.py -q -x -k "backward or train or wgrad or bench_launch or empty" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu --mode bilevel > $O/bench_c3.log 2>&1
CMD="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --mode bilevel --clock-ms 0"
timeout 300 $CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv --log-file $O/launches.csv $CMD > $O/ncu.log 2>&1
echo done
