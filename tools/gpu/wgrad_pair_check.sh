set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_backward.py -q -x > gpurun_out/pt_bwd.log 2>&1; echo "rc=$?" >> gpurun_out/pt_bwd.log
for v in 1 0; do SMILE_WGRAD_CTA_PAIR=$v timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu --mode bilevel > gpurun_out/c3_wpair$v.log 2>&1; done
CMD3="python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --mode bilevel --clock-ms 0"
timeout 300 $CMD3 > gpurun_out/plain3.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:wgrad -c 6 --csv --log-file gpurun_out/wgrad.csv $CMD3 > gpurun_out/ncu_w.log 2>&1
echo done
