set -x
O=gpurun_out/r02tb
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_topk.py tests/test_gpu_backward.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --mode flat --topk 2 --config c3 --steps 10 --no-cpu > $O/bench_c3_flat_top2.log 2>&1
echo done
