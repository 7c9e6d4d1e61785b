set -x
O=gpurun_out/r02tb2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_topk.py -q -k backward > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
echo done
