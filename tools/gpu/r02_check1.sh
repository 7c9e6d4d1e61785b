# Round 2 check 1: build, single-GPU tests, smoke, default bench line, box facts.
set -x
O=gpurun_out/r02c1
mkdir -p $O
nproc > $O/nproc.txt; lscpu > $O/lscpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "not multigpu" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py --steps 50 > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
echo done
