# after the 128-row-tile heuristic for small experts: all GPU tests, C2 and C5 bench
set -x
mkdir -p gpurun_out/cg
O=gpurun_out/cg
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "not multigpu" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python bench.py --no-cpu --no-e2e --steps 100 --mode bilevel > $O/bench_c2.log 2>&1
timeout 300 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu > $O/bench_c5.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
echo done
