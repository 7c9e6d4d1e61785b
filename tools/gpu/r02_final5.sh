# Round 2 final HEAD (A multicast default, gate / MMA-issuer work): smoke, every single-GPU
# test, default / C4 / C5 bench lines.
set -x
O=gpurun_out/r02f5
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 3000 python -m pytest tests -m gpu -q -x -k "not multigpu" > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_default.log 2>&1
for c in c4 c5; do timeout 900 python bench.py --config $c --steps 20 --no-cpu > $O/bench_$c.log 2>&1; done
echo done
