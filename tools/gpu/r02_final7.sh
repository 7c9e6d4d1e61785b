# Final HEAD bench lines (default contract run, graph, reference arm) and smoke.
set -x
O=gpurun_out/r02f7
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_default.log 2>&1
timeout 600 python bench.py --steps 100 --no-cpu --graph > $O/bench_graph.log 2>&1
timeout 900 python bench.py --config c3 --steps 20 --no-cpu > $O/bench_c3.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.log 2>&1
echo done
