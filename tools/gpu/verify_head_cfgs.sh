# Re-entry check of HEAD on one B200: the C3 (training), C4 and C5 bench lines and the reference arm.
set -x
O=gpurun_out/headc
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for c in c3 c4 c5; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu > $O/bench_$c.log 2>&1; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.log 2>&1
echo done
