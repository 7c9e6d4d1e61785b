# scan1 / scan2 over V x nb blocks: parity + C2 / C4 / C5 gate phases + launch list.
set -x
O=gpurun_out/r02scan2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -k "not multigpu" > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python bench.py --steps 50 --no-cpu --no-e2e > $O/c2.log 2>&1
timeout 300 python bench.py --config c4 --steps 10 --no-cpu --no-e2e > $O/c4.log 2>&1
timeout 300 python bench.py --config c5 --steps 10 --no-cpu --no-e2e > $O/c5.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"scan1|scan2|gate1|rank2" -c 4 --csv --log-file $O/ncu_c5.csv \
    python bench.py --config c5 --mode bilevel --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > /dev/null 2>&1
echo done
