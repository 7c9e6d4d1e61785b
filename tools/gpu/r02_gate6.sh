# Round 2: same-box A/B of the r01 gate kernel (old_r01/, git-ignored copy of commit 02343a3)
# against the ranged gate (in-kernel scan vs separate scan kernel), phase times + ncu.
set -x
O=gpurun_out/r02g6
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
(cd old_r01 && python -c "from paper_2212_05191_b200 import build; build.build()") > $O/build_old.log 2>&1
for i in 1 2; do
  (cd old_r01 && timeout 300 python bench.py --steps 50 --no-cpu --no-e2e --mode bilevel) > $O/old_c2_$i.log 2>&1
  timeout 300 python bench.py --steps 50 --no-cpu --no-e2e --mode bilevel > $O/new_c2_$i.log 2>&1
  SMILE_GATE_DIAG=4 timeout 300 python bench.py --steps 50 --no-cpu --no-e2e --mode bilevel > $O/new4_c2_$i.log 2>&1
done
(cd old_r01 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gate1|scan1|router_split" -c 6 --csv --log-file ../$O/l_old.csv \
    python bench.py --config c2 --mode bilevel --steps 2 --warmup 1 --no-e2e --no-cpu --clock-ms 0) > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gate1|scan1|router_split" -c 6 --csv --log-file $O/l_new.csv \
    python bench.py --config c2 --mode bilevel --steps 2 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > /dev/null 2>&1
SMILE_GATE_DIAG=4 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gate1|scan1|router_split" -c 6 --csv --log-file $O/l_new4.csv \
    python bench.py --config c2 --mode bilevel --steps 2 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gate1 -c 2 -o $O/ncu_new \
    python bench.py --config c2 --mode bilevel --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > /dev/null 2>&1
echo done
