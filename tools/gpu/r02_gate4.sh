# Round 2: isolate the ranged gate's slowdown (SMILE_GATE_DIAG bits: 1 W box 128 rows, 2 split kernel, 4 scan kernel)
set -x
O=gpurun_out/r02g4
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for sch in contig rounds; do for dg in 0 1 2 4 7; do
  SMILE_GATE_SCHED=$sch SMILE_GATE_DIAG=$dg timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gate1 -c 3 --csv --log-file $O/l_${sch}_$dg.csv \
    python bench.py --config c2 --mode bilevel --steps 2 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > /dev/null 2>&1
done; done
SMILE_GATE_SWAP=0 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:gate1 -c 3 --csv --log-file $O/l_swap0.csv \
    python bench.py --config c2 --mode bilevel --steps 2 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > /dev/null 2>&1
git -C . log --oneline -1 > $O/rev.txt 2>&1
echo done
