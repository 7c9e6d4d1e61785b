# row mover register budget A/B (SMILE_MOVE_MINB 1 / 3), N = 1, alternating on one box
set -x
O=gpurun_out/mb
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
SMILE_MOVE_MINB=3 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "peer or out_direct or dispatch or combine" > $O/pt3.log 2>&1; echo "rc=$?" >> $O/pt3.log
for rep in 1 2; do for b in 3 1; do
  SMILE_MOVE_MINB=$b timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e > $O/n1_mb${b}_$rep.log 2>&1
  SMILE_MOVE_MINB=$b timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu --no-e2e > $O/c4_mb${b}_$rep.log 2>&1
done; done
echo done
