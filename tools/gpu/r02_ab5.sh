# Resident split router build (column-parallel loads): gate parity + C2 timeline + A/B.
set -x
O=gpurun_out/r02ab6
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_topk.py tests/test_gpu_backward.py -q -x > $O/pytest_gate.log 2>&1; echo "rc=$?" >> $O/pytest_gate.log
SMILE_TRACE=gate timeout 300 python tools/gpu/trace_kernels.py --config c2 --mode bilevel > $O/trace_c2_gate.log 2>&1
for round in 1 2; do
for v in new resw0; do
  if [ $v = resw0 ]; then export SMILE_GATE_RESW=0; else unset SMILE_GATE_RESW; fi
  timeout 300 python bench.py --steps 50 --no-cpu --no-e2e > $O/c2_${v}_$round.log 2>&1
done
done
unset SMILE_GATE_RESW
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"gate1|scan1" -c 4 --csv \
    --log-file $O/launch_c2.csv python bench.py --config c2 --mode bilevel --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > /dev/null 2>&1
echo done
