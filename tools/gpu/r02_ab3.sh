# Gate epilogue rework (chunked statistics, scaled-on-read softmax, resident split router in the
# swapped kernel): parity, timelines, same-box A/B against HEAD.
set -x
O=gpurun_out/r02ab4
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -q -x -m gpu -k "not multigpu" > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for cfg in c2 c4 c5; do
  SMILE_TRACE=gate timeout 300 python tools/gpu/trace_kernels.py --config $cfg --mode bilevel > $O/trace_${cfg}_gate.log 2>&1
done
SMILE_TRACE=gate SMILE_GATE_RESW=0 timeout 300 python tools/gpu/trace_kernels.py --config c2 --mode bilevel > $O/trace_c2_gate_resw0.log 2>&1
for round in 1 2; do
for v in head new resw0; do
  if [ $v = head ]; then export SMILE_LIB_PATH=$PWD/ab/libsmile_head.so; else unset SMILE_LIB_PATH; fi
  if [ $v = resw0 ]; then export SMILE_GATE_RESW=0; else unset SMILE_GATE_RESW; fi
  timeout 300 python bench.py --steps 50 --no-cpu --no-e2e > $O/c2_${v}_$round.log 2>&1
  if [ $v != resw0 ]; then
    timeout 300 python bench.py --config c4 --steps 10 --no-cpu --no-e2e > $O/c4_${v}_$round.log 2>&1
    timeout 300 python bench.py --config c5 --steps 10 --no-cpu --no-e2e > $O/c5_${v}_$round.log 2>&1
  fi
done
done
unset SMILE_LIB_PATH SMILE_GATE_RESW
for cfg in c2 c4 c5; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"gate1|scan1" -c 4 --csv \
    --log-file $O/launch_${cfg}.csv python bench.py --config $cfg --mode bilevel --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > /dev/null 2>&1
done
echo done
