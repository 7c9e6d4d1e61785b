# ncu --set full of one C5 and one C4 step (gate, movers, FFN) on the final HEAD.
set -x
O=gpurun_out/r02nf
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
K='gate1|scan1|row_move|ffn_gemm'
for c in c5 c4; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$K" -c 6 -o $O/ncu_${c}_step \
    python bench.py --config $c --mode bilevel --steps 1 --warmup 1 --no-e2e --no-cpu --clock-ms 0 > $O/ncu_${c}_step.log 2>&1
done
echo done
