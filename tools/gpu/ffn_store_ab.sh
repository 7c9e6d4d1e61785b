# FFN epilogue output path A/B on one B200: TMA tensor stores (default) vs st.global.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for ts in 1 0; do
  SMILE_FFN_TMA_STORE=$ts timeout 600 python bench.py --no-cpu --no-e2e --steps 100 > gpurun_out/ab_tmastore$ts.log 2>&1
  SMILE_FFN_TMA_STORE=$ts timeout 600 python bench.py --no-cpu --no-e2e --steps 10 --config c4 --mode bilevel > gpurun_out/ab_c4_tmastore$ts.log 2>&1
done
echo done
