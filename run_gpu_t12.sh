set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in 2 4; do
  timeout 300 python bench.py --chunks $c --mode both --steps 50 --warmup 3 > gpurun_out/pipe_c$c.log 2>&1
  SMILE_FFN_MAX_CTAS=128 timeout 300 python bench.py --chunks $c --mode both --steps 50 --warmup 3 > gpurun_out/pipe_c${c}_128.log 2>&1
  SMILE_FFN_MAX_CTAS=112 timeout 300 python bench.py --chunks $c --mode both --steps 50 --warmup 3 > gpurun_out/pipe_c${c}_112.log 2>&1
done
timeout 300 python bench.py --mode both --steps 50 --no-e2e --no-cpu > gpurun_out/pipe_c1.log 2>&1
python - > gpurun_out/cublas_shapes.log 2>&1 <<'PY'
import torch
torch.backends.cuda.matmul.allow_tf32=False
for (M,K,N) in [(131072,768,3072),(131072,3072,768),(8192,8192,8192)]:
    a=torch.randn(M,K,device='cuda',dtype=torch.bfloat16); b=torch.randn(K,N,device='cuda',dtype=torch.bfloat16)
    for _ in range(3): c=a@b
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): c=a@b
    e1.record(); torch.cuda.synchronize()
    t=e0.elapsed_time(e1)/20
    print(M,K,N, f"{t:.3f} ms", f"{2*M*K*N/t/1e9:.0f} TFLOP/s")
PY
echo done
