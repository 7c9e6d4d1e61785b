"""PCIe probe: pinned H2D / D2H bandwidth, one vs two streams, uni- and bidirectional."""
import torch
N = 201326592
h = torch.empty(N, dtype=torch.uint8).pin_memory()
h2 = torch.empty(N, dtype=torch.uint8).pin_memory()
d = torch.empty(N, dtype=torch.uint8, device="cuda")
d2 = torch.empty(N, dtype=torch.uint8, device="cuda")
s = [torch.cuda.Stream() for _ in range(4)]


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    for st in s:
        torch.cuda.current_stream().wait_stream(st)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d(k):
    def f():
        ch = N // k
        for i in range(k):
            with torch.cuda.stream(s[i]):
                d[i * ch:(i + 1) * ch].copy_(h[i * ch:(i + 1) * ch], non_blocking=True)
    return f


def d2h(k):
    def f():
        ch = N // k
        for i in range(k):
            with torch.cuda.stream(s[i]):
                h2[i * ch:(i + 1) * ch].copy_(d2[i * ch:(i + 1) * ch], non_blocking=True)
    return f


def both(k):
    def f():
        h2d(k)()
        ch = N // k
        for i in range(k):
            with torch.cuda.stream(s[(i + 2) % 4]):
                h2[i * ch:(i + 1) * ch].copy_(d2[i * ch:(i + 1) * ch], non_blocking=True)
    return f


for k in (1, 2, 4):
    t = timed(h2d(k))
    print(f"H2D {k} streams: {t:.3f} ms = {N / t / 1e6:.1f} GB/s")
    t = timed(d2h(k))
    print(f"D2H {k} streams: {t:.3f} ms = {N / t / 1e6:.1f} GB/s")
for k in (1, 2):
    t = timed(both(k))
    print(f"H2D+D2H concurrent ({k} streams each): {t:.3f} ms = {N / t / 1e6:.1f} GB/s per direction")
