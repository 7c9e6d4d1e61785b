"""ncclAlltoAll-only bus bandwidth per group size ("an ncclAlltoAll-only
microbenchmark per group size (2-, 4- and 8-way) gives achievable busBW").

    torchrun --nproc-per-node N tools/nccl_busbw.py [--mb 6,12,25] [--iters 20]

For every group size g in {2, 4, ..., N} (consecutive ranks, like the intra level; the
strided inter groups give the same numbers on one NVSwitch box) and every per-peer
message size, times torch.distributed.all_to_all_single (the torch-bundled NCCL 2.28, the
library libsmile links) with CUDA events, max over ranks, and prints one JSON line:
busBW = (g - 1) / g * bytes per rank / time (= bytes each rank sends to its peers / time),
in GB/s per direction.  Message sizes default to the capacity-padded chunks of the C2
layer: flat 4096 x 1536 B = 6.3 MB, intra (e * C2) 12.6 MB, inter (C1) 25.2 MB."""
import argparse
import json
import os

import torch
import torch.distributed as dist


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", default="0.25,1,6.29,12.58,25.17")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    sizes = [float(x) for x in args.mb.split(",")]
    res = []
    g = 2
    while g <= world:
        groups = [dist.new_group(list(range(b, b + g))) for b in range(0, world, g)]
        mine = groups[rank // g]
        for mb in sizes:
            per_peer = int(mb * 1e6) // 16 * 16
            src = torch.empty(g * per_peer, dtype=torch.uint8, device=dev)
            dst = torch.empty_like(src)
            for _ in range(args.warmup):
                dist.all_to_all_single(dst, src, group=mine)
            torch.cuda.synchronize()
            dist.barrier()
            e0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.iters)]
            e1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.iters)]
            for i in range(args.iters):
                e0[i].record()
                dist.all_to_all_single(dst, src, group=mine)
                e1[i].record()
            torch.cuda.synchronize()
            ts = sorted(e0[i].elapsed_time(e1[i]) for i in range(args.iters))
            t = torch.tensor([ts[len(ts) // 2]], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
            bus = (g - 1) * per_peer / (ms / 1e3) / 1e9
            res.append({"group": g, "per_peer_bytes": per_peer, "ms": ms, "busbw_GBps_per_direction": bus})
        g *= 2
    if rank == 0:
        env = {k: v for k, v in os.environ.items() if k.startswith("NCCL_")}
        print(json.dumps({"tool": "nccl_busbw", "world": world, "nccl_env": env,
                          "nccl_version": ".".join(map(str, torch.cuda.nccl.version())), "results": res}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
