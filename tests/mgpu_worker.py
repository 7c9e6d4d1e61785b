"""torchrun worker for the multi-GPU parity test (tests/test_multigpu.py).

Every process builds the whole seeded problem (synth), runs its V = G/nprocs resident
ranks through libsmile (NCCL exchanges between processes, device copies inside one),
and rank 0 gathers every output and compares it with the CPU oracle."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from harness import Case, assert_close_scaled  # noqa: E402
from paper_2212_05191_b200 import SmileLayer, smile as smb  # noqa: E402


def main():
    cases = json.loads(sys.argv[1])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    failures = []
    for c in cases:
        case = Case(**{k: v for k, v in c.items() if not k.startswith("_")})
        G, V = case.G, case.G // world
        r0 = rank * V
        buf = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(smb.unique_id()), dtype=torch.uint8))
        dist.broadcast(buf, 0)
        topk = int(c.get("_topk", 1))
        layer = SmileLayer(case.n, case.m, case.e, case.d, case.d_ff, case.T, case.cf, case.dtype, case.mode,
                           nprocs=world, proc=rank, device=local, ffn_impl=case.ffn_impl,
                           nccl_id=bytes(buf.cpu().numpy().tobytes()), topk=topk)
        if c.get("_peer"):
            layer.alloc_workspace()

            def allgather(b):
                t = torch.frombuffer(bytearray(b), dtype=torch.uint8).to(dev)
                outs = [torch.empty_like(t) for _ in range(world)]
                dist.all_gather(outs, t)
                return b"".join(bytes(o.cpu().numpy().tobytes()) for o in outs)

            layer.enable_peer_exchange(allgather)
            dist.barrier()
        g = case.gpu_tensors(dev)
        e = case.e
        sl = lambda t, k=1: None if t is None else t[r0 * k:(r0 + V) * k].contiguous()
        out = torch.empty_like(sl(g["x"]))
        loss = torch.empty(V, dtype=torch.float64, device=dev)
        bwd = bool(c.get("_bwd"))
        xin, lin = sl(g["x"]), sl(g["logits"])
        fwd = lambda: layer.forward(xin, sl(g["W1t"], e), sl(g["b1"], e), sl(g["W2t"], e), sl(g["b2"], e), out, loss,
                                    logits=lin, w_router=g["w_router"], alpha=case.alpha, beta=case.beta, train=bwd)
        fwd()
        torch.cuda.synchronize()
        # routing state of every resident rank for the bit-exact route check (snapshot before
        # any graph replay overwrites it with the replayed inputs' routes)
        vw = {k: t.clone() for k, t in layer.view().items()}
        out_base, loss_base = out.clone(), loss.clone()
        graph_checks = []
        if c.get("_graph"):
            # smile_forward captured once as a CUDA graph and replayed on new inputs copied into
            # the captured buffers: the peer barriers' epochs must advance on the device per
            # replay (a host-side epoch would let replay 2 pass every barrier at once)
            torch.cuda.synchronize()
            dist.barrier()
            cg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(cg):
                fwd()
            for k in (1, 2):
                ck = Case(**{kk: (v + k if kk == "seed" else v) for kk, v in c.items() if not kk.startswith("_")})
                ck.W1, ck.b1, ck.W2, ck.b2, ck.w_router = case.W1, case.b1, case.W2, case.b2, case.w_router
                gk = ck.gpu_tensors(dev)
                xin.copy_(sl(gk["x"]))
                if lin is not None:
                    lin.copy_(sl(gk["logits"]))
                out.fill_(float("nan"))
                torch.cuda.synchronize()
                dist.barrier()
                cg.replay()
                torch.cuda.synchronize()
                outs_k = [torch.empty_like(out) for _ in range(world)]
                dist.all_gather(outs_k, out)
                losses_k = [torch.empty_like(loss) for _ in range(world)]
                dist.all_gather(losses_k, loss)
                graph_checks.append((ck, torch.cat(outs_k).float().cpu().numpy(), torch.cat(losses_k).cpu().numpy()))
            del cg
        grads = None
        if bwd:
            # a16-a19 over the same exchange; gout seeded identically on every process
            tdt = g["x"].dtype
            rs = np.random.default_rng(100)
            gout_np = rs.normal(size=(case.G, case.T, case.d)).astype(np.float32)
            if case.dtype == "bf16":
                import synth
                gout_np = synth.round_bf16(gout_np)
            gout = torch.from_numpy(gout_np).to(dev).to(tdt)
            W1 = torch.from_numpy(case.W1).to(dev).to(tdt)
            W2 = torch.from_numpy(case.W2).to(dev).to(tdt)
            f32 = dict(dtype=torch.float32, device=dev)
            NEl = V * e
            grads = dict(dx=torch.empty_like(out), dW1=torch.empty(NEl, case.d, case.d_ff, **f32),
                         db1=torch.empty(NEl, case.d_ff, **f32), dW2=torch.empty(NEl, case.d_ff, case.d, **f32),
                         db2=torch.empty(NEl, case.d, **f32),
                         dW=torch.empty(case.cfg.logit_width, case.d, **f32) if case.fused else None)
            layer.backward(sl(gout), grads["dx"], sl(W1, e), sl(W2, e), grads["dW1"], grads["db1"], grads["dW2"],
                           grads["db2"], dW_router=grads["dW"], lam=2.0)
        torch.cuda.synchronize()
        err = layer.get_error()
        outs = [torch.empty_like(out) for _ in range(world)]
        losses = [torch.empty_like(loss) for _ in range(world)]
        dist.all_gather(outs, out_base)
        dist.all_gather(losses, loss_base)
        rkeys = ["dest1", "dest2", "slot1", "counts1", "hist1"] + ([] if case.flat else ["rmeta1", "slot2", "counts2"])
        routes = {}
        for k in rkeys:
            parts = [torch.empty_like(vw[k]) for _ in range(world)]
            dist.all_gather(parts, vw[k].contiguous())
            # top-k: dest1 / slot1 are [k, V, T] choice-major -- ranks along dim 1
            routes[k] = torch.cat(parts, dim=1 if (topk > 1 and k in ("dest1", "slot1")) else 0).cpu().numpy()
        gathered = {}
        if grads is not None:
            for k, t in grads.items():
                if t is None:
                    continue
                if k == "dW":                     # each process holds its ranks' share of the tied router gradient
                    tot = t.clone()
                    dist.all_reduce(tot)
                    gathered[k] = tot
                else:
                    parts = [torch.empty_like(t) for _ in range(world)]
                    dist.all_gather(parts, t)
                    gathered[k] = torch.cat(parts)
        if rank == 0:
            try:
                assert err == 0, f"device error {err}"
                lg_or = None
                if case.fused:
                    lg_or = oracle.logits(case.x.reshape(-1, case.d), case.w_router).reshape(case.G, case.T, -1)
                if topk > 1:
                    # the FLAT top-k layer (Eq. 2, R29-R32) across processes
                    rt = oracle.route_topk(case.cfg, topk, case.logits)
                    np.testing.assert_array_equal(routes["dest1"], rt.dest)
                    np.testing.assert_array_equal(routes["slot1"], rt.slot)
                    np.testing.assert_array_equal(routes["counts1"], rt.counts)
                    got = torch.cat(outs).float().cpu().numpy().reshape(-1, case.d)
                    assert_close_scaled(got, oracle.out_rows_topk(case.cfg, rt, case.x, case.W1, case.b1, case.W2,
                                                                  case.b2), 2e-2 if case.dtype == "bf16" else 1e-5,
                                        f"mgpu top-{topk} {c}")
                    np.testing.assert_allclose(torch.cat(losses).cpu().numpy(), rt.loss, rtol=1e-6)
                    raise StopIteration
                r = case.oracle_route()
                # routing indices, capacity slots, drop masks and counts: bit-exact (north star).
                # Fused router: the GPU's fp32 logits may differ from the oracle's in the last
                # ulp, so compare where the top-2 margin is clear and require agreement there.
                if not case.fused:
                    np.testing.assert_array_equal(routes["dest1"], r.dest1)
                    np.testing.assert_array_equal(routes["dest2"], r.dest2 if not case.flat else 0 * r.dest2)
                    np.testing.assert_array_equal(routes["slot1"], r.slot1)
                    np.testing.assert_array_equal(routes["counts1"], r.counts1)
                    np.testing.assert_array_equal(routes["hist1"], r.A1)
                    if not case.flat:
                        np.testing.assert_array_equal(routes["rmeta1"], r.jin)
                        valid = r.jin >= 0
                        np.testing.assert_array_equal(routes["slot2"][valid], r.slot2[valid])
                        np.testing.assert_array_equal(routes["counts2"], r.counts2)
                else:
                    K1 = case.n if not case.flat else lg_or.shape[-1]
                    srt = np.sort(lg_or[:, :, :K1], axis=-1)
                    clear = (srt[..., -1] - srt[..., -2]) > 1e-4
                    np.testing.assert_array_equal(routes["dest1"][clear], r.dest1[clear])
                got = torch.cat(outs).float().cpu().numpy().reshape(-1, case.d)
                ref = case.oracle_out(r)
                assert_close_scaled(got, ref, 2e-2 if case.dtype == "bf16" else 1e-5, f"mgpu {c}")
                keep = r.keep.reshape(-1).astype(bool)
                assert (got[~keep] == 0).all()
                np.testing.assert_allclose(torch.cat(losses).cpu().numpy(), r.loss, rtol=1e-6)
                for ck, ok, lk in graph_checks:
                    rk = ck.oracle_route()
                    assert_close_scaled(ok.reshape(-1, case.d), ck.oracle_out(rk), 2e-2 if case.dtype == "bf16" else 1e-5,
                                        f"mgpu graph replay {c}")
                    np.testing.assert_allclose(lk, rk.loss, rtol=1e-6)
                if gathered:
                    ref = oracle.backward(case.cfg, r, case.x, case.W1, case.b1, case.W2, case.b2, gout_np, lam=2.0,
                                          W=case.w_router if case.fused else None,
                                          logits=None if case.fused else case.logits)
                    tol = 3e-2 if case.dtype == "bf16" else 1e-4
                    for k, t in gathered.items():
                        assert_close_scaled(t.float().cpu().numpy().reshape(ref[k].shape), ref[k], tol, f"mgpu bwd {k}")
            except StopIteration:
                pass
            except AssertionError as ex:
                failures.append(f"{c}: {ex}")
        torch.cuda.synchronize()
        dist.barrier()          # every peer is done with our workspace before it is freed
        layer.close()
        if rank == 0:
            print("MGPU_CASE_DONE", c, flush=True)
    dist.destroy_process_group()
    if rank == 0:
        print("MGPU_RESULT", json.dumps({"failures": failures, "cases": len(cases)}))
        sys.exit(1 if failures else 0)


if __name__ == "__main__":
    main()
