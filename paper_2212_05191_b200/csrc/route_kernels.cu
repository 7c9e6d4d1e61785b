// route_kernels.cu -- gate, capacity scan, permute, un-permute, combine and aux-loss
// kernels of the SMILE layer.
//
// The capacity rule (R5, R8) assigns every token a slot = number of EARLIER tokens of
// its rank with the same destination.  It is computed exactly (integers, so the result
// is order-independent and deterministic) in two steps: the gate kernel ranks tokens
// inside a block with __match_any_sync + a cross-warp scan and publishes the block's
// per-destination histogram; a scan kernel turns the histograms into per-block offsets;
// the permute kernel adds the offset and moves the row.
#include "smile_internal.h"
#include "gate_common.cuh"

#include <math.h>
#include <stdlib.h>

namespace smile {
namespace {


__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ float load_elem(const void *p, int64_t i, int bf16) {
    return bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16 *>(p)[i])
                : reinterpret_cast<const float *>(p)[i];
}

// Copy one row of `nvec` 16-byte vectors with a warp (4 loads in flight per lane).
__device__ __forceinline__ void warp_copy_row(int4 *__restrict__ dst, const int4 *__restrict__ src,
                                              int nvec, int lane) {
    int i = lane;
    for (; i + 96 < nvec; i += 128) {
        int4 a = __ldg(src + i), b = __ldg(src + i + 32), c = __ldg(src + i + 64), d = __ldg(src + i + 96);
        dst[i] = a; dst[i + 32] = b; dst[i + 64] = c; dst[i + 96] = d;
    }
    for (; i < nvec; i += 32) dst[i] = __ldg(src + i);
}

__device__ __forceinline__ void warp_zero_row(int4 *dst, int nvec, int lane) {
    const int4 z = make_int4(0, 0, 0, 0);
    for (int i = lane; i < nvec; i += 32) dst[i] = z;
}

// a1: fused router for one block's tokens.  One warp computes RT tokens at a time: each
// lane loads 16-byte chunks of the RT rows of x, multiplies them with the matching
// chunk of every router row (fp32, staged in smem when KW*d*4 <= kRouterSmem), and the
// partial dot products are reduced with a butterfly (fixed order: deterministic).
constexpr int kRT = 4;
constexpr int kRouterSmem = 48 * 1024;

template <bool BF16>
__device__ void router_tile(const GateArgs &a, float *s_lg, int lds, float *s_w, int64_t tok0, int nt) {
    constexpr int EPV = BF16 ? 8 : 4;          // elements per 16-byte vector
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = blockDim.x >> 5;
    const int KW = a.KW, d = a.d, nchunk = d / EPV;
    const bool wsm = (size_t)KW * d * 4 <= (size_t)kRouterSmem;
    if (wsm) {
        const float4 *src = reinterpret_cast<const float4 *>(a.w);
        float4 *dst = reinterpret_cast<float4 *>(s_w);
        for (int i = threadIdx.x; i < KW * d / 4; i += blockDim.x) dst[i] = __ldg(src + i);
        __syncthreads();
    }
    const float *W = wsm ? s_w : a.w;
    for (int tt0 = w * kRT; tt0 < nt; tt0 += NW * kRT) {
        for (int k0 = 0; k0 < KW; k0 += 8) {
            float acc[kRT][8];
#pragma unroll
            for (int r = 0; r < kRT; ++r)
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) acc[r][kk] = 0.f;
            for (int c = lane; c < nchunk; c += 32) {
                float xv[kRT][EPV];
#pragma unroll
                for (int r = 0; r < kRT; ++r) {
                    if (tt0 + r < nt) {
                        const int4 u = __ldg(reinterpret_cast<const int4 *>(
                            static_cast<const char *>(a.x) + ((tok0 + tt0 + r) * d + (int64_t)c * EPV) * (BF16 ? 2 : 4)));
                        if (BF16) {
                            const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
                            for (int z = 0; z < 4; ++z) {
                                const float2 f = __bfloat1622float2(h[z]);
                                xv[r][2 * z] = f.x;
                                xv[r][2 * z + 1] = f.y;
                            }
                        } else {
                            const float *f = reinterpret_cast<const float *>(&u);
#pragma unroll
                            for (int z = 0; z < EPV; ++z) xv[r][z] = f[z];
                        }
                    } else {
#pragma unroll
                        for (int z = 0; z < EPV; ++z) xv[r][z] = 0.f;
                    }
                }
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    if (k0 + kk >= KW) break;
                    const float *wr = W + (int64_t)(k0 + kk) * d + c * EPV;
                    float wv[EPV];
#pragma unroll
                    for (int z = 0; z < EPV; z += 4) {
                        const float4 q = wsm ? *reinterpret_cast<const float4 *>(wr + z)
                                             : __ldg(reinterpret_cast<const float4 *>(wr + z));
                        wv[z] = q.x; wv[z + 1] = q.y; wv[z + 2] = q.z; wv[z + 3] = q.w;
                    }
#pragma unroll
                    for (int r = 0; r < kRT; ++r)
#pragma unroll
                        for (int z = 0; z < EPV; ++z) acc[r][kk] = fmaf(xv[r][z], wv[z], acc[r][kk]);
                }
            }
#pragma unroll
            for (int r = 0; r < kRT; ++r)
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    float v = acc[r][kk];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
                    if (lane == 0 && k0 + kk < KW && tt0 + r < nt) s_lg[(tt0 + r) * lds + k0 + kk] = v;
                }
        }
    }
}

// ---------------------------------------------------------------------------------
// a1-a3: level-1 gate.  grid (nblk, V), block TB threads (one token per thread).
// smem: logits tile [TB][lds] fp32 | s_j [TB] | warp hist [NW][K1] | block hist [K1]
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 2) gate1_kernel(GateArgs a) {
    pdl_wait();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float *s_lg = reinterpret_cast<float *>(smem_raw);
    const int lds = gate_lds(a.KW);
    int *s_j = reinterpret_cast<int *>(s_lg + (size_t)a.TB * lds);
    int *s_wh = s_j + a.TB;
    int *s_bh = s_wh + (((a.TB / 32) * a.K1 + 3) & ~3);               // 16-byte aligned below
    double *s_part = reinterpret_cast<double *>(s_bh + ((a.K1 + 3) & ~3));   // gate_finish scratch
    float *s_w = reinterpret_cast<float *>(reinterpret_cast<unsigned char *>(s_part) +
                                           ((gate_scratch_bytes(a.TB, a.KW, a.K2) + 15) & ~(size_t)15));   // [KW, d] when it fits

    const int v = blockIdx.y, blk = blockIdx.x, tid = threadIdx.x;
    const int64_t t0 = (int64_t)blk * a.TB;
    const int nt = (int)imin64(a.TB, a.T - t0);
    const int KW = a.KW, K1 = a.K1, K2 = a.K2;
    const int64_t tok0 = (int64_t)v * a.T + t0;

    // Phase A: the block's logits tile (Eq. 1: r = W x).
    if (a.logits) {
        const float *src = a.logits + tok0 * KW;
        for (int i = tid; i < nt * KW; i += blockDim.x) s_lg[(i / KW) * lds + i % KW] = __ldg(src + i);
    } else if (a.bf16) {
        router_tile<true>(a, s_lg, lds, s_w, tok0, nt);
    } else {
        router_tile<false>(a, s_lg, lds, s_w, tok0, nt);
    }
    __syncthreads();
    if (a.logits_out && !a.logits)
        for (int i = tid; i < nt * KW; i += blockDim.x) a.logits_out[tok0 * KW + i] = s_lg[(i / KW) * lds + i % KW];
    if (a.logits_out && !a.logits) __syncthreads();

    gate_finish<BlockSync>(a, s_lg, lds, s_j, s_wh, s_bh, s_part, tok0, nt, (int64_t)v * a.nblk + blk);
}

// Level-1 scan over the per-chunk tables (gate_common.cuh scan1_rank), grid = V.
// grid = V x nb: the rank's independent jobs (one scan / sum per destination or statistic,
// a warp each) are spread over nb blocks, so a wide router's 100+ jobs run in one round
// (C5: 132 jobs, 18 -> a few us).
__global__ void scan1_kernel(Scan1Args a) {
    pdl_wait();
    const int nb = gridDim.x / a.V;
    const int v = blockIdx.x / nb, bi = blockIdx.x - v * nb;
    if (a.lb_flag && bi == 0)                        // the fused gate's look-back flags, for the next call
        for (int b = threadIdx.x; b < a.nlb; b += blockDim.x) a.lb_flag[(int64_t)v * a.nlb + b] = 0;
    const int wpb = blockDim.x >> 5;
    scan1_rank(a, v, bi * wpb + (threadIdx.x >> 5), nb * wpb);
}

// a6: level-2 gate at the intermediate: rank valid received slots per j, in received
// order (source node ascending, then slot: the flat index s*C1 + c, R8).
__global__ void rank2_kernel(Rank2Args a) {
    pdl_wait();
    __shared__ int s_wh[(kRank2Items / 32) * 256];
    __shared__ int s_bh[256];
    const int v = blockIdx.y, blk = blockIdx.x;
    const int64_t x = (int64_t)blk * kRank2Items + threadIdx.x;
    int b = -1;
    if (x < a.items) {
        b = a.recv_meta[(int64_t)v * a.items + x];
        if (b >= a.K2) { set_err(a.err, SMILE_EINDEX); b = -1; }
    }
    const int lr = block_rank<BlockSync>(b, a.K2, s_wh, s_bh);
    if (x < a.items) a.slot2[(int64_t)v * a.items + x] = lr;
    for (int k = threadIdx.x; k < a.K2; k += blockDim.x)
        a.blk_hist2[((int64_t)v * a.nblk + blk) * a.K2 + k] = s_bh[k];
}

// grid = V x nb: a rank's K2 destination scans (a warp each) spread over nb blocks
__global__ void scan2_kernel(Rank2Args a) {
    pdl_wait();
    const int nb = gridDim.x / a.V;
    const int v = blockIdx.x / nb, bi = blockIdx.x - v * nb;
    const int w = bi * (blockDim.x >> 5) + (threadIdx.x >> 5), NW = nb * (blockDim.x >> 5), lane = threadIdx.x & 31;
    for (int k = w; k < a.K2; k += NW) {
        const int64_t o = (int64_t)v * a.nblk * a.K2 + k;
        const int tot = warp_exclusive_scan(a.blk_hist2 + o, a.nblk, a.K2, a.blk_off2 + o);
        if (lane == 0) {
            a.counts2[v * a.K2 + k] = (int32_t)imin64(tot, a.C2);
            if (a.peer.bases) {                    // rcounts[(i, k / e)][l][k % e] of the expert rank
                const PeerMap &P = a.peer;
                const int rk = P.rank0 + v, i = rk / P.m, l = rk % P.m, q = i * P.m + k / P.e;
                reinterpret_cast<int32_t *>(P.bases[q / P.V] + P.off_rcounts)[((int64_t)(q % P.V) * P.m + l) * P.e + k % P.e] =
                    (int32_t)imin64(tot, a.C2);
            }
        }
    }
}

// Row movers (a4, a7, a11, a13): plan_row resolves each row's source / destination (and
// the slot bookkeeping); row_move_body moves the rows warp by warp with 16-byte loads,
// several rows' loads in flight per lane (see there).  A source of nullptr writes a zero
// row (a dropped token, a13); a scale != 1 multiplies by the gate (a13).
enum MoveKind { MOVE_DISPATCH1 = 0, MOVE_DISPATCH2 = 1, MOVE_COMBINE2 = 2, MOVE_COMBINE1 = 3, MOVE_GRAD2 = 4 };

struct MoveArgs {
    int kind;
    int64_t rows;            // total rows (V * items)
    int64_t rowbytes;
    Dispatch1Args d1;
    Dispatch2Args d2;
    Combine2Args c2;
    Combine1Args c1;
};

struct RowPlan {
    const char *src;         // nullptr: zero row
    char *dst;               // nullptr: nothing to store
    float scale;             // != 1: multiply (combine1)
};

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ RowPlan plan_row(const MoveArgs &m, int64_t g) {   // g: the mover's row (item) index
    RowPlan r{nullptr, nullptr, 1.f};
    if (m.kind == MOVE_DISPATCH1) {
        // item gi = choice j of token g (top-k: choice-major, R31; top-1: gi = g)
        const Dispatch1Args &a = m.d1;
        const int64_t gi = g;
        const int64_t VT = (int64_t)a.V * a.T;
        const int jc = (int)(gi / VT);
        g = gi - (int64_t)jc * VT;
        const int v = (int)(g / a.T);
        const int64_t t = g - (int64_t)v * a.T;
        const int i = a.route.dest1[gi];
        const int slot = a.blk_off1[(((int64_t)v * a.topk + jc) * a.nblk + t / a.TB) * a.K1 + i] + a.route.slot1[gi];
        a.route.slot1[gi] = slot;                                     // finalise (R5, R8, R31)
        if (slot < a.C1) {
            r.src = static_cast<const char *>(a.x) + g * a.rowbytes;
            if (a.peer.bases) {
                // peer store straight into the receive buffer of the level-1 destination
                const PeerMap &P = a.peer;
                const int rk = P.rank0 + v;
                int q;
                int64_t row;
                if (a.meta) {                      // bi-level: (s, l) -> intermediate (i, l), chunk s
                    const int s_ = rk / P.m, l = rk % P.m;
                    q = i * P.m + l;
                    row = ((int64_t)(q % P.V) * P.n + s_) * a.C1 + slot;
                } else {                           // flat: expert E = i on rank E / e, chunk (src, E % e)
                    q = i / P.e;
                    row = (((int64_t)(q % P.V) * P.G + rk) * P.e + i % P.e) * a.C1 + slot;
                }
                char *base = P.bases[q / P.V];
                r.dst = base + P.off_recv1 + row * a.rowbytes;
                if (a.meta) {
                    reinterpret_cast<int32_t *>(base + P.off_rmeta1)[row] = a.route.dest2[g];
                    reinterpret_cast<int32_t *>(base + P.off_rtok1)[row] = (int32_t)t;   // source token
                } else {
                    // flat: the received row IS the expert's input row -- its source token
                    // lets GEMM 2 write the output row straight to out[t] (smile_set_output)
                    reinterpret_cast<int32_t *>(base + P.off_rtok2)[row] = (int32_t)t;
                }
            } else {
                const int64_t dst_row = ((int64_t)v * a.K1 + i) * a.C1 + slot;
                r.dst = static_cast<char *>(a.send) + dst_row * a.rowbytes;
                if (a.meta) a.meta[dst_row] = a.route.dest2[g];
            }
        } else if (a.out) {
            r.dst = static_cast<char *>(a.out) + g * a.rowbytes;     // dropped (R8): zero output row
        }
    } else if (m.kind == MOVE_DISPATCH2) {
        const Dispatch2Args &a = m.d2;
        const int j = a.recv_meta[g];
        if (j >= 0 && j < a.K2) {
            const int v = (int)(g / a.items);
            const int64_t x = g - (int64_t)v * a.items;
            const int slot = a.blk_off2[((int64_t)v * a.nblk + x / kRank2Items) * a.K2 + j] + a.slot2[g];
            a.slot2[g] = slot;
            if (slot < a.C2) {
                r.src = static_cast<const char *>(a.recv1) + g * a.rowbytes;
                if (a.peer.bases) {
                    // peer store into the expert rank (i, j / e), chunk (l, j % e), and the
                    // row's place in this rank's ret1 (row g), where the expert's GEMM 2
                    // will store its output (a10 + a11 fused into the FFN)
                    const PeerMap &P = a.peer;
                    const int rk = P.rank0 + v, i = rk / P.m, l = rk % P.m;
                    const int q = i * P.m + j / P.e;
                    const int64_t row = (((int64_t)(q % P.V) * P.m + l) * P.e + j % P.e) * a.C2 + slot;
                    r.dst = P.bases[q / P.V] + P.off_recv2 + row * a.rowbytes;
                    reinterpret_cast<int32_t *>(P.bases[q / P.V] + P.off_rrow)[row] = (int32_t)g;
                    reinterpret_cast<int32_t *>(P.bases[q / P.V] + P.off_rtok2)[row] =
                        reinterpret_cast<const int32_t *>(P.bases[P.rank0 / P.V] + P.off_rtok1)[g];
                } else {
                    r.dst = static_cast<char *>(a.send2) + (((int64_t)v * a.K2 + j) * a.C2 + slot) * a.rowbytes;
                }
            } else if (a.peer.bases && a.ret1) {
                // dropped at level 2 (R8): its return row is zero (written now; the fused
                // GEMM 2 writes only kept rows)
                r.dst = static_cast<char *>(a.ret1) + g * a.rowbytes;
                if (a.out) {
                    // output bound: when the source rank and the expert share this process the
                    // combine skips the token, so its zero output row is written here too
                    const PeerMap &P = a.peer;
                    const int rk = P.rank0 + v, i = rk / P.m, l = rk % P.m;
                    const int us = (int)(x / (a.items / P.n)) * P.m + l;    // source (s, l): x = s C1 + c
                    const int q = i * P.m + j / P.e;
                    const int me = P.rank0 / P.V;
                    if (us / P.V == me && q / P.V == me) {
                        const int tt = reinterpret_cast<const int32_t *>(P.bases[me] + P.off_rtok1)[g];
                        int4 *o = reinterpret_cast<int4 *>(static_cast<char *>(a.out) +
                                                           ((int64_t)(us % P.V) * a.T + tt) * a.rowbytes);
                        for (int k = 0; k < (int)(a.rowbytes / 16); ++k) o[k] = make_int4(0, 0, 0, 0);
                    }
                }
            }
        }
    } else if (m.kind == MOVE_GRAD2) {
        // gradient rows follow the forward route with the forward's final slot2 (a16)
        const Dispatch2Args &a = m.d2;
        const int j = a.recv_meta[g];
        if (j >= 0 && j < a.K2) {
            const int v = (int)(g / a.items);
            const int slot = a.slot2[g];
            if (slot < a.C2) {
                r.src = static_cast<const char *>(a.recv1) + g * a.rowbytes;
                if (a.peer.bases) {
                    // PEER: straight into the expert's Y buffer (where dY is consumed), at the
                    // row the forward permute used for this token
                    const PeerMap &P = a.peer;
                    const int rk = P.rank0 + v, i = rk / P.m, l = rk % P.m;
                    const int q = i * P.m + j / P.e;
                    const int64_t row = (((int64_t)(q % P.V) * P.m + l) * P.e + j % P.e) * a.C2 + slot;
                    r.dst = P.bases[q / P.V] + P.off_Y + row * a.rowbytes;
                } else {
                    r.dst = static_cast<char *>(a.send2) + (((int64_t)v * a.K2 + j) * a.C2 + slot) * a.rowbytes;
                }
            }
        }
    } else if (m.kind == MOVE_COMBINE2) {
        const Combine2Args &a = m.c2;
        const int j = a.recv_meta[g];
        if (j >= 0 && j < a.K2) {
            const int v = (int)(g / a.items);
            const int s2 = a.slot2[g];
            r.dst = static_cast<char *>(a.ret1) + g * a.rowbytes;
            if (s2 < a.C2) {
                if (a.peer.bases) {
                    // peer load of the expert output from rank (i, j / e), chunk (l, j % e)
                    const PeerMap &P = a.peer;
                    const int rk = P.rank0 + v, i = rk / P.m, l = rk % P.m;
                    const int q = i * P.m + j / P.e;
                    if (a.skip_local && q / P.V == P.rank0 / P.V) {
                        r.dst = nullptr;              // stored here by the expert's GEMM 2
                        return r;
                    }
                    const int64_t row = (((int64_t)(q % P.V) * P.m + l) * P.e + j % P.e) * a.C2 + s2;
                    r.src = P.bases[q / P.V] + P.off_Y + row * a.rowbytes;
                } else {
                    r.src = static_cast<const char *>(a.ret2) + (((int64_t)v * a.K2 + j) * a.C2 + s2) * a.rowbytes;
                }
            }
        }
    } else {
        const Combine1Args &a = m.c1;
        const int64_t rb = m.rowbytes;
        const int v = (int)(g / a.T);
        const int i = a.route.dest1[g];
        const int s1 = a.route.slot1[g];
        r.dst = static_cast<char *>(a.out) + g * rb;
        if (s1 < a.C1) {
            if (a.peer.bases) {
                const PeerMap &P = a.peer;
                const int rk = P.rank0 + v;
                if (P.n > 0) {   // bi-level: peer load from the intermediate (i, l), chunk s
                    const int s_ = rk / P.m, l = rk % P.m, u = i * P.m + l;
                    if (a.skip_direct) {
                        const int q = i * P.m + a.route.dest2[g] / P.e, me = P.rank0 / P.V;
                        if (u / P.V == me && q / P.V == me) {     // written by the expert's GEMM 2
                            r.dst = nullptr;
                            return r;
                        }
                    }
                    r.src = P.bases[u / P.V] + P.off_ret1 + (((int64_t)(u % P.V) * P.n + s_) * a.C1 + s1) * rb;
                } else {         // flat: peer load of Y from the expert rank E / e
                    const int q = i / P.e;
                    if (a.skip_direct && q / P.V == P.rank0 / P.V) {   // written by the expert's GEMM 2
                        r.dst = nullptr;
                        return r;
                    }
                    r.src = P.bases[q / P.V] + P.off_Y + ((((int64_t)(q % P.V) * P.G + rk) * P.e + i % P.e) * a.C1 + s1) * rb;
                }
            } else {
                r.src = static_cast<const char *>(a.back1) + (((int64_t)v * a.K1 + i) * a.C1 + s1) * rb;
            }
            r.scale = a.nogate ? 1.f : a.route.gate[g];
        } else {
            r.scale = 0.f;
        }
    }
    return r;
}

constexpr int kMoveThreads = 256;
constexpr int kMoveRowsPerWarp = 4;     // rows whose metadata 4 lanes resolve in parallel
constexpr int kMoveColUnroll = 3;       // 16-byte vectors per lane per row in flight

// One warp moves kMoveRowsPerWarp rows at a time: lanes 0..3 resolve one row each
// (independent dependent-load chains), the pointers are broadcast, then every lane keeps
// rows x kMoveColUnroll 16-byte loads in flight before its stores.
template <int RW>
__device__ __forceinline__ void row_move_body(const MoveArgs &m) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int nvec = (int)(m.rowbytes / 16);
    const bool combine1 = m.kind == MOVE_COMBINE1;
    const bool bf16 = m.c1.bf16 != 0;
    constexpr int CU = kMoveColUnroll;
    // The next batch's row plan (dependent metadata loads: slot offsets, routes) is
    // resolved while the current batch's row loads are in flight.
    RowPlan mine{nullptr, nullptr, 1.f};
    if (lane < RW && gw * RW + lane < m.rows) mine = plan_row(m, gw * RW + lane);
    for (int64_t g0 = gw * RW; g0 < m.rows; g0 += warps * RW) {
        const char *src[RW];
        char *dst[RW];
        float sc[RW];
#pragma unroll
        for (int r = 0; r < RW; ++r) {
            src[r] = reinterpret_cast<const char *>(__shfl_sync(kFull, reinterpret_cast<unsigned long long>(mine.src), r));
            dst[r] = reinterpret_cast<char *>(__shfl_sync(kFull, reinterpret_cast<unsigned long long>(mine.dst), r));
            sc[r] = __shfl_sync(kFull, mine.scale, r);
        }
        const int64_t gn = g0 + warps * RW;
        bool planned = false;
        for (int c0 = lane; c0 < nvec; c0 += 32 * CU) {
            int4 val[RW][CU];
#pragma unroll
            for (int r = 0; r < RW; ++r)
#pragma unroll
                for (int u = 0; u < CU; ++u) {
                    const int c = c0 + 32 * u;
                    val[r][u] = (dst[r] && src[r] && c < nvec) ? __ldg(reinterpret_cast<const int4 *>(src[r]) + c)
                                                               : make_int4(0, 0, 0, 0);
                }
            if (!planned) {
                RowPlan nxt{nullptr, nullptr, 1.f};
                if (lane < RW && gn + lane < m.rows) nxt = plan_row(m, gn + lane);
                mine = nxt;
                planned = true;
            }
#pragma unroll
            for (int r = 0; r < RW; ++r) {
                if (!dst[r]) continue;
#pragma unroll
                for (int u = 0; u < CU; ++u) {
                    const int c = c0 + 32 * u;
                    if (c >= nvec) continue;
                    int4 w = val[r][u];
                    if (combine1 && sc[r] != 1.f) {
                        if (bf16) {
                            __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&w);
#pragma unroll
                            for (int z = 0; z < 4; ++z) {
                                const float2 f = __bfloat1622float2(h[z]);
                                h[z] = __floats2bfloat162_rn(__fmul_rn(sc[r], f.x), __fmul_rn(sc[r], f.y));
                            }
                        } else {
                            float *f = reinterpret_cast<float *>(&w);
#pragma unroll
                            for (int z = 0; z < 4; ++z) f[z] = __fmul_rn(sc[r], f[z]);
                        }
                    }
                    reinterpret_cast<int4 *>(dst[r])[c] = w;
                }
            }
        }
        if (!planned) {                        // rows narrower than this lane's first vector
            RowPlan nxt{nullptr, nullptr, 1.f};
            if (lane < RW && gn + lane < m.rows) nxt = plan_row(m, gn + lane);
            mine = nxt;
        }
    }
    pdl_trigger();
}

template <int RW>
__global__ void __launch_bounds__(kMoveThreads) row_move_kernel(MoveArgs m) { row_move_body<RW>(m); }

// the same with the register budget fitted to MINB resident blocks per SM (SMILE_MOVE_MINB)
template <int RW, int MINB>
__global__ void __launch_bounds__(kMoveThreads, MINB) row_move_kernel_mb(MoveArgs m) { row_move_body<RW>(m); }

// a13 for the FLAT top-k layer (Eq. 2): warp per token, out[t] = dtype(sum over
// the token's kept choices j (ascending) of gate_j * row_j), fp32 accumulation; the rows
// come from back1 [V, K1, C1, d] or, with the peer-store exchange, straight from the
// expert's Y.  A token whose every choice was dropped gets a zero row (R9).
__global__ void __launch_bounds__(256) combine_topk_kernel(Combine1Args a) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t VT = (int64_t)a.V * a.T;
    const int64_t rb = (int64_t)a.d * (a.bf16 ? 2 : 4);
    const int nvec = (int)(rb / 16);
    for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g < VT; g += warps) {
        const int v = (int)(g / a.T);
        const char *src[4];
        float w[4];
        int nsrc = 0;
        for (int j = 0; j < a.topk; ++j) {
            const int64_t gi = (int64_t)j * VT + g;
            const int i = a.route.dest1[gi];
            const int s1 = a.route.slot1[gi];
            if (s1 >= a.C1) continue;
            const char *p;
            if (a.peer.bases) {
                const PeerMap &P = a.peer;
                const int rk = P.rank0 + v, q = i / P.e;
                p = P.bases[q / P.V] + P.off_Y + ((((int64_t)(q % P.V) * P.G + rk) * P.e + i % P.e) * a.C1 + s1) * rb;
            } else {
                p = static_cast<const char *>(a.back1) + (((int64_t)v * a.K1 + i) * a.C1 + s1) * rb;
            }
            src[nsrc] = p;
            w[nsrc] = a.nogate ? 1.f : a.route.gate[gi];       // a18 (dX return): rows already carry the gate
            ++nsrc;
        }
        int4 *dst = reinterpret_cast<int4 *>(static_cast<char *>(a.out) + g * rb);
        for (int c = lane; c < nvec; c += 32) {
            float acc[8];
#pragma unroll
            for (int z = 0; z < 8; ++z) acc[z] = 0.f;
            int4 uu[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)                      // every choice's 16 B in flight together
                if (k < nsrc) uu[k] = __ldg(reinterpret_cast<const int4 *>(src[k]) + c);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (k >= nsrc) break;
                const int4 u = uu[k];
                if (a.bf16) {
                    const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
                    for (int z = 0; z < 4; ++z) {
                        const float2 f = __bfloat1622float2(h[z]);
                        acc[2 * z] = fmaf(w[k], f.x, acc[2 * z]);
                        acc[2 * z + 1] = fmaf(w[k], f.y, acc[2 * z + 1]);
                    }
                } else {
                    const float *f = reinterpret_cast<const float *>(&u);
#pragma unroll
                    for (int z = 0; z < 4; ++z) acc[z] = fmaf(w[k], f[z], acc[z]);
                }
            }
            int4 o;
            if (a.bf16) {
                __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
                for (int z = 0; z < 4; ++z) h[z] = __floats2bfloat162_rn(acc[2 * z], acc[2 * z + 1]);
            } else {
                float *f = reinterpret_cast<float *>(&o);
#pragma unroll
                for (int z = 0; z < 4; ++z) f[z] = acc[z];
            }
            dst[c] = o;
        }
    }
}

// dispatch1 also fills meta = -1 for the empty slots [count, C1) of every destination.
__global__ void meta_fill_kernel(Dispatch1Args a) {
    pdl_wait();
    if (!a.meta && !a.peer.bases) return;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    const int64_t tot = (int64_t)a.V * a.K1 * a.C1;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < tot; idx += nthr) {
        const int64_t vi = idx / a.C1, cc = idx - vi * a.C1;   // vi = v*K1 + i
        const int64_t v = vi / a.K1, i = vi - v * a.K1;
        const int64_t last = ((v * a.topk + a.topk - 1) * a.nblk + a.nblk - 1) * a.K1 + i;   // total = off + hist of the last block
        if (cc >= (int64_t)a.blk_off1[last] + a.blk_hist1[last]) {
            if (a.peer.bases) {
                const PeerMap &P = a.peer;
                const int rk = P.rank0 + (int)v, s_ = rk / P.m, l = rk % P.m, q = (int)i * P.m + l;
                reinterpret_cast<int32_t *>(P.bases[q / P.V] + P.off_rmeta1)[((int64_t)(q % P.V) * P.n + s_) * a.C1 + cc] = -1;
            } else {
                a.meta[idx] = -1;
            }
        }
    }
}

// a14: Eq. (4) per resident rank in fp64.
__global__ void aux_kernel(smile_stats s, double alpha, double beta, double *loss, int V, int K1,
                           int K2, int64_t T, int flat) {
    pdl_wait();
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= V) return;
    const double Td = (double)T;
    double l1 = 0.0, l2 = 0.0;
    for (int k = 0; k < K1; ++k) l1 += ((double)s.hist1[v * K1 + k] / Td) * (s.psum1[v * K1 + k] / Td);
    for (int k = 0; k < K2; ++k) l2 += ((double)s.hist2[v * K2 + k] / Td) * (s.psum2[v * K2 + k] / Td);
    loss[v] = alpha * (double)K1 * l1 + (flat ? 0.0 : beta * (double)K2 * l2);
}

// Device-copy exchange for pairs of ranks resident on this device (the All2All of a
// level when several ranks share a GPU).  grid (V*P*nsub, row chunks).
constexpr int kCopyRows = 32;
__global__ void exchange_copy_kernel(CopyXArgs a) {
    pdl_wait();
    const int pair = blockIdx.x / a.nsub, k = blockIdx.x % a.nsub;
    const int v = pair / a.P, p = pair % a.P;
    const int q = a.member_local[v * a.P + p];
    if (q < 0) return;
    if (a.fabric && (a.rank0 + v) / a.m != (a.rank0 + q) / a.m) return;   // carried by the emulated NIC
    const int pos = a.mypos[v];
    const int64_t src_chunk = ((int64_t)v * a.P + p) * a.nsub + k;
    const int64_t dst_chunk = ((int64_t)q * a.P + pos) * a.nsub + k;
    int64_t rows = a.Csub;
    if (a.cnt) {
        rows = a.rev ? a.cnt[((int64_t)q * a.P + pos) * a.nsub + k] : a.cnt[src_chunk];
        rows = imin64((rows > 0 ? rows : (int64_t)0), a.Csub);
    }
    const int64_t r0 = (int64_t)blockIdx.y * kCopyRows;
    const int nvec = (int)(a.rowbytes / 16);
    if (r0 < rows) {
        const int64_t nr = imin64(kCopyRows, rows - r0);
        const int4 *src = reinterpret_cast<const int4 *>(a.send + (src_chunk * a.Csub + r0) * a.rowbytes);
        int4 *dst = reinterpret_cast<int4 *>(a.recv + (dst_chunk * a.Csub + r0) * a.rowbytes);
        const int64_t nv = nr * nvec;
        int64_t i = threadIdx.x;
        for (; i + 3 * blockDim.x < nv; i += 4 * blockDim.x) {
            int4 x0 = __ldg(src + i), x1 = __ldg(src + i + blockDim.x), x2 = __ldg(src + i + 2 * blockDim.x),
                 x3 = __ldg(src + i + 3 * blockDim.x);
            dst[i] = x0; dst[i + blockDim.x] = x1; dst[i + 2 * blockDim.x] = x2; dst[i + 3 * blockDim.x] = x3;
        }
        for (; i < nv; i += blockDim.x) dst[i] = __ldg(src + i);
    }
    if (!a.rev && a.sint && blockIdx.y == 0 && k == 0) {
        for (int i = threadIdx.x; i < a.ipp; i += blockDim.x)
            a.rint[((int64_t)q * a.P + pos) * a.ipp + i] = a.sint[((int64_t)v * a.P + p) * a.ipp + i];
    }
}

// Emulated heterogeneous fabric (smile_set_fabric): the NIC of sending
// rank v = the kFabricCtas CTAs (b, v).  It sends v's cross-node messages (one per group
// member on another node: all of the pair's sub-chunks and side ints) one after another:
// message k occupies the window [W_k, W_k + latency + bytes_k * ns_per_byte) of wall time
// (%globaltimer), W_0 = the CTA's start, W_{k+1} = the end of window k; each CTA copies its
// share of the message's rows as soon as the window opens and then waits for the window's
// end (a share that takes longer than the window delays the next one: the emulation is then
// bounded by the copy rate of kFabricCtas SMs).
constexpr int kFabricCtas = 16;
__global__ void fabric_copy_kernel(CopyXArgs a) {
    __shared__ unsigned long long s_w;
    pdl_wait();
    const int v = blockIdx.y, b = blockIdx.x, NB = gridDim.x;
    const int pos = a.mypos[v];
    const int nvec = (int)(a.rowbytes / 16);
    if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        s_w = t;
    }
    __syncthreads();
    unsigned long long w = s_w;
    for (int p = 0; p < a.P; ++p) {
        const int q = a.member_local[v * a.P + p];
        if (q < 0 || (a.rank0 + v) / a.m == (a.rank0 + q) / a.m) continue;
        int64_t bytes = 0;
        for (int k = 0; k < a.nsub; ++k) {
            const int64_t src_chunk = ((int64_t)v * a.P + p) * a.nsub + k;
            const int64_t dst_chunk = ((int64_t)q * a.P + pos) * a.nsub + k;
            int64_t rows = a.Csub;
            if (a.cnt) {
                rows = a.rev ? a.cnt[((int64_t)q * a.P + pos) * a.nsub + k] : a.cnt[src_chunk];
                rows = imin64((rows > 0 ? rows : (int64_t)0), a.Csub);
            }
            bytes += rows * a.rowbytes;
            const int64_t r0 = rows * b / NB, r1 = rows * (b + 1) / NB;     // this CTA's share
            const int4 *src = reinterpret_cast<const int4 *>(a.send + (src_chunk * a.Csub + r0) * a.rowbytes);
            int4 *dst = reinterpret_cast<int4 *>(a.recv + (dst_chunk * a.Csub + r0) * a.rowbytes);
            const int64_t nv = (r1 - r0) * nvec;
            int64_t i = threadIdx.x;
            for (; i + 3 * blockDim.x < nv; i += 4 * blockDim.x) {
                int4 x0 = __ldg(src + i), x1 = __ldg(src + i + blockDim.x), x2 = __ldg(src + i + 2 * blockDim.x),
                     x3 = __ldg(src + i + 3 * blockDim.x);
                dst[i] = x0; dst[i + blockDim.x] = x1; dst[i + 2 * blockDim.x] = x2; dst[i + 3 * blockDim.x] = x3;
            }
            for (; i < nv; i += blockDim.x) dst[i] = __ldg(src + i);
        }
        if (!a.rev && a.sint) {
            bytes += (int64_t)a.ipp * 4;
            if (b == 0)
                for (int i = threadIdx.x; i < a.ipp; i += blockDim.x)
                    a.rint[((int64_t)q * a.P + pos) * a.ipp + i] = a.sint[((int64_t)v * a.P + p) * a.ipp + i];
        }
        w += (unsigned long long)(a.latency_ns + (double)bytes * a.ns_per_byte);   // end of this message's window
        __syncthreads();
        if (threadIdx.x == 0) {
            for (;;) {
                unsigned long long t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                if (t >= w) break;
            }
        }
        __syncthreads();
    }
}

// Process-level barrier over NVLink (peer-store exchange): advance this level's epoch
// counter (device memory: every launch, graph replays included, gets the next epoch),
// after a fence write it into flag[level][me] of every peer process's workspace, then
// wait until every peer has written at least that epoch into ours.  One thread.  A wait
// longer than timeout_ns (0 = forever) sets the sticky SMILE_ETIMEOUT flag and returns.
__global__ void peer_barrier_kernel(char *const *bases, int64_t off_flags, int me, const int32_t *peers, int npeers,
                                    int level, long long *epoch_ctr, unsigned long long timeout_ns, int *err) {
    pdl_wait();
    if (threadIdx.x != 0) return;
    const long long epoch = *epoch_ctr + 1;
    *epoch_ctr = epoch;
    __threadfence_system();
    for (int i = 0; i < npeers; ++i) {
        long long *f = reinterpret_cast<long long *>(bases[peers[i]] + off_flags) + level * kMaxProcs + me;
        asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(f), "l"(epoch) : "memory");
    }
    const long long *mine = reinterpret_cast<const long long *>(bases[me] + off_flags) + level * kMaxProcs;
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < npeers; ++i) {
        long long v = 0;
        for (;;) {
            asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(mine + peers[i]) : "memory");
            if (v >= epoch) break;
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (timeout_ns && t - t0 > timeout_ns) {     // the peer never came: report, never hang
                set_err(err, SMILE_ETIMEOUT);
                __threadfence_system();
                return;
            }
        }
    }
    __threadfence_system();
}

inline int grid_for(int64_t warps_needed, int per_block_warps, int cap) {
    int64_t b = (warps_needed + per_block_warps - 1) / per_block_warps;
    if (b < 1) b = 1;
    return (int)(b < cap ? b : cap);
}

}  // namespace

void launch_gate1(const GateArgs &a, cudaStream_t st) {
    if (a.T == 0) return;
    size_t smem = (size_t)a.TB * gate_lds(a.KW) * 4 + (size_t)a.TB * 4 + (size_t)(((a.TB / 32) * a.K1 + 3) & ~3) * 4 +
                  (size_t)((a.K1 + 3) & ~3) * 4 + ((gate_scratch_bytes(a.TB, a.KW, a.K2) + 15) & ~(size_t)15);
    if (!a.logits && (size_t)a.KW * a.d * 4 <= (size_t)kRouterSmem) smem += (size_t)a.KW * a.d * 4;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(gate1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        attr_set = true;
    }
    note_launch();
    launch_k(gate1_kernel, dim3(a.nblk, a.V), dim3(a.TB), smem, st, a);
}

void launch_scan1(const Scan1Args &a, cudaStream_t st) {
    if (a.T == 0) return;
    const int jobs = a.K1 + (a.K1 + a.K2) + a.K2;             // scan1_rank's jobs per rank
    int nb = (jobs + 15) / 16;                               // 16 warps per block
    if (nb > 16) nb = 16;
    note_launch();
    launch_k(scan1_kernel, dim3(a.V * nb), dim3(512), 0, st, a);
}

void launch_rank2(const Rank2Args &a, cudaStream_t st) {
    if (a.items == 0) return;
    note_launch();
    launch_k(rank2_kernel, dim3(a.nblk, a.V), dim3(kRank2Items), 0, st, a);
    int nb = (a.K2 + 15) / 16;                               // 16 warps per block
    if (nb > 16) nb = 16;
    note_launch();
    launch_k(scan2_kernel, dim3(a.V * nb), dim3(512), 0, st, a);
}

// Rows per warp batch: SMILE_MOVE_RW = 4 (default) or 8.
static int move_rw() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("SMILE_MOVE_RW");
        v = (e && e[0] == '8') ? 8 : kMoveRowsPerWarp;
    }
    return v;
}

// Grid cap of the movers in blocks per SM: SMILE_MOVE_GRIDMUL (default 8).
// resident 256-thread blocks per SM the register budget is fitted to (SMILE_MOVE_MINB: 1 = the
// unconstrained 118-register kernel, 2 blocks per SM; 3 = 80 registers, 216 B spilled)
static int move_minb() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("SMILE_MOVE_MINB");
        v = e ? atoi(e) : 1;
        if (v != 3) v = 1;
    }
    return v;
}

static int move_gridmul() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("SMILE_MOVE_GRIDMUL");
        v = e ? atoi(e) : 8;
        if (v < 1) v = 8;
    }
    return v;
}

static void launch_move(MoveArgs &m, cudaStream_t st) {
    if (m.rows <= 0) return;
    const int rw = move_rw();
    const int64_t per_block = (int64_t)(kMoveThreads / 32) * rw;
    int64_t grid = (m.rows + per_block - 1) / per_block;
    if (grid > 148 * move_gridmul()) grid = 148 * move_gridmul();
    note_launch();
    const int minb = move_minb();
    if (rw == 8) launch_k(row_move_kernel<8>, dim3((unsigned)grid), dim3(kMoveThreads), 0, st, m);
    else if (minb == 3) launch_k(row_move_kernel_mb<kMoveRowsPerWarp, 3>, dim3((unsigned)grid), dim3(kMoveThreads), 0, st, m);
    else launch_k(row_move_kernel<kMoveRowsPerWarp>, dim3((unsigned)grid), dim3(kMoveThreads), 0, st, m);
}

void launch_dispatch1(const Dispatch1Args &a, cudaStream_t st) {
    if (a.T == 0) return;
    MoveArgs m{};
    m.kind = MOVE_DISPATCH1; m.rows = (int64_t)a.topk * a.V * a.T; m.rowbytes = a.rowbytes; m.d1 = a;
    launch_move(m, st);
    if (a.meta || a.peer.bases && a.peer.n > 0) {
        note_launch();
        launch_k(meta_fill_kernel, dim3(148 * 4), dim3(256), 0, st, a);
    }
}

void launch_meta_fill(const Dispatch1Args &a, cudaStream_t st) {
    if (a.T == 0) return;
    if (a.meta || a.peer.bases && a.peer.n > 0) {
        note_launch();
        launch_k(meta_fill_kernel, dim3(148 * 4), dim3(256), 0, st, a);
    }
}

void launch_dispatch2(const Dispatch2Args &a, cudaStream_t st) {
    if (a.items == 0) return;
    MoveArgs m{};
    m.kind = MOVE_DISPATCH2; m.rows = (int64_t)a.V * a.items; m.rowbytes = a.rowbytes; m.d2 = a;
    launch_move(m, st);
}

void launch_grad_dispatch2(const Dispatch2Args &a, cudaStream_t st) {
    if (a.items == 0) return;
    MoveArgs m{};
    m.kind = MOVE_GRAD2; m.rows = (int64_t)a.V * a.items; m.rowbytes = a.rowbytes; m.d2 = a;
    launch_move(m, st);
}

void launch_combine2(const Combine2Args &a, cudaStream_t st) {
    if (a.items == 0) return;
    MoveArgs m{};
    m.kind = MOVE_COMBINE2; m.rows = (int64_t)a.V * a.items; m.rowbytes = a.rowbytes; m.c2 = a;
    launch_move(m, st);
}

void launch_combine1(const Combine1Args &a, cudaStream_t st) {
    if (a.T == 0) return;
    if (a.topk > 1) {
        const int64_t warps = (int64_t)a.V * a.T;
        int64_t grid = (warps + 7) / 8;
        if (grid > 148 * 8) grid = 148 * 8;
        note_launch();
        launch_k(combine_topk_kernel, dim3((unsigned)grid), dim3(256), 0, st, a);
        return;
    }
    MoveArgs m{};
    m.kind = MOVE_COMBINE1; m.rows = (int64_t)a.V * a.T; m.rowbytes = (int64_t)a.d * (a.bf16 ? 2 : 4); m.c1 = a;
    launch_move(m, st);
}

void launch_aux(const smile_stats &s, double alpha, double beta, double *loss, int V, int K1, int K2,
                int64_t T, int flat, cudaStream_t st) {
    note_launch();
    launch_k(aux_kernel, dim3((V + 127) / 128), dim3(128), 0, st, s, alpha, beta, loss, V, K1, K2, T, flat);
}

void launch_peer_barrier(char *const *bases, int64_t off_flags, int me, const int32_t *peers, int npeers, int level,
                         long long *epoch, unsigned long long timeout_ns, int *err, cudaStream_t st) {
    if (npeers <= 0) return;
    note_launch();
    launch_k(peer_barrier_kernel, dim3(1), dim3(32), 0, st, bases, off_flags, me, peers, npeers, level, epoch, timeout_ns,
             err);
}

void launch_fabric_copy(const CopyXArgs &a, cudaStream_t st) {
    note_launch();
    launch_k(fabric_copy_kernel, dim3(kFabricCtas, a.V), dim3(256), 0, st, a);
}

void launch_exchange_copy(const CopyXArgs &a, cudaStream_t st) {
    const int64_t chunks = (a.Csub + kCopyRows - 1) / kCopyRows;
    dim3 grid((unsigned)(a.V * a.P * a.nsub), (unsigned)(chunks > 0 ? chunks : 1));
    note_launch();
    launch_k(exchange_copy_kernel, grid, dim3(256), 0, st, a);
}

}  // namespace smile
