// gate_common.cuh -- the per-tile part of the level-1 gate shared
// by the SIMT gate (route_kernels.cu: gate1_kernel, one thread block per tile) and the
// tensor-core gate (gate_tcgen05.cu: the tile's 4 epilogue warps).  Given one tile's fp32
// logits in shared memory it takes the routing decisions, the in-tile capacity ranks and
// the LB-statistic partials of the tile.  `Sync` names the threads that cooperate on a
// tile: the whole block, or a named barrier over the epilogue warps.
#pragma once
#include "smile_internal.h"

#include <math.h>

namespace smile {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void set_err(int *err, int code) {
    if (err) atomicCAS(err, 0, code);
}

struct BlockSync {
    static __device__ __forceinline__ void sync() { __syncthreads(); }
    static __device__ __forceinline__ int tid() { return threadIdx.x; }
    static __device__ __forceinline__ int nthr() { return blockDim.x; }
};

// Epilogue group G (4 warps, threads 128 + 128 G .. 255 + 128 G) of the tensor-core
// gate, on named barrier 1 + G.
template <int G>
struct EpiSync {
    static __device__ __forceinline__ void sync() { asm volatile("bar.sync %0, 128;" ::"n"(1 + G) : "memory"); }
    static __device__ __forceinline__ int tid() { return threadIdx.x - 128 - 128 * G; }
    static __device__ __forceinline__ int nthr() { return 128; }
};

// Rank of this thread's item among the tile's earlier items with the same bucket
// (bucket < 0: no item).  s_wh: [NW][K] ints, s_bh: [K] ints.  Writes the tile
// histogram to s_bh and returns the tile-local rank (or -1).  Items are ordered by
// thread index, i.e. warp-major then lane, matching item order.
template <class Sync>
__device__ int block_rank(int b, int K, int *s_wh, int *s_bh) {
    const int tid = Sync::tid(), nthr = Sync::nthr();
    const int lane = tid & 31, w = tid >> 5, NW = nthr >> 5;
    for (int i = tid; i < NW * K; i += nthr) s_wh[i] = 0;
    Sync::sync();
    const unsigned peers = __match_any_sync(kFull, b);
    const int lr = __popc(peers & ((1u << lane) - 1u));
    if (b >= 0 && lane == __ffs(peers) - 1) s_wh[w * K + b] = __popc(peers);
    Sync::sync();
    for (int k = tid; k < K; k += nthr) {
        int acc = 0;
        for (int ww = 0; ww < NW; ++ww) {
            const int c = s_wh[ww * K + k];
            s_wh[ww * K + k] = acc;
            acc += c;
        }
        s_bh[k] = acc;
    }
    Sync::sync();
    return b >= 0 ? s_wh[w * K + b] + lr : -1;
}

// Odd row stride for a [tokens][KW] fp32 tile that threads (tokens) walk in lockstep:
// conflict-free shared-memory banks for any KW (KW = 64 would otherwise be 32-way).
__host__ __device__ __forceinline__ int gate_lds(int KW) { return KW | 1; }

// Phases B and C of the level-1 gate over one tile of nt <= Sync::nthr() tokens whose
// logits are s_lg [nt][lds] (entries 0..K1-1: inter router W_p; K1..KW-1: intra W_q).
// tok0: global index of the tile's first token; bo = v * nblk + blk: the tile's index in
// the per-tile tables (with top-k, choice j of the tile is table row (v * topk + j) * nblk
// + blk).  Must be entered by all Sync threads after the logits are visible to them.
// Thread-per-token row passes of phase B over one token's logits in smem, four entries per
// step with their loads issued together (the per-entry load -> use chains of a plain loop
// bound the epilogue of the wide routers).  Same results, bit for bit, as the plain loops:
// the arg max is the FIRST index of the strict maximum (R2, R28: '>' over ascending k, a
// running max in a register), the sum is accumulated in ascending k.
__device__ __forceinline__ void row_argmax(const float *L, int K, int &arg, float &mx, bool &finite) {
    float m = L[0];
    int b = 0;
    finite &= isfinite(m);
    int k = 1;
    for (; k + 3 < K; k += 4) {
        const float x0 = L[k], x1 = L[k + 1], x2 = L[k + 2], x3 = L[k + 3];
        finite &= isfinite(x0) & isfinite(x1) & isfinite(x2) & isfinite(x3);
        if (x0 > m) { m = x0; b = k; }
        if (x1 > m) { m = x1; b = k + 1; }
        if (x2 > m) { m = x2; b = k + 2; }
        if (x3 > m) { m = x3; b = k + 3; }
    }
    for (; k < K; ++k) {
        const float x = L[k];
        finite &= isfinite(x);
        if (x > m) { m = x; b = k; }
    }
    arg = b;
    mx = m;
}
// e_k = expf(L_k - mx) written over L_k; returns sum_k e_k (ascending k)
__device__ __forceinline__ float row_exp_sum(float *L, int K, float mx) {
    float s = 0.f;
    int k = 0;
    for (; k + 3 < K; k += 4) {
        const float e0 = expf(L[k] - mx), e1 = expf(L[k + 1] - mx), e2 = expf(L[k + 2] - mx), e3 = expf(L[k + 3] - mx);
        L[k] = e0; L[k + 1] = e1; L[k + 2] = e2; L[k + 3] = e3;
        s += e0; s += e1; s += e2; s += e3;
    }
    for (; k < K; ++k) {
        const float e = expf(L[k] - mx);
        L[k] = e;
        s += e;
    }
    return s;
}
struct GateTok {
    int i;       // level-1 destination of this thread's token (-1: no token)
    int lr;      // its rank among the tile's tokens with the same destination
};

// Scratch of gate_finish's statistics (shared memory, per tile in flight): s_part [ceil(TB / 32)
// x KW] fp64 chunk partials, s_h2 [K2] int counts, s_sc [2][TB] fp32 per-token p and q.
__host__ __device__ __forceinline__ size_t gate_scratch_bytes(int TB, int KW, int K2) {
    return (size_t)((TB + 31) / 32) * KW * 8 + (size_t)((K2 + 1) & ~1) * 4 + (size_t)2 * TB * 4;
}

template <class Sync>
__device__ GateTok gate_finish(const GateArgs &a, float *s_lg, int lds, int *s_j, int *s_wh, int *s_bh, double *s_part,
                               int64_t tok0, int nt, int64_t bo, unsigned long long *trace = nullptr, int tslot = 0) {
    const int tid = Sync::tid(), nthr = Sync::nthr();
    const bool tr = trace && tid == 0;           // SMILE_TRACE=gate: stamps of the epilogue's phases
    const int KW = a.KW, K1 = a.K1, K2 = a.K2;
    const int topk = a.topk > 1 ? a.topk : 1;
    const int64_t VT = (int64_t)a.V * a.T;
    // Phase B: one thread per token -- argmax (R2, R3), top-1 probabilities (R4), and
    // the softmax entries for the LB statistics, written back over the logits.  Top-k
    // (FLAT, R29): the further choices by repeated first-argmax over the logits not chosen
    // yet, taken before the logits are transformed.
    int *s_h2 = reinterpret_cast<int *>(s_part + (size_t)((nthr + 31) >> 5) * KW);
    float *s_p = reinterpret_cast<float *>(s_h2 + ((K2 + 1) & ~1)), *s_q = s_p + nthr;
    for (int k = tid; k < K2; k += nthr) s_h2[k] = 0;      // (block_rank's barriers order it)
    int i = -1, j = 0;
    int ch[4] = {-1, -1, -1, -1};
    if (tid < nt) {
        float *L = s_lg + tid * lds;
        bool finite = true;
        // level 1: argmax, then (top-k) the further choices before the logits are transformed
        float mi;
        row_argmax(L, K1, i, mi, finite);
        ch[0] = i;
        for (int c = 1; c < topk; ++c) {
            int best = -1;
            for (int k = 0; k < K1; ++k) {
                bool taken = false;
                for (int cc = 0; cc < c; ++cc) taken |= ch[cc] == k;
                if (!taken && (best < 0 || L[k] > L[best])) best = k;
            }
            ch[c] = best;
        }
        // one expf per entry: e_k = exp(r_k - r_max) is kept, the softmax entry for the
        // statistics is e_k * (1 / sum) (within 1.5 ulp of e_k / sum; the LB loss
        // tolerance is 1e-6 relative), and the top-1 probability is 1 / sum exactly.
        // The rows keep e_k; the statistics pass scales them by p (level 1) or q (level 2)
        // as it reads them (the same fp32 products e_k * p, e_k * q).
        const float p = __frcp_rn(row_exp_sum(L, K1, mi));
        float q = 1.f;
        if (!a.flat) {
            float *L2 = L + K1;
            float mj;
            row_argmax(L2, K2, j, mj, finite);
            q = __frcp_rn(row_exp_sum(L2, K2, mj));
        }
        if (!finite) set_err(a.err, SMILE_ENONFINITE);
        s_p[tid] = p;
        s_q[tid] = q;
        const int64_t g = tok0 + tid;
        a.route.dest1[g] = i;
        a.route.dest2[g] = j;
        a.route.p[g] = p;
        a.route.q[g] = q;
        a.route.gate[g] = __fmul_rn(p, q);
        for (int c = 1; c < topk; ++c) {              // Eq. (2) weights p_e of the further choices (R30)
            a.route.dest1[c * VT + g] = ch[c];
            a.route.gate[c * VT + g] = L[ch[c]] * p;
        }
        if (i < 0 || i >= K1) set_err(a.err, SMILE_EINDEX);
    }
    s_j[tid] = (tid < nt) ? j : -1;
    if (tr) trace_clock(trace, tslot);

    // Phase C: tile-local capacity rank of dest1 (R5, R8) -- per choice with top-k, whose
    // tables are laid out choice-major per rank so the scan gives choice-major slots (R31).
    const int64_t v = bo / a.nblk, blk = bo - v * a.nblk;
    const int64_t bo0 = (v * topk) * a.nblk + blk;              // choice 0's table row
    const int lr = block_rank<Sync>(i, K1, s_wh, s_bh);
    if (tid < nt) a.route.slot1[tok0 + tid] = lr;
    for (int k = tid; k < K1; k += nthr) a.blk_hist1[bo0 * K1 + k] = s_bh[k];
    if (tr) trace_clock(trace, tslot + 1);
    for (int c = 1; c < topk; ++c) {
        Sync::sync();                                             // s_bh of the previous choice consumed
        const int lrc = block_rank<Sync>(tid < nt ? ch[c] : -1, K1, s_wh, s_bh);
        if (tid < nt) a.route.slot1[c * VT + tok0 + tid] = lrc;
        for (int k = tid; k < K1; k += nthr) a.blk_hist1[(bo0 + (int64_t)c * a.nblk) * K1 + k] = s_bh[k];
    }
    // LB statistics partials of the tile: fp64 sums of the probabilities (R13) and the
    // level-2 top-1 counts, in a fixed order that depends only on the tile's token count and
    // KW (deterministic, the same in every kernel that calls this).  Counts: warp-aggregated
    // shared-memory adds (exact).  Narrow routers (KW < 32): a warp per statistic, lanes
    // stride over the tokens, fixed butterfly.  Wide routers: per 32-token chunk c and
    // statistic k, four interleaved accumulators over the chunk's tokens in ascending order,
    // then the chunks in ascending order, the (chunk, 32-statistic block) items spread over
    // all warps (one warp per 32 statistics walking every token left most warps idle and
    // bounded the epilogue of C4 / C5).
    {
        const int lane = tid & 31, w = tid >> 5, NW = nthr >> 5;
        const int jj = (tid < nt) ? j : -1;
        const unsigned peers = __match_any_sync(kFull, jj);
        if (jj >= 0 && lane == __ffs(peers) - 1) atomicAdd(&s_h2[jj], __popc(peers));
        if (KW < 32) {
            for (int k = w; k < KW; k += NW) {
                const float *sc = k < K1 ? s_p : s_q;         // softmax entry = e_k * p or e_k * q
                double acc = 0.0;
                for (int tt = lane; tt < nt; tt += 32) acc += (double)(s_lg[tt * lds + k] * sc[tt]);
                for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
                if (lane == 0) a.blk_psum[bo0 * (K1 + K2) + k] = acc;
            }
            Sync::sync();
        } else {
            const int nch = (nt + 31) >> 5, ncb = (KW + 31) >> 5;
            for (int item = w; item < nch * ncb; item += NW) {
                const int c = item / ncb, k = (item - c * ncb) * 32 + lane;
                if (k < KW) {
                    const float *sc = k < K1 ? s_p : s_q;
                    const int t1 = min(nt, c * 32 + 32);
                    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
                    int tt = c * 32;
                    for (; tt + 3 < t1; tt += 4) {
                        a0 += (double)(s_lg[tt * lds + k] * sc[tt]);
                        a1 += (double)(s_lg[(tt + 1) * lds + k] * sc[tt + 1]);
                        a2 += (double)(s_lg[(tt + 2) * lds + k] * sc[tt + 2]);
                        a3 += (double)(s_lg[(tt + 3) * lds + k] * sc[tt + 3]);
                    }
                    for (; tt < t1; ++tt) a0 += (double)(s_lg[tt * lds + k] * sc[tt]);
                    s_part[c * KW + k] = (a0 + a1) + (a2 + a3);
                }
            }
            Sync::sync();
            for (int k = tid; k < KW; k += nthr) {
                double acc = 0.0;
                for (int c = 0; c < nch; ++c) acc += s_part[c * KW + k];
                a.blk_psum[bo0 * (K1 + K2) + k] = acc;
            }
        }
        for (int k = tid; k < K2; k += nthr) a.blk_hist2a[bo0 * K2 + k] = s_h2[k];
        if (a.flat && tid == 0) a.blk_psum[bo0 * (K1 + K2) + K1] = (double)nt;
    }
    if (tr) trace_clock(trace, tslot + 2);
    return GateTok{i, topk > 1 ? -1 : lr};
}

// Warp-cooperative scans / sums over n entries at stride st, in batches of 32 * kScanR
// entries: lane l owns the kScanR consecutive entries [b0 + l kScanR, +kScanR) of a batch
// and loads them all before combining (one memory round trip per batch instead of one per
// 32 entries -- these run at the tail of the gate kernel, latency-bound).  Fixed order
// (lane-serial, then the warp's shuffles): deterministic.
constexpr int kScanR = 16;
__device__ __forceinline__ int warp_exclusive_scan(const int32_t *p, int n, int64_t st, int32_t *out_excl) {
    const int lane = threadIdx.x & 31;
    int carry = 0;
    for (int b0 = 0; b0 < n; b0 += 32 * kScanR) {
        const int i0 = b0 + lane * kScanR;
        int v[kScanR];
#pragma unroll
        for (int r = 0; r < kScanR; ++r) v[r] = i0 + r < n ? __ldcg(p + (int64_t)(i0 + r) * st) : 0;
        int tot = 0;
#pragma unroll
        for (int r = 0; r < kScanR; ++r) { const int x = v[r]; v[r] = tot; tot += x; }   // lane-local exclusive
        int x = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += y;
        }
        const int base = carry + x - tot;                 // exclusive prefix of this lane's entries
#pragma unroll
        for (int r = 0; r < kScanR; ++r)
            if (i0 + r < n) out_excl[(int64_t)(i0 + r) * st] = base + v[r];
        carry += __shfl_sync(kFull, x, 31);
    }
    return carry;
}
__device__ __forceinline__ double warp_sum_f64(const double *p, int n, int64_t st) {
    const int lane = threadIdx.x & 31;
    double acc = 0.0;
    for (int b0 = 0; b0 < n; b0 += 32 * kScanR) {
        const int i0 = b0 + lane * kScanR;
        double v[kScanR];
#pragma unroll
        for (int r = 0; r < kScanR; ++r) v[r] = i0 + r < n ? __ldcg(p + (int64_t)(i0 + r) * st) : 0.0;
#pragma unroll
        for (int r = 0; r < kScanR; ++r) acc += v[r];
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    return acc;
}
__device__ __forceinline__ int warp_sum_i32(const int32_t *p, int n, int64_t st) {
    const int lane = threadIdx.x & 31;
    int acc = 0;
    for (int b0 = 0; b0 < n; b0 += 32 * kScanR) {
        const int i0 = b0 + lane * kScanR;
        int v[kScanR];
#pragma unroll
        for (int r = 0; r < kScanR; ++r) v[r] = i0 + r < n ? __ldcg(p + (int64_t)(i0 + r) * st) : 0;
#pragma unroll
        for (int r = 0; r < kScanR; ++r) acc += v[r];
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    return acc;
}

__device__ __forceinline__ void scan1_rank(const Scan1Args &a, int v, int w, int NW) {
    const int lane = threadIdx.x & 31;
    const int KS = a.K1 + a.K2;
    const int topk = a.topk > 1 ? a.topk : 1;
    const int64_t rb = (int64_t)v * topk * a.nblk;               // the rank's first table row
    const int jobs = a.K1 + KS + a.K2;
    for (int jb = w; jb < jobs; jb += NW) {
        if (jb < a.K1) {
            const int k = jb;
            const int64_t o = rb * a.K1 + k;
            // top-k: the rank's items in choice-major order (R31) -- offsets over every choice
            const int tot = warp_exclusive_scan(a.blk_hist1 + o, topk * a.nblk, a.K1, a.blk_off1 + o);
            // f counts choice 0 only (R13, R32)
            const int top1 = topk > 1 ? warp_sum_i32(a.blk_hist1 + o, a.nblk, a.K1) : tot;
            if (lane == 0) {
                const int32_t cnt = (int32_t)(tot < a.C1 ? tot : a.C1);
                a.stats.hist1[v * a.K1 + k] = top1;
                a.counts1[v * a.K1 + k] = cnt;
                if (a.peer.bases && a.flat) {      // counts travel with the rows: rcounts[q][src][k % e]
                    const PeerMap &P = a.peer;
                    const int rk = P.rank0 + v, q = k / P.e;
                    reinterpret_cast<int32_t *>(P.bases[q / P.V] + P.off_rcounts)[((int64_t)(q % P.V) * P.G + rk) * P.e + k % P.e] = cnt;
                }
            }
        } else if (jb < a.K1 + KS) {
            const int k = jb - a.K1;
            const double sum = warp_sum_f64(a.blk_psum + rb * KS + k, a.nblk, KS);
            if (lane == 0) {
                if (k < a.K1) a.stats.psum1[v * a.K1 + k] = sum;
                else a.stats.psum2[v * a.K2 + (k - a.K1)] = sum;
            }
        } else {
            const int k = jb - a.K1 - KS;
            const int c = warp_sum_i32(a.blk_hist2a + rb * a.K2 + k, a.nblk, a.K2);
            if (lane == 0) a.stats.hist2[v * a.K2 + k] = c;
        }
    }
}

}  // namespace smile
