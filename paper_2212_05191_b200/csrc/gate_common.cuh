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
struct GateTok {
    int i;       // level-1 destination of this thread's token (-1: no token)
    int lr;      // its rank among the tile's tokens with the same destination
};

template <class Sync>
__device__ GateTok gate_finish(const GateArgs &a, float *s_lg, int lds, int *s_j, int *s_wh, int *s_bh, int64_t tok0,
                               int nt, int64_t bo) {
    const int tid = Sync::tid(), nthr = Sync::nthr();
    const int KW = a.KW, K1 = a.K1, K2 = a.K2;
    const int topk = a.topk > 1 ? a.topk : 1;
    const int64_t VT = (int64_t)a.V * a.T;
    // Phase B: one thread per token -- argmax (R2, R3), top-1 probabilities (R4), and
    // the softmax entries for the LB statistics, written back over the logits.  Top-k
    // (FLAT, R29): the further choices by repeated first-argmax over the logits not chosen
    // yet, taken before the logits are transformed.
    int i = -1, j = 0;
    int ch[4] = {-1, -1, -1, -1};
    if (tid < nt) {
        float *L = s_lg + tid * lds;
        bool finite = true;
        for (int k = 0; k < KW; ++k) finite &= isfinite(L[k]);
        if (!finite) set_err(a.err, SMILE_ENONFINITE);
        i = 0;
        for (int k = 1; k < K1; ++k)
            if (L[k] > L[i]) i = k;
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
        const float mi = L[i];
        float s1 = 0.f;
        for (int k = 0; k < K1; ++k) {
            const float ek = expf(L[k] - mi);
            L[k] = ek;
            s1 += ek;
        }
        const float p = __frcp_rn(s1);
        float q = 1.f;
        if (!a.flat) {
            float *L2 = L + K1;
            j = 0;
            for (int k = 1; k < K2; ++k)
                if (L2[k] > L2[j]) j = k;
            const float mj = L2[j];
            float s2 = 0.f;
            for (int k = 0; k < K2; ++k) {
                const float ek = expf(L2[k] - mj);
                L2[k] = ek;
                s2 += ek;
            }
            q = __frcp_rn(s2);
            for (int k = 0; k < K2; ++k) L2[k] *= q;
        }
        for (int k = 0; k < K1; ++k) L[k] *= p;
        const int64_t g = tok0 + tid;
        a.route.dest1[g] = i;
        a.route.dest2[g] = j;
        a.route.p[g] = p;
        a.route.q[g] = q;
        a.route.gate[g] = __fmul_rn(p, q);
        for (int c = 1; c < topk; ++c) {              // Eq. (2) weights p_e of the further choices (R30)
            a.route.dest1[c * VT + g] = ch[c];
            a.route.gate[c * VT + g] = L[ch[c]];
        }
        if (i < 0 || i >= K1) set_err(a.err, SMILE_EINDEX);
    }
    s_j[tid] = (tid < nt) ? j : -1;

    // Phase C: tile-local capacity rank of dest1 (R5, R8) -- per choice with top-k, whose
    // tables are laid out choice-major per rank so the scan gives choice-major slots (R31).
    const int64_t v = bo / a.nblk, blk = bo - v * a.nblk;
    const int64_t bo0 = (v * topk) * a.nblk + blk;              // choice 0's table row
    const int lr = block_rank<Sync>(i, K1, s_wh, s_bh);
    if (tid < nt) a.route.slot1[tok0 + tid] = lr;
    for (int k = tid; k < K1; k += nthr) a.blk_hist1[bo0 * K1 + k] = s_bh[k];
    for (int c = 1; c < topk; ++c) {
        Sync::sync();                                             // s_bh of the previous choice consumed
        const int lrc = block_rank<Sync>(tid < nt ? ch[c] : -1, K1, s_wh, s_bh);
        if (tid < nt) a.route.slot1[c * VT + tok0 + tid] = lrc;
        for (int k = tid; k < K1; k += nthr) a.blk_hist1[(bo0 + (int64_t)c * a.nblk) * K1 + k] = s_bh[k];
    }
    // LB statistics partials of the tile (fp64 for the probability sums), deterministic
    // (fixed summation order).  Wide routers (KW >= 32): a warp per block of 32
    // statistics, lane = statistic, tokens in ascending order over 4 interleaved fp64
    // accumulators (conflict-free row reads; the per-statistic shuffle trees of the narrow
    // case cost C5's 66-wide gate most of its epilogue).  Narrow routers: one warp per
    // statistic, lanes stride over tokens, fixed butterfly.
    if (KW >= 32) {
        const int lane = tid & 31, w = tid >> 5, NW = nthr >> 5;
        for (int cb = w; cb < (KW + 31) / 32; cb += NW) {
            const int k = cb * 32 + lane;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            if (k < KW) {
                int tt = 0;
                for (; tt + 3 < nt; tt += 4) {
                    a0 += (double)s_lg[tt * lds + k];
                    a1 += (double)s_lg[(tt + 1) * lds + k];
                    a2 += (double)s_lg[(tt + 2) * lds + k];
                    a3 += (double)s_lg[(tt + 3) * lds + k];
                }
                for (; tt < nt; ++tt) a0 += (double)s_lg[tt * lds + k];
                a.blk_psum[bo0 * (K1 + K2) + k] = (a0 + a1) + (a2 + a3);
            }
        }
        for (int cb = w; cb < (K2 + 31) / 32; cb += NW) {
            const int k = cb * 32 + lane;
            int c = 0;
            for (int tt = 0; tt < nt; ++tt) c += (s_j[tt] == k);
            if (k < K2) a.blk_hist2a[bo0 * K2 + k] = c;
        }
        if (a.flat && tid == 0) a.blk_psum[bo0 * (K1 + K2) + K1] = (double)nt;
    } else {
        const int lane = tid & 31, w = tid >> 5, NW = nthr >> 5;
        for (int k = w; k < KW; k += NW) {
            double acc = 0.0;
            for (int tt = lane; tt < nt; tt += 32) acc += (double)s_lg[tt * lds + k];
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
            if (lane == 0) a.blk_psum[bo0 * (K1 + K2) + k] = acc;
        }
        for (int k = w; k < K2; k += NW) {
            int c = 0;
            for (int tt = lane; tt < nt; tt += 32) c += (s_j[tt] == k);
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
            if (lane == 0) a.blk_hist2a[bo0 * K2 + k] = c;
        }
        if (a.flat && tid == 0) a.blk_psum[bo0 * (K1 + K2) + K1] = (double)nt;
    }
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
