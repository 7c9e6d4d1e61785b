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
// tok0: global index of the tile's first token; bo: the tile's index in the per-tile
// tables.  Must be entered by all Sync threads after the logits are visible to them.
struct GateTok {
    int i;       // level-1 destination of this thread's token (-1: no token)
    int lr;      // its rank among the tile's tokens with the same destination
};

template <class Sync>
__device__ GateTok gate_finish(const GateArgs &a, float *s_lg, int lds, int *s_j, int *s_wh, int *s_bh, int64_t tok0,
                               int nt, int64_t bo) {
    const int tid = Sync::tid(), nthr = Sync::nthr();
    const int KW = a.KW, K1 = a.K1, K2 = a.K2;
    // Phase B: one thread per token -- argmax (R2, R3), top-1 probabilities (R4), and
    // the softmax entries for the LB statistics, written back over the logits.
    int i = -1, j = 0;
    if (tid < nt) {
        float *L = s_lg + tid * lds;
        bool finite = true;
        for (int k = 0; k < KW; ++k) finite &= isfinite(L[k]);
        if (!finite) set_err(a.err, SMILE_ENONFINITE);
        i = 0;
        for (int k = 1; k < K1; ++k)
            if (L[k] > L[i]) i = k;
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
        if (i < 0 || i >= K1) set_err(a.err, SMILE_EINDEX);
    }
    s_j[tid] = (tid < nt) ? j : -1;

    // Phase C: tile-local capacity rank of dest1 (R5, R8).
    const int lr = block_rank<Sync>(i, K1, s_wh, s_bh);
    if (tid < nt) a.route.slot1[tok0 + tid] = lr;
    for (int k = tid; k < K1; k += nthr) a.blk_hist1[bo * K1 + k] = s_bh[k];
    // LB statistics partials of the tile (fp64 for the probability sums): one warp per
    // statistic, lanes stride over tokens, fixed butterfly order => deterministic.
    {
        const int lane = tid & 31, w = tid >> 5, NW = nthr >> 5;
        for (int k = w; k < KW; k += NW) {
            double acc = 0.0;
            for (int tt = lane; tt < nt; tt += 32) acc += (double)s_lg[tt * lds + k];
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
            if (lane == 0) a.blk_psum[bo * (K1 + K2) + k] = acc;
        }
        for (int k = w; k < K2; k += NW) {
            int c = 0;
            for (int tt = lane; tt < nt; tt += 32) c += (s_j[tt] == k);
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
            if (lane == 0) a.blk_hist2a[bo * K2 + k] = c;
        }
        if (a.flat && tid == 0) a.blk_psum[bo * (K1 + K2) + K1] = (double)nt;
    }
    return GateTok{i, lr};
}

}  // namespace smile
