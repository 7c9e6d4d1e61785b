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

struct GateTok {
    int i;       // level-1 destination of this thread's token (-1: no token)
    int lr;      // its rank among the tile's tokens with the same destination
};

// fp64 sums of 32 values per lane over the warp's lanes, transposed: afterwards lane l holds
// the warp total of v[l] (the butterfly halves the vector each step; fixed order).
__device__ __forceinline__ double transpose_reduce32_f64(double (&v)[32], int lane) {
#pragma unroll
    for (int h = 16; h >= 1; h >>= 1) {
        const bool up = (lane & h) != 0;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const double send = up ? v[i] : v[i + h];
            const double keep = up ? v[i + h] : v[i];
            v[i] = keep + __shfl_xor_sync(kFull, send, h);
        }
    }
    return v[0];
}

// Per-chunk (32-token) tables of the level-1 capacity scan and the LB statistics.  A
// chunk is one warp's tokens; chunk indices run rank-major, ch = v * nch + t / 32, so the
// tables do not depend on how a kernel tiles the tokens (tiles are whole chunks of one
// rank).  Written for every chunk that holds tokens.
__device__ __forceinline__ void chunk_tables(const GateArgs &a, const float *s_lg, int lds, int i, int j, bool has,
                                             int64_t ch, int lane, int tok) {
    const int K1 = a.K1, K2 = a.K2, KW = a.KW, KS = K1 + K2;
    // destination histograms (argmax counts before capacity, R13)
    for (int k0 = 0; k0 < K1; k0 += 32) {
        int mine = 0;
        for (int kk = 0; kk < 32 && k0 + kk < K1; ++kk) {
            const int c = __popc(__ballot_sync(kFull, has && i == k0 + kk));
            if (lane == kk) mine = c;
        }
        if (k0 + lane < K1) a.blk_hist1[ch * K1 + k0 + lane] = mine;
    }
    for (int k0 = 0; k0 < K2; k0 += 32) {
        int mine = 0;
        for (int kk = 0; kk < 32 && k0 + kk < K2; ++kk) {
            const int c = __popc(__ballot_sync(kFull, has && j == k0 + kk));
            if (lane == kk) mine = c;
        }
        if (k0 + lane < K2) a.blk_hist2a[ch * K2 + k0 + lane] = mine;
    }
    // softmax-entry sums in fp64, fixed order (deterministic)
    if (KW <= 6) {
        for (int k = 0; k < KW; ++k) {
            double acc = has ? (double)s_lg[tok * lds + k] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
            if (lane == 0) a.blk_psum[ch * KS + k] = acc;
        }
    } else {
        for (int k0 = 0; k0 < KW; k0 += 32) {
            double v[32];
#pragma unroll
            for (int kk = 0; kk < 32; ++kk) v[kk] = (has && k0 + kk < KW) ? (double)s_lg[tok * lds + k0 + kk] : 0.0;
            const double tot = transpose_reduce32_f64(v, lane);
            if (k0 + lane < KW) a.blk_psum[ch * KS + k0 + lane] = tot;
        }
    }
    if (a.flat) {                                    // FLAT: the second statistic counts the tokens
        const int cnt = __popc(__ballot_sync(kFull, has));
        if (lane == 0) a.blk_psum[ch * KS + K1] = (double)cnt;
    }
}

// Phases B and C of the level-1 gate over one tile of nt <= Sync::nthr() tokens whose
// logits are s_lg [nt][lds] (entries 0..K1-1: inter router W_p; K1..KW-1: intra W_q).
// tok0: global index of the tile's first token (a multiple of 32 within its rank); ch0:
// the chunk index of that token (v * nch + t / 32).  Must be entered by all Sync threads
// after the logits are visible to them.
template <class Sync>
__device__ GateTok gate_finish(const GateArgs &a, float *s_lg, int lds, int *s_wh, int *s_bh, int64_t tok0,
                               int nt, int64_t ch0) {
    const int tid = Sync::tid();
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
    // Phase C: capacity ranks (R5, R8) -- the rank of the token among the earlier tokens of
    // its 32-token chunk with the same destination (the scan adds the chunk's offset), the
    // chunk's histograms and LB partials; with the fused permute also the tile-wide rank.
    const int lane = tid & 31, w = tid >> 5;
    const bool has = tid < nt;
    const unsigned peers = __match_any_sync(kFull, i);
    const int lrw = __popc(peers & ((1u << lane) - 1u));
    if (has && !a.fuse_dispatch) a.route.slot1[tok0 + tid] = lrw;
    if (32 * w < nt) chunk_tables(a, s_lg, lds, i, j, has, ch0 + w, lane, tid);
    int lr = lrw;
    if (a.fuse_dispatch) lr = block_rank<Sync>(i, K1, s_wh, s_bh);
    return GateTok{i, lr};
}

// Level-1 scan of one rank over its chunk tables: exclusive prefix over
// chunks of each destination's count (the chunk offsets the permute adds to the chunk-local
// ranks), totals -> hist1, counts1 = min(hist1, C1) (R5), and the LB statistics reduced over
// chunks in fixed order (deterministic).  Work split over the NW warps w of the caller.
__device__ __forceinline__ int warp_exclusive_scan(const int32_t *p, int n, int64_t st, int32_t *out_excl) {
    const int lane = threadIdx.x & 31;
    int carry = 0;
    for (int b0 = 0; b0 < n; b0 += 32) {
        const int i = b0 + lane;
        const int v = i < n ? __ldcg(p + (int64_t)i * st) : 0;
        int x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += y;
        }
        if (i < n) out_excl[(int64_t)i * st] = carry + x - v;
        carry += __shfl_sync(kFull, x, 31);
    }
    return carry;
}
__device__ __forceinline__ double warp_sum_f64(const double *p, int n, int64_t st) {
    const int lane = threadIdx.x & 31;
    double acc = 0.0;
    for (int i = lane; i < n; i += 32) acc += __ldcg(p + (int64_t)i * st);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    return acc;
}
__device__ __forceinline__ int warp_sum_i32(const int32_t *p, int n, int64_t st) {
    const int lane = threadIdx.x & 31;
    int acc = 0;
    for (int i = lane; i < n; i += 32) acc += __ldcg(p + (int64_t)i * st);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    return acc;
}

__device__ __forceinline__ void scan1_rank(const Scan1Args &a, int v, int w, int NW) {
    const int lane = threadIdx.x & 31;
    const int KS = a.K1 + a.K2;
    const int jobs = a.K1 + KS + a.K2;
    for (int jb = w; jb < jobs; jb += NW) {
        if (jb < a.K1) {
            const int k = jb;
            const int64_t o = (int64_t)v * a.nblk * a.K1 + k;
            const int tot = warp_exclusive_scan(a.blk_hist1 + o, a.nblk, a.K1, a.blk_off1 + o);
            if (lane == 0) {
                const int32_t cnt = (int32_t)(tot < a.C1 ? tot : a.C1);
                a.stats.hist1[v * a.K1 + k] = tot;
                a.counts1[v * a.K1 + k] = cnt;
                if (a.peer.bases && a.flat) {      // counts travel with the rows: rcounts[q][src][k % e]
                    const PeerMap &P = a.peer;
                    const int rk = P.rank0 + v, q = k / P.e;
                    reinterpret_cast<int32_t *>(P.bases[q / P.V] + P.off_rcounts)[((int64_t)(q % P.V) * P.G + rk) * P.e + k % P.e] = cnt;
                }
            }
        } else if (jb < a.K1 + KS) {
            const int k = jb - a.K1;
            const double sum = warp_sum_f64(a.blk_psum + (int64_t)v * a.nblk * KS + k, a.nblk, KS);
            if (lane == 0) {
                if (k < a.K1) a.stats.psum1[v * a.K1 + k] = sum;
                else a.stats.psum2[v * a.K2 + (k - a.K1)] = sum;
            }
        } else {
            const int k = jb - a.K1 - KS;
            const int c = warp_sum_i32(a.blk_hist2a + (int64_t)v * a.nblk * a.K2 + k, a.nblk, a.K2);
            if (lane == 0) a.stats.hist2[v * a.K2 + k] = c;
        }
    }
}

}  // namespace smile
