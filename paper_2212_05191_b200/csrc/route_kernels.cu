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

#include <math.h>

namespace smile {
namespace {

constexpr unsigned kFull = 0xffffffffu;

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ float load_elem(const void *p, int64_t i, int bf16) {
    return bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16 *>(p)[i])
                : reinterpret_cast<const float *>(p)[i];
}

__device__ __forceinline__ void set_err(int *err, int code) {
    if (err) atomicCAS(err, 0, code);
}

// Rank of this thread's item among the block's earlier items with the same bucket
// (bucket < 0: no item).  s_wh: [NW][K] ints, s_bh: [K] ints.  Writes the block
// histogram to s_bh and returns the block-local rank (or -1).  Items are ordered by
// threadIdx.x, i.e. warp-major then lane, matching item order.
__device__ int block_rank(int b, int K, int *s_wh, int *s_bh) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = blockDim.x >> 5;
    for (int i = threadIdx.x; i < NW * K; i += blockDim.x) s_wh[i] = 0;
    __syncthreads();
    const unsigned peers = __match_any_sync(kFull, b);
    const int lr = __popc(peers & ((1u << lane) - 1u));
    if (b >= 0 && lane == __ffs(peers) - 1) s_wh[w * K + b] = __popc(peers);
    __syncthreads();
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        int acc = 0;
        for (int ww = 0; ww < NW; ++ww) {
            const int c = s_wh[ww * K + k];
            s_wh[ww * K + k] = acc;
            acc += c;
        }
        s_bh[k] = acc;
    }
    __syncthreads();
    return b >= 0 ? s_wh[w * K + b] + lr : -1;
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
__device__ void router_tile(const GateArgs &a, float *s_lg, float *s_w, int64_t tok0, int nt) {
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
                    if (lane == 0 && k0 + kk < KW && tt0 + r < nt) s_lg[(tt0 + r) * KW + k0 + kk] = v;
                }
        }
    }
}

// ---------------------------------------------------------------------------------
// a1-a3: level-1 gate.  grid (nblk, V), block TB threads (one token per thread).
// smem: logits tile [TB][KW] fp32 | s_j [TB] | warp hist [NW][K1] | block hist [K1]
// ---------------------------------------------------------------------------------
__global__ void gate1_kernel(GateArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float *s_lg = reinterpret_cast<float *>(smem_raw);
    int *s_j = reinterpret_cast<int *>(s_lg + (size_t)a.TB * a.KW);
    int *s_wh = s_j + a.TB;
    int *s_bh = s_wh + (a.TB / 32) * a.K1;
    float *s_w = reinterpret_cast<float *>(s_bh + ((a.K1 + 3) & ~3));   // [KW, d] when it fits

    const int v = blockIdx.y, blk = blockIdx.x, tid = threadIdx.x;
    const int64_t t0 = (int64_t)blk * a.TB;
    const int nt = (int)imin64(a.TB, a.T - t0);
    const int KW = a.KW, K1 = a.K1, K2 = a.K2;
    const int64_t tok0 = (int64_t)v * a.T + t0;

    // Phase A: the block's logits tile (Eq. 1: r = W x).
    if (a.logits) {
        const float *src = a.logits + tok0 * KW;
        for (int i = tid; i < nt * KW; i += blockDim.x) s_lg[i] = __ldg(src + i);
    } else if (a.bf16) {
        router_tile<true>(a, s_lg, s_w, tok0, nt);
    } else {
        router_tile<false>(a, s_lg, s_w, tok0, nt);
    }
    __syncthreads();
    if (a.logits_out && !a.logits)
        for (int i = tid; i < nt * KW; i += blockDim.x) a.logits_out[tok0 * KW + i] = s_lg[i];
    if (a.logits_out && !a.logits) __syncthreads();

    // Phase B: one thread per token -- argmax (R2, R3), top-1 probabilities (R4), and
    // the softmax entries for the LB statistics, written back over the logits.
    int i = -1, j = 0;
    if (tid < nt) {
        float *L = s_lg + tid * KW;
        bool finite = true;
        for (int k = 0; k < KW; ++k) finite &= isfinite(L[k]);
        if (!finite) set_err(a.err, SMILE_ENONFINITE);
        i = 0;
        for (int k = 1; k < K1; ++k)
            if (L[k] > L[i]) i = k;
        float s1 = 0.f;
        for (int k = 0; k < K1; ++k) s1 += expf(L[k] - L[i]);
        const float p = __frcp_rn(s1);
        float q = 1.f;
        if (!a.flat) {
            float *L2 = L + K1;
            j = 0;
            for (int k = 1; k < K2; ++k)
                if (L2[k] > L2[j]) j = k;
            float s2 = 0.f;
            for (int k = 0; k < K2; ++k) s2 += expf(L2[k] - L2[j]);
            q = __frcp_rn(s2);
            const float mj = L2[j];
            for (int k = 0; k < K2; ++k) L2[k] = __fdiv_rn(expf(L2[k] - mj), s2);
        }
        const float mi = L[i];
        for (int k = 0; k < K1; ++k) L[k] = __fdiv_rn(expf(L[k] - mi), s1);
        const int64_t g = tok0 + tid;
        a.route.dest1[g] = i;
        a.route.dest2[g] = j;
        a.route.p[g] = p;
        a.route.q[g] = q;
        a.route.gate[g] = __fmul_rn(p, q);
        if (i < 0 || i >= K1) set_err(a.err, SMILE_EINDEX);
    }
    s_j[tid] = (tid < nt) ? j : -1;

    // Phase C: block-local capacity rank of dest1 (R5, R8).
    const int lr = block_rank(i, K1, s_wh, s_bh);
    if (tid < nt) a.route.slot1[tok0 + tid] = lr;
    const int64_t bo = (int64_t)v * a.nblk + blk;
    for (int k = tid; k < K1; k += blockDim.x) a.blk_hist1[bo * K1 + k] = s_bh[k];
    // LB statistics partials, summed over the block's tokens in token order (fp64).
    for (int k = tid; k < KW; k += blockDim.x) {
        double acc = 0.0;
        for (int tt = 0; tt < nt; ++tt) acc += (double)s_lg[tt * KW + k];
        a.blk_psum[bo * (K1 + K2) + k] = acc;
    }
    if (a.flat && tid == 0) a.blk_psum[bo * (K1 + K2) + K1] = (double)nt;
    for (int k = tid; k < K2; k += blockDim.x) {
        int c = 0;
        for (int tt = 0; tt < nt; ++tt) c += (s_j[tt] == k);
        a.blk_hist2a[bo * K2 + k] = c;
    }
}

// Level-1 scan: per rank, exclusive prefix over blocks of each destination's count;
// totals -> hist1, counts1 = min(hist1, C1); stats reduced over blocks in fixed order.
__global__ void scan1_kernel(Scan1Args a) {
    const int v = blockIdx.x;
    const int KS = a.K1 + a.K2;
    for (int k = threadIdx.x; k < a.K1; k += blockDim.x) {
        int acc = 0;
        for (int b = 0; b < a.nblk; ++b) {
            const int64_t o = ((int64_t)v * a.nblk + b) * a.K1 + k;
            a.blk_off1[o] = acc;
            acc += a.blk_hist1[o];
        }
        a.stats.hist1[v * a.K1 + k] = acc;
        a.counts1[v * a.K1 + k] = (int32_t)imin64(acc, a.C1);
    }
    for (int k = threadIdx.x; k < KS; k += blockDim.x) {
        double s = 0.0;
        for (int b = 0; b < a.nblk; ++b) s += a.blk_psum[((int64_t)v * a.nblk + b) * KS + k];
        if (k < a.K1) a.stats.psum1[v * a.K1 + k] = s;
        else a.stats.psum2[v * a.K2 + (k - a.K1)] = s;
    }
    for (int k = threadIdx.x; k < a.K2; k += blockDim.x) {
        int c = 0;
        for (int b = 0; b < a.nblk; ++b) c += a.blk_hist2a[((int64_t)v * a.nblk + b) * a.K2 + k];
        a.stats.hist2[v * a.K2 + k] = c;
    }
}

// a6: level-2 gate at the intermediate: rank valid received slots per j, in received
// order (source node ascending, then slot: the flat index s*C1 + c, R8).
__global__ void rank2_kernel(Rank2Args a) {
    __shared__ int s_wh[(kRank2Items / 32) * 256];
    __shared__ int s_bh[256];
    const int v = blockIdx.y, blk = blockIdx.x;
    const int64_t x = (int64_t)blk * kRank2Items + threadIdx.x;
    int b = -1;
    if (x < a.items) {
        b = a.recv_meta[(int64_t)v * a.items + x];
        if (b >= a.K2) { set_err(a.err, SMILE_EINDEX); b = -1; }
    }
    const int lr = block_rank(b, a.K2, s_wh, s_bh);
    if (x < a.items) a.slot2[(int64_t)v * a.items + x] = lr;
    for (int k = threadIdx.x; k < a.K2; k += blockDim.x)
        a.blk_hist2[((int64_t)v * a.nblk + blk) * a.K2 + k] = s_bh[k];
}

__global__ void scan2_kernel(Rank2Args a) {
    const int v = blockIdx.x;
    for (int k = threadIdx.x; k < a.K2; k += blockDim.x) {
        int acc = 0;
        for (int b = 0; b < a.nblk; ++b) {
            const int64_t o = ((int64_t)v * a.nblk + b) * a.K2 + k;
            a.blk_off2[o] = acc;
            acc += a.blk_hist2[o];
        }
        a.counts2[v * a.K2 + k] = (int32_t)imin64(acc, a.C2);
    }
}

// a4: level-1 permute.  One warp per token: slot1 = block offset + block-local rank;
// kept rows are copied to send[v, i, slot1] with 16-byte vectors; meta = j.
// The same launch fills meta = -1 for the empty slots [counts1[i], C1).
__global__ void dispatch1_kernel(Dispatch1Args a) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int nvec = (int)(a.rowbytes / 16);
    const int64_t total = (int64_t)a.V * a.T;
    for (int64_t g = gw; g < total; g += warps) {
        const int v = (int)(g / a.T);
        const int64_t t = g - (int64_t)v * a.T;
        const int i = a.route.dest1[g];
        const int blk = (int)(t / a.TB);
        const int slot = a.blk_off1[((int64_t)v * a.nblk + blk) * a.K1 + i] + a.route.slot1[g];
        __syncwarp();
        if (lane == 0) a.route.slot1[g] = slot;
        if (slot < a.C1) {
            const int64_t dst_row = ((int64_t)v * a.K1 + i) * a.C1 + slot;
            warp_copy_row(reinterpret_cast<int4 *>(static_cast<char *>(a.send) + dst_row * a.rowbytes),
                          reinterpret_cast<const int4 *>(static_cast<const char *>(a.x) + g * a.rowbytes),
                          nvec, lane);
            if (a.meta && lane == 0) a.meta[dst_row] = a.route.dest2[g];
        }
    }
    if (a.meta) {
        const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
        const int64_t tot = (int64_t)a.V * a.K1 * a.C1;
        for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < tot; idx += nthr) {
            const int64_t vi = idx / a.C1, c = idx - vi * a.C1;   // vi = v*K1 + i
            const int64_t v = vi / a.K1, i = vi - v * a.K1;
            const int64_t last = ((v * a.nblk) + a.nblk - 1) * a.K1 + i;   // total = off + hist of the last block
            if (c >= (int64_t)a.blk_off1[last] + a.blk_hist1[last]) a.meta[idx] = -1;
        }
    }
}

// a7: level-2 permute at the intermediate.  One warp per received slot (s, c) with a
// valid j: slot2 = block offset + block-local rank; kept rows go to send2[v, j, slot2].
__global__ void dispatch2_kernel(Dispatch2Args a) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int nvec = (int)(a.rowbytes / 16);
    const int64_t total = (int64_t)a.V * a.items;
    for (int64_t g = gw; g < total; g += warps) {
        const int j = a.recv_meta[g];
        if (j < 0 || j >= a.K2) continue;
        const int v = (int)(g / a.items);
        const int64_t x = g - (int64_t)v * a.items;
        const int blk = (int)(x / kRank2Items);
        const int slot = a.blk_off2[((int64_t)v * a.nblk + blk) * a.K2 + j] + a.slot2[g];
        __syncwarp();
        if (lane == 0) a.slot2[g] = slot;
        if (slot < a.C2) {
            const int64_t dst_row = ((int64_t)v * a.K2 + j) * a.C2 + slot;
            warp_copy_row(reinterpret_cast<int4 *>(static_cast<char *>(a.send2) + dst_row * a.rowbytes),
                          reinterpret_cast<const int4 *>(static_cast<const char *>(a.recv1) + g * a.rowbytes),
                          nvec, lane);
        }
    }
}

// a11: level-2 un-permute: ret1[s, c] = keep2 ? ret2[j, slot2] : 0 for valid slots.
__global__ void combine2_kernel(Combine2Args a) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int nvec = (int)(a.rowbytes / 16);
    const int64_t total = (int64_t)a.V * a.items;
    for (int64_t g = gw; g < total; g += warps) {
        const int j = a.recv_meta[g];
        if (j < 0 || j >= a.K2) continue;
        const int v = (int)(g / a.items);
        const int s2 = a.slot2[g];
        int4 *dst = reinterpret_cast<int4 *>(static_cast<char *>(a.ret1) + g * a.rowbytes);
        if (s2 < a.C2) {
            const int64_t src_row = ((int64_t)v * a.K2 + j) * a.C2 + s2;
            warp_copy_row(dst, reinterpret_cast<const int4 *>(static_cast<const char *>(a.ret2) + src_row * a.rowbytes),
                          nvec, lane);
        } else {
            warp_zero_row(dst, nvec, lane);
        }
    }
}

// a13: level-1 combine (Eq. 3): out[t] = keep1 ? dtype(gate * back1[i, slot1]) : 0.
template <bool BF16>
__global__ void combine1_kernel(Combine1Args a) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    constexpr int kPer = BF16 ? 8 : 4;             // elements per 16-byte vector
    const int nvec = a.d / kPer;
    const int64_t total = (int64_t)a.V * a.T;
    for (int64_t g = gw; g < total; g += warps) {
        const int v = (int)(g / a.T);
        const int i = a.route.dest1[g];
        const int s1 = a.route.slot1[g];
        int4 *dst = reinterpret_cast<int4 *>(static_cast<char *>(a.out) + g * (int64_t)a.d * (BF16 ? 2 : 4));
        if (s1 < a.C1) {
            const float gt = a.route.gate[g];
            const int64_t src_row = ((int64_t)v * a.K1 + i) * a.C1 + s1;
            const int4 *src = reinterpret_cast<const int4 *>(static_cast<const char *>(a.back1) +
                                                             src_row * (int64_t)a.d * (BF16 ? 2 : 4));
            for (int k = lane; k < nvec; k += 32) {
                int4 u = __ldg(src + k);
                if (BF16) {
                    __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&u);
#pragma unroll
                    for (int z = 0; z < 4; ++z) {
                        float2 f = __bfloat1622float2(h[z]);
                        h[z] = __floats2bfloat162_rn(__fmul_rn(gt, f.x), __fmul_rn(gt, f.y));
                    }
                } else {
                    float *f = reinterpret_cast<float *>(&u);
#pragma unroll
                    for (int z = 0; z < 4; ++z) f[z] = __fmul_rn(gt, f[z]);
                }
                dst[k] = u;
            }
        } else {
            warp_zero_row(dst, nvec, lane);
        }
    }
}

// a14: Eq. (4) per resident rank in fp64.
__global__ void aux_kernel(smile_stats s, double alpha, double beta, double *loss, int V, int K1,
                           int K2, int64_t T, int flat) {
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
    const int pair = blockIdx.x / a.nsub, k = blockIdx.x % a.nsub;
    const int v = pair / a.P, p = pair % a.P;
    const int q = a.member_local[v * a.P + p];
    if (q < 0) return;
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

inline int grid_for(int64_t warps_needed, int per_block_warps, int cap) {
    int64_t b = (warps_needed + per_block_warps - 1) / per_block_warps;
    if (b < 1) b = 1;
    return (int)(b < cap ? b : cap);
}

}  // namespace

void launch_gate1(const GateArgs &a, cudaStream_t st) {
    if (a.T == 0) return;
    size_t smem = (size_t)a.TB * a.KW * 4 + (size_t)a.TB * 4 + (size_t)(a.TB / 32) * a.K1 * 4 + (size_t)((a.K1 + 3) & ~3) * 4;
    if (!a.logits && (size_t)a.KW * a.d * 4 <= (size_t)kRouterSmem) smem += (size_t)a.KW * a.d * 4;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(gate1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        attr_set = true;
    }
    gate1_kernel<<<dim3(a.nblk, a.V), a.TB, smem, st>>>(a);
}

void launch_scan1(const Scan1Args &a, cudaStream_t st) {
    if (a.T == 0) return;
    scan1_kernel<<<a.V, 128, 0, st>>>(a);
}

void launch_rank2(const Rank2Args &a, cudaStream_t st) {
    if (a.items == 0) return;
    rank2_kernel<<<dim3(a.nblk, a.V), kRank2Items, 0, st>>>(a);
    scan2_kernel<<<a.V, 128, 0, st>>>(a);
}

void launch_dispatch1(const Dispatch1Args &a, cudaStream_t st) {
    if (a.T == 0) return;
    dispatch1_kernel<<<grid_for((int64_t)a.V * a.T, 8, 148 * 16), 256, 0, st>>>(a);
}

void launch_dispatch2(const Dispatch2Args &a, cudaStream_t st) {
    if (a.items == 0) return;
    dispatch2_kernel<<<grid_for((int64_t)a.V * a.items, 8, 148 * 16), 256, 0, st>>>(a);
}

void launch_combine2(const Combine2Args &a, cudaStream_t st) {
    if (a.items == 0) return;
    combine2_kernel<<<grid_for((int64_t)a.V * a.items, 8, 148 * 16), 256, 0, st>>>(a);
}

void launch_combine1(const Combine1Args &a, cudaStream_t st) {
    if (a.T == 0) return;
    const int g = grid_for((int64_t)a.V * a.T, 8, 148 * 16);
    if (a.bf16) combine1_kernel<true><<<g, 256, 0, st>>>(a);
    else combine1_kernel<false><<<g, 256, 0, st>>>(a);
}

void launch_aux(const smile_stats &s, double alpha, double beta, double *loss, int V, int K1, int K2,
                int64_t T, int flat, cudaStream_t st) {
    aux_kernel<<<(V + 127) / 128, 128, 0, st>>>(s, alpha, beta, loss, V, K1, K2, T, flat);
}

void launch_exchange_copy(const CopyXArgs &a, cudaStream_t st) {
    const int64_t chunks = (a.Csub + kCopyRows - 1) / kCopyRows;
    dim3 grid((unsigned)(a.V * a.P * a.nsub), (unsigned)(chunks > 0 ? chunks : 1));
    exchange_copy_kernel<<<grid, 256, 0, st>>>(a);
}

}  // namespace smile
