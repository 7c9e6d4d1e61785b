// backward_kernels.cu -- routing-side backward of the SMILE layer.
//
// The paper trains the layer (Eq. 5) but gives no backward; the gradients
// are the chain rule of Eq. (3) and Eq. (4) with the dispatch fractions f held constant
// (S:L240), as in oracle_backward.
#include "smile_internal.h"

namespace smile {
namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ float warp_sum(float v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

__device__ __forceinline__ float ld_el(const void *p, int64_t i, int bf16) {
    return bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16 *>(p)[i]) : reinterpret_cast<const float *>(p)[i];
}

__device__ __forceinline__ void st_el(void *p, int64_t i, float v, int bf16) {
    if (bf16) reinterpret_cast<__nv_bfloat16 *>(p)[i] = __float2bfloat16_rn(v);
    else reinterpret_cast<float *>(p)[i] = v;
}

// Softmax derivative terms of one level for one token (serial over k):
//   dl_k = dtop * ptop * (delta_k,top - p_k) + coef * p_k * (f_k - sum_i f_i p_i)
__device__ void level_dlogits_thread(const float *L, int K, int top, float dtop, float coef, const int32_t *hist,
                                     float invT, float *dl) {
    const float mx = L[top];
    float s = 0.f;
    for (int k = 0; k < K; ++k) s += expf(L[k] - mx);
    const float inv = __frcp_rn(s);
    float fp = 0.f;
    for (int k = 0; k < K; ++k) fp += (float)hist[k] * invT * (expf(L[k] - mx) * inv);
    for (int k = 0; k < K; ++k) {
        const float pk = expf(L[k] - mx) * inv;
        const float fk = (float)hist[k] * invT;
        dl[k] = dtop * inv * ((k == top ? 1.f : 0.f) - pk) + coef * pk * (fk - fp);
    }
}

// FLAT top-k (Eq. 2, R29-R32): dl_k = sum_j dgate_j p_{e_j} (delta_{k, e_j} - p_k)
//                                  + coef p_k (f_k - sum_i f_i p_i)        (serial over k)
__device__ void topk_dlogits_thread(const float *L, int K, const int *e, const float *dg, int topk, float coef,
                                    const int32_t *hist, float invT, float *dl) {
    const float mx = L[e[0]];                   // choice 0 is the argmax (R29)
    float s = 0.f;
    for (int k = 0; k < K; ++k) s += expf(L[k] - mx);
    const float inv = __frcp_rn(s);
    float pe[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) pe[j] = j < topk ? expf(L[e[j]] - mx) * inv : 0.f;
    float fp = 0.f;
    for (int k = 0; k < K; ++k) fp += (float)hist[k] * invT * (expf(L[k] - mx) * inv);
    for (int k = 0; k < K; ++k) {
        const float pk = expf(L[k] - mx) * inv;
        const float fk = (float)hist[k] * invT;
        float v = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (j < topk) v += dg[j] * pe[j] * ((k == e[j] ? 1.f : 0.f) - pk);
        dl[k] = v + coef * pk * (fk - fp);
    }
}

// a16 + a19: one warp per token.  dgate = <gout, back1[i, slot1]> (fp32); the gradient
// row gate * gout goes to dsend[i, slot1] (the forward route); dlogits from Eq. (3)'s
// p_i q_j and Eq. (4)'s LB terms.
__global__ void combine_bwd_kernel(CombineBwdArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t total = (int64_t)a.V * a.T;
    const float invT = 1.f / (float)a.T;
    // a warp takes 32 consecutive tokens: their rows one after the other (16-byte
    // vectors, warp-wide dot product for dgate), then lane t computes token t's dlogits
    const int64_t wg = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int topk = a.topk > 1 ? a.topk : 1;
    for (int64_t g0 = wg * 32; g0 < total; g0 += warps * 32) {
      float my_dgate[4] = {0.f, 0.f, 0.f, 0.f};
      for (int tt = 0; tt < 32 && g0 + tt < total; ++tt) {
      const int64_t g = g0 + tt;
      const int v = (int)(g / a.T);
      for (int jc = 0; jc < topk; ++jc) {        // top-k: every choice of the token (choice-major route)
        const int64_t gi = (int64_t)jc * total + g;
        const int i = a.route.dest1[gi];
        const int s1 = a.route.slot1[gi];
        float dgate = 0.f;
        if (s1 < a.C1) {
            const float gt = a.route.gate[gi];
            const void *bsrc = a.back1;
            void *gdst = a.dsend;
            int64_t brow = ((int64_t)v * a.K1 + i) * a.C1 + s1, grow = brow;
            if (a.peer.bases) {
                // PEER: the forward output row lives at its owner (bi-level: the intermediate's
                // ret1; flat: the expert's Y) and the gradient row goes where the forward row
                // went (bi-level: the intermediate's recv1; flat: the expert's Y, read first)
                const PeerMap &P = a.peer;
                const int rk = P.rank0 + v;
                const int64_t esz = a.bf16 ? 2 : 4;
                if (P.n > 0) {
                    const int s_ = rk / P.m, l = rk % P.m, u = i * P.m + l;
                    const int64_t row = ((int64_t)(u % P.V) * P.n + s_) * a.C1 + s1;
                    bsrc = P.bases[u / P.V] + P.off_ret1;
                    gdst = P.bases[u / P.V] + P.off_recv1;
                    brow = grow = row;
                } else {
                    const int q = i / P.e;
                    const int64_t row = (((int64_t)(q % P.V) * P.G + rk) * P.e + i % P.e) * a.C1 + s1;
                    bsrc = P.bases[q / P.V] + P.off_Y;
                    gdst = P.bases[q / P.V] + P.off_Y;
                    brow = grow = row;
                }
                (void)esz;
            }
            // 16-byte vectors: lane handles elements [8v, 8v + 8) (bf16) / [4v, 4v + 4) (fp32)
            const int epv = a.bf16 ? 8 : 4, nv = a.d / epv;
            const int64_t esz = a.bf16 ? 2 : 4;
            const uint4 *gv = reinterpret_cast<const uint4 *>(static_cast<const char *>(a.gout) + g * a.d * esz);
            const uint4 *bv = reinterpret_cast<const uint4 *>(static_cast<const char *>(bsrc) + brow * a.d * esz);
            uint4 *dv = reinterpret_cast<uint4 *>(static_cast<char *>(gdst) + grow * a.d * esz);
            float acc = 0.f;
            uint4 gk[4];
            int nk = 0;
            for (int vi = lane; vi < nv; vi += 32) {
                const uint4 gg = gv[vi], bb = bv[vi];
                if (nk < 4) gk[nk] = gg;
                ++nk;
                if (a.bf16) {
                    const __nv_bfloat162 *g2 = reinterpret_cast<const __nv_bfloat162 *>(&gg);
                    const __nv_bfloat162 *b2 = reinterpret_cast<const __nv_bfloat162 *>(&bb);
#pragma unroll
                    for (int z = 0; z < 4; ++z) {
                        const float2 fg = __bfloat1622float2(g2[z]), fb = __bfloat1622float2(b2[z]);
                        acc = fmaf(fg.x, fb.x, acc);
                        acc = fmaf(fg.y, fb.y, acc);
                    }
                } else {
                    const float *fg = reinterpret_cast<const float *>(&gg);
                    const float *fb = reinterpret_cast<const float *>(&bb);
#pragma unroll
                    for (int z = 0; z < 4; ++z) acc = fmaf(fg[z], fb[z], acc);
                }
            }
            __syncwarp();                      // (flat PEER: the row is read before it is overwritten)
            nk = 0;
            for (int vi = lane; vi < nv; vi += 32, ++nk) {
                const uint4 gg = nk < 4 ? gk[nk] : gv[vi];
                uint4 o;
                if (a.bf16) {
                    const __nv_bfloat162 *g2 = reinterpret_cast<const __nv_bfloat162 *>(&gg);
                    __nv_bfloat162 *o2 = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
                    for (int z = 0; z < 4; ++z) {
                        const float2 fg = __bfloat1622float2(g2[z]);
                        o2[z] = __floats2bfloat162_rn(gt * fg.x, gt * fg.y);
                    }
                } else {
                    const float *fg = reinterpret_cast<const float *>(&gg);
                    float *fo = reinterpret_cast<float *>(&o);
#pragma unroll
                    for (int z = 0; z < 4; ++z) fo[z] = gt * fg[z];
                }
                dv[vi] = o;
            }
            dgate = warp_sum(acc);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (j == jc && lane == tt) my_dgate[j] = dgate;
      }
      }
      const int64_t g = g0 + lane;
      if (g < total) {
        const int v = (int)(g / a.T);
        const float *L = a.logits + g * a.KW;
        float *dl = a.dlogits + g * a.KW;
        const float p = a.route.p[g], q = a.route.q[g];
        const float c1 = (float)(a.lam * a.alpha * (double)a.K1) * invT;
        if (topk > 1) {
            int e[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) e[j] = j < topk ? a.route.dest1[(int64_t)j * total + g] : 0;
            topk_dlogits_thread(L, a.K1, e, my_dgate, topk, c1, a.stats.hist1 + (int64_t)v * a.K1, invT, dl);
            continue;
        }
        level_dlogits_thread(L, a.K1, a.route.dest1[g], q * my_dgate[0], c1, a.stats.hist1 + (int64_t)v * a.K1, invT, dl);
        if (!a.flat) {
            const float c2 = (float)(a.lam * a.beta * (double)a.K2) * invT;
            level_dlogits_thread(L + a.K1, a.K2, a.route.dest2[g], p * my_dgate[0], c2,
                                 a.stats.hist2 + (int64_t)v * a.K2, invT, dl + a.K1);
        }
      }
    }
}

// a19 router, two streams (each with few registers, so many tokens stay in flight):
//   router_dx_kernel:  dx[t, c] += sum_k dlogits[t, k] W[k, c]   (reads + writes dx)
//   router_dw_kernel:  partial[chunk, k, c] = sum over the chunk's tokens of
//                      dlogits[t, k] x[t, c] (fixed order)       (reads x)
// A thread owns RB_C adjacent columns (one 16-byte vector: 8 bf16 or 4 fp32) of kRbTok
// tokens; router rows go kRbK at a time (W / the accumulators in registers), and kRbU
// tokens' vectors are loaded before any is used.  The chunk's dlogits are staged in smem
// once per pass (broadcast reads in the token loop).
constexpr int kRbTok = 256, kRbK = 8, kRbU = 8, kRbUw = 16, kRbThreads = 128;   // kRbUw: dW stream (reads only)

template <bool BF16>
__device__ __forceinline__ void vec_to_float(const uint4 &v, float *f) {
    if (BF16) {
        const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&v);
#pragma unroll
        for (int z = 0; z < 4; ++z) {
            const float2 t = __bfloat1622float2(h[z]);
            f[2 * z] = t.x;
            f[2 * z + 1] = t.y;
        }
    } else {
        const float *t = reinterpret_cast<const float *>(&v);
#pragma unroll
        for (int z = 0; z < 4; ++z) f[z] = t[z];
    }
}

template <bool BF16>
__global__ void __launch_bounds__(kRbThreads) router_dx_kernel(RouterBwdArgs a) {
    constexpr int RB_C = BF16 ? 8 : 4, EB = BF16 ? 2 : 4;
    __shared__ float s_dl[kRbTok][kRbK];
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) * RB_C;
    const bool ok = c < a.d;
    const int64_t t0 = (int64_t)blockIdx.y * kRbTok;
    const int64_t t1 = (t0 + kRbTok < a.rows) ? t0 + kRbTok : a.rows;
    char *__restrict__ dx = static_cast<char *>(a.dx);
    for (int k0 = 0; k0 < a.KW; k0 += kRbK) {
        const int nk = min(kRbK, a.KW - k0);
        __syncthreads();
        for (int z = threadIdx.x; z < kRbTok * kRbK; z += blockDim.x) {
            const int tt = z / kRbK, k = z % kRbK;
            s_dl[tt][k] = (t0 + tt < t1 && k < nk) ? a.dlogits[(t0 + tt) * a.KW + k0 + k] : 0.f;
        }
        __syncthreads();
        if (!ok) continue;
        float w[kRbK][RB_C];
#pragma unroll
        for (int k = 0; k < kRbK; ++k)
#pragma unroll
            for (int j = 0; j < RB_C; ++j) w[k][j] = k < nk ? a.w[(int64_t)(k0 + k) * a.d + c + j] : 0.f;
        for (int64_t tb = t0; tb < t1; tb += kRbU) {
            uint4 dv[kRbU];
#pragma unroll
            for (int u = 0; u < kRbU; ++u)
                dv[u] = tb + u < t1 ? *reinterpret_cast<const uint4 *>(dx + ((tb + u) * a.d + c) * EB)
                                    : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < kRbU; ++u) {
                if (tb + u >= t1) break;
                const float *dl = s_dl[tb + u - t0];
                float df[RB_C];
                vec_to_float<BF16>(dv[u], df);
#pragma unroll
                for (int k = 0; k < kRbK; ++k) {
                    const float l = dl[k];            // 0 for k >= nk
#pragma unroll
                    for (int j = 0; j < RB_C; ++j) df[j] = fmaf(l, w[k][j], df[j]);
                }
                uint4 o;
                if (BF16) {
                    __nv_bfloat162 *ho = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
                    for (int z = 0; z < 4; ++z) ho[z] = __floats2bfloat162_rn(df[2 * z], df[2 * z + 1]);
                } else {
                    float *fo = reinterpret_cast<float *>(&o);
#pragma unroll
                    for (int z = 0; z < 4; ++z) fo[z] = df[z];
                }
                *reinterpret_cast<uint4 *>(dx + ((tb + u) * a.d + c) * EB) = o;
            }
        }
    }
}

template <bool BF16>
__global__ void __launch_bounds__(kRbThreads) router_dw_kernel(RouterBwdArgs a) {
    constexpr int RB_C = BF16 ? 8 : 4, EB = BF16 ? 2 : 4;
    __shared__ float s_dl[kRbTok][kRbK];
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) * RB_C;
    const bool ok = c < a.d;
    const int64_t t0 = (int64_t)blockIdx.y * kRbTok;
    const int64_t t1 = (t0 + kRbTok < a.rows) ? t0 + kRbTok : a.rows;
    const char *__restrict__ x = static_cast<const char *>(a.x);
    for (int k0 = 0; k0 < a.KW; k0 += kRbK) {
        const int nk = min(kRbK, a.KW - k0);
        __syncthreads();
        for (int z = threadIdx.x; z < kRbTok * kRbK; z += blockDim.x) {
            const int tt = z / kRbK, k = z % kRbK;
            s_dl[tt][k] = (t0 + tt < t1 && k < nk) ? a.dlogits[(t0 + tt) * a.KW + k0 + k] : 0.f;
        }
        __syncthreads();
        if (!ok) continue;
        float acc[kRbK][RB_C];
#pragma unroll
        for (int k = 0; k < kRbK; ++k)
#pragma unroll
            for (int j = 0; j < RB_C; ++j) acc[k][j] = 0.f;
        for (int64_t tb = t0; tb < t1; tb += kRbUw) {
            uint4 xv[kRbUw];
#pragma unroll
            for (int u = 0; u < kRbUw; ++u)
                xv[u] = tb + u < t1 ? __ldg(reinterpret_cast<const uint4 *>(x + ((tb + u) * a.d + c) * EB))
                                    : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < kRbUw; ++u) {
                if (tb + u >= t1) break;
                const float *dl = s_dl[tb + u - t0];
                float xf[RB_C];
                vec_to_float<BF16>(xv[u], xf);
#pragma unroll
                for (int k = 0; k < kRbK; ++k) {
                    const float l = dl[k];
#pragma unroll
                    for (int j = 0; j < RB_C; ++j) acc[k][j] = fmaf(l, xf[j], acc[k][j]);
                }
            }
        }
        for (int k = 0; k < nk; ++k)
#pragma unroll
            for (int j = 0; j < RB_C; ++j) a.partial[((int64_t)blockIdx.y * a.KW + k0 + k) * a.d + c + j] = acc[k][j];
    }
}

// dW[i] = sum over chunks of partial[chunk][i]: a block owns 32 consecutive elements,
// warp w sums chunks w, w + 8, ... (4 loads in flight), then the 8 warp sums are added in
// warp order (fixed order: deterministic).
__global__ void __launch_bounds__(256) router_bwd_reduce(RouterBwdArgs a) {
    __shared__ float s_part[8][32];
    const int64_t n = (int64_t)a.KW * a.d;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t i = (int64_t)blockIdx.x * 32 + lane;
    float s = 0.f;
    if (i < n) {
        int ch = w;
        for (; ch + 24 < a.nchunk; ch += 32) {
            const float v0 = a.partial[(int64_t)ch * n + i], v1 = a.partial[(int64_t)(ch + 8) * n + i];
            const float v2 = a.partial[(int64_t)(ch + 16) * n + i], v3 = a.partial[(int64_t)(ch + 24) * n + i];
            s += v0; s += v1; s += v2; s += v3;
        }
        for (; ch < a.nchunk; ch += 8) s += a.partial[(int64_t)ch * n + i];
    }
    s_part[w][lane] = s;
    __syncthreads();
    if (w == 0 && i < n) {
        float t = 0.f;
        for (int k = 0; k < 8; ++k) t += s_part[k][lane];
        a.dW[i] = t;
    }
}

}  // namespace

void launch_combine_bwd(const CombineBwdArgs &a, cudaStream_t st) {
    if (a.T == 0) return;
    int64_t warps = ((int64_t)a.V * a.T + 31) / 32;          // 32 tokens per warp
    int grid = (int)((warps + 7) / 8);
    if (grid > 148 * 16) grid = 148 * 16;
    note_launch();
    combine_bwd_kernel<<<grid, 256, 0, st>>>(a);
}

size_t router_bwd_partial_floats(int64_t rows, int d, int KW) {
    const int64_t nchunk = (rows + kRbTok - 1) / kRbTok;
    return (size_t)(nchunk > 0 ? nchunk : 1) * KW * d;
}

void launch_router_bwd(const RouterBwdArgs &a0, cudaStream_t st) {
    if (a0.rows == 0) return;
    RouterBwdArgs a = a0;
    a.nchunk = (int)((a.rows + kRbTok - 1) / kRbTok);
    const int per = a.bf16 ? 8 : 4;                       // columns per thread
    int thr = ((a.d / per + 31) / 32) * 32;
    thr = thr < 32 ? 32 : (thr > kRbThreads ? kRbThreads : thr);
    dim3 grid((a.d + thr * per - 1) / (thr * per), a.nchunk);
    note_launch();
    if (a.bf16) router_dw_kernel<true><<<grid, thr, 0, st>>>(a);
    else router_dw_kernel<false><<<grid, thr, 0, st>>>(a);
    note_launch();
    if (a.bf16) router_dx_kernel<true><<<grid, thr, 0, st>>>(a);
    else router_dx_kernel<false><<<grid, thr, 0, st>>>(a);
    note_launch();
    router_bwd_reduce<<<(int)(((int64_t)a.KW * a.d + 31) / 32), 256, 0, st>>>(a);
}

}  // namespace smile
