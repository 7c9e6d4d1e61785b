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

// Softmax derivative terms of one level for one token, lanes over k (warp-cooperative).
//   dl_k = dtop * ptop * (delta_k,top - p_k) + coef * p_k * (f_k - sum_i f_i p_i)
__device__ void level_dlogits(const float *L, int K, int top, float dtop, float coef, const int32_t *hist,
                              float invT, float *dl) {
    const int lane = threadIdx.x & 31;
    const float mx = L[top];
    float s = 0.f, fp = 0.f;
    for (int k = lane; k < K; k += 32) s += expf(L[k] - mx);
    s = warp_sum(s);
    for (int k = lane; k < K; k += 32) fp += (float)hist[k] * invT * __fdiv_rn(expf(L[k] - mx), s);
    fp = warp_sum(fp);
    const float ptop = __frcp_rn(s);
    for (int k = lane; k < K; k += 32) {
        const float pk = __fdiv_rn(expf(L[k] - mx), s);
        const float fk = (float)hist[k] * invT;
        dl[k] = dtop * ptop * ((k == top ? 1.f : 0.f) - pk) + coef * pk * (fk - fp);
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
    for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g < total; g += warps) {
        const int v = (int)(g / a.T);
        const int i = a.route.dest1[g];
        const int s1 = a.route.slot1[g];
        float dgate = 0.f;
        if (s1 < a.C1) {
            const float gt = a.route.gate[g];
            const int64_t row = ((int64_t)v * a.K1 + i) * a.C1 + s1;
            float acc = 0.f;
            for (int c = lane; c < a.d; c += 32) {
                const float go = ld_el(a.gout, g * a.d + c, a.bf16);
                acc = fmaf(go, ld_el(a.back1, row * a.d + c, a.bf16), acc);
                st_el(a.dsend, row * a.d + c, gt * go, a.bf16);
            }
            dgate = warp_sum(acc);
        }
        const float *L = a.logits + g * a.KW;
        float *dl = a.dlogits + g * a.KW;
        const float p = a.route.p[g], q = a.route.q[g];
        const float c1 = (float)(a.lam * a.alpha * (double)a.K1) * invT;
        level_dlogits(L, a.K1, i, q * dgate, c1, a.stats.hist1 + (int64_t)v * a.K1, invT, dl);
        if (!a.flat) {
            const float c2 = (float)(a.lam * a.beta * (double)a.K2) * invT;
            level_dlogits(L + a.K1, a.K2, a.route.dest2[g], p * dgate, c2, a.stats.hist2 + (int64_t)v * a.K2, invT,
                          dl + a.K1);
        }
    }
}

// a19 router: dx[t, c] += sum_k dlogits[t, k] W[k, c]; partial[chunk, k, c] = sum over the
// chunk's tokens of dlogits[t, k] x[t, c] (thread per column; fixed order).
constexpr int kRbCols = 128, kRbTok = 512, kRbK = 8;

__global__ void router_bwd_kernel(RouterBwdArgs a) {
    __shared__ float s_dl[64][kRbK];
    const int c = blockIdx.x * kRbCols + threadIdx.x;
    const int64_t t0 = (int64_t)blockIdx.y * kRbTok;
    const int64_t t1 = (t0 + kRbTok < a.rows) ? t0 + kRbTok : a.rows;
    for (int k0 = 0; k0 < a.KW; k0 += kRbK) {
        const int nk = min(kRbK, a.KW - k0);
        float acc[kRbK], w[kRbK];
#pragma unroll
        for (int k = 0; k < kRbK; ++k) {
            acc[k] = 0.f;
            w[k] = (k < nk && c < a.d) ? a.w[(int64_t)(k0 + k) * a.d + c] : 0.f;
        }
        for (int64_t tb = t0; tb < t1; tb += 64) {
            __syncthreads();
            for (int z = threadIdx.x; z < 64 * kRbK; z += blockDim.x) {
                const int tt = z / kRbK, k = z % kRbK;
                s_dl[tt][k] = (tb + tt < t1 && k < nk) ? a.dlogits[(tb + tt) * a.KW + k0 + k] : 0.f;
            }
            __syncthreads();
            if (c < a.d) {
                const int nt = (int)((t1 - tb) < 64 ? (t1 - tb) : 64);
                for (int tt = 0; tt < nt; ++tt) {
                    const int64_t t = tb + tt;
                    const float xv = ld_el(a.x, t * a.d + c, a.bf16);
                    float dxa = 0.f;
#pragma unroll
                    for (int k = 0; k < kRbK; ++k) {
                        acc[k] = fmaf(s_dl[tt][k], xv, acc[k]);
                        dxa = fmaf(s_dl[tt][k], w[k], dxa);
                    }
                    st_el(a.dx, t * a.d + c, ld_el(a.dx, t * a.d + c, a.bf16) + dxa, a.bf16);
                }
            }
        }
        if (c < a.d)
            for (int k = 0; k < nk; ++k) a.partial[((int64_t)blockIdx.y * a.KW + k0 + k) * a.d + c] = acc[k];
    }
}

__global__ void router_bwd_reduce(RouterBwdArgs a) {
    const int64_t n = (int64_t)a.KW * a.d;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float s = 0.f;
        for (int ch = 0; ch < a.nchunk; ++ch) s += a.partial[(int64_t)ch * n + i];
        a.dW[i] = s;
    }
}

}  // namespace

void launch_combine_bwd(const CombineBwdArgs &a, cudaStream_t st) {
    if (a.T == 0) return;
    int64_t warps = (int64_t)a.V * a.T;
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
    dim3 grid((a.d + kRbCols - 1) / kRbCols, a.nchunk);
    note_launch();
    router_bwd_kernel<<<grid, kRbCols, 0, st>>>(a);
    note_launch();
    router_bwd_reduce<<<148, 256, 0, st>>>(a);
}

}  // namespace smile
