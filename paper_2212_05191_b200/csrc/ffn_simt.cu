// ffn_simt.cu -- grouped expert FFN on the FP32 SIMT pipe.
//
// Y = GELU(X W1 + b1) W2 + b2 for every resident expert over its S capacity-padded
// segments, as two grouped GEMMs D = A B^T + bias with B stored K-major ([N, K]).
// This is the path of the fp32 layer (C1: rtol 1e-5 rules out TF32) and the bf16
// debugging fallback; the bf16 product path is ffn_tcgen05.cu.
//
// Work list: segment g = (v, s, k) holds counts[g] valid rows at row g*Cseg of X; its
// expert is v*e + k.  Tiles of 64 rows x 64 columns are enumerated on the device from
// the counts (no host sync), so padding rows cost nothing.
#include "smile_internal.h"
#include "tiles.cuh"

namespace smile {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, NTHR = 256, MAXSEG = 4096;

struct GemmArgs {
    const void *A; const void *B; const float *bias; void *D; const int32_t *counts;
    int nseg, e, S; int64_t Cseg; int N, K; int gelu; int bf16;
};

__device__ __forceinline__ float ld(const void *p, int64_t i, int bf16) {
    return bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16 *>(p)[i])
                : reinterpret_cast<const float *>(p)[i];
}

__device__ __forceinline__ float gelu_erf(float z) {
    return 0.5f * z * (1.0f + erff(z * 0.70710678118654752f));   // R21: exact erf GELU
}

__global__ void __launch_bounds__(NTHR) grouped_gemm_simt(GemmArgs a) {
    __shared__ int s_pref[MAXSEG + 1];
    __shared__ int s_warp[32];
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const int tid = threadIdx.x;
    tile_prefix<BM>(a.counts, a.nseg, s_pref, s_warp);
    const int ntn = a.N / BN;
    const int64_t total = (int64_t)s_pref[a.nseg] * ntn;
    const int tx = tid % 16, ty = tid / 16;
    for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
        const int nt = (int)(tile % ntn);
        const int mtg = (int)(tile / ntn);
        const int g = tile_segment(s_pref, a.nseg, mtg);
        const int mt = mtg - s_pref[g];
        const int cnt = a.counts[g];
        const int v = g / (a.S * a.e), k = g % a.e;
        const int64_t expert = (int64_t)v * a.e + k;
        const int64_t row0 = (int64_t)g * a.Cseg + (int64_t)mt * BM;
        const int rows = min(BM, cnt - mt * BM);
        const int n0 = nt * BN;
        const int64_t boff = expert * (int64_t)a.N * a.K;
        float acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
        for (int k0 = 0; k0 < a.K; k0 += BK) {
#pragma unroll
            for (int z = 0; z < 4; ++z) {
                const int idx = tid + z * NTHR;     // 0..1023 over [64 rows][16 k]
                const int r = idx / BK, kk = idx % BK;
                As[kk][r] = (r < rows) ? ld(a.A, (row0 + r) * a.K + k0 + kk, a.bf16) : 0.f;
                Bs[kk][r] = ld(a.B, boff + (int64_t)(n0 + r) * a.K + k0 + kk, a.bf16);
            }
            __syncthreads();
#pragma unroll
            for (int kk = 0; kk < BK; ++kk) {
                float av[4], bv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) { av[i] = As[kk][ty * 4 + i]; bv[i] = Bs[kk][tx * 4 + i]; }
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
            }
            __syncthreads();
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = ty * 4 + i;
            if (r >= rows) continue;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int n = n0 + tx * 4 + j;
                float y = acc[i][j] + a.bias[expert * a.N + n];
                if (a.gelu) y = gelu_erf(y);
                const int64_t o = (row0 + r) * a.N + n;
                if (a.bf16) reinterpret_cast<__nv_bfloat16 *>(a.D)[o] = __float2bfloat16_rn(y);
                else reinterpret_cast<float *>(a.D)[o] = y;
            }
        }
    }
}

}  // namespace

void launch_ffn_simt(const FfnArgs &f, cudaStream_t st) {
    const int nseg = f.V * f.S * f.e;
    const int grid = f.num_sms * 4;
    GemmArgs g1{f.X, f.W1t, f.b1, f.H, f.counts, nseg, f.e, f.S, f.Cseg, f.d_ff, f.d, 1, f.bf16};
    grouped_gemm_simt<<<grid, NTHR, 0, st>>>(g1);
    GemmArgs g2{f.H, f.W2t, f.b2, f.Y, f.counts, nseg, f.e, f.S, f.Cseg, f.d, f.d_ff, 0, f.bf16};
    grouped_gemm_simt<<<grid, NTHR, 0, st>>>(g2);
}

bool ffn_simt_supported(int nseg, int d, int d_ff) {
    return nseg <= MAXSEG && d % BN == 0 && d_ff % BN == 0 && d % BK == 0 && d_ff % BK == 0;
}

}  // namespace smile
