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

// mode: 0 = act(acc + bias) (act = GELU when gelu), 1 = also D2 = GELU'(acc + bias)
//       (training: the activation derivative the backward needs), 2 = acc * aux (backward
//       dZ = dH . GELU'(A1) with aux = the saved GELU'(A1)), 3 = acc (backward dX).
struct GemmArgs {
    const void *A; const void *B; const float *bias; void *D; const int32_t *counts;
    int nseg, e, S; int64_t Cseg; int N, K; int gelu; int bf16;
    int mode; void *D2; const void *aux;
};

__device__ __forceinline__ float ld(const void *p, int64_t i, int bf16) {
    return bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16 *>(p)[i])
                : reinterpret_cast<const float *>(p)[i];
}

__device__ __forceinline__ float gelu_erf(float z) {
    return 0.5f * z * (1.0f + erff(z * 0.70710678118654752f));   // R21: exact erf GELU
}

__device__ __forceinline__ float gelu_grad(float z) {            // Phi(z) + z phi(z)
    return 0.5f * (1.0f + erff(z * 0.70710678118654752f)) + z * 0.3989422804014327f * expf(-0.5f * z * z);
}

__device__ __forceinline__ void st(void *p, int64_t o, float v, int bf16) {
    if (bf16) reinterpret_cast<__nv_bfloat16 *>(p)[o] = __float2bfloat16_rn(v);
    else reinterpret_cast<float *>(p)[o] = v;
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
                const int64_t o = (row0 + r) * a.N + n;
                float y = acc[i][j];
                if (a.mode <= 1) y += a.bias[expert * a.N + n];
                if (a.mode == 1) st(a.D2, o, gelu_grad(y), a.bf16);
                if ((a.mode == 0 && a.gelu) || a.mode == 1) y = gelu_erf(y);
                if (a.mode == 2) y *= ld(a.aux, o, a.bf16);
                st(a.D, o, y, a.bf16);
            }
        }
    }
}

}  // namespace

void launch_ffn_simt(const FfnArgs &f, cudaStream_t st) {
    const int nseg = f.V * f.S * f.e;
    const int grid = f.num_sms * 4;
    GemmArgs g1{f.X, f.W1t, f.b1, f.H, f.counts, nseg, f.e, f.S, f.Cseg, f.d_ff, f.d, 1, f.bf16, 0, nullptr, nullptr};
    note_launch();
    grouped_gemm_simt<<<grid, NTHR, 0, st>>>(g1);
    GemmArgs g2{f.H, f.W2t, f.b2, f.Y, f.counts, nseg, f.e, f.S, f.Cseg, f.d, f.d_ff, 0, f.bf16, 0, nullptr, nullptr};
    note_launch();
    grouped_gemm_simt<<<grid, NTHR, 0, st>>>(g2);
}

cudaError_t launch_ffn_tcgen05_train(const FfnArgs &f, void *A1, cudaStream_t st);
cudaError_t launch_ffn_tcgen05_dgrad(const FfnBwdArgs &b, int part, cudaStream_t st);

cudaError_t launch_ffn_fwd_train(const FfnArgs &f, void *A1, bool tc, cudaStream_t st) {
    if (tc) return launch_ffn_tcgen05_train(f, A1, st);
    const int nseg = f.V * f.S * f.e;
    const int grid = f.num_sms * 4;
    GemmArgs g1{f.X, f.W1t, f.b1, f.H, f.counts, nseg, f.e, f.S, f.Cseg, f.d_ff, f.d, 1, f.bf16, 1, A1, nullptr};
    note_launch();
    grouped_gemm_simt<<<grid, NTHR, 0, st>>>(g1);
    GemmArgs g2{f.H, f.W2t, f.b2, f.Y, f.counts, nseg, f.e, f.S, f.Cseg, f.d, f.d_ff, 0, f.bf16, 0, nullptr, nullptr};
    note_launch();
    grouped_gemm_simt<<<grid, NTHR, 0, st>>>(g2);
    return cudaGetLastError();
}

namespace {

// Weight gradient of one expert (a17): Dw[e][m][n] = sum over the expert's valid rows r
// of A[r][m] * B[r][n] (A [rows, M], B [rows, N] row-major, segment-padded like X).
// Tile 64 x 64 per block, rows in chunks of 16 staged through smem; fp32 accumulation.
struct WgradArgs {
    const void *A; const void *B; float *Dw; const int32_t *counts;
    int e, S; int64_t Cseg; int M, N; int bf16;
};

__global__ void __launch_bounds__(NTHR) wgrad_simt(WgradArgs a) {
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
    const int ex = blockIdx.z, v = ex / a.e, k = ex % a.e;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    for (int s = 0; s < a.S; ++s) {
        const int g = (v * a.S + s) * a.e + k;
        const int cnt = a.counts[g];
        const int64_t base = (int64_t)g * a.Cseg;
        for (int r0 = 0; r0 < cnt; r0 += BK) {
#pragma unroll
            for (int z = 0; z < 4; ++z) {
                const int idx = tid + z * NTHR;      // [16 rows][64 cols]
                const int rr = idx / BM, cc = idx % BM;
                const bool ok = r0 + rr < cnt;
                As[rr][cc] = (ok && m0 + cc < a.M) ? ld(a.A, (base + r0 + rr) * a.M + m0 + cc, a.bf16) : 0.f;
                Bs[rr][cc] = (ok && n0 + cc < a.N) ? ld(a.B, (base + r0 + rr) * a.N + n0 + cc, a.bf16) : 0.f;
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
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
            if (m < a.M && n < a.N) a.Dw[((int64_t)ex * a.M + m) * a.N + n] = acc[i][j];
        }
}

}  // namespace

// Order: dZ, then everything that reads dY (dW2, db2), then dX -- so dX may overwrite dY
// in place (the peer-store exchange returns dX from the Y buffer) -- then dW1, db1.
cudaError_t launch_ffn_bwd(const FfnBwdArgs &b, bool tc, cudaStream_t st) {
    const int nseg = b.V * b.S * b.e;
    const int NE = b.V * b.e;
    const int grid = b.num_sms * 4;
    const bool tcw = tc && wgrad_tc_supported(b.bf16, b.d, b.d_ff, b.S);
    // dZ = (dY W2^T) . GELU'(A1): B operand = W2 [NE, d_ff, d] as [N = d_ff, K = d]
    if (tc) {
        // the dZ GEMM's epilogue also writes per-strip column sums of dZ: db1 = 1^T dZ
        // (reduced now, before the db2 column sums reuse the workspace)
        cudaError_t e = launch_ffn_tcgen05_dgrad(b, 1, st);
        if (e != cudaSuccess) return e;
        launch_colsum_strips(b.colsum_ws, b.db1, b.counts, NE, b.e, b.S, (int)((b.Cseg + 31) / 32), b.d_ff, st);
    } else {
        GemmArgs g1{b.dY, b.W2, nullptr, b.dZ, b.counts, nseg, b.e, b.S, b.Cseg, b.d_ff, b.d, 0, b.bf16, 2, nullptr, b.A1};
        note_launch();
        grouped_gemm_simt<<<grid, NTHR, 0, st>>>(g1);
    }
    // dW2 = H^T dY [NE, d_ff, d]; db2 = 1^T dY (fixed-order two-pass column sums)
    if (tcw) {
        // tcgen05 wgrad: padding rows up to the next 64-row K block must be zero
        launch_pad_rows_zero(const_cast<void *>(b.X), b.counts, nseg, b.Cseg, b.d, st);
        launch_pad_rows_zero(const_cast<void *>(b.dY), b.counts, nseg, b.Cseg, b.d, st);
        launch_pad_rows_zero(const_cast<void *>(b.H), b.counts, nseg, b.Cseg, b.d_ff, st);
        launch_pad_rows_zero(b.dZ, b.counts, nseg, b.Cseg, b.d_ff, st);
        cudaError_t e = launch_wgrad_tc(b.H, b.d_ff, b.dY, b.d, b.dW2, b.counts, b.V, b.S, b.e, b.Cseg, b.num_sms, st);
        if (e != cudaSuccess) return e;
    } else {
        WgradArgs w2{b.H, b.dY, b.dW2, b.counts, b.e, b.S, b.Cseg, b.d_ff, b.d, b.bf16};
        note_launch();
        wgrad_simt<<<dim3((b.d + BN - 1) / BN, (b.d_ff + BM - 1) / BM, NE), NTHR, 0, st>>>(w2);
    }
    launch_colsum(b.dY, b.db2, b.colsum_ws, b.counts, NE, b.e, b.S, b.Cseg, b.d, b.bf16, st);
    // dX = dZ W1^T: B operand = W1 [NE, d, d_ff] as [N = d, K = d_ff]
    if (tc) {
        cudaError_t e = launch_ffn_tcgen05_dgrad(b, 2, st);
        if (e != cudaSuccess) return e;
    } else {
        GemmArgs g2{b.dZ, b.W1, nullptr, b.dX, b.counts, nseg, b.e, b.S, b.Cseg, b.d, b.d_ff, 0, b.bf16, 3, nullptr, nullptr};
        note_launch();
        grouped_gemm_simt<<<grid, NTHR, 0, st>>>(g2);
    }
    // dW1 = X^T dZ [NE, d, d_ff]; db1 = 1^T dZ (SIMT path; the tcgen05 dZ GEMM made it above)
    if (tcw) {
        cudaError_t e = launch_wgrad_tc(b.X, b.d, b.dZ, b.d_ff, b.dW1, b.counts, b.V, b.S, b.e, b.Cseg, b.num_sms, st);
        if (e != cudaSuccess) return e;
    } else {
        WgradArgs w1{b.X, b.dZ, b.dW1, b.counts, b.e, b.S, b.Cseg, b.d, b.d_ff, b.bf16};
        note_launch();
        wgrad_simt<<<dim3((b.d_ff + BN - 1) / BN, (b.d + BM - 1) / BM, NE), NTHR, 0, st>>>(w1);
    }
    if (!tc) launch_colsum(b.dZ, b.db1, b.colsum_ws, b.counts, NE, b.e, b.S, b.Cseg, b.d_ff, b.bf16, st);
    return cudaGetLastError();
}

bool ffn_simt_supported(int nseg, int d, int d_ff) {
    return nseg <= MAXSEG && d % BN == 0 && d_ff % BN == 0 && d % BK == 0 && d_ff % BK == 0;
}

}  // namespace smile
