// wgrad_tcgen05.cu -- weight and bias gradients of the grouped expert FFN (SURVEY §8(a)
// a17, configuration C3) on Blackwell tensor cores.
//
//   dW2[E] = H_E^T dY_E   [d_ff, d]        dW1[E] = X_E^T dZ_E   [d, d_ff]
//   db2[E] = 1^T dY_E     [d]              db1[E] = 1^T dZ_E     [d_ff]
//
// where the rows of expert E are the valid rows of its S capacity-padded segments.  The
// contraction runs over tokens, so both operands are read "transposed": A[m][k] =
// X[row k][col m] and B[n][k] = dZ[row k][col n] are MN-major, which tcgen05 consumes
// directly (instruction-descriptor bits 15/16, MN-major SWIZZLE_128B smem descriptors) --
// no transposed copies.  TMA loads 64-row x 64-column boxes through 3-D tensor maps
// [segment][row][col], so a box never reads past its segment; the rows between a
// segment's count and the next multiple of 64 are zeroed first (pad_rows_zero_kernel),
// since the permutes never write padding rows and 0 * garbage could be NaN.
//
// One persistent, warp-specialised kernel: warp 0 TMA producer (4-stage ring of A 128 x 64
// and B BN x 64 K-blocks), warp 1 single-thread tcgen05.mma issuer (M = 128, N = BN, K = 16
// per instruction, fp32 accumulation in a double-buffered TMEM accumulator), warp 2 TMEM
// allocator, warps 4-7 epilogue (tcgen05.ld -> fp32 dW rows).  Tiles (E, m-tile, n-tile),
// n fastest; the K loop walks every segment of the expert.
//
// Bias gradients: two passes with fixed-order sums (deterministic): per (expert, segment,
// 128-row chunk) column partials, then their sum in chunk order.
#include "smile_internal.h"
#include "tc_util.cuh"

#include <stdlib.h>
#include <string.h>

namespace smile {
namespace {

using namespace tc;

constexpr int WG_BM = 128, WG_BK = 64, WG_STAGES = 4;
constexpr int WG_THREADS = 256;
constexpr int WG_A_BYTES = WG_BM * WG_BK * 2;        // 16 KB: two 64-column boxes
constexpr int WG_BOX_BYTES = 64 * WG_BK * 2;         // 8 KB: one 64 x 64 box
constexpr int WG_MAXSEG_S = 64;                      // segments per expert (S <= world size)
constexpr int COLSUM_ROWS = 128;     // rows per partial: short sequential chains, many blocks

__global__ void pad_rows_zero_kernel(void *buf, const int32_t *counts, int nseg, int64_t Cseg, int cols) {
    // rows [count, min(ceil64(count), Cseg)) of every segment; cols % 8 == 0 (16-byte stores)
    const int g = blockIdx.x;
    if (g >= nseg) return;
    const int cnt = counts[g];
    const int64_t end = ((int64_t)cnt + WG_BK - 1) / WG_BK * WG_BK;
    const int64_t stop = end < Cseg ? end : Cseg;
    const int vec = cols / 8;
    uint4 *base = reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(buf) + (int64_t)g * Cseg * cols);
    const uint4 z = make_uint4(0, 0, 0, 0);
    for (int64_t i = threadIdx.x; i < (stop - cnt) * vec; i += blockDim.x) base[(int64_t)cnt * vec + i] = z;
}

struct WgArgs {
    float *Dw;                 // [NE, M, N]
    const int32_t *counts;     // [nseg]
    int e, S;
    int64_t Cseg;
    int M, N, BN, NE;
};

// CG = 2: a CTA pair (cluster of 2) per 256-row tile of dW, tcgen05.mma.cta_group::2
// issued by the leader; each CTA loads its 128 rows of A and half of B's columns, which
// cuts the bytes each SM receives per MAC by a third (the wgrad GEMMs are bound by that).
template <int CG>
__global__ void __launch_bounds__(WG_THREADS, 1)
wgrad_tcgen05(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, WgArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *base = reinterpret_cast<unsigned char *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int b_bytes = (a.BN / CG / 64) * WG_BOX_BYTES;       // this CTA's share of B per stage
    unsigned char *sA = base;
    unsigned char *sB = sA + WG_STAGES * WG_A_BYTES;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sB + WG_STAGES * b_bytes);
    uint64_t *full = bars, *empty = bars + WG_STAGES, *tfull = bars + 2 * WG_STAGES, *tempty = bars + 2 * WG_STAGES + 2;
    uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bars + 2 * WG_STAGES + 4);
    int *s_kb = reinterpret_cast<int *>(tmem_holder + 4);     // [NE] K-blocks of each expert

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = CG == 2 ? (int)cluster_ctarank() : 0;
    const bool leader = rank == 0;
    const int cid = blockIdx.x / CG, ncl = gridDim.x / CG;
    if (threadIdx.x == 0) {
        for (int s = 0; s < WG_STAGES; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(smem_u32(&tfull[s]), 1);
            mbar_init(smem_u32(&tempty[s]), 4 * CG);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        if (CG == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                             smem_u32(tmem_holder))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                             smem_u32(tmem_holder))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    for (int E = threadIdx.x; E < a.NE; E += blockDim.x) {
        const int v = E / a.e, k = E % a.e;
        int kb = 0;
        for (int s = 0; s < a.S; ++s) kb += (a.counts[(v * a.S + s) * a.e + k] + WG_BK - 1) / WG_BK;
        s_kb[E] = kb;
    }
    tc_fence_before();
    __syncthreads();
    if (CG == 2) cluster_sync_all();          // the leader's barriers exist before any remote arrive
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const int mtn = a.M / (WG_BM * CG), ntn = a.N / a.BN;
    const int total = a.NE * mtn * ntn;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer ----------------
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = cid; tile < total; tile += ncl) {
                const int E = tile / (mtn * ntn), rem = tile % (mtn * ntn);
                const int m0 = (rem / ntn) * WG_BM * CG + rank * WG_BM, n0 = (rem % ntn) * a.BN + rank * (a.BN / CG);
                const int v = E / a.e, k = E % a.e;
                for (int s = 0; s < a.S; ++s) {
                    const int g = (v * a.S + s) * a.e + k;
                    const int cnt = a.counts[g];
                    for (int r0 = 0; r0 < cnt; r0 += WG_BK) {
                        mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
                        const uint32_t fb = smem_u32(&full[stage]);
                        unsigned char *pa = sA + stage * WG_A_BYTES, *pb = sB + stage * b_bytes;
                        if (CG == 1) {
                            mbar_arrive_tx(fb, WG_A_BYTES + b_bytes);
                            tma_load_3d(smem_u32(pa), &mapA, m0, r0, g, fb);
                            tma_load_3d(smem_u32(pa + WG_BOX_BYTES), &mapA, m0 + 64, r0, g, fb);
                            for (int j = 0; j < a.BN / 64; ++j)
                                tma_load_3d(smem_u32(pb + j * WG_BOX_BYTES), &mapB, n0 + 64 * j, r0, g, fb);
                        } else {
                            // the leader's full barrier counts both CTAs' bytes
                            if (leader) mbar_arrive_tx(fb, CG * (WG_A_BYTES + b_bytes));
                            const uint32_t fbl = mapa_shared(fb, 0);
                            tma_load_3d_pair(smem_u32(pa), &mapA, m0, r0, g, fbl);
                            tma_load_3d_pair(smem_u32(pa + WG_BOX_BYTES), &mapA, m0 + 64, r0, g, fbl);
                            for (int j = 0; j < a.BN / CG / 64; ++j)
                                tma_load_3d_pair(smem_u32(pb + j * WG_BOX_BYTES), &mapB, n0 + 64 * j, r0, g, fbl);
                        }
                        if (++stage == WG_STAGES) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {
            // ---------------- MMA issuer: A and B both MN-major ----------------
            // (whole warp, warp-uniform descriptors; one elected lane issues: tc_util.cuh)
            const uint32_t idesc = make_idesc(WG_BM * CG, a.BN) | (1u << 15) | (1u << 16);
            const uint64_t adesc0 = sw128_mn_desc(smem_u32(sA), WG_BOX_BYTES);
            const uint64_t bdesc0 = sw128_mn_desc(smem_u32(sB), WG_BOX_BYTES);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int tile = cid; tile < total; tile += ncl, ++it) {
                const int E = tile / (mtn * ntn);
                const int nk = s_kb[E];
                const int acc = it & 1;
                mbar_wait(smem_u32(&tempty[acc]), ((uint32_t)(it >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t tmem_d = tmem_base + acc * 256;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(smem_u32(&full[stage]), phase);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint64_t ad = adesc0 + (uint64_t)((uint32_t)(stage * WG_A_BYTES) >> 4);
                        const uint64_t bd = bdesc0 + (uint64_t)((uint32_t)(stage * b_bytes) >> 4);
#pragma unroll
                        for (int kk = 0; kk < WG_BK / 16; ++kk) {  // 16 K-rows = two 1024 B swizzle atoms
                            if (CG == 1)
                                mma_bf16(tmem_d, ad + (uint64_t)(kk * 128), bd + (uint64_t)(kk * 128), idesc,
                                         (kb | kk) ? 1u : 0u);
                            else
                                mma_bf16_pair(tmem_d, ad + (uint64_t)(kk * 128), bd + (uint64_t)(kk * 128), idesc,
                                              (kb | kk) ? 1u : 0u);
                        }
                        if (CG == 1) mma_commit(smem_u32(&empty[stage]));
                        else mma_commit_pair(smem_u32(&empty[stage]));
                    }
                    __syncwarp();
                    if (++stage == WG_STAGES) { stage = 0; phase ^= 1; }
                }
                if (elect_one()) {
                    if (CG == 1) mma_commit(smem_u32(&tfull[acc]));
                    else mma_commit_pair(smem_u32(&tfull[acc]));
                }
                __syncwarp();
            }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: thread = row m of the tile ----------------
        const int q = warp & 3;
        const int row = q * 32 + lane;
        int it = 0;
        for (int tile = cid; tile < total; tile += ncl, ++it) {
            const int E = tile / (mtn * ntn), rem = tile % (mtn * ntn);
            const int m0 = (rem / ntn) * WG_BM * CG + rank * WG_BM, n0 = (rem % ntn) * a.BN;
            const bool empty_k = s_kb[E] == 0;                    // no rows: the gradient is 0
            const int acc = it & 1;
            mbar_wait(smem_u32(&tfull[acc]), (uint32_t)(it >> 1) & 1);
            tc_fence_after();
            const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + acc * 256;
            float4 *dst = reinterpret_cast<float4 *>(a.Dw + ((int64_t)E * a.M + m0 + row) * a.N + n0);
            for (int c = 0; c < a.BN / 32; ++c) {
                float v[32];
                tmem_ld32(tb + c * 32, v);
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    dst[c * 8 + i] = empty_k ? make_float4(0.f, 0.f, 0.f, 0.f)
                                             : make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (CG == 1) mbar_arrive(smem_u32(&tempty[acc]));
                else mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
            }
        }
    }
    __syncthreads();
    if (CG == 2) cluster_sync_all();
    if (warp == 2) {
        tc_fence_after();
        if (CG == 2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
    }
}

// ---- bias gradients -----------------------------------------------------------------
struct ColsumArgs {
    const void *B; float *part; float *db; const int32_t *counts;
    int e, S; int64_t Cseg; int N, NE, nch; int bf16;
};

// part[E][s * nch + c][n] = sum of rows [128 c, 128 c + 128) of segment s (valid rows
// only).  A thread owns 8 (bf16) / 4 (fp32) adjacent columns: 16-byte loads, 4 rows in
// flight; rows summed in order (deterministic).
__global__ void colsum_partial_kernel(ColsumArgs a) {
    const int epv = a.bf16 ? 8 : 4;
    const int n0 = (blockIdx.x * blockDim.x + threadIdx.x) * epv;
    const int E = blockIdx.y, sc = blockIdx.z;
    const int s = sc / a.nch, c = sc % a.nch;
    if (n0 >= a.N) return;
    const int v = E / a.e, k = E % a.e;
    const int g = (v * a.S + s) * a.e + k;
    const int cnt = a.counts[g];
    const int r0 = c * COLSUM_ROWS, r1 = min(cnt, r0 + COLSUM_ROWS);
    const int64_t base = (int64_t)g * a.Cseg;
    const int64_t esz = a.bf16 ? 2 : 4;
    const char *B = static_cast<const char *>(a.B);
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.f;
    for (int r = r0; r < r1; r += 4) {
        uint4 u[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            u[q] = r + q < r1 ? *reinterpret_cast<const uint4 *>(B + ((base + r + q) * a.N + n0) * esz)
                              : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (a.bf16) {
                const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u[q]);
#pragma unroll
                for (int z = 0; z < 4; ++z) {
                    const float2 f = __bfloat1622float2(h[z]);
                    acc[2 * z] += f.x;
                    acc[2 * z + 1] += f.y;
                }
            } else {
                const float *f = reinterpret_cast<const float *>(&u[q]);
#pragma unroll
                for (int z = 0; z < 4; ++z) acc[z] += f[z];
            }
        }
    }
    float *dst = a.part + ((int64_t)E * a.S * a.nch + sc) * a.N + n0;
    for (int i = 0; i < epv; ++i) dst[i] = acc[i];
}

__global__ void colsum_reduce_kernel(ColsumArgs a) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    const int E = blockIdx.y;
    if (n >= a.N) return;
    float acc = 0.f;
    for (int sc = 0; sc < a.S * a.nch; ++sc) acc += a.part[((int64_t)E * a.S * a.nch + sc) * a.N + n];
    a.db[(int64_t)E * a.N + n] = acc;
}

int pick_wg_bn(int N) {
    for (int bn = 256; bn >= 64; bn -= 64)
        if (N % bn == 0) return bn;
    return 0;
}

}  // namespace

size_t colsum_ws_bytes(int NE, int S, int64_t Cseg, int maxN) {
    // room for either layout: 128-row chunk partials (launch_colsum) or 32-row strip
    // partials of the dZ GEMM's epilogue (launch_colsum_strips)
    const int64_t nstr = (Cseg + 31) / 32;
    return (size_t)NE * S * (nstr > 0 ? nstr : 1) * maxN * 4;
}

namespace {
// Block (32 columns, expert E): warp w sums strips u = w, w + 8, ... of every segment of E
// in order (4 loads in flight), then the 8 warp sums are added in warp order.
__global__ void __launch_bounds__(256) colsum_strip_reduce_kernel(const float *__restrict__ part, float *db,
                                                                  const int32_t *counts, int e, int S, int nstr,
                                                                  int N) {
    __shared__ float s_w[8][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int n = blockIdx.x * 32 + lane, E = blockIdx.y;
    const int v = E / e, k = E % e;
    float acc = 0.f;
    if (n < N)
        for (int s = 0; s < S; ++s) {
            const int g = (v * S + s) * e + k;
            const int ns = (counts[g] + 31) / 32;
            const float *p = part + (int64_t)g * nstr * N + n;
            int u = w;
            for (; u + 24 < ns; u += 32) {
                const float a0 = p[(int64_t)u * N], a1 = p[(int64_t)(u + 8) * N];
                const float a2 = p[(int64_t)(u + 16) * N], a3 = p[(int64_t)(u + 24) * N];
                acc += a0; acc += a1; acc += a2; acc += a3;
            }
            for (; u < ns; u += 8) acc += p[(int64_t)u * N];
        }
    s_w[w][lane] = acc;
    __syncthreads();
    if (w == 0 && n < N) {
        float t = 0.f;
        for (int i = 0; i < 8; ++i) t += s_w[i][lane];
        db[(int64_t)E * N + n] = t;
    }
}
}  // namespace

void launch_colsum_strips(const float *part, float *db, const int32_t *counts, int NE, int e, int S, int nstr, int N,
                          cudaStream_t st) {
    note_launch();
    colsum_strip_reduce_kernel<<<dim3((N + 31) / 32, NE), 256, 0, st>>>(part, db, counts, e, S, nstr, N);
}

void launch_colsum(const void *B, float *db, float *part, const int32_t *counts, int NE, int e, int S, int64_t Cseg,
                   int N, int bf16, cudaStream_t st) {
    ColsumArgs a{B, part, db, counts, e, S, Cseg, N, NE, (int)((Cseg + COLSUM_ROWS - 1) / COLSUM_ROWS), bf16};
    if (a.nch < 1) a.nch = 1;
    note_launch();
    const int per_blk = 128 * (bf16 ? 8 : 4);
    colsum_partial_kernel<<<dim3((N + per_blk - 1) / per_blk, NE, S * a.nch), 128, 0, st>>>(a);
    note_launch();
    colsum_reduce_kernel<<<dim3((N + 255) / 256, NE), 256, 0, st>>>(a);
}

bool wgrad_tc_supported(int bf16, int d, int d_ff, int S) {
    return bf16 && d % WG_BM == 0 && d_ff % WG_BM == 0 && pick_wg_bn(d) && pick_wg_bn(d_ff) && S <= WG_MAXSEG_S &&
           encode_fn() != nullptr;
}

// Dw[E] = A_E^T B_E over the experts' valid rows; A, B [V, S, e, Cseg, M|N] bf16.
cudaError_t launch_wgrad_tc(const void *A, int M, const void *B, int N, float *Dw, const int32_t *counts, int V, int S,
                            int e, int64_t Cseg, int num_sms, cudaStream_t st) {
    const int nseg = V * S * e, NE = V * e;
    const int BN = pick_wg_bn(N);
    CUtensorMap mA, mB;           // 64 x 64 boxes: A (M-major) two per CTA, B (N-major) BN / CG / 64 per CTA
    if (!make_map_3d(&mA, A, nseg, Cseg, M, WG_BK)) return cudaErrorNotSupported;
    if (!make_map_3d(&mB, B, nseg, Cseg, N, WG_BK)) return cudaErrorNotSupported;
    WgArgs a;
    memset(&a, 0, sizeof(a));
    a.Dw = Dw; a.counts = counts; a.e = e; a.S = S; a.Cseg = Cseg; a.M = M; a.N = N; a.BN = BN; a.NE = NE;
    // CTA pairs when the 256-row tiles divide M and half of BN is whole 64-column boxes
    const char *ep = getenv("SMILE_WGRAD_CTA_PAIR");
    const int CG = (!(ep && ep[0] == '0') && M % (2 * WG_BM) == 0 && (BN / 2) % 64 == 0 && num_sms >= 2) ? 2 : 1;
    const size_t smem = 1024 + WG_STAGES * (WG_A_BYTES + (BN / CG / 64) * WG_BOX_BYTES) + (2 * WG_STAGES + 4) * 8 + 16 +
                        (size_t)NE * 4;
    const int total = NE * (M / (WG_BM * CG)) * (N / BN);
    note_launch();
    if (CG == 1) {
        static bool attr1 = false;
        if (!attr1) {
            cudaFuncSetAttribute(wgrad_tcgen05<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
            attr1 = true;
        }
        wgrad_tcgen05<1><<<total < num_sms ? total : num_sms, WG_THREADS, smem, st>>>(mA, mB, a);
        return cudaGetLastError();
    }
    static bool attr2 = false;
    if (!attr2) {
        cudaFuncSetAttribute(wgrad_tcgen05<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr2 = true;
    }
    const int grid = 2 * (total < num_sms / 2 ? total : num_sms / 2);
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(WG_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = 2;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, wgrad_tcgen05<2>, mA, mB, a);
}

void launch_pad_rows_zero(void *buf, const int32_t *counts, int nseg, int64_t Cseg, int cols, cudaStream_t st) {
    note_launch();
    pad_rows_zero_kernel<<<nseg, 256, 0, st>>>(buf, counts, nseg, Cseg, cols);
}

}  // namespace smile
