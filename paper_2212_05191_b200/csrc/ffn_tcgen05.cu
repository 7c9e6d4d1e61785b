// ffn_tcgen05.cu -- the grouped expert FFN on Blackwell tensor cores.
//
// Y = GELU(X W1 + b1) W2 + b2 for every resident expert over its capacity-padded
// segments, as two launches of one persistent, warp-specialised grouped GEMM
//     D[rows, N] = A[rows, K] . B[expert][N, K]^T + bias[expert][N]   (+ exact erf GELU)
// with bf16 operands, fp32 accumulation in TMEM and bf16 output (H, then Y).
//
//   warp 0      TMA producer: A (128 x 64) and B (BN x 64) tiles, SWIZZLE_128B, into a
//               4-stage smem ring guarded by full/empty mbarriers
//   warp 1      MMA issuer: one thread issues tcgen05.mma.cta_group::1.kind::f16
//               (M = 128, N = BN, K = 16) into a double-buffered TMEM accumulator
//               (2 x 256 columns) and commits to the empty / tmem_full mbarriers
//   warp 2      TMEM allocator (512 columns)
//   warps 4-11  epilogue: two warps per TMEM lane quadrant, each on half of the columns:
//               tcgen05.ld 32x32b -> +bias -> GELU -> bf16 -> a 32x32 box in smem ->
//               TMA tensor store (partial boxes at a segment's end: masked st.global of
//               the valid rows only); the 8 warps release the accumulator buffer
//
// Work list: tiles of 128 rows of one segment x BN columns, enumerated on the device
// from the segment counts (tiles.cuh), n fastest so the CTAs running concurrently share
// the A tile and the expert's weights in L2.  One CTA per SM (grid = #SMs).
#include "smile_internal.h"
#include "tiles.cuh"

#include <cuda.h>
#include <string.h>

namespace smile {
namespace {

constexpr int BM = 128, BK = 64, STAGES = 4, MAXSEG = 1024;
constexpr int EPI_WARPS = 8;                  // 2 warps per TMEM lane quadrant, split by columns
constexpr int NTHREADS = 128 + 32 * EPI_WARPS;
constexpr int A_BYTES = BM * BK * 2;          // 16 KB
constexpr int B_BYTES_MAX = 256 * BK * 2;     // 32 KB
constexpr int ACC_COLS = 256;                 // TMEM columns per accumulator buffer
constexpr int OUT_BOX_BYTES = 32 * 32 * 2;    // per epilogue warp: 32 rows x 32 bf16 staged for a TMA store

struct TcArgs {
    const float *bias;       // [NE, N]
    __nv_bfloat16 *D;        // [rows_total, N]
    __nv_bfloat16 *D2;       // EPI_BIAS_SAVE: the pre-activation output
    const int32_t *counts;   // [nseg]
    int nseg, e, S;
    int64_t Cseg;
    int N, K, BN;
    int gelu;
    int mode;                  // EPI_* below
    const __nv_bfloat16 *aux;  // EPI_DGELU: the saved pre-activation A1 [rows_total, N]
    int stages;                // smem pipeline depth (3 when two output boxes per warp)
    int *err;
};

// Epilogue modes of the grouped GEMM.
enum { EPI_BIAS = 0,        // D = act(acc + bias), act = GELU when gelu != 0 (forward)
       EPI_BIAS_SAVE = 1,   // D = GELU(acc + bias) and D2 = acc + bias (training forward: H and A1)
       EPI_DGELU = 2,       // D = acc * GELU'(aux) (backward: dZ = dH . GELU'(A1))
       EPI_PLAIN = 3 };     // D = acc (backward: dX)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    for (uint32_t spin = 0;; ++spin) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
        if (ok) return;
        if (spin > (1u << 26)) __trap();   // never hang the GPU: a lost arrival aborts the kernel
    }
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Shared-memory matrix descriptor of a K-major SWIZZLE_128B tile (rows of 64 bf16 =
// 128 B, 8-row atoms 1024 B apart): start>>4, LBO = 16 B (unused for this layout),
// SBO = 1024 B, version 1 (sm_100), layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// kind::f16 instruction descriptor: D = F32, A = B = BF16, both K-major, M = 128, N.
__device__ __forceinline__ uint32_t make_idesc(int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// GELU(z) = z Phi(z) = 0.5 z + 0.5 |z| erf(|z| / sqrt 2) (R21, erf form).  erf by Abramowitz &
// Stegun 7.1.28, 1 - (1 + a1 x + ... + a6 x^6)^-16: |error| <= 1.8e-6 on erf and 8.8e-7 on GELU
// over all z (checked against scipy in fp32 emulation), ~14 instructions with one
// MUFU reciprocal instead of erff's ~30 -- the bf16 H it feeds has a half-ulp of >= 2^-9 |H|.
__device__ __forceinline__ float gelu_erf(float z) {
    const float ax = fabsf(z) * 0.70710678118654752f;
    float p = 4.30638e-5f;
    p = fmaf(p, ax, 2.765672e-4f);
    p = fmaf(p, ax, 1.520143e-4f);
    p = fmaf(p, ax, 9.2705272e-3f);
    p = fmaf(p, ax, 4.22820123e-2f);
    p = fmaf(p, ax, 7.05230784e-2f);
    p = fmaf(p, ax, 1.0f);
    p = p * p;
    p = p * p;
    p = p * p;
    p = p * p;
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(p));
    return fmaf(0.5f * fabsf(z), 1.0f - r, 0.5f * z);
}

// GELU'(z) = Phi(z) + z phi(z), with Phi from the same erf approximation.
__device__ __forceinline__ float gelu_grad(float z) {
    const float ax = fabsf(z) * 0.70710678118654752f;
    float p = 4.30638e-5f;
    p = fmaf(p, ax, 2.765672e-4f);
    p = fmaf(p, ax, 1.520143e-4f);
    p = fmaf(p, ax, 9.2705272e-3f);
    p = fmaf(p, ax, 4.22820123e-2f);
    p = fmaf(p, ax, 7.05230784e-2f);
    p = fmaf(p, ax, 1.0f);
    p = p * p;
    p = p * p;
    p = p * p;
    p = p * p;
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(p));
    const float erf_abs = 1.0f - r;
    const float Phi = 0.5f + 0.5f * copysignf(erf_abs, z);
    return Phi + z * 0.3989422804014327f * __expf(-0.5f * z * z);
}

struct TileInfo {
    int g, mt, nt, rows;
    int64_t a_row, b_row, d_row, expert;
};

__device__ __forceinline__ TileInfo tile_info(const TcArgs &a, const int *s_pref, int tile, int ntn) {
    TileInfo t;
    t.nt = tile % ntn;
    const int mtg = tile / ntn;
    t.g = tile_segment(s_pref, a.nseg, mtg);
    t.mt = mtg - s_pref[t.g];
    const int v = t.g / (a.S * a.e), k = t.g % a.e;
    t.expert = (int64_t)v * a.e + k;
    t.rows = min(BM, a.counts[t.g] - t.mt * BM);
    t.a_row = (int64_t)t.g * a.Cseg + (int64_t)t.mt * BM;
    t.d_row = t.a_row;
    t.b_row = t.expert * a.N + (int64_t)t.nt * a.BN;
    return t;
}

__global__ void __launch_bounds__(NTHREADS, 1)
ffn_gemm_tcgen05(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                 const __grid_constant__ CUtensorMap mapD, const __grid_constant__ CUtensorMap mapD2, TcArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte aligned carve-up: [A stages][B stages][barriers][tmem holder][prefix]
    unsigned char *base = reinterpret_cast<unsigned char *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    unsigned char *sA = base;
    const int STAGES = a.stages;
    const int nbox = a.mode == EPI_BIAS_SAVE ? 2 : 1;
    unsigned char *sB = sA + STAGES * A_BYTES;
    unsigned char *sOut = sB + STAGES * B_BYTES_MAX;                 // EPI_WARPS x nbox x 2 KB
    uint64_t *bars = reinterpret_cast<uint64_t *>(sOut + nbox * EPI_WARPS * OUT_BOX_BYTES);
    uint64_t *full = bars, *empty = bars + STAGES, *tfull = bars + 2 * STAGES, *tempty = bars + 2 * STAGES + 2;
    uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bars + 2 * STAGES + 4);
    int *s_warp = reinterpret_cast<int *>(tmem_holder + 4);
    int *s_pref = s_warp + 32;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(smem_u32(&tfull[s]), 1);
            mbar_init(smem_u32(&tempty[s]), EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapD)) : "memory");
        if (nbox == 2) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapD2)) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_holder))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tile_prefix<BM>(a.counts, a.nseg, s_pref, s_warp);   // ends with __syncthreads
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const int ntn = a.N / a.BN;
    const int total = s_pref[a.nseg] * ntn;
    const int nk = a.K / BK;
    const uint32_t b_bytes = (uint32_t)a.BN * BK * 2;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer ----------------
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
                const TileInfo t = tile_info(a, s_pref, tile, ntn);
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
                    const uint32_t fb = smem_u32(&full[stage]);
                    mbar_arrive_tx(fb, A_BYTES + b_bytes);
                    tma_load_2d(smem_u32(sA + stage * A_BYTES), &mapA, kb * BK, (int)t.a_row, fb);
                    tma_load_2d(smem_u32(sB + stage * B_BYTES_MAX), &mapB, kb * BK, (int)t.b_row, fb);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer (single thread) ----------------
            const uint32_t idesc = make_idesc(a.BN);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
                const int acc = it & 1;
                const uint32_t use = (uint32_t)(it >> 1) & 1;
                mbar_wait(smem_u32(&tempty[acc]), use ^ 1);
                tc_fence_after();
                const uint32_t tmem_d = tmem_base + acc * ACC_COLS;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(smem_u32(&full[stage]), phase);
                    tc_fence_after();
                    const uint64_t ad = sw128_desc(smem_u32(sA + stage * A_BYTES));
                    const uint64_t bd = sw128_desc(smem_u32(sB + stage * B_BYTES_MAX));
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)   // +32 B along K inside the 128 B swizzle atom
                        mma_bf16(tmem_d, ad + (uint64_t)(2 * k), bd + (uint64_t)(2 * k), idesc, (kb | k) ? 1u : 0u);
                    mma_commit(smem_u32(&empty[stage]));
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                mma_commit(smem_u32(&tfull[acc]));
            }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: 8 warps; quadrant q = rows 32q..32q+31 ----------------
        const int q = warp & 3;
        const int half = (warp - 4) >> 2;
        const int row = q * 32 + lane;
        const int nch = a.BN / 32;
        const int c_beg = half ? (nch + 1) / 2 : 0, c_end = half ? nch : (nch + 1) / 2;
        int it = 0;
        for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
            const TileInfo t = tile_info(a, s_pref, tile, ntn);
            const int acc = it & 1;
            mbar_wait(smem_u32(&tfull[acc]), (uint32_t)(it >> 1) & 1);
            tc_fence_after();
            const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * ACC_COLS;
            const bool has_bias = a.mode == EPI_BIAS || a.mode == EPI_BIAS_SAVE;
            const float4 *bias4 = reinterpret_cast<const float4 *>(a.bias + t.expert * a.N + (int64_t)t.nt * a.BN);
            const int64_t dcol0 = (int64_t)t.nt * a.BN;
            __nv_bfloat16 *drow = a.D + (t.d_row + row) * (int64_t)a.N + dcol0;
            unsigned char *box = sOut + (warp - 4) * nbox * OUT_BOX_BYTES;
            const bool full_box = q * 32 + 32 <= t.rows;
            for (int c = c_beg; c < c_end; ++c) {
                float v[32];
                tmem_ld32(tbase + c * 32, v);
                if (has_bias) {
#pragma unroll
                    for (int i4 = 0; i4 < 8; ++i4) {
                        const float4 b = __ldg(bias4 + c * 8 + i4);
                        v[4 * i4] += b.x; v[4 * i4 + 1] += b.y; v[4 * i4 + 2] += b.z; v[4 * i4 + 3] += b.w;
                    }
                }
                uint4 pk[4], pk2[4];
                uint32_t *pw = reinterpret_cast<uint32_t *>(pk);
                uint32_t *pw2 = reinterpret_cast<uint32_t *>(pk2);
                if (a.mode == EPI_BIAS_SAVE) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
                        pw2[i] = *reinterpret_cast<uint32_t *>(&h);
                    }
                }
                if (a.mode == EPI_DGELU && row < t.rows) {
                    const uint4 *ap = reinterpret_cast<const uint4 *>(a.aux + (t.d_row + row) * (int64_t)a.N + dcol0 + c * 32);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint4 u = __ldg(ap + i);
                        const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
                        for (int z = 0; z < 4; ++z) {
                            const float2 f = __bfloat1622float2(h[z]);
                            v[8 * i + 2 * z] *= gelu_grad(f.x);
                            v[8 * i + 2 * z + 1] *= gelu_grad(f.y);
                        }
                    }
                }
                const bool act = (a.mode == EPI_BIAS && a.gelu) || a.mode == EPI_BIAS_SAVE;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    float y0 = v[2 * i], y1 = v[2 * i + 1];
                    if (act) { y0 = gelu_erf(y0); y1 = gelu_erf(y1); }
                    __nv_bfloat162 h = __floats2bfloat162_rn(y0, y1);
                    pw[i] = *reinterpret_cast<uint32_t *>(&h);
                }
                if (full_box) {
                    // stage the 32 x 32 box(es), then TMA tensor stores (full 64 B row segments)
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    __syncwarp();
                    uint4 *srow = reinterpret_cast<uint4 *>(box + lane * 64);
#pragma unroll
                    for (int i = 0; i < 4; ++i) srow[i] = pk[i];
                    if (nbox == 2) {
                        uint4 *srow2 = reinterpret_cast<uint4 *>(box + OUT_BOX_BYTES + lane * 64);
#pragma unroll
                        for (int i = 0; i < 4; ++i) srow2[i] = pk2[i];
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                                         reinterpret_cast<uint64_t>(&mapD)),
                                     "r"((int)dcol0 + c * 32), "r"((int)(t.d_row + q * 32)), "r"(smem_u32(box))
                                     : "memory");
                        if (nbox == 2)
                            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                                             reinterpret_cast<uint64_t>(&mapD2)),
                                         "r"((int)dcol0 + c * 32), "r"((int)(t.d_row + q * 32)),
                                         "r"(smem_u32(box + OUT_BOX_BYTES))
                                         : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                } else if (row < t.rows) {
                    uint4 *dst = reinterpret_cast<uint4 *>(drow + c * 32);
#pragma unroll
                    for (int i = 0; i < 4; ++i) dst[i] = pk[i];
                    if (nbox == 2) {
                        uint4 *dst2 = reinterpret_cast<uint4 *>(a.D2 + (t.d_row + row) * (int64_t)a.N + dcol0 + c * 32);
#pragma unroll
                        for (int i = 0; i < 4; ++i) dst2[i] = pk2[i];
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&tempty[acc]));
        }
    }
    if (warp >= 4 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
    }
}

// ---- host: tensor maps ------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// 2D bf16 row-major [rows, K] map with a (box_cols x box_rows) box, SWIZZLE_128B for the
// 64-column operand boxes, none for the 32 x 32 output boxes.
bool make_map(CUtensorMap *m, const void *ptr, int64_t rows, int64_t K, int box_rows, int box_cols = BK) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, box_cols == BK ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int pick_bn(int N) {
    for (int bn = 256; bn >= 32; bn -= 32)
        if (N % bn == 0) return bn;
    return 0;
}

size_t smem_bytes(int stages, int nbox) {
    return 1024 + stages * (A_BYTES + B_BYTES_MAX) + nbox * EPI_WARPS * OUT_BOX_BYTES + (2 * stages + 4) * 8 + 16 +
           32 * 4 + (MAXSEG + 1) * 4;
}

// One grouped GEMM launch: D[rows, N] = epi(A[rows, K] . B[expert][N, K]^T).
cudaError_t launch_gemm(const void *A, int64_t rows_total, const void *B, int NE, const float *bias, void *D,
                        void *D2, const void *aux, const FfnArgs &f, int N, int K, int mode, int gelu,
                        cudaStream_t st) {
    const int BN = pick_bn(N);
    CUtensorMap mA, mB, mD, mD2;
    if (!make_map(&mA, A, rows_total, K, BM)) return cudaErrorNotSupported;
    if (!make_map(&mB, B, (int64_t)NE * N, K, BN)) return cudaErrorNotSupported;
    if (!make_map(&mD, D, rows_total, N, 32, 32)) return cudaErrorNotSupported;
    mD2 = mD;
    if (D2 && !make_map(&mD2, D2, rows_total, N, 32, 32)) return cudaErrorNotSupported;
    TcArgs a;
    memset(&a, 0, sizeof(a));
    a.bias = bias; a.D = reinterpret_cast<__nv_bfloat16 *>(D); a.D2 = reinterpret_cast<__nv_bfloat16 *>(D2);
    a.counts = f.counts;
    a.nseg = f.V * f.S * f.e; a.e = f.e; a.S = f.S; a.Cseg = f.Cseg; a.N = N; a.K = K; a.BN = BN; a.gelu = gelu;
    a.mode = mode; a.aux = reinterpret_cast<const __nv_bfloat16 *>(aux);
    const int nbox = mode == EPI_BIAS_SAVE ? 2 : 1;
    a.stages = nbox == 2 ? 3 : STAGES;
    a.err = nullptr;
    const size_t smem = smem_bytes(a.stages, nbox);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(ffn_gemm_tcgen05, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes(STAGES, 1));
        attr = true;
    }
    ffn_gemm_tcgen05<<<f.num_sms, NTHREADS, smem, st>>>(mA, mB, mD, mD2, a);
    return cudaGetLastError();
}

}  // namespace

static bool tc_supported(const FfnArgs &f) {
    const int nseg = f.V * f.S * f.e;
    if (!f.bf16 || nseg > MAXSEG || f.d % BK || f.d_ff % BK || !pick_bn(f.d) || !pick_bn(f.d_ff)) return false;
    return (int64_t)nseg * f.Cseg < ((int64_t)1 << 31);
}

cudaError_t launch_ffn_tcgen05(const FfnArgs &f, cudaStream_t st) {
    if (!tc_supported(f)) return cudaErrorNotSupported;
    const int64_t rows_total = (int64_t)f.V * f.S * f.e * f.Cseg;
    const int NE = f.V * f.e;
    cudaError_t e = launch_gemm(f.X, rows_total, f.W1t, NE, f.b1, f.H, nullptr, nullptr, f, f.d_ff, f.d, EPI_BIAS, 1, st);
    if (e != cudaSuccess) return e;
    return launch_gemm(f.H, rows_total, f.W2t, NE, f.b2, f.Y, nullptr, nullptr, f, f.d, f.d_ff, EPI_BIAS, 0, st);
}

// Training forward on tcgen05: GEMM1 also stores the pre-activation A1 (for GELU').
cudaError_t launch_ffn_tcgen05_train(const FfnArgs &f, void *A1, cudaStream_t st) {
    if (!tc_supported(f)) return cudaErrorNotSupported;
    const int64_t rows_total = (int64_t)f.V * f.S * f.e * f.Cseg;
    const int NE = f.V * f.e;
    cudaError_t e = launch_gemm(f.X, rows_total, f.W1t, NE, f.b1, f.H, A1, nullptr, f, f.d_ff, f.d, EPI_BIAS_SAVE, 1, st);
    if (e != cudaSuccess) return e;
    return launch_gemm(f.H, rows_total, f.W2t, NE, f.b2, f.Y, nullptr, nullptr, f, f.d, f.d_ff, EPI_BIAS, 0, st);
}

// Backward data GEMMs on tcgen05 (a17): dZ = (dY W2^T) . GELU'(A1); dX = dZ W1^T.
// W1 [NE, d, d_ff] and W2 [NE, d_ff, d] in their math layouts are the K-major B operands.
cudaError_t launch_ffn_tcgen05_dgrad(const FfnBwdArgs &b, cudaStream_t st) {
    FfnArgs f{};
    f.counts = b.counts; f.V = b.V; f.S = b.S; f.e = b.e; f.Cseg = b.Cseg; f.d = b.d; f.d_ff = b.d_ff; f.bf16 = b.bf16;
    f.num_sms = b.num_sms;
    if (!tc_supported(f)) return cudaErrorNotSupported;
    const int64_t rows_total = (int64_t)f.V * f.S * f.e * f.Cseg;
    const int NE = f.V * f.e;
    cudaError_t e = launch_gemm(b.dY, rows_total, b.W2, NE, nullptr, b.dZ, nullptr, b.A1, f, f.d_ff, f.d, EPI_DGELU, 0, st);
    if (e != cudaSuccess) return e;
    return launch_gemm(b.dZ, rows_total, b.W1, NE, nullptr, b.dX, nullptr, nullptr, f, f.d, f.d_ff, EPI_PLAIN, 0, st);
}

}  // namespace smile
