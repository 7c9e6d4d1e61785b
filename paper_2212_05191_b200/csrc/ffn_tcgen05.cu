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
#include "tc_util.cuh"

#include <cuda.h>
#include <stdlib.h>
#include <string.h>

namespace smile {
namespace {

using namespace tc;

constexpr int BM = 128, BK = 64, MAXSEG = 1024;
// Epilogue warps: EPI_WARPS / 4 per TMEM lane quadrant, splitting the tile's columns.  8
// measured faster than round 1's 16 (same box: C5 FFN 3.12-3.13 vs 3.37-3.46 ms, C2 GEMM 1
// 547 vs 559 us; 12 in between; profiles/r02_ffn_c5.md) -- fewer warps competing with the
// producer / MMA warps for issue slots and with the MMAs for TMEM / shared-memory bandwidth.
// The dZ epilogue (EPI_DGELU: saved GELU' loads, the product, the db1 column sums) keeps 16:
// with 8 the C3 backward measured 1-3 % slower.
#ifndef SMILE_FFN_EPI_WARPS
#define SMILE_FFN_EPI_WARPS 8
#endif
constexpr int epi_warps(int ek) { return ek == 2 ? 16 : SMILE_FFN_EPI_WARPS; }
constexpr int nthreads(int ek) { return 128 + 32 * epi_warps(ek); }
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
    const __nv_bfloat16 *aux;  // EPI_DGELU: the saved GELU'(A1) [rows_total, N]
    int stages;                // smem pipeline depth
    int tma_store;             // 1: full 32 x 32 boxes leave through smem + TMA; 0: st.global from registers
    int box64;                 // 1: 32 x 64 boxes (two chunks per TMA store; every warp owns 2k chunks)
    float *colsum;             // EPI_DGELU: per-strip column sums of D (fp32, before rounding):
                               // colsum[(seg * nstr + strip) * N + n], or nullptr
    int nstr;                  // strips per segment, ceil(Cseg / 32)
    // GEMM 2 in the peer-store exchange: each output row goes straight to its intermediate's
    // ret1 (row rrow[row] of process (rank0 + v) / m * m + l's workspace), not to D
    char *const *rbases;
    const int32_t *rrow;
    int64_t roff_ret1;
    int rrank0, rm, rV;
    // ... and, with the layer output bound, rows whose source rank is in this process too go
    // to out[t] as bf16(gate[t] * bf16(y)) (the level-1 combine's arithmetic, R24)
    char *out;
    const float *gate;
    const int32_t *rtok2;
    int64_t T, C1;
    int n;
    int flat_out;              // FLAT: segment l of an expert holds source rank l's rows; rows of
                               // in-process sources go to out[t] as bf16(p[t] * bf16(y))
    int diag;                  // measurement only (SMILE_FFN_DIAG; wrong results): 1 no activation,
                               // 2 no stores, 4 no TMEM reads / epilogue math (release only),
                               // 8 TMA stores into rows [0, 1024) only (L2-resident)
    int *err;
    unsigned long long *trace;   // SMILE_TRACE=ffn1 / ffn2 timeline (smile_internal.h), or null
};

// Epilogue modes of the grouped GEMM.
enum { EPI_BIAS = 0,        // D = act(acc + bias), act = GELU when gelu != 0 (forward)
       EPI_BIAS_SAVE = 1,   // D = GELU(acc + bias) and D2 = GELU'(acc + bias) (training forward:
                            // H and the activation derivative, sharing one erf evaluation)
       EPI_DGELU = 2,       // D = acc * aux (backward: dZ = dH . GELU'(A1), aux = saved GELU'(A1))
       EPI_PLAIN = 3 };     // D = acc (backward: dX)

// GELU(z) = z Phi(z) = 0.5 z + 0.5 |z| erf(|z| / sqrt 2) (R21, erf form).  erf by Abramowitz &
// Stegun 7.1.28, 1 - (1 + a1 x + ... + a6 x^6)^-16: |error| <= 1.8e-6 on erf and 8.8e-7 on GELU
// over all z (checked against scipy in fp32 emulation), with one MUFU reciprocal
// instead of erff's ~30 instructions -- the bf16 H it feeds has a half-ulp of >= 2^-9 |H|.
// Evaluated on pairs of values with Blackwell's packed fp32x2 pipe (FFMA2 / FMUL2: two
// lanes of fp32 arithmetic per instruction, identical rounding per lane), which halves
// the epilogue's ALU work -- the bias + GELU epilogue of the first FFN GEMM is otherwise
// slower than its MMAs.  The polynomial is evaluated directly in |z| with the
// coefficients a_i / sqrt(2)^i.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pack2(float a, float b) {
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void unpack2(f32x2 r, float &a, float &b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); }
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
    f32x2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
    f32x2 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f32x2 splat2(float a) { return pack2(a, a); }

__device__ __forceinline__ f32x2 gelu_erf2(f32x2 z) {
    const f32x2 az = z & 0x7fffffff7fffffffull;
    // a_i / sqrt(2)^i, a_i of A&S 7.1.28
    f32x2 p = splat2(4.30638e-5f * 0.125f);
    p = fma2(p, az, splat2(2.765672e-4f * 0.17677669529663688f));
    p = fma2(p, az, splat2(1.520143e-4f * 0.25f));
    p = fma2(p, az, splat2(9.2705272e-3f * 0.35355339059327373f));
    p = fma2(p, az, splat2(4.22820123e-2f * 0.5f));
    p = fma2(p, az, splat2(7.05230784e-2f * 0.70710678118654752f));
    p = fma2(p, az, splat2(1.0f));
    p = mul2(p, p);
    p = mul2(p, p);
    p = mul2(p, p);
    p = mul2(p, p);
    float p0, p1, r0, r1;
    unpack2(p, p0, p1);
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(p0));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(p1));
    const f32x2 erfa = fma2(pack2(r0, r1), splat2(-1.0f), splat2(1.0f));   // erf(|z| / sqrt 2)
    return mul2(fma2(az, erfa, z), splat2(0.5f));                          // (z + |z| erf) / 2
}

// GELU(z) and GELU'(z) = Phi(z) + z phi(z) on a pair from one erf evaluation (the training
// forward saves GELU' for the backward's dZ): Phi from the same erf approximation, phi(z) =
// exp(-z^2 / 2) / sqrt(2 pi) via ex2.approx (|error| <= 9e-7 on GELU').
__device__ __forceinline__ void gelu_and_grad2(f32x2 z, f32x2 &g, f32x2 &gp) {
    const f32x2 az = z & 0x7fffffff7fffffffull;
    f32x2 p = splat2(4.30638e-5f * 0.125f);
    p = fma2(p, az, splat2(2.765672e-4f * 0.17677669529663688f));
    p = fma2(p, az, splat2(1.520143e-4f * 0.25f));
    p = fma2(p, az, splat2(9.2705272e-3f * 0.35355339059327373f));
    p = fma2(p, az, splat2(4.22820123e-2f * 0.5f));
    p = fma2(p, az, splat2(7.05230784e-2f * 0.70710678118654752f));
    p = fma2(p, az, splat2(1.0f));
    p = mul2(p, p);
    p = mul2(p, p);
    p = mul2(p, p);
    p = mul2(p, p);
    float p0, p1, r0, r1;
    unpack2(p, p0, p1);
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(p0));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(p1));
    f32x2 erfa = fma2(pack2(r0, r1), splat2(-1.0f), splat2(1.0f));        // erf(|z| / sqrt 2)
    g = mul2(fma2(az, erfa, z), splat2(0.5f));                             // (z + |z| erf) / 2
    erfa |= z & 0x8000000080000000ull;                                     // erf(z / sqrt 2)
    const f32x2 Phi = fma2(erfa, splat2(0.5f), splat2(0.5f));
    const f32x2 ex = mul2(mul2(z, z), splat2(-0.72134752044448170f));
    float e0, e1;
    unpack2(ex, e0, e1);
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(e0));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(e1));
    gp = fma2(mul2(z, splat2(0.3989422804014327f)), pack2(e0, e1), Phi);
}

// Column sums of a warp's 32 x 32 tile (lane = row): 31 shuffles, after which lane j holds
// the sum of column j in v[0].  Fixed order (deterministic).
__device__ __forceinline__ void transpose_reduce32(float (&v)[32], int lane) {
#pragma unroll
    for (int h = 16; h >= 1; h >>= 1) {
        const bool up = (lane & h) != 0;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const float send = up ? v[i] : v[i + h];
            const float keep = up ? v[i + h] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, h);
        }
    }
}

struct TileInfo {
    int nt, E, u0;            // n-tile, expert, first strip of this CTA
    int64_t b_row;
};

// Tile `tile` of the work list: 4 * CG * NSUB strips (32 rows each) of one expert x BN
// columns.  With NSUB = 2 a CTA pair computes two M = 256 sub-tiles (consecutive 8-strip
// M-tiles of the expert) that share the N-tile: `sub` selects one.
// For a CTA pair, `rank` selects this CTA's 4 strips (its 128 rows of the M = 256 MMA)
// and its BN/2-row half of B.  Strip u0 + j of the expert goes to TMEM lanes 32j..32j+31;
// a missing strip (the expert's last tile) has 0 rows and points at row 0 (loaded,
// computed, never stored).
template <int CG, int NSUB, int MC = 0>
__device__ __forceinline__ TileInfo tile_info(const TcArgs &a, const int *s_pref, int tile, int ntn, int rank,
                                              int sub) {
    TileInfo t;
    if (MC) {
        // A-multicast cluster (CG = 1): work item `tile` = (M-tile, pair of N-tiles); cluster
        // rank r takes N-tile 2 p + r (>= ntn: a dummy that only shares its half of A)
        const int ntp = (ntn + 1) >> 1;
        t.nt = 2 * (tile % ntp) + rank;
        const int mtg = tile / ntp;
        const int NE = a.nseg / a.S;
        t.E = tile_segment(s_pref, NE, mtg);
        t.u0 = (mtg - s_pref[t.E]) * 4;
        t.b_row = (int64_t)t.E * a.N + (int64_t)t.nt * a.BN;
        return t;
    }
    t.nt = tile % ntn;
    const int mtg = tile / ntn;
    const int NE = a.nseg / a.S;
    t.E = tile_segment(s_pref, NE, mtg);
    t.u0 = (((mtg - s_pref[t.E]) * NSUB + sub) * CG + rank) * 4;
    t.b_row = (int64_t)t.E * a.N + (int64_t)t.nt * a.BN + rank * (a.BN / CG);
    return t;
}

// CG = 1: one CTA per tile (M = 128).  CG = 2: a CTA pair (cluster of 2) per tile
// (M = 256, tcgen05.mma.cta_group::2 issued by the leader), each CTA loading half of A
// and half of B, which halves the shared-memory operand traffic per SM.
// NSUB = 2 (CG = 2): every stage holds two A tiles and one B tile; the two sub-tiles'
// accumulators fill TMEM (2 x 256 columns), so each B byte delivered from L2 feeds twice
// the MACs: 24 instead of 32 KB per CTA per 128 x 256 x 64 MACs.  The price is the
// double-buffered accumulator: the epilogue drains sub-tile 0 first and releases it, and
// the next tile's MMAs run the first K blocks on sub-tile 0 alone until sub-tile 1 is
// drained too.  Measured slower at C2 (GEMM1 705 vs 572 us, GEMM2 449 vs 455 us: the main
// loop is at the tensor peak already; profiles/r01_ffn_epilogue_diagnostics.md), so opt-in.
// EK: epilogue kind, one instantiation each so the forward kernel carries no backward
// registers: 0 = EPI_BIAS / EPI_PLAIN, 1 = EPI_BIAS_SAVE, 2 = EPI_DGELU.
// MC = 1 (CG = 1, NSUB = 1, forward): clusters of 2 CTAs computing two N-tiles of the same
// 128-row M-tile; each CTA TMA-loads 2 of the tile's 4 A strips multicast into both CTAs,
// so A crosses L2 -> SM once per pair of N-tiles (C5: the operand traffic from L2 bounds
// the 128-row tiles; r02_ffn_c5.md).  A stage is refilled only after both CTAs' MMAs have
// released it (each commit multicasts to both CTAs' empty barrier, count 2).
template <int CG, int NSUB, int EK, int MC = 0>
__global__ void __launch_bounds__(nthreads(EK), 1)
ffn_gemm_tcgen05(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapA128,
                 const __grid_constant__ CUtensorMap mapB,
                 const __grid_constant__ CUtensorMap mapD, const __grid_constant__ CUtensorMap mapD2, TcArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    pdl_wait();
    // 1024-byte aligned carve-up: [A stages][B stages][out boxes][barriers][tmem holder][prefix]
    unsigned char *base = reinterpret_cast<unsigned char *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    unsigned char *sA = base;
    const int STAGES = a.stages;
    constexpr int nbox = EK == 1 ? 2 : 1;
    const int b_stage_bytes = B_BYTES_MAX / CG;
    constexpr int A_STAGE = NSUB * A_BYTES;                           // NSUB A tiles per stage
    unsigned char *sB = sA + STAGES * A_STAGE;
    constexpr int EPI_WARPS = epi_warps(EK);
    unsigned char *sOut = sB + STAGES * b_stage_bytes;                // EPI_WARPS x nbox x 2 KB
    uint64_t *bars = reinterpret_cast<uint64_t *>(
        sOut + (a.tma_store ? nbox * EPI_WARPS * OUT_BOX_BYTES * (a.box64 ? 2 : 1) : 0));
    uint64_t *full = bars, *empty = bars + STAGES, *tfull = bars + 2 * STAGES, *tempty = bars + 2 * STAGES + 2;
    uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bars + 2 * STAGES + 4);
    int *s_warp = reinterpret_cast<int *>(tmem_holder + 4);
    int *s_pref = s_warp + 32;
    int *s_cnt = s_pref + a.nseg + 1;                                 // [nseg] segment row counts

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    static_assert(!MC || (CG == 1 && NSUB == 1), "A multicast: single-CTA tiles only");
    constexpr int CS = MC ? 2 : CG;                             // cluster size
    const int rank = CS > 1 ? (int)cluster_ctarank() : 0;
    const bool leader = MC ? true : rank == 0;                  // this CTA issues its own MMAs
    const uint32_t lead = 0;                                    // cluster rank of the pair's leader
    const int cid = blockIdx.x / CS, ncl = gridDim.x / CS;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), MC ? 2 : 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(smem_u32(&tfull[s]), 1);
            mbar_init(smem_u32(&tempty[s]), CG * EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA128)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapD)) : "memory");
        if (nbox == 2) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapD2)) : "memory");
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
    for (int g = threadIdx.x; g < a.nseg; g += blockDim.x) s_cnt[g] = a.counts[g];
    __syncthreads();
    expert_tile_prefix<4 * CG * NSUB>(s_cnt, a.nseg / a.S, a.S, a.e, s_pref, s_warp);   // ends with __syncthreads
    if (CS > 1) cluster_sync_all();                          // peer barriers initialised before any remote arrive
    tc_fence_after();
    trace_begin(a.trace);
    const uint32_t tmem_base = *tmem_holder;
    const int ntn = a.N / a.BN;
    const int total = s_pref[a.nseg / a.S] * (MC ? (ntn + 1) >> 1 : ntn);
    const int nk = a.K / BK;
    const uint32_t b_bytes = (uint32_t)(a.BN / CG) * BK * 2;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer (both CTAs of a pair) ----------------
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = cid; tile < total; tile += ncl) {
                // A: one 128-row box when a sub-tile's 4 strips are consecutive rows (fewer
                // TMA requests), else four
                // 32-row strip boxes (4 KB each, stacked = the same SW128 tile); rows
                // resolved once per tile
                int srow[NSUB][4];
                bool contig[NSUB];
                int64_t b_row = 0;
#pragma unroll
                for (int u = 0; u < NSUB; ++u) {
                    const TileInfo t = tile_info<CG, NSUB, MC>(a, s_pref, tile, ntn, rank, u);
                    b_row = t.b_row;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        int64_t r;
                        int nr;
                        expert_strip(s_cnt, t.E, a.S, a.e, a.Cseg, t.u0 + j, r, nr);
                        srow[u][j] = (int)r;
                    }
                    contig[u] = srow[u][1] == srow[u][0] + 32 && srow[u][2] == srow[u][0] + 64 &&
                                srow[u][3] == srow[u][0] + 96;
                }
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
                    const uint32_t fb = smem_u32(&full[stage]);
                    unsigned char *sAs = sA + stage * A_STAGE;
                    if (MC) {
                        // strips 2 rank, 2 rank + 1 of the tile into both CTAs (the peer sends the
                        // other two); this CTA's own B
                        mbar_arrive_tx(fb, A_STAGE + b_bytes);
#pragma unroll
                        for (int j = 2 * rank; j < 2 * rank + 2; ++j)
                            tma_load_2d_mc(smem_u32(sAs + j * (A_BYTES / 4)), &mapA, kb * BK, srow[0][j], fb, (uint16_t)3);
                        tma_load_2d(smem_u32(sB + stage * b_stage_bytes), &mapB, kb * BK, (int)b_row, fb);
                    } else if (CG == 1) {
                        mbar_arrive_tx(fb, A_STAGE + b_bytes);
#pragma unroll
                        for (int u = 0; u < NSUB; ++u) {
                            if (contig[u])
                                tma_load_2d(smem_u32(sAs + u * A_BYTES), &mapA128, kb * BK, srow[u][0], fb);
                            else
                                for (int j = 0; j < 4; ++j)
                                    tma_load_2d(smem_u32(sAs + u * A_BYTES + j * (A_BYTES / 4)), &mapA, kb * BK,
                                                srow[u][j], fb);
                        }
                        tma_load_2d(smem_u32(sB + stage * b_stage_bytes), &mapB, kb * BK, (int)b_row, fb);
                    } else {
                        // the leader's full barrier counts the bytes of both CTAs' loads
                        if (leader) mbar_arrive_tx(fb, CG * (A_STAGE + b_bytes));
                        const uint32_t fbl = mapa_shared(fb, lead);
#pragma unroll
                        for (int u = 0; u < NSUB; ++u) {
                            if (contig[u])
                                tma_load_2d_pair(smem_u32(sAs + u * A_BYTES), &mapA128, kb * BK, srow[u][0], fbl);
                            else
                                for (int j = 0; j < 4; ++j)
                                    tma_load_2d_pair(smem_u32(sAs + u * A_BYTES + j * (A_BYTES / 4)), &mapA,
                                                     kb * BK, srow[u][j], fbl);
                        }
                        tma_load_2d_pair(smem_u32(sB + stage * b_stage_bytes), &mapB, kb * BK, (int)b_row, fbl);
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
            trace_clock(a.trace, 5);
        }
    } else if (warp == 1) {
        if (leader) {
            // ---------------- MMA issuer (warp 1 of the leader) ----------------
            // The whole warp runs the loop so descriptors and loop state stay warp-uniform
            // (uniform registers; a single-lane loop pays a register-to-uniform broadcast loop
            // per MMA), and one elected lane issues the MMAs and commits.
            const uint32_t idesc = make_idesc(BM * CG, a.BN);
            const uint64_t adesc0 = sw128_desc(smem_u32(sA)), bdesc0 = sw128_desc(smem_u32(sB));
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            // the 4 K = 16 MMAs of one K block of sub-tile / buffer `acc` on stage `st`
            // (elected lane only)
            auto kblock = [&](int st, int u, int acc, bool first) {
                const uint32_t tmem_d = tmem_base + acc * ACC_COLS;
                const uint64_t ad = adesc0 + (uint64_t)((uint32_t)(st * A_STAGE + u * A_BYTES) >> 4);
                const uint64_t bd = bdesc0 + (uint64_t)((uint32_t)(st * b_stage_bytes) >> 4);
#pragma unroll
                for (int k = 0; k < BK / 16; ++k) {   // +32 B along K inside the 128 B swizzle atom
                    const uint32_t accum = (first && k == 0) ? 0u : 1u;
                    if (CG == 1) mma_bf16(tmem_d, ad + (uint64_t)(2 * k), bd + (uint64_t)(2 * k), idesc, accum);
                    else mma_bf16_pair(tmem_d, ad + (uint64_t)(2 * k), bd + (uint64_t)(2 * k), idesc, accum);
                }
            };
            auto release = [&](uint64_t *bar) {
                if (CG == 1) mma_commit(smem_u32(bar));
                else mma_commit_pair(smem_u32(bar), (uint16_t)3);
            };
            auto release_stage = [&](uint64_t *bar) {    // a smem stage: both CTAs' with A multicast
                if (MC) mma_commit_mc(smem_u32(bar), (uint16_t)3);
                else release(bar);
            };
            for (int tile = cid; tile < total; tile += ncl, ++it) {
                if (NSUB == 1) {
                    // double-buffered accumulator: tile `it` uses buffer it & 1
                    const int acc = it & 1;
                    mbar_wait(smem_u32(&tempty[acc]), ((uint32_t)(it >> 1) & 1) ^ 1);
                    tc_fence_after();
                    if (lane == 0 && it < 240) trace_clock(a.trace, 8 + 2 * it);
                    for (int kb = 0; kb < nk; ++kb) {
                        mbar_wait(smem_u32(&full[stage]), phase);
                        tc_fence_after();
                        if (elect_one()) {
                            kblock(stage, 0, acc, kb == 0);
                            release_stage(&empty[stage]);
                        }
                        __syncwarp();
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                    if (elect_one()) release(&tfull[acc]);
                    __syncwarp();
                    if (lane == 0 && it < 240) trace_clock(a.trace, 9 + 2 * it);
                } else {
                    // sub-tile u accumulates in buffer u; both are drained after every tile.
                    // The first P K blocks go to sub-tile 0 alone (their stages stay held)
                    // while the epilogue still drains sub-tile 1; then sub-tile 1 catches up.
                    const uint32_t par = ((uint32_t)it & 1) ^ 1;
                    const int P = min(nk, STAGES);
                    mbar_wait(smem_u32(&tempty[0]), par);
                    tc_fence_after();
                    const int st0 = stage;
                    const uint32_t ph0 = phase;
                    for (int kb = 0; kb < P; ++kb) {
                        mbar_wait(smem_u32(&full[stage]), phase);
                        tc_fence_after();
                        if (elect_one()) kblock(stage, 0, 0, kb == 0);
                        __syncwarp();
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                    mbar_wait(smem_u32(&tempty[1]), par);
                    tc_fence_after();
                    stage = st0;
                    phase = ph0;
                    for (int kb = 0; kb < P; ++kb) {
                        if (elect_one()) {
                            kblock(stage, 1, 1, kb == 0);
                            release(&empty[stage]);
                        }
                        __syncwarp();
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                    for (int kb = P; kb < nk; ++kb) {
                        mbar_wait(smem_u32(&full[stage]), phase);
                        tc_fence_after();
                        if (elect_one()) {
                            kblock(stage, 0, 0, false);
                            kblock(stage, 1, 1, false);
                            release(&empty[stage]);
                        }
                        __syncwarp();
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                    if (elect_one()) release(&tfull[0]);
                    __syncwarp();
                }
            }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: EPI_WARPS warps ----------------
        // Warp w reads TMEM lane quadrant q = w & 3 (the tile's strip q) and column group
        // h = (w - 4) >> 2 of EPI_WARPS / 4, in 32-column chunks: tcgen05.ld -> bias / GELU
        // in packed fp32x2 -> bf16 -> a 32 x 32 SWIZZLE_64B box in smem -> one TMA tensor
        // store.
        const int q = warp & 3;
        const int h = (warp - 4) >> 2;
        constexpr int ngc = EPI_WARPS / 4;                  // column groups per quadrant
        const int nch = a.BN / 32;
        const int c_beg = (h * nch) / ngc, c_end = ((h + 1) * nch) / ngc;
        int it = 0;
        unsigned char *box = sOut + (warp - 4) * nbox * OUT_BOX_BYTES * (a.box64 ? 2 : 1);
        for (int tile = cid, sub = 0; tile < total;) {
            const TileInfo t = tile_info<CG, NSUB, MC>(a, s_pref, tile, ntn, rank, sub);
            const bool nt_ok = !MC || t.nt < ntn;                 // MC: a dummy N-tile stores nothing
            const int acc = NSUB == 2 ? sub : it & 1;
            const bool has_bias = a.mode == EPI_BIAS || a.mode == EPI_BIAS_SAVE;
            const bool act = ((a.mode == EPI_BIAS && a.gelu) || a.mode == EPI_BIAS_SAVE) && !(a.diag & 1);
            constexpr bool dgelu = EK == 2;                 // EPI_DGELU / EPI_BIAS_SAVE: own instantiations
            const float4 *bias4 = reinterpret_cast<const float4 *>(a.bias + (int64_t)t.E * a.N + (int64_t)(nt_ok ? t.nt : 0) * a.BN);
            const int64_t dcol0 = (int64_t)t.nt * a.BN;
            int64_t d_row;                                  // this warp's strip
            int srows;
            expert_strip(s_cnt, t.E, a.S, a.e, a.Cseg, t.u0 + q, d_row, srows);
            if (!nt_ok) srows = 0;
            const int st_row = (a.diag & 8) ? (int)(d_row & 1023) : (int)d_row;   // diag 8: L2-resident store window
            // ret mode: rows whose intermediate (i, l) lives in this process go straight to
            // its ret1 (this lane's row: rdst); a strip is one segment, so one l and one
            // decision per warp.  Rows for other processes' intermediates go to D (Y) as
            // usual and smile_combine(2) fetches them over NVLink.
            bool rlocal = false, rout = false;
            char *rdst = nullptr;
            float rgate = 0.f;
            if (EK == 0 && a.rbases && srows > 0 && a.flat_out) {
                // FLAT (Switch): segment l is source rank l; one decision per warp
                const int64_t seg = d_row / a.Cseg;                    // (v * G + l) * e + k
                const int l = (int)((seg / a.e) % a.S);
                rlocal = l / a.rV == a.rrank0 / a.rV;
                if (rlocal && lane < srows) {
                    const int64_t tok = (int64_t)(l % a.rV) * a.T + a.rtok2[d_row + lane];
                    rdst = a.out + tok * a.N * 2 + dcol0 * 2;
                    rgate = a.gate[tok];
                    rout = true;
                }
            } else if (EK == 0 && a.rbases && srows > 0) {
                const int64_t seg = d_row / a.Cseg;                    // (v * S + l) * e + k
                const int vv = (int)(seg / ((int64_t)a.S * a.e)), l = (int)((seg / a.e) % a.S);
                const int u = (a.rrank0 + vv) / a.rm * a.rm + l;       // intermediate (i, l)
                rlocal = u / a.rV == a.rrank0 / a.rV;
                if (rlocal && lane < srows) {
                    const int32_t rr = a.rrow[d_row + lane];
                    rdst = a.rbases[u / a.rV] + a.roff_ret1 + (int64_t)rr * a.N * 2 + dcol0 * 2;
                    if (a.out) {
                        const int us = (int)((rr % (a.n * a.C1)) / a.C1) * a.rm + l;   // source (s, l)
                        if (us / a.rV == a.rrank0 / a.rV) {
                            const int64_t tok = (int64_t)(us % a.rV) * a.T + a.rtok2[d_row + lane];
                            rdst = a.out + tok * a.N * 2 + dcol0 * 2;
                            rgate = a.gate[tok];
                            rout = true;
                        }
                    }
                }
            }
            const bool full_box = srows == 32 && !(a.diag & 2);
            // EPI_DGELU: chunk c's saved GELU'(A1) is loaded before its accumulator
            // columns (the first chunk's while this tile's MMAs still run)
            const uint4 *aux_row =
                reinterpret_cast<const uint4 *>(a.aux + (d_row + (lane < srows ? lane : 0)) * (int64_t)a.N + dcol0);
            uint4 acur[4];
            if (dgelu && c_beg < c_end && srows > 0)
#pragma unroll
                for (int i = 0; i < 4; ++i) acur[i] = __ldg(aux_row + c_beg * 4 + i);
            if (NSUB == 1) mbar_wait(smem_u32(&tfull[acc]), (uint32_t)(it >> 1) & 1);
            else if (sub == 0) mbar_wait(smem_u32(&tfull[0]), (uint32_t)it & 1);
            tc_fence_after();
            const bool tr = warp == 4 && lane == 0 && it < 240;
            if (tr) trace_clock(a.trace, 520 + 2 * it);
            const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * ACC_COLS;
            for (int c = c_beg; c < c_end && srows > 0 && !(a.diag & 4); ++c) {
                if (dgelu && c > c_beg)
#pragma unroll
                    for (int i = 0; i < 4; ++i) acur[i] = __ldg(aux_row + c * 4 + i);
                float w[32];
                tmem_ld32(tbase + c * 32, w);
                if (has_bias) {
#pragma unroll
                    for (int i4 = 0; i4 < 8; ++i4) {
                        const float4 b = __ldg(bias4 + c * 8 + i4);
                        const f32x2 lo = add2(pack2(w[4 * i4], w[4 * i4 + 1]), pack2(b.x, b.y));
                        const f32x2 hi = add2(pack2(w[4 * i4 + 2], w[4 * i4 + 3]), pack2(b.z, b.w));
                        unpack2(lo, w[4 * i4], w[4 * i4 + 1]);
                        unpack2(hi, w[4 * i4 + 2], w[4 * i4 + 3]);
                    }
                }
                uint4 pk[4], pks[4];
                constexpr bool save = EK == 1;
                if (save) {
                    // H = GELU(z) into w, GELU'(z) into pks (one erf evaluation for both)
                    uint32_t *pw2 = reinterpret_cast<uint32_t *>(pks);
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        f32x2 gg, gp;
                        gelu_and_grad2(pack2(w[2 * i], w[2 * i + 1]), gg, gp);
                        unpack2(gg, w[2 * i], w[2 * i + 1]);
                        float q0, q1;
                        unpack2(gp, q0, q1);
                        __nv_bfloat162 hh = __floats2bfloat162_rn(q0, q1);
                        pw2[i] = *reinterpret_cast<uint32_t *>(&hh);
                    }
                }
                if (dgelu) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint4 u = acur[i];
                        const __nv_bfloat162 *hh = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
                        for (int z = 0; z < 4; ++z) {
                            const float2 f = __bfloat1622float2(hh[z]);
                            const f32x2 gg = mul2(pack2(w[8 * i + 2 * z], w[8 * i + 2 * z + 1]), pack2(f.x, f.y));
                            unpack2(gg, w[8 * i + 2 * z], w[8 * i + 2 * z + 1]);
                        }
                    }
                }
                uint32_t *pw = reinterpret_cast<uint32_t *>(pk);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    float y0 = w[2 * i], y1 = w[2 * i + 1];
                    if (act && !save) unpack2(gelu_erf2(pack2(y0, y1)), y0, y1);
                    __nv_bfloat162 hh = __floats2bfloat162_rn(y0, y1);
                    pw[i] = *reinterpret_cast<uint32_t *>(&hh);
                }
                if (dgelu && a.colsum) {
                    // db1 (a17): this strip's column sums of dZ (valid rows only)
                    if (lane >= srows)
#pragma unroll
                        for (int i = 0; i < 32; ++i) w[i] = 0.f;
                    transpose_reduce32(w, lane);
                    const int64_t seg = d_row / a.Cseg;
                    const int64_t u = (d_row - seg * a.Cseg) >> 5;
                    a.colsum[(seg * a.nstr + u) * a.N + dcol0 + c * 32 + lane] = w[0];
                }
                if (EK == 0 && rlocal) {
                    if (rdst) {
                        if (rout) {
                            __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(pk);
#pragma unroll
                            for (int z = 0; z < 16; ++z) {
                                const float2 f = __bfloat1622float2(h[z]);
                                h[z] = __floats2bfloat162_rn(rgate * f.x, rgate * f.y);
                            }
                        }
                        uint4 *d4 = reinterpret_cast<uint4 *>(rdst + c * 64);
#pragma unroll
                        for (int i = 0; i < 4; ++i) d4[i] = pk[i];
                    }
                } else if (full_box && a.tma_store && a.box64) {
                    // 32 x 64 box (SWIZZLE_128B: 16-byte unit j of row r at j ^ (r & 7)) over
                    // two consecutive chunks: the first waits for the box's previous store,
                    // the second fences and issues one TMA store (128-byte row segments)
                    const int hf = (c - c_beg) & 1;
                    if (hf == 0) {
                        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                        __syncwarp();
                    }
                    uint4 *srow = reinterpret_cast<uint4 *>(box + lane * 128);
#pragma unroll
                    for (int j = 0; j < 4; ++j) srow[(4 * hf + j) ^ (lane & 7)] = pk[j];
                    if (hf == 1) {
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        __syncwarp();
                        if (lane == 0) {
                            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                                             reinterpret_cast<uint64_t>(&mapD)),
                                         "r"((int)dcol0 + (c - 1) * 32), "r"(st_row), "r"(smem_u32(box))
                                         : "memory");
                            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                        }
                    }
                } else if (full_box && a.tma_store) {
                    // the box's previous store has finished reading smem; then the 32 x 32 box
                    // in the SWIZZLE_64B layout (16-byte chunk j of row r at j ^ ((r >> 1) & 3))
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    __syncwarp();
                    uint4 *srow = reinterpret_cast<uint4 *>(box + lane * 64);
                    const int sw = (lane >> 1) & 3;
#pragma unroll
                    for (int j = 0; j < 4; ++j) srow[j ^ sw] = pk[j];
                    if (nbox == 2) {
                        uint4 *srow2 = reinterpret_cast<uint4 *>(box + OUT_BOX_BYTES + lane * 64);
#pragma unroll
                        for (int j = 0; j < 4; ++j) srow2[j ^ sw] = pks[j];
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) {
                        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                                         reinterpret_cast<uint64_t>(&mapD)),
                                     "r"((int)dcol0 + c * 32), "r"(st_row), "r"(smem_u32(box))
                                     : "memory");
                        if (nbox == 2)
                            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                                             reinterpret_cast<uint64_t>(&mapD2)),
                                         "r"((int)dcol0 + c * 32), "r"((int)d_row), "r"(smem_u32(box + OUT_BOX_BYTES))
                                         : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                } else if (lane < srows && !(a.diag & 2)) {
                    // partial strips (a segment's last rows), or tma_store == 0: st.global of
                    // this lane's row (64 contiguous bytes per output), valid rows only
                    uint4 *dst = reinterpret_cast<uint4 *>(a.D + (d_row + lane) * (int64_t)a.N + dcol0 + c * 32);
#pragma unroll
                    for (int i = 0; i < 4; ++i) dst[i] = pk[i];
                    if (nbox == 2) {
                        uint4 *dst2 = reinterpret_cast<uint4 *>(a.D2 + (d_row + lane) * (int64_t)a.N + dcol0 + c * 32);
#pragma unroll
                        for (int i = 0; i < 4; ++i) dst2[i] = pks[i];
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (CG == 1) mbar_arrive(smem_u32(&tempty[acc]));
                else mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), lead));   // the leader's MMA waits on it
            }
            if (tr) trace_clock(a.trace, 521 + 2 * it);
            if (++sub == NSUB) {
                sub = 0;
                tile += ncl;
                ++it;
            }
        }
    }
    if (warp >= 4 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    pdl_trigger();
    __syncthreads();
    trace_end(a.trace);
    if (CS > 1) cluster_sync_all();           // no remote arrive / MMA into a CTA that has left
    if (warp == 2) {
        tc_fence_after();
        if (CG == 2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
    }
}

// ---- host: tensor maps ------------------------------------------------------------
int pick_bn(int N) {
    for (int bn = 256; bn >= 32; bn -= 32)
        if (N % bn == 0) return bn;
    return 0;
}

size_t smem_bytes(int CG, int nsub, int stages, int nbox, int tma_store, int box64, int nseg, int ek) {
    return 1024 + stages * (nsub * A_BYTES + B_BYTES_MAX / CG) +
           (tma_store ? nbox * epi_warps(ek) * OUT_BOX_BYTES * (box64 ? 2 : 1) : 0) +
           (2 * stages + 4) * 8 +
           16 + 32 * 4 + (nseg + 1) * 4 + nseg * 4;
}

constexpr size_t kSmemLimit = 227 * 1024;

// Epilogue output path: full 32 x 32 boxes staged in smem and written by TMA tensor
// stores (default), or SMILE_FFN_TMA_STORE=0: st.global from registers.  Measured at C2:
// GEMM1 (which writes H, 4x the bytes of Y) 687 us with st.global vs ~600 us with TMA
// stores; the FFN 1.15 vs 1.04 ms.
int pick_tma_store() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("SMILE_FFN_TMA_STORE");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v;
}

int pick_stages(int CG, int nsub, int nbox, int tma_store, int box64, int nseg, int ek) {
    int st = 8;
    while (st > 2 && smem_bytes(CG, nsub, st, nbox, tma_store, box64, nseg, ek) > kSmemLimit) --st;
    return st;
}

// CTA pairs (256-row tiles) unless an expert can hold at most 2048 rows (S * Cseg: then
// the experts' last, partly empty tiles dominate -- C5, ~512 rows per expert: 128-row
// tiles 3.68 vs 3.93 ms), the grid is odd, or SMILE_FFN_CTA_PAIR=0 / =1 forces it.
int pick_cg(int num_sms, int BN, int64_t rows_per_expert) {
    const char *e = getenv("SMILE_FFN_CTA_PAIR");          // read per launch (tests switch it)
    const int env = e ? (e[0] == '0' ? 0 : 1) : -1;
    const bool want = env >= 0 ? env == 1 : rows_per_expert > 2048;
    return (want && num_sms >= 2 && (BN / 2) % 16 == 0) ? 2 : 1;
}

// Sub-tiles per CTA-pair tile: SMILE_FFN_NSUB=2 (two M = 256 sub-tiles sharing each B
// stage; TMEM holds both accumulators) or 1 (one sub-tile, double-buffered accumulator).
int pick_nsub() {                                          // read per launch (tests switch it)
    const char *e = getenv("SMILE_FFN_NSUB");
    return (e && e[0] == '2') ? 2 : 1;
}

template <int CG, int NSUB, int EK, int MC = 0>
cudaError_t launch_tc(const CUtensorMap &mA, const CUtensorMap &mA128, const CUtensorMap &mB, const CUtensorMap &mD,
                      const CUtensorMap &mD2, const TcArgs &a, size_t smem, int num_sms, cudaStream_t st) {
    constexpr int CS = MC ? 2 : CG;
    static int grid = 0;
    if (!grid) {
        cudaFuncSetAttribute(ffn_gemm_tcgen05<CG, NSUB, EK, MC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemLimit);
        grid = num_sms / CS * CS;
        // SMILE_FFN_MAX_CTAS caps the persistent grid (leaves SMs to kernels of other
        // streams, e.g. the permutes of the next chunk in the pipelined layer)
        if (const char *e = getenv("SMILE_FFN_MAX_CTAS")) {
            const int cap = atoi(e) / CS * CS;
            if (cap >= CS && cap < grid) grid = cap;
        }
    }
    note_launch();
    if (CS == 1)
        return launch_k(ffn_gemm_tcgen05<CG, NSUB, EK, MC>, dim3(grid), dim3(nthreads(EK)), smem, st, mA, mA128, mB, mD, mD2, a);
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(nthreads(EK));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attrs[2];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = CS;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL (smile_internal.h)
    attrs[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, ffn_gemm_tcgen05<CG, NSUB, EK, MC>, mA, mA128, mB, mD, mD2, a);
}

// One grouped GEMM launch: D[rows, N] = epi(A[rows, K] . B[expert][N, K]^T).
cudaError_t launch_gemm(const void *A, int64_t rows_total, const void *B, int NE, const float *bias, void *D,
                        void *D2, const void *aux, const FfnArgs &f, int N, int K, int mode, int gelu,
                        cudaStream_t st, float *colsum = nullptr) {
    const int BN = pick_bn(N);
    const int CG = pick_cg(f.num_sms, BN, (int64_t)f.S * f.Cseg);
    // sub-tiles: SMILE_FFN_NSUB=2 (both tile shapes; single CTAs with two 128-row sub-tiles
    // sharing each B stage halve the B operand bytes of C5's small experts)
    const int NSUB = pick_nsub();
    CUtensorMap mA, mA128, mB, mD, mD2;
    if (!make_map(&mA, A, rows_total, K, 32)) return cudaErrorNotSupported;        // 32-row strip boxes
    if (!make_map(&mA128, A, rows_total, K, BM)) return cudaErrorNotSupported;     // 128-row tile box
    if (!make_map(&mB, B, (int64_t)NE * N, K, BN / CG)) return cudaErrorNotSupported;
    if (!make_map(&mD, D, rows_total, N, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B)) return cudaErrorNotSupported;
    CUtensorMap mD64;
    if (!make_map(&mD64, D, rows_total, N, 32, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorNotSupported;
    mD2 = mD;
    if (D2 && !make_map(&mD2, D2, rows_total, N, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B)) return cudaErrorNotSupported;
    TcArgs a;
    memset(&a, 0, sizeof(a));
    a.bias = bias; a.D = reinterpret_cast<__nv_bfloat16 *>(D); a.D2 = reinterpret_cast<__nv_bfloat16 *>(D2);
    a.counts = f.counts;
    a.nseg = f.V * f.S * f.e; a.e = f.e; a.S = f.S; a.Cseg = f.Cseg; a.N = N; a.K = K; a.BN = BN; a.gelu = gelu;
    a.mode = mode; a.aux = reinterpret_cast<const __nv_bfloat16 *>(aux);
    const int nbox = mode == EPI_BIAS_SAVE ? 2 : 1;
    a.tma_store = pick_tma_store();
    if (nbox == 2) {                      // training forward (H and A1): SMILE_FFN_SAVE_TMA=0 -> st.global
        const char *e = getenv("SMILE_FFN_SAVE_TMA");
        if (e && e[0] == '0') a.tma_store = 0;
    }
    // 32 x 64 output boxes for the GELU GEMM (the one that writes H, 4x the bytes of Y)
    // when every epilogue warp owns an even number of 32-column chunks
    {
        const char *e = getenv("SMILE_FFN_BOX64");
        const bool want = e ? (e[0] == '1' && gelu) || e[0] == '2' : false;     // 2: both GEMMs
        a.box64 = (want && a.tma_store && nbox == 1 && mode != EPI_DGELU && (BN / 32) % 8 == 0) ? 1 : 0;
    }
    const int ek = mode == EPI_DGELU ? 2 : (mode == EPI_BIAS_SAVE ? 1 : 0);
    a.stages = pick_stages(CG, NSUB, nbox, a.tma_store, a.box64, a.nseg, ek);
    if (const char *e = getenv("SMILE_FFN_STAGES")) {
        const int s = atoi(e);
        if (s >= 2 && s < a.stages) a.stages = s;
    }
    if (const char *e = getenv("SMILE_FFN_DIAG")) a.diag = atoi(e);
    a.colsum = colsum;
    a.nstr = (int)((f.Cseg + 31) / 32);
    if (mode == EPI_BIAS && !gelu && f.ret.bases) {
        a.rbases = f.ret.bases; a.rrow = f.rrow; a.roff_ret1 = f.ret.off_ret1;
        a.rrank0 = f.ret.rank0; a.rm = f.ret.m; a.rV = f.ret.V;
        if (f.out) {
            a.out = static_cast<char *>(f.out); a.gate = f.gate; a.rtok2 = f.rtok2;
            a.T = f.T; a.C1 = f.C1; a.n = f.n;
        }
        a.flat_out = f.flat_out;
        if (f.flat_out && !f.out) a.rbases = nullptr;       // nothing to fuse without the output
    }
    a.err = nullptr;
    a.trace = trace_buffer(mode == EPI_BIAS ? (gelu ? "ffn1" : "ffn2") : "ffn_bwd");
    const size_t smem = smem_bytes(CG, NSUB, a.stages, nbox, a.tma_store, a.box64, a.nseg, ek);
    if (a.box64) mD = mD64;                   // the output map with 32 x 64 SWIZZLE_128B boxes
#define SMILE_LAUNCH_TC(cg, ns)                                                                    \
    return ek == 2 ? launch_tc<cg, ns, 2>(mA, mA128, mB, mD, mD2, a, smem, f.num_sms, st)          \
                   : (ek == 1 ? launch_tc<cg, ns, 1>(mA, mA128, mB, mD, mD2, a, smem, f.num_sms, st) \
                              : launch_tc<cg, ns, 0>(mA, mA128, mB, mD, mD2, a, smem, f.num_sms, st))
    // A multicast across clusters of 2 single-CTA tiles (forward GEMMs of 128-row tiles)
    // when the N-tiles pair up evenly: C5 GEMM 2 1.94 -> 1.82 ms, while GEMM 1 (25 N-tiles:
    // a dummy every 13th pair) measured 1.57 -> 1.63 ms (r02_ffn_c5.md).  SMILE_FFN_MCAST=0
    // turns it off, =1 forces it for odd N-tile counts too (read per launch).
    {
        const char *mc = getenv("SMILE_FFN_MCAST");
        const int env = mc ? (mc[0] == '1' ? 1 : 0) : -1;
        const bool even = (N / BN) % 2 == 0;
        if (CG == 1 && NSUB == 1 && ek == 0 && f.num_sms >= 2 && (env == 1 || (env < 0 && even)))
            return launch_tc<1, 1, 0, 1>(mA, mA128, mB, mD, mD2, a, smem, f.num_sms, st);
    }
    if (CG == 2 && NSUB == 2) SMILE_LAUNCH_TC(2, 2);
    if (CG == 1 && NSUB == 2) SMILE_LAUNCH_TC(1, 2);
    if (CG == 2) SMILE_LAUNCH_TC(2, 1);
    SMILE_LAUNCH_TC(1, 1);
#undef SMILE_LAUNCH_TC
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

// Training forward on tcgen05: GEMM1 also stores GELU'(A1) (the backward's dZ multiplier).
cudaError_t launch_ffn_tcgen05_train(const FfnArgs &f, void *A1, cudaStream_t st) {
    if (!tc_supported(f)) return cudaErrorNotSupported;
    const int64_t rows_total = (int64_t)f.V * f.S * f.e * f.Cseg;
    const int NE = f.V * f.e;
    cudaError_t e = launch_gemm(f.X, rows_total, f.W1t, NE, f.b1, f.H, A1, nullptr, f, f.d_ff, f.d, EPI_BIAS_SAVE, 1, st);
    if (e != cudaSuccess) return e;
    return launch_gemm(f.H, rows_total, f.W2t, NE, f.b2, f.Y, nullptr, nullptr, f, f.d, f.d_ff, EPI_BIAS, 0, st);
}

// Backward data GEMMs on tcgen05 (a17): part 1: dZ = (dY W2^T) . GELU'(A1); part 2:
// dX = dZ W1^T.  W1 [NE, d, d_ff] and W2 [NE, d_ff, d] in their math layouts are the
// K-major B operands.
cudaError_t launch_ffn_tcgen05_dgrad(const FfnBwdArgs &b, int part, cudaStream_t st) {
    FfnArgs f{};
    f.counts = b.counts; f.V = b.V; f.S = b.S; f.e = b.e; f.Cseg = b.Cseg; f.d = b.d; f.d_ff = b.d_ff; f.bf16 = b.bf16;
    f.num_sms = b.num_sms;
    if (!tc_supported(f)) return cudaErrorNotSupported;
    const int64_t rows_total = (int64_t)f.V * f.S * f.e * f.Cseg;
    const int NE = f.V * f.e;
    if (part == 1)
        return launch_gemm(b.dY, rows_total, b.W2, NE, nullptr, b.dZ, nullptr, b.A1, f, f.d_ff, f.d, EPI_DGELU, 0, st,
                           b.colsum_ws);
    return launch_gemm(b.dZ, rows_total, b.W1, NE, nullptr, b.dX, nullptr, nullptr, f, f.d, f.d_ff, EPI_PLAIN, 0, st);
}

}  // namespace smile
