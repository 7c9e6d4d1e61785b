// gate_tcgen05.cu -- the level-1 gate with the router on Blackwell tensor cores (SURVEY
// §8(a) a1-a3, bf16 tokens, fused router).
//
// a1 (Eq. 1; tied routers W_p, W_q) is logit[t, k] = sum_c x[t, c] W[k, c]
// with fp32 W and, by R3/R23, fp32 logits.  The tokens are bf16; the router rows are
// split exactly into three bf16 pieces W = W^(0) + W^(1) + W^(2) (each piece the bf16
// rounding of the remainder, so the split is exact to ~2^-27 |W|), every product
// x * W^(p) is exact in fp32, and the tensor core accumulates in fp32: the logits match
// an fp32 dot product to within fp32 accumulation error, while the token stream runs
// at HBM speed on the tensor pipe instead of the FMA pipe (which cannot keep up once
// K1 + K2 reaches a few tens: SURVEY §7 hard part 4).
//
// One persistent, warp-specialised kernel (grid = min(#tiles, #SMs), 256 threads):
//   warp 0      TMA producer: the tile's x block (128 tokens x 64 columns, SWIZZLE_128B)
//               and the matching block of the split router (NP x 64), into an smem ring
//   warp 1      MMA issuer: tcgen05.mma.cta_group::1.kind::f16, M = 128 tokens,
//               N = NP = 3 * KW rounded up to 32 (columns 3k..3k+2 hold the three
//               pieces of logit k), into a double-buffered TMEM accumulator
//   warp 2      TMEM allocator
//   warps 4-11  two epilogue groups of 4 warps, taking alternate tiles (group g owns
//               accumulator buffer g): tcgen05.ld the tile's accumulator (thread =
//               token), sum the three pieces in order, logits to the group's smem,
//               release the accumulator, then the gate's phases B and C
//               (gate_common.cuh) on named barrier 1 + g.
// Tiles are 128 consecutive tokens of one rank, the same tiles as the capacity scan's
// (TB1 = 128): tile index = v * nblk + blk.
#include "smile_internal.h"
#include "gate_common.cuh"
#include "tc_util.cuh"

#include <stdlib.h>
#include <string.h>

namespace smile {
namespace {

using namespace tc;

constexpr int GT_BM = 128, GT_BK = 64;
constexpr int GT_THREADS = 384;
constexpr int GT_A_BYTES = GT_BM * GT_BK * 2;   // 16 KB per 64-column sub-block
constexpr int GT_MAX_NP = 384;                  // 3 * KW <= 384 (KW <= 128)

// W fp32 [KW, d] -> Wb bf16 [NP, d]: row 3k+p = piece p of W[k], rows >= 3 KW zero.
// r0 = W, piece_p = bf16_rn(r_p), r_{p+1} = r_p - piece_p (exact in fp32).
// quad10 = 1 (the swapped kernel): row r = 32 Q + w holds piece w % 3 of logit 10 Q + w / 3
// for w < 30 (rows 30, 31 of every 32-row group zero), so a logit's three pieces share a
// 32-lane TMEM quadrant.
__global__ void router_split_kernel(const float *__restrict__ w, __nv_bfloat16 *__restrict__ wb, int KW, int d,
                                    int NP, int quad10) {
    pdl_wait();
    const int64_t n = (int64_t)NP * d;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / d), c = (int)(i - (int64_t)r * d);
        int k = r / 3, p = r - 3 * k;
        if (quad10) {
            const int q = r >> 5, ww = r & 31;
            k = ww < 30 ? 10 * q + ww / 3 : KW;
            p = ww % 3;
        }
        float out = 0.f;
        if (k < KW) {
            float rem = w[(int64_t)k * d + c];
            for (int q = 0; q < p; ++q) rem -= __bfloat162float(__float2bfloat16_rn(rem));
            out = rem;
        }
        wb[i] = __float2bfloat16_rn(out);
    }
}

// In-kernel level-1 scan of the tensor-core gates (a3): flags [V * nblk] tagged with the
// call's epoch (2 e + 1: the tile's aggregate published, 2 e + 2: its inclusive prefix), so
// nothing is reset between calls; the last CTA of a call advances *epoch_ctr.
struct Lookback {
    int on;
    Scan1Args s;     // tables (blk_hist1 = aggregates, blk_off1, psum, hist2a), stats, counts1, lb_inc
    int *flags;
    int *epoch_ctr;
};

struct GateTcArgs {
    GateArgs g;
    int NP;          // accumulator columns (3 * KW rounded up to 32)
    int nbuf;        // TMEM accumulator buffers (2 when 2 * NP <= 512)
    int stages;
    int ntiles;
    int nsub;        // 64-column sub-blocks per pipeline stage (2 when d % 128 == 0: fewer,
                     // larger stages -- the single MMA thread's per-stage overhead halves)
    int resident_b;  // 1: every CTA builds the split router (NP x d bf16, SWIZZLE_128B K-major)
                     // in its own smem at start from the fp32 W -- no split kernel, and the
                     // pipeline stages carry x only
    Lookback lb;     // in-kernel level-1 scan (non-fused gates)
    int *done;       // CTA arrival counter (the last CTA advances the look-back epoch)
    unsigned long long *trace;   // SMILE_TRACE=gate timeline (smile_internal.h), or null
};

__device__ __forceinline__ int ld_acquire_gpu(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Level-1 scan of one tile by decoupled look-back (a3; R5, R8): the tile's destination
// histogram s_bh (gate_finish's block_rank) is already in blk_hist1; publish it, look back
// over the rank's earlier tiles (warp 0: lane = predecessor, aggregates summed up to the
// nearest inclusive prefix), write the tile's exclusive offsets to blk_off1 (what the
// permute adds to the tile-local ranks) and its inclusive prefix.  The rank's LAST tile
// then holds the totals: hist1, counts1 = min(total, C1) (and FLAT peer counts), and -- once
// every tile of the rank has published -- reduces the rank's LB statistics over its tiles in
// tile order (lane = statistic: deterministic).  Tiles run in increasing order on every CTA
// and every CTA is resident, so every wait terminates.
template <class Sync>
__device__ void lookback_scan(const GateArgs &a, const Lookback &lb, const int *s_bh, int *s_off, int tile,
                              int epoch) {
    const Scan1Args &sc = lb.s;
    const int tid = Sync::tid(), lane = tid & 31, w = tid >> 5, NW = Sync::nthr() >> 5;
    const int K1 = a.K1, v = tile / a.nblk, blk = tile - v * a.nblk;
    int *flag = lb.flags + tile;
    const int f_agg = 2 * epoch + 1, f_inc = 2 * epoch + 2;
    // 1. publish (the first tile of a rank: directly its inclusive prefix)
    for (int k = tid; k < K1; k += Sync::nthr()) {
        if (blk == 0) sc.lb_inc[(int64_t)tile * K1 + k] = s_bh[k];
        s_off[k] = 0;
    }
    // the threads that wrote this tile's table entries (blk_hist1, lb_inc: tid < K1; psum /
    // hist2a: lane 0 of the narrow loops, every lane of the wide ones) make them visible
    if (lane == 0 || tid < K1 || a.KW >= 32) __threadfence();
    Sync::sync();
    if (tid == 0) st_release_gpu(flag, blk == 0 ? f_inc : f_agg);
    // 2. look back (warp 0)
    if (blk > 0 && w == 0) {
        const int base = v * a.nblk;
        for (int p = blk - 1;; p -= 32) {
            const int pb = p - lane;
            int fl = f_inc;                             // before the rank's first tile: zero, inclusive
            if (pb >= 0) {
                uint64_t spin = 0;
                while ((fl = ld_acquire_gpu(lb.flags + base + pb)) < f_agg)
                    if (++spin > (1ull << 28)) __trap();   // a tile that never publishes: abort, never hang
            }
            const unsigned incm = __ballot_sync(kFull, fl == f_inc);
            const int stop = incm ? __ffs(incm) - 1 : 32;
            for (int k = 0; k < K1; ++k) {
                int val = 0;
                if (pb >= 0 && lane < stop) val = __ldcg(sc.blk_hist1 + ((int64_t)base + pb) * K1 + k);
                else if (pb >= 0 && lane == stop) val = __ldcg(sc.lb_inc + ((int64_t)base + pb) * K1 + k);
                for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(kFull, val, o);
                if (lane == 0) s_off[k] += val;
            }
            if (incm) break;
        }
    }
    Sync::sync();
    // 3. offsets for the permute, the inclusive prefix for the successors
    for (int k = tid; k < K1; k += Sync::nthr()) {
        sc.blk_off1[(int64_t)tile * K1 + k] = s_off[k];
        if (blk > 0) sc.lb_inc[(int64_t)tile * K1 + k] = s_off[k] + s_bh[k];
    }
    if (blk > 0) {
        __threadfence();
        Sync::sync();
        if (tid == 0) st_release_gpu(flag, f_inc);
    }
    // 4. the rank's last tile: totals and the LB statistics
    if (blk == a.nblk - 1) {
        for (int k = tid; k < K1; k += Sync::nthr()) {
            const int tot = s_off[k] + s_bh[k];
            const int32_t cnt = (int32_t)(tot < sc.C1 ? tot : sc.C1);
            sc.stats.hist1[v * K1 + k] = tot;
            sc.counts1[v * K1 + k] = cnt;
            if (sc.peer.bases && sc.flat) {             // counts travel with the rows: rcounts[q][src][k % e]
                const PeerMap &P = sc.peer;
                const int rk = P.rank0 + v, q = k / P.e;
                reinterpret_cast<int32_t *>(P.bases[q / P.V] + P.off_rcounts)[((int64_t)(q % P.V) * P.G + rk) * P.e + k % P.e] = cnt;
            }
        }
        if (w == 0) {                                   // every tile of the rank has published its partials
            for (int p = lane; p < a.nblk; p += 32) {
                uint64_t spin = 0;
                while (ld_acquire_gpu(lb.flags + v * a.nblk + p) < f_agg)
                    if (++spin > (1ull << 28)) __trap();
            }
        }
        __threadfence();
        Sync::sync();
        const int KS = K1 + a.K2;
        const int64_t rb = (int64_t)v * a.nblk;
        for (int cb = w; cb < (KS + 31) / 32; cb += NW) {
            const int k = cb * 32 + lane;
            if (k < KS) {
                double acc = 0.0;
                for (int p0 = 0; p0 < a.nblk; p0 += 16) {        // 16 loads in flight, summed in tile order
                    double t[16];
#pragma unroll
                    for (int u = 0; u < 16; ++u) t[u] = p0 + u < a.nblk ? __ldcg(sc.blk_psum + (rb + p0 + u) * KS + k) : 0.0;
#pragma unroll
                    for (int u = 0; u < 16; ++u) acc += t[u];
                }
                if (k < K1) sc.stats.psum1[v * K1 + k] = acc;
                else sc.stats.psum2[v * a.K2 + (k - K1)] = acc;
            }
        }
        for (int cb = w; cb < (a.K2 + 31) / 32; cb += NW) {
            const int k = cb * 32 + lane;
            if (k < a.K2) {
                int c = 0;
                for (int p0 = 0; p0 < a.nblk; p0 += 16) {
                    int t[16];
#pragma unroll
                    for (int u = 0; u < 16; ++u) t[u] = p0 + u < a.nblk ? __ldcg(sc.blk_hist2a + (rb + p0 + u) * a.K2 + k) : 0;
#pragma unroll
                    for (int u = 0; u < 16; ++u) c += t[u];
                }
                sc.stats.hist2[v * a.K2 + k] = c;
            }
        }
    }
}

// Fused level-1 permute (a4) in the gate's epilogue.  The tile's destination histogram
// s_bh is published (flag 1); warp 0 of the group looks back over the rank's earlier
// tiles 32 at a time (lane = one predecessor): aggregates are summed up to the nearest
// tile that has published its inclusive prefix (flag 2), giving this tile's exclusive
// offsets s_off; the inclusive prefix is published (flag 2).  Tiles run in increasing
// order on every CTA and all CTAs are resident, so every look-back terminates.  Then
// slot1 = s_off[dest1] + in-tile rank (R5, R8: earliest token first), and each warp
// moves its kept tokens' rows (16-byte vectors, 4 rows in flight) to the slot -- into
// send1 / meta1, or straight into the destination's receive buffer (peer stores).
template <class Sync>
__device__ void fused_dispatch(const GateArgs &a, const GateTok tk, const int *s_bh, int *s_off, int64_t tok0,
                               int nt, int tile) {
    const int tid = Sync::tid(), lane = tid & 31, w = tid >> 5;
    const int K1 = a.K1, v = tile / a.nblk, blk = tile - v * a.nblk;
    int *flag = a.lb_flag + tile;
    // 1. publish the aggregate (the first tile of a rank: directly the inclusive prefix)
    for (int k = tid; k < K1; k += Sync::nthr()) {
        a.lb_agg[(int64_t)tile * K1 + k] = s_bh[k];
        if (blk == 0) a.lb_inc[(int64_t)tile * K1 + k] = s_bh[k];
        s_off[k] = 0;
    }
    __threadfence();
    Sync::sync();
    if (tid == 0) st_release_gpu(flag, blk == 0 ? 2 : 1);
    // 2. look back (warp 0)
    if (blk > 0 && w == 0) {
        const int base = v * a.nblk;
        for (int p = blk - 1;; p -= 32) {
            const int pb = p - lane;
            int fl = 2;                                  // before the rank's first tile: zero, inclusive
            if (pb >= 0) {
                uint64_t spin = 0;
                while ((fl = ld_acquire_gpu(a.lb_flag + base + pb)) == 0)
                    if (++spin > (1ull << 28)) __trap();  // a tile that never publishes: abort, never hang
            }
            const unsigned incm = __ballot_sync(kFull, fl == 2);
            const int stop = incm ? __ffs(incm) - 1 : 32;   // nearest predecessor with an inclusive prefix
            for (int k = 0; k < K1; ++k) {
                int val = 0;
                if (pb >= 0 && lane < stop) val = a.lb_agg[((int64_t)base + pb) * K1 + k];
                else if (pb >= 0 && lane == stop) val = a.lb_inc[((int64_t)base + pb) * K1 + k];
                for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(kFull, val, o);
                if (lane == 0) s_off[k] += val;
            }
            if (incm) break;
        }
    }
    Sync::sync();
    // 3. publish the inclusive prefix
    if (blk > 0) {
        for (int k = tid; k < K1; k += Sync::nthr()) a.lb_inc[(int64_t)tile * K1 + k] = s_off[k] + s_bh[k];
        __threadfence();
        Sync::sync();
        if (tid == 0) st_release_gpu(flag, 2);
    }
    // 4. final slots, meta, destinations
    const char *src = nullptr;
    char *dst = nullptr;
    if (tid < nt && tk.i >= 0) {
        const int64_t g = tok0 + tid;
        const int slot = s_off[tk.i] + tk.lr;
        a.route.slot1[g] = slot;
        if (slot < a.C1) {
            src = static_cast<const char *>(a.x) + g * a.rowbytes;
            const int j = a.route.dest2[g];
            if (a.peer.bases) {
                const PeerMap &P = a.peer;
                const int rk = P.rank0 + v;
                int q;
                int64_t row;
                if (!a.flat) {                   // bi-level: (s, l) -> intermediate (i, l), chunk s
                    const int s_ = rk / P.m, l = rk % P.m;
                    q = tk.i * P.m + l;
                    row = ((int64_t)(q % P.V) * P.n + s_) * a.C1 + slot;
                } else {                         // flat: expert i on rank i / e, chunk (src, i % e)
                    q = tk.i / P.e;
                    row = (((int64_t)(q % P.V) * P.G + rk) * P.e + tk.i % P.e) * a.C1 + slot;
                }
                char *b = P.bases[q / P.V];
                dst = b + P.off_recv1 + row * a.rowbytes;
                if (!a.flat) reinterpret_cast<int32_t *>(b + P.off_rmeta1)[row] = j;
            } else {
                const int64_t row = ((int64_t)v * K1 + tk.i) * a.C1 + slot;
                dst = static_cast<char *>(a.send) + row * a.rowbytes;
                if (a.meta) a.meta[row] = j;
            }
        }
    }
    // 5. the warp's 32 rows, 4 at a time: every lane moves 16-byte vectors of each
    const int nvec = (int)(a.rowbytes / 16);
    for (int r0 = 0; r0 < 32; r0 += 4) {
        const char *sr[4];
        char *dr[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            sr[r] = reinterpret_cast<const char *>(__shfl_sync(kFull, reinterpret_cast<unsigned long long>(src), r0 + r));
            dr[r] = reinterpret_cast<char *>(__shfl_sync(kFull, reinterpret_cast<unsigned long long>(dst), r0 + r));
        }
        for (int c0 = lane; c0 < nvec; c0 += 96) {
            int4 val[4][3];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int u = 0; u < 3; ++u) {
                    const int c = c0 + 32 * u;
                    val[r][u] = (dr[r] && c < nvec) ? *reinterpret_cast<const int4 *>(sr[r] + (int64_t)c * 16)
                                                    : make_int4(0, 0, 0, 0);
                }
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int u = 0; u < 3; ++u) {
                    const int c = c0 + 32 * u;
                    if (dr[r] && c < nvec) *reinterpret_cast<int4 *>(dr[r] + (int64_t)c * 16) = val[r][u];
                }
        }
    }
}

// After the group's logits of one tile are in smem: (optional) logits_out copy, the
// gate's phases B and C, and (fused) the level-1 permute of the tile.
template <class Sync>
__device__ __forceinline__ void finish_tile(const GateArgs &a, float *s_lg, int *s_j, int *s_wh, int *s_bh,
                                            double *s_part, int *s_off, int64_t tok0, int nt, int tile,
                                            unsigned long long *trace = nullptr, int tslot = 0) {
    Sync::sync();
    if (a.logits_out) {
        const int lds = gate_lds(a.KW);
        for (int i = Sync::tid(); i < nt * a.KW; i += Sync::nthr())
            a.logits_out[tok0 * a.KW + i] = s_lg[(i / a.KW) * lds + i % a.KW];
        Sync::sync();
    }
    const GateTok tk = gate_finish<Sync>(a, s_lg, gate_lds(a.KW), s_j, s_wh, s_bh, s_part, tok0, nt, (int64_t)tile, trace,
                                         tslot);
    if (a.fuse_dispatch) fused_dispatch<Sync>(a, tk, s_bh, s_off, tok0, nt, tile);
    Sync::sync();
}

__global__ void __launch_bounds__(GT_THREADS, 1)
gate1_tc_kernel(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapW, GateTcArgs ta) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    pdl_wait();
    const GateArgs &a = ta.g;
    const int NP = ta.NP, ST = ta.stages, KW = a.KW;
    const int nsub = ta.nsub;
    const int a_bytes = nsub * GT_A_BYTES;                 // per stage
    const bool resb = ta.resident_b != 0;
    const int b_bytes = resb ? 0 : nsub * NP * GT_BK * 2;     // per stage (streamed split router)
    unsigned char *base = reinterpret_cast<unsigned char *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    unsigned char *sA = base;
    unsigned char *sB = sA + ST * a_bytes;                   // resident: [d / 64][NP rows][128 B]
    const int b_region = resb ? NP * a.d * 2 : ST * b_bytes;
    // per epilogue group g: gate_finish scratch (fp64 first) | logits [128][lds] | s_j [128] |
    // s_wh [4][K1] | s_bh [K1] | s_off [K1] (fused permute); an even int count per group keeps
    // every group's scratch 8-byte aligned
    const int lds = gate_lds(KW);
    const int scr_ints = (int)(gate_scratch_bytes(GT_BM, KW, a.K2) / 4);
    const int grp_ints = (scr_ints + GT_BM * lds + GT_BM + 6 * a.K1 + 1) & ~1;
    int *grp0 = reinterpret_cast<int *>(sB + b_region);
    uint64_t *bars = reinterpret_cast<uint64_t *>(((uintptr_t)(grp0 + ta.nbuf * grp_ints) + 7) & ~(uintptr_t)7);
    uint64_t *full = bars, *empty = bars + ST, *tfull = bars + 2 * ST, *tempty = bars + 2 * ST + 2;
    uint64_t *b_ready = bars + 2 * ST + 4;                     // resident split router built
    uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bars + 2 * ST + 5);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int epoch = ta.lb.on ? *reinterpret_cast<volatile int *>(ta.lb.epoch_ctr) : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(smem_u32(&tfull[s]), 1);
            mbar_init(smem_u32(&tempty[s]), 4);
        }
        mbar_init(smem_u32(b_ready), (GT_THREADS - 96) / 32);        // one arrive per building warp
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapX)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapW)) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_holder))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    trace_begin(ta.trace);
    const uint32_t tmem_base = *tmem_holder;
    const int nk = a.d / (GT_BK * nsub);
    const int nbuf = ta.nbuf;
    const int nchunk_n = NP > 256 ? 2 : 1;
    const int NPc = NP / nchunk_n;                     // N of one MMA

    if (resb && warp >= 3) {
        // warps 3.. build the exact 3-piece bf16 split of W (row 3k + p = piece p of W[k];
        // rows >= 3 KW zero) in the canonical SWIZZLE_128B K-major layout the MMA reads
        // (per 64-column block: rows of 128 B, 16-byte unit u of row r at u ^ (r & 7)),
        // while the producer already streams x; the MMA thread waits on b_ready.
        __nv_bfloat16 *bs = reinterpret_cast<__nv_bfloat16 *>(sB);
        const int nthr = GT_THREADS - 96, t0 = threadIdx.x - 96;
        const int total = NP * a.d;
        for (int i0 = t0; i0 < total; i0 += nthr * 4) {
            float wv[4];
#pragma unroll
            for (int z = 0; z < 4; ++z) {
                const int idx = i0 + z * nthr;
                const int r = idx / a.d, c = idx - r * a.d, k = r / 3;
                wv[z] = (idx < total && k < KW) ? __ldg(a.w + (int64_t)k * a.d + c) : 0.f;
            }
#pragma unroll
            for (int z = 0; z < 4; ++z) {
                const int idx = i0 + z * nthr;
                if (idx >= total) break;
                const int r = idx / a.d, c = idx - r * a.d, k = r / 3, p = r - 3 * k;
                float rem = wv[z];
                for (int q = 0; q < p; ++q) rem -= __bfloat162float(__float2bfloat16_rn(rem));
                const int kb = c >> 6, u = (c & 63) >> 3;
                bs[((size_t)kb * NP + r) * 64 + ((u ^ (r & 7)) << 3) + (c & 7)] = __float2bfloat16_rn(k < KW ? rem : 0.f);
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor-core reads
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(b_ready));
    }

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer ----------------
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < ta.ntiles; tile += gridDim.x) {
                const int v = tile / a.nblk, blk = tile - v * a.nblk;
                const int row0 = (int)((int64_t)v * a.T + (int64_t)blk * GT_BM);
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
                    const uint32_t fb = smem_u32(&full[stage]);
                    mbar_arrive_tx(fb, a_bytes + b_bytes);
                    for (int u = 0; u < nsub; ++u) {
                        const int col = (kb * nsub + u) * GT_BK;
                        tma_load_2d(smem_u32(sA + stage * a_bytes + u * GT_A_BYTES), &mapX, col, row0, fb);
                        if (!resb)
                            for (int h = 0; h < nchunk_n; ++h)
                                tma_load_2d(smem_u32(sB + stage * b_bytes + u * NP * 128 + h * NPc * 128), &mapW,
                                            col, h * NPc, fb);
                    }
                    if (++stage == ST) { stage = 0; phase ^= 1; }
                }
            }
            trace_clock(ta.trace, 5);
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer: the whole warp runs the loop (warp-uniform descriptors,
        // advanced by adding 16-byte units to the start-address field), one elected lane issues
        if (resb) mbar_wait(smem_u32(b_ready), 0);
        const uint32_t idesc = make_idesc(GT_BM, NPc);
        const uint64_t adesc0 = sw128_desc(smem_u32(sA)), bdesc0 = sw128_desc(smem_u32(sB));
        const uint32_t a_st = (uint32_t)a_bytes >> 4, b_st = (uint32_t)b_bytes >> 4;
        const uint32_t b_sub = (uint32_t)(NP * 128) >> 4, b_half = (uint32_t)(NPc * 128) >> 4;
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        for (int tile = blockIdx.x; tile < ta.ntiles; tile += gridDim.x, ++it) {
            const int buf = it % nbuf;
            const uint32_t use = (uint32_t)(it / nbuf) & 1;
            mbar_wait(smem_u32(&tempty[buf]), use ^ 1);
            tc_fence_after();
            if (lane == 0 && it < 120) trace_clock(ta.trace, 8 + 2 * it);
            const uint32_t tmem_d = tmem_base + buf * NP;
            for (int kb = 0; kb < nk; ++kb) {
                mbar_wait(smem_u32(&full[stage]), phase);
                tc_fence_after();
                if (elect_one()) {
                    for (int u = 0; u < nsub; ++u) {
                        const uint64_t ad = adesc0 + (uint64_t)(stage * a_st + u * (GT_A_BYTES >> 4));
                        const uint64_t bd = bdesc0 + (uint64_t)(resb ? (uint32_t)(kb * nsub + u) * b_sub
                                                                      : stage * b_st + u * b_sub);
#pragma unroll
                        for (int k = 0; k < GT_BK / 16; ++k) {
                            const uint32_t acc = (kb | u | k) ? 1u : 0u;
                            mma_bf16(tmem_d, ad + (uint64_t)(2 * k), bd + (uint64_t)(2 * k), idesc, acc);
                            if (nchunk_n == 2)
                                mma_bf16(tmem_d + NPc, ad + (uint64_t)(2 * k), bd + (uint64_t)(b_half + 2 * k), idesc,
                                         acc);
                        }
                    }
                    mma_commit(smem_u32(&empty[stage]));
                }
                __syncwarp();
                if (++stage == ST) { stage = 0; phase ^= 1; }
            }
            if (elect_one()) mma_commit(smem_u32(&tfull[buf]));
            __syncwarp();
            if (lane == 0 && it < 120) trace_clock(ta.trace, 9 + 2 * it);
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: thread = token (TMEM lane) ----------------
        const int grp = (warp - 4) >> 2;
        const int q = warp & 3;
        const int row = q * 32 + lane;
        double *s_part = reinterpret_cast<double *>(grp0 + grp * grp_ints);
        float *s_lg = reinterpret_cast<float *>(grp0 + grp * grp_ints + scr_ints);
        int *s_j = reinterpret_cast<int *>(s_lg + GT_BM * lds);
        int *s_wh = s_j + GT_BM;
        int *s_bh = s_wh + 4 * a.K1;
        int *s_off = s_bh + a.K1;
        // with a single accumulator buffer (NP > 256) one group takes every tile: the
        // tfull / tempty parities then count every tile of the CTA
        const int ngrp = nbuf;
        int it = grp;
        for (int tile = blockIdx.x + grp * gridDim.x; grp < ngrp && tile < ta.ntiles;
             tile += ngrp * gridDim.x, it += ngrp) {
            const int v = tile / a.nblk, blk = tile - v * a.nblk;
            const int64_t t0 = (int64_t)blk * GT_BM;
            const int nt = (int)(a.T - t0 < GT_BM ? a.T - t0 : GT_BM);
            const int64_t tok0 = (int64_t)v * a.T + t0;
            const int buf = it % nbuf;
            mbar_wait(smem_u32(&tfull[buf]), (uint32_t)(it / nbuf) & 1);
            tc_fence_after();
            const bool tr = q == 0 && lane == 0 && it < 120;
            if (tr) trace_clock(ta.trace, 256 + 4 * it);
            const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + buf * NP;
            // logit k = (piece0 + piece1) + piece2 from columns 3k, 3k+1, 3k+2: 32 logits per
            // group of three 32-column loads in flight (one wait), unrolled so every column's
            // register is fixed at compile time.  The last group may read past this buffer's
            // NP columns (into the other buffer or unused columns: discarded, k >= KW); when it
            // would pass the 512 allocated columns, the column-at-a-time loop instead.
            const int ng = (KW + 31) / 32;
            if (buf * NP + ng * 96 <= 512) {
                for (int g3 = 0; g3 < ng; ++g3) {
                    float v0[32], v1[32], v2[32];
                    tmem_ld32_nowait(tb + g3 * 96, v0);
                    tmem_ld32_nowait(tb + g3 * 96 + 32, v1);
                    tmem_ld32_nowait(tb + g3 * 96 + 64, v2);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int f = 3 * i;
                        const float x0 = f < 32 ? v0[f] : f < 64 ? v1[f - 32] : v2[f - 64];
                        const float x1 = f + 1 < 32 ? v0[f + 1] : f + 1 < 64 ? v1[f - 31] : v2[f - 63];
                        const float x2 = f + 2 < 32 ? v0[f + 2] : f + 2 < 64 ? v1[f - 30] : v2[f - 62];
                        const int k = g3 * 32 + i;
                        if (k < KW) s_lg[row * lds + k] = (x0 + x1) + x2;
                    }
                }
            } else {
                float accv = 0.f;
                for (int c = 0; c < NP / 32; ++c) {
                    float vv[32];
                    tmem_ld32(tb + c * 32, vv);
                    int k = (c * 32) / 3, pc = (c * 32) - 3 * k;
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        if (k < KW) {
                            accv = pc == 0 ? vv[i] : accv + vv[i];
                            if (pc == 2) s_lg[row * lds + k] = accv;
                        }
                        if (++pc == 3) { pc = 0; ++k; }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&tempty[buf]));
            if (tr) trace_clock(ta.trace, 257 + 4 * it);
            if (grp == 0) {
                finish_tile<EpiSync<0>>(a, s_lg, s_j, s_wh, s_bh, s_part, s_off, tok0, nt, tile, it < 100 ? ta.trace : nullptr,
                                        600 + 4 * it);
                if (ta.lb.on) lookback_scan<EpiSync<0>>(a, ta.lb, s_bh, s_off, tile, epoch);
            } else {
                finish_tile<EpiSync<1>>(a, s_lg, s_j, s_wh, s_bh, s_part, s_off, tok0, nt, tile, it < 100 ? ta.trace : nullptr,
                                        600 + 4 * it);
                if (ta.lb.on) lookback_scan<EpiSync<1>>(a, ta.lb, s_bh, s_off, tile, epoch);
            }
            if (tr) trace_clock(ta.trace, 258 + 4 * it);
        }
    }
    pdl_trigger();
    __syncthreads();
    trace_end(ta.trace);
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
    }
    if (threadIdx.x == 0 && ta.lb.on) {
        // every CTA has read the epoch: the last one advances it for the next call
        __threadfence();
        if (atomicAdd(ta.done, 1) == (int)gridDim.x - 1) {
            *ta.done = 0;
            *ta.lb.epoch_ctr = epoch + 1;
            __threadfence();
        }
    }
}

// ---------------------------------------------------------------------------------
// Swapped-role tensor-core gate (default for KW <= 40): M = the split router (its
// 32 * ceil(KW / 10) rows zero-padded to 128 by TMA), N = 256 TOKENS per MMA.  With the
// tokens on M (gate1_tc_kernel) every tcgen05.mma is 128 x NP x 16 with NP as small as
// 32, and the MMA count per token -- each costs a near-fixed ~350 cycles there (ncu: the
// producer waits on stage releases while the MMA thread never waits for data) -- is what
// bounds the kernel; here one MMA covers 256 tokens.  The accumulator [piece rows x 256
// tokens] is transposed by the epilogue: lane r of quadrant q holds piece r % 3 of logit
// 10 q + r / 3 for 32 tokens; two shuffles sum the pieces in order, and the logits land in
// s_lg [token][KW] for the same gate_finish (8 warps, 256 tokens per tile, TB1 = 256).
// The exact three-piece bf16 split of the fp32 router (R3, R23) is built into `wsplit` by
// the epilogue warps of the first CTAs while the producers already stream x; a producer
// issues the router loads of its first stages once the split is published (release /
// acquire counter + async-proxy fence) -- no separate split kernel.  The last CTA to finish
// resets the counter (graph-replay safe).
// (Round 2 measured two alternatives on the same box and kept neither: contiguous per-CTA
// token ranges with 32-token scan tables (no partial last wave) 48-51 us + a 4x larger
// scan, and 128-token tables with 256/128-token tiles 57-59 us, against this kernel's
// 45 us; profiles/r02_gate_schedule_ab.md.)
// ---------------------------------------------------------------------------------
constexpr int GS_TOK = 256, GS_THREADS = 128 + 256;
constexpr int kResWMaxKW = 20;                     // resident split router: KW <= 20 (NPT <= 64),
constexpr int kResWCols = 4;                       // d <= 1024
constexpr int GS_X_BYTES = GS_TOK * GT_BK * 2;    // 32 KB per stage
constexpr int GS_W_BYTES = 128 * GT_BK * 2;       // 16 KB per stage

template <int G>
struct EpiSync256 {
    static __device__ __forceinline__ void sync() { asm volatile("bar.sync %0, 256;" ::"n"(1 + G) : "memory"); }
    static __device__ __forceinline__ int tid() { return threadIdx.x - 128; }
    static __device__ __forceinline__ int nthr() { return 256; }
};

struct GateTArgs {
    GateArgs g;
    int NPT;         // split-router rows (32 * ceil(KW / 10))
    int stages;
    int ntiles;
    int nbuilders;   // CTAs that build the split router (0: built by router_split_kernel)
    int *split_ready, *done;
    __nv_bfloat16 *wsplit;   // [NPT, d] the split router
    int resw;        // 1: every CTA builds the split router into its own smem (NPT x d bf16,
                     // resident; small routers) and the stages carry x only -- no global split,
                     // no publish / poll before the first MMA
    // level-1 scan by decoupled look-back inside the kernel (lookback != 0): per-tile flags
    // carry the call's epoch (2 e + 1: aggregate published, 2 e + 2: inclusive prefix), so
    // nothing is reset between calls; the last CTA advances *epoch_ctr
    Lookback lb;     // in-kernel level-1 scan
    unsigned long long *trace;   // SMILE_TRACE=gate timeline (smile_internal.h), or null
};

__global__ void __launch_bounds__(GS_THREADS, 1)
gate1_tcT_kernel(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapW, GateTArgs ta) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    pdl_wait();
    const GateArgs &a = ta.g;
    const int ST = ta.stages, KW = a.KW, NQ = ta.NPT / 32;
    unsigned char *base = reinterpret_cast<unsigned char *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    unsigned char *sW = base;
    const bool resw = ta.resw != 0;
    // resident: [d / 64][NPT rows][128 B] (4 KB-aligned k blocks).  The M = 128 MMA also reads
    // rows NPT..127 past each block -- the next blocks', or the x stages' bytes after the last
    // one: they only feed TMEM lanes >= NPT, which the epilogue never reads
    unsigned char *sX = sW + (resw ? (size_t)ta.NPT * a.d * 2 : (size_t)ST * GS_W_BYTES);
    const int lds = gate_lds(KW);
    float *s_lg = reinterpret_cast<float *>(sX + ST * GS_X_BYTES);    // [256][lds]
    int *s_j = reinterpret_cast<int *>(s_lg + GS_TOK * lds);          // [256]
    int *s_wh = s_j + GS_TOK;                                         // [8][K1]
    int *s_bh = s_wh + 8 * a.K1;                                      // [K1]
    int *s_off = s_bh + a.K1;                                         // [K1] look-back offsets
    double *s_part = reinterpret_cast<double *>(((uintptr_t)(s_off + a.K1) + 7) & ~(uintptr_t)7);   // gate_finish scratch
    uint64_t *bars = reinterpret_cast<uint64_t *>(
        ((uintptr_t)s_part + gate_scratch_bytes(GS_TOK, KW, a.K2) + 7) & ~(uintptr_t)7);
    uint64_t *full = bars, *empty = bars + ST, *tfull = bars + 2 * ST, *tempty = bars + 2 * ST + 2;
    uint64_t *w_ready = bars + 2 * ST + 4;     // [kResWCols] resident split: columns 256 r.. built
    uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bars + 2 * ST + 4 + kResWCols);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // the call's look-back epoch: read before any CTA can advance it (the last CTA to finish)
    const int epoch = ta.lb.on ? *reinterpret_cast<volatile int *>(ta.lb.epoch_ctr) : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(smem_u32(&tfull[s]), 1);
            mbar_init(smem_u32(&tempty[s]), 8);
        }
        for (int r = 0; r < kResWCols; ++r) mbar_init(smem_u32(&w_ready[r]), 8);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapX)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapW)) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_holder))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    trace_begin(ta.trace);
    const uint32_t tmem_base = *tmem_holder;
    const int nk = a.d / GT_BK;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            // router loads wait for the in-kernel split: the first ST stages get their x
            // loads at once and their router loads once the split is published
            bool wready = ta.nbuilders == 0;
            int npend = 0;
            for (int tile = blockIdx.x; tile < ta.ntiles; tile += gridDim.x) {
                const int v = tile / a.nblk, blk = tile - v * a.nblk;
                const int row0 = (int)((int64_t)v * a.T + (int64_t)blk * GS_TOK);
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
                    const uint32_t fb = smem_u32(&full[stage]);
                    mbar_arrive_tx(fb, resw ? GS_X_BYTES : GS_W_BYTES + GS_X_BYTES);
                    tma_load_2d(smem_u32(sX + stage * GS_X_BYTES), &mapX, kb * GT_BK, row0, fb);
                    if (resw) {
                    } else if (wready) {
                        tma_load_2d(smem_u32(sW + stage * GS_W_BYTES), &mapW, kb * GT_BK, 0, fb);
                    } else if (++npend == ST) {
                        // stages 0..ST-1 hold k blocks 0..ST-1 of this CTA's first tile(s)
                        while (ld_acquire_gpu(ta.split_ready) < ta.nbuilders) { }
                        asm volatile("fence.proxy.async.global;" ::: "memory");   // generic writes -> TMA reads
                        for (int i = 0; i < ST; ++i)
                            tma_load_2d(smem_u32(sW + i * GS_W_BYTES), &mapW, (i % nk) * GT_BK, 0, smem_u32(&full[i]));
                        wready = true;
                        trace_clock(ta.trace, 4);
                    }
                    if (++stage == ST) { stage = 0; phase ^= 1; }
                }
            }
            if (!wready && npend) {
                while (ld_acquire_gpu(ta.split_ready) < ta.nbuilders) { }
                asm volatile("fence.proxy.async.global;" ::: "memory");
                for (int i = 0; i < npend; ++i)
                    tma_load_2d(smem_u32(sW + i * GS_W_BYTES), &mapW, (i % nk) * GT_BK, 0, smem_u32(&full[i]));
            }
            trace_clock(ta.trace, 5);
        }
    } else if (warp == 1) {
        // MMA issuer (one lane: this kernel's MMAs are few and wide -- one per 256 tokens x 16
        // columns -- and the whole-warp issuer of gate1_tc_kernel measured slower here,
        // 68 vs 64 us gate phase at C2)
        if (lane == 0) {
            const uint32_t idesc = make_idesc(128, GS_TOK);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;

            for (int tile = blockIdx.x; tile < ta.ntiles; tile += gridDim.x, ++it) {
                const int buf = it & 1;
                mbar_wait(smem_u32(&tempty[buf]), ((uint32_t)(it >> 1) & 1) ^ 1);
                tc_fence_after();
                if (it < 120) trace_clock(ta.trace, 8 + 2 * it);
                const uint32_t tmem_d = tmem_base + buf * GS_TOK;
                for (int kb = 0; kb < nk; ++kb) {
                    // the resident split is built in rounds of 256 columns (4 k blocks): the
                    // first tile's MMAs follow the build round by round
                    if (resw && it == 0 && (kb & 3) == 0) mbar_wait(smem_u32(&w_ready[kb >> 2]), 0);
                    mbar_wait(smem_u32(&full[stage]), phase);
                    tc_fence_after();
                    const uint64_t ad = sw128_desc(smem_u32(resw ? sW + (size_t)kb * ta.NPT * 128 : sW + stage * GS_W_BYTES));
                    const uint64_t bd = sw128_desc(smem_u32(sX + stage * GS_X_BYTES));
#pragma unroll
                    for (int k = 0; k < GT_BK / 16; ++k)
                        mma_bf16(tmem_d, ad + (uint64_t)(2 * k), bd + (uint64_t)(2 * k), idesc, (kb | k) ? 1u : 0u);
                    mma_commit(smem_u32(&empty[stage]));
                    if (++stage == ST) { stage = 0; phase ^= 1; }
                }
                mma_commit(smem_u32(&tfull[buf]));
                if (it < 120) trace_clock(ta.trace, 9 + 2 * it);
            }
        }
    } else if (warp >= 4) {
        // the exact three-piece split of W into wsplit ("quad10" rows: row 32 Q + w holds
        // piece w % 3 of logit 10 Q + w / 3 for w < 30, rows 30, 31 of each group zero)
        if (resw) {
            // ... or into this CTA's resident copy, in the SWIZZLE_128B K-major layout the MMA
            // reads (16-byte unit u of row r of a 64-column block at u ^ (r & 7))
            // Thread = column (up to kResWCols of them, d <= 256 kResWCols): all its router
            // entries are loaded first (one memory latency for the CTA's whole build), then its
            // NPT <= 64 rows are produced from registers (loops unrolled: static indices).
            __nv_bfloat16 *bs = reinterpret_cast<__nv_bfloat16 *>(sW);
            const int etid = threadIdx.x - 128, NPT = ta.NPT;
            float wv[kResWCols][kResWMaxKW];
#pragma unroll
            for (int ci = 0; ci < kResWCols; ++ci) {
                const int c = etid + 256 * ci;
#pragma unroll
                for (int k = 0; k < kResWMaxKW; ++k)
                    wv[ci][k] = (c < a.d && k < KW) ? __ldg(a.w + (int64_t)k * a.d + c) : 0.f;
            }
#pragma unroll
            for (int ci = 0; ci < kResWCols; ++ci) {
                const int c = etid + 256 * ci;
                if (256 * ci >= a.d) break;
                const int kb = c >> 6, u = (c & 63) >> 3;
                __nv_bfloat16 *col = bs + (size_t)kb * NPT * 64 + (c & 7);
#pragma unroll
                for (int r = 0; r < 2 * 32; ++r) {
                    if (r >= NPT || c >= a.d) break;     // (every warp still arrives below)
                    const int ww = r & 31, k = 10 * (r >> 5) + ww / 3, p = ww % 3;
                    float rem = (ww < 30 && k < KW) ? wv[ci][k] : 0.f;
                    for (int q = 0; q < p; ++q) rem -= __bfloat162float(__float2bfloat16_rn(rem));
                    col[(size_t)r * 64 + ((u ^ (r & 7)) << 3)] = __float2bfloat16_rn(rem);
                }
                // round ci (columns 256 ci .. 256 ci + 255 = k blocks 4 ci .. 4 ci + 3) is built
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor-core reads
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&w_ready[ci]));
            }
            if (threadIdx.x == 128) trace_clock(ta.trace, 6);
        } else if ((int)blockIdx.x < ta.nbuilders) {
            const int etid = threadIdx.x - 128;
            for (int r = blockIdx.x; r < ta.NPT; r += gridDim.x) {
                const int q = r >> 5, ww = r & 31;
                const int k = ww < 30 ? 10 * q + ww / 3 : KW, p = ww % 3;
                for (int c = etid; c < a.d; c += 256) {
                    float out = 0.f;
                    if (k < KW) {
                        float rem = __ldg(a.w + (int64_t)k * a.d + c);
                        for (int z = 0; z < p; ++z) rem -= __bfloat162float(__float2bfloat16_rn(rem));
                        out = rem;
                    }
                    ta.wsplit[(int64_t)r * a.d + c] = __float2bfloat16_rn(out);
                }
            }
            asm volatile("fence.proxy.async.global;" ::: "memory");
            __threadfence();
            EpiSync256<0>::sync();
            if (etid == 0) atomicAdd(ta.split_ready, 1);
            if (etid == 0) trace_clock(ta.trace, 6);
        }
        const int q = warp & 3, hc = (warp - 4) >> 2;    // TMEM lane quadrant, token-column half
        int it = 0;
        for (int tile = blockIdx.x; tile < ta.ntiles; tile += gridDim.x, ++it) {
            const int v = tile / a.nblk, blk = tile - v * a.nblk;
            const int64_t t0 = (int64_t)blk * GS_TOK;
            const int nt = (int)(a.T - t0 < GS_TOK ? a.T - t0 : GS_TOK);
            const int64_t tok0 = (int64_t)v * a.T + t0;
            const int buf = it & 1;
            mbar_wait(smem_u32(&tfull[buf]), (uint32_t)(it >> 1) & 1);
            tc_fence_after();
            const bool tr = threadIdx.x == 128 && it < 120;
            if (tr) trace_clock(ta.trace, 256 + 4 * it);
            if (q < NQ) {
                const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + buf * GS_TOK + hc * 128;
                const int k = 10 * q + lane / 3;
                const bool head = (lane % 3 == 0) && lane < 30 && k < KW;
                for (int c = 0; c < 4; ++c) {
                    float vv[32];
                    tmem_ld32(tb + c * 32, vv);
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float p1 = __shfl_down_sync(kFull, vv[j], 1);
                        const float p2 = __shfl_down_sync(kFull, vv[j], 2);
                        if (head) s_lg[(hc * 128 + c * 32 + j) * lds + k] = (vv[j] + p1) + p2;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&tempty[buf]));
            if (tr) trace_clock(ta.trace, 257 + 4 * it);
            EpiSync256<0>::sync();
            if (a.logits_out) {
                for (int i = EpiSync256<0>::tid(); i < nt * KW; i += 256)
                    a.logits_out[tok0 * KW + i] = s_lg[(i / KW) * lds + i % KW];
                EpiSync256<0>::sync();
            }
            gate_finish<EpiSync256<0>>(a, s_lg, lds, s_j, s_wh, s_bh, s_part, tok0, nt, (int64_t)tile,
                                       it < 100 ? ta.trace : nullptr, 600 + 4 * it);
            if (tr) trace_clock(ta.trace, 258 + 4 * it);
            if (ta.lb.on) lookback_scan<EpiSync256<0>>(a, ta.lb, s_bh, s_off, tile, epoch);
            EpiSync256<0>::sync();
            if (tr) trace_clock(ta.trace, 259 + 4 * it);
        }
    }
    pdl_trigger();
    __syncthreads();
    trace_end(ta.trace);
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
    }
    if (threadIdx.x == 0 && (ta.nbuilders > 0 || ta.lb.on)) {
        // every CTA is past its split wait and has read the epoch: the last one resets the
        // split counter and advances the look-back epoch for the next call
        __threadfence();
        if (atomicAdd(ta.done, 1) == (int)gridDim.x - 1) {
            *ta.split_ready = 0;
            *ta.done = 0;
            if (ta.lb.on) *ta.lb.epoch_ctr = epoch + 1;
            __threadfence();
        }
    }
}

size_t gate_tcT_smem(int KW, int K1, int K2, int stages, size_t resw_bytes = 0) {
    return 1024 + (resw_bytes ? resw_bytes + (size_t)stages * GS_X_BYTES : (size_t)stages * (GS_W_BYTES + GS_X_BYTES)) +
           ((size_t)GS_TOK * gate_lds(KW) + GS_TOK + 10 * K1) * 4 + 8 + gate_scratch_bytes(GS_TOK, KW, K2) + 8 +
           (2 * stages + 4 + kResWCols) * 8 + 16;
}

size_t gate_tc_smem(int NP, int KW, int K1, int K2, int stages, int nsub, int resident_b = 0, int d = 0) {
    const int groups = 2 * NP <= 512 ? 2 : 1;          // = nbuf
    const size_t grp_ints = ((gate_scratch_bytes(GT_BM, KW, K2) / 4 + (size_t)GT_BM * gate_lds(KW) + GT_BM + 6 * K1 + 1) &
                             ~(size_t)1);
    return 1024 + (size_t)stages * nsub * (GT_A_BYTES + (resident_b ? 0 : NP * GT_BK * 2)) +
           (resident_b ? (size_t)NP * d * 2 : 0) + 8 + groups * grp_ints * 4 + 8 + (2 * stages + 5) * 8 + 16;
}

}  // namespace

int gate_tc_np(int KW) { return ((3 * KW + 31) / 32) * 32; }

// The swapped-role kernel (256-token tiles) for KW <= 40 unless SMILE_GATE_SWAP=0.
bool gate_tc_swapped(int KW) {                // read at every smile_create
    const char *e = getenv("SMILE_GATE_SWAP");
    const bool on = !(e && e[0] == '0');
    return on && KW <= 40;
}

int gate_tc_rows(int KW) {                    // rows of the split-router buffer (both layouts)
    const int a = gate_tc_np(KW), b = 32 * ((KW + 9) / 10);
    return a > b ? a : b;
}

bool gate_tc_supported(int bf16, int d, int KW) {
    return bf16 && d % GT_BK == 0 && d >= GT_BK && gate_tc_np(KW) <= GT_MAX_NP && encode_fn() != nullptr;
}

cudaError_t launch_gate1_tc(const GateArgs &a, __nv_bfloat16 *wsplit, int num_sms, int *gate_sync, const Scan1Args *scan,
                            bool *scanned, cudaStream_t st) {
    if (scanned) *scanned = false;
    if (a.T == 0) return cudaSuccess;
    if (a.logits || !gate_tc_supported(a.bf16, a.d, a.KW)) return cudaErrorNotSupported;
    if (a.swapped) {
        if (a.TB != GS_TOK || a.fuse_dispatch || !gate_sync) return cudaErrorNotSupported;   // 256-token tiles
        const int NPT = 32 * ((a.KW + 9) / 10);
        CUtensorMap mX, mW;
        if (!make_map(&mX, a.x, (int64_t)a.V * a.T, a.d, GS_TOK)) return cudaErrorNotSupported;
        if (!make_map(&mW, wsplit, NPT, a.d, 128)) return cudaErrorNotSupported;    // rows >= NPT: zero fill
        GateTArgs ta;
        memset(&ta, 0, sizeof(ta));
        ta.g = a;
        ta.NPT = NPT;
        ta.ntiles = a.V * a.nblk;
        // resident split router when it is small (C2 / C3: 32 rows x 768 = 48 KB) and 4+ x
        // stages still fit; SMILE_GATE_RESW=0 streams it with x instead
        const char *rwe = getenv("SMILE_GATE_RESW");             // read per call (A/B, tests)
        const size_t rbytes = (size_t)NPT * a.d * 2;
        ta.resw = (!(rwe && rwe[0] == '0') && a.KW <= kResWMaxKW && a.d <= 256 * kResWCols && rbytes <= 64 * 1024 &&
                   gate_tcT_smem(a.KW, a.K1, a.K2, 4, rbytes) <= 227 * 1024) ? 1 : 0;
        int stages = 8;
        while (stages > 2 && gate_tcT_smem(a.KW, a.K1, a.K2, stages, ta.resw ? rbytes : 0) > 227 * 1024) --stages;
        ta.stages = stages;
        const size_t smem = gate_tcT_smem(a.KW, a.K1, a.K2, stages, ta.resw ? rbytes : 0);
        static bool attrT = false;
        if (!attrT) {
            cudaFuncSetAttribute(gate1_tcT_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
            attrT = true;
        }
        const int grid = ta.ntiles < num_sms ? ta.ntiles : num_sms;
        ta.nbuilders = ta.resw ? 0 : (NPT < grid ? NPT : grid);
        ta.trace = trace_buffer("gate");
        ta.split_ready = gate_sync; ta.done = gate_sync + 1;
        ta.wsplit = wsplit;
        // the level-1 scan by look-back inside the kernel: opt-in (SMILE_GATE_LOOKBACK=1) --
        // measured slower than the separate scan kernel (C2: 83-85 us vs 50 + 4.4 us, the
        // look-back waits stall the epilogue; profiles/r02_gate_schedule_ab.md)
        const char *lbe = getenv("SMILE_GATE_LOOKBACK");        // read per call (tests switch it)
        const int lb_env = (lbe && lbe[0] == '1') ? 1 : 0;   // opt-in: measured slower
        if (lb_env && scan && scan->lb_flag && scan->lb_inc && a.topk <= 1) {
            ta.lb.on = 1;
            ta.lb.s = *scan;
            ta.lb.flags = scan->lb_flag;
            ta.lb.epoch_ctr = gate_sync + 2;
        }
        const char *e2 = getenv("SMILE_GATE_SPLIT_KERNEL");      // 1: the separate split kernel (A/B)
        if (e2 && e2[0] == '1' && !ta.resw) {
            note_launch();
            launch_k(router_split_kernel, dim3((NPT * a.d + 255) / 256 < 1024 ? (NPT * a.d + 255) / 256 : 1024),
                     dim3(256), 0, st, a.w, wsplit, a.KW, a.d, NPT, 1);
            ta.nbuilders = 0;
        }
        note_launch();
        launch_k(gate1_tcT_kernel, dim3(grid), dim3(GS_THREADS), smem, st, mX, mW, ta);
        if (scanned) *scanned = ta.lb.on != 0;
        return cudaGetLastError();
    }
    if (a.TB != GT_BM) return cudaErrorNotSupported;
    const int NP = gate_tc_np(a.KW);
    // The split router is made once per call by router_split_kernel and streamed by TMA
    // with x.  SMILE_GATE_RESIDENT_B=1: small routers (<= 64 KB) are instead built by every
    // CTA in its own smem -- measured slower at C2 (69 vs ~45 us: each CTA's MMAs wait for
    // its ~10 us build, and a CTA only has ~7 tiles), so off by default.
    static int env_resb = -1;
    if (env_resb < 0) {
        const char *e = getenv("SMILE_GATE_RESIDENT_B");
        env_resb = (e && e[0] == '1') ? 1 : 0;
    }
    const int resb = (env_resb && (size_t)NP * a.d * 2 <= 64 * 1024) ? 1 : 0;
    if (!resb) {
        note_launch();
        launch_k(router_split_kernel, dim3((NP * a.d + 255) / 256 < 1024 ? (NP * a.d + 255) / 256 : 1024), dim3(256), 0,
                 st, a.w, wsplit, a.KW, a.d, NP, 0);
    }
    CUtensorMap mX, mW;
    if (!make_map(&mX, a.x, (int64_t)a.V * a.T, a.d, GT_BM)) return cudaErrorNotSupported;
    if (!make_map(&mW, wsplit, NP, a.d, NP > 256 ? NP / 2 : NP)) return cudaErrorNotSupported;
    GateTcArgs ta;
    memset(&ta, 0, sizeof(ta));
    ta.g = a;
    ta.NP = NP;
    ta.nbuf = 2 * NP <= 512 ? 2 : 1;
    ta.ntiles = a.V * a.nblk;
    ta.resident_b = resb;
    ta.trace = trace_buffer("gate");
    // two 64-column sub-blocks per stage when d allows and 3+ such stages fit (same box,
    // C2: 53-55 us vs 58-59 us with one; SMILE_GATE_NSUB=1 forces one)
    static int env_nsub = -1;
    if (env_nsub < 0) {
        const char *e = getenv("SMILE_GATE_NSUB");
        env_nsub = (e && e[0] == '1') ? 1 : 2;
    }
    ta.nsub = (env_nsub == 2 && a.d % (2 * GT_BK) == 0 &&
               gate_tc_smem(NP, a.KW, a.K1, a.K2, 3, 2, resb, a.d) <= 227 * 1024) ? 2 : 1;
    int stages = 8;
    while (stages > 2 && gate_tc_smem(NP, a.KW, a.K1, a.K2, stages, ta.nsub, resb, a.d) > 227 * 1024) --stages;
    ta.stages = stages;
    const size_t smem = gate_tc_smem(NP, a.KW, a.K1, a.K2, stages, ta.nsub, resb, a.d);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(gate1_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr = true;
    }
    const int grid = ta.ntiles < num_sms ? ta.ntiles : num_sms;
    // the level-1 scan by look-back inside the kernel (not with the fused permute, which has
    // its own look-back): opt-in SMILE_GATE_LOOKBACK=1, measured slower (C4 flat 1.77 ms)
    {
        const char *lbe = getenv("SMILE_GATE_LOOKBACK");
        const int lb_env = (lbe && lbe[0] == '1') ? 1 : 0;   // opt-in: measured slower
        if (lb_env && !a.fuse_dispatch && scan && scan->lb_flag && scan->lb_inc && gate_sync && a.topk <= 1) {
            ta.lb.on = 1;
            ta.lb.s = *scan;
            ta.lb.flags = scan->lb_flag;
            ta.lb.epoch_ctr = gate_sync + 2;
            ta.done = gate_sync + 1;
        }
    }
    note_launch();
    launch_k(gate1_tc_kernel, dim3(grid), dim3(GT_THREADS), smem, st, mX, mW, ta);
    if (scanned) *scanned = ta.lb.on != 0;
    return cudaGetLastError();
}

}  // namespace smile
