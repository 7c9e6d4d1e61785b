// tiles.cuh -- device-side work list of the grouped expert GEMMs: prefix sums of the
// row tiles of every capacity-padded segment, computed from the device counts (no host
// sync).  Shared by ffn_simt.cu and ffn_tcgen05.cu.
#pragma once
#include <stdint.h>

namespace smile {

// s_pref[g] = sum_{g' < g} ceil(counts[g'] / BM), s_pref[nseg] = total; needs
// blockDim.x % 32 == 0, blockDim.x <= 1024 and s_warp[32].  Ends with __syncthreads().
template <int BM>
__device__ void tile_prefix(const int32_t *counts, int nseg, int *s_pref, int *s_warp) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int per = (nseg + nthr - 1) / nthr;
    const int beg = min(tid * per, nseg), end = min(beg + per, nseg);
    int local = 0;
    for (int g = beg; g < end; ++g) {
        const int c = counts[g];
        const int t = c > 0 ? (c + BM - 1) / BM : 0;
        s_pref[g] = t;
        local += t;
    }
    // inclusive warp scan of `local`
    const int lane = tid & 31, w = tid >> 5;
    int x = local;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    if (w == 0) {
        int z = lane < (nthr >> 5) ? s_warp[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= o) z += y;
        }
        if (lane < (nthr >> 5)) s_warp[lane] = z;     // inclusive per warp
    }
    __syncthreads();
    int run = x - local + (w > 0 ? s_warp[w - 1] : 0);   // exclusive start of this thread
    for (int g = beg; g < end; ++g) {
        const int t = s_pref[g];
        s_pref[g] = run;
        run += t;
    }
    if (tid == nthr - 1) s_pref[nseg] = run;
    __syncthreads();
}

// Strip work list of the grouped GEMMs: an expert's rows are its S segments' valid rows,
// cut into 32-row strips (a segment's last strip may be partial); a tile is SPT
// consecutive strips of one expert, so a tile can span segment boundaries and the
// padding between segments costs at most one partial strip per segment.
// Segment of (expert E = v * e + k, source s): g = (v * S + s) * e + k.
__device__ __forceinline__ int expert_strips(const int32_t *counts, int E, int S, int e) {
    const int v = E / e, k = E % e;
    int n = 0;
    for (int s = 0; s < S; ++s) n += (counts[(v * S + s) * e + k] + 31) / 32;
    return n;
}

// s_pref[E] = sum_{E' < E} ceil(strips(E') / SPT), s_pref[NE] = total tiles.  Same
// block-wide scan as tile_prefix; ends with __syncthreads().
template <int SPT>
__device__ void expert_tile_prefix(const int32_t *counts, int NE, int S, int e, int *s_pref, int *s_warp) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int per = (NE + nthr - 1) / nthr;
    const int beg = min(tid * per, NE), end = min(beg + per, NE);
    int local = 0;
    for (int E = beg; E < end; ++E) {
        const int t = (expert_strips(counts, E, S, e) + SPT - 1) / SPT;
        s_pref[E] = t;
        local += t;
    }
    const int lane = tid & 31, w = tid >> 5;
    int x = local;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    if (w == 0) {
        int z = lane < (nthr >> 5) ? s_warp[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, z, o);
            if (lane >= o) z += y;
        }
        if (lane < (nthr >> 5)) s_warp[lane] = z;
    }
    __syncthreads();
    int run = x - local + (w > 0 ? s_warp[w - 1] : 0);
    for (int E = beg; E < end; ++E) {
        const int t = s_pref[E];
        s_pref[E] = run;
        run += t;
    }
    if (tid == nthr - 1) s_pref[NE] = run;
    __syncthreads();
}

// Strip u (0-based, in segment order) of expert E: its first row in the [nseg, Cseg]
// row space and its valid rows (1..32); rows = 0 when the expert has fewer strips.
__device__ __forceinline__ void expert_strip(const int32_t *counts, int E, int S, int e, int64_t Cseg, int u,
                                             int64_t &row, int &rows) {
    const int v = E / e, k = E % e;
    for (int s = 0; s < S; ++s) {
        const int g = (v * S + s) * e + k;
        const int c = counts[g];
        const int ns = (c + 31) / 32;
        if (u < ns) {
            row = (int64_t)g * Cseg + 32 * u;
            rows = min(32, c - 32 * u);
            return;
        }
        u -= ns;
    }
    row = 0;
    rows = 0;
}

// Largest g with s_pref[g] <= mt (segments with zero tiles are skipped).
__device__ __forceinline__ int tile_segment(const int *s_pref, int nseg, int mt) {
    int lo = 0, hi = nseg;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_pref[mid] <= mt) lo = mid; else hi = mid;
    }
    return lo;
}

}  // namespace smile
