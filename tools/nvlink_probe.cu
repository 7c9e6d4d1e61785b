// nvlink_probe.cu -- how fast can SM-issued row moves cross NVLink?  (measurement tool)
//
// Two GPUs in one process with peer access.  Each GPU moves R rows of `rb` bytes to the
// other (both directions at once, as in the layer's exchanges) with a scattered
// destination permutation, by:
//   simt-push  warp copies, 16-byte ld.global (local) -> st.global (peer)
//   simt-pull  warp copies, 16-byte ld.global (peer)  -> st.global (local)
//   tma-push   one thread per CTA: cp.async.bulk global -> smem (local), then
//              cp.async.bulk smem -> global (peer), NSLOT rows in flight
//   tma-pull   the same with the bulk loads from the peer and the stores local
//   ce         cudaMemcpyPeerAsync of the same bytes, contiguous (copy engines)
// Prints GB/s per direction (bytes one GPU sends / time of the slower GPU).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvlink_probe tools/nvlink_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

__global__ void simt_move(const char *__restrict__ src, char *__restrict__ dst, const int *__restrict__ perm,
                          int64_t R, int rb) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int nvec = rb / 16;
    for (int64_t r0 = gw * 4; r0 < R; r0 += warps * 4)
        for (int c0 = 0; c0 < nvec; c0 += 96) {
            int4 v[4][3];
            int64_t d[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t r = r0 + k;
                d[k] = r < R ? perm[r] : -1;
#pragma unroll
                for (int u = 0; u < 3; ++u) {
                    const int c = c0 + lane + 32 * u;
                    if (r < R && c < nvec) v[k][u] = reinterpret_cast<const int4 *>(src + r * rb)[c];
                }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int u = 0; u < 3; ++u) {
                    const int c = c0 + lane + 32 * u;
                    if (d[k] >= 0 && c < nvec) reinterpret_cast<int4 *>(dst + d[k] * rb)[c] = v[k][u];
                }
        }
}

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// TMA with a store ring: loads run NSLOT ahead; a slot is reused once the store issued
// from it NSLOT-1 stores ago has read smem (wait_group.read NSLOT-1 keeps the others flying).
template <int NSLOT>
__global__ void tma_move2(const char *__restrict__ src, char *__restrict__ dst, const int *__restrict__ perm,
                          int64_t R, int rb) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar[NSLOT];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < NSLOT; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int64_t per = (R + gridDim.x - 1) / gridDim.x;
    const int64_t b = blockIdx.x * per, e = b + per < R ? b + per : R;
    const int64_t n = e > b ? e - b : 0;
    for (int64_t k = 0; k < n + NSLOT; ++k) {
        // step k: store row k - NSLOT/2 ... keep it simple: load row k into slot k % NSLOT
        // after the store of row k - NSLOT (same slot) has read smem; store row k - NSLOT/2
        if (k < n) {
            if (k >= NSLOT) {
                // stores issued so far: rows 0 .. k - NSLOT/2 - 1; the one that used this slot
                // is row k - NSLOT, so at most NSLOT/2 - 1 younger stores may still be pending
                asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NSLOT / 2 - 1) : "memory");
            }
            const int s = (int)(k % NSLOT);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(rb)
                         : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             su32(sm + s * rb)),
                         "l"(src + (b + k) * rb), "r"(rb), "r"(su32(&bar[s]))
                         : "memory");
        }
        const int64_t j = k - NSLOT / 2;
        if (j >= 0 && j < n) {
            const int s = (int)(j % NSLOT);
            const uint32_t par = (uint32_t)((j / NSLOT) & 1);
            asm volatile(
                "{\n .reg .pred p;\n W2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W2;\n}" ::"r"(
                    su32(&bar[s])),
                "r"(par)
                : "memory");
            const int64_t drow = perm[b + j];
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + drow * rb),
                         "r"(su32(sm + s * rb)), "r"(rb)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char **argv) {
    const int64_t R = argc > 1 ? atoll(argv[1]) : 32768;
    const int rb = argc > 2 ? atoi(argv[2]) : 1536;
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (ndev < 2) {
        printf("needs 2 GPUs\n");
        return 0;
    }
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    char *buf[2][2];
    int *perm[2];
    cudaStream_t st[2];
    cudaEvent_t e0[2], e1[2];
    std::vector<int> hp(R);
    for (int64_t i = 0; i < R; ++i) hp[i] = (int)i;
    srand(1);
    for (int64_t i = R - 1; i > 0; --i) {
        const int64_t j = rand() % (i + 1);
        std::swap(hp[i], hp[j]);
    }
    for (int g = 0; g < 2; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaDeviceEnablePeerAccess(1 - g, 0));
        CK(cudaMalloc(&buf[g][0], R * rb));
        CK(cudaMalloc(&buf[g][1], R * rb));
        CK(cudaMemset(buf[g][0], g + 1, R * rb));
        CK(cudaMalloc(&perm[g], R * 4));
        CK(cudaMemcpy(perm[g], hp.data(), R * 4, cudaMemcpyHostToDevice));
        CK(cudaStreamCreate(&st[g]));
        CK(cudaEventCreate(&e0[g]));
        CK(cudaEventCreate(&e1[g]));
    }
    const double bytes = (double)R * rb;
    auto run = [&](const char *name, auto launch) {
        float best = 1e30f;
        for (int rep = 0; rep < 6; ++rep) {
            for (int g = 0; g < 2; ++g) {
                CK(cudaSetDevice(g));
                CK(cudaDeviceSynchronize());
            }
            for (int g = 0; g < 2; ++g) {
                CK(cudaSetDevice(g));
                CK(cudaEventRecord(e0[g], st[g]));
                launch(g);
                CK(cudaGetLastError());
                CK(cudaEventRecord(e1[g], st[g]));
            }
            float worst = 0.f;
            for (int g = 0; g < 2; ++g) {
                CK(cudaSetDevice(g));
                CK(cudaEventSynchronize(e1[g]));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
                worst = ms > worst ? ms : worst;
            }
            if (rep > 0 && worst < best) best = worst;
        }
        printf("%-28s %8.1f us  %7.1f GB/s per direction\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9);
    };
    // push: GPU g reads its buf[g][0], writes the peer's buf[1-g][1]; pull: reads the
    // peer's buf[1-g][0], writes its own buf[g][1]
    for (int mul : {1, 2, 4, 8}) {
        char nm[64];
        snprintf(nm, sizeof nm, "simt-push grid %dxSM", mul);
        run(nm, [&](int g) { simt_move<<<nsm * mul, 256, 0, st[g]>>>(buf[g][0], buf[1 - g][1], perm[g], R, rb); });
        snprintf(nm, sizeof nm, "simt-pull grid %dxSM", mul);
        run(nm, [&](int g) { simt_move<<<nsm * mul, 256, 0, st[g]>>>(buf[1 - g][0], buf[g][1], perm[g], R, rb); });
        snprintf(nm, sizeof nm, "simt-local grid %dxSM", mul);
        run(nm, [&](int g) { simt_move<<<nsm * mul, 256, 0, st[g]>>>(buf[g][0], buf[g][1], perm[g], R, rb); });
    }
    for (int g = 0; g < 2; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaFuncSetAttribute(tma_move2<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * rb));
        CK(cudaFuncSetAttribute(tma_move2<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * rb));
        CK(cudaFuncSetAttribute(tma_move2<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * rb));
    }
    for (int mul : {1, 2, 4}) {
        char nm[64];
        snprintf(nm, sizeof nm, "tma-push 16 slots %dxSM", mul);
        run(nm, [&](int g) { tma_move2<16><<<nsm * mul, 32, 16 * rb, st[g]>>>(buf[g][0], buf[1 - g][1], perm[g], R, rb); });
        snprintf(nm, sizeof nm, "tma-push 32 slots %dxSM", mul);
        run(nm, [&](int g) { tma_move2<32><<<nsm * mul, 32, 32 * rb, st[g]>>>(buf[g][0], buf[1 - g][1], perm[g], R, rb); });
        snprintf(nm, sizeof nm, "tma-pull 32 slots %dxSM", mul);
        run(nm, [&](int g) { tma_move2<32><<<nsm * mul, 32, 32 * rb, st[g]>>>(buf[1 - g][0], buf[g][1], perm[g], R, rb); });
        snprintf(nm, sizeof nm, "tma-local 32 slots %dxSM", mul);
        run(nm, [&](int g) { tma_move2<32><<<nsm * mul, 32, 32 * rb, st[g]>>>(buf[g][0], buf[g][1], perm[g], R, rb); });
    }
    run("tma-push 64 slots 1xSM", [&](int g) { tma_move2<64><<<nsm, 32, 64 * rb, st[g]>>>(buf[g][0], buf[1 - g][1], perm[g], R, rb); });
    run("ce memcpyPeer contiguous", [&](int g) {
        CK(cudaMemcpyPeerAsync(buf[1 - g][1], 1 - g, buf[g][0], g, R * rb, st[g]));
    });
    // one direction only (GPU 0 -> GPU 1) for reference
    {
        float best = 1e30f;
        for (int rep = 0; rep < 6; ++rep) {
            CK(cudaSetDevice(0));
            CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(e0[0], st[0]));
            simt_move<<<nsm * 4, 256, 0, st[0]>>>(buf[0][0], buf[1][1], perm[0], R, rb);
            CK(cudaEventRecord(e1[0], st[0]));
            CK(cudaEventSynchronize(e1[0]));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0[0], e1[0]));
            if (rep > 0 && ms < best) best = ms;
        }
        printf("%-28s %8.1f us  %7.1f GB/s (one direction only)\n", "simt-push 4xSM 0->1", best * 1e3,
               bytes / (best * 1e-3) / 1e9);
    }
    return 0;
}
