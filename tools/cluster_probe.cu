// Probe: how many thread-block clusters of size 1/2/4/8 with ~201 KB smem and 640
// threads can be co-resident on this GPU (cudaOccupancyMaxActiveClusters).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_probe(int *p) { if (p) p[threadIdx.x] = 0; }
int main() {
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(sms / cs * cs);
        cfg.blockDim = dim3(640);
        cfg.dynamicSmemBytes = 201 * 1024;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_probe, &cfg);
        printf("cluster %2d: max active clusters %d (%d SMs busy of %d) %s\n", cs, n, n * cs, sms, cudaGetErrorString(e));
    }
    return 0;
}
