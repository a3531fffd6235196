// How many clusters of 2/4/8 CTAs (one CTA per SM, ~200 KB smem each) can be
// co-resident on this GPU: the question behind a 4-CTA multicast cluster for
// the C3 kernel. Build: nvcc -arch=sm_100a -o /tmp/co tools/cluster_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) { extern __shared__ int s[]; if (p) p[0] = s[0]; }
int main() {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    printf("SMs %d\n", prop.multiProcessorCount);
    for (int smem_kb : {100, 200, 227}) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024);
        cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        for (int cs : {1, 2, 4, 8, 16}) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(cs * 64);
            cfg.blockDim = dim3(448);
            cfg.dynamicSmemBytes = smem_kb * 1024;
            cudaLaunchAttribute at;
            at.id = cudaLaunchAttributeClusterDimension;
            at.val.clusterDim.x = cs; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
            cfg.attrs = &at; cfg.numAttrs = 1;
            int n = -1;
            cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
            printf("smem %3d KB cluster %2d: %d clusters (%d SMs)%s%s\n", smem_kb, cs, n, n * cs,
                   e ? " err " : "", e ? cudaGetErrorString(e) : "");
        }
    }
    return 0;
}
