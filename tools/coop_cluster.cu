// Probe: can a cooperative launch also carry a cluster dimension, and how many
// clusters of 2/4/8 CTAs with ~225 KB smem each fit at once on this GPU?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a tools/coop_cluster.cu -o tools/_bin/coop_cluster
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(int* out) {
    extern __shared__ int s[];
    s[threadIdx.x] = threadIdx.x;
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(out, 1);
}

int main() {
    int* d;
    cudaMalloc(&d, 4);
    const int smem = 225 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg{};
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeCooperative;
        at[1].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(cs);
        int nclusters = -1;
        cudaError_t e0 = cudaOccupancyMaxActiveClusters(&nclusters, k, &cfg);
        const int grid = (148 / cs) * cs;
        cfg.gridDim = dim3(grid);
        cfg.numAttrs = 2;
        cudaMemset(d, 0, 4);
        cudaError_t e1 = cudaLaunchKernelEx(&cfg, k, d);
        cudaError_t e2 = cudaDeviceSynchronize();
        int h = 0;
        cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
        printf("cluster %2d: max active clusters %d (%s) -> %d CTAs; coop+cluster launch of %d: %s / %s, ran %d\n", cs,
               nclusters, cudaGetErrorString(e0), nclusters * cs, grid, cudaGetErrorString(e1),
               cudaGetErrorString(e2), h);
        cudaGetLastError();
    }
    return 0;
}
