// Micro-benchmark: pinned host -> device copy rate with 1, 2 and 4 streams
// splitting the same bytes (does a second copy engine raise the H2D rate?).
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/h2d_rate.cu -o tools/_bin/h2d_rate
#include <cstdio>
#include <cuda_runtime.h>

int main() {
    const size_t total = 1ull << 30;
    char *h, *d;
    cudaHostAlloc(&h, total, cudaHostAllocDefault);
    cudaMalloc(&d, total);
    for (size_t i = 0; i < total; i += 4096) h[i] = 1;
    cudaStream_t s[4];
    for (auto& x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (size_t chunk : {size_t(2) << 20, size_t(64) << 20}) {
        for (int ns : {1, 2, 4}) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaDeviceSynchronize();
                cudaEventRecord(e0, s[0]);
                for (int k = 1; k < ns; ++k) cudaStreamWaitEvent(s[k], e0, 0);
                size_t i = 0;
                for (size_t off = 0; off < total; off += chunk, ++i)
                    cudaMemcpyAsync(d + off, h + off, chunk, cudaMemcpyHostToDevice, s[i % ns]);
                for (int k = 1; k < ns; ++k) {
                    cudaEvent_t ek;
                    cudaEventCreate(&ek);
                    cudaEventRecord(ek, s[k]);
                    cudaStreamWaitEvent(s[0], ek, 0);
                }
                cudaEventRecord(e1, s[0]);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep) printf("chunk %4zu MB, %d streams: %.2f GB/s\n", chunk >> 20, ns, total / (ms * 1e6));
            }
        }
    }
    return 0;
}
