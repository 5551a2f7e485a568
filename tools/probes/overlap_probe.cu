// Does a pinned H2D copy on one stream overlap a kernel on another on this box?
//   nvcc -O2 -arch=sm_100a overlap_probe.cu -o overlap_probe && ./overlap_probe
#include <cstdio>
#include <cuda_runtime.h>
__global__ void spin(float* x, long n, int reps) {
    for (int r = 0; r < reps; ++r)
        for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
            x[i] = x[i] * 0.999f + 1.f;
}
int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    printf("%s asyncEngineCount=%d concurrentKernels=%d unifiedAddressing=%d\n", p.name, p.asyncEngineCount,
           p.concurrentKernels, p.unifiedAddressing);
    const size_t bytes = 1ull << 30;
    float *h, *d, *w;
    cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
    cudaMalloc(&d, bytes);
    const long n = 1l << 28;
    cudaMalloc(&w, n * sizeof(float));
    cudaStream_t a, b;
    cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    auto time_it = [&](bool k, bool c) {
        cudaDeviceSynchronize();
        cudaEventRecord(e0, 0);
        if (k) spin<<<148 * 8, 256, 0, a>>>(w, n, 40);
        if (c) cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, b);
        cudaDeviceSynchronize();
        cudaEventRecord(e1, 0);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        return ms;
    };
    for (int rep = 0; rep < 2; ++rep)
        printf("kernel %.1f ms, copy %.1f ms, both %.1f ms\n", time_it(true, false), time_it(false, true),
               time_it(true, true));
    return 0;
}
