// FP64 pipe throughput probe: many independent DFMA chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void dlat_kernel(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x;
    for (int i = 0; i < iters; ++i) x0 = fma(x0, a, b);
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0;
}
int main() {
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, sizeof(double) * sms * 64 * 1024);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int iters = 1 << 16;
    for (int blocksPerSm : {4, 8, 16}) {
        int blocks = sms * blocksPerSm, threads = 256;
        dfma_kernel<<<blocks, threads>>>(out, 1024, 0.999, 0.001);
        cudaEventRecord(e0);
        dfma_kernel<<<blocks, threads>>>(out, iters, 0.999, 0.001);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = 8.0 * iters * blocks * threads;
        printf("dfma throughput: %d blocks/SM: %.3f T DFMA/s (%.1f TFLOP/s)\n", blocksPerSm, ops / ms / 1e9, 2 * ops / ms / 1e9);
    }
    dlat_kernel<<<1, 32>>>(out, 1024, 0.999, 0.001);
    cudaEventRecord(e0);
    dlat_kernel<<<1, 32>>>(out, iters, 0.999, 0.001);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int khz = 0; cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    printf("dependent DFMA latency: %.2f ns = %.1f cycles @ %d MHz\n", ms * 1e6 / iters, ms * 1e6 / iters * khz / 1e6, khz / 1000);
    return 0;
}
