// Measured FP32 instruction-rate peak of this B200 (the denominator of the
// traversal's "alu" roofline): independent FFMA chains, 8 per thread, full
// occupancy, CUDA events.  Prints thread-level FFMA instructions per second.
// Build/run on the GPU box: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp32_peak tools/fp32_peak.cu && /tmp/fp32_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k_ffma(float* out, int iters, float a, float b) {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
            x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
        }
    }
    if (x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 == 12345.0f) out[0] = x0;  // keep the chains live
}

int main() {
    int sms = 0, dev = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    float* out;
    cudaMalloc(&out, 4);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    k_ffma<<<blocks, threads>>>(out, 16, 0.999f, 0.001f);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_ffma<<<blocks, threads>>>(out, iters, 0.999f, 0.001f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double inst = (double)blocks * threads * iters * 16 * 8;
        const double rate = inst / (ms * 1e-3);
        if (rate > best) best = rate;
    }
    printf("{\"fp32_ffma_inst_per_s\": %.4e, \"sms\": %d, \"clock_mhz_attr\": %d, \"nominal_at_1965\": %.4e}\n", best, sms,
           clk / 1000, 148.0 * 128 * 1965e6);
    return 0;
}
