// FP64 vector (DFMA) throughput of this GPU, the compute ceiling behind the
// step kernel's roofline discussion.  Independent FMA chains
// per thread, all SMs, CUDA-event timed.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && /tmp/fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 8;
constexpr int ITERS = 4096;

__global__ void k_dfma(double *out, double a, double b) {
    double x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;  // keep the chains live
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, 8);
    const int threads = 256, blocks = sms * 8;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_dfma<<<blocks, threads>>>(out, 0.999999, 1e-9);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int r = 0; r < reps; ++r) k_dfma<<<blocks, threads>>>(out, 0.999999, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fmas = (double)reps * blocks * threads * ITERS * CHAINS;
    printf("FP64 DFMA: %.2f TFLOP/s (2 flops per FMA) on %d SMs, %.3f ms per launch\n",
           2.0 * fmas / (ms * 1e-3) / 1e12, sms, ms / reps);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("per SM per cycle at the %.0f MHz attribute clock: %.1f DFMA\n", clk / 1e3,
           fmas / (ms * 1e-3) / sms / (clk * 1e3));
    return 0;
}
