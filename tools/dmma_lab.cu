// FP64 tensor-core (mma.sync m8n8k4 f64) issue-rate probe: W warps per CTA,
// one CTA per SM, NACC independent accumulators per warp, operands in registers.
// Usage: ./dmma_lab   (prints TFLOP/s per (W, NACC))
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int NACC>
__global__ void k(int iters, double* out, double a0, double b0) {
    double c[NACC][2];
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = 0.0;
    double a = a0 + threadIdx.x * 1e-9, b = b0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
}
template <int NACC>
void run(int W, int sms) {
    const int iters = 20000;
    double* out; cudaMalloc(&out, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<NACC><<<sms, 32 * W>>>(iters / 10, out, 1.0, 1.0);
    cudaEventRecord(e0);
    k<NACC><<<sms, 32 * W>>>(iters, out, 1.0, 1.0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double flop = 512.0 * NACC * iters * W * sms;
    printf("W=%2d NACC=%2d  %.3f ms  %.1f TFLOP/s\n", W, NACC, ms, flop / ms / 1e9);
    cudaFree(out);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int W : {4, 8, 16, 32}) { run<4>(W, sms); run<8>(W, sms); run<16>(W, sms); }
    return 0;
}
