// FMA-pipe microbenchmark: FFMA (scalar), FFMA2 (packed f32x2) and DFMA (FP64) with
// independent accumulator chains, to measure the SIMT FP32 roofline and the FP64
// roofline of the FP64-output option on B200.
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void k_ffma(float *out, float a, float b, int iters) {
    float acc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) acc[i] = fmaf(acc[i], a, b);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += acc[i];
    if (s == 12345.f) out[0] = s;
}

template <int NACC>
__global__ void k_ffma2(float *out, float a, float b, int iters) {
    float2 acc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    const float2 bb = make_float2(b, b);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) acc[i] = __ffma2_rn(acc[i], make_float2(a, a), bb);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += acc[i].x + acc[i].y;
    if (s == 12345.f) out[0] = s;
}

template <int NACC>
__global__ void k_dfma(double *out, double a, double b, int iters) {
    double acc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += acc[i];
    if (s == 12345.) out[0] = s;
}

int main() {
    float *d;
    cudaMalloc(&d, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000, threads = 512, blocks = sms * 4;
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        k_ffma<16><<<blocks, threads>>>(d, 0.999f, 1e-3f, 100);
        cudaEventRecord(e0);
        k_ffma<16><<<blocks, threads>>>(d, 0.999f, 1e-3f, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 16 * (double)iters * threads * blocks;
        printf("FFMA : %.1f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
        k_ffma2<8><<<blocks, threads>>>(d, 0.999f, 1e-3f, 100);
        cudaEventRecord(e0);
        k_ffma2<8><<<blocks, threads>>>(d, 0.999f, 1e-3f, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("FFMA2: %.1f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
        k_dfma<16><<<blocks, threads>>>((double *)d, 0.999, 1e-3, 100);
        cudaEventRecord(e0);
        k_dfma<16><<<blocks, threads>>>((double *)d, 0.999, 1e-3, iters / 4);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("DFMA : %.2f TFLOP/s (%.3f ms)\n", fl / 4 / ms / 1e9, ms);
    }
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("SMs %d, max clock %d MHz, nominal FP32 = %.1f TFLOP/s\n", sms, clk / 1000, sms * 128.0 * 2 * clk / 1e9);
    return 0;
}
