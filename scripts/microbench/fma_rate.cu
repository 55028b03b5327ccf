// FMA-pipe throughput on this GPU: FFMA (3-reg), FFMA2 (fma.rn.f32x2), FHFMA.BF16 (fma.rn.f32.bf16),
// FFMA2 with a broadcast scalar. Prints FMAs per SM per clock (clock = %clock64 inside the kernel).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fma_rate fma_rate.cu && ./fma_rate
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096, kChains = 8;

template <int KIND>
__global__ void bench(float *out, unsigned long long *clk, float a0, float b0) {
    float acc[kChains][2];
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c][0] = acc[c][1] = threadIdx.x * 1e-7f + c;
    float a = a0 + threadIdx.x * 1e-9f, b = b0;
    unsigned int ab = __float_as_uint(a), bb = __float_as_uint(b);
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            if (KIND == 0) {
                acc[c][0] = fmaf(acc[c][0], a, b);
                acc[c][1] = fmaf(acc[c][1], b, a);
            } else if (KIND == 1) {
                unsigned long long v, x, y;
                asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "f"(acc[c][0]), "f"(acc[c][1]));
                asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a), "f"(b));
                asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(b), "f"(a));
                asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(v) : "l"(x), "l"(y));
                asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[c][0]), "=f"(acc[c][1]) : "l"(v));
            } else if (KIND == 2) {
                asm volatile("{.reg .b16 al, ah, bl, bh;\n\tmov.b32 {al, ah}, %2;\n\tmov.b32 {bl, bh}, %3;\n\t"
                             "fma.rn.f32.bf16 %0, al, bl, %0;\n\tfma.rn.f32.bf16 %1, ah, bh, %1;}"
                             : "+f"(acc[c][0]), "+f"(acc[c][1]) : "r"(ab), "r"(bb));
            } else {
                unsigned long long v, x;
                asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "f"(acc[c][0]), "f"(acc[c][1]));
                asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a), "f"(b));
                asm volatile("{.reg .b64 s;\n\tmov.b64 s, {%2, %2};\n\tfma.rn.f32x2 %0, %1, s, %0;}"
                             : "+l"(v) : "l"(x), "f"(b0));
                asm("mov.b64 {%0, %1}, %2;" : "=f"(acc[c][0]), "=f"(acc[c][1]) : "l"(v));
            }
        }
    }
    const unsigned long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += acc[c][0] + acc[c][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int KIND>
void run(const char *name, int sms, int ctas_per_sm, int threads) {
    const int grid = sms * ctas_per_sm;
    float *out;
    unsigned long long *clk;
    cudaMalloc(&out, (size_t)grid * threads * 4);
    cudaMalloc(&clk, grid * 8);
    bench<KIND><<<grid, threads>>>(out, clk, 1.0001f, 0.9999f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    bench<KIND><<<grid, threads>>>(out, clk, 1.0001f, 0.9999f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[4096];
    cudaMemcpy(h, clk, grid * 8, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
    const double fmas = (double)grid * threads * kIters * kChains * 2;
    printf("%-14s threads/SM %5d: %8.1f FMA/SM/clk (clock64), %6.2f TFMA/s (events, %.3f ms)\n", name,
           ctas_per_sm * threads, fmas / sms / (double)mx, fmas / (ms * 1e-3) / 1e12, ms);
    cudaFree(out);
    cudaFree(clk);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int tpsm : {256, 512, 1024}) {
        run<0>("FFMA", sms, 1, tpsm);
        run<1>("FFMA2", sms, 1, tpsm);
        run<2>("FHFMA.BF16", sms, 1, tpsm);
        run<3>("FFMA2.bcast", sms, 1, tpsm);
    }
    return 0;
}
