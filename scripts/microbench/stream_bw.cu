// stream_bw.cu -- read-bandwidth microbenchmark on B200: what a 117 MB weight stream can reach.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bw stream_bw.cu && ./stream_bw
// Variants: (A) LDG.128 warp-contiguous streaming, (B) cp.async.bulk ring into shared memory with
// consumers reading every byte from smem (1 CTA/SM, several stage sizes / depths), (C) same with
// 2 CTAs/SM. Each reported as GB/s over a buffer rotation that defeats L2.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint4 ldg_stream(const void *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

template <int UNR>
__global__ void ldg_kernel(const uint4 *__restrict__ a, size_t n16, unsigned *out) {
    unsigned acc = 0;
    size_t i = (size_t)blockIdx.x * blockDim.x * UNR + threadIdx.x;
    const size_t step = (size_t)gridDim.x * blockDim.x * UNR;
    for (; i < n16; i += step) {
        uint4 r[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            size_t j = i + (size_t)u * blockDim.x;
            r[u] = j < n16 ? ldg_stream(a + j) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) acc ^= r[u].x ^ r[u].y ^ r[u].z ^ r[u].w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// bulk ring: CTA takes tiles dynamically (atomic) of `tile` bytes; S stages; consumers XOR all smem.
__global__ void bulk_kernel(const char *__restrict__ a, size_t nbytes, uint32_t tile, int S, unsigned *ctr,
                            unsigned *out) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)S * tile);
    int *stile = reinterpret_cast<int *>(full + S);
    const unsigned ntiles = (unsigned)((nbytes + tile - 1) / tile);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    auto fill = [&](int s) {
        unsigned t = atomicAdd(ctr, 1u);
        if (t < ntiles) {
            stile[s] = t;
            uint32_t bytes = (uint32_t)min((size_t)tile, nbytes - (size_t)t * tile);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(bytes));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(smem + (size_t)s * tile)), "l"(a + (size_t)t * tile), "r"(bytes),
                         "r"(smem_u32(&full[s])) : "memory");
        } else {
            stile[s] = -1;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 0;" ::"r"(smem_u32(&full[s])));
        }
    };
    if (threadIdx.x == 0) for (int s = 0; s < S; ++s) fill(s);
    unsigned acc = 0;
    for (int g = 0;; ++g) {
        int s = g % S;
        uint32_t par = (g / S) & 1, ok = 0;
        while (!ok) {
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                         : "=r"(ok) : "r"(smem_u32(&full[s])), "r"(par) : "memory");
        }
        if (stile[s] < 0) break;
        const uint4 *p = reinterpret_cast<const uint4 *>(smem + (size_t)s * tile);
        for (uint32_t i = threadIdx.x; i < tile / 16; i += blockDim.x) { uint4 r = p[i]; acc ^= r.x ^ r.w; }
        __syncthreads();
        if (threadIdx.x == 0) fill(s);
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    const size_t chunk = 117440512;   // 117 MB: one Mistral W_gate
    const int ncopies = 8;
    char *buf;
    CK(cudaMalloc(&buf, chunk * ncopies));
    CK(cudaMemset(buf, 1, chunk * ncopies));
    unsigned *out, *ctr;
    CK(cudaMalloc(&out, 4));
    CK(cudaMalloc(&ctr, 64 * 16 * 4));
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char *name, auto launch) {
        for (int i = 0; i < 4; ++i) launch(i % ncopies);
        cudaDeviceSynchronize();
        const int reps = 40;
        cudaEventRecord(e0);
        for (int i = 0; i < reps; ++i) launch(i % ncopies);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double us = ms * 1e3 / reps;
        printf("%-44s %8.2f us  %7.1f GB/s\n", name, us, chunk / us / 1e3);
        cudaError_t err = cudaGetLastError();
        if (err != cudaSuccess) printf("  error %s\n", cudaGetErrorString(err));
    };
    const size_t n16 = chunk / 16;
    for (int threads : {256, 512, 1024}) {
        for (int bps : {1, 2, 4}) {
            if (threads * bps > 2048) continue;
            char name[128];
            snprintf(name, sizeof name, "LDG unr8 %d thr x %d CTA/SM", threads, bps);
            timeit(name, [&](int c) { ldg_kernel<8><<<nsm * bps, threads>>>((const uint4 *)(buf + c * chunk), n16, out); });
            snprintf(name, sizeof name, "LDG unr16 %d thr x %d CTA/SM", threads, bps);
            timeit(name, [&](int c) { ldg_kernel<16><<<nsm * bps, threads>>>((const uint4 *)(buf + c * chunk), n16, out); });
        }
    }
    for (uint32_t tile : {16384u, 32768u, 65536u}) {
        for (int S : {2, 3, 4, 6, 8, 12}) {
            for (int bps : {1, 2}) {
                size_t smem = (size_t)S * tile + S * 12 + 64;
                if (smem * bps > 228 * 1024 - 2048) continue;
                CK(cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                char name[128];
                snprintf(name, sizeof name, "bulk tile %uKB x %d stages, %d CTA/SM", tile / 1024, S, bps);
                int it = 0;
                CK(cudaMemset(ctr, 0, 64 * 16 * 4));
                timeit(name, [&](int c) {
                    bulk_kernel<<<nsm * bps, 512, smem>>>(buf + c * chunk, chunk, tile, S, ctr + 16 * (it++), out);
                });
            }
        }
    }
    return 0;
}
