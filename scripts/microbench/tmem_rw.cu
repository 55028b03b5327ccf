// TMEM round trip check: per-warp lane-quarter stores (tcgen05.st 32x32b.x16) read back with tcgen05.ld
#include <cstdint>
__global__ void k(const uint32_t *in, uint32_t *out) {
    __shared__ uint32_t s_taddr;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        uint32_t sa = (uint32_t)__cvta_generic_to_shared(&s_taddr);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa), "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = s_taddr + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(warp >> 2) * 64u;
    uint32_t r[16];
    for (int i = 0; i < 16; ++i) r[i] = in[threadIdx.x * 16 + i];
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
                 ::"r"(base), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                   "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    uint32_t q[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
                 : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]),
                   "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15])
                 : "r"(base) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 16; ++i) out[threadIdx.x * 16 + i] = q[i];
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_taddr), "r"(512u));
}
#include <cstdio>
int main() {
    const int n = 256 * 16;
    uint32_t *a, *b; cudaMalloc(&a, n * 4); cudaMalloc(&b, n * 4);
    uint32_t h[n]; for (int i = 0; i < n; ++i) h[i] = i * 2654435761u;
    cudaMemcpy(a, h, n * 4, cudaMemcpyHostToDevice);
    k<<<148, 256>>>(a, b);
    cudaError_t e = cudaDeviceSynchronize();
    uint32_t g[n]; cudaMemcpy(g, b, n * 4, cudaMemcpyDeviceToHost);
    int bad = 0; for (int i = 0; i < n; ++i) bad += g[i] != h[i];
    printf("err=%s bad=%d\n", cudaGetErrorString(e), bad);
}
