// cats_device.cuh -- device-side primitives shared by the libcats kernels (sm_100a only).
//
// 128-bit streaming loads, bf16 unpacking, mbarrier + cp.async.bulk (the TMA bulk-copy engine)
// wrappers, programmatic-dependent-launch controls and warp reductions. Nothing here knows about
// CATS; the method's arithmetic lives in mlp_fused.cu / mlp_split.cu / xsparse.cu / calib.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libcats is written for sm_100a (B200) only"
#endif

// Debug build (python -m paper_2404_08763_b200.build --debug -> libcats_debug.so): device-side bounds and
// invariant checks that trap on failure -- the pool's stand-in for compute-sanitizer, which is closed here.
#ifdef CATS_DEBUG_CHECKS
#include <cstdio>
#define CATS_DCHECK(cond)                                                                                   \
    do {                                                                                                    \
        if (!(cond)) {                                                                                      \
            printf("CATS_DCHECK failed %s:%d: %s (block %d, thread %d)\n", __FILE__, __LINE__, #cond,       \
                   (int)blockIdx.x, (int)threadIdx.x);                                                      \
            __trap();                                                                                       \
        }                                                                                                   \
    } while (0)
#else
#define CATS_DCHECK(cond) \
    do {                  \
    } while (0)
#endif

namespace cats {

using bf16_bits = uint16_t;  // bfloat16 stored as its bit pattern

template <typename T> struct VecTraits;
template <> struct VecTraits<float> { static constexpr int kVec = 4; };      // fp32 per 16 B
template <> struct VecTraits<bf16_bits> { static constexpr int kVec = 8; };  // bf16 per 16 B

__device__ __forceinline__ float bf16_to_f32(uint32_t bits16) { return __uint_as_float(bits16 << 16); }

// 16 bytes -> VEC fp32 values (exact widening)
__device__ __forceinline__ void unpack16(const uint4 &r, float (&f)[8]) {
    f[0] = __uint_as_float(r.x << 16); f[1] = __uint_as_float(r.x & 0xffff0000u);
    f[2] = __uint_as_float(r.y << 16); f[3] = __uint_as_float(r.y & 0xffff0000u);
    f[4] = __uint_as_float(r.z << 16); f[5] = __uint_as_float(r.z & 0xffff0000u);
    f[6] = __uint_as_float(r.w << 16); f[7] = __uint_as_float(r.w & 0xffff0000u);
}
__device__ __forceinline__ void unpack16(const uint4 &r, float (&f)[4]) {
    f[0] = __uint_as_float(r.x); f[1] = __uint_as_float(r.y);
    f[2] = __uint_as_float(r.z); f[3] = __uint_as_float(r.w);
}

// Streaming read-only 128-bit global load: bypass L1 allocation, mark the line evict-first in L2
// (weights are touched once per step).
__device__ __forceinline__ uint4 ldg_stream(const void *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

__device__ __forceinline__ uint4 lds128(uint32_t saddr) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(saddr));
    return r;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier (transaction-count barrier used by the bulk-copy engine) ----
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar_addr, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok) : "r"(bar_addr), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    while (!mbar_try_wait(a, parity)) {
    }
}

// cp.async.bulk global -> shared (TMA bulk engine, SASS UBLKCP), completion counted in bytes on
// the mbarrier. dst/src 16-byte aligned, bytes a multiple of 16. L2 evict-first policy: each
// weight row is read once per decode step.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s(void *dst_smem, const void *src, uint32_t bytes, uint64_t *bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_u32(dst_smem)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// ---- TMA bulk reduction shared -> global (SASS UBLKRED), bulk-group completion ----
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void bulk_reduce_add_u64(unsigned long long *gdst, const void *ssrc, uint32_t bytes) {
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u64 [%0], [%1], %2;"
                 ::"l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit_and_wait_all() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---- dot products on 16-byte chunks ----
// FHFMA.BF16 (fma.rn.f32.bf16) multiplies the bf16 halves of the packed registers directly: no
// unpack instructions, products exact, fp32 accumulation in element order (= unpack + FFMA).
// acc + sum_e w[e] * x[e] over one 16-byte chunk; products exact, fp32 accumulation in e order
template <typename T>
__device__ __forceinline__ float dot16(const uint4 &w, const uint4 &x, float acc);
template <>
__device__ __forceinline__ float dot16<bf16_bits>(const uint4 &w, const uint4 &x, float acc) {
    asm("{\n\t.reg .b16 a0, a1, b0, b1;\n\t"
        "mov.b32 {a0, a1}, %1;\n\tmov.b32 {b0, b1}, %5;\n\t"
        "fma.rn.f32.bf16 %0, a0, b0, %0;\n\tfma.rn.f32.bf16 %0, a1, b1, %0;\n\t"
        "mov.b32 {a0, a1}, %2;\n\tmov.b32 {b0, b1}, %6;\n\t"
        "fma.rn.f32.bf16 %0, a0, b0, %0;\n\tfma.rn.f32.bf16 %0, a1, b1, %0;\n\t"
        "mov.b32 {a0, a1}, %3;\n\tmov.b32 {b0, b1}, %7;\n\t"
        "fma.rn.f32.bf16 %0, a0, b0, %0;\n\tfma.rn.f32.bf16 %0, a1, b1, %0;\n\t"
        "mov.b32 {a0, a1}, %4;\n\tmov.b32 {b0, b1}, %8;\n\t"
        "fma.rn.f32.bf16 %0, a0, b0, %0;\n\tfma.rn.f32.bf16 %0, a1, b1, %0;\n\t}"
        : "+f"(acc)
        : "r"(w.x), "r"(w.y), "r"(w.z), "r"(w.w), "r"(x.x), "r"(x.y), "r"(x.z), "r"(x.w));
    return acc;
}
template <>
__device__ __forceinline__ float dot16<float>(const uint4 &w, const uint4 &x, float acc) {
    acc = fmaf(__uint_as_float(w.x), __uint_as_float(x.x), acc);
    acc = fmaf(__uint_as_float(w.y), __uint_as_float(x.y), acc);
    acc = fmaf(__uint_as_float(w.z), __uint_as_float(x.z), acc);
    acc = fmaf(__uint_as_float(w.w), __uint_as_float(x.w), acc);
    return acc;
}

// ---- programmatic dependent launch ----
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait_primary() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
template <int NTHREADS>
__device__ __forceinline__ void consumer_barrier() {  // named barrier 1: the consumer threads only
    asm volatile("bar.sync 1, %0;" ::"n"(NTHREADS) : "memory");
}

// ---- diagnostics: per-CTA %globaltimer stamps into the workspace trace area (null = off) ----
constexpr int kTraceCtas = 512, kTraceSlots = 8, kTraceKernels = 3;
__device__ __forceinline__ void trace_stamp(unsigned long long *tr, int kernel, int slot) {
    if (tr != nullptr && threadIdx.x == 0 && blockIdx.x < kTraceCtas) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        tr[((size_t)kernel * kTraceCtas + blockIdx.x) * kTraceSlots + slot] = t;
    }
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void trace_put(unsigned long long *tr, int kernel, int slot, unsigned long long v) {
    if (tr != nullptr && blockIdx.x < kTraceCtas) tr[((size_t)kernel * kTraceCtas + blockIdx.x) * kTraceSlots + slot] = v;
}

// ---- exact fixed point for order-independent (deterministic) accumulation ----
// A value y is accumulated as the integer q = round(y * 2^38) held in two int32 halves,
// q = hi * 2^30 + lo with lo kept in [0, 2^30). The caller pre-scales t = y * 2^8 (exact);
// hi += round(t) via the fp32 "magic number" trick (t + 1.5*2^23: full-rate FADD / IADD), the exact
// remainder f = t - round(t) (|f| <= 1/2) gives lo += round(f * 2^30) (|.| <= 2^29), and a carry
// renormalises lo after every add. Only f * 2^30 is rounded, so each add is exactly round(y * 2^38)
// (|t| < 2^21; larger |t| take a slow int64 path). Resolution 2^-38 (3.6e-12) absolute; range:
// |y| < 2^25 (3.4e7) for the int64 total, |partial of one thread| < 2^23.
constexpr int kFixLoBits = 30;
constexpr float kFixPre = 256.0f;                  // 2^8: callers pre-scale y by this (exact)
constexpr float kFixMagic = 12582912.0f;           // 1.5 * 2^23
constexpr int kFixMagicBits = 0x4B400000;
__device__ __forceinline__ void fix_acc(int &hi, int &lo, float t) {
    if (fabsf(t) < 2097152.0f) {  // 2^21
        const float h = t + kFixMagic;
        hi += __float_as_int(h) - kFixMagicBits;
        const float f = t - (h - kFixMagic);
        lo += __float2int_rn(f * 1073741824.0f);  // round(f * 2^30), |f| <= 1/2
    } else {
        const long long q = __float2ll_rn(t * 1073741824.0f);
        hi += (int)(q >> kFixLoBits);
        lo += (int)(q & ((1ll << kFixLoBits) - 1));
    }
    const int c = lo >> kFixLoBits;  // carry (floor): lo back into [0, 2^30)
    hi += c;
    lo -= c << kFixLoBits;
}
__device__ __forceinline__ long long fix_value(int hi, int lo) { return ((long long)hi << kFixLoBits) + lo; }
constexpr int kFixShift = 38;  // q is in units of 2^-38
// one correct rounding int64 -> fp32, then an exact power-of-two scale
__device__ __forceinline__ float fix_to_float(long long q) { return __ll2float_rn(q) * 3.637978807091713e-12f; }

// ---- warp reductions (fixed xor-butterfly: every lane ends with the same, order-fixed sum) ----
__device__ __forceinline__ float warp_allreduce_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace cats
