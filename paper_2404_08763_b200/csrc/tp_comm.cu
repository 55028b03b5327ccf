// tp_comm.cu -- one-shot cross-rank reduction of the tensor-parallel partials over NVLink peer memory
// (DESIGN.md §7).
//
// Tensor parallelism splits the intermediate dimension m into P contiguous neuron blocks; every rank's
// decode yields a partial y_p (b x d fp32) and y = sum_p y_p is the layer output (the one exchange step
// of the path; the threshold t is layer-global, so the masks need no communication -- Eq. 5 is per
// neuron). The paper measures one GPU and motivates removing synchronisation overhead
// (App. D); this is the B200 design of that exchange:
//
//   * every rank owns a symmetric buffer (same layout on all ranks, mapped into every peer's address
//     space with CUDA IPC over NVLink): per-CTA epoch counters, then two parity slots of world x n
//     8-byte words (value, epoch);
//   * ONE launch per call: CTA c takes slice c of the n values and pushes this rank's slice into slot
//     [epoch & 1][rank] of EVERY rank's buffer, each float in one 8-byte word with the call's epoch
//     (16-byte stores over NVLink, self included) -- the data is its own flag (no fences, no flag
//     round trip); every thread then polls its own words of each rank's row until they carry the epoch
//     and sums them in fixed rank order 0..P-1 -- the same additions in the same order on every rank,
//     so y is bit-identical across ranks;
//   * epochs are per CTA and live on the device (CUDA-graph safe); two parity slots make a call's pushes
//     land in the slot no rank can still be reading (a rank pushes call e+1 only after its call e saw
//     every rank's call-e data, i.e. after every rank finished call e-1).
//
// On one device (this pool) the P ranks are emulated as ONE cooperative launch over all ranks' data
// (blocks of virtual rank r = blockIdx.x / C), so the flag waits are between co-resident CTAs.
#include <cuda_runtime.h>

#include <cstring>
#include <new>

#include "cats_device.cuh"
#include "cats_internal.h"

namespace cats {

constexpr int kTpMaxWorld = 8;
constexpr int kTpThreads = 256;
constexpr int kTpMaxCtas = 64;
constexpr size_t kTpHeaderBytes = 256;  // per-CTA epochs ep[kTpMaxCtas], u32

struct TpLaunch {
    int world, ctas, nlocal, rank0;       // nlocal ranks handled by this launch: rank0 .. rank0 + nlocal - 1
    unsigned long long n, slot_floats;    // values per call, floats per (parity, rank) slot
    unsigned char *bufs[kTpMaxWorld][kTpMaxWorld];  // [local rank][peer]: peer's symmetric buffer as mapped here
    const float *x[kTpMaxWorld];          // [local rank] partial
    float *y[kTpMaxWorld];                // [local rank] output
};


__device__ __forceinline__ void st_volatile_v4(uint4 *p, const uint4 &v) {
    asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ uint4 ld_volatile_v4(const uint4 *p) {
    uint4 v;
    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p) : "memory");
    return v;
}

// Low-latency protocol: every pushed float travels with the call's epoch in the same 8-byte word
// (value bits, epoch), so a reader accepts a value exactly when its word carries the epoch -- no flags,
// no fences, no barrier between the push and the wait (each thread waits for its own words only).
// 8-byte words are written and read whole, so a word is either entirely this call's or stale.
__global__ void __launch_bounds__(kTpThreads) tp_allreduce_kernel(const __grid_constant__ TpLaunch L) {
    const int lr = blockIdx.x / L.ctas, c = blockIdx.x % L.ctas;  // local rank, slice
    const int me = L.rank0 + lr, W = L.world;
    unsigned char *const *bufs = L.bufs[lr];
    unsigned int *own_hdr = reinterpret_cast<unsigned int *>(bufs[me]);
    // slice of this CTA (16-byte aligned boundaries: n is a multiple of 4)
    const unsigned long long n4 = L.n / 4;
    const unsigned long long s0 = n4 * c / L.ctas, s1 = n4 * (c + 1) / L.ctas;
    CATS_DCHECK(lr < L.nlocal && me < W && s1 <= n4 && L.n <= L.slot_floats);
    __shared__ unsigned int s_ep;
    pdl_launch_dependents();  // the next layer's decode may start streaming its static W_gate tiles
    pdl_wait_primary();       // x (and this CTA's epoch word) may come from the kernels launched before us
    if (threadIdx.x == 0) s_ep = own_hdr[c] + 1u;  // this CTA's epoch (only CTA c of this rank writes ep[c])
    __syncthreads();
    const unsigned int ep = s_ep;
    if (threadIdx.x == 0) own_hdr[c] = ep;
    // slots: [parity][rank][slot_floats] of (value, epoch) 8-byte words
    const size_t slot_words = (size_t)L.slot_floats;
    const size_t slot_off = kTpHeaderBytes + (size_t)(ep & 1u) * W * slot_words * 8;
    // push: this rank's slice into slot [ep & 1][me] of every rank (NVLink stores; self is local)
    const float4 *x4 = reinterpret_cast<const float4 *>(L.x[lr]);
    for (unsigned long long i = s0 + threadIdx.x; i < s1; i += blockDim.x) {
        const float4 v = __ldcg(x4 + i);
        const uint4 lo = make_uint4(__float_as_uint(v.x), ep, __float_as_uint(v.y), ep);
        const uint4 hi = make_uint4(__float_as_uint(v.z), ep, __float_as_uint(v.w), ep);
        for (int r = 0; r < W; ++r) {
            uint4 *dst = reinterpret_cast<uint4 *>(bufs[r] + slot_off + (size_t)me * slot_words * 8) + 2 * i;
            st_volatile_v4(dst, lo);
            st_volatile_v4(dst + 1, hi);
        }
    }
    // y = sum over ranks in fixed order 0..W-1 (identical on every rank), each word once it carries the epoch
    const uint4 *slots = reinterpret_cast<const uint4 *>(bufs[me] + slot_off);
    float4 *y4 = reinterpret_cast<float4 *>(L.y[lr]);
    const size_t rstride = slot_words / 2;  // uint4 per rank row
    for (unsigned long long i = s0 + threadIdx.x; i < s1; i += blockDim.x) {
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int r = 0; r < W; ++r) {
            const uint4 *src = slots + (size_t)r * rstride + 2 * i;
            uint4 lo, hi;
            do {
                lo = ld_volatile_v4(src);
                hi = ld_volatile_v4(src + 1);
            } while (lo.y != ep || lo.w != ep || hi.y != ep || hi.w != ep);
            if (r == 0) {
                a = make_float4(__uint_as_float(lo.x), __uint_as_float(lo.z), __uint_as_float(hi.x), __uint_as_float(hi.z));
            } else {
                a.x += __uint_as_float(lo.x); a.y += __uint_as_float(lo.z);
                a.z += __uint_as_float(hi.x); a.w += __uint_as_float(hi.z);
            }
        }
        y4[i] = a;
    }
}

}  // namespace cats

using namespace cats;

struct cats_tp_comm {
    int rank, world, device, ctas;
    uint64_t n_max;
    unsigned char *bufs[kTpMaxWorld];  // every rank's symmetric buffer as mapped in this process
};

namespace {
inline cats_status_t cuda_status_tp(cudaError_t e) {
    if (e == cudaSuccess) return CATS_OK;
    set_last_cuda_error(e);
    return CATS_E_CUDA;
}
size_t tp_buffer_bytes(int world, uint64_t n) { return kTpHeaderBytes + 2 * (size_t)world * ((n + 3) / 4 * 4) * 8; }
int tp_ctas(uint64_t n) {  // ~1 KB of the call's values per CTA and slice, at most kTpMaxCtas
    const uint64_t c = (n + 255) / 256;
    return (int)(c < 1 ? 1 : c > (uint64_t)kTpMaxCtas ? kTpMaxCtas : c);
}
}  // namespace

extern "C" cats_status_t cats_tp_buffer_bytes(int world, uint64_t n_max, size_t *bytes) {
    if (!bytes) return CATS_E_NULL;
    if (world < 1 || world > kTpMaxWorld || n_max == 0 || n_max % 4) return CATS_E_SHAPE;
    *bytes = tp_buffer_bytes(world, n_max);
    return CATS_OK;
}

extern "C" cats_status_t cats_tp_buffer_alloc(size_t bytes, int device, void **dev_ptr_out) {
    if (!dev_ptr_out) return CATS_E_NULL;
    if (bytes == 0) return CATS_E_SHAPE;
    void *p = nullptr;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaMalloc(&p, bytes);  // its own allocation: an IPC handle maps exactly it
    if (e == cudaSuccess) e = cudaMemset(p, 0, bytes);  // epochs start at 0 (blocking)
    if (e != cudaSuccess) {
        if (p) cudaFree(p);
        return cuda_status_tp(e);
    }
    *dev_ptr_out = p;
    return CATS_OK;
}

extern "C" cats_status_t cats_tp_buffer_free(void *dev_ptr) {
    if (!dev_ptr) return CATS_E_NULL;
    return cuda_status_tp(cudaFree(dev_ptr));
}

extern "C" cats_status_t cats_ipc_handle_get(const void *dev_ptr, uint8_t *handle_out) {
    if (!dev_ptr || !handle_out) return CATS_E_NULL;
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void *>(dev_ptr));
    if (e != cudaSuccess) return cuda_status_tp(e);
    static_assert(sizeof(h) == CATS_IPC_HANDLE_BYTES, "cudaIpcMemHandle_t size");
    std::memcpy(handle_out, &h, sizeof h);
    return CATS_OK;
}

extern "C" cats_status_t cats_ipc_handle_open(const uint8_t *handle, int device, void **dev_ptr_out) {
    if (!handle || !dev_ptr_out) return CATS_E_NULL;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
    return cuda_status_tp(e);
}

extern "C" cats_status_t cats_ipc_handle_close(void *dev_ptr) {
    if (!dev_ptr) return CATS_E_NULL;
    return cuda_status_tp(cudaIpcCloseMemHandle(dev_ptr));
}

extern "C" cats_status_t cats_tp_comm_create(int rank, int world, uint64_t n_max, void *const *bufs, int device,
                                             cats_tp_comm_t **out) {
    if (!bufs || !out) return CATS_E_NULL;
    if (world < 1 || world > kTpMaxWorld || rank < 0 || rank >= world || n_max == 0 || n_max % 4) return CATS_E_SHAPE;
    for (int r = 0; r < world; ++r) {
        if (!bufs[r]) return CATS_E_NULL;
        if (reinterpret_cast<uintptr_t>(bufs[r]) & 15u) return CATS_E_ALIGN;
    }
    cats_tp_comm *c = new (std::nothrow) cats_tp_comm;
    if (!c) return CATS_E_CUDA;
    c->rank = rank;
    c->world = world;
    c->device = device;
    c->n_max = n_max;
    c->ctas = tp_ctas(n_max);
    for (int r = 0; r < kTpMaxWorld; ++r) c->bufs[r] = r < world ? static_cast<unsigned char *>(bufs[r]) : nullptr;
    *out = c;
    return CATS_OK;
}

extern "C" void cats_tp_comm_destroy(cats_tp_comm_t *comm) { delete comm; }

namespace {
cats_status_t tp_launch(cats_tp_comm_t *const *comms, int nlocal, const float *const *x, float *const *y, uint64_t n,
                        cudaStream_t s, bool cooperative) {
    const cats_tp_comm *c0 = comms[0];
    if (n == 0 || n % 4 || n > c0->n_max) return CATS_E_SHAPE;
    TpLaunch L{};
    L.world = c0->world;
    L.ctas = c0->ctas;
    L.nlocal = nlocal;
    L.rank0 = c0->rank;
    L.n = n;
    L.slot_floats = (c0->n_max + 3) / 4 * 4;
    for (int l = 0; l < nlocal; ++l) {
        const cats_tp_comm *c = comms[l];
        if (!c || !x[l] || !y[l]) return CATS_E_NULL;
        if (c->world != c0->world || c->n_max != c0->n_max || c->rank != c0->rank + l) return CATS_E_SHAPE;
        if ((reinterpret_cast<uintptr_t>(x[l]) | reinterpret_cast<uintptr_t>(y[l])) & 15u) return CATS_E_ALIGN;
        for (int r = 0; r < c->world; ++r) L.bufs[l][r] = c->bufs[r];
        L.x[l] = x[l];
        L.y[l] = y[l];
    }
    cudaError_t e = cudaSetDevice(c0->device);
    if (e != cudaSuccess) return cuda_status_tp(e);
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(nlocal * c0->ctas));
    cfg.blockDim = dim3(kTpThreads);
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cooperative) {  // emulated ranks wait on one another: co-residency guaranteed (or the launch fails)
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
    } else {            // one rank: start while the decode drains (programmatic dependent launch)
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
    }
    e = cudaLaunchKernelEx(&cfg, tp_allreduce_kernel, L);
    if (e == cudaSuccess) e = cudaGetLastError();
    return cuda_status_tp(e);
}
}  // namespace

extern "C" cats_status_t cats_tp_allreduce(const cats_tp_comm_t *comm, const float *x, float *y, uint64_t n,
                                           cats_stream_t s) {
    if (!comm || !x || !y) return CATS_E_NULL;
    cats_tp_comm_t *c = const_cast<cats_tp_comm_t *>(comm);
    return tp_launch(&c, 1, &x, &y, n, static_cast<cudaStream_t>(s), false);
}

extern "C" cats_status_t cats_tp_allreduce_emulated(cats_tp_comm_t *const *comms, int world, const float *const *x,
                                                    float *const *y, uint64_t n, cats_stream_t s) {
    if (!comms || !x || !y) return CATS_E_NULL;
    if (world < 1 || world > kTpMaxWorld) return CATS_E_SHAPE;
    for (int r = 0; r < world; ++r)
        if (!comms[r]) return CATS_E_NULL;
    if (comms[0]->rank != 0 || comms[0]->world != world) return CATS_E_SHAPE;
    return tp_launch(comms, world, x, y, n, static_cast<cudaStream_t>(s), true);
}
