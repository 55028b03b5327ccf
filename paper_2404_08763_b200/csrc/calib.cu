// calib.cu -- K-cal: windowed histogram pass for the Eq. 3 threshold (radix-select style).
//
// Paper: Stage 1, Eq. 3: t = min{t' : F(t') >= k}, F the empirical CDF of
// |activations|. t is an order statistic of the |activations|, so it is found exactly by
// histogramming keys = |bit pattern| (sign cleared; for finite IEEE values the unsigned order of
// the key equals the order of |value|).
//
// One pass streams the activations once with 128-bit loads and, per element, only compares the
// key against a window [lo, hi]: keys below/above are counted in registers; keys inside go to a
// shared-memory histogram (bin = (key - lo) >> shift). A strided sample pass first aims the window
// at the rank, so the atomics touch ~1% of elements; the host step (api.cu) narrows the window until
// one key remains. NaN/Inf (key >= exponent-all-ones) are counted and rejected.
#include <algorithm>

#include "cats_device.cuh"
#include "cats_internal.h"

namespace cats {

constexpr int kCalThreads = 512;
constexpr int kCalUnroll = 8;

template <typename K> struct KeyTraits;
template <> struct KeyTraits<uint16_t> {  // bf16
    static constexpr int kPerVec = 8;
    static constexpr uint32_t kMask = 0x7fffu, kInf = 0x7f80u;
    __device__ static inline uint32_t key(const uint4 &r, int e) {
        const uint32_t w = (e >> 1) == 0 ? r.x : (e >> 1) == 1 ? r.y : (e >> 1) == 2 ? r.z : r.w;
        return ((e & 1) ? (w >> 16) : w) & kMask;
    }
};
template <> struct KeyTraits<uint32_t> {  // fp32
    static constexpr int kPerVec = 4;
    static constexpr uint32_t kMask = 0x7fffffffu, kInf = 0x7f800000u;
    __device__ static inline uint32_t key(const uint4 &r, int e) {
        const uint32_t w = e == 0 ? r.x : e == 1 ? r.y : e == 2 ? r.z : r.w;
        return w & kMask;
    }
};

template <typename K>
__global__ void __launch_bounds__(kCalThreads)
calib_hist_kernel(const K *__restrict__ acts, uint64_t n, uint32_t lo, uint32_t hi, uint32_t shift, uint32_t nbins,
                  uint64_t stride, unsigned long long *__restrict__ hist, unsigned long long *__restrict__ counts) {
    using KT = KeyTraits<K>;
    constexpr int E = KT::kPerVec;
    extern __shared__ uint32_t sh[];  // [nbins]
    __shared__ unsigned long long scount[4];
    for (uint32_t i = threadIdx.x; i < nbins; i += blockDim.x) sh[i] = 0u;
    if (threadIdx.x < 4) scount[threadIdx.x] = 0ull;
    __syncthreads();

    // Branch-free counters on the common path (no divergence); only keys inside the window (a small
    // fraction after the sample pass) take the histogram path. above = seen - below - inwin - nonfin.
    uint32_t below = 0, nonfin = 0, inwin = 0, seen = 0;
    uint32_t cur_bin = 0xffffffffu, cur_cnt = 0;  // run-length cache against same-bin contention
    const uint32_t span = hi - lo;
    auto classify_in = [&](uint32_t key) {  // key known to lie in [lo, hi]
        ++inwin;
        const uint32_t bin = (key - lo) >> shift;
        CATS_DCHECK(bin < nbins);
        if (bin == cur_bin) {
            ++cur_cnt;
        } else {
            if (cur_cnt) atomicAdd(&sh[cur_bin], cur_cnt);
            cur_bin = bin;
            cur_cnt = 1;
        }
    };
    auto classify = [&](uint32_t key) {
        below += key < lo ? 1u : 0u;
        nonfin += key >= KT::kInf ? 1u : 0u;
        const uint32_t rel = key - lo;  // unsigned: wraps for key < lo
        if (rel <= span) classify_in(key);
    };
    uint32_t seen_main = 0;

    const uint64_t nvec = n / E;
    const uint64_t nwork = stride ? (nvec + stride - 1) / stride : nvec;
    const uint4 *v4 = reinterpret_cast<const uint4 *>(acts);
    const uint64_t gstride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t step = stride ? stride : 1;
    // main loop: kCalUnroll independent 16-byte loads in flight per thread
    uint32_t nge2 = 0, kmax2 = 0;  // bf16 word path: keys >= lo, running max of the key pairs
    for (; i + (kCalUnroll - 1) * gstride < nwork; i += kCalUnroll * gstride) {
        uint4 r[kCalUnroll];
        if (step == 1) {  // full pass: no 64-bit multiply per load
#pragma unroll
            for (int u = 0; u < kCalUnroll; ++u) r[u] = ldg_stream(v4 + i + u * gstride);
        } else {
#pragma unroll
            for (int u = 0; u < kCalUnroll; ++u) r[u] = ldg_stream(v4 + (i + u * gstride) * step);
        }
        if constexpr (sizeof(K) == 2) {
            // two keys per 32-bit word, SIMD within the register: per 16-bit half,
            // (0x8000 + key) - lo has bit 15 set iff key >= lo, (0x8000 + hi) - key iff key <= hi
            // (no borrow crosses halves: both differences stay >= 1). ~6 instructions per key.
            const uint32_t lo2 = lo * 0x10001u;
            const uint32_t hi2x = (min(hi, KT::kMask) * 0x10001u) | 0x80008000u;
#pragma unroll
            for (int u = 0; u < kCalUnroll; ++u) {
                const uint32_t wv[4] = {r[u].x, r[u].y, r[u].z, r[u].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t gl = ((wv[q] | 0x80008000u) - lo2) & 0x80008000u;
                    nge2 += __popc(gl);
                    const uint32_t k2 = wv[q] & 0x7fff7fffu;
                    kmax2 = __vmaxu2(kmax2, k2);
                    const uint32_t iw = (hi2x - k2) & gl;
                    if (iw) {  // in-window keys: the minority once the sample pass aimed the window
                        if (iw & 0x8000u) classify_in(k2 & 0xffffu);
                        if (iw & 0x80000000u) classify_in(k2 >> 16);
                    }
                }
            }
        } else {
#pragma unroll
            for (int u = 0; u < kCalUnroll; ++u)
#pragma unroll
                for (int e = 0; e < E; ++e) classify(KT::key(r[u], e));
        }
        seen_main += kCalUnroll * E;
    }
    if constexpr (sizeof(K) == 2) {
        below += seen_main - nge2;
        // non-finite keys (always > hi) are flagged once per thread: CATS_CALIB_NONFINITE is then
        // nonzero iff any NaN/Inf was seen (the calibration is rejected; cats.h)
        nonfin += ((kmax2 & 0xffffu) >= KT::kInf || (kmax2 >> 16) >= KT::kInf) ? 1u : 0u;
    }
    seen += seen_main;
    for (; i < nwork; i += gstride) {
        const uint4 r = ldg_stream(v4 + i * step);
#pragma unroll
        for (int e = 0; e < E; ++e) classify(KT::key(r, e));
        seen += E;
    }
    // scalar tail (full passes only)
    if (!stride && blockIdx.x == 0) {
        for (uint64_t j = nvec * E + threadIdx.x; j < n; j += blockDim.x) {
            classify((uint32_t)acts[j] & KT::kMask);
            ++seen;
        }
    }
    const uint32_t above = seen - below - inwin - nonfin;
    if (cur_cnt) atomicAdd(&sh[cur_bin], cur_cnt);

    // block-reduce the register counters, one global atomic per counter per block
    const unsigned long long c4[4] = {below, inwin, above, nonfin};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        unsigned long long v = c4[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&scount[q], v);
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x)
        if (sh[b]) atomicAdd(&hist[b], (unsigned long long)sh[b]);
    if (threadIdx.x < 4 && scount[threadIdx.x]) atomicAdd(&counts[threadIdx.x], scount[threadIdx.x]);
}

// ---------------------------------------------------------------------------------------------
// Full-pass kernel: the data streams through a shared-memory ring fed by the TMA bulk-copy engine
// (cp.async.bulk + mbarrier), so the HBM stream never waits for the key arithmetic and the
// arithmetic never waits for HBM (the register-load loop above keeps 8 loads per thread in flight
// only between its compute phases). One producer warp claims 32 KB chunks from a global counter
// (dynamic: SMs with more bandwidth take more chunks) and keeps kCalStages of them in flight;
// 16 consumer warps classify the keys from shared memory. Bytes beyond the last whole chunk (and a
// sub-16-byte tail) are classified by CTA 0 straight from global memory.
constexpr int kCalStageBytes = 32 * 1024;
constexpr int kCalMaxStages = 6;
constexpr int kCalClaim = 4;  // chunks per claim
constexpr int kCalConsumerWarps = 16;
constexpr int kCalRegBins = 8;  // windows of <= 8 bins are counted in registers
constexpr int kCalTmaThreads = (kCalConsumerWarps + 1) * 32;

template <typename K>
__global__ void __launch_bounds__(kCalTmaThreads, 2)
calib_hist_tma_kernel(const K *__restrict__ acts, uint64_t n, uint32_t lo, uint32_t hi, uint32_t shift,
                      uint32_t nbins, int kCalStages, unsigned long long *__restrict__ hist,
                      unsigned long long *__restrict__ counts) {
    using KT = KeyTraits<K>;
    constexpr int E = KT::kPerVec;
    constexpr int NC = kCalConsumerWarps * 32;
    constexpr int VPT = kCalStageBytes / 16 / NC;  // 16-byte vectors per consumer thread per stage
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char *ring = smem;
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + (size_t)kCalStages * kCalStageBytes);
    uint64_t *empty = full + kCalStages;
    int *chunk_of = reinterpret_cast<int *>(empty + kCalStages);  // [kCalStages] chunk id per stage (-1 = end)
    uint32_t *sh = reinterpret_cast<uint32_t *>(chunk_of + kCalStages);  // [nbins]
    __shared__ unsigned long long scount[4];
    __shared__ unsigned int s_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (uint32_t i = tid; i < nbins; i += blockDim.x) sh[i] = 0u;
    if (tid < 4) scount[tid] = 0ull;
    if (tid == 0) {
        for (int s = 0; s < kCalStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kCalConsumerWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const uint64_t nbytes = n * sizeof(K);
    const uint64_t nchunks = nbytes / kCalStageBytes;
    unsigned int *ctr = reinterpret_cast<unsigned int *>(counts + 4);  // [0] chunk counter, [2] exit tickets

    uint32_t below = 0, nonfin = 0, inwin = 0, seen = 0;
    if (warp == kCalConsumerWarps) {
        // ---------------- producer: claim chunks, keep kCalStages bulk copies in flight ----------------
        if (lane == 0) {
            // chunks are claimed kCalClaim at a time, the next group's atomic in flight while the current
            // group streams (a blocking claim per chunk would put an L2 atomic round trip on every 32 KB)
            const uint64_t policy = l2_evict_first_policy();
            unsigned int grp = atomicAdd(ctr, (unsigned)kCalClaim);
            unsigned int nxt = atomicAdd(ctr, (unsigned)kCalClaim);
            int in_grp = 0;
            for (int j = 0;; ++j) {
                const int s = j % kCalStages;
                if (j >= kCalStages) mbar_wait(&empty[s], (uint32_t)((j / kCalStages) - 1) & 1u);
                if (in_grp == kCalClaim) {
                    grp = nxt;
                    in_grp = 0;
                    nxt = atomicAdd(ctr, (unsigned)kCalClaim);
                }
                const unsigned int c = grp + (unsigned)in_grp++;
                if ((uint64_t)c >= nchunks) {
                    chunk_of[s] = -1;
                    mbar_arrive_expect_tx(&full[s], 0u);  // END
                    break;
                }
                chunk_of[s] = (int)c;
                mbar_arrive_expect_tx(&full[s], (uint32_t)kCalStageBytes);
                bulk_g2s(ring + (size_t)s * kCalStageBytes, reinterpret_cast<const unsigned char *>(acts) +
                         (size_t)c * kCalStageBytes, (uint32_t)kCalStageBytes, &full[s], policy);
            }
        }
    } else {
        // ---------------- consumers ----------------
        // in-window keys: a window of <= kCalRegBins bins (the usual case: the sample pass aims it at a
        // key or two) is counted in registers (unrolled compare-adds, no shared atomics on a hot bin);
        // wider windows go to the shared-memory histogram with a run-length cache
        const bool regbins = nbins <= (uint32_t)kCalRegBins;
        uint32_t rc[kCalRegBins];
#pragma unroll
        for (int j = 0; j < kCalRegBins; ++j) rc[j] = 0u;
        uint32_t cur_bin = 0xffffffffu, cur_cnt = 0;
        const uint32_t span = hi - lo;
        auto classify_in = [&](uint32_t key) {
            ++inwin;
            const uint32_t bin = (key - lo) >> shift;
            CATS_DCHECK(bin < nbins);
            if (regbins) {
#pragma unroll
                for (int j = 0; j < kCalRegBins; ++j) rc[j] += bin == (uint32_t)j ? 1u : 0u;
            } else if (bin == cur_bin) {
                ++cur_cnt;
            } else {
                if (cur_cnt) atomicAdd(&sh[cur_bin], cur_cnt);
                cur_bin = bin;
                cur_cnt = 1;
            }
        };
        auto classify = [&](uint32_t key) {
            below += key < lo ? 1u : 0u;
            nonfin += key >= KT::kInf ? 1u : 0u;
            if (key - lo <= span) classify_in(key);
        };
        uint32_t nge2 = 0, kmax2 = 0, seen_main = 0;
        const uint32_t lo2 = lo * 0x10001u;
        const uint32_t hi2x = (min(hi, KT::kMask) * 0x10001u) | 0x80008000u;
        for (int j = 0;; ++j) {
            const int s = j % kCalStages;
            mbar_wait(&full[s], (uint32_t)(j / kCalStages) & 1u);
            if (chunk_of[s] < 0) break;
            const uint32_t sb = smem_u32(ring + (size_t)s * kCalStageBytes);
            uint4 r[VPT];
#pragma unroll
            for (int u = 0; u < VPT; ++u) r[u] = lds128(sb + (uint32_t)((u * NC + tid) * 16));
            if constexpr (sizeof(K) == 2) {
                // two keys per 32-bit word, SIMD within the register (see calib_hist_kernel)
                // (k2 + C1, C1 = 0x8000 - lo per half: bit 15 of a half set iff key >= lo, no carry across
                //  halves -- one ALU-pipe operation fewer than (w | 0x80008000) - lo2; the loop saturates the ALU pipe)
                const uint32_t C1 = 0x80008000u - lo2;
                uint32_t hit = 0;  // words holding an in-window key: handled after the sweep, from smem
#pragma unroll
                for (int u = 0; u < VPT; ++u) {
                    const uint32_t wv[4] = {r[u].x, r[u].y, r[u].z, r[u].w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t k2 = wv[q] & 0x7fff7fffu;
                        const uint32_t gl = (k2 + C1) & 0x80008000u;
                        nge2 += __popc(gl);
                        kmax2 = __vmaxu2(kmax2, k2);
                        hit |= ((hi2x - k2) & gl) ? (1u << (u * 4 + q)) : 0u;
                    }
                }
                while (hit) {  // rare: re-read the word from the (still owned) stage
                    const int wq = __ffs(hit) - 1;
                    hit &= hit - 1;
                    uint32_t w;
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w)
                                 : "r"(sb + (uint32_t)(((wq >> 2) * NC + tid) * 16 + (wq & 3) * 4)));
                    const uint32_t gl = ((w | 0x80008000u) - lo2) & 0x80008000u;
                    const uint32_t k2 = w & 0x7fff7fffu;
                    const uint32_t iw = (hi2x - k2) & gl;
                    if (iw & 0x8000u) classify_in(k2 & 0xffffu);
                    if (iw & 0x80000000u) classify_in(k2 >> 16);
                }
                seen_main += VPT * E;
            } else {
#pragma unroll
                for (int u = 0; u < VPT; ++u)
#pragma unroll
                    for (int e = 0; e < E; ++e) classify(KT::key(r[u], e));
                seen += VPT * E;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);  // stage consumed: the producer may refill it
        }
        if constexpr (sizeof(K) == 2) {
            below += seen_main - nge2;
            nonfin += ((kmax2 & 0xffffu) >= KT::kInf || (kmax2 >> 16) >= KT::kInf) ? 1u : 0u;
            seen += seen_main;
        }
        // bytes past the last whole chunk: CTA 0's consumers, from global memory
        if (blockIdx.x == 0) {
            const uint64_t e0 = nchunks * (kCalStageBytes / sizeof(K));
            for (uint64_t i = e0 + tid; i < n; i += NC) {
                classify((uint32_t)acts[i] & KT::kMask);
                ++seen;
            }
        }
        if (cur_cnt) atomicAdd(&sh[cur_bin], cur_cnt);
        if (regbins) {
#pragma unroll
            for (int j = 0; j < kCalRegBins; ++j) {
                uint32_t v = rc[j];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0 && v) atomicAdd(&sh[j], v);
            }
        }
    }
    const uint32_t above = seen - below - inwin - nonfin;
    const unsigned long long c4[4] = {below, inwin, above, nonfin};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        unsigned long long v = c4[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && v) atomicAdd(&scount[q], v);
    }
    __syncthreads();
    for (uint32_t b = tid; b < nbins; b += blockDim.x)
        if (sh[b]) atomicAdd(&hist[b], (unsigned long long)sh[b]);
    if (tid < 4 && scount[tid]) atomicAdd(&counts[tid], scount[tid]);
    // the last CTA re-arms the pass scratch (chunk counter, tickets) for the next pass
    if (tid == 0) s_last = atomicAdd(ctr + 4, 1u) == gridDim.x - 1 ? 1u : 0u;
    __syncthreads();
    if (s_last && tid == 0) {
        ctr[0] = 0u;
        ctr[4] = 0u;
    }
}

cudaError_t launch_calib_hist(const void *acts, uint64_t n, cats_dtype_t dt, const cats_calib_window_t &w,
                              uint64_t *hist, uint64_t *counts, cudaStream_t s) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = (size_t)w.nbins * 4;
    const int per_vec = dt == CATS_BF16 ? 8 : 4;
    const uint64_t nvec = n / per_vec;
    const uint64_t nwork = w.sample_stride ? (nvec + w.sample_stride - 1) / w.sample_stride : nvec;
    const int blocks_per_sm = smem <= 48 * 1024 ? 2 : 1;
    uint64_t want = (nwork + kCalThreads - 1) / kCalThreads;
    if (want < 1) want = 1;
    const int grid = (int)std::min<uint64_t>(want, (uint64_t)nsm * blocks_per_sm);
    auto *h = reinterpret_cast<unsigned long long *>(hist);
    auto *c = reinterpret_cast<unsigned long long *>(counts);
    // two CTAs per SM (two producers, 2 x 16 consumer warps), each with a ring of 32 KB stages
    const size_t bins_smem = w.nbins <= (uint32_t)kCalRegBins ? 64 : (size_t)w.nbins * 4;
    const size_t tbudget = 110 * 1024;
    const int tstages = bins_smem >= tbudget ? 0
                      : (int)std::min<size_t>(kCalMaxStages, (tbudget - bins_smem) / (kCalStageBytes + 20));
    if (!w.sample_stride && tstages >= 2 && (uint64_t)n * (dt == CATS_BF16 ? 2 : 4) >= (uint64_t)kCalStageBytes * nsm) {
        // full pass over a large buffer: the TMA-ring kernel, one CTA per SM
        const size_t tsmem = (size_t)tstages * (kCalStageBytes + 16 + 4) + (size_t)w.nbins * 4;
        const int tgrid = 2 * nsm;
        if (dt == CATS_BF16) {
            auto kern = calib_hist_tma_kernel<uint16_t>;
            cudaError_t e = ensure_smem_attr(reinterpret_cast<const void *>(kern), tsmem);
            if (e != cudaSuccess) return e;
            kern<<<tgrid, kCalTmaThreads, tsmem, s>>>(static_cast<const uint16_t *>(acts), n, w.lo, w.hi, w.shift,
                                                     w.nbins, tstages, h, c);
        } else {
            auto kern = calib_hist_tma_kernel<uint32_t>;
            cudaError_t e = ensure_smem_attr(reinterpret_cast<const void *>(kern), tsmem);
            if (e != cudaSuccess) return e;
            kern<<<tgrid, kCalTmaThreads, tsmem, s>>>(static_cast<const uint32_t *>(acts), n, w.lo, w.hi, w.shift,
                                                     w.nbins, tstages, h, c);
        }
        return cudaGetLastError();
    }
    if (dt == CATS_BF16) {
        auto kern = calib_hist_kernel<uint16_t>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        kern<<<grid, kCalThreads, smem, s>>>(static_cast<const uint16_t *>(acts), n, w.lo, w.hi, w.shift, w.nbins,
                                             w.sample_stride, h, c);
    } else {
        auto kern = calib_hist_kernel<uint32_t>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        kern<<<grid, kCalThreads, smem, s>>>(static_cast<const uint32_t *>(acts), n, w.lo, w.hi, w.shift, w.nbins,
                                             w.sample_stride, h, c);
    }
    return cudaGetLastError();
}

}  // namespace cats
