// k2_sparse.cu -- K2: fused sparse up x v and down projection; K3: deterministic split-K reduce.
//
// Paper: Custom GPU Kernel "MLP using CATS" lines 4-5:
//     x1 <- (x W_up[Mask]) * v[Mask];   y <- x1 W_down[Mask]
// with Optimization 1, the x v multiply fused into the x W_up tile so x1 never touches HBM
// (P:305-306), and App. D eq. y = (v' * (x W'_up)) W'_down.
//
// B200 design (K2/K3):
//  * Only active neurons' rows of W_up and of the neuron-major W_down are read: each is one
//    contiguous 2d-byte row, moved HBM -> shared memory by the TMA bulk-copy engine
//    (cp.async.bulk + mbarrier transaction counts) into an S-stage ring, NS neurons per stage.
//  * The union active list produced by K1 (per-tile segments) is split into P equal, contiguous
//    slices, one per persistent CTA: static and balanced, so every CTA's partial sum has a fixed
//    composition (bit-reproducible y), and no atomics.
//  * Thread t owns fixed 16-byte column chunks {t, t+NT, ...} of d: it keeps x and its slice of the
//    y partial in registers. Per stage: partial up-dots, a fixed xor butterfly per warp, ONE
//    __syncthreads, then every warp forms the cross-warp sums itself (fixed tree; identical in all
//    warps), scales by v (Optimization 1) and does the down axpy from the staged W_down rows.
//  * The paper's fp16 tl.atomic_add into Y is replaced by a deterministic two-phase
//    split-K: each CTA writes its fp32 partial y_p, K3 sums the P partials in a fixed order.
#include "cats_device.cuh"
#include "cats_internal.h"

namespace cats {

template <typename T, int B, int CPT, int NS>
__global__ void __launch_bounds__(kK2Threads, 1)
k2_sparse_up_down(const T *__restrict__ x, const T *__restrict__ Wu, const T *__restrict__ Wd, int d, int m,
                  int ntiles, int tile_rows, int p2, int stages, int l_max, const int32_t *__restrict__ idx,
                  const float *__restrict__ vals, const int32_t *__restrict__ cnt, float *__restrict__ ypart) {
    constexpr int VEC = VecTraits<T>::kVec;
    constexpr int NT = kK2Threads;
    constexpr int NW = NT / 32;
    constexpr int NP = NS * B;
    static_assert(NW == 16, "cross-warp reduction assumes 16 warps");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int p = blockIdx.x;
    const int nch = d * (int)sizeof(T) / 16;
    const uint32_t row_bytes = (uint32_t)d * (uint32_t)sizeof(T);
    const uint32_t stage_bytes = (uint32_t)NS * 2u * row_bytes;

    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char *ring = smem;                                                          // [stages][NS][2][row]
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + (size_t)stages * stage_bytes);  // [stages]
    int *pref = reinterpret_cast<int *>(full + stages);                                  // [ntiles + 1]
    int *slist = pref + (ntiles + 1);                                                    // [l_max] neuron ids
    float *svals = reinterpret_cast<float *>(slist + l_max);                             // [l_max][B]
    float *red = svals + (size_t)l_max * B;                                              // [2][NW][NP]

    pdl_launch_dependents();

    if (tid == 0) {
        for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }

    // x -> registers (fp32), own chunks only. x is not written by K1, so this overlaps K1's tail.
    float xr[B][CPT][VEC];
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int ch = tid + k * NT;
#pragma unroll
        for (int tk = 0; tk < B; ++tk) {
            if (ch < nch) {
                unpack16(*reinterpret_cast<const uint4 *>(x + (size_t)tk * d + (size_t)ch * VEC), xr[tk][k]);
            } else {
#pragma unroll
                for (int e = 0; e < VEC; ++e) xr[tk][k][e] = 0.f;
            }
        }
    }

    // ---- wait for K1 (programmatic dependent launch) ----
    pdl_wait_primary();

    // exclusive prefix over K1's per-tile active counts -> union size U and this CTA's slice
    {
        const int per = (ntiles + NT - 1) / NT;
        const int lo = tid * per, hi = min(ntiles, lo + per);
        int s = 0;
        for (int i = lo; i < hi; ++i) s += cnt[i];
        // block exclusive scan of s (warp scan + warp totals)
        int inc = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
        }
        __shared__ int wtot[NW];
        if (lane == 31) wtot[warp] = inc;
        __syncthreads();
        int woff = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) woff += (w < warp) ? wtot[w] : 0;
        int run = woff + inc - s;
        for (int i = lo; i < hi; ++i) {
            pref[i] = run;
            run += cnt[i];
        }
        if (tid == NT - 1) pref[ntiles] = run;
    }
    __syncthreads();
    const int U = pref[ntiles];
    const int a0 = (int)((int64_t)p * U / p2), a1 = (int)((int64_t)(p + 1) * U / p2);
    const int L = a1 - a0;

    // gather the slice's neuron ids and v values (global position q -> K1 tile segment)
    for (int q = a0 + tid; q < a1; q += NT) {
        int lo = 0, hi = ntiles - 1;  // largest tile with pref[tile] <= q
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (pref[mid] <= q) lo = mid; else hi = mid - 1;
        }
        const int64_t pos = (int64_t)lo * tile_rows + (q - pref[lo]);
        slist[q - a0] = idx[pos];
#pragma unroll
        for (int tk = 0; tk < B; ++tk) svals[(size_t)(q - a0) * B + tk] = vals[(size_t)pos * B + tk];
    }
    __syncthreads();

    const int ngroups = (L + NS - 1) / NS;
    uint64_t policy = 0;
    auto issue = [&](int g) {  // thread 0 only
        const int s = g % stages;  // (once per stage refill)
        const int n_in = min(NS, L - g * NS);
        mbar_arrive_expect_tx(&full[s], (uint32_t)n_in * 2u * row_bytes);
        unsigned char *dst = ring + (size_t)s * stage_bytes;
        for (int i = 0; i < n_in; ++i) {
            const size_t j = (size_t)slist[g * NS + i];
            bulk_g2s(dst + (size_t)(2 * i) * row_bytes, Wu + j * d, row_bytes, &full[s], policy);
            bulk_g2s(dst + (size_t)(2 * i + 1) * row_bytes, Wd + j * d, row_bytes, &full[s], policy);
        }
    };
    if (tid == 0) {
        policy = l2_evict_first_policy();
        const int first = min(stages, ngroups);
        for (int g = 0; g < first; ++g) issue(g);
    }

    float yr[B][CPT][VEC];
#pragma unroll
    for (int tk = 0; tk < B; ++tk)
#pragma unroll
        for (int k = 0; k < CPT; ++k)
#pragma unroll
            for (int e = 0; e < VEC; ++e) yr[tk][k][e] = 0.f;

    int s = 0;
    uint32_t phase = 0;
    for (int g = 0; g < ngroups; ++g) {
        const int n_in = min(NS, L - g * NS);
        mbar_wait(&full[s], phase);
        const uint32_t sbase = smem_u32(ring + (size_t)s * stage_bytes);

        // ---- own chunks of the staged W_up and W_down rows -> registers (frees the stage early) ----
        uint4 wu[NS][CPT], wd[NS][CPT];
#pragma unroll
        for (int i = 0; i < NS; ++i)
#pragma unroll
            for (int k = 0; k < CPT; ++k) {
                const int ch = tid + k * NT;
                const bool ok = i < n_in && ch < nch;
                wu[i][k] = ok ? lds128(sbase + (uint32_t)(2 * i) * row_bytes + (uint32_t)ch * 16u) : make_uint4(0u, 0u, 0u, 0u);
                wd[i][k] = ok ? lds128(sbase + (uint32_t)(2 * i + 1) * row_bytes + (uint32_t)ch * 16u) : make_uint4(0u, 0u, 0u, 0u);
            }

        // ---- up: partial dots of x with this thread's chunks of each W_up row ----
        float part[NS][B];
#pragma unroll
        for (int i = 0; i < NS; ++i) {
#pragma unroll
            for (int tk = 0; tk < B; ++tk) part[i][tk] = 0.f;
#pragma unroll
            for (int k = 0; k < CPT; ++k) {
                float wf[VEC];
                unpack16(wu[i][k], wf);
#pragma unroll
                for (int tk = 0; tk < B; ++tk)
#pragma unroll
                    for (int e = 0; e < VEC; ++e) part[i][tk] = fmaf(xr[tk][k][e], wf[e], part[i][tk]);
            }
        }
        float *rb = red + (size_t)(g & 1) * NW * NP;
#pragma unroll
        for (int i = 0; i < NS; ++i)
#pragma unroll
            for (int tk = 0; tk < B; ++tk) {
                const float r = warp_allreduce_sum(part[i][tk]);
                if (lane == 0) rb[warp * NP + i * B + tk] = r;
            }
        __syncthreads();  // red[g&1] complete; every thread has read stage s -> refill it now
        if (tid == 0 && g + stages < ngroups) issue(g + stages);

        // ---- cross-warp sums, computed redundantly by every warp in one fixed tree:
        //      lane l reads warp (l & 15)'s partial of pair 2c + (l >> 4); xor 8,4,2,1 sums the 16.
        float a[NP];
#pragma unroll
        for (int c = 0; c < (NP + 1) / 2; ++c) {
            const int pp = 2 * c + (lane >> 4);
            float v = (pp < NP) ? rb[(lane & 15) * NP + pp] : 0.f;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            a[2 * c] = __shfl_sync(0xffffffffu, v, 0);
            if (2 * c + 1 < NP) a[2 * c + 1] = __shfl_sync(0xffffffffu, v, 16);
        }

        // ---- down: y_p += x1_j * W_down[j, own chunks], x1_j = (x W_up[j]) * v_j (Optimization 1) ----
#pragma unroll
        for (int i = 0; i < NS; ++i) {
            if (i < n_in) {
                float x1[B];
#pragma unroll
                for (int tk = 0; tk < B; ++tk) x1[tk] = a[i * B + tk] * svals[(size_t)(g * NS + i) * B + tk];
#pragma unroll
                for (int k = 0; k < CPT; ++k) {
                    float wf[VEC];
                    unpack16(wd[i][k], wf);
#pragma unroll
                    for (int tk = 0; tk < B; ++tk)
#pragma unroll
                        for (int e = 0; e < VEC; ++e) yr[tk][k][e] = fmaf(x1[tk], wf[e], yr[tk][k][e]);
                }
            }
        }
        if (++s == stages) { s = 0; phase ^= 1u; }
    }

    // ---- phase 1 output: this CTA's fp32 partial y_p[b][d] ----
    float *yp = ypart + (size_t)p * B * d;
#pragma unroll
    for (int tk = 0; tk < B; ++tk)
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            const int ch = tid + k * NT;
            if (ch < nch) {
                float4 *dst = reinterpret_cast<float4 *>(yp + (size_t)tk * d + (size_t)ch * VEC);
#pragma unroll
                for (int q = 0; q < VEC / 4; ++q)
                    dst[q] = make_float4(yr[tk][k][4 * q], yr[tk][k][4 * q + 1], yr[tk][k][4 * q + 2], yr[tk][k][4 * q + 3]);
            }
        }
}

// K3: y[b][d] = sum_{p=0}^{P-1} y_p[b][d] in a fixed order: lane l of the warp owning a float4
// column group adds p = l, l+32, ... sequentially (all loads issued up front), then a fixed xor
// butterfly. Bit-reproducible.
__global__ void __launch_bounds__(kK3Threads)
k3_splitk_reduce(const float4 *__restrict__ ypart, int p2, int n4, float4 *__restrict__ y) {
    constexpr int kMaxPerLane = 8;
    pdl_wait_primary();
    const int lane = threadIdx.x & 31;
    const int f = (int)((blockIdx.x * (size_t)kK3Threads + threadIdx.x) >> 5);
    if (f >= n4) return;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int base = 0; base < p2; base += 32 * kMaxPerLane) {
        float4 v[kMaxPerLane];
#pragma unroll
        for (int i = 0; i < kMaxPerLane; ++i) {
            const int pp = base + lane + 32 * i;
            v[i] = pp < p2 ? ypart[(size_t)pp * n4 + f] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < kMaxPerLane; ++i) {
            acc.x += v[i].x; acc.y += v[i].y; acc.z += v[i].z; acc.w += v[i].w;
        }
    }
    acc.x = warp_allreduce_sum(acc.x);
    acc.y = warp_allreduce_sum(acc.y);
    acc.z = warp_allreduce_sum(acc.z);
    acc.w = warp_allreduce_sum(acc.w);
    if (lane == 0) y[f] = acc;
}

size_t k2_smem_bytes(int esize, int d, int ns, int stages, int b, int l_max, int ntiles) {
    size_t s = (size_t)stages * ns * 2 * (size_t)d * esize;   // ring
    s += (size_t)stages * 8;                                   // mbarriers
    s += (size_t)(ntiles + 1) * 4;                             // prefix
    s += (size_t)l_max * 4 + (size_t)l_max * b * 4;            // slice ids + v
    s = (s + 15) & ~(size_t)15;
    s += (size_t)2 * (kK2Threads / 32) * ns * b * 4;           // cross-warp partials
    return (s + 127) & ~(size_t)127;
}

static cudaError_t launch_ex(const void *func, dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                             void **args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelExC(&cfg, func, args);
}

template <typename T, int B, int CPT, int NS>
static cudaError_t launch_k2_t(const PlanData &p, int b, const void *x, const void *Wu, const void *Wd, void *ws,
                               cudaStream_t s, bool pdl) {
    auto kern = k2_sparse_up_down<T, B, CPT, NS>;
    const int tile_rows = k1_rows_per_tile(p, b);
    int ntiles = k1_ntiles(p, b);
    int stages = k2_stages(p, b);
    const size_t smem = k2_smem_bytes((int)sizeof(T), p.d, NS, stages, B, p.l_max, ntiles);
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void *>(kern), smem);
    if (e != cudaSuccess) return e;
    char *w = static_cast<char *>(ws);
    const T *xp = static_cast<const T *>(x);
    const T *wu = static_cast<const T *>(Wu);
    const T *wd = static_cast<const T *>(Wd);
    int d = p.d, m = p.m, p2 = p.p2, l_max = p.l_max, tr = tile_rows;
    const int32_t *idx = reinterpret_cast<const int32_t *>(w + p.off_idx);
    const float *vals = reinterpret_cast<const float *>(w + p.off_vals);
    const int32_t *cnt = reinterpret_cast<const int32_t *>(w + p.off_cnt);
    float *ypart = reinterpret_cast<float *>(w + p.off_ypart);
    void *args[] = {&xp, &wu, &wd, &d, &m, &ntiles, &tr, &p2, &stages, &l_max, &idx, &vals, &cnt, &ypart};
    return launch_ex(reinterpret_cast<const void *>(kern), dim3(p.p2), dim3(kK2Threads), smem, s, pdl, args);
}

template <typename T, int B>
static cudaError_t launch_k2_b(const PlanData &p, const void *x, const void *Wu, const void *Wd, void *ws,
                               cudaStream_t s, bool pdl) {
    const bool ns4 = k2_neurons_per_stage(p, B) == 4;
    switch (p.cpt) {
        case 1: return ns4 ? launch_k2_t<T, B, 1, 4>(p, B, x, Wu, Wd, ws, s, pdl)
                           : launch_k2_t<T, B, 1, 2>(p, B, x, Wu, Wd, ws, s, pdl);
        case 2: return ns4 ? launch_k2_t<T, B, 2, 4>(p, B, x, Wu, Wd, ws, s, pdl)
                           : launch_k2_t<T, B, 2, 2>(p, B, x, Wu, Wd, ws, s, pdl);
        default: return cudaErrorInvalidValue;
    }
}

template <typename T>
static cudaError_t launch_k2_dt(const PlanData &p, const void *x, int b, const void *Wu, const void *Wd, void *ws,
                                cudaStream_t s, bool pdl) {
    switch (b) {
        case 1: return launch_k2_b<T, 1>(p, x, Wu, Wd, ws, s, pdl);
        case 2: return launch_k2_b<T, 2>(p, x, Wu, Wd, ws, s, pdl);
        case 3: return launch_k2_b<T, 3>(p, x, Wu, Wd, ws, s, pdl);
        case 4: return launch_k2_b<T, 4>(p, x, Wu, Wd, ws, s, pdl);
        case 5: return launch_k2_b<T, 5>(p, x, Wu, Wd, ws, s, pdl);
        case 6: return launch_k2_b<T, 6>(p, x, Wu, Wd, ws, s, pdl);
        case 7: return launch_k2_b<T, 7>(p, x, Wu, Wd, ws, s, pdl);
        case 8: return launch_k2_b<T, 8>(p, x, Wu, Wd, ws, s, pdl);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_k2(const PlanData &p, const void *x, int b, const void *Wu, const void *Wd, void *ws,
                      cudaStream_t s, bool pdl) {
    if (p.dt == CATS_BF16) return launch_k2_dt<bf16_bits>(p, x, b, Wu, Wd, ws, s, pdl);
    return launch_k2_dt<float>(p, x, b, Wu, Wd, ws, s, pdl);
}

cudaError_t launch_k3(const PlanData &p, int b, const void *ws, float *y, cudaStream_t s, bool pdl) {
    const char *w = static_cast<const char *>(ws);
    const float4 *ypart = reinterpret_cast<const float4 *>(w + p.off_ypart);
    int p2 = p.p2;
    int n4 = b * p.d / 4;
    float4 *y4 = reinterpret_cast<float4 *>(y);
    const int warps_per_block = kK3Threads / 32;
    const int grid = (n4 + warps_per_block - 1) / warps_per_block;
    void *args[] = {&ypart, &p2, &n4, &y4};
    return launch_ex(reinterpret_cast<const void *>(k3_splitk_reduce), dim3(grid), dim3(kK3Threads), 0, s, pdl,
                     args);
}

}  // namespace cats
