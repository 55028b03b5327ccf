// k1_gate.cu -- K1: gate GEMV + SiLU + CATS threshold + ballot/prefix compaction.
//
// Paper: Eq. 1 x W_gate, Eq. 2 SiLU, Eq. 4/5 CATS_t,
// Custom GPU Kernel "MLP using CATS" lines 2-3 and App. D Alg. 1 line 4
// "idcs <- indices where Mask = 1". The paper builds idcs by atomic appends;
// here each CTA owns a contiguous neuron range and compacts it with warp ballots + a CTA prefix
// sum: no atomics, deterministic ascending order.
//
// Work: every row of W_gate (neuron-major [m][d]) is read exactly once with 128-bit coalesced
// streaming loads (lane l of a warp reads 16-byte chunks l, l+32, ... of the row), dotted in fp32
// against x staged in shared memory, reduced with a fixed xor butterfly. HBM-bound: 2*d*m bytes
// (bf16) per launch, independent of the batch (K1 roofline).
//
// Outputs (workspace, see api.cu): for CTA c with rows [r0, r1) and cnt[c] active rows, entries
// [r0, r0 + cnt[c]) of idx / tokmask / vals hold the active neuron ids (ascending), their
// per-token keep bits, and v (fp32, 0 where the token's |v| < t) [row][b].
#include "cats_device.cuh"
#include "cats_internal.h"

namespace cats {

__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(bf16_bits v) { return bf16_to_f32(v); }

template <typename T, int B, int ROWS, int UNR>
__global__ void __launch_bounds__(kK1Threads, 1)
k1_gate_silu_cats_compact(const T *__restrict__ x, const T *__restrict__ Wg, int d, int m, int g1, int r_max,
                          float t, int dense, int32_t *__restrict__ idx, uint8_t *__restrict__ tokmask,
                          float *__restrict__ vals, int32_t *__restrict__ cnt, float *__restrict__ acts) {
    constexpr int VEC = VecTraits<T>::kVec;
    constexpr int NW = kK1Threads / 32;
    extern __shared__ __align__(16) unsigned char smem[];
    float *xs = reinterpret_cast<float *>(smem);                  // [B][d] fp32 copy of x
    float *sv = xs + (size_t)B * d;                               // [r_max][B]  v = SiLU(u)
    int *wsum = reinterpret_cast<int *>(sv + (size_t)r_max * B);  // [NW]
    uint8_t *sk = reinterpret_cast<uint8_t *>(wsum + NW);         // [r_max] keep bits per token

    // Let K2 get scheduled as soon as SMs free up; K2 blocks in griddepcontrol.wait until this
    // grid has completed and its writes are visible.
    pdl_launch_dependents();

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x;
    const int64_t r0 = k1_row0(c, m, g1);
    const int R = (int)(k1_row0(c + 1, m, g1) - r0);
    const int nch = d / VEC;

    for (int i = tid; i < B * d; i += kK1Threads) xs[i] = to_f32(x[i]);
    __syncthreads();

    // ---- u = x W_gate[:, j]  (one warp per ROWS rows; all loads of a UNR-batch in flight) ----
    for (int rl = warp * ROWS; rl < R; rl += NW * ROWS) {
        float acc[ROWS][B];
#pragma unroll
        for (int rr = 0; rr < ROWS; ++rr)
#pragma unroll
            for (int tk = 0; tk < B; ++tk) acc[rr][tk] = 0.f;

        for (int cb = 0; cb < nch; cb += 32 * UNR) {
            uint4 w[ROWS][UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const int ch = cb + u * 32 + lane;
#pragma unroll
                for (int rr = 0; rr < ROWS; ++rr) {
                    if (ch < nch && rl + rr < R)
                        w[rr][u] = ldg_stream(Wg + (size_t)(r0 + rl + rr) * d + (size_t)ch * VEC);
                    else
                        w[rr][u] = make_uint4(0u, 0u, 0u, 0u);
                }
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const int ch = cb + u * 32 + lane;
                if (ch < nch) {
                    float wf[ROWS][VEC];
#pragma unroll
                    for (int rr = 0; rr < ROWS; ++rr) unpack16(w[rr][u], wf[rr]);
#pragma unroll
                    for (int tk = 0; tk < B; ++tk) {
                        const float4 *xp = reinterpret_cast<const float4 *>(xs + (size_t)tk * d + (size_t)ch * VEC);
                        float xv[VEC];
#pragma unroll
                        for (int q = 0; q < VEC / 4; ++q) {
                            const float4 f = xp[q];
                            xv[4 * q + 0] = f.x; xv[4 * q + 1] = f.y; xv[4 * q + 2] = f.z; xv[4 * q + 3] = f.w;
                        }
#pragma unroll
                        for (int rr = 0; rr < ROWS; ++rr)
#pragma unroll
                            for (int e = 0; e < VEC; ++e) acc[rr][tk] = fmaf(xv[e], wf[rr][e], acc[rr][tk]);
                    }
                }
            }
        }
#pragma unroll
        for (int rr = 0; rr < ROWS; ++rr)
#pragma unroll
            for (int tk = 0; tk < B; ++tk) acc[rr][tk] = warp_allreduce_sum(acc[rr][tk]);

        // ---- v = SiLU(u) (Eq. 2); keep = |v| >= t (Eq. 4, ties kept) ----
#pragma unroll
        for (int rr = 0; rr < ROWS; ++rr) {
            const int r = rl + rr;
            if (r < R && lane == 0) {
                uint32_t bits = 0;
#pragma unroll
                for (int tk = 0; tk < B; ++tk) {
                    const float u = acc[rr][tk];
                    const float v = u / (1.0f + __expf(-u));
                    const bool keep = dense || (fabsf(v) >= t);
                    bits |= (keep ? 1u : 0u) << tk;
                    sv[(size_t)r * B + tk] = v;
                    if (acts) acts[(size_t)tk * m + (size_t)(r0 + r)] = v;
                }
                sk[r] = (uint8_t)bits;
            }
        }
    }
    __syncthreads();

    // ---- compaction of the union mask: ballot + CTA prefix, ascending neuron order ----
    int base = 0;
    for (int i0 = 0; i0 < R; i0 += kK1Threads) {
        const int i = i0 + tid;
        const uint32_t bits = (i < R) ? sk[i] : 0u;
        const bool f = bits != 0u;
        const uint32_t bal = __ballot_sync(0xffffffffu, f);
        const int wpre = __popc(bal & ((1u << lane) - 1u));
        if (lane == 0) wsum[warp] = __popc(bal);
        __syncthreads();
        int woff = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const int s = wsum[w];
            woff += (w < warp) ? s : 0;
            tot += s;
        }
        if (f) {
            const int64_t pos = r0 + base + woff + wpre;
            idx[pos] = (int32_t)(r0 + i);
            tokmask[pos] = (uint8_t)bits;
#pragma unroll
            for (int tk = 0; tk < B; ++tk)
                vals[(size_t)pos * B + tk] = ((bits >> tk) & 1u) ? sv[(size_t)i * B + tk] : 0.0f;
        }
        base += tot;
        __syncthreads();
    }
    if (tid == 0) cnt[c] = base;
}

size_t k1_smem_bytes(const PlanData &p, int b) {
    size_t s = (size_t)b * p.d * 4 + (size_t)p.r_max * b * 4 + (kK1Threads / 32) * 4 + (size_t)p.r_max;
    return (s + 15) & ~(size_t)15;
}

template <typename T, int B>
static cudaError_t launch_k1_t(const PlanData &p, const void *x, const void *Wg, float t, int dense, float *acts,
                               void *ws, cudaStream_t s) {
    constexpr int ROWS = B <= 2 ? 1 : (B <= 4 ? 2 : 4);
    constexpr int UNR = B <= 2 ? 16 : (B <= 4 ? 8 : 4);
    auto kern = k1_gate_silu_cats_compact<T, B, ROWS, UNR>;
    const size_t smem = k1_smem_bytes(p, B);
    static size_t configured = 0;  // per instantiation
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    char *w = static_cast<char *>(ws);
    kern<<<p.g1, kK1Threads, smem, s>>>(static_cast<const T *>(x), static_cast<const T *>(Wg), p.d, p.m, p.g1,
                                         p.r_max, t, dense, reinterpret_cast<int32_t *>(w + p.off_idx),
                                         reinterpret_cast<uint8_t *>(w + p.off_tokmask),
                                         reinterpret_cast<float *>(w + p.off_vals),
                                         reinterpret_cast<int32_t *>(w + p.off_cnt), acts);
    return cudaGetLastError();
}

template <typename T>
static cudaError_t launch_k1_b(const PlanData &p, const void *x, int b, const void *Wg, float t, int dense,
                               float *acts, void *ws, cudaStream_t s) {
    switch (b) {
        case 1: return launch_k1_t<T, 1>(p, x, Wg, t, dense, acts, ws, s);
        case 2: return launch_k1_t<T, 2>(p, x, Wg, t, dense, acts, ws, s);
        case 3: return launch_k1_t<T, 3>(p, x, Wg, t, dense, acts, ws, s);
        case 4: return launch_k1_t<T, 4>(p, x, Wg, t, dense, acts, ws, s);
        case 5: return launch_k1_t<T, 5>(p, x, Wg, t, dense, acts, ws, s);
        case 6: return launch_k1_t<T, 6>(p, x, Wg, t, dense, acts, ws, s);
        case 7: return launch_k1_t<T, 7>(p, x, Wg, t, dense, acts, ws, s);
        case 8: return launch_k1_t<T, 8>(p, x, Wg, t, dense, acts, ws, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_k1(const PlanData &p, const void *x, int b, const void *Wg, float t, int dense, float *acts_out,
                      void *ws, cudaStream_t s) {
    if (p.dt == CATS_BF16) return launch_k1_b<bf16_bits>(p, x, b, Wg, t, dense, acts_out, ws, s);
    return launch_k1_b<float>(p, x, b, Wg, t, dense, acts_out, ws, s);
}

}  // namespace cats
