// k1_gate.cu -- K1: gate GEMV + SiLU + CATS threshold + ballot compaction.
//
// Paper: Eq. 1 x W_gate, Eq. 2 SiLU, Eq. 4/5 CATS_t,
// Custom GPU Kernel "MLP using CATS" lines 2-3 and App. D Alg. 1 line 4
// "idcs <- indices where Mask = 1". The paper builds idcs by atomic appends;
// here every tile of NR consecutive neurons is compacted by one warp ballot into its own segment of
// the index list: no atomics on the data, deterministic ascending order.
//
// B200 design (K1):
//  * W_gate (neuron-major [m][d]) is streamed HBM -> shared memory by the TMA bulk-copy engine
//    (cp.async.bulk + mbarrier transaction counts) into an S-stage ring; one stage = one tile of
//    NR rows. Every row is read exactly once: 2*d*m bytes per launch, the K1 roofline.
//  * Tiles are handed out dynamically (one global atomic per tile, prefetched one tile ahead) so SMs
//    that get more bandwidth take more tiles: no static-partition tail. Results do not depend on
//    which CTA processes a tile (each tile's dot products, SiLU and compaction are self-contained).
//  * Thread t owns 16-byte column chunks {t, t+NT, ...}; x stays in registers (fp32) and each thread
//    forms partial dots of its chunks; a fixed xor butterfly and a fixed-order cross-warp sum give u.
//    One __syncthreads per tile.
//
// Outputs (workspace, see api.cu): tile tau covers rows [tau*NR, tau*NR + NR); its cnt[tau] active
// rows are written at positions [tau*NR, tau*NR + cnt[tau]) of idx / tokmask / vals (vals = v in
// fp32, 0 where the token's |v| < t), ascending.
#include "cats_device.cuh"
#include "cats_internal.h"

namespace cats {

template <typename T, int B, int NR, int CPT>
__global__ void __launch_bounds__(kK1Threads, 1)
k1_gate_silu_cats_compact(const T *__restrict__ x, const T *__restrict__ Wg, int d, int m, int stages, float t,
                          int dense, int32_t *__restrict__ idx, uint8_t *__restrict__ tokmask,
                          float *__restrict__ vals, int32_t *__restrict__ cnt, float *__restrict__ acts,
                          unsigned int *__restrict__ sched) {
    constexpr int VEC = VecTraits<T>::kVec;
    constexpr int NT = kK1Threads;
    constexpr int NW = NT / 32;
    constexpr int NP = NR * B;  // (row, token) dot products per tile
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nch = d * (int)sizeof(T) / 16;
    const uint32_t row_bytes = (uint32_t)d * (uint32_t)sizeof(T);
    const uint32_t stage_bytes = (uint32_t)NR * row_bytes;
    const int ntiles = (m + NR - 1) / NR;

    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char *ring = smem;                                                          // [stages][NR][row]
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + (size_t)stages * stage_bytes);  // [stages]
    int *stile = reinterpret_cast<int *>(full + stages);                                 // [stages] tile ids
    float *red = reinterpret_cast<float *>(stile + stages);                              // [2][NW][NP]

    pdl_launch_dependents();

    // x -> registers (fp32), own chunks only
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

    // ---- producer state (thread 0): prefetched next tile id ----
    uint64_t policy = 0;
    unsigned int next_tile = 0;
    auto fill = [&](int s, unsigned int tile) {  // thread 0: stage s <- tile (or end marker)
        if (tile < (unsigned)ntiles) {
            const int r0 = (int)tile * NR;
            const int nr = min(NR, m - r0);
            stile[s] = (int)tile;
            mbar_arrive_expect_tx(&full[s], (uint32_t)nr * row_bytes);
            bulk_g2s(ring + (size_t)s * stage_bytes, Wg + (size_t)r0 * d, (uint32_t)nr * row_bytes, &full[s], policy);
        } else {
            stile[s] = -1;
            mbar_arrive_expect_tx(&full[s], 0u);
        }
    };
    if (tid == 0) {
        for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
        policy = l2_evict_first_policy();
        const unsigned int base = atomicAdd(&sched[0], (unsigned)stages);  // first `stages` tiles at once
        next_tile = atomicAdd(&sched[0], 1u);                              // prefetch: used at the next fill
        for (int s = 0; s < stages; ++s) fill(s, base + s);
    }
    __syncthreads();

    int s = 0;
    uint32_t phase = 0;
    for (int g = 0;; ++g) {
        mbar_wait(&full[s], phase);
        const int tile = stile[s];
        if (tile < 0) break;
        const int r0 = tile * NR;
        const int nr = min(NR, m - r0);
        const uint32_t sbase = smem_u32(ring + (size_t)s * stage_bytes);

        // ---- u = x W_gate[:, j]: own chunks of the tile's rows -> registers, partial dots ----
        uint4 wr[NR][CPT];
#pragma unroll
        for (int r = 0; r < NR; ++r)
#pragma unroll
            for (int k = 0; k < CPT; ++k) {
                const int ch = tid + k * NT;
                wr[r][k] = (r < nr && ch < nch) ? lds128(sbase + (uint32_t)r * row_bytes + (uint32_t)ch * 16u)
                                                : make_uint4(0u, 0u, 0u, 0u);
            }
        float part[NR][B];
#pragma unroll
        for (int r = 0; r < NR; ++r) {
#pragma unroll
            for (int tk = 0; tk < B; ++tk) part[r][tk] = 0.f;
#pragma unroll
            for (int k = 0; k < CPT; ++k) {
                float wf[VEC];
                unpack16(wr[r][k], wf);
#pragma unroll
                for (int tk = 0; tk < B; ++tk)
#pragma unroll
                    for (int e = 0; e < VEC; ++e) part[r][tk] = fmaf(xr[tk][k][e], wf[e], part[r][tk]);
            }
        }
        float *rb = red + (size_t)(g & 1) * NW * NP;
#pragma unroll
        for (int r = 0; r < NR; ++r)
#pragma unroll
            for (int tk = 0; tk < B; ++tk) {
                const float v = warp_allreduce_sum(part[r][tk]);
                if (lane == 0) rb[warp * NP + r * B + tk] = v;
            }
        __syncthreads();  // red[g&1] complete; every thread has read stage s -> refill it now
        if (tid == 0) {
            const unsigned int nt = next_tile;
            if (nt < (unsigned)ntiles) next_tile = atomicAdd(&sched[0], 1u);
            fill(s, nt);
        }

        // ---- warp 0: u -> v = SiLU(u) (Eq. 2) -> keep = |v| >= t (Eq. 4) -> compaction ----
        if (warp == 0) {
            // lane r < NR holds row r; tokens looped. Cross-warp sum in the fixed order w = 0..NW-1.
            uint32_t bits = 0;
            float vrow[B];
#pragma unroll
            for (int tk = 0; tk < B; ++tk) {
                float u = 0.f;
                if (lane < nr) {
#pragma unroll
                    for (int w = 0; w < NW; ++w) u += rb[w * NP + lane * B + tk];
                }
                const float v = u / (1.0f + __expf(-u));
                vrow[tk] = v;
                const bool keep = dense || (fabsf(v) >= t);
                bits |= (keep ? 1u : 0u) << tk;
                if (acts && lane < nr) acts[(size_t)tk * m + (size_t)(r0 + lane)] = v;
            }
            const bool act = (lane < nr) && bits != 0u;
            const uint32_t bal = __ballot_sync(0xffffffffu, act);
            if (act) {
                const int pos = r0 + __popc(bal & ((1u << lane) - 1u));
                idx[pos] = r0 + lane;
                tokmask[pos] = (uint8_t)bits;
#pragma unroll
                for (int tk = 0; tk < B; ++tk) vals[(size_t)pos * B + tk] = ((bits >> tk) & 1u) ? vrow[tk] : 0.0f;
            }
            if (lane == 0) cnt[tile] = __popc(bal);
        }
        if (++s == stages) { s = 0; phase ^= 1u; }
    }

    // ---- last CTA out resets the tile scheduler for the next launch ----
    if (tid == 0) {
        __threadfence();
        const unsigned int prev = atomicAdd(&sched[1], 1u);
        if (prev == gridDim.x - 1) {
            sched[0] = 0u;
            sched[1] = 0u;
            __threadfence();
        }
    }
}

size_t k1_smem_bytes(const PlanData &p, int b) {
    const int nr = k1_rows_per_tile(p, b);
    const int stages = k1_stages(p, b);
    size_t s = (size_t)stages * nr * (size_t)p.d * p.esize;
    s += (size_t)stages * 8 + (size_t)stages * 4;
    s = (s + 15) & ~(size_t)15;
    s += (size_t)2 * (kK1Threads / 32) * nr * b * 4;
    return (s + 127) & ~(size_t)127;
}

template <typename T, int B, int NR, int CPT>
static cudaError_t launch_k1_t(const PlanData &p, const void *x, const void *Wg, float t, int dense, float *acts,
                               void *ws, cudaStream_t s) {
    auto kern = k1_gate_silu_cats_compact<T, B, NR, CPT>;
    const size_t smem = k1_smem_bytes(p, B);
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void *>(kern), smem);
    if (e != cudaSuccess) return e;
    char *w = static_cast<char *>(ws);
    kern<<<p.g1, kK1Threads, smem, s>>>(static_cast<const T *>(x), static_cast<const T *>(Wg), p.d, p.m,
                                         k1_stages(p, B), t, dense, reinterpret_cast<int32_t *>(w + p.off_idx),
                                         reinterpret_cast<uint8_t *>(w + p.off_tokmask),
                                         reinterpret_cast<float *>(w + p.off_vals),
                                         reinterpret_cast<int32_t *>(w + p.off_cnt), acts,
                                         reinterpret_cast<unsigned int *>(w + p.off_sched));
    return cudaGetLastError();
}

template <typename T, int B, int NR>
static cudaError_t launch_k1_r(const PlanData &p, const void *x, const void *Wg, float t, int dense, float *acts,
                               void *ws, cudaStream_t s) {
    switch (p.cpt) {
        case 1: return launch_k1_t<T, B, NR, 1>(p, x, Wg, t, dense, acts, ws, s);
        case 2: return launch_k1_t<T, B, NR, 2>(p, x, Wg, t, dense, acts, ws, s);
        default: return cudaErrorInvalidValue;
    }
}

template <typename T, int B>
static cudaError_t launch_k1_c(const PlanData &p, const void *x, const void *Wg, float t, int dense, float *acts,
                               void *ws, cudaStream_t s) {
    constexpr int NR0 = k1_rows_per_tile_c(B);
    switch (k1_rows_per_tile(p, B)) {
        case NR0: return launch_k1_r<T, B, NR0>(p, x, Wg, t, dense, acts, ws, s);
        case (NR0 > 2 ? NR0 / 2 : 1): return launch_k1_r<T, B, (NR0 > 2 ? NR0 / 2 : 2)>(p, x, Wg, t, dense, acts, ws, s);
        case (NR0 > 4 ? NR0 / 4 : 0): return launch_k1_r<T, B, (NR0 > 4 ? NR0 / 4 : 2)>(p, x, Wg, t, dense, acts, ws, s);
        default: return cudaErrorInvalidValue;
    }
}

template <typename T>
static cudaError_t launch_k1_b(const PlanData &p, const void *x, int b, const void *Wg, float t, int dense,
                               float *acts, void *ws, cudaStream_t s) {
    switch (b) {
        case 1: return launch_k1_c<T, 1>(p, x, Wg, t, dense, acts, ws, s);
        case 2: return launch_k1_c<T, 2>(p, x, Wg, t, dense, acts, ws, s);
        case 3: return launch_k1_c<T, 3>(p, x, Wg, t, dense, acts, ws, s);
        case 4: return launch_k1_c<T, 4>(p, x, Wg, t, dense, acts, ws, s);
        case 5: return launch_k1_c<T, 5>(p, x, Wg, t, dense, acts, ws, s);
        case 6: return launch_k1_c<T, 6>(p, x, Wg, t, dense, acts, ws, s);
        case 7: return launch_k1_c<T, 7>(p, x, Wg, t, dense, acts, ws, s);
        case 8: return launch_k1_c<T, 8>(p, x, Wg, t, dense, acts, ws, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_k1(const PlanData &p, const void *x, int b, const void *Wg, float t, int dense, float *acts_out,
                      void *ws, cudaStream_t s) {
    if (p.dt == CATS_BF16) return launch_k1_b<bf16_bits>(p, x, b, Wg, t, dense, acts_out, ws, s);
    return launch_k1_b<float>(p, x, b, Wg, t, dense, acts_out, ws, s);
}

}  // namespace cats
