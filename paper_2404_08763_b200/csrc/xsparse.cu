// xsparse.cu -- App. B: CATS on the hidden vector before the attention projections.
//
//     y = CATS_t(x) W,   CATS_t(x)_i = x_i if |x_i| >= t else 0   (Eq. 4, on x itself)
//
// with W stored input-major [d_in][d_out] (row i = the weights input i feeds; q/k/v_proj.weight.T),
// so only the rows of inputs that survive the threshold are read from HBM: an input-sparse GEMV.
//
// ONE kernel (XS), launched as Q x R CTAs in clusters of R:
//   * every CTA thresholds x itself (b x d_in values, L2-resident after the first CTA) into a bitmask
//     of kept inputs (union over the b tokens) and scans it: the kept list is known to every CTA
//     without a second kernel or a global handshake;
//   * CTA (q, r) owns output columns [q*C, (q+1)*C) and the r-th of R equal ranges of the kept list;
//     its 8 warps stream the C-column segments of those rows (128-512 B each) with 16-byte
//     non-allocating loads, xs_unroll(b) rows in flight per thread, and accumulate y_part[b][C] in fp32
//     (measured: per-row cp.async.bulk copies of such short segments ran at ~0.6 TB/s chip-wide);
//   * the R partials of a column part are summed through distributed shared memory inside the
//     cluster in rank order: no workspace partials, no grid barrier, bit-identical y per input.
#include "cats_device.cuh"
#include "cats_internal.h"

namespace cats {

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void xs_mma_bf16(float (&dd)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                            uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
                 "{%8, %9}, {%0, %1, %2, %3};"
                 : "+f"(dd[0]), "+f"(dd[1]), "+f"(dd[2]), "+f"(dd[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void xs_ldsm_x4_trans(uint32_t saddr, uint32_t &r0, uint32_t &r1, uint32_t &r2,
                                                 uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(saddr)
                 : "memory");
}

// MT > 0: bf16 tensor-core main loop (C = 16 MT columns, b >= kXsMmaMinB); MT = 0: CUDA-core FFMA2
template <typename T, int B, int MT>
__global__ void __launch_bounds__(kXsThreads, 2)
xs_gemv(const T *__restrict__ x, const T *__restrict__ W, float *__restrict__ y, int d_in, int d_out, int C,
        float t, int maxr, uint8_t *__restrict__ kin, unsigned long long *__restrict__ trace) {
    constexpr int VEC = 16 / (int)sizeof(T);  // columns per 16-byte chunk
    constexpr int NW_ = kXsThreads / 32, UN = xs_unroll(B);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t rank = cluster_rank();
    uint32_t csize;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
    const int q = blockIdx.x / (int)csize;
    const int nch = C * (int)sizeof(T) / 16;  // threads per row segment (divides 32)
    const int G = kXsThreads / nch;           // rows in flight across the CTA per unroll slot
    const int NW = (d_in + 31) / 32;

    extern __shared__ __align__(128) unsigned char smem[];
    T *xs = reinterpret_cast<T *>(smem);                            // [B][d_in] staged x
    float *wred = reinterpret_cast<float *>(smem);                  // [NW_][B][C] per-warp partials (after xs)
    unsigned char *tiles = smem;                                    // MT > 0: [NW_][16][C + 8] bf16 (after xs)
    const size_t tile_bytes = MT > 0 ? (size_t)NW_ * 16 * (C * 2 + 16) : 0;
    const size_t a_bytes = (max((size_t)NW_ * B * C * 4, tile_bytes) + 15) & ~(size_t)15;
    float *slots = reinterpret_cast<float *>(smem + a_bytes);       // [R][B][C] rank partials (rank 0, after xs)
    const size_t region = max((size_t)B * d_in * sizeof(T), a_bytes + (size_t)csize * B * C * 4);
    uint32_t *kmask = reinterpret_cast<uint32_t *>(smem + ((region + 15) & ~(size_t)15));  // [NW]
    int *woff = reinterpret_cast<int *>(kmask + NW);                // [NW + 1]
    int *lj = woff + NW + 1;                                        // [maxr] kept inputs of this range
    // [maxr][LXS] CATS_t(x) of those inputs: bf16 (exact: x itself or 0) in pairs of tokens, or fp32
    constexpr int LXS = sizeof(T) == 2 ? (B + 1) & ~1 : B;
    T *lx = reinterpret_cast<T *>(lj + maxr);

    trace_stamp(trace, 0, 0);
    pdl_wait_primary();  // x comes from the predecessor; y may still be read by it
    pdl_launch_dependents();

    // ---- stage x (b x d_in, L2-resident after the first CTA) in shared memory ----
    if ((d_in * (int)sizeof(T)) % 16 == 0) {
        const uint4 *xv = reinterpret_cast<const uint4 *>(x);
        uint4 *xsv = reinterpret_cast<uint4 *>(xs);
        for (int v = tid; v < B * d_in / VEC; v += kXsThreads) xsv[v] = __ldg(xv + v);
    } else {
        for (int i = tid; i < B * d_in; i += kXsThreads) xs[i] = x[i];
    }
    __syncthreads();
    trace_stamp(trace, 0, 5);
    auto keep_bits = [&](int i) {  // bit tk: |x[tk][i]| >= t  (Eq. 4, ties kept: reading G1)
        uint32_t bits = 0;
#pragma unroll
        for (int tk = 0; tk < B; ++tk) {
            float v;
            if constexpr (sizeof(T) == 2) v = bf16_to_f32((uint32_t)xs[(size_t)tk * d_in + i]); else v = xs[(size_t)tk * d_in + i];
            bits |= (fabsf(v) >= t ? 1u : 0u) << tk;
        }
        return bits;
    };
    // ---- keep bits of every input (union over the b tokens) into 32-input words kmask[] ----
    const bool vec_x = (d_in * (int)sizeof(T)) % 16 == 0;
    if (vec_x) {  // 16-byte chunks of VEC inputs; the 32 / VEC lanes of one word OR their bits together
        constexpr int LPW = 32 / VEC;
        const int NV = d_in / VEC, nvp = (NW * 32 / VEC + 31) / 32 * 32;  // whole warps per pass
        const uint4 *xsv = reinterpret_cast<const uint4 *>(xs);
        for (int c = tid; c < nvp; c += kXsThreads) {
            uint32_t any = 0, tb[VEC];
#pragma unroll
            for (int e = 0; e < VEC; ++e) tb[e] = 0u;
            if (c < NV) {
#pragma unroll
                for (int tk = 0; tk < B; ++tk) {
                    float f[VEC];
                    unpack16(xsv[(size_t)tk * NV + c], f);
#pragma unroll
                    for (int e = 0; e < VEC; ++e) tb[e] |= (fabsf(f[e]) >= t ? 1u : 0u) << tk;  // Eq. 4, ties kept
                }
#pragma unroll
                for (int e = 0; e < VEC; ++e) any |= (tb[e] != 0u ? 1u : 0u) << e;
                if (blockIdx.x == 0)  // introspection (cats_mlp_last_active)
#pragma unroll
                    for (int e = 0; e < VEC; ++e) kin[(size_t)c * VEC + e] = (uint8_t)tb[e];
            }
            uint32_t wbits = any << ((c * VEC) & 31);
#pragma unroll
            for (int o = 1; o < LPW; o <<= 1) wbits |= __shfl_xor_sync(0xffffffffu, wbits, o);
            if ((lane & (LPW - 1)) == 0 && c * VEC < NW * 32) kmask[(c * VEC) >> 5] = wbits;
        }
    } else {  // ragged d_in: one input per thread, one ballot per word
        for (int i = tid; i < NW * 32; i += kXsThreads) {
            const uint32_t bits = i < d_in ? keep_bits(i) : 0u;
            if (blockIdx.x == 0 && i < d_in) kin[i] = (uint8_t)bits;
            const uint32_t bal = __ballot_sync(0xffffffffu, bits != 0u);
            if (lane == 0) kmask[i >> 5] = bal;
        }
    }
    __syncthreads();
    trace_stamp(trace, 0, 6);
    // ---- exclusive prefix of the word popcounts, block-wide, 256 words per pass:
    //      woff[w] = kept inputs before word w, woff[NW] = U ----
    __shared__ int wsum[kXsThreads / 32];
    __shared__ int s_wr[2];
    int carry = 0, my_off = 0, my_pc = 0;  // my_*: word tid (kept when NW fits one pass)
    for (int base = 0; base < NW; base += kXsThreads) {
        const int w = base + tid;
        const int pc = w < NW ? __popc(kmask[w]) : 0;
        int incl = pc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        int before = carry;
#pragma unroll
        for (int k = 0; k < NW_; ++k) before += k < warp ? wsum[k] : 0;
        if (w < NW) woff[w] = before + incl - pc;
        my_off = before + incl - pc;
        my_pc = pc;
#pragma unroll
        for (int k = 0; k < NW_; ++k) carry += wsum[k];
        __syncthreads();
    }
    if (tid == 0) woff[NW] = carry;
    trace_stamp(trace, 0, 7);
    // ---- this CTA's range [lo, hi) of the kept list (equal split into csize ranges): the words
    //      [wa, we) that hold its first and last kept input, then one thread per input of those ----
    const long long U = carry;
    const int lo = (int)(U * rank / csize), hi = (int)(U * (rank + 1) / csize), len = hi - lo;
    int wa = 0, we = 0;
    if (NW <= kXsThreads) {  // the owning threads know it from the prefix pass
        if (tid < NW && my_pc > 0) {
            if (my_off <= lo && lo < my_off + my_pc) s_wr[0] = tid;
            if (my_off <= hi - 1 && hi - 1 < my_off + my_pc) s_wr[1] = tid + 1;
        }
        __syncthreads();
        wa = s_wr[0];
        we = s_wr[1];
    } else {  // binary searches on woff: last word with woff <= lo, first word with woff >= hi
        int a = 0, b2 = NW;
        while (b2 - a > 1) {
            const int mid = (a + b2) >> 1;
            if (woff[mid] <= lo) a = mid; else b2 = mid;
        }
        wa = a;
        a = 0, b2 = NW;
        while (b2 - a > 1) {
            const int mid = (a + b2) >> 1;
            if (woff[mid] < hi) a = mid; else b2 = mid;
        }
        we = a + 1;
    }
    if (len == 0) wa = we = 0;
    trace_stamp(trace, 1, 0);
    const int iend = min(we * 32, d_in);
#pragma unroll 2
    for (int i = wa * 32 + tid; i < iend; i += kXsThreads) {
        const int w = i >> 5;
        const uint32_t m = kmask[w];
        if (!((m >> (i & 31)) & 1u)) continue;
        const int gi = woff[w] + __popc(m & ((1u << (i & 31)) - 1u));
        if (gi < lo || gi >= hi) continue;
        lj[gi - lo] = i;
#pragma unroll
        for (int tk = 0; tk < LXS; ++tk) {  // CATS_t(x) per token (Eq. 4); the pad token is 0
            const T xv = tk < B ? xs[(size_t)tk * d_in + i] : T(0);
            float v;
            if constexpr (sizeof(T) == 2) v = bf16_to_f32((uint32_t)xv); else v = xv;
            lx[(size_t)(gi - lo) * LXS + tk] = fabsf(v) >= t ? xv : T(0);
        }
    }
    trace_stamp(trace, 1, 1);
    __syncthreads();
    trace_stamp(trace, 1, 2);
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");  // this CTA is done with xs

    trace_stamp(trace, 0, 1);
    // ---- acc[tk][e] += CATS_t(x)[tk][i] * W[i][col]: thread (g, ch) takes rows g, g + G, ... of the
    //      range in list order, UN rows' 16-byte chunks in flight ----
    const int g = tid / nch, ch = tid % nch;
    if constexpr (MT > 0) {
        // ---- tensor cores: warp w takes 16-row groups w, w + 8, ... of the range; a group's C-column
        //      segments go through the warp's shared-memory tile (zero rows past the range), A = W^T by
        //      ldmatrix .trans, B = CATS_t(x) (exact bf16), D[16 cols x 8 tokens] in fp32; the next
        //      group's loads are issued before this group's MMAs ----
        static_assert(sizeof(T) == 2, "MMA path is bf16");
        constexpr int NL = MT;  // 16-byte chunks per lane per group: 16 rows x 2 MT chunks / 32 lanes
        const int ng = (len + 15) / 16;
        const uint32_t tst = (uint32_t)C * 2u + 16u;  // padded row stride: conflict-free ldmatrix
        const uint32_t tile = smem_u32(tiles) + (uint32_t)warp * 16u * tst;
        const int g4 = lane >> 2, t4 = lane & 3, mat = lane >> 3, r8 = lane & 7;
        float dacc[MT][4];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int e = 0; e < 4; ++e) dacc[mt][e] = 0.f;
        auto load_group = [&](uint4 (&v)[NL], int grp) {
#pragma unroll
            for (int j = 0; j < NL; ++j) {
                const int idx = lane + 32 * j, r = idx / (2 * MT), chk = idx % (2 * MT), row = grp * 16 + r;
                v[j] = row < len ? ldg_stream(W + (size_t)lj[row] * d_out + (size_t)q * C + (size_t)chk * 8)
                                 : make_uint4(0u, 0u, 0u, 0u);
            }
        };
        uint4 cur[NL], nxt[NL];
        if (warp < ng) load_group(cur, warp);
        for (int grp = warp; grp < ng; grp += NW_) {
            if (grp + NW_ < ng) load_group(nxt, grp + NW_);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < NL; ++j) {
                const int idx = lane + 32 * j, r = idx / (2 * MT), chk = idx % (2 * MT);
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(tile + (uint32_t)r * tst + (uint32_t)chk * 16u),
                             "r"(cur[j].x), "r"(cur[j].y), "r"(cur[j].z), "r"(cur[j].w) : "memory");
            }
            __syncwarp();
            // B fragments: rows 2 t4, 2 t4 + 1 (b0) and 2 t4 + 8, + 9 (b1) of the group, token g4
            uint32_t bf[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int k0 = grp * 16 + 2 * t4 + 8 * h;
                const uint32_t lo16 = (g4 < B && k0 < len) ? (uint32_t)lx[(size_t)k0 * LXS + g4] : 0u;
                const uint32_t hi16 = (g4 < B && k0 + 1 < len) ? (uint32_t)lx[(size_t)(k0 + 1) * LXS + g4] : 0u;
                bf[h] = lo16 | (hi16 << 16);
            }
            const uint32_t abase = tile + (uint32_t)(r8 + 8 * (mat >> 1)) * tst + (uint32_t)(8 * (mat & 1)) * 2u;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                uint32_t a0, a1, a2, a3;
                xs_ldsm_x4_trans(abase + (uint32_t)mt * 32u, a0, a1, a2, a3);
                xs_mma_bf16(dacc[mt], a0, a1, a2, a3, bf[0], bf[1]);
            }
#pragma unroll
            for (int j = 0; j < NL; ++j) cur[j] = nxt[j];
        }
        __syncthreads();  // every warp is past its tile: wred may overwrite the tiles
        trace_stamp(trace, 0, 2);
        // lane (g4, t4): D[col 16 mt + g4 (+8)][token 2 t4 (+1)]
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int c = mt * 16 + g4 + 8 * (e >> 1), tk = 2 * t4 + (e & 1);
                if (tk < B) wred[((size_t)warp * B + tk) * C + c] = dacc[mt][e];
            }
        __syncthreads();
    } else {
    const T *wcol = W + (size_t)q * C + (size_t)ch * VEC;
    float2 acc2[B][VEC / 2];  // column pairs: one FFMA2 per pair (same rounding as two FFMAs)
#pragma unroll
    for (int tk = 0; tk < B; ++tk)
#pragma unroll
        for (int e = 0; e < VEC / 2; ++e) acc2[tk][e] = make_float2(0.f, 0.f);
    auto fma_row = [&](const uint4 &wv, int r) {
        float f[VEC];
        unpack16(wv, f);
        float xv[LXS];
        if constexpr (sizeof(T) == 2) {  // one 32-bit load per token pair
            const uint32_t *xr = reinterpret_cast<const uint32_t *>(lx + (size_t)r * LXS);
#pragma unroll
            for (int k = 0; k < LXS / 2; ++k) {
                const uint32_t u = xr[k];
                xv[2 * k] = __uint_as_float(u << 16);
                xv[2 * k + 1] = __uint_as_float(u & 0xffff0000u);
            }
        } else {
#pragma unroll
            for (int tk = 0; tk < B; ++tk) xv[tk] = lx[(size_t)r * LXS + tk];
        }
#pragma unroll
        for (int tk = 0; tk < B; ++tk) {
            const float2 xx = make_float2(xv[tk], xv[tk]);
#pragma unroll
            for (int e = 0; e < VEC / 2; ++e) acc2[tk][e] = __ffma2_rn(xx, make_float2(f[2 * e], f[2 * e + 1]), acc2[tk][e]);
        }
    };
    for (int r = g; r < len; r += UN * G) {  // the tail batch is predicated, not a serial chain
        uint4 wv[UN];
#pragma unroll
        for (int u = 0; u < UN; ++u)
            if (r + u * G < len) wv[u] = ldg_stream(wcol + (size_t)lj[r + u * G] * d_out);
#pragma unroll
        for (int u = 0; u < UN; ++u)
            if (r + u * G < len) fma_row(wv[u], r + u * G);
    }

    // ---- in-CTA reduction, fixed order: lanes sharing a column chunk (shuffle butterfly), then the
    //      warps in warp order (wred overwrites xs: every thread is past its last row) ----
    float acc[B][VEC];
#pragma unroll
    for (int tk = 0; tk < B; ++tk)
#pragma unroll
        for (int e = 0; e < VEC / 2; ++e) {
            acc[tk][2 * e] = acc2[tk][e].x;
            acc[tk][2 * e + 1] = acc2[tk][e].y;
        }
#pragma unroll
    for (int tk = 0; tk < B; ++tk)
#pragma unroll
        for (int e = 0; e < VEC; ++e)
            for (int o = nch; o < 32; o <<= 1) acc[tk][e] += __shfl_xor_sync(0xffffffffu, acc[tk][e], o);
    __syncthreads();
    trace_stamp(trace, 0, 2);
    if (lane < nch) {
#pragma unroll
        for (int tk = 0; tk < B; ++tk)
#pragma unroll
            for (int e = 0; e < VEC; ++e) wred[((size_t)warp * B + tk) * C + ch * VEC + e] = acc[tk][e];
    }
    __syncthreads();
    }  // MT
    // ---- cluster reduction, fixed order: every rank stores its partial (sum over its warps in warp
    //      order) into slot [rank] of rank 0's shared memory (DSMEM), one cluster barrier, then rank 0
    //      writes y[tk][q*C + c] = sum over ranks 0..R-1 in order. The slots alias rank 0's x staging:
    //      the wait below (paired with the arrive after the prologue) orders them after its last use. ----
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    trace_stamp(trace, 0, 3);
    {
        const uint32_t slot0 = smem_u32(slots) + 4u * (uint32_t)(rank * B * C);
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(slot0));
        for (int e = tid; e < B * C; e += kXsThreads) {
            float sum = 0.f;
#pragma unroll
            for (int w = 0; w < NW_; ++w) sum += wred[(size_t)w * B * C + e];
            asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(remote + 4u * (uint32_t)e), "f"(sum) : "memory");
        }
    }
    cluster_sync_all();
    if (rank == 0) {
        for (int e = tid; e < B * C; e += kXsThreads) {
            float sum = 0.f;
            for (uint32_t rk = 0; rk < csize; ++rk) sum += slots[(size_t)rk * B * C + e];
            const int tk = e / C, c = e % C;
            y[(size_t)tk * d_out + (size_t)q * C + c] = sum;
        }
    }
    trace_stamp(trace, 0, 4);
}

int xs_mt(const PlanData &p, int b) {  // tensor-core tile count per warp for batch b (0 = FFMA2 path)
    const int c = p.xs[b].cols;
    return (p.esize == 2 && b >= kXsMmaMinB && !p.xs_no_mma && (c == 64 || c == 128)) ? c / 16 : 0;
}

size_t xs_smem_bytes(const PlanData &p, int b) {
    const int nw = (p.m + 31) / 32;
    const int maxr = xs_maxr(p, b);
    const int c = p.xs[b].cols, mt = xs_mt(p, b);
    const size_t tiles = mt > 0 ? (size_t)(kXsThreads / 32) * 16 * (c * 2 + 16) : 0;
    const size_t a_bytes = (std::max((size_t)(kXsThreads / 32) * b * c * 4, tiles) + 15) & ~(size_t)15;
    const size_t region = std::max((size_t)b * p.m * p.esize, a_bytes + (size_t)p.xs[b].r * b * c * 4);
    const int lxs = p.esize == 2 ? (b + 1) & ~1 : b;
    return ((region + 15) & ~(size_t)15) + (size_t)nw * 4 + (size_t)(nw + 1) * 4 +
           (size_t)maxr * 4 + (size_t)maxr * lxs * p.esize;
}

template <typename T, int B>
static decltype(&xs_gemv<T, B, 0>) xs_kernel(const PlanData &p) {
    if constexpr (sizeof(T) == 2 && B >= kXsMmaMinB) {
        const int mt = xs_mt(p, B);
        if (mt == 4) return xs_gemv<T, B, 4>;
        if (mt == 8) return xs_gemv<T, B, 8>;
    }
    return xs_gemv<T, B, 0>;
}

template <typename T, int B>
static cudaError_t launch_xs_b(const PlanData &p, const void *x, const void *W, float t, float *y, void *ws,
                               cudaStream_t s) {
    const size_t smem = xs_smem_bytes(p, B);
    auto kern = xs_kernel<T, B>(p);
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void *>(kern), smem);
    if (e != cudaSuccess) return e;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = (unsigned)p.xs[B].r;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(p.xs[B].q * p.xs[B].r));
    cfg.blockDim = dim3((unsigned)kXsThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    char *w = static_cast<char *>(ws);
    return cudaLaunchKernelEx(&cfg, kern, static_cast<const T *>(x), static_cast<const T *>(W), y, p.m, p.d,
                              p.xs[B].cols, t, xs_maxr(p, B), reinterpret_cast<uint8_t *>(w + p.off_tokmask),
                              p.trace ? reinterpret_cast<unsigned long long *>(w + p.off_trace) : nullptr);
}

template <typename T, int B>
static int xs_active_clusters_b(const PlanData &p) {
    const size_t smem = xs_smem_bytes(p, B);
    auto kern = xs_kernel<T, B>(p);
    if (ensure_smem_attr(reinterpret_cast<const void *>(kern), smem) != cudaSuccess) return -1;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)p.xs[B].r;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(p.xs[B].q * p.xs[B].r));
    cfg.blockDim = dim3((unsigned)kXsThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
        (void)cudaGetLastError();
        return -1;
    }
    return n;
}

// clusters of p.xs[b].r CTAs of the batch-b kernel that can be resident at once (-1: no device to ask)
int xs_active_clusters(const PlanData &p, int b) {
    const bool bf = p.dt == CATS_BF16;
    switch (b) {
        case 1: return bf ? xs_active_clusters_b<bf16_bits, 1>(p) : xs_active_clusters_b<float, 1>(p);
        case 2: return bf ? xs_active_clusters_b<bf16_bits, 2>(p) : xs_active_clusters_b<float, 2>(p);
        case 3: return bf ? xs_active_clusters_b<bf16_bits, 3>(p) : xs_active_clusters_b<float, 3>(p);
        case 4: return bf ? xs_active_clusters_b<bf16_bits, 4>(p) : xs_active_clusters_b<float, 4>(p);
        case 5: return bf ? xs_active_clusters_b<bf16_bits, 5>(p) : xs_active_clusters_b<float, 5>(p);
        case 6: return bf ? xs_active_clusters_b<bf16_bits, 6>(p) : xs_active_clusters_b<float, 6>(p);
        case 7: return bf ? xs_active_clusters_b<bf16_bits, 7>(p) : xs_active_clusters_b<float, 7>(p);
        default: return bf ? xs_active_clusters_b<bf16_bits, 8>(p) : xs_active_clusters_b<float, 8>(p);
    }
}

template <typename T>
static cudaError_t launch_xs_dt(const PlanData &p, const void *x, int b, const void *W, float t, float *y, void *ws,
                                cudaStream_t s) {
    switch (b) {
        case 1: return launch_xs_b<T, 1>(p, x, W, t, y, ws, s);
        case 2: return launch_xs_b<T, 2>(p, x, W, t, y, ws, s);
        case 3: return launch_xs_b<T, 3>(p, x, W, t, y, ws, s);
        case 4: return launch_xs_b<T, 4>(p, x, W, t, y, ws, s);
        case 5: return launch_xs_b<T, 5>(p, x, W, t, y, ws, s);
        case 6: return launch_xs_b<T, 6>(p, x, W, t, y, ws, s);
        case 7: return launch_xs_b<T, 7>(p, x, W, t, y, ws, s);
        case 8: return launch_xs_b<T, 8>(p, x, W, t, y, ws, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_xsparse(const PlanData &p, const void *x, int b, const void *W, float t, float *y, void *ws,
                           cudaStream_t s) {
    if (p.dt == CATS_BF16) return launch_xs_dt<bf16_bits>(p, x, b, W, t, y, ws, s);
    return launch_xs_dt<float>(p, x, b, W, t, y, ws, s);
}

}  // namespace cats
