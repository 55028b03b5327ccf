// mlp_split.cu -- the CATS-MLP decode for batches b >= 2: two persistent kernels, KA and KB.
//
// Paper: Custom GPU Kernel "MLP using CATS":
//     v <- SiLU(x W_gate); Mask <- |v| >= t; x1 <- (x W_up[Mask]) * v[Mask]; y <- x1 W_down[Mask]
// with the batch semantics of DESIGN.md reading G6: a neuron's W_up / W_down rows are read once if it
// is active for ANY of the b tokens (the union), and token i uses v_i = 0 where |v_i| < t.
//
// Why a second path. K12 keeps x and the exact fixed-point y partial of every token
// in registers: 2*b*d values per CTA, which is the whole register file at b = 8. Here the two
// register-heavy halves run in different kernels, each with its own work decomposition:
//
//  * KA (gate + up, dynamic): the K12 dataflow (persistent CTAs, tile counter, TMA bulk rings) with x
//    staged once in shared memory and TWO independent job streams per CTA (each: a producer warp, a
//    ring, 8 consumer warps -- one producer per SM was the bottleneck). Jobs are GATE(tile of NR
//    W_gate rows) and UP(<= NR active neurons' W_up rows, gathered across tiles from a FIFO). Every
//    job is the same consumer work, NR x b dot products, in one of two engines: b <= 2 FHFMA.BF16
//    (fma.rn.f32.bf16 on the packed registers) + one warp reduce-scatter (NR*b - 1 shuffles);
//    b >= 3 (bf16) warp-level mma.sync m16n8k16 bf16 -> fp32 (x = A, the job's rows = B; x from
//    tensor memory where d % 1024 == 0, else ldmatrix from 16-byte-padded rows). The producer sums the group's 8 warp partials in fixed order and
//    turns GATE results into u -> v = SiLU(u) -> keep = |v| >= t -> ballot compaction (idx / tokmask /
//    vals / cnt, the same per-tile layout as K12, plus one mask word per tile for KB) and UP results
//    into x1 = (x W_up[j]) * v_j (Optimization 1), written per compact position.
//    Each neuron's u and x1 are computed entirely inside one CTA in a fixed order: deterministic.
//  * KB (down, static): starts from KA's per-tile mask words while KA drains; the compact active list
//    (prefix-summed in every CTA) is cut into R equal ranges; CTA (r, q) streams the W_down rows of
//    range r, column part q, accumulates y_r = sum_j x1_j W_down[j] in fp32 in list order (CUDA
//    cores at b = 1 and for fp32; bf16 from b = 2 MMA with W_down^T via ldmatrix.trans and x1 as exact
//    bf16 hi + lo),
//    writes the partial; the last 64 CTAs to finish (no grid barrier) each sum a slice of the R partials in
//    fixed order r = 0..R-1 into y: the deterministic two-phase split-K reduction of the north star. The
//    tapered ranges balance the data-dependent work.
//
// KA -> KB -> next decode run as programmatic dependent launches: a kernel's CTAs become resident
// while its predecessor drains and wait (griddepcontrol.wait) only before touching its outputs.
#include <cuda_bf16.h>

#include "cats_device.cuh"
#include "cats_internal.h"

namespace cats {

enum : int { kSJobEnd = 0, kSJobGate = 1, kSJobUp = 2 };

// ------------------------------------------------------------------------------ arithmetic helpers
// Sum a[P] over the 32 lanes of a warp; afterwards lane l holds the warp total of a[l % P].
// Halving rounds (xor P/2 .. 1): a lane keeps the half selected by its lane bit and adds the
// partner's copy of it (P - 1 shuffles in all), then xor rounds P .. 16 combine the lane groups.
// A fixed tree: the same bits every run.
template <int P>
__device__ __forceinline__ float warp_reduce_scatter(float (&a)[P], int lane) {
#pragma unroll
    for (int h = P / 2; h >= 1; h >>= 1) {
        const bool up = (lane & h) != 0;
#pragma unroll
        for (int j = 0; j < h; ++j) {
            const float keep = up ? a[h + j] : a[j];
            const float send = up ? a[j] : a[h + j];
            a[j] = keep + __shfl_xor_sync(0xffffffffu, send, h);
        }
    }
    float v = a[0];
#pragma unroll
    for (int o = P; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

constexpr int pow2_ceil(int v) { return v <= 1 ? 1 : 2 * pow2_ceil((v + 1) / 2); }

// warp-level bf16 MMA, fp32 accumulate (D += A B), m16n8k16, A row-major, B column-major
__device__ __forceinline__ void mma_bf16_16816(float (&dd)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
                 "{%8, %9}, {%0, %1, %2, %3};"
                 : "+f"(dd[0]), "+f"(dd[1]), "+f"(dd[2]), "+f"(dd[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4_trans(uint32_t saddr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(saddr)
                 : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t saddr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(saddr)
                 : "memory");
}

// tensor memory: columns to allocate (a power of two >= 32), and 16-column (x16) stores / loads of one warp's
// 32 lanes (lane quarter = warp % 4 of the CTA), 32-bit per column
constexpr uint32_t tmem_cols_c(int n) { return n <= 32 ? 32u : n <= 64 ? 64u : n <= 128 ? 128u : n <= 256 ? 256u : 512u; }
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                 "%13, %14, %15, %16};" ::"r"(taddr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
                 "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
                 : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
                 "%14, %15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr)
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void claim_async(unsigned int &t, unsigned int *ctr, bool pred) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p atom.global.add.u32 %0, [%1], 1;\n\t}"
                 : "+r"(t)
                 : "l"(ctr), "r"((unsigned)pred)
                 : "memory");
}
constexpr unsigned int kNoTileS = 0xffffffffu;

// ======================================================================================== KA
template <typename T, int B, int NR, int KS>
__global__ void __launch_bounds__(kSplitAThreads, 1)
ka_gate_up(const T *__restrict__ x, const T *__restrict__ Wg, const T *__restrict__ Wu, int d, int m, int stages,
           float t, int mode, int32_t *__restrict__ idx, uint8_t *__restrict__ tokmask, float *__restrict__ vals,
           int32_t *__restrict__ cnt, unsigned int *__restrict__ tmask, float *__restrict__ x1out,
           unsigned int *__restrict__ sched, int lazy_tail, unsigned long long *__restrict__ trace) {
    constexpr int NW = kSplitAWarps;    // consumer warps (both groups)
    constexpr int NC = NW * 32;
    constexpr int NG = kSplitAGroups;    // independent job streams (producer + ring + consumers)
    constexpr int NWG = NW / NG;         // consumer warps per group
    constexpr int NCG = NWG * 32;
    constexpr int NP = NR * B;          // (row, token) dot products per job
    constexpr int PP = pow2_ceil(NP);   // padded to a power of two for the reduce-scatter
    constexpr bool CS = KS == 2;        // tensor cores in column parts (ka_colsplit)
    constexpr bool MP = CS || NP > 32;  // two (row, token) pairs per producer lane (8-row / 6-row tiles at b > 5)
    constexpr int NS = MP ? (NP + 31) / 32 : 1;  // (row, token) pairs per producer lane
    constexpr int FIFO = CS ? kSplitFifoCs : kSplitFifo;
    static_assert(MP ? PP <= 64 : PP <= 32, "one or two (row, token) pairs per lane");
    static_assert(!CS || NR == 8, "column parts use 8-row tiles");
    constexpr uint32_t TKM = (1u << B) - 1u;
    using Desc = SplitDesc<NR, B>;
    using Ent = SplitFifoEntry<B>;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = warp < NW ? warp / NWG : warp - NW;  // this warp's group
    const int nch = d * (int)sizeof(T) / 16;
    const uint32_t row_bytes = (uint32_t)d * (uint32_t)sizeof(T);
    // column parts (CS): a job is H consecutive stages, part h = columns [h C, (h + 1) C), C = kKaPartCols
    const int H = CS ? d / kKaPartCols : 1;
    const uint32_t srow_bytes = CS ? (uint32_t)kKaPartCols * (uint32_t)sizeof(T) : row_bytes;  // a stage row
    // stage rows are padded by 16 B: the NR rows of a stage start in different shared-memory bank
    // groups (conflict-free ldmatrix) and the zeroed pad absorbs a half 16-wide k-step at the row end
    const uint32_t rs_bytes = srow_bytes + 16u;
    const uint32_t stage_bytes = (uint32_t)NR * rs_bytes;
    const int ntiles = (m + NR - 1) / NR;

    // shared memory: x, then per group: ring, barriers, descriptors, FIFO, partial sums
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char *xs = smem;  // x: [B][d] (dot-product path) or [B][d + 8] (tensor-core path, padded rows)
    // (KS == 3 keeps x in tensor memory, not here)
    unsigned char *ring0 = xs + (KS == 3 ? (size_t)0 : (size_t)B * (KS > 0 ? row_bytes + 16u : row_bytes));  // [NG][stages][stage]
    uint64_t *full0 = reinterpret_cast<uint64_t *>(ring0 + (size_t)NG * stages * stage_bytes);  // [NG][stages]
    uint64_t *empty0 = full0 + NG * stages;                                               // [NG][stages]
    Desc *desc0 = reinterpret_cast<Desc *>(empty0 + NG * stages);                         // [NG][stages]
    Ent *fifo0 = reinterpret_cast<Ent *>(desc0 + NG * stages);                            // [NG][FIFO]
    float *red0 = reinterpret_cast<float *>(fifo0 + NG * FIFO);                           // [NG][stages][NWG][PP]
    Desc *jt0 = reinterpret_cast<Desc *>(red0 + (size_t)NG * stages * NWG * PP);          // CS: [NG] job in flight
    unsigned char *ring = ring0 + (size_t)g * stages * stage_bytes;
    uint64_t *full = full0 + g * stages;
    uint64_t *empty = empty0 + g * stages;
    Desc *desc = desc0 + g * stages;
    Ent *fifo = fifo0 + g * FIFO;
    float *red = red0 + (size_t)g * stages * NWG * PP;

    trace_stamp(trace, 0, 0);
    // (griddepcontrol.launch_dependents comes after each thread's griddepcontrol.wait: KB may only
    //  start once this grid's predecessor -- the previous decode -- has completed, because KB reads
    //  the per-tile masks and counters that decode re-armed)
    if (tid == 0) {
        for (int s = 0; s < NG * stages; ++s) {
            mbar_init(&full0[s], 1);
            mbar_init(&empty0[s], NWG);
        }
        fence_mbar_init();
    }
    for (int i = tid; i < NG * stages * NR; i += blockDim.x)  // row pads (never written by copies)
        *reinterpret_cast<uint4 *>(ring0 + (size_t)i * rs_bytes + srow_bytes) = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();

    if (warp >= NW) {
        // ===================================== PRODUCER WARPS ====================================
        // one per group; the groups share the tile counter and x, nothing else
        const bool dense = mode == kModeDense;
        const uint64_t policy = l2_evict_first_policy();
        unsigned int res0 = kNoTileS, res1 = kNoTileS;  // reserved tiles (raw counter values)
        int rsel = 0;                                    // slot the next GATE issue uses
        const int nstreams = (int)gridDim.x * NG;  // job streams in the grid
        // static tiles per stream: enough to fill the ring (a tile is H stages in column parts)
        const int batch = max(1, min((stages + H - 1) / H, ntiles / nstreams));
        const unsigned int dyn_base = (unsigned)nstreams * (unsigned)batch;
        int prod = 0, ps = 0, retire = 0;
        int q_head = 0, q_tail = 0;  // active-neuron FIFO (uniform across the warp)
        int gates_inflight = 0;
        bool ended = false;
        Desc &J = jt0[g];            // CS: the job being streamed part by part
        int cur_part = 0;            // CS: its next column part (0 = no job in progress)

        // CS: stage s <- column part `part` of job J (descriptor copy, then one copy per row)
        auto issue_part = [&](int s, int part) {
            const int *src = reinterpret_cast<const int *>(&J);
            int *dst = reinterpret_cast<int *>(&desc[s]);
            for (int i = lane; i < (int)(sizeof(Desc) / 4); i += 32) dst[i] = src[i];
            __syncwarp();
            const int n = J.n;
            if (lane == 0) {
                desc[s].part = part;
                mbar_arrive_expect_tx(&full[s], (uint32_t)n * srow_bytes);
            }
            __syncwarp();
            if (lane < n) {
                const size_t row = J.type == kSJobGate ? (size_t)(J.tile * NR + lane) : (size_t)J.id[lane];
                bulk_g2s(ring + (size_t)s * stage_bytes + (size_t)lane * rs_bytes,
                         (J.type == kSJobGate ? Wg : Wu) + row * d + (size_t)part * kKaPartCols, srow_bytes,
                         &full[s], policy);
            }
        };
        auto issue_up = [&](int n) {  // UP job: W_up rows of the next n FIFO neurons
            const int s = ps;
            Desc &D = CS ? J : desc[s];
            if (lane < n) {
                const Ent &E = fifo[(q_head + lane) & (FIFO - 1)];
                D.id[lane] = E.id;
                D.pos[lane] = E.pos;
#pragma unroll
                for (int tk = 0; tk < B; ++tk) D.v[lane][tk] = E.v[tk];
            }
            if constexpr (CS) {
                if (lane == 0) {
                    J.type = kSJobUp;
                    J.n = n;
                }
                __syncwarp();
                issue_part(s, 0);
                cur_part = H > 1 ? 1 : 0;
            } else {
                if (lane == 0) {
                    D.type = kSJobUp;
                    D.n = n;
                    mbar_arrive_expect_tx(&full[s], (uint32_t)n * row_bytes);
                }
                __syncwarp();
                if (lane < n)
                    bulk_g2s(ring + (size_t)s * stage_bytes + (size_t)lane * rs_bytes, Wu + (size_t)D.id[lane] * d,
                             row_bytes, &full[s], policy);
            }
            q_head += n;
        };
        auto issue_job = [&]() -> bool {
            const int s = ps;
            if constexpr (CS) {
                if (cur_part != 0) {  // the next column part of the job in flight
                    issue_part(s, cur_part);
                    if (++cur_part == H) cur_part = 0;
                    __syncwarp();
                    ++prod;
                    if (++ps == stages) ps = 0;
                    return true;
                }
            }
            const int qn = q_tail - q_head;
            if (qn >= NR) {
                issue_up(NR);
            } else {
                // next tile: the reservation claimed two GATE issues ago (two slots used in turn,
                // selected by branches so no instruction waits on the newest atomic); a slot that
                // came back past the end is parked there and the other one is tried
                unsigned int tile = kNoTileS;
                if (lane == 0) {
                    for (int tries = 0; tries < 2; ++tries) {
                        unsigned int raw;
                        if (rsel == 0) {
                            raw = res0;
                            if (raw == kNoTileS) raw = atomicAdd(&sched[0], 1u);
                        } else {
                            raw = res1;
                            if (raw == kNoTileS) raw = atomicAdd(&sched[0], 1u);
                        }
                        if (raw + dyn_base < (unsigned)ntiles) {
                            tile = raw + dyn_base;
                            break;
                        }
                        if (rsel == 0) res0 = raw; else res1 = raw;
                        rsel ^= 1;
                    }
                }
                tile = __shfl_sync(0xffffffffu, tile, 0);
                if (tile < (unsigned)ntiles) {
                    const int r0 = (int)tile * NR;
                    const int nr = min(NR, m - r0);
                    if (lane == 0) {
                        const bool more = tile + 1u + (unsigned)lazy_tail < (unsigned)ntiles;
                        if (rsel == 0) {
                            res0 = kNoTileS;
                            claim_async(res0, sched, more);
                        } else {
                            res1 = kNoTileS;
                            claim_async(res1, sched, more);
                        }
                        rsel ^= 1;
                    }
                    if constexpr (CS) {
                        if (lane == 0) {
                            J.type = kSJobGate;
                            J.tile = (int)tile;
                            J.n = nr;
                        }
                        __syncwarp();
                        issue_part(s, 0);
                        cur_part = H > 1 ? 1 : 0;
                    } else {
                        if (lane == 0) {
                            desc[s].type = kSJobGate;
                            desc[s].tile = (int)tile;
                            desc[s].n = nr;
                            mbar_arrive_expect_tx(&full[s], (uint32_t)nr * row_bytes);
                        }
                        __syncwarp();
                        if (lane < nr)  // one copy per (padded) row
                            bulk_g2s(ring + (size_t)s * stage_bytes + (size_t)lane * rs_bytes,
                                     Wg + (size_t)(r0 + lane) * d, row_bytes, &full[s], policy);
                    }
                    ++gates_inflight;
                } else {
                    if (qn > 0) {
                        issue_up(qn);  // drain a partial UP job
                    } else if (gates_inflight != 0) {
                        return false;  // an in-flight GATE job may still add neurons
                    } else {
                        if (lane == 0) {
                            desc[s].type = kSJobEnd;
                            desc[s].n = 0;
                            mbar_arrive_expect_tx(&full[s], 0u);
                        }
                        ended = true;
                    }
                }
            }
            __syncwarp();
            ++prod;
            if (++ps == stages) ps = 0;
            return true;
        };

        int nstatic = 0;  // static tiles started
        if (lane == 0) {  // static first batch (weights only: safe before the PDL wait)
            const unsigned int base = (blockIdx.x * NG + g) * (unsigned)batch;
            for (int s = 0; s < batch; ++s) {
                if (base + s >= (unsigned)ntiles) break;  // tiny layers: fewer tiles than streams
                const int r0 = (int)(base + s) * NR;
                const int nr = min(NR, m - r0);
                ++nstatic;
                // CS: the tile's column parts in consecutive stages while the ring has room; a tile cut
                // off by the ring's end continues from J / cur_part (the first dynamic issues)
                for (int part = 0; part < H && prod < stages; ++part) {
                    desc[prod].type = kSJobGate;
                    desc[prod].tile = (int)(base + s);
                    desc[prod].n = nr;
                    desc[prod].part = part;
                    mbar_arrive_expect_tx(&full[prod], (uint32_t)nr * srow_bytes);
                    for (int r = 0; r < nr; ++r)
                        bulk_g2s(ring + (size_t)prod * stage_bytes + (size_t)r * rs_bytes,
                                 Wg + (size_t)(r0 + r) * d + (size_t)part * (srow_bytes / sizeof(T)), srow_bytes,
                                 &full[prod], policy);
                    ++prod;
                    if (CS && part + 1 < H && prod == stages) {
                        J = desc[prod - 1];
                        cur_part = part + 1;
                    }
                }
            }
        }
        prod = __shfl_sync(0xffffffffu, prod, 0);
        cur_part = __shfl_sync(0xffffffffu, cur_part, 0);
        ps = prod % stages;
        gates_inflight = __shfl_sync(0xffffffffu, nstatic, 0);
        __syncwarp();
        pdl_wait_primary();
        pdl_launch_dependents();
        if (lane == 0) {
            claim_async(res0, sched, dyn_base + (unsigned)lazy_tail < (unsigned)ntiles);
            claim_async(res1, sched, dyn_base + 1u + (unsigned)lazy_tail < (unsigned)ntiles);
        }
        if (prod == 0) {  // no static tile: claim (or end) right away
            while (!ended && issue_job()) {
            }
        }

        int rs = 0;
        uint32_t rphase = 0;
        const int r = lane / B, tk = lane % B;  // this lane's (row, token) pair
        unsigned long long p_wait = 0;           // diagnostics (options.trace)
        int n_gate = 0, n_up = 0;
        // retire every job in order; after END (the last job issued, never released by the
        // consumers) is queued, the UP jobs still in flight are retired before the loop exits
        while (!ended || retire < prod - 1) {
            const unsigned long long tw0 = trace ? gtimer() : 0ull;
            mbar_wait(&empty[rs], rphase);
            if (trace) p_wait += gtimer() - tw0;
            const Desc &D = desc[rs];
            if (trace) { if (D.type == kSJobGate) ++n_gate; else ++n_up; }
            const int n = D.n;
            if constexpr (MP) {
                // column parts: the consumers accumulate across a job's H stages and publish the warp
                // partials with the last part; earlier parts only free their stage. Also the retire of
                // tiles with more (row, token) pairs than lanes (two per lane).
                if (!CS || D.part == H - 1) {
                    float u[NS];
                    bool ok[NS];
#pragma unroll
                    for (int j = 0; j < NS; ++j) {
                        const int p = lane + 32 * j;
                        ok[j] = p < NP && p / B < n;
                        u[j] = 0.f;
                        if (ok[j]) {
                            const float *rb = red + (size_t)rs * NWG * PP + p;
#pragma unroll
                            for (int w = 0; w < NWG; ++w) u[j] += rb[w * PP];
                        }
                    }
                    if (D.type == kSJobGate) {
                        const int tile = D.tile, r0 = tile * NR;
                        float v[NS];
                        bool keep[NS];
                        unsigned long long m64 = 0ull;  // bit p: pair p = (row p / B, token p % B) kept
#pragma unroll
                        for (int j = 0; j < NS; ++j) {
                            v[j] = __fdividef(u[j], 1.0f + __expf(-u[j]));  // SiLU (Eq. 2)
                            keep[j] = ok[j] && (dense || fabsf(v[j]) >= t);  // Eq. 4, ties kept
                            m64 |= (unsigned long long)__ballot_sync(0xffffffffu, keep[j]) << (32 * j);
                        }
                        uint32_t rowact = 0;
#pragma unroll
                        for (int rr = 0; rr < NR; ++rr)
                            if ((m64 >> (rr * B)) & TKM) rowact |= 1u << rr;
                        const int nact = __popc(rowact);
#pragma unroll
                        for (int j = 0; j < NS; ++j) {
                            const int p = lane + 32 * j, rj = p / B, tj = p % B;
                            if (ok[j] && ((rowact >> rj) & 1u)) {
                                const int rank = __popc(rowact & ((1u << rj) - 1u));
                                const int pos = r0 + rank;
                                const float vk = keep[j] ? v[j] : 0.f;
                                vals[(size_t)pos * B + tj] = vk;
                                Ent &E = fifo[(q_tail + rank) & (FIFO - 1)];
                                E.v[tj] = vk;
                                if (tj == 0) {
                                    idx[pos] = r0 + rj;
                                    tokmask[pos] = (uint8_t)((m64 >> (rj * B)) & TKM);
                                    E.id = r0 + rj;
                                    E.pos = pos;
                                }
                            }
                        }
                        if (lane == 0) {
                            cnt[tile] = nact;
                            asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(tmask + tile),
                                         "r"(0x80000000u | rowact)
                                         : "memory");
                        }
                        q_tail += nact;
                        --gates_inflight;
                    } else {  // UP: x1 = (x W_up[j]) * v_j, per token
#pragma unroll
                        for (int j = 0; j < NS; ++j) {
                            const int p = lane + 32 * j, rj = p / B, tj = p % B;
                            if (ok[j]) x1out[(size_t)D.pos[rj] * B + tj] = u[j] * D.v[rj][tj];
                        }
                    }
                }
                __syncwarp();
                ++retire;
                if (++rs == stages) { rs = 0; rphase ^= 1u; }
                while (!ended && prod < retire + stages && issue_job()) {
                }
                continue;
            }
            const bool mine = lane < NP && r < n;
            float u = 0.f;
            if (mine) {
                const float *rb = red + (size_t)rs * NWG * PP + lane;
#pragma unroll
                for (int w = 0; w < NWG; ++w) u += rb[w * PP];
            }
            // everything the retire needs from the stage's descriptor and partials; on the tensor-core
            // path the stage is refilled first, so its load latency starts before the retire arithmetic
            // (the refill may not see this job's FIFO entries yet; they go out with the next issue).
            // Measured (A/B): 1-1.4 % faster at b = 4 / 8; on the FHFMA path (b <= 3) 1-2.6 % slower.
            const int jtype = D.type, jtile = D.tile;
            int jpos = 0;
            float jv = 0.f;
            if (mine && jtype != kSJobGate) {
                jpos = D.pos[r];
                jv = D.v[r][tk];
            }
            __syncwarp();
            ++retire;
            if (++rs == stages) { rs = 0; rphase ^= 1u; }
            if constexpr (KS == 1 || KS == 3) {
                while (!ended && prod < retire + stages && issue_job()) {
                }
            }
            if (jtype == kSJobGate) {
                // u -> v = SiLU(u) (Eq. 2) -> keep = |v| >= t (Eq. 4, ties kept) -> compaction
                const int tile = jtile, r0 = tile * NR;
                const float v = __fdividef(u, 1.0f + __expf(-u));
                const bool keep = mine && (dense || fabsf(v) >= t);
                const uint32_t bal = __ballot_sync(0xffffffffu, keep);
                uint32_t rowact = 0;
#pragma unroll
                for (int rr = 0; rr < NR; ++rr)
                    if ((bal >> (rr * B)) & TKM) rowact |= 1u << rr;
                const int nact = __popc(rowact);
                if (lane < NP && ((rowact >> r) & 1u)) {
                    const int rank = __popc(rowact & ((1u << r) - 1u));
                    const int pos = r0 + rank;
                    const float vk = keep ? v : 0.f;
                    vals[(size_t)pos * B + tk] = vk;
                    Ent &E = fifo[(q_tail + rank) & (FIFO - 1)];
                    E.v[tk] = vk;
                    if (tk == 0) {
                        idx[pos] = r0 + r;
                        tokmask[pos] = (uint8_t)((bal >> (r * B)) & TKM);
                        E.id = r0 + r;
                        E.pos = pos;
                    }
                }
                if (lane == 0) {
                    cnt[tile] = nact;
                    // one self-contained word per tile (valid bit + active rows): KB starts from these
                    // while KA is still running its UP jobs
                    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(tmask + tile), "r"(0x80000000u | rowact)
                                 : "memory");
                }
                q_tail += nact;
                --gates_inflight;
            } else if (mine) {  // UP: x1 = (x W_up[j]) * v_j, per token
                x1out[(size_t)jpos * B + tk] = u * jv;
            }
            __syncwarp();
            while (!ended && prod < retire + stages && issue_job()) {
            }
        }
        if (lane == 0) {
            trace_put(trace, 2, 0, p_wait);
            trace_put(trace, 2, 2, (unsigned long long)retire);
            trace_put(trace, 2, 4, (unsigned long long)n_gate);
            trace_put(trace, 2, 5, (unsigned long long)n_up);
        }
    } else {
        // ===================================== CONSUMER WARPS ====================================
        pdl_wait_primary();  // x may come from the predecessor
        pdl_launch_dependents();
        trace_stamp(trace, 0, 4);  // this CTA's consumers have released KB's launch
        const int ctid = tid - g * NCG;  // consumer thread index within the group
        const int cwarp = warp - g * NWG;
        int s = 0;
        uint32_t phase = 0;
        unsigned long long c_wait = 0;
        if constexpr (KS == 3) {
            // ---- tensor cores with x in TENSOR MEMORY: warp w's A fragments (x rows = tokens, its k-steps
            //      [w spw, (w + 1) spw)) are written once into TMEM columns of the warp's lane quarter and
            //      re-read per stage with tcgen05.ld, so no x lives in shared memory (the ring gets that
            //      space: three 4-row stages per job stream at b = 8) and no ldmatrix of x competes with
            //      the stage reads. The warps of both groups that own the same k-steps share columns. ----
            __shared__ uint32_t s_tmem;
            const int nsteps = d / 16, spw = nsteps / NWG;  // a multiple of 8: d % 1024 == 0 (split_ka_ks)
            const uint32_t tcols = tmem_cols_c(4 * spw);
            if (warp == 0) {
                asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                             "r"(tcols));
                asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            consumer_barrier<NC>();
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const int g4 = lane >> 2, t4 = lane & 3;
            // lane quarter = warp % 4; within it, cwarp 0-3 and 4-7 own different k-steps (column blocks)
            const uint32_t taddr = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((cwarp >> 2) * 2 * spw);
            if (g == 0) {  // fill: column 2j = a0, 2j + 1 = a2 of k-step j (A row = token g4, or token 0)
                const uint32_t *xw = reinterpret_cast<const uint32_t *>(x) + (size_t)(g4 < B ? g4 : 0) * (d / 2);
                for (int j0 = 0; j0 < spw; j0 += 8) {
                    uint32_t r[16];
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) {
                        const int kk = (cwarp * spw + j0 + jj) * 16;
                        r[2 * jj] = __ldg(xw + (kk >> 1) + t4);
                        r[2 * jj + 1] = __ldg(xw + ((kk + 8) >> 1) + t4);
                    }
                    tmem_st16(taddr + (uint32_t)(2 * j0), r);
                }
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            consumer_barrier<NC>();
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t koff = (uint32_t)(lane >> 3) * 16u + (uint32_t)(cwarp * spw) * 32u;
            const uint32_t brow = (uint32_t)((lane & 7) % NR) * rs_bytes + koff;
            for (;;) {
                const unsigned long long cw0 = trace ? gtimer() : 0ull;
                mbar_wait(&full[s], phase);
                if (trace) c_wait += gtimer() - cw0;
                if (desc[s].type == kSJobEnd) break;
                const uint32_t sb = smem_u32(ring + (size_t)s * stage_bytes) + brow;
                float dacc[4] = {0.f, 0.f, 0.f, 0.f}, dacc2[4] = {0.f, 0.f, 0.f, 0.f};
                for (int j0 = 0; j0 < spw; j0 += 8) {  // 8 k-steps (16 TMEM columns) per load
                    uint32_t a[16];
                    tmem_ld16(taddr + (uint32_t)(2 * j0), a);
#pragma unroll
                    for (int jj = 0; jj < 8; jj += 2) {
                        uint32_t b0, b1, b2, b3;
                        ldsm_x4(sb + (uint32_t)(j0 + jj) * 32u, b0, b1, b2, b3);
                        mma_bf16_16816(dacc, a[2 * jj], a[2 * jj], a[2 * jj + 1], a[2 * jj + 1], b0, b1);
                        mma_bf16_16816(dacc2, a[2 * jj + 2], a[2 * jj + 2], a[2 * jj + 3], a[2 * jj + 3], b2, b3);
                    }
                }
                float *rb = red + ((size_t)s * NWG + cwarp) * PP;
                if (g4 < B && 2 * t4 < NR) rb[(2 * t4) * B + g4] = dacc[0] + dacc2[0];
                if (g4 < B && 2 * t4 + 1 < NR) rb[(2 * t4 + 1) * B + g4] = dacc[1] + dacc2[1];
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                if (++s == stages) { s = 0; phase ^= 1u; }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            consumer_barrier<NC>();
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem), "r"(tcols));
        } else if constexpr (KS > 0) {
            // ---- tensor-core dot products (bf16): D[16 x 8] += A[16 x 16] B[16 x 8] per 16-wide k-step,
            //      A = x (rows = tokens; rows >= b repeat token 0 and are ignored), B = W^T (columns =
            //      the job's NR rows; the other 8 - NR columns repeat them and are ignored). Warp w of the
            //      group owns k-steps [w*spw, (w+1)*spw). Both operands come from shared memory with
            //      ldmatrix (x rows and stage rows padded by 16 B: conflict-free). ----
            {
                const uint4 *xg = reinterpret_cast<const uint4 *>(x);
                const uint32_t xrs = row_bytes + 16u;
                for (int i = tid; i < B * nch; i += NC)
                    *reinterpret_cast<uint4 *>(xs + (size_t)(i / nch) * xrs + (size_t)(i % nch) * 16) = xg[i];
                if (tid < B) *reinterpret_cast<uint4 *>(xs + (size_t)tid * xrs + row_bytes) = make_uint4(0u, 0u, 0u, 0u);
            }
            consumer_barrier<NC>();
            const int g4 = lane >> 2, t4 = lane & 3;
            if constexpr (CS) {
                // column parts: warp w owns k-steps [w SPW, (w + 1) SPW) of every part; the 8 B columns are
                // the tile's 8 distinct rows; D accumulates over the job's H consecutive stages
                constexpr int SPW = kKaPartCols / 16 / NWG;
                static_assert(SPW % 2 == 0, "two k-steps per ldmatrix.x4");
                const uint32_t koff = (uint32_t)(lane >> 3) * 16u + (uint32_t)(cwarp * SPW) * 32u;
                const uint32_t arow =
                    smem_u32(xs) + (uint32_t)((lane & 7) < B ? (lane & 7) : 0) * (row_bytes + 16u) + koff;
                const uint32_t brow = (uint32_t)(lane & 7) * rs_bytes + koff;
                float dacc[4] = {0.f, 0.f, 0.f, 0.f};
                for (;;) {
                    const unsigned long long cw0 = trace ? gtimer() : 0ull;
                    mbar_wait(&full[s], phase);
                    if (trace) c_wait += gtimer() - cw0;
                    if (desc[s].type == kSJobEnd) break;
                    const int part = desc[s].part;
                    if (part == 0) dacc[0] = dacc[1] = dacc[2] = dacc[3] = 0.f;
                    const uint32_t sb = smem_u32(ring + (size_t)s * stage_bytes) + brow;
                    const uint32_t ab = arow + (uint32_t)part * srow_bytes;
#pragma unroll
                    for (int j = 0; j < SPW; j += 2) {
                        uint32_t a0, a2, a4, a6, b0, b1, b2, b3;
                        ldsm_x4(ab + (uint32_t)j * 32u, a0, a2, a4, a6);
                        ldsm_x4(sb + (uint32_t)j * 32u, b0, b1, b2, b3);
                        mma_bf16_16816(dacc, a0, a0, a2, a2, b0, b1);  // rows 8..15 of A: ignored copies
                        mma_bf16_16816(dacc, a4, a4, a6, a6, b2, b3);
                    }
                    if (part == H - 1 && g4 < B) {  // lane (g4, t4): D[token g4][rows 2 t4, 2 t4 + 1]
                        float *rb = red + ((size_t)s * NWG + cwarp) * PP;
                        rb[(2 * t4) * B + g4] = dacc[0];
                        rb[(2 * t4 + 1) * B + g4] = dacc[1];
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[s]);
                    if (++s == stages) { s = 0; phase ^= 1u; }
                }
            } else {
            const int nsteps = (d + 15) / 16;
            const int spw = (nsteps + NWG - 1) / NWG;
            const int j0 = cwarp * spw, j1 = min(nsteps, j0 + spw);
            // ldmatrix.x4 row addresses: lane i -> matrix i/8 (k offset 8*(i/8)), row i%8
            const uint32_t koff = (uint32_t)(lane >> 3) * 16u + (uint32_t)j0 * 32u;
            const uint32_t arow = smem_u32(xs) + (uint32_t)((lane & 7) < B ? (lane & 7) : 0) * (row_bytes + 16u) + koff;
            const uint32_t brow = (uint32_t)((lane & 7) % NR) * rs_bytes + koff;
            for (;;) {
                const unsigned long long cw0 = trace ? gtimer() : 0ull;
                mbar_wait(&full[s], phase);
                if (trace) c_wait += gtimer() - cw0;
                if (desc[s].type == kSJobEnd) break;
                const uint32_t sb = smem_u32(ring + (size_t)s * stage_bytes) + brow;
                // two accumulator chains (even / odd k-steps): half the dependent-MMA latency per stage
                float dacc[4] = {0.f, 0.f, 0.f, 0.f}, dacc2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
                for (int j = j0; j < j1; j += 2) {
                    const uint32_t o = (uint32_t)(j - j0) * 32u;
                    uint32_t a0, a2, a4, a6, b0, b1, b2, b3;
                    ldsm_x4(arow + o, a0, a2, a4, a6);  // steps j (a0, a2) and j + 1 (a4, a6)
                    ldsm_x4(sb + o, b0, b1, b2, b3);    // steps j (b0, b1) and j + 1 (b2, b3)
                    mma_bf16_16816(dacc, a0, a0, a2, a2, b0, b1);  // rows 8..15 of A: ignored copies
                    if (j + 1 < j1) mma_bf16_16816(dacc2, a4, a4, a6, a6, b2, b3);
                }
                // lane (g4, t4) holds D[token g4][row 2 t4] and D[g4][2 t4 + 1]
                float *rb = red + ((size_t)s * NWG + cwarp) * PP;
                if (g4 < B && 2 * t4 < NR) rb[(2 * t4) * B + g4] = dacc[0] + dacc2[0];
                if (g4 < B && 2 * t4 + 1 < NR) rb[(2 * t4 + 1) * B + g4] = dacc[1] + dacc2[1];
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                if (++s == stages) { s = 0; phase ^= 1u; }
            }
            }
        } else {
        {
            const uint4 *xg = reinterpret_cast<const uint4 *>(x);
            uint4 *xd = reinterpret_cast<uint4 *>(xs);
            for (int i = tid; i < B * nch; i += NC) xd[i] = xg[i];
        }
        consumer_barrier<NC>();
        const uint32_t xbase = smem_u32(xs);
        for (;;) {
            const unsigned long long cw0 = trace ? gtimer() : 0ull;
            mbar_wait(&full[s], phase);
            if (trace) c_wait += gtimer() - cw0;
            const int type = desc[s].type;
            if (type == kSJobEnd) break;
            const uint32_t sbase = smem_u32(ring + (size_t)s * stage_bytes);
            float acc[PP];
#pragma unroll
            for (int p = 0; p < PP; ++p) acc[p] = 0.f;
            for (int ch = ctid; ch < nch; ch += NCG) {
                uint4 xv[B];
#pragma unroll
                for (int tk = 0; tk < B; ++tk) xv[tk] = lds128(xbase + (uint32_t)tk * row_bytes + (uint32_t)ch * 16u);
                // rows r >= n of a short job hold stale shared memory: their sums are computed
                // anyway (no branches) and ignored by the producer
#pragma unroll
                for (int r = 0; r < NR; ++r) {
                    const uint4 w = lds128(sbase + (uint32_t)r * rs_bytes + (uint32_t)ch * 16u);
#pragma unroll
                    for (int tk = 0; tk < B; ++tk) acc[r * B + tk] = dot16<T>(w, xv[tk], acc[r * B + tk]);
                }
            }
            const float v = warp_reduce_scatter<PP>(acc, lane);
            if (lane < PP) red[((size_t)s * NWG + cwarp) * PP + lane] = v;
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == stages) { s = 0; phase ^= 1u; }
        }
        }
        if (tid == 0) trace_put(trace, 2, 3, c_wait);
    }
    trace_stamp(trace, 0, 2);
    __syncthreads();
    if (tid == 0 && atomicAdd(&sched[1], 1u) == gridDim.x - 1) {  // last CTA: reset the tile scheduler
        sched[0] = 0u;
        sched[1] = 0u;
        sched[2] = 0u;  // KB's arrival-ticket counter
    }
    trace_stamp(trace, 0, 3);
}

// ======================================================================================== KB
template <typename T, int B, int EPT, int MT>
__global__ void __launch_bounds__(kSplitBMaxThreads, 1)
kb_down(const T *__restrict__ Wd, int d, int ntiles, int nr_tile, int Q, int R, int stages, int rows_per_stage,
        int maxr, unsigned int *__restrict__ tmask, const float *__restrict__ x1in, float *__restrict__ part,
        float *__restrict__ y, unsigned int *__restrict__ sched, unsigned long long *__restrict__ trace) {
    constexpr int EB = EPT * (int)sizeof(T);  // bytes of a thread's columns in one row (8 or 16)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nth = blockDim.x, NCW = nth / 32 - 1, NCt = NCW * 32;  // consumer warps / threads
    const int q = blockIdx.x % Q;  // column part; the range index rr is taken in arrival order below
    const int part_cols = d / Q;
    const uint32_t seg_bytes = (uint32_t)part_cols * (uint32_t)sizeof(T);
    const uint32_t sst = seg_bytes + 16u;  // stage row stride (padded: conflict-free ldmatrix)
    const uint32_t stage_bytes = (uint32_t)rows_per_stage * sst;

    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char *ring = smem;                                                               // [stages][stage]
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + (size_t)stages * stage_bytes);       // [stages]
    uint64_t *empty = full + stages;                                                          // [stages]
    // x1 of the range (8-byte aligned): fp32 [maxr][B], or on the MMA path bf16x2 hi + lo per neuron pair
    float *lx = reinterpret_cast<float *>(empty + stages);
    const int lxn = MT > 0 ? (maxr + 15) / 16 * 16 * B : maxr * B;
    int *pre = reinterpret_cast<int *>(lx + lxn);                                             // [ntiles + 1]
    int *wsum = pre + ntiles + 1;                                                             // [32]
    int *lj = wsum + 32;                                                                      // [maxr]
    int *lpos = lj + maxr;                                                                    // [maxr]
    uint8_t *rowm = reinterpret_cast<uint8_t *>(lpos + maxr);                                 // [ntiles]
    __shared__ int s_rr;

    trace_stamp(trace, 1, 0);
    pdl_launch_dependents();
    // this CTA's arrival ticket for column part q, taken at start: the atomic's round trip overlaps the
    // mask reads below (KB starts only after the previous decode's KB completed and re-armed the tickets:
    // KA waits for it before letting KB launch)
    unsigned int rr_ticket = 0;
    if (tid == 0) rr_ticket = atomicAdd(&sched[8 + q], 1u);
    if (tid == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        fence_mbar_init();
    }
    // ---- per-tile active-row masks, published by KA's GATE retire (valid bit 31). KB does NOT wait
    //      for KA to finish here: the list and the first W_down loads overlap KA's UP tail. ----
    if (tid == 0) pre[0] = 0;
    for (int base = 0; base < ntiles; base += 8 * nth) {  // 8 loads in flight per thread
        unsigned int c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = base + u * nth + tid;
            c[u] = 0x80000000u;
            if (i < ntiles) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(c[u]) : "l"(tmask + i) : "memory");
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = base + u * nth + tid;
            if (i < ntiles) {
                while (!(c[u] & 0x80000000u)) {  // that tile's GATE job has not retired yet
                    __nanosleep(128);
                    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(c[u]) : "l"(tmask + i) : "memory");
                }
                rowm[i] = (uint8_t)(c[u] & 0xffu);
                pre[i + 1] = __popc(c[u] & 0xffu);
            }
        }
    }
    trace_stamp(trace, 1, 5);
    __syncthreads();
    {
        const int per = (ntiles + nth - 1) / nth;
        const int a = min(ntiles, tid * per), e = min(ntiles, a + per);
        int sum = 0;
        for (int i = a; i < e; ++i) sum += pre[i + 1];
        int incl = sum;  // inclusive scan of the thread sums within the warp
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            const int nwarps = nth / 32;
            int w = lane < nwarps ? wsum[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += v;
            }
            if (lane < nwarps) wsum[lane] = w;  // inclusive over warps
        }
        __syncthreads();
        int run = (warp > 0 ? wsum[warp - 1] : 0) + incl - sum;  // exclusive start of this thread
        for (int i = a; i < e; ++i) {
            run += pre[i + 1];
            pre[i + 1] = run;
        }
    }
    __syncthreads();
    trace_stamp(trace, 1, 6);
    // Ranges in ARRIVAL order with tapered sizes: KB's CTAs become resident as KA's CTAs drain (a few
    // us apart), so the r-th CTA of part q to arrive takes range r, and range sizes shrink linearly
    // (weights 4R - r : 4R - r ... about +-14%) so that late arrivals finish with the early ones. The
    // boundaries are a fixed function of (U, R) and the partials are summed in range order: which CTA
    // computes which range does not change a bit of y.
    if (tid == 0) s_rr = (int)rr_ticket;
    __syncthreads();
    trace_stamp(trace, 1, 7);  // range ticket known
    const int rr = s_rr;
    const long long U = pre[ntiles];
    auto wcum = [R](long long r) { return r * (4LL * R + 1) - r * (r - 1) / 2; };  // sum_{i<r} (4R - i)
    const int lo = (int)(U * wcum(rr) / wcum(R)), hi = (int)(U * wcum(rr + 1) / wcum(R)), len = hi - lo;
    CATS_DCHECK(rr < R && 0 <= lo && lo <= hi && hi <= U && len <= maxr);

    // ---- this range's neurons: one thread per tile scatters the tile's active rows whose compact ranks
    //      g = pre[tau] + k fall in [lo, hi) (no search: every tile is one independent shared-memory read) ----
    for (int tau = tid; tau < ntiles; tau += nth) {
        const int p0 = pre[tau], p1 = pre[tau + 1];
        if (p1 <= lo || p0 >= hi) continue;
        unsigned int msk = rowm[tau];
        for (int g = p0; g < p1; ++g, msk &= msk - 1u) {  // k-th set row of the tile = rank p0 + k
            if (g < lo || g >= hi) continue;
            lj[g - lo] = tau * nr_tile + (__ffs(msk) - 1);
            lpos[g - lo] = tau * nr_tile + (g - p0);
            CATS_DCHECK(msk != 0u && g - p0 < nr_tile);
        }
    }
    __syncthreads();
    trace_stamp(trace, 1, 1);
    const int njobs = (len + rows_per_stage - 1) / rows_per_stage;

    if (warp == NCW) {
        // ---- producer: W_down row segments [j][q*part_cols, (q+1)*part_cols) into the ring ----
        const uint64_t policy = l2_evict_first_policy();
        for (int jn = 0; jn < njobs; ++jn) {
            const int s = jn % stages;
            if (jn >= stages) mbar_wait(&empty[s], (uint32_t)((jn / stages) - 1) & 1u);
            const int r0 = jn * rows_per_stage, nrow = min(rows_per_stage, len - r0);
            if (lane == 0) mbar_arrive_expect_tx(&full[s], (uint32_t)nrow * seg_bytes);
            __syncwarp();
            if (lane < nrow)
                bulk_g2s(ring + (size_t)s * stage_bytes + (size_t)lane * sst,
                         Wd + (size_t)lj[r0 + lane] * d + (size_t)q * part_cols, seg_bytes, &full[s], policy);
        }
    } else {
        // ---- consumers: y[tk][c] += x1[j][tk] * W_down[j][c] over the range, list order, fp32 ----
        pdl_wait_primary();  // x1 comes from KA's UP jobs: KA must have completed
        if constexpr (MT > 0) {
            // the MMA B operand, built once per CTA instead of once per warp and k-step: per neuron pair
            // (2 i, 2 i + 1) and token, the bf16x2 hi and lo parts of x1 (zero past the range, up to the
            // next 16-neuron k-step)
            uint2 *lxp = reinterpret_cast<uint2 *>(lx);
            const int npair = ((len + 15) / 16) * 8;
            for (int i = tid; i < npair * B; i += NCt) {
                const int pr = i / B, tk = i % B, r = 2 * pr;
                const float v0 = r < len ? __ldcg(x1in + (size_t)lpos[r] * B + tk) : 0.f;
                const float v1 = r + 1 < len ? __ldcg(x1in + (size_t)lpos[r + 1] * B + tk) : 0.f;
                const __nv_bfloat162 hi = __floats2bfloat162_rn(v0, v1);
                const float2 hf = __bfloat1622float2(hi);
                const __nv_bfloat162 lo = __floats2bfloat162_rn(v0 - hf.x, v1 - hf.y);
                lxp[i] = make_uint2(*reinterpret_cast<const uint32_t *>(&hi), *reinterpret_cast<const uint32_t *>(&lo));
            }
        } else {
            for (int i = tid; i < len * B; i += NCt) lx[i] = __ldcg(x1in + (size_t)lpos[i / B] * B + (i % B));
        }
        asm volatile("bar.sync 1, %0;" ::"r"(NCt) : "memory");  // consumers only
        if constexpr (MT > 0) {
            // ---- tensor cores (bf16): D[16 cols x 8 tokens] += A[16 cols x 16 neurons] B[16 neurons x 8]
            //      A = W_down^T from the stage (ldmatrix .trans), B = x1 split exactly enough into
            //      bf16 hi + lo (two MMAs; |x1 - hi - lo| <= 2^-16 |x1|). Warp w owns MT 16-column
            //      tiles; 16 neurons (one stage) per k-step, in list order: deterministic. ----
            const int g4 = lane >> 2, t4 = lane & 3;
            const int col0 = warp * MT * 16;  // within the part
            float dacc[MT][4];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int e = 0; e < 4; ++e) dacc[mt][e] = 0.f;
            const int mat = lane >> 3, r8 = lane & 7;
            for (int jn = 0; jn < njobs; ++jn) {
                const int s = jn % stages;
                mbar_wait(&full[s], (uint32_t)(jn / stages) & 1u);
                const int rs0 = jn * rows_per_stage, nrs = min(rows_per_stage, len - rs0);
                // one 16-neuron MMA k-step per 16 rows of the stage (rows_per_stage = 16 or 32)
                for (int k0 = 0; k0 < nrs; k0 += 16) {
                const int r0 = rs0 + k0, nrow = min(16, nrs - k0);
                // B fragments: x1 of neurons 2 t4, 2 t4 + 1 (b0) and 2 t4 + 8, + 9 (b1), token g4, as the
                // precomputed bf16 hi + lo pairs (|x1 - hi - lo| <= 2^-16 |x1|)
                uint32_t bh[2], bl[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint2 v = g4 < B ? reinterpret_cast<const uint2 *>(lx)[(size_t)((r0 >> 1) + 4 * h + t4) * B + g4]
                                           : make_uint2(0u, 0u);
                    bh[h] = v.x;
                    bl[h] = v.y;
                }
                // A: lane -> neuron row r8 + 8 (mat / 2) (rows past nrow repeat row 0: finite, x1 = 0),
                //    columns + 8 (mat % 2)
                const int arow = r8 + 8 * (mat >> 1);
                const uint32_t abase = smem_u32(ring + (size_t)s * stage_bytes) + (uint32_t)(k0 + (arow < nrow ? arow : 0)) * sst +
                                       (uint32_t)(col0 + 8 * (mat & 1)) * 2u;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    uint32_t a0, a1, a2, a3;
                    ldsm_x4_trans(abase + (uint32_t)mt * 32u, a0, a1, a2, a3);
                    mma_bf16_16816(dacc[mt], a0, a1, a2, a3, bh[0], bh[1]);
                    mma_bf16_16816(dacc[mt], a0, a1, a2, a3, bl[0], bl[1]);
                }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }
            // lane (g4, t4): D[col g4 (+8)][token 2 t4 (+1)]
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int c = col0 + mt * 16 + g4 + 8 * (e >> 1), tk = 2 * t4 + (e & 1);
                    if (tk < B) part[((size_t)rr * B + tk) * d + (size_t)q * part_cols + c] = dacc[mt][e];
                }
            }
        } else {
        const int c0 = tid * EPT;  // first column of this thread within the part
        const bool own = c0 < part_cols;
        float acc[B][EPT];
#pragma unroll
        for (int tk = 0; tk < B; ++tk)
#pragma unroll
            for (int e = 0; e < EPT; ++e) acc[tk][e] = 0.f;
        for (int jn = 0; jn < njobs; ++jn) {
            const int s = jn % stages;
            mbar_wait(&full[s], (uint32_t)(jn / stages) & 1u);
            const int r0 = jn * rows_per_stage, nrow = min(rows_per_stage, len - r0);
            if (own) {
                const uint32_t sb = smem_u32(ring + (size_t)s * stage_bytes) + (uint32_t)c0 * sizeof(T);
                for (int i = 0; i < nrow; ++i) {
                    float wf[EPT];
                    if constexpr (EB == 16) {
                        unpack16(lds128(sb + (uint32_t)i * sst), wf);
                    } else {  // 8 bytes = 4 bf16
                        uint32_t w0, w1;
                        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w0), "=r"(w1) : "r"(sb + (uint32_t)i * sst));
                        wf[0] = __uint_as_float(w0 << 16);
                        wf[1] = __uint_as_float(w0 & 0xffff0000u);
                        wf[2] = __uint_as_float(w1 << 16);
                        wf[3] = __uint_as_float(w1 & 0xffff0000u);
                    }
                    const float *xr = lx + (size_t)(r0 + i) * B;
#pragma unroll
                    for (int tk = 0; tk < B; ++tk) {
                        const float a = xr[tk];
#pragma unroll
                        for (int e = 0; e < EPT; ++e) acc[tk][e] = fmaf(a, wf[e], acc[tk][e]);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        if (own) {  // partial of range rr, columns of part q
#pragma unroll
            for (int tk = 0; tk < B; ++tk) {
                float *dst = part + ((size_t)rr * B + tk) * d + (size_t)q * part_cols + c0;
#pragma unroll
                for (int e = 0; e < EPT; e += 4)
                    *reinterpret_cast<float4 *>(dst + e) = make_float4(acc[tk][e], acc[tk][e + 1], acc[tk][e + 2], acc[tk][e + 3]);
            }
        }
        }
    }
    trace_stamp(trace, 1, 2);

    // ---- phase 2 by the LAST kKbReducers CTAs to finish phase 1 (no grid barrier) ----
    // Every CTA takes an arrival ticket after its partial is written; the CTAs with the last K tickets
    // wait until all G have arrived and then each sums a slice of the R partials in fixed order
    // r = 0..R-1 into y. The others exit at once (their SMs go to the next kernel). A reducer only ever
    // waits for CTAs that have not arrived yet, and at most K of the SM slots are held by reducers, so
    // the kernel completes whenever more than K CTAs fit on the device at once -- no co-residency of the
    // whole grid is assumed (the planner checks the occupancy).
    __shared__ unsigned int s_ticket;
    __syncthreads();
    if (tid == 0) {
        __threadfence();  // this CTA's partial is visible before its ticket
        s_ticket = atomicAdd(&sched[2], 1u);
    }
    __syncthreads();
    const int G = gridDim.x;
    const int K = min(G, kKbReducers);
    const int red_idx = (int)s_ticket - (G - K);  // < 0: not a reducer
    if (red_idx < 0) {
        trace_stamp(trace, 1, 3);
        trace_stamp(trace, 1, 4);
        return;
    }
    if (tid == 0) {
        unsigned int seen;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(sched + 2) : "memory");
        } while (seen < (unsigned)G);
    }
    __syncthreads();
    trace_stamp(trace, 1, 3);
    for (int i = red_idx * nth + tid; i < ntiles; i += K * nth) tmask[i] = 0u;  // for the next call
    if (red_idx == 0 && tid < Q) sched[8 + tid] = 0u;  // arrival tickets (all taken before the tickets)

    // ---- fixed-order reduction: y[e] = sum_{r=0..R-1} part[r][e], this reducer's slice of B*d ----
    {
        const int total4 = B * d / 4;
        const int g0 = (int)((long long)total4 * red_idx / K), g1 = (int)((long long)total4 * (red_idx + 1) / K);
        const int ng = g1 - g0;
        // r-slices per float4 group: enough that each thread has <= 8 partials (one batch of loads)
        const int ns = ng > 0 ? max(1, min(min(R, nth / ng), max((R + 7) / 8, 4))) : 1;
        const float4 *p4 = reinterpret_cast<const float4 *>(part);
        if (ns == 1) {  // (few CTAs) each thread sums whole columns
            for (int i = tid; i < ng; i += nth) {
                float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
                for (int r = 0; r < R; r += 8) {
                    float4 v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        v[u] = r + u < R ? __ldcg(p4 + (size_t)(r + u) * total4 + g0 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        a.x += v[u].x; a.y += v[u].y; a.z += v[u].z; a.w += v[u].w;
                    }
                }
                reinterpret_cast<float4 *>(y)[g0 + i] = a;
            }
        } else {  // ng * ns <= nth: slice sums into the (idle) ring, then a fixed-order sum of slices
            float4 *red4 = reinterpret_cast<float4 *>(ring);
            if (tid < ng * ns) {
                const int grp = tid % ng, sl = tid / ng;
                float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
                for (int r = sl; r < R; r += 8 * ns) {  // 8 loads in flight, summed in r order
                    float4 v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        v[u] = r + u * ns < R ? __ldcg(p4 + (size_t)(r + u * ns) * total4 + g0 + grp)
                                              : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        a.x += v[u].x; a.y += v[u].y; a.z += v[u].z; a.w += v[u].w;
                    }
                }
                red4[sl * ng + grp] = a;
            }
            __syncthreads();
            if (tid < ng) {
                float4 a = red4[tid];
                for (int sl = 1; sl < ns; ++sl) {
                    const float4 v = red4[sl * ng + tid];
                    a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
                }
                reinterpret_cast<float4 *>(y)[g0 + tid] = a;
            }
        }
    }
    trace_stamp(trace, 1, 4);
}

// ================================================================================== host side
// KA dot-product engine: 1 = warp-level bf16 MMA (bf16 weights, b >= kSplitMmaMinB), 0 = FHFMA.BF16 / FFMA.
// Measured (Llama2-7B): the MMA path wins from b = 4 (b = 8: KA 58 -> 38 us); at b = 2 its ldmatrix
// traffic (x re-read per job, half the B columns duplicated) made it slower than FHFMA. With x in tensor
// memory it wins from b = 3 (Llama2-7B 47.9 vs 52.4 us, Mistral 58.8 vs 63.6, Llama2-13B 69.6 vs 73.7;
// b = 2 still 0.1-1.2 us slower, A/B on one box).
// 2 = MMA in column parts (ka_colsplit: 8-row tiles, jobs of d / kKaPartCols stages)
// 3 = MMA with x in tensor memory (d % 1024 == 0: each warp's k-steps come in whole 8-step TMEM loads)
int split_ka_ks(const PlanData &p, int b) {
    if (ka_colsplit(p, b)) return 2;
    if (p.esize == 2 && b >= kSplitMmaMinB) return ka_x_in_tmem(p, b) ? 3 : 1;
    return 0;
}
static size_t ka_stage_row_bytes(const PlanData &p, int b) {  // bytes of one row in a ring stage (unpadded)
    return (size_t)(ka_colsplit(p, b) ? kKaPartCols : p.d) * p.esize;
}
// KA shared memory: x [b][d] (FHFMA path only), then per group (kSplitAGroups): the ring of padded
// rows, 2 mbarriers, a descriptor and the warp partial sums per stage, and the FIFO. `stages` counts
// stages per group.
static size_t split_ka_per_stage_nr(const PlanData &p, int b, int nr) {
    const size_t desc = (4 + 2 * (size_t)nr + (size_t)nr * b) * 4;  // sizeof(SplitDesc<nr, b>)
    return (size_t)nr * ((size_t)p.d * p.esize + 16) + 16 + desc +
           (size_t)(kSplitAWarps / kSplitAGroups) * pow2_ceil(nr * b) * 4;
}
// KA ring stages per group with tiles of nr rows (used by k12_rows_per_tile to pick nr at b >= 2)
int split_ka_stages_nr(const PlanData &p, int b, int nr) {
    const size_t ent = (2 + (size_t)b) * 4;
    const size_t xs = ka_x_in_tmem(p, b) ? 0
                      : (size_t)b * ((size_t)p.d * p.esize + ((p.esize == 2 && b >= kSplitMmaMinB) ? 16 : 0));
    const size_t fixed = xs + kSplitAGroups * kSplitFifo * ent;
    if (fixed >= kSmemBudget) return 0;
    return (int)std::min<size_t>((kSmemBudget - fixed) / (kSplitAGroups * split_ka_per_stage_nr(p, b, nr)), kMaxStages);
}
static size_t split_ka_per_stage(const PlanData &p, int b) {
    const int nr = split_rows_per_tile(p, b);
    const size_t desc = (4 + 2 * (size_t)nr + (size_t)nr * b) * 4;  // sizeof(SplitDesc<nr, b>)
    return (size_t)nr * (ka_stage_row_bytes(p, b) + 16) + 16 + desc +
           (size_t)(kSplitAWarps / kSplitAGroups) * pow2_ceil(nr * b) * 4;
}
size_t split_ka_smem(const PlanData &p, int b, int stages) {
    const size_t ent = (2 + (size_t)b) * 4;  // sizeof(SplitFifoEntry<b>)
    const size_t desc = (4 + 2 * (size_t)split_rows_per_tile(p, b) + (size_t)split_rows_per_tile(p, b) * b) * 4;
    const int ks = split_ka_ks(p, b);
    const size_t xs = ks == 3 ? 0 : (size_t)b * ((size_t)p.d * p.esize + (ks > 0 ? 16 : 0));
    // column parts: one more descriptor per group (the job being streamed part by part)
    const size_t fifo = split_ka_ks(p, b) == 2 ? kSplitFifoCs : kSplitFifo;
    return xs + kSplitAGroups * ((size_t)stages * split_ka_per_stage(p, b) + fifo * ent +
                                 (split_ka_ks(p, b) == 2 ? desc : 0));
}
int split_ka_stages(const PlanData &p, int b) {
    const size_t fixed = split_ka_smem(p, b, 0);
    if (fixed >= kSmemBudget) return 0;
    return (int)std::min<size_t>((kSmemBudget - fixed) / (kSplitAGroups * split_ka_per_stage(p, b)), kMaxStages);
}
static int split_kb_maxr(const PlanData &p, int b) {  // the largest (first) tapered range, + rounding
    const long long R = split_ranges(p, b);
    const long long wtot = R * (4 * R + 1) - R * (R - 1) / 2;
    return (int)(((long long)p.m * 4 * R + wtot - 1) / wtot) + 2;
}
static size_t split_kb_fixed_smem(const PlanData &p, int b) {  // everything but the ring's stages
    const int ntiles = split_ntiles(p, b), maxr = split_kb_maxr(p, b);
    // x1 of the range: fp32 [maxr][b], or (MMA path) bf16x2 hi + lo per neuron pair up to a whole k-step
    const size_t lx = split_kb_mma(p, b) ? (size_t)((maxr + 15) / 16) * 16 * b * 4 : (size_t)maxr * b * 4;
    return (size_t)(ntiles + 1 + 32) * 4 + (size_t)maxr * 8 + lx + (size_t)ntiles;
}
static int split_kb_rows_per_stage(const PlanData &p, int b) {
    // (rows per stage <= 32: one bulk copy per producer lane)
    if (split_kb_mma(p, b)) {  // 16-neuron MMA k-steps: two per stage where 3 such stages fit, else one
        const size_t seg = (size_t)split_part_cols(p, b) * p.esize + 16;
        return 3 * (32 * seg + 16) + split_kb_fixed_smem(p, b) <= kSmemBudget ? 32 : 16;
    }
    // CUDA cores: ~32 KB stages; ~64 KB at b = 1 (KB runs at b = 1 only for d >= 5120: Llama2-13B and
    // its TP shards, 51.4 / 16.9 vs 52.3 / 17.2 us; at b = 2 the larger stages measured 0.1-0.6 us slower)
    const size_t seg = (size_t)split_part_cols(p, b) * p.esize;
    return (int)std::max<size_t>(1, std::min<size_t>(32, ((b == 1 ? 64 : 32) * 1024) / seg));
}
size_t split_kb_smem(const PlanData &p, int b, int stages) {
    const size_t seg = (size_t)split_part_cols(p, b) * p.esize + 16;  // padded rows
    const size_t stage = (size_t)split_kb_rows_per_stage(p, b) * seg;
    return (size_t)stages * stage + (size_t)stages * 16 + split_kb_fixed_smem(p, b);
}
int split_kb_stages(const PlanData &p, int b) {
    const size_t seg = (size_t)split_part_cols(p, b) * p.esize + 16;  // padded rows
    const size_t stage = (size_t)split_kb_rows_per_stage(p, b) * seg;
    const size_t fixed = split_kb_smem(p, b, 0);
    if (fixed >= kSmemBudget) return 0;
    int st = (int)std::min<size_t>((kSmemBudget - fixed) / (stage + 16), kMaxStages);
    // the reduction scratch (one float4 per thread) lives in the ring
    while (st > 0 && (size_t)st * stage < (size_t)kSplitBMaxThreads * 16) ++st;
    return st;
}
bool kb_supported(const PlanData &p, int b) {  // KB alone fits this shape and batch
    if (b < 1 || b > 8) return false;
    if (p.d % (split_q(p, b) * split_ept(p, b)) != 0) return false;
    if (((size_t)split_part_cols(p, b) * p.esize) % 16 != 0) return false;
    if (split_kb_consumers(p, b) + 32 > kSplitBMaxThreads) return false;
    const int sb = split_kb_stages(p, b);
    return sb >= 2 && split_kb_smem(p, b, sb) <= kSmemBudget;
}
bool split_supported(const PlanData &p, int b) {
    // KB's phase 2 holds up to kKbReducers CTAs (one per SM) waiting for the rest: more SMs than that
    if (p.num_sms <= kKbReducers) return false;
    if (b < 1 || b > 8 || !kb_supported(p, b)) return false;
    const int sa = split_ka_stages(p, b);
    return sa >= 2 && split_ka_smem(p, b, sa) <= kSmemBudget;  // >= 2 stages per group
}

static cudaLaunchConfig_t pdl_config(cudaLaunchAttribute *attr, int grid, int threads, size_t smem,
                                     cudaStream_t s) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cfg;
}

template <typename T, int B, int NR, int KS>
static cudaError_t launch_ka(const PlanData &p, const void *x, const void *Wg, const void *Wu, float t, int mode,
                             void *ws, cudaStream_t s) {
    static_assert(sizeof(SplitDesc<NR, B>) == (4 + 2 * NR + NR * B) * 4, "split_ka_smem layout");
    static_assert(sizeof(SplitFifoEntry<B>) == (2 + B) * 4, "split_ka_smem layout");
    auto kern = ka_gate_up<T, B, NR, KS>;
    const int stages = split_ka_stages(p, B);
    const size_t smem = split_ka_smem(p, B, stages);
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void *>(kern), smem);
    if (e != cudaSuccess) return e;
    char *w = static_cast<char *>(ws);
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = pdl_config(attr, split_ka_grid(p, B), kSplitAThreads, smem, s);
    return cudaLaunchKernelEx(&cfg, kern, static_cast<const T *>(x), static_cast<const T *>(Wg),
                              static_cast<const T *>(Wu), p.d, p.m, stages, t, mode,
                              reinterpret_cast<int32_t *>(w + p.off_idx), reinterpret_cast<uint8_t *>(w + p.off_tokmask),
                              reinterpret_cast<float *>(w + p.off_vals), reinterpret_cast<int32_t *>(w + p.off_cnt),
                              reinterpret_cast<unsigned int *>(w + p.off_tmask), reinterpret_cast<float *>(w + p.off_x1),
                              reinterpret_cast<unsigned int *>(w + p.off_sched),
                              p.lazy_tail * split_ka_grid(p, B),
                              p.trace ? reinterpret_cast<unsigned long long *>(w + p.off_trace) : nullptr);
}

template <typename T, int B, int EPT, int MT>
static cudaError_t launch_kb(const PlanData &p, const void *Wd, float *y, void *ws, cudaStream_t s) {
    auto kern = kb_down<T, B, EPT, MT>;
    const int stages = split_kb_stages(p, B);
    const size_t smem = split_kb_smem(p, B, stages);
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void *>(kern), smem);
    if (e != cudaSuccess) return e;
    char *w = static_cast<char *>(ws);
    cudaLaunchAttribute attr[1];
    const int threads = split_kb_consumers(p, B) + 32;
    cudaLaunchConfig_t cfg = pdl_config(attr, split_kb_grid(p, B), threads, smem, s);
    return cudaLaunchKernelEx(&cfg, kern, static_cast<const T *>(Wd), p.d, split_ntiles(p, B), split_rows_per_tile(p, B),
                              split_q(p, B), split_ranges(p, B), stages, split_kb_rows_per_stage(p, B),
                              split_kb_maxr(p, B), reinterpret_cast<unsigned int *>(w + p.off_tmask),
                              reinterpret_cast<const float *>(w + p.off_x1), reinterpret_cast<float *>(w + p.off_part), y,
                              reinterpret_cast<unsigned int *>(w + p.off_sched),
                              p.trace ? reinterpret_cast<unsigned long long *>(w + p.off_trace) : nullptr);
}

// KB for batch B: tensor-core variant where instantiated (split_kb_mt), else CUDA cores
template <typename T, int B>
static cudaError_t launch_kb_b(const PlanData &p, const void *Wd, float *y, void *ws, cudaStream_t s) {
    constexpr int EPT = 4;  // = split_ept()
    if constexpr (sizeof(T) == 2 && B >= kSplitKbMmaMinB) {
        const int mt = split_kb_mt(p, B);
        if (mt == 1) return launch_kb<T, B, EPT, 1>(p, Wd, y, ws, s);
        if (mt == 4) return launch_kb<T, B, EPT, 4>(p, Wd, y, ws, s);
        if (mt == 5) return launch_kb<T, B, EPT, 5>(p, Wd, y, ws, s);
        if (mt != 0) return cudaErrorInvalidValue;
    }
    return launch_kb<T, B, EPT, 0>(p, Wd, y, ws, s);
}

template <typename T, int B>
static cudaError_t launch_split_b(const PlanData &p, const void *x, const void *Wg, const void *Wu, const void *Wd,
                                  float t, int mode, float *y, void *ws, cudaStream_t s, cudaEvent_t ev_mid) {
    cudaError_t e;
    const int ks = split_ka_ks(p, B);
    if constexpr (sizeof(T) == 2 && B >= kSplitMmaMinB) {
        const int nr = split_rows_per_tile(p, B);
        if (ks == 2) {
            e = launch_ka<T, B, 8, 2>(p, x, Wg, Wu, t, mode, ws, s);
        } else if (nr == 6) {
            e = launch_ka<T, B, 6, 3>(p, x, Wg, Wu, t, mode, ws, s);
        } else if (nr == 4) {
            e = ks == 3 ? launch_ka<T, B, 4, 3>(p, x, Wg, Wu, t, mode, ws, s)
                        : launch_ka<T, B, 4, 1>(p, x, Wg, Wu, t, mode, ws, s);
        } else {
            e = ks == 3 ? launch_ka<T, B, 2, 3>(p, x, Wg, Wu, t, mode, ws, s)
                        : launch_ka<T, B, 2, 1>(p, x, Wg, Wu, t, mode, ws, s);
        }
    } else {
        const int nr = split_rows_per_tile(p, B);
        // 6-row tiles: b = 1 on large layers (the split path at b = 1: options), bf16 b = 2, 3 (ka_nr6)
        constexpr bool kNr6 = B == 1 || (sizeof(T) == 2 && B < kSplitMmaMinB);
        if constexpr (kNr6) {
            if (nr == 6) e = launch_ka<T, B, 6, 0>(p, x, Wg, Wu, t, mode, ws, s);
        }
        if (nr != 6) e = nr == 4 ? launch_ka<T, B, 4, 0>(p, x, Wg, Wu, t, mode, ws, s)
                                 : launch_ka<T, B, 2, 0>(p, x, Wg, Wu, t, mode, ws, s);
        else if (!kNr6) e = cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    if (ev_mid) {
        e = cudaEventRecord(ev_mid, s);
        if (e != cudaSuccess) return e;
    }
    return launch_kb_b<T, B>(p, Wd, y, ws, s);
}

template <typename T>
static cudaError_t launch_split_dt(const PlanData &p, const void *x, int b, const void *Wg, const void *Wu,
                                   const void *Wd, float t, int mode, float *y, void *ws, cudaStream_t s,
                                   cudaEvent_t ev) {
    switch (b) {
        case 1: return launch_split_b<T, 1>(p, x, Wg, Wu, Wd, t, mode, y, ws, s, ev);
        case 2: return launch_split_b<T, 2>(p, x, Wg, Wu, Wd, t, mode, y, ws, s, ev);
        case 3: return launch_split_b<T, 3>(p, x, Wg, Wu, Wd, t, mode, y, ws, s, ev);
        case 4: return launch_split_b<T, 4>(p, x, Wg, Wu, Wd, t, mode, y, ws, s, ev);
        case 5: return launch_split_b<T, 5>(p, x, Wg, Wu, Wd, t, mode, y, ws, s, ev);
        case 6: return launch_split_b<T, 6>(p, x, Wg, Wu, Wd, t, mode, y, ws, s, ev);
        case 7: return launch_split_b<T, 7>(p, x, Wg, Wu, Wd, t, mode, y, ws, s, ev);
        case 8: return launch_split_b<T, 8>(p, x, Wg, Wu, Wd, t, mode, y, ws, s, ev);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_split(const PlanData &p, const void *x, int b, const void *Wg, const void *Wu, const void *Wd,
                         float t, int mode, float *y, void *ws, cudaStream_t s, cudaEvent_t ev_mid) {
    if (p.dt == CATS_BF16) return launch_split_dt<bf16_bits>(p, x, b, Wg, Wu, Wd, t, mode, y, ws, s, ev_mid);
    return launch_split_dt<float>(p, x, b, Wg, Wu, Wd, t, mode, y, ws, s, ev_mid);
}

}  // namespace cats
