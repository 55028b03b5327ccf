// mlp_fused.cu -- the CATS-MLP decode as ONE persistent dataflow kernel (K12).
//
// Paper: Custom GPU Kernel "MLP using CATS":
//     v <- SiLU(x W_gate); Mask <- |v| >= t; x1 <- (x W_up[Mask]) * v[Mask]; y <- x1 W_down[Mask]
// Eq. 1, Eq. 2 SiLU, Eq. 4/5 CATS_t, Optimization 1 -- the x v
// multiply fused into the up tile so x1 never touches HBM, and App. D
// Alg. 1 line 4 "idcs <- indices where Mask = 1" done per tile with a warp ballot (no
// atomic appends).
//
// B200 design:
//  * Work unit = a tile of NR consecutive neurons (6 / 4 / 2, k12_rows_per_tile). Persistent CTAs
//    (two per SM at b = 1, one at b >= 2) take their first tiles statically -- issued before
//    griddepcontrol.wait, so they stream while the previous kernel drains -- and the rest from a
//    global counter (one tile reserved ahead, none in the last 8 x grid tiles): SMs with more
//    bandwidth take more tiles, and there is no grid-wide barrier between the gate GEMV and the
//    sparse up/down projection.
//  * Each CTA runs a ring of S shared-memory stages fed by the TMA bulk-copy engine
//    (cp.async.bulk + mbarrier transaction counts, L2 evict-first). A stage holds one JOB:
//        GATE(tile): the tile's NR rows of W_gate (neuron-major, contiguous: one copy);
//        UD(<= NU = NR/2 active neurons of one tile): their W_up and W_down rows (one copy per row).
//  * Warp specialisation: 8 (b = 1) or 16 consumer warps do the arithmetic; one producer warp retires
//    jobs in order (full/empty mbarrier pair per stage), turns a GATE job's partial dot products into
//    u -> v = SiLU(u) -> keep = |v| >= t -> ballot compaction, queues the tile's active neurons as
//    UD jobs, and refills freed stages (UD jobs first, else a new GATE tile). UD rows are requested
//    S-1 jobs before they are consumed, so the mask -> load dependency is hidden and only active
//    neurons' W_up / W_down rows are ever read (the paper's memory saving).
//  * Consumer thread t owns 16-byte column chunks {t, t + NC, ...} of d; x stays in registers,
//    packed; dot products use FHFMA.BF16 (bf16 x bf16 -> fp32 straight from the packed registers),
//    a fixed xor butterfly per warp, then a fixed-order sum over the warps. GATE jobs need no
//    consumer barrier; UD jobs one named barrier.
//  * Determinism under dynamic scheduling: a UD job's contribution y_job[c] = sum_i x1_i Wd[i][c]
//    (<= NU neurons of ONE tile, ascending, fp32, fixed order) is converted once to an exact
//    fixed-point integer round(y_job * 2^38) (split into two int32 halves, cats_device.cuh
//    fix_acc) and added to the thread's integer accumulator. Integer
//    addition is associative, so y does not depend on which CTA took which tile or in which order:
//    bit-reproducible. (Replaces the paper's fp16 tl.atomic_add into Y.)
//  * Split-K reduction: each CTA stages its integer partial in the (idle) ring and bulk-reduces it
//    (TMA cp.reduce.async.bulk .add.u64) into one global accumulator; the last CTA converts it to
//    fp32 once, writes y and re-arms the tile counter. Two accumulators alternate per call: the next
//    call's CTAs zero the one just converted, so the last CTA only reads.
//
// Workspace outputs for introspection: tile tau's cnt[tau] active neurons are written ascending at
// positions [tau*NR, tau*NR + cnt[tau]) of idx / tokmask / vals (v in fp32, 0 where |v| < t).
//
// The App. D ablation modes (Alg. 2 mask-predicated loads, Alg. 1 atomic appends + list launch; DESIGN.md
// §5.9) are a separate instantiation of the same kernel (template flag ABL), so the product kernel
// carries none of their branches.
#include "cats_device.cuh"
#include "cats_internal.h"

namespace cats {

enum : int { kJobEnd = 0, kJobGate = 1, kJobUD = 2 };



template <int NU, int B>
struct JobDesc {
    int type;        // kJobEnd / kJobGate / kJobUD
    int tile;        // tile id
    int n;           // rows (GATE) or neurons (UD) in the stage
    int id[NU];      // UD: neuron ids, ascending
    float v[NU][B];  // UD: v = SiLU(u) per token, 0 where the token's |v| < t
};

constexpr unsigned int kNoTile = 0xffffffffu;

// if (pred) t = atomicAdd(sched, 1) without a select on the result: the destination is written by a
// predicated ATOM, so the warp only waits for it where t is next read.
__device__ __forceinline__ void claim_tile_async(unsigned int &t, unsigned int *sched, bool pred) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p atom.global.add.u32 %0, [%1], 1;\n\t}"
                 : "+r"(t)
                 : "l"(sched), "r"((unsigned)pred)
                 : "memory");
}

// ABL: the App. D ablation modes (kModePredicated, kModeAtomicGate, kModeAtomicList) are compiled in.
// The default instantiation (ABL = false) carries only the CATS / dense / gate-only paths: the ablation
// branches cost registers and issue slots in the producer's refill loop even when never taken
// (measured: 42.3 vs 41.8 us per Mistral-7B layer with them compiled into the default kernel).
template <typename T, int B, int NR, int CPT, bool ABL>
__global__ void __launch_bounds__(k12_threads_c(B), k12_ctas_per_sm_c(B))
k12_cats_mlp(const T *__restrict__ x, const T *__restrict__ Wg, const T *__restrict__ Wu, const T *__restrict__ Wd,
             int d, int m, int stages, float t, int mode, int32_t *__restrict__ idx, uint8_t *__restrict__ tokmask,
             float *__restrict__ vals, int32_t *__restrict__ cnt, float *__restrict__ acts,
             unsigned long long *__restrict__ yacc, float *__restrict__ y, unsigned int *__restrict__ sched,
             int32_t *__restrict__ gidx, float *__restrict__ gval,
             int ystride, int lazy_tail, int eager, int l2pf, unsigned long long *__restrict__ trace) {
    constexpr int NU = NR / 2;   // neurons per UD job (2 rows each) = the bytes of a GATE job
    constexpr int VEC = VecTraits<T>::kVec;
    constexpr int NW = k12_consumer_warps_c(B);
    constexpr int NC = NW * 32;
    static_assert(32 % NW == 0, "cross-warp reduction packs 32 / NW pairs per round");
    constexpr int NPG = NR * B;  // (row, token) gate dot products per GATE job
    constexpr int NPU = NU * B;  // (neuron, token) up dot products per UD job
    constexpr int NPMAX = NPG > NPU ? NPG : NPU;
    constexpr int QCAP = 64;     // pending UD jobs (each retired GATE adds <= 2, each refill takes 1)
    static_assert(NR <= 32, "a GATE tile is compacted by one warp ballot");
    using Desc = JobDesc<NU, B>;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nch = d * (int)sizeof(T) / 16;
    const uint32_t row_bytes = (uint32_t)d * (uint32_t)sizeof(T);
    const uint32_t stage_bytes = (uint32_t)NR * row_bytes;
    const int ntiles = (m + NR - 1) / NR;
    const bool list_mode = ABL && mode == kModeAtomicList;  // App. D Alg. 1, launch 2: work units = chunks of idcs
    const bool atomic_gate = ABL && mode == kModeAtomicGate;  // App. D Alg. 1, launch 1: gate + atomic appends
    const bool has_y = mode != kModeGateOnly && !atomic_gate;

    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char *ring = smem;                                                           // [stages][stage_bytes]
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + (size_t)stages * stage_bytes);   // [stages]
    uint64_t *empty = full + stages;                                                      // [stages]
    Desc *desc = reinterpret_cast<Desc *>(empty + stages);                                // [stages]
    Desc *queue = desc + stages;                                                          // [QCAP]
    float *red = reinterpret_cast<float *>(queue + QCAP);                                 // [stages][NW][NPMAX]

    trace_stamp(trace, 0, 0);
    pdl_launch_dependents();  // a PDL successor may be scheduled once every CTA has started

    if (tid == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == NW) {
        // ===================================== PRODUCER WARP =====================================
        const bool dense = mode == kModeDense;
        const bool gate_only = mode == kModeGateOnly || atomic_gate;  // no UD jobs from this launch
        const bool predicated = ABL && mode == kModePredicated;
        const uint64_t policy = l2_evict_first_policy();
        // Tile claims (lane 0). While many tiles remain, the next GATE tile is reserved one issue ahead
        // (t_res: a predicated atomic whose round trip overlaps the jobs in between; nothing reads
        // it until the next GATE issue). For the last `lazy_tail` tiles no CTA reserves: a tile is
        // claimed when a stage is free to stream it, so no CTA sits on unstarted work while others
        // drain (balanced tail), and small layers spread over all CTAs.
        unsigned int t_res = kNoTile;  // raw counter value; tile id = dyn_base + counter
        unsigned int sched_list_n = 0; // list mode: length of the global idcs list
        // static first tiles per CTA: `stages` of them go straight into the ring, up to l2pf more are
        // prefetched into L2 (cp.async.bulk.prefetch) -- both before griddepcontrol.wait, so they use
        // the HBM time while the previous kernel drains -- and taken in order before any claim
        const int batch = list_mode ? 0 : max(1, min(stages + l2pf, ntiles / (int)gridDim.x));
        int ntl = ntiles;            // claimable work units: GATE tiles, or (list mode) idcs chunks of NU
        const unsigned int dyn_base = gridDim.x * (unsigned)batch;        // first dynamically claimed tile
        const unsigned int sbase = blockIdx.x * (unsigned)batch;          // this CTA's static tiles
        int snext = min(batch, stages);                                    // next static tile to issue
        int prod = 0;                // jobs issued; job j lives in stage j % stages
        int ps = 0;                  // = prod % stages
        int retire = 0;              // jobs retired (consumed and post-processed), in order
        int q_head = 0, q_tail = 0;  // pending UD jobs
        int gates_inflight = 0;      // GATE jobs issued, not yet retired
        bool ended = false;
        unsigned long long p_wait = 0, p_busy = 0, p_issue = 0, t_last_gate = 0;  // diagnostics (options.trace)

        // issue job `prod` into its stage; returns false if nothing can be issued yet
        auto issue_job = [&]() -> bool {
            const int s = ps;
            Desc &D = desc[s];
            unsigned char *dst = ring + (size_t)s * stage_bytes;
            if (q_head != q_tail) {  // UD job: W_up and W_down rows of <= NU active neurons
                const Desc &Q = queue[q_head % QCAP];
                const int qn = Q.n;
                // a negative id marks a row whose load Mask predicates off (Alg. 2 mode): no copy, read as 0
                bool has = lane < 2 * qn;
                uint32_t nrows = (uint32_t)qn * 2u;
                if constexpr (ABL) {
                    has = has && Q.id[lane >> 1] >= 0;
                    nrows = (uint32_t)__popc(__ballot_sync(0xffffffffu, has));
                }
                if (lane == 0) {
                    D = Q;
                    mbar_arrive_expect_tx(&full[s], nrows * row_bytes);
                }
                __syncwarp();
                CATS_DCHECK(q_tail - q_head <= QCAP);
                if (has) {  // one bulk copy per lane: row (lane & 1) of neuron lane >> 1
                    const int i = lane >> 1;
                    const size_t j = (size_t)Q.id[i];
                    CATS_DCHECK(j < (size_t)m && (size_t)(lane + 1) * row_bytes <= stage_bytes);
                    bulk_g2s(dst + (size_t)lane * row_bytes, ((lane & 1) ? Wd : Wu) + j * d, row_bytes, &full[s],
                             policy);
                }
                ++q_head;
            } else if (list_mode) {  // Alg. 1 list kernel: UD job = the next NU entries of the global idcs
                unsigned int tile = t_res;
                if (lane == 0 && tile == kNoTile) tile = atomicAdd(&sched[0], 1u);
                tile = __shfl_sync(0xffffffffu, tile, 0);
                if (tile < (unsigned)ntl) {
                    if (lane == 0) {
                        t_res = kNoTile;
                        claim_tile_async(t_res, sched, tile + (unsigned)lazy_tail < (unsigned)ntl);
                    }
                    const int base = (int)tile * NU;
                    const int qn = min(NU, (int)sched_list_n - base);
                    CATS_DCHECK(qn >= 1 && sched_list_n <= (unsigned)m);
                    if (lane < qn) {
                        D.id[lane] = __ldcg(gidx + base + lane);
#pragma unroll
                        for (int tk = 0; tk < B; ++tk) D.v[lane][tk] = __ldcg(gval + (size_t)(base + lane) * B + tk);
                    }
                    __syncwarp();
                    if (lane == 0) {
                        D.type = kJobUD;
                        D.tile = (int)tile;
                        D.n = qn;
                        mbar_arrive_expect_tx(&full[s], (uint32_t)qn * 2u * row_bytes);
                    }
                    __syncwarp();
                    if (lane < 2 * qn)
                        bulk_g2s(dst + (size_t)lane * row_bytes, ((lane & 1) ? Wd : Wu) + (size_t)D.id[lane >> 1] * d,
                                 row_bytes, &full[s], policy);
                } else {
                    if (lane == 0) {
                        t_res = tile;  // past the end: keep it, no further claims
                        D.type = kJobEnd;
                        D.n = 0;
                        mbar_arrive_expect_tx(&full[s], 0u);
                    }
                    ended = true;
                }
            } else {
                unsigned int tile;
                const bool from_static = snext < batch;
                if (from_static) {  // a static tile (L2-prefetched at start)
                    tile = sbase + (unsigned)snext;
                } else {
                    tile = t_res;
                    if (lane == 0 && tile == kNoTile) tile = atomicAdd(&sched[0], 1u);  // claim now
                    tile = __shfl_sync(0xffffffffu, tile, 0) + dyn_base;
                }
                if (tile < (unsigned)ntiles) {  // GATE job: a new tile of W_gate rows
                    const int r0 = (int)tile * NR;
                    const int nr = min(NR, m - r0);
                    CATS_DCHECK(r0 >= 0 && nr >= 1 && r0 + nr <= m && (uint32_t)nr * row_bytes <= stage_bytes);
                    if (from_static) {
                        ++snext;
                    } else if (lane == 0) {
                        t_res = kNoTile;
                        claim_tile_async(t_res, sched, tile + (unsigned)lazy_tail < (unsigned)ntl);
                    }
                    if (lane == 0) {
                        D.type = kJobGate;
                        D.tile = (int)tile;
                        D.n = nr;
                        mbar_arrive_expect_tx(&full[s], (uint32_t)nr * row_bytes);
                        bulk_g2s(dst, Wg + (size_t)r0 * d, (uint32_t)nr * row_bytes, &full[s], policy);
                    }
                    ++gates_inflight;
                    if (trace) t_last_gate = gtimer();
                } else {
                    if (lane == 0) t_res = tile - dyn_base;  // past the end: keep it, no further claims
                    if (gates_inflight != 0) return false;  // an in-flight GATE job may add UD work
                    // no tiles left and nothing in flight can create UD work: end the ring
                    if (lane == 0) {
                        D.type = kJobEnd;
                        D.n = 0;
                        mbar_arrive_expect_tx(&full[s], 0u);
                    }
                    ended = true;
                }
            }
            __syncwarp();
            ++prod;
            if (++ps == stages) ps = 0;
            return true;
        };

        if (lane == 0) {
            // Prime the ring with this CTA's static first batch of GATE tiles (at most its fair share,
            // so small layers spread over all CTAs). Weights are read-only, so the loads may start
            // before the PDL predecessor has finished; everything it writes (tile counter, y
            // accumulator, x, index lists) is touched only after griddepcontrol.wait below.
            for (int s = batch > stages ? stages : batch; s < batch; ++s) {  // the rest of the static tiles -> L2
                const int r0 = (int)(sbase + s) * NR;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Wg + (size_t)r0 * d),
                             "r"((uint32_t)min(NR, m - r0) * row_bytes)
                             : "memory");
            }
            for (int s = 0; s < min(batch, stages); ++s) {
                const unsigned int tile = sbase + s;  // grid * batch <= ntiles
                const int r0 = (int)tile * NR;
                const int nr = min(NR, m - r0);
                desc[s].type = kJobGate;
                desc[s].tile = (int)tile;
                desc[s].n = nr;
                mbar_arrive_expect_tx(&full[s], (uint32_t)nr * row_bytes);
                bulk_g2s(ring + (size_t)s * stage_bytes, Wg + (size_t)r0 * d, (uint32_t)nr * row_bytes, &full[s],
                         policy);
                ++prod;
            }
        }
        pdl_wait_primary();
        if (list_mode) {  // the gate launch's atomic appends are complete: chunks of NU list entries
            unsigned int n_app = 0;
            if (lane == 0) n_app = *reinterpret_cast<volatile unsigned int *>(sched + 3);
            sched_list_n = __shfl_sync(0xffffffffu, n_app, 0);
            ntl = (int)((sched_list_n + NU - 1) / NU);
        }
        if (lane == 0) claim_tile_async(t_res, sched, dyn_base + (unsigned)lazy_tail < (unsigned)ntl);
        prod = __shfl_sync(0xffffffffu, prod, 0);
        ps = prod % stages;
        gates_inflight = prod;
        // the rest of the ring fills as jobs retire (UD work first); with `eager` (small layers, and the
        // list kernel, which has no static GATE tiles to prime the ring) the free stages are filled now
        if (eager || list_mode) {
            while (!ended && prod < stages && issue_job()) {
            }
        }
        trace_stamp(trace, 0, 1);

        int rs = 0;                  // = retire % stages
        uint32_t rphase = 0;         // = (retire / stages) & 1
        while (!ended) {
            // ---- retire job `retire` in order ----
            const unsigned long long tw0 = trace ? gtimer() : 0ull;
            mbar_wait(&empty[rs], rphase);
            const unsigned long long tw1 = trace ? gtimer() : 0ull;
            p_wait += tw1 - tw0;
            if (desc[rs].type == kJobGate) {
                // u (fixed-order sum over the 16 consumer warps) -> v = SiLU(u) (Eq. 2) ->
                // keep = |v| >= t (Eq. 4, ties kept) -> ballot compaction of the tile
                const int tile = desc[rs].tile, n = desc[rs].n, r0 = tile * NR;
                const float *rb = red + (size_t)rs * NW * NPMAX;
                uint32_t bits = 0;
                float vrow[B];
#pragma unroll
                for (int tk = 0; tk < B; ++tk) {
                    float u = 0.f;
                    if (lane < n) {
#pragma unroll
                        for (int w = 0; w < NW; ++w) u += rb[w * NPMAX + lane * B + tk];
                    }
                    const float v = __fdividef(u, 1.0f + __expf(-u));
                    vrow[tk] = v;
                    const bool keep = dense || mode == kModeGateOnly || (fabsf(v) >= t);
                    bits |= (keep ? 1u : 0u) << tk;
                    if (acts && lane < n) acts[(size_t)tk * m + (size_t)(r0 + lane)] = v;
                }
                // (ablation mode: every row of the tile is queued -- the paper's Alg. 2 mask-predicated
                //  loads at tile granularity; inactive rows carry v = 0, so y is unchanged)
                const bool act = (lane < n) && bits != 0u;
                const uint32_t bal = __ballot_sync(0xffffffffu, act);
                const int rank = __popc(bal & ((1u << lane) - 1u));
                const int nact = __popc(bal);
                if (predicated && lane < n) {
                    // App. D Alg. 2 (no compaction): the tile's rows in two fixed halves, one UD job each
                    // whatever the mask; Mask predicates each row's load (negative id = not loaded, 0)
                    Desc &Q = queue[(q_tail + lane / NU) % QCAP];
                    const int i = lane % NU;
                    Q.id[i] = act ? r0 + lane : -1 - (r0 + lane);
#pragma unroll
                    for (int tk = 0; tk < B; ++tk) Q.v[i][tk] = ((bits >> tk) & 1u) ? vrow[tk] : 0.0f;
                    if (i == 0) {
                        Q.type = kJobUD;
                        Q.tile = tile;
                        Q.n = min(NU, n - lane);
                    }
                }
                if (act) {
                    const int pos = r0 + rank;
                    CATS_DCHECK(pos < m && rank < n);
                    idx[pos] = r0 + lane;
                    tokmask[pos] = (uint8_t)bits;
#pragma unroll
                    for (int tk = 0; tk < B; ++tk) vals[(size_t)pos * B + tk] = ((bits >> tk) & 1u) ? vrow[tk] : 0.0f;
                    if (atomic_gate) {  // App. D Alg. 1 line 4: append (j, v_j) to the global idcs
                        const unsigned int ap = atomicAdd(&sched[3], 1u);
                        CATS_DCHECK(ap < (unsigned)m);
                        gidx[ap] = r0 + lane;
#pragma unroll
                        for (int tk = 0; tk < B; ++tk) gval[(size_t)ap * B + tk] = ((bits >> tk) & 1u) ? vrow[tk] : 0.0f;
                    }
                    if (!gate_only && !predicated) {  // queue the tile's active neurons, NU per UD job, ascending
                        Desc &Q = queue[(q_tail + rank / NU) % QCAP];
                        const int i = rank % NU;
                        Q.id[i] = r0 + lane;
#pragma unroll
                        for (int tk = 0; tk < B; ++tk) Q.v[i][tk] = ((bits >> tk) & 1u) ? vrow[tk] : 0.0f;
                        if (i == 0) {
                            Q.type = kJobUD;
                            Q.tile = tile;
                            Q.n = min(NU, nact - rank);
                        }
                    }
                }
                if (lane == 0) cnt[tile] = nact;
                if (predicated) q_tail += (n + NU - 1) / NU;
                else if (!gate_only) q_tail += (nact + NU - 1) / NU;
                --gates_inflight;
                __syncwarp();
            }
            ++retire;
            if (++rs == stages) { rs = 0; rphase ^= 1u; }
            const unsigned long long tw2 = trace ? gtimer() : 0ull;
            // ---- refill every free stage (UD jobs first, else new GATE tiles, else END) ----
            while (!ended && prod < retire + stages && issue_job()) {
            }
            if (trace) {
                const unsigned long long tw3 = gtimer();
                p_busy += tw3 - tw1;
                p_issue += tw3 - tw2;
            }
        }
        if (lane == 0) {
            trace_put(trace, 2, 0, p_wait);
            trace_put(trace, 2, 1, p_busy);
            trace_put(trace, 2, 2, (unsigned long long)retire);
            trace_put(trace, 2, 6, p_issue);
            trace_put(trace, 2, 7, t_last_gate);
        }
    } else {
        // ===================================== CONSUMER WARPS ====================================
        pdl_wait_primary();     // x (and the accumulators) may come from the PDL predecessor
        // Two int64 accumulators, alternating per decode (parity in sched[4]): the previous decode's
        // converting CTA left the first sched[5] x d words of its buffer dirty; this call's CTAs zero
        // them here, a slice each, off the critical path (that conversion completed before
        // griddepcontrol.wait returned), so the last CTA of a call only reads its accumulator.
        const unsigned int par = *reinterpret_cast<volatile unsigned int *>(sched + 4) & 1u;
        const int dirty = min(ystride, (int)*reinterpret_cast<volatile unsigned int *>(sched + 5) * d);
        yacc += (size_t)par * ystride;
        {
            longlong2 *yo = reinterpret_cast<longlong2 *>(par ? yacc - ystride : yacc + ystride);
            for (int c = (int)blockIdx.x * NC + tid; c < dirty / 2; c += (int)gridDim.x * NC)
                yo[c] = make_longlong2(0, 0);
        }
        uint4 xr[B][CPT];  // x, own chunks, packed (bf16 pairs or fp32), 0 past the row end
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            const int ch = tid + k * NC;
#pragma unroll
            for (int tk = 0; tk < B; ++tk)
                xr[tk][k] = ch < nch ? *reinterpret_cast<const uint4 *>(x + (size_t)tk * d + (size_t)ch * VEC)
                                     : make_uint4(0u, 0u, 0u, 0u);
        }
        int yhi[B][CPT][VEC], ylo[B][CPT][VEC];  // exact fixed-point partial of y (units 2^-38), own chunks
#pragma unroll
        for (int tk = 0; tk < B; ++tk)
#pragma unroll
            for (int k = 0; k < CPT; ++k)
#pragma unroll
                for (int e = 0; e < VEC; ++e) yhi[tk][k][e] = ylo[tk][k][e] = 0;

        int s = 0;
        uint32_t phase = 0;
        unsigned long long c_wait = 0;
        int n_gate = 0, n_ud = 0;
        for (;;) {
            const unsigned long long cw0 = trace ? gtimer() : 0ull;
            mbar_wait(&full[s], phase);
            if (trace) c_wait += gtimer() - cw0;
            const int type = desc[s].type;
            if (type == kJobEnd) break;
            const int n = desc[s].n;
            const uint32_t sbase = smem_u32(ring + (size_t)s * stage_bytes);
            float *rb = red + (size_t)s * NW * NPMAX;

            if (type == kJobGate) {
                ++n_gate;
                // ---- u = x W_gate[:, j] partials for the tile's rows ----
                uint4 wr[NR][CPT];
#pragma unroll
                for (int r = 0; r < NR; ++r)
#pragma unroll
                    for (int k = 0; k < CPT; ++k) {
                        const int ch = tid + k * NC;
                        wr[r][k] = (r < n && ch < nch) ? lds128(sbase + (uint32_t)r * row_bytes + (uint32_t)ch * 16u)
                                                       : make_uint4(0u, 0u, 0u, 0u);
                    }
                float part[NR][B];
#pragma unroll
                for (int r = 0; r < NR; ++r) {
#pragma unroll
                    for (int tk = 0; tk < B; ++tk) part[r][tk] = 0.f;
#pragma unroll
                    for (int k = 0; k < CPT; ++k)
#pragma unroll
                        for (int tk = 0; tk < B; ++tk) part[r][tk] = dot16<T>(wr[r][k], xr[tk][k], part[r][tk]);
                }
#pragma unroll
                for (int r = 0; r < NR; ++r)
#pragma unroll
                    for (int tk = 0; tk < B; ++tk) {
                        const float v = warp_allreduce_sum(part[r][tk]);
                        if (lane == 0) rb[warp * NPMAX + r * B + tk] = v;
                    }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);  // stage read + partials written -> producer
            } else {  // kJobUD
                ++n_ud;
                float vj[NU][B];  // descriptor -> registers before releasing the stage
                bool live[NU];    // row loaded (false: predicated off by Mask in Alg. 2 mode -> zeros)
#pragma unroll
                for (int i = 0; i < NU; ++i) {
                    live[i] = i < n && (!ABL || mode != kModePredicated || desc[s].id[i] >= 0);
#pragma unroll
                    for (int tk = 0; tk < B; ++tk) vj[i][tk] = desc[s].v[i][tk];
                }
                uint4 wu[NU][CPT], wd[NU][CPT];
#pragma unroll
                for (int i = 0; i < NU; ++i)
#pragma unroll
                    for (int k = 0; k < CPT; ++k) {
                        const int ch = tid + k * NC;
                        const bool ok = live[i] && ch < nch;
                        wu[i][k] = ok ? lds128(sbase + (uint32_t)(2 * i) * row_bytes + (uint32_t)ch * 16u)
                                      : make_uint4(0u, 0u, 0u, 0u);
                        wd[i][k] = ok ? lds128(sbase + (uint32_t)(2 * i + 1) * row_bytes + (uint32_t)ch * 16u)
                                      : make_uint4(0u, 0u, 0u, 0u);
                    }
                // ---- up: partial dots x . W_up[j] ----
                float part[NU][B];
#pragma unroll
                for (int i = 0; i < NU; ++i) {
#pragma unroll
                    for (int tk = 0; tk < B; ++tk) part[i][tk] = 0.f;
#pragma unroll
                    for (int k = 0; k < CPT; ++k)
#pragma unroll
                        for (int tk = 0; tk < B; ++tk) part[i][tk] = dot16<T>(wu[i][k], xr[tk][k], part[i][tk]);
                }
#pragma unroll
                for (int i = 0; i < NU; ++i)
#pragma unroll
                    for (int tk = 0; tk < B; ++tk) {
                        const float v = warp_allreduce_sum(part[i][tk]);
                        if (lane == 0) rb[warp * NPMAX + i * B + tk] = v;
                    }
                consumer_barrier<NC>();  // all 16 warps' partials are in red[s]
                // ---- cross-warp sums (fixed tree, identical in every warp): lane l reads warp
                //      (l % NW)'s partial of pair c*PPR + l/NW; an xor butterfly over NW lanes sums them.
                constexpr int PPR = 32 / NW;
                float a[NPU];
#pragma unroll
                for (int c = 0; c < (NPU + PPR - 1) / PPR; ++c) {
                    const int pp = c * PPR + lane / NW;
                    float v = (pp < NPU) ? rb[(lane % NW) * NPMAX + pp] : 0.f;
#pragma unroll
                    for (int o = NW / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
#pragma unroll
                    for (int q = 0; q < PPR; ++q)
                        if (c * PPR + q < NPU) a[c * PPR + q] = __shfl_sync(0xffffffffu, v, q * NW);
                }
                // stage data, descriptor and red[s] are no longer needed: release the stage
                if (lane == 0) mbar_arrive(&empty[s]);
                // x1_j = (x W_up[j]) * v_j  (Optimization 1), pre-scaled by 2^8 for the fixed-point split
                // (a power of two: the fp32 products and sums below are exactly 2^8 times unscaled ones)
                float x1[NU][B];
#pragma unroll
                for (int i = 0; i < NU; ++i)
#pragma unroll
                    for (int tk = 0; tk < B; ++tk) x1[i][tk] = (i < n) ? (a[i * B + tk] * vj[i][tk]) * kFixPre : 0.f;
                // ---- down: y_job[c] = sum_i x1_i W_down[i][c] (fp32, fixed order) -> fixed point ----
#pragma unroll
                for (int k = 0; k < CPT; ++k) {
                    float wf[NU][VEC];
#pragma unroll
                    for (int i = 0; i < NU; ++i) unpack16(wd[i][k], wf[i]);
#pragma unroll
                    for (int tk = 0; tk < B; ++tk)
#pragma unroll
                        for (int e = 0; e < VEC; ++e) {
                            float yj = 0.f;
#pragma unroll
                            for (int i = 0; i < NU; ++i) yj = fmaf(x1[i][tk], wf[i][e], yj);
                            fix_acc(yhi[tk][k][e], ylo[tk][k][e], yj);
                        }
                }
            }
            if (++s == stages) { s = 0; phase ^= 1u; }
        }
        trace_stamp(trace, 0, 2);
        if (tid == 0) {
            trace_put(trace, 2, 3, c_wait);
            trace_put(trace, 2, 4, (unsigned long long)n_gate);
            trace_put(trace, 2, 5, (unsigned long long)n_ud);
        }

        // ---- split-K reduction through the TMA bulk-reduce engine ----
        // The CTA's exact int64 partial is staged in shared memory (the ring is idle after END)
        // and added into the global accumulator yacc[b][d] with cp.reduce.async.bulk .add.u64
        // (integer adds performed at L2, any order -> deterministic). The last CTA to finish converts
        // yacc to fp32 once, writes y, flips the accumulator parity and re-arms the tile scheduler.
        __shared__ unsigned int s_last;
        if (has_y) {
            consumer_barrier<NC>();  // every consumer warp is past its last job: the ring is idle
            trace_stamp(trace, 0, 5);
            unsigned long long *sbuf = reinterpret_cast<unsigned long long *>(ring);
            const int tpc = min(B, (int)(((size_t)stages * stage_bytes) / ((size_t)d * 8)));  // tokens per chunk
            for (int t0 = 0; t0 < B; t0 += tpc) {
                const int tn = min(tpc, B - t0);
#pragma unroll
                for (int tk = 0; tk < B; ++tk) {
                    if (tk < t0 || tk >= t0 + tn) continue;
#pragma unroll
                    for (int k = 0; k < CPT; ++k) {
                        const int ch = tid + k * NC;
                        if (ch < nch) {
                            ulonglong2 *dst =
                                reinterpret_cast<ulonglong2 *>(sbuf + (size_t)(tk - t0) * d + (size_t)ch * VEC);
                            ulonglong2 qv[VEC / 2];
#pragma unroll
                            for (int q = 0; q < VEC / 2; ++q)
                                qv[q] = make_ulonglong2(
                                    (unsigned long long)fix_value(yhi[tk][k][2 * q], ylo[tk][k][2 * q]),
                                    (unsigned long long)fix_value(yhi[tk][k][2 * q + 1], ylo[tk][k][2 * q + 1]));
                            // a thread's 16-byte pieces in lane-rotated order: the 32 lanes' stores of one
                            // instruction then spread over all banks (4 wavefronts instead of 16 at VEC = 8)
#pragma unroll
                            for (int q2 = 0; q2 < VEC / 2; ++q2) {
                                const int q = (q2 + lane) & (VEC / 2 - 1);
                                ulonglong2 v = qv[0];
#pragma unroll
                                for (int j = 1; j < VEC / 2; ++j) v = q == j ? qv[j] : v;
                                dst[q] = v;
                            }
                        }
                    }
                }
                fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the bulk engine
                consumer_barrier<NC>();
                if (tid == 0) {
                    trace_stamp(trace, 0, 6);
                    bulk_reduce_add_u64(yacc + (size_t)t0 * d, sbuf, (uint32_t)((size_t)tn * d * 8));
                    bulk_commit_and_wait_all();
                    trace_stamp(trace, 0, 7);
                }
                consumer_barrier<NC>();  // sbuf reusable
            }
            if (tid == 0) {
                fence_proxy_async_global();
                __threadfence();
            }
        }
        consumer_barrier<NC>();
        trace_stamp(trace, 0, 4);  // partial reduced into yacc
        if (tid == 0) s_last = (atomicAdd(&sched[1], 1u) == gridDim.x - 1) ? 1u : 0u;
        consumer_barrier<NC>();
        if (s_last) {
            __threadfence();
            if (has_y) {
                // 8 independent L2 loads in flight per thread (the accumulator was just written by
                // the bulk-reduce engine of every SM; a serial loop would pay one L2 trip per step)
                const int n2 = B * d / 2;
                for (int c0 = 0; c0 < n2; c0 += 8 * NC) {
                    longlong2 v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int c = c0 + u * NC + tid;
                        v[u] = c < n2 ? __ldcg(reinterpret_cast<const longlong2 *>(yacc) + c) : make_longlong2(0, 0);
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int c = c0 + u * NC + tid;
                        if (c < n2) {
                            reinterpret_cast<float2 *>(y)[c] = make_float2(fix_to_float(v[u].x), fix_to_float(v[u].y));
                        }
                    }
                }
            }
            if (tid == 0) {
                sched[0] = 0u;
                sched[1] = 0u;
                if (list_mode) sched[3] = 0u;  // the idcs list was consumed: re-arm the append counter
                if (has_y) {
                    sched[4] = par ^ 1u;     // the next decode accumulates into the other (zeroed) buffer
                    sched[5] = (unsigned)B;  // ... and zeroes these B x d words of this one
                }
            }
        }
        trace_stamp(trace, 0, 3);
    }
}

size_t k12_smem_bytes(const PlanData &p, int b, int stages) {
    const int nr = k12_rows_per_tile(p, b);
    const int nu = nr / 2;
    size_t s = (size_t)stages * nr * (size_t)p.d * p.esize;  // ring
    s += (size_t)stages * 16;                                // full + empty mbarriers
    const size_t desc = (size_t)(3 + nu) * 4 + (size_t)nu * b * 4;
    s += (size_t)(stages + 64) * desc;                       // stage descriptors + UD queue
    s = (s + 15) & ~(size_t)15;
    s += (size_t)stages * k12_consumer_warps_c(b) * std::max(nr, nu) * b * 4;  // per-stage warp partials
    return (s + 127) & ~(size_t)127;
}

template <typename T, int B, int NR, int CPT, bool ABL>
static cudaError_t launch_k12_t(const PlanData &p, const void *x, const void *Wg, const void *Wu, const void *Wd,
                                float t, int mode, float *acts, float *y, void *ws, cudaStream_t s) {
    auto kern = k12_cats_mlp<T, B, NR, CPT, ABL>;
    const int stages = p.k12_max_stages > 0 ? std::min(p.k12_max_stages, k12_stages(p, B)) : k12_stages(p, B);
    const size_t smem = k12_smem_bytes(p, B, stages);
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void *>(kern), smem);
    if (e != cudaSuccess) return e;
    char *w = static_cast<char *>(ws);
    // Programmatic dependent launch: the CTAs of this decode may become resident while the previous
    // kernel on the stream drains, and start streaming their static W_gate tiles (see the kernel).
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)k12_grid(p, B));
    cfg.blockDim = dim3((unsigned)k12_threads_c(B));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(
        &cfg, kern, static_cast<const T *>(x), static_cast<const T *>(Wg), static_cast<const T *>(Wu),
        static_cast<const T *>(Wd), p.d, p.m, stages, t, mode, reinterpret_cast<int32_t *>(w + p.off_idx),
        reinterpret_cast<uint8_t *>(w + p.off_tokmask), reinterpret_cast<float *>(w + p.off_vals),
        reinterpret_cast<int32_t *>(w + p.off_cnt), acts, reinterpret_cast<unsigned long long *>(w + p.off_ypart), y,
        reinterpret_cast<unsigned int *>(w + p.off_sched), reinterpret_cast<int32_t *>(w + p.off_gidx),
        reinterpret_cast<float *>(w + p.off_gval), p.max_batch * p.d, p.lazy_tail * k12_grid(p, B),
        p.k12_eager, p.k12_l2pf,
        p.trace ? reinterpret_cast<unsigned long long *>(w + p.off_trace) : nullptr);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <typename T, int B, int NR, bool ABL>
static cudaError_t launch_k12_a(const PlanData &p, const void *x, const void *Wg, const void *Wu, const void *Wd,
                                float t, int mode, float *acts, float *y, void *ws, cudaStream_t s) {
    switch (k12_cpt(p, B)) {
        case 1: return launch_k12_t<T, B, NR, 1, ABL>(p, x, Wg, Wu, Wd, t, mode, acts, y, ws, s);
        case 2: return launch_k12_t<T, B, NR, 2, ABL>(p, x, Wg, Wu, Wd, t, mode, acts, y, ws, s);
        case 3:
            return B == 1 ? launch_k12_t<T, B, NR, (B == 1 ? 3 : 2), ABL>(p, x, Wg, Wu, Wd, t, mode, acts, y, ws, s)
                          : cudaErrorInvalidValue;
        case 4:
            return B == 1 ? launch_k12_t<T, B, NR, (B == 1 ? 4 : 2), ABL>(p, x, Wg, Wu, Wd, t, mode, acts, y, ws, s)
                          : cudaErrorInvalidValue;
        default: return cudaErrorInvalidValue;
    }
}

template <typename T, int B, int NR>
static cudaError_t launch_k12_r(const PlanData &p, const void *x, const void *Wg, const void *Wu, const void *Wd,
                                float t, int mode, float *acts, float *y, void *ws, cudaStream_t s) {
    const bool abl = mode == kModePredicated || mode == kModeAtomicGate || mode == kModeAtomicList;
    return abl ? launch_k12_a<T, B, NR, true>(p, x, Wg, Wu, Wd, t, mode, acts, y, ws, s)
               : launch_k12_a<T, B, NR, false>(p, x, Wg, Wu, Wd, t, mode, acts, y, ws, s);
}

template <typename T, int B>
static cudaError_t launch_k12_b(const PlanData &p, const void *x, const void *Wg, const void *Wu, const void *Wd,
                                float t, int mode, float *acts, float *y, void *ws, cudaStream_t s) {
    switch (k12_rows_per_tile(p, B)) {
        case 4: return launch_k12_r<T, B, 4>(p, x, Wg, Wu, Wd, t, mode, acts, y, ws, s);
        case 2: return launch_k12_r<T, B, 2>(p, x, Wg, Wu, Wd, t, mode, acts, y, ws, s);
        case 6:
            if constexpr (B == 1) return launch_k12_r<T, B, 6>(p, x, Wg, Wu, Wd, t, mode, acts, y, ws, s);
            return cudaErrorInvalidValue;
        default: return cudaErrorInvalidValue;
    }
}

template <typename T>
static cudaError_t launch_k12_dt(const PlanData &p, const void *x, int b, const void *Wg, const void *Wu,
                                 const void *Wd, float t, int mode, float *acts, float *y, void *ws, cudaStream_t s) {
    switch (b) {
        case 1: return launch_k12_b<T, 1>(p, x, Wg, Wu, Wd, t, mode, acts, y, ws, s);
        case 2: return launch_k12_b<T, 2>(p, x, Wg, Wu, Wd, t, mode, acts, y, ws, s);
        case 3: return launch_k12_b<T, 3>(p, x, Wg, Wu, Wd, t, mode, acts, y, ws, s);
        case 4: return launch_k12_b<T, 4>(p, x, Wg, Wu, Wd, t, mode, acts, y, ws, s);
        case 5: return launch_k12_b<T, 5>(p, x, Wg, Wu, Wd, t, mode, acts, y, ws, s);
        case 6: return launch_k12_b<T, 6>(p, x, Wg, Wu, Wd, t, mode, acts, y, ws, s);
        case 7: return launch_k12_b<T, 7>(p, x, Wg, Wu, Wd, t, mode, acts, y, ws, s);
        case 8: return launch_k12_b<T, 8>(p, x, Wg, Wu, Wd, t, mode, acts, y, ws, s);
        default: return cudaErrorInvalidValue;
    }
}

// cats_mlp_decode_host with a mapped (pinned) x: x crosses PCIe in a small kernel instead of a copy-engine
// transfer, so the decode kernel that follows can use programmatic dependent launch -- its CTAs become
// resident and stream their static W_gate tiles while x is in flight (they read x after
// griddepcontrol.wait, which also orders this kernel's stores before their loads).
__global__ void x_stage_kernel(const uint4 *__restrict__ src, uint4 *__restrict__ dst, int n16) {
    pdl_launch_dependents();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x) dst[i] = src[i];
}

cudaError_t launch_x_stage(const void *x_mapped, void *xd, size_t bytes, cudaStream_t s) {
    const int n16 = (int)(bytes / 16);
    const int grid = std::max(1, std::min(64, (n16 + 255) / 256));
    x_stage_kernel<<<grid, 256, 0, s>>>(static_cast<const uint4 *>(x_mapped), static_cast<uint4 *>(xd), n16);
    return cudaGetLastError();
}

cudaError_t launch_k12(const PlanData &p, const void *x, int b, const void *Wg, const void *Wu, const void *Wd,
                       float t, int mode, float *acts, float *y, void *ws, cudaStream_t s) {
    if (p.dt == CATS_BF16) return launch_k12_dt<bf16_bits>(p, x, b, Wg, Wu, Wd, t, mode, acts, y, ws, s);
    return launch_k12_dt<float>(p, x, b, Wg, Wu, Wd, t, mode, acts, y, ws, s);
}

}  // namespace cats
