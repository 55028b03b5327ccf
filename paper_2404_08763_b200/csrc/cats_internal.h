// cats_internal.h -- host-side plumbing shared by the libcats translation units (not exported).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <algorithm>

#include "../../include/cats.h"

namespace cats {

// K12 CTA shapes: b = 1 runs two CTAs per SM with 8 consumer warps each (two independent job streams
// hide per-job latency); b >= 2 runs one CTA per SM with 16 consumer warps (half the columns per
// thread, so x and the fixed-point y partials of every token fit in registers).
constexpr int k12_consumer_warps_c(int b) { return b == 1 ? 8 : 16; }
constexpr int k12_ctas_per_sm_c(int b) { return b == 1 ? 2 : 1; }
constexpr int k12_threads_c(int b) { return k12_consumer_warps_c(b) * 32 + 32; }  // + 1 producer warp
constexpr size_t k12_smem_budget_c(int b) { return b == 1 ? 112 * 1024 : 224 * 1024; }
constexpr size_t kSmemBudget = 224 * 1024;  // dynamic shared memory per CTA, one CTA per SM
constexpr int kMaxCPT = 4;            // 16-byte chunks of a row owned per consumer (d <= 8192 bf16)
constexpr int kMaxStages = 8;

// K12 launch modes
constexpr int kModeCats = 0;          // CATS_t decode
constexpr int kModeDense = 1;         // every neuron active (the library's dense MLP)
constexpr int kModeGateOnly = 2;      // SiLU(x W_gate) only (calibration data collection)
constexpr int kModePredicated = 3;    // App. D Alg. 2 (CATS_COMPACT_PREDICATED): no compaction, UD jobs = fixed
                                      // tile halves, Mask predicates the row loads (inactive rows read as 0)
constexpr int kModeAtomicGate = 4;    // App. D Alg. 1 (CATS_COMPACT_ATOMIC), launch 1: gate + SiLU + Mask +
                                      // atomic appends of (id, v) to the global idcs list
constexpr int kModeAtomicList = 5;    // App. D Alg. 1, launch 2: up / down over the idcs list (no GATE jobs)

struct PlanData {
    int d, m, max_batch;
    cats_dtype_t dt;
    int device, num_sms;
    int esize;          // bytes per element
    int vec;            // elements per 16 bytes
    int nchunks;        // d * esize / 16
    int g1;             // max K12 CTAs over batch sizes (sizes the partial buffer)
    // workspace layout (byte offsets)
    size_t off_sched, off_idx, off_tokmask, off_vals, off_cnt, off_ypart, off_xstage, off_ystage, ws_bytes;
    bool trace;         // options.trace: kernels stamp %globaltimer into the workspace
    int lazy_tail;      // K12 stops reserving tile ids for the last lazy_tail * grid tiles (options.lazy_tail)
    int split_min_b;    // batches b >= split_min_b run the split path KA + KB (9 = never: options.path FUSED)
    int k12_max_stages; // 0 = as many K12 stages as fit (options.max_stages caps it)
    int k12_min_tiles;  // K12 grid <= ntiles / k12_min_tiles (options.min_tiles)
    int k12_eager;      // K12 fills every stage with claimed tiles at start (options.eager)
    int k12_l2pf;       // K12 static tiles per CTA prefetched into L2 at start (options.l2_prefetch)
    int nr_force;       // 0 = automatic tile height; 2 / 4 / 6 forces it (options.rows_per_tile)
    int compaction;     // cats_compaction_t (options.compaction)
    int kind;           // 0 = gated-MLP plan, 1 = App. B input-sparse projection plan (d = d_out, m = d_in)
    struct XsCfg {            // kind 1 (xsparse.cu), per batch size b = 1..8:
        int cols, q, r;       //   columns per CTA, column parts, cluster size (ranges of the kept list)
        int clusters;         //   clusters resident at once (-1: planned without a device)
    } xs[9];
    bool xs_no_mma;           // options.xs_mma = 0: XS keeps the FFMA2 path at every batch (experiments)
    size_t off_x1, off_part;  // split path: x1 per compact position [m][max_b]; KB partials [R][max_b][d]
    size_t off_tmask;         // split path: per-tile active-row mask words (KA -> KB), zero between calls
    size_t off_trace, trace_bytes;
    size_t off_gidx, off_gval;  // App. D Alg. 1 mode: the global idcs list (ids, v per token), arbitrary order
};

int split_ka_stages_nr(const PlanData &p, int b, int nr);  // mlp_split.cu

// K12 tile height NR (W_gate rows per GATE job; a UD job carries NR/2 neurons = the same bytes).
// The split path (KA, KB) shares the tile geometry at b >= 2.
inline int k12_rows_per_tile(const PlanData &p, int b) {
    if (p.nr_force == 2 || p.nr_force == 4 || (p.nr_force == 6 && b == 1)) return p.nr_force;  // options
    // b >= 2: 2-row tiles where x [b][d] staged in KA's shared memory leaves < 2 stages of 4-row tiles per
    // job stream (Llama2-13B d = 5120 from b = 6) -- otherwise the planner would fall back to K12, whose
    // x and y partials do not fit in registers there (measured 3.5 ms per step at b = 8)
    if (b >= 2 && split_ka_stages_nr(p, b, 4) < 2) return 2;
    // 4-row tiles whenever two 4-row stages fit (measured at d = 5120, b = 1: 4 rows x 2 stages beats
    // 2 rows x 5 stages, 55.6 vs 60.6 us; per-job costs are per row pair)
    const size_t row = (size_t)p.d * p.esize;
    // b = 1 on large layers: 6-row tiles (two 48 KB stages at d = 4096; fewer, larger jobs: Mistral-7B
    // 42.6 -> 41.9 us); small layers keep 4 rows (more tiles to balance)
    if (b == 1 && p.m >= 8192 && 6 * row * 2 <= k12_smem_budget_c(b) - 8 * 1024) return 6;
    return 4 * row * 2 <= k12_smem_budget_c(b) - 8 * 1024 ? 4 : 2;
}
inline int k12_ntiles(const PlanData &p, int b) { return (p.m + k12_rows_per_tile(p, b) - 1) / k12_rows_per_tile(p, b); }
inline int k12_cpt(const PlanData &p, int b) {
    const int nc = k12_consumer_warps_c(b) * 32;
    return (p.nchunks + nc - 1) / nc;
}
inline int k12_grid(const PlanData &p, int b) {  // >= k12_min_tiles tiles per CTA on small layers
    const int mt = std::max(1, p.k12_min_tiles);
    return std::max(1, std::min(p.num_sms * k12_ctas_per_sm_c(b), (k12_ntiles(p, b) + mt - 1) / mt));
}
size_t k12_smem_bytes(const PlanData &p, int b, int stages);
inline int k12_stages(const PlanData &p, int b) {
    const size_t stage = (size_t)k12_rows_per_tile(p, b) * p.d * p.esize;
    const size_t extra = k12_smem_bytes(p, b, 0) + kMaxStages * 256;
    if (extra >= k12_smem_budget_c(b)) return 0;
    return (int)std::min<size_t>((k12_smem_budget_c(b) - extra) / stage, kMaxStages);
}

// ---- split path for b >= 2 (mlp_split.cu): KA = gate + up (dynamic tiles), KB = down (static balanced
// ranges of the compact active list x column parts, fixed-order two-phase reduction) ----
constexpr int kSplitAWarps = 16;                         // KA consumer warps (both groups)
constexpr int kSplitAGroups = 2;                         // KA job streams per CTA (one producer warp each)
constexpr int kSplitAThreads = (kSplitAWarps + kSplitAGroups) * 32;
constexpr int kSplitBMaxThreads = 672;                   // KB: <= 20 consumer warps + 1 producer warp
constexpr int kSplitFifo = 64;                           // KA active-neuron FIFO (power of two)
constexpr int kSplitFifoCs = 128;                        // the same with 8-row tiles (ka_colsplit)
constexpr int kKbReducers = 64;                          // KB: the last K CTAs to finish sum the partials

template <int NR, int B>
struct SplitDesc {   // one KA ring stage: GATE(tile) or UP(<= NR active neurons), column part `part`
    int type, tile, n, part;
    int id[NR];      // UP: neuron ids
    int pos[NR];     // UP: compact positions (tile * NR + rank)
    float v[NR][B];  // UP: v = SiLU(u), 0 for tokens where |v| < t
};
template <int B>
struct SplitFifoEntry {  // one active neuron waiting for its UP job
    int id, pos;
    float v[B];
};

// KB on tensor cores (bf16, d a multiple of 1024: 4 column parts of 16-column tiles over 16 warps)
// KB's tensor-core path from b = 2 (A/B: Llama2-13B b = 2 62.1 vs 64.3 us, its TP4 shard 25.4 vs 26.6,
// Llama2-7B 44.7 vs 44.9, Mistral 53.1 vs 53.3), KA's from b = 3 (below)
constexpr int kSplitKbMmaMinB = 2;
constexpr int kSplitMmaMinB = 3;  // batches from which KA / KB use warp-level bf16 MMA (measured crossover, DESIGN 5.2)
// KA's tensor-core path in column parts (bf16, b >= kSplitMmaMinB, d a multiple of kKaPartCols): tiles of
// 8 rows -- all 8 columns of the m16n8k16 B operand distinct rows -- and every GATE / UP job streamed as
// d / kKaPartCols consecutive ring stages of 8 rows x kKaPartCols columns, the consumers accumulating in
// registers across the parts: x [b][d] is read (ldmatrix) once per 8 rows instead of once per NR.
// Taken where full-row jobs would shrink to 2-row tiles (x leaves room for fewer than 2 stages of 4 rows
// per job stream: d = 5120 from b = 6). Measured (A/B, one box): Llama2-13B b = 8 89.6 vs 112.9 us, the
// TP8 shard at b = 8 25.8 vs 27.2; but at d = 4096 (4-row full-row jobs fit) 70.3 vs 59.4 us at b = 8:
// next to x, the 8-row partial buffers and the larger FIFO only 3 stages of 16.5 KB fit per stream
// (ncu: shared-memory wavefronts 54 -> 25 % of peak, but DRAM 4.1 -> 3.4 TB/s, consumers waiting on data).
constexpr int kKaPartCols = 1024;
// KA keeps x in tensor memory on its tensor-core path where each warp's k-steps come in whole 8-step
// TMEM loads (d % 1024 == 0) -- then x takes no shared memory (split_ka_stages_nr, split_ka_smem)
inline bool ka_x_in_tmem(const PlanData &p, int b) {
    return p.esize == 2 && b >= kSplitMmaMinB && p.d % 1024 == 0 && p.d <= 8192;
}
inline bool ka_colsplit(const PlanData &p, int b) {
    return p.esize == 2 && b >= kSplitMmaMinB && p.d % kKaPartCols == 0 && split_ka_stages_nr(p, b, 4) < 2;
}
// tile height of the split path (KA's tiles, KB's per-tile masks)
// 6-row tiles on the x-in-TMEM path (6 of the 8 B-operand columns distinct, a third fewer jobs than 4-row
// tiles) where two such stages fit per job stream; on the CUDA-core path (b = 2, 3) of large bf16 layers
// likewise (K12's b = 1 shape: fewer, larger jobs where the per-job chain bounds the rate)
inline bool ka_nr6(const PlanData &p, int b) {
    if (p.nr_force != 0 || ka_colsplit(p, b)) return false;
    if (ka_x_in_tmem(p, b)) return split_ka_stages_nr(p, b, 6) >= 2;
    return p.esize == 2 && b >= 2 && b < kSplitMmaMinB && p.m >= 8192 && split_ka_stages_nr(p, b, 6) >= 2;
}
inline int split_rows_per_tile(const PlanData &p, int b) {
    return ka_colsplit(p, b) ? 8 : ka_nr6(p, b) ? 6 : k12_rows_per_tile(p, b);
}
inline int split_ntiles(const PlanData &p, int b) {
    return (p.m + split_rows_per_tile(p, b) - 1) / split_rows_per_tile(p, b);
}
inline bool split_kb_mma(const PlanData &p, int b) {  // instantiated for 1, 4, 5 tiles per warp
    return b >= kSplitKbMmaMinB && p.esize == 2 && (p.d == 1024 || p.d == 4096 || p.d == 5120);
}
// scheduler words at the workspace base: [0..1] tile counter / CTA exits, [2] KB arrival tickets,
// [3] App. D Alg. 1 append counter, [4] K12 accumulator parity, [5] tokens the last K12 call left in the
// other accumulator, [8 + q] KB range tickets of column part q (q < 16)
constexpr size_t kSchedBytes = 128;
inline int split_q(const PlanData &p, int b) {  // KB column parts (<= 16)
    if (split_kb_mma(p, b)) return 4;
    for (int q = 2; q <= 16; ++q)  // CUDA-core path: <= 640 consumer threads of 4 columns each
        if (p.d % (4 * q) == 0 && ((size_t)(p.d / q) * p.esize) % 16 == 0 && p.d / q / 4 <= 640) return q;
    return 2;
}
inline int split_ept(const PlanData &, int) { return 4; }  // KB (FFMA path) columns per thread
inline int split_part_cols(const PlanData &p, int b) { return p.d / split_q(p, b); }
inline int split_kb_mt(const PlanData &p, int b) {  // 16-column MMA tiles per KB warp (0 = FFMA path)
    return split_kb_mma(p, b) ? split_part_cols(p, b) / (16 * 16) : 0;
}
inline int split_kb_consumers(const PlanData &p, int b) {
    if (split_kb_mma(p, b)) return 16 * 32;
    const int c = (split_part_cols(p, b) + split_ept(p, b) - 1) / split_ept(p, b);
    return (c + 31) / 32 * 32;
}
inline int split_ranges(const PlanData &p, int b) {  // R: static ranges of the active list
    return std::max(1, std::min(p.num_sms / split_q(p, b), p.m / 8));
}
inline int split_kb_grid(const PlanData &p, int b) { return split_ranges(p, b) * split_q(p, b); }
inline int split_ka_grid(const PlanData &p, int b) {
    return std::max(1, std::min(p.num_sms, (split_ntiles(p, b) + kSplitAGroups - 1) / kSplitAGroups));
}
int split_ka_ks(const PlanData &p, int b);
size_t split_ka_smem(const PlanData &p, int b, int stages);
size_t split_kb_smem(const PlanData &p, int b, int stages);
int split_ka_stages(const PlanData &p, int b);
int split_kb_stages(const PlanData &p, int b);
bool split_supported(const PlanData &p, int b);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel / size (thread-safe)
cudaError_t ensure_smem_attr(const void *func, size_t smem);

// launchers: return cudaError_t of the launch
// K12 = the whole decode (gate ... down projection and the split-K reduction; y written by the last CTA)
cudaError_t launch_x_stage(const void *x_mapped, void *xd, size_t bytes, cudaStream_t s);  // mlp_fused.cu
cudaError_t launch_k12(const PlanData &p, const void *x, int b, const void *Wg, const void *Wu, const void *Wd,
                       float t, int mode, float *acts, float *y, void *ws, cudaStream_t s);

// split path (b >= 2): KA then KB, both PDL launches; ev (optional) = event recorded between them
cudaError_t launch_split(const PlanData &p, const void *x, int b, const void *Wg, const void *Wu, const void *Wd,
                         float t, int mode, float *y, void *ws, cudaStream_t s, cudaEvent_t ev_mid);

// KB alone for batch b (1..8), and the App. B input-sparse projection (KX then KB)
// ---- App. B input-sparse projection (xsparse.cu): one kernel XS, clusters of xs[b].r CTAs ----
constexpr int kXsThreads = 256;
// W rows in flight per thread: as many as the registers left by the b x 8 accumulators allow (each
// thread's rows are a latency chain of ceil(rows / unroll) HBM round trips)
__host__ __device__ constexpr int xs_unroll(int b) { return b <= 2 ? 16 : b <= 4 ? 12 : 8; }
constexpr size_t kXsSmemBudget = 113 * 1024;  // two CTAs per SM (228 KB less 1 KB reserved per CTA)
inline int xs_maxr(const PlanData &p, int b) { return (p.m + p.xs[b].r - 1) / p.xs[b].r; }  // longest kept range
// XS uses bf16 MMA from b = 2 whenever its column slab is 64 or 128 wide; from b = 4 the slab width is
// restricted to those (measured: b = 2 4096 -> 6144 13.8 -> 13.0 us, 4096 -> 4096 14.3 -> 11.1; forcing
// 128 columns at 4096 -> 12288 b = 2 cost 20.5 -> 23.5, so below b = 4 the width stays free)
constexpr int kXsMmaMinB = 2;
constexpr int kXsMmaForceB = 4;
int xs_mt(const PlanData &p, int b);
size_t xs_smem_bytes(const PlanData &p, int b);
int xs_active_clusters(const PlanData &p, int b);  // occupancy query (-1 without a device)
cudaError_t launch_xsparse(const PlanData &p, const void *x, int b, const void *W, float t, float *y, void *ws,
                           cudaStream_t s);
bool kb_supported(const PlanData &p, int b);

cudaError_t launch_calib_hist(const void *acts, uint64_t n, cats_dtype_t dt, const cats_calib_window_t &w,
                              uint64_t *hist, uint64_t *counts, cudaStream_t s);

void set_last_cuda_error(cudaError_t e);

}  // namespace cats
