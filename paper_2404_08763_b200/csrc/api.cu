// api.cu -- the exported C ABI of libcats (declared in include/cats.h): validation, planning,
// workspace layout, launch sequencing and the host side of the calibration radix select.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "cats_device.cuh"
#include "cats_internal.h"

using namespace cats;

struct cats_mlp_plan {
    PlanData p;
};

namespace cats {
static thread_local std::string g_last_cuda_error;
void set_last_cuda_error(cudaError_t e) {
    g_last_cuda_error = std::string(cudaGetErrorName(e)) + ": " + cudaGetErrorString(e);
}
}  // namespace cats

namespace {

constexpr uint32_t kKeyMaxBF16 = 0x7f7fu;       // largest finite |bf16| key
constexpr uint32_t kKeyMaxF32 = 0x7f7fffffu;    // largest finite |fp32| key
constexpr uint32_t kFullPassBins = 4096;        // shared-memory bins of a full-data pass
constexpr size_t kCalibHistOff = 0;
constexpr size_t kCalibCountOff = (size_t)CATS_CALIB_MAX_BINS * 8;
constexpr size_t kCalibWsBytes = kCalibCountOff + CATS_CALIB_COUNTS_LEN * 8;

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

inline cats_status_t cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return CATS_OK;
    set_last_cuda_error(e);
    return CATS_E_CUDA;
}

#define CATS_TRY(...)                                                    \
    try {                                                                \
        __VA_ARGS__                                                      \
    } catch (const std::bad_alloc &) {                                   \
        g_last_cuda_error = "host allocation failed";                    \
        return CATS_E_CUDA;                                              \
    } catch (...) {                                                      \
        g_last_cuda_error = "unexpected host exception";                 \
        return CATS_E_CUDA;                                              \
    }

uint32_t key_max(cats_dtype_t dt) { return dt == CATS_BF16 ? kKeyMaxBF16 : kKeyMaxF32; }

void make_window(uint32_t lo, uint32_t hi, uint32_t maxbins, cats_calib_window_t *w) {
    uint32_t shift = 0;
    while (((hi - lo) >> shift) + 1u > maxbins) ++shift;
    w->lo = lo;
    w->hi = hi;
    w->shift = shift;
    w->nbins = ((hi - lo) >> shift) + 1u;
    w->sample_stride = 0;
}

// exact ceil(k * n) on the IEEE-754 bits of k (0 <= k < 1): k = M * 2^-(1075 - E)
uint64_t exact_rank(double k, uint64_t n) {
    uint64_t bits;
    std::memcpy(&bits, &k, sizeof bits);
    const uint64_t E = (bits >> 52) & 0x7ffu;
    const uint64_t frac = bits & ((1ull << 52) - 1);
    if (E == 0 && frac == 0) return 0;
    const uint64_t M = E ? (frac | (1ull << 52)) : frac;
    const int sh = (int)(1075 - (E ? E : 1));
    const unsigned __int128 prod = (unsigned __int128)M * n;
    if (prod == 0) return 0;
    if (sh >= 128) return 1;
    const unsigned __int128 q = prod >> sh;
    return (uint64_t)(((q << sh) == prod) ? q : q + 1);
}

bool valid_k(double k) { return k >= 0.0 && k < 1.0; }  // false for NaN

}  // namespace

// =============================================================================== misc
extern "C" const char *cats_status_string(cats_status_t s) {
    switch (s) {
        case CATS_OK: return "CATS_OK";
        case CATS_E_NULL: return "CATS_E_NULL";
        case CATS_E_SHAPE: return "CATS_E_SHAPE";
        case CATS_E_DTYPE: return "CATS_E_DTYPE";
        case CATS_E_ALIGN: return "CATS_E_ALIGN";
        case CATS_E_SPARSITY: return "CATS_E_SPARSITY";
        case CATS_E_EMPTY: return "CATS_E_EMPTY";
        case CATS_E_NONFINITE: return "CATS_E_NONFINITE";
        case CATS_E_THRESHOLD: return "CATS_E_THRESHOLD";
        case CATS_E_BATCH: return "CATS_E_BATCH";
        case CATS_E_WORKSPACE: return "CATS_E_WORKSPACE";
        case CATS_E_CUDA: return "CATS_E_CUDA";
        case CATS_E_UNSUPPORTED: return "CATS_E_UNSUPPORTED";
    }
    return "CATS_E_UNKNOWN";
}

extern "C" const char *cats_last_cuda_error(void) { return g_last_cuda_error.c_str(); }
extern "C" int cats_version(void) { return CATS_VERSION; }

// =============================================================================== calibration
extern "C" cats_status_t cats_calib_rank(double k, uint64_t n, uint64_t *r) {
    if (!r) return CATS_E_NULL;
    if (!valid_k(k)) return CATS_E_SPARSITY;
    *r = exact_rank(k, n);
    return CATS_OK;
}

extern "C" cats_status_t cats_calibrate_workspace_bytes(uint64_t n, cats_dtype_t dt, size_t *bytes) {
    (void)n;
    if (!bytes) return CATS_E_NULL;
    if (dt != CATS_BF16 && dt != CATS_F32) return CATS_E_DTYPE;
    *bytes = kCalibWsBytes;
    return CATS_OK;
}

extern "C" cats_status_t cats_calib_window_init(uint64_t n, cats_dtype_t dt, cats_calib_window_t *w) {
    if (!w) return CATS_E_NULL;
    if (dt != CATS_BF16 && dt != CATS_F32) return CATS_E_DTYPE;
    make_window(0, key_max(dt), CATS_CALIB_MAX_BINS, w);
    const uint64_t nvec = n / (dt == CATS_BF16 ? 8 : 4);
    // sample ~2^20 vectors (~8M bf16 values) when the data is large; odd stride against aliasing. The
    // sample's 6-sigma margin is then ~0.1% of the mass: the full pass's window holds a key or two
    w->sample_stride = nvec > (1ull << 24) ? ((nvec >> 20) | 1ull) : 0ull;
    return CATS_OK;
}

extern "C" cats_status_t cats_calib_hist(const void *acts, uint64_t n, cats_dtype_t dt, const cats_calib_window_t *w,
                                         uint64_t *hist_dev, uint64_t *counts_dev, cats_stream_t s) {
    if (!acts || !w || !hist_dev || !counts_dev) return CATS_E_NULL;
    if (dt != CATS_BF16 && dt != CATS_F32) return CATS_E_DTYPE;
    if (!aligned16(acts)) return CATS_E_ALIGN;
    if (w->hi < w->lo || w->hi > key_max(dt) || w->nbins == 0 || w->nbins > CATS_CALIB_MAX_BINS ||
        w->shift > 31 || ((w->hi - w->lo) >> w->shift) + 1u != w->nbins)
        return CATS_E_SHAPE;
    if (n == 0) return CATS_OK;
    return cuda_status(launch_calib_hist(acts, n, dt, *w, hist_dev, counts_dev, static_cast<cudaStream_t>(s)));
}

extern "C" cats_status_t cats_calib_step(const uint64_t *hist, const uint64_t *counts, uint64_t n, cats_dtype_t dt,
                                         double k, cats_calib_window_t *w, int *done, uint32_t *t_bits,
                                         uint64_t *count_lt, uint64_t *count_le) {
    if (!hist || !counts || !w || !done || !t_bits || !count_lt || !count_le) return CATS_E_NULL;
    if (dt != CATS_BF16 && dt != CATS_F32) return CATS_E_DTYPE;
    if (!valid_k(k)) return CATS_E_SPARSITY;
    if (n == 0) return CATS_E_EMPTY;
    *done = 0;
    const uint32_t kmax = key_max(dt);
    const uint64_t below = counts[CATS_CALIB_BELOW], inwin = counts[CATS_CALIB_INWIN];
    const uint64_t above = counts[CATS_CALIB_ABOVE], nonfin = counts[CATS_CALIB_NONFINITE];
    if (nonfin) return CATS_E_NONFINITE;
    const uint64_t r = exact_rank(k, n);

    if (w->sample_stride) {
        // aim a full-data window at the rank with a 6-sigma binomial margin (statistics only steer
        // the window; exactness comes from the full passes, which re-aim if the rank is missed)
        const uint64_t ns = below + inwin + above;
        if (r == 0) { make_window(0, 0, kFullPassBins, w); return CATS_OK; }
        if (ns == 0) { make_window(0, kmax, CATS_CALIB_MAX_BINS, w); return CATS_OK; }
        const double rs = k * (double)ns;
        const double delta = 6.0 * std::sqrt((double)ns * k * (1.0 - k)) + 16.0;
        const double rlo = rs - delta, rhi = rs + delta;
        uint32_t lo = 0, hi = kmax;
        if (rlo > (double)below) {
            uint64_t cum = below;
            for (uint32_t b = 0; b < w->nbins; ++b) {
                cum += hist[b];
                if ((double)cum >= rlo) { lo = w->lo + (b << w->shift); break; }
            }
        }
        if (rhi <= (double)(below + inwin)) {
            uint64_t cum = below;
            for (uint32_t b = 0; b < w->nbins; ++b) {
                cum += hist[b];
                if ((double)cum >= rhi) {
                    const uint64_t h = (uint64_t)w->lo + ((uint64_t)(b + 1) << w->shift) - 1;
                    hi = (uint32_t)std::min<uint64_t>(h, w->hi);
                    break;
                }
            }
        }
        make_window(lo, hi, kFullPassBins, w);
        return CATS_OK;
    }

    if (below + inwin + above != n) return CATS_E_SHAPE;
    if (r == 0) {  // k = 0: t = 0 (reading G4); count_le = #{|a| == 0}
        if (w->lo == 0 && w->shift == 0) {
            *t_bits = 0;
            *count_lt = 0;
            *count_le = hist[0];
            *done = 1;
        } else {
            make_window(0, 0, kFullPassBins, w);
        }
        return CATS_OK;
    }
    if (r <= below) { make_window(0, w->lo - 1, kFullPassBins, w); return CATS_OK; }
    if (r > below + inwin) { make_window(w->hi + 1, kmax, kFullPassBins, w); return CATS_OK; }
    uint64_t cum = below;
    uint32_t b = 0;
    for (; b < w->nbins; ++b) {
        if (cum + hist[b] >= r) break;
        cum += hist[b];
    }
    if (b == w->nbins) return CATS_E_SHAPE;  // histogram inconsistent with counts
    if (w->shift == 0) {
        *t_bits = w->lo + b;
        *count_lt = cum;
        *count_le = cum + hist[b];
        *done = 1;
        return CATS_OK;
    }
    const uint32_t lo = w->lo + (b << w->shift);
    const uint32_t hi = (uint32_t)std::min<uint64_t>((uint64_t)lo + (1ull << w->shift) - 1, w->hi);
    make_window(lo, hi, kFullPassBins, w);
    return CATS_OK;
}

extern "C" cats_status_t cats_calibrate_threshold(const void *acts, uint64_t n, cats_dtype_t dt, double k, void *ws,
                                                  size_t ws_bytes, cats_stream_t s, float *t_out,
                                                  cats_calib_info_t *info) {
    if (!acts || !t_out) return CATS_E_NULL;
    if (dt != CATS_BF16 && dt != CATS_F32) return CATS_E_DTYPE;
    if (!valid_k(k)) return CATS_E_SPARSITY;
    if (n == 0) return CATS_E_EMPTY;
    if (!aligned16(acts)) return CATS_E_ALIGN;
    if (!ws || ws_bytes < kCalibWsBytes) return CATS_E_WORKSPACE;
    if (!aligned16(ws)) return CATS_E_ALIGN;
    CATS_TRY({
        cudaStream_t st = static_cast<cudaStream_t>(s);
        uint64_t *hist = reinterpret_cast<uint64_t *>(static_cast<char *>(ws) + kCalibHistOff);
        uint64_t *cnt = reinterpret_cast<uint64_t *>(static_cast<char *>(ws) + kCalibCountOff);
        std::vector<uint64_t> h_hist(CATS_CALIB_MAX_BINS);
        uint64_t h_cnt[CATS_CALIB_NCOUNTS];
        cats_calib_window_t w;
        cats_calib_window_init(n, dt, &w);
        uint32_t passes = 0, t_bits = 0;
        uint64_t lt = 0, le = 0;
        int done = 0;
        for (int it = 0; it < 32 && !done; ++it) {
            cudaError_t e = cudaMemsetAsync(hist, 0, (size_t)w.nbins * 8, st);
            if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, CATS_CALIB_COUNTS_LEN * 8, st);
            if (e == cudaSuccess) e = launch_calib_hist(acts, n, dt, w, hist, cnt, st);
            if (e == cudaSuccess) e = cudaMemcpyAsync(h_hist.data(), hist, (size_t)w.nbins * 8, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaMemcpyAsync(h_cnt, cnt, sizeof h_cnt, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) return cuda_status(e);
            if (!w.sample_stride) ++passes;
            cats_status_t rc = cats_calib_step(h_hist.data(), h_cnt, n, dt, k, &w, &done, &t_bits, &lt, &le);
            if (rc != CATS_OK) return rc;
        }
        if (!done) { g_last_cuda_error = "calibration did not converge"; return CATS_E_CUDA; }
        uint32_t f32bits = dt == CATS_BF16 ? (t_bits << 16) : t_bits;
        float t;
        std::memcpy(&t, &f32bits, sizeof t);
        *t_out = t;
        if (info) {
            info->n = n;
            info->rank_r = exact_rank(k, n);
            info->count_lt = lt;
            info->count_le = le;
            info->t_bits = t_bits;
            info->passes = passes;
        }
        return CATS_OK;
    })
}

// =============================================================================== planning
namespace cats {

static std::mutex g_attr_mu;
static std::vector<std::pair<const void *, size_t>> g_attr;  // (kernel, configured smem) per process

cudaError_t ensure_smem_attr(const void *func, size_t smem) {
    if (smem <= 48 * 1024) return cudaSuccess;
    int dev = 0;
    cudaGetDevice(&dev);
    const void *key = reinterpret_cast<const char *>(func) + dev;  // distinct per device
    std::lock_guard<std::mutex> lk(g_attr_mu);
    for (auto &kv : g_attr)
        if (kv.first == key && kv.second >= smem) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    g_attr.emplace_back(key, smem);
    return cudaSuccess;
}

}  // namespace cats

namespace {
// kind 0: gated-MLP plan (d, m); kind 1: App. B input-sparse projection plan (d = d_out, m = d_in)
cats_status_t plan_create(int d, int m, int max_batch, cats_dtype_t dt, int device, int num_sms, int kind,
                          const cats_mlp_plan_options_t *opt_in, cats_mlp_plan_t **out) {
    if (!out) return CATS_E_NULL;
    cats_mlp_plan_options_t o;
    cats_mlp_plan_options_init(&o);
    if (opt_in) {
        if (opt_in->size != sizeof(cats_mlp_plan_options_t)) return CATS_E_SHAPE;
        o = *opt_in;
    }
    if (o.path < CATS_PATH_AUTO || o.path > CATS_PATH_SPLIT) return CATS_E_UNSUPPORTED;
    if (o.compaction < CATS_COMPACT_BALLOT || o.compaction > CATS_COMPACT_ATOMIC) return CATS_E_UNSUPPORTED;
    if (o.lazy_tail < 0 || o.min_tiles < 1 || o.l2_prefetch < 0 || o.max_stages < 0 || o.max_stages == 1 ||
        (o.rows_per_tile != 0 && o.rows_per_tile != 2 && o.rows_per_tile != 4 && o.rows_per_tile != 6) ||
        o.xs_cols < 0 || o.xs_ranges < 0 || o.xs_ranges > 8)
        return CATS_E_SHAPE;
    if (d <= 0 || m <= 0) return CATS_E_SHAPE;
    if (dt != CATS_BF16 && dt != CATS_F32) return CATS_E_DTYPE;
    if (max_batch < 1 || max_batch > CATS_MAX_BATCH) return CATS_E_BATCH;
    const int esize = dt == CATS_BF16 ? 2 : 4;
    if (((size_t)d * esize) % 16 != 0) return CATS_E_ALIGN;
    const bool query_device = num_sms <= 0;
    if (num_sms <= 0) {
        cudaError_t e = cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, device);
        if (e != cudaSuccess) return cuda_status(e);
    }
    CATS_TRY({
        PlanData p{};
        p.d = d;
        p.m = m;
        p.max_batch = max_batch;
        p.dt = dt;
        p.device = device;
        p.num_sms = num_sms;
        p.esize = esize;
        p.vec = 16 / esize;
        p.nchunks = d * esize / 16;
        p.compaction = kind == 0 ? o.compaction : CATS_COMPACT_BALLOT;
        p.nr_force = o.rows_per_tile;
        p.trace = o.trace != 0;
        p.kind = kind;
        p.g1 = 0;
        if (kind == 1) {  // App. B: kernel XS only (xsparse.cu)
            // per batch size b: column parts of C = 16 * nch / esize columns (nch | 32 threads per row
            // segment), clusters of R <= 8 ranges of the kept list; the most CTAs up to `cps` per SM whose
            // shared memory fits, ties to the widest segment; segments under 128 B only when no wider one
            // divides d_out. Two CTAs per SM unless x (staged in shared memory) needs the whole SM.
            p.xs_no_mma = o.xs_mma == 0;
            for (int b = 1; b <= max_batch; ++b) {
                PlanData::XsCfg &c = p.xs[b];
                bool fits = false;
                for (int cps = 2; cps >= 1 && !fits; --cps) {
                    const int slots = cps * num_sms;
                    const size_t budget = cps == 2 ? kXsSmemBudget : kSmemBudget;
                    int best = 0;
                    bool wide_ok = false;  // some segment of >= 128 B divides d_out
                    // tensor-core batches take 64- or 128-column slabs when d_out allows
                    const bool mma = esize == 2 && b >= kXsMmaForceB && !p.xs_no_mma && d % 64 == 0;
                    for (int nch = 32; nch >= 1; nch /= 2) {
                        const int cols = 16 * nch / esize;
                        if (d % cols != 0 || (nch < 8 && wide_ok)) continue;
                        if (mma && cols != 64 && cols != 128) continue;
                        if (nch >= 8) wide_ok = true;
                        const PlanData::XsCfg keep = c;
                        c.cols = cols;
                        c.q = d / cols;
                        c.r = std::max(1, std::min(8, slots / c.q));
                        const int qr = c.q * c.r;
                        const int score = qr <= slots ? qr : 1;  // Q alone over a wave: last resort
                        if (score > best && xs_smem_bytes(p, b) <= budget) best = score;
                        else c = keep;
                    }
                    fits = best > 0;
                }
                if (!fits) return CATS_E_UNSUPPORTED;
                if (o.xs_cols > 0 && d % o.xs_cols == 0 && (o.xs_cols * esize) % 16 == 0 && o.xs_cols * esize <= 512) {
                    c.cols = o.xs_cols;
                    c.q = d / c.cols;
                }
                if (o.xs_ranges >= 1) c.r = o.xs_ranges;
                if (xs_smem_bytes(p, b) > kSmemBudget) return CATS_E_UNSUPPORTED;
                // with a device: shrink the clusters until every one of them is resident at once (the GPCs'
                // SM counts need not be multiples of the cluster footprint)
                c.clusters = -1;
                if (query_device && !o.xs_no_shrink && cudaSetDevice(device) == cudaSuccess) {
                    for (;;) {
                        c.clusters = xs_active_clusters(p, b);
                        if (c.clusters < 0 || c.clusters >= c.q || c.r == 1) break;
                        --c.r;
                    }
                }
            }
            size_t off = 0;
            p.off_sched = off;   off = align_up(off + kSchedBytes, 256);
            p.off_tokmask = off; off = align_up(off + (size_t)m, 256);  // per-input keep bits (introspection)
            p.off_trace = off;
            p.trace_bytes = p.trace ? (size_t)kTraceKernels * kTraceCtas * kTraceSlots * 8 : 0;
            off = align_up(off + p.trace_bytes, 256);
            p.ws_bytes = off;
            cats_mlp_plan *plan = new cats_mlp_plan;
            plan->p = p;
            *out = plan;
            return CATS_OK;
        }
        for (int b = 1; b <= max_batch; ++b) {
            // K12: persistent CTAs pulling NR-row tiles from a global counter
            if (k12_cpt(p, b) > (b == 1 ? kMaxCPT : 2)) return CATS_E_UNSUPPORTED;
            if (k12_stages(p, b) < 2 || k12_smem_bytes(p, b, k12_stages(p, b)) > k12_smem_budget_c(b))
                return CATS_E_UNSUPPORTED;
            p.g1 = std::max(p.g1, k12_grid(p, b));
        }
        // workspace
        size_t off = 0;
        p.off_sched = off;   off = align_up(off + kSchedBytes, 256);
        p.off_idx = off;     off = align_up(off + (size_t)m * 4, 256);
        p.off_tokmask = off; off = align_up(off + (size_t)m, 256);
        p.off_vals = off;    off = align_up(off + (size_t)m * max_batch * 4, 256);
        p.off_cnt = off;     off = align_up(off + (size_t)((m + 1) / 2) * 4, 256);  // per-tile counts (tiles >= 2 rows)
        p.off_ypart = off;   off = align_up(off + (size_t)2 * max_batch * d * 8, 256);  // 2 int64 y accumulators (K12)
        p.off_xstage = off;  off = align_up(off + (size_t)max_batch * d * esize, 256);
        p.off_ystage = off;  off = align_up(off + (size_t)max_batch * d * 4, 256);
        // split path (b >= 2): x1 per compact position and the KB range partials
        // non-default compaction modes (the App. D ablation) run K12-based kernels at every batch size
        // AUTO: K12 at b = 1 while a consumer thread holds <= 2 chunks of a row (d <= 4096 bf16); wider rows
        // (Llama2-13B, d = 5120: K12 needs 3 chunks per thread and 4-row tiles) take KA + KB from b = 1
        // (measured, 13B b = 1: 51.9 vs 57.6 us unsharded, 17.4 vs 19.1 us at the TP8 shard)
        p.split_min_b = (o.path == CATS_PATH_FUSED || p.compaction != CATS_COMPACT_BALLOT) ? CATS_MAX_BATCH + 1
                        : (o.path == CATS_PATH_SPLIT || (esize == 2 && k12_cpt(p, 1) >= 3)) ? 1 : 2;
        size_t part_bytes = 0, x1_bytes = 0;
        for (int b = p.split_min_b; b <= max_batch; ++b) {
            if (!split_supported(p, b)) continue;
            part_bytes = std::max(part_bytes, (size_t)split_ranges(p, b) * b * d * 4);
            x1_bytes = std::max(x1_bytes, (size_t)split_ntiles(p, b) * split_rows_per_tile(p, b) * b * 4);
        }
        p.off_x1 = off;      off = align_up(off + x1_bytes, 256);
        p.off_tmask = off;   off = align_up(off + (size_t)((m + 1) / 2) * 4, 256);
        p.off_part = off;    off = align_up(off + part_bytes, 256);
        const bool atomic_list = p.compaction == CATS_COMPACT_ATOMIC;  // App. D Alg. 1: global idcs list
        p.off_gidx = off;    off = align_up(off + (atomic_list ? (size_t)m * 4 : 0), 256);
        p.off_gval = off;    off = align_up(off + (atomic_list ? (size_t)m * max_batch * 4 : 0), 256);
        p.k12_min_tiles = o.min_tiles;
        p.k12_l2pf = o.l2_prefetch;  // measured: prefetching only slows the drain (default 0)
        p.k12_eager = o.eager;
        p.k12_max_stages = o.max_stages;
        p.lazy_tail = o.lazy_tail;
        p.off_trace = off;
        p.trace_bytes = p.trace ? (size_t)kTraceKernels * kTraceCtas * kTraceSlots * 8 : 0;
        off = align_up(off + p.trace_bytes, 256);
        p.ws_bytes = off;
        cats_mlp_plan *plan = new cats_mlp_plan;
        plan->p = p;
        *out = plan;
        return CATS_OK;
    })
}
}  // namespace

extern "C" cats_status_t cats_mlp_plan_options_init(cats_mlp_plan_options_t *o) {
    if (!o) return CATS_E_NULL;
    std::memset(o, 0, sizeof *o);
    o->size = sizeof *o;
    o->path = CATS_PATH_AUTO;
    o->compaction = CATS_COMPACT_BALLOT;
    o->lazy_tail = 8;
    o->min_tiles = 2;
    o->xs_mma = 1;
    return CATS_OK;
}

extern "C" cats_status_t cats_mlp_plan_create(int d, int m, int max_batch, cats_dtype_t dt, int device, int num_sms,
                                              cats_mlp_plan_t **out) {
    return plan_create(d, m, max_batch, dt, device, num_sms, 0, nullptr, out);
}

extern "C" cats_status_t cats_mlp_plan_create_ex(int d, int m, int max_batch, cats_dtype_t dt, int device, int num_sms,
                                                 const cats_mlp_plan_options_t *opt, cats_mlp_plan_t **out) {
    return plan_create(d, m, max_batch, dt, device, num_sms, 0, opt, out);
}

extern "C" cats_status_t cats_xsparse_plan_create(int d_in, int d_out, int max_batch, cats_dtype_t dt, int device,
                                                  int num_sms, cats_mlp_plan_t **out) {
    return plan_create(d_out, d_in, max_batch, dt, device, num_sms, 1, nullptr, out);
}

extern "C" cats_status_t cats_xsparse_plan_create_ex(int d_in, int d_out, int max_batch, cats_dtype_t dt, int device,
                                                     int num_sms, const cats_mlp_plan_options_t *opt,
                                                     cats_mlp_plan_t **out) {
    return plan_create(d_out, d_in, max_batch, dt, device, num_sms, 1, opt, out);
}

extern "C" cats_status_t cats_xsparse_gemv(const cats_mlp_plan_t *plan, const void *x, int b, const void *W_in_major,
                                           float t, float *y, void *ws, size_t ws_bytes, cats_stream_t s) {
    if (!plan || !x || !W_in_major || !y) return CATS_E_NULL;
    if (plan->p.kind != 1) return CATS_E_UNSUPPORTED;
    if (b < 1 || b > plan->p.max_batch) return CATS_E_BATCH;
    if (!ws || ws_bytes < plan->p.ws_bytes) return CATS_E_WORKSPACE;
    if (!aligned16(x) || !aligned16(W_in_major) || !aligned16(y) || !aligned16(ws)) return CATS_E_ALIGN;
    if (!(t >= 0.0f) || std::isinf(t)) return CATS_E_THRESHOLD;
    cudaError_t e = cudaSetDevice(plan->p.device);
    if (e == cudaSuccess) e = launch_xsparse(plan->p, x, b, W_in_major, t, y, ws, static_cast<cudaStream_t>(s));
    return cuda_status(e);
}

extern "C" void cats_mlp_plan_destroy(cats_mlp_plan_t *plan) { delete plan; }

extern "C" cats_status_t cats_mlp_plan_info(const cats_mlp_plan_t *plan, cats_mlp_plan_info_t *info) {
    if (!plan || !info) return CATS_E_NULL;
    const PlanData &p = plan->p;
    const int b = p.max_batch;
    info->d = p.d;
    info->m = p.m;
    info->max_batch = p.max_batch;
    info->w_dtype = p.dt;
    info->device = p.device;
    info->num_sms = p.num_sms;
    if (p.kind == 1) {  // kernel XS: Q x R CTAs (clusters of R), W rows per ring stage
        info->grid = p.xs[b].q * p.xs[b].r;
        info->threads = kXsThreads;
        info->rows_per_tile = p.xs[b].r;  // cluster size: ranges of the kept list per column part
        info->stages = p.xs[b].clusters;  // clusters resident at once (-1: planned without a device)
        info->smem = xs_smem_bytes(p, b);
    } else {
        info->grid = k12_grid(p, b);
        info->threads = k12_threads_c(b);
        info->rows_per_tile = k12_rows_per_tile(p, b);
        info->stages = k12_stages(p, b);
        info->smem = k12_smem_bytes(p, b, info->stages);
    }
    info->workspace_bytes = p.ws_bytes;
    return CATS_OK;
}

extern "C" cats_status_t cats_mlp_workspace_bytes(const cats_mlp_plan_t *plan, size_t *bytes) {
    if (!plan || !bytes) return CATS_E_NULL;
    *bytes = plan->p.ws_bytes;
    return CATS_OK;
}

extern "C" cats_status_t cats_mlp_workspace_init(const cats_mlp_plan_t *plan, void *ws, size_t ws_bytes,
                                                 cats_stream_t s) {
    if (!plan) return CATS_E_NULL;
    if (!ws || ws_bytes < plan->p.ws_bytes) return CATS_E_WORKSPACE;
    if (!aligned16(ws)) return CATS_E_ALIGN;
    cudaError_t e = cudaSetDevice(plan->p.device);
    if (e == cudaSuccess) e = cudaMemsetAsync(static_cast<char *>(ws) + plan->p.off_sched, 0, kSchedBytes,
                                              static_cast<cudaStream_t>(s));
    if (plan->p.kind == 1) return cuda_status(e);  // XS keeps no state between calls
    if (e == cudaSuccess)
        e = cudaMemsetAsync(static_cast<char *>(ws) + plan->p.off_ypart, 0, (size_t)2 * plan->p.max_batch * plan->p.d * 8,
                            static_cast<cudaStream_t>(s));
    if (e == cudaSuccess)
        e = cudaMemsetAsync(static_cast<char *>(ws) + plan->p.off_tmask, 0, (size_t)((plan->p.m + 1) / 2) * 4,
                            static_cast<cudaStream_t>(s));
    return cuda_status(e);
}

// =============================================================================== decode
namespace {

cats_status_t validate_common(const cats_mlp_plan_t *plan, const void *x, int b, const void *a, const void *bptr,
                              const void *c, const void *y, const void *ws, size_t ws_bytes) {
    if (!plan || !x || !a || !bptr || !c || !y) return CATS_E_NULL;
    if (plan->p.kind != 0) return CATS_E_UNSUPPORTED;  // an input-sparse projection plan
    if (b < 1 || b > plan->p.max_batch) return CATS_E_BATCH;
    if (!ws || ws_bytes < plan->p.ws_bytes) return CATS_E_WORKSPACE;
    if (!aligned16(x) || !aligned16(a) || !aligned16(bptr) || !aligned16(c) || !aligned16(y) || !aligned16(ws))
        return CATS_E_ALIGN;
    return CATS_OK;
}

// b = 1 (or a shape the split path does not take): K12, one kernel. b >= split_min_b: KA + KB.
cudaError_t launch_mlp(const PlanData &p, const void *x, int b, const void *Wg, const void *Wu, const void *Wd,
                       float t, int mode, float *y, void *ws, cudaStream_t st, cudaEvent_t ev_mid) {
    if (b >= p.split_min_b && split_supported(p, b)) return launch_split(p, x, b, Wg, Wu, Wd, t, mode, y, ws, st, ev_mid);
    cudaError_t e = launch_k12(p, x, b, Wg, Wu, Wd, t, mode, nullptr, y, ws, st);
    if (e == cudaSuccess && ev_mid) e = cudaEventRecord(ev_mid, st);
    return e;
}

cats_status_t run_mlp(const PlanData &p, const void *x, int b, const void *Wg, const void *Wu, const void *Wd, float t,
                      int dense, float *y, void *ws, cudaStream_t st, cudaEvent_t ev_mid = nullptr) {
    cudaError_t e = cudaSetDevice(p.device);
    if (e != cudaSuccess) return cuda_status(e);
    if (!dense && p.compaction == CATS_COMPACT_ATOMIC) {
        // App. D Alg. 1: launch 1 = gate GEMV, SiLU, Mask and atomic appends to idcs; launch 2 = sparse up x v
        // and down projection over idcs (both K12 instantiations, chained by programmatic dependent launch)
        e = launch_k12(p, x, b, Wg, Wu, Wd, t, kModeAtomicGate, nullptr, y, ws, st);
        if (e == cudaSuccess && ev_mid) e = cudaEventRecord(ev_mid, st);
        if (e == cudaSuccess) e = launch_k12(p, x, b, Wg, Wu, Wd, t, kModeAtomicList, nullptr, y, ws, st);
        return cuda_status(e);
    }
    const int mode = dense ? kModeDense : (p.compaction == CATS_COMPACT_PREDICATED ? kModePredicated : kModeCats);
    e = launch_mlp(p, x, b, Wg, Wu, Wd, t, mode, y, ws, st, ev_mid);
    return cuda_status(e);
}

}  // namespace

extern "C" cats_status_t cats_mlp_decode(const cats_mlp_plan_t *plan, const void *x, int b, const void *W_gate,
                                         const void *W_up, const void *W_down_nm, float t, float *y, void *ws,
                                         size_t ws_bytes, cats_stream_t s) {
    cats_status_t rc = validate_common(plan, x, b, W_gate, W_up, W_down_nm, y, ws, ws_bytes);
    if (rc != CATS_OK) return rc;
    if (!(t >= 0.0f) || std::isinf(t)) return CATS_E_THRESHOLD;  // NaN fails t >= 0
    return run_mlp(plan->p, x, b, W_gate, W_up, W_down_nm, t, 0, y, ws, static_cast<cudaStream_t>(s));
}

extern "C" cats_status_t cats_mlp_decode_profiled(const cats_mlp_plan_t *plan, const void *x, int b,
                                                  const void *W_gate, const void *W_up, const void *W_down_nm,
                                                  float t, float *y, void *ws, size_t ws_bytes, cats_stream_t s,
                                                  void *const *events) {
    cats_status_t rc = validate_common(plan, x, b, W_gate, W_up, W_down_nm, y, ws, ws_bytes);
    if (rc != CATS_OK) return rc;
    if (!events || !events[0] || !events[1] || !events[2]) return CATS_E_NULL;
    if (!(t >= 0.0f) || std::isinf(t)) return CATS_E_THRESHOLD;
    const PlanData &p = plan->p;
    cudaStream_t st = static_cast<cudaStream_t>(s);
    cudaEvent_t ev[3];
    for (int i = 0; i < 3; ++i) ev[i] = static_cast<cudaEvent_t>(events[i]);
    cudaError_t e = cudaSetDevice(p.device);
    if (e == cudaSuccess) e = cudaEventRecord(ev[0], st);
    if (e != cudaSuccess) return cuda_status(e);
    // K12: ev[1] right after the kernel (= ev[2]); two-launch paths: ev[1] between the launches
    rc = run_mlp(p, x, b, W_gate, W_up, W_down_nm, t, 0, y, ws, st, ev[1]);
    if (rc != CATS_OK) return rc;
    return cuda_status(cudaEventRecord(ev[2], st));
}

extern "C" cats_status_t cats_mlp_dense(const cats_mlp_plan_t *plan, const void *x, int b, const void *W_gate,
                                        const void *W_up, const void *W_down_nm, float *y, void *ws, size_t ws_bytes,
                                        cats_stream_t s) {
    cats_status_t rc = validate_common(plan, x, b, W_gate, W_up, W_down_nm, y, ws, ws_bytes);
    if (rc != CATS_OK) return rc;
    return run_mlp(plan->p, x, b, W_gate, W_up, W_down_nm, 0.0f, 1, y, ws, static_cast<cudaStream_t>(s));
}

extern "C" cats_status_t cats_mlp_decode_host(const cats_mlp_plan_t *plan, const void *x_host, int b,
                                              const void *W_gate, const void *W_up, const void *W_down_nm, float t,
                                              float *y_host, void *ws, size_t ws_bytes, cats_stream_t s) {
    if (!plan || !x_host || !y_host || !W_gate || !W_up || !W_down_nm) return CATS_E_NULL;
    if (plan->p.kind != 0) return CATS_E_UNSUPPORTED;  // an input-sparse projection plan
    if (b < 1 || b > plan->p.max_batch) return CATS_E_BATCH;
    if (!ws || ws_bytes < plan->p.ws_bytes) return CATS_E_WORKSPACE;
    if (!aligned16(ws) || !aligned16(W_gate) || !aligned16(W_up) || !aligned16(W_down_nm)) return CATS_E_ALIGN;
    if (!(t >= 0.0f) || std::isinf(t)) return CATS_E_THRESHOLD;
    const PlanData &p = plan->p;
    cudaStream_t st = static_cast<cudaStream_t>(s);
    char *w = static_cast<char *>(ws);
    void *xd = w + p.off_xstage;
    float *yd = reinterpret_cast<float *>(w + p.off_ystage);
    cudaError_t e = cudaSetDevice(p.device);
    if (e != cudaSuccess) return cuda_status(e);
    // pinned (mapped) host buffers: a small kernel pulls x across PCIe (the decode kernel then overlaps its
    // start with it through programmatic dependent launch) and the kernel writes y straight into host memory
    // (one small PCIe write from the converting CTAs); pageable buffers go through copies
    auto mapped = [](const void *h) -> void * {
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, h) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer &&
            aligned16(pa.devicePointer))
            return pa.devicePointer;
        (void)cudaGetLastError();  // clear a pageable-pointer query error
        return nullptr;
    };
    const size_t x_bytes = (size_t)b * p.d * p.esize;
    const void *x_direct = mapped(x_host);
    float *y_direct = static_cast<float *>(mapped(y_host));
    e = x_direct ? launch_x_stage(x_direct, xd, x_bytes, st)
                 : cudaMemcpyAsync(xd, x_host, x_bytes, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_status(e);
    cats_status_t rc = run_mlp(p, xd, b, W_gate, W_up, W_down_nm, t, 0, y_direct ? y_direct : yd, ws, st);
    if (rc != CATS_OK) return rc;
    if (!y_direct) e = cudaMemcpyAsync(y_host, yd, (size_t)b * p.d * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return cuda_status(e);
}

struct cats_mlp_host_call {
    cudaGraphExec_t exec;
    cudaStream_t stream;
    int device;
};

extern "C" cats_status_t cats_mlp_host_call_create(const cats_mlp_plan_t *plan, const void *x_host, int b,
                                                   const void *W_gate, const void *W_up, const void *W_down_nm,
                                                   float t, float *y_host, void *ws, size_t ws_bytes, cats_stream_t s,
                                                   cats_mlp_host_call_t **out) {
    if (!out) return CATS_E_NULL;
    *out = nullptr;
    // validation, attribute setup and one uncaptured call (also the pageable-buffer errors)
    cats_status_t rc = cats_mlp_decode_host(plan, x_host, b, W_gate, W_up, W_down_nm, t, y_host, ws, ws_bytes, s);
    if (rc != CATS_OK) return rc;
    const PlanData &p = plan->p;
    auto mapped = [](const void *h) -> void * {
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, h) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer &&
            aligned16(pa.devicePointer))
            return pa.devicePointer;
        (void)cudaGetLastError();
        return nullptr;
    };
    const void *xm = mapped(x_host);
    float *ym = static_cast<float *>(mapped(y_host));
    if (!xm || !ym) return CATS_E_UNSUPPORTED;
    cudaStream_t st = static_cast<cudaStream_t>(s);
    char *w = static_cast<char *>(ws);
    void *xd = w + p.off_xstage;
    // captured on a private stream (s may be the legacy default stream, which cannot capture); the graph
    // is launched on s. The uncaptured call above has completed (it blocks), so nothing is pending.
    cudaStream_t cs = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_status(e);
    e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    cats_status_t rr = CATS_OK;
    if (e == cudaSuccess) {
        e = launch_x_stage(xm, xd, (size_t)b * p.d * p.esize, cs);
        if (e == cudaSuccess) rr = run_mlp(p, xd, b, W_gate, W_up, W_down_nm, t, 0, ym, ws, cs);
        const cudaError_t ee = cudaStreamEndCapture(cs, &graph);
        if (e == cudaSuccess) e = ee;
    }
    if (e == cudaSuccess && rr == CATS_OK) e = cudaGraphInstantiate(&exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    cudaStreamDestroy(cs);
    if (e != cudaSuccess || rr != CATS_OK) {
        const cats_status_t out_rc = e != cudaSuccess ? cuda_status(e) : rr;
        (void)cudaGetLastError();  // a failed capture must not leak into the next call's launch checks
        return out_rc;
    }
    cats_mlp_host_call_t *c = new (std::nothrow) cats_mlp_host_call{exec, st, p.device};
    if (!c) {
        cudaGraphExecDestroy(exec);
        g_last_cuda_error = "host allocation failed";
        return CATS_E_CUDA;
    }
    *out = c;
    return CATS_OK;
}

extern "C" cats_status_t cats_mlp_host_call_run(cats_mlp_host_call_t *c) {
    if (!c) return CATS_E_NULL;
    cudaError_t e = cudaSetDevice(c->device);
    if (e == cudaSuccess) e = cudaGraphLaunch(c->exec, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    return cuda_status(e);
}

extern "C" void cats_mlp_host_call_destroy(cats_mlp_host_call_t *c) {
    if (!c) return;
    cudaGraphExecDestroy(c->exec);
    delete c;
}

extern "C" cats_status_t cats_mlp_gate_act(const cats_mlp_plan_t *plan, const void *x, int b, const void *W_gate,
                                           float *acts, void *ws, size_t ws_bytes, cats_stream_t s) {
    if (!plan || !x || !W_gate || !acts) return CATS_E_NULL;
    if (plan->p.kind != 0) return CATS_E_UNSUPPORTED;  // an input-sparse projection plan
    if (b < 1 || b > plan->p.max_batch) return CATS_E_BATCH;
    if (!ws || ws_bytes < plan->p.ws_bytes) return CATS_E_WORKSPACE;
    if (!aligned16(x) || !aligned16(W_gate) || !aligned16(ws)) return CATS_E_ALIGN;
    cudaError_t e = cudaSetDevice(plan->p.device);
    if (e == cudaSuccess)
        e = launch_k12(plan->p, x, b, W_gate, W_gate, W_gate, 0.0f, kModeGateOnly, acts, nullptr, ws,
                       static_cast<cudaStream_t>(s));
    return cuda_status(e);
}

extern "C" cats_status_t cats_mlp_last_active(const cats_mlp_plan_t *plan, const void *ws, int b, int32_t *idx_host,
                                              uint8_t *tokmask_host, uint32_t *nnz_union, uint32_t *nnz_per_token,
                                              cats_stream_t s) {
    if (!plan || !ws || !idx_host || !tokmask_host || !nnz_union) return CATS_E_NULL;
    if (b < 1 || b > plan->p.max_batch) return CATS_E_BATCH;
    const PlanData &p = plan->p;
    CATS_TRY({
        cudaStream_t st = static_cast<cudaStream_t>(s);
        const char *w = static_cast<const char *>(ws);
        if (p.kind == 1) {  // XS: one keep-bit byte per input, written by CTA 0
            std::vector<uint8_t> kin(p.m);
            cudaError_t e = cudaSetDevice(p.device);
            if (e == cudaSuccess) e = cudaMemcpyAsync(kin.data(), w + p.off_tokmask, (size_t)p.m, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) return cuda_status(e);
            uint32_t k = 0;
            if (nnz_per_token) std::fill(nnz_per_token, nnz_per_token + b, 0u);
            for (int i = 0; i < p.m; ++i) {
                if (!kin[i]) continue;
                idx_host[k] = i;
                tokmask_host[k] = kin[i];
                if (nnz_per_token)
                    for (int tk = 0; tk < b; ++tk) nnz_per_token[tk] += (kin[i] >> tk) & 1u;
                ++k;
            }
            *nnz_union = k;
            return CATS_OK;
        }
        // per-tile segments: the tile geometry of the kernel that ran (K12, or KA's 8-row tiles in
        // column parts on the split path)
        const bool split = b >= p.split_min_b && split_supported(p, b);
        const int ntiles = split ? split_ntiles(p, b) : k12_ntiles(p, b);
        const int nr = split ? split_rows_per_tile(p, b) : k12_rows_per_tile(p, b);
        std::vector<int32_t> idx(p.m), cnt(ntiles);
        std::vector<uint8_t> tm(p.m);
        cudaError_t e = cudaSetDevice(p.device);
        if (e == cudaSuccess) e = cudaMemcpyAsync(idx.data(), w + p.off_idx, (size_t)p.m * 4, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(tm.data(), w + p.off_tokmask, (size_t)p.m, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(cnt.data(), w + p.off_cnt, (size_t)ntiles * 4, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return cuda_status(e);
        uint32_t k = 0;
        if (nnz_per_token) std::fill(nnz_per_token, nnz_per_token + b, 0u);
        for (int c = 0; c < ntiles; ++c) {
            const int64_t r0 = (int64_t)c * nr;
            const int64_t R = std::min<int64_t>(r0 + nr, p.m) - r0;
            if (cnt[c] < 0 || cnt[c] > R) return CATS_E_SHAPE;
            for (int i = 0; i < cnt[c]; ++i) {
                idx_host[k] = idx[r0 + i];
                tokmask_host[k] = tm[r0 + i];
                if (nnz_per_token)
                    for (int tk = 0; tk < b; ++tk) nnz_per_token[tk] += (tm[r0 + i] >> tk) & 1u;
                ++k;
            }
        }
        *nnz_union = k;
        return CATS_OK;
    })
}

extern "C" cats_status_t cats_mlp_kernels_per_call(const cats_mlp_plan_t *plan, int b, int *kernels) {
    if (!plan || !kernels) return CATS_E_NULL;
    if (b < 1 || b > plan->p.max_batch) return CATS_E_BATCH;
    const PlanData &p = plan->p;
    *kernels = p.kind == 1 ? 1 : p.compaction == CATS_COMPACT_ATOMIC ? 2
                               : (b >= p.split_min_b && split_supported(p, b)) ? 2 : 1;
    return CATS_OK;
}

extern "C" cats_status_t cats_mlp_trace_info(const cats_mlp_plan_t *plan, size_t *offset, size_t *bytes) {
    if (!plan || !offset || !bytes) return CATS_E_NULL;
    *offset = plan->p.off_trace;
    *bytes = plan->p.trace_bytes;
    return CATS_OK;
}
