// cats_internal.h -- host-side plumbing shared by the libcats translation units (not exported).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <algorithm>

#include "../../include/cats.h"

namespace cats {

constexpr int kConsumerWarps = 8;     // K12: consumer warps per CTA (column owners)
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kK12Threads = kConsumers + 32;  // + 1 producer warp
constexpr int kCtasPerSm = 2;         // two independent job streams per SM hide per-job latency
constexpr int kK3Threads = 256;
constexpr size_t kSmemBudget = 112 * 1024;  // dynamic shared memory per K12 CTA (2 per SM)
constexpr int kMaxCPT = 4;            // 16-byte chunks of a row owned per consumer (d <= 8192 bf16)
constexpr int kMaxStages = 8;
constexpr int kFixShift = 36;         // y partials: exact 64-bit fixed point, resolution 2^-36

// K12 launch modes
constexpr int kModeCats = 0;          // CATS_t decode
constexpr int kModeDense = 1;         // every neuron active (the library's dense MLP)
constexpr int kModeGateOnly = 2;      // SiLU(x W_gate) only (calibration data collection)

struct PlanData {
    int d, m, max_batch;
    cats_dtype_t dt;
    int device, num_sms;
    int esize;          // bytes per element
    int vec;            // elements per 16 bytes
    int nchunks;        // d * esize / 16
    int cpt;            // chunks per consumer thread
    int g1;             // K12 CTAs (persistent, dynamic tile scheduler)
    // workspace layout (byte offsets)
    size_t off_sched, off_idx, off_tokmask, off_vals, off_cnt, off_ypart, off_xstage, off_ystage, ws_bytes;
    bool trace;         // CATS_TRACE=1 at plan creation: kernels stamp %globaltimer into the workspace
    size_t off_trace, trace_bytes;
};

// K12 tile height NR (W_gate rows per GATE job; a UD job carries NR/2 neurons = the same bytes).
inline int k12_rows_per_tile(const PlanData &p, int b) {
    const size_t row = (size_t)p.d * p.esize;
    (void)b;
    return 4 * row * 3 <= kSmemBudget - 8 * 1024 ? 4 : 2;
}
inline int k12_ntiles(const PlanData &p, int b) { return (p.m + k12_rows_per_tile(p, b) - 1) / k12_rows_per_tile(p, b); }
size_t k12_smem_bytes(const PlanData &p, int b, int stages);
inline int k12_stages(const PlanData &p, int b) {
    const size_t stage = (size_t)k12_rows_per_tile(p, b) * p.d * p.esize;
    const size_t extra = k12_smem_bytes(p, b, 0) + kMaxStages * 256;
    if (extra >= kSmemBudget) return 0;
    return (int)std::min<size_t>((kSmemBudget - extra) / stage, kMaxStages);
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel / size (thread-safe)
cudaError_t ensure_smem_attr(const void *func, size_t smem);

// launchers: return cudaError_t of the launch
cudaError_t launch_k12(const PlanData &p, const void *x, int b, const void *Wg, const void *Wu, const void *Wd,
                       float t, int mode, float *acts, void *ws, cudaStream_t s);
cudaError_t launch_k3(const PlanData &p, int b, void *ws, float *y, cudaStream_t s, bool pdl);

cudaError_t launch_calib_hist(const void *acts, uint64_t n, cats_dtype_t dt, const cats_calib_window_t &w,
                              uint64_t *hist, uint64_t *counts, cudaStream_t s);

void set_last_cuda_error(cudaError_t e);

}  // namespace cats
