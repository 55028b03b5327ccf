// cats_internal.h -- host-side plumbing shared by the libcats translation units (not exported).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/cats.h"

namespace cats {

constexpr int kK1Threads = 512;       // 16 warps, one persistent CTA per SM
constexpr int kK2Threads = 512;       // 16 warps, one persistent CTA per SM
constexpr int kK3Threads = 256;
constexpr size_t kSmemBudget = 227 * 1024;  // usable dynamic shared memory per CTA on sm_100
constexpr int kMaxCPT = 2;            // 16-byte chunks of a row owned per thread (d <= 8192 bf16)
constexpr int kMaxStages = 8;

struct PlanData {
    int d, m, max_batch;
    cats_dtype_t dt;
    int device, num_sms;
    int esize;          // bytes per element
    int vec;            // elements per 16 bytes
    int nchunks;        // d * esize / 16
    int cpt;            // chunks per thread (K1 and K2, 512 threads)
    int g1;             // K1 CTAs (dynamic tile scheduler)
    int p2;             // K2 CTAs (split-K slices of the active list)
    int l_max;          // max active neurons per K2 CTA slice
    // workspace layout (byte offsets)
    size_t off_sched, off_idx, off_tokmask, off_vals, off_cnt, off_ypart, off_xstage, off_ystage, ws_bytes;
};

// K1 tile height (rows of W_gate per ring stage) for batch b: keeps the per-thread partial dot
// products (rows x tokens) in registers; halved for very wide rows so >= 3 stages fit in smem.
__host__ __device__ constexpr int k1_rows_per_tile_c(int b) { return b <= 2 ? 8 : (b <= 4 ? 4 : 2); }
inline int k1_rows_per_tile(const PlanData &p, int b) {
    int nr = k1_rows_per_tile_c(b);
    const size_t row = (size_t)p.d * p.esize;
    while (nr > 2 && 3 * (size_t)nr * row > kSmemBudget - 16 * 1024) nr /= 2;
    return nr;
}
inline int k1_ntiles(const PlanData &p, int b) { return (p.m + k1_rows_per_tile(p, b) - 1) / k1_rows_per_tile(p, b); }

size_t k1_smem_bytes(const PlanData &p, int b);
int k1_stages(const PlanData &p, int b);
size_t k2_smem_bytes(int esize, int d, int ns, int stages, int b, int l_max, int ntiles);
int k2_neurons_per_stage(const PlanData &p, int b);  // 4, or 2 for very wide rows
int k2_stages(const PlanData &p, int b);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel / size (thread-safe)
cudaError_t ensure_smem_attr(const void *func, size_t smem);

// launchers: return cudaError_t of the launch
cudaError_t launch_k1(const PlanData &p, const void *x, int b, const void *Wg, float t, int dense,
                      float *acts_out, void *ws, cudaStream_t s);
cudaError_t launch_k2(const PlanData &p, const void *x, int b, const void *Wu, const void *Wd, void *ws,
                      cudaStream_t s, bool pdl);
cudaError_t launch_k3(const PlanData &p, int b, const void *ws, float *y, cudaStream_t s, bool pdl);

cudaError_t launch_calib_hist(const void *acts, uint64_t n, cats_dtype_t dt, const cats_calib_window_t &w,
                              uint64_t *hist, uint64_t *counts, cudaStream_t s);

void set_last_cuda_error(cudaError_t e);

}  // namespace cats
