// cats_internal.h -- host-side plumbing shared by the libcats translation units (not exported).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/cats.h"

namespace cats {

constexpr int kK1Threads = 512;       // 16 warps: one CTA per SM, persistent over its row range
constexpr int kK3Threads = 256;
constexpr size_t kSmemBudget = 227 * 1024;  // usable dynamic shared memory per CTA on sm_100
constexpr int kMaxCPT = 4;            // K2: 16-byte chunks of a row owned per thread

struct PlanData {
    int d, m, max_batch;
    cats_dtype_t dt;
    int device, num_sms;
    int esize;          // bytes per element
    int vec;            // elements per 16 bytes
    int nchunks;        // d * esize / 16
    // K1
    int g1;             // CTAs; CTA c owns neuron rows [c*m/g1, (c+1)*m/g1)
    int r_max;          // max rows per CTA
    // K2
    int p2;             // CTAs (split-K slices of the active list)
    int k2_threads;
    int cpt;            // chunks per thread
    int ns;             // neurons per ring stage
    int stages;         // ring depth
    size_t k2_smem;
    int l_max;          // max active neurons per K2 CTA slice
    // K3
    int k3_grid_max;
    // workspace layout (byte offsets)
    size_t off_idx, off_tokmask, off_vals, off_cnt, off_ypart, off_xstage, off_ystage, ws_bytes;
};

// row range of K1 CTA c (shared by K1, K2 and the host introspection: the compaction layout)
__host__ __device__ inline int64_t k1_row0(int c, int m, int g1) { return (int64_t)c * m / g1; }

size_t k1_smem_bytes(const PlanData &p, int b);
size_t k2_smem_bytes(int dt_esize, int d, int ns, int stages, int b, int l_max, int g1, int threads);

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
