/*
 * cats.h -- C ABI of libcats: the B200 (sm_100a) hot path of CATS
 * (Contextually-Aware Thresholding for Sparsity, arXiv 2404.08763).
 *
 * Citations: "P:n" = PAPER.md line n (section / equation named alongside).
 *
 * What is computed
 *   Calibration, Stage 1 (Eq. 3):  t := min{ t' : F(t') >= k }, F the empirical
 *     CDF of |activations| of one Gated-MLP block. Returned exactly: t is the r-th smallest
 *     |a_i| with r = ceil(k*N) on the binary value of the double k (t = 0 when k = 0).
 *   Decode, Stage 2 (Eq. 1/2/4/5; Custom GPU Kernel "MLP using CATS" P:289-298):
 *     v = SiLU(x W_gate);  Mask = |v| >= t;  x1 = (x W_up[Mask]) * v[Mask];  y = x1 W_down[Mask]
 *     for a batch of b in [1, 8] tokens, each token with its own mask (Eq. 5 is elementwise).
 *
 * Conventions (all calls)
 *   - Tensors are row-major, contiguous, device memory unless the name says _host.
 *   - W_gate, W_up, W_down_nm are NEURON-MAJOR [m][d]: row j holds neuron j's d weights.
 *     (= HF gate_proj.weight, up_proj.weight, down_proj.weight.T.contiguous(); the paper's
 *     d x m W_gate / W_up are their transposes; "columns of W_up and rows of
 *     W_down are the experts".)
 *   - x has the weights' dtype; y is fp32 [b][d]. Accumulation is fp32, never rounded in between.
 *   - Every device pointer is 16-byte aligned and d * sizeof(dtype) is a multiple of 16
 *     (d % 8 == 0 for bf16, d % 4 == 0 for fp32): 128-bit loads and cp.async.bulk need it.
 *   - Ownership: the caller owns every buffer (torch allocates them); a plan owns only host
 *     metadata. A decode workspace is initialised once (cats_mlp_workspace_init); its contents
 *     persist until the next call that uses it.
 *   - Concurrency: plans are immutable and may be shared by threads; concurrent calls need
 *     distinct workspaces and outputs.
 *   - Errors: every entry point returns a cats_status_t; nothing throws or aborts across the
 *     ABI. Arguments are validated before anything is launched; on error nothing is launched
 *     and outputs are untouched. A failed launch returns CATS_E_CUDA (message in
 *     cats_last_cuda_error()). Asynchronous device faults surface at the caller's next sync.
 *   - Streams: cats_stream_t is a cudaStream_t (0 = legacy default stream). Calls that do not
 *     say "blocks" are stream-ordered and asynchronous, with no allocation and no host sync.
 */
#ifndef CATS_H_
#define CATS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CATS_VERSION 1
#define CATS_MAX_BATCH 8

typedef enum {
    CATS_OK = 0,
    CATS_E_NULL = 1,         /* a required pointer is NULL */
    CATS_E_SHAPE = 2,        /* d, m or n out of range / inconsistent */
    CATS_E_DTYPE = 3,        /* unknown dtype */
    CATS_E_ALIGN = 4,        /* pointer not 16-byte aligned or row bytes not a multiple of 16 */
    CATS_E_SPARSITY = 5,     /* k outside [0, 1) or NaN ("desired sparsity level k") */
    CATS_E_EMPTY = 6,        /* n = 0 activations */
    CATS_E_NONFINITE = 7,    /* calibration input holds NaN or +-Inf */
    CATS_E_THRESHOLD = 8,    /* t < 0 or NaN ("t >= 0") */
    CATS_E_BATCH = 9,        /* b outside [1, plan max_batch] */
    CATS_E_WORKSPACE = 10,   /* workspace NULL or smaller than required */
    CATS_E_CUDA = 11,        /* CUDA runtime error; see cats_last_cuda_error() */
    CATS_E_UNSUPPORTED = 12  /* shape beyond what the kernels were built for */
} cats_status_t;

typedef enum {
    CATS_F32 = 0,   /* IEEE binary32 */
    CATS_BF16 = 1   /* bfloat16 */
} cats_dtype_t;

typedef void *cats_stream_t; /* cudaStream_t */

/* Human-readable name of a status code (static storage). */
const char *cats_status_string(cats_status_t s);
/* Message of the last CUDA error seen by this thread ("" if none). Thread-local storage. */
const char *cats_last_cuda_error(void);
/* CATS_VERSION of the loaded library. */
int cats_version(void);

/* =============================================================================================
 * Calibration (Stage 1; Eq. 3 at P:226-233)
 * ========================================================================================== */

/* The single normative rank rule (reading G5 in DESIGN.md): *r = ceil(k * n) computed exactly
 * on the binary value of the double k (0 when k == 0). Host-only.
 * Errors: CATS_E_NULL (r), CATS_E_SPARSITY (k not in [0,1) or NaN). */
cats_status_t cats_calib_rank(double k, uint64_t n, uint64_t *r);

typedef struct {
    uint64_t n;         /* number of activations */
    uint64_t rank_r;    /* r = ceil(k n) */
    uint64_t count_lt;  /* #{ |a_i| <  t } */
    uint64_t count_le;  /* #{ |a_i| <= t }  -- invariant count_lt < k n <= count_le (r > 0) */
    uint32_t t_bits;    /* bit pattern of t in the INPUT dtype (bf16: 16 bits, fp32: 32 bits) */
    uint32_t passes;    /* full passes over the data the GPU made (sample pass not counted) */
} cats_calib_info_t;

/* Device workspace needed by cats_calibrate_threshold / cats_calib_hist (histogram bins and
 * counters). Host-only. Errors: CATS_E_NULL, CATS_E_DTYPE. */
cats_status_t cats_calibrate_workspace_bytes(uint64_t n, cats_dtype_t dt, size_t *bytes);

/* Eq. 3 threshold of one MLP block. acts: n post-SiLU activations (device, 16-B aligned; signed
 * values -- the library takes |.|, so magnitudes also work). k: target sparsity in [0,1).
 * Writes t (fp32; exactly an input value widened, or 0 for k = 0) and, if info != NULL, the
 * exact rank bookkeeping. GPU histogram / radix-select: a strided sample pass picks a key
 * window around the rank, then full passes histogram only the window.
 * BLOCKS on stream s (returns a host scalar).
 * Errors: CATS_E_NULL, CATS_E_DTYPE, CATS_E_ALIGN, CATS_E_SPARSITY, CATS_E_EMPTY,
 *         CATS_E_NONFINITE (any NaN/Inf in acts), CATS_E_WORKSPACE, CATS_E_CUDA. */
cats_status_t cats_calibrate_threshold(const void *acts, uint64_t n, cats_dtype_t dt, double k,
                                       void *ws, size_t ws_bytes, cats_stream_t s,
                                       float *t_out, cats_calib_info_t *info);

/* ---- building blocks (sharded / streamed calibration: all-reduce the histograms between
 *      steps and every rank selects the same t) -------------------------------------------- */

/* A key window: keys are |bit patterns| (sign cleared, 15 bits for bf16, 31 for fp32), whose
 * unsigned order equals the order of |value| for finite values. Bin of key q in [lo, hi] is
 * (q - lo) >> shift; nbins = ((hi - lo) >> shift) + 1 <= CATS_CALIB_MAX_BINS. */
#define CATS_CALIB_MAX_BINS 32768
typedef struct {
    uint32_t lo, hi;     /* inclusive key range, hi <= largest finite key */
    uint32_t shift;      /* bin width = 2^shift keys */
    uint32_t nbins;
    uint64_t sample_stride; /* 0: every element; s > 0: only 16-byte vectors v with v % s == 0 */
} cats_calib_window_t;

/* Counter slots written by cats_calib_hist (accumulated with +=). */
#define CATS_CALIB_BELOW 0     /* finite keys < lo */
#define CATS_CALIB_INWIN 1     /* keys in [lo, hi] */
#define CATS_CALIB_ABOVE 2     /* finite keys > hi */
#define CATS_CALIB_NONFINITE 3 /* NaN / Inf: nonzero iff any was seen (the bf16 pass flags once per
                                  thread instead of counting every value; ABOVE is exact only when 0) */
#define CATS_CALIB_NCOUNTS 4
#define CATS_CALIB_COUNTS_LEN 8 /* length of counts_dev: [0, 4) the counts above, [4, 8) scratch of a
                                   pass (zero on entry; every pass leaves it zero again) */

/* Initial window for n values: the whole finite key range, coarse bins; strided sampling when n
 * is large (the sample only steers the window; it never decides t). Host-only. */
cats_status_t cats_calib_window_init(uint64_t n, cats_dtype_t dt, cats_calib_window_t *w);

/* Device pass: hist_dev[0..w->nbins) += histogram of keys in the window, counts_dev[0..4) +=
 * the CATS_CALIB_* counts, over acts (or its sample). counts_dev holds CATS_CALIB_COUNTS_LEN
 * uint64. Caller zeroes both buffers first (or keeps accumulating chunks / ranks). Asynchronous. Errors: CATS_E_NULL, CATS_E_DTYPE, CATS_E_ALIGN,
 * CATS_E_SHAPE (bad window), CATS_E_CUDA. */
cats_status_t cats_calib_hist(const void *acts, uint64_t n, cats_dtype_t dt, const cats_calib_window_t *w,
                              uint64_t *hist_dev, uint64_t *counts_dev, cats_stream_t s);

/* Host step after a pass over ALL n values (hist/counts summed over every chunk and rank):
 * if the rank-r key is resolved to a single key, *done = 1 and t_bits / count_lt / count_le are
 * set; otherwise *w becomes the next, narrower (or re-aimed) window and *done = 0.
 * If the window came from a sample (w->sample_stride > 0), sample_k_rank is used to aim the
 * next full-data window with a statistical margin instead. Errors: CATS_E_NONFINITE,
 * CATS_E_NULL, CATS_E_SHAPE (counts inconsistent with n). */
cats_status_t cats_calib_step(const uint64_t *hist_host, const uint64_t *counts_host, uint64_t n,
                              cats_dtype_t dt, double k, cats_calib_window_t *w, int *done,
                              uint32_t *t_bits, uint64_t *count_lt, uint64_t *count_le);

/* =============================================================================================
 * Decode (Stage 2; App. D)
 * ========================================================================================== */

typedef struct cats_mlp_plan cats_mlp_plan_t;

typedef struct {
    int d, m, max_batch;
    cats_dtype_t w_dtype;
    int device, num_sms;
    /* K12 (the fused kernel) at b = max_batch: */
    int grid, threads;            /* persistent CTAs (two per SM at b = 1, one at b >= 2) */
    int rows_per_tile;            /* W_gate rows per GATE job; a UD job carries rows_per_tile/2 neurons */
    int stages;                   /* shared-memory ring depth (one job per stage) */
    size_t smem;                  /* dynamic shared memory bytes per CTA */
    size_t workspace_bytes;
} cats_mlp_plan_info_t;

/* Host-only planning (tile and grid choices from the SM count; no device allocation).
 * num_sms <= 0 queries `device`; num_sms > 0 plans for that many SMs without touching a GPU.
 * d: hidden size, m: intermediate size (this rank's shard under tensor parallelism).
 * Errors: CATS_E_NULL, CATS_E_SHAPE (d, m <= 0), CATS_E_DTYPE, CATS_E_ALIGN (row bytes % 16),
 *         CATS_E_BATCH (max_batch not in [1, 8]), CATS_E_UNSUPPORTED (d too large for the
 *         register/shared-memory tiling), CATS_E_CUDA (device query failed). */
cats_status_t cats_mlp_plan_create(int d, int m, int max_batch, cats_dtype_t w_dtype, int device,
                                   int num_sms, cats_mlp_plan_t **out);

/* ---- explicit plan options (kernel-path selection, the App. D ablation, tuning knobs) ---------
 * The library reads no environment variables: every choice that changes which kernels run is an
 * explicit field here, fixed at plan creation. cats_mlp_plan_create(...) == _ex(..., NULL). */
typedef enum {
    CATS_PATH_AUTO = 0,   /* K12 at b = 1; KA + KB at b >= 2 where their shared memory fits */
    CATS_PATH_FUSED = 1,  /* K12 (the single fused kernel) at every batch size */
    CATS_PATH_SPLIT = 2   /* KA + KB wherever they fit, b = 1 included (small tensor-parallel shards) */
} cats_path_t;

/* How the active set reaches the sparse up / down projection (App. D; the ablation
 * figure). Every mode computes the same y (Eq. 5); they differ in launches and traffic. */
typedef enum {
    CATS_COMPACT_BALLOT = 0,     /* default: per-tile warp ballot + popc prefix inside K12 / KA (no atomics) */
    CATS_COMPACT_PREDICATED = 1, /* App. D Alg. 2 (Triton P:803-866): no index list; every tile's rows
                                    are visited in fixed halves and Mask predicates the row loads (inactive rows
                                    are not read, they enter the arithmetic as zeros). K12 only */
    CATS_COMPACT_ATOMIC = 2      /* App. D Alg. 1: "idcs <- indices where Mask = 1" by atomic appends
                                    into one global list (arbitrary order), then a second kernel walks idcs.
                                    Two launches (gate kernel, list kernel) */
} cats_compaction_t;

typedef struct {
    uint32_t size;           /* = sizeof(cats_mlp_plan_options_t) (ABI check; CATS_E_SHAPE otherwise) */
    int32_t path;            /* cats_path_t */
    int32_t compaction;      /* cats_compaction_t (gated-MLP plans; non-default modes always run K12 kernels) */
    int32_t trace;           /* 1: kernels stamp %globaltimer into the workspace (cats_mlp_trace_info) */
    /* tuning (measurement knobs; cats_mlp_plan_options_init sets the planner's defaults) */
    int32_t rows_per_tile;   /* K12 tile height NR: 0 = auto, else 2, 4 or (b = 1 only) 6 */
    int32_t max_stages;      /* K12 ring depth cap: 0 = as many stages as fit, else >= 2 */
    int32_t lazy_tail;       /* K12 / KA reserve no tile ahead for the last lazy_tail x grid tiles (>= 0) */
    int32_t min_tiles;       /* K12 grid <= ntiles / min_tiles (>= 1) */
    int32_t eager;           /* K12 fills every ring stage with claimed tiles at start (0 / 1) */
    int32_t l2_prefetch;     /* K12 static tiles per CTA prefetched into L2 before griddepcontrol.wait (>= 0) */
    int32_t xs_cols;         /* App. B XS: columns per CTA (0 = auto) */
    int32_t xs_ranges;       /* App. B XS: cluster size R (0 = auto, else 1..8) */
    int32_t xs_mma;          /* App. B XS: 1 = tensor cores where the slab allows (default), 0 = FFMA2 only */
    int32_t xs_no_shrink;    /* App. B XS: 1 = keep R even when not every cluster is co-resident */
} cats_mlp_plan_options_t;

/* Fill *opt with the defaults (size set, path AUTO, compaction BALLOT, lazy_tail 8, min_tiles 2,
 * xs_mma 1, the rest 0). Errors: CATS_E_NULL. */
cats_status_t cats_mlp_plan_options_init(cats_mlp_plan_options_t *opt);
/* cats_mlp_plan_create with options (opt == NULL: the defaults). Additional errors: CATS_E_SHAPE
 * (opt->size mismatch or a tuning field out of range), CATS_E_UNSUPPORTED (unknown path / compaction). */
cats_status_t cats_mlp_plan_create_ex(int d, int m, int max_batch, cats_dtype_t w_dtype, int device, int num_sms,
                                      const cats_mlp_plan_options_t *opt, cats_mlp_plan_t **out);
void cats_mlp_plan_destroy(cats_mlp_plan_t *plan);
cats_status_t cats_mlp_plan_info(const cats_mlp_plan_t *plan, cats_mlp_plan_info_t *info);
cats_status_t cats_mlp_workspace_bytes(const cats_mlp_plan_t *plan, size_t *bytes);
/* Initialise a freshly allocated workspace once (zeroes the scheduler counters, the int64 y
 * accumulator and the per-tile mask words, which every launch leaves zeroed again on exit).
 * Required before the first call that uses `ws`. Asynchronous on s.
 * Errors: CATS_E_NULL, CATS_E_WORKSPACE, CATS_E_ALIGN, CATS_E_CUDA. */
cats_status_t cats_mlp_workspace_init(const cats_mlp_plan_t *plan, void *ws, size_t ws_bytes, cats_stream_t s);

/* y[b][d] = CATS_t gated MLP of x[b][d] over this plan's m neurons (under tensor parallelism y
 * is the rank's partial; the caller all-reduces). t >= 0; t = 0 gives dense semantics.
 * b = 1 (d <= 4096): ONE kernel launch on s (K12), a persistent dataflow kernel doing the gate GEMV,
 * SiLU, threshold, compaction, sparse up x v, down projection and the split-K reduction (TMA
 * bulk-reduce of exact fixed-point partials; the last CTA writes y).
 * b >= 2, and b = 1 at d >= 5120: TWO launches (KA: gate + up with compaction; KB: down projection
 * over balanced ranges of the active list + a fixed-order two-phase reduction); bf16 at b >= 3 uses
 * warp-level bf16 MMA for the dot products (KA's x operand held in tensor memory where d % 1024 == 0). cats_mlp_kernels_per_call() tells which. All launches use programmatic dependent
 * launch (a successor's CTAs start streaming weights while the predecessor drains).
 * KB has no grid barrier: the last 64 of its CTAs to finish do the fixed-order reduction while the
 * others exit, so it completes whenever more than 64 of its CTAs (one per SM) can be resident at once;
 * plans for <= 64 SMs take K12 at every batch size.
 * Deterministic: bit-identical y for identical inputs, whatever the dynamic tile schedule.
 * Errors: CATS_E_NULL, CATS_E_ALIGN, CATS_E_BATCH, CATS_E_THRESHOLD, CATS_E_WORKSPACE,
 *         CATS_E_CUDA. */
cats_status_t cats_mlp_decode(const cats_mlp_plan_t *plan, const void *x, int b, const void *W_gate,
                              const void *W_up, const void *W_down_nm, float t, float *y,
                              void *ws, size_t ws_bytes, cats_stream_t s);

/* The library's own dense gated MLP (Eq. 1, the "Dense" baseline of P:530): same kernels with
 * every neuron active. Same arguments / errors as cats_mlp_decode without t. */
cats_status_t cats_mlp_dense(const cats_mlp_plan_t *plan, const void *x, int b, const void *W_gate,
                             const void *W_up, const void *W_down_nm, float *y,
                             void *ws, size_t ws_bytes, cats_stream_t s);

/* End-to-end variant for host activations: brings x_host [b][d] into the workspace, runs
 * cats_mlp_decode and delivers y to y_host [b][d] fp32. Pinned (mapped) x_host: a small kernel reads
 * it across PCIe and the decode kernel overlaps its start with that read (programmatic dependent
 * launch); pageable x_host: a host-to-device copy. Pinned y_host: written by the kernel straight
 * into host memory; pageable: a device-to-host copy. BLOCKS on s. */
cats_status_t cats_mlp_decode_host(const cats_mlp_plan_t *plan, const void *x_host, int b,
                                   const void *W_gate, const void *W_up, const void *W_down_nm,
                                   float t, float *y_host, void *ws, size_t ws_bytes, cats_stream_t s);

/* A bound end-to-end call for a serving loop: the work of cats_mlp_decode_host for fixed arguments,
 * captured once into a CUDA graph (the x staging kernel, the decode kernels chained by programmatic
 * dependent launch, y written by the kernel into host memory), replayed by cats_mlp_host_call_run, which
 * BLOCKS until y_host holds the call's y. Every run re-reads the CURRENT contents of x_host; weights, t,
 * the workspace and the stream are fixed at creation. x_host and y_host must be pinned and mapped
 * (cudaHostAlloc / cudaHostRegister; torch's pin_memory()), else CATS_E_UNSUPPORTED. Creation validates
 * like cats_mlp_decode_host and runs the call once (uncaptured). Not thread-safe per handle. */
typedef struct cats_mlp_host_call cats_mlp_host_call_t;
cats_status_t cats_mlp_host_call_create(const cats_mlp_plan_t *plan, const void *x_host, int b, const void *W_gate,
                                        const void *W_up, const void *W_down_nm, float t, float *y_host, void *ws,
                                        size_t ws_bytes, cats_stream_t s, cats_mlp_host_call_t **out);
cats_status_t cats_mlp_host_call_run(cats_mlp_host_call_t *call);
void cats_mlp_host_call_destroy(cats_mlp_host_call_t *call);

/* Measurement variant of cats_mlp_decode: the identical launch bracketed by events[0] and events[1]
 * (cudaEvent_t created by the caller with timing enabled; events[2] is recorded right after
 * events[1]) -- the kernel's device time for the roofline report. */
cats_status_t cats_mlp_decode_profiled(const cats_mlp_plan_t *plan, const void *x, int b, const void *W_gate,
                                       const void *W_up, const void *W_down_nm, float t, float *y,
                                       void *ws, size_t ws_bytes, cats_stream_t s, void *const *events);

/* Calibration data collection (S "collect_activations"): acts[b][m] = SiLU(x W_gate)
 * in fp32 for b tokens -- the activations Eq. 3 is evaluated on. Uses K1. Asynchronous. */
cats_status_t cats_mlp_gate_act(const cats_mlp_plan_t *plan, const void *x, int b, const void *W_gate,
                                float *acts, void *ws, size_t ws_bytes, cats_stream_t s);

/* Introspection of the last decode on `ws` with batch b: the union of active neurons in
 * ascending order (idx_host[0..*nnz_union)), each one's per-token keep bits (bit i = token i;
 * tokmask_host, same order), and per-token active counts (nnz_per_token[b]). idx_host and
 * tokmask_host must hold m entries; nnz_per_token may be NULL. BLOCKS on s. */
cats_status_t cats_mlp_last_active(const cats_mlp_plan_t *plan, const void *ws, int b, int32_t *idx_host,
                                   uint8_t *tokmask_host, uint32_t *nnz_union, uint32_t *nnz_per_token,
                                   cats_stream_t s);

/* Which kernels a cats_mlp_decode / cats_mlp_dense call with batch b launches on this plan
 * (DESIGN.md §6): *kernels = 1 for the fused single-kernel path K12 (b = 1, or shapes the split path
 * does not take), 2 for the split path KA (gate + up) then KB (down + the two-phase reduction).
 * Errors: CATS_E_NULL, CATS_E_BATCH (b outside [1, max_batch]). Host-only. */
cats_status_t cats_mlp_kernels_per_call(const cats_mlp_plan_t *plan, int b, int *kernels);

/* ---- App. B: CATS on the attention input -------------------------------------------
 * y[b][d_out] = CATS_t(x) W for x[b][d_in], CATS_t(x)_i = x_i if |x_i| >= t else 0 (Eq. 4 applied
 * to the hidden vector itself, ties kept), W stored INPUT-major [d_in][d_out] row-major (row i = the
 * weights input i feeds, i.e. the transpose of a q/k/v_proj weight; several projections sharing
 * the input may be concatenated along d_out). Only the rows of inputs kept for at least one of the
 * b tokens are read from HBM.
 * The plan is a cats_mlp_plan_t of a second kind: cats_mlp_plan_destroy / _info / _workspace_bytes /
 * _workspace_init / _last_active / _kernels_per_call accept it (last_active reports the kept INPUT
 * dimensions); the gated-MLP calls reject it with CATS_E_UNSUPPORTED, and cats_xsparse_gemv rejects
 * a gated-MLP plan the same way.
 * cats_mlp_plan_info on this kind: grid = CTAs, rows_per_tile = cluster size (ranges of the kept
 * list per column slab), stages = clusters resident at once (-1 when planned without a device),
 * smem = dynamic shared memory at max_batch.
 * Errors of _plan_create: as cats_mlp_plan_create (d_out plays d: d_out * esize % 16 == 0;
 * CATS_E_UNSUPPORTED when x [max_batch][d_in] does not fit in shared memory: b x d_in x esize
 * above ~200 KB). */
cats_status_t cats_xsparse_plan_create(int d_in, int d_out, int max_batch, cats_dtype_t w_dtype, int device,
                                       int num_sms, cats_mlp_plan_t **out);
/* with explicit options (only trace and the xs_* fields apply; NULL = defaults) */
cats_status_t cats_xsparse_plan_create_ex(int d_in, int d_out, int max_batch, cats_dtype_t w_dtype, int device,
                                          int num_sms, const cats_mlp_plan_options_t *opt, cats_mlp_plan_t **out);
/* x [b][d_in] (w_dtype), W_in_major [d_in][d_out] (w_dtype), y [b][d_out] fp32, all device memory
 * with 16-byte aligned bases; t >= 0 finite (t = 0 keeps every input: the dense GEMV).
 * ONE launch on s (DESIGN.md §5 XS, thread-block clusters + programmatic dependent launch): every CTA
 * thresholds x and ranks the kept inputs; the CTAs of a cluster stream equal ranges of the kept rows
 * for one slab of output columns and sum their partials in rank order through distributed shared
 * memory: bit-identical y for identical inputs. The workspace holds only the introspection bytes
 * (no state between calls; cats_mlp_workspace_init only zeroes the scheduler words). Asynchronous.
 * Errors: CATS_E_NULL, CATS_E_UNSUPPORTED (plan kind), CATS_E_BATCH, CATS_E_WORKSPACE, CATS_E_ALIGN,
 *         CATS_E_THRESHOLD (t < 0, NaN or Inf), CATS_E_CUDA. */
cats_status_t cats_xsparse_gemv(const cats_mlp_plan_t *plan, const void *x, int b, const void *W_in_major,
                                float t, float *y, void *ws, size_t ws_bytes, cats_stream_t s);

/* ---- Tensor parallelism: one-shot cross-rank reduction over NVLink peer memory ------
 * Each of the P ranks (one process per GPU) holds its m / P neuron block; its cats_mlp_decode returns a
 * partial y_p and y = sum_p y_p (the exchange step; masking needs none: t is layer-global, Eq. 5 is per
 * neuron). Instead of an NCCL all-reduce, every rank allocates one SYMMETRIC buffer of
 * cats_tp_buffer_bytes (device memory, zero-initialised once), exports it with cats_ipc_handle_get, opens
 * every peer's with cats_ipc_handle_open (CUDA IPC over NVLink / NVSwitch) and builds a comm; then
 * cats_tp_allreduce is ONE launch that pushes this rank's partial into every rank's buffer (each float in an
 * 8-byte word with the call's epoch: the data is its own flag), waits until every rank's words of its slice
 * carry the epoch and sums the P partials in fixed rank order 0..P-1: bit-identical y on every rank.
 * Epochs live on the device (graph-capturable); two parity slots make back-to-back calls safe.
 * Requirements: P <= 8; n (floats per call) a multiple of 4 and <= n_max; every rank calls with the same
 * n in the same order; buffers 16-byte aligned. Errors: CATS_E_NULL, CATS_E_SHAPE, CATS_E_ALIGN, CATS_E_CUDA. */
#define CATS_IPC_HANDLE_BYTES 64
typedef struct cats_tp_comm cats_tp_comm_t;
cats_status_t cats_tp_buffer_bytes(int world, uint64_t n_max, size_t *bytes);
/* The symmetric buffer as its own cudaMalloc allocation, zeroed (an IPC handle maps a whole allocation: a
 * sub-range of a caching allocator's block would open at the block's base in the peers). Blocks. */
cats_status_t cats_tp_buffer_alloc(size_t bytes, int device, void **dev_ptr_out);
cats_status_t cats_tp_buffer_free(void *dev_ptr);
cats_status_t cats_ipc_handle_get(const void *dev_ptr, uint8_t *handle_out /* [CATS_IPC_HANDLE_BYTES] */);
cats_status_t cats_ipc_handle_open(const uint8_t *handle, int device, void **dev_ptr_out);
cats_status_t cats_ipc_handle_close(void *dev_ptr);
/* bufs[r] = rank r's symmetric buffer as mapped in this process (bufs[rank] = the local allocation). Host-only. */
cats_status_t cats_tp_comm_create(int rank, int world, uint64_t n_max, void *const *bufs, int device,
                                  cats_tp_comm_t **out);
void cats_tp_comm_destroy(cats_tp_comm_t *comm);
/* y[n] = sum over ranks (order 0..P-1) of every rank's x[n] (fp32, device). Asynchronous on s (programmatic
 * dependent launch: it may start while the decode that writes x drains). x and y may alias. */
cats_status_t cats_tp_allreduce(const cats_tp_comm_t *comm, const float *x, float *y, uint64_t n, cats_stream_t s);
/* The same step for `world` ranks emulated on ONE device (testing without P GPUs): comms[r] built with
 * rank r over buffers on this device, x[r] / y[r] the ranks' partials / outputs; one cooperative launch runs
 * every rank's CTAs (they wait on one another's flags, so they must be co-resident). */
cats_status_t cats_tp_allreduce_emulated(cats_tp_comm_t *const *comms, int world, const float *const *x,
                                         float *const *y, uint64_t n, cats_stream_t s);

/* Diagnostics. When the plan was created with options.trace = 1, the kernels
 * record %globaltimer stamps (ns) per CTA into a trace area of the workspace:
 * uint64 trace[3][512 CTAs][8 slots] at byte `offset` (bytes = 0 when tracing is off).
 * [0] K12 / KA slots: 0 start, 1 ring primed, 2 jobs done, 3 exit, 4 K12 partial reduced, 5 all consumer
 *     warps done, 6 partial staged (bulk reduce issued), 7 bulk reduce complete;
 * [1] KB slots: 0 start, 1 list ready, 2 jobs done, 3 reducer released (last-64 reducers only), 4 exit,
 *     5 masks read, 6 prefix done;
 * [2] per-CTA producer/consumer statistics (see scripts/trace_decode.py). */
cats_status_t cats_mlp_trace_info(const cats_mlp_plan_t *plan, size_t *offset, size_t *bytes);

#ifdef __cplusplus
}
#endif
#endif /* CATS_H_ */
