/*
 * sparse_assembly.h -- C ABI of the B200-native sparse assembly library
 * (libsa_b200.so).  Matlab-compatible S = sparse(i,j,s,m,n[,nzmax]):
 * 1-based (row, column, value) triplets in, compressed-column storage
 * (jc / ir / pr, int32 / int32 / float64) out, duplicates summed in input
 * order (pr = ((+0.0 + v1) + v2) + ..., bit-exact with the reference).
 *
 * Reference interfaces this ABI replaces (file:line in the reference package
 * /root/reference/pkg/src/sparseasm):
 *   sa_assemble_async + sa_finish  <- serial.assemble_serial      serial.py:111-168
 *                                     parallel.assemble_parallel  parallel.py:361-389
 *                                     (and the kernel-module protocol they drive,
 *                                     _kernels.pyx:20-89 count_rows / build_rank /
 *                                     compress / accumulate / scatter)
 *   sa_host_upload / sa_host_dims /  <- __init__.assemble          __init__.py:36-46
 *   sa_host_assemble / sa_host_fetch    (host arrays in, host CSC out)
 *   sa_convert_indices             <- types._convert_index_array  types.py:121-138
 *                                     parallel.find_max_parallel  parallel.py:87-122
 *                                     _kernels.validate_chunk     _kernels.pyx:92-110
 *   sa_infer_dims                  <- AssemblyRequest.effective_dims (inferred) types.py:102-118
 *   sa_prune_zeros                 <- types.prune_explicit_zeros types.py:204-213
 *   sa_block_histogram             <- (new: the sampled column-block histogram that sets
 *                                     the multi-GPU rank boundaries)
 *   sa_partition                   <- (new: multi-GPU column-block sharding, SURVEY 8(e);
 *                                     the reference's threaded driver partitions by
 *                                     element range, parallel.py:28-35, 267-358)
 *
 * Conventions
 *   - Every call returns an sa_status (0 = SA_OK).  sa_last_error() gives a
 *     human-readable message for the last failure on that context.
 *   - One context per host thread; calls on one context are serialised on
 *     its CUDA stream (sa_set_stream may substitute the caller's stream).
 *   - "d_" pointers are device pointers (CUDA global memory), "h_" pointers
 *     host pointers (pinned memory gives full PCIe bandwidth; pageable works).
 *   - Indices are validated on the device.  Errors mirror the reference's
 *     exception types: SA_ERR_BAD_INDEX <-> errors.BadIndex (first bad
 *     position, rows checked before columns, types.py:161-162),
 *     SA_ERR_DIM_TOO_SMALL <-> errors.DimensionTooSmall (types.py:113-117).
 *   - nzmax is an allocation hint only (types.py:78-86): the caller passes
 *     the capacity of its ir/pr buffers; SA_ERR_CAPACITY if nnz exceeds it.
 */
#ifndef SPARSE_ASSEMBLY_H
#define SPARSE_ASSEMBLY_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sa_ctx sa_ctx;

typedef enum sa_status {
    SA_OK = 0,
    SA_ERR_CUDA = 1,           /* a CUDA runtime call failed                 */
    SA_ERR_BAD_INDEX = 2,      /* index < 1, non-integral, NaN/Inf, > 2^31-1 */
    SA_ERR_DIM_TOO_SMALL = 3,  /* explicit m/n cannot hold the indices       */
    SA_ERR_CAPACITY = 4,       /* nnz exceeds the caller's ir/pr capacity    */
    SA_ERR_INVALID_ARG = 5,    /* null pointer, negative size, bad dtype ... */
    SA_ERR_NOMEM = 6,          /* device or pinned-host allocation failed    */
    SA_ERR_INTERNAL = 7        /* device-side consistency check failed       */
} sa_status;

/* raw index dtypes accepted by sa_convert_indices */
enum { SA_DTYPE_INT32 = 0, SA_DTYPE_INT64 = 1, SA_DTYPE_FLOAT64 = 2 };

/* which array a SA_ERR_BAD_INDEX refers to */
enum { SA_WHICH_ROW = 0, SA_WHICH_COL = 1 };

/* context options (sa_set_option); value -1 = automatic (the default), 0 or 1
 * forces a pipeline variant.  They select between code paths that produce the
 * SAME bits (tests force each variant); none changes a result. */
enum {
    SA_OPT_FOLD_STAGED = 0,     /* fold outputs staged + k_tile_emit pass       */
    SA_OPT_SCATTER_STAGED = 1,  /* column scatter through shared-memory staging */
    SA_OPT_PATH = 2,            /* 0: column-cursor pipeline, 1: column-block radix
                                   path (sa_radix.cu), -1: chosen per input    */
    SA_OPT_RPASS_TMA = 3        /* radix partition passes with TMA-staged input
                                   (k_rpass_tma) or register loads (k_rpass)   */
};

/* ABI version (bumped on any signature change). */
int sa_version(void);

/* Create a context on CUDA device `device` (own non-blocking stream). */
int sa_create(int device, sa_ctx **out);
/* Destroy a context and free its device / pinned workspace. */
void sa_destroy(sa_ctx *ctx);
/* Run subsequent work on `stream` (a cudaStream_t; 0/NULL = the legacy
 * default stream).  A new context starts on its own non-blocking stream. */
int sa_set_stream(sa_ctx *ctx, void *stream);
/* Set a context option (SA_OPT_*) to -1 (automatic), 0 or 1.  Replaces no
 * reference interface: the reference has one code path per backend. */
int sa_set_option(sa_ctx *ctx, int option, int value);
/* Message describing the last failure on this context ("" if none). */
const char *sa_last_error(const sa_ctx *ctx);

/*
 * Validate and convert one raw index array on the device (types.py:121-138).
 * dtype SA_DTYPE_INT64: valid iff 1 <= x <= 2^31-1.  SA_DTYPE_FLOAT64: valid
 * iff x >= 1, integral, <= 2^31-1 (NaN/Inf invalid).  SA_DTYPE_INT32: valid
 * iff x >= 1 (d_out may alias d_raw).  Synchronous.  *first_bad receives the
 * first invalid position or -1; *max_out the maximum (0 for L == 0).
 */
int sa_convert_indices(sa_ctx *ctx, const void *d_raw, int dtype, int64_t L,
                       int32_t *d_out, int64_t *first_bad, int32_t *max_out);

/*
 * Dimension inference for int32 indices (types.py:102-118, 163-165).
 * Synchronous.  On SA_ERR_BAD_INDEX, *bad_pos / *bad_which name the first
 * invalid entry (rows before columns).
 */
int sa_infer_dims(sa_ctx *ctx, const int32_t *d_ii, const int32_t *d_jj, int64_t L,
                  int32_t *M, int32_t *N, int64_t *bad_pos, int *bad_which);

/*
 * Enqueue the whole assembly on the context stream; no host synchronisation.
 *   d_ii, d_jj : int32[L], 1-based (validated on device)
 *   d_s        : float64 values; s_stride 1 (vector) or 0 (scalar broadcast,
 *                folded as repeated adds exactly like the reference's np.full)
 *   M, N       : matrix dimensions (explicit or from sa_infer_dims)
 *   d_jc       : int32[N+1] output
 *   d_ir, d_pr : int32[cap], float64[cap] outputs (cap >= nnz; L always suffices)
 * Workspace is held by the context and reused across calls.
 */
int sa_assemble_async(sa_ctx *ctx, const int32_t *d_ii, const int32_t *d_jj,
                      const double *d_s, int64_t s_stride, int64_t L,
                      int32_t M, int32_t N,
                      int32_t *d_jc, int32_t *d_ir, double *d_pr, int64_t cap);

/*
 * The same pipeline over up to 3 input segments read in place and
 * concatenated in order (input positions, which order the duplicate fold,
 * run through the segments one after the other) -- the sharded path: a
 * rank's own chunk, in place, between the triplets received from lower and
 * from higher ranks.  Columns are j - col_lo; columns outside [1, N] are
 * another rank's and are skipped (the chunks were validated by
 * sa_partition).  Per segment: d_ii[g], d_jj[g] (int32), d_s[g] (float64,
 * s_stride[g] 0 or 1), len[g].
 */
int sa_assemble_segments_async(sa_ctx *ctx, int nseg, const int32_t *const *d_ii,
                               const int32_t *const *d_jj, const double *const *d_s,
                               const int64_t *s_stride, const int64_t *len, int32_t col_lo,
                               int32_t M, int32_t N, int32_t *d_jc, int32_t *d_ir, double *d_pr,
                               int64_t cap);

/*
 * Synchronise the stream and report the outcome of the last
 * sa_assemble_async: *nnz, and for SA_ERR_BAD_INDEX *bad_pos / *bad_which.
 */
int sa_finish(sa_ctx *ctx, int64_t *nnz, int64_t *bad_pos, int *bad_which);

/*
 * Device pointer to the int64 nnz of the last sa_assemble_async (valid until
 * the next call on this context); lets callers chain device work without a
 * host round trip.
 */
const int64_t *sa_device_nnz(sa_ctx *ctx);

/*
 * Host-buffer protocol (the reference-facing call, __init__.py:36-46: host
 * arrays in, a fresh host CSC out).  nnz is unknown until the device has
 * assembled, so -- as in the reference, which sizes ir/pr after Part 4
 * (serial.py:153-158) -- the caller allocates its outputs between steps:
 *   1. sa_host_upload   : enqueue host->device copies of the triplets in
 *                         chunks (pinned host memory gives full PCIe
 *                         bandwidth); the validation / maxima pass of each
 *                         chunk runs on a second stream as soon as the
 *                         chunk has landed, overlapped with the next copy
 *                         (types.py:121-138, 163-165 fused into the upload)
 *   2. sa_host_dims     : optional, M = max(i), N = max(j) or the first bad
 *                         index from that pass (sync; no further pass)
 *   3. sa_host_assemble : assemble the uploaded triplets (sync), -> nnz
 *   4. sa_host_fetch    : copy jc[N+1], ir[nnz], pr[nnz] to the host (sync)
 */
int sa_host_upload(sa_ctx *ctx, const int32_t *h_ii, const int32_t *h_jj, const double *h_s,
                   int64_t s_stride, int64_t L);
int sa_host_dims(sa_ctx *ctx, int32_t *M, int32_t *N, int64_t *bad_pos, int *bad_which);
int sa_host_assemble(sa_ctx *ctx, int32_t M, int32_t N, int64_t *nnz, int64_t *bad_pos,
                     int *bad_which);
int sa_host_fetch(sa_ctx *ctx, int32_t *h_jc, int32_t *h_ir, double *h_pr);

/*
 * Page-locked host buffers from a process-wide cache (size classes of powers
 * of two), for host outputs that the device->host copies fill at full link
 * bandwidth.  The process keeps at most 8 GB of released blocks for reuse and
 * hands out at most 16 GB at a time; sa_host_buffer returns NULL beyond that
 * or on failure (callers then use pageable memory).
 */
void *sa_host_buffer(uint64_t bytes);
void sa_host_buffer_release(void *ptr);

/*
 * Matlab-style post-pass on a device CSC (types.py:204-213): drop entries
 * stored as exactly 0.0 (either sign; NaN is kept), keep the order, recompact
 * jc.  d_jc_out[N+1], d_ir_out / d_pr_out (capacity nnz) must not alias the
 * inputs.  Synchronous; *nnz_out receives the pruned count.
 */
int sa_prune_zeros(sa_ctx *ctx, const int32_t *d_jc, const int32_t *d_ir, const double *d_pr,
                   int32_t N, int64_t nnz, int32_t *d_jc_out, int32_t *d_ir_out,
                   double *d_pr_out, int64_t *nnz_out);

/*
 * Sampled column-block histogram (multi-GPU rank boundaries): d_hist[b]
 * (nblocks <= 8192 entries, zeroed here) += step for every step-th triplet
 * whose column j falls in block b = (j-1) / bsize (clamped to [0, nblocks)).
 * Asynchronous on the context's stream.
 */
int sa_block_histogram(sa_ctx *ctx, const int32_t *d_jj, int64_t L, int64_t step, int32_t nblocks,
                       int64_t bsize, uint64_t *d_hist);

/*
 * Multi-GPU column-block sharding (one process per GPU).  sa_partition
 * groups a rank's triplets by destination rank -- the owner of the column,
 * h_bounds[r] <= j-1 < h_bounds[r+1] for r < world (<= 8) -- into the arrays
 * d_ii_out, d_jj_out (global columns), d_s_out (capacity L each):
 * destinations in rank order, input order inside each (stable).  The
 * triplets of rank `self` (>= 0) are counted but not written: they stay in
 * place and the rank's assembly reads them there
 * (sa_assemble_segments_async); self = -1 writes every destination.  The
 * chunk is validated on the way: SA_ERR_BAD_INDEX with *bad_pos
 * (chunk-local) / *bad_which, SA_ERR_DIM_TOO_SMALL for indices above the
 * global M / N.  Synchronous; h_counts[r] = triplets for rank r.
 */
int sa_partition(sa_ctx *ctx, const int32_t *d_ii, const int32_t *d_jj, const double *d_s,
                 int64_t s_stride, int64_t L, int32_t M, int32_t N, int32_t world, int32_t self,
                 const int32_t *h_bounds, int32_t *d_ii_out, int32_t *d_jj_out, double *d_s_out,
                 int64_t *h_counts, int64_t *bad_pos, int *bad_which);

/* Number of kernel launches enqueued by the last sa_assemble_async. */
int sa_last_launch_count(const sa_ctx *ctx);

/*
 * Per-kernel timing with CUDA events recorded on the launching stream
 * (profiling aid; off by default).  After an sa_assemble_async with timing
 * on, sa_last_kernel_times synchronises and writes up to `max` per-launch
 * durations (milliseconds) and static kernel names; returns the count.
 */
int sa_enable_timing(sa_ctx *ctx, int on);
int sa_last_kernel_times(sa_ctx *ctx, int max, float *ms, const char **names);

#ifdef __cplusplus
}
#endif

#endif /* SPARSE_ASSEMBLY_H */
