// sa_internal.cuh -- shared device helpers and launch declarations for the
// B200 sparse-assembly kernels (sm_100a).  Not part of the public ABI.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sa {

constexpr unsigned FULL = 0xffffffffu;

// Record space.  Columns with at most BIGCOL triplets ("small") are laid out
// in column order in [0, Lsmall); longer ("big") columns get their own space
// [Lsmall, L) and are folded by k_bigcol.  Column words carry BIGFLAG for big
// columns; the low 31 bits are an offset.
constexpr uint32_t BIGFLAG = 0x80000000u;
constexpr uint32_t POSMASK = 0x7fffffffu;
// k_col_scan: threads per CTA and consecutive columns per thread
constexpr int SCAN_NT = 256;
constexpr int SCAN_IPT = 8;  // multiple of 4 (16-byte vectors)
constexpr int SCAN_TILE = SCAN_NT * SCAN_IPT;

// Fold geometry (k_tile_fold).  Tile b owns the columns whose small-space
// start lies in [b*TILE, (b+1)*TILE); inside the CTA every thread owns a
// contiguous range of the tile's columns.  A tile holds at most
// TILE + BIGCOL - 1 small records.
constexpr int TILE = 1792;
constexpr int TILE_THREADS = 128;
constexpr int BIGCOL = 256;
constexpr int TCAP = TILE + BIGCOL;
// Columns of at most SHORT_COL triplets are sorted by one thread's register
// network in the fold; longer small columns go to its warp-level long pass.
constexpr int SHORT_COL = 24;

// One big column (k_col_scan appends, k_bigcol folds, k_tile_fold copies out).
struct BigCol {
    uint32_t col;     // column index
    uint32_t start;   // absolute record offset (Lsmall + big-space offset)
    uint32_t n;       // triplets
    uint32_t u;       // unique rows (after k_bigcol) | BIGFLAG if keys ended in buffer B
};

// The triplet input: up to MAXSEG segments read in place, concatenated in
// order (sa_assemble_segments_async; one segment for sa_assemble_async).
// A triplet's input position = pos0 of its segment + its index there.
constexpr int MAXSEG = 3;
struct Segs {
    const int32_t *ii[MAXSEG];
    const int32_t *jj[MAXSEG];
    const double *s[MAXSEG];
    int64_t stride[MAXSEG];   // value stride (0: one value broadcast)
    int64_t len[MAXSEG];
    int64_t pos0[MAXSEG];     // global position of the first triplet
    int64_t ch0[MAXSEG + 1];  // first CHUNK of each segment; ch0[nseg] = chunks in total
    int vec[MAXSEG];          // ii and jj 16-byte aligned
    int nseg;
    int col_lo;               // columns are j - col_lo
    int skip_foreign;         // columns outside [1, N] are another rank's: skipped, not errors
};

// Address of the value of input position p.
__device__ __forceinline__ const double *seg_value(const Segs &S, int64_t p) {
    const double *v = S.s[0] + (p - S.pos0[0]) * S.stride[0];
#pragma unroll
    for (int q = 1; q < MAXSEG; ++q)
        if (q < S.nseg && p >= S.pos0[q]) v = S.s[q] + (p - S.pos0[q]) * S.stride[q];
    return v;
}

// Device-side outcome of one assembly (zeroed / reset before every call).
struct ErrState {
    unsigned long long bad_i;   // first row index < 1 (or invalid raw value)
    unsigned long long bad_j;   // first column index < 1
    unsigned int over_m;        // a valid row index exceeded M
    unsigned int over_n;        // a valid column index exceeded N
    unsigned int max_i;         // maxima, for dimension inference
    unsigned int max_j;
    unsigned int cap_exceeded;  // nnz > caller capacity
    unsigned int internal;      // device consistency check failed
    long long nnz;              // written by the last tile
    unsigned int tile_ticket;   // dynamic tile counters (forward progress)
    unsigned int scan_ticket;
    unsigned int nbig;          // number of big columns
    unsigned int lsmall;        // triplets in small columns (small record space)
    unsigned int long_cols;     // some small column is long (> SHORT_COL): the fold's long pass runs
    // radix path (sa_radix.cu)
    unsigned int rbig_n;        // oversize sub-buckets listed by k_rbounds
    unsigned int rvalid;        // triplets with a valid column (partitioned)
};

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// x86 SSE `addsd acc, v` semantics, which the reference's compiled scatter
// (_kernels.pyx:82-89, `pr[k] += sr[i]`) obeys.  B200 add.f64 agrees except
// when both operands are NaN: it returns the second operand's payload while
// x86 keeps the first (probe: tools/probe/nanprobe.cu).  A NaN accumulator
// is already quiet (it came out of an add), so keeping it is exact.
__device__ __forceinline__ double fold_add(double acc, double v) {
    return (acc != acc) ? acc : __dadd_rn(acc, v);
}

// Ordered fold, from +0.0, of the n values (bit patterns) at v by one warp:
// the values are read 32 at a time (the next 32 in flight) and handed round
// by shuffles, every lane running the same chain of adds -- the chain is
// the floor of a long run of repeats.  Whole blocks of 32 use plain adds
// (fold_add's bits unless the sum turns NaN: NaN is sticky, so a non-NaN
// result met no NaN on the way; the block is redone by the rule otherwise),
// which keeps the rule's compare and select off the dependent chain.
__device__ __forceinline__ double warp_fold_run(const unsigned long long *v, int64_t n, int stride = 1) {
    const int lane = threadIdx.x & 31;
    double acc = 0.0;
    unsigned long long x = (lane < n) ? v[(int64_t)lane * stride] : 0ull;
    for (int64_t k0 = 0; k0 < n; k0 += 32) {
        const unsigned long long xn = (k0 + 32 + lane < n) ? v[(k0 + 32 + lane) * stride] : 0ull;
        if (n - k0 >= 32) {
            double t = acc;
#pragma unroll
            for (int j = 0; j < 32; ++j)
                t = __dadd_rn(t, __longlong_as_double((long long)__shfl_sync(0xffffffffu, x, j)));
            if (t != t) {
                t = acc;
                for (int j = 0; j < 32; ++j)
                    t = fold_add(t, __longlong_as_double((long long)__shfl_sync(0xffffffffu, x, j)));
            }
            acc = t;
        } else {
            const int cnt = (int)(n - k0);
            for (int j = 0; j < cnt; ++j)
                acc = fold_add(acc, __longlong_as_double((long long)__shfl_sync(0xffffffffu, x, j)));
        }
        x = xn;
    }
    return acc;
}

// ---- decoupled look-back (single-pass chained scan) ----------------------
// status word: bits 63:62 flag (0 empty, 1 aggregate, 2 inclusive prefix),
// bits 61:0 value.
constexpr unsigned long long LB_VALMASK = (1ull << 62) - 1;
// A status word carries its own payload (flag and value in one 64-bit
// store), and consumers read nothing else the producer wrote, so publishing
// needs no memory fence: a fence would only add ~0.5 us per chain hop.
// One status word per 128-byte line: the words of neighbouring tiles land in
// different L2 slices, so the polling of hundreds of CTAs does not queue on
// one slice.
constexpr int LB_STRIDE = 16;
__device__ __forceinline__ unsigned long long lb_pack(unsigned flag, unsigned long long v) {
    return (static_cast<unsigned long long>(flag) << 62) | v;
}

// Called by one full warp of tile `b`.  Publishes `agg`, returns the
// exclusive prefix of all tiles < b, and publishes the inclusive prefix.
__device__ __forceinline__ unsigned long long lookback_warp(
    unsigned long long *st, long long b, unsigned long long agg) {
    const int lane = threadIdx.x & 31;
    volatile unsigned long long *vst = st;
    if (b == 0) {
        if (lane == 0) {
            vst[(0) * LB_STRIDE] = lb_pack(2, agg);
        }
        return 0;
    }
    if (lane == 0) {
        vst[(b) * LB_STRIDE] = lb_pack(1, agg);
    }
    unsigned long long excl = 0;
    long long base = b - 1;
    while (true) {
        long long idx = base - lane;
        unsigned long long w = (idx >= 0) ? vst[(idx) * LB_STRIDE] : lb_pack(2, 0);
        unsigned flag = static_cast<unsigned>(w >> 62);
        if (__any_sync(FULL, flag == 0)) continue;  // predecessors not published yet
        unsigned pm = __ballot_sync(FULL, flag == 2);
        int stop = pm ? (__ffs(pm) - 1) : 31;
        unsigned long long v = (lane <= stop) ? (w & LB_VALMASK) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        excl += v;
        if (pm) break;
        base -= 32;
    }
    if (lane == 0) {
        vst[(b) * LB_STRIDE] = lb_pack(2, excl + agg);
    }
    return excl;
}

// Block-wide look-back: each round reads NT predecessor words at once (one
// per thread), so a CTA reaches the nearest inclusive prefix in one or two
// L2 round trips even when hundreds of predecessors are in flight.  All
// threads call it; returns the exclusive prefix of tile b.  s_red needs NT/32
// slots.  Ends with a barrier.
template <int NT>
__device__ __forceinline__ unsigned long long lookback_block(unsigned long long *st, long long b,
                                                             unsigned long long agg,
                                                             unsigned long long *s_red,
                                                             int *s_stop) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    volatile unsigned long long *vst = st;
    if (tid == 0) {
        vst[(b) * LB_STRIDE] = lb_pack(b == 0 ? 2 : 1, agg);
    }
    if (b == 0) return 0;
    unsigned long long excl = 0;
    long long base = b - 1;
    while (true) {
        const long long idx = base - tid;
        unsigned long long wd;
        do {
            wd = (idx >= 0) ? vst[(idx) * LB_STRIDE] : lb_pack(2, 0);
        } while ((wd >> 62) == 0);  // predecessor not published yet
        if (tid == 0) *s_stop = NT;
        __syncthreads();
        const unsigned inc = __ballot_sync(FULL, (wd >> 62) == 2);
        if (lane == 0 && inc) atomicMin(s_stop, w * 32 + __ffs(inc) - 1);
        __syncthreads();
        const int stop = *s_stop;
        unsigned long long v = (tid <= stop) ? (wd & LB_VALMASK) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        if (lane == 0) s_red[w] = v;
        __syncthreads();
        unsigned long long t = 0;
#pragma unroll
        for (int k = 0; k < NT / 32; ++k) t += s_red[k];
        excl += t;
        __syncthreads();  // s_red / s_stop reused next round
        if (stop < NT) break;
        base -= NT;
    }
    if (tid == 0) {
        vst[(b) * LB_STRIDE] = lb_pack(2, excl + agg);
    }
    return excl;
}

// ---- block scans ----------------------------------------------------------
// Exclusive sum over one value per thread; returns the exclusive prefix and
// the block total.  s_warp needs NT/32 slots.  Ends with a barrier.
template <int NT, typename T>
__device__ __forceinline__ T block_excl_sum(T v, T *s_warp, T &total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    if (w == 0) {
        T t = (lane < NT / 32) ? s_warp[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(FULL, t, o);
            if (lane >= o) t += y;
        }
        if (lane < NT / 32) s_warp[lane] = t;
    }
    __syncthreads();
    T wpre = w ? s_warp[w - 1] : T(0);
    total = s_warp[NT / 32 - 1];
    __syncthreads();
    return wpre + x - v;
}

// The same with one barrier: every warp scans the NT/32 warp totals itself.
// No trailing barrier: the caller must pass a barrier before s_warp is
// written again (and NT/32 <= 32).
template <int NT, typename T>
__device__ __forceinline__ T block_excl_sum1(T v, T *s_warp, T &total) {
    static_assert(NT / 32 <= 32, "one lane per warp total");
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    T t = (lane < NT / 32) ? s_warp[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(FULL, t, o);
        if (lane >= o) t += y;
    }
    total = __shfl_sync(FULL, t, NT / 32 - 1);
    const T winc = __shfl_sync(FULL, t, w);  // inclusive over warps 0..w
    const T wtot = __shfl_sync(FULL, x, 31);
    return winc - wtot + x - v;
}

// In-place exclusive sum over arr[0..n) in shared memory (n <= NT*IPT).
// Returns the total.  Each thread owns IPT consecutive entries.
template <int NT, int IPT, typename T>
__device__ __forceinline__ T smem_excl_scan(T *arr, int n, T *s_warp) {
    const int base = threadIdx.x * IPT;
    T loc[IPT];
    T sum = 0;
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
        loc[k] = (base + k < n) ? arr[base + k] : T(0);
        sum += loc[k];
    }
    T total;
    T pre = block_excl_sum<NT, T>(sum, s_warp, total);
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
        if (base + k < n) arr[base + k] = pre;
        pre += loc[k];
    }
    __syncthreads();
    return total;
}

// In-place inclusive max-scan over arr[0..n) (non-negative ints).
template <int NT, int IPT>
__device__ __forceinline__ void smem_incl_max(int *arr, int n, int *s_warp) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int base = threadIdx.x * IPT;
    int loc[IPT];
    int run = 0;
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
        int v = (base + k < n) ? arr[base + k] : 0;
        run = max(run, v);
        loc[k] = run;
    }
    int x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x = max(x, y);
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    if (w == 0) {
        int t = (lane < NT / 32) ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(FULL, t, o);
            if (lane >= o) t = max(t, y);
        }
        if (lane < NT / 32) s_warp[lane] = t;
    }
    __syncthreads();
    int wpre = w ? s_warp[w - 1] : 0;
    int tpre = __shfl_up_sync(FULL, x, 1);
    if (lane == 0) tpre = 0;
    int pre = max(wpre, tpre);
#pragma unroll
    for (int k = 0; k < IPT; ++k)
        if (base + k < n) arr[base + k] = max(pre, loc[k]);
    __syncthreads();
}

constexpr int BIG_NT = 1024;
constexpr int BIG_NW = BIG_NT / 32;

// One stable LSD radix pass (8-bit digit at `shift`) of n keys src -> dst by
// one CTA: every warp owns a contiguous segment; per-warp digit counts, one
// block scan over (digit, warp), then each warp places its segment in order
// (match.any ranks + a warp-private running counter per digit) -- no block
// barrier inside the loops.
__device__ __forceinline__ void big_radix_pass(const unsigned long long *src,
                                               unsigned long long *dst, int64_t n, int shift,
                                               uint32_t (*s_cnt)[256], uint32_t *s_warp) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const unsigned lt = lanemask_lt();
    for (int k = tid; k < BIG_NW * 256; k += BIG_NT) (&s_cnt[0][0])[k] = 0;
    __syncthreads();
    const int64_t lo = (int64_t)w * n / BIG_NW, hi = (int64_t)(w + 1) * n / BIG_NW;
    for (int64_t p = lo + lane; p < hi; p += 32) atomicAdd(&s_cnt[w][(src[p] >> shift) & 255], 1u);
    __syncthreads();
    {  // digit-major exclusive scan: thread t owns entries 8t .. 8t+7 of (digit, warp)
        uint32_t v[8], sum = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int q = 8 * tid + k;
            v[k] = s_cnt[q % BIG_NW][q / BIG_NW];
            sum += v[k];
        }
        uint32_t tot;
        uint32_t pre = block_excl_sum<BIG_NT, uint32_t>(sum, s_warp, tot);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int q = 8 * tid + k;
            s_cnt[q % BIG_NW][q / BIG_NW] = pre;
            pre += v[k];
        }
    }
    __syncthreads();
    for (int64_t b0 = lo; b0 < hi; b0 += 32) {
        const int64_t p = b0 + lane;
        const bool valid = p < hi;
        const unsigned long long key = valid ? src[p] : 0ull;
        const int d = valid ? (int)((key >> shift) & 255) : 256;
        const unsigned peers = __match_any_sync(FULL, d);
        const uint32_t base = valid ? s_cnt[w][d] : 0u;
        if (valid) dst[base + __popc(peers & lt)] = key;
        __syncwarp();
        if (valid && (peers & lt) == 0u) s_cnt[w][d] = base + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
}

// ---- programmatic dependent launch -------------------------------------------
// Every kernel of the assembly chain is launched with programmatic stream
// serialisation: it may start (smem set-up) while its predecessor drains,
// and waits at pdl_wait() before touching global memory the predecessor
// writes or reads.  pdl_trigger() lets the successor launch once every CTA
// of this grid has started.  Both are no-ops for a plain launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// cudaFuncAttributeMaxDynamicSharedMemorySize for `fn` on the CURRENT device
// (the attribute is per device): set once per (kernel, device), thread-safe.
cudaError_t ensure_smem_attr(const void *fn, int bytes);

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t stream, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---- launchers (sa_kernels.cu) ---------------------------------------------
struct Launch {
    cudaStream_t stream;
    int num_sms;
    int launches;  // incremented per kernel launch
    // context options (sa_set_option): -1 = automatic choice
    int fold_staged = -1;     // SA_OPT_FOLD_STAGED: staged fold outputs + k_tile_emit
    int scatter_staged = -1;  // SA_OPT_SCATTER_STAGED: k_scatter_staged
    int rpass_tma = -1;       // SA_OPT_RPASS_TMA: radix passes with TMA-staged input (k_rpass_tma)
};

cudaError_t launch_convert(Launch &lc, const void *raw, int dtype, int64_t L, int32_t *out,
                           ErrState *err);
cudaError_t launch_hist(Launch &lc, const int32_t *ii, const int32_t *jj, int64_t L,
                        int32_t M, int32_t N, uint32_t *cnt, ErrState *err, bool infer,
                        int64_t pos0 = 0);
cudaError_t launch_col_scan(Launch &lc, const uint32_t *cnt, uint32_t *sstart, uint32_t *cur,
                            int32_t N, int2 *tile_info, uint8_t *tile_big,
                            int64_t ntiles, BigCol *big_list, uint32_t *bigk,
                            unsigned long long *scan_state, uint2 *perm, ErrState *err,
                            int tile_sz);
cudaError_t launch_colcount(Launch &lc, const Segs &S, int32_t N, uint32_t *cnt, ErrState *err);
cudaError_t launch_scatter(Launch &lc, const Segs &S, int32_t M, int32_t N, uint32_t *cur,
                           uint2 *perm, ErrState *err);
cudaError_t launch_bigcol(Launch &lc, BigCol *big_list, const ErrState *err, int4 *rec,
                          const uint2 *perm, const Segs &S, int idx_bits, int passes);
cudaError_t launch_tile_fold(Launch &lc, const uint32_t *sstart, const int2 *tile_info,
                             const uint8_t *tile_big, int64_t ntiles, const int2 *entries,
                             const Segs &S, const int4 *rec,
                             const BigCol *big_list, const uint32_t *bigk,
                             unsigned long long *tile_state, int32_t N, int32_t *jc, int32_t *ir,
                             double *pr, int64_t cap, ErrState *err, int4 *stage,
                             int2 *tile_cnt);

// ---- radix path (sa_radix.cu) -------------------------------------------------
constexpr int RP_NT = 1024;                 // partition pass: threads per CTA (one CTA per SM)
constexpr int RP_NW = RP_NT / 32;
// (12: chunks of 12288 triplets, two TMA-staged halves of 6144 -- 192 KB of
// staging, 226 KB of shared memory per CTA, the most an SM has; longer digit
// runs per half and fewer per-half overheads than with 8: cfg4 passes 5.07 /
// 4.62 -> 4.43 / 4.08 ms; 10: 4.62 / 4.28)
#ifndef SA_RP_IPT
#define SA_RP_IPT 12
#endif
constexpr int RP_IPT = SA_RP_IPT;           // triplets per thread
constexpr int RP_CHUNK = RP_NT * RP_IPT;    // triplets per chunk (CTA)
constexpr int RP_MAXBITS = 9;               // digit bits per pass
constexpr int RP_MAXD = 1 << RP_MAXBITS;
constexpr int RP_MAXPASS = 4;
constexpr int RP_BLK = 64;                  // chunks per upsweep block
constexpr int RF_CAP = 4096;                // fold: largest sub-bucket held in shared memory
constexpr int RF_WMAX = 256;                // fold: columns per sub-bucket (2^w)

struct RadixPassArgs {
    const int32_t *ii_in, *jj_in;  // the first pass's input (the caller's arrays)
    const int2 *rc_in;             // the later passes' input: {row, col} pairs
    const double *s_in;
    int64_t s_stride;
    int32_t *ii_out, *jj_out;  // (SA_PAIRS == 0: output rows / columns of every pass but the last)
    double *s_out;             // output values
    int2 *rc_out;              // output {row, col} pairs (8 B each)
    int64_t L;
    int32_t M, N;
    int shift, bits;          // this pass's digit: (key >> shift) & (2^bits - 1) of the key
    int rbits;                // key = (col - 1) << rbits | (row - 1)
    const uint32_t *off;      // nchunk x RP_MAXD: global position of every chunk's digits
};

// SA_AOS = 1: the last pass writes 16-byte {row, col, value} records (one
// store per triplet, one write stream of 128-byte digit runs) and the fold's
// views rc / s of the record array step by RF_STRIDE = 2 elements per
// triplet.  Measured on cfg4: last pass 4.66 -> 4.30 ms, but the fold reads
// keys and values in separate phases and then pulls every line twice from
// L2: 6.13 -> 6.62 ms.  Off.
#ifndef SA_AOS
#define SA_AOS 0
#endif
constexpr int RF_STRIDE = SA_AOS ? 2 : 1;

struct RadixFoldArgs {
    const int2 *rc;          // partitioned triplets (sorted by sub-bucket, stable): {row, col} of
    const double *s;         // triplet k at rc[k * RF_STRIDE], its value at s[k * RF_STRIDE]
    const uint32_t *bnd;     // nsub + 1 sub-bucket starts
    const uint32_t *biglist; // oversize sub-buckets
    uint32_t *bigu;          // per oversize sub-bucket: results | BIGFLAG (keys in scrB)
    unsigned long long *scrA, *scrB;  // oversize scratch (L entries each)
    unsigned long long *lbf; // look-back words, nsub x LB_STRIDE
    unsigned tag;
    int z, rbits;            // sub-bucket s = the keys [s << z, (s + 1) << z), key as above
    int32_t N, nsub;
    int32_t nres;            // fold CTAs in flight (set by launch_rfold)
    int32_t *jc, *ir;
    double *pr;
    int64_t cap;
};

cudaError_t launch_rup(Launch &lc, bool first, const int32_t *ii, const int32_t *jj, const int2 *rc, int64_t L,
                       int32_t N,
                       int shift, int bits, int rbits, uint16_t *cnt, uint32_t *bsum, uint32_t *off,
                       ErrState *err);
int rup_cpb(int64_t nchunk, int num_sms);  // chunks per upsweep block
cudaError_t launch_rpass(Launch &lc, const RadixPassArgs &A, bool first, bool last, int nseg, ErrState *err);
cudaError_t launch_rbounds(Launch &lc, const int2 *rc, int z, int rbits, int32_t nsub, uint32_t *bnd,
                           uint32_t *biglist, ErrState *err);
cudaError_t launch_rbig(Launch &lc, const RadixFoldArgs &F, ErrState *err);
cudaError_t launch_rfold(Launch &lc, const RadixFoldArgs &F, ErrState *err);

cudaError_t launch_prune(Launch &lc, const int32_t *jc, const int32_t *ir, const double *pr,
                         int32_t N, int64_t nnz, int32_t *jc_out, int32_t *ir_out,
                         double *pr_out, unsigned long long *state, long long *nnz_out);
int64_t prune_tiles(int64_t nnz);
cudaError_t launch_partition(Launch &lc, const int32_t *ii, const int32_t *jj, const double *s,
                             int64_t s_stride, int64_t L, int world, int self, const int32_t *bounds,
                             int32_t M, int32_t *tile_cnt, int64_t *tile_off, int64_t *counts,
                             int32_t *out_i, int32_t *out_j, double *out_s, ErrState *err);
int64_t partition_tiles(int64_t L);
cudaError_t launch_block_hist(Launch &lc, const int32_t *jj, int64_t L, int64_t step, int nblocks,
                              int64_t bsize, unsigned long long *hist);

}  // namespace sa
