// sa_kernels.cu -- hand-written sm_100a kernels for sparse(i,j,s,m,n).
//
// Pipeline (one stream, no host round trip, programmatic dependent launch):
//   k_init          reset counters, look-back words, error state (sa_capi.cu)
//   k_colcount_win  column histogram + column-index validation: runs of equal
//                   columns per thread, a shared-memory window per 2048-triplet
//                   chunk, one global atomic per touched column and chunk
//   k_col_scan      single-pass decoupled-look-back exclusive scan of the column
//                   counts -> column cursors; the tile -> first-column map and
//                   the list of big columns
//   k_scatter       counting-sort scatter by column of 8-byte entries {row,
//                   input position} (shared-memory hash aggregation, one cursor
//                   reservation per column and chunk) + row validation
//   k_bigcol        columns longer than BIGCOL: LSD radix sort by (row, input
//                   position) in one 1024-thread CTA, ordered fold
//   k_tile_fold     (sa_tile.cu) per tile of columns: TMA entries, cp.async
//                   value gather, per-column sort by (row, position), fold from
//                   +0.0 in input order (bit-exact with the reference scatter,
//                   _kernels.pyx:82-89), decoupled look-back of the unique
//                   counts -> jc, ir, pr written once.
// Helpers: k_hist (dimension inference / validation-only path), k_convert
// (raw index arrays), k_prune (sa_prune.cu), the sharding partition
// (sa_shard.cu).
//
// Reference algorithm: serial.py:111-168 / _kernels.pyx:20-89 (row-first
// counting sort).  This pipeline is column-first; it produces the same CSC
// because both order entries by (column, row) and fold duplicates in
// ascending input order.

#include <cstdlib>
#include <mutex>
#include <set>
#include <utility>

#include "sa_internal.cuh"

namespace sa {

// ---------------------------------------------------------------------------
// index validation / conversion of raw (non-int32) index arrays
// ---------------------------------------------------------------------------
__global__ void k_convert(const void *__restrict__ raw, int dtype, int64_t L,
                          int32_t *__restrict__ out, ErrState *err) {
    unsigned mx = 0;
    unsigned long long bad = ~0ull;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < L; t += stride) {
        bool ok;
        int32_t v = 0;
        if (dtype == 1) {
            long long x = static_cast<const long long *>(raw)[t];
            ok = x >= 1 && x <= 2147483647LL;
            v = (int32_t)x;
        } else if (dtype == 2) {
            double x = static_cast<const double *>(raw)[t];
            ok = (x >= 1.0) && (x == ceil(x)) && (x <= 2147483647.0);
            v = ok ? (int32_t)x : 0;
        } else {
            int32_t x = static_cast<const int32_t *>(raw)[t];
            ok = x >= 1;
            v = x;
        }
        if (!ok) bad = min(bad, (unsigned long long)t);
        else {
            out[t] = v;
            mx = max(mx, (unsigned)v);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mx = max(mx, __shfl_xor_sync(FULL, mx, o));
        bad = min(bad, __shfl_xor_sync(FULL, bad, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (mx) atomicMax(&err->max_i, mx);
        if (bad != ~0ull) atomicMin(&err->bad_i, bad);
    }
}

cudaError_t launch_convert(Launch &lc, const void *raw, int dtype, int64_t L, int32_t *out,
                           ErrState *err) {
    if (L <= 0) return cudaSuccess;
    int64_t want = (L + 255) / 256;
    int grid = (int)std::min<int64_t>(want, (int64_t)lc.num_sms * 8);
    k_convert<<<grid, 256, 0, lc.stream>>>(raw, dtype, L, out, err);
    lc.launches++;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// k_hist: column histogram + validation.  infer != 0: inference mode
// (validation and maxima only).  Warp-aggregated: lanes holding the same
// column issue one atomic (FEM element order makes neighbours share columns).
// ---------------------------------------------------------------------------
struct HistAcc {
    unsigned long long bad_i = ~0ull, bad_j = ~0ull;
    unsigned maxi = 0, maxj = 0;
    unsigned over_m = 0, over_n = 0;
};

__device__ __forceinline__ void hist_one(int64_t t, int32_t i, int32_t j, bool live, int32_t M,
                                         int32_t N, uint32_t *__restrict__ cnt, HistAcc &a) {
    const bool bi = live && i < 1, bj = live && j < 1;
    if (bi) a.bad_i = min(a.bad_i, (unsigned long long)t);
    if (bj) a.bad_j = min(a.bad_j, (unsigned long long)t);
    const bool valid = live && !bi && !bj;
    if (valid) {
        a.maxi = max(a.maxi, (unsigned)i);
        a.maxj = max(a.maxj, (unsigned)j);
    }
    if (cnt == nullptr) return;  // inference mode (warp-uniform)
    const bool ok = valid && i <= M && j <= N;
    if (valid && !ok) {
        if (i > M) a.over_m = 1;
        if (j > N) a.over_n = 1;
    }
    const unsigned act = __ballot_sync(FULL, ok);
    if (ok) {
        const unsigned peers = __match_any_sync(act, j);
        const int leader = __ffs(peers) - 1;
        if ((threadIdx.x & 31) == leader) atomicAdd(&cnt[j - 1], (uint32_t)__popc(peers));
    }
}

__global__ void __launch_bounds__(256) k_hist(const int32_t *__restrict__ ii,
                                              const int32_t *__restrict__ jj, int64_t L,
                                              int32_t M, int32_t N, uint32_t *__restrict__ cnt,
                                              ErrState *err, int vec, int infer, int64_t pos0) {
    HistAcc a;
    if (infer) cnt = nullptr;
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t wbase0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
    int64_t tail0 = 0;
    if (vec) {
        const int64_t nq = L >> 2;
        const int4 *ii4 = reinterpret_cast<const int4 *>(ii);
        const int4 *jj4 = reinterpret_cast<const int4 *>(jj);
        for (int64_t qb = wbase0; qb < nq; qb += stride) {
            const int64_t q = qb + lane;
            const bool live = q < nq;
            int4 vi = make_int4(1, 1, 1, 1), vj = make_int4(1, 1, 1, 1);
            if (live) {
                vi = __ldg(ii4 + q);
                vj = __ldg(jj4 + q);
            }
            hist_one(4 * q + 0, vi.x, vj.x, live, M, N, cnt, a);
            hist_one(4 * q + 1, vi.y, vj.y, live, M, N, cnt, a);
            hist_one(4 * q + 2, vi.z, vj.z, live, M, N, cnt, a);
            hist_one(4 * q + 3, vi.w, vj.w, live, M, N, cnt, a);
        }
        tail0 = nq << 2;
    }
    for (int64_t tb = tail0 + wbase0; tb < L; tb += stride) {
        const int64_t t = tb + lane;
        const bool live = t < L;
        int32_t i = live ? ii[t] : 1, j = live ? jj[t] : 1;
        hist_one(t, i, j, live, M, N, cnt, a);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a.bad_i = min(a.bad_i, __shfl_xor_sync(FULL, a.bad_i, o));
        a.bad_j = min(a.bad_j, __shfl_xor_sync(FULL, a.bad_j, o));
        a.maxi = max(a.maxi, __shfl_xor_sync(FULL, a.maxi, o));
        a.maxj = max(a.maxj, __shfl_xor_sync(FULL, a.maxj, o));
        a.over_m |= __shfl_xor_sync(FULL, a.over_m, o);
        a.over_n |= __shfl_xor_sync(FULL, a.over_n, o);
    }
    if (lane == 0) {  // (positions of this array slice + pos0: global input positions)
        if (a.bad_i != ~0ull) atomicMin(&err->bad_i, a.bad_i + (unsigned long long)pos0);
        if (a.bad_j != ~0ull) atomicMin(&err->bad_j, a.bad_j + (unsigned long long)pos0);
        if (infer) {
            if (a.maxi) atomicMax(&err->max_i, a.maxi);
            if (a.maxj) atomicMax(&err->max_j, a.maxj);
        }
        if (a.over_m) err->over_m = 1;
        if (a.over_n) err->over_n = 1;
    }
}

static inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

cudaError_t launch_hist(Launch &lc, const int32_t *ii, const int32_t *jj, int64_t L, int32_t M,
                        int32_t N, uint32_t *cnt, ErrState *err, bool infer, int64_t pos0) {
    if (L <= 0) return cudaSuccess;
    const int vec = aligned16(ii) && aligned16(jj);
    int64_t want = ((vec ? (L >> 2) : L) + 255) / 256 + 1;
    int grid = (int)std::min<int64_t>(want, (int64_t)lc.num_sms * 8);
    k_hist<<<grid, 256, 0, lc.stream>>>(ii, jj, L, M, N, cnt, err, vec, infer ? 1 : 0, pos0);
    lc.launches++;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// k_col_scan: one pass over the column counts (decoupled look-back across
// CTAs, ticket-ordered for forward progress).  Two exclusive prefixes at once,
// packed (big << 31 | small): small columns (<= BIGCOL triplets) get offsets
// in the small record space, big columns in the big space.  Emits
//   sstart[c]     small-space start of column c (| BIGFLAG if big; a big
//                 column sits at the start of the next small column)
//   cur[c]        scatter cursor (small start, or big-space start | BIGFLAG)
//   tile_info[t]  {min{c : sstart(c) >= t*tile}, its sstart}, 0 <= t <= ntiles
//                 (tile = the call's tile size, TILE or smaller for small inputs)
//                 (the fold tile t owns the columns starting in its range)
//   tile_big[b]   tile b owns a big column
//   big_list[]    big columns {col, big-space start, n}; bigk[c] = list index
//   err->lsmall   size of the small space
// ---------------------------------------------------------------------------
constexpr unsigned long long SMALL_MASK = (1ull << 31) - 1;
#ifdef SA_TRACE
__device__ unsigned long long g_trace[1 << 16][4];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smid_() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
#define TRACE(b, k) if (threadIdx.x == 0 && (b) < (1 << 16)) g_trace[b][k] = gtime() | ((unsigned long long)smid_() << 54)
#else
#define TRACE(b, k)
#endif

// One column's contribution to the packed (big << 31 | small) prefix.
__device__ __forceinline__ unsigned long long scan_word(uint32_t n) {
    return (n > (uint32_t)BIGCOL) ? (((unsigned long long)n << 31) | 1ull) : n;
}

// Each thread owns SCAN_IPT = 8 consecutive columns: 16-byte loads of the
// counts, 16-byte stores of sstart / cur, so the kernel streams at HBM speed;
// small CTAs keep many of them resident per SM for memory parallelism.
// Tile index of small-space offset x for the runtime tile size d: the high
// half of x * ceil(2^64 / d), exact for x < 2^32 (the error x * (m/2^64 -
// 1/d) < 2^-32 stays below the distance 1/d to the next integer).
__device__ __forceinline__ int64_t tile_of(uint64_t x, uint64_t tmagic) {
    return (int64_t)__umul64hi(x, tmagic);
}

__global__ void __launch_bounds__(SCAN_NT) k_col_scan(const uint32_t *cnt,
                                                      uint32_t *__restrict__ sstart,
                                                      uint32_t *cur, int32_t N,
                                                      int2 *__restrict__ tile_info,
                                                      uint8_t *__restrict__ tile_big, int64_t ntiles,
                                                      BigCol *__restrict__ big_list,
                                                      uint32_t *__restrict__ bigk,
                                                      unsigned long long *scan_state,
                                                      uint2 *__restrict__ perm,
                                                      ErrState *err, uint64_t tmagic) {
    __shared__ unsigned long long s_warp[SCAN_NT / 32];
    __shared__ long long s_b;
    __shared__ unsigned long long s_excl;
    __shared__ long long s_tail;
    __shared__ int s_tot;
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x == 0) s_b = atomicAdd(&err->scan_ticket, 1u);
    __syncthreads();
    const long long b = s_b;
    TRACE(b, 0);
    const int64_t c0 = b * SCAN_TILE + (int64_t)threadIdx.x * SCAN_IPT;
    uint32_t loc[SCAN_IPT];
    if (c0 + SCAN_IPT <= N) {
#pragma unroll
        for (int v = 0; v < SCAN_IPT / 4; ++v) {
            const uint4 q = *reinterpret_cast<const uint4 *>(cnt + c0 + 4 * v);
            loc[4 * v] = q.x; loc[4 * v + 1] = q.y; loc[4 * v + 2] = q.z; loc[4 * v + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < SCAN_IPT; ++k) loc[k] = (c0 + k < N) ? cnt[c0 + k] : 0u;
    }
    unsigned long long sum = 0;
    bool long_col = false;
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k) {
        sum += scan_word(loc[k]);
        long_col |= loc[k] > (uint32_t)SHORT_COL && loc[k] <= (uint32_t)BIGCOL;
    }
    if (__any_sync(FULL, long_col) && (threadIdx.x & 31) == 0) err->long_cols = 1u;
    unsigned long long total;
    const unsigned long long pre = block_excl_sum<SCAN_NT, unsigned long long>(sum, s_warp, total);
    TRACE(b, 1);
    if (threadIdx.x < 32) {
        const unsigned long long e = lookback_warp(scan_state, b, total);
        if (threadIdx.x == 0) s_excl = e;
    }
    __syncthreads();
    TRACE(b, 2);
    const unsigned long long run0 = s_excl + pre;
    uint64_t small = run0 & SMALL_MASK;
    uint64_t bigp = run0 >> 31;
    uint32_t o_s[SCAN_IPT], o_c[SCAN_IPT];
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k) {
        const int64_t c = c0 + k;
        const uint32_t n = loc[k];
        const bool big = n > (uint32_t)BIGCOL;
        o_s[k] = (uint32_t)small | (big ? BIGFLAG : 0u);
        o_c[k] = big ? ((uint32_t)bigp | BIGFLAG) : (uint32_t)small;
        if (c < N) {
            if (big) {
                const unsigned slot = atomicAdd(&err->nbig, 1u);
                big_list[slot] = BigCol{(uint32_t)c, (uint32_t)bigp, n, 0u};
                bigk[c] = slot;
                perm[small] = make_uint2(0u, 0xffffffffu);  // placeholder slot: nothing to gather
                int64_t tb = tile_of(small, tmagic);
                if (tb > ntiles - 1) tb = ntiles - 1;
                tile_big[tb] = 1;
            }
            // fold tiles t with small < t*tile <= small + extent start at column c+1
            const uint32_t ext = big ? 1u : n;
            if (ext) {
                int64_t t = tile_of(small, tmagic) + 1;
                const int64_t last = min(tile_of(small + ext, tmagic), ntiles - 1);
                for (; t <= last; ++t) tile_info[t] = make_int2((int)(c + 1), (int)(small + ext));
            }
            if (c == N - 1) {
                const uint64_t tot_small = small + ext;
                err->lsmall = (unsigned)tot_small;
                sstart[N] = (uint32_t)tot_small;
                s_tail = (long long)tile_of(tot_small, tmagic) + 1;
                s_tot = (int)tot_small;
            }
        }
        if (big) {
            bigp += n;
            small += 1;
        } else {
            small += n;
        }
    }
    if (c0 + SCAN_IPT <= N) {
#pragma unroll
        for (int v = 0; v < SCAN_IPT / 4; ++v) {
            *reinterpret_cast<uint4 *>(sstart + c0 + 4 * v) =
                make_uint4(o_s[4 * v], o_s[4 * v + 1], o_s[4 * v + 2], o_s[4 * v + 3]);
            *reinterpret_cast<uint4 *>(cur + c0 + 4 * v) =
                make_uint4(o_c[4 * v], o_c[4 * v + 1], o_c[4 * v + 2], o_c[4 * v + 3]);
        }
    } else {
#pragma unroll
        for (int k = 0; k < SCAN_IPT; ++k)
            if (c0 + k < N) {
                sstart[c0 + k] = o_s[k];
                cur[c0 + k] = o_c[k];
            }
    }
    if (b == 0 && threadIdx.x == 0) tile_info[0] = make_int2(0, 0);
    TRACE(b, 3);
    // tiles past the small space (and past dropped invalid triplets) are
    // empty; the CTA holding column N-1 fills them together
    if (b == (long long)(N - 1) / SCAN_TILE) {
        __syncthreads();
        for (int64_t t = s_tail + threadIdx.x; t <= ntiles; t += SCAN_NT)
            tile_info[t] = make_int2(N, s_tot);
    }
}

cudaError_t launch_col_scan(Launch &lc, const uint32_t *cnt, uint32_t *sstart, uint32_t *cur,
                            int32_t N, int2 *tile_info, uint8_t *tile_big,
                            int64_t ntiles, BigCol *big_list, uint32_t *bigk,
                            unsigned long long *scan_state, uint2 *perm, ErrState *err,
                            int tile_sz) {
    if (N <= 0) return cudaSuccess;
    const uint64_t tmagic = ~0ull / (uint64_t)tile_sz + 1;  // ceil(2^64 / tile_sz)
    int grid = (int)((N + SCAN_TILE - 1) / SCAN_TILE);
    cudaError_t e = launch_pdl(k_col_scan, dim3(grid), dim3(SCAN_NT), 0, lc.stream, cnt, sstart, cur, N,
                               tile_info, tile_big, ntiles, big_list, bigk, scan_state, perm, err,
                               tmagic);
    if (e != cudaSuccess) return e;
    lc.launches++;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// The triplet input of an assembly: up to MAXSEG segments read in place, in
// order (one segment on one GPU; a rank's own chunk between the triplets
// received from lower and from higher ranks in the sharded path).  A CTA
// takes CHUNK consecutive triplets of one segment (CPT per thread, 16-byte
// vector loads, the next chunk in flight in registers).  The input position
// of a triplet -- its order for the duplicate fold -- is the segment's pos0
// plus its index.  Columns are j - col_lo; with skip_foreign, columns
// outside [1, N] belong to another rank and are skipped, not errors.
// ---------------------------------------------------------------------------
constexpr int AGG_NT = 256;
constexpr int CPT = 8;
constexpr int CHUNK = AGG_NT * CPT;
constexpr int HT = 2 * CHUNK;

struct SegChunk {  // one chunk of one segment
    const int32_t *ii, *jj;
    int64_t t0;    // segment-local index of the chunk's first triplet
    int64_t len;   // segment length
    int64_t pos0;  // global position of the segment's first triplet
    int vec;
};

__device__ __forceinline__ SegChunk seg_chunk(const Segs &S, int64_t ch) {
    int g = 0;
#pragma unroll
    for (int q = 1; q < MAXSEG; ++q)
        if (q < S.nseg && ch >= S.ch0[q]) g = q;
    SegChunk c{S.ii[0], S.jj[0], 0, S.len[0], S.pos0[0], S.vec[0]};
#pragma unroll
    for (int q = 1; q < MAXSEG; ++q)
        if (q == g) c = SegChunk{S.ii[q], S.jj[q], 0, S.len[q], S.pos0[q], S.vec[q]};
    c.t0 = (ch - (g == 0 ? 0 : (g == 1 ? S.ch0[1] : S.ch0[2]))) * CHUNK;
    return c;
}

// seg_chunk with a one-array fast path (the single-GPU call): the column
// pass spends ~15 % of its instructions on the segment search otherwise (in
// the scatter the same branch costs more than it saves)
__device__ __forceinline__ SegChunk seg_chunk_1(const Segs &S, int64_t ch) {
    if (S.nseg == 1) return SegChunk{S.ii[0], S.jj[0], ch * CHUNK, S.len[0], S.pos0[0], S.vec[0]};
    return seg_chunk(S, ch);
}

struct AggSmem {
    int key[HT];        // column + 1 (0 = empty)
    int ctr[HT];        // per column: triplets in the chunk, then the reserved cursor word
    int used[CHUNK];    // used slots
    int nused;
};

// Append `item` to a shared list when `take`; the lanes of the calling
// (possibly partial) warp share one atomic on the list counter.
__device__ __forceinline__ void list_push(int *list, int *count, bool take, int item) {
    const unsigned act = __activemask();
    const unsigned m = __ballot_sync(act, take);
    if (m == 0u) return;
    const int leader = __ffs(m) - 1;
    int base = 0;
    if ((int)(threadIdx.x & 31) == leader) base = atomicAdd(count, __popc(m));
    base = __shfl_sync(act, base, leader);
    if (take) list[base + __popc(m & lanemask_lt())] = item;
}

__device__ __forceinline__ int agg_insert(AggSmem &A, int col) {
    const int key = col + 1;
    unsigned h = ((unsigned)key * 0x9E3779B1u) >> (32 - 12);  // HT = 4096
    bool fresh = false;
    while (true) {
        const int old = atomicCAS(&A.key[h], 0, key);
        if (old == 0) {
            fresh = true;
            break;
        }
        if (old == key) break;
        h = (h + 1) & (HT - 1);
    }
    list_push(A.used, &A.nused, fresh, (int)h);
    return (int)h;
}

// load CPT consecutive int32 (vector path when aligned and complete)
__device__ __forceinline__ void load_run(const int32_t *__restrict__ p, int64_t t0, int64_t L,
                                         int vec, int (&v)[CPT], int fill) {
    if (vec && t0 + CPT <= L) {
        const int4 *q = reinterpret_cast<const int4 *>(p + t0);
#pragma unroll
        for (int k = 0; k < CPT / 4; ++k) {
            const int4 x = __ldg(q + k);
            v[4 * k] = x.x;
            v[4 * k + 1] = x.y;
            v[4 * k + 2] = x.z;
            v[4 * k + 3] = x.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < CPT; ++k) v[k] = (t0 + k < L) ? p[t0 + k] : fill;
    }
}

// Runs of equal columns inside a thread's CPT consecutive triplets (FEM
// element order emits each column 3-4 times in a row): only a run's head
// touches the shared-memory aggregation, with the run length.  Bit k of
// `heads` starts a run of valid triplets; a head's run length is the
// distance to the next set bit of `stops` (a new run, an invalid slot, or
// the end).
struct Runs {
    unsigned heads, stops;
};
__device__ __forceinline__ Runs run_masks(const int (&j)[CPT], unsigned vmask) {
    unsigned eq = 0;
#pragma unroll
    for (int k = 1; k < CPT; ++k)
        if (j[k] == j[k - 1]) eq |= 1u << k;
    eq &= vmask & (vmask << 1);
    return Runs{vmask & ~eq, ~eq | (1u << CPT)};
}
__device__ __forceinline__ int run_len(const Runs &r, int k) { return __ffs(r.stops >> (k + 1)); }

// Column validity of a thread's run (relabelled columns): one min/max test,
// per-slot checks only when something is off.  Out-of-range columns are
// errors (first bad position, over_n) unless skip_foreign.
__device__ __forceinline__ unsigned column_mask(const int (&j)[CPT], int64_t t0, int64_t len,
                                               int64_t pos0, int32_t N, bool skip_foreign,
                                               unsigned long long &bad, unsigned &over) {
    int lo = j[0], hi = j[0];
#pragma unroll
    for (int k = 1; k < CPT; ++k) {
        lo = min(lo, j[k]);
        hi = max(hi, j[k]);
    }
    if (lo >= 1 && hi <= N && t0 + CPT <= len) return (1u << CPT) - 1;
    unsigned vmask = 0;
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const bool live = t0 + k < len;
        if (!skip_foreign) {
            if (live && j[k] < 1) bad = min(bad, (unsigned long long)(pos0 + t0 + k));
            if (live && j[k] > N) over = 1;
        }
        if (live && j[k] >= 1 && j[k] <= N) vmask |= 1u << k;
    }
    return vmask;
}

// ---------------------------------------------------------------------------
// k_colcount_win: column histogram + column-index validation.  Each CTA
// takes a contiguous range of chunks (element-ordered input keeps the
// range's columns within a few mesh rows) and counts runs into a directly
// indexed shared-memory window of WB columns with non-returning shared adds.
// The window starts just behind the range's first column and is flushed to
// global memory (the touched bin range only: one global atomic per touched
// column) at the end of the range, or when a chunk's first column has left
// the window's first half -- at most every RECENTER chunks, so shuffled
// input does not flush every chunk.  Columns outside the window go to
// global memory directly.
// ---------------------------------------------------------------------------
constexpr int WB = 8192;
constexpr int WBACK = 512;    // window bins behind the first column
constexpr int RECENTER = 4;   // chunks between window moves, at least

struct WinSmem {
    uint32_t bin[WB];  // per window column: triplets of the CTA's range
    int lo, hi;        // touched bin range
};

// Window bins [lo, hi] touched since the last flush -> global counts; the
// bins are zeroed and the touched range reset.  Called by the whole CTA.
__device__ __forceinline__ void flush_window(WinSmem &W, int &blo, int &bhi, int cb,
                                             uint32_t *__restrict__ cnt) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        blo = min(blo, __shfl_xor_sync(FULL, blo, o));
        bhi = max(bhi, __shfl_xor_sync(FULL, bhi, o));
    }
    if ((threadIdx.x & 31) == 0 && bhi >= 0) {
        atomicMin(&W.lo, blo);
        atomicMax(&W.hi, bhi);
    }
    __syncthreads();
    const int lo = W.lo, hi = W.hi;
    for (int b = lo + (int)threadIdx.x; b <= hi; b += AGG_NT) {
        const uint32_t v = W.bin[b];
        if (v) {
            atomicAdd(&cnt[cb + b], v);
            W.bin[b] = 0;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        W.lo = WB;
        W.hi = -1;
    }
    __syncthreads();
    blo = WB;
    bhi = -1;
}

__global__ void __launch_bounds__(AGG_NT) k_colcount_win(Segs S, int32_t N,
                                                         uint32_t *__restrict__ cnt,
                                                         ErrState *err) {
    __shared__ WinSmem W;
    const int tid = threadIdx.x;
    for (int k = tid; k < WB; k += AGG_NT) W.bin[k] = 0;
    if (tid == 0) {
        W.lo = WB;
        W.hi = -1;
    }
    __syncthreads();
    pdl_wait();
    pdl_trigger();
    unsigned long long bad = ~0ull;
    unsigned over = 0;
    const int64_t nchunk = S.ch0[S.nseg];
    const bool skip = S.skip_foreign != 0;
    const int64_t per = (nchunk + gridDim.x - 1) / gridDim.x;
    const int64_t c_begin = (int64_t)blockIdx.x * per, c_end = min(nchunk, c_begin + per);
    int blo = WB, bhi = -1;
    int cb = 0;  // window base (column index of bin 0)
    int64_t moved = c_begin;
    int jn[CPT], fn = 0;  // the next chunk's columns and first column, in flight
    if (c_begin < c_end) {
        const SegChunk c = seg_chunk_1(S, c_begin);
        fn = __ldg(c.jj + c.t0);
        cb = fn - S.col_lo - 1 - WBACK;  // the range runs forward in the mesh
        load_run(c.jj, c.t0 + (int64_t)tid * CPT, c.len, c.vec, jn, 0x7fffffff);
    }
    for (int64_t ch = c_begin; ch < c_end; ++ch) {
        const SegChunk c = seg_chunk_1(S, ch);
        const int64_t t0 = c.t0 + (int64_t)tid * CPT;
        const int first = fn - S.col_lo - 1;
        if (ch - moved >= RECENTER && (first < cb || first >= cb + WB / 2)) {  // CTA-uniform
            flush_window(W, blo, bhi, cb, cnt);
            cb = first - WBACK;
            moved = ch;
        }
        int j[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) j[k] = jn[k] - S.col_lo;
        if (ch + 1 < c_end) {  // prefetch the next chunk while this one is counted
            const SegChunk cn = seg_chunk_1(S, ch + 1);
            fn = __ldg(cn.jj + cn.t0);
            load_run(cn.jj, cn.t0 + (int64_t)tid * CPT, cn.len, cn.vec, jn, 0x7fffffff);
        }
        const unsigned vmask = column_mask(j, t0, c.len, c.pos0, N, skip, bad, over);
        const Runs R = run_masks(j, vmask);
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            if (R.heads & (1u << k)) {
                const int len = run_len(R, k);
                const unsigned b = (unsigned)(j[k] - 1 - cb);
                if (b < (unsigned)WB) {
                    atomicAdd(&W.bin[b], (uint32_t)len);
                    blo = min(blo, (int)b);
                    bhi = max(bhi, (int)b);
                } else {
                    atomicAdd(&cnt[j[k] - 1], (uint32_t)len);
                }
            }
        }
    }
    flush_window(W, blo, bhi, cb, cnt);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        bad = min(bad, __shfl_xor_sync(FULL, bad, o));
        over |= __shfl_xor_sync(FULL, over, o);
    }
    if ((tid & 31) == 0) {
        if (bad != ~0ull) atomicMin(&err->bad_j, bad);
        if (over) err->over_n = 1;
    }
}

cudaError_t ensure_smem_attr(const void *fn, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(mu);
    if (done.count({fn, dev})) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.insert({fn, dev});
    return e;
}

constexpr int COLCOUNT_CTAS = 5;  // resident CTAs per SM of the column pass

cudaError_t launch_colcount(Launch &lc, const Segs &S, int32_t N, uint32_t *cnt, ErrState *err) {
    const int64_t nchunk = S.ch0[S.nseg];
    if (nchunk <= 0) return cudaSuccess;
    // at least the resident CTAs; large inputs: about 32 chunks per CTA
    // (cfg5 1.84 -> 1.62 ms with 16x the resident CTAs; cfg2 slower with more)
    const int64_t grid = std::min<int64_t>(nchunk, std::max<int64_t>((int64_t)lc.num_sms * COLCOUNT_CTAS, nchunk / 32));
    cudaError_t e = launch_pdl(k_colcount_win, dim3((unsigned)grid), dim3(AGG_NT), 0, lc.stream, S, N, cnt, err);
    lc.launches++;
    return e;
}

// ---------------------------------------------------------------------------
// k_scatter: counting-sort scatter by column of 8-byte entries {row, input
// position} (the fold gathers the values by position, so the 8-byte values
// are read once, by the fold).  Per chunk: (1) each column run gets
// chunk-local slots from a shared-memory hash counter, (2) one global
// atomicAdd per distinct column reserves the chunk's slots on the column
// cursor, (3) entries are written.  Row indices are validated here for every
// triplet (first bad position, rows above M).  The slot order inside a
// column is arbitrary; the fold restores input order from the position.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(AGG_NT) k_scatter(Segs S, int32_t M, int32_t N,
                                                    uint32_t *__restrict__ cur,
                                                    uint2 *__restrict__ perm, ErrState *err) {
    __shared__ AggSmem A;
    const int tid = threadIdx.x;
    for (int k = tid; k < HT; k += AGG_NT) {
        A.key[k] = 0;
        A.ctr[k] = 0;
    }
    if (tid == 0) A.nused = 0;
    __syncthreads();
    pdl_wait();
    pdl_trigger();
    const uint32_t lsmall = err->lsmall;
    unsigned long long bad = ~0ull, badj = ~0ull;
    unsigned over = 0, overj = 0;
    const int64_t nchunk = S.ch0[S.nseg];
    const bool skip = S.skip_foreign != 0;
    int in_[CPT], jn[CPT];
    if ((int64_t)blockIdx.x < nchunk) {
        const SegChunk c = seg_chunk(S, blockIdx.x);
        const int64_t t0 = c.t0 + (int64_t)tid * CPT;
        load_run(c.ii, t0, c.len, c.vec, in_, 1);
        load_run(c.jj, t0, c.len, c.vec, jn, 0);
    }
    for (int64_t ch = blockIdx.x; ch < nchunk; ch += gridDim.x) {
        const SegChunk c = seg_chunk(S, ch);
        const int64_t t0 = c.t0 + (int64_t)tid * CPT;
        int i[CPT], j[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            i[k] = in_[k];
            j[k] = jn[k] - S.col_lo;
        }
        if (ch + gridDim.x < nchunk) {  // next chunk in flight
            const SegChunk cn = seg_chunk(S, ch + gridDim.x);
            const int64_t t1 = cn.t0 + (int64_t)tid * CPT;
            load_run(cn.ii, t1, cn.len, cn.vec, in_, 1);
            load_run(cn.jj, t1, cn.len, cn.vec, jn, 0);
        }
        {  // rows: one min/max test, per-slot checks only when needed
            int ilo = i[0], ihi = i[0];
#pragma unroll
            for (int k = 1; k < CPT; ++k) {
                ilo = min(ilo, i[k]);
                ihi = max(ihi, i[k]);
            }
            if (ilo < 1 || ihi > M || t0 + CPT > c.len) {
#pragma unroll
                for (int k = 0; k < CPT; ++k) {
                    const bool live = t0 + k < c.len;
                    if (live && i[k] < 1) bad = min(bad, (unsigned long long)(c.pos0 + t0 + k));
                    if (live && i[k] > M) over = 1;
                }
            }
        }
        const unsigned vmask = column_mask(j, t0, c.len, c.pos0, N, true, badj, overj);
        const Runs R = run_masks(j, vmask);
        int hk[CPT], rk[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            hk[k] = -1;
            rk[k] = 0;
            if (R.heads & (1u << k)) {
                hk[k] = agg_insert(A, j[k] - 1);
                rk[k] = atomicAdd(&A.ctr[hk[k]], run_len(R, k));
            } else if (vmask & (1u << k)) {  // continues the run of slot k-1
                hk[k] = hk[k > 0 ? k - 1 : 0];
                rk[k] = rk[k > 0 ? k - 1 : 0] + 1;
            }
        }
        __syncthreads();
        const int nu = A.nused;
        for (int e = tid; e < nu; e += AGG_NT) {
            const int h = A.used[e];
            A.ctr[h] = (int)atomicAdd(&cur[A.key[h] - 1], (uint32_t)A.ctr[h]);
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            if (hk[k] < 0) continue;
            const uint32_t bw = (uint32_t)A.ctr[hk[k]];
            const uint32_t pos = (bw & POSMASK) + ((bw & BIGFLAG) ? lsmall : 0u) + (uint32_t)rk[k];
            perm[pos] = make_uint2((uint32_t)i[k], (uint32_t)(c.pos0 + t0 + k));
        }
        __syncthreads();
        for (int e = tid; e < nu; e += AGG_NT) {
            const int h = A.used[e];
            A.key[h] = 0;
            A.ctr[h] = 0;
        }
        if (tid == 0) A.nused = 0;
        __syncthreads();
    }
    (void)skip;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        bad = min(bad, __shfl_xor_sync(FULL, bad, o));
        over |= __shfl_xor_sync(FULL, over, o);
    }
    if ((tid & 31) == 0) {
        if (bad != ~0ull) atomicMin(&err->bad_i, bad);
        if (over) err->over_m = 1;
    }
}

// Staged variant (chosen for N > 4M columns; SA_OPT_SCATTER_STAGED forces
// either): 128-thread CTAs on half chunks (1024 triplets); after the
// reservation every entry is first placed in
// shared memory grouped by column (each column's run of the half chunk is
// contiguous there), then copied out so that consecutive lanes write
// consecutive slots of one column.
constexpr int SNT = 128;
constexpr int SCH = SNT * CPT;   // 1024 triplets per half chunk
constexpr int SHT = 2 * SCH;     // hash slots
struct StgSmem {
    int key[SHT];       // column + 1 (0 = empty); after the reservation: staging base
    int ctr[SHT];       // triplets of the column in the half chunk, then the cursor word
    int used[SCH];
    uint2 ent[SCH];     // staged entries {row, position}
    uint32_t dst[SCH];  // their slots
    int nused;
    int top;
};

__device__ __forceinline__ int stg_insert(StgSmem &A, int col) {
    const int key = col + 1;
    unsigned h = ((unsigned)key * 0x9E3779B1u) >> (32 - 11);  // SHT = 2048
    bool fresh = false;
    while (true) {
        const int old = atomicCAS(&A.key[h], 0, key);
        if (old == 0) {
            fresh = true;
            break;
        }
        if (old == key) break;
        h = (h + 1) & (SHT - 1);
    }
    list_push(A.used, &A.nused, fresh, (int)h);
    return (int)h;
}

__global__ void __launch_bounds__(SNT) k_scatter_staged(Segs S, int32_t M, int32_t N,
                                                        uint32_t *__restrict__ cur,
                                                        uint2 *__restrict__ perm, ErrState *err) {
    __shared__ StgSmem A;
    const int tid = threadIdx.x;
    for (int k = tid; k < SHT; k += SNT) {
        A.key[k] = 0;
        A.ctr[k] = 0;
    }
    if (tid == 0) {
        A.nused = 0;
        A.top = 0;
    }
    __syncthreads();
    pdl_wait();
    pdl_trigger();
    const uint32_t lsmall = err->lsmall;
    unsigned long long bad = ~0ull, badj = ~0ull;
    unsigned over = 0, overj = 0;
    const int64_t nh = 2 * S.ch0[S.nseg];
    int in_[CPT], jn[CPT];
    auto prefetch = [&](int64_t hc) {
        const SegChunk c = seg_chunk(S, hc >> 1);
        const int64_t t = c.t0 + (hc & 1) * SCH + (int64_t)tid * CPT;
        load_run(c.ii, t, c.len, c.vec, in_, 1);
        load_run(c.jj, t, c.len, c.vec, jn, 0);
    };
    if ((int64_t)blockIdx.x < nh) prefetch(blockIdx.x);
    for (int64_t hc = blockIdx.x; hc < nh; hc += gridDim.x) {
        const SegChunk c = seg_chunk(S, hc >> 1);
        const int64_t t0 = c.t0 + (hc & 1) * SCH + (int64_t)tid * CPT;
        int i[CPT], j[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            i[k] = in_[k];
            j[k] = jn[k] - S.col_lo;
        }
        if (hc + gridDim.x < nh) prefetch(hc + gridDim.x);
        {
            int ilo = i[0], ihi = i[0];
#pragma unroll
            for (int k = 1; k < CPT; ++k) {
                ilo = min(ilo, i[k]);
                ihi = max(ihi, i[k]);
            }
            if (ilo < 1 || ihi > M || t0 + CPT > c.len) {
#pragma unroll
                for (int k = 0; k < CPT; ++k) {
                    const bool live = t0 + k < c.len;
                    if (live && i[k] < 1) bad = min(bad, (unsigned long long)(c.pos0 + t0 + k));
                    if (live && i[k] > M) over = 1;
                }
            }
        }
        const unsigned vmask = column_mask(j, t0, c.len, c.pos0, N, true, badj, overj);
        const Runs R = run_masks(j, vmask);
        int hk[CPT], rk[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            hk[k] = -1;
            rk[k] = 0;
            if (R.heads & (1u << k)) {
                hk[k] = stg_insert(A, j[k] - 1);
                rk[k] = atomicAdd(&A.ctr[hk[k]], run_len(R, k));
            } else if (vmask & (1u << k)) {
                hk[k] = hk[k > 0 ? k - 1 : 0];
                rk[k] = rk[k > 0 ? k - 1 : 0] + 1;
            }
        }
        __syncthreads();
        const int nu = A.nused;
        for (int e = tid; e < nu; e += SNT) {
            const int h = A.used[e];
            const int cnt = A.ctr[h];
            A.ctr[h] = (int)atomicAdd(&cur[A.key[h] - 1], (uint32_t)cnt);
            A.key[h] = atomicAdd(&A.top, cnt);  // the column's run in the staging area
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            if (hk[k] < 0) continue;
            const uint32_t bw = (uint32_t)A.ctr[hk[k]];
            const int x = A.key[hk[k]] + rk[k];
            A.ent[x] = make_uint2((uint32_t)i[k], (uint32_t)(c.pos0 + t0 + k));
            A.dst[x] = (bw & POSMASK) + ((bw & BIGFLAG) ? lsmall : 0u) + (uint32_t)rk[k];
        }
        __syncthreads();
        const int nst = A.top;
        for (int x = tid; x < nst; x += SNT) perm[A.dst[x]] = A.ent[x];
        __syncthreads();
        for (int e = tid; e < nu; e += SNT) {
            const int h = A.used[e];
            A.key[h] = 0;
            A.ctr[h] = 0;
        }
        if (tid == 0) {
            A.nused = 0;
            A.top = 0;
        }
        __syncthreads();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        bad = min(bad, __shfl_xor_sync(FULL, bad, o));
        over |= __shfl_xor_sync(FULL, over, o);
    }
    if ((tid & 31) == 0) {
        if (bad != ~0ull) atomicMin(&err->bad_i, bad);
        if (over) err->over_m = 1;
    }
}

// Staged writes pay off when the column cursors (4 N bytes) and the columns'
// slot regions no longer stay in L2 between the chunks that fill them (cfg5,
// N = 6.4e7: 14.3 -> 6.7 ms with its grid below; a rank's cfg5 block at 8
// GPUs, N = 8e6: 2.92 -> 2.48 ms for its local assembly); with L2-resident
// cursors (cfg2 / cfg3, N = 1e6) the plain scatter is faster (109 vs 166 us
// on cfg2, 459 vs 619 us on cfg3).  The context option
// SA_OPT_SCATTER_STAGED overrides the choice (tests force both variants).
static bool scatter_staged(const Launch &lc, int32_t N) {
    return lc.scatter_staged >= 0 ? lc.scatter_staged == 1 : N > (4 << 20);
}

cudaError_t launch_scatter(Launch &lc, const Segs &S, int32_t M, int32_t N, uint32_t *cur,
                           uint2 *perm, ErrState *err) {
    const int64_t nchunk = S.ch0[S.nseg];
    if (nchunk <= 0) return cudaSuccess;
    cudaError_t e;
    if (scatter_staged(lc, N)) {
        // many short-lived CTAs, about 16 half chunks each (cfg5: 10.6 ms with
        // the 7 resident CTAs per SM walking all chunks, 6.6 ms like this)
        const int64_t grid = std::min<int64_t>(2 * nchunk, std::max<int64_t>((int64_t)lc.num_sms * 7, 2 * nchunk / 16));
        e = launch_pdl(k_scatter_staged, dim3((unsigned)grid), dim3(SNT), 0, lc.stream, S, M, N, cur, perm, err);
    } else {
        const int64_t grid = std::min<int64_t>(nchunk, (int64_t)lc.num_sms * 4);
        e = launch_pdl(k_scatter, dim3((unsigned)grid), dim3(AGG_NT), 0, lc.stream, S, M, N, cur, perm, err);
    }
    lc.launches++;
    return e;
}

// ---------------------------------------------------------------------------
// k_bigcol: columns longer than BIGCOL (grid-stride over the device-side
// list).  Results: row-1 in the key buffer, value bits in the other buffer,
// at index = run number; bigu[c] = runs | (BIGFLAG if keys ended in buffer
// B).  The column's two 8-byte buffers A|B are its 16-byte slots of the big
// scratch.  Two paths by length:
//  * medium (n <= MED_CAP): one 256-thread quarter of the CTA per column
//    (named barrier per quarter), entirely in shared memory: keys
//    (row-1) << idx_bits | input position, bitonic sort, values gathered by
//    position, each run of equal rows folded from +0.0 in position order by
//    the thread owning its head, heads compacted by a quarter-wide scan;
//  * long: the whole CTA, keys in A|B, stable LSD radix passes (8-bit
//    digits, warp match + per-warp digit counts), values gathered into the
//    other buffer, runs folded and compacted in place.
// ---------------------------------------------------------------------------
constexpr int MED_NT = 256;                 // threads per medium-column quarter
constexpr int MED_Q = BIG_NT / MED_NT;      // quarters per CTA
constexpr int MED_CAP = 1024;               // longest medium column
constexpr size_t BIG_DSMEM = (size_t)MED_Q * 2 * MED_CAP * sizeof(unsigned long long);

__device__ __forceinline__ void quarter_sync(int q) {
    asm volatile("bar.sync %0, %1;" ::"r"(q + 1), "n"(MED_NT) : "memory");
}

// One medium column (n <= MED_CAP) by quarter q (threads qt = 0..MED_NT-1).
__device__ __forceinline__ void med_column(BigCol *bcp, uint32_t st, int n, unsigned long long *A,
                                           const uint2 *__restrict__ perm, const Segs &S,
                                           int idx_bits, unsigned long long *K,
                                           unsigned long long *V, uint32_t *s_qw, int q, int qt) {
    const unsigned long long idx_mask = (1ull << idx_bits) - 1;
    int np2 = 32;
    while (np2 < n) np2 <<= 1;
    for (int p = qt; p < np2; p += MED_NT) {
        unsigned long long key = ~0ull;
        if (p < n) {
            const uint2 e = perm[st + p];
            key = ((unsigned long long)(e.x - 1u) << idx_bits) | e.y;
        }
        K[p] = key;
    }
    quarter_sync(q);
    for (int k = 2; k <= np2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int t = qt; t < (np2 >> 1); t += MED_NT) {
                const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
                const unsigned long long a = K[i], b = K[i + j];
                if ((a > b) == ((i & k) == 0)) {
                    K[i] = b;
                    K[i + j] = a;
                }
            }
            quarter_sync(q);
        }
    }
    for (int p = qt; p < n; p += MED_NT)
        V[p] = (unsigned long long)__double_as_longlong(*seg_value(S, (int64_t)(K[p] & idx_mask)));
    quarter_sync(q);
    // thread qt owns entries [4 qt, 4 qt + 4) (MED_CAP = 4 * MED_NT)
    constexpr int PER = MED_CAP / MED_NT;
    const int p0 = PER * qt;
    bool head[PER];
    uint32_t cnt = 0;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int p = p0 + u;
        head[u] = p < n && (p == 0 || (K[p] >> idx_bits) != (K[p - 1] >> idx_bits));
        cnt += head[u];
    }
    // quarter-wide exclusive scan of the head counts
    const int lane = qt & 31, w = qt >> 5;
    uint32_t incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, incl, d);
        if (lane >= d) incl += y;
    }
    if (lane == 31) s_qw[w] = incl;
    quarter_sync(q);
    uint32_t run = incl - cnt;
    for (int k = 0; k < w; ++k) run += s_qw[k];
    unsigned long long *B = A + n;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        if (!head[u]) continue;
        const int p = p0 + u;
        const unsigned long long row = K[p] >> idx_bits;
        double acc = fold_add(0.0, __longlong_as_double((long long)V[p]));
        for (int r = p + 1; r < n && (K[r] >> idx_bits) == row; ++r)
            acc = fold_add(acc, __longlong_as_double((long long)V[r]));
        A[run] = row;
        B[run] = (unsigned long long)__double_as_longlong(acc);
        ++run;
    }
    if (qt == MED_NT - 1) {
        bcp->start = st;  // absolute from here on
        bcp->u = run;     // keys in A
    }
    quarter_sync(q);  // K, V and s_qw are free for the next column
}

constexpr int BIGC_LONGRUN = 256;  // runs of equal rows longer than this are folded by a warp
constexpr int BIGC_NLONG = 256;    // listed long runs per column (more: walked by their thread)
__global__ void __launch_bounds__(BIG_NT, 2) k_bigcol(BigCol *__restrict__ big_list,
                                                   const ErrState *err, int4 *rec,
                                                   const uint2 *__restrict__ perm, Segs S,
                                                   int idx_bits, int passes, int med_cap) {
    __shared__ uint32_t s_cnt[BIG_NW][256];
    __shared__ uint32_t s_warp[BIG_NW];
    __shared__ unsigned long long s_prevrow;
    __shared__ uint2 s_long[BIGC_NLONG];  // long runs of the column: [first, end)
    __shared__ int s_nlong;
    extern __shared__ unsigned long long s_med[];  // [MED_Q][2 * MED_CAP]
    const int tid = threadIdx.x;
    pdl_wait();
    pdl_trigger();
    const unsigned nbig = *((volatile const unsigned *)&err->nbig);
    if (blockIdx.x >= nbig) return;  // no column for this CTA in either loop
    const unsigned lsmall = *((volatile const unsigned *)&err->lsmall);
    const unsigned long long idx_mask = (1ull << idx_bits) - 1;
    {  // medium columns: one quarter each
        const int q = tid / MED_NT, qt = tid % MED_NT;
        unsigned long long *K = s_med + (size_t)q * 2 * MED_CAP;
        uint32_t *s_qw = &s_cnt[0][0] + q * (MED_NT / 32);
        for (unsigned kb = blockIdx.x * MED_Q + q; kb < nbig; kb += gridDim.x * MED_Q) {
            const int n = (int)big_list[kb].n;
            if (n > med_cap) continue;
            const uint32_t st = big_list[kb].start + lsmall;
            med_column(&big_list[kb], st, n, reinterpret_cast<unsigned long long *>(rec + st), perm,
                       S, idx_bits, K, K + MED_CAP, s_qw, q, qt);
        }
    }
    __syncthreads();
    for (unsigned kb = blockIdx.x; kb < nbig; kb += gridDim.x) {
        const int64_t n = big_list[kb].n;
        if (n <= med_cap) continue;
        const uint32_t st = big_list[kb].start + lsmall;
        unsigned long long *A = reinterpret_cast<unsigned long long *>(rec + st);
        unsigned long long *B = A + n;
        // entries {row, position} -> keys in A (8 loads per thread in flight)
        for (int64_t p0 = 0; p0 < n; p0 += 8 * BIG_NT) {
            uint2 e[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t p = p0 + u * BIG_NT + tid;
                e[u] = (p < n) ? perm[st + p] : make_uint2(0u, 0u);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t p = p0 + u * BIG_NT + tid;
                if (p < n) A[p] = ((unsigned long long)(e[u].x - 1u) << idx_bits) | e[u].y;
            }
        }
        __syncthreads();
        unsigned long long *src = A, *dst = B;
        for (int ps = 0; ps < passes; ++ps) {
            big_radix_pass(src, dst, n, 8 * ps, s_cnt, s_warp);
            unsigned long long *tmp = src;
            src = dst;
            dst = tmp;
        }
        // gather values in sorted order into the other buffer (8 in flight)
        for (int64_t p0 = 0; p0 < n; p0 += 8 * BIG_NT) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t p = p0 + u * BIG_NT + tid;
                v[u] = (p < n) ? *seg_value(S, (int64_t)(src[p] & idx_mask)) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t p = p0 + u * BIG_NT + tid;
                if (p < n) dst[p] = (unsigned long long)__double_as_longlong(v[u]);
            }
        }
        __syncthreads();
        // ordered fold of runs of equal rows, all runs at once: thread t folds
        // the runs whose head lies in its segment (a run may extend past it);
        // the result lands at the run's head (row in src, value in dst)
        // A run longer than BIGC_LONGRUN (a heavy hitter: one entry repeated
        // over and over) is only listed (its end by binary search: the rows are
        // sorted) and folded by a warp afterwards (warp_fold_run): one thread
        // walking it through global memory costs ~100+ cycles per repeat.
        if (tid == 0) s_nlong = 0;
        __syncthreads();
        {
            const int64_t lo = (int64_t)tid * n / BIG_NT, hi = (int64_t)(tid + 1) * n / BIG_NT;
            int64_t p = lo;
            while (p < hi) {
                const unsigned long long row = src[p] >> idx_bits;
                if (p > 0 && (src[p - 1] >> idx_bits) == row) {  // not a head: skip to the next one
                    ++p;
                    continue;
                }
                if (p + BIGC_LONGRUN < n && (src[p + BIGC_LONGRUN] >> idx_bits) == row) {
                    int64_t a2 = p + BIGC_LONGRUN + 1, b2 = n;  // first index in [a2, b2] of another row
                    while (a2 < b2) {
                        const int64_t mid = (a2 + b2) >> 1;
                        if ((src[mid] >> idx_bits) == row) a2 = mid + 1;
                        else b2 = mid;
                    }
                    const int e = atomicAdd(&s_nlong, 1);
                    if (e < BIGC_NLONG) {
                        s_long[e] = make_uint2((uint32_t)p, (uint32_t)a2);
                        p = a2;
                        continue;
                    }
                }
                double acc = fold_add(0.0, __longlong_as_double((long long)dst[p]));
                int64_t q = p + 1;
                while (q < n && (src[q] >> idx_bits) == row) {
                    acc = fold_add(acc, __longlong_as_double((long long)dst[q]));
                    ++q;
                }
                dst[p] = (unsigned long long)__double_as_longlong(acc);
                p = q;
            }
        }
        __syncthreads();
        {
            const int nl = min(s_nlong, BIGC_NLONG);
            for (int e = tid >> 5; e < nl; e += BIG_NT / 32) {
                const uint32_t q0 = s_long[e].x, q1 = s_long[e].y;
                const double acc = warp_fold_run(dst + q0, (int64_t)q1 - q0);
                __syncwarp();
                if ((tid & 31) == 0) dst[q0] = (unsigned long long)__double_as_longlong(acc);
            }
        }
        __syncthreads();
        if (tid == 0) s_prevrow = ~0ull;
        __syncthreads();
        // compact the heads to [0, runs) in order
        uint32_t carry = 0;
        for (int64_t base = 0; base < n; base += BIG_NT) {
            const int64_t p = base + tid;
            const bool valid = p < n;
            const unsigned long long row = valid ? (src[p] >> idx_bits) : 0ull;
            const unsigned long long prev =
                (tid == 0) ? s_prevrow : (valid ? (src[p - 1] >> idx_bits) : 0ull);
            const bool head = valid && row != prev;
            const unsigned long long val = head ? dst[p] : 0ull;
            uint32_t tot;
            const uint32_t run = block_excl_sum<BIG_NT, uint32_t>(head ? 1u : 0u, s_warp, tot) + carry;
            if (p == base + BIG_NT - 1 && valid) s_prevrow = row;
            if (!valid && tid == BIG_NT - 1) s_prevrow = row;
            __syncthreads();  // the chunk is read before any of it is overwritten
            if (head) {
                src[run] = row;  // row - 1 (key stores row-1)
                dst[run] = val;
            }
            carry += tot;
            __syncthreads();
        }
        if (tid == 0) {
            big_list[kb].start = st;  // absolute from here on
            big_list[kb].u = carry | ((src == B) ? BIGFLAG : 0u);
        }
        __syncthreads();
    }
}

cudaError_t launch_bigcol(Launch &lc, BigCol *big_list, const ErrState *err, int4 *rec,
                          const uint2 *perm, const Segs &S, int idx_bits, int passes) {
    cudaError_t e = ensure_smem_attr((const void *)k_bigcol, (int)BIG_DSMEM);
    if (e != cudaSuccess) return e;
    const int grid = 2 * lc.num_sms;
    e = launch_pdl(k_bigcol, dim3(grid), dim3(BIG_NT), BIG_DSMEM, lc.stream, big_list, err, rec,
                   perm, S, idx_bits, passes, MED_CAP);
    if (e != cudaSuccess) return e;
    lc.launches++;
    return cudaGetLastError();
}

}  // namespace sa

#ifdef SA_TRACE
extern "C" int sa_debug_trace(void *host, int n) {
    return (int)cudaMemcpyFromSymbol(host, sa::g_trace, (size_t)n * 32);
}
#endif
