// sa_kernels.cu -- hand-written sm_100a kernels for sparse(i,j,s,m,n).
//
// Pipeline (one stream, no host round trip):
//   k_hist       column histogram of the triplets + index validation
//                (types.py:121-165 semantics), warp-aggregated atomics
//   k_col_scan   single-pass decoupled-look-back exclusive scan of the column
//                counts -> column cursors; also the tile -> first-column map
//                and the list of big columns
//   k_scatter    counting-sort scatter by column: 16-byte records
//                {row, input position, value} at cursor positions
//   k_bigcol     columns longer than BIGCOL: in-place LSD radix sort by
//                (row, input position), ordered fold
//   k_tile_fold  per tile of columns, in shared memory: hash (column,row)
//                groups, order each group by input position, fold from +0.0
//                in input order (bit-exact with the reference scatter,
//                _kernels.pyx:82-89), order groups by row, chained scan of
//                the unique counts -> jc, ir, pr written once.
//
// Reference algorithm: serial.py:111-168 / _kernels.pyx:20-89 (row-first
// counting sort).  This pipeline is column-first; it produces the same CSC
// because both order entries by (column, row) and fold duplicates in
// ascending input order.

#include <cstdlib>

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
                                              ErrState *err, int vec, int infer) {
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
    if (lane == 0) {
        if (a.bad_i != ~0ull) atomicMin(&err->bad_i, a.bad_i);
        if (a.bad_j != ~0ull) atomicMin(&err->bad_j, a.bad_j);
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
                        int32_t N, uint32_t *cnt, ErrState *err, bool infer) {
    if (L <= 0) return cudaSuccess;
    const int vec = aligned16(ii) && aligned16(jj);
    int64_t want = ((vec ? (L >> 2) : L) + 255) / 256 + 1;
    int grid = (int)std::min<int64_t>(want, (int64_t)lc.num_sms * 8);
    k_hist<<<grid, 256, 0, lc.stream>>>(ii, jj, L, M, N, cnt, err, vec, infer ? 1 : 0);
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
//   tile_info[t]  {min{c : sstart(c) >= t*TILE}, its sstart}, 0 <= t <= ntiles
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
__global__ void __launch_bounds__(SCAN_NT) k_col_scan(const uint32_t *cnt,
                                                      uint32_t *__restrict__ sstart,
                                                      uint32_t *cur, int32_t N,
                                                      int2 *__restrict__ tile_info,
                                                      uint8_t *__restrict__ tile_big, int64_t ntiles,
                                                      BigCol *__restrict__ big_list,
                                                      uint32_t *__restrict__ bigk,
                                                      unsigned long long *scan_state,
                                                      uint2 *__restrict__ perm,
                                                      ErrState *err) {
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
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k) sum += scan_word(loc[k]);
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
                int64_t tb = (int64_t)(small / TILE);
                if (tb > ntiles - 1) tb = ntiles - 1;
                tile_big[tb] = 1;
            }
            // fold tiles t with small < t*TILE <= small + extent start at column c+1
            const uint32_t ext = big ? 1u : n;
            if (ext) {
                int64_t t = (int64_t)(small / TILE) + 1;
                const int64_t last = min((int64_t)((small + ext) / TILE), ntiles - 1);
                for (; t <= last; ++t) tile_info[t] = make_int2((int)(c + 1), (int)(small + ext));
            }
            if (c == N - 1) {
                const uint64_t tot_small = small + ext;
                err->lsmall = (unsigned)tot_small;
                sstart[N] = (uint32_t)tot_small;
                s_tail = (long long)(tot_small / TILE) + 1;
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
                            unsigned long long *scan_state, uint2 *perm, ErrState *err) {
    if (N <= 0) return cudaSuccess;
    int grid = (int)((N + SCAN_TILE - 1) / SCAN_TILE);
    cudaError_t e = launch_pdl(k_col_scan, dim3(grid), dim3(SCAN_NT), 0, lc.stream, cnt, sstart, cur, N,
                               tile_info, tile_big, ntiles, big_list, bigk, scan_state, perm, err);
    if (e != cudaSuccess) return e;
    lc.launches++;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// CTA-scope column aggregation shared by k_colcount and k_scatter.  A CTA
// takes CHUNK consecutive triplets (CPT per thread, loaded with 16-byte
// vector loads) and counts their columns in a shared-memory hash (open
// addressing, HT slots, list of used slots so only those are visited again).
// Element-ordered FEM input touches ~CHUNK/9 distinct columns per chunk, so
// global atomics drop by an order of magnitude and stay independent.
// ---------------------------------------------------------------------------
constexpr int AGG_NT = 256;
constexpr int CPT = 8;
constexpr int CHUNK = AGG_NT * CPT;
constexpr int HT = 2 * CHUNK;

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
// touches the shared-memory hash, with the run length.  len[k] = triplets
// from k to the end of its run.
__device__ __forceinline__ void run_lengths(const int (&j)[CPT], const bool (&v)[CPT],
                                            int (&len)[CPT]) {
    int run = 0;
#pragma unroll
    for (int k = CPT - 1; k >= 0; --k) {
        const bool cont = (k + 1 < CPT) && v[k] && v[k < CPT - 1 ? k + 1 : k] &&
                          j[k < CPT - 1 ? k + 1 : k] == j[k];
        run = v[k] ? (cont ? run + 1 : 1) : 0;
        len[k] = run;
    }
}

// The same runs as bit masks over the CPT slots: bit k of `heads` starts a
// run of valid triplets, and a head's run length is the distance to the next
// set bit of `stops` (a new run or an invalid slot, or the end).
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

__device__ __forceinline__ bool run_head(const int (&j)[CPT], const bool (&v)[CPT], int k) {
    return !(k > 0 && v[k > 0 ? k - 1 : 0] && j[k > 0 ? k - 1 : 0] == j[k]);
}

// ---------------------------------------------------------------------------
// k_colcount: column histogram of the assembly path (reads jj only; rows
// are validated by k_scatter, which reads them anyway).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(AGG_NT) k_colcount(const int32_t *__restrict__ jj, int64_t L,
                                                     int32_t N, uint32_t *__restrict__ cnt,
                                                     ErrState *err, int vec) {
    __shared__ AggSmem A;
    const int tid = threadIdx.x;
    for (int k = tid; k < HT; k += AGG_NT) {
        A.key[k] = 0;
        A.ctr[k] = 0;
    }
    if (tid == 0) A.nused = 0;
    __syncthreads();
    unsigned long long bad = ~0ull;
    unsigned over = 0;
    const int64_t nchunk = (L + CHUNK - 1) / CHUNK;
    int jn[CPT];
    if ((int64_t)blockIdx.x < nchunk)
        load_run(jj, (int64_t)blockIdx.x * CHUNK + (int64_t)tid * CPT, L, vec, jn, 0x7fffffff);
    for (int64_t ch = blockIdx.x; ch < nchunk; ch += gridDim.x) {
        const int64_t t0 = ch * CHUNK + (int64_t)tid * CPT;
        int j[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) j[k] = jn[k];
        if (ch + gridDim.x < nchunk)  // prefetch the next chunk while this one is counted
            load_run(jj, (ch + gridDim.x) * CHUNK + (int64_t)tid * CPT, L, vec, jn, 0x7fffffff);
        bool vk[CPT];
        int len[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            const bool live = t0 + k < L;
            if (live && j[k] < 1) bad = min(bad, (unsigned long long)(t0 + k));
            if (live && j[k] > N) over = 1;
            vk[k] = live && j[k] >= 1 && j[k] <= N;
        }
        run_lengths(j, vk, len);
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            if (vk[k] && run_head(j, vk, k)) {
                const int h = agg_insert(A, j[k] - 1);
                atomicAdd(&A.ctr[h], len[k]);
            }
        }
        __syncthreads();
        const int nu = A.nused;
        for (int e = tid; e < nu; e += AGG_NT) {
            const int h = A.used[e];
            atomicAdd(&cnt[A.key[h] - 1], (uint32_t)A.ctr[h]);
            A.key[h] = 0;
            A.ctr[h] = 0;
        }
        __syncthreads();
        if (tid == 0) A.nused = 0;
        __syncthreads();
    }
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

// Direct variant: each column run (per thread, CPT consecutive triplets)
// issues one global reduction, with no shared-memory aggregation.
__global__ void __launch_bounds__(AGG_NT) k_colcount_direct(const int32_t *__restrict__ jj,
                                                            int64_t L, int32_t N,
                                                            uint32_t *__restrict__ cnt,
                                                            ErrState *err, int vec) {
    unsigned long long bad = ~0ull;
    unsigned over = 0;
    const int64_t nrun = (L + CPT - 1) / CPT;
    for (int64_t r = (int64_t)blockIdx.x * AGG_NT + threadIdx.x; r < nrun;
         r += (int64_t)gridDim.x * AGG_NT) {
        const int64_t t0 = r * CPT;
        int j[CPT];
        load_run(jj, t0, L, vec, j, 0x7fffffff);
        bool vk[CPT];
        int len[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            const bool live = t0 + k < L;
            if (live && j[k] < 1) bad = min(bad, (unsigned long long)(t0 + k));
            if (live && j[k] > N) over = 1;
            vk[k] = live && j[k] >= 1 && j[k] <= N;
        }
        run_lengths(j, vk, len);
#pragma unroll
        for (int k = 0; k < CPT; ++k)
            if (vk[k] && run_head(j, vk, k)) atomicAdd(&cnt[j[k] - 1], (uint32_t)len[k]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        bad = min(bad, __shfl_xor_sync(FULL, bad, o));
        over |= __shfl_xor_sync(FULL, over, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (bad != ~0ull) atomicMin(&err->bad_j, bad);
        if (over) err->over_n = 1;
    }
}

// ---------------------------------------------------------------------------
// Window aggregation (k_colcount_win, k_scatter_win).  A CTA takes CHUNK
// consecutive triplets; element-ordered input keeps a chunk's columns near
// the chunk's first column, so the column runs (per thread) count into a
// directly indexed shared-memory window of WB bins around it (one shared
// atomic per run, no hashing).  The first touch of a bin lists it; after
// the chunk, every listed bin issues one global atomic.  Columns outside
// the window go to global memory directly.
// ---------------------------------------------------------------------------
constexpr int WB = 8192;

struct WinSmem {
    uint32_t bin[WB];      // per window column: triplets of the chunk, then the cursor word
    int used[CHUNK];       // listed bins
    int nused;
};

__device__ __forceinline__ int window_base(const int32_t *__restrict__ jj, int64_t t) {
    return __ldg(jj + t) - 1 - WB / 2;
}

__global__ void __launch_bounds__(AGG_NT) k_colcount_win(const int32_t *__restrict__ jj, int64_t L,
                                                         int32_t N, uint32_t *__restrict__ cnt,
                                                         ErrState *err, int vec) {
    __shared__ WinSmem W;
    const int tid = threadIdx.x;
    for (int k = tid; k < WB; k += AGG_NT) W.bin[k] = 0;
    if (tid == 0) W.nused = 0;
    __syncthreads();
    pdl_wait();
    pdl_trigger();
    unsigned long long bad = ~0ull;
    unsigned over = 0;
    const int64_t nchunk = (L + CHUNK - 1) / CHUNK;
    int jn[CPT];
    if ((int64_t)blockIdx.x < nchunk)
        load_run(jj, (int64_t)blockIdx.x * CHUNK + (int64_t)tid * CPT, L, vec, jn, 0x7fffffff);
    for (int64_t ch = blockIdx.x; ch < nchunk; ch += gridDim.x) {
        const int64_t t0 = ch * CHUNK + (int64_t)tid * CPT;
        const int cb = window_base(jj, ch * CHUNK);
        int j[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) j[k] = jn[k];
        if (ch + gridDim.x < nchunk)  // prefetch the next chunk while this one is counted
            load_run(jj, (ch + gridDim.x) * CHUNK + (int64_t)tid * CPT, L, vec, jn, 0x7fffffff);
        // validity: one min/max over the run; per-slot checks only when needed
        unsigned vmask = (1u << CPT) - 1;
        {
            int lo = j[0], hi = j[0];
#pragma unroll
            for (int k = 1; k < CPT; ++k) {
                lo = min(lo, j[k]);
                hi = max(hi, j[k]);
            }
            if (lo < 1 || hi > N || t0 + CPT > L) {
                vmask = 0;
#pragma unroll
                for (int k = 0; k < CPT; ++k) {
                    const bool live = t0 + k < L;
                    if (live && j[k] < 1) bad = min(bad, (unsigned long long)(t0 + k));
                    if (live && j[k] > N) over = 1;
                    if (live && j[k] >= 1 && j[k] <= N) vmask |= 1u << k;
                }
            }
        }
        const Runs R = run_masks(j, vmask);
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            if (R.heads & (1u << k)) {
                const int len = run_len(R, k);
                const unsigned b = (unsigned)(j[k] - 1 - cb);
                if (b < (unsigned)WB) {
                    if (atomicAdd(&W.bin[b], (uint32_t)len) == 0u) W.used[atomicAdd(&W.nused, 1)] = (int)b;
                } else {
                    atomicAdd(&cnt[j[k] - 1], (uint32_t)len);
                }
            }
        }
        __syncthreads();
        const int nu = W.nused;
        for (int e = tid; e < nu; e += AGG_NT) {
            const int b = W.used[e];
            atomicAdd(&cnt[cb + b], W.bin[b]);
            W.bin[b] = 0;
        }
        __syncthreads();
        if (tid == 0) W.nused = 0;
        __syncthreads();
    }
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

// Aggregation variants (measured on cfg2/cfg3/cfg4), chosen
// by SA_COLCOUNT_MODE / SA_SCATTER_MODE = 0 direct, 1 hash, 2 window.
bool pdl_enabled() {
    static int m = -1;
    if (m < 0) {
        const char *e = getenv("SA_PDL");
        m = (e && e[0] == '0') ? 0 : 1;
    }
    return m == 1;
}

static int env_mode(const char *name, int dflt) {
    const char *e = getenv(name);
    return (e && e[0] >= '0' && e[0] <= '2') ? e[0] - '0' : dflt;
}
// 0 direct, 1 shared-memory hash, 2 shared-memory window
static int colcount_mode() {
    static int m = -1;
    if (m < 0) m = env_mode("SA_COLCOUNT_MODE", 2);
    return m;
}
static int scatter_mode() {
    static int m = -1;
    if (m < 0) m = env_mode("SA_SCATTER_MODE", 1);
    return m;
}

cudaError_t launch_colcount(Launch &lc, const int32_t *jj, int64_t L, int32_t N, uint32_t *cnt,
                            ErrState *err) {
    if (L <= 0) return cudaSuccess;
    const int vec = aligned16(jj);
    const int64_t nchunk = (L + CHUNK - 1) / CHUNK;
    int grid = (int)std::min<int64_t>(nchunk, (int64_t)lc.num_sms * 4);
    if (colcount_mode() == 1) {
        k_colcount<<<grid, AGG_NT, 0, lc.stream>>>(jj, L, N, cnt, err, vec);
    } else if (colcount_mode() == 2) {
        cudaError_t e = launch_pdl(k_colcount_win, dim3(grid), dim3(AGG_NT), 0, lc.stream, jj, L, N, cnt,
                                   err, vec);
        if (e != cudaSuccess) return e;
    } else {
        const int64_t want = ((L + CPT - 1) / CPT + AGG_NT - 1) / AGG_NT;
        const int g = (int)std::min<int64_t>(want, (int64_t)lc.num_sms * 8);
        k_colcount_direct<<<g, AGG_NT, 0, lc.stream>>>(jj, L, N, cnt, err, vec);
    }
    lc.launches++;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// k_scatter: counting-sort scatter by column of 8-byte entries {row,
// input position} (the fold gathers the values by position, so the 8-byte
// values are read once, by the fold).  Per chunk: (1) each column run gets
// chunk-local slots from a shared-memory counter, (2) one global atomicAdd
// per distinct column reserves the chunk's slots on the column cursor, (3)
// entries are written.  Row indices are validated here for every triplet
// (first bad position, rows above M).  The slot order inside a column is
// arbitrary; the fold restores input order from the position.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(AGG_NT) k_scatter(const int32_t *__restrict__ ii,
                                                    const int32_t *__restrict__ jj, int64_t L,
                                                    int32_t M, int32_t N,
                                                    uint32_t *__restrict__ cur,
                                                    uint2 *__restrict__ perm, int vec,
                                                    ErrState *err) {
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
    unsigned long long bad = ~0ull;
    unsigned over = 0;
    const int64_t nchunk = (L + CHUNK - 1) / CHUNK;
    int in_[CPT], jn[CPT];
    if ((int64_t)blockIdx.x < nchunk) {
        const int64_t t0 = (int64_t)blockIdx.x * CHUNK + (int64_t)tid * CPT;
        load_run(ii, t0, L, vec, in_, 1);
        load_run(jj, t0, L, vec, jn, 0);
    }
    for (int64_t ch = blockIdx.x; ch < nchunk; ch += gridDim.x) {
        const int64_t t0 = ch * CHUNK + (int64_t)tid * CPT;
        int i[CPT], j[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            i[k] = in_[k];
            j[k] = jn[k];
        }
        if (ch + gridDim.x < nchunk) {  // next chunk in flight
            const int64_t t1 = (ch + gridDim.x) * CHUNK + (int64_t)tid * CPT;
            load_run(ii, t1, L, vec, in_, 1);
            load_run(jj, t1, L, vec, jn, 0);
        }
        // validity: min/max over the run; per-slot checks only when needed
        unsigned vmask = (1u << CPT) - 1;
        {
            int jlo = j[0], jhi = j[0], ilo = i[0], ihi = i[0];
#pragma unroll
            for (int k = 1; k < CPT; ++k) {
                jlo = min(jlo, j[k]);
                jhi = max(jhi, j[k]);
                ilo = min(ilo, i[k]);
                ihi = max(ihi, i[k]);
            }
            if (jlo < 1 || jhi > N || ilo < 1 || ihi > M || t0 + CPT > L) {
                vmask = 0;
#pragma unroll
                for (int k = 0; k < CPT; ++k) {
                    const bool live = t0 + k < L;
                    if (live && i[k] < 1) bad = min(bad, (unsigned long long)(t0 + k));
                    if (live && i[k] > M) over = 1;
                    if (live && j[k] >= 1 && j[k] <= N) vmask |= 1u << k;
                }
            }
        }
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
            perm[pos] = make_uint2((uint32_t)i[k], (uint32_t)(t0 + k));
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

// Direct variant: one global cursor reservation (atomicAdd with return) per
// column run; all of a thread's reservations are in flight together.
__global__ void __launch_bounds__(AGG_NT) k_scatter_direct(const int32_t *__restrict__ ii,
                                                           const int32_t *__restrict__ jj,
                                                           int64_t L, int32_t M, int32_t N,
                                                           uint32_t *__restrict__ cur,
                                                           uint2 *__restrict__ perm, int vec,
                                                           ErrState *err) {
    const uint32_t lsmall = err->lsmall;
    unsigned long long bad = ~0ull;
    unsigned over = 0;
    const int64_t nrun = (L + CPT - 1) / CPT;
    for (int64_t r = (int64_t)blockIdx.x * AGG_NT + threadIdx.x; r < nrun;
         r += (int64_t)gridDim.x * AGG_NT) {
        const int64_t t0 = r * CPT;
        int i[CPT], j[CPT];
        load_run(ii, t0, L, vec, i, 1);
        load_run(jj, t0, L, vec, j, 0);
        bool vk[CPT];
        int len[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            const bool live = t0 + k < L;
            if (live && i[k] < 1) bad = min(bad, (unsigned long long)(t0 + k));
            if (live && i[k] > M) over = 1;
            vk[k] = live && j[k] >= 1 && j[k] <= N;
        }
        run_lengths(j, vk, len);
        uint32_t w[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            w[k] = 0;
            if (vk[k] && run_head(j, vk, k)) w[k] = atomicAdd(&cur[j[k] - 1], (uint32_t)len[k]);
        }
        uint32_t slot = 0;
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            if (!vk[k]) continue;
            if (run_head(j, vk, k)) slot = (w[k] & POSMASK) + ((w[k] & BIGFLAG) ? lsmall : 0u);
            else slot += 1;
            perm[slot] = make_uint2((uint32_t)i[k], (uint32_t)(t0 + k));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        bad = min(bad, __shfl_xor_sync(FULL, bad, o));
        over |= __shfl_xor_sync(FULL, over, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (bad != ~0ull) atomicMin(&err->bad_i, bad);
        if (over) err->over_m = 1;
    }
}

__global__ void __launch_bounds__(AGG_NT, 4) k_scatter_win(const int32_t *__restrict__ ii,
                                                        const int32_t *__restrict__ jj, int64_t L,
                                                        int32_t M, int32_t N,
                                                        uint32_t *__restrict__ cur,
                                                        uint2 *__restrict__ perm, int vec,
                                                        ErrState *err) {
    __shared__ WinSmem W;
    const int tid = threadIdx.x;
    for (int k = tid; k < WB; k += AGG_NT) W.bin[k] = 0;
    if (tid == 0) W.nused = 0;
    __syncthreads();
    const uint32_t lsmall = err->lsmall;
    unsigned long long bad = ~0ull;
    unsigned over = 0;
    const int64_t nchunk = (L + CHUNK - 1) / CHUNK;
    int in_[CPT], jn[CPT];
    if ((int64_t)blockIdx.x < nchunk) {
        const int64_t t0 = (int64_t)blockIdx.x * CHUNK + (int64_t)tid * CPT;
        load_run(ii, t0, L, vec, in_, 1);
        load_run(jj, t0, L, vec, jn, 0);
    }
    for (int64_t ch = blockIdx.x; ch < nchunk; ch += gridDim.x) {
        const int64_t t0 = ch * CHUNK + (int64_t)tid * CPT;
        const int cb = window_base(jj, ch * CHUNK);
        int i[CPT], j[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            i[k] = in_[k];
            j[k] = jn[k];
        }
        if (ch + gridDim.x < nchunk) {  // next chunk in flight
            const int64_t t1 = (ch + gridDim.x) * CHUNK + (int64_t)tid * CPT;
            load_run(ii, t1, L, vec, in_, 1);
            load_run(jj, t1, L, vec, jn, 0);
        }
        unsigned vmask = (1u << CPT) - 1;
        {
            int jlo = j[0], jhi = j[0], ilo = i[0], ihi = i[0];
#pragma unroll
            for (int k = 1; k < CPT; ++k) {
                jlo = min(jlo, j[k]);
                jhi = max(jhi, j[k]);
                ilo = min(ilo, i[k]);
                ihi = max(ihi, i[k]);
            }
            if (jlo < 1 || jhi > N || ilo < 1 || ihi > M || t0 + CPT > L) {
                vmask = 0;
#pragma unroll
                for (int k = 0; k < CPT; ++k) {
                    const bool live = t0 + k < L;
                    if (live && i[k] < 1) bad = min(bad, (unsigned long long)(t0 + k));
                    if (live && i[k] > M) over = 1;
                    if (live && j[k] >= 1 && j[k] <= N) vmask |= 1u << k;
                }
            }
        }
        const Runs R = run_masks(j, vmask);
        uint32_t rk[CPT];
        // heads: rank inside the window bin, or (outside the window) the
        // global cursor word itself
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            rk[k] = 0;
            if (R.heads & (1u << k)) {
                const unsigned b = (unsigned)(j[k] - 1 - cb);
                if (b < (unsigned)WB) {
                    rk[k] = atomicAdd(&W.bin[b], (uint32_t)run_len(R, k));
                    if (rk[k] == 0u) W.used[atomicAdd(&W.nused, 1)] = (int)b;
                } else {
                    rk[k] = atomicAdd(&cur[j[k] - 1], (uint32_t)run_len(R, k));
                }
            }
        }
        __syncthreads();
        const int nu = W.nused;
        for (int e = tid; e < nu; e += AGG_NT) {
            const int b = W.used[e];
            W.bin[b] = atomicAdd(&cur[cb + b], W.bin[b]);
        }
        __syncthreads();
        uint32_t slot = 0;
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            if (!(vmask & (1u << k))) continue;
            if (R.heads & (1u << k)) {
                const unsigned b = (unsigned)(j[k] - 1 - cb);
                const uint32_t w = (b < (unsigned)WB) ? W.bin[b] + rk[k] : rk[k];
                slot = (w & POSMASK) + ((w & BIGFLAG) ? lsmall : 0u);
            } else {
                slot += 1;
            }
            perm[slot] = make_uint2((uint32_t)i[k], (uint32_t)(t0 + k));
        }
        __syncthreads();
        for (int e = tid; e < nu; e += AGG_NT) W.bin[W.used[e]] = 0;
        if (tid == 0) W.nused = 0;
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

cudaError_t launch_scatter(Launch &lc, const int32_t *ii, const int32_t *jj, int64_t L, int32_t M,
                           int32_t N, uint32_t *cur, uint2 *perm, ErrState *err) {
    if (L <= 0) return cudaSuccess;
    const int vec = aligned16(ii) && aligned16(jj);
    const int64_t nchunk = (L + CHUNK - 1) / CHUNK;
    int grid = (int)std::min<int64_t>(nchunk, (int64_t)lc.num_sms * 4);
    if (scatter_mode() == 1) {
        cudaError_t e = launch_pdl(k_scatter, dim3(grid), dim3(AGG_NT), 0, lc.stream, ii, jj, L, M, N, cur,
                                   perm, vec, err);
        if (e != cudaSuccess) return e;
    } else if (scatter_mode() == 2) {
        k_scatter_win<<<grid, AGG_NT, 0, lc.stream>>>(ii, jj, L, M, N, cur, perm, vec, err);
    } else {
        const int64_t want = ((L + CPT - 1) / CPT + AGG_NT - 1) / AGG_NT;
        const int g = (int)std::min<int64_t>(want, (int64_t)lc.num_sms * 8);
        k_scatter_direct<<<g, AGG_NT, 0, lc.stream>>>(ii, jj, L, M, N, cur, perm, vec, err);
    }
    lc.launches++;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// k_bigcol: one CTA per big column (grid-stride over the device-side list).
// The column's entries {row, position} (big space) become keys
// key = (row-1) << idx_bits | input position in two 8-byte buffers A|B
// (the column's 16-byte slots of the big scratch).  Stable LSD radix
// passes (8-bit digits, warp match + per-warp digit counts) sort by (row,
// position); values are gathered from the input by position; each run of
// equal rows is folded from +0.0 in position order.  Results: row-1 in the
// key buffer, value bits in the other buffer, at index = run number;
// bigu[c] = runs | (BIGFLAG if keys ended in buffer B).
// ---------------------------------------------------------------------------
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

__global__ void __launch_bounds__(BIG_NT) k_bigcol(BigCol *__restrict__ big_list,
                                                   const ErrState *err, int4 *rec,
                                                   const uint2 *__restrict__ perm,
                                                   const double *__restrict__ s, int64_t s_stride,
                                                   int idx_bits, int passes) {
    __shared__ uint32_t s_cnt[BIG_NW][256];
    __shared__ uint32_t s_warp[BIG_NW];
    __shared__ unsigned long long s_prevrow;
    const int tid = threadIdx.x;
    pdl_wait();
    pdl_trigger();
    const unsigned nbig = *((volatile const unsigned *)&err->nbig);
    if (blockIdx.x >= nbig) return;
    const unsigned lsmall = *((volatile const unsigned *)&err->lsmall);
    const unsigned long long idx_mask = (1ull << idx_bits) - 1;
    for (unsigned kb = blockIdx.x; kb < nbig; kb += gridDim.x) {
        const uint32_t st = big_list[kb].start + lsmall;
        const int64_t n = big_list[kb].n;
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
                v[u] = (p < n) ? s[(src[p] & idx_mask) * s_stride] : 0.0;
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
        {
            const int64_t lo = (int64_t)tid * n / BIG_NT, hi = (int64_t)(tid + 1) * n / BIG_NT;
            int64_t p = lo;
            while (p < hi) {
                const unsigned long long row = src[p] >> idx_bits;
                if (p > 0 && (src[p - 1] >> idx_bits) == row) {  // not a head: skip to the next one
                    ++p;
                    continue;
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
                          const uint2 *perm, const double *s, int64_t s_stride, int idx_bits,
                          int passes) {
    int grid = lc.num_sms;
    cudaError_t e = launch_pdl(k_bigcol, dim3(grid), dim3(BIG_NT), 0, lc.stream, big_list, err, rec, perm, s,
                               s_stride, idx_bits, passes);
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
