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
//   win_first[w]  min{c : sstart(c) >= w*WIN}, 0 <= w <= nwin (fold windows)
//   tile_big[b]   tile b owns a big column
//   big_list[]    big columns {col, big-space start, n}; bigk[c] = list index
//   err->lsmall   size of the small space
// ---------------------------------------------------------------------------
constexpr int SCAN_NT = 256;
constexpr int SCAN_IPT = 16;
constexpr int SCAN_TILE = SCAN_NT * SCAN_IPT;
constexpr unsigned long long SMALL_MASK = (1ull << 31) - 1;

__global__ void __launch_bounds__(SCAN_NT) k_col_scan(const uint32_t *__restrict__ cnt,
                                                      uint32_t *__restrict__ sstart,
                                                      uint32_t *__restrict__ cur, int32_t N,
                                                      int64_t nwin, int32_t *__restrict__ win_first,
                                                      uint8_t *__restrict__ tile_big, int64_t ntiles,
                                                      BigCol *__restrict__ big_list,
                                                      uint32_t *__restrict__ bigk,
                                                      unsigned long long *scan_state,
                                                      ErrState *err) {
    __shared__ uint32_t s_v[SCAN_TILE];
    __shared__ unsigned long long s_warp[SCAN_NT / 32];
    __shared__ long long s_b;
    __shared__ unsigned long long s_excl;
    if (threadIdx.x == 0) s_b = atomicAdd(&err->scan_ticket, 1u);
    __syncthreads();
    const long long b = s_b;
    const int64_t c_base = b * SCAN_TILE;
    for (int k = threadIdx.x; k < SCAN_TILE; k += SCAN_NT) {
        const int64_t c = c_base + k;
        s_v[k] = (c < N) ? cnt[c] : 0u;
    }
    __syncthreads();
    uint32_t loc[SCAN_IPT];
    unsigned long long sum = 0;
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k) {
        loc[k] = s_v[threadIdx.x * SCAN_IPT + k];
        // a big column adds its triplets to the big space and one placeholder
        // slot to the small space (so every column has a distinct fold position)
        sum += (loc[k] > (uint32_t)BIGCOL) ? (((unsigned long long)loc[k] << 31) | 1ull) : loc[k];
    }
    unsigned long long total;
    unsigned long long pre = block_excl_sum<SCAN_NT, unsigned long long>(sum, s_warp, total);
    if (threadIdx.x < 32) {
        const unsigned long long e = lookback_warp(scan_state, b, total);
        if (threadIdx.x == 0) s_excl = e;
    }
    __syncthreads();
    const unsigned long long run0 = s_excl + pre;
    uint64_t small = run0 & SMALL_MASK;
    uint64_t bigp = run0 >> 31;
#pragma unroll
    for (int k = 0; k < SCAN_IPT; ++k) {
        const int64_t c = c_base + threadIdx.x * SCAN_IPT + k;
        const uint32_t n = loc[k];
        const bool big = n > (uint32_t)BIGCOL;
        if (c < N) {
            sstart[c] = (uint32_t)small | (big ? BIGFLAG : 0u);
            if (big) {
                cur[c] = (uint32_t)bigp | BIGFLAG;
                const unsigned slot = atomicAdd(&err->nbig, 1u);
                big_list[slot] = BigCol{(uint32_t)c, (uint32_t)bigp, n, 0u};
                bigk[c] = slot;
                int64_t tb = (int64_t)(small / TILE);
                if (tb > ntiles - 1) tb = ntiles - 1;
                tile_big[tb] = 1;
            } else {
                cur[c] = (uint32_t)small;
            }
            // fold windows w with small < w*WIN <= small + extent start at column c+1
            const uint32_t ext = big ? 1u : n;
            if (ext) {
                int64_t first = (int64_t)(small / WIN) + 1;
                int64_t last = (int64_t)((small + ext) / WIN);
                if (last > nwin - 1) last = nwin - 1;
                for (int64_t w = first; w <= last; ++w) win_first[w] = (int32_t)(c + 1);
            }
            if (c == N - 1) {
                const uint64_t tot_small = small + (big ? 1 : n);
                err->lsmall = (unsigned)tot_small;
                sstart[N] = (uint32_t)tot_small;
                // windows past the small space (and past dropped invalid triplets) are empty
                for (int64_t w = (int64_t)(tot_small / WIN) + 1; w <= nwin; ++w) win_first[w] = N;
            }
        }
        if (big) {
            bigp += n;
            small += 1;
        } else {
            small += n;
        }
    }
    if (b == 0 && threadIdx.x == 0) {
        win_first[0] = 0;
        win_first[nwin] = N;
    }
}

cudaError_t launch_col_scan(Launch &lc, const uint32_t *cnt, uint32_t *sstart, uint32_t *cur,
                            int32_t N, int64_t nwin, int32_t *win_first, uint8_t *tile_big,
                            int64_t ntiles, BigCol *big_list, uint32_t *bigk,
                            unsigned long long *scan_state, ErrState *err) {
    if (N <= 0) return cudaSuccess;
    int grid = (int)((N + SCAN_TILE - 1) / SCAN_TILE);
    k_col_scan<<<grid, SCAN_NT, 0, lc.stream>>>(cnt, sstart, cur, N, nwin, win_first, tile_big,
                                               ntiles, big_list, bigk, scan_state, err);
    lc.launches++;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// k_colcount: column histogram of the assembly path.  Reads only jj (row
// indices are validated by k_scatter, which reads them anyway).  Each thread
// walks a run of RUN consecutive triplets with a 4-entry column cache in
// registers (element-ordered FEM input revisits a handful of columns), and
// flushes evicted counts with fire-and-forget reductions.
// ---------------------------------------------------------------------------
constexpr int RUN = 16;

__global__ void __launch_bounds__(256) k_colcount(const int32_t *__restrict__ jj, int64_t L,
                                                  int32_t N, uint32_t *__restrict__ cnt,
                                                  ErrState *err, int vec) {
    const int64_t nrun = (L + RUN - 1) / RUN;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    unsigned long long bad = ~0ull;
    unsigned over = 0;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrun; r += stride) {
        const int64_t t0 = r * RUN;
        int j[RUN];
        if (vec && t0 + RUN <= L) {
            const int4 *p = reinterpret_cast<const int4 *>(jj + t0);
#pragma unroll
            for (int q = 0; q < RUN / 4; ++q) {
                const int4 v = __ldg(p + q);
                j[4 * q] = v.x;
                j[4 * q + 1] = v.y;
                j[4 * q + 2] = v.z;
                j[4 * q + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < RUN; ++k) j[k] = (t0 + k < L) ? jj[t0 + k] : 0x7fffffff;
        }
        int key[4] = {0, 0, 0, 0};
        unsigned cn[4] = {0u, 0u, 0u, 0u};
        int victim = 0;
#pragma unroll
        for (int k = 0; k < RUN; ++k) {
            const int c = j[k];
            const bool live = t0 + k < L;
            if (live && c < 1) bad = min(bad, (unsigned long long)(t0 + k));
            if (live && c > N) over = 1;
            if (!(live && c >= 1 && c <= N)) continue;
            bool hit = false;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (key[e] == c) {
                    cn[e] += 1u;
                    hit = true;
                }
            }
            if (!hit) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    if (e == victim) {
                        if (cn[e]) atomicAdd(&cnt[key[e] - 1], cn[e]);
                        key[e] = c;
                        cn[e] = 1u;
                    }
                }
                victim = (victim + 1) & 3;
            }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (cn[e]) atomicAdd(&cnt[key[e] - 1], cn[e]);
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

cudaError_t launch_colcount(Launch &lc, const int32_t *jj, int64_t L, int32_t N, uint32_t *cnt,
                            ErrState *err) {
    if (L <= 0) return cudaSuccess;
    const int vec = aligned16(jj);
    const int64_t nrun = (L + RUN - 1) / RUN;
    int grid = (int)std::min<int64_t>((nrun + 255) / 256, (int64_t)lc.num_sms * 8);
    k_colcount<<<grid, 256, 0, lc.stream>>>(jj, L, N, cnt, err, vec);
    lc.launches++;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// k_scatter: counting-sort scatter by column.  Record = {row, input position,
// value lo, value hi}.  Each thread takes a run of SRUN consecutive
// triplets: duplicates of a column inside the run share one reservation
// (atomicAdd of the run's count on the column cursor), and the run's
// reservations are independent, so their round trips overlap.  Row indices
// are validated here (first bad position, rows above M).  Within a column
// the slot order is whatever the reservations produce; the fold restores
// input order from the stored position.
// ---------------------------------------------------------------------------
constexpr int SRUN = 8;

__global__ void __launch_bounds__(256) k_scatter(const int32_t *__restrict__ ii,
                                                 const int32_t *__restrict__ jj,
                                                 const double *__restrict__ s, int64_t s_stride,
                                                 int64_t L, int32_t M, int32_t N,
                                                 uint32_t *__restrict__ cur,
                                                 int4 *__restrict__ rec, int vec,
                                                 ErrState *err) {
    const uint32_t lsmall = err->lsmall;
    const int64_t nrun = (L + SRUN - 1) / SRUN;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const double s0v = s_stride ? 0.0 : __ldg(s);
    unsigned long long bad = ~0ull;
    unsigned over = 0;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrun; r += stride) {
        const int64_t t0 = r * SRUN;
        int iv[SRUN], jv[SRUN];
        double vv[SRUN];
        if (vec && t0 + SRUN <= L) {
            const int4 *pi = reinterpret_cast<const int4 *>(ii + t0);
            const int4 *pj = reinterpret_cast<const int4 *>(jj + t0);
#pragma unroll
            for (int q = 0; q < SRUN / 4; ++q) {
                const int4 a = __ldg(pi + q), b = __ldg(pj + q);
                iv[4 * q] = a.x; iv[4 * q + 1] = a.y; iv[4 * q + 2] = a.z; iv[4 * q + 3] = a.w;
                jv[4 * q] = b.x; jv[4 * q + 1] = b.y; jv[4 * q + 2] = b.z; jv[4 * q + 3] = b.w;
            }
            if (s_stride) {
                const double2 *ps = reinterpret_cast<const double2 *>(s + t0);
#pragma unroll
                for (int q = 0; q < SRUN / 2; ++q) {
                    const double2 d = __ldg(ps + q);
                    vv[2 * q] = d.x;
                    vv[2 * q + 1] = d.y;
                }
            } else {
#pragma unroll
                for (int k = 0; k < SRUN; ++k) vv[k] = s0v;
            }
        } else {
#pragma unroll
            for (int k = 0; k < SRUN; ++k) {
                const bool live = t0 + k < L;
                iv[k] = live ? ii[t0 + k] : 1;
                jv[k] = live ? jj[t0 + k] : 0;
                vv[k] = live ? s[(t0 + k) * s_stride] : 0.0;
            }
        }
        // columns scattered: valid column index (k_colcount validated/counted
        // exactly these); rows are data here, validated for the error report
        bool ok[SRUN];
#pragma unroll
        for (int k = 0; k < SRUN; ++k) {
            const bool live = t0 + k < L;
            ok[k] = live && jv[k] >= 1 && jv[k] <= N;
            if (live && iv[k] < 1) bad = min(bad, (unsigned long long)(t0 + k));
            if (live && iv[k] > M) over = 1;
        }
        // first occurrence of each column in the run, rank, and run counts
        int first[SRUN], rank[SRUN];
        unsigned cnt[SRUN];
#pragma unroll
        for (int k = 0; k < SRUN; ++k) {
            first[k] = k;
            rank[k] = 0;
            cnt[k] = 0u;
        }
#pragma unroll
        for (int k = 0; k < SRUN; ++k) {
#pragma unroll
            for (int q = 0; q < k; ++q) {
                if (ok[k] && ok[q] && jv[q] == jv[k]) {
                    rank[k] += 1;
                    first[k] = min(first[k], q);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < SRUN; ++k)
#pragma unroll
            for (int q = 0; q < SRUN; ++q)
                if (ok[k] && first[k] == q) cnt[q] += 1u;
        uint32_t base[SRUN];
#pragma unroll
        for (int k = 0; k < SRUN; ++k) {
            base[k] = 0u;
            if (ok[k] && first[k] == k) base[k] = atomicAdd(&cur[jv[k] - 1], cnt[k]);
        }
#pragma unroll
        for (int k = 0; k < SRUN; ++k) {
            if (!ok[k]) continue;
            uint32_t bw = 0u;
#pragma unroll
            for (int q = 0; q < SRUN; ++q)
                if (first[k] == q) bw = base[q];
            const uint32_t pos = (bw & POSMASK) + ((bw & BIGFLAG) ? lsmall : 0u) + (uint32_t)rank[k];
            rec[pos] = make_int4(iv[k], (int)(t0 + k), __double2loint(vv[k]), __double2hiint(vv[k]));
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

cudaError_t launch_scatter(Launch &lc, const int32_t *ii, const int32_t *jj, const double *s,
                           int64_t s_stride, int64_t L, int32_t M, int32_t N, uint32_t *cur,
                           int4 *rec, ErrState *err) {
    if (L <= 0) return cudaSuccess;
    const int vec = aligned16(ii) && aligned16(jj) && (s_stride == 0 || aligned16(s));
    const int64_t nrun = (L + SRUN - 1) / SRUN;
    int grid = (int)std::min<int64_t>((nrun + 255) / 256, (int64_t)lc.num_sms * 8);
    k_scatter<<<grid, 256, 0, lc.stream>>>(ii, jj, s, s_stride, L, M, N, cur, rec, vec, err);
    lc.launches++;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// k_bigcol: one CTA per big column (grid-stride over the device-side list).
// The column's 16-byte records are reused in place as two 8-byte key
// buffers A|B: key = (row-1) << idx_bits | input position.  Stable LSD radix
// passes (8-bit digits, warp match + per-warp digit counts) sort by (row,
// position); values are gathered from the input by position; each run of
// equal rows is folded from +0.0 in position order.  Results: row-1 in the
// key buffer, value bits in the other buffer, at index = run number;
// bigu[c] = runs | (BIGFLAG if keys ended in buffer B).
// ---------------------------------------------------------------------------
constexpr int BIG_NT = 256;

__global__ void __launch_bounds__(BIG_NT) k_bigcol(BigCol *__restrict__ big_list,
                                                   const ErrState *err, int4 *rec,
                                                   const double *__restrict__ s, int64_t s_stride,
                                                   int idx_bits, int passes) {
    __shared__ uint32_t s_hist[256];
    __shared__ uint32_t s_bin[256];
    __shared__ uint16_t s_wcnt[BIG_NT / 32][257];
    __shared__ uint32_t s_warp[BIG_NT / 32];
    __shared__ unsigned long long s_prevrow;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned nbig = *((volatile const unsigned *)&err->nbig);
    const unsigned lsmall = *((volatile const unsigned *)&err->lsmall);
    for (int k = tid; k < (BIG_NT / 32) * 257; k += BIG_NT) (&s_wcnt[0][0])[k] = 0;
    __syncthreads();
    const unsigned long long idx_mask = (1ull << idx_bits) - 1;
    for (unsigned kb = blockIdx.x; kb < nbig; kb += gridDim.x) {
        const uint32_t st = big_list[kb].start + lsmall;
        const int64_t n = big_list[kb].n;
        unsigned long long *A = reinterpret_cast<unsigned long long *>(rec + st);
        unsigned long long *B = A + n;
        // pack records -> keys in A (ascending chunks; reads stay ahead of writes)
        for (int64_t base = 0; base < n; base += BIG_NT) {
            const int64_t p = base + tid;
            int4 r = make_int4(0, 0, 0, 0);
            if (p < n) r = rec[st + p];
            __syncthreads();
            if (p < n)
                A[p] = ((unsigned long long)(uint32_t)(r.x - 1) << idx_bits) | (uint32_t)r.y;
            __syncthreads();
        }
        unsigned long long *src = A, *dst = B;
        for (int ps = 0; ps < passes; ++ps) {
            const int shift = 8 * ps;
            for (int k = tid; k < 256; k += BIG_NT) s_hist[k] = 0;
            __syncthreads();
            for (int64_t p = tid; p < n; p += BIG_NT) atomicAdd(&s_hist[(src[p] >> shift) & 255], 1u);
            __syncthreads();
            {
                uint32_t tot;
                uint32_t v = s_hist[tid];
                uint32_t pre = block_excl_sum<BIG_NT, uint32_t>(v, s_warp, tot);
                s_bin[tid] = pre;
            }
            __syncthreads();
            for (int64_t base = 0; base < n; base += BIG_NT) {
                const int64_t p = base + tid;
                const bool valid = p < n;
                const unsigned long long key = valid ? src[p] : 0ull;
                const int d = valid ? (int)((key >> shift) & 255) : 256;
                const unsigned peers = __match_any_sync(FULL, d);
                const int leader = __ffs(peers) - 1;
                const int wrank = __popc(peers & lanemask_lt());
                if (lane == leader) s_wcnt[warp][d] = (uint16_t)__popc(peers);
                __syncthreads();
                if (valid) {
                    uint32_t pre = s_bin[d];
                    for (int w2 = 0; w2 < warp; ++w2) pre += s_wcnt[w2][d];
                    dst[pre + wrank] = key;
                }
                __syncthreads();
                if (lane == leader) {
                    if (valid) atomicAdd(&s_bin[d], (uint32_t)__popc(peers));
                    s_wcnt[warp][d] = 0;
                }
                __syncthreads();
            }
            unsigned long long *tmp = src;
            src = dst;
            dst = tmp;
        }
        // gather values in sorted order into the other buffer
        for (int64_t p = tid; p < n; p += BIG_NT) {
            const unsigned long long idx = src[p] & idx_mask;
            dst[p] = (unsigned long long)__double_as_longlong(s[idx * s_stride]);
        }
        if (tid == 0) s_prevrow = ~0ull;
        __syncthreads();
        // ordered fold of runs of equal rows
        uint32_t carry = 0;
        for (int64_t base = 0; base < n; base += BIG_NT) {
            const int64_t p = base + tid;
            const bool valid = p < n;
            const unsigned long long row = valid ? (src[p] >> idx_bits) : 0ull;
            const unsigned long long prev =
                (tid == 0) ? s_prevrow : (valid ? (src[p - 1] >> idx_bits) : 0ull);
            const bool head = valid && row != prev;
            uint32_t tot;
            uint32_t run = block_excl_sum<BIG_NT, uint32_t>(head ? 1u : 0u, s_warp, tot) + carry;
            double acc = 0.0;
            if (head) {
                int64_t q = p;
                bool more = true;
                while (more) {
                    unsigned long long kk[8], vv[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const bool in = q + u < n;
                        kk[u] = in ? src[q + u] : ~0ull;
                        vv[u] = in ? dst[q + u] : 0ull;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        if (more && (kk[u] >> idx_bits) == row)
                            acc = fold_add(acc, __longlong_as_double((long long)vv[u]));
                        else
                            more = false;
                    }
                    q += 8;
                }
            }
            if (p == base + BIG_NT - 1 && valid) s_prevrow = row;
            if (!valid && tid == BIG_NT - 1) s_prevrow = row;
            __syncthreads();
            if (head) {
                src[run] = row;  // row - 1 (key stores row-1)
                dst[run] = (unsigned long long)__double_as_longlong(acc);
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
                          const double *s, int64_t s_stride, int idx_bits, int passes) {
    int grid = lc.num_sms;
    k_bigcol<<<grid, BIG_NT, 0, lc.stream>>>(big_list, err, rec, s, s_stride, idx_bits, passes);
    lc.launches++;
    return cudaGetLastError();
}

}  // namespace sa
