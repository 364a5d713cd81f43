// sa_tile.cu -- k_tile_fold: the ordered segmented fold (sm_100a).
//
// Input: 16-byte records {row, input position, value} already grouped by
// column (k_scatter), column cursors cur[] (end of column c, k_col_scan +
// k_scatter), tile_first[] (first column of each TILE-wide window of record
// positions).  Output: jc, ir, pr.
//
// Persistent CTAs take tiles in ticket order.  Per tile, entirely in shared
// memory:
//   1. column pass: the tile's columns, their record ranges, big columns
//   2. records arrive by TMA bulk copy (cp.async.bulk, issued one tile ahead)
//   3. (column,row) groups through a shared-memory hash table
//   4. each group ordered by input position; fold from +0.0 in that order
//      (the reference's scatter contract, _kernels.pyx:82-89), x86 NaN rule
//   5. groups ordered by row inside each column -> staged (row, value) in
//      final CSC order, tile unique count U published (decoupled look-back)
//   6. one tile LATER (so the look-back has resolved meanwhile): block-wide
//      look-back for the tile prefix P, coalesced writes of ir/pr/jc.
// Tiles holding a column longer than BIGCOL use the synchronous path (the
// column itself was folded by k_bigcol).

#include "sa_internal.cuh"

namespace sa {

namespace {

constexpr int HS = 2 * TCAP;   // hash slots (load factor <= 0.5)
constexpr int CCAP = TILE;     // non-empty columns per tile (distinct starts in a TILE window)
constexpr int NT = TILE_THREADS;
constexpr int IPT = TCAP / NT;

struct OutStage {
    int row[TCAP];           // ir values (row - 1), tile-local CSC order
    double val[TCAP];        // pr values
    int ci_base[CCAP + 1];   // tile-local output offset of each non-empty column
    int c0, c1, n_ci, U;
    long long tile;
};

struct TileSmem {
    int4 rec[2][TCAP];                 // double-buffered records (TMA destination)
    unsigned long long mbar[2];
    int col[TCAP];                     // head marks -> column-local index + 1
    union {
        struct {
            unsigned long long key[HS];
            int16_t gid[HS];
        } h;
        struct {
            double sval[TCAP];         // group values in input order
            int16_t members[TCAP];     // record ids grouped by (column,row)
            int16_t colgrp[TCAP];      // group ids grouped by column
        } o;
    } u;
    int g_cnt[TCAP];
    int g_base[TCAP];
    int16_t g_first[TCAP];
    int16_t g_crank[TCAP];
    int16_t r_gid[TCAP];
    int16_t r_arr[TCAP];
    int ci_col[CCAP];
    int ci_start[CCAP];
    int ci_q[CCAP];
    int ci_cnt[CCAP];
    int ci_u[CCAP];
    OutStage out[2];
    int warp_tmp[NT / 32];
    long long red_ll[NT / 32];
    int n_groups, overflow;
    long long next_tile;
    int pre_r0[2], pre_n[2];           // prefetched record range per buffer
    long long P;
};

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long *bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tma_load(void *dst, const void *src, unsigned bytes,
                                         unsigned long long *bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}

__device__ __forceinline__ unsigned hash_slot(unsigned long long key) {
    return (unsigned)((key * 0x9E3779B97F4A7C15ull) >> 40) & (HS - 1);
}

__device__ __forceinline__ int col_start(const uint32_t *cur, int c) {
    return c > 0 ? (int)(cur[c - 1] & POSMASK) : 0;
}

// Block-wide decoupled look-back: exclusive prefix of tile b (all tiles < b),
// then publish b's inclusive prefix.  NT predecessors are inspected per L2
// round trip.  Must be called by all threads.
__device__ long long lookback_block(unsigned long long *st, long long b, unsigned long long agg,
                                   TileSmem &S) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    volatile unsigned long long *vst = st;
    long long excl = 0;
    long long base = b - 1;
    while (base >= 0) {
        const long long idx = base - tid;
        const unsigned long long word = (idx >= 0) ? vst[idx] : lb_pack(2, 0);
        const unsigned flag = (unsigned)(word >> 62);
        if (__syncthreads_or(flag == 0)) continue;
        // nearest inclusive prefix = smallest tid with flag 2
        int stop = (flag == 2) ? tid : NT;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) stop = min(stop, __shfl_xor_sync(FULL, stop, o));
        if (lane == 0) S.warp_tmp[w] = stop;
        __syncthreads();
        stop = NT;
#pragma unroll
        for (int k = 0; k < NT / 32; ++k) stop = min(stop, S.warp_tmp[k]);
        long long v = (tid <= stop) ? (long long)(word & LB_VALMASK) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        if (lane == 0) S.red_ll[w] = v;
        __syncthreads();
        long long sum = 0;
#pragma unroll
        for (int k = 0; k < NT / 32; ++k) sum += S.red_ll[k];
        excl += sum;
        __syncthreads();
        if (stop < NT) break;
        base -= NT;
    }
    if (tid == 0) {
        __threadfence();
        vst[b] = lb_pack(2, (unsigned long long)excl + agg);
    }
    return excl;
}

// Issue the record prefetch of tile t into buffer `buf` (thread 0 only).
__device__ void prefetch_tile(TileSmem &S, int buf, long long t, long long ntiles,
                              const int32_t *tile_first, const uint32_t *cur, const int4 *rec,
                              unsigned *phase) {
    S.pre_n[buf] = -1;
    if (t >= ntiles) return;
    const int c0 = tile_first[t], c1 = tile_first[t + 1];
    const int r0 = col_start(cur, c0), r1 = col_start(cur, c1);
    const int n = r1 - r0;
    S.pre_r0[buf] = r0;
    if (n > 0 && n <= TCAP) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tma_load(S.rec[buf], rec + r0, (unsigned)n * 16u, &S.mbar[buf]);
        S.pre_n[buf] = n;
    } else {
        S.pre_n[buf] = (n == 0) ? 0 : -1;
    }
    (void)phase;
}

// Write the staged outputs of a finished tile (after its look-back).
__device__ void finish_tile(TileSmem &S, const OutStage &O, unsigned long long *tile_state,
                            long long ntiles, const uint32_t *cur, int32_t N, int32_t *jc,
                            int32_t *ir, double *pr, int64_t cap, ErrState *err) {
    const int tid = threadIdx.x;
    const long long P = lookback_block(tile_state, O.tile, (unsigned long long)O.U, S);
    bool over = false;
    for (int k = tid; k < O.U; k += NT) {
        const long long o = P + k;
        if (o < cap) {
            ir[o] = O.row[k];
            pr[o] = O.val[k];
        } else {
            over = true;
        }
    }
    if (over) atomicExch(&err->cap_exceeded, 1u);
    int ne_run = 0;
    for (int cb = O.c0; cb < O.c1; cb += NT) {
        const int c = cb + tid;
        const bool in = c < O.c1;
        const int e = in ? (int)(cur[c] & POSMASK) : 0;
        const int st = in ? col_start(cur, c) : 0;
        const int ne = (in && e > st) ? 1 : 0;
        int tot;
        const int k = block_excl_sum<NT, int>(ne, S.warp_tmp, tot) + ne_run;
        if (in) jc[c] = (int32_t)(P + O.ci_base[min(k, O.n_ci)]);
        ne_run += tot;
    }
    if (O.tile == ntiles - 1 && tid == 0) {
        const long long nnz = P + O.U;
        jc[N] = (int32_t)nnz;
        err->nnz = nnz;
        if (nnz > cap) atomicExch(&err->cap_exceeded, 1u);
    }
}

}  // namespace

__global__ void __launch_bounds__(NT, 2) k_tile_fold(const uint32_t *__restrict__ cur,
                                                      const int32_t *__restrict__ tile_first,
                                                      int64_t ntiles, const int4 *__restrict__ rec,
                                                      const uint32_t *__restrict__ bigu,
                                                      unsigned long long *tile_state, int32_t N,
                                                      int32_t *__restrict__ jc,
                                                      int32_t *__restrict__ ir,
                                                      double *__restrict__ pr, int64_t cap,
                                                      ErrState *err) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    TileSmem &S = *reinterpret_cast<TileSmem *>(smem_raw);
    const int tid = threadIdx.x;
    unsigned phase[2] = {0u, 0u};

    if (tid == 0) {
        mbar_init(&S.mbar[0]);
        mbar_init(&S.mbar[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const long long t0 = atomicAdd(&err->tile_ticket, 1u);
        S.next_tile = t0;
        prefetch_tile(S, 0, t0, ntiles, tile_first, cur, rec, phase);
    }
    __syncthreads();
    long long b = S.next_tile;
    int buf = 0, ob = 0;
    long long pending = -1;

    while (b < ntiles) {
        // ---- claim the next tile and start its record prefetch ------------
        if (tid == 0) {
            const long long t1 = atomicAdd(&err->tile_ticket, 1u);
            S.next_tile = t1;
            prefetch_tile(S, buf ^ 1, t1, ntiles, tile_first, cur, rec, phase);
            S.n_groups = 0;
            S.overflow = 0;
        }
        for (int k = tid; k < TCAP; k += NT) {
            S.col[k] = 0;
            S.g_cnt[k] = 0;
        }
        for (int k = tid; k < HS; k += NT) S.u.h.key[k] = 0ull;
        const int c0 = tile_first[b], c1 = tile_first[b + 1];
        __syncthreads();

        // ---- phase 1: columns of the tile ---------------------------------
        int n_ci = 0, n_small = 0, has_big = 0;
        const int r0 = col_start(cur, c0);
        for (int cb = c0; cb < c1; cb += NT) {
            const int c = cb + tid;
            const bool in = c < c1;
            const uint32_t ew = in ? cur[c] : 0u;
            const int e = (int)(ew & POSMASK);
            const int big = (int)(ew >> 31);
            const int st = in ? col_start(cur, c) : 0;
            const int cnt = in ? e - st : 0;
            const int ne = cnt > 0 ? 1 : 0;
            const int sc = (ne && !big) ? cnt : 0;
            int tot_ne, tot_sc;
            const int ci = block_excl_sum<NT, int>(ne, S.warp_tmp, tot_ne) + n_ci;
            const int q = block_excl_sum<NT, int>(sc, S.warp_tmp, tot_sc) + n_small;
            const int anybig = __syncthreads_or(ne && big);
            if (ne) {
                if (ci < CCAP && q + sc <= TCAP) {
                    S.ci_col[ci] = c;
                    S.ci_start[ci] = st;
                    S.ci_q[ci] = big ? -1 : q;
                    S.ci_cnt[ci] = big ? 0 : cnt;
                    S.ci_u[ci] = big ? (int)(bigu[c] & POSMASK) : 0;
                    if (!big) S.col[q] = ci + 1;
                } else {
                    S.overflow = 1;
                }
            }
            n_ci += tot_ne;
            n_small += tot_sc;
            has_big |= anybig;
        }
        __syncthreads();
        if (S.overflow) {
            if (tid == 0) atomicExch(&err->internal, 1u);
            n_ci = 0;
            n_small = 0;
            has_big = 1;  // no staging: take the synchronous path with nothing to write
        }

        // ---- phase 2: records in shared memory --------------------------------
        int4 *R = S.rec[buf];
        const int pn = S.pre_n[buf];
        if (pn > 0) {  // a TMA load was issued for this buffer: wait for it
            mbar_wait(&S.mbar[buf], phase[buf]);
            phase[buf] ^= 1u;
        }
        if (has_big) {
            __syncthreads();  // everyone past the wait before overwriting
            for (int ci = 0; ci < n_ci; ++ci) {
                const int q = S.ci_q[ci];
                if (q < 0) continue;
                const int st = S.ci_start[ci], cnt = S.ci_cnt[ci];
                for (int p = tid; p < cnt; p += NT) R[q + p] = rec[st + p];
            }
        } else if (pn < 0 && n_small > 0) {
            for (int p = tid; p < n_small; p += NT) R[p] = rec[r0 + p];
        }
        smem_incl_max<NT, IPT>(S.col, n_small, S.warp_tmp);  // ends with a barrier

        // ---- phase 3: (column,row) groups via a shared-memory hash -------------
        for (int p = tid; p < n_small; p += NT) {
            const int row = R[p].x;
            const int ci = S.col[p] - 1;
            const unsigned long long key = ((unsigned long long)(unsigned)ci << 32) | (unsigned)row;
            unsigned h = hash_slot(key);
            while (true) {
                const unsigned long long old = atomicCAS(&S.u.h.key[h], 0ull, key);
                if (old == 0ull) {
                    const int g = atomicAdd(&S.n_groups, 1);
                    S.u.h.gid[h] = (int16_t)g;
                    S.g_first[g] = (int16_t)p;
                    S.g_crank[g] = (int16_t)atomicAdd(&S.ci_u[ci], 1);
                    break;
                }
                if (old == key) break;
                h = (h + 1) & (HS - 1);
            }
            S.r_gid[p] = (int16_t)h;
        }
        __syncthreads();
        for (int p = tid; p < n_small; p += NT) {
            const int g = S.u.h.gid[S.r_gid[p]];
            S.r_gid[p] = (int16_t)g;
            S.r_arr[p] = (int16_t)atomicAdd(&S.g_cnt[g], 1);
        }
        __syncthreads();
        const int n_groups = S.n_groups;

        // ---- phase 4: group offsets, column offsets, publish the aggregate -----
        OutStage &O = S.out[ob];
        for (int g = tid; g < n_groups; g += NT) S.g_base[g] = S.g_cnt[g];
        for (int k = tid; k < n_ci; k += NT) O.ci_base[k] = S.ci_u[k];
        __syncthreads();
        smem_excl_scan<NT, IPT, int>(S.g_base, n_groups, S.warp_tmp);
        const int U = smem_excl_scan<NT, (CCAP + NT - 1) / NT, int>(O.ci_base, n_ci, S.warp_tmp);
        if (tid == 0) {
            O.ci_base[n_ci] = U;
            O.c0 = c0;
            O.c1 = c1;
            O.n_ci = n_ci;
            O.U = U;
            O.tile = b;
            volatile unsigned long long *vst = tile_state;
            __threadfence();
            if (b == 0) vst[0] = lb_pack(2, (unsigned long long)U);
            else vst[b] = lb_pack(1, (unsigned long long)U);
        }

        // ---- phase 5: members by group, groups by column -----------------------
        for (int p = tid; p < n_small; p += NT) {
            const int g = S.r_gid[p];
            S.u.o.members[S.g_base[g] + S.r_arr[p]] = (int16_t)p;
        }
        for (int g = tid; g < n_groups; g += NT) {
            const int ci = S.col[S.g_first[g]] - 1;
            S.u.o.colgrp[O.ci_base[ci] + S.g_crank[g]] = (int16_t)g;
        }
        __syncthreads();
        // ---- phase 6: order each group by input position -----------------------
        for (int p = tid; p < n_small; p += NT) {
            const int g = S.r_gid[p];
            const int base = S.g_base[g], sz = S.g_cnt[g];
            const int4 r = R[p];
            int rank = 0;
            if (sz > 1) {
                for (int k = 0; k < sz; ++k) rank += (R[S.u.o.members[base + k]].y < r.y);
            }
            S.u.o.sval[base + rank] = __hiloint2double(r.w, r.z);
        }
        __syncthreads();
        // ---- phase 7: fold each group, order groups by row, stage outputs -----
        for (int g = tid; g < n_groups; g += NT) {
            const int p0 = S.g_first[g];
            const int row = R[p0].x;
            const int ci = S.col[p0] - 1;
            const int cb = O.ci_base[ci], cu = S.ci_u[ci];
            int rank = 0;
            for (int k = 0; k < cu; ++k) rank += (R[S.g_first[S.u.o.colgrp[cb + k]]].x < row);
            const int base = S.g_base[g], sz = S.g_cnt[g];
            double acc = 0.0;
            for (int k = 0; k < sz; ++k) acc = fold_add(acc, S.u.o.sval[base + k]);
            if (!has_big) {
                O.row[cb + rank] = row - 1;
                O.val[cb + rank] = acc;
            } else {
                S.u.o.sval[base] = acc;  // keep for the synchronous write below
                S.g_cnt[g] = cb + rank;  // tile-local output index
            }
        }
        __syncthreads();

        if (!has_big) {
            // ---- deferred output of the previous tile ------------------------
            if (pending >= 0) finish_tile(S, S.out[ob ^ 1], tile_state, ntiles, cur, N, jc, ir, pr, cap, err);
            pending = b;
            ob ^= 1;
        } else {
            // ---- synchronous path (tile with a big column) --------------------
            const long long P = lookback_block(tile_state, b, (unsigned long long)U, S);
            bool over = false;
            for (int g = tid; g < n_groups; g += NT) {
                const int p0 = S.g_first[g];
                const long long o = P + S.g_cnt[g];
                if (o < cap) {
                    ir[o] = R[p0].x - 1;
                    pr[o] = S.u.o.sval[S.g_base[g]];
                } else {
                    over = true;
                }
            }
            for (int ci = 0; ci < n_ci; ++ci) {
                if (S.ci_q[ci] >= 0) continue;
                const int c = S.ci_col[ci];
                const uint32_t w = bigu[c];
                const int ub = (int)(w & POSMASK);
                const int st = S.ci_start[ci];
                const int n = (int)((cur[c] & POSMASK) - (uint32_t)st);
                const unsigned long long *RR = reinterpret_cast<const unsigned long long *>(rec + st);
                const unsigned long long *K = (w & BIGFLAG) ? RR + n : RR;
                const unsigned long long *V = (w & BIGFLAG) ? RR : RR + n;
                for (int k = tid; k < ub; k += NT) {
                    const long long o = P + O.ci_base[ci] + k;
                    if (o < cap) {
                        ir[o] = (int32_t)K[k];
                        pr[o] = __longlong_as_double((long long)V[k]);
                    } else {
                        over = true;
                    }
                }
            }
            if (over) atomicExch(&err->cap_exceeded, 1u);
            int ne_run = 0;
            for (int cb = c0; cb < c1; cb += NT) {
                const int c = cb + tid;
                const bool in = c < c1;
                const int e = in ? (int)(cur[c] & POSMASK) : 0;
                const int st = in ? col_start(cur, c) : 0;
                const int ne = (in && e > st) ? 1 : 0;
                int tot;
                const int k = block_excl_sum<NT, int>(ne, S.warp_tmp, tot) + ne_run;
                if (in) jc[c] = (int32_t)(P + O.ci_base[min(k, n_ci)]);
                ne_run += tot;
            }
            if (b == ntiles - 1 && tid == 0) {
                const long long nnz = P + U;
                jc[N] = (int32_t)nnz;
                err->nnz = nnz;
                if (nnz > cap) atomicExch(&err->cap_exceeded, 1u);
            }
        }
        __syncthreads();
        b = S.next_tile;
        buf ^= 1;
    }
    if (pending >= 0) finish_tile(S, S.out[ob ^ 1], tile_state, ntiles, cur, N, jc, ir, pr, cap, err);
    // drain a prefetch that was issued past the end (none: t >= ntiles issues nothing)
}

cudaError_t launch_tile_fold(Launch &lc, const uint32_t *cur, const int32_t *tile_first,
                             int64_t ntiles, const int4 *rec, const uint32_t *bigu,
                             unsigned long long *tile_state, int32_t N, int32_t *jc, int32_t *ir,
                             double *pr, int64_t cap, ErrState *err) {
    if (ntiles <= 0) return cudaSuccess;
    const size_t smem = sizeof(TileSmem);
    cudaError_t e = cudaFuncSetAttribute(k_tile_fold, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tile_fold, NT, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    int64_t grid = std::min<int64_t>(ntiles, (int64_t)lc.num_sms * per_sm);
    k_tile_fold<<<(unsigned)grid, NT, smem, lc.stream>>>(cur, tile_first, ntiles, rec, bigu,
                                                        tile_state, N, jc, ir, pr, cap, err);
    lc.launches++;
    return cudaGetLastError();
}


}  // namespace sa
