// sa_tile.cu -- k_tile_fold: the ordered segmented fold (sm_100a).
//
// Input: 16-byte records {row, input position, value} grouped by column
// (k_scatter), column cursors cur[] (cur[c] = end of column c), tile_first[]
// (first column whose records start in each TILE-wide window).  Output: jc,
// ir, pr.
//
// Persistent CTAs take tiles in ticket order.  Per tile:
//   block  column pass: the tile's non-empty columns and record ranges
//   TMA    records arrive by cp.async.bulk, issued one tile ahead
//   warps  each warp owns the columns starting in its TILE/8 window and, with
//          warp-synchronous code only (no block barriers):
//            (a) column id of each record
//            (b) (column,row) groups: warp-private shared-memory hash,
//                group ids by ballot
//            (c) group sizes / arrival ranks, (d) warp scans of group and
//                column offsets, (e) member lists, (f) members ordered by
//                input position
//   block  tile unique count U -> decoupled look-back aggregate; the
//          PREVIOUS tile (whose look-back had a whole tile of time to
//          resolve) is finished: block-wide look-back, coalesced ir/pr/jc
//   warps  (g) fold each group from +0.0 in input order (the reference's
//          scatter contract, _kernels.pyx:82-89; x86 NaN rule), order groups
//          by row inside each column, stage (row, value) in CSC order.
// Tiles with a column longer than BIGCOL (folded by k_bigcol) take a
// synchronous path that writes straight to global memory.

#include "sa_internal.cuh"

namespace sa {

namespace {

constexpr int NT = TILE_THREADS;
constexpr int NW = NT / 32;
constexpr int WIN = TILE / NW;  // record-position window per warp
constexpr int HSZ = 2 * TCAP;   // hash slots: 2 per record position
constexpr int CCAP = TILE;      // non-empty columns per tile (distinct starts in a TILE window)

struct TileSmem {
    int4 rec[2][TCAP];                 // double-buffered records (TMA destination)
    unsigned long long mbar[2];
    int col[TCAP];                     // column heads -> column-local index + 1
    // One 16-byte cell per record position k: first the two hash slots 2k,
    // 2k+1 of the owning warp's private table, then (hash dead) per-index
    // fields.  Warps only touch cells of their own record range.
    union HCell {
        unsigned long long key[2];
        struct {
            double sval;               // group values ordered by input position
            int g_base;                // group offset (index qa + gid)
            int16_t mem;               // member lists (record ids), per group
            int16_t cgrp;              // group ids listed per column
        } o;
    } hc[TCAP];
    int16_t hgid[HSZ];
    int g_cnt[TCAP];                   // per group (indexed qa + gid)
    int cg_base[CCAP];                 // warp-relative offset of a column in cgrp
    int16_t g_first[TCAP];
    int16_t g_crank[TCAP];
    int16_t r_gid[TCAP];               // per record
    int16_t r_arr[TCAP];
    int ci_col[CCAP];
    int ci_start[CCAP];
    int ci_q[CCAP];
    int ci_cnt[CCAP];                  // 0 for big columns
    int ci_u[CCAP];                    // groups per column (or k_bigcol's count)
    int ci_base[2][CCAP + 1];          // tile-local output offsets (current / pending)
    int st_row[TCAP];                  // staged outputs of the pending tile
    double st_val[TCAP];
    int w_u[NW], w_base[NW];
    int warp_tmp[NW];
    long long red_ll[NW];
    int pre_n[2];
    long long next_tile;
    // pending tile metadata
    long long p_tile;
    int p_c0, p_c1, p_nci, p_U;
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

__device__ __forceinline__ int col_start(const uint32_t *cur, int c) {
    return c > 0 ? (int)(cur[c - 1] & POSMASK) : 0;
}

// warp-level inclusive sum / max
__device__ __forceinline__ int warp_incl_sum(int x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

__device__ __forceinline__ int warp_incl_max(int x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x = max(x, y);
    }
    return x;
}

// In-place warp exclusive scan over a[lo, hi) (lanes stride 32); returns total.
__device__ __forceinline__ int warp_excl_scan(int *a, int lo, int hi) {
    const int lane = threadIdx.x & 31;
    int carry = 0;
    for (int p0 = lo; p0 < hi; p0 += 32) {
        const int p = p0 + lane;
        const int v = (p < hi) ? a[p] : 0;
        const int inc = warp_incl_sum(v);
        if (p < hi) a[p] = carry + inc - v;
        carry += __shfl_sync(FULL, inc, 31);
    }
    return carry;
}

// Block-wide decoupled look-back: exclusive prefix of tile b, then publish
// b's inclusive prefix.  NT predecessors per L2 round trip.  All threads.
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
        int stop = (flag == 2) ? tid : NT;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) stop = min(stop, __shfl_xor_sync(FULL, stop, o));
        if (lane == 0) S.warp_tmp[w] = stop;
        __syncthreads();
        stop = NT;
#pragma unroll
        for (int k = 0; k < NW; ++k) stop = min(stop, S.warp_tmp[k]);
        long long v = (tid <= stop) ? (long long)(word & LB_VALMASK) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        if (lane == 0) S.red_ll[w] = v;
        __syncthreads();
        long long sum = 0;
#pragma unroll
        for (int k = 0; k < NW; ++k) sum += S.red_ll[k];
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

// Record prefetch of tile t into buffer buf (thread 0).
__device__ void prefetch_tile(TileSmem &S, int buf, long long t, long long ntiles,
                              const int32_t *tile_first, const uint32_t *cur, const int4 *rec) {
    S.pre_n[buf] = -1;
    if (t >= ntiles) return;
    const int c0 = tile_first[t], c1 = tile_first[t + 1];
    const int r0 = col_start(cur, c0), r1 = col_start(cur, c1);
    const int n = r1 - r0;
    if (n > 0 && n <= TCAP) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tma_load(S.rec[buf], rec + r0, (unsigned)n * 16u, &S.mbar[buf]);
        S.pre_n[buf] = n;
    } else {
        S.pre_n[buf] = (n == 0) ? 0 : -1;
    }
}

// jc entries of columns [c0, c1): jc[c] = P + base[# non-empty columns before c]
__device__ void write_jc(TileSmem &S, const uint32_t *cur, int c0, int c1, int n_ci,
                         const int *base, long long P, int32_t *jc) {
    const int tid = threadIdx.x;
    int ne_run = 0;
    for (int cb = c0; cb < c1; cb += NT) {
        const int c = cb + tid;
        const bool in = c < c1;
        const int e = in ? (int)(cur[c] & POSMASK) : 0;
        const int st = in ? col_start(cur, c) : 0;
        const int ne = (in && e > st) ? 1 : 0;
        int tot;
        const int k = block_excl_sum<NT, int>(ne, S.warp_tmp, tot) + ne_run;
        if (in) jc[c] = (int32_t)(P + base[min(k, n_ci)]);
        ne_run += tot;
    }
}

// Finish the pending tile: look-back, staged ir/pr, jc, nnz.
__device__ void finish_pending(TileSmem &S, unsigned long long *tile_state, long long ntiles,
                               const uint32_t *cur, int32_t N, int32_t *jc, int32_t *ir,
                               double *pr, int64_t cap, ErrState *err, int pb) {
    const int tid = threadIdx.x;
    const long long t = S.p_tile;
    const int U = S.p_U;
    const long long P = lookback_block(tile_state, t, (unsigned long long)U, S);
    bool over = false;
    for (int k = tid; k < U; k += NT) {
        const long long o = P + k;
        if (o < cap) {
            ir[o] = S.st_row[k];
            pr[o] = S.st_val[k];
        } else {
            over = true;
        }
    }
    if (over) atomicExch(&err->cap_exceeded, 1u);
    write_jc(S, cur, S.p_c0, S.p_c1, S.p_nci, S.ci_base[pb], P, jc);
    if (t == ntiles - 1 && tid == 0) {
        const long long nnz = P + U;
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
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = lanemask_lt();
    unsigned phase0 = 0u, phase1 = 0u;

    if (tid == 0) {
        mbar_init(&S.mbar[0]);
        mbar_init(&S.mbar[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const long long t0 = atomicAdd(&err->tile_ticket, 1u);
        S.next_tile = t0;
        prefetch_tile(S, 0, t0, ntiles, tile_first, cur, rec);
    }
    __syncthreads();
    long long b = S.next_tile;
    int buf = 0, cbuf = 0;
    bool pending = false;

    while (b < ntiles) {
        // ---- claim the next tile, prefetch its records ----------------------
        if (tid == 0) {
            const long long t1 = atomicAdd(&err->tile_ticket, 1u);
            S.next_tile = t1;
            prefetch_tile(S, buf ^ 1, t1, ntiles, tile_first, cur, rec);
        }
        for (int k = tid; k < TCAP; k += NT) S.col[k] = 0;
        const int c0 = tile_first[b], c1 = tile_first[b + 1];
        __syncthreads();

        // ---- column pass (block) ---------------------------------------------
        // packed scan: bits 0-11 non-empty count, 12-23 small records, 24+ big
        int n_ci = 0, n_small = 0, has_big = 0, overflow = 0;
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
            const int scc = min(sc, 4095);
            const int packed = ne | (scc << 12) | ((ne && big) ? (1 << 24) : 0);
            int tot;
            const int pre = block_excl_sum<NT, int>(packed, S.warp_tmp, tot);
            const int ci = n_ci + (pre & 4095);
            const int q = n_small + ((pre >> 12) & 4095);
            if (ne) {
                if (ci < CCAP && q + sc <= TCAP) {
                    S.ci_col[ci] = c;
                    S.ci_start[ci] = st;
                    S.ci_q[ci] = q;
                    S.ci_cnt[ci] = big ? 0 : cnt;
                    S.ci_u[ci] = big ? (int)(bigu[c] & POSMASK) : 0;
                    if (!big) S.col[q] = ci + 1;
                } else {
                    overflow = 1;
                }
            }
            n_ci += tot & 4095;
            n_small += (tot >> 12) & 4095;
            has_big |= (tot >> 24) != 0;
            overflow |= (n_ci > CCAP) || (n_small > TCAP);
        }
        overflow = __syncthreads_or(overflow);
        if (overflow) {  // cannot happen for consistent cursors; fail loudly
            if (tid == 0) atomicExch(&err->internal, 1u);
            n_ci = 0;
            n_small = 0;
            has_big = 1;
        }

        // ---- records in shared memory ----------------------------------------
        int4 *R = S.rec[buf];
        const int pn = S.pre_n[buf];
        if (pn > 0) {
            if (buf == 0) {
                mbar_wait(&S.mbar[0], phase0);
                phase0 ^= 1u;
            } else {
                mbar_wait(&S.mbar[1], phase1);
                phase1 ^= 1u;
            }
        }
        if (has_big) {
            __syncthreads();
            for (int ci = 0; ci < n_ci; ++ci) {
                const int cnt = S.ci_cnt[ci];
                if (cnt == 0) continue;
                const int q = S.ci_q[ci], st = S.ci_start[ci];
                for (int p = tid; p < cnt; p += NT) R[q + p] = rec[st + p];
            }
            __syncthreads();
        } else if (pn < 0 && n_small > 0) {
            const int r0 = S.ci_start[0];
            for (int p = tid; p < n_small; p += NT) R[p] = rec[r0 + p];
            __syncthreads();
        }

        // ---- warp window: columns whose first record lies in [w*WIN, (w+1)*WIN)
        int cw_lo, cw_hi;
        {
            // lower_bound over ci_q (non-decreasing) for the two window edges
            int lo = 0, hi = n_ci;
            const int key_lo = warp * WIN;
            while (lo < hi) {
                int mid = (lo + hi) >> 1;
                if (S.ci_q[mid] < key_lo) lo = mid + 1; else hi = mid;
            }
            cw_lo = lo;
            hi = n_ci;
            const int key_hi = (warp == NW - 1) ? 0x7fffffff : (warp + 1) * WIN;
            while (lo < hi) {
                int mid = (lo + hi) >> 1;
                if (S.ci_q[mid] < key_hi) lo = mid + 1; else hi = mid;
            }
            cw_hi = lo;
        }
        const int qa = (cw_lo < n_ci) ? S.ci_q[cw_lo] : n_small;
        const int qb = (cw_hi < n_ci) ? S.ci_q[cw_hi] : n_small;

        // (a) column id of each record: warp max-scan of the head marks
        {
            int carry = 0;
            for (int p0 = qa; p0 < qb; p0 += 32) {
                const int p = p0 + lane;
                const int v = (p < qb) ? S.col[p] : 0;
                const int m = max(warp_incl_max(v), carry);
                if (p < qb) S.col[p] = m;
                carry = __shfl_sync(FULL, m, 31);
            }
        }
        // clear this warp's hash region and group counters
        const int hb = 2 * qa, hn = 2 * (qb - qa);  // hash slots of this warp
        for (int k = qa + lane; k < qb; k += 32) {
            S.hc[k].key[0] = 0ull;
            S.hc[k].key[1] = 0ull;
        }
        for (int k = qa + lane; k < qb; k += 32) S.g_cnt[k] = 0;
        __syncwarp();

        // (b) (column,row) groups: hash insert, group ids by ballot
        int ng = 0;
        for (int p0 = qa; p0 < qb; p0 += 32) {
            const int p = p0 + lane;
            const bool act = p < qb;
            bool leader = false;
            int h = 0, ci = 0;
            if (act) {
                const int row = R[p].x;
                ci = S.col[p] - 1;
                const unsigned long long key = ((unsigned long long)(unsigned)ci << 32) | (unsigned)row;
                const unsigned hk = (unsigned)((key * 0x9E3779B97F4A7C15ull) >> 32);
                h = hb + (int)(((unsigned long long)hk * (unsigned)hn) >> 32);
                while (true) {
                    const unsigned long long old = atomicCAS(&S.hc[h >> 1].key[h & 1], 0ull, key);
                    if (old == 0ull) { leader = true; break; }
                    if (old == key) break;
                    h = (h + 1 == hb + hn) ? hb : h + 1;
                }
            }
            const unsigned lm = __ballot_sync(FULL, leader);
            if (leader) {
                const int g = ng + __popc(lm & lt);
                S.hgid[h] = (int16_t)g;
                S.g_first[qa + g] = (int16_t)p;
                S.g_crank[qa + g] = (int16_t)atomicAdd(&S.ci_u[ci], 1);
            }
            if (act) S.r_gid[p] = (int16_t)h;
            ng += __popc(lm);
        }
        __syncwarp();
        // (c) group of each record, arrival rank inside its group
        for (int p = qa + lane; p < qb; p += 32) {
            const int g = S.hgid[S.r_gid[p]];
            S.r_gid[p] = (int16_t)g;
            S.r_arr[p] = (int16_t)atomicAdd(&S.g_cnt[qa + g], 1);
        }
        __syncwarp();
        // (d) group offsets (relative to qa), column offsets (relative to the
        //     warp; with and without big columns)
        for (int k = qa + lane; k < qa + ng; k += 32) S.hc[k].o.g_base = S.g_cnt[k];
        int *cib = S.ci_base[cbuf];
        for (int k = cw_lo + lane; k < cw_hi; k += 32) {
            cib[k] = S.ci_u[k];
            S.cg_base[k] = (S.ci_cnt[k] > 0) ? S.ci_u[k] : 0;
        }
        __syncwarp();
        {
            int carry = 0;
            for (int p0 = qa; p0 < qa + ng; p0 += 32) {
                const int p = p0 + lane;
                const int v = (p < qa + ng) ? S.hc[p].o.g_base : 0;
                const int inc = warp_incl_sum(v);
                if (p < qa + ng) S.hc[p].o.g_base = carry + inc - v;
                carry += __shfl_sync(FULL, inc, 31);
            }
        }
        const int Uw = warp_excl_scan(cib, cw_lo, cw_hi);
        warp_excl_scan(S.cg_base, cw_lo, cw_hi);
        __syncwarp();
        // (e) member lists by group, group lists by column
        for (int p = qa + lane; p < qb; p += 32) {
            const int g = S.r_gid[p];
            S.hc[qa + S.hc[qa + g].o.g_base + S.r_arr[p]].o.mem = (int16_t)p;
        }
        for (int g = lane; g < ng; g += 32) {
            const int ci = S.col[S.g_first[qa + g]] - 1;
            S.hc[qa + S.cg_base[ci] + S.g_crank[qa + g]].o.cgrp = (int16_t)g;
        }
        __syncwarp();
        // (f) order each group by input position
        for (int p = qa + lane; p < qb; p += 32) {
            const int g = S.r_gid[p];
            const int base = qa + S.hc[qa + g].o.g_base, sz = S.g_cnt[qa + g];
            const int4 r = R[p];
            int rank = 0;
            for (int k = 0; k < sz; ++k) rank += (R[S.hc[base + k].o.mem].y < r.y);
            S.hc[base + rank].o.sval = __hiloint2double(r.w, r.z);
        }
        if (lane == 0) S.w_u[warp] = Uw;
        __syncthreads();

        // ---- tile count, aggregate, warp output bases --------------------------
        if (tid < 32) {
            const int v = (tid < NW) ? S.w_u[tid] : 0;
            const int inc = warp_incl_sum(v);
            if (tid < NW) S.w_base[tid] = inc - v;
            if (tid == NW - 1) {
                const int U = inc;
                cib[n_ci] = U;
                volatile unsigned long long *vst = tile_state;
                __threadfence();
                if (b == 0) vst[0] = lb_pack(2, (unsigned long long)U);
                else vst[b] = lb_pack(1, (unsigned long long)U);
                S.warp_tmp[0] = U;
            }
        }
        __syncthreads();
        const int U = S.warp_tmp[0];
        const int wbase = S.w_base[warp];
        for (int k = cw_lo + lane; k < cw_hi; k += 32) cib[k] += wbase;
        __syncthreads();

        // ---- finish the previous tile (its look-back had a tile of time) -------
        if (pending) finish_pending(S, tile_state, ntiles, cur, N, jc, ir, pr, cap, err, cbuf ^ 1);

        long long P = 0;
        if (has_big) P = lookback_block(tile_state, b, (unsigned long long)U, S);
        __syncthreads();

        // (g) fold each group in input order, order groups by row, stage/write
        bool over = false;
        for (int g = lane; g < ng; g += 32) {
            const int p0 = S.g_first[qa + g];
            const int row = R[p0].x;
            const int ci = S.col[p0] - 1;
            const int cl = S.cg_base[ci];        // warp-relative column offset in cgrp
            const int cu = S.ci_u[ci];
            int rank = 0;
            for (int k = 0; k < cu; ++k) rank += (R[S.g_first[qa + S.hc[qa + cl + k].o.cgrp]].x < row);
            const int base = qa + S.hc[qa + g].o.g_base, sz = S.g_cnt[qa + g];
            double acc = 0.0;
            for (int k = 0; k < sz; ++k) acc = fold_add(acc, S.hc[base + k].o.sval);
            const int o = cib[ci] + rank;        // tile-local output index
            if (!has_big) {
                S.st_row[o] = row - 1;
                S.st_val[o] = acc;
            } else {
                const long long go = P + o;
                if (go < cap) {
                    ir[go] = row - 1;
                    pr[go] = acc;
                } else {
                    over = true;
                }
            }
        }
        if (has_big) {
            __syncthreads();
            for (int ci = 0; ci < n_ci; ++ci) {
                if (S.ci_cnt[ci] != 0) continue;  // small column: done above
                const int c = S.ci_col[ci];
                const uint32_t w = bigu[c];
                const int ub = (int)(w & POSMASK);
                const int st = S.ci_start[ci];
                const int n = (int)((cur[c] & POSMASK) - (uint32_t)st);
                const unsigned long long *RR = reinterpret_cast<const unsigned long long *>(rec + st);
                const unsigned long long *K = (w & BIGFLAG) ? RR + n : RR;
                const unsigned long long *V = (w & BIGFLAG) ? RR : RR + n;
                for (int k = tid; k < ub; k += NT) {
                    const long long go = P + cib[ci] + k;
                    if (go < cap) {
                        ir[go] = (int32_t)K[k];
                        pr[go] = __longlong_as_double((long long)V[k]);
                    } else {
                        over = true;
                    }
                }
            }
            if (over) atomicExch(&err->cap_exceeded, 1u);
            write_jc(S, cur, c0, c1, n_ci, cib, P, jc);
            if (b == ntiles - 1 && tid == 0) {
                const long long nnz = P + U;
                jc[N] = (int32_t)nnz;
                err->nnz = nnz;
                if (nnz > cap) atomicExch(&err->cap_exceeded, 1u);
            }
            pending = false;
        } else {
            if (tid == 0) {
                S.p_tile = b;
                S.p_c0 = c0;
                S.p_c1 = c1;
                S.p_nci = n_ci;
                S.p_U = U;
            }
            pending = true;
            cbuf ^= 1;
        }
        __syncthreads();
        b = S.next_tile;
        buf ^= 1;
    }
    if (pending) finish_pending(S, tile_state, ntiles, cur, N, jc, ir, pr, cap, err, cbuf ^ 1);
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
