// sa_tile.cu -- k_tile_fold: the ordered segmented fold (sm_100a).
//
// Input: 16-byte records {row, input position, value} grouped by column
// (k_scatter) in the small record space; sstart[c] = small-space start of
// column c (| BIGFLAG for a big column, which occupies one placeholder
// slot); win_first[w] = first column starting in fold window w.
// Output: jc, ir, pr.
//
// Persistent CTAs take tiles (TILE_WARPS consecutive windows) in ticket
// order; a tile's records arrive by one TMA bulk copy issued a tile ahead.
// Each warp folds the columns starting in its window, warp-synchronously:
//   A  one pass over its records: column slot (max-scan of head marks),
//      (slot,row) -> group via a warp-private shared-memory hash (group ids
//      by ballot), arrival rank inside the group by match.any in position
//      order (deterministic, no atomics)
//   B  warp scans: group offsets, column offsets
//   C  group-major member list (input position, value)
//   D  members ranked by input position inside their group
// the block then adds the warp counts into the tile count U (decoupled
// look-back aggregate) and finishes the PREVIOUS tile (warp-0 look-back,
// which had a whole tile of time to resolve; coalesced ir/pr; jc per warp);
// then each warp
//   E  folds every group from +0.0 in input order (the reference's scatter
//      contract, _kernels.pyx:82-89; x86 NaN rule) and places it by row
//      inside its column, staging (row-1, value) in CSC order.
// Tiles holding a big column (folded by k_bigcol) write straight to global
// memory after an inline look-back.

#include "sa_internal.cuh"

namespace sa {

namespace {

constexpr int NT = TILE_THREADS;
constexpr int NW = TILE_WARPS;
constexpr int WSTRIDE = WIN + 1;  // per-warp column slots + sentinel

struct TileSmem {
    int4 rec[2][TCAP];                 // double-buffered records (TMA destination)
    unsigned long long mbar[2];
    // One 16-byte cell per record position k of the owning warp's range:
    // first hash slots 2k, 2k+1; after the hash is dead, group-major fields.
    union HCell {
        unsigned long long key[2];
        struct {
            double sval;               // values ordered by input position
            int midx;                  // member input positions (arrival order)
            int pad;
        } o;
    } hc[TCAP];
    double mval[TCAP];                 // member values (arrival order)
    int ga[TCAP];                      // per record: gid << 16 | arrival rank
    int crow[TCAP];                    // rows of a column's groups (column-major)
    int g_row[TCAP];                   // per group (index qa + gid)
    int16_t hgid[2 * TCAP];
    int16_t col[TCAP];                 // column heads -> column slot + 1
    int16_t g_cnt[TCAP];
    int16_t g_base[TCAP];
    int16_t g_slot[TCAP];
    int16_t g_crank[TCAP];
    int ci_c[TILE];                    // per column slot (warp w: [w*WIN, w*WIN+WIN))
    int ci_q[TILE];
    int ci_n[TILE];                    // small record count (0 for a big placeholder)
    int ci_u[TILE];                    // groups, or k_bigcol's unique count
    int cg_base[TILE];                 // warp-relative offset of the column in crow
    int cib[2][NW * WSTRIDE];          // warp-relative output offsets (+ sentinel), 2 tiles
    int w_base[2][NW];                 // warp output base inside the tile, 2 tiles
    int w_u[NW];
    int st_row[TCAP];                  // staged outputs of the pending tile
    double st_val[TCAP];
    int pre_n[2];
    int U_cur;
    long long P_bc;
    long long P_big;
    long long next_tile;
    long long p_tile;
    int p_U;
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

// Warp-level decoupled look-back (32 predecessors per L2 round trip):
// exclusive prefix of tile b; publishes b's inclusive prefix.
__device__ long long lookback_warp32(unsigned long long *st, long long b, unsigned long long agg) {
    const int lane = threadIdx.x & 31;
    volatile unsigned long long *vst = st;
    unsigned long long excl = 0;
    long long base = b - 1;
    while (base >= 0) {
        const long long idx = base - lane;
        const unsigned long long w = (idx >= 0) ? vst[idx] : lb_pack(2, 0);
        const unsigned flag = (unsigned)(w >> 62);
        if (__any_sync(FULL, flag == 0)) continue;
        const unsigned pm = __ballot_sync(FULL, flag == 2);
        const int stop = pm ? (__ffs(pm) - 1) : 31;
        unsigned long long v = (lane <= stop) ? (w & LB_VALMASK) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        excl += v;
        if (pm) break;
        base -= 32;
    }
    if (lane == 0) {
        __threadfence();
        vst[b] = lb_pack(2, excl + agg);
    }
    return (long long)excl;
}

__device__ __forceinline__ int tile_r0(const uint32_t *sstart, const int32_t *win_first,
                                       long long t) {
    return (int)(sstart[win_first[t * NW]] & POSMASK);
}

// Record prefetch of tile t into buffer buf (thread 0).
__device__ void prefetch_tile(TileSmem &S, int buf, long long t, long long ntiles,
                              const int32_t *win_first, const uint32_t *sstart, const int4 *rec) {
    S.pre_n[buf] = -1;
    if (t >= ntiles) return;
    const int r0 = tile_r0(sstart, win_first, t);
    const int r1 = (int)(sstart[win_first[(t + 1) * NW]] & POSMASK);
    const int n = r1 - r0;
    if (n > 0 && n <= TCAP) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tma_load(S.rec[buf], rec + r0, (unsigned)n * 16u, &S.mbar[buf]);
        S.pre_n[buf] = n;
    } else {
        S.pre_n[buf] = (n == 0) ? 0 : -1;
    }
}

// jc of one warp's columns: jc[c] = P + cib[first non-empty column >= c]
__device__ void warp_write_jc(const uint32_t *sstart, int c_lo, int c_hi, const int *cibw,
                              long long Pw, int32_t *jc) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt();
    int k0 = 0;
    for (int cb = c_lo; cb < c_hi; cb += 32) {
        const int c = cb + lane;
        const bool in = c < c_hi;
        int ne = 0;
        if (in) ne = (sstart[c + 1] & POSMASK) > (sstart[c] & POSMASK);
        const unsigned m = __ballot_sync(FULL, ne);
        if (in) jc[c] = (int32_t)(Pw + cibw[k0 + __popc(m & lt)]);
        k0 += __popc(m);
    }
}

// Finish a staged tile: look-back (warp 0), coalesced ir/pr, jc per warp.
__device__ void finish_staged(TileSmem &S, unsigned long long *tile_state, long long ntiles,
                              const uint32_t *sstart, const int32_t *win_first, int32_t N,
                              int32_t *jc, int32_t *ir, double *pr, int64_t cap, ErrState *err,
                              int pb) {
    const int tid = threadIdx.x, warp = tid >> 5;
    const long long pt = S.p_tile;
    const int pU = S.p_U;
    if (warp == 0) {
        const long long P = lookback_warp32(tile_state, pt, (unsigned long long)pU);
        if (tid == 0) S.P_bc = P;
    }
    __syncthreads();
    const long long P = S.P_bc;
    for (int k = tid; k < pU; k += NT) {
        const long long o = P + k;
        if (o < cap) {
            ir[o] = S.st_row[k];
            pr[o] = S.st_val[k];
        }
    }
    const int pgw = (int)(pt * NW) + warp;
    warp_write_jc(sstart, win_first[pgw], win_first[pgw + 1], &S.cib[pb][warp * WSTRIDE],
                  P + S.w_base[pb][warp], jc);
    if (pt == ntiles - 1 && tid == 0) {
        jc[N] = (int32_t)(P + pU);
        err->nnz = P + pU;
    }
    if (tid == 0 && P + pU > cap) atomicExch(&err->cap_exceeded, 1u);
}

}  // namespace

__global__ void __launch_bounds__(NT, 2) k_tile_fold(const uint32_t *__restrict__ sstart,
                                                      const int32_t *__restrict__ win_first,
                                                      const uint8_t *__restrict__ tile_big,
                                                      int64_t ntiles, const int4 *__restrict__ rec,
                                                      const BigCol *__restrict__ big_list,
                                                      const uint32_t *__restrict__ bigk,
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
        prefetch_tile(S, 0, t0, ntiles, win_first, sstart, rec);
    }
    __syncthreads();
    long long b = S.next_tile;
    int buf = 0, cb2 = 0;
    bool pending = false;

    while (b < ntiles) {
        if (tid == 0) {
            const long long t1 = atomicAdd(&err->tile_ticket, 1u);
            S.next_tile = t1;
            prefetch_tile(S, buf ^ 1, t1, ntiles, win_first, sstart, rec);
        }
        const bool has_big = tile_big[b] != 0;
        const int r0 = tile_r0(sstart, win_first, b);
        const int gw = (int)(b * NW) + warp;
        const int c_lo = win_first[gw], c_hi = win_first[gw + 1];
        const int slot0 = warp * WIN;
        int *cibw = &S.cib[cb2][warp * WSTRIDE];

        // ---- the warp's non-empty columns (lanes over columns) ------------------
        int ncw = 0;
        for (int cb = c_lo; cb < c_hi; cb += 32) {
            const int c = cb + lane;
            const bool in = c < c_hi;
            uint32_t w0 = 0, w1 = 0;
            if (in) {
                w0 = sstart[c];
                w1 = sstart[c + 1];
            }
            const int s0 = (int)(w0 & POSMASK), s1 = (int)(w1 & POSMASK);
            const bool ne = in && s1 > s0;
            const unsigned m = __ballot_sync(FULL, ne);
            if (ne) {
                const int k = ncw + __popc(m & lt);
                if (k < WIN) {
                    const int sl = slot0 + k;
                    const bool big = (w0 & BIGFLAG) != 0;
                    S.ci_c[sl] = c;
                    S.ci_q[sl] = s0 - r0;
                    S.ci_n[sl] = big ? 0 : s1 - s0;
                    S.ci_u[sl] = big ? (int)(big_list[bigk[c]].u & POSMASK) : 0;
                } else {
                    atomicExch(&err->internal, 1u);
                }
            }
            ncw += __popc(m);
        }
        ncw = min(ncw, WIN);
        int qa = 0, qb = 0;
        if (ncw) {
            qa = (int)(sstart[c_lo] & POSMASK) - r0;
            qb = (int)(sstart[c_hi] & POSMASK) - r0;
        }
        for (int p = qa + lane; p < qb; p += 32) {
            S.col[p] = 0;
            S.hc[p].key[0] = 0ull;
            S.hc[p].key[1] = 0ull;
        }
        __syncwarp();
        for (int k = lane; k < ncw; k += 32) S.col[S.ci_q[slot0 + k]] = (int16_t)(slot0 + k + 1);

        // ---- records arrive (TMA) ------------------------------------------------
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
        } else if (pn < 0 && tid == 0) {
            atomicExch(&err->internal, 1u);  // cannot happen: tiles hold small columns only
        }
        __syncwarp();

        // ---- A: slot, group, arrival rank (one pass, position order) -------------
        const int hb = 2 * qa, hn = 2 * (qb - qa);
        int ng = 0, carry = 0;
        for (int p0 = qa; p0 < qb; p0 += 32) {
            const int p = p0 + lane;
            const bool inr = p < qb;
            const int hm = inr ? (int)S.col[p] : 0;
            const int sl = max(warp_incl_max(hm), carry) - 1;
            carry = __shfl_sync(FULL, sl + 1, 31);
            const bool act = inr && S.ci_n[sl] > 0;  // skip big placeholders
            int row = 0, h = -1;
            bool leader = false;
            if (act) {
                row = R[p].x;
                const unsigned long long key = ((unsigned long long)(unsigned)sl << 32) | (unsigned)row;
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
                S.g_row[qa + g] = row;
                S.g_slot[qa + g] = (int16_t)sl;
                S.g_cnt[qa + g] = 0;
                S.g_crank[qa + g] = (int16_t)atomicAdd(&S.ci_u[sl], 1);
            }
            ng += __popc(lm);
            __syncwarp();
            const int g = act ? (int)S.hgid[h] : -1 - lane;  // unique dummy keys for idle lanes
            const unsigned peers = __match_any_sync(FULL, g);
            const int before = act ? (int)S.g_cnt[qa + g] : 0;
            __syncwarp();
            if (act) {
                const int arr = before + __popc(peers & lt);
                S.ga[p] = (g << 16) | arr;
                if ((peers & lt) == 0) S.g_cnt[qa + g] = (int16_t)(before + __popc(peers));
            } else if (inr) {
                S.ga[p] = -1;
            }
            __syncwarp();
        }

        // ---- B: group offsets, column offsets -------------------------------------
        {
            int gc = 0;
            for (int g0 = 0; g0 < ng; g0 += 32) {
                const int g = g0 + lane;
                const int v = (g < ng) ? (int)S.g_cnt[qa + g] : 0;
                const int inc = warp_incl_sum(v);
                if (g < ng) S.g_base[qa + g] = (int16_t)(gc + inc - v);
                gc += __shfl_sync(FULL, inc, 31);
            }
        }
        int Uw = 0;
        {
            int cc = 0, gcc = 0;
            for (int k0 = 0; k0 < ncw; k0 += 32) {
                const int k = k0 + lane;
                const int u = (k < ncw) ? S.ci_u[slot0 + k] : 0;
                const int gu = (k < ncw && S.ci_n[slot0 + k] > 0) ? u : 0;
                const int inc = warp_incl_sum(u);
                const int ginc = warp_incl_sum(gu);
                if (k < ncw) {
                    cibw[k] = cc + inc - u;
                    S.cg_base[slot0 + k] = gcc + ginc - gu;
                }
                cc += __shfl_sync(FULL, inc, 31);
                gcc += __shfl_sync(FULL, ginc, 31);
            }
            Uw = cc;
            if (lane == 0) cibw[ncw] = Uw;
        }
        __syncwarp();
        // ---- C: group-major members; group rows per column ---------------------
        for (int p = qa + lane; p < qb; p += 32) {
            const int ga = S.ga[p];
            if (ga < 0) continue;
            const int g = ga >> 16;
            const int j = qa + S.g_base[qa + g] + (ga & 0xffff);
            const int4 r = R[p];
            S.hc[j].o.midx = r.y;
            S.mval[j] = __hiloint2double(r.w, r.z);
        }
        for (int g = lane; g < ng; g += 32)
            S.crow[qa + S.cg_base[S.g_slot[qa + g]] + S.g_crank[qa + g]] = S.g_row[qa + g];
        __syncwarp();
        // ---- D: members ranked by input position inside their group -------------
        for (int p = qa + lane; p < qb; p += 32) {
            const int ga = S.ga[p];
            if (ga < 0) continue;
            const int g = ga >> 16;
            const int base = qa + S.g_base[qa + g];
            const int sz = S.g_cnt[qa + g];
            const int j = base + (ga & 0xffff);
            int rank = 0;
            if (sz > 1) {
                const int my = S.hc[j].o.midx;
                for (int k = base; k < base + sz; ++k) rank += (S.hc[k].o.midx < my);
            }
            S.hc[base + rank].o.sval = S.mval[j];
        }
        if (lane == 0) S.w_u[warp] = Uw;
        __syncthreads();

        // ---- tile count, aggregate ---------------------------------------------
        if (tid < 32) {
            const int v = (tid < NW) ? S.w_u[tid] : 0;
            const int inc = warp_incl_sum(v);
            if (tid < NW) S.w_base[cb2][tid] = inc - v;
            if (tid == NW - 1) {
                volatile unsigned long long *vst = tile_state;
                __threadfence();
                if (b == 0) vst[0] = lb_pack(2, (unsigned long long)inc);
                else vst[b] = lb_pack(1, (unsigned long long)inc);
                S.U_cur = inc;
            }
        }
        __syncthreads();
        const int U = S.U_cur;
        const int wbase = S.w_base[cb2][warp];

        // ---- finish the previous tile -------------------------------------------
        if (pending) {
            finish_staged(S, tile_state, ntiles, sstart, win_first, N, jc, ir, pr, cap, err, cb2 ^ 1);
            pending = false;
        }
        long long P = 0;
        if (has_big) {
            if (warp == 0) {
                const long long Pb = lookback_warp32(tile_state, b, (unsigned long long)U);
                if (tid == 0) S.P_big = Pb;
            }
        }
        __syncthreads();
        if (has_big) P = S.P_big;

        // ---- E: fold each group in input order, place it by row ------------------
        bool over = false;
        for (int g = lane; g < ng; g += 32) {
            const int row = S.g_row[qa + g];
            const int sl = S.g_slot[qa + g];
            const int cl = qa + S.cg_base[sl];
            const int cu = S.ci_u[sl];
            int rank = 0;
            for (int k = cl; k < cl + cu; ++k) rank += (S.crow[k] < row);
            const int base = qa + S.g_base[qa + g];
            const int sz = S.g_cnt[qa + g];
            double acc = 0.0;
            for (int k = base; k < base + sz; ++k) acc = fold_add(acc, S.hc[k].o.sval);
            const int o = wbase + cibw[sl - slot0] + rank;  // tile-local output index
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
            for (int k = 0; k < ncw; ++k) {  // big columns of this warp: k_bigcol's results
                const int sl = slot0 + k;
                if (S.ci_n[sl] != 0) continue;
                const BigCol bc = big_list[bigk[S.ci_c[sl]]];
                const int ub = (int)(bc.u & POSMASK);
                const unsigned long long *RR = reinterpret_cast<const unsigned long long *>(rec + bc.start);
                const unsigned long long *K = (bc.u & BIGFLAG) ? RR + bc.n : RR;
                const unsigned long long *V = (bc.u & BIGFLAG) ? RR : RR + bc.n;
                const long long ob = P + wbase + cibw[k];
                for (int e = lane; e < ub; e += 32) {
                    if (ob + e < cap) {
                        ir[ob + e] = (int32_t)K[e];
                        pr[ob + e] = __longlong_as_double((long long)V[e]);
                    } else {
                        over = true;
                    }
                }
            }
            if (over) atomicExch(&err->cap_exceeded, 1u);
            warp_write_jc(sstart, c_lo, c_hi, cibw, P + wbase, jc);
            if (b == ntiles - 1 && tid == 0) {
                jc[N] = (int32_t)(P + U);
                err->nnz = P + U;
                if (P + U > cap) atomicExch(&err->cap_exceeded, 1u);
            }
        } else {
            if (tid == 0) {
                S.p_tile = b;
                S.p_U = U;
            }
            pending = true;
            cb2 ^= 1;
        }
        __syncthreads();
        b = S.next_tile;
        buf ^= 1;
    }
    if (pending) finish_staged(S, tile_state, ntiles, sstart, win_first, N, jc, ir, pr, cap, err, cb2 ^ 1);
}

cudaError_t launch_tile_fold(Launch &lc, const uint32_t *sstart, const int32_t *win_first,
                             const uint8_t *tile_big, int64_t ntiles, const int4 *rec,
                             const BigCol *big_list, const uint32_t *bigk,
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
    k_tile_fold<<<(unsigned)grid, NT, smem, lc.stream>>>(sstart, win_first, tile_big, ntiles, rec,
                                                        big_list, bigk, tile_state, N, jc, ir, pr,
                                                        cap, err);
    lc.launches++;
    return cudaGetLastError();
}

}  // namespace sa
