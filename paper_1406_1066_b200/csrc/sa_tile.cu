// sa_tile.cu -- k_tile_fold: the ordered segmented fold (sm_100a).
//
// Input: 16-byte records {row, input position, value} grouped by column
// (k_scatter) in the small record space; sstart[c] = small-space start of
// column c (| BIGFLAG for a big column, which occupies one placeholder
// slot); tile_info[t] = {first column of tile t, its start}.  Thread tid
// owns the columns starting in its window of WIN = 16 record positions.
// Output: jc, ir, pr.
//
// One CTA per tile (TILE = 2048 record positions, ticket order for
// forward progress); the tile's records arrive by one TMA bulk copy
// (cp.async.bulk) into shared memory.  Then every THREAD owns the columns
// starting in its window and folds each of them alone -- a column is short
// (FEM: 18 / 93 triplets), and ~1e6 independent columns hide the latency of
// thread-sequential shared-memory code while keeping every lane busy:
//   * short columns (<= 24 records): insertion sort of the records by
//     (row, input position), then one pass that folds each run of equal rows
//   * longer columns: row selection -- per distinct row (ascending), gather
//     its records to the front, insertion-sorted by input position, fold
// Each fold starts from +0.0 and adds in ascending input position (the
// reference's scatter contract, _kernels.pyx:82-89; x86 NaN rule,
// fold_add).  Results are written in place (row-1, value), compacted to the
// column's front.  A block scan of the per-thread unique counts gives the
// tile count U (decoupled look-back, warp 0) and each thread's output base;
// outputs are staged in CSC order and written coalesced.  Tiles holding a
// big column (folded by k_bigcol) copy its results from the big space.

#include <cstdlib>

#include "sa_internal.cuh"
#include "sa_network.cuh"

namespace sa {

namespace {

constexpr int NT = TILE_THREADS;
constexpr int SHORT_COL = 24;

constexpr int NWARP = NT / 32;
constexpr int LCAP = TILE / (SHORT_COL + 1) + 2;  // long columns per tile
constexpr int SCAP = 256;                         // staged column starts per tile
constexpr int MAXU = 96;                          // distinct rows of a long column (warp table)

struct WarpScratchGroups {
    uint8_t gid[BIGCOL];               // group (table entry) of each record
    int16_t arr[BIGCOL];               // arrival rank inside the group
    int16_t mem[BIGCOL];               // group-major member list (record slots)
    int gcnt[MAXU];
    int gbase[MAXU];
};
union WarpScratch {
    WarpScratchGroups g;               // fold_column_warp (fallback)
    unsigned long long skey[256];      // fold_column_bitonic: sorted keys
};

template <int NBUF>
struct TileSmem {
    int4 rec[NBUF][TCAP];              // tile records {row, position, value} (NBUF buffers)
    uint8_t perm[TCAP];                // per column: sorted order, then output slots
    WarpScratch ws[NWARP];
    int lcol[LCAP];                    // long columns: record offset | (count << 16)
    uint32_t scol[NBUF][SCAP];         // sstart of the tile's columns (when they fit)
    int nlong;
    int warp_u[NWARP];
    long long P;
};

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// Ampere-style asynchronous copies (LDGSTS): the gathered row / value of a
// record land in shared memory without passing through registers, so a
// tile's gather is in flight while the previous tile is folded.
__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// (row, position) order of two records (both non-negative int32)
__device__ __forceinline__ unsigned long long rec_key(const int4 &a) {
    return ((unsigned long long)(unsigned)a.x << 32) | (unsigned)a.y;
}
__device__ __forceinline__ bool rec_less(const int4 &a, const int4 &b) {
    return rec_key(a) < rec_key(b);
}

__device__ __forceinline__ double rec_val(const int4 &r) { return __hiloint2double(r.w, r.z); }

// Fold one column of c records in place; returns the number of distinct rows
// u; R[0..u) then hold {row-1, -, value} in ascending row order.
__device__ int fold_column(int4 *R, int c) {
    if (c <= SHORT_COL) {
        // insertion sort by (row, position)
        for (int i = 1; i < c; ++i) {
            const int4 x = R[i];
            int j = i;
            while (j > 0) {
                const int4 y = R[j - 1];
                if (!rec_less(x, y)) break;
                R[j] = y;
                --j;
            }
            R[j] = x;
        }
        int u = 0;
        int k = 0;
        while (k < c) {
            const int row = R[k].x;
            double acc = fold_add(0.0, rec_val(R[k]));
            int e = k + 1;
            while (e < c) {
                const int4 y = R[e];
                if (y.x != row) break;
                acc = fold_add(acc, rec_val(y));
                ++e;
            }
            R[u] = make_int4(row - 1, 0, __double2loint(acc), __double2hiint(acc));
            ++u;
            k = e;
        }
        R[0].y = u;  // the column's output count travels with its outputs
        return u;
    }
    // row selection: per distinct row, ascending
    int u = 0;
    int k = 0;
    while (k < c) {
        int m = R[k].x;
        for (int i = k + 1; i < c; ++i) m = min(m, R[i].x);
        int g = 0;
        for (int i = k; i < c; ++i) {
            const int4 x = R[i];
            if (x.x != m) continue;
            if (k + g < i) R[i] = R[k + g];
            int j = k + g;
            while (j > k) {
                const int4 y = R[j - 1];
                if (y.y < x.y) break;
                R[j] = y;
                --j;
            }
            R[j] = x;
            ++g;
        }
        double acc = 0.0;
        for (int i = k; i < k + g; ++i) acc = fold_add(acc, rec_val(R[i]));
        R[u] = make_int4(m - 1, 0, __double2loint(acc), __double2hiint(acc));
        ++u;
        k += g;
    }
    R[0].y = u;
    return u;
}

// Short column (c <= W records): static Batcher sorting network on the
// (row, position) keys held in registers -- compare-exchanges within a layer
// are independent, so the sort runs at instruction throughput.  The key is
// packed with the record slot so a compare-exchange is a min/max pair:
//   32-bit  (row - rmin) | (pos - pmin) | slot   when the spans fit 27 bits
//   64-bit  row | (pos - pmin) | slot            when the position span fits 27
//   64-bit  row | pos, slot carried separately   otherwise
// Writes the sorted order (record slots) to perm and returns the number of
// distinct rows u; the values are folded later (fold_from_perm).
__device__ __forceinline__ int span_bits(unsigned x) { return x ? 32 - __clz(x) : 0; }

template <int W, typename K>
__device__ __forceinline__ void run_network(K (&k)[W]) {
#define SA_CE(i, j)                         \
    {                                       \
        const K lo_ = k[i] < k[j] ? k[i] : k[j]; \
        const K hi_ = k[i] < k[j] ? k[j] : k[i]; \
        k[i] = lo_;                         \
        k[j] = hi_;                         \
    }
    if constexpr (W == 8) {
        SA_NET8(SA_CE)
    } else if constexpr (W == 12) {
        SA_NET12(SA_CE)
    } else if constexpr (W == 16) {
        SA_NET16(SA_CE)
    } else if constexpr (W == 18) {
        SA_NET18(SA_CE)
    } else {
        SA_NET24(SA_CE)
    }
#undef SA_CE
}

template <int W>
__device__ int fold_short_net(const int4 *R, int c, uint8_t *perm) {
    int rowv[W], posv[W];
    unsigned rmin = 0xffffffffu, rmax = 0u, pmin = 0xffffffffu, pmax = 0u;
#pragma unroll
    for (int w = 0; w < W; ++w) {
        if (w < c) {
            const int2 kk = *reinterpret_cast<const int2 *>(&R[w]);
            rowv[w] = kk.x;
            posv[w] = kk.y;
            rmin = min(rmin, (unsigned)kk.x);
            rmax = max(rmax, (unsigned)kk.x);
            pmin = min(pmin, (unsigned)kk.y);
            pmax = max(pmax, (unsigned)kk.y);
        } else {
            rowv[w] = 0;
            posv[w] = 0;
        }
    }
    const int rb = span_bits(rmax - rmin), pb = span_bits(pmax - pmin);
    int u = 1;
    if (rb + pb <= 27) {
        const int sh = pb + 5;
        unsigned k[W];
#pragma unroll
        for (int w = 0; w < W; ++w)
            k[w] = (w < c) ? (unsigned)(((unsigned long long)((unsigned)rowv[w] - rmin) << sh) |
                                        (((unsigned)posv[w] - pmin) << 5) | w)
                           : 0xffffffffu;
        run_network<W, unsigned>(k);
#pragma unroll
        for (int w = 0; w < W; ++w) {
            if (w < c) perm[w] = (uint8_t)(k[w] & 31u);
            if (w > 0 && w < c && ((unsigned long long)k[w] >> sh) != ((unsigned long long)k[w - 1] >> sh)) ++u;
        }
    } else if (pb <= 27) {
        unsigned long long k[W];
#pragma unroll
        for (int w = 0; w < W; ++w)
            k[w] = (w < c) ? (((unsigned long long)(unsigned)rowv[w] << 32) |
                              ((((unsigned)posv[w] - pmin) << 5) | w))
                           : ~0ull;
        run_network<W, unsigned long long>(k);
#pragma unroll
        for (int w = 0; w < W; ++w) {
            if (w < c) perm[w] = (uint8_t)(k[w] & 31u);
            if (w > 0 && w < c && (k[w] >> 32) != (k[w - 1] >> 32)) ++u;
        }
    } else {
        // full (row, position) keys with the slot carried alongside
        unsigned long long k[W];
        int sl[W];
#pragma unroll
        for (int w = 0; w < W; ++w) {
            k[w] = (w < c) ? (((unsigned long long)(unsigned)rowv[w] << 32) | (unsigned)posv[w])
                           : ~0ull - (unsigned long long)(W - w);
            sl[w] = w;
        }
#define SA_CE(i, j)                                            \
    {                                                          \
        const bool sw = k[j] < k[i];                           \
        const unsigned long long lo_ = sw ? k[j] : k[i];       \
        const unsigned long long hi_ = sw ? k[i] : k[j];       \
        const int sa_ = sw ? sl[j] : sl[i];                    \
        const int sb_ = sw ? sl[i] : sl[j];                    \
        k[i] = lo_;                                            \
        k[j] = hi_;                                            \
        sl[i] = sa_;                                           \
        sl[j] = sb_;                                           \
    }
        if constexpr (W == 8) {
            SA_NET8(SA_CE)
        } else if constexpr (W == 12) {
            SA_NET12(SA_CE)
        } else if constexpr (W == 16) {
            SA_NET16(SA_CE)
        } else if constexpr (W == 18) {
            SA_NET18(SA_CE)
        } else {
            SA_NET24(SA_CE)
        }
#undef SA_CE
#pragma unroll
        for (int w = 0; w < W; ++w) {
            if (w < c) perm[w] = (uint8_t)sl[w];
            if (w > 0 && w < c && (k[w] >> 32) != (k[w - 1] >> 32)) ++u;
        }
    }
    return u;
}

// Fold a short column from its sorted order: each run of equal rows from
// +0.0 in input-position order.  A run's output (row-1, value) is stored in
// the slot of the run's first record (already read, never read again),
// with un (the column's output count) in its .y, and perm[j] becomes the
// slot of output j.
__device__ void fold_from_perm(int4 *R, uint8_t *perm, int c, int un) {
    int head = perm[0];
    int4 x = R[head];
    int prev = x.x;
    double acc = fold_add(0.0, rec_val(x));
    int u = 0;
    for (int w = 1; w < c; ++w) {
        const int sl = perm[w];
        const int4 y = R[sl];
        if (y.x != prev) {
            R[head] = make_int4(prev - 1, un, __double2loint(acc), __double2hiint(acc));
            perm[u++] = (uint8_t)head;
            head = sl;
            prev = y.x;
            acc = fold_add(0.0, rec_val(y));
        } else {
            acc = fold_add(acc, rec_val(y));
        }
    }
    R[head] = make_int4(prev - 1, un, __double2loint(acc), __double2hiint(acc));
    perm[u] = (uint8_t)head;
}

__device__ __forceinline__ int warp_incl_sum(int x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

__device__ __forceinline__ int tab_get(const int (&tab)[3], int k) {
    return (k == 0) ? tab[0] : ((k == 1) ? tab[1] : tab[2]);
}

// Warp-cooperative fold of one column with c > SHORT_COL records (all 32
// lanes call it; returns u, warp-uniform).  Lanes hold a table of the
// column's distinct rows (entry t in lane t%32); each batch of 32 records
// looks its rows up by shuffles, appends new rows, and takes arrival ranks
// in position order (match.any; deterministic).  Then per group (lane per
// group): members ordered by input position, folded from +0.0, placed by row.
// More than MAXU distinct rows: lane 0 folds the column alone.
__device__ int fold_column_warp(int4 *R, int c, WarpScratchGroups &W) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt();
    int tab[3] = {0, 0, 0};
    int u = 0;
    bool overflow = false;
    for (int t = lane; t < MAXU; t += 32) W.gcnt[t] = 0;
    __syncwarp();
    for (int b0 = 0; b0 < c && !overflow; b0 += 32) {
        const int i = b0 + lane;
        const bool act = i < c;
        const int r = act ? R[i].x : -1;
        int gid = -1;
        for (int t = 0; t < u; ++t) {
            const int rt = __shfl_sync(FULL, tab_get(tab, t >> 5), t & 31);
            if (r == rt) gid = t;
        }
        unsigned miss = __ballot_sync(FULL, act && gid < 0);
        while (miss) {
            if (u >= MAXU) {
                overflow = true;
                break;
            }
            const int rl = __shfl_sync(FULL, r, __ffs(miss) - 1);
            if (act && gid < 0 && r == rl) gid = u;
            if (lane == (u & 31)) {
                const int k = u >> 5;
                if (k == 0) tab[0] = rl;
                else if (k == 1) tab[1] = rl;
                else tab[2] = rl;
            }
            ++u;
            miss = __ballot_sync(FULL, act && gid < 0);
        }
        if (overflow) break;
        const unsigned peers = __match_any_sync(FULL, act ? gid : -1 - lane);
        const int leader = __ffs(peers) - 1;
        int base = 0;
        if (act && lane == leader) base = atomicAdd(&W.gcnt[gid], __popc(peers));
        base = __shfl_sync(FULL, base, leader);
        if (act) {
            W.gid[i] = (uint8_t)gid;
            W.arr[i] = (int16_t)(base + __popc(peers & lt));
        }
    }
    if (overflow) {
        int uu = 0;
        if (lane == 0) uu = fold_column(R, c);
        __syncwarp();
        return __shfl_sync(FULL, uu, 0);
    }
    __syncwarp();
    {
        int carry = 0;
        for (int t0 = 0; t0 < u; t0 += 32) {
            const int t = t0 + lane;
            const int v = (t < u) ? W.gcnt[t] : 0;
            const int inc = warp_incl_sum(v);
            if (t < u) W.gbase[t] = carry + inc - v;
            carry += __shfl_sync(FULL, inc, 31);
        }
    }
    __syncwarp();
    for (int i = lane; i < c; i += 32) W.mem[W.gbase[W.gid[i]] + W.arr[i]] = (int16_t)i;
    __syncwarp();
    // rank of every record inside its group by input position:
    // small groups -- each record compares against its group's members
    for (int i = lane; i < c; i += 32) {
        const int t = W.gid[i];
        const int g = W.gcnt[t];
        if (g > 8) continue;
        int rank = 0;
        if (g > 1) {
            const int base = W.gbase[t], my = R[i].y;
            for (int k = 0; k < g; ++k) rank += (R[W.mem[base + k]].y < my);
        }
        W.arr[i] = (int16_t)rank;
    }
    // large groups -- the whole warp, member positions exchanged by shuffles
    for (int t = 0; t < u; ++t) {
        const int g = W.gcnt[t];
        if (g <= 8) continue;
        const int base = W.gbase[t];
        if (g <= 32) {
            const int sl = (lane < g) ? (int)W.mem[base + lane] : 0;
            const int my = (lane < g) ? R[sl].y : 0x7fffffff;
            int rank = 0;
            for (int m = 0; m < g; ++m) rank += (__shfl_sync(FULL, my, m) < my);
            if (lane < g) W.arr[sl] = (int16_t)rank;
        } else {
            for (int k = lane; k < g; k += 32) {
                const int sl = W.mem[base + k];
                const int my = R[sl].y;
                int rank = 0;
                for (int m = 0; m < g; ++m) rank += (R[W.mem[base + m]].y < my);
                W.arr[sl] = (int16_t)rank;
            }
        }
    }
    __syncwarp();
    // group-major list in input-position order
    for (int i = lane; i < c; i += 32) W.mem[W.gbase[W.gid[i]] + W.arr[i]] = (int16_t)i;
    __syncwarp();
    double acc[3] = {0.0, 0.0, 0.0};
    int rank[3] = {0, 0, 0};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int t = lane + 32 * k;
        if (t < u) {
            const int base = W.gbase[t], g = W.gcnt[t];
            double sacc = 0.0;
            for (int a = base; a < base + g; ++a) sacc = fold_add(sacc, rec_val(R[W.mem[a]]));
            acc[k] = sacc;
        }
    }
    for (int t2 = 0; t2 < u; ++t2) {
        const int rt = __shfl_sync(FULL, tab_get(tab, t2 >> 5), t2 & 31);
#pragma unroll
        for (int k = 0; k < 3; ++k) rank[k] += (rt < tab[k]);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int t = lane + 32 * k;
        if (t < u) R[rank[k]] = make_int4(tab[k] - 1, u, __double2loint(acc[k]), __double2hiint(acc[k]));
    }
    __syncwarp();
    return u;
}

// Warp-wide bitonic sort of 32*E 64-bit keys, blocked layout (lane holds
// elements lane*E .. lane*E+E-1): partner distances >= E are shuffles,
// shorter ones are register compare-exchanges.
template <int E>
__device__ __forceinline__ void warp_bitonic(unsigned long long (&k)[E]) {
    const int lane = threadIdx.x & 31;
    constexpr int P = 32 * E;
#pragma unroll
    for (int size = 2; size <= P; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride >= E) {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int i = lane * E + e;
                    const unsigned long long o = __shfl_xor_sync(FULL, k[e], stride / E);
                    const bool up = (i & size) == 0;
                    const bool lower = (i & stride) == 0;
                    const bool take = (lower == up) ? (o < k[e]) : (k[e] < o);
                    k[e] = take ? o : k[e];
                }
            } else {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int q = e ^ stride;
                    if (q > e) {
                        const bool up = ((lane * E + e) & size) == 0;
                        const unsigned long long a = k[e], b = k[q];
                        const bool sw = up ? (b < a) : (a < b);
                        k[e] = sw ? b : a;
                        k[q] = sw ? a : b;
                    }
                }
            }
        }
    }
}

// Warp-cooperative fold of one column of c (<= 32*E) records: one bitonic
// sort of the packed key (row - rmin) << (PB+SB) | (pos - pmin) << SB | slot
// puts the records in (row, input position) order; the lane holding a run
// head folds the run of equal rows from +0.0 in that order (the reference's
// order, _kernels.pyx:82-89).  Outputs (row-1, u, value) at R[0..u).
// Returns u, or -1 (nothing written) when the spans do not fit 64 bits.
template <int E>
__device__ int fold_column_bitonic(int4 *R, int c, unsigned long long *skey) {
    constexpr int SB = (E == 1) ? 5 : (E == 2) ? 6 : (E == 4) ? 7 : (E == 8) ? 8 : 9;
    const int lane = threadIdx.x & 31;
    int2 rp[E];
    unsigned rmin = 0xffffffffu, rmax = 0u, pmin = 0xffffffffu, pmax = 0u;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = lane * E + e;
        rp[e] = (i < c) ? *reinterpret_cast<const int2 *>(&R[i]) : make_int2(0, 0);
        if (i < c) {
            rmin = min(rmin, (unsigned)rp[e].x);
            rmax = max(rmax, (unsigned)rp[e].x);
            pmin = min(pmin, (unsigned)rp[e].y);
            pmax = max(pmax, (unsigned)rp[e].y);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        rmin = min(rmin, __shfl_xor_sync(FULL, rmin, o));
        rmax = max(rmax, __shfl_xor_sync(FULL, rmax, o));
        pmin = min(pmin, __shfl_xor_sync(FULL, pmin, o));
        pmax = max(pmax, __shfl_xor_sync(FULL, pmax, o));
    }
    const int pb = span_bits(pmax - pmin), rb = span_bits(rmax - rmin);
    if (rb + pb + SB > 63) return -1;
    const int rs = pb + SB;
    unsigned long long k[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = lane * E + e;
        k[e] = (i < c) ? ((((unsigned long long)((unsigned)rp[e].x - rmin)) << rs) |
                          ((unsigned long long)((unsigned)rp[e].y - pmin) << SB) | (unsigned)i)
                       : ~0ull;
    }
    warp_bitonic<E>(k);
#pragma unroll
    for (int e = 0; e < E; ++e)
        if (lane * E + e < c) skey[lane * E + e] = k[e];
    // run heads and their output ranks
    const unsigned long long prev_last = __shfl_up_sync(FULL, k[E - 1], 1);
    unsigned hmask = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = lane * E + e;
        const unsigned long long pk = (e > 0) ? k[e > 0 ? e - 1 : 0] : prev_last;
        if (i < c && (i == 0 || (k[e] >> rs) != (pk >> rs))) hmask |= 1u << e;
    }
    const int hc = __popc(hmask);
    int incl = hc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    const int u = __shfl_sync(FULL, incl, 31);
    int oidx = incl - hc;
    __syncwarp();
    constexpr unsigned SMASK = (1u << SB) - 1;
    double acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        acc[e] = 0.0;
        if (!(hmask & (1u << e))) continue;
        const int i = lane * E + e;
        const unsigned long long rk = k[e] >> rs;
        double sacc = fold_add(0.0, rec_val(R[(unsigned)k[e] & SMASK]));
        for (int j = i + 1; j < c; ++j) {
            const unsigned long long y = skey[j];
            if ((y >> rs) != rk) break;
            sacc = fold_add(sacc, rec_val(R[(unsigned)y & SMASK]));
        }
        acc[e] = sacc;
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; ++e) {
        if (!(hmask & (1u << e))) continue;
        const int orow = (int)(rmin + (unsigned)(k[e] >> rs));
        R[oidx] = make_int4(orow - 1, u, __double2loint(acc[e]), __double2hiint(acc[e]));
        ++oidx;
    }
    __syncwarp();
    return u;
}

// Publish tile b's aggregate (the inclusive prefix right away for tile 0).
__device__ __forceinline__ void lookback_publish(unsigned long long *st, long long b,
                                                 unsigned long long agg) {
    volatile unsigned long long *vst = st;
    vst[(b) * LB_STRIDE] = lb_pack(b == 0 ? 2 : 1, agg);
}

// Warp-level decoupled look-back (32 predecessors per L2 round trip, with
// back-off); the aggregate was published before.  Returns the exclusive
// prefix and publishes the inclusive one.
__device__ long long lookback_warp32(unsigned long long *st, long long b, unsigned long long agg) {
    const int lane = threadIdx.x & 31;
    volatile unsigned long long *vst = st;
    if (b == 0) return 0;
    unsigned long long excl = 0;
    long long base = b - 1;
    while (base >= 0) {
        const long long idx = base - lane;
        const unsigned long long w = (idx >= 0) ? vst[(idx) * LB_STRIDE] : lb_pack(2, 0);
        const unsigned flag = (unsigned)(w >> 62);
        if (__any_sync(FULL, flag == 0)) {
            __nanosleep(64);
            continue;
        }
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
        vst[(b) * LB_STRIDE] = lb_pack(2, excl + agg);
    }
    return (long long)excl;
}

// Per-tile descriptor (loaded two tiles ahead).
struct TileDesc {
    int c_a, c_b;  // first column of the tile, first column of the next tile
    int r0, n;     // small-space start, records
};

__device__ __forceinline__ TileDesc tile_desc(const int2 *__restrict__ tile_info, long long t,
                                              int64_t ntiles) {
    TileDesc d{0, 0, 0, 0};
    if (t < ntiles) {
        const int2 a = tile_info[t], b = tile_info[t + 1];
        d.c_a = a.x;
        d.c_b = b.x;
        d.r0 = a.y;
        d.n = b.y - a.y;
    }
    return d;
}

constexpr int GPT = (TCAP + NT - 1) / NT;  // record slots per thread
constexpr uint32_t NOPOS = 0xffffffffu;    // placeholder slot of a big column

// Entries {position, row} of a tile's record slots (tid + q*NT) into registers.
__device__ __forceinline__ void load_entries(const uint2 *__restrict__ perm, const TileDesc &d,
                                             uint2 (&p)[GPT]) {
    const int tid = threadIdx.x;
#pragma unroll
    for (int q = 0; q < GPT; ++q) {
        const int k = tid + q * NT;
        p[q] = (k < d.n && d.n <= TCAP) ? __ldg(perm + d.r0 + k) : make_uint2(NOPOS, 0u);
    }
}

// Gather of a tile: {row, position} by a plain store, the value by position
// asynchronously (cp.async) into R; the column starts into cs.
__device__ __forceinline__ void issue_gather(int4 *R, uint32_t *cs, const TileDesc &d,
                                             const uint2 (&p)[GPT],
                                             const double *__restrict__ sv, int64_t s_stride,
                                             const uint32_t *__restrict__ sstart) {
    const int tid = threadIdx.x;
#pragma unroll
    for (int q = 0; q < GPT; ++q) {
        const int k = tid + q * NT;
        if (k < d.n) {
            int *r = reinterpret_cast<int *>(&R[k]);
            *reinterpret_cast<int2 *>(r) = make_int2((int)p[q].y, (int)p[q].x);
            if (p[q].x != NOPOS) cp_async8(r + 2, sv + (int64_t)p[q].x * s_stride);
        }
    }
    const int ncols = d.c_b - d.c_a;
    if (ncols < SCAP)
        for (int k = tid; k <= ncols; k += NT) cp_async4(cs + k, sstart + d.c_a + k);
    cp_async_commit();
}

}  // namespace

// Persistent, software-pipelined fold: CTA g folds tiles g, g+G, g+2G, ...
// (cooperative launch, so every CTA is resident and the look-back always
// progresses).  While tile t is folded from buffer t&1, the gather of tile
// t+G is in flight into the other buffer and the positions of tile t+2G are
// loading into registers.
template <int NBUF>
__global__ void __launch_bounds__(NT, 4) k_tile_fold(const uint32_t *__restrict__ sstart,
                                                     const int2 *__restrict__ tile_info,
                                                     const uint8_t *__restrict__ tile_big,
                                                     int64_t ntiles,
                                                     const uint2 *__restrict__ perm,
                                                     const double *__restrict__ sv,
                                                     int64_t s_stride,
                                                     const int4 *__restrict__ rec,
                                                     const BigCol *__restrict__ big_list,
                                                     const uint32_t *__restrict__ bigk,
                                                     unsigned long long *tile_state, int32_t N,
                                                     int32_t *__restrict__ jc,
                                                     int32_t *__restrict__ ir,
                                                     double *__restrict__ pr, int64_t cap,
                                                     ErrState *err) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    TileSmem<NBUF> &S = *reinterpret_cast<TileSmem<NBUF> *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long G = gridDim.x;
    long long b = blockIdx.x;
    if (b >= ntiles) return;

    // prologue: gather of the first tile, positions of the second
    TileDesc d0 = tile_desc(tile_info, b, ntiles);
    TileDesc d1 = tile_desc(tile_info, b + G, ntiles);
    uint2 pn[GPT];
    load_entries(perm, d0, pn);
    issue_gather(S.rec[0], S.scol[0], d0, pn, sv, s_stride, sstart);
    load_entries(perm, d1, pn);
    bool over_cap = false;

    for (int it = 0; b < ntiles; ++it, b += G) {
        const int buf = (NBUF == 2) ? (it & 1) : 0;
        cp_async_wait_all();
        __syncthreads();  // tile b's records are in; every use of the other buffer is done
        const TileDesc d2 = tile_desc(tile_info, b + 2 * G, ntiles);
        if (NBUF == 2 && b + G < ntiles)
            issue_gather(S.rec[buf ^ 1], S.scol[buf ^ 1], d1, pn, sv, s_stride, sstart);
        load_entries(perm, d2, pn);

        int4 *R = S.rec[buf];
        const int c_a = d0.c_a, r0 = d0.r0, n = d0.n;
        const int ncols = d0.c_b - c_a;
        if (n > TCAP && tid == 0) atomicExch(&err->internal, 1u);
        const bool staged = n <= TCAP;
        const uint32_t *cs = (ncols < SCAP) ? S.scol[buf] : sstart + c_a;
        if (tid == 0) S.nlong = 0;
        __syncthreads();
        // thread tid owns the contiguous columns [k_lo, k_hi) of the tile
        const int k_lo = (int)(((long long)tid * ncols) / NT);
        const int k_hi = (int)(((long long)(tid + 1) * ncols) / NT);

        // ---- pass 1: each thread sorts its short columns; long ones are listed ----
        if (staged) {
            const int nmine = k_hi - k_lo;
            int maxcols = nmine;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) maxcols = max(maxcols, __shfl_xor_sync(FULL, maxcols, o));
            for (int k = 0; k < maxcols; ++k) {
                const int c = k_lo + k;
                int cnt = 0, off = 0;
                if (k < nmine) {
                    const uint32_t w0 = cs[c];
                    const int s0 = (int)(w0 & POSMASK), s1 = (int)(cs[c + 1] & POSMASK);
                    if (!(w0 & BIGFLAG) && s1 > s0) {
                        cnt = s1 - s0;
                        off = s0 - r0;
                    }
                }
                if (cnt > SHORT_COL) {
                    const int e = atomicAdd(&S.nlong, 1);
                    if (e < LCAP) S.lcol[e] = off | (cnt << 16);
                    else atomicExch(&err->internal, 1u);
                    cnt = 0;
                }
                int wmax = cnt;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) wmax = max(wmax, __shfl_xor_sync(FULL, wmax, o));
                if (wmax == 0) continue;
                int u = 0;
                if (wmax <= 8) {
                    if (cnt) u = fold_short_net<8>(&R[off], cnt, &S.perm[off]);
                } else if (wmax <= 12) {
                    if (cnt) u = fold_short_net<12>(&R[off], cnt, &S.perm[off]);
                } else if (wmax <= 16) {
                    if (cnt) u = fold_short_net<16>(&R[off], cnt, &S.perm[off]);
                } else if (wmax <= 18) {
                    if (cnt) u = fold_short_net<18>(&R[off], cnt, &S.perm[off]);
                } else {
                    if (cnt) u = fold_short_net<24>(&R[off], cnt, &S.perm[off]);
                }
                if (cnt) R[off].y = u;  // input positions are no longer needed
            }
        }
        __syncthreads();
        // ---- pass 2: warps fold the long columns ---------------------------------
        {
            const int nl = min(S.nlong, LCAP);
            for (int e = warp; e < nl; e += NWARP) {
                const int v = S.lcol[e];
                const int off = v & 0xffff;
                const int c = v >> 16;
                int u = -1;  // outputs at R[0..u)
                if (c <= 64) u = fold_column_bitonic<2>(&R[off], c, S.ws[warp].skey);
                else if (c <= 128) u = fold_column_bitonic<4>(&R[off], c, S.ws[warp].skey);
                else if (c <= 256) u = fold_column_bitonic<8>(&R[off], c, S.ws[warp].skey);
                if (u < 0) fold_column_warp(&R[off], c, S.ws[warp].g);
            }
        }
        __syncthreads();

        // ---- tile count and thread output bases; publish the aggregate early ------
        int ut = 0;
        for (int c = k_lo; c < k_hi; ++c) {
            const uint32_t w0 = cs[c];
            const int s0 = (int)(w0 & POSMASK), s1 = (int)(cs[c + 1] & POSMASK);
            if (w0 & BIGFLAG) ut += (int)(big_list[bigk[c_a + c]].u & POSMASK);
            else if (s1 > s0 && staged) ut += R[s0 - r0].y;
        }
        const int inc = warp_incl_sum(ut);
        if (lane == 31) S.warp_u[warp] = inc;
        __syncthreads();
        int wpre = 0, U = 0;
#pragma unroll
        for (int k = 0; k < NWARP; ++k) {
            const int v = S.warp_u[k];
            if (k < warp) wpre += v;
            U += v;
        }
        const int tbase = wpre + inc - ut;  // this thread's first output, tile-local
        if (tid == 0) lookback_publish(tile_state, b, (unsigned long long)U);

        // ---- pass 3: fold the short columns' values (predecessors publish meanwhile)
        if (staged) {
            for (int c = k_lo; c < k_hi; ++c) {
                const uint32_t w0 = cs[c];
                if (w0 & BIGFLAG) continue;
                const int s0 = (int)(w0 & POSMASK), s1 = (int)(cs[c + 1] & POSMASK);
                const int cnt = s1 - s0;
                if (cnt > 0 && cnt <= SHORT_COL)
                    fold_from_perm(&R[s0 - r0], &S.perm[s0 - r0], cnt, R[s0 - r0].y);
            }
        }
        if (warp == 0) {
            const long long P = lookback_warp32(tile_state, b, (unsigned long long)U);
            if (lane == 0) S.P = P;
        }
        __syncthreads();
        const long long P = S.P;

        // ---- outputs (each thread: its columns, contiguous) and column pointers ----
        long long o = P + tbase;
        for (int c = k_lo; c < k_hi; ++c) {
            jc[c_a + c] = (int32_t)o;
            const uint32_t w0 = cs[c];
            const int s0 = (int)(w0 & POSMASK), s1 = (int)(cs[c + 1] & POSMASK);
            if (w0 & BIGFLAG) {
                const BigCol bc = big_list[bigk[c_a + c]];
                const int ub = (int)(bc.u & POSMASK);
                const unsigned long long *RR = reinterpret_cast<const unsigned long long *>(rec + bc.start);
                const unsigned long long *K = (bc.u & BIGFLAG) ? RR + bc.n : RR;
                const unsigned long long *V = (bc.u & BIGFLAG) ? RR : RR + bc.n;
                for (int e = 0; e < ub; ++e) {
                    if (o + e < cap) {
                        ir[o + e] = (int32_t)K[e];
                        pr[o + e] = __longlong_as_double((long long)V[e]);
                    } else {
                        over_cap = true;
                    }
                }
                o += ub;
            } else if (s1 > s0 && staged) {
                const int4 *Rc = &R[s0 - r0];
                const uint8_t *pm = &S.perm[s0 - r0];
                const bool shrt = s1 - s0 <= SHORT_COL;  // short: outputs at slots pm[k]
                const int u = Rc[shrt ? pm[0] : 0].y;    // every output record carries u
                for (int k = 0; k < u; ++k) {
                    const int4 r = Rc[shrt ? pm[k] : k];
                    if (o + k < cap) {
                        ir[o + k] = r.x;
                        pr[o + k] = rec_val(r);
                    } else {
                        over_cap = true;
                    }
                }
                o += u;
            }
        }
        if (b == ntiles - 1 && tid == 0) {
            jc[N] = (int32_t)(P + U);
            err->nnz = P + U;
            if (P + U > cap) atomicExch(&err->cap_exceeded, 1u);
        }
        d0 = d1;
        d1 = d2;
    }
    cp_async_wait_all();
    if (over_cap) atomicExch(&err->cap_exceeded, 1u);
}

cudaError_t launch_tile_fold(Launch &lc, const uint32_t *sstart, const int2 *tile_info,
                             const uint8_t *tile_big, int64_t ntiles, const uint2 *perm,
                             const double *s, int64_t s_stride, const int4 *rec,
                             const BigCol *big_list, const uint32_t *bigk,
                             unsigned long long *tile_state, int32_t N, int32_t *jc, int32_t *ir,
                             double *pr, int64_t cap, ErrState *err) {
    if (ntiles <= 0) return cudaSuccess;
    // SA_FOLD_PERSIST=1: persistent double-buffered CTAs (cooperative launch);
    // default: one CTA per tile, single buffer
    static int mode = -1;
    static int occ = -1;
    if (mode < 0) {
        const char *ev = getenv("SA_FOLD_PERSIST");
        mode = (ev && ev[0] == '1') ? 1 : 0;
        cudaError_t e = cudaFuncSetAttribute(k_tile_fold<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sizeof(TileSmem<2>));
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(k_tile_fold<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(TileSmem<1>));
        if (e != cudaSuccess) return e;
        int o = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_tile_fold<2>, NT, sizeof(TileSmem<2>));
        if (e != cudaSuccess) return e;
        if (o < 1) return cudaErrorInvalidConfiguration;
        occ = o;
    }
    cudaError_t e;
    if (mode == 1) {
        const int64_t grid = std::min<int64_t>(ntiles, (int64_t)occ * lc.num_sms);
        void *args[] = {(void *)&sstart, (void *)&tile_info, (void *)&tile_big, (void *)&ntiles,
                        (void *)&perm, (void *)&s, (void *)&s_stride,
                        (void *)&rec, (void *)&big_list, (void *)&bigk, (void *)&tile_state,
                        (void *)&N, (void *)&jc, (void *)&ir, (void *)&pr, (void *)&cap, (void *)&err};
        e = cudaLaunchCooperativeKernel((const void *)k_tile_fold<2>, dim3((unsigned)grid), dim3(NT),
                                        args, sizeof(TileSmem<2>), lc.stream);
    } else {
        k_tile_fold<1><<<(unsigned)ntiles, NT, sizeof(TileSmem<1>), lc.stream>>>(
            sstart, tile_info, tile_big, ntiles, perm, s, s_stride, rec, big_list, bigk,
            tile_state, N, jc, ir, pr, cap, err);
        e = cudaGetLastError();
    }
    lc.launches++;
    return e;
}

}  // namespace sa
