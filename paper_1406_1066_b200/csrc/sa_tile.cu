// sa_tile.cu -- k_tile_fold: the ordered segmented fold (sm_100a).
//
// Input: 8-byte entries {row, input position} grouped by column (k_scatter)
// in the small record space; sstart[c] = small-space start of column c
// (| BIGFLAG for a big column, which occupies one placeholder slot);
// tile_info[t] = {first column of tile t, its start}.  Output: jc, ir, pr.
//
// One CTA (128 threads) per tile of TILE = 1792 record positions (plus the
// last column's overhang, TCAP):
//   1. one TMA bulk copy (cp.async.bulk) brings the tile's entries into
//      shared memory (keys K[k] = {row, position}); the values are gathered
//      by position with cp.async (8 bytes each, no register staging) into
//      V[k] while the short columns are already being sorted;
//   2. every thread owns a contiguous range of the tile's columns; a short
//      column (<= SHORT_COL triplets) is sorted by (row, position) with a
//      register sorting network (sa_network.cuh); longer ones go to a warp
//      each: a hash-group fold (rows grouped in a per-warp hash table,
//      members ranked by position in grouped order) when they have <= 64
//      distinct rows, else a sub-warp bitonic sort of packed 64-bit keys;
//   3. each run of equal rows is folded from +0.0 in ascending input
//      position -- the reference's scatter order (_kernels.pyx:82-89, x86 NaN
//      rule in fold_add) -- so pr is bit-exact;
//   4. a block scan of the per-thread unique counts gives the tile count U,
//      published for the decoupled look-back before the values are folded
//      (or, for long-column inputs, staged outputs chained by k_tile_emit);
//   5. an output map (tile-local CSC index -> slot) lets all threads write
//      jc / ir / pr with coalesced stores.
// The kernel dispatches on the column scan's flag: inputs without long small
// columns run a body compiled without step 2's warp paths (inline, the
// fall-through code); the long-column body is out of line.  Tiles holding a
// big column (folded by k_bigcol) copy its results from the big space.

#include <cstdlib>

#include "sa_internal.cuh"
#include "sa_network.cuh"

namespace sa {

#ifdef SA_TRACE
// per-tile timeline (tools/fold_trace.py): 8 stamps per tile, globaltimer ns
__device__ unsigned long long g_ftrace[1 << 15][8];
#define FTRACE(b, k)                                                                   \
    if (threadIdx.x == 0 && (b) < (1 << 15)) {                                         \
        unsigned long long t_;                                                         \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                        \
        g_ftrace[b][k] = t_;                                                           \
    }
#else
#define FTRACE(b, k)
#endif

#ifndef SA_FOLD_MINB
#define SA_FOLD_MINB 5  // resident CTAs per SM the fold is compiled for (96 registers)
#endif

namespace {

constexpr int NT = TILE_THREADS;
constexpr int NWARP = NT / 32;
constexpr int LCAP = TILE / (SHORT_COL + 1) + 2;  // long columns per tile
constexpr int SCAP = 256;                         // staged column starts per tile
constexpr int LONGCAP = 256;                     // warp bitonic capacity
constexpr uint32_t NOPOS = 0xffffffffu;           // placeholder slot of a big column

struct TileSmem {
    int2 kbuf[TCAP + 2];               // TMA destination (16-byte aligned start)
    double val[TCAP];                  // gathered values
    uint8_t perm[TCAP];                // per short column: sorted order, then output slots
    union {
        unsigned long long skey[NWARP][LONGCAP];  // pass 2: long columns' sorted keys
        uint16_t omap[TCAP];                       // pass 3+: tile-local output index -> slot
    };
    int lcol[4][LCAP];                 // long columns by class (<=64, <=128, <=256, fallback):
                                       // offset | (count << 16)
    int ncls[4];
    uint32_t scol[SCAP];               // sstart of the tile's columns (when they fit)
    unsigned long long mbar;
    int warp_u[NWARP];
    int warp_b[NWARP];
    long long P;
};

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
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

// Ampere-style asynchronous 8-byte copy (LDGSTS): a gathered value lands in
// shared memory without passing through registers.
__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Fallback for a long column whose (row, position) spans do not fit the
// packed bitonic key: one lane, row selection (per distinct row, ascending:
// gather its records to the front ordered by position, fold).  Outputs
// (row-1, u) in K[0..u), values in V[0..u).
__device__ __noinline__ int fold_column_serial(int2 *K, double *V, int c) {
    int u = 0;
    int k = 0;
    while (k < c) {
        int m = K[k].x;
        for (int i = k + 1; i < c; ++i) m = min(m, K[i].x);
        int g = 0;
        for (int i = k; i < c; ++i) {
            const int2 x = K[i];
            if (x.x != m) continue;
            const double xv = V[i];
            if (k + g < i) {
                K[i] = K[k + g];
                V[i] = V[k + g];
            }
            int j = k + g;
            while (j > k) {
                const int2 y = K[j - 1];
                if (y.y < x.y) break;
                K[j] = y;
                V[j] = V[j - 1];
                --j;
            }
            K[j] = x;
            V[j] = xv;
            ++g;
        }
        double acc = 0.0;
        for (int i = k; i < k + g; ++i) acc = fold_add(acc, V[i]);
        K[u] = make_int2(m - 1, 0);
        V[u] = acc;
        ++u;
        k += g;
    }
    for (int i = 0; i < u; ++i) K[i].y = u;
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
__device__ int fold_short_net(const int2 *K, int c, uint8_t *perm) {
    int rowv[W], posv[W];
    unsigned rmin = 0xffffffffu, rmax = 0u, pmin = 0xffffffffu, pmax = 0u;
#pragma unroll
    for (int w = 0; w < W; ++w) {
        if (w < c) {
            const int2 kk = K[w];
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
        const unsigned rmask = (sh >= 32) ? 0u : (~0u << sh);  // the row bits of a key
#pragma unroll
        for (int w = 0; w < W; ++w) {
            if (w < c) perm[w] = (uint8_t)(k[w] & 31u);
            if (w > 0 && w < c && ((k[w] ^ k[w - 1]) & rmask)) ++u;
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
// +0.0 in input-position order.  A run's output (row-1, u) / value is stored
// in the slot of the run's first record (already read, never read again),
// and perm[j] becomes the slot of output j; with an output map `om`, its
// tile-local slot (off + slot) goes to om[j] as well.
__device__ void fold_from_perm(int2 *K, double *V, uint8_t *perm, int c, int un, uint16_t *om,
                               int off) {
    int head = perm[0];
    int prev = K[head].x;
    double acc = fold_add(0.0, V[head]);
    int u = 0;
    for (int w = 1; w < c; ++w) {
        const int sl = perm[w];
        const int row = K[sl].x;
        const double v = V[sl];
        if (row != prev) {
            K[head] = make_int2(prev - 1, un);
            V[head] = acc;
            if (om) om[u] = (uint16_t)(off + head);
            perm[u++] = (uint8_t)head;
            head = sl;
            prev = row;
            acc = fold_add(0.0, v);
        } else {
            acc = fold_add(acc, v);
        }
    }
    K[head] = make_int2(prev - 1, un);
    V[head] = acc;
    if (om) om[u] = (uint16_t)(off + head);
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

// Bitonic sort of G*E 64-bit keys held by a group of G lanes (E per lane,
// blocked layout); 32/G groups of one warp sort independent sequences at
// once, so the shuffle latency of one is hidden behind the others.
template <int G, int E>
__device__ __forceinline__ void group_bitonic(unsigned long long (&k)[E]) {
    const int li = threadIdx.x & (G - 1);
    constexpr int P = G * E;
#pragma unroll
    for (int size = 2; size <= P; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride >= E) {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int i = li * E + e;
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
                        const bool up = ((li * E + e) & size) == 0;
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

// Up to 32/G long columns (list entries: offset | count << 16, count <=
// G*E) folded at once by one warp, G lanes per column: one group bitonic
// sort of the packed key (row - rmin) << (PB+SB) | (pos - pmin) << SB | slot,
// then the lane holding a run head folds the run of equal rows from +0.0 in
// input-position order (the reference's order, _kernels.pyx:82-89).
// Outputs (row-1, u) in K[off..off+u), values in V[off..off+u).  A column
// whose spans do not fit 64 bits is appended to `fb` instead.
template <int G, int E>
__device__ __noinline__ void fold_columns_group(int2 *K, double *V, const int *list, int count,
                                   unsigned long long *skey, int *fb, int *nfb) {
    constexpr int P = G * E;
    constexpr int SB = (P <= 32) ? 5 : (P <= 64) ? 6 : (P <= 128) ? 7 : 8;
    constexpr unsigned SMASK = (1u << SB) - 1;
    const int lane = threadIdx.x & 31, g = lane / G, li = lane & (G - 1);
    const bool has = g < count;
    const int ent = has ? list[g] : 0;
    const int off = ent & 0xffff, c = has ? (ent >> 16) : 0;
    int2 *Kc = K + off;
    double *Vc = V + off;
    unsigned long long *sk = skey + g * P;
    int2 rp[E];
    unsigned rmin = 0xffffffffu, rmax = 0u, pmin = 0xffffffffu, pmax = 0u;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = li * E + e;
        rp[e] = (i < c) ? Kc[i] : make_int2(0, 0);
        if (i < c) {
            rmin = min(rmin, (unsigned)rp[e].x);
            rmax = max(rmax, (unsigned)rp[e].x);
            pmin = min(pmin, (unsigned)rp[e].y);
            pmax = max(pmax, (unsigned)rp[e].y);
        }
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
        rmin = min(rmin, __shfl_xor_sync(FULL, rmin, o));
        rmax = max(rmax, __shfl_xor_sync(FULL, rmax, o));
        pmin = min(pmin, __shfl_xor_sync(FULL, pmin, o));
        pmax = max(pmax, __shfl_xor_sync(FULL, pmax, o));
    }
    const int pb = span_bits(pmax - pmin), rb = span_bits(rmax - rmin);
    const bool fits = rb + pb + SB <= 63;
    if (has && !fits && li == 0) {
        const int e = atomicAdd(nfb, 1);
        if (e < LCAP) fb[e] = ent;
    }
    const bool act = has && fits;
    const int rs = pb + SB;
    unsigned long long k[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = li * E + e;
        k[e] = (act && i < c) ? ((((unsigned long long)((unsigned)rp[e].x - rmin)) << rs) |
                                 ((unsigned long long)((unsigned)rp[e].y - pmin) << SB) | (unsigned)i)
                              : ~0ull;
    }
    group_bitonic<G, E>(k);
#pragma unroll
    for (int e = 0; e < E; ++e)
        if (act && li * E + e < c) sk[li * E + e] = k[e];
    // run heads and their output ranks inside the group
    const unsigned long long prev_last = __shfl_up_sync(FULL, k[E - 1], 1, G);
    unsigned hmask = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = li * E + e;
        const unsigned long long pk = (e > 0) ? k[e > 0 ? e - 1 : 0] : prev_last;
        if (act && i < c && (i == 0 || (k[e] >> rs) != (pk >> rs))) hmask |= 1u << e;
    }
    const int hc = __popc(hmask);
    int incl = hc;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o, G);
        if (li >= o) incl += y;
    }
    const int u = __shfl_sync(FULL, incl, G - 1, G);
    int oidx = incl - hc;
    __syncwarp();
    double acc[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        acc[e] = 0.0;
        if (!(hmask & (1u << e))) continue;
        const int i = li * E + e;
        const unsigned long long rk = k[e] >> rs;
        double sacc = fold_add(0.0, Vc[(unsigned)k[e] & SMASK]);
        for (int j = i + 1; j < c; ++j) {
            const unsigned long long y = sk[j];
            if ((y >> rs) != rk) break;
            sacc = fold_add(sacc, Vc[(unsigned)y & SMASK]);
        }
        acc[e] = sacc;
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; ++e) {
        if (!(hmask & (1u << e))) continue;
        const int orow = (int)(rmin + (unsigned)(k[e] >> rs));
        Kc[oidx] = make_int2(orow - 1, u);
        Vc[oidx] = acc[e];
        ++oidx;
    }
    __syncwarp();
}

// ---- hash-group fold of one long column by one warp ------------------------
// Groups the column's entries by row in a per-warp hash table instead of
// sorting them: distinct rows are ranked by counting (at most HU of them),
// each group gets its output offset, the entries are placed by group (as
// {position, entry} in the column's own key slots, free once loaded) and
// ranked inside it by input position, and one lane per group folds it from
// +0.0 in ascending position (the reference's order, _kernels.pyx:82-89).
// Far fewer instructions than the 64-bit bitonic for columns with few
// distinct rows (FEM, repeated triplets).  Returns false, leaving the column
// untouched, when it has more than HU distinct rows.
constexpr int HT = 128;  // hash slots per warp
constexpr int HU = 64;   // most distinct rows
struct HashScratch {
    int row[HT];       // slot -> row (0: empty; rows are >= 1)
    int cnt[HT];       // slot -> entries
    uint16_t off[HT];  // slot -> first entry of its group (sorted order)
    int2 dl[HU];       // distinct rows (compacted): {row, entries}
    uint8_t ds[HU];    // their slots
};
static_assert(sizeof(HashScratch) <= LONGCAP * sizeof(unsigned long long), "per-warp scratch");

__device__ __forceinline__ int row_hash(int r) { return (int)(((unsigned)r * 0x9E3779B1u) >> 25); }

// Ordered fold of one row group (members M[m0 .. m0+n), value slots in .y)
// from +0.0.  Plain adds give the bits of fold_add's x86 rule unless the sum
// turns NaN (only then can two NaN payloads meet), so the rule's select is
// kept off the dependent chain and the fold is redone exactly in that case.
__device__ __forceinline__ double fold_group_exact(const double *Vc, const int2 *M, int m0, int n) {
    double a = fold_add(0.0, Vc[M[m0].y]);
    for (int k = 1; k < n; ++k) a = fold_add(a, Vc[M[m0 + k].y]);
    return a;
}
__device__ __forceinline__ double fold_group(const double *Vc, const int2 *M, int m0, int n) {
    double a = __dadd_rn(0.0, Vc[M[m0].y]);
#pragma unroll 4
    for (int k = 1; k < n; ++k) a = __dadd_rn(a, Vc[M[m0 + k].y]);
    return (a != a) ? fold_group_exact(Vc, M, m0, n) : a;
}

__device__ bool fold_column_hash(int2 *Kc, double *Vc, int c, HashScratch &H) {
    constexpr int EPL = LONGCAP / 32;
    const int lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int k = lane; k < HT; k += 32) {
        H.row[k] = 0;
        H.cnt[k] = 0;
    }
    __syncwarp();
    const int nb = (c + 31) >> 5;
    uint32_t hs[EPL];  // slot | arrival << 8
    int pp[EPL];       // input positions
    bool over = false;
#pragma unroll
    for (int q = 0; q < EPL; ++q) {
        hs[q] = 0;
        pp[q] = 0;
        if (q < nb) {
            const int i = q * 32 + lane;
            const bool v = i < c;
            const int2 e = v ? Kc[i] : make_int2(0, 0);
            pp[q] = e.y;
            const unsigned peers = __match_any_sync(FULL, v ? e.x : 0);
            const int leader = __ffs(peers) - 1;
            // first 32 rows mostly distinct: a short column is cheaper in the
            // 4-columns-per-warp bitonic, a longer one will exceed HU rows
            if (q == 0 && c > 32) {
                const int nd = __popc(__ballot_sync(FULL, v && lane == leader));
                if (nd >= (c <= 64 ? 24 : 30)) return false;
            }
            int h = 0, a = 0;
            if (v && lane == leader) {
                h = row_hash(e.x);
                for (int probe = 0;; ++probe) {
                    const int old = atomicCAS(&H.row[h], 0, e.x);
                    if (old == 0 || old == e.x) break;
                    h = (h + 1) & (HT - 1);
                    if (probe == HT) {
                        over = true;
                        break;
                    }
                }
                a = atomicAdd(&H.cnt[h], __popc(peers));
            }
            h = __shfl_sync(FULL, h, leader);
            a = __shfl_sync(FULL, a, leader) + __popc(peers & lt);
            hs[q] = (uint32_t)h | ((uint32_t)a << 8);
        }
    }
    __syncwarp();
    // compact the distinct rows (slot order)
    int D = 0;
#pragma unroll
    for (int m = 0; m < HT / 32; ++m) {
        const int s = lane + 32 * m;
        const int r = H.row[s];
        const unsigned bal = __ballot_sync(FULL, r != 0);
        const int k = D + __popc(bal & lt);
        if (r != 0 && k < HU) {
            H.dl[k] = make_int2(r, H.cnt[s]);
            H.ds[k] = (uint8_t)s;
        }
        D += __popc(bal);
    }
    if (__any_sync(FULL, over) || D > HU) return false;
    __syncwarp();
    // rank and group offset of distinct rows lane and lane + 32
    const int ra = lane < D ? H.dl[lane].x : 0x7fffffff;
    const int rb = lane + 32 < D ? H.dl[lane + 32].x : 0x7fffffff;
    int ka = 0, kb = 0, oa = 0, ob = 0;
#pragma unroll 4
    for (int k = 0; k < D; ++k) {
        const int2 x = H.dl[k];
        if (x.x < ra) {
            ++ka;
            oa += x.y;
        }
        if (x.x < rb) {
            ++kb;
            ob += x.y;
        }
    }
    const int sa_ = lane < D ? H.ds[lane] : 0, sb_ = lane + 32 < D ? H.ds[lane + 32] : 0;
    if (lane < D) H.off[sa_] = (uint16_t)oa;
    if (lane + 32 < D) H.off[sb_] = (uint16_t)ob;
    __syncwarp();
    // members grouped by row, {position, entry}, in the column's key slots
    int2 *M = Kc;
#pragma unroll
    for (int q = 0; q < EPL; ++q) {
        const int i = q * 32 + lane;
        if (q < nb && i < c) M[H.off[hs[q] & 255] + (hs[q] >> 8)] = make_int2(pp[q], i | (int)((hs[q] & 255) << 8));
    }
    __syncwarp();
    const int na = lane < D ? H.dl[lane].y : 0, nb2 = lane + 32 < D ? H.dl[lane + 32].y : 0;
    // rank inside the group by input position, members taken in grouped
    // order (M[x] = {position, slot | group slot << 8}): consecutive lanes
    // hold members of one group, so a warp iterates about as long as its
    // own groups, and no group needs a sort
    int mp[EPL], mw[EPL];
#pragma unroll
    for (int q = 0; q < EPL; ++q) {
        const int x = q * 32 + lane;
        mp[q] = 0;
        mw[q] = -1;
        if (q < nb && x < c) {
            const int2 w = M[x];
            mp[q] = w.x;
            mw[q] = w.y;
        }
    }
    __syncwarp();  // every member word is read before the slots are written
#pragma unroll
    for (int q = 0; q < EPL; ++q) {
        if (mw[q] < 0) continue;
        const int s = mw[q] >> 8;
        const int b0 = H.off[s], n = H.cnt[s];
        const int me = mp[q];
        const int e = b0 + n;
        int r = 0;
        for (int k = b0; k < e; k += 4)  // 4 per step, the tail predicated (groups of 4-6 are common)
            r += (M[k].x < me) + (k + 1 < e && M[k + 1].x < me) + (k + 2 < e && M[k + 2].x < me) +
                 (k + 3 < e && M[k + 3].x < me);
        M[b0 + r].y = mw[q] & 255;  // (positions in .x are only read)
    }
    __syncwarp();
    // one lane per group folds it in position order
    double acc_a = 0.0, acc_b = 0.0;
    if (lane < D) {
        const int n = na;
        acc_a = fold_group(Vc, M, oa, n);
    }
    if (lane + 32 < D) {
        const int n = nb2;
        acc_b = fold_group(Vc, M, ob, n);
    }
    __syncwarp();
    if (lane < D) {
        Kc[ka] = make_int2(ra - 1, D);
        Vc[ka] = acc_a;
    }
    if (lane + 32 < D) {
        Kc[kb] = make_int2(rb - 1, D);
        Vc[kb] = acc_b;
    }
    __syncwarp();
    return true;
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
    unsigned ns = 32;  // exponential back-off: a waiting warp leaves the issue slots to others
    while (base >= 0) {
        const long long idx = base - lane;
        const unsigned long long w = (idx >= 0) ? vst[(idx) * LB_STRIDE] : lb_pack(2, 0);
        const unsigned flag = (unsigned)(w >> 62);
        if (__any_sync(FULL, flag == 0)) {
            __nanosleep(ns);
            ns = min(ns * 2, 1024u);
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

}  // namespace

// The fold of one tile.  LONGP: the input has long small columns (the
// column scan's flag); the body without the long pass is compiled on its
// own, so short-column inputs (2D FEM) run code free of its registers and
// instructions.
template <bool STAGED, bool LONGP>
__device__ __forceinline__ void tile_fold_body(const uint32_t *__restrict__ sstart,
                                                     const int2 *__restrict__ tile_info,
                                                     const uint8_t *__restrict__ tile_big,
                                                     int64_t ntiles,
                                                     const int2 *__restrict__ entries, Segs SG,
                                                     const int4 *__restrict__ rec,
                                                     const BigCol *__restrict__ big_list,
                                                     const uint32_t *__restrict__ bigk,
                                                     unsigned long long *tile_state, int32_t N,
                                                     int32_t *__restrict__ jc,
                                                     int32_t *__restrict__ ir,
                                                     double *__restrict__ pr, int64_t cap,
                                                     ErrState *err, int hash_fold,
                                                     int4 *__restrict__ stage,
                                                     int2 *__restrict__ tile_cnt) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    TileSmem &S = *reinterpret_cast<TileSmem *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long b = blockIdx.x;
    FTRACE(b, 0);
    const int2 ti0 = tile_info[b], ti1 = tile_info[b + 1];
    const int c_a = ti0.x, r0 = ti0.y;
    int n = ti1.y - r0;
    if (n > TCAP) {  // cannot happen (tiles end at column starts); keep the chain alive
        if (tid == 0) atomicExch(&err->internal, 1u);
        n = 0;
    }
    const int ncols = ti1.x - c_a;
    const bool has_big = tile_big[b] != 0;  // outputs written per thread (no output map)
    const int shift = r0 & 1;  // TMA source must be 16-byte aligned
    if (tid == 0) {
        S.ncls[0] = S.ncls[1] = S.ncls[2] = S.ncls[3] = 0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&S.mbar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (n > 0)
            tma_load(S.kbuf, entries + (r0 - shift), (unsigned)((n + shift + 1) & ~1) * 8u, &S.mbar);
    }
    const bool cs_staged = ncols < SCAP;
    if (cs_staged)
        for (int k = tid; k <= ncols; k += NT) S.scol[k] = sstart[c_a + k];
    __syncthreads();
    const uint32_t *cs = cs_staged ? S.scol : sstart + c_a;
    int2 *K = S.kbuf + shift;
    double *V = S.val;
    if (n > 0) mbar_wait(&S.mbar, 0u);
    FTRACE(b, 1);
    if (SG.nseg == 1) {  // one input array (the single-GPU path)
        const double *sv = SG.s[0];
        const int64_t st = SG.stride[0];
        for (int k = tid; k < n; k += NT) {
            const uint32_t pos = (uint32_t)K[k].y;
            if (pos != NOPOS) cp_async8(&V[k], sv + (int64_t)pos * st);
        }
    } else {
        for (int k = tid; k < n; k += NT) {
            const uint32_t pos = (uint32_t)K[k].y;
            if (pos != NOPOS) cp_async8(&V[k], seg_value(SG, (int64_t)pos));
        }
    }
    cp_async_commit();
    __syncthreads();  // every position is read before pass 1 reuses the field
    // thread tid owns the contiguous columns [k_lo, k_hi) of the tile
    const int k_lo = (int)(((long long)tid * ncols) / NT);
    const int k_hi = (int)(((long long)(tid + 1) * ncols) / NT);

    // ---- pass 1: each thread sorts its short columns (keys only); long ones are listed
    {
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
                const int cls = (cnt <= 64) ? 0 : (cnt <= 128) ? 1 : (cnt <= LONGCAP) ? 2 : 3;
                const int e = atomicAdd(&S.ncls[cls], 1);
                if (e < LCAP) S.lcol[cls][e] = off | (cnt << 16);
                else atomicExch(&err->internal, 1u);
                cnt = 0;
            }
            int wmax = cnt;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) wmax = max(wmax, __shfl_xor_sync(FULL, wmax, o));
            if (wmax == 0) continue;
            int u = 0;
            if (wmax > 16 && wmax <= 18) {  // 2D FEM columns first (the fall-through code)
                if (cnt) u = fold_short_net<18>(&K[off], cnt, &S.perm[off]);
            } else if (wmax <= 8) {
                if (cnt) u = fold_short_net<8>(&K[off], cnt, &S.perm[off]);
            } else if (wmax <= 12) {
                if (cnt) u = fold_short_net<12>(&K[off], cnt, &S.perm[off]);
            } else if (wmax <= 16) {
                if (cnt) u = fold_short_net<16>(&K[off], cnt, &S.perm[off]);
            } else {
                if (cnt) u = fold_short_net<24>(&K[off], cnt, &S.perm[off]);
            }
            if (cnt) K[off].y = u;  // input positions of a sorted column are no longer needed
        }
    }
    FTRACE(b, 2);
    cp_async_wait_all();
    __syncthreads();  // values in; long-column list complete
    FTRACE(b, 3);
    if constexpr (LONGP) {
    // ---- pass 2: warps fold the long columns: hash groups, one column per warp;
    // columns with too many distinct rows by the group bitonic, 4 / 2 / 1 per warp
    if (hash_fold && (S.ncls[0] | S.ncls[1] | S.ncls[2])) {
        const int n0 = min(S.ncls[0], LCAP), n1 = min(S.ncls[1], LCAP), n2 = min(S.ncls[2], LCAP);
        HashScratch &H = *reinterpret_cast<HashScratch *>(S.skey[warp]);
        for (int t = warp; t < n0 + n1 + n2; t += NWARP) {
            int *ent = (t < n0) ? &S.lcol[0][t] : (t < n0 + n1) ? &S.lcol[1][t - n0]
                                                               : &S.lcol[2][t - n0 - n1];
            const int v = *ent;
            const bool ok = fold_column_hash(&K[v & 0xffff], &V[v & 0xffff], v >> 16, H);
            if (!ok && lane == 0) *ent = v | (int)0x80000000u;  // left for the bitonic
        }
        __syncthreads();
        if (warp < 3) {  // keep only the marked entries, in order
            const int n = min(S.ncls[warp], LCAP);
            int kept = 0;
            for (int base = 0; base < n; base += 32) {
                const int e = (base + lane < n) ? S.lcol[warp][base + lane] : 0;
                const unsigned bal = __ballot_sync(FULL, e < 0);
                __syncwarp();
                if (e < 0) S.lcol[warp][kept + __popc(bal & lanemask_lt())] = e & 0x7fffffff;
                kept += __popc(bal);
            }
            if (lane == 0) S.ncls[warp] = kept;
        }
        __syncthreads();
    }
    {
        const int n0 = min(S.ncls[0], LCAP), n1 = min(S.ncls[1], LCAP), n2 = min(S.ncls[2], LCAP);
        const int b0 = (n0 + 3) / 4, b1 = (n1 + 1) / 2;
        for (int t = warp; t < b0 + b1 + n2; t += NWARP) {
            if (t < b0)
                fold_columns_group<8, 8>(K, V, &S.lcol[0][4 * t], min(4, n0 - 4 * t), S.skey[warp],
                                         S.lcol[3], &S.ncls[3]);
            else if (t < b0 + b1)
                fold_columns_group<16, 8>(K, V, &S.lcol[1][2 * (t - b0)], min(2, n1 - 2 * (t - b0)),
                                          S.skey[warp], S.lcol[3], &S.ncls[3]);
            else
                fold_columns_group<32, 8>(K, V, &S.lcol[2][t - b0 - b1], 1, S.skey[warp], S.lcol[3],
                                          &S.ncls[3]);
        }
    }
    __syncthreads();
    {  // columns whose spans do not fit the packed key (and counts above LONGCAP)
        const int nf = min(S.ncls[3], LCAP);
        for (int e = tid; e < nf; e += NT) {
            const int v = S.lcol[3][e];
            fold_column_serial(&K[v & 0xffff], &V[v & 0xffff], v >> 16);
        }
    }
    __syncthreads();

    }  // LONGP
    // ---- tile count and thread output bases; publish the aggregate early ------
    int ut = 0, bt = 0;  // outputs of this thread's columns; of its big columns
    for (int c = k_lo; c < k_hi; ++c) {
        const uint32_t w0 = cs[c];
        const int s0 = (int)(w0 & POSMASK), s1 = (int)(cs[c + 1] & POSMASK);
        if (w0 & BIGFLAG) {
            const int ub = (int)(big_list[bigk[c_a + c]].u & POSMASK);
            ut += ub;
            if (STAGED) bt += ub;
        } else if (s1 > s0) {
            ut += K[s0 - r0].y;
        }
    }
    const int inc = warp_incl_sum(ut);
    const int incb = (STAGED && has_big) ? warp_incl_sum(bt) : 0;
    if (lane == 31) {
        S.warp_u[warp] = inc;
        S.warp_b[warp] = incb;
    }
    __syncthreads();
    int wpre = 0, U = 0, bpre = 0, UB = 0;
#pragma unroll
    for (int k = 0; k < NWARP; ++k) {
        const int v = S.warp_u[k], vb = S.warp_b[k];
        if (k < warp) {
            wpre += v;
            bpre += vb;
        }
        U += v;
        UB += vb;
    }
    const int tbase = wpre + inc - ut;  // this thread's first output, tile-local
    // staged: this thread's first small-column output among the tile's staged ones
    const int sbase = tbase - (bpre + incb - bt);
    if (tid == 0) {
        if (STAGED) tile_cnt[b] = make_int2(U, U - UB);
        lookback_publish(tile_state, b, (unsigned long long)U);
    }
    FTRACE(b, 4);

    // ---- pass 3: fold the short columns' values; output map -------------------
    {
        int o = tbase;
        for (int c = k_lo; c < k_hi; ++c) {
            const uint32_t w0 = cs[c];
            if (w0 & BIGFLAG) continue;
            const int s0 = (int)(w0 & POSMASK), s1 = (int)(cs[c + 1] & POSMASK);
            const int cnt = s1 - s0;
            if (cnt <= 0) continue;
            const int off = s0 - r0;
            const int u = K[off].y;
            if (cnt <= SHORT_COL)  // (writes the output map itself)
                fold_from_perm(&K[off], &V[off], &S.perm[off], cnt, u, has_big ? nullptr : &S.omap[o], off);
            else if (!has_big)
                for (int k = 0; k < u; ++k) S.omap[o + k] = (uint16_t)(off + k);
            o += u;
        }
    }
    FTRACE(b, 5);
    if (warp == 0) {  // staged: tile-local outputs, k_tile_emit adds the tile offset
        const long long P = STAGED ? 0 : lookback_warp32(tile_state, b, (unsigned long long)U);
        if (lane == 0) S.P = P;
    }
    __syncthreads();
    const long long P = S.P;
    FTRACE(b, 6);

    // ---- column pointers and, in tiles with a big column, all outputs per thread
    bool over = false;
    // big columns are copied by the whole CTA below: (tile-local output base,
    // big-list index) pairs in the (now free) long-column lists
    int *bcopy = &S.lcol[0][0];
    constexpr int BCAP = (int)(sizeof(S.lcol) / (2 * sizeof(int)));
    if (tid == 0) S.ncls[0] = 0;
    __syncthreads();
    {
        long long o = P + tbase;
        int so = sbase;  // staged index of the next small-column output
        for (int c = k_lo; c < k_hi; ++c) {
            jc[c_a + c] = (int32_t)o;
            const uint32_t w0 = cs[c];
            const int s0 = (int)(w0 & POSMASK), s1 = (int)(cs[c + 1] & POSMASK);
            if (w0 & BIGFLAG) {
                const uint32_t kb = bigk[c_a + c];
                const BigCol bc = big_list[kb];
                const int ub = (int)(bc.u & POSMASK);
                if (STAGED) {  // copied by k_tile_emit
                    o += ub;
                    continue;
                }
                const int e = atomicAdd(&S.ncls[0], 1);
                if (e < BCAP) {
                    bcopy[2 * e] = (int)(o - P);
                    bcopy[2 * e + 1] = (int)kb;
                } else {  // (more big columns in one tile than list slots) copy alone
                    const unsigned long long *RR = reinterpret_cast<const unsigned long long *>(rec + bc.start);
                    const unsigned long long *BK = (bc.u & BIGFLAG) ? RR + bc.n : RR;
                    const unsigned long long *BV = (bc.u & BIGFLAG) ? RR : RR + bc.n;
                    for (int q = 0; q < ub; ++q) {
                        if (o + q < cap) {
                            ir[o + q] = (int32_t)BK[q];
                            pr[o + q] = __longlong_as_double((long long)BV[q]);
                        } else {
                            over = true;
                        }
                    }
                }
                o += ub;
            } else if (s1 > s0) {
                const int off = s0 - r0;
                const int u = K[off].y;
                if (STAGED && has_big) {
                    const bool shrt = s1 - s0 <= SHORT_COL;
                    for (int k = 0; k < u; ++k) {
                        const int sl = off + (shrt ? S.perm[off + k] : k);
                        const long long vb = __double_as_longlong(V[sl]);
                        stage[r0 + so + k] = make_int4(K[sl].x, (int)(unsigned)vb,
                                                       (int)(unsigned)(vb >> 32), (int)(o + k));
                    }
                    so += u;
                } else if (has_big) {
                    const bool shrt = s1 - s0 <= SHORT_COL;
                    for (int k = 0; k < u; ++k) {
                        const int sl = off + (shrt ? S.perm[off + k] : k);
                        if (o + k < cap) {
                            ir[o + k] = K[sl].x;
                            pr[o + k] = V[sl];
                        } else {
                            over = true;
                        }
                    }
                }
                o += u;
            }
        }
    }
    __syncthreads();
    {  // the tile's big columns, each copied by all threads
        const int nb = min(S.ncls[0], BCAP);
        for (int e = 0; e < nb; ++e) {
            const long long o = P + bcopy[2 * e];
            const BigCol bc = big_list[bcopy[2 * e + 1]];
            const int ub = (int)(bc.u & POSMASK);
            const unsigned long long *RR = reinterpret_cast<const unsigned long long *>(rec + bc.start);
            const unsigned long long *BK = (bc.u & BIGFLAG) ? RR + bc.n : RR;
            const unsigned long long *BV = (bc.u & BIGFLAG) ? RR : RR + bc.n;
            for (int q0 = 0; q0 < ub; q0 += 8 * NT) {  // 8 loads per thread in flight
                unsigned long long kk[8], vv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int q = q0 + u * NT + tid;
                    kk[u] = (q < ub) ? BK[q] : 0ull;
                    vv[u] = (q < ub) ? BV[q] : 0ull;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int q = q0 + u * NT + tid;
                    if (q >= ub) continue;
                    if (o + q < cap) {
                        ir[o + q] = (int32_t)kk[u];
                        pr[o + q] = __longlong_as_double((long long)vv[u]);
                    } else {
                        over = true;
                    }
                }
            }
        }
    }
    // ---- coalesced row indices and values ---------------------------------------
    if (STAGED && !has_big) {
        for (int x = tid; x < U; x += NT) {
            const int sl = S.omap[x];
            const long long vb = __double_as_longlong(V[sl]);
            stage[r0 + x] = make_int4(K[sl].x, (int)(unsigned)vb, (int)(unsigned)(vb >> 32), x);
        }
    } else if (!has_big) {
        for (int x = tid; x < U; x += NT) {
            const int sl = S.omap[x];
            if (P + x < cap) {
                ir[P + x] = K[sl].x;
                pr[P + x] = V[sl];
            } else {
                over = true;
            }
        }
    }
    if (over) atomicExch(&err->cap_exceeded, 1u);
    FTRACE(b, 7);
    if (!STAGED && b == ntiles - 1 && tid == 0) {
        jc[N] = (int32_t)(P + U);
        err->nnz = P + U;
        if (P + U > cap) atomicExch(&err->cap_exceeded, 1u);
    }
}

// The long-column body out of line: the short body stays on the kernel's
// fall-through path with its own code layout.
template <bool STAGED>
__device__ __noinline__ void tile_fold_long(
    const uint32_t *__restrict__ sstart, const int2 *__restrict__ tile_info,
    const uint8_t *__restrict__ tile_big, int64_t ntiles, const int2 *__restrict__ entries, Segs SG,
    const int4 *__restrict__ rec, const BigCol *__restrict__ big_list,
    const uint32_t *__restrict__ bigk, unsigned long long *tile_state, int32_t N,
    int32_t *__restrict__ jc, int32_t *__restrict__ ir, double *__restrict__ pr, int64_t cap,
    ErrState *err, int hash_fold, int4 *__restrict__ stage, int2 *__restrict__ tile_cnt) {
    tile_fold_body<STAGED, true>(sstart, tile_info, tile_big, ntiles, entries, SG, rec, big_list, bigk,
                                 tile_state, N, jc, ir, pr, cap, err, hash_fold, stage, tile_cnt);
}

template <bool STAGED>
__global__ void __launch_bounds__(NT, SA_FOLD_MINB) k_tile_fold(
    const uint32_t *__restrict__ sstart, const int2 *__restrict__ tile_info,
    const uint8_t *__restrict__ tile_big, int64_t ntiles, const int2 *__restrict__ entries, Segs SG,
    const int4 *__restrict__ rec, const BigCol *__restrict__ big_list,
    const uint32_t *__restrict__ bigk, unsigned long long *tile_state, int32_t N,
    int32_t *__restrict__ jc, int32_t *__restrict__ ir, double *__restrict__ pr, int64_t cap,
    ErrState *err, int hash_fold, int4 *__restrict__ stage, int2 *__restrict__ tile_cnt) {
    pdl_wait();
    pdl_trigger();
    if (!err->long_cols)  // (the short body first: the fall-through path)
        tile_fold_body<STAGED, false>(sstart, tile_info, tile_big, ntiles, entries, SG, rec, big_list,
                                      bigk, tile_state, N, jc, ir, pr, cap, err, hash_fold, stage,
                                      tile_cnt);
    else
        tile_fold_long<STAGED>(sstart, tile_info, tile_big, ntiles, entries, SG, rec, big_list, bigk,
                               tile_state, N, jc, ir, pr, cap, err, hash_fold, stage, tile_cnt);
}

// ---- staged outputs (long-column inputs): no look-back in k_tile_fold ------
// With many long columns a tile spends a fifth of its life waiting for its
// predecessors' counts.  In staged mode k_tile_fold writes each tile's
// small-column outputs as {row, value, tile-local index} records into the
// free small space of the record scratch (tile b at its record start), and
// its column pointers tile-local, and publishes its count; k_tile_emit
// chains the tile offsets (decoupled look-back over counts that are all
// already published) and copies every tile to its place (and the big
// columns from the big space), adding the offset to the column pointers.

constexpr int EMIT_NT = 256;

constexpr int EMIT_TILES = 8;  // tiles per k_tile_emit CTA

__global__ void __launch_bounds__(EMIT_NT) k_tile_emit(
    const uint32_t *__restrict__ sstart, const int2 *__restrict__ tile_info,
    const uint8_t *__restrict__ tile_big, int64_t ntiles, const int2 *__restrict__ tile_cnt,
    unsigned long long *tile_state, const int4 *__restrict__ stage,
    const int4 *__restrict__ rec, const BigCol *__restrict__ big_list,
    const uint32_t *__restrict__ bigk, int32_t N, int32_t *__restrict__ jc,
    int32_t *__restrict__ ir, double *__restrict__ pr, int64_t cap, ErrState *err) {
    __shared__ int2 s_big[TCAP];  // (tile-local output base, big-list index)
    __shared__ int s_nbig;
    __shared__ long long s_P[EMIT_TILES];
    pdl_wait();
    pdl_trigger();
    const int tid = threadIdx.x, lane = tid & 31;
    const long long b0 = (long long)blockIdx.x * EMIT_TILES;
    const int nt = (int)min((long long)EMIT_TILES, ntiles - b0);
    if (tid < 32) {  // every count is published already: one look-back for the first tile,
                     // the others by a prefix over their counts (and published as inclusive)
        const int cv = lane < nt ? tile_cnt[b0 + lane].x : 0;
        int incl = cv;
#pragma unroll
        for (int o = 1; o < EMIT_TILES; o <<= 1) {
            const int y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        const long long p0 = lookback_warp32(tile_state, b0, (unsigned long long)__shfl_sync(FULL, cv, 0));
        const long long P = p0 + incl - cv;
        if (lane < nt) {
            s_P[lane] = P;
            if (lane > 0)
                reinterpret_cast<volatile unsigned long long *>(tile_state)[(b0 + lane) * LB_STRIDE] =
                    lb_pack(2, (unsigned long long)(P + cv));
        }
    }
    __syncthreads();
    bool over = false;
    for (int t = 0; t < nt; ++t) {
        const long long b = b0 + t;
        const int2 ti0 = tile_info[b], ti1 = tile_info[b + 1];
        const int c_a = ti0.x, r0 = ti0.y, ncols = ti1.x - c_a;
        const long long P = s_P[t];
        const int2 uc = tile_cnt[b];
        for (int k = tid; k < uc.y; k += EMIT_NT) {
            const int4 r = stage[r0 + k];
            const long long x = P + r.w;
            if (x < cap) {
                ir[x] = r.x;
                pr[x] = __hiloint2double(r.z, r.y);
            } else {
                over = true;
            }
        }
        const bool has_big = tile_big[b] != 0;
        if (has_big) {
            if (tid == 0) s_nbig = 0;
            __syncthreads();
        }
        for (int c = tid; c < ncols; c += EMIT_NT) {
            const int o = jc[c_a + c];
            if (has_big && (sstart[c_a + c] & BIGFLAG)) {
                const int e = atomicAdd(&s_nbig, 1);
                if (e < TCAP) s_big[e] = make_int2(o, (int)bigk[c_a + c]);
                else atomicExch(&err->internal, 1u);
            }
            jc[c_a + c] = (int32_t)(P + o);
        }
        if (has_big) {
            __syncthreads();
            const int nb = min(s_nbig, TCAP);
            for (int e = 0; e < nb; ++e) {
                const long long o = P + s_big[e].x;
                const BigCol bc = big_list[s_big[e].y];
                const int ub = (int)(bc.u & POSMASK);
                const unsigned long long *RR = reinterpret_cast<const unsigned long long *>(rec + bc.start);
                const unsigned long long *BK = (bc.u & BIGFLAG) ? RR + bc.n : RR;
                const unsigned long long *BV = (bc.u & BIGFLAG) ? RR : RR + bc.n;
                for (int q = tid; q < ub; q += EMIT_NT) {
                    if (o + q < cap) {
                        ir[o + q] = (int32_t)BK[q];
                        pr[o + q] = __longlong_as_double((long long)BV[q]);
                    } else {
                        over = true;
                    }
                }
            }
            __syncthreads();  // s_big / s_nbig are reused by the next tile
        }
        if (b == ntiles - 1 && tid == 0) {
            jc[N] = (int32_t)(P + uc.x);
            err->nnz = P + uc.x;
            if (P + uc.x > cap) atomicExch(&err->cap_exceeded, 1u);
        }
    }
    if (over) atomicExch(&err->cap_exceeded, 1u);
}

cudaError_t launch_tile_fold(Launch &lc, const uint32_t *sstart, const int2 *tile_info,
                             const uint8_t *tile_big, int64_t ntiles, const int2 *entries,
                             const Segs &SG, const int4 *rec, const BigCol *big_list,
                             const uint32_t *bigk, unsigned long long *tile_state, int32_t N,
                             int32_t *jc, int32_t *ir, double *pr, int64_t cap, ErrState *err,
                             int4 *stage, int2 *tile_cnt) {
    if (ntiles <= 0) return cudaSuccess;
    constexpr int hash_fold = 1;
    cudaError_t e = ensure_smem_attr((const void *)k_tile_fold<false>, (int)sizeof(TileSmem));
    if (e == cudaSuccess) e = ensure_smem_attr((const void *)k_tile_fold<true>, (int)sizeof(TileSmem));
    if (e != cudaSuccess) return e;
    e = stage ? launch_pdl(k_tile_fold<true>, dim3((unsigned)ntiles), dim3(NT),
                                       sizeof(TileSmem), lc.stream, sstart, tile_info, tile_big,
                                       ntiles, entries, SG, rec, big_list, bigk, tile_state, N, jc,
                                       ir, pr, cap, err, hash_fold, stage, tile_cnt)
                          : launch_pdl(k_tile_fold<false>, dim3((unsigned)ntiles), dim3(NT),
                                       sizeof(TileSmem), lc.stream, sstart, tile_info, tile_big,
                                       ntiles, entries, SG, rec, big_list, bigk, tile_state, N, jc,
                                       ir, pr, cap, err, hash_fold, stage, tile_cnt);
    lc.launches++;
    if (e != cudaSuccess || !stage) return e;
    e = launch_pdl(k_tile_emit, dim3((unsigned)((ntiles + EMIT_TILES - 1) / EMIT_TILES)), dim3(EMIT_NT), 0,
                   lc.stream, sstart, tile_info,
                   tile_big, ntiles, (const int2 *)tile_cnt, tile_state, (const int4 *)stage, rec,
                   big_list, bigk, N, jc, ir, pr, cap, err);
    lc.launches++;
    return e;
}

}  // namespace sa

#ifdef SA_TRACE
extern "C" int sa_debug_ftrace(void *host, int n) {
    return (int)cudaMemcpyFromSymbol(host, sa::g_ftrace, (size_t)n * 64);
}
#endif
