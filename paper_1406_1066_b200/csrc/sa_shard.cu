// sa_shard.cu -- multi-GPU column-block sharding: the stable partition of a
// rank's triplet chunk by destination rank (distributed.py).
//
// The destination of a triplet is the rank owning its column block:
// bounds[r] <= j-1 < bounds[r+1] (0-based column boundaries, world <= 8).
// Output: the arrays {i}, {j}, {s} of the triplets bound for other ranks,
// grouped by destination in rank order and, inside a destination, in input
// order (the rank's own triplets stay in place: its assembly reads its chunk
// directly, sa_assemble_segments_async) -- the receiver places what it gets
// from lower ranks before and from higher ranks after its own chunk, which
// keeps the global input order, so the per-rank assemblies stay
// bit-identical to one GPU.  The chunk's indices are validated on the way
// (first bad row / column position, maxima).
//
// Three launches (a single pass over the triplets each):
//   k_part_count    per tile (2048 triplets) and destination: counts
//   k_part_scan     one CTA: exclusive scan over tiles per destination
//   k_part_scatter  per tile: block scan of packed per-thread counts (4 x
//                   16-bit fields per 64-bit word), entries written
// Invalid columns (outside [1, bounds[world]]) go to no destination; the
// validation reports them (bad_j, or max_j above the global N).

#include "sa_internal.cuh"

namespace sa {

namespace {

constexpr int PT_NT = 256;
constexpr int PT_NW = PT_NT / 32;
constexpr int PT_IPT = 8;                 // rows of a tile: element (k, tid) = tile + k*PT_NT + tid
constexpr int PT_TILE = PT_NT * PT_IPT;   // 2048 triplets
constexpr int PT_MAXW = 8;

struct Bounds {
    int b[PT_MAXW + 1];
    int world;
    int n;  // b[world]
};

__device__ __forceinline__ int dest_of(const Bounds &B, int j) {
    const int c = j - 1;
    if (c < 0 || c >= B.n) return -1;
    int d = 0;
    for (int r = 1; r < B.world; ++r)  // warp-uniform trip count
        if (c >= B.b[r]) d = r;
    return d;
}

// first column of destination d (no dynamic indexing into the parameter)
__device__ __forceinline__ int block_lo(const Bounds &B, int d) {
    int v = 0;
#pragma unroll
    for (int r = 1; r < PT_MAXW; ++r)
        if (r == d) v = B.b[r];
    return v;
}

// first bad position (< 1) and maximum of the CTA's indices -> one slot per
// tile (no same-address atomics across the grid; k_part_reduce folds them)
struct TileCheck {
    unsigned long long bad;
    unsigned mx;
    unsigned pad;
};

__device__ __forceinline__ void check_finish(unsigned long long b, unsigned m, TileCheck *out,
                                             TileCheck *s_chk) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        b = min(b, __shfl_xor_sync(FULL, b, o));
        m = max(m, __shfl_xor_sync(FULL, m, o));
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) s_chk[w] = TileCheck{b, m, 0u};
    __syncthreads();
    if (threadIdx.x == 0) {
        TileCheck c = s_chk[0];
        for (int k = 1; k < PT_NW; ++k) {
            c.bad = min(c.bad, s_chk[k].bad);
            c.mx = max(c.mx, s_chk[k].mx);
        }
        *out = c;
    }
}

// Per (row k, warp w) and destination d: triplets of the warp's 32 consecutive
// elements that go to d; lane d of the warp writes cnt[k][w][d].
__device__ __forceinline__ void warp_dest_counts(int dk, int world, int *cnt_kw) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int r = 0; r < PT_MAXW; ++r) {
        const unsigned m = __ballot_sync(FULL, dk == r);
        if (lane == r && r < world) cnt_kw[r] = __popc(m);
    }
}

__global__ void __launch_bounds__(PT_NT) k_part_count(const int32_t *__restrict__ jj, int64_t L,
                                                      Bounds B, int32_t *__restrict__ tile_cnt,
                                                      TileCheck *__restrict__ chk_j) {
    __shared__ int s_cnt[PT_NW][PT_MAXW];
    __shared__ TileCheck s_chk[PT_NW];
    const long long t = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    unsigned long long bad = ~0ull;
    unsigned mx = 0;
    // per-thread counts in 4-bit fields (<= PT_IPT = 8 per destination)
    unsigned long long acc = 0;
    int jv[PT_IPT];
#pragma unroll
    for (int k = 0; k < PT_IPT; ++k) {  // all loads in flight before any use
        const int64_t e = t * PT_TILE + (int64_t)k * PT_NT + tid;
        jv[k] = (e < L) ? __ldg(jj + e) : 0;
    }
#pragma unroll
    for (int k = 0; k < PT_IPT; ++k) {
        const int64_t e = t * PT_TILE + (int64_t)k * PT_NT + tid;
        const int j = jv[k];
        const int d = (e < L) ? dest_of(B, j) : -1;
        if (e < L) {
            if (j < 1) bad = min(bad, (unsigned long long)e);
            else mx = max(mx, (unsigned)j);
        }
        if (d >= 0) acc += 1ull << (4 * d);
    }
    // widen to 16-bit fields (4 destinations per word) and reduce over the warp
    unsigned long long lo = 0, hi = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        lo |= ((acc >> (4 * r)) & 15ull) << (16 * r);
        hi |= ((acc >> (4 * (r + 4))) & 15ull) << (16 * r);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo += __shfl_xor_sync(FULL, lo, o);
        hi += __shfl_xor_sync(FULL, hi, o);
    }
    const int acc_l = (lane < 4) ? (int)((lo >> (16 * lane)) & 0xffff)
                                 : (int)((hi >> (16 * (lane & 3))) & 0xffff);
    if (lane < PT_MAXW) s_cnt[w][lane] = acc_l;
    check_finish(bad, mx, &chk_j[t], s_chk);  // ends with a barrier
    if (tid < B.world) {
        int tot = 0;
        for (int q = 0; q < PT_NW; ++q) tot += s_cnt[q][tid];
        tile_cnt[t * B.world + tid] = tot;
    }
}

// CTA d: tile_off[t][d] = sum over tiles < t of tile_cnt[.][d]; counts[d] =
// records for destination d (the scatter derives the destination bases)
__global__ void __launch_bounds__(1024) k_part_scan(const int32_t *__restrict__ tile_cnt,
                                                    int64_t ntiles, int world,
                                                    int64_t *__restrict__ tile_off,
                                                    int64_t *__restrict__ counts) {
    __shared__ long long s_warp[32];
    __shared__ long long s_carry;
    const int d = blockIdx.x;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < ntiles; base += 1024) {
        const int64_t t = base + threadIdx.x;
        const long long v = (t < ntiles) ? tile_cnt[t * world + d] : 0;
        long long total;
        const long long pre = block_excl_sum<1024, long long>(v, s_warp, total);
        if (t < ntiles) tile_off[t * world + d] = s_carry + pre;
        __syncthreads();
        if (threadIdx.x == 0) s_carry += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) counts[d] = s_carry;
}

// Element (k, tid) of a tile is its k*PT_NT + tid-th triplet; the stable
// order inside the tile is (k, warp, lane).  The per-(k, warp) destination
// counts are scanned in that order (one warp per destination), and every
// lane adds its rank among the warp's lanes with the same destination:
// lanes writing one destination write consecutive slots.
__global__ void __launch_bounds__(PT_NT) k_part_scatter(const int32_t *__restrict__ ii,
                                                        const int32_t *__restrict__ jj,
                                                        const double *__restrict__ s,
                                                        int64_t s_stride, int64_t L, Bounds B,
                                                        const int64_t *__restrict__ tile_off,
                                                        const int64_t *__restrict__ counts,
                                                        int32_t *__restrict__ out_i,
                                                        int32_t *__restrict__ out_j,
                                                        double *__restrict__ out_s, int self,
                                                        TileCheck *__restrict__ chk_i) {
    __shared__ int s_cnt[PT_MAXW][PT_IPT * PT_NW];  // [dest][k*NW + w], then exclusive prefixes
    __shared__ TileCheck s_chk[PT_NW];
    const long long t = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const unsigned lt = lanemask_lt();
    int d[PT_IPT], j[PT_IPT], iv[PT_IPT];
    unsigned long long bad = ~0ull;
    unsigned mx = 0;
    double sv[PT_IPT];
    unsigned pm[PT_IPT];
    for (int x = tid; x < PT_MAXW * PT_IPT * PT_NW; x += PT_NT) (&s_cnt[0][0])[x] = 0;
#pragma unroll
    for (int k = 0; k < PT_IPT; ++k) {  // all loads in flight before any use
        const int64_t e = t * PT_TILE + (int64_t)k * PT_NT + tid;
        j[k] = (e < L) ? __ldg(jj + e) : 0;
        iv[k] = (e < L) ? __ldg(ii + e) : 1;
        sv[k] = (e < L) ? __ldg(s + e * s_stride) : 0.0;
    }
    __syncthreads();  // counters zeroed
#pragma unroll
    for (int k = 0; k < PT_IPT; ++k) {
        const int64_t e = t * PT_TILE + (int64_t)k * PT_NT + tid;
        d[k] = (e < L) ? dest_of(B, j[k]) : -1;
        if (e < L) {
            if (iv[k] < 1) bad = min(bad, (unsigned long long)e);
            else mx = max(mx, (unsigned)iv[k]);
        }
        pm[k] = __match_any_sync(FULL, d[k]);  // lanes with the same destination
        if (d[k] >= 0 && (pm[k] & lt) == 0u) {  // group leader
#pragma unroll
            for (int r = 0; r < PT_MAXW; ++r)
                if (r == d[k]) s_cnt[r][k * PT_NW + w] = __popc(pm[k]);
        }
    }
    __syncthreads();
    // exclusive scan of s_cnt[d][0..64) in (k, w) order: warp d, 2 entries per lane
    if (w < B.world) {
        static_assert(PT_IPT * PT_NW == 64, "two (k, warp) entries per lane");
        const int a0 = s_cnt[w][2 * lane], a1 = s_cnt[w][2 * lane + 1];
        int x = a0 + a1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x += y;
        }
        long long base = tile_off[t * B.world + w];
        for (int r = 0; r < w; ++r)  // destinations before w (the rank's own stay in place)
            if (r != self) base += counts[r];
        const int ex = x - a0 - a1;
        s_cnt[w][2 * lane] = (int)ex;
        s_cnt[w][2 * lane + 1] = (int)(ex + a0);
        if (lane == 0) s_chk[w].bad = (unsigned long long)base;  // stash the base
    }
    __syncthreads();
    long long dbase[PT_MAXW];
#pragma unroll
    for (int r = 0; r < PT_MAXW; ++r) dbase[r] = (r < B.world) ? (long long)s_chk[r].bad : 0;
#pragma unroll
    for (int k = 0; k < PT_IPT; ++k) {
        const int64_t e = t * PT_TILE + (int64_t)k * PT_NT + tid;
        const unsigned peers = pm[k];
        if (d[k] < 0 || d[k] == self) continue;
        long long pos = 0;
        int pre = 0;
#pragma unroll
        for (int r = 0; r < PT_MAXW; ++r)
            if (r == d[k]) {
                pos = dbase[r];
                pre = s_cnt[r][k * PT_NW + w];
            }
        pos += pre + __popc(peers & lt);
        out_i[pos] = iv[k];
        out_j[pos] = j[k];
        out_s[pos] = sv[k];
    }
    __syncthreads();  // s_chk is reused below
    check_finish(bad, mx, &chk_i[t], s_chk);
}

// one CTA: the tiles' index checks -> the context's error state
__global__ void __launch_bounds__(1024) k_part_reduce(const TileCheck *__restrict__ chk_i,
                                                      const TileCheck *__restrict__ chk_j,
                                                      int64_t ntiles, ErrState *err) {
    unsigned long long bi = ~0ull, bj = ~0ull;
    unsigned mi = 0, mj = 0;
    for (int64_t t = threadIdx.x; t < ntiles; t += 1024) {
        bi = min(bi, chk_i[t].bad);
        bj = min(bj, chk_j[t].bad);
        mi = max(mi, chk_i[t].mx);
        mj = max(mj, chk_j[t].mx);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        bi = min(bi, __shfl_xor_sync(FULL, bi, o));
        bj = min(bj, __shfl_xor_sync(FULL, bj, o));
        mi = max(mi, __shfl_xor_sync(FULL, mi, o));
        mj = max(mj, __shfl_xor_sync(FULL, mj, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (bi != ~0ull) atomicMin(&err->bad_i, bi);
        if (bj != ~0ull) atomicMin(&err->bad_j, bj);
        if (mi) atomicMax(&err->max_i, mi);
        if (mj) atomicMax(&err->max_j, mj);
    }
}

}  // namespace

int64_t partition_tiles(int64_t L) { return (L + PT_TILE - 1) / PT_TILE; }
size_t partition_check_bytes(int64_t L) { return 2 * (size_t)partition_tiles(L) * sizeof(TileCheck); }

cudaError_t launch_partition(Launch &lc, const int32_t *ii, const int32_t *jj, const double *s,
                             int64_t s_stride, int64_t L, int world, int self, const int32_t *bounds,
                             int32_t *tile_cnt, int64_t *tile_off, int64_t *counts,
                             int32_t *out_i, int32_t *out_j, double *out_s, void *checks,
                             ErrState *err) {
    if (world < 1 || world > PT_MAXW) return cudaErrorInvalidValue;
    Bounds B;
    for (int r = 0; r <= PT_MAXW; ++r) B.b[r] = (r <= world) ? bounds[r] : bounds[world];
    B.world = world;
    B.n = bounds[world];
    const int64_t ntiles = partition_tiles(L);
    if (ntiles == 0) return cudaMemsetAsync(counts, 0, 2 * PT_MAXW * sizeof(int64_t), lc.stream);
    TileCheck *chk_j = reinterpret_cast<TileCheck *>(checks), *chk_i = chk_j + ntiles;
    k_part_count<<<(unsigned)ntiles, PT_NT, 0, lc.stream>>>(jj, L, B, tile_cnt, chk_j);
    k_part_scan<<<world, 1024, 0, lc.stream>>>(tile_cnt, ntiles, world, tile_off, counts);
    k_part_scatter<<<(unsigned)ntiles, PT_NT, 0, lc.stream>>>(ii, jj, s, s_stride, L, B, tile_off,
                                                              counts, out_i, out_j, out_s, self,
                                                              chk_i);
    k_part_reduce<<<1, 1024, 0, lc.stream>>>(chk_i, chk_j, ntiles, err);
    lc.launches += 4;
    return cudaGetLastError();
}

}  // namespace sa
