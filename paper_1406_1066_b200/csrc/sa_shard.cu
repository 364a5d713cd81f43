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
// (first bad row / column position, indices beyond the global dimensions).
//
// Three launches (values are read only for the triplets that leave):
//   k_part_count    per tile (2048 triplets, 8 consecutive per thread) and
//                   destination: counts; column checks
//   k_part_scan     one CTA per destination: exclusive scan over tiles
//   k_part_scatter  per tile: lane / warp prefixes of packed per-thread
//                   counts (16-bit fields), leaving triplets written; row
//                   checks; tiles whose triplets all stay exit early
// Invalid columns (outside [1, bounds[world]]) go to no destination; the
// checks report them (first bad position, or an index beyond the global
// dimensions).

#include "sa_internal.cuh"

namespace sa {

namespace {

constexpr int PT_NT = 256;
constexpr int PT_NW = PT_NT / 32;
constexpr int PT_IPT = 8;                 // triplets per thread: element k of thread tid = tile + tid*PT_IPT + k
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
#pragma unroll
    for (int r = 1; r < PT_MAXW; ++r)  // static indices: the bounds stay in the parameter bank
        if (r < B.world && c >= B.b[r]) d = r;
    return d;
}

// Element k of thread tid of a tile is the tile's (tid * PT_IPT + k)-th
// triplet (thread-contiguous: two 16-byte loads per index array); the stable
// order inside a tile is (thread, k).  Index checks go straight to the error
// state with rare atomics: a warp reports only when it saw a bad index (first
// position, atomicMin) or one beyond the global dimensions (a flag).

__device__ __forceinline__ void load8(const int32_t *__restrict__ p, int64_t e0, int64_t L, bool vec,
                                      int (&v)[PT_IPT], int fill) {
    if (vec && e0 + PT_IPT <= L) {
        const int4 a = __ldg(reinterpret_cast<const int4 *>(p + e0));
        const int4 b = __ldg(reinterpret_cast<const int4 *>(p + e0) + 1);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
        v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
        for (int k = 0; k < PT_IPT; ++k) v[k] = (e0 + k < L) ? __ldg(p + e0 + k) : fill;
    }
}

__device__ __forceinline__ void report(unsigned long long bad, bool over,
                                       unsigned long long *err_bad, unsigned *err_over) {
    if (!__any_sync(FULL, bad != ~0ull || over)) return;  // the common case
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bad = min(bad, __shfl_xor_sync(FULL, bad, o));
    const bool ov = __any_sync(FULL, over);
    if ((threadIdx.x & 31) == 0) {
        if (bad != ~0ull) atomicMin(err_bad, bad);
        if (ov) atomicExch(err_over, 1u);
    }
}

// A thread's destination counts (<= PT_IPT = 8 each) as 4-bit fields of one
// word, widened to 16-bit fields, two destinations per word (sums over a
// whole tile fit).
__device__ __forceinline__ void widen(unsigned c4, unsigned (&w)[PT_MAXW / 2]) {
#pragma unroll
    for (int q = 0; q < PT_MAXW / 2; ++q)
        w[q] = ((c4 >> (8 * q)) & 15u) | (((c4 >> (8 * q + 4)) & 15u) << 16);
}
__device__ __forceinline__ int field(const unsigned (&w)[PT_MAXW / 2], int d) {
    int v = 0;
#pragma unroll
    for (int q = 0; q < PT_MAXW / 2; ++q)
        if (q == (d >> 1)) v = (int)((w[q] >> (16 * (d & 1))) & 0xffffu);
    return v;
}

// Destinations of a thread's PT_IPT consecutive triplets.  The destination
// is monotone in the column, so when the smallest and largest column of the
// run go to the same rank (FEM element order: nearly always) the per-triplet
// search is skipped.  Returns the 4-bit per-destination counts.
__device__ __forceinline__ unsigned run_dests(const Bounds &B, const int (&j)[PT_IPT], int64_t e0,
                                              int64_t L, int (&d)[PT_IPT]) {
    int lo = j[0], hi = j[0];
#pragma unroll
    for (int k = 1; k < PT_IPT; ++k) {
        lo = min(lo, j[k]);
        hi = max(hi, j[k]);
    }
    if (e0 + PT_IPT <= L && lo >= 1 && hi <= B.n) {
        const int dl = dest_of(B, lo);
        if (dl == dest_of(B, hi)) {
#pragma unroll
            for (int k = 0; k < PT_IPT; ++k) d[k] = dl;
            return (unsigned)PT_IPT << (4 * dl);
        }
    }
    unsigned c4 = 0;
#pragma unroll
    for (int k = 0; k < PT_IPT; ++k) {
        d[k] = (e0 + k < L) ? dest_of(B, j[k]) : -1;
        if (d[k] >= 0) c4 += 1u << (4 * d[k]);
    }
    return c4;
}

__global__ void __launch_bounds__(PT_NT) k_part_count(const int32_t *__restrict__ ii,
                                                      const int32_t *__restrict__ jj, int64_t L,
                                                      Bounds B, int vec, int32_t M,
                                                      int32_t *__restrict__ tile_cnt, ErrState *err) {
    __shared__ unsigned s_w[PT_NW][PT_MAXW / 2];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t ntiles = (L + PT_TILE - 1) / PT_TILE;
    unsigned long long bad = ~0ull, badi = ~0ull;
    bool over = false, overi = false;
    // the next tile's indices, in flight while this one is counted; rows are
    // validated here so that the scatter pass touches only tiles with
    // triplets that leave
    int jn[PT_IPT], in_[PT_IPT];
    if ((int64_t)blockIdx.x < ntiles) {
        const int64_t e1 = (int64_t)blockIdx.x * PT_TILE + (int64_t)tid * PT_IPT;
        load8(jj, e1, L, vec != 0, jn, 1);
        load8(ii, e1, L, vec != 0, in_, 1);
    }
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t e0 = t * PT_TILE + (int64_t)tid * PT_IPT;
        int jv[PT_IPT], iv[PT_IPT];
#pragma unroll
        for (int k = 0; k < PT_IPT; ++k) {
            jv[k] = jn[k];
            iv[k] = in_[k];
        }
        if (t + gridDim.x < ntiles) {
            load8(jj, e0 + (int64_t)gridDim.x * PT_TILE, L, vec != 0, jn, 1);
            load8(ii, e0 + (int64_t)gridDim.x * PT_TILE, L, vec != 0, in_, 1);
        }
        int d[PT_IPT];
        const unsigned c4 = run_dests(B, jv, e0, L, d);
#pragma unroll
        for (int k = 0; k < PT_IPT; ++k) {
            const bool live = e0 + k < L;
            if (live && jv[k] < 1) bad = min(bad, (unsigned long long)(e0 + k));
            if (live && jv[k] > B.n) over = true;
            if (live && iv[k] < 1) badi = min(badi, (unsigned long long)(e0 + k));
            if (live && iv[k] > M) overi = true;
        }
        unsigned wd[PT_MAXW / 2];
        widen(c4, wd);
#pragma unroll
        for (int q = 0; q < PT_MAXW / 2; ++q)
            if (2 * q < B.world) wd[q] = __reduce_add_sync(FULL, wd[q]);
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < PT_MAXW / 2; ++q) s_w[w][q] = wd[q];
        __syncthreads();
        if (tid < B.world) {
            int tot = 0;
            for (int q = 0; q < PT_NW; ++q) tot += (int)((s_w[q][tid >> 1] >> (16 * (tid & 1))) & 0xffffu);
            tile_cnt[(int64_t)tid * ntiles + t] = tot;  // destination-major
        }
        __syncthreads();  // s_w is rewritten by the next tile
    }
    report(bad, over, &err->bad_j, &err->over_n);
    report(badi, overi, &err->bad_i, &err->over_m);
}

// CTA d: tile_off[d][t] = sum over tiles < t of tile_cnt[d][.]
// (destination-major rows; every thread scans a contiguous run of up to
// SC_RUN tiles held in registers, more in a second pass); counts[d] =
// records for destination d
constexpr int SC_RUN = 12;
__global__ void __launch_bounds__(1024) k_part_scan(const int32_t *__restrict__ tile_cnt,
                                                    int64_t ntiles, int world,
                                                    int64_t *__restrict__ tile_off,
                                                    int64_t *__restrict__ counts) {
    __shared__ long long s_warp[32];
    const int d = blockIdx.x;
    const int32_t *row = tile_cnt + (int64_t)d * ntiles;
    int64_t *orow = tile_off + (int64_t)d * ntiles;
    const int64_t per = (ntiles + 1023) / 1024;
    const int64_t t0 = min(ntiles, (int64_t)threadIdx.x * per), t1 = min(ntiles, t0 + per);
    int v[SC_RUN];
    long long sum = 0;
#pragma unroll
    for (int k = 0; k < SC_RUN; ++k) {
        v[k] = (t0 + k < t1) ? row[t0 + k] : 0;
        sum += v[k];
    }
    for (int64_t t = t0 + SC_RUN; t < t1; ++t) sum += row[t];
    long long total;
    long long run = block_excl_sum<1024, long long>(sum, s_warp, total);
#pragma unroll
    for (int k = 0; k < SC_RUN; ++k)
        if (t0 + k < t1) {
            orow[t0 + k] = run;
            run += v[k];
        }
    for (int64_t t = t0 + SC_RUN; t < t1; ++t) {
        orow[t] = run;
        run += row[t];
    }
    if (threadIdx.x == 0) counts[d] = total;
}

// Stable scatter of the triplets bound for other ranks.  A thread's base
// for destination d = tile offset + the counts of the warps and lanes before
// it (16-bit fields); its own triplets to d follow in k order.  Values are
// loaded only for triplets that leave (element-ordered FEM keeps ~99.9 %
// of them at home).
__global__ void __launch_bounds__(PT_NT, 3) k_part_scatter(const int32_t *__restrict__ ii,
                                                        const int32_t *__restrict__ jj,
                                                        const double *__restrict__ s,
                                                        int64_t s_stride, int64_t L, Bounds B,
                                                        int vec,
                                                        const int32_t *__restrict__ tile_cnt,
                                                        const int64_t *__restrict__ tile_off,
                                                        const int64_t *__restrict__ counts,
                                                        int32_t *__restrict__ out_i,
                                                        int32_t *__restrict__ out_j,
                                                        double *__restrict__ out_s, int self) {
    __shared__ unsigned s_w[PT_NW][PT_MAXW / 2];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t ntiles = (L + PT_TILE - 1) / PT_TILE;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        // a tile none of whose triplets leave (the count pass's per-tile
        // counts) is not read at all: FEM element order keeps ~99.9 % home
        bool any = false;
        for (int r = 0; r < B.world; ++r)
            if (r != self) any |= __ldg(tile_cnt + (int64_t)r * ntiles + t) != 0;
        if (!any) continue;
        const int64_t e0 = t * PT_TILE + (int64_t)tid * PT_IPT;
        int jv[PT_IPT], iv[PT_IPT], d[PT_IPT];
        load8(jj, e0, L, vec != 0, jv, 1);
        load8(ii, e0, L, vec != 0, iv, 1);
        const unsigned c4 = run_dests(B, jv, e0, L, d);
        unsigned leave = 0;
#pragma unroll
        for (int k = 0; k < PT_IPT; ++k)
            if (d[k] >= 0 && d[k] != self) leave |= 1u << k;
        double sv[PT_IPT];
#pragma unroll
        for (int k = 0; k < PT_IPT; ++k) sv[k] = (leave >> k & 1u) ? __ldg(s + (e0 + k) * s_stride) : 0.0;
        // exclusive prefix of the fields over the lanes, then over the warps
        unsigned own[PT_MAXW / 2], x[PT_MAXW / 2];
        widen(c4, own);
#pragma unroll
        for (int q = 0; q < PT_MAXW / 2; ++q) x[q] = own[q];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
            for (int q = 0; q < PT_MAXW / 2; ++q) {
                const unsigned y = __shfl_up_sync(FULL, x[q], o);
                if (lane >= o) x[q] += y;
            }
        }
        if (lane == 31)
#pragma unroll
            for (int q = 0; q < PT_MAXW / 2; ++q) s_w[w][q] = x[q];
#pragma unroll
        for (int q = 0; q < PT_MAXW / 2; ++q) x[q] -= own[q];
        __syncthreads();
        for (int p = 0; p < w; ++p)
#pragma unroll
            for (int q = 0; q < PT_MAXW / 2; ++q) x[q] += s_w[p][q];
        if (leave) {
            long long base[PT_MAXW];
            {
                long long acc = 0;  // destinations before r (the rank's own stay in place)
#pragma unroll
                for (int r = 0; r < PT_MAXW; ++r) {
                    base[r] = 0;
                    if (r < B.world) {
                        base[r] = acc + tile_off[(int64_t)r * ntiles + t] + field(x, r);
                        if (r != self) acc += counts[r];
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < PT_IPT; ++k) {
                if (!(leave >> k & 1u)) continue;  // (every triplet to a destination r != self leaves)
                long long pos = 0;
#pragma unroll
                for (int r = 0; r < PT_MAXW; ++r) {  // predicated: base stays in registers
                    const bool m = r == d[k];
                    pos = m ? base[r] : pos;
                    base[r] += m ? 1 : 0;
                }
                out_i[pos] = iv[k];
                out_j[pos] = jv[k];
                out_s[pos] = sv[k];
            }
        }
        __syncthreads();  // s_w is rewritten by the next tile
    }
}

// Sampled column-block histogram for the rank boundaries (distributed.py):
// every `step`-th triplet's column, in `nblocks` blocks of `bsize` columns
// (columns outside [1, N] clamped into the end blocks), counts scaled by
// `step`.  Shared-memory bins per CTA, one global add per touched bin.
constexpr int BH_NT = 256;
constexpr int BH_MAXB = 8192;
__global__ void __launch_bounds__(BH_NT) k_block_hist(const int32_t *__restrict__ jj, int64_t L,
                                                      int64_t step, int nblocks, int64_t bsize,
                                                      unsigned long long *__restrict__ hist) {
    __shared__ unsigned bins[BH_MAXB];
    for (int b = threadIdx.x; b < nblocks; b += BH_NT) bins[b] = 0;
    __syncthreads();
    const int64_t ns = (L + step - 1) / step;
    for (int64_t q = (int64_t)blockIdx.x * BH_NT + threadIdx.x; q < ns; q += (int64_t)gridDim.x * BH_NT) {
        int64_t b = ((int64_t)__ldg(jj + q * step) - 1) / bsize;
        b = b < 0 ? 0 : (b >= nblocks ? nblocks - 1 : b);
        atomicAdd(&bins[b], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nblocks; b += BH_NT)
        if (bins[b]) atomicAdd(&hist[b], (unsigned long long)bins[b] * (unsigned long long)step);
}

}  // namespace

int64_t partition_tiles(int64_t L) { return (L + PT_TILE - 1) / PT_TILE; }

cudaError_t launch_block_hist(Launch &lc, const int32_t *jj, int64_t L, int64_t step, int nblocks,
                              int64_t bsize, unsigned long long *hist) {
    if (nblocks < 1 || nblocks > BH_MAXB || step < 1 || bsize < 1) return cudaErrorInvalidValue;
    cudaError_t e = cudaMemsetAsync(hist, 0, (size_t)nblocks * sizeof(unsigned long long), lc.stream);
    if (e != cudaSuccess || L <= 0) return e;
    const int64_t ns = (L + step - 1) / step;
    const int grid = (int)std::min<int64_t>((ns + BH_NT - 1) / BH_NT, (int64_t)lc.num_sms * 2);
    k_block_hist<<<grid, BH_NT, 0, lc.stream>>>(jj, L, step, nblocks, bsize, hist);
    lc.launches++;
    return cudaGetLastError();
}

cudaError_t launch_partition(Launch &lc, const int32_t *ii, const int32_t *jj, const double *s,
                             int64_t s_stride, int64_t L, int world, int self, const int32_t *bounds,
                             int32_t M, int32_t *tile_cnt, int64_t *tile_off, int64_t *counts,
                             int32_t *out_i, int32_t *out_j, double *out_s, ErrState *err) {
    if (world < 1 || world > PT_MAXW) return cudaErrorInvalidValue;
    Bounds B;
    for (int r = 0; r <= PT_MAXW; ++r) B.b[r] = (r <= world) ? bounds[r] : bounds[world];
    B.world = world;
    B.n = bounds[world];
    const int64_t ntiles = partition_tiles(L);
    if (ntiles == 0) return cudaMemsetAsync(counts, 0, 2 * PT_MAXW * sizeof(int64_t), lc.stream);
    const int vec = ((reinterpret_cast<uintptr_t>(ii) | reinterpret_cast<uintptr_t>(jj)) & 15) == 0;
    const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)lc.num_sms * 8);
    k_part_count<<<grid, PT_NT, 0, lc.stream>>>(ii, jj, L, B, vec, M, tile_cnt, err);
    k_part_scan<<<world, 1024, 0, lc.stream>>>(tile_cnt, ntiles, world, tile_off, counts);
    k_part_scatter<<<grid, PT_NT, 0, lc.stream>>>(ii, jj, s, s_stride, L, B, vec, tile_cnt, tile_off,
                                                  counts, out_i, out_j, out_s, self);
    lc.launches += 3;
    return cudaGetLastError();
}

}  // namespace sa
