// sa_prune.cu -- device prune_explicit_zeros (sm_100a).
//
// Reference: types.py:204-213 (`prune_explicit_zeros`): drop the entries
// stored as exactly 0.0 (+0.0 and -0.0; NaN is kept because NaN != 0.0) and
// recompact jc.  Entry order is preserved, so ir stays strictly increasing
// inside every column.
//
// One pass, single kernel: tiles of PR_TILE consecutive entries; each thread
// owns PR_IPT consecutive entries (16-byte vector loads of pr), a block scan
// of the keep flags gives the tile's kept count, the decoupled look-back
// (sa_internal.cuh) its output offset; kept entries are written compacted.
// Column pointers: the tile holding entry jc[c] (the first entry of column c)
// writes jc_out[c] = kept entries before it; trailing columns (jc[c] == nnz)
// are written by the last tile.

#include "sa_internal.cuh"

namespace sa {

namespace {

constexpr int PR_NT = 256;
constexpr int PR_IPT = 8;
constexpr int PR_TILE = PR_NT * PR_IPT;

// first c in [lo, hi) with jc[c] >= key (jc non-decreasing)
__device__ __forceinline__ int lower_bound_jc(const int32_t *__restrict__ jc, int lo, int hi,
                                              long long key) {
    while (lo < hi) {
        const int mid = lo + ((hi - lo) >> 1);
        if ((long long)jc[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(PR_NT) k_prune(const int32_t *__restrict__ jc,
                                                 const int32_t *__restrict__ ir,
                                                 const double *__restrict__ pr, int32_t N,
                                                 int64_t nnz, int32_t *__restrict__ jc_out,
                                                 int32_t *__restrict__ ir_out,
                                                 double *__restrict__ pr_out,
                                                 unsigned long long *state, long long *nnz_out) {
    __shared__ int kpre[PR_TILE + 1];  // kept entries of the tile before each entry
    __shared__ int s_warp[PR_NT / 32];
    __shared__ long long s_P;
    const int tid = threadIdx.x;
    const long long b = blockIdx.x;
    const long long t0 = b * PR_TILE + (long long)tid * PR_IPT;
    double v[PR_IPT];
    int r[PR_IPT];
    bool keep[PR_IPT];
    int kc = 0;
#pragma unroll
    for (int k = 0; k < PR_IPT; ++k) {
        const bool live = t0 + k < nnz;
        v[k] = live ? pr[t0 + k] : 0.0;
        r[k] = live ? ir[t0 + k] : 0;
        keep[k] = live && v[k] != 0.0;  // NaN != 0.0 is true: NaN is kept
        kc += keep[k];
    }
    int total;
    const int pre = block_excl_sum<PR_NT, int>(kc, s_warp, total);
    {
        int run = pre;
#pragma unroll
        for (int k = 0; k < PR_IPT; ++k) {
            kpre[tid * PR_IPT + k] = run;
            run += keep[k];
        }
        if (tid == PR_NT - 1) kpre[PR_TILE] = run;
    }
    if (tid < 32) {
        const unsigned long long e = lookback_warp(state, b, (unsigned long long)total);
        if (tid == 0) s_P = (long long)e;
    }
    __syncthreads();
    const long long P = s_P;
    {
        long long o = P + pre;
#pragma unroll
        for (int k = 0; k < PR_IPT; ++k) {
            if (keep[k]) {
                ir_out[o] = r[k];
                pr_out[o] = v[k];
                ++o;
            }
        }
    }
    // column pointers of the columns that start inside this tile
    const long long tbeg = b * PR_TILE;
    const long long tend = min(tbeg + PR_TILE, (long long)nnz);
    const bool last = (b == (long long)gridDim.x - 1);
    const int c_lo = lower_bound_jc(jc, 0, N + 1, tbeg);
    const int c_hi = last ? N + 1 : lower_bound_jc(jc, c_lo, N + 1, tend);
    for (int c = c_lo + tid; c < c_hi; c += PR_NT) {
        const long long q = (long long)jc[c] - tbeg;
        jc_out[c] = (int32_t)(P + (q < PR_TILE ? kpre[q] : kpre[PR_TILE]));
    }
    if (last && tid == 0) *nnz_out = P + total;
}

}  // namespace

cudaError_t launch_prune(Launch &lc, const int32_t *jc, const int32_t *ir, const double *pr,
                         int32_t N, int64_t nnz, int32_t *jc_out, int32_t *ir_out,
                         double *pr_out, unsigned long long *state, long long *nnz_out) {
    if (nnz <= 0) {
        cudaError_t e = cudaMemsetAsync(jc_out, 0, ((size_t)N + 1) * sizeof(int32_t), lc.stream);
        if (e != cudaSuccess) return e;
        return cudaMemsetAsync(nnz_out, 0, sizeof(long long), lc.stream);
    }
    const int64_t ntiles = (nnz + PR_TILE - 1) / PR_TILE;
    cudaError_t e = cudaMemsetAsync(state, 0, (size_t)ntiles * LB_STRIDE * sizeof(unsigned long long),
                                    lc.stream);
    if (e != cudaSuccess) return e;
    k_prune<<<(unsigned)ntiles, PR_NT, 0, lc.stream>>>(jc, ir, pr, N, nnz, jc_out, ir_out, pr_out,
                                                     state, nnz_out);
    lc.launches++;
    return cudaGetLastError();
}

int64_t prune_tiles(int64_t nnz) { return nnz > 0 ? (nnz + PR_TILE - 1) / PR_TILE : 0; }

}  // namespace sa
