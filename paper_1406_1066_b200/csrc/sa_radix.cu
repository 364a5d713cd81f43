// sa_radix.cu -- the column-block ("radix") path of sparse(i,j,s,m,n) for
// inputs without column locality (shuffled / random triplets, BASELINE cfg4).
//
// The legacy pipeline (sa_kernels.cu, sa_tile.cu) scatters 8-byte entries to
// per-column cursors.  On shuffled input its N write fronts (N = 1e7 on cfg4)
// do not fit in L2 and every entry costs a DRAM read-modify-write of a
// sector; the fold then gathers every value at random.  This path instead
// moves the triplets themselves through a stable LSD radix partition on the
// HIGH column bits, so that every later access stays inside one small
// column block ("sub-bucket", W = 2^w columns, ~3k triplets):
//
//   k_init     error state, tickets, digit histograms reset (sa_capi.cu)
//   k_rhist    histogram of the first pass's digit + column validation
//   k_rpass    one stable partition pass (onesweep: chunk-local stable rank
//              by warp match + per-warp running counters, decoupled
//              look-back per digit across chunks, coalesced scatter through
//              shared memory), 16 B per triplet in and out; the first pass
//              validates rows, every pass histograms the next pass's digit
//   k_rbounds  sub-bucket boundaries in the partitioned arrays (binary search)
//              and the list of oversize sub-buckets
//   k_rbig     oversize sub-buckets (> RF_CAP triplets: skewed input), one
//              1024-thread CTA each: stable LSD radix sort of (column, row)
//              keys in global scratch, ordered run folds
//   k_rfold    one CTA per sub-bucket, all in shared memory: (column, row)
//              groups by hashing, members of each group folded from +0.0 in
//              input order (the partition is stable, so input order = array
//              order), groups ordered by (column, row), decoupled look-back of
//              the distinct counts across sub-buckets -> jc, ir, pr written
//              once, coalesced.
//
// Bit-exactness: identical contract to the legacy path (reference
// _kernels.pyx:82-89, pr[k] = ((+0.0 + v1) + v2) + ... in ascending input
// position): every pass is stable, so within a (column, row) group the
// members keep input order, and each group is folded sequentially with the
// x86 NaN rule (fold_add).
//
// Look-back words carry a 16-bit tag (call epoch << 2 | pass) so the state
// arrays never need resetting between calls.

#include <cstdint>

#include "sa_internal.cuh"

namespace sa {

// ---- epoch-tagged look-back words: [63:48] tag, [47:46] flag, [45:0] value --
constexpr unsigned long long EP_VMASK = (1ull << 46) - 1;
__device__ __forceinline__ unsigned long long ep_pack(unsigned tag, unsigned flag,
                                                      unsigned long long v) {
    return (static_cast<unsigned long long>(tag) << 48) |
           (static_cast<unsigned long long>(flag) << 46) | v;
}
__device__ __forceinline__ unsigned ep_flag(unsigned long long w, unsigned tag) {
    return (static_cast<unsigned>(w >> 48) == tag) ? static_cast<unsigned>((w >> 46) & 3u) : 0u;
}

// Exclusive prefix of tile b (its aggregate already published by the caller)
// over tiles < b; one full warp.  Tiles publish 1 (aggregate) or 2
// (inclusive prefix) under `tag`; anything else reads as "not yet".
__device__ __forceinline__ unsigned long long ep_walk_warp(const unsigned long long *st, long long b,
                                                           unsigned tag) {
    const int lane = threadIdx.x & 31;
    const volatile unsigned long long *vst = st;
    unsigned long long excl = 0;
    long long base = b - 1;
    while (base >= 0) {
        const long long idx = base - lane;
        const unsigned long long w = (idx >= 0) ? vst[idx * LB_STRIDE] : ep_pack(tag, 2, 0);
        const unsigned f = ep_flag(w, tag);
        if (__any_sync(FULL, f == 0)) continue;
        const unsigned pm = __ballot_sync(FULL, f == 2);
        const int stop = pm ? (__ffs(pm) - 1) : 31;
        unsigned long long v = (lane <= stop) ? (w & EP_VMASK) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        excl += v;
        if (pm) break;
        base -= 32;
    }
    return excl;
}

// ---------------------------------------------------------------------------
// k_rhist: histogram of the first pass's digit over the valid triplets and
// column validation (first column index < 1, any index > N).
// ---------------------------------------------------------------------------
constexpr int RH_NT = 256;
constexpr int RH_U = 8;

__global__ void __launch_bounds__(RH_NT) k_rhist(const int32_t *__restrict__ jj, int64_t L,
                                                 int32_t N, int shift, int bits,
                                                 uint32_t *__restrict__ hist, ErrState *err) {
    __shared__ uint32_t h[RP_MAXD];
    for (int k = threadIdx.x; k < RP_MAXD; k += RH_NT) h[k] = 0;
    __syncthreads();
    pdl_wait();
    const unsigned dmask = (1u << bits) - 1u;
    unsigned long long bad = ~0ull;
    unsigned over = 0;
    const int64_t step = (int64_t)gridDim.x * RH_NT * RH_U;
    for (int64_t t0 = (int64_t)blockIdx.x * RH_NT * RH_U + threadIdx.x; t0 < L; t0 += step) {
        int v[RH_U];
#pragma unroll
        for (int u = 0; u < RH_U; ++u) {
            const int64_t t = t0 + (int64_t)u * RH_NT;
            v[u] = (t < L) ? __ldg(jj + t) : 1;
        }
#pragma unroll
        for (int u = 0; u < RH_U; ++u) {
            const int64_t t = t0 + (int64_t)u * RH_NT;
            if (t >= L) continue;
            const int c = v[u];
            if (c < 1) bad = min(bad, (unsigned long long)t);
            else if (c > N) over = 1;
            else atomicAdd(&h[((unsigned)(c - 1) >> shift) & dmask], 1u);
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k <= (int)dmask; k += RH_NT)
        if (h[k]) atomicAdd(&hist[k], h[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        bad = min(bad, __shfl_xor_sync(FULL, bad, o));
        over |= __shfl_xor_sync(FULL, over, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (bad != ~0ull) atomicMin(&err->bad_j, bad);
        if (over) err->over_n = 1;
    }
    pdl_trigger();
}

// ---------------------------------------------------------------------------
// k_rpass: one stable LSD partition pass by the digit (col-1) >> shift.
// A chunk of RP_CHUNK consecutive triplets per CTA (ticket order); warp w
// owns the chunk's w-th run of RP_IPT x 32 triplets and walks it in order,
// 32 at a time: __match_any_sync groups equal digits, a per-warp running
// counter per digit gives every triplet its rank -- stable by construction.
// A block scan over (digit, warp) makes the ranks chunk-local; a decoupled
// look-back per digit (one thread each) over the previous chunks gives the
// chunk's global base per digit.  The triplets are then reordered in shared
// memory by digit and written out so that consecutive threads write
// consecutive addresses of one digit run.
// ---------------------------------------------------------------------------
struct PassSmem {
    uint16_t cnt[RP_NW][RP_MAXD];      // per warp and digit: running count, then chunk-local base
    unsigned long long buf[RP_CHUNK];  // reorder buffer (values, then row << 32 | col)
    uint16_t sdig[RP_CHUNK];           // digit of the reordered triplet
    uint32_t cbase[RP_MAXD];           // global position of the digit's chunk-local slot 0
    uint32_t hnext[RP_MAXD];           // histogram of the next pass's digit
    uint32_t red[RP_NW];
    int b;
};

template <bool FIRST>
__global__ void __launch_bounds__(RP_NT, 2) k_rpass(RadixPassArgs A, ErrState *err) {
    extern __shared__ __align__(16) unsigned char rp_smem[];
    PassSmem &S = *reinterpret_cast<PassSmem *>(rp_smem);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int ndig = 1 << A.bits;
    const unsigned dmask = (unsigned)ndig - 1u;
    const unsigned nmask = (1u << A.nbits) - 1u;
    const unsigned lt = lanemask_lt();
    {
        uint32_t *c32 = reinterpret_cast<uint32_t *>(&S.cnt[0][0]);
        for (int k = tid; k < RP_NW * RP_MAXD / 2; k += RP_NT) c32[k] = 0;
        for (int k = tid; k < RP_MAXD; k += RP_NT) S.hnext[k] = 0;
    }
    pdl_wait();
    // global start of every digit: exclusive scan of this pass's histogram
    uint32_t htot;
    const uint32_t gstart =
        block_excl_sum<RP_NT, uint32_t>((tid < ndig) ? A.hist[tid] : 0u, S.red, htot);
    if (tid == 0) S.b = (int)atomicAdd(&err->rp_ticket[A.pass], 1u);
    __syncthreads();
    const int64_t b = S.b;
    const int64_t base = b * RP_CHUNK + (int64_t)w * (RP_IPT * 32) + lane;
    {  // the chunk's rows and values into L2 now; they are read after the ranking
        const int64_t c0 = b * RP_CHUNK;
        const int64_t nrow = max((int64_t)0, min((int64_t)RP_CHUNK, A.L - c0));  // upper bound (Lp <= L)
        if (A.s_stride) {
            const char *vb = reinterpret_cast<const char *>(A.s_in + c0);
            for (int64_t o = (int64_t)tid * 128; o < nrow * 8; o += RP_NT * 128)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(vb + o));
        }
        const char *rb = reinterpret_cast<const char *>(A.ii_in + c0);
        for (int64_t o = (int64_t)tid * 128; o < nrow * 4; o += RP_NT * 128)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(rb + o));
    }

    // passes after the first read the valid triplets the first one wrote
    const int64_t Lp = FIRST ? A.L : (int64_t)*((volatile const unsigned *)&err->rvalid);
    int col[RP_IPT];
#pragma unroll
    for (int r = 0; r < RP_IPT; ++r) {
        const int64_t idx = base + r * 32;
        col[r] = (idx < Lp) ? __ldg(A.jj_in + idx) : 0;
    }
    unsigned long long bad = ~0ull;
    unsigned over = 0, nval = 0;
    uint32_t rk[RP_IPT / 2];  // ranks, two 16-bit halves per word
#pragma unroll
    for (int r = 0; r < RP_IPT; ++r) {
        const int64_t idx = base + r * 32;
        const bool live = idx < Lp;
        const bool valid = live && col[r] >= 1 && col[r] <= A.N;
        const unsigned c0 = (unsigned)(col[r] - 1);
        const unsigned d = valid ? ((c0 >> A.shift) & dmask) : (unsigned)ndig;
        if (A.nbits && valid) atomicAdd(&S.hnext[(c0 >> A.nshift) & nmask], 1u);
        nval += valid;
        const unsigned peers = __match_any_sync(FULL, d);
        unsigned c = 0;
        if (valid) c = S.cnt[w][d];
        __syncwarp();
        if (valid && (peers & lt) == 0u) S.cnt[w][d] = (uint16_t)(c + __popc(peers));
        __syncwarp();
        const unsigned rr = c + __popc(peers & lt);
        if (r & 1) rk[r >> 1] |= rr << 16;
        else rk[r >> 1] = rr;
    }
    __syncthreads();
    // (digit, warp) digit-major scan: chunk-local base of every warp's run of a digit
    uint32_t tot = 0;
    if (tid < ndig) {
#pragma unroll
        for (int ww = 0; ww < RP_NW; ++ww) {
            const uint32_t c = S.cnt[ww][tid];
            S.cnt[ww][tid] = (uint16_t)tot;
            tot += c;
        }
    }
    uint32_t ctot;
    const uint32_t dstart = block_excl_sum<RP_NT, uint32_t>(tot, S.red, ctot);
    if (tid < ndig) {
#pragma unroll
        for (int ww = 0; ww < RP_NW; ++ww) S.cnt[ww][tid] = (uint16_t)(S.cnt[ww][tid] + dstart);
        // decoupled look-back of this digit's count across the chunks
        volatile unsigned long long *vlb = A.lb + b * ndig;
        unsigned long long excl = 0;
        if (b == 0) {
            vlb[tid] = ep_pack(A.tag, 2, tot);
        } else {
            vlb[tid] = ep_pack(A.tag, 1, tot);
            const volatile unsigned long long *p = A.lb + (b - 1) * ndig + tid;
            while (true) {
                unsigned long long wd;
                unsigned f;
                do {
                    wd = *p;
                    f = ep_flag(wd, A.tag);
                } while (f == 0);
                excl += wd & EP_VMASK;
                if (f == 2) break;
                p -= ndig;
            }
            vlb[tid] = ep_pack(A.tag, 2, excl + tot);
        }
        S.cbase[tid] = (uint32_t)(gstart + excl) - dstart;
    }
    __syncthreads();
    // values -> reorder buffer
#pragma unroll
    for (int r = 0; r < RP_IPT; ++r) {
        const int64_t idx = base + r * 32;
        const bool valid = idx < Lp && col[r] >= 1 && col[r] <= A.N;
        if (valid) {
            const unsigned d = ((unsigned)(col[r] - 1) >> A.shift) & dmask;
            const unsigned pos = S.cnt[w][d] + ((rk[r >> 1] >> ((r & 1) * 16)) & 0xffffu);
            S.buf[pos] = (unsigned long long)__double_as_longlong(__ldg(A.s_in + idx * A.s_stride));
            S.sdig[pos] = (uint16_t)d;
        }
    }
    __syncthreads();
    for (int k = tid; k < (int)ctot; k += RP_NT)
        A.s_out[S.cbase[S.sdig[k]] + (uint32_t)k] = __longlong_as_double((long long)S.buf[k]);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RP_IPT; ++r) {  // rows (re-read: the chunk is still in L2), validated once
        const int64_t idx = base + r * 32;
        const bool live = idx < Lp;
        const int row = live ? __ldg(A.ii_in + idx) : 1;
        if (FIRST && live) {
            if (row < 1) bad = min(bad, (unsigned long long)idx);
            else if (row > A.M) over = 1;
        }
        if (live && col[r] >= 1 && col[r] <= A.N) {
            const unsigned d = ((unsigned)(col[r] - 1) >> A.shift) & dmask;
            const unsigned pos = S.cnt[w][d] + ((rk[r >> 1] >> ((r & 1) * 16)) & 0xffffu);
            S.buf[pos] = ((unsigned long long)(uint32_t)row << 32) | (uint32_t)col[r];
        }
    }
    __syncthreads();
    for (int k = tid; k < (int)ctot; k += RP_NT) {
        const unsigned long long v = S.buf[k];
        const uint32_t o = S.cbase[S.sdig[k]] + (uint32_t)k;
        A.ii_out[o] = (int32_t)(v >> 32);
        A.jj_out[o] = (int32_t)(uint32_t)v;
    }
    pdl_trigger();
    if (A.nbits)
        for (int k = tid; k <= (int)nmask; k += RP_NT)
            if (S.hnext[k]) atomicAdd(&A.hist_next[k], S.hnext[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        bad = min(bad, __shfl_xor_sync(FULL, bad, o));
        over |= __shfl_xor_sync(FULL, over, o);
        nval += __shfl_xor_sync(FULL, nval, o);
    }
    if (lane == 0) {
        if (FIRST) {
            if (bad != ~0ull) atomicMin(&err->bad_i, bad);
            if (over) err->over_m = 1;
        }
        if (A.pass == 0 && nval) atomicAdd(&err->rvalid, nval);
    }
}

// ---------------------------------------------------------------------------
// k_rbounds: start of every sub-bucket s = (col-1) >> w in the partitioned
// column array (lower bound; the array is sorted by sub-bucket), and the
// list of sub-buckets longer than RF_CAP.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t sub_lower_bound(const int32_t *__restrict__ jj, uint32_t n,
                                                    int w, uint32_t s) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (((uint32_t)(__ldg(jj + mid) - 1) >> w) < s) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void k_rbounds(const int32_t *__restrict__ jj, int w, int32_t nsub,
                          uint32_t *__restrict__ bnd, uint32_t *__restrict__ biglist,
                          ErrState *err) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    pdl_wait();
    if (s <= nsub) {
        const uint32_t n = *((volatile const unsigned *)&err->rvalid);
        const uint32_t a = (s == 0) ? 0u : (s == nsub ? n : sub_lower_bound(jj, n, w, (uint32_t)s));
        bnd[s] = a;
        if (s < nsub) {
            const uint32_t e = (s + 1 == nsub) ? n : sub_lower_bound(jj, n, w, (uint32_t)s + 1);
            if (e - a > (uint32_t)RF_CAP) biglist[atomicAdd(&err->rbig_n, 1u)] = (uint32_t)s;
        }
    }
    pdl_trigger();
}

// ---------------------------------------------------------------------------
// k_rbig: oversize sub-buckets, one 1024-thread CTA each (grid-stride over
// the list).  Keys (col_local << rbits | row-1) << 32 | k in scratch A, a
// stable LSD radix sort on the key bits (big_radix_pass, 8-bit digits, A <->
// B), values gathered in sorted order, each run of equal keys folded from
// +0.0 in k (= input) order, heads compacted.  Result: keys (high 32 bits)
// in one buffer, value bits in the other, bigu[s] = U | BIGFLAG if the keys
// ended in B.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(BIG_NT, 1) k_rbig(RadixFoldArgs F, ErrState *err) {
    __shared__ uint32_t s_cnt[BIG_NW][256];
    __shared__ uint32_t s_warp[BIG_NW];
    __shared__ unsigned long long s_prev;
    const int tid = threadIdx.x;
    pdl_wait();
    const unsigned nbig = *((volatile const unsigned *)&err->rbig_n);
    const int kbits = F.w + F.rbits;
    const int passes = (kbits + 7) / 8;
    for (unsigned q = blockIdx.x; q < nbig; q += gridDim.x) {
        const uint32_t s = F.biglist[q];
        const uint32_t a = F.bnd[s], n = F.bnd[s + 1] - a;
        const uint32_t c0 = s << F.w;
        unsigned long long *A = F.scrA + a;
        unsigned long long *B = F.scrB + a;
        for (uint32_t k = tid; k < n; k += BIG_NT) {
            const uint32_t key = ((uint32_t)(F.jj[a + k] - 1) - c0) << F.rbits | (uint32_t)(F.ii[a + k] - 1);
            A[k] = ((unsigned long long)key << 32) | k;
        }
        __syncthreads();
        unsigned long long *src = A, *dst = B;
        for (int p = 0; p < passes; ++p) {
            big_radix_pass(src, dst, n, 32 + 8 * p, s_cnt, s_warp);
            unsigned long long *t = src;
            src = dst;
            dst = t;
        }
        for (uint32_t k = tid; k < n; k += BIG_NT)
            dst[k] = (unsigned long long)__double_as_longlong(__ldg(F.s + a + (uint32_t)src[k]));
        __syncthreads();
        {  // ordered fold of every run; the result lands at the run's head
            const uint32_t lo = (uint32_t)((uint64_t)tid * n / BIG_NT);
            const uint32_t hi = (uint32_t)((uint64_t)(tid + 1) * n / BIG_NT);
            uint32_t p = lo;
            while (p < hi) {
                const uint32_t key = (uint32_t)(src[p] >> 32);
                if (p > 0 && (uint32_t)(src[p - 1] >> 32) == key) {
                    ++p;
                    continue;
                }
                double acc = fold_add(0.0, __longlong_as_double((long long)dst[p]));
                uint32_t r = p + 1;
                while (r < n && (uint32_t)(src[r] >> 32) == key) {
                    acc = fold_add(acc, __longlong_as_double((long long)dst[r]));
                    ++r;
                }
                dst[p] = (unsigned long long)__double_as_longlong(acc);
                p = r;
            }
        }
        __syncthreads();
        if (tid == 0) s_prev = ~0ull;
        __syncthreads();
        uint32_t carry = 0;
        for (uint32_t b0 = 0; b0 < n; b0 += BIG_NT) {
            const uint32_t p = b0 + tid;
            const bool valid = p < n;
            const unsigned long long key = valid ? (src[p] >> 32) : 0ull;
            const unsigned long long prev = (tid == 0) ? s_prev : (valid ? (src[p - 1] >> 32) : 0ull);
            const bool head = valid && key != prev;
            const unsigned long long val = head ? dst[p] : 0ull;
            uint32_t tot;
            const uint32_t run = block_excl_sum<BIG_NT, uint32_t>(head ? 1u : 0u, s_warp, tot) + carry;
            if (tid == BIG_NT - 1) s_prev = valid ? key : s_prev;
            __syncthreads();
            if (head) {
                src[run] = key << 32;
                dst[run] = val;
            }
            carry += tot;
            __syncthreads();
        }
        if (tid == 0) F.bigu[s] = carry | ((src == B) ? BIGFLAG : 0u);
        __syncthreads();
    }
    pdl_trigger();
}

// ---------------------------------------------------------------------------
// k_rfold: one CTA per sub-bucket (ticket order), everything in shared
// memory.  Records k = 0..n-1 are the sub-bucket's triplets in input order.
//   1. hash (col_local, row) -> slot; per slot a member count; a fresh slot
//      becomes group g (glist[g] = slot) and counts its column;
//   2. the sub-bucket's distinct count U is published (look-back aggregate);
//   3. member lists: group starts by a block scan, members placed with shared
//      atomics (unordered); groups of more than 32 members are rebuilt in
//      order by a warp ballot-scan;
//   4. output order: groups placed per column, each column's groups sorted by
//      row (insertion sort; a CTA bitonic sort of all groups when a column has
//      more than 32 distinct rows);
//   5. look-back walk -> global offset; thread per output entry: the group's
//      members sorted by k (insertion sort, <= 32) and folded from +0.0;
//      ir / pr / jc written coalesced.
// ---------------------------------------------------------------------------
constexpr int RF_NT = 256;
constexpr int RF_HS = 2 * RF_CAP;
constexpr int RF_BIGG = 128;  // groups of > 32 members per sub-bucket (<= RF_CAP / 33)

struct FoldSmem {
    uint32_t key[RF_HS];          // hash keys (key + 1; 0 = empty); sort items in the fallback
    uint32_t cnt[RF_HS];          // members per slot, then member cursor
    uint16_t gid[RF_CAP];         // slot of record k; then: group of output entry p
    uint16_t memb[RF_CAP];        // member records, grouped
    uint16_t glist[RF_CAP];       // slot of group g
    uint16_t gstart[RF_CAP + 1];  // first member of group g
    uint16_t ord[RF_CAP];         // groups listed per column (unordered)
    uint32_t colst[RF_WMAX + 1];  // distinct groups per column -> column start
    uint32_t colcur[RF_WMAX];
    uint16_t bigg[RF_BIGG];       // groups of more than 32 members
    uint32_t red[RF_NT / 32];
    int U, nbigg, sortall, b;
    long long off;
};

__device__ __forceinline__ unsigned rf_insert(uint32_t *key, int hbits, uint32_t k, bool &fresh) {
    const unsigned hmask = (1u << hbits) - 1u;
    unsigned h = (k * 0x9E3779B1u) >> (32 - hbits);
    while (true) {
        const uint32_t old = atomicCAS(&key[h], 0u, k);
        if (old == 0u) {
            fresh = true;
            return h;
        }
        if (old == k) {
            fresh = false;
            return h;
        }
        h = (h + 1) & hmask;
    }
}

__device__ __forceinline__ void rf_isort16(uint16_t *a, int n) {  // ascending, in place
    for (int i = 1; i < n; ++i) {
        const uint16_t x = a[i];
        int j = i - 1;
        while (j >= 0 && a[j] > x) {
            a[j + 1] = a[j];
            --j;
        }
        a[j + 1] = x;
    }
}

__global__ void __launch_bounds__(RF_NT, 2) k_rfold(RadixFoldArgs F, ErrState *err) {
    extern __shared__ __align__(16) unsigned char rf_smem[];
    FoldSmem &S = *reinterpret_cast<FoldSmem *>(rf_smem);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = lanemask_lt();
    pdl_wait();
    if (tid == 0) S.b = (int)atomicAdd(&err->rf_ticket, 1u);
    __syncthreads();
    const int64_t s = S.b;
    const uint32_t a = F.bnd[s], n = F.bnd[s + 1] - a;
    const int64_t c0 = s << F.w;
    const int ncol = (int)min((int64_t)1 << F.w, (int64_t)F.N - c0);
    const uint32_t rmask = (F.rbits >= 32) ? 0xffffffffu : ((1u << F.rbits) - 1u);
    unsigned long long *lbs = F.lbf + s * LB_STRIDE;
    bool over = false;

    if (n > (uint32_t)RF_CAP) {  // oversize: k_rbig left U sorted results in scratch
        const uint32_t ub = F.bigu[s];
        const uint32_t U = ub & POSMASK;
        const unsigned long long *RK = (ub & BIGFLAG) ? F.scrB + a : F.scrA + a;
        const unsigned long long *RV = (ub & BIGFLAG) ? F.scrA + a : F.scrB + a;
        if (warp == 0) {
            if (lane == 0) ((volatile unsigned long long *)lbs)[0] = ep_pack(F.tag, s == 0 ? 2 : 1, U);
            const unsigned long long e = ep_walk_warp(F.lbf, s, F.tag);
            if (lane == 0) {
                ((volatile unsigned long long *)lbs)[0] = ep_pack(F.tag, 2, e + U);
                S.off = (long long)e;
            }
        }
        __syncthreads();
        const long long off = S.off;
        for (int c = tid; c < ncol; c += RF_NT) {  // first result of column c
            uint32_t lo = 0, hi = U;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if ((uint32_t)(RK[mid] >> 32) >> F.rbits < (uint32_t)c) lo = mid + 1;
                else hi = mid;
            }
            F.jc[c0 + c] = (int32_t)(off + lo);
        }
        for (uint32_t p = tid; p < U; p += RF_NT) {
            if (off + p < F.cap) {
                F.ir[off + p] = (int32_t)((uint32_t)(RK[p] >> 32) & rmask);
                F.pr[off + p] = __longlong_as_double((long long)RV[p]);
            } else {
                over = true;
            }
        }
        if (s == F.nsub - 1 && tid == 0) {
            F.jc[F.N] = (int32_t)(off + U);
            err->nnz = off + U;
            if (off + U > F.cap) atomicExch(&err->cap_exceeded, 1u);
        }
        if (over) atomicExch(&err->cap_exceeded, 1u);
        pdl_trigger();
        return;
    }

    // ---- 1. groups -------------------------------------------------------
    {  // the sub-bucket's values into L1 while the groups are built (the fold reads them)
        const char *vb = reinterpret_cast<const char *>(F.s + a);
        const uint32_t nb = n * 8u;
        for (uint32_t o = (uint32_t)tid * 128u; o < nb; o += RF_NT * 128u)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(vb + o));
    }
    int hbits = 6;
    while ((1u << hbits) < 2 * n) ++hbits;
    const int hs = 1 << hbits;
    for (int k = tid; k < hs; k += RF_NT) {
        S.key[k] = 0u;
        S.cnt[k] = 0;
    }
    for (int c = tid; c <= ncol; c += RF_NT) S.colst[c] = 0;
    if (tid == 0) {
        S.U = 0;
        S.nbigg = 0;
        S.sortall = 0;
    }
    constexpr int RIPT = RF_CAP / RF_NT;
    uint32_t kk[RIPT];  // (col_local << rbits | row-1) + 1 of records tid + u * RF_NT
#pragma unroll
    for (int u = 0; u < RIPT; ++u) {
        const uint32_t k = tid + u * RF_NT;
        kk[u] = 0u;
        if (k < n) {
            const uint32_t cl = (uint32_t)(__ldg(F.jj + a + k) - 1) - (uint32_t)c0;
            kk[u] = ((cl << F.rbits) | (uint32_t)(__ldg(F.ii + a + k) - 1)) + 1u;
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < RIPT; ++u) {
        const uint32_t k = tid + u * RF_NT;
        if (k < n) {
            bool fresh;
            const unsigned h = rf_insert(S.key, hbits, kk[u], fresh);
            S.gid[k] = (uint16_t)h;
            atomicAdd(&S.cnt[h], 1u);
            if (fresh) {
                S.glist[atomicAdd(&S.U, 1)] = (uint16_t)h;
                atomicAdd(&S.colst[(kk[u] - 1u) >> F.rbits], 1u);
            }
        }
    }
    __syncthreads();
    const int U = S.U;
    if (tid == 0) ((volatile unsigned long long *)lbs)[0] = ep_pack(F.tag, s == 0 ? 2 : 1, (unsigned)U);

    // ---- 2. member starts, column starts ------------------------------------
    {  // exclusive scan of the member counts in group order -> gstart
        const int g0 = tid * RIPT;
        uint32_t loc[RIPT], sum = 0;
#pragma unroll
        for (int u = 0; u < RIPT; ++u) {
            loc[u] = (g0 + u < U) ? S.cnt[S.glist[g0 + u]] : 0u;
            sum += loc[u];
        }
        uint32_t tot;
        uint32_t pre = block_excl_sum<RF_NT, uint32_t>(sum, S.red, tot);
#pragma unroll
        for (int u = 0; u < RIPT; ++u) {
            if (g0 + u < U) S.gstart[g0 + u] = (uint16_t)pre;
            pre += loc[u];
        }
    }
    smem_excl_scan<RF_NT, 1, uint32_t>(S.colst, ncol, S.red);
    for (int g = tid; g < U; g += RF_NT) {
        const unsigned h = S.glist[g];
        const int m = S.cnt[h];
        S.cnt[h] = S.gstart[g];  // member cursor
        if (m > 32) {
            const int q = atomicAdd(&S.nbigg, 1);
            if (q < RF_BIGG) S.bigg[q] = (uint16_t)g;
        }
    }
    for (int c = tid; c < ncol; c += RF_NT) S.colcur[c] = S.colst[c];
    if (tid == 0) {
        S.gstart[U] = (uint16_t)n;
        S.colst[ncol] = (uint32_t)U;
    }
    __syncthreads();
    // ---- 3. members (unordered), groups per column ---------------------------------
#pragma unroll
    for (int u = 0; u < RIPT; ++u) {
        const uint32_t k = tid + u * RF_NT;
        if (k < n) S.memb[atomicAdd(&S.cnt[S.gid[k]], 1u)] = (uint16_t)k;
    }
    for (int g = tid; g < U; g += RF_NT) {
        const uint32_t cl = (S.key[S.glist[g]] - 1u) >> F.rbits;
        S.ord[atomicAdd(&S.colcur[cl], 1u)] = (uint16_t)g;  // column lists (unordered)
    }
    __syncthreads();
    for (int q = warp; q < min(S.nbigg, RF_BIGG); q += RF_NT / 32) {  // big groups: rebuilt in order
        const int g = S.bigg[q];
        const unsigned h = S.glist[g];
        int cur = S.gstart[g];
        for (uint32_t k0 = 0; k0 < n; k0 += 32) {
            const uint32_t k = k0 + lane;
            const bool mine = k < n && S.gid[k] == h;
            const unsigned bal = __ballot_sync(FULL, mine);
            if (mine) S.memb[cur + __popc(bal & lt)] = (uint16_t)k;
            cur += __popc(bal);
        }
    }
    // ---- 4. output order: rank of every group among its column's groups ----------
    uint16_t opos[RIPT];
#pragma unroll
    for (int u = 0; u < RIPT; ++u) {
        const int g = tid + u * RF_NT;
        opos[u] = 0;
        if (g < U) {
            const uint32_t kx = S.key[S.glist[g]];
            const int st = S.colst[(kx - 1u) >> F.rbits], en = S.colst[((kx - 1u) >> F.rbits) + 1];
            if (en - st > 64) {
                S.sortall = 1;
            } else {
                int r = st;
                for (int q = st; q < en; ++q) r += S.key[S.glist[S.ord[q]]] < kx;
                opos[u] = (uint16_t)r;
            }
        }
    }
    __syncthreads();
    const bool sortall = S.sortall != 0;
    unsigned long long *items = reinterpret_cast<unsigned long long *>(S.key);  // fallback only
    if (!sortall) {
#pragma unroll
        for (int u = 0; u < RIPT; ++u) {
            const int g = tid + u * RF_NT;
            if (g < U) S.gid[opos[u]] = (uint16_t)g;  // gid := group of output entry
        }
    } else {  // CTA bitonic sort of all groups by key (a column with > 64 distinct rows)
        int np2 = 1;
        while (np2 < U) np2 <<= 1;
        unsigned long long it[RIPT];
#pragma unroll
        for (int u = 0; u < RIPT; ++u) {
            const int g = tid + u * RF_NT;
            it[u] = (g < U) ? (((unsigned long long)S.key[S.glist[g]] << 16) | (unsigned)g) : ~0ull;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < RIPT; ++u) {
            const int g = tid + u * RF_NT;
            if (g < np2) items[g] = it[u];
        }
        __syncthreads();
        for (int k = 2; k <= np2; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int t = tid; t < (np2 >> 1); t += RF_NT) {
                    const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
                    const unsigned long long x = items[i], y = items[i + j];
                    if ((x > y) == ((i & k) == 0)) {
                        items[i] = y;
                        items[i + j] = x;
                    }
                }
                __syncthreads();
            }
        }
        for (int p = tid; p < U; p += RF_NT) S.gid[p] = (uint16_t)(items[p] & 0xffffu);
    }
    // ---- 5. offset, fold, outputs -------------------------------------------------
    if (warp == 0) {
        const unsigned long long e = ep_walk_warp(F.lbf, s, F.tag);
        if (lane == 0) {
            ((volatile unsigned long long *)lbs)[0] = ep_pack(F.tag, 2, e + (unsigned)U);
            S.off = (long long)e;
        }
    }
    __syncthreads();
    const long long off = S.off;
    const double *__restrict__ sv = F.s + a;
    for (int p = tid; p < U; p += RF_NT) {
        const int g = S.gid[p];
        const int st = S.gstart[g], en = S.gstart[g + 1];
        const uint32_t kx = sortall ? (uint32_t)(items[p] >> 16) : S.key[S.glist[g]];
        if (en - st <= 32) rf_isort16(S.memb + st, en - st);
        double acc = 0.0;
        for (int q = st; q < en; ++q) acc = fold_add(acc, __ldg(sv + S.memb[q]));
        if (off + p < F.cap) {
            F.ir[off + p] = (int32_t)((kx - 1u) & rmask);
            F.pr[off + p] = acc;
        } else {
            over = true;
        }
    }
    for (int c = tid; c < ncol; c += RF_NT) F.jc[c0 + c] = (int32_t)(off + S.colst[c]);
    if (s == F.nsub - 1 && tid == 0) {
        F.jc[F.N] = (int32_t)(off + U);
        err->nnz = off + U;
        if (off + U > F.cap) atomicExch(&err->cap_exceeded, 1u);
    }
    if (over) atomicExch(&err->cap_exceeded, 1u);
    pdl_trigger();
}

// ---- launchers -----------------------------------------------------------------
cudaError_t launch_rhist(Launch &lc, const int32_t *jj, int64_t L, int32_t N, int shift, int bits,
                         uint32_t *hist, ErrState *err) {
    if (L <= 0) return cudaSuccess;
    const int64_t want = (L + RH_NT * RH_U - 1) / (RH_NT * RH_U);
    const int grid = (int)std::min<int64_t>(want, (int64_t)lc.num_sms * 8);
    cudaError_t e = launch_pdl(k_rhist, dim3(grid), dim3(RH_NT), 0, lc.stream, jj, L, N, shift, bits,
                               hist, err);
    lc.launches++;
    return e;
}

cudaError_t launch_rpass(Launch &lc, const RadixPassArgs &A, bool first, int64_t nchunk,
                         ErrState *err) {
    if (nchunk <= 0) return cudaSuccess;
    const int smem = (int)sizeof(PassSmem);
    cudaError_t e = first ? ensure_smem_attr((const void *)k_rpass<true>, smem)
                          : ensure_smem_attr((const void *)k_rpass<false>, smem);
    if (e != cudaSuccess) return e;
    e = first ? launch_pdl(k_rpass<true>, dim3((unsigned)nchunk), dim3(RP_NT), smem, lc.stream, A, err)
              : launch_pdl(k_rpass<false>, dim3((unsigned)nchunk), dim3(RP_NT), smem, lc.stream, A, err);
    lc.launches++;
    return e;
}

cudaError_t launch_rbounds(Launch &lc, const int32_t *jj, int w, int32_t nsub, uint32_t *bnd,
                           uint32_t *biglist, ErrState *err) {
    const int64_t n = (int64_t)nsub + 1;
    cudaError_t e = launch_pdl(k_rbounds, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, lc.stream,
                               jj, w, nsub, bnd, biglist, err);
    lc.launches++;
    return e;
}

cudaError_t launch_rbig(Launch &lc, const RadixFoldArgs &F, ErrState *err) {
    cudaError_t e = launch_pdl(k_rbig, dim3((unsigned)lc.num_sms), dim3(BIG_NT), 0, lc.stream, F, err);
    lc.launches++;
    return e;
}

cudaError_t launch_rfold(Launch &lc, const RadixFoldArgs &F, ErrState *err) {
    const int smem = (int)sizeof(FoldSmem);
    cudaError_t e = ensure_smem_attr((const void *)k_rfold, smem);
    if (e != cudaSuccess) return e;
    e = launch_pdl(k_rfold, dim3((unsigned)F.nsub), dim3(RF_NT), smem, lc.stream, F, err);
    lc.launches++;
    return e;
}

}  // namespace sa
