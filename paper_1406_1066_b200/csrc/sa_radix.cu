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
//   per pass (stable LSD partition on one digit of the column):
//   k_rup      per-segment digit histograms of the pass input (S contiguous
//              segments, one per resident partition CTA); the first also
//              validates the columns
//   k_rscan    every segment's global base per digit
//   k_rpass    the partition: CTA s walks its segment's chunks in order
//              (chunk-local stable rank from per-warp running counters over
//              digit ballots, a running base per digit in shared memory,
//              coalesced scatter through shared memory), 16 B per triplet
//              in and out; the first pass validates the rows
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

#include <cstddef>
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
// Partition passes without a look-back chain ("reduce, then scan").  The
// upsweep histograms the pass input chunk by chunk (RP_CHUNK triplets) --
// one CTA per block of RP_BLK chunks, which also sums its block -- a small
// scan turns the block sums into every block's global base per digit, and a
// third kernel turns them into every chunk's base per digit.  The
// partition CTAs then need no look-back: concurrently running CTAs take
// adjacent chunks (chunk = CTA + k x grid), so the output digit runs of
// neighbouring chunks are written at about the same time and L2 completes
// their sectors before they leave it.  (A decoupled look-back per digit spent
// a quarter of the pass's instructions spinning; contiguous per-CTA segments
// without it left ~150k partially written write fronts in L2 and cost 50 %
// extra DRAM traffic in read-modify-writes.)
// ---------------------------------------------------------------------------
constexpr int RU_NT = 512;

// Digit of the sort key (col - 1) << rbits | (row - 1) at bit `shift`.  The
// column-block plan only uses digits of the column bits (shift >= rbits);
// the row-split plan (few, long columns) also the row bits.
__device__ __forceinline__ unsigned key_digit(int col, int row, int shift, int rbits, unsigned dmask) {
    if (shift >= rbits) return ((unsigned)(col - 1) >> (shift - rbits)) & dmask;
    const unsigned long long key = ((unsigned long long)(unsigned)(col - 1) << rbits) | (unsigned)(row - 1);
    return (unsigned)(key >> shift) & dmask;
}

// Sort key of a (valid) triplet.
__device__ __forceinline__ unsigned long long tkey(int col, int row, int rbits) {
    return ((unsigned long long)(unsigned)(col - 1) << rbits) | (unsigned)(row - 1);
}

// Key relative to the first key of its sub-bucket (K0 = c0 << rbits | roff),
// in 32 bits: column-block plan (z >= rbits, roff = 0) the local column and
// the row; row-split plan (one column) the row offset.
__device__ __forceinline__ uint32_t lkey(int col, int row, int z, int rbits, uint32_t c0, uint32_t roff) {
    return z >= rbits ? (((uint32_t)(col - 1) - c0) << rbits) | (uint32_t)(row - 1)
                      : (uint32_t)(row - 1) - roff;
}

// Any index error: the call fails, the fold's work is moot (and rows beyond
// M would spill into the column bits of the fold's keys).
__device__ __forceinline__ bool call_failed(const ErrState *err) {
    return err->bad_i != ~0ull || err->bad_j != ~0ull || err->over_m || err->over_n;
}

// Intermediate partition buffers hold {row, col} pairs (as the last pass's
// output) instead of separate row and column arrays.
#ifndef SA_PAIRS
#define SA_PAIRS 1
#endif
#ifndef SA_RUP_PRED
#define SA_RUP_PRED 1
#endif

// k_rup: per-chunk digit histograms cnt[c][d] (16-bit) of the pass input (jj)
// and the block's sums bsum[B][d].  The first pass also validates the
// columns (first index < 1, any index > N) and counts the valid triplets
// (err->rvalid, the length the later passes read).
template <bool FIRST, bool ROWKEY>
__global__ void __launch_bounds__(RU_NT) k_rup(const int32_t *__restrict__ ii, const int32_t *__restrict__ jj,
                                               const int2 *__restrict__ rc, int64_t L, int32_t N, int shift, int bits, int rbits, int cpb,
                                               uint16_t *__restrict__ cnt, uint32_t *__restrict__ bsum,
                                               ErrState *err) {
    // two histograms: chunk c counts into h[c & 1] while the loads of chunk
    // c + 1 are in flight; one barrier per chunk (the owner of digit k writes
    // out and clears its counter for chunk c + 2)
    __shared__ uint32_t h[2][RP_MAXD];
    for (int k = threadIdx.x; k < 2 * RP_MAXD; k += RU_NT) h[k >> RP_MAXBITS][k & (RP_MAXD - 1)] = 0;
    pdl_wait();
    const int64_t Lp = FIRST ? L : (int64_t)*((volatile const unsigned *)&err->rvalid);
    const int64_t nchunk = (Lp + RP_CHUNK - 1) / RP_CHUNK;
    const unsigned dmask = (1u << bits) - 1u;
    const int ndig = 1 << bits;
    unsigned long long bad = ~0ull;
    unsigned over = 0, nval = 0;
    uint32_t bs = 0;  // block sum of digit threadIdx.x
    // a chunk is counted in RU_SUB pieces (at most 8 K triplets each: the piece in
    // hand and the one in flight stay in registers)
    constexpr int RU_SUB = RP_CHUNK > 8192 ? 2 : 1;
    constexpr int RU_PIECE = RP_CHUNK / RU_SUB;
    constexpr int UPT = RU_PIECE / RU_NT;
    static_assert(RU_PIECE % (2 * RU_NT) == 0, "16- and 8-byte loads of whole pieces");
    const int64_t cb = (int64_t)blockIdx.x * cpb, ce = min(nchunk, cb + cpb);
    // Whole chunks of a 16-byte aligned array are read with 16-byte loads
    // (thread t holds the elements 4 (t + 512 u) .. + 3: a histogram does not
    // care which thread counts what), a partial last chunk or an unaligned
    // array element by element.  Valid columns take the short way (one
    // unsigned compare); the position of a bad one is worked out only then.
    constexpr bool PAIRS = !FIRST && SA_PAIRS;  // input: {row, col} pairs (rc)
    const bool al16 = ((PAIRS ? reinterpret_cast<uintptr_t>(rc) : reinterpret_cast<uintptr_t>(jj)) & 15) == 0;
    const int csh = shift - rbits;
    int v[UPT];
#if SA_PAIRS
    if (PAIRS) {
        // thread t holds the pairs 2 (t + RU_NT u), + 1 of a whole chunk (one
        // 16-byte load each), or t + RU_NT u of a partial / unaligned one
        int vr[ROWKEY ? UPT : 1], vnr[ROWKEY ? UPT : 1];
        auto vecmode = [&](int64_t q) { return al16 && (q + 1) * RU_PIECE <= Lp; };
        auto load = [&](int64_t c, int (&x)[UPT], int (&xr)[ROWKEY ? UPT : 1]) {
            const int64_t lo = c * RU_PIECE;
            if (vecmode(c)) {
                const int4 *p4 = reinterpret_cast<const int4 *>(rc + lo) + threadIdx.x;
#pragma unroll
                for (int u = 0; u < UPT / 2; ++u) {
                    const int4 q = __ldcs(p4 + u * RU_NT);
                    x[2 * u] = q.y;
                    x[2 * u + 1] = q.w;
                    if (ROWKEY) {
                        xr[2 * u] = q.x;
                        xr[2 * u + 1] = q.z;
                    }
                }
            } else {
                const int64_t hi = min(Lp, lo + RU_PIECE);
#pragma unroll
                for (int u = 0; u < UPT; ++u) {
                    const int64_t t = lo + threadIdx.x + (int64_t)u * RU_NT;
                    const int2 q = (t < hi) ? __ldcs(rc + t) : make_int2(1, 0);  // (column 0: padding)
                    x[u] = q.y;
                    if (ROWKEY) xr[u] = q.x;
                }
            }
        };
        if (cb < ce) load(cb * RU_SUB, v, vr);
        __syncthreads();
        for (int64_t c = cb * RU_SUB; c < ce * RU_SUB; ++c) {  // c: piece; chunk c / RU_SUB
            int vn[UPT];
            if (c + 1 < ce * RU_SUB) load(c + 1, vn, vnr);
            uint32_t *hc = h[(c / RU_SUB) & 1];
#if SA_RUP_PRED
            if (!ROWKEY && vecmode(c)) {  // whole chunk of stored (valid) columns: no tests
#pragma unroll
                for (int u = 0; u < UPT; ++u) atomicAdd(&hc[((unsigned)(v[u] - 1) >> csh) & dmask], 1u);
            } else
#endif
#pragma unroll
            for (int u = 0; u < UPT; ++u) {
                const int cc = v[u];
                if (cc < 1) continue;  // padding of a partial chunk (stored columns are valid)
                if (ROWKEY) atomicAdd(&hc[key_digit(cc, vr[ROWKEY ? u : 0], shift, rbits, dmask)], 1u);
                else atomicAdd(&hc[((unsigned)(cc - 1) >> csh) & dmask], 1u);
            }
            if (c % RU_SUB == RU_SUB - 1) {  // the chunk's last piece
                __syncthreads();
                for (int k = threadIdx.x; k < ndig; k += RU_NT) {
                    cnt[(c / RU_SUB) * RP_MAXD + k] = (uint16_t)hc[k];
                    bs += hc[k];  // RU_NT == RP_MAXD: thread k owns digit k
                    hc[k] = 0;
                }
            }
#pragma unroll
            for (int u = 0; u < UPT; ++u) {
                v[u] = vn[u];
                if (ROWKEY) vr[u] = vnr[u];
            }
        }
        if (threadIdx.x < ndig) bsum[(int64_t)blockIdx.x * RP_MAXD + threadIdx.x] = bs;
        pdl_trigger();
        return;
    }
#endif
    auto vecmode = [&](int64_t q) { return al16 && (q + 1) * RU_PIECE <= Lp; };
    auto load = [&](int64_t c, int (&x)[UPT]) {
        const int64_t lo = c * RU_PIECE;
        if (vecmode(c)) {
            const int4 *p4 = reinterpret_cast<const int4 *>(jj + lo) + threadIdx.x;
#pragma unroll
            for (int u = 0; u < UPT / 4; ++u) {
                const int4 q = __ldcs(p4 + u * RU_NT);
                x[4 * u] = q.x;
                x[4 * u + 1] = q.y;
                x[4 * u + 2] = q.z;
                x[4 * u + 3] = q.w;
            }
            if (UPT % 4) {  // the piece's tail: one 8-byte load (UPT % 4 == 2)
                constexpr int U4 = UPT / 4 * 4;
                const int2 q = __ldcs(reinterpret_cast<const int2 *>(jj + lo + U4 * RU_NT) + threadIdx.x);
                x[U4] = q.x;
                x[U4 + 1] = q.y;
            }
        } else {
            const int64_t hi = min(Lp, lo + RU_PIECE);
#pragma unroll
            for (int u = 0; u < UPT; ++u) {
                const int64_t t = lo + threadIdx.x + (int64_t)u * RU_NT;
                x[u] = (t < hi) ? __ldcs(jj + t) : 1;  // (padding: a valid column, not counted)
            }
        }
    };
    if (cb < ce) load(cb * RU_SUB, v);
    __syncthreads();
    for (int64_t c = cb * RU_SUB; c < ce * RU_SUB; ++c) {  // c: piece; chunk c / RU_SUB
        int vn[UPT];
        if (c + 1 < ce * RU_SUB) load(c + 1, vn);
        uint32_t *hc = h[(c / RU_SUB) & 1];
        const int64_t lo = c * RU_PIECE, hi = min(Lp, lo + RU_PIECE);
        const bool vec = vecmode(c);
        // element index of v[u] within the chunk
        auto eidx = [&](int u) -> int {
            constexpr int U4 = UPT / 4 * 4;
            if (!vec) return (int)threadIdx.x + u * RU_NT;
            return u < U4 ? 4 * ((int)threadIdx.x + (u >> 2) * RU_NT) + (u & 3)
                          : U4 * RU_NT + 2 * (int)threadIdx.x + (u - U4);
        };
#if SA_RUP_PRED
        if (vec && !ROWKEY) {
            // whole chunk, column digits: branch-free -- a predicated shared
            // reduction per element, the valid ones counted; the (rare) bad
            // indices are looked at afterwards
            const unsigned hb = (unsigned)__cvta_generic_to_shared(hc);
            unsigned nok = 0, nbad = 0;
#pragma unroll
            for (int u = 0; u < UPT; ++u) {
                const unsigned c1 = (unsigned)v[u] - 1u;
                const unsigned ok = (!FIRST || c1 < (unsigned)N) ? 1u : 0u;
                const unsigned a = hb + (((c1 >> csh) & dmask) << 2);
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t@p red.shared.add.u32 [%0], 1;\n\t}"
                             ::"r"(a), "r"(ok) : "memory");
                nok += ok;
                nbad += 1u - ok;
            }
            nval += nok;
            if (FIRST && nbad) {
#pragma unroll
                for (int u = 0; u < UPT; ++u) {
                    const int cc = v[u];
                    if ((unsigned)(cc - 1) < (unsigned)N) continue;
                    if (cc < 1) bad = min(bad, (unsigned long long)(lo + eidx(u)));
                    else over = 1;
                }
            }
        } else
#endif
#pragma unroll
        for (int u = 0; u < UPT; ++u) {
            const int cc = v[u];
            if (!FIRST || (unsigned)(cc - 1) < (unsigned)N) {
                if (!vec && lo + eidx(u) >= hi) continue;  // padding of a partial chunk
                if (ROWKEY)  // the digit takes row bits (row-split plan)
                    atomicAdd(&hc[key_digit(cc, __ldcs(ii + lo + eidx(u)), shift, rbits, dmask)], 1u);
                else
                    atomicAdd(&hc[((unsigned)(cc - 1) >> csh) & dmask], 1u);
                ++nval;
            } else {
                if (cc < 1) bad = min(bad, (unsigned long long)(lo + eidx(u)));
                else over = 1;
            }
        }
        if (c % RU_SUB == RU_SUB - 1) {  // the chunk's last piece
            __syncthreads();
            for (int k = threadIdx.x; k < ndig; k += RU_NT) {
                cnt[(c / RU_SUB) * RP_MAXD + k] = (uint16_t)hc[k];
                bs += hc[k];  // RU_NT == RP_MAXD: thread k owns digit k
                hc[k] = 0;
            }
        }
#pragma unroll
        for (int u = 0; u < UPT; ++u) v[u] = vn[u];
    }
    if (threadIdx.x < ndig) bsum[(int64_t)blockIdx.x * RP_MAXD + threadIdx.x] = bs;
    if (FIRST) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            bad = min(bad, __shfl_xor_sync(FULL, bad, o));
            over |= __shfl_xor_sync(FULL, over, o);
            nval += __shfl_xor_sync(FULL, nval, o);
        }
        if ((threadIdx.x & 31) == 0) {
            if (bad != ~0ull) atomicMin(&err->bad_j, bad);
            if (over) err->over_n = 1;
            if (nval) atomicAdd(&err->rvalid, nval);
        }
    }
    pdl_trigger();
}

// k_rscan: bsum[B][d] := the count of digit d in blocks < B; tot[d] := the
// digit's total.  One warp per digit (lane q takes blocks q, q + 32, ...).
__global__ void __launch_bounds__(256) k_rscan(uint32_t *__restrict__ bsum, uint32_t *__restrict__ tot, int nblk,
                                               int bits) {
    const int lane = threadIdx.x & 31;
    const int d = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    pdl_wait();
    if (d < (1 << bits)) {
        uint32_t run = 0;
        for (int q0 = 0; q0 < nblk; q0 += 32) {
            const int q = q0 + lane;
            const uint32_t c = (q < nblk) ? bsum[(int64_t)q * RP_MAXD + d] : 0u;
            uint32_t x = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL, x, o);
                if (lane >= o) x += y;
            }
            if (q < nblk) bsum[(int64_t)q * RP_MAXD + d] = run + x - c;
            run += __shfl_sync(FULL, x, 31);
        }
        if (lane == 0) tot[d] = run;
    }
    pdl_trigger();
}

// k_roff: off[c][d] = the global position of chunk c's first digit-d triplet
// (the digit's base -- an exclusive scan of the digit totals, redone by
// every CTA -- plus the digit's count in earlier blocks and chunks).
__global__ void __launch_bounds__(RP_MAXD) k_roff(const uint16_t *__restrict__ cnt,
                                                  const uint32_t *__restrict__ bsum,
                                                  const uint32_t *__restrict__ tot, int bits,
                                                  uint32_t *__restrict__ off, ErrState *err, int64_t L,
                                                  int first, int cpb) {
    __shared__ uint32_t red[RP_MAXD / 32];
    const int d = threadIdx.x;
    pdl_wait();
    const int64_t Lp = first ? L : (int64_t)*((volatile const unsigned *)&err->rvalid);
    const int64_t nchunk = (Lp + RP_CHUNK - 1) / RP_CHUNK;
    const bool live = d < (1 << bits);
    uint32_t total;
    const uint32_t g = block_excl_sum<RP_MAXD, uint32_t>(live ? tot[d] : 0u, red, total);
    if (live) {
        uint32_t run = g + bsum[(int64_t)blockIdx.x * RP_MAXD + d];
        const int64_t cb = (int64_t)blockIdx.x * cpb;
        for (int64_t c = cb; c < min(nchunk, cb + cpb); ++c) {
            off[c * RP_MAXD + d] = run;
            run += cnt[c * RP_MAXD + d];
        }
    }
    pdl_trigger();
}

// L2 eviction priority "last" for the partition's output stores: a digit run
// of a chunk fills only part of a sector, the neighbouring chunk's run the
// rest; keeping the lines in L2 until both arrive avoids a DRAM
// read-modify-write of the sector.
__device__ __forceinline__ unsigned long long l2_evict_last() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st_last(int32_t *a, int32_t v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(a), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_last(double *a, double v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_last(uint4 *a, uint4 v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(a), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_last(int2 *a, int2 v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.v2.b32 [%0], {%1, %2}, %3;" ::"l"(a), "r"(v.x), "r"(v.y), "l"(pol)
                 : "memory");
}

// One sorted record {row, col, value bits} out: the last pass writes the
// {row, col} pair as one 8-byte store (what the fold and the bounds read),
// the others separate row and column arrays (the next upsweep reads the
// columns alone); the values go to their own array either way.
template <bool LAST>
__device__ __forceinline__ void put_rec(const RadixPassArgs &A, uint32_t o, uint4 v, unsigned long long pol) {
    if (LAST && SA_AOS) {  // one 16-byte record (the fold's and the bounds' input)
        st_last(reinterpret_cast<uint4 *>(A.rc_out) + o, v, pol);
        return;
    }
    if (LAST || SA_PAIRS) {
        st_last(A.rc_out + o, make_int2((int)v.x, (int)v.y), pol);
    } else {
        st_last(A.ii_out + o, (int32_t)v.x, pol);
        st_last(A.jj_out + o, (int32_t)v.y, pol);
    }
    st_last(A.s_out + o, __longlong_as_double((long long)(((unsigned long long)v.w << 32) | v.z)), pol);
}

// ---------------------------------------------------------------------------
// Pass building blocks shared by k_rpass and k_rpass_tma.
//
// Per-warp digit counters: RP_NW rows of RP_MAXD / 2 words (digits 2p and
// 2p + 1 in the 16-bit halves of word p), row stride RP_CS = 257 words so that
// the block-wide scan below (4 adjacent lanes per digit pair, 8 rows each)
// reads 32 distinct banks.
// ---------------------------------------------------------------------------
#ifndef SA_PASS_V2
#define SA_PASS_V2 1
#endif
#ifndef SA_SCAN1
#define SA_SCAN1 1
#endif
#ifndef SA_PASS_NOIDX
#define SA_PASS_NOIDX 1
#endif
#if SA_PASS_V2
constexpr int RP_CS = RP_MAXD / 2 + 1;
#else
constexpr int RP_CS = RP_MAXD / 2;
#endif

// Stable rank of a triplet among its warp's triplets of digit d so far (the
// running counter of (warp, d) advances by the step's group size).  Optimistic:
// every valid lane reads the counter, then takes a slot with its own shared
// atomic (one warp's shared-memory operations complete in program order, so
// all lanes of a step read the count from before the step).  A lane whose
// atomic returned something else shares its digit with another lane of this
// step; only those digits are re-ranked in lane order (a ballot per distinct
// conflicting digit) -- with 2^9 digits about one pair per step, against one
// ballot per digit bit for every step.
__device__ __forceinline__ unsigned rp_rank(uint32_t *cntw, unsigned d, bool valid, unsigned lt) {
    const unsigned sh = (d & 1u) * 16u;
    const unsigned addr = (unsigned)__cvta_generic_to_shared(cntw + (d >> 1));
    unsigned c0 = 0, rr = 0;
    if (valid) {
        unsigned w0, w1;
        asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(w0) : "r"(addr) : "memory");
        asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(w1) : "r"(addr), "r"(1u << sh) : "memory");
        c0 = (w0 >> sh) & 0xffffu;
        rr = (w1 >> sh) & 0xffffu;
    }
    unsigned fl = __ballot_sync(FULL, rr != c0);
    while (fl) {
        const int f = __ffs(fl) - 1;
        const unsigned df = __shfl_sync(FULL, d, f);
        const bool mine = valid && d == df;
        const unsigned same = __ballot_sync(FULL, mine);
        if (mine) rr = c0 + __popc(same & lt);
        fl &= ~same;
    }
    return rr;
}

// (digit, warp) digit-major exclusive scan of the per-warp counters, all
// RP_NT threads: thread (p = tid / 4, q = tid % 4) owns digit pair p in the
// warp rows 8 q .. 8 q + 7 (packed 16-bit adds; a half never exceeds the chunk
// size).  Every counter becomes the chunk-local start of its (digit, warp)
// run; returns through t0 / t1 / ex (valid for q == 0, p < npair) the pair's
// digit totals and the chunk-local start of digit 2p, and the chunk total.
template <int BITS>
__device__ __forceinline__ void rp_scan(uint32_t *cnt, uint32_t *red, uint32_t &t0, uint32_t &t1, uint32_t &ex,
                                        uint32_t &ctot) {
    static_assert(RP_NT == 1024 && RP_NW == 32, "rp_scan layout");
    constexpr int npair = ((1 << BITS) + 1) >> 1;
    const int tid = threadIdx.x, lane = tid & 31, p = tid >> 2, q = tid & 3;
    uint32_t c[8], part = 0;
    uint32_t *cp = cnt + (q * 8) * RP_CS + p;
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = (p < npair) ? cp[i * RP_CS] : 0u;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t x = c[i];
        c[i] = part;
        part += x;
    }
    uint32_t inc = part;
    uint32_t y = __shfl_up_sync(FULL, inc, 1);
    if (q >= 1) inc += y;
    y = __shfl_up_sync(FULL, inc, 2);
    if (q >= 2) inc += y;
    const uint32_t before = inc - part;  // rows of lower q (packed)
    const uint32_t totp = __shfl_sync(FULL, inc, lane | 3);
    t0 = totp & 0xffffu;
    t1 = totp >> 16;
#if SA_SCAN1
    // (one barrier; red is next written a chunk half later, barriers away)
    const uint32_t exq = block_excl_sum1<RP_NT, uint32_t>(q == 0 ? t0 + t1 : 0u, red, ctot);
#else
    const uint32_t exq = block_excl_sum<RP_NT, uint32_t>(q == 0 ? t0 + t1 : 0u, red, ctot);
#endif
    ex = __shfl_sync(FULL, exq, lane & ~3);
    if (p < npair) {
        const uint32_t add = (ex + (before & 0xffffu)) | ((ex + t0 + (before >> 16)) << 16);
#pragma unroll
        for (int i = 0; i < 8; ++i) cp[i * RP_CS] = c[i] + add;
    }
}

// ---------------------------------------------------------------------------
// k_rpass: one stable LSD partition pass by the digit (col-1) >> shift (the
// downsweep).  CTA s walks the RP_CHUNK-triplet chunks of segment s in order;
// warp w owns the chunk's w-th run of RP_IPT x 32 triplets.  All of a
// thread's triplets (row, column, value) are loaded up front.  The warp walks
// its run in order, 32 at a time: lanes of equal digit are found by one
// ballot per digit bit, and a per-warp running counter per digit (a shared
// atomic by the group's first lane) gives every triplet its rank -- stable by
// construction.  A scan over (digit, warp) makes the ranks chunk-local; the
// segment's running base per digit places the chunk.  Each triplet is then
// put, as one 16-byte record with its output index, at its sorted slot in
// shared memory, and the chunk is written out so that consecutive threads
// write consecutive addresses of one digit run.
// ---------------------------------------------------------------------------
struct PassSmem {
    uint4 rec[RP_CHUNK];              // reordered {row, col, value}
#if !SA_PASS_NOIDX
    uint32_t oidx[RP_CHUNK];          // output index of reordered slot k
#endif
    uint32_t cnt[RP_NW][RP_CS];       // per warp, digit pair (16-bit halves): running count, then base
    uint32_t run[RP_MAXD];            // the chunk's global base per digit
    uint32_t red[RP_NW];
};

template <bool FIRST, bool LAST, int BITS>
__global__ void __launch_bounds__(RP_NT, 1) k_rpass(RadixPassArgs A, ErrState *err) {
    extern __shared__ __align__(16) unsigned char rp_smem[];
    PassSmem &S = *reinterpret_cast<PassSmem *>(rp_smem);
    constexpr int ndig = 1 << BITS;
    constexpr unsigned dmask = (unsigned)ndig - 1u;
    constexpr int npair = (ndig + 1) >> 1;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const unsigned lt = lanemask_lt();
    pdl_wait();
    // passes after the first read the valid triplets the first one wrote
    const int64_t Lp = FIRST ? A.L : (int64_t)*((volatile const unsigned *)&err->rvalid);
    const int64_t nchunk = (Lp + RP_CHUNK - 1) / RP_CHUNK;
    const int shift = A.shift;
    const int32_t M = A.M, N = A.N;
    unsigned long long bad = ~0ull;
    unsigned over = 0;
    for (int64_t c = blockIdx.x; c < nchunk; c += gridDim.x) {
        const int64_t c0 = c * RP_CHUNK;
        const int64_t seg_hi = min(Lp, c0 + RP_CHUNK);
        {
            uint32_t *c32 = &S.cnt[0][0];
            for (int k = tid; k < RP_NW * npair; k += RP_NT) c32[(k / npair) * RP_CS + k % npair] = 0;
            for (int k = tid; k < ndig; k += RP_NT) S.run[k] = A.off[c * RP_MAXD + k];
        }
        const int64_t base = c0 + (int64_t)w * (RP_IPT * 32) + lane;
        const int nlive = (int)max((int64_t)0, min((int64_t)(RP_IPT * 32), seg_hi - (base - lane)));  // warp-uniform
        const int32_t *jp = A.jj_in + base, *ip = A.ii_in + base;
        const double *sp = A.s_in + (A.s_stride ? base : 0);
        const int sstep = A.s_stride ? 32 : 0;
        int col[RP_IPT], row[RP_IPT];
        double val[RP_IPT];
#pragma unroll
        for (int r = 0; r < RP_IPT; ++r) {
            const bool live = r * 32 + lane < nlive;
            // streaming loads (evict-first): the input must not push the
            // partially written output lines out of L2
            if (!FIRST && SA_PAIRS) {
                const int2 pr2 = live ? __ldcs(A.rc_in + base + r * 32) : make_int2(1, 0);
                row[r] = pr2.x;
                col[r] = pr2.y;
            } else {
                col[r] = live ? __ldcs(jp + r * 32) : 0;
                row[r] = live ? __ldcs(ip + r * 32) : 1;
            }
            val[r] = live ? __ldcs(sp + r * sstep) : 0.0;
        }
        __syncthreads();  // counters cleared (and the previous chunk's buffers drained)
        uint32_t rk[RP_IPT / 2];  // ranks: two 16-bit halves per word
#pragma unroll
        for (int r = 0; r < RP_IPT; ++r) {
            const bool live = r * 32 + lane < nlive;
            if (FIRST && live) {
                if (row[r] < 1) bad = min(bad, (unsigned long long)(base + r * 32));
                else if (row[r] > M) over = 1;
            }
            const bool valid = live && (unsigned)(col[r] - 1) < (unsigned)N;
            const unsigned d = key_digit(col[r], row[r], shift, A.rbits, dmask);
#if SA_PASS_V2
            const unsigned rr = rp_rank(&S.cnt[w][0], d, valid, lt);
#else
            // lanes with the same digit: one ballot per digit bit
            // (__match_any_sync runs on the slow ADU pipe)
            unsigned peers = __ballot_sync(FULL, valid);
#pragma unroll
            for (int i = 0; i < BITS; ++i) {
                const unsigned bb = __ballot_sync(FULL, (d >> i) & 1u);
                peers &= bb ^ (((d >> i) & 1u) - 1u);  // bit set: bb; clear: ~bb
            }
            // rank = the warp's running count of digit d (returned by the
            // group's first lane's shared atomic; one warp's shared atomics
            // complete in program order)
            const int leader = __ffs(peers) - 1;
            const unsigned sh = (d & 1u) * 16u;
            unsigned old = 0;
            if (lane == leader && valid) old = atomicAdd(&S.cnt[w][d >> 1], (unsigned)__popc(peers) << sh);
            const unsigned rr = ((__shfl_sync(FULL, old, leader & 31) >> sh) & 0xffffu) + __popc(peers & lt);
#endif
            if (r & 1) rk[r >> 1] |= rr << 16;
            else rk[r >> 1] = rr;
        }
        __syncthreads();
#if SA_PASS_V2
        uint32_t t0, t1, ex, ctot;
        rp_scan<BITS>(&S.cnt[0][0], S.red, t0, t1, ex, ctot);
        if ((tid & 3) == 0 && (tid >> 2) < npair) {
            // global position of chunk-local slot 0 of each digit: run - local start
            const int pp = tid >> 2;
            S.run[2 * pp] -= ex;
            if (2 * pp + 1 < ndig) S.run[2 * pp + 1] -= ex + t0;
        }
#else
        // (digit, warp) digit-major scan: thread t owns the digit pair (2t, 2t+1)
        uint32_t t0 = 0, t1 = 0;
        if (tid < npair) {
#pragma unroll 8
            for (int ww = 0; ww < RP_NW; ++ww) {
                const uint32_t c = S.cnt[ww][tid];
                S.cnt[ww][tid] = t0 | (t1 << 16);
                t0 += c & 0xffffu;
                t1 += c >> 16;
            }
        }
        uint32_t ctot;
        const uint32_t ex = block_excl_sum<RP_NT, uint32_t>(t0 + t1, S.red, ctot);
        if (tid < npair) {
            const uint32_t add = ex | ((ex + t0) << 16);  // chunk-local starts of digits 2t, 2t+1
#pragma unroll 8
            for (int ww = 0; ww < RP_NW; ++ww) S.cnt[ww][tid] += add;
            // global position of chunk-local slot 0 of each digit: run - local start
            S.run[2 * tid] -= ex;
            if (2 * tid + 1 < ndig) S.run[2 * tid + 1] -= ex + t0;
        }
#endif
        __syncthreads();
#pragma unroll
        for (int r = 0; r < RP_IPT; ++r) {  // records to their sorted slots
            if (r * 32 + lane < nlive && (unsigned)(col[r] - 1) < (unsigned)N) {
                const unsigned d = key_digit(col[r], row[r], shift, A.rbits, dmask);
                const unsigned pos = ((S.cnt[w][d >> 1] >> ((d & 1u) * 16u)) & 0xffffu) +
                                     ((rk[r >> 1] >> ((r & 1) * 16)) & 0xffffu);
                const unsigned long long vb = (unsigned long long)__double_as_longlong(val[r]);
                S.rec[pos] = make_uint4((uint32_t)row[r], (uint32_t)col[r], (uint32_t)vb, (uint32_t)(vb >> 32));
#if !SA_PASS_NOIDX
                S.oidx[pos] = S.run[d] + pos;
#endif
            }
        }
        __syncthreads();
        const unsigned long long pol = l2_evict_last();
#if SA_PASS_NOIDX
        for (int k = tid; k < (int)ctot; k += RP_NT) {  // (output index from the record's own digit)
            const uint4 v = S.rec[k];
            put_rec<LAST>(A, S.run[key_digit((int)v.y, (int)v.x, shift, A.rbits, dmask)] + (uint32_t)k, v, pol);
        }
#else
        for (int k = tid; k < (int)ctot; k += RP_NT) put_rec<LAST>(A, S.oidx[k], S.rec[k], pol);
#endif
    }
    pdl_trigger();
    if (FIRST) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            bad = min(bad, __shfl_xor_sync(FULL, bad, o));
            over |= __shfl_xor_sync(FULL, over, o);
        }
        if (lane == 0) {
            if (bad != ~0ull) atomicMin(&err->bad_i, bad);
            if (over) err->over_m = 1;
        }
    }
}

// ---------------------------------------------------------------------------
// k_rpass_tma: the same stable partition pass with the input staged by TMA.
// A chunk (RP_CHUNK triplets, the unit of the histograms and bases) is
// processed as two halves of RT_HALF; each half's rows, columns and values
// arrive by cp.async.bulk into one of two shared-memory buffers while the
// previous half is ranked, placed and written out, so the loads never stall
// the CTA (k_rpass holds a whole chunk in registers and waits for it).  The
// records are then placed in sorted order in the same buffer (every thread
// has its triplets in registers by then) and written out as in k_rpass.
// Needs 16-byte aligned input arrays (the host checks; k_rpass otherwise).
// ---------------------------------------------------------------------------
constexpr int RT_HALF = RP_CHUNK / 2;
constexpr int RT_IPT = RT_HALF / RP_NT;
struct PassTmaSmem {
    uint4 buf[2][RT_HALF];            // staged {ii[], jj[], s[]} of a half, then its sorted records
#if !SA_PASS_NOIDX
    uint32_t oidx[RT_HALF];           // output index of sorted slot k
#endif
    uint32_t cnt[RP_NW][RP_CS];       // per warp, digit pair (16-bit halves)
    uint32_t run[RP_MAXD];
    uint32_t red[RP_NW];
    unsigned long long mbar[2];
};

__device__ __forceinline__ unsigned rt_smem(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

// Stage half h (triplets [h0, h0 + nh)) into buffer `b` (thread 0).
template <bool PAIRS>
__device__ __forceinline__ void rt_issue(PassTmaSmem &S, int b, const RadixPassArgs &A, int64_t h0, int nh) {
    int32_t *si = reinterpret_cast<int32_t *>(&S.buf[b][0]);
    int32_t *sj = si + RT_HALF;
    double *ss = reinterpret_cast<double *>(sj + RT_HALF);
    const unsigned bi = (unsigned)nh * 4u, bs = A.s_stride ? (unsigned)nh * 8u : 0u;
    const unsigned bar = rt_smem(&S.mbar[b]);
    // the buffer was last written by the generic proxy (sorted records)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(2 * bi + bs) : "memory");
    if (PAIRS) {  // {row, col} pairs: one copy into the si | sj regions
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(rt_smem(si)), "l"(A.rc_in + h0), "r"(2 * bi), "r"(bar) : "memory");
    } else {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(rt_smem(si)), "l"(A.ii_in + h0), "r"(bi), "r"(bar) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(rt_smem(sj)), "l"(A.jj_in + h0), "r"(bi), "r"(bar) : "memory");
    }
    if (bs)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(rt_smem(ss)), "l"(A.s_in + h0), "r"(bs), "r"(bar) : "memory");
}

__device__ __forceinline__ void rt_wait(unsigned long long *bar, unsigned parity) {
    unsigned done = 0;
    while (!done) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(rt_smem(bar)), "r"(parity) : "memory");
    }
}

template <bool FIRST, bool LAST, int BITS>
__global__ void __launch_bounds__(RP_NT, 1) k_rpass_tma(RadixPassArgs A, ErrState *err) {
    extern __shared__ __align__(128) unsigned char rt_smem_raw[];
    PassTmaSmem &S = *reinterpret_cast<PassTmaSmem *>(rt_smem_raw);
    constexpr int ndig = 1 << BITS;
    constexpr unsigned dmask = (unsigned)ndig - 1u;
    constexpr int npair = (ndig + 1) >> 1;
    constexpr bool PAIRS = !FIRST && SA_PAIRS;  // input: {row, col} pairs
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const unsigned lt = lanemask_lt();
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(rt_smem(&S.mbar[0])) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(rt_smem(&S.mbar[1])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait();
    const int64_t Lp = FIRST ? A.L : (int64_t)*((volatile const unsigned *)&err->rvalid);
    const int64_t nchunk = (Lp + RP_CHUNK - 1) / RP_CHUNK;
    const int shift = A.shift;
    const int32_t M = A.M, N = A.N;
    const double sc = A.s_stride ? 0.0 : A.s_in[0];
    unsigned long long bad = ~0ull;
    unsigned over = 0;
    // this CTA's halves: chunks blockIdx.x + i * grid, two halves each
    const int64_t nmine = (nchunk > blockIdx.x) ? 2 * ((nchunk - 1 - blockIdx.x) / gridDim.x + 1) : 0;
    auto half_start = [&](int64_t k) -> int64_t {
        return ((int64_t)blockIdx.x + (k >> 1) * gridDim.x) * RP_CHUNK + (k & 1) * RT_HALF;
    };
    auto half_len = [&](int64_t k) -> int { return (int)max((int64_t)0, min((int64_t)RT_HALF, Lp - half_start(k))); };
    // TMA only for whole halves (16-byte multiples); a partial tail half is
    // loaded by the threads
    if (tid == 0 && nmine > 0 && half_len(0) == RT_HALF) rt_issue<PAIRS>(S, 0, A, half_start(0), RT_HALF);
    // the chunk's digit bases live in the registers of the scan's pair owners
    // (thread 4 p: digits 2 p, 2 p + 1), fetched one chunk ahead
    static_assert(RP_MAXD / 2 * 4 <= RP_NT && RP_MAXD % 2 == 0, "one digit pair per owner thread");
    const bool owner = (tid & 3) == 0 && (tid >> 2) < npair;
    const uint2 *offp = reinterpret_cast<const uint2 *>(A.off) + (tid >> 2);  // (+ chunk * RP_MAXD / 2)
    uint2 hbn = (owner && nmine > 0) ? offp[(int64_t)blockIdx.x * (RP_MAXD / 2)] : make_uint2(0u, 0u);
    uint32_t hb0 = 0, hb1 = 0;
    for (int64_t k = 0; k < nmine; ++k) {
        const int b = (int)(k & 1);
        const int64_t h0 = half_start(k);
        const int nh = half_len(k);
        const int64_t c = blockIdx.x + (k >> 1) * gridDim.x;
        {
            // (no barrier closes an iteration: the counters were last read
            // before the previous half's write-out barrier)
            static_assert(sizeof(S.cnt) % 16 == 0 && offsetof(PassTmaSmem, cnt) % 16 == 0, "vector clear");
            uint4 *c128 = reinterpret_cast<uint4 *>(&S.cnt[0][0]);
            for (int q = tid; q < (int)(sizeof(S.cnt) / 16); q += RP_NT) c128[q] = make_uint4(0u, 0u, 0u, 0u);
            if ((k & 1) == 0 && owner) {
                hb0 = hbn.x;
                hb1 = hbn.y;
                if (k + 2 < nmine) hbn = offp[(c + gridDim.x) * (RP_MAXD / 2)];
            }
        }
        int32_t *si = reinterpret_cast<int32_t *>(&S.buf[b][0]);
        int32_t *sj = si + RT_HALF;
        double *ss = reinterpret_cast<double *>(sj + RT_HALF);
        if (nh == RT_HALF) {
            rt_wait(&S.mbar[b], (unsigned)((k >> 1) & 1));
        } else {  // tail half: plain loads into the buffer
            for (int q = tid; q < nh; q += RP_NT) {
                if (PAIRS) {
                    reinterpret_cast<int2 *>(si)[q] = A.rc_in[h0 + q];
                } else {
                    si[q] = A.ii_in[h0 + q];
                    sj[q] = A.jj_in[h0 + q];
                }
                if (A.s_stride) ss[q] = A.s_in[h0 + q];
            }
            __syncthreads();
        }
        // warp w owns the half's w-th run of RT_IPT x 32 triplets, striped
        const int o0 = w * (RT_IPT * 32) + lane;
        int col[RT_IPT], row[RT_IPT];
        double val[RT_IPT];
#pragma unroll
        for (int r = 0; r < RT_IPT; ++r) {
            const int q = o0 + r * 32;
            const bool live = q < nh;
            if (PAIRS) {
                const int2 pr2 = live ? reinterpret_cast<const int2 *>(si)[q] : make_int2(1, 0);
                row[r] = pr2.x;
                col[r] = pr2.y;
            } else {
                col[r] = live ? sj[q] : 0;
                row[r] = live ? si[q] : 1;
            }
            val[r] = live ? (A.s_stride ? ss[q] : sc) : 0.0;
        }
        __syncthreads();  // counters cleared; the buffer is read (it now takes the sorted records)
        // every thread is past the previous half's write-out: its buffer
        // takes the next half while this one is ranked, placed and written
        if (tid == 0 && k + 1 < nmine && half_len(k + 1) == RT_HALF)
            rt_issue<PAIRS>(S, b ^ 1, A, half_start(k + 1), RT_HALF);
        uint32_t rk[(RT_IPT + 1) / 2];
#pragma unroll
        for (int r = 0; r < RT_IPT; ++r) {
            const bool live = o0 + r * 32 < nh;
            if (FIRST && live) {
                if (row[r] < 1) bad = min(bad, (unsigned long long)(h0 + o0 + r * 32));
                else if (row[r] > M) over = 1;
            }
            const bool valid = live && (unsigned)(col[r] - 1) < (unsigned)N;
            const unsigned d = key_digit(col[r], row[r], shift, A.rbits, dmask);
            const unsigned rr = rp_rank(&S.cnt[w][0], d, valid, lt);
            if (r & 1) rk[r >> 1] |= rr << 16;
            else rk[r >> 1] = rr;
        }
        __syncthreads();
        uint32_t t0, t1, ex, ctot;
        rp_scan<BITS>(&S.cnt[0][0], S.red, t0, t1, ex, ctot);
        if (owner) {
            // global position of the half-local slot 0 of each digit; the next
            // half of the chunk starts where this one ends
            const int pp = tid >> 2;
            S.run[2 * pp] = hb0 - ex;
            hb0 += t0;
            if (2 * pp + 1 < ndig) {
                S.run[2 * pp + 1] = hb1 - (ex + t0);
                hb1 += t1;
            }
        }
        __syncthreads();
        uint4 *rec = &S.buf[b][0];
#pragma unroll
        for (int r = 0; r < RT_IPT; ++r) {
            if (o0 + r * 32 < nh && (unsigned)(col[r] - 1) < (unsigned)N) {
                const unsigned d = key_digit(col[r], row[r], shift, A.rbits, dmask);
                const unsigned pos = ((S.cnt[w][d >> 1] >> ((d & 1u) * 16u)) & 0xffffu) +
                                     ((rk[r >> 1] >> ((r & 1) * 16)) & 0xffffu);
                const unsigned long long vb = (unsigned long long)__double_as_longlong(val[r]);
                rec[pos] = make_uint4((uint32_t)row[r], (uint32_t)col[r], (uint32_t)vb, (uint32_t)(vb >> 32));
#if !SA_PASS_NOIDX
                S.oidx[pos] = S.run[d] + pos;
#endif
            }
        }
        __syncthreads();
        const unsigned long long pol = l2_evict_last();
#if SA_PASS_NOIDX
        // output index from the record's own digit: consecutive slots share a
        // digit, so the base reads are near-broadcasts (a stored index per slot
        // cost a scattered store and a scattered base read in the loop above)
        for (int q = tid; q < (int)ctot; q += RP_NT) {
            const uint4 v = rec[q];
            put_rec<LAST>(A, S.run[key_digit((int)v.y, (int)v.x, shift, A.rbits, dmask)] + (uint32_t)q, v, pol);
        }
#else
        for (int q = tid; q < (int)ctot; q += RP_NT) put_rec<LAST>(A, S.oidx[q], rec[q], pol);
#endif
    }
    pdl_trigger();
    if (FIRST) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            bad = min(bad, __shfl_xor_sync(FULL, bad, o));
            over |= __shfl_xor_sync(FULL, over, o);
        }
        if (lane == 0) {
            if (bad != ~0ull) atomicMin(&err->bad_i, bad);
            if (over) err->over_m = 1;
        }
    }
}

// ---------------------------------------------------------------------------
// k_rbounds: start of every sub-bucket s = key >> z in the partitioned
// arrays (lower bound; the arrays are sorted by sub-bucket), and the list of
// sub-buckets longer than RF_CAP.  Column-block plan (z >= rbits): s =
// (col - 1) >> (z - rbits), the columns alone decide.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long sub_of(const int2 *__restrict__ rcp, uint32_t k, int z,
                                                     int rbits) {
    const int2 rc = __ldg(rcp + (size_t)k * RF_STRIDE);  // {row, col}
    if (z >= rbits) return (unsigned long long)((uint32_t)(rc.y - 1) >> (z - rbits));
    return tkey(rc.y, rc.x, rbits) >> z;
}

__device__ __forceinline__ uint32_t sub_lower_bound(const int2 *__restrict__ rec, uint32_t n, int z,
                                                    int rbits, uint32_t s) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (sub_of(rec, mid, z, rbits) < s) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void k_rbounds(const int2 *__restrict__ rec, int z, int rbits, int32_t nsub,
                          uint32_t *__restrict__ bnd, uint32_t *__restrict__ biglist, ErrState *err) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    pdl_wait();
    if (s <= nsub) {
        const uint32_t n = *((volatile const unsigned *)&err->rvalid);
        const uint32_t a = (s == 0) ? 0u : (s == nsub ? n : sub_lower_bound(rec, n, z, rbits, (uint32_t)s));
        bnd[s] = a;
        if (s < nsub) {
            const uint32_t e = (s + 1 == nsub) ? n : sub_lower_bound(rec, n, z, rbits, (uint32_t)s + 1);
            if (e - a > (uint32_t)RF_CAP) biglist[atomicAdd(&err->rbig_n, 1u)] = (uint32_t)s;
        }
    }
    pdl_trigger();
}

// ---------------------------------------------------------------------------
// k_rbig: oversize sub-buckets, one 1024-thread CTA each (grid-stride over
// the list).  Keys (key - the sub-bucket's first key) << 32 | k in scratch A, a
// stable LSD radix sort on the key bits (big_radix_pass, 8-bit digits, A <->
// B), values gathered in sorted order, each run of equal keys folded from
// +0.0 in k (= input) order, heads compacted.  Result: keys (high 32 bits)
// in one buffer, value bits in the other, bigu[s] = U | BIGFLAG if the keys
// ended in B.
// ---------------------------------------------------------------------------
constexpr int BIG_LONGRUN = 256;  // runs longer than this are folded by a warp
constexpr int BIG_NLONG = 512;    // listed long runs per sub-bucket (more: walked by their thread)
__global__ void __launch_bounds__(BIG_NT, 1) k_rbig(RadixFoldArgs F, ErrState *err) {
    __shared__ uint32_t s_cnt[BIG_NW][256];
    __shared__ uint32_t s_warp[BIG_NW];
    __shared__ unsigned long long s_prev;
    __shared__ uint2 s_long[BIG_NLONG];  // long runs of the sub-bucket: [first, end)
    __shared__ int s_nlong;
    const int tid = threadIdx.x;
    pdl_wait();
    const unsigned nbig = *((volatile const unsigned *)&err->rbig_n);
    if (call_failed(err)) {
        pdl_trigger();
        return;
    }
    const int passes = (F.z + 7) / 8;
    if (passes == 0) {
        // z == 0: a sub-bucket is one (row, col) key, i.e. one run of n > RF_CAP
        // repeats already in input order (the partition is stable).  Nothing to
        // sort: one warp per sub-bucket reads the values 32 at a time (the next
        // 32 in flight) and every lane folds them in order through shuffles --
        // the chain of n ordered adds is the floor; with a CTA per sub-bucket
        // one thread walked the run through global memory (1e7 triplets on
        // 1000 keys: 7.7 ms).
        const int lane = tid & 31;
        const unsigned wpg = gridDim.x * (BIG_NT / 32);
        for (unsigned q = blockIdx.x * (BIG_NT / 32) + (tid >> 5); q < nbig; q += wpg) {
            const uint32_t s = F.biglist[q];
            const uint32_t a = F.bnd[s], n = F.bnd[s + 1] - a;
            const double acc = warp_fold_run(reinterpret_cast<const unsigned long long *>(F.s + (size_t)a * RF_STRIDE), n,
                                             RF_STRIDE);
            if (lane == 0) {  // one result: local key 0 in A, its value in B
                F.scrA[a] = 0ull;
                F.scrB[a] = (unsigned long long)__double_as_longlong(acc);
                F.bigu[s] = 1u;
            }
        }
        pdl_trigger();
        return;
    }
    for (unsigned q = blockIdx.x; q < nbig; q += gridDim.x) {
        const uint32_t s = F.biglist[q];
        const uint32_t a = F.bnd[s], n = F.bnd[s + 1] - a;
        const unsigned long long K0 = (unsigned long long)s << F.z;
        const uint32_t c0 = (uint32_t)(K0 >> F.rbits);
        const uint32_t roff = (uint32_t)K0 & ((F.rbits >= 32) ? 0xffffffffu : ((1u << F.rbits) - 1u));
        unsigned long long *A = F.scrA + a;
        unsigned long long *B = F.scrB + a;
        for (uint32_t k = tid; k < n; k += BIG_NT) {
            const int2 rc = __ldg(F.rc + (size_t)(a + k) * RF_STRIDE);
            const uint32_t key = lkey(rc.y, rc.x, F.z, F.rbits, c0, roff);
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
            dst[k] = (unsigned long long)__double_as_longlong(__ldg(F.s + ((size_t)a + (uint32_t)src[k]) * RF_STRIDE));
        __syncthreads();
        if (tid == 0) s_nlong = 0;
        __syncthreads();
        {  // ordered fold of every run; the result lands at the run's head.  A
           // run longer than BIG_LONGRUN is only listed here (its end found by
           // binary search: the keys are sorted) and folded by a warp below --
           // one thread walking a heavy hitter's run through global memory
           // costs ~100 cycles per repeat, the warp ~12
            const uint32_t lo = (uint32_t)((uint64_t)tid * n / BIG_NT);
            const uint32_t hi = (uint32_t)((uint64_t)(tid + 1) * n / BIG_NT);
            uint32_t p = lo;
            while (p < hi) {
                const uint32_t key = (uint32_t)(src[p] >> 32);
                if (p > 0 && (uint32_t)(src[p - 1] >> 32) == key) {
                    ++p;
                    continue;
                }
                if (p + BIG_LONGRUN < n && (uint32_t)(src[p + BIG_LONGRUN] >> 32) == key) {
                    uint32_t a2 = p + BIG_LONGRUN + 1, b2 = n;  // first index in [a2, b2] of another key
                    while (a2 < b2) {
                        const uint32_t mid = (a2 + b2) >> 1;
                        if ((uint32_t)(src[mid] >> 32) == key) a2 = mid + 1;
                        else b2 = mid;
                    }
                    const int e = atomicAdd(&s_nlong, 1);
                    if (e < BIG_NLONG) {
                        s_long[e] = make_uint2(p, a2);
                        p = a2;
                        continue;
                    }
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
        {  // the listed long runs: one warp each, values 32 at a time (the next
           // 32 in flight), every lane folding them in order through shuffles
            const int lane = tid & 31;
            const int nl = min(s_nlong, BIG_NLONG);
            for (int e = tid >> 5; e < nl; e += BIG_NT / 32) {
                const uint32_t p0 = s_long[e].x, p1 = s_long[e].y;
                const double acc = warp_fold_run(dst + p0, (int64_t)p1 - p0);
                __syncwarp();
                if (lane == 0) dst[p0] = (unsigned long long)__double_as_longlong(acc);
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
#ifndef SA_FOLD_GBAL
#define SA_FOLD_GBAL 1
#endif
#ifndef SA_FOLD_CWARP
#define SA_FOLD_CWARP 1
#endif
#ifndef SA_FOLD_PF
#define SA_FOLD_PF 1
#endif
#ifndef SA_FOLD_XOR
#define SA_FOLD_XOR 1
#endif
#ifndef SA_FOLD_K32
#define SA_FOLD_K32 1
#endif
#ifndef SA_FOLD_LRANK
#define SA_FOLD_LRANK 1
#endif
#ifndef SA_RF_NT
#define SA_RF_NT 512
#endif
// 512 threads, two sub-buckets in flight per SM (8192 hash slots, 98 KB of
// shared memory); 256 threads fit three (4096 slots, 74 KB) but measured
// slower (cfg4 fold 8.5 -> 8.9 ms)
constexpr int RF_NT = SA_RF_NT;
constexpr int RF_MINB = RF_NT == 256 ? 3 : 2;
constexpr int RF_HS = RF_NT == 256 ? RF_CAP : 2 * RF_CAP;
constexpr int RF_HS_BITS = RF_NT == 256 ? 12 : 13;
static_assert((1 << RF_HS_BITS) == RF_HS, "hash table size");
constexpr int RF_BIGG = 128;  // groups of > 32 members per sub-bucket (<= RF_CAP / 33)

#ifdef SA_RTRACE
// per-sub-bucket phase stamps of k_rfold (tools/rfold_trace.py): SM cycles
__device__ long long g_rtrace[1 << 15][10];
#define RTRACE(k) \
    if (threadIdx.x == 0 && blockIdx.x < (1 << 15)) g_rtrace[blockIdx.x][k] = clock64();
#else
#define RTRACE(k)
#endif

struct FoldSmem {
    // key, cnt2 and glist are dead by the output phase: together (>= 8 RF_CAP
    // bytes) they take the staged values (or the fallback's sort items)
    uint32_t key[RF_HS];          // hash keys (key + 1; 0 = empty); then the column lists' keys
                                  // (ckey)
    uint32_t cnt2[RF_HS / 2];     // per slot (16-bit halves): members, then member cursor
    uint16_t glist[RF_CAP];       // slot of group g
    uint32_t gkey[RF_CAP];        // key + 1 of group g
    uint16_t gid[RF_CAP];         // slot of record k; then: group of output entry p
    uint16_t memb[RF_CAP];        // member records, grouped
    uint16_t gstart[RF_CAP + 1];  // first member of group g
    uint32_t colst[RF_WMAX + 1];  // distinct groups per column -> column start
    uint32_t colcur[RF_WMAX];
    uint16_t bigg[RF_BIGG];       // groups of more than 32 members
    uint16_t cgrp[RF_CAP];        // group of column-list entry q
    uint32_t red[RF_NT / 32];
    int U, nbigg, sortall, ndef;
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

__device__ __forceinline__ void rf_cp_async8(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src) : "memory");
}

// Batcher's odd-even merge network on 8 keys (19 compare-exchanges), ascending.
__device__ __forceinline__ void rf_cx(uint32_t &a, uint32_t &b) {
    const uint32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}
__device__ __forceinline__ void rf_net8(uint32_t (&m)[8]) {
    rf_cx(m[0], m[1]); rf_cx(m[2], m[3]); rf_cx(m[4], m[5]); rf_cx(m[6], m[7]);
    rf_cx(m[0], m[2]); rf_cx(m[1], m[3]); rf_cx(m[4], m[6]); rf_cx(m[5], m[7]);
    rf_cx(m[1], m[2]); rf_cx(m[5], m[6]);
    rf_cx(m[0], m[4]); rf_cx(m[1], m[5]); rf_cx(m[2], m[6]); rf_cx(m[3], m[7]);
    rf_cx(m[2], m[4]); rf_cx(m[3], m[5]);
    rf_cx(m[1], m[2]); rf_cx(m[3], m[4]); rf_cx(m[5], m[6]);
}

// 16 keys: two sorted halves (rf_net8), then merged -- compare k with 15 - k
// (every key of the low half is then <= every key of the high half and both
// halves are bitonic) and a bitonic clean-up of each half (70 compare-exchanges).
__device__ __forceinline__ void rf_net16(uint32_t (&m)[16]) {
    uint32_t(&lo)[8] = *reinterpret_cast<uint32_t(*)[8]>(&m[0]);
    uint32_t(&hi)[8] = *reinterpret_cast<uint32_t(*)[8]>(&m[8]);
    rf_net8(lo);
    rf_net8(hi);
#pragma unroll
    for (int k = 0; k < 8; ++k) rf_cx(m[k], m[15 - k]);
#pragma unroll
    for (int d = 4; d >= 1; d >>= 1)
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if ((k & d) == 0) rf_cx(m[k], m[k + d]);
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

__global__ void __launch_bounds__(RF_NT, RF_MINB) k_rfold(RadixFoldArgs F, ErrState *err) {
    extern __shared__ __align__(16) unsigned char rf_smem[];
    FoldSmem &S = *reinterpret_cast<FoldSmem *>(rf_smem);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = lanemask_lt();
    pdl_wait();
    // sub-bucket = block index (blocks are dispatched in index order, so the
    // look-back below only waits on started predecessors, as in the tile fold);
    // the error flags and the bounds are read concurrently
    RTRACE(0)
    const int64_t s = blockIdx.x;
    const bool failed = call_failed(err);
    const uint32_t a = F.bnd[s], n = F.bnd[s + 1] - a;
    if (failed) {
        pdl_trigger();
        return;
    }
    // sub-bucket keys [K0, K0 + 2^z): column-block plan (z >= rbits) -- the
    // columns c0 .. c0 + 2^(z - rbits) - 1, whole; row-split plan (z < rbits)
    // -- rows roff .. roff + 2^z - 1 of column c0 (it starts the column when
    // roff == 0).  A local key kl = key - K0 belongs to local column
    // (roff + kl) >> rbits and row (roff + kl) & rmask.
    const unsigned long long K0 = (unsigned long long)s << F.z;
    const int64_t c0 = (int64_t)(K0 >> F.rbits);
    const uint32_t rmask = (F.rbits >= 32) ? 0xffffffffu : ((1u << F.rbits) - 1u);
    const uint32_t roff = (uint32_t)K0 & rmask;
    // local columns (group bookkeeping) and the columns whose jc this
    // sub-bucket writes (a row-split sub-bucket only if it starts its column)
    const int ncol = F.z >= F.rbits ? (int)min((int64_t)1 << (F.z - F.rbits), (int64_t)F.N - c0) : 1;
    const int njc = (F.z >= F.rbits || roff == 0) ? ncol : 0;
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
        for (int c = tid; c < njc; c += RF_NT) {  // first result of column c
            uint32_t lo = 0, hi = U;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if ((roff + (uint32_t)(RK[mid] >> 32)) >> F.rbits < (uint32_t)c) lo = mid + 1;
                else hi = mid;
            }
            F.jc[c0 + c] = (int32_t)(off + lo);
        }
        for (uint32_t p = tid; p < U; p += RF_NT) {
            if (off + p < F.cap) {
                F.ir[off + p] = (int32_t)((roff + (uint32_t)(RK[p] >> 32)) & rmask);
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
    {  // the sub-bucket's values into L2 while the groups are built (staged later)
        // (16-byte records: keys and values share their lines)
        const char *vb = SA_AOS ? reinterpret_cast<const char *>(F.rc + (size_t)a * RF_STRIDE)
                                : reinterpret_cast<const char *>(F.s + a);
        const uint32_t nb = n * 8u * RF_STRIDE;
        for (uint32_t o = (uint32_t)tid * 128u; o < nb; o += RF_NT * 128u)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(vb + o));
    }
    // table of 2^hbits >= 2 n slots (64 .. RF_HS), cleared with 16-byte stores
    const int hbits = n ? min(RF_HS_BITS, max(6, 32 - __clz((int)(2u * n) - 1))) : 6;
    const int hs = 1 << hbits;
    static_assert(offsetof(FoldSmem, key) % 16 == 0 && offsetof(FoldSmem, cnt2) % 16 == 0, "vector clear");
    {
        uint4 *k4 = reinterpret_cast<uint4 *>(S.key), *c4 = reinterpret_cast<uint4 *>(S.cnt2);
        for (int k = tid; k < hs / 4; k += RF_NT) k4[k] = make_uint4(0u, 0u, 0u, 0u);
        for (int k = tid; k < hs / 8; k += RF_NT) c4[k] = make_uint4(0u, 0u, 0u, 0u);
    }
    for (int c = tid; c <= ncol; c += RF_NT) S.colst[c] = 0;
    if (tid == 0) {
        S.U = 0;
        S.nbigg = 0;
        S.sortall = 0;
        S.ndef = 0;
    }
    constexpr int RIPT = RF_CAP / RF_NT;
#if SA_FOLD_K32
    const int ksh = min(F.rbits, 31);  // (rbits == 32 only with one column block: the shifted term is 0)
#endif
    uint32_t kk[RIPT];  // local key + 1 of records tid + u * RF_NT
#pragma unroll
    for (int u = 0; u < RIPT; ++u) {
        const uint32_t k = tid + u * RF_NT;
        kk[u] = 0u;
        if (k < n) {
            const int2 rc = __ldg(F.rc + (size_t)(a + k) * RF_STRIDE);  // {row, col}
#if SA_FOLD_K32
            // local key + 1 in 32 bits: ((col - 1 - c0) << rbits) + row - roff
            // (column-block plan: roff = 0; row-split plan: col - 1 == c0)
            kk[u] = (((uint32_t)(rc.y - 1) - (uint32_t)c0) << ksh) + (uint32_t)rc.x - roff;
#else
            kk[u] = (uint32_t)(tkey(rc.y, rc.x, F.rbits) - K0) + 1u;
#endif
        }
    }
#if SA_FOLD_PF
    {  // the keys of the sub-bucket that takes this CTA's place when it retires: into L2
        const int64_t sp = s + F.nres;
        if (sp < F.nsub) {
            const uint32_t a2 = F.bnd[sp], n2 = min(F.bnd[sp + 1] - a2, (uint32_t)RF_CAP);
            const char *kb = reinterpret_cast<const char *>(F.rc + (size_t)a2 * RF_STRIDE);
            for (uint32_t o = (uint32_t)tid * 128u; o < n2 * 8u * RF_STRIDE; o += RF_NT * 128u)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(kb + o));
        }
    }
#endif
    __syncthreads();
    RTRACE(1)
#pragma unroll
    for (int u = 0; u < RIPT; ++u) {
        const uint32_t k = tid + u * RF_NT;
        bool fresh = false;
        unsigned h = 0;
        if (k < n) {
            h = rf_insert(S.key, hbits, kk[u], fresh);
            S.gid[k] = (uint16_t)h;
            atomicAdd(&S.cnt2[h >> 1], 1u << ((h & 1u) * 16u));
        }
        if (fresh) {
            const int g = atomicAdd(&S.U, 1);
            S.glist[g] = (uint16_t)h;
            S.gkey[g] = kk[u];
            atomicAdd(&S.colst[(roff + kk[u] - 1u) >> F.rbits], 1u);
        }
    }
    __syncthreads();
    RTRACE(2)
    const int U = S.U;
    if (tid == 0) ((volatile unsigned long long *)lbs)[0] = ep_pack(F.tag, s == 0 ? 2 : 1, (unsigned)U);

    // ---- 2. member starts, column starts ------------------------------------
#if SA_FOLD_CWARP
    if (warp == RF_NT / 32 - 1) {  // column starts: one warp's scan (no block-wide barriers)
        constexpr int CPL = RF_WMAX / 32;
        uint32_t v[CPL], sum = 0;
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            const int c = lane * CPL + i;
            v[i] = (c < ncol) ? S.colst[c] : 0u;
            sum += v[i];
        }
        uint32_t x = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x += y;
        }
        uint32_t ex = x - sum;
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            const int c = lane * CPL + i;
            if (c < ncol) {
                S.colst[c] = ex;
                S.colcur[c] = ex;
            }
            ex += v[i];
        }
        if (lane == 31) S.colst[ncol] = ex;  // = U
    }
#endif
    {  // exclusive scan of the member counts in group order -> gstart; the slot's
       // count becomes its member cursor
#if SA_FOLD_GBAL
        const int G = (U + RF_NT - 1) / RF_NT;  // groups per thread (<= RIPT)
#else
        const int G = RIPT;
#endif
        const int g0 = tid * G;
        uint32_t loc[RIPT], sum = 0;
#pragma unroll
        for (int u = 0; u < RIPT; ++u) {
            loc[u] = 0u;
            if (u < G && g0 + u < U) {
                const unsigned h = S.glist[g0 + u];
                loc[u] = (S.cnt2[h >> 1] >> ((h & 1u) * 16u)) & 0xffffu;
            }
            sum += loc[u];
        }
        uint32_t tot;
        uint32_t pre = block_excl_sum<RF_NT, uint32_t>(sum, S.red, tot);
#pragma unroll
        for (int u = 0; u < RIPT; ++u) {
            const int g = g0 + u;
            if (u < G && g < U) {
                S.gstart[g] = (uint16_t)pre;
                const unsigned h = S.glist[g], sh = (h & 1u) * 16u;
#if SA_FOLD_XOR
                atomicXor(&S.cnt2[h >> 1], (loc[u] ^ pre) << sh);  // count -> first member
#else
                atomicAnd(&S.cnt2[h >> 1], ~(0xffffu << sh));
                atomicOr(&S.cnt2[h >> 1], pre << sh);
#endif
                if (loc[u] > 32u) {
                    const int q = atomicAdd(&S.nbigg, 1);
                    if (q < RF_BIGG) S.bigg[q] = (uint16_t)g;
                }
            }
            pre += loc[u];
        }
    }
#if !SA_FOLD_CWARP
    smem_excl_scan<RF_NT, 1, uint32_t>(S.colst, ncol, S.red);
    for (int c = tid; c < ncol; c += RF_NT) S.colcur[c] = S.colst[c];
    if (tid == 0) S.colst[ncol] = (uint32_t)U;
#endif
    if (tid == 0) S.gstart[U] = (uint16_t)n;
    __syncthreads();
    RTRACE(3)
    // ---- 3. members (unordered), groups per column ---------------------------------
    uint32_t *ckey = S.key;  // the hash table is dead: column lists' keys
#pragma unroll
    for (int u = 0; u < RIPT; ++u) {
        const uint32_t k = tid + u * RF_NT;
        if (k < n) {
            const unsigned h = S.gid[k], sh = (h & 1u) * 16u;
            S.memb[(atomicAdd(&S.cnt2[h >> 1], 1u << sh) >> sh) & 0xffffu] = (uint16_t)k;
        }
    }
    for (int g = tid; g < U; g += RF_NT) {
        const uint32_t kx = S.gkey[g];
        const uint32_t q = atomicAdd(&S.colcur[(roff + kx - 1u) >> F.rbits], 1u);
        ckey[q] = kx;  // column lists of the groups' keys (unordered)
        S.cgrp[q] = (uint16_t)g;
    }
    __syncthreads();
    RTRACE(4)
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
    // (walked in list order: the lanes of a warp share a few columns, so the
    // list reads below are near-broadcasts; in group order every lane walked
    // its own column's list)
    uint32_t opos[RIPT];  // output position | group << 16
    // output entries whose group has more than 8 members, listed over the
    // dead member cursors (folded by the last threads of the CTA, below)
    uint16_t *dl = reinterpret_cast<uint16_t *>(S.cnt2);
#pragma unroll
    for (int u = 0; u < RIPT; ++u) {
        const int t = tid + u * RF_NT;
        opos[u] = 0;
        if (t < U) {
#if SA_FOLD_LRANK
            const uint32_t kx = ckey[t];
#else
            const uint32_t kx = S.gkey[t];
#endif
            const uint32_t cl = (roff + kx - 1u) >> F.rbits;
            const int st = S.colst[cl], en = S.colst[cl + 1];
            if (en - st > 64) {
                S.sortall = 1;
            } else {
                int r = st;
                for (int q = st; q < en; ++q) r += ckey[q] < kx;
#if SA_FOLD_LRANK
                const uint32_t g = S.cgrp[t];
                opos[u] = (uint32_t)r | (g << 16);
                if (S.gstart[g + 1] - S.gstart[g] > 8) dl[atomicAdd(&S.ndef, 1)] = (uint16_t)r;
#else
                opos[u] = (uint32_t)r | ((uint32_t)t << 16);
#endif
            }
        }
    }
    __syncthreads();
    RTRACE(5)
    const bool sortall = S.sortall != 0;
    // the sub-bucket's values into shared memory (the dead hash table, member
    // counts and group slots: the ranking above was the last reader of ckey),
    // in flight while the offset is looked back; the fallback sort below
    // uses the same space first
    static_assert(sizeof(uint32_t) * (RF_HS + RF_HS / 2) + sizeof(uint16_t) * RF_CAP >= 8 * RF_CAP,
                  "staged values");
    double *Vs = reinterpret_cast<double *>(&S.key[0]);
    if (!sortall) {
#pragma unroll
        for (int u = 0; u < RIPT; ++u) {
            if (tid + u * RF_NT < U) S.gid[opos[u] & 0xffffu] = (uint16_t)(opos[u] >> 16);  // gid := group of output entry
        }
    } else {  // CTA bitonic sort of all groups by key (a column with > 64 distinct rows)
        unsigned long long *items = reinterpret_cast<unsigned long long *>(S.key);
        int np2 = 1;
        while (np2 < U) np2 <<= 1;
        for (int g = tid; g < np2; g += RF_NT)
            items[g] = (g < U) ? (((unsigned long long)S.gkey[g] << 16) | (unsigned)g) : ~0ull;
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
        if (tid == 0) S.ndef = 0;  // (the ranking above listed some entries before it gave up)
        __syncthreads();
        for (int p = tid; p < U; p += RF_NT) {
            const int g = S.gid[p];
            if (S.gstart[g + 1] - S.gstart[g] > 8) dl[atomicAdd(&S.ndef, 1)] = (uint16_t)p;
        }
    }
    {  // (after the sort, if any: its items were last read before the barrier above)
        const double *sg = F.s + (size_t)a * RF_STRIDE;
        for (uint32_t k = tid; k < n; k += RF_NT) rf_cp_async8(&Vs[k], sg + (size_t)k * RF_STRIDE);
        asm volatile("cp.async.commit_group;" ::: "memory");
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
    RTRACE(6)
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    RTRACE(7)
    const long long off = S.off;
    const double *__restrict__ sv = Vs;
    // groups of more than 8 members (Poisson(5) repeats: 7 % of the groups)
    // were listed by the ranking: folded one per thread, taken from the last
    // thread down -- the warps with the fewest entries of the loop below -- so
    // the 16-key network and the general loop run in a warp or two instead
    // of in every warp for a few lanes each, and beside the small groups
    // instead of after them
    {
        const int ndef = S.ndef;
        for (int t = RF_NT - 1 - tid; t < ndef; t += RF_NT) {
            const int p = dl[t];
            const int g = S.gid[p];
            const int st = S.gstart[g], en = S.gstart[g + 1];
            const int nm = en - st;
            double acc = 0.0;
            if (nm <= 16) {
                uint32_t m[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) m[q] = (q < nm) ? (uint32_t)S.memb[st + q] : 0xffffu;
                rf_net16(m);
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    if (q < nm) acc = fold_add(acc, sv[m[q]]);
            } else {
                if (nm <= 32) rf_isort16(S.memb + st, nm);
                for (int q = st; q < en; ++q) acc = fold_add(acc, sv[S.memb[q]]);
            }
            if (off + p < F.cap) {
                F.ir[off + p] = (int32_t)((roff + S.gkey[g] - 1u) & rmask);
                F.pr[off + p] = acc;
            } else {
                over = true;
            }
        }
    }
    for (int p = tid; p < U; p += RF_NT) {
        const int g = S.gid[p];
        const int st = S.gstart[g], en = S.gstart[g + 1];
        const int nm = en - st;
        if (nm <= 8) {
            // member indices sorted by a register network, then every value
            // load in flight at once before the ordered chain of adds
            uint32_t m[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) m[q] = (q < nm) ? (uint32_t)S.memb[st + q] : 0xffffu;
            rf_net8(m);
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = (q < nm) ? sv[m[q]] : 0.0;
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q < nm) acc = fold_add(acc, v[q]);
            if (off + p < F.cap) {
                F.ir[off + p] = (int32_t)((roff + S.gkey[g] - 1u) & rmask);
                F.pr[off + p] = acc;
            } else {
                over = true;
            }
        }
    }
    for (int c = tid; c < njc; c += RF_NT) F.jc[c0 + c] = (int32_t)(off + S.colst[c]);
    if (s == F.nsub - 1 && tid == 0) {
        F.jc[F.N] = (int32_t)(off + U);
        err->nnz = off + U;
        if (off + U > F.cap) atomicExch(&err->cap_exceeded, 1u);
    }
    if (over) atomicExch(&err->cap_exceeded, 1u);
    RTRACE(9)
    pdl_trigger();
}

#ifdef SA_RTRACE
}  // namespace sa
extern "C" int sa_debug_rtrace(void *host, int n) {
    return (int)cudaMemcpyFromSymbol(host, sa::g_rtrace, (size_t)n * 80);
}
namespace sa {
#endif

// ---- launchers -----------------------------------------------------------------
// Chunks per upsweep block: about RP_BLK / 2, sized so that the blocks fill
// whole waves of the two resident CTAs per SM (cfg4, 40691 chunks: blocks of
// 64 made 2.15 waves -- 0.46 + 0.65 ms; 32: 0.42 + 0.63 ms); fewer for small
// inputs so that every SM gets about four blocks.
int rup_cpb(int64_t nchunk, int num_sms) {
    const int64_t slots = 2 * (int64_t)num_sms, tgt = RP_BLK / 2;
    if (nchunk >= 2 * tgt * slots) {
        const int64_t waves = (nchunk + tgt * slots / 2) / (tgt * slots);
        return (int)((nchunk + waves * slots - 1) / (waves * slots));
    }
    return (int)std::max<int64_t>(1, std::min<int64_t>(tgt, nchunk / (4 * (int64_t)num_sms)));
}

cudaError_t launch_rup(Launch &lc, bool first, const int32_t *ii, const int32_t *jj, const int2 *rc, int64_t L,
                       int32_t N,
                       int shift, int bits, int rbits, uint16_t *cnt, uint32_t *bsum, uint32_t *off,
                       ErrState *err) {
    // grid sized for L (an upper bound of the valid count the later passes read)
    const int64_t nchunk = (L + RP_CHUNK - 1) / RP_CHUNK;
    const int cpb = rup_cpb(nchunk, lc.num_sms);
    const int nblk = (int)std::max<int64_t>(1, (nchunk + cpb - 1) / cpb);
    const bool rowkey = shift < rbits;
    auto kern = first ? (rowkey ? k_rup<true, true> : k_rup<true, false>)
                      : (rowkey ? k_rup<false, true> : k_rup<false, false>);
    cudaError_t e = launch_pdl(kern, dim3((unsigned)nblk), dim3(RU_NT), 0, lc.stream, ii, jj, rc, L, N, shift, bits,
                               rbits, cpb, cnt, bsum, err);
    lc.launches++;
    if (e != cudaSuccess) return e;
    // (the digit totals live behind the block sums: bsum has room for nblk + 1 rows)
    uint32_t *tot = bsum + (int64_t)nblk * RP_MAXD;
    e = launch_pdl(k_rscan, dim3((unsigned)((RP_MAXD + 7) / 8)), dim3(256), 0, lc.stream, bsum, tot, nblk, bits);
    lc.launches++;
    if (e != cudaSuccess) return e;
    e = launch_pdl(k_roff, dim3((unsigned)nblk), dim3(RP_MAXD), 0, lc.stream, (const uint16_t *)cnt,
                   (const uint32_t *)bsum, (const uint32_t *)tot, bits, off, err, L, first ? 1 : 0, cpb);
    lc.launches++;
    return e;
}

template <bool FIRST, bool LAST, int BITS>
static cudaError_t launch_rpass_t(Launch &lc, const RadixPassArgs &A, int nseg, ErrState *err) {
    auto al16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    // TMA-staged input (cfg4: pass 1 8.3 -> 7.0 ms, pass 2 7.0 -> 6.1 ms)
    const bool tma = lc.rpass_tma != 0;
    const bool in16 = (!FIRST && SA_PAIRS) ? al16(A.rc_in) : (al16(A.ii_in) && al16(A.jj_in));
    if (tma && in16 && (A.s_stride == 0 || al16(A.s_in))) {
        const int smem = (int)sizeof(PassTmaSmem);
        cudaError_t e = ensure_smem_attr((const void *)k_rpass_tma<FIRST, LAST, BITS>, smem);
        if (e != cudaSuccess) return e;
        // grid: the first pass runs best on several waves of short-lived CTAs
        // (cfg4, 40691 chunks of 12288: 5.54 ms at one CTA per SM; 4.52 / 4.44 /
        // 4.38 / 4.33 / 4.31 / 4.28 / 4.37 ms at 2 / 3 / 4 / 6 / 8 / 12 / 16 chunks per
        // CTA -- 12 and 16 differ by the last, partly filled wave, so large
        // inputs get whole waves of about SA_RP_FIRST_CPC chunks per CTA), the
        // later ones with one CTA per SM (4.07 ms; 2 chunks per CTA: 4.21 ms)
        // -- measured, tools/abn.sh
#ifndef SA_RP_FIRST_CPC
#define SA_RP_FIRST_CPC 12
#endif
#ifndef SA_RP_LATER_CPC
#define SA_RP_LATER_CPC 0
#endif
        const int64_t nch = (A.L + RP_CHUNK - 1) / RP_CHUNK;
        int64_t grid = lc.num_sms;
        if (FIRST && SA_RP_FIRST_CPC) {
            const int64_t per_wave = (int64_t)SA_RP_FIRST_CPC * lc.num_sms;
            if (nch >= 2 * per_wave) grid = (nch + per_wave / 2) / per_wave * lc.num_sms;  // whole waves
            else grid = std::max<int64_t>(lc.num_sms, (nch + 2) / 3);                      // 3 chunks per CTA
        } else if (!FIRST && SA_RP_LATER_CPC) {
            constexpr int64_t lc_cpc = SA_RP_LATER_CPC ? SA_RP_LATER_CPC : 1;
            grid = std::max<int64_t>(lc.num_sms, (nch + lc_cpc - 1) / lc_cpc);
        }
        return launch_pdl(k_rpass_tma<FIRST, LAST, BITS>, dim3((unsigned)grid), dim3(RP_NT), smem, lc.stream,
                          A, err);
    }
    const int smem = (int)sizeof(PassSmem);
    cudaError_t e = ensure_smem_attr((const void *)k_rpass<FIRST, LAST, BITS>, smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(k_rpass<FIRST, LAST, BITS>, dim3((unsigned)nseg), dim3(RP_NT), smem, lc.stream, A, err);
    // (nseg = the number of resident partition CTAs; they walk the chunks with stride nseg)
}

template <bool FIRST, bool LAST>
static cudaError_t launch_rpass_b(Launch &lc, const RadixPassArgs &A, int nseg, ErrState *err) {
    switch (A.bits) {  // the digit width is a compile-time constant of the kernel
        case 0: return launch_rpass_t<FIRST, LAST, 0>(lc, A, nseg, err);
        case 1: return launch_rpass_t<FIRST, LAST, 1>(lc, A, nseg, err);
        case 2: return launch_rpass_t<FIRST, LAST, 2>(lc, A, nseg, err);
        case 3: return launch_rpass_t<FIRST, LAST, 3>(lc, A, nseg, err);
        case 4: return launch_rpass_t<FIRST, LAST, 4>(lc, A, nseg, err);
        case 5: return launch_rpass_t<FIRST, LAST, 5>(lc, A, nseg, err);
        case 6: return launch_rpass_t<FIRST, LAST, 6>(lc, A, nseg, err);
        case 7: return launch_rpass_t<FIRST, LAST, 7>(lc, A, nseg, err);
        case 8: return launch_rpass_t<FIRST, LAST, 8>(lc, A, nseg, err);
        case 9: return launch_rpass_t<FIRST, LAST, 9>(lc, A, nseg, err);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_rpass(Launch &lc, const RadixPassArgs &A, bool first, bool last, int nseg, ErrState *err) {
    cudaError_t e = first ? (last ? launch_rpass_b<true, true>(lc, A, nseg, err)
                                  : launch_rpass_b<true, false>(lc, A, nseg, err))
                          : (last ? launch_rpass_b<false, true>(lc, A, nseg, err)
                                  : launch_rpass_b<false, false>(lc, A, nseg, err));
    lc.launches++;
    return e;
}

cudaError_t launch_rbounds(Launch &lc, const int2 *rec, int z, int rbits, int32_t nsub, uint32_t *bnd,
                           uint32_t *biglist, ErrState *err) {
    const int64_t n = (int64_t)nsub + 1;
    cudaError_t e = launch_pdl(k_rbounds, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, lc.stream,
                               rec, z, rbits, nsub, bnd, biglist, err);
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
    RadixFoldArgs G = F;
    G.nres = lc.num_sms * RF_MINB;  // CTAs in flight
    e = launch_pdl(k_rfold, dim3((unsigned)F.nsub), dim3(RF_NT), smem, lc.stream, G, err);
    lc.launches++;
    return e;
}

}  // namespace sa
