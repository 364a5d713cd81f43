// sa_capi.cu -- the C ABI (include/sparse_assembly.h): contexts, workspace,
// launch sequencing and error mapping.  No torch types cross this boundary.

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "../../include/sparse_assembly.h"
#include "sa_internal.cuh"

using namespace sa;

struct sa_ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    std::string last_error;
    int launches = 0;

    // device workspace (grown on demand, reused across calls)
    uint32_t *cur = nullptr;              size_t cur_cap = 0;     // N (counts, then cursors)
    uint32_t *sstart = nullptr;           size_t st_cap = 0;      // N+1 small-space starts
    uint2 *perm = nullptr;                size_t perm_cap = 0;    // L + placeholders (+2): {row, position} by column
    int4 *rec = nullptr;                  size_t rec_cap = 0;     // big-column scratch (16 B per slot)
    int2 *tile_info = nullptr;            size_t ti_cap = 0;      // ntiles+1
    uint8_t *tile_big = nullptr;          size_t tb_cap = 0;      // ntiles
    unsigned long long *tile_state = nullptr; size_t ts_cap = 0;  // ntiles
    int2 *tile_cnt = nullptr;             size_t tc_cap = 0;      // staged fold: {U, small U} per tile
    unsigned long long *scan_state = nullptr; size_t ss_cap = 0;  // scan CTAs
    BigCol *big_list = nullptr;           size_t bl_cap = 0;      // L/(BIGCOL+1)+1
    uint32_t *bigk = nullptr;             size_t bk_cap = 0;      // N
    unsigned long long *pr_state = nullptr; size_t prs_cap = 0;  // prune look-back words
    long long *pr_nnz = nullptr;          // prune: device nnz of the result
    int32_t *pt_cnt = nullptr;            size_t ptc_cap = 0;    // partition: tile x rank counts
    int64_t *pt_off = nullptr;            size_t pto_cap = 0;    // partition: tile x rank offsets
    int64_t *pt_counts = nullptr;         // partition: per-rank counts and bases (16)
    // radix path (sa_radix.cu): partition buffers X / Y (one 16-byte-per-triplet
    // block each: the arrays ii | jj | s of the passes before the last, the
    // last pass's {row, col} pairs | s), histograms, look-back words
    uint4 *rx = nullptr; int32_t *rx_i = nullptr, *rx_j = nullptr; double *rx_s = nullptr;  size_t rx_cap = 0;
    uint4 *ry = nullptr; int32_t *ry_i = nullptr, *ry_j = nullptr; double *ry_s = nullptr;  size_t ry_cap = 0;
    uint16_t *rcnt = nullptr;             size_t rcnt_cap = 0;         // nchunk x RP_MAXD chunk histograms
    uint32_t *roff = nullptr;             size_t roff_cap = 0;         // nchunk x RP_MAXD chunk bases
    uint32_t *rbsum = nullptr;            size_t rbsum_cap = 0;        // (nblk + 1) x RP_MAXD: block bases, digit totals
    unsigned long long *rlbf = nullptr;   size_t rlbf_cap = 0;         // nsub x LB_STRIDE
    uint32_t *rbnd = nullptr;             size_t rbnd_cap = 0;         // nsub + 1
    uint32_t *rbig = nullptr;             size_t rbig_cap = 0;         // nsub (oversize list)
    uint32_t *rbigu = nullptr;            size_t rbigu_cap = 0;        // nsub
    unsigned rp_epoch = 0;                                             // look-back tag epoch
    ErrState *err = nullptr;              // device
    ErrState *err_host = nullptr;         // pinned mirror
    // host protocol: the dimension / validation pass runs on up_stream over
    // each uploaded chunk while the next one is copied (sa_host_upload), its
    // outcome in err_up; up_done marks its end
    cudaStream_t up_stream = nullptr;
    ErrState *err_up = nullptr;
    ErrState *err_up_host = nullptr;
    cudaEvent_t up_done = nullptr;
    static constexpr int MAXUP = 64;
    cudaEvent_t up_ev[MAXUP] = {};

    // buffers of the host-pointer entry point
    int32_t *h_ii = nullptr;                   size_t hii_cap = 0;
    int32_t *h_jj = nullptr;                   size_t hjj_cap = 0;
    double *h_s = nullptr;                     size_t hs_cap = 0;
    int32_t *o_jc = nullptr;                   size_t ojc_cap = 0;
    int32_t *o_ir = nullptr;                   size_t oir_cap = 0;
    double *o_pr = nullptr;                    size_t opr_cap = 0;
    // optional per-kernel event timing
    static constexpr int MAXEV = 16;
    int timing = 0;
    int nev = 0;
    cudaEvent_t ev[MAXEV + 1] = {};
    const char *ev_name[MAXEV] = {};

    // options (sa_set_option); -1 = automatic
    int opt_fold_staged = -1;
    int opt_scatter_staged = -1;
    int opt_path = -1;
    int opt_rpass_tma = -1;
    std::map<std::tuple<const void *, int64_t, int32_t, int32_t>, bool> path_cache;  // choose_radix

    int64_t host_L = -1;
    int host_radix = -1;  // path choice made at sa_host_upload from the host columns
    int64_t host_stride = 1;
    int32_t host_N = 0;
    int64_t host_nnz = -1;
};

namespace {

int fail(sa_ctx *ctx, int code, const std::string &msg) {
    if (ctx) ctx->last_error = msg;
    return code;
}

int cuda_fail(sa_ctx *ctx, cudaError_t e, const char *where) {
    std::string m = std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    return fail(ctx, e == cudaErrorMemoryAllocation ? SA_ERR_NOMEM : SA_ERR_CUDA, m);
}

#define SA_CUDA(ctx, expr)                                    \
    do {                                                      \
        cudaError_t _e = (expr);                              \
        if (_e != cudaSuccess) return cuda_fail(ctx, _e, #expr); \
    } while (0)

template <typename T>
cudaError_t ensure(T *&ptr, size_t &cap, size_t need) {
    if (need <= cap && ptr) return cudaSuccess;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    size_t n = std::max<size_t>(need, 1);
    cudaError_t e = cudaMalloc(reinterpret_cast<void **>(&ptr), n * sizeof(T));
    if (e == cudaSuccess) cap = n;
    return e;
}

int bits_for(uint64_t v) {  // bits needed to represent v (0 -> 0)
    int b = 0;
    while (v) {
        ++b;
        v >>= 1;
    }
    return b;
}

// One launch that resets the per-call device state.
__global__ void k_init(ErrState *err, uint32_t *cur, int64_t ncur, unsigned long long *ts,
                       int64_t nts, unsigned long long *ss, int64_t nss, uint8_t *tb,
                       uint32_t *z, int nz) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    pdl_wait();  // the previous call's fold may still read the look-back words
    pdl_trigger();
    if (t0 == 0) {
        ErrState e;
        memset(&e, 0, sizeof(e));
        e.bad_i = ~0ull;
        e.bad_j = ~0ull;
        *err = e;
    }
    // cur: 16-byte stores where possible
    const int64_t nq = ncur >> 2;
    uint4 *cur4 = reinterpret_cast<uint4 *>(cur);
    for (int64_t k = t0; k < nq; k += stride) cur4[k] = make_uint4(0, 0, 0, 0);
    for (int64_t k = (nq << 2) + t0; k < ncur; k += stride) cur[k] = 0;
    for (int64_t k = t0; k < nts; k += stride) {
        ts[k * LB_STRIDE] = 0ull;
        tb[k] = 0;
    }
    for (int64_t k = t0; k < nss; k += stride) ss[k * LB_STRIDE] = 0ull;
    for (int64_t k = t0; k < nz; k += stride) z[k] = 0u;
}

int launch_init(sa_ctx *ctx, Launch &lc, int64_t ncur, int64_t nts, int64_t nss,
                uint32_t *z = nullptr, int nz = 0) {
    int64_t work = std::max<int64_t>({ncur / 4, nts, nss, (int64_t)nz, 1});
    int grid = (int)std::min<int64_t>((work + 255) / 256, (int64_t)ctx->num_sms * 4);
    SA_CUDA(ctx, launch_pdl(k_init, dim3(grid), dim3(256), 0, lc.stream, ctx->err, ctx->cur, ncur,
                            ctx->tile_state, nts, ctx->scan_state, nss, ctx->tile_big, z, nz));
    lc.launches++;
    return SA_OK;
}

int decode(sa_ctx *ctx, const ErrState &e, int64_t *nnz, int64_t *bad_pos, int *bad_which) {
    if (bad_pos) *bad_pos = -1;
    if (bad_which) *bad_which = -1;
    if (e.bad_i != ~0ull || e.bad_j != ~0ull) {
        const bool row = e.bad_i != ~0ull;
        const int64_t pos = (int64_t)(row ? e.bad_i : e.bad_j);
        if (bad_pos) *bad_pos = pos;
        if (bad_which) *bad_which = row ? SA_WHICH_ROW : SA_WHICH_COL;
        char buf[96];
        snprintf(buf, sizeof buf, "bad %s index at position %lld", row ? "row" : "column",
                 (long long)pos);
        return fail(ctx, SA_ERR_BAD_INDEX, buf);
    }
    if (e.over_m || e.over_n) return fail(ctx, SA_ERR_DIM_TOO_SMALL, "indices exceed the explicit dimensions");
    if (e.internal) return fail(ctx, SA_ERR_INTERNAL, "device consistency check failed");
    if (e.cap_exceeded) {
        if (nnz) *nnz = e.nnz;
        return fail(ctx, SA_ERR_CAPACITY, "nnz exceeds the ir/pr capacity");
    }
    if (nnz) *nnz = e.nnz;
    ctx->last_error.clear();
    return SA_OK;
}

// Record a timing event before the next launch (name) or after the last (nullptr).
int mark(sa_ctx *ctx, const char *name) {
    if (!ctx->timing) return SA_OK;
    if (ctx->nev > sa_ctx::MAXEV) return SA_OK;
    cudaEvent_t &e = ctx->ev[ctx->nev];
    if (!e) SA_CUDA(ctx, cudaEventCreate(&e));
    SA_CUDA(ctx, cudaEventRecord(e, ctx->stream));
    if (name && ctx->nev < sa_ctx::MAXEV) ctx->ev_name[ctx->nev] = name;
    ctx->nev++;
    return SA_OK;
}

}  // namespace

// ---- process-wide cache of page-locked host buffers ------------------------
namespace {
struct PinnedCache {
    std::mutex mu;
    std::map<uint64_t, std::vector<void *>> free_by_class;  // class bytes -> blocks
    std::unordered_map<void *, uint64_t> live;               // block -> class bytes
    uint64_t cached = 0;      // bytes in free blocks
    uint64_t live_bytes = 0;  // bytes handed out and not yet released
    // bounds on the host RAM this library keeps page-locked: free blocks kept
    // for reuse, and results handed out (beyond it callers get nullptr and
    // fall back to pageable memory)
    static constexpr uint64_t kMaxCached = 8ull << 30;
    static constexpr uint64_t kMaxLive = 16ull << 30;
};
PinnedCache &pinned_cache() {
    static PinnedCache *c = new PinnedCache();  // leaked on purpose (process lifetime)
    return *c;
}
uint64_t size_class(uint64_t b) {
    uint64_t c = 1ull << 16;
    while (c < b) c <<= 1;
    return c;
}
}  // namespace

extern "C" {

void *sa_host_buffer(uint64_t bytes) {
    PinnedCache &pc = pinned_cache();
    const uint64_t cls = size_class(std::max<uint64_t>(bytes, 1));
    {
        std::lock_guard<std::mutex> g(pc.mu);
        auto it = pc.free_by_class.find(cls);
        if (it != pc.free_by_class.end() && !it->second.empty()) {
            void *p = it->second.back();
            it->second.pop_back();
            pc.cached -= cls;
            pc.live[p] = cls;
            pc.live_bytes += cls;
            return p;
        }
        if (pc.live_bytes + cls > PinnedCache::kMaxLive) return nullptr;
    }
    void *p = nullptr;
    if (cudaHostAlloc(&p, cls, cudaHostAllocPortable) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> g(pc.mu);
    pc.live[p] = cls;
    pc.live_bytes += cls;
    return p;
}

void sa_host_buffer_release(void *ptr) {
    if (!ptr) return;
    PinnedCache &pc = pinned_cache();
    uint64_t cls = 0;
    {
        std::lock_guard<std::mutex> g(pc.mu);
        auto it = pc.live.find(ptr);
        if (it == pc.live.end()) return;
        cls = it->second;
        pc.live.erase(it);
        pc.live_bytes -= cls;
        if (pc.cached + cls <= PinnedCache::kMaxCached) {
            pc.free_by_class[cls].push_back(ptr);
            pc.cached += cls;
            return;
        }
    }
    cudaFreeHost(ptr);
}

int sa_enable_timing(sa_ctx *ctx, int on) {
    if (!ctx) return SA_ERR_INVALID_ARG;
    ctx->timing = on ? 1 : 0;
    ctx->nev = 0;
    return SA_OK;
}

int sa_last_kernel_times(sa_ctx *ctx, int max, float *ms, const char **names) {
    if (!ctx) return SA_ERR_INVALID_ARG;
    if (ctx->nev < 2) return 0;
    SA_CUDA(ctx, cudaEventSynchronize(ctx->ev[ctx->nev - 1]));
    int n = std::min(ctx->nev - 1, max);
    for (int k = 0; k < n; ++k) {
        float t = 0.f;
        SA_CUDA(ctx, cudaEventElapsedTime(&t, ctx->ev[k], ctx->ev[k + 1]));
        if (ms) ms[k] = t;
        if (names) names[k] = ctx->ev_name[k];
    }
    return n;
}

int sa_version(void) { return 2; }

int sa_create(int device, sa_ctx **out) {
    if (!out) return SA_ERR_INVALID_ARG;
    *out = nullptr;
    sa_ctx *ctx = new sa_ctx();
    ctx->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void **>(&ctx->err), sizeof(ErrState));
    if (e == cudaSuccess) e = cudaMallocHost(reinterpret_cast<void **>(&ctx->err_host), sizeof(ErrState));
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->up_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void **>(&ctx->err_up), sizeof(ErrState));
    if (e == cudaSuccess) e = cudaMallocHost(reinterpret_cast<void **>(&ctx->err_up_host), sizeof(ErrState));
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->up_done, cudaEventDisableTiming);
    for (int k = 0; k < sa_ctx::MAXUP && e == cudaSuccess; ++k)
        e = cudaEventCreateWithFlags(&ctx->up_ev[k], cudaEventDisableTiming);
    if (e != cudaSuccess) {
        int rc = cuda_fail(ctx, e, "sa_create");
        sa_destroy(ctx);
        return rc;
    }
    ctx->stream = ctx->own_stream;
    *out = ctx;
    return SA_OK;
}

void sa_destroy(sa_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->up_stream) {
        cudaStreamSynchronize(ctx->up_stream);
        cudaStreamDestroy(ctx->up_stream);
    }
    cudaFree(ctx->err_up);
    cudaFreeHost(ctx->err_up_host);
    if (ctx->up_done) cudaEventDestroy(ctx->up_done);
    for (auto ev : ctx->up_ev)
        if (ev) cudaEventDestroy(ev);
    cudaFree(ctx->cur);
    cudaFree(ctx->sstart);
    cudaFree(ctx->rec);
    cudaFree(ctx->perm);
    cudaFree(ctx->tile_info);
    cudaFree(ctx->tile_big);
    cudaFree(ctx->tile_state);
    cudaFree(ctx->tile_cnt);
    cudaFree(ctx->scan_state);
    cudaFree(ctx->big_list);
    cudaFree(ctx->bigk);
    cudaFree(ctx->err);
    cudaFree(ctx->pr_state);
    cudaFree(ctx->pt_cnt);
    cudaFree(ctx->pt_off);
    cudaFree(ctx->pt_counts);
    cudaFree(ctx->pr_nnz);
    for (void *p : {(void *)ctx->rx, (void *)ctx->ry, (void *)ctx->rcnt, (void *)ctx->roff, (void *)ctx->rbsum,
                    (void *)ctx->rlbf, (void *)ctx->rbnd, (void *)ctx->rbig, (void *)ctx->rbigu})
        cudaFree(p);
    cudaFree(ctx->h_ii);
    cudaFree(ctx->h_jj);
    cudaFree(ctx->h_s);
    cudaFree(ctx->o_jc);
    cudaFree(ctx->o_ir);
    cudaFree(ctx->o_pr);
    if (ctx->err_host) cudaFreeHost(ctx->err_host);
    for (int k = 0; k <= sa_ctx::MAXEV; ++k)
        if (ctx->ev[k]) cudaEventDestroy(ctx->ev[k]);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
}

int sa_set_option(sa_ctx *ctx, int option, int value) {
    if (!ctx) return SA_ERR_INVALID_ARG;
    if (value < -1 || value > 1) return fail(ctx, SA_ERR_INVALID_ARG, "sa_set_option: value must be -1, 0 or 1");
    switch (option) {
        case SA_OPT_FOLD_STAGED: ctx->opt_fold_staged = value; return SA_OK;
        case SA_OPT_SCATTER_STAGED: ctx->opt_scatter_staged = value; return SA_OK;
        case SA_OPT_PATH: ctx->opt_path = value; return SA_OK;
        case SA_OPT_RPASS_TMA: ctx->opt_rpass_tma = value; return SA_OK;
        default: return fail(ctx, SA_ERR_INVALID_ARG, "sa_set_option: unknown option");
    }
}

int sa_set_stream(sa_ctx *ctx, void *stream) {
    if (!ctx) return SA_ERR_INVALID_ARG;
    ctx->stream = reinterpret_cast<cudaStream_t>(stream);  // 0 = the legacy default stream
    return SA_OK;
}

const char *sa_last_error(const sa_ctx *ctx) { return ctx ? ctx->last_error.c_str() : "null context"; }

int sa_last_launch_count(const sa_ctx *ctx) { return ctx ? ctx->launches : 0; }

const int64_t *sa_device_nnz(sa_ctx *ctx) {
    return ctx ? reinterpret_cast<const int64_t *>(&ctx->err->nnz) : nullptr;
}

int sa_convert_indices(sa_ctx *ctx, const void *d_raw, int dtype, int64_t L, int32_t *d_out,
                       int64_t *first_bad, int32_t *max_out) {
    if (!ctx) return SA_ERR_INVALID_ARG;
    if (L < 0 || (L > 0 && (!d_raw || !d_out)) || dtype < 0 || dtype > 2)
        return fail(ctx, SA_ERR_INVALID_ARG, "sa_convert_indices: bad arguments");
    SA_CUDA(ctx, cudaSetDevice(ctx->device));
    Launch lc{ctx->stream, ctx->num_sms, 0};
    int rc = launch_init(ctx, lc, 0, 0, 0);
    if (rc) return rc;
    static const int kmap[3] = {0, 1, 2};
    SA_CUDA(ctx, launch_convert(lc, d_raw, kmap[dtype], L, d_out, ctx->err));
    SA_CUDA(ctx, cudaMemcpyAsync(ctx->err_host, ctx->err, sizeof(ErrState), cudaMemcpyDeviceToHost, ctx->stream));
    SA_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    ctx->launches = lc.launches;
    if (first_bad) *first_bad = ctx->err_host->bad_i == ~0ull ? -1 : (int64_t)ctx->err_host->bad_i;
    if (max_out) *max_out = (int32_t)ctx->err_host->max_i;
    return SA_OK;
}

int sa_infer_dims(sa_ctx *ctx, const int32_t *d_ii, const int32_t *d_jj, int64_t L, int32_t *M,
                  int32_t *N, int64_t *bad_pos, int *bad_which) {
    if (!ctx) return SA_ERR_INVALID_ARG;
    if (L < 0 || (L > 0 && (!d_ii || !d_jj)))
        return fail(ctx, SA_ERR_INVALID_ARG, "sa_infer_dims: bad arguments");
    SA_CUDA(ctx, cudaSetDevice(ctx->device));
    Launch lc{ctx->stream, ctx->num_sms, 0};
    int rc = launch_init(ctx, lc, 0, 0, 0);
    if (rc) return rc;
    SA_CUDA(ctx, launch_hist(lc, d_ii, d_jj, L, 0, 0, nullptr, ctx->err, true));
    SA_CUDA(ctx, cudaMemcpyAsync(ctx->err_host, ctx->err, sizeof(ErrState), cudaMemcpyDeviceToHost, ctx->stream));
    SA_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    ctx->launches = lc.launches;
    if (M) *M = (int32_t)ctx->err_host->max_i;
    if (N) *N = (int32_t)ctx->err_host->max_j;
    ErrState e = *ctx->err_host;
    e.nnz = 0;
    return decode(ctx, e, nullptr, bad_pos, bad_which);
}

namespace {

// ---- radix path (sa_radix.cu) -------------------------------------------------
struct RadixPlan {
    bool ok = false;
    int z = 0, rbits = 0, npass = 0;
    int shift[RP_MAXPASS] = {}, bits[RP_MAXPASS] = {};
    int32_t nsub = 0;
    int64_t nchunk = 0;
};

// The sort key of a triplet is (col - 1) << rbits | (row - 1); sub-bucket s
// holds the keys [s << z, (s + 1) << z) and the passes partition on the key
// bits above z (at most RP_MAXPASS passes of at most RP_MAXBITS bits).
// Column-block plan: z = rbits + w, sub-buckets of W = 2^w whole columns --
// the largest w whose expected sub-bucket (L W / N triplets) stays within 4/5
// of the fold's shared-memory capacity, with the local key inside 31 bits.
// Row-split plan, when even single columns are longer than that on average
// (few, long columns: L > 4/5 RF_CAP N): z < rbits, sub-buckets of 2^z rows
// of one column, expected (L / N) 2^z / M triplets.
RadixPlan radix_plan(int64_t L, int32_t M, int32_t N) {
    RadixPlan P;
    if (L <= 0 || N <= 0 || M <= 0) return P;
    P.rbits = bits_for((uint64_t)(M - 1));
    const int cbits = bits_for((uint64_t)(N - 1));
    const int64_t cap = 4 * RF_CAP / 5;
    int z;
    if (L <= cap * (int64_t)N || P.rbits == 0) {
        int w = 0;
        while (w < 8 && w < cbits && w + 1 + P.rbits <= 31 && (L << (w + 1)) <= cap * (int64_t)N) ++w;
        z = w + P.rbits;
    } else {
        z = 0;
        while (z + 1 < P.rbits && (double)L / N * (double)(1ll << (z + 1)) / M <= (double)cap) ++z;
    }
    if (z > 31) return P;
    const int R = cbits + P.rbits - z;
    const int npass = std::max(1, (R + RP_MAXBITS - 1) / RP_MAXBITS);
    if (npass > RP_MAXPASS) return P;
    int sh = z;
    for (int p = 0; p < npass; ++p) {
        P.bits[p] = R / npass + (p < R % npass ? 1 : 0);
        P.shift[p] = sh;
        sh += P.bits[p];
    }
    const uint64_t kmax = ((uint64_t)(N - 1) << P.rbits) | (uint64_t)(M - 1);
    if ((kmax >> z) >= (uint64_t)INT32_MAX) return P;
    P.z = z;
    P.npass = npass;
    P.nsub = (int32_t)((kmax >> z) + 1);
    P.nchunk = (L + RP_CHUNK - 1) / RP_CHUNK;
    P.ok = true;
    return P;
}

// One partition buffer of 16 bytes per triplet for `need` triplets: viewed as
// the column arrays ii, jj (int32) and s (float64), each 16-byte aligned, or
// as `need` records.
cudaError_t ensure_trip(uint4 *&blk, int32_t *&i, int32_t *&j, double *&v, size_t &cap, size_t need) {
    if (need <= cap && blk) return cudaSuccess;
    cudaFree(blk);
    blk = nullptr;
    i = j = nullptr;
    v = nullptr;
    cap = 0;
    need = (std::max<size_t>(need, 1) + 3) & ~size_t(3);
    cudaError_t e = cudaMalloc(reinterpret_cast<void **>(&blk), need * 16);
    if (e != cudaSuccess) return e;
    cap = need;
    i = reinterpret_cast<int32_t *>(blk);
    j = i + need;
    v = reinterpret_cast<double *>(j + need);
    return e;
}

// ensure() for look-back word arrays: fresh memory is zeroed (tag 0 = never
// published); returns true in `fresh` when the array was (re)allocated.
cudaError_t ensure_lb(unsigned long long *&p, size_t &cap, size_t need, cudaStream_t st, bool &fresh) {
    fresh = false;
    if (need <= cap && p) return cudaSuccess;
    cudaError_t e = ensure(p, cap, need);
    if (e == cudaSuccess) e = cudaMemsetAsync(p, 0, cap * sizeof(unsigned long long), st);
    fresh = true;
    return e;
}

int assemble_radix(sa_ctx *ctx, const RadixPlan &P, const int32_t *ii, const int32_t *jj,
                   const double *s, int64_t s_stride, int64_t L, int32_t M, int32_t N,
                   int32_t *d_jc, int32_t *d_ir, double *d_pr, int64_t cap) {
    Launch lc{ctx->stream, ctx->num_sms, 0};
    lc.rpass_tma = ctx->opt_rpass_tma;
    const size_t nl = (size_t)L;
    const size_t nsub = (size_t)P.nsub;
    // X and Y: the passes alternate X, Y, X, ...; the last one writes records.
    // (With one pass Y is the oversize scratch B.)
    SA_CUDA(ctx, ensure_trip(ctx->rx, ctx->rx_i, ctx->rx_j, ctx->rx_s, ctx->rx_cap, nl));
    SA_CUDA(ctx, ensure_trip(ctx->ry, ctx->ry_i, ctx->ry_j, ctx->ry_s, ctx->ry_cap, nl));
    SA_CUDA(ctx, ensure(ctx->perm, ctx->perm_cap, nl + 2));  // oversize scratch A
    // partition CTAs: the resident ones (2 per SM), walking the chunks with that stride
    const int nseg = (int)std::max<int64_t>(1, std::min<int64_t>(P.nchunk, (int64_t)ctx->num_sms * (2048 / RP_NT)));
    const int cpb = rup_cpb(P.nchunk, ctx->num_sms);
    const int64_t nblk = (P.nchunk + cpb - 1) / cpb;
    SA_CUDA(ctx, ensure(ctx->rcnt, ctx->rcnt_cap, (size_t)P.nchunk * RP_MAXD));
    SA_CUDA(ctx, ensure(ctx->roff, ctx->roff_cap, (size_t)P.nchunk * RP_MAXD));
    SA_CUDA(ctx, ensure(ctx->rbsum, ctx->rbsum_cap, (size_t)(std::max<int64_t>(nblk, 1) + 1) * RP_MAXD));  // + the digit totals
    bool f2 = false;
    SA_CUDA(ctx, ensure_lb(ctx->rlbf, ctx->rlbf_cap, nsub * LB_STRIDE, ctx->stream, f2));
    SA_CUDA(ctx, ensure(ctx->rbnd, ctx->rbnd_cap, nsub + 1));
    SA_CUDA(ctx, ensure(ctx->rbig, ctx->rbig_cap, nsub));
    SA_CUDA(ctx, ensure(ctx->rbigu, ctx->rbigu_cap, nsub));
    // look-back tags: (epoch << 2 | pass), epoch in [1, 16383]; on wrap-around
    // every word is cleared once so no stale word can carry a live tag
    if (++ctx->rp_epoch >= 16384) {
        if (!f2) SA_CUDA(ctx, cudaMemsetAsync(ctx->rlbf, 0, ctx->rlbf_cap * 8, ctx->stream));
        ctx->rp_epoch = 1;
    }
    const unsigned ep = ctx->rp_epoch << 2;

    ctx->nev = 0;
    int rc = mark(ctx, "k_init");
    if (rc) return rc;
    if ((rc = launch_init(ctx, lc, 0, 0, 0))) return rc;
    int32_t *bi[2] = {ctx->rx_i, ctx->ry_i}, *bj[2] = {ctx->rx_j, ctx->ry_j};
    double *bs[2] = {ctx->rx_s, ctx->ry_s};
    uint4 *br[2] = {ctx->rx, ctx->ry};
    static const char *pname[RP_MAXPASS] = {"k_rpass0", "k_rpass1", "k_rpass2", "k_rpass3"};
    static const char *uname[RP_MAXPASS] = {"k_rup0", "k_rup1", "k_rup2", "k_rup3"};
    for (int p = 0; p < P.npass; ++p) {
        RadixPassArgs A{};
        A.ii_in = p ? bi[(p - 1) & 1] : ii;
        A.jj_in = p ? bj[(p - 1) & 1] : jj;
        A.rc_in = p ? reinterpret_cast<const int2 *>(bi[(p - 1) & 1]) : nullptr;  // (the ii | jj regions)
        A.s_in = p ? bs[(p - 1) & 1] : s;
        A.s_stride = p ? 1 : s_stride;
        A.ii_out = bi[p & 1];
        A.jj_out = bj[p & 1];
        A.s_out = bs[p & 1];
        A.rc_out = reinterpret_cast<int2 *>(bi[p & 1]);  // the ii | jj regions of the block
        A.L = L;
        A.M = M;
        A.N = N;
        A.shift = P.shift[p];
        A.bits = P.bits[p];
        A.rbits = P.rbits;
        A.off = ctx->roff;
        if ((rc = mark(ctx, uname[p]))) return rc;
        SA_CUDA(ctx, launch_rup(lc, p == 0, A.ii_in, A.jj_in, A.rc_in, L, N, A.shift, A.bits, P.rbits, ctx->rcnt,
                                ctx->rbsum, ctx->roff, ctx->err));
        if ((rc = mark(ctx, pname[p]))) return rc;
        SA_CUDA(ctx, launch_rpass(lc, A, p == 0, p == P.npass - 1, nseg, ctx->err));
    }
    const int fb = (P.npass - 1) & 1;  // buffer holding the partitioned records
    RadixFoldArgs F{};
    F.rc = reinterpret_cast<const int2 *>(bi[fb]);
    // (16-byte records: the value sits behind its {row, col} pair)
    F.s = SA_AOS ? reinterpret_cast<const double *>(br[fb]) + 1 : bs[fb];
    F.bnd = ctx->rbnd;
    F.biglist = ctx->rbig;
    F.bigu = ctx->rbigu;
    F.scrA = reinterpret_cast<unsigned long long *>(ctx->perm);
    F.scrB = reinterpret_cast<unsigned long long *>(br[fb ^ 1]);
    F.lbf = ctx->rlbf;
    F.tag = ep | 3u;
    F.z = P.z;
    F.rbits = P.rbits;
    F.N = N;
    F.nsub = P.nsub;
    F.jc = d_jc;
    F.ir = d_ir;
    F.pr = d_pr;
    F.cap = cap;
    if ((rc = mark(ctx, "k_rbounds"))) return rc;
    SA_CUDA(ctx, launch_rbounds(lc, F.rc, P.z, P.rbits, P.nsub, ctx->rbnd, ctx->rbig, ctx->err));
    if ((rc = mark(ctx, "k_rbig"))) return rc;
    SA_CUDA(ctx, launch_rbig(lc, F, ctx->err));
    if ((rc = mark(ctx, "k_rfold"))) return rc;
    SA_CUDA(ctx, launch_rfold(lc, F, ctx->err));
    if ((rc = mark(ctx, nullptr))) return rc;
    ctx->launches = lc.launches;
    return SA_OK;
}

// ---- path choice -----------------------------------------------------------------
// The column-cursor pipeline wins when consecutive triplets touch nearby
// columns (element-ordered FEM input: its scatter write front and its value
// gathers stay in L2); the radix path wins when they do not (shuffled input:
// cfg4 70.7 vs 25.7 ms; cfg2 0.32 vs 1.1 ms the other way).  The choice looks
// at RADIX_WIN windows of RADIX_WLEN consecutive column indices spread over
// the input: the median number of distinct 64-column blocks per window.
// The sample costs one small synchronous copy, so the decision is cached per
// (input pointer, L, M, N): re-assembling the same buffers reuses it (a stale
// choice after the caller rewrites the buffers only costs speed -- both paths
// give the same bits).
constexpr int64_t RADIX_MIN_L = 1 << 21;
constexpr int64_t RADIX_LONG_L = 1 << 16;  // long-column inputs take the radix path from this size
constexpr int RADIX_WIN = 8;
constexpr int RADIX_WLEN = 1024;
constexpr int RADIX_BLOCKS = RADIX_WLEN / 4;  // more distinct blocks per window: no locality

int64_t window_at(int64_t L, int wdx) {
    return std::max<int64_t>(0, std::min<int64_t>(L - RADIX_WLEN, L * (2 * wdx + 1) / (2 * RADIX_WIN)));
}
bool sample_says_radix(const std::vector<int32_t> &smp);

int choose_radix(sa_ctx *ctx, const int32_t *jj, int64_t L, int32_t M, int32_t N, bool &radix) {
    const std::tuple<const void *, int64_t, int32_t, int32_t> key{jj, L, M, N};
    auto it = ctx->path_cache.find(key);
    if (it != ctx->path_cache.end()) {
        radix = it->second;
        return SA_OK;
    }
    std::vector<int32_t> smp((size_t)RADIX_WIN * RADIX_WLEN);
    for (int wdx = 0; wdx < RADIX_WIN; ++wdx)
        SA_CUDA(ctx, cudaMemcpyAsync(smp.data() + (size_t)wdx * RADIX_WLEN, jj + window_at(L, wdx),
                                     RADIX_WLEN * 4, cudaMemcpyDeviceToHost, ctx->stream));
    SA_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    radix = sample_says_radix(smp);
    if (ctx->path_cache.size() > 64) ctx->path_cache.clear();
    ctx->path_cache[key] = radix;
    return SA_OK;
}

bool sample_says_radix(const std::vector<int32_t> &smp) {
    std::vector<int> distinct(RADIX_WIN);
    for (int wdx = 0; wdx < RADIX_WIN; ++wdx) {
        std::vector<int32_t> b(smp.begin() + (size_t)wdx * RADIX_WLEN, smp.begin() + (size_t)(wdx + 1) * RADIX_WLEN);
        for (auto &x : b) x >>= 6;
        std::sort(b.begin(), b.end());
        distinct[wdx] = (int)(std::unique(b.begin(), b.end()) - b.begin());
    }
    std::nth_element(distinct.begin(), distinct.begin() + RADIX_WIN / 2, distinct.end());
    return distinct[RADIX_WIN / 2] > RADIX_BLOCKS;
}

// The assembly pipeline over a segment table (Ltot triplets in total).
int assemble_segments(sa_ctx *ctx, const Segs &S, int64_t L, int32_t M, int32_t N, int32_t *d_jc,
                      int32_t *d_ir, double *d_pr, int64_t cap) {
    SA_CUDA(ctx, cudaSetDevice(ctx->device));
    if (S.nseg == 1 && L > 0 && N > 0 && M > 0 && ctx->opt_path != 0) {
        const RadixPlan P = radix_plan(L, M, N);
        bool radix = P.ok && ctx->opt_path == 1;
        if (P.ok && ctx->opt_path == -1 && L >= RADIX_LONG_L && P.z < P.rbits) {
            // columns longer than a fold sub-bucket on average: the row-split
            // plan spreads each column over many CTAs (the column-cursor
            // pipeline folds a big column in one CTA)
            radix = true;
        } else if (P.ok && ctx->opt_path == -1 && L >= RADIX_MIN_L) {
            if (S.jj[0] == ctx->h_jj && ctx->host_radix >= 0) {
                radix = ctx->host_radix == 1;  // host protocol: chosen at upload
            } else {
                int rc = choose_radix(ctx, S.jj[0], L, M, N, radix);
                if (rc) return rc;
            }
        }
        if (radix)
            return assemble_radix(ctx, P, S.ii[0], S.jj[0], S.s[0], S.stride[0], L, M, N, d_jc, d_ir,
                                  d_pr, cap);
    }
    Launch lc{ctx->stream, ctx->num_sms, 0};
    lc.fold_staged = ctx->opt_fold_staged;
    lc.scatter_staged = ctx->opt_scatter_staged;

    if (L == 0 || N == 0) {
        // nothing to assemble (L > 0 with N == 0 means every column index is
        // out of range: k_hist still flags it)
        int rc = launch_init(ctx, lc, 0, 0, 0);
        if (rc) return rc;
        // L > 0 with N == 0: validation only; every valid column index then
        // exceeds N and k_hist flags DimensionTooSmall (no histogram writes)
        if (L > 0 && !S.skip_foreign)
            for (int g = 0; g < S.nseg; ++g)
                SA_CUDA(ctx, launch_hist(lc, S.ii[g], S.jj[g], S.len[g], M, N, ctx->cur, ctx->err, false,
                                         S.pos0[g]));
        SA_CUDA(ctx, cudaMemsetAsync(d_jc, 0, ((size_t)N + 1) * sizeof(int32_t), ctx->stream));
        ctx->launches = lc.launches;
        return SA_OK;
    }

    const int64_t nbig_max = L / (BIGCOL + 1) + 1;
    // fold tile size: TILE, or smaller so that a small input still gives every
    // SM two tiles (cfg1: 56 tiles of 1792 slots would leave 92 SMs idle)
    int tile_sz = TILE;
    if ((L + nbig_max + TILE - 1) / TILE < 2 * (int64_t)ctx->num_sms)
        tile_sz = (int)std::max<int64_t>(256, (L + nbig_max + 2 * ctx->num_sms - 1) / (2 * ctx->num_sms));
    const int64_t ntiles = (L + nbig_max + tile_sz - 1) / tile_sz;
    const int64_t nscan = (N + SCAN_TILE - 1) / SCAN_TILE;
    SA_CUDA(ctx, ensure(ctx->cur, ctx->cur_cap, (size_t)N + 4));
    SA_CUDA(ctx, ensure(ctx->sstart, ctx->st_cap, (size_t)N + 1));
    SA_CUDA(ctx, ensure(ctx->perm, ctx->perm_cap, (size_t)(L + nbig_max + 2)));  // TMA over-read
    SA_CUDA(ctx, ensure(ctx->rec, ctx->rec_cap, (size_t)(L + nbig_max)));
    SA_CUDA(ctx, ensure(ctx->tile_info, ctx->ti_cap, (size_t)ntiles + 1));
    SA_CUDA(ctx, ensure(ctx->tile_big, ctx->tb_cap, (size_t)ntiles));
    SA_CUDA(ctx, ensure(ctx->tile_state, ctx->ts_cap, (size_t)ntiles * LB_STRIDE));
    SA_CUDA(ctx, ensure(ctx->scan_state, ctx->ss_cap, (size_t)nscan * LB_STRIDE));
    SA_CUDA(ctx, ensure(ctx->big_list, ctx->bl_cap, (size_t)nbig_max));
    SA_CUDA(ctx, ensure(ctx->bigk, ctx->bk_cap, (size_t)N));

    ctx->nev = 0;
    int rc = mark(ctx, "k_init");
    if (rc) return rc;
    rc = launch_init(ctx, lc, N, ntiles, nscan);
    if (rc) return rc;
    if ((rc = mark(ctx, "k_colcount"))) return rc;
    SA_CUDA(ctx, launch_colcount(lc, S, N, ctx->cur, ctx->err));
    if ((rc = mark(ctx, "k_col_scan"))) return rc;
    SA_CUDA(ctx, launch_col_scan(lc, ctx->cur, ctx->sstart, ctx->cur, N, ctx->tile_info,
                                 ctx->tile_big, ntiles, ctx->big_list, ctx->bigk, ctx->scan_state,
                                 ctx->perm, ctx->err, tile_sz));
    if ((rc = mark(ctx, "k_scatter"))) return rc;
    SA_CUDA(ctx, launch_scatter(lc, S, M, N, ctx->cur, ctx->perm, ctx->err));
    if (L > BIGCOL) {
        const int idx_bits = std::max(1, bits_for((uint64_t)(L - 1)));
        const int row_bits = bits_for((uint64_t)(M > 0 ? M - 1 : 0));
        const int passes = std::max(1, (idx_bits + row_bits + 7) / 8);
        if ((rc = mark(ctx, "k_bigcol"))) return rc;
        SA_CUDA(ctx, launch_bigcol(lc, ctx->big_list, ctx->err, ctx->rec, ctx->perm, S, idx_bits,
                                   passes));
    }
    // long columns dominate: stage the outputs instead of chaining tile offsets
    const bool staged = ctx->opt_fold_staged >= 0
                            ? ctx->opt_fold_staged == 1
                            : (L >= 40 * (int64_t)N && ntiles >= 16 * ctx->num_sms);
    if (staged) {
        SA_CUDA(ctx, ensure(ctx->tile_cnt, ctx->tc_cap, (size_t)ntiles));
    }
    if ((rc = mark(ctx, "k_tile_fold"))) return rc;
    SA_CUDA(ctx, launch_tile_fold(lc, ctx->sstart, ctx->tile_info, ctx->tile_big, ntiles,
                                  reinterpret_cast<const int2 *>(ctx->perm), S, ctx->rec,
                                  ctx->big_list, ctx->bigk, ctx->tile_state, N, d_jc, d_ir, d_pr,
                                  cap, ctx->err, staged ? ctx->rec : nullptr, ctx->tile_cnt));
    if ((rc = mark(ctx, nullptr))) return rc;
    ctx->launches = lc.launches;
    return SA_OK;
}

bool aligned16p(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Segment table; false if a segment is malformed.
bool make_segs(int nseg, const int32_t *const *ii, const int32_t *const *jj,
               const double *const *s, const int64_t *s_stride, const int64_t *len, int32_t col_lo,
               int skip_foreign, Segs &S, int64_t &total) {
    constexpr int64_t CH = 2048;  // = CHUNK of sa_kernels.cu
    S = Segs{};
    S.nseg = nseg;
    S.col_lo = col_lo;
    S.skip_foreign = skip_foreign;
    total = 0;
    int64_t ch = 0;
    for (int g = 0; g < nseg; ++g) {
        if (len[g] < 0 || (s_stride[g] != 0 && s_stride[g] != 1)) return false;
        if (len[g] > 0 && (!ii[g] || !jj[g] || !s[g])) return false;
        S.ii[g] = ii[g];
        S.jj[g] = jj[g];
        S.s[g] = s[g];
        S.stride[g] = s_stride[g];
        S.len[g] = len[g];
        S.pos0[g] = total;
        S.ch0[g] = ch;
        S.vec[g] = aligned16p(ii[g]) && aligned16p(jj[g]);
        total += len[g];
        ch += (len[g] + CH - 1) / CH;
    }
    S.ch0[nseg] = ch;
    return true;
}

}  // namespace

int sa_assemble_async(sa_ctx *ctx, const int32_t *d_ii, const int32_t *d_jj, const double *d_s,
                      int64_t s_stride, int64_t L, int32_t M, int32_t N, int32_t *d_jc,
                      int32_t *d_ir, double *d_pr, int64_t cap) {
    if (!ctx) return SA_ERR_INVALID_ARG;
    if (L < 0 || M < 0 || N < 0 || cap < 0 || !d_jc || (s_stride != 0 && s_stride != 1))
        return fail(ctx, SA_ERR_INVALID_ARG, "sa_assemble_async: bad arguments");
    if (L > 0 && (!d_ii || !d_jj || !d_s))
        return fail(ctx, SA_ERR_INVALID_ARG, "sa_assemble_async: null triplet pointer");
    if (L > (int64_t)POSMASK)
        return fail(ctx, SA_ERR_INVALID_ARG, "sa_assemble_async: more than 2^31-1 triplets");
    Segs S;
    int64_t total = 0;
    make_segs(1, &d_ii, &d_jj, &d_s, &s_stride, &L, 0, 0, S, total);
    return assemble_segments(ctx, S, L, M, N, d_jc, d_ir, d_pr, cap);
}

int sa_assemble_segments_async(sa_ctx *ctx, int nseg, const int32_t *const *d_ii,
                               const int32_t *const *d_jj, const double *const *d_s,
                               const int64_t *s_stride, const int64_t *len, int32_t col_lo,
                               int32_t M, int32_t N, int32_t *d_jc, int32_t *d_ir, double *d_pr,
                               int64_t cap) {
    if (!ctx) return SA_ERR_INVALID_ARG;
    if (nseg < 1 || nseg > MAXSEG || !d_ii || !d_jj || !d_s || !s_stride || !len || M < 0 ||
        N < 0 || col_lo < 0 || cap < 0 || !d_jc)
        return fail(ctx, SA_ERR_INVALID_ARG, "sa_assemble_segments_async: bad arguments");
    Segs S;
    int64_t total = 0;
    if (!make_segs(nseg, d_ii, d_jj, d_s, s_stride, len, col_lo, 1, S, total))
        return fail(ctx, SA_ERR_INVALID_ARG, "sa_assemble_segments_async: bad segment");
    if (total > (int64_t)POSMASK)
        return fail(ctx, SA_ERR_INVALID_ARG, "sa_assemble_segments_async: more than 2^31-1 triplets");
    return assemble_segments(ctx, S, total, M, N, d_jc, d_ir, d_pr, cap);
}

int sa_finish(sa_ctx *ctx, int64_t *nnz, int64_t *bad_pos, int *bad_which) {
    if (!ctx) return SA_ERR_INVALID_ARG;
    SA_CUDA(ctx, cudaSetDevice(ctx->device));
    SA_CUDA(ctx, cudaMemcpyAsync(ctx->err_host, ctx->err, sizeof(ErrState), cudaMemcpyDeviceToHost, ctx->stream));
    SA_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return decode(ctx, *ctx->err_host, nnz, bad_pos, bad_which);
}

int sa_host_upload(sa_ctx *ctx, const int32_t *h_ii, const int32_t *h_jj, const double *h_s,
                   int64_t s_stride, int64_t L) {
    if (!ctx) return SA_ERR_INVALID_ARG;
    if (L < 0 || (L > 0 && (!h_ii || !h_jj || !h_s)) || (s_stride != 0 && s_stride != 1))
        return fail(ctx, SA_ERR_INVALID_ARG, "sa_host_upload: bad arguments");
    SA_CUDA(ctx, cudaSetDevice(ctx->device));
    ctx->host_nnz = -1;
    ctx->host_L = L;
    ctx->host_stride = s_stride;
    ctx->host_radix = -1;
    if (L >= RADIX_MIN_L) {  // the path choice from the host copy of the columns
        std::vector<int32_t> smp((size_t)RADIX_WIN * RADIX_WLEN);
        for (int wdx = 0; wdx < RADIX_WIN; ++wdx)
            memcpy(smp.data() + (size_t)wdx * RADIX_WLEN, h_jj + window_at(L, wdx), RADIX_WLEN * 4);
        ctx->host_radix = sample_says_radix(smp) ? 1 : 0;
    }
    const size_t nl = (size_t)std::max<int64_t>(L, 1);
    const size_t ns = s_stride ? nl : 1;
    // the previous upload's dimension pass may still read the buffers (the
    // assembly itself never waits for it)
    SA_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->up_done, 0));
    SA_CUDA(ctx, cudaStreamSynchronize(ctx->up_stream));
    SA_CUDA(ctx, ensure(ctx->h_ii, ctx->hii_cap, nl));
    SA_CUDA(ctx, ensure(ctx->h_jj, ctx->hjj_cap, nl));
    SA_CUDA(ctx, ensure(ctx->h_s, ctx->hs_cap, ns));
    // the dimension / validation pass (types.py:121-138, 163-165: maxima and
    // first bad positions) is fused into the upload: it runs on up_stream
    // over each chunk as soon as it has landed, overlapped with the copy of
    // the next one, so sa_host_dims only reads its outcome
    {
        ErrState z{};
        z.bad_i = ~0ull;
        z.bad_j = ~0ull;
        *ctx->err_up_host = z;
    }
    SA_CUDA(ctx, cudaMemcpyAsync(ctx->err_up, ctx->err_up_host, sizeof(ErrState), cudaMemcpyHostToDevice,
                                 ctx->stream));
    if (L > 0) {
        const int64_t nch = std::min<int64_t>(sa_ctx::MAXUP, std::max<int64_t>(1, L >> 24));  // >= 16M per chunk
        Launch lc{ctx->up_stream, ctx->num_sms, 0};
        for (int64_t k = 0; k < nch; ++k) {
            const int64_t a = (L * k / nch) & ~(int64_t)3, b = (k + 1 == nch) ? L : ((L * (k + 1) / nch) & ~(int64_t)3);
            if (b <= a) continue;
            SA_CUDA(ctx, cudaMemcpyAsync(ctx->h_ii + a, h_ii + a, (size_t)(b - a) * 4, cudaMemcpyHostToDevice, ctx->stream));
            SA_CUDA(ctx, cudaMemcpyAsync(ctx->h_jj + a, h_jj + a, (size_t)(b - a) * 4, cudaMemcpyHostToDevice, ctx->stream));
            if (s_stride)
                SA_CUDA(ctx, cudaMemcpyAsync(ctx->h_s + a, h_s + a, (size_t)(b - a) * 8, cudaMemcpyHostToDevice, ctx->stream));
            SA_CUDA(ctx, cudaEventRecord(ctx->up_ev[k], ctx->stream));
            SA_CUDA(ctx, cudaStreamWaitEvent(ctx->up_stream, ctx->up_ev[k], 0));
            SA_CUDA(ctx, launch_hist(lc, ctx->h_ii + a, ctx->h_jj + a, b - a, 0, 0, nullptr, ctx->err_up, true, a));
        }
        if (!s_stride) SA_CUDA(ctx, cudaMemcpyAsync(ctx->h_s, h_s, 8, cudaMemcpyHostToDevice, ctx->stream));
    }
    SA_CUDA(ctx, cudaEventRecord(ctx->up_done, ctx->up_stream));
    return SA_OK;
}

int sa_host_dims(sa_ctx *ctx, int32_t *M, int32_t *N, int64_t *bad_pos, int *bad_which) {
    if (!ctx) return SA_ERR_INVALID_ARG;
    if (ctx->host_L < 0) return fail(ctx, SA_ERR_INVALID_ARG, "sa_host_dims: nothing uploaded");
    SA_CUDA(ctx, cudaSetDevice(ctx->device));
    // the outcome of the pass the upload ran (no further pass over the data)
    SA_CUDA(ctx, cudaMemcpyAsync(ctx->err_up_host, ctx->err_up, sizeof(ErrState), cudaMemcpyDeviceToHost,
                                 ctx->up_stream));
    SA_CUDA(ctx, cudaStreamSynchronize(ctx->up_stream));
    ErrState e = *ctx->err_up_host;
    if (M) *M = (int32_t)e.max_i;
    if (N) *N = (int32_t)e.max_j;
    e.nnz = 0;
    return decode(ctx, e, nullptr, bad_pos, bad_which);
}

int sa_host_assemble(sa_ctx *ctx, int32_t M, int32_t N, int64_t *nnz, int64_t *bad_pos,
                     int *bad_which) {
    if (!ctx) return SA_ERR_INVALID_ARG;
    if (ctx->host_L < 0) return fail(ctx, SA_ERR_INVALID_ARG, "sa_host_assemble: nothing uploaded");
    if (M < 0 || N < 0) return fail(ctx, SA_ERR_INVALID_ARG, "sa_host_assemble: negative dimensions");
    ctx->host_nnz = -1;
    SA_CUDA(ctx, cudaSetDevice(ctx->device));
    const size_t nl = (size_t)std::max<int64_t>(ctx->host_L, 1);
    SA_CUDA(ctx, ensure(ctx->o_jc, ctx->ojc_cap, (size_t)N + 1));
    SA_CUDA(ctx, ensure(ctx->o_ir, ctx->oir_cap, nl));
    SA_CUDA(ctx, ensure(ctx->o_pr, ctx->opr_cap, nl));
    int rc = sa_assemble_async(ctx, ctx->h_ii, ctx->h_jj, ctx->h_s, ctx->host_stride, ctx->host_L,
                               M, N, ctx->o_jc, ctx->o_ir, ctx->o_pr, (int64_t)nl);
    if (rc) return rc;
    int64_t z = 0;
    rc = sa_finish(ctx, &z, bad_pos, bad_which);
    if (rc) return rc;
    if (nnz) *nnz = z;
    ctx->host_nnz = z;
    ctx->host_N = N;
    return SA_OK;
}

int sa_host_fetch(sa_ctx *ctx, int32_t *h_jc, int32_t *h_ir, double *h_pr) {
    if (!ctx) return SA_ERR_INVALID_ARG;
    if (ctx->host_nnz < 0) return fail(ctx, SA_ERR_INVALID_ARG, "sa_host_fetch: no assembled result");
    if (!h_jc || (ctx->host_nnz > 0 && (!h_ir || !h_pr)))
        return fail(ctx, SA_ERR_INVALID_ARG, "sa_host_fetch: null output");
    SA_CUDA(ctx, cudaSetDevice(ctx->device));
    SA_CUDA(ctx, cudaMemcpyAsync(h_jc, ctx->o_jc, ((size_t)ctx->host_N + 1) * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (ctx->host_nnz > 0) {
        SA_CUDA(ctx, cudaMemcpyAsync(h_ir, ctx->o_ir, (size_t)ctx->host_nnz * 4, cudaMemcpyDeviceToHost, ctx->stream));
        SA_CUDA(ctx, cudaMemcpyAsync(h_pr, ctx->o_pr, (size_t)ctx->host_nnz * 8, cudaMemcpyDeviceToHost, ctx->stream));
    }
    SA_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return SA_OK;
}

int sa_prune_zeros(sa_ctx *ctx, const int32_t *d_jc, const int32_t *d_ir, const double *d_pr,
                   int32_t N, int64_t nnz, int32_t *d_jc_out, int32_t *d_ir_out,
                   double *d_pr_out, int64_t *nnz_out) {
    if (!ctx) return SA_ERR_INVALID_ARG;
    if (N < 0 || nnz < 0 || !d_jc || !d_jc_out || (nnz > 0 && (!d_ir || !d_pr || !d_ir_out || !d_pr_out)))
        return fail(ctx, SA_ERR_INVALID_ARG, "sa_prune_zeros: bad arguments");
    SA_CUDA(ctx, cudaSetDevice(ctx->device));
    Launch lc{ctx->stream, ctx->num_sms, 0};
    SA_CUDA(ctx, ensure(ctx->pr_state, ctx->prs_cap, (size_t)std::max<int64_t>(prune_tiles(nnz), 1) * LB_STRIDE));
    if (!ctx->pr_nnz) SA_CUDA(ctx, cudaMalloc(reinterpret_cast<void **>(&ctx->pr_nnz), sizeof(long long)));
    SA_CUDA(ctx, launch_prune(lc, d_jc, d_ir, d_pr, N, nnz, d_jc_out, d_ir_out, d_pr_out,
                              ctx->pr_state, ctx->pr_nnz));
    long long h = 0;
    SA_CUDA(ctx, cudaMemcpyAsync(&h, ctx->pr_nnz, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
    SA_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    ctx->launches = lc.launches;
    if (nnz_out) *nnz_out = h;
    return SA_OK;
}

int sa_block_histogram(sa_ctx *ctx, const int32_t *d_jj, int64_t L, int64_t step, int32_t nblocks,
                       int64_t bsize, uint64_t *d_hist) {
    if (!ctx) return SA_ERR_INVALID_ARG;
    if (L < 0 || step < 1 || nblocks < 1 || nblocks > 8192 || bsize < 1 || !d_hist || (L > 0 && !d_jj))
        return fail(ctx, SA_ERR_INVALID_ARG, "sa_block_histogram: bad arguments");
    SA_CUDA(ctx, cudaSetDevice(ctx->device));
    Launch lc{ctx->stream, ctx->num_sms, 0};
    SA_CUDA(ctx, launch_block_hist(lc, d_jj, L, step, nblocks, bsize,
                                   reinterpret_cast<unsigned long long *>(d_hist)));
    ctx->launches = lc.launches;
    return SA_OK;
}

int sa_partition(sa_ctx *ctx, const int32_t *d_ii, const int32_t *d_jj, const double *d_s,
                 int64_t s_stride, int64_t L, int32_t M, int32_t N, int32_t world, int32_t self,
                 const int32_t *h_bounds, int32_t *d_ii_out, int32_t *d_jj_out, double *d_s_out,
                 int64_t *h_counts, int64_t *bad_pos, int *bad_which) {
    if (!ctx) return SA_ERR_INVALID_ARG;
    if (L < 0 || M < 0 || N < 0 || world < 1 || world > 8 || self < -1 || self >= world ||
        !h_bounds || !h_counts ||
        (s_stride != 0 && s_stride != 1) ||
        (L > 0 && (!d_ii || !d_jj || !d_s || !d_ii_out || !d_jj_out || !d_s_out)))
        return fail(ctx, SA_ERR_INVALID_ARG, "sa_partition: bad arguments");
    SA_CUDA(ctx, cudaSetDevice(ctx->device));
    Launch lc{ctx->stream, ctx->num_sms, 0};
    const size_t nt = (size_t)std::max<int64_t>(partition_tiles(L), 1) * (size_t)world;
    SA_CUDA(ctx, ensure(ctx->pt_cnt, ctx->ptc_cap, nt));
    SA_CUDA(ctx, ensure(ctx->pt_off, ctx->pto_cap, nt));
    if (!ctx->pt_counts) SA_CUDA(ctx, cudaMalloc(reinterpret_cast<void **>(&ctx->pt_counts), 16 * sizeof(int64_t)));
    int rc = launch_init(ctx, lc, 0, 0, 0);  // error state
    if (rc) return rc;
    SA_CUDA(ctx, launch_partition(lc, d_ii, d_jj, d_s, s_stride, L, world, self, h_bounds, M,
                                  ctx->pt_cnt, ctx->pt_off, ctx->pt_counts, d_ii_out, d_jj_out,
                                  d_s_out, ctx->err));
    int64_t h[16];
    SA_CUDA(ctx, cudaMemcpyAsync(h, ctx->pt_counts, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    SA_CUDA(ctx, cudaMemcpyAsync(ctx->err_host, ctx->err, sizeof(ErrState), cudaMemcpyDeviceToHost, ctx->stream));
    SA_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    for (int r = 0; r < world; ++r) h_counts[r] = h[r];
    ctx->launches = lc.launches;
    ErrState e = *ctx->err_host;  // over_m / over_n: an index beyond the global dimensions
    e.nnz = 0;
    return decode(ctx, e, nullptr, bad_pos, bad_which);
}

}  // extern "C"
