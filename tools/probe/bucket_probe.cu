// bucket_probe.cu -- design probe for the column-block ("bucket") partition of
// shuffled input (cfg4 shape: L = 5e8, M = N = 1e7).  Times, on synthetic
// random (i, j):
//   copy      16 B read + 16 B write per triplet, coalesced (the floor)
//   count     per-CTA shared histogram of buckets (jj only)
//   gatomic   bucket scatter through global cursors (warp-aggregated atomics)
//   matrix    bucket scatter through per-CTA offsets (count matrix), shared cursors
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bucket_probe bucket_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t hsh(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return (uint32_t)x;
}
__global__ void k_gen(int32_t *ii, int32_t *jj, double *s, int64_t L, int M, int N) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < L; t += (int64_t)gridDim.x * blockDim.x) {
        ii[t] = 1 + (int)(hsh(2 * t) % (uint32_t)M);
        jj[t] = 1 + (int)(hsh(2 * t + 1) % (uint32_t)N);
        s[t] = (double)(hsh(3 * t) & 0xffff) - 30000.0;
    }
}
__global__ void k_copy(const int4 *a, const int4 *b, const double2 *c, int4 *x, int4 *y, double2 *z, int64_t n4) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n4; t += (int64_t)gridDim.x * blockDim.x) {
        x[t] = a[t];
        y[t] = b[t];
        z[2 * t] = c[2 * t];
        z[2 * t + 1] = c[2 * t + 1];
    }
}
constexpr int NT = 512;
// per-CTA histogram of buckets over the CTA's contiguous range -> cnt[g*B + b]
__global__ void __launch_bounds__(NT) k_count(const int32_t *jj, int64_t L, int shift, int B, uint32_t *cnt) {
    extern __shared__ uint32_t h[];
    for (int k = threadIdx.x; k < B; k += NT) h[k] = 0;
    __syncthreads();
    const int64_t per = (L + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * per, hi = min(L, lo + per);
    const int4 *j4 = reinterpret_cast<const int4 *>(jj);
    for (int64_t q = lo / 4 + threadIdx.x; q < hi / 4; q += NT) {
        int4 v = __ldg(j4 + q);
        atomicAdd(&h[(v.x - 1) >> shift], 1u);
        atomicAdd(&h[(v.y - 1) >> shift], 1u);
        atomicAdd(&h[(v.z - 1) >> shift], 1u);
        atomicAdd(&h[(v.w - 1) >> shift], 1u);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < B; k += NT) cnt[(int64_t)blockIdx.x * B + k] = h[k];
}
// column-wise exclusive scan of cnt (G x B) + bucket totals
__global__ void k_colscan(uint32_t *cnt, int G, int B, uint32_t *tot) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    uint32_t run = 0;
    for (int g = 0; g < G; ++g) {
        uint32_t v = cnt[(int64_t)g * B + b];
        cnt[(int64_t)g * B + b] = run;
        run += v;
    }
    tot[b] = run;
}
__global__ void k_addbase(uint32_t *cnt, int G, int B, const uint32_t *base) {
    int64_t n = (int64_t)G * B;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        cnt[t] += base[t % B];
}
__device__ __forceinline__ unsigned lanemask_lt() { unsigned m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }

// matrix scatter: shared cursors initialised from the CTA's offsets row
__global__ void __launch_bounds__(NT) k_mscatter(const int32_t *ii, const int32_t *jj, const double *s, int64_t L,
                                                 int shift, int B, const uint32_t *off, int rb, int pb,
                                                 unsigned long long *key, double *val) {
    extern __shared__ uint32_t cur[];
    for (int k = threadIdx.x; k < B; k += NT) cur[k] = off[(int64_t)blockIdx.x * B + k];
    __syncthreads();
    const int64_t per = (L + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * per, hi = min(L, lo + per);
    const int4 *i4 = reinterpret_cast<const int4 *>(ii);
    const int4 *j4 = reinterpret_cast<const int4 *>(jj);
    const double2 *s2 = reinterpret_cast<const double2 *>(s);
    const unsigned long long cmask = (1ull << shift) - 1;
    for (int64_t q = lo / 4 + threadIdx.x; q < hi / 4; q += NT) {
        int4 vi = __ldg(i4 + q), vj = __ldg(j4 + q);
        double2 sa = __ldg(s2 + 2 * q), sb = __ldg(s2 + 2 * q + 1);
        int I[4] = {vi.x, vi.y, vi.z, vi.w}, J[4] = {vj.x, vj.y, vj.z, vj.w};
        double S[4] = {sa.x, sa.y, sb.x, sb.y};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = J[u] - 1;
            const uint32_t slot = atomicAdd(&cur[c >> shift], 1u);
            key[slot] = (((unsigned long long)c & cmask) << (rb + pb)) | ((unsigned long long)(I[u] - 1) << pb) | (unsigned long long)(4 * q + u);
            val[slot] = S[u];
        }
    }
}
// global-cursor scatter: warp-aggregated global atomics
template <int PAD>
__global__ void __launch_bounds__(256) k_gscatter(const int32_t *ii, const int32_t *jj, const double *s, int64_t L,
                                                  int shift, uint32_t *gcur, int rb, int pb,
                                                  unsigned long long *key, double *val) {
    const int4 *i4 = reinterpret_cast<const int4 *>(ii);
    const int4 *j4 = reinterpret_cast<const int4 *>(jj);
    const double2 *s2 = reinterpret_cast<const double2 *>(s);
    const unsigned long long cmask = (1ull << shift) - 1;
    const unsigned lt = lanemask_lt();
    const int lane = threadIdx.x & 31;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < L / 4; q += (int64_t)gridDim.x * blockDim.x) {
        int4 vi = __ldg(i4 + q), vj = __ldg(j4 + q);
        double2 sa = __ldg(s2 + 2 * q), sb = __ldg(s2 + 2 * q + 1);
        int I[4] = {vi.x, vi.y, vi.z, vi.w}, J[4] = {vj.x, vj.y, vj.z, vj.w};
        double S[4] = {sa.x, sa.y, sb.x, sb.y};
        uint32_t base[4];
        unsigned pe[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int b = (J[u] - 1) >> shift;
            pe[u] = __match_any_sync(0xffffffffu, b);
            const int leader = __ffs(pe[u]) - 1;
            uint32_t v = 0;
            if (lane == leader) v = atomicAdd(&gcur[(int64_t)b * PAD], (uint32_t)__popc(pe[u]));
            base[u] = __shfl_sync(0xffffffffu, v, leader);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = J[u] - 1;
            const uint32_t slot = base[u] + __popc(pe[u] & lt);
            key[slot] = (((unsigned long long)c & cmask) << (rb + pb)) | ((unsigned long long)(I[u] - 1) << pb) | (unsigned long long)(4 * q + u);
            val[slot] = S[u];
        }
    }
}
__global__ void k_setcur(uint32_t *gcur, const uint32_t *base, int B, int pad) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < B) gcur[(int64_t)b * pad] = base[b];
}
// global reductions to per-column counters (the current colcount on shuffled input)
__global__ void k_colred(const int32_t *jj, int64_t L, uint32_t *cnt) {
    const int4 *j4 = reinterpret_cast<const int4 *>(jj);
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < L / 4; q += (int64_t)gridDim.x * blockDim.x) {
        int4 v = __ldg(j4 + q);
        atomicAdd(&cnt[v.x - 1], 1u); atomicAdd(&cnt[v.y - 1], 1u);
        atomicAdd(&cnt[v.z - 1], 1u); atomicAdd(&cnt[v.w - 1], 1u);
    }
}


// bucket count by global reductions (one RED per triplet, no shared histogram)
__global__ void k_bred(const int32_t *jj, int64_t L, int shift, uint32_t *cnt) {
    const int4 *j4 = reinterpret_cast<const int4 *>(jj);
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < L / 4; q += (int64_t)gridDim.x * blockDim.x) {
        int4 v = __ldcs(j4 + q);
        atomicAdd(&cnt[(v.x - 1) >> shift], 1u); atomicAdd(&cnt[(v.y - 1) >> shift], 1u);
        atomicAdd(&cnt[(v.z - 1) >> shift], 1u); atomicAdd(&cnt[(v.w - 1) >> shift], 1u);
    }
}
// record scatter: one returning global atomic per triplet (no aggregation), one
// 16-byte record {local key, position, value} per triplet; Q quads per thread
template <int Q>
__global__ void __launch_bounds__(256) k_rscatter(const int32_t *ii, const int32_t *jj, const double *s, int64_t L,
                                                  int shift, uint32_t *gcur, int rb, uint4 *rec) {
    const int4 *i4 = reinterpret_cast<const int4 *>(ii);
    const int4 *j4 = reinterpret_cast<const int4 *>(jj);
    const double2 *s2 = reinterpret_cast<const double2 *>(s);
    const int64_t q0 = ((int64_t)blockIdx.x * 256) * Q + threadIdx.x;
    int I[4 * Q], J[4 * Q];
    double S[4 * Q];
#pragma unroll
    for (int u = 0; u < Q; ++u) {
        const int64_t q = q0 + u * 256;
        int4 vi = make_int4(1, 1, 1, 1), vj = make_int4(0, 0, 0, 0);
        double2 sa = make_double2(0, 0), sb = sa;
        if (q < L / 4) { vi = __ldcs(i4 + q); vj = __ldcs(j4 + q); sa = __ldcs(s2 + 2 * q); sb = __ldcs(s2 + 2 * q + 1); }
        I[4*u] = vi.x; I[4*u+1] = vi.y; I[4*u+2] = vi.z; I[4*u+3] = vi.w;
        J[4*u] = vj.x; J[4*u+1] = vj.y; J[4*u+2] = vj.z; J[4*u+3] = vj.w;
        S[4*u] = sa.x; S[4*u+1] = sa.y; S[4*u+2] = sb.x; S[4*u+3] = sb.y;
    }
    uint32_t slot[4 * Q];
#pragma unroll
    for (int k = 0; k < 4 * Q; ++k) slot[k] = J[k] > 0 ? atomicAdd(&gcur[(J[k] - 1) >> shift], 1u) : 0u;
    const uint32_t cm = (1u << shift) - 1u;
#pragma unroll
    for (int k = 0; k < 4 * Q; ++k) {
        if (J[k] <= 0) continue;
        const int64_t pos = 4 * (q0 + (k >> 2) * 256) + (k & 3);
        const unsigned long long vb = (unsigned long long)__double_as_longlong(S[k]);
        rec[slot[k]] = make_uint4((((uint32_t)(J[k] - 1) & cm) << rb) | (uint32_t)(I[k] - 1), (uint32_t)pos,
                                  (uint32_t)vb, (uint32_t)(vb >> 32));
    }
}

int main(int argc, char **argv) {
    const int64_t L = argc > 1 ? atoll(argv[1]) : 500000000LL;
    const int M = 10000000, N = 10000000;
    const int shift = argc > 2 ? atoi(argv[2]) : 10;
    const int B = ((N - 1) >> shift) + 1;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    int32_t *ii, *jj; double *s, *val; unsigned long long *key;
    int4 *x, *y; double2 *z;
    CK(cudaMalloc(&ii, L * 4)); CK(cudaMalloc(&jj, L * 4)); CK(cudaMalloc(&s, L * 8));
    CK(cudaMalloc(&key, L * 8)); CK(cudaMalloc(&val, L * 8));
    k_gen<<<sms * 8, 256>>>(ii, jj, s, L, M, N);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto tm = [&](const char *name, auto fn, double bytes) {
        fn(); CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        const int R = 3;
        for (int r = 0; r < R; ++r) fn();
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= R;
        printf("%-28s %9.3f ms  %7.1f GB/s\n", name, ms, bytes / (ms * 1e-3) / 1e9);
    };
    x = reinterpret_cast<int4 *>(key); y = reinterpret_cast<int4 *>(val);
    int32_t *cp_j; CK(cudaMalloc(&cp_j, L * 4)); z = nullptr;
    double2 *zz; CK(cudaMalloc(&zz, L * 8));
    tm("copy 16B/16B", [&] { k_copy<<<sms * 4, 512>>>((const int4 *)ii, (const int4 *)jj, (const double2 *)s, x, (int4 *)cp_j, zz, L / 4); }, 32.0 * L);
    CK(cudaFree(cp_j)); CK(cudaFree(zz));

    {
        uint32_t *bc, *gcur; uint4 *rec;
        CK(cudaMalloc(&bc, (size_t)B * 4)); CK(cudaMalloc(&gcur, (size_t)B * 4)); CK(cudaMalloc(&rec, (size_t)L * 16));
        char nm[64];
        for (int gm : {8, 32}) {
            snprintf(nm, 64, "bucket RED count grid=%dx", gm);
            tm(nm, [&] { cudaMemsetAsync(bc, 0, (size_t)B * 4); k_bred<<<sms * gm, 256>>>(jj, L, shift, bc); }, 4.0 * L);
        }
        std::vector<uint32_t> h(B);
        CK(cudaMemcpy(h.data(), bc, B * 4, cudaMemcpyDeviceToHost));
        uint32_t r = 0, mx = 0;
        for (int b = 0; b < B; ++b) { uint32_t v = h[b]; h[b] = r; r += v; mx = v > mx ? v : mx; }
        printf("   B=%d max bucket %u\n", B, mx);
        uint32_t *base; CK(cudaMalloc(&base, (size_t)B * 4));
        CK(cudaMemcpy(base, h.data(), B * 4, cudaMemcpyHostToDevice));
        tm("record scatter Q=1", [&] { cudaMemcpyAsync(gcur, base, B * 4, cudaMemcpyDeviceToDevice);
             k_rscatter<1><<<(unsigned)((L / 4 + 255) / 256), 256>>>(ii, jj, s, L, shift, gcur, 24, rec); }, 32.0 * L);
        tm("record scatter Q=2", [&] { cudaMemcpyAsync(gcur, base, B * 4, cudaMemcpyDeviceToDevice);
             k_rscatter<2><<<(unsigned)((L / 4 + 511) / 512), 256>>>(ii, jj, s, L, shift, gcur, 24, rec); }, 32.0 * L);
        tm("record scatter Q=4", [&] { cudaMemcpyAsync(gcur, base, B * 4, cudaMemcpyDeviceToDevice);
             k_rscatter<4><<<(unsigned)((L / 4 + 1023) / 1024), 256>>>(ii, jj, s, L, shift, gcur, 24, rec); }, 32.0 * L);
        CK(cudaFree(bc)); CK(cudaFree(gcur)); CK(cudaFree(rec)); CK(cudaFree(base));
    }
    if (argc > 3) { printf("done\n"); return 0; }
    const int rb = 24, pb = 29;
    for (int gmul : {1}) {
        const int G = sms * gmul;
        uint32_t *cnt, *tot, *base;
        CK(cudaMalloc(&cnt, (size_t)G * B * 4)); CK(cudaMalloc(&tot, B * 4)); CK(cudaMalloc(&base, B * 4));
        CK(cudaFuncSetAttribute(k_count, cudaFuncAttributeMaxDynamicSharedMemorySize, B * 4));
        CK(cudaFuncSetAttribute(k_mscatter, cudaFuncAttributeMaxDynamicSharedMemorySize, B * 4));
        char nm[64];
        snprintf(nm, 64, "count G=%d", G);
        tm(nm, [&] { k_count<<<G, NT, B * 4>>>(jj, L, shift, B, cnt); }, 4.0 * L);
        k_colscan<<<(B + 255) / 256, 256>>>(cnt, G, B, tot);
        std::vector<uint32_t> h(B);
        CK(cudaMemcpy(h.data(), tot, B * 4, cudaMemcpyDeviceToHost));
        uint32_t r = 0, mx = 0;
        for (int b = 0; b < B; ++b) { uint32_t v = h[b]; h[b] = r; r += v; mx = v > mx ? v : mx; }
        CK(cudaMemcpy(base, h.data(), B * 4, cudaMemcpyHostToDevice));
        k_addbase<<<sms * 4, 256>>>(cnt, G, B, base);
        snprintf(nm, 64, "colscan G=%d", G);
        tm(nm, [&] { k_colscan<<<(B + 255) / 256, 256>>>(cnt, G, B, tot); }, 8.0 * G * B);
        // restore offsets (colscan above re-scanned the offsets)
        k_count<<<G, NT, B * 4>>>(jj, L, shift, B, cnt);
        k_colscan<<<(B + 255) / 256, 256>>>(cnt, G, B, tot);
        k_addbase<<<sms * 4, 256>>>(cnt, G, B, base);
        CK(cudaDeviceSynchronize());
        snprintf(nm, 64, "matrix scatter G=%d", G);
        tm(nm, [&] { k_mscatter<<<G, NT, B * 4>>>(ii, jj, s, L, shift, B, cnt, rb, pb, key, val); }, 32.0 * L);
        if (gmul == 1) printf("   B=%d max bucket %u (%.1f KB at 16 B)\n", B, mx, mx * 16 / 1024.0);
        if (gmul == 1) {
            uint32_t *gcur; CK(cudaMalloc(&gcur, (size_t)B * 4 * 32));
            for (int gm2 : {8, 16}) {
                snprintf(nm, 64, "gatomic scatter grid=%dx", gm2);
                tm(nm, [&] { k_setcur<<<(B + 255) / 256, 256>>>(gcur, base, B, 1);
                             k_gscatter<1><<<sms * gm2, 256>>>(ii, jj, s, L, shift, gcur, rb, pb, key, val); }, 32.0 * L);
                snprintf(nm, 64, "gatomic pad8 grid=%dx", gm2);
                tm(nm, [&] { k_setcur<<<(B + 255) / 256, 256>>>(gcur, base, B, 8);
                             k_gscatter<8><<<sms * gm2, 256>>>(ii, jj, s, L, shift, gcur, rb, pb, key, val); }, 32.0 * L);
                snprintf(nm, 64, "gatomic pad32 grid=%dx", gm2);
                tm(nm, [&] { k_setcur<<<(B + 255) / 256, 256>>>(gcur, base, B, 32);
                             k_gscatter<32><<<sms * gm2, 256>>>(ii, jj, s, L, shift, gcur, rb, pb, key, val); }, 32.0 * L);
            }
            CK(cudaFree(gcur));
        }
        CK(cudaFree(cnt)); CK(cudaFree(tot)); CK(cudaFree(base));
    }
    uint32_t *cc; CK(cudaMalloc(&cc, (size_t)N * 4));
    tm("colred (global RED per triplet)", [&] { cudaMemsetAsync(cc, 0, (size_t)N * 4); k_colred<<<sms * 8, 256>>>(jj, L, cc); }, 4.0 * L);
    CK(cudaDeviceSynchronize());
    printf("done\n");
    return 0;
}
