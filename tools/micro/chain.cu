// Synthetic level chain on one CTA: L levels x 22 rows, each row 21 early + 3 mid + 3 late
// columns (sources in levels <= l-3, l-2, l-1), SELL layout in shared memory, per-level
// mbarriers, 3 level teams -- the k_trsv_lvl scheme without TMA ring / cluster / pushes.
// Prints cycles per level.  mode 0: mbarrier teams; mode 1: one warp does every level
// (no cross-warp hop, __syncwarp only).
#include <cstdio>
__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ long long clk() { long long t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)); return t; }
__device__ __forceinline__ void mwait(unsigned a) {
    unsigned ok = 0;
    while (!ok)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(a) : "memory");
}
constexpr int L = 200, NE = 21, NM = 3, NL = 3, NC = NE + NM + NL, ROWS = 22;
__global__ void k(int mode, long long *out, double *sink) {
    extern __shared__ __align__(16) unsigned char sm[];
    unsigned long long *mb = reinterpret_cast<unsigned long long *>(sm);
    double *xh = reinterpret_cast<double *>(sm + 8 * L) + 6 * 32;   // 6 zero levels below level 0
    int *code = reinterpret_cast<int *>(sm + 8 * L + 8 * (L + 6) * 32);
    double *val = reinterpret_cast<double *>(sm + 8 * L + 8 * (L + 6) * 32 + 4 * NC * 32);
    for (int i = threadIdx.x; i < (L + 6) * 32; i += blockDim.x) xh[i - 6 * 32] = i < 6 * 32 ? 0.0 : 1.0;
    for (int i = threadIdx.x; i < NC * 32; i += blockDim.x) {   // one template level: code = d*32 - row
        const int c = i / 32, lane = i % 32;
        const int d = c < NE ? 3 + (c % 3) : c < NE + NM ? 2 : 1;
        code[i] = d * 32 - ((lane * 7 + c * 5) % ROWS);
        val[i] = 1e-3;
    }
    for (int l = threadIdx.x; l < L; l += blockDim.x)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&mb[l])), "r"(ROWS) : "memory");
    __syncthreads();
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    long long t0 = clk();
    int waited = 0;
    for (int l = 0; l < L; ++l) {
        if (mode == 0 && l % 3 != wid) continue;
        if (mode == 1 && wid != 0) break;
        const int base = lane;
        const double *xl = xh + l * 32;   // x of source (l - d, row) at xl[-code]
        if (mode == 0) for (; waited < l - 2; ++waited) mwait(su32(&mb[waited]));
        double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
        int e = base, kq = 0;
        for (; kq + 8 <= NE; kq += 8, e += 256) {
            int cd[8]; double v[8], xv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) { cd[u] = code[e + 32 * u]; v[u] = val[e + 32 * u]; }
#pragma unroll
            for (int u = 0; u < 8; ++u) xv[u] = xl[-cd[u]];
            s0 = fma(v[0], xv[0], s0); s1 = fma(v[1], xv[1], s1); s2 = fma(v[2], xv[2], s2); s3 = fma(v[3], xv[3], s3);
            s0 = fma(v[4], xv[4], s0); s1 = fma(v[5], xv[5], s1); s2 = fma(v[6], xv[6], s2); s3 = fma(v[7], xv[7], s3);
        }
        for (; kq < NE; ++kq, e += 32) s0 = fma(val[e], xl[-code[e]], s0);
        int mc[NM], lc[NL]; double mv[NM], lv[NL];
#pragma unroll
        for (int u = 0; u < NM; ++u) { mc[u] = code[e + 32 * u]; mv[u] = val[e + 32 * u]; }
#pragma unroll
        for (int u = 0; u < NL; ++u) { lc[u] = code[e + 32 * (NM + u)]; lv[u] = val[e + 32 * (NM + u)]; }
        double sum = (s0 + s1) + (s2 + s3);
        if (mode == 0 && waited < l - 1) { mwait(su32(&mb[l - 2])); waited = l - 1; }
        else if (mode == 1) __syncwarp();
#pragma unroll
        for (int u = 0; u < NM; ++u) sum = fma(mv[u], xl[-mc[u]], sum);
        if (mode == 0 && waited < l) { mwait(su32(&mb[l - 1])); waited = l; }
        else if (mode == 1) __syncwarp();
        double t0_ = 0, t1_ = 0;
#pragma unroll
        for (int u = 0; u < NL; ++u) { if (u & 1) t1_ = fma(lv[u], xl[-lc[u]], t1_); else t0_ = fma(lv[u], xl[-lc[u]], t0_); }
        sum += t0_ + t1_;
        if (lane < ROWS) xh[l * 32 + lane] = (1.0 - sum) * 0.5;
        __syncwarp();
        if (mode == 0 && lane == 0)
            asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mb[l])), "r"(ROWS) : "memory");
    }
    long long t1 = clk();
    if (threadIdx.x == 0 || (mode == 0 && wid == (L - 1) % 3 && lane == 0)) out[mode * 2 + (threadIdx.x != 0)] = t1 - t0;
    if (threadIdx.x == 0) sink[0] = xh[(L - 1) * 32];
}
int main() {
    long long *d, h[4] = {0};
    double *sink;
    cudaMalloc(&d, 32); cudaMalloc(&sink, 64);
    cudaMemset(d, 0, 32);
    size_t smem = 8 * L + 8 * (L + 6) * 32 + 12 * NC * 32 + 64;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<1, 96, smem>>>(0, d, sink);
    k<<<1, 32, smem>>>(1, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("smem %zu B: mbarrier teams %lld cycles/level (last team %lld) | single warp %lld cycles/level\n", smem,
           h[0] / L, h[1] / L, h[2] / L);
    return 0;
}
