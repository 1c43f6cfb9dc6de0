// Cycles for one warp's SELL-chunk dot product (27 columns, conflict-free code/val, gathered x)
// in isolation -- the k_trsv_lvl early loop without any synchronisation around it.
#include <cstdio>
__device__ __forceinline__ long long clk() { long long t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)); return t; }
__global__ void k(int ncol, int reps, long long *out, double *sink) {
    extern __shared__ __align__(16) unsigned char sm[];
    double *xh = reinterpret_cast<double *>(sm);                  // 8192 doubles
    int *code = reinterpret_cast<int *>(sm + 8192 * 8);            // ncol*32
    double *val = reinterpret_cast<double *>(sm + 8192 * 8 + ncol * 32 * 4);
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) xh[i] = 1.0 + (i & 7) * 1e-3;
    for (int i = threadIdx.x; i < ncol * 32; i += blockDim.x) {
        const int lane = i & 31, k = i >> 5;
        code[i] = (lane * 37 + k * 301 + ((k * lane) & 15)) & 8191;
        val[i] = 0.25;
    }
    __syncthreads();
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    double tot = 0;
    long long best = 1ll << 60, sum_t = 0;
    for (int r = 0; r < reps; ++r) {
        long long t0 = clk();
        double s = 0.0;
        int e = lane;
#pragma unroll 4
        for (int k = 0; k < ncol; ++k, e += 32) s += val[e] * xh[code[e]];
        long long sink_dep = __double_as_longlong(s) & 1;   // consume s before the stop time
        long long t1 = clk() + sink_dep * 0;
        if (s == 12345.0) sink[0] = s;
        tot += s;
        best = min(best, t1 - t0);
        sum_t += t1 - t0;
    }
    if (lane == 0) { out[0] = best; out[1] = sum_t / reps; }
    sink[1 + lane] = tot;
}
int main() {
    long long *d, h[2];
    double *sink;
    cudaMalloc(&d, 16); cudaMalloc(&sink, 64 * 8);
    for (int ncol : {4, 8, 16, 27, 32}) {
        size_t smem = 8192 * 8 + ncol * 32 * 12 + 64;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<1, 160, smem>>>(ncol, 200, d, sink);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("ncol %2d: best %lld cycles, mean %lld  (%.1f per column)\n", ncol, h[0], h[1], (double)h[1] / ncol);
    }
    return 0;
}
