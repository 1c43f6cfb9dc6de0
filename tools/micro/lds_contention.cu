// Does an LDS-gather dot product (the sweep's row loop) slow down while other warps of the
// CTA sit in mbarrier try_wait loops?  Cycles per entry for warp 0, 25-entry rows, G=1.
#include <cstdio>
__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ long long clk() { long long t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)); return t; }

__global__ void k(int mode, int rows, long long *out, double *sink) {
    extern __shared__ __align__(16) unsigned char sm[];
    unsigned long long *mb = reinterpret_cast<unsigned long long *>(sm);
    double *xh = reinterpret_cast<double *>(sm + 64);          // 4096 doubles
    int *code = reinterpret_cast<int *>(sm + 64 + 4096 * 8);     // rows*25 ints
    double *val = reinterpret_cast<double *>(sm + 64 + 4096 * 8 + ((rows * 25 * 4 + 15) & ~15));
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) xh[i] = 1.0 + (i & 7);
    for (int i = threadIdx.x; i < rows * 25; i += blockDim.x) { code[i] = (i * 2654435761u) >> 20 & 4095; val[i] = 0.5; }
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(mb)) : "memory");
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (w > 0) {
        if (mode == 1) {   // sleep on the mbarrier until warp 0 is done
            unsigned ok = 0;
            while (!ok)
                asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
                             : "=r"(ok) : "r"(su32(mb)) : "memory");
        } else if (mode == 2) {   // spin on a volatile shared flag
            volatile double *f = xh;
            while (f[4095] > 0.0) {}
        }
        return;
    }
    double s = 0;
    long long t0 = clk();
    for (int r = lane; r < rows; r += 32) {
        const int e0 = r * 25;
#pragma unroll 4
        for (int e = e0; e < e0 + 25; ++e) s += val[e] * xh[code[e]];
    }
    if (s == 1234.5) sink[0] = s;
    long long t1 = clk();
    if (lane == 0) out[mode] = (t1 - t0) / ((rows + 31) / 32 * 25);
    __syncwarp();
    if (lane == 0) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(mb)) : "memory");
        xh[4095] = -1.0;
    }
    sink[1 + lane] = s;
}

int main() {
    long long *d, h[3];
    double *sink;
    cudaMalloc(&d, 24); cudaMalloc(&sink, 64 * 8);
    int rows = 256;
    size_t smem = 64 + 4096 * 8 + rows * 25 * 12 + 64;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int nthr : {32, 160, 1024}) {
        for (int mode = 0; mode < 3; ++mode) k<<<1, nthr, smem>>>(mode, rows, d, sink);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
        printf("threads %4d: cycles/entry (per warp-row-step) idle-exit %lld | try_wait sleepers %lld | volatile spinners %lld\n", nthr, h[0], h[1], h[2]);
    }
    return 0;
}
