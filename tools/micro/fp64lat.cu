// Latency probes (cycles) for the triangular-sweep critical path on sm_100a:
// DFMA / DADD / DMUL dependent chains, FP64 shuffle round, LDS round trip,
// mbarrier arrive (warp A) -> try_wait wake-up (warp B) ping-pong, STS -> volatile-LDS poll ping-pong.
#include <cstdio>
__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ long long clk() { long long t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)); return t; }

__global__ void k_alu(double a, double b, int iters, long long *out, double *sink) {
    __shared__ double sh[64];
    __shared__ int idx[64];
    if (threadIdx.x < 64) { sh[threadIdx.x] = 1.0 + threadIdx.x; idx[threadIdx.x] = (threadIdx.x * 7) & 63; }
    __syncthreads();
    if (threadIdx.x >= 32) return;
    double x = a;
    long long t0 = clk();
    for (int i = 0; i < iters; ++i) x = fma(x, b, a);
    long long t1 = clk();
    double y = a;
    for (int i = 0; i < iters; ++i) y = y + b;
    long long t2 = clk();
    double z = x + y;
    for (int i = 0; i < iters; ++i) z += __shfl_xor_sync(0xffffffffu, z, 1);
    long long t3 = clk();
    int p = threadIdx.x;
    for (int i = 0; i < iters; ++i) p = idx[p];
    long long t4 = clk();
    double w = z;
    for (int i = 0; i < iters; ++i) w = w * b;
    long long t5 = clk();
    // LDS-dependent gather + DFMA (the sweep's code -> xh -> fma chain)
    double s = 0; int q = p & 63;
    for (int i = 0; i < iters; ++i) { s = fma(sh[idx[q]], b, s); q = (q + (int)(s > 1e300)) & 63; }
    long long t6 = clk();
    if (threadIdx.x == 0) {
        out[0] = (t1 - t0) / iters; out[1] = (t2 - t1) / iters; out[2] = (t3 - t2) / iters;
        out[3] = (t4 - t3) / iters; out[4] = (t5 - t4) / iters; out[5] = (t6 - t5) / iters;
    }
    sink[threadIdx.x] = x + y + z + w + p + s;
}

// warp 0 and warp 1 ping-pong through per-step mbarriers (arrive / try_wait) or polled STS
__global__ void k_pp(int mode, int iters, long long *out) {
    __shared__ __align__(8) unsigned long long mb[512];
    __shared__ __align__(8) volatile double v[512];
    if (threadIdx.x == 0)
        for (int i = 0; i < iters; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mb[i])) : "memory");
            v[i] = -1.0;
        }
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (w > 1) {   // bystander warps (mode 2: spin on shared memory like a polling sweep)
        if (mode == 2) { double acc = 0; for (int i = 0; i < 20000; ++i) acc += v[(lane * 13 + i) & 511]; if (acc == 12345.0) out[9] = 1; }
        return;
    }
    long long t0 = clk();
    for (int i = 0; i < iters; ++i) {
        const bool mine = (i & 1) == w;
        if (mine) {
            if (mode == 0) { if (lane == 0) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su32(&mb[i])) : "memory"); }
            else { if (lane == 0) v[i] = 1.0; }
        } else {
            if (mode == 0) {
                asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}" ::"r"(su32(&mb[i])) : "memory");
            } else {
                while (__any_sync(0xffffffffu, v[i] < 0.0)) {}
            }
        }
        __syncwarp();
    }
    long long t1 = clk();
    if (threadIdx.x == 0) out[6 + (mode > 0)] = (t1 - t0) / iters;
}

int main() {
    long long *d, h[10] = {0};
    double *sink;
    cudaMalloc(&d, 80); cudaMalloc(&sink, 256 * 8);
    cudaMemset(d, 0, 80);
    k_alu<<<1, 64>>>(1.0000001, 0.9999999, 1000, d, sink);
    k_pp<<<1, 64>>>(0, 500, d);
    k_pp<<<1, 64>>>(1, 500, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, 80, cudaMemcpyDeviceToHost);
    printf("latency cycles: DFMA %lld | DADD %lld | SHFL.f64+DADD %lld | LDS (dep) %lld | DMUL %lld | LDS idx->LDS x->DFMA %lld\n",
           h[0], h[1], h[2], h[3], h[4], h[5]);
    printf("one-way warp hop: mbarrier arrive->try_wait %lld | STS->polled LDS %lld\n", h[6], h[7]);
    k_pp<<<1, 1024>>>(1, 500, d);
    k_pp<<<1, 1024>>>(0, 500, d);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 80, cudaMemcpyDeviceToHost);
    printf("with 30 idle warps: mbarrier %lld | STS->poll %lld\n", h[6], h[7]);
    k_pp<<<1, 1024>>>(2, 500, d);   // mode 2 = poll hop with 30 warps spinning on shared memory
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 80, cudaMemcpyDeviceToHost);
    printf("with 30 smem-spinning warps: STS->poll %lld\n", h[7]);
    return 0;
}
