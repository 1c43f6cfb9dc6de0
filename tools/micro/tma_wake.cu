// Wake-up latency of a warp waiting on an mbarrier whose phase is completed by a bulk copy
// (complete_tx from the async proxy): try_wait loop vs test_wait polling.  The issuing warp
// records when the copy completes (its own test_wait spin); the waiter records when it woke.
#include <cstdio>
__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ long long gclk() { long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ long long clk() { long long t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)); return t; }
__global__ void k(const unsigned char *src, int bytes, int mode, long long *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    unsigned long long *mb = reinterpret_cast<unsigned long long *>(sm);
    unsigned char *buf = sm + 128;
    __shared__ volatile long long t_done[64], t_wake[64];
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(mb)) : "memory");
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int it = 0; it < 64; ++it) {
        const unsigned ph = it & 1;
        if (w == 0 && lane == 0) {
            const long long t = clk();
            while (clk() - t < 3000) {}
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(mb)), "r"(bytes) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su32(buf)), "l"(src + (it % 16) * bytes), "r"(bytes), "r"(su32(mb)) : "memory");
            unsigned ok = 0;
            while (!ok) asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(su32(mb)), "r"(ph) : "memory");
            t_done[it] = clk();
        }
        if (w == 1) {
            unsigned ok = 0;
            if (mode == 0)
                while (!ok) asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(su32(mb)), "r"(ph) : "memory");
            else
                while (!ok) asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(su32(mb)), "r"(ph) : "memory");
            if (lane == 0) t_wake[it] = clk();
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        long long s = 0, mx = 0;
        for (int it = 0; it < 64; ++it) { long long d = t_wake[it] - t_done[it]; s += d; mx = d > mx ? d : mx; }
        out[0] = s / 64; out[1] = mx;
    }
}
int main() {
    unsigned char *src; long long *d, h[2];
    cudaMalloc(&src, 16 << 20); cudaMalloc(&d, 16);
    for (int bytes : {4096, 24576}) for (int mode = 0; mode < 2; ++mode) {
        const size_t smem = 128 + bytes;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<1, 64, smem>>>(src, bytes, mode, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("bytes %5d %s: waiter wakes %lld cycles (max %lld) after the copy completed\n", bytes,
               mode == 0 ? "try_wait " : "test_wait", h[0], h[1]);
    }
    return 0;
}
