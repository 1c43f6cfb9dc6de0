// Does a warp issuing bulk copies (cp.async.bulk, 24 KB every ~2k cycles) slow an LDS-latency
// chain running on the SAME SM sub-partition (warp 0 + warp 4) vs a different one (warp 0 + 1)?
#include <cstdio>
__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ long long clk() { long long t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)); return t; }
__global__ void k(const unsigned char *src, int copier, int bytes, int gap, long long *out, int *sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    unsigned long long *mb = reinterpret_cast<unsigned long long *>(sm);
    int *chain = reinterpret_cast<int *>(sm + 128);            // 4096 ints
    unsigned char *buf = sm + 128 + 16384;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) chain[i] = (i * 97 + 13) & 4095;
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(mb)) : "memory");
    __syncthreads();
    __shared__ volatile int stop;
    if (threadIdx.x == 0) stop = 0;
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (w == copier && lane == 0) {
        unsigned ph = 0;
        long long issued = 0;
        while (!stop) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(mb)), "r"(bytes) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su32(buf)), "l"(src + (issued % 64) * bytes), "r"(bytes), "r"(su32(mb)) : "memory");
            unsigned ok = 0;
            while (!ok) asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(su32(mb)), "r"(ph) : "memory");
            ph ^= 1;
            ++issued;
            const long long t = clk();
            while (clk() - t < gap) __nanosleep(64);
        }
        out[1] = issued;
    }
    if (w == 0) {
        int p = lane;
        const long long t0 = clk();
        for (int i = 0; i < 20000; ++i) p = chain[(p + i) & 4095];
        const long long t1 = clk();
        if (lane == 0) { out[0] = (t1 - t0) / 20000; stop = 1; }
        sink[lane] = p;
    }
}
int main() {
    unsigned char *src; long long *d, h[2]; int *sink;
    cudaMalloc(&src, 64 << 20); cudaMalloc(&d, 16); cudaMalloc(&sink, 128);
    const int bytes = 24576;
    const size_t smem = 128 + 16384 + bytes;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int copier : {-1, 1, 4}) for (int gap : {0, 2000}) {
        k<<<1, 256, smem>>>(src, copier, bytes, gap, d, sink);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("copier warp %2d (%s) gap %4d: LDS chain %lld cycles per load, copies %lld\n", copier,
               copier < 0 ? "none" : copier % 4 == 0 ? "same sub-partition" : "other sub-partition", gap, h[0], copier < 0 ? 0 : h[1]);
    }
    return 0;
}
