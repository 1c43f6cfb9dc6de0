// Per-SM bulk-copy (cp.async.bulk global -> shared) throughput and latency: one CTA streams a
// buffer through a 2 x `chunk` ring; also with 16 CTAs at once.  Bytes per SM cycle.
#include <cstdio>
__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ long long clk() { long long t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)); return t; }
__global__ void k(const unsigned char *src, size_t bytes, int chunk, int nslot, long long *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    unsigned long long *mb = reinterpret_cast<unsigned long long *>(sm);
    unsigned char *ring = sm + 128;
    if (threadIdx.x < nslot) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mb[threadIdx.x])) : "memory");
    __syncthreads();
    if (threadIdx.x != 0) return;
    const unsigned char *s = src + (size_t)blockIdx.x * bytes;
    const int n = (int)(bytes / chunk);
    long long t0 = clk(), first = 0;
    for (int i = 0; i < n + nslot; ++i) {
        if (i >= nslot) {   // wait for copy i - nslot
            const int j = i - nslot, sl = j % nslot;
            unsigned ok = 0;
            while (!ok) asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                                     : "=r"(ok) : "r"(su32(&mb[sl])), "r"((unsigned)((j / nslot) & 1)) : "memory");
            if (j == 0) first = clk() - t0;
        }
        if (i < n) {
            const int sl = i % nslot;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mb[sl])), "r"(chunk) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su32(ring + (size_t)sl * chunk)), "l"(s + (size_t)i * chunk), "r"(chunk), "r"(su32(&mb[sl])) : "memory");
        }
    }
    long long t1 = clk();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = first; }
}
int main() {
    const size_t bytes = 4 << 20;
    unsigned char *src;
    long long *d, h[2];
    cudaMalloc(&src, bytes * 16);
    cudaMemset(src, 1, bytes * 16);
    cudaMalloc(&d, 16);
    for (int chunk : {8192, 32768, 65536}) for (int nslot : {2, 3}) for (int grid : {1, 16}) {
        const size_t smem = 128 + (size_t)chunk * nslot;
        if (smem > 227 * 1024) continue;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<grid, 32, smem>>>(src, bytes, chunk, nslot, d);   // warm (L2 holds 64 MB)
        k<<<grid, 32, smem>>>(src, bytes, chunk, nslot, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("chunk %6d slots %d grid %2d: %.1f B/cycle per SM, first copy latency %lld cycles\n", chunk, nslot, grid,
               (double)bytes / h[0], h[1]);
    }
    return 0;
}
