// Issue cost of remote stores inside a 2-CTA cluster, one warp, 32 lanes each storing:
//  mode 0: st.async.shared::cluster.mbarrier::complete_tx (8 B)  mode 1: st.relaxed.cluster.shared::cluster
//  mode 2: local st.shared (reference)
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa(unsigned a, int r) { unsigned o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ long long clk() { long long t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)); return t; }
__global__ void __cluster_dims__(2, 1, 1) k(int mode, int iters, long long *out) {
    __shared__ __align__(8) unsigned long long mb;
    __shared__ __align__(8) double buf[4096];
    cg::cluster_group cl = cg::this_cluster();
    const int r = cl.block_rank();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mb)) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mb)), "r"(iters * 32 * 8) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    cl.sync();
    if (r == 0 && threadIdx.x < 32) {
        const unsigned rb = mapa(su32(buf), 1), rm = mapa(su32(&mb), 1);
        long long t0 = clk();
        for (int i = 0; i < iters; ++i) {
            const unsigned a = rb + 8u * ((i * 32 + threadIdx.x) & 4095);
            if (mode == 0)
                asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(a), "l"(1ll), "r"(rm) : "memory");
            else if (mode == 1)
                asm volatile("st.relaxed.cluster.shared::cluster.b64 [%0], %1;" ::"r"(a), "l"(1ll) : "memory");
            else
                buf[(i * 32 + threadIdx.x) & 4095] = 1.0;
        }
        long long t1 = clk();
        if (threadIdx.x == 0) out[mode] = (t1 - t0) / iters;
    }
    if (r == 1 && mode == 0 && threadIdx.x == 0) {
        unsigned ok = 0;
        while (!ok) asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(su32(&mb)) : "memory");
    }
    cl.sync();
}
int main() {
    long long *d, h[3];
    cudaMalloc(&d, 24);
    for (int m = 0; m < 3; ++m) k<<<2, 64>>>(m, 64, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("cycles per warp-wide store: st.async %lld | st.relaxed.cluster %lld | local STS %lld\n", h[0], h[1], h[2]);
    return 0;
}
