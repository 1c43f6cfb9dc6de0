// Round-trip latency between two CTAs of a cluster (cycles), three mechanisms:
//  0: st.async + mbarrier complete_tx, receiver mbarrier.try_wait
//  1: st.shared::cluster (relaxed remote store) + local volatile polling on a sentinel
//  2: barrier.cluster.arrive.relaxed / wait (no data)
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa(unsigned a, int r) { unsigned o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }

__global__ void __cluster_dims__(2, 1, 1) k_pp(int mode, int iters, unsigned long long *out) {
    __shared__ __align__(8) unsigned long long mb[1024];
    __shared__ __align__(8) double val[1024];
    cg::cluster_group cl = cg::this_cluster();
    const int k = cl.block_rank(), other = 1 - k;
    if (threadIdx.x == 0) {
        for (int i = 0; i < iters; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mb[i])) : "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 8;" ::"r"(su32(&mb[i])) : "memory");
            val[i] = -1.0;
        }
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    cl.sync();
    if (threadIdx.x != 0) return;
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const bool my_turn = (i & 1) == k;
        if (mode == 0) {
            if (my_turn) {
                asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
                             ::"r"(mapa(su32(&val[i]), other)), "l"(1ll), "r"(mapa(su32(&mb[i]), other)) : "memory");
            } else {
                asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}"
                             ::"r"(su32(&mb[i])) : "memory");
            }
        } else if (mode == 1) {
            if (my_turn) {
                asm volatile("st.relaxed.cluster.shared::cluster.f64 [%0], %1;" ::"r"(mapa(su32(&val[i]), other)), "d"(1.0) : "memory");
            } else {
                volatile double *v = &val[i];
                while (*v < 0.0) {}
            }
        } else {
            asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
        }
    }
    const unsigned long long t1 = clock64();
    if (k == 0) out[mode] = (t1 - t0) / iters;   // cycles per one-way hop
}

int main() {
    unsigned long long *d, h[3];
    cudaMalloc(&d, 24);
    for (int mode = 0; mode < 3; ++mode) {
        // mode 2 needs every thread of both CTAs at the barrier: use 32 threads and let all run
        k_pp<<<2, mode == 2 ? 1 : 1>>>(mode, 1000, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("mode %d error %s\n", mode, cudaGetErrorString(e)); return 1; }
    }
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("one-way hop cycles: st.async+mbarrier %llu | remote st + poll %llu | cluster barrier %llu\n", h[0], h[1], h[2]);
    return 0;
}
