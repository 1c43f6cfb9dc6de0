// Microbenchmark: cost of one cluster barrier (and __syncthreads) per iteration.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int MODE>
__global__ void kbar(int iters, unsigned long long *out) {
    __shared__ double xs[1024];
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (MODE == 0) __syncthreads();
        if (MODE == 1) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (MODE == 2) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (MODE == 3) {  // CTA barrier + one warp does the cluster barrier... (all threads must arrive: not valid) -> use relaxed+wait only
            asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
        }
        xs[threadIdx.x] += 1.0;
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(int C, int T) {
    unsigned long long *d;
    cudaMalloc(&d, 64 * sizeof(unsigned long long));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(T);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaFuncSetAttribute(kbar<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int iters = 10000;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaLaunchKernelEx(&cfg, kbar<MODE>, 100, d);
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, kbar<MODE>, iters, d);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("mode %d C=%2d T=%4d : %7.1f ns/iter  %6.0f cycles/iter  %s\n", MODE, C, T, ms * 1e6 / iters, (double)h / iters, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    for (int T : {128, 512, 1024}) {
        run<0>(1, T);
        for (int C : {2, 4, 8, 16}) { run<1>(C, T); run<2>(C, T); }
    }
    return 0;
}
