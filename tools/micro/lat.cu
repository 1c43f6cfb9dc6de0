// Dependent-chain latencies (cycles) on one warp: DFMA, DADD, SHFL (64-bit via 2x32), LDS.64
#include <cstdio>
__global__ void k(int iters, double seed, long long *out) {
    __shared__ double sm[1024];
    __shared__ int si[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sm[i] = 1.0 + i * 1e-9; si[i] = (i * 7 + 3) & 1023; }
    __syncthreads();
    double a = seed, b = 1.0000001, c = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) a = fma(a, b, c);
    long long t1 = clock64();
    for (int i = 0; i < iters; ++i) a = a + c;
    long long t2 = clock64();
    for (int i = 0; i < iters; ++i) a += __shfl_xor_sync(0xffffffffu, a, 1);
    long long t3 = clock64();
    int j = threadIdx.x;
    for (int i = 0; i < iters; ++i) j = si[j];
    long long t4 = clock64();
    double x = 0; int p = threadIdx.x;
    for (int i = 0; i < iters; ++i) { x = sm[(p + (int)x) & 1023]; }
    long long t5 = clock64();
    if (threadIdx.x == 0) {
        out[0] = (t1 - t0) / iters; out[1] = (t2 - t1) / iters; out[2] = (t3 - t2) / iters;
        out[3] = (t4 - t3) / iters; out[4] = (t5 - t4) / iters; out[5] = (long long)(a + j + x);
    }
}
int main() {
    long long *d, h[6];
    cudaMalloc(&d, sizeof(h));
    k<<<1, 32>>>(4096, 1.0, d);
    k<<<1, 32>>>(4096, 1.0, d);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("latency cycles: DFMA %lld | DADD %lld | SHFL.f64+DADD %lld | LDS.32 dep %lld | LDS.64 dep (+cvt) %lld\n",
           h[0], h[1], h[2], h[3], h[4]);
}
