// Block-sequential triangular sweep for small, deep triangles (coarse AMG levels).
//
// The Gauss-Seidel sweeps of the reference's V-cycle (linalg.py:383-385) on the
// first coarse level have hundreds of dependency levels for a few thousand rows
// (691 levels on 5,593 rows at config 2), so any
// level-by-level schedule pays a barrier per ~8 rows.  Here consecutive rows are
// grouped into blocks of BS = 32; the dense inverse of each diagonal block is
// formed at setup (an exact-arithmetic rewrite of the same sweep), and the
// sweep becomes n/BS dependent steps, each
//     r_K = b_K - T_{K,outside} x      (one warp per row, sparse)
//     x_K = inv(T_KK) r_K              (one warp per row, dense 32-wide)
// on a single CTA with x in shared memory and every block's data streamed
// into a shared-memory ring by TMA bulk copies several steps ahead.
#include <cub/cub.cuh>

#include <cstdio>

#include "dpp_internal.cuh"

namespace dpp {

constexpr int BS = 32;                 // rows per block
constexpr int BT = 1024;               // threads (32 warps: one per block row)
constexpr int BNST = 4;                // max ring stages (runtime nst <= BNST)
constexpr size_t BSMEM_LIMIT = 227 * 1024;

__host__ __device__ __forceinline__ int bpad16(long long b) { return (int)((b + 15) & ~15LL); }
// block layout: [int nr, int ne, pad, pad][int rend[BS]][double dinv[BS][BS]][int cidx[ne]][double val[ne]]
__host__ __device__ __forceinline__ long long block_bytes(int ne) {
    return 16 + 4 * BS + 8 * BS * BS + bpad16(4LL * ne) + 8LL * ne;
}

__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bmbar_init(unsigned long long *m) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(m)) : "memory");
}
__device__ __forceinline__ void bmbar_wait(unsigned long long *m, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAITB_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAITB_%=;\n}" ::"r"(su32(m)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bissue(const unsigned char *src, unsigned bytes, unsigned char *dst,
                                       unsigned long long *m) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(m)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(m)) : "memory");
}

__global__ void __launch_bounds__(BT, 1)
    k_trsv_block(int n, int nblk, int backward, int stage, int nst, const unsigned char *__restrict__ blocks,
                 const long long *__restrict__ boff, const double *__restrict__ b, double *__restrict__ x,
                 const double *__restrict__ xadd, double *__restrict__ xout) {
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned long long *mbar = reinterpret_cast<unsigned long long *>(smem);
    double *rs = reinterpret_cast<double *>(smem + 128);              // r of the current block
    double *xs = reinterpret_cast<double *>(smem + 128 + 8 * BS);
    unsigned char *ring = smem + 128 + 8 * BS + bpad16(8LL * n);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x < nst) bmbar_init(&mbar[threadIdx.x]);
    for (int i = threadIdx.x; i < n; i += BT) xs[i] = b[i];
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0)
        for (int s = 0; s < nst - 1 && s < nblk; ++s)
            bissue(blocks + boff[s], (unsigned)(boff[s + 1] - boff[s]), ring + (size_t)s * stage, &mbar[s]);
    int slot = 0;
    unsigned phase = 0;
    for (int t = 0; t < nblk; ++t) {
        // step t processes block K (forward: K = t, backward: K = nblk-1-t); blocks are stored in step order
        const int K = backward ? nblk - 1 - t : t;
        const int row0 = K * BS;
        if (threadIdx.x == 0) bmbar_wait(&mbar[slot], phase);
        __syncthreads();   // block data landed; x of step t-1 visible; stage of t-1 reusable
        if (threadIdx.x == 0 && t + nst - 1 < nblk) {
            const int s = (slot + nst - 1) % nst;
            bissue(blocks + boff[t + nst - 1], (unsigned)(boff[t + nst] - boff[t + nst - 1]),
                   ring + (size_t)s * stage, &mbar[s]);
        }
        const unsigned char *blk = ring + (size_t)slot * stage;
        const int nr = reinterpret_cast<const int *>(blk)[0];
        const int *rend = reinterpret_cast<const int *>(blk + 16);
        const double *dinv = reinterpret_cast<const double *>(blk + 16 + 4 * BS);
        const int ne = nr ? rend[nr - 1] : 0;
        const int *cidx = reinterpret_cast<const int *>(blk + 16 + 4 * BS + 8 * BS * BS);
        const double *val = reinterpret_cast<const double *>(blk + 16 + 4 * BS + 8 * BS * BS + bpad16(4LL * ne));
        if (w < nr) {   // r_w = b_w - T_{w,outside} x
            const int e0 = w ? rend[w - 1] : 0, e1 = rend[w];
            double s = 0.0;
            for (int e = e0 + lane; e < e1; e += 32) s += val[e] * xs[cidx[e]];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) rs[w] = xs[row0 + w] - s;
        }
        __syncthreads();
        if (w < nr) {   // x_w = sum_j inv(T_KK)_wj r_j
            double s = lane < nr ? dinv[w * BS + lane] * rs[lane] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) xs[row0 + w] = s;
        }
        if (++slot == nst) { slot = 0; phase ^= 1u; }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += BT) {
        x[i] = xs[i];
        if (xout) xout[i] = xadd[i] + xs[i];
    }
}

// ----------------------------------------------------------------- plan
// entries of row r outside its diagonal block, per block in step order
__global__ void k_blk_count(int n, int nblk, int backward, const int *ptr, const int *idx, int *cnt) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const int K = r / BS;
        int c = 0;
        for (int p = ptr[r]; p < ptr[r + 1]; ++p) c += idx[p] / BS != K;
        cnt[r] = c;
        (void)nblk;
        (void)backward;
    }
}
__global__ void k_blk_bytes(int nblk, int n, int backward, const int *rp, long long *bytes) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nblk; t += gridDim.x * blockDim.x) {
        const int K = backward ? nblk - 1 - t : t;
        const int r0 = K * BS, r1 = min(n, r0 + BS);
        bytes[t] = bpad16(block_bytes(rp[r1] - rp[r0]));
    }
}
// one warp per block: outside entries, then the dense inverse of the diagonal block
__global__ void k_blk_fill(int n, int nblk, int backward, const int *ptr, const int *idx, const double *val,
                           const double *diag, const int *rp, const long long *boff, unsigned char *blocks) {
    __shared__ double T[BS][BS + 1];
    const int lane = threadIdx.x & 31;
    for (int t = blockIdx.x; t < nblk; t += gridDim.x) {
        const int K = backward ? nblk - 1 - t : t;
        const int r0 = K * BS, nr = min(n, r0 + BS) - r0;
        unsigned char *B = blocks + boff[t];
        const int ne = rp[r0 + nr] - rp[r0];
        int *rend = reinterpret_cast<int *>(B + 16);
        double *dinv = reinterpret_cast<double *>(B + 16 + 4 * BS);
        int *cidx = reinterpret_cast<int *>(B + 16 + 4 * BS + 8 * BS * BS);
        double *vv = reinterpret_cast<double *>(B + 16 + 4 * BS + 8 * BS * BS + bpad16(4LL * ne));
        if (lane == 0) { reinterpret_cast<int *>(B)[0] = nr; reinterpret_cast<int *>(B)[1] = ne; }
        for (int i = 0; i < BS; ++i) T[i][lane] = (i == lane && i >= nr) ? 1.0 : 0.0;
        __syncwarp();
        for (int i = 0; i < nr; ++i) {
            const int r = r0 + i;
            if (lane == 0) rend[i] = rp[r + 1] - rp[r0];
            int w = rp[r] - rp[r0];
            // outside entries keep their stored order; inside entries go to the dense block
            for (int p = ptr[r]; p < ptr[r + 1]; ++p) {
                const int j = idx[p];
                if (j / BS != K) {
                    if (lane == 0) { cidx[w] = j; vv[w] = val[p]; }
                    ++w;
                } else if (lane == 0) {
                    T[i][j - r0] += val[p];
                }
            }
            if (lane == 0) T[i][i] += diag ? diag[r] : 1.0;
        }
        for (int i = nr; i < BS; ++i)
            if (lane == 0) rend[i] = ne;
        __syncwarp();
        // column `lane` of inv(T): forward substitution (lower) or backward (upper)
        double xcol[BS];
        if (!backward) {
            for (int i = 0; i < BS; ++i) {
                double s = i == lane ? 1.0 : 0.0;
                for (int j = 0; j < i; ++j) s -= T[i][j] * xcol[j];
                xcol[i] = s / T[i][i];
            }
        } else {
            for (int i = BS - 1; i >= 0; --i) {
                double s = i == lane ? 1.0 : 0.0;
                for (int j = i + 1; j < BS; ++j) s -= T[i][j] * xcol[j];
                xcol[i] = s / T[i][i];
            }
        }
        for (int i = 0; i < BS; ++i) dinv[i * BS + lane] = xcol[i];
        __syncwarp();
    }
}

static size_t bsmem_fixed(int n) { return 128 + 8 * BS + (size_t)bpad16(8LL * n); }

bool block_plan(Ctx *c, Tri &T) {
    const int n = T.n;
    if (n == 0) return false;
    const int nblk = (n + BS - 1) / BS;
    DBuf<int> cnt(n, c->s), rp;
    k_blk_count<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, nblk, T.backward, T.strict.ptr.p, T.strict.idx.p,
                                                          cnt.p);
    launched(c);
    counts_to_ptr(c, cnt.p, n, rp);
    DBuf<long long> bytes((size_t)nblk + 1, c->s), boff((size_t)nblk + 1, c->s);
    CK(cudaMemsetAsync(bytes.p + nblk, 0, sizeof(long long), c->s));
    k_blk_bytes<<<grid_for(nblk, 256, c->sms), 256, 0, c->s>>>(nblk, n, T.backward, rp.p, bytes.p);
    launched(c);
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, bytes.p, boff.p, nblk + 1, c->s));
    {
        DBuf<char> t(tb, c->s);
        CK(cub::DeviceScan::ExclusiveSum(t.p, tb, bytes.p, boff.p, nblk + 1, c->s));
        launched(c);
    }
    std::vector<long long> hb = bytes.to_host();
    long long mx = 16;
    for (int i = 0; i < nblk; ++i) mx = std::max(mx, hb[i]);
    const int stage = (int)((mx + 127) & ~127LL);
    const int nst = (int)std::min<long long>(BNST, ((long long)BSMEM_LIMIT - (long long)bsmem_fixed(n)) / stage);
    if (TraceScope::on())
        std::fprintf(stderr, "[dpp-trace]   block_plan n=%d nblk=%d stage=%d nst=%d\n", n, nblk, stage, nst);
    if (nst < 2) return false;
    long long total = 0;
    CK(cudaMemcpyAsync(&total, boff.p + nblk, sizeof(long long), cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    auto P = std::make_unique<BlockPlan>();
    P->nblk = nblk;
    P->stage = stage;
    P->nst = nst;
    P->blocks.alloc((size_t)total, c->s);
    P->boff = std::move(boff);
    k_blk_fill<<<std::min(nblk, c->sms * 8), 32, 0, c->s>>>(n, nblk, T.backward, T.strict.ptr.p, T.strict.idx.p,
                                                           T.strict.val.p, T.diag.n ? T.diag.p : nullptr, rp.p,
                                                           P->boff.p, P->blocks.p);
    launched(c);
    CK(cudaStreamSynchronize(c->s));
    static bool attr = false;
    if (!attr) {
        CK(cudaFuncSetAttribute(k_trsv_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BSMEM_LIMIT));
        attr = true;
    }
    T.bl = std::move(P);
    return true;
}

void trsv_block(Ctx *c, const Tri &T, const double *b, double *x, const double *xadd, double *xout,
                cudaStream_t st) {
    const BlockPlan &P = *T.bl;
    k_trsv_block<<<1, BT, bsmem_fixed(T.n) + (size_t)P.nst * P.stage, st>>>(
        T.n, P.nblk, T.backward, P.stage, P.nst, P.blocks.p, P.boff.p, b, x, xadd, xout);
    launched(c);
}

}  // namespace dpp
