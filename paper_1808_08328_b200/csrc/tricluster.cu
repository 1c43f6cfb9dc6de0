// Level-synchronous sparse triangular sweep on one thread-block cluster.
//
// The exact preconditioner (reference linalg.py:225-227 ILU(0) apply and
// :383-385 Gauss-Seidel sweeps) is a chain of hundreds of dependent levels
// (SURVEY 7 H1).  Going through L2 for every level (sync-free flags) costs
// ~2 us per level; here:
//   * the solution vector lives in the distributed shared memory of one
//     cluster (<= 16 CTAs, each owns a contiguous slice of rows); x is seeded
//     with b, so a row only reads its own slot before overwriting it;
//   * every (CTA, level) has one contiguous, 16-byte aligned block in HBM
//     [header | local row ids | row ends | diagonal | column codes | values],
//     streamed into a shared-memory ring with cp.async NST-1 levels ahead,
//     so no global load sits on the dependency chain;
//   * levels are separated by one hardware cluster barrier; reads of x are
//     local or DSMEM loads (column codes = owner << 24 | local offset);
//   * rows are reduced by G-lane groups with a fixed shuffle tree.
// Arithmetic per row is the textbook b_i - sum_j t_ij x_j (/ t_ii) in
// dependency order -- exact-arithmetic identical to the reference sweep.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include "dpp_internal.cuh"

namespace cg = cooperative_groups;

namespace dpp {

constexpr int CL_THREADS = 1024;
constexpr int CL_MAX = 16;
constexpr int NST_MAX = 32;            // ring stages (upper bound)
constexpr int XS_MAX = 14000;          // rows per CTA (x slice in shared memory)
constexpr size_t SMEM_LIMIT = 227 * 1024;

__host__ __device__ __forceinline__ int pad16(int b) { return (b + 15) & ~15; }

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *m, unsigned cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *m, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *m, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(m)), "r"(parity) : "memory");
}
// TMA 1-D bulk copy global -> shared, completion counted on an mbarrier
__device__ __forceinline__ void bulk_copy(void *dst, const void *src, unsigned bytes, unsigned long long *m) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(m)) : "memory");
}

// level barrier: hardware cluster barrier with release/acquire at cluster scope
// (cg::cluster_group::sync() adds a GPU-scope MEMBAR + ERRBAR per call), or a
// plain CTA barrier when the "cluster" is a single CTA
__device__ __forceinline__ void level_barrier(int C) {
    if (C == 1) {
        __syncthreads();
    } else {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
}

// thread 0: start the copy of this CTA's level l into its ring stage
__device__ __forceinline__ void issue_level(const unsigned char *__restrict__ blocks, const long long *boff_s,
                                            int l, unsigned char *ring, int stage, int nst,
                                            unsigned long long *mbar) {
    const int s = l % nst;
    const unsigned bytes = (unsigned)(boff_s[l + 1] - boff_s[l]);
    mbar_expect_tx(&mbar[s], bytes);
    bulk_copy(ring + (size_t)s * stage, blocks + boff_s[l], bytes, &mbar[s]);
}

template <int G>
__global__ void __launch_bounds__(CL_THREADS, 1)
    k_trsv_cluster(int n, int chunk, int L, int C, int stage, int nst, const unsigned char *__restrict__ blocks,
                   const long long *__restrict__ boff, const double *__restrict__ b,
                   double *__restrict__ x, const double *__restrict__ xadd, double *__restrict__ xout) {
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned long long *mbar = reinterpret_cast<unsigned long long *>(smem);          // NST_MAX barriers
    double *xs = reinterpret_cast<double *>(smem + 8 * NST_MAX);
    long long *boff_s = reinterpret_cast<long long *>(smem + 8 * NST_MAX + pad16(chunk * 8));
    unsigned char *ring = smem + 8 * NST_MAX + pad16(chunk * 8) + pad16(8 * (L + 1));
    cg::cluster_group cl = cg::this_cluster();
    const int k = (int)cl.block_rank();
    const int gl = threadIdx.x & (G - 1), grp = threadIdx.x / G, ngrp = blockDim.x / G;
    const int lane = threadIdx.x & 31;
    const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1) << (lane & ~(G - 1)));
    const int base = k * chunk;
    const int mine = min(chunk, n - base);
    const int b0 = k * L;   // this CTA's first block
    if (threadIdx.x < nst) mbar_init(&mbar[threadIdx.x], 1);
    for (int i = threadIdx.x; i < mine; i += blockDim.x) xs[i] = b[base + i];
    for (int i = threadIdx.x; i <= L; i += blockDim.x) boff_s[i] = boff[b0 + i];
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0)
        for (int l = 0; l < min(nst - 1, L); ++l) issue_level(blocks, boff_s, l, ring, stage, nst, mbar);
    if (C > 1) level_barrier(C);    // every CTA's x slice is seeded before any remote read
    for (int l = 0; l < L; ++l) {
        // thread 0 waits for level l's block; the barrier then publishes it to the CTA,
        // together with the x values of level l-1 to the whole cluster
        if (threadIdx.x == 0) mbar_wait(&mbar[l % nst], (unsigned)((l / nst) & 1));
        level_barrier(C);
        if (threadIdx.x == 0 && l + nst - 1 < L) issue_level(blocks, boff_s, l + nst - 1, ring, stage, nst, mbar);
        const unsigned char *blk = ring + (size_t)(l % nst) * stage;
        const int nr = reinterpret_cast<const int *>(blk)[0];
        const int *lrow = reinterpret_cast<const int *>(blk + 16);
        const int *rend = reinterpret_cast<const int *>(blk + 16 + pad16(4 * nr));
        const double *dg = reinterpret_cast<const double *>(blk + 16 + 2 * pad16(4 * nr));
        const int ne = nr ? rend[nr - 1] : 0;
        const int *cidx = reinterpret_cast<const int *>(blk + 16 + 2 * pad16(4 * nr) + 8 * nr);
        const double *val = reinterpret_cast<const double *>(blk + 16 + 2 * pad16(4 * nr) + 8 * nr + pad16(4 * ne));
        for (int q = grp; q < nr; q += ngrp) {
            const int r = lrow[q];
            const int e0 = q ? rend[q - 1] : 0, e1 = rend[q];
            double sum = 0.0;
            for (int e = e0 + gl; e < e1; e += G) {
                const int c = cidx[e];
                const int o = c >> 24, loc = c & 0xFFFFFF;
                const double *src = o == k ? xs : cl.map_shared_rank(xs, o);
                sum += val[e] * src[loc];
            }
#pragma unroll
            for (int s = G / 2; s > 0; s >>= 1) sum += __shfl_xor_sync(gmask, sum, s, G);
            if (gl == 0) xs[r] = (xs[r] - sum) * dg[q];   // dg = 1/t_ii (as SuperLU's pre-scaled solve)
        }
    }
    level_barrier(C);
    for (int i = threadIdx.x; i < mine; i += blockDim.x) {
        x[base + i] = xs[i];
        if (xout) xout[base + i] = xadd[base + i] + xs[i];
    }
}

static size_t smem_fixed(int chunk, int L) { return 8 * NST_MAX + (size_t)pad16(chunk * 8) + (size_t)pad16(8 * (L + 1)); }

// ----------------------------------------------------------------- plan
__global__ void k_owner_keys(int n, int chunk, int L, const int *lev, int *key, int *rows) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        key[r] = (r / chunk) * L + lev[r];
        rows[r] = r;
    }
}
// lp[v] = first sorted position with key >= v, v in [0, nkeys]
__global__ void k_key_ptr(int n, const int *skey, int nkeys, int *lp) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x) {
        const int v = i < n ? skey[i] : nkeys;
        const int prev = i ? skey[i - 1] : -1;
        for (int k = prev + 1; k <= v && k <= nkeys; ++k) lp[k] = i;
    }
}
__global__ void k_perm_len(int n, const int *perm, const int *ptr, int *len) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x)
        len[q] = ptr[perm[q] + 1] - ptr[perm[q]];
}
// block bytes from (rows, entries) of each (CTA, level)
__global__ void k_block_bytes(int nblk, const int *lp, const int *rptr, long long *bytes) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nblk; i += gridDim.x * blockDim.x) {
        const int nr = lp[i + 1] - lp[i];
        const int ne = rptr[lp[i + 1]] - rptr[lp[i]];
        long long by = 16 + 2 * pad16(4 * nr) + 8LL * nr + pad16(4 * ne) + 8LL * ne;
        bytes[i] = (by + 15) & ~15LL;
    }
}
__global__ void k_block_fill(int n, int chunk, const int *skey, const int *perm, const int *lp,
                             const int *rptr, const long long *boff, const int *ptr, const int *idx,
                             const double *val, const double *diag, unsigned char *blocks) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        const int blk = skey[q];
        const int q0 = lp[blk], nr = lp[blk + 1] - q0, i = q - q0;
        const int ne = rptr[lp[blk + 1]] - rptr[q0];
        unsigned char *B = blocks + boff[blk];
        const int r = perm[q];
        const int owner = r / chunk;
        if (i == 0) { reinterpret_cast<int *>(B)[0] = nr; reinterpret_cast<int *>(B)[1] = ne; }
        reinterpret_cast<int *>(B + 16)[i] = r - owner * chunk;
        reinterpret_cast<int *>(B + 16 + pad16(4 * nr))[i] = rptr[q + 1] - rptr[q0];
        reinterpret_cast<double *>(B + 16 + 2 * pad16(4 * nr))[i] = diag ? 1.0 / diag[r] : 1.0;
        int *ci = reinterpret_cast<int *>(B + 16 + 2 * pad16(4 * nr) + 8 * nr);
        double *vv = reinterpret_cast<double *>(B + 16 + 2 * pad16(4 * nr) + 8 * nr + pad16(4 * ne));
        int w = rptr[q] - rptr[q0];
        for (int p = ptr[r]; p < ptr[r + 1]; ++p, ++w) {
            const int j = idx[p];
            const int o = j / chunk;
            ci[w] = (o << 24) | (j - o * chunk);
            vv[w] = val[p];
        }
    }
}
__global__ void k_block_headers(int nblk, const int *lp, unsigned char *blocks, const long long *boff) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nblk; i += gridDim.x * blockDim.x)
        if (lp[i + 1] == lp[i]) {
            reinterpret_cast<int *>(blocks + boff[i])[0] = 0;
            reinterpret_cast<int *>(blocks + boff[i])[1] = 0;
        }
}

static bool try_plan(Ctx *c, Tri &T, const DBuf<int> &lev, int L, int C) {
    const int n = T.n;
    const int chunk = (n + C - 1) / C;
    const int nblk = C * L;
    DBuf<int> key(n, c->s), skey(n, c->s), rows(n, c->s), perm(n, c->s), len(n, c->s),
        lp((size_t)nblk + 1, c->s);
    k_owner_keys<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, chunk, L, lev.p, key.p, rows.p);
    launched(c);
    int bits = 1;
    while (bits < 31 && (1 << bits) <= nblk) ++bits;
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, skey.p, rows.p, perm.p, n, 0, bits, c->s));
    {
        DBuf<char> t(tb, c->s);
        CK(cub::DeviceRadixSort::SortPairs(t.p, tb, key.p, skey.p, rows.p, perm.p, n, 0, bits, c->s));
        launched(c);
    }
    k_key_ptr<<<grid_for(n + 1, 256, c->sms), 256, 0, c->s>>>(n, skey.p, nblk, lp.p);
    launched(c);
    k_perm_len<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, perm.p, T.strict.ptr.p, len.p);
    launched(c);
    DBuf<int> rptr;
    counts_to_ptr(c, len.p, n, rptr);
    DBuf<long long> bytes((size_t)nblk + 1, c->s), boff((size_t)nblk + 1, c->s);
    CK(cudaMemsetAsync(bytes.p + nblk, 0, sizeof(long long), c->s));
    k_block_bytes<<<grid_for(nblk, 256, c->sms), 256, 0, c->s>>>(nblk, lp.p, rptr.p, bytes.p);
    launched(c);
    size_t tb2 = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb2, bytes.p, boff.p, nblk + 1, c->s));
    {
        DBuf<char> t(tb2, c->s);
        CK(cub::DeviceScan::ExclusiveSum(t.p, tb2, bytes.p, boff.p, nblk + 1, c->s));
        launched(c);
    }
    std::vector<long long> hb = bytes.to_host();
    long long mx = 16;
    for (int i = 0; i < nblk; ++i) mx = std::max(mx, hb[i]);
    std::vector<int> hlp = lp.to_host();
    int widest = 1;
    for (int i = 0; i < nblk; ++i) widest = std::max(widest, hlp[i + 1] - hlp[i]);
    const size_t fixed = smem_fixed(chunk, L);
    if (fixed >= SMEM_LIMIT) return false;
    const long long stage = (mx + 127) & ~127LL;
    const int nst = (int)std::min<long long>(NST_MAX, (long long)(SMEM_LIMIT - fixed) / stage);
    if (nst < 2) return false;
    long long total = 0;
    CK(cudaMemcpyAsync(&total, boff.p + nblk, sizeof(long long), cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    auto P = std::make_unique<ClusterPlan>();
    P->C = C;
    P->chunk = chunk;
    P->L = L;
    P->stage = (int)stage;
    P->nst = nst;
    const double avg = (double)T.strict.nnz / n;
    // ~4 entries per lane; threads sized to the widest (CTA, level) so idle warps
    // do not pay the per-level instruction overhead
    P->G = 2;
    while (P->G < 32 && P->G * 4 < avg) P->G *= 2;
    int threads = 64;
    while (threads < CL_THREADS && (threads / P->G) < widest) threads *= 2;
    P->threads = threads;
    P->blocks.alloc((size_t)total, c->s);
    P->boff = std::move(boff);
    k_block_headers<<<grid_for(nblk, 256, c->sms), 256, 0, c->s>>>(nblk, lp.p, P->blocks.p, P->boff.p);
    launched(c);
    k_block_fill<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, chunk, skey.p, perm.p, lp.p, rptr.p,
                                                           P->boff.p, T.strict.ptr.p, T.strict.idx.p,
                                                           T.strict.val.p, T.diag.n ? T.diag.p : nullptr,
                                                           P->blocks.p);
    launched(c);
    CK(cudaStreamSynchronize(c->s));
    T.cl = std::move(P);
    return true;
}


bool cluster_plan(Ctx *c, Tri &T, const DBuf<int> &lev, int L) {
    const int n = T.n;
    if (n == 0 || L < 1) return false;
    static bool attr = false;
    if (!attr) {
        auto setk = [](const void *f) {
            CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_LIMIT));
            CK(cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        };
        setk((const void *)k_trsv_cluster<2>);
        setk((const void *)k_trsv_cluster<4>);
        setk((const void *)k_trsv_cluster<8>);
        setk((const void *)k_trsv_cluster<16>);
        setk((const void *)k_trsv_cluster<32>);
        attr = true;
    }
    // as many CTAs as useful: each keeps >= ~2k rows of x
    int C0 = std::max((n + XS_MAX - 1) / XS_MAX, std::min(CL_MAX, (n + 2047) / 2048));
    for (int C = C0; C <= CL_MAX; ++C)
        if (try_plan(c, T, lev, L, C)) return true;
    return false;
}

void trsv_cluster(Ctx *c, const Tri &T, const double *b, double *x, const double *xadd, double *xout,
                  cudaStream_t st) {
    const ClusterPlan &P = *T.cl;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P.C, 1, 1);
    cfg.blockDim = dim3(P.threads, 1, 1);
    cfg.dynamicSmemBytes = smem_fixed(P.chunk, P.L) + (size_t)P.nst * P.stage;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = P.C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const unsigned char *B = P.blocks.p;
    const long long *O = P.boff.p;
    cudaError_t e;
    switch (P.G) {
        case 2: e = cudaLaunchKernelEx(&cfg, k_trsv_cluster<2>, T.n, P.chunk, P.L, P.C, P.stage, P.nst, B, O, b, x, xadd, xout); break;
        case 4: e = cudaLaunchKernelEx(&cfg, k_trsv_cluster<4>, T.n, P.chunk, P.L, P.C, P.stage, P.nst, B, O, b, x, xadd, xout); break;
        case 8: e = cudaLaunchKernelEx(&cfg, k_trsv_cluster<8>, T.n, P.chunk, P.L, P.C, P.stage, P.nst, B, O, b, x, xadd, xout); break;
        case 16: e = cudaLaunchKernelEx(&cfg, k_trsv_cluster<16>, T.n, P.chunk, P.L, P.C, P.stage, P.nst, B, O, b, x, xadd, xout); break;
        default: e = cudaLaunchKernelEx(&cfg, k_trsv_cluster<32>, T.n, P.chunk, P.L, P.C, P.stage, P.nst, B, O, b, x, xadd, xout); break;
    }
    CK(e);
    launched(c);
}

}  // namespace dpp
