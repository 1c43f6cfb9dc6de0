// Level-scheduled sparse triangular sweep on one thread-block cluster, with
// point-to-point x exchange (push) instead of a cluster barrier per level.
//
// Same problem and arithmetic as tricluster.cu (reference linalg.py:225-227 ILU(0)
// apply, :383-385 Gauss-Seidel sweeps): each CTA owns a contiguous slice of rows
// (x seeded with b in shared memory), rows are processed level by level, and
// every (CTA, level) block is streamed into a shared-memory ring by TMA.  The
// difference is how a level's results reach the CTAs that need them:
//
//   * at setup, every cross-CTA dependency (consumer CTA d reads row j owned by
//     another CTA) gets a slot in d's halo buffer; a row's block entry carries
//     its push list (destination CTA, halo slot), and column codes address
//     either the own slice or the halo;
//   * when a row is solved, its value is written with st.async straight into
//     every consumer's halo, counting 8 bytes on the consumer's mbarrier of
//     the producing level (one single-use mbarrier per level, armed at launch
//     with the exact byte count the CTA will receive for that level);
//   * before level l a CTA waits only on its level l-1 mbarrier (all values
//     it will ever read from level l-1) and on a CTA barrier for its own rows.
//
// So a level costs one push latency on the critical path instead of a
// release/acquire cluster barrier (MEMBAR.GPU + ERRBAR + barrier round trip).
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <cstdio>
#include <cstdlib>

#include "dpp_internal.cuh"

namespace cg = cooperative_groups;

namespace dpp {

namespace {

constexpr int PU_THREADS = 1024;
constexpr int PU_MAX = 16;
constexpr int PU_NST_MAX = 16;
constexpr int PU_LMAX = 4096;              // one mbarrier per level in shared memory (32 KB)
constexpr size_t PU_SMEM_LIMIT = 226 * 1024;   // dynamic; leaves room for static shared memory

__host__ __device__ __forceinline__ long long p16(long long b) { return (b + 15) & ~15LL; }
__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa_u32(unsigned a, int rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// bounded wait: a miscounted exchange traps (~2 s) instead of hanging the device
__device__ __forceinline__ void mwait(unsigned a, unsigned parity) {
    unsigned ok = 0;
    const long long t0 = clock64();
    while (true) {
        asm volatile(
            "{\n .reg .pred p;\n"
            " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(a), "r"(parity) : "memory");
        if (ok) return;
        if (clock64() - t0 > (4ll << 30)) __trap();
    }
}

// shared memory: ring mbarriers | level mbarriers [L] | xh = [x slice (chunk, padded) | halo (hmax)] |
//                boff [smax+1] | peer addresses | ring
// A CTA walks its own list of steps: the non-empty (level, part) blocks of its rows in
// level order (a level's block is cut into parts that fit one ring stage).
__host__ __device__ inline int pu_chunkp(int chunk) { return (int)(p16(8LL * chunk) / 8); }
__host__ __device__ inline size_t pu_fixed(int chunk, int L, int hmax, int smax) {
    return 8 * PU_NST_MAX + p16(8LL * L) + p16(8LL * chunk) + p16(8LL * hmax) + p16(8LL * (smax + 1)) + 8 * PU_MAX;
}

// block layout (16-byte aligned):
//   int4 {nr, ne, np, level} | int4 row[nr] = {local row, e0, e1, p0 << 4 | npush} | double dg[nr] |
//   int code[ne] (index into xh) | (16) double val[ne] | int push[np] (dest << 28 | halo slot)
__host__ __device__ inline long long pu_off_code(long long nr) { return 16 + 24 * nr; }
__host__ __device__ inline long long pu_off_val(long long nr, long long ne) { return p16(pu_off_code(nr) + 4 * ne); }
__host__ __device__ inline long long pu_block_bytes(long long nr, long long ne, long long np) {
    return p16(pu_off_val(nr, ne) + 8 * ne + 4 * np);
}

template <int G>
__global__ void __launch_bounds__(PU_THREADS, 1)
    k_trsv_push(int n, int ncomp, int chunk, int L, int smax, int hmax, int stage, int nst,
                const unsigned char *__restrict__ blocks, const long long *__restrict__ boff,
                const int *__restrict__ sstart, const int *__restrict__ tx, const int *__restrict__ wptr,
                const int *__restrict__ widx, const double *__restrict__ wval, const double *__restrict__ b,
                double *__restrict__ x, const double *__restrict__ xadd, double *__restrict__ xout, int l2pf,
                unsigned long long *dbg) {
    extern __shared__ __align__(128) unsigned char smem[];
    // debug timeline (DPP_PU_DEBUG): per step {level, rows, t ring landed, t levels landed,
    // t barrier passed, t last row pushed} in %globaltimer ns, row [cta][step] of dbg
    __shared__ unsigned long long t_done[2][32];   // per warp (no atomics on the timed path)
    unsigned long long tB = 0, tC = 0;
    unsigned long long *mring = reinterpret_cast<unsigned long long *>(smem);
    unsigned long long *mlev = mring + PU_NST_MAX;
    double *xh = reinterpret_cast<double *>(smem + 8 * PU_NST_MAX + p16(8LL * L));
    long long *boff_s = reinterpret_cast<long long *>(xh + pu_chunkp(chunk) + p16(8LL * hmax) / 8);
    unsigned *peer = reinterpret_cast<unsigned *>(boff_s + p16(8LL * (smax + 1)) / 8);   // [0,16): halo, [16,32): mlev
    unsigned char *ring = smem + pu_fixed(chunk, L, hmax, smax);
    cg::cluster_group cl = cg::this_cluster();
    const int k = (int)cl.block_rank(), C = (int)cl.num_blocks();
    const int comp = blockIdx.x / C;   // one cluster per Kronecker component (x[r * ncomp + comp])
    const int s0 = sstart[k], S = sstart[k + 1] - s0;
    const int gl = threadIdx.x & (G - 1), grp = threadIdx.x / G, ngrp = blockDim.x / G;
    const int lane = threadIdx.x & 31;
    const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1) << (lane & ~(G - 1)));
    const int base = k * chunk, mine = min(chunk, n - base);
    const int b0 = k * L;
    if (threadIdx.x < nst)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mring[threadIdx.x])) : "memory");
    for (int l = threadIdx.x; l < L; l += blockDim.x) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mlev[l])) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mlev[l])), "r"(tx[b0 + l])
                     : "memory");
    }
    if (threadIdx.x < C) {   // every peer's halo / level-mbarrier base in the cluster window
        peer[threadIdx.x] = mapa_u32(su32(xh + pu_chunkp(chunk)), threadIdx.x);
        peer[16 + threadIdx.x] = mapa_u32(su32(mlev), threadIdx.x);
    }
    for (int i = threadIdx.x; i <= S; i += blockDim.x) boff_s[i] = boff[s0 + i];
    pdl_wait();   // b is the previous kernel's output (the prologue above reads static plan data only)
    if (wptr) {   // level-merged sweep: right-hand side W b
        for (int i = threadIdx.x; i < mine; i += blockDim.x) {
            double v = 0.0;
            for (int p = wptr[base + i]; p < wptr[base + i + 1]; ++p) v += wval[p] * b[(size_t)widx[p] * ncomp + comp];
            xh[i] = v;
        }
    } else {
        for (int i = threadIdx.x; i < mine; i += blockDim.x) xh[i] = b[(size_t)(base + i) * ncomp + comp];
    }
    if (dbg && threadIdx.x < 64) t_done[threadIdx.x >> 5][threadIdx.x & 31] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    auto issue = [&](int l, int s) {
        const unsigned bytes = (unsigned)(boff_s[l + 1] - boff_s[l]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mring[s])), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(ring + (size_t)s * stage)), "l"(blocks + boff_s[l]), "r"(bytes), "r"(su32(&mring[s]))
                     : "memory");
    };
    // blocks further ahead than the ring are pulled into L2, so the ring's
    // copies come from L2 rather than HBM
    auto prefetch = [&](int l) {
        const unsigned bytes = (unsigned)(boff_s[l + 1] - boff_s[l]);
        if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(blocks + boff_s[l]), "r"(bytes) : "memory");
    };
    if (threadIdx.x == blockDim.x - 32) {
        for (int l = 0; l < min(nst - 1, S); ++l) issue(l, l);
        for (int l = nst - 1; l < min(nst - 1 + l2pf, S); ++l) prefetch(l);
    }
    // every CTA's level mbarriers are armed before the first push
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    int slot = 0, islot = nst - 1, waited = 0;
    unsigned phase = 0;
    for (int st = 0; st < S; ++st) {
        // the producer is lane 0 of the LAST warp: rows are dealt to lane groups from
        // group 0 up, so warp 0 (which holds every level's first rows) starts its rows
        // right after the barrier instead of first issuing the next TMA copy
        const bool producer = threadIdx.x == blockDim.x - 32;
        const unsigned char *blk = ring + (size_t)slot * stage;
        if (producer) {
            mwait(su32(&mring[slot]), phase);
            if (dbg) tB = gtimer();
            // every value this CTA reads from levels below this step's level landed
            const int lv = reinterpret_cast<const int4 *>(blk)->w;
            while (waited < lv) mwait(su32(&mlev[waited++]), 0);
            if (dbg) tC = gtimer();
        }
        __syncthreads();   // ... and its own rows of earlier steps are written
        if (dbg && producer) {
            unsigned long long *o = dbg + ((size_t)blockIdx.x * smax + st) * 6;
            o[0] = reinterpret_cast<const int4 *>(blk)->w;
            o[1] = reinterpret_cast<const int4 *>(blk)->x;
            o[2] = tB; o[3] = tC; o[4] = gtimer();
            if (st > 0) {
                unsigned long long m = 0;
                for (int w = 0; w < 32; ++w) { m = max(m, t_done[(st - 1) & 1][w]); t_done[(st - 1) & 1][w] = 0; }
                dbg[((size_t)blockIdx.x * smax + st - 1) * 6 + 5] = m;
            }
        }
        if (producer) {
            if (st + nst - 1 < S) issue(st + nst - 1, islot);   // the slot of step st-1 is free
            if (st + nst - 1 + l2pf < S) prefetch(st + nst - 1 + l2pf);
        }
        if (++slot == nst) { slot = 0; phase ^= 1u; }
        if (++islot == nst) islot = 0;
        const int4 hd = *reinterpret_cast<const int4 *>(blk);
        const int nr = hd.x, ne = hd.y, lvl = hd.w;
        const int4 *rows = reinterpret_cast<const int4 *>(blk + 16);
        const double *dg = reinterpret_cast<const double *>(blk + 16 + 16LL * nr);
        const int *code = reinterpret_cast<const int *>(blk + pu_off_code(nr));
        const double *val = reinterpret_cast<const double *>(blk + pu_off_val(nr, ne));
        const int *pl = reinterpret_cast<const int *>(val + ne);
        for (int q = grp; q < nr; q += ngrp) {
            const int4 R = rows[q];
            const double dq = dg[q];
            double sum = 0.0;
            for (int e = R.y + gl; e < R.z; e += G) sum += val[e] * xh[code[e]];
#pragma unroll
            for (int s = G / 2; s > 0; s >>= 1) sum += __shfl_xor_sync(gmask, sum, s, G);
            const double xr = (xh[R.x] - sum) * dq;   // dq = 1/t_ii (as SuperLU's pre-scaled solve)
            __syncwarp(gmask);
            if (gl == 0) xh[R.x] = xr;
            const int p0 = R.w >> 4, pc = R.w & 15;
            for (int u = gl; u < pc; u += G) {
                const int pe = pl[p0 + u];
                const int dst = (int)((unsigned)pe >> 28);
                const unsigned sl = (unsigned)pe & 0x0fffffffu;
                asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
                             ::"r"(peer[dst] + 8u * sl), "l"(__double_as_longlong(xr)), "r"(peer[16 + dst] + 8u * lvl)
                             : "memory");
            }
        }
        if (dbg) { __syncwarp(); if (lane == 0) t_done[st & 1][threadIdx.x >> 5] = gtimer(); }
    }
    __syncthreads();
    pdl_trigger();   // the dependent kernel's launch overlaps the x write-out below
    if (dbg && threadIdx.x == blockDim.x - 32 && S > 0) {
        unsigned long long m = 0;
        for (int w = 0; w < 32; ++w) m = max(m, t_done[(S - 1) & 1][w]);
        dbg[((size_t)blockIdx.x * smax + S - 1) * 6 + 5] = m;
    }
    for (int i = threadIdx.x; i < mine; i += blockDim.x) {
        const size_t g = (size_t)(base + i) * ncomp + comp;
        x[g] = xh[i];
        if (xout) xout[g] = xadd[g] + xh[i];
    }
}

// ----------------------------------------------------------------- dataflow variant
// Same plan, same arithmetic, no per-level synchronisation: x slots (own slice and
// halo) start as a NaN sentinel, a solved row is stored into its own slot and pushed
// with plain remote stores into its consumers' halo slots, and every entry a row reads
// is polled until it is no longer the sentinel.  A lane group moves on to its next row
// as soon as that row's inputs exist, so the critical path is the dependency chain
// (mostly shared-memory hops inside a CTA) instead of levels x (slowest producer + push
// + barrier).  The blocks are streamed by a dedicated producer warp through a ring of
// full / empty mbarriers (consumer warps release a slot after its rows).
constexpr unsigned long long PU_SENT = 0xFFFFFFFFFFFFFFFFull;
__device__ __forceinline__ double ld_vol_shared(unsigned a) {
    unsigned long long v;
    asm volatile("ld.volatile.shared.b64 %0, [%1];" : "=l"(v) : "r"(a));
    return __longlong_as_double((long long)v);
}
__device__ __forceinline__ void st_vol_shared(unsigned a, double v) {
    asm volatile("st.volatile.shared.b64 [%0], %1;" ::"r"(a), "l"(__double_as_longlong(v)) : "memory");
}
__device__ __forceinline__ int ld_vol_u8(unsigned a) {
    unsigned short v;
    asm volatile("ld.volatile.shared.u8 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void st_vol_u8(unsigned a, int v) {
    asm volatile("st.volatile.shared.u8 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ void st_remote(unsigned a, double v) {
    asm volatile("st.relaxed.cluster.shared::cluster.b64 [%0], %1;" ::"r"(a), "l"(__double_as_longlong(v)) : "memory");
}

template <int G>
__global__ void __launch_bounds__(PU_THREADS, 1)
    k_trsv_flow(int n, int ncomp, int chunk, int L, int smax, int hmax, int stage, int nst,
                const unsigned char *__restrict__ blocks, const long long *__restrict__ boff,
                const int *__restrict__ sstart, const double *__restrict__ b, double *__restrict__ x,
                const double *__restrict__ xadd, double *__restrict__ xout, int l2pf, unsigned long long *dbg) {
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned long long *mfull = reinterpret_cast<unsigned long long *>(smem);
    unsigned long long *mempty = mfull + PU_NST_MAX;   // the level-mbarrier area (L >= nst)
    double *xh = reinterpret_cast<double *>(smem + 8 * PU_NST_MAX + p16(8LL * L));
    long long *boff_s = reinterpret_cast<long long *>(xh + pu_chunkp(chunk) + p16(8LL * hmax) / 8);
    unsigned *peer = reinterpret_cast<unsigned *>(boff_s + p16(8LL * (smax + 1)) / 8);
    unsigned char *ring = smem + pu_fixed(chunk, L, hmax, smax);
    cg::cluster_group cl = cg::this_cluster();
    const int k = (int)cl.block_rank(), C = (int)cl.num_blocks();
    const int comp = blockIdx.x / C;
    const int s0 = sstart[k], S = sstart[k + 1] - s0;
    const int nw = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gl = threadIdx.x & (G - 1), grp = threadIdx.x / G, ngrp = (blockDim.x - 32) / G;
    const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1) << (lane & ~(G - 1)));
    const int base = k * chunk, mine = min(chunk, n - base);
    const int chunkp = pu_chunkp(chunk);
    if (threadIdx.x < nst) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mfull[threadIdx.x])) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&mempty[threadIdx.x])), "r"(nw - 1) : "memory");
    }
    if (threadIdx.x < C) peer[threadIdx.x] = mapa_u32(su32(xh + chunkp), threadIdx.x);
    for (int i = threadIdx.x; i <= S; i += blockDim.x) boff_s[i] = boff[s0 + i];
    // own rows: x slot seeded with b (as the level-synchronous kernel), readiness in a
    // byte flag behind the ring; halo slots: the NaN sentinel until the push lands
    pdl_wait();   // b is the previous kernel's output
    double *bsl = reinterpret_cast<double *>(ring + (size_t)nst * stage);
    const double sent = __longlong_as_double((long long)PU_SENT);
    for (int i = threadIdx.x; i < mine; i += blockDim.x) {
        bsl[i] = b[(size_t)(base + i) * ncomp + comp];
        xh[i] = sent;
    }
    for (int i = threadIdx.x; i < hmax; i += blockDim.x) xh[chunkp + i] = sent;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    // every CTA's slots hold the sentinel before anyone pushes
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    // ring slots of `stage` bytes hold runs of consecutive (CTA, level) blocks (contiguous in
    // the plan): one TMA copy, one full / empty mbarrier round per run instead of per level
    auto run_end = [&](int a) {
        int e = a + 1;
        while (e < S && boff_s[e + 1] - boff_s[a] <= stage) ++e;
        return e;
    };
    if (wid == nw - 1) {   // producer warp: TMA ring
        if (lane == 0) {
            int pa = 0, pq = 0;   // L2 prefetch cursor (runs ahead of the copies)
            for (int a = 0, j = 0; a < S; ++j) {
                const int e = run_end(a), sl = j % nst;
                if (j >= nst) mwait(su32(&mempty[sl]), (unsigned)((j / nst - 1) & 1));
                const unsigned bytes = (unsigned)(boff_s[e] - boff_s[a]);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mfull[sl])), "r"(bytes)
                             : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(su32(ring + (size_t)sl * stage)), "l"(blocks + boff_s[a]), "r"(bytes),
                             "r"(su32(&mfull[sl]))
                             : "memory");
                while (l2pf && pa < S && pq < j + nst + l2pf) {
                    const int pe = run_end(pa);
                    if (pq >= j + nst) {
                        const unsigned pb = (unsigned)(boff_s[pe] - boff_s[pa]);
                        if (pb) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(blocks + boff_s[pa]), "r"(pb) : "memory");
                    }
                    pa = pe;
                    ++pq;
                }
                a = e;
            }
        }
    } else {
        const unsigned xh_s = su32(xh);
        for (int a = 0, j = 0; a < S; ++j) {
          const int e_run = run_end(a), sl = j % nst;
          mwait(su32(&mfull[sl]), (unsigned)((j / nst) & 1));
          unsigned long long t_land = 0;
          if (dbg && lane == 0) t_land = gtimer();
          for (int t = a; t < e_run; ++t) {
            const unsigned char *blk = ring + (size_t)sl * stage + (boff_s[t] - boff_s[a]);
            const int4 hd = *reinterpret_cast<const int4 *>(blk);
            const int nr = hd.x, ne = hd.y;
            const int4 *rows = reinterpret_cast<const int4 *>(blk + 16);
            const double *dg = reinterpret_cast<const double *>(blk + 16 + 16LL * nr);
            const int *code = reinterpret_cast<const int *>(blk + pu_off_code(nr));
            const double *val = reinterpret_cast<const double *>(blk + pu_off_val(nr, ne));
            const int *pl = reinterpret_cast<const int *>(val + ne);
            // warp-uniform row loop and polling (a spinning lane group must not hold back
            // the other groups of its warp): the groups of a warp take consecutive rows
            const int g0 = (wid * 32) / G;   // first group of this warp
            for (int q0 = g0; q0 < nr; q0 += ngrp) {
                const int q = q0 + (grp - g0);
                const bool act = q < nr;
                int4 R = make_int4(0, 0, 0, 0);
                double dq = 0.0, bi = 0.0;
                if (act) {
                    R = rows[q];
                    dq = dg[q];
                    bi = bsl[R.x];
                }
                int len = R.z - R.y;
                len = __reduce_max_sync(0xffffffffu, len);
                // RND entries per lane loaded before any is waited on (independent loads in
                // flight); per lane the products are added in the same e order as before
                constexpr int RND = 4;
                double sum = 0.0;
                for (int e0 = 0; e0 < len; e0 += G * RND) {
                    unsigned xa[RND];
                    double v[RND], xv[RND];
                    bool has[RND];
#pragma unroll
                    for (int r = 0; r < RND; ++r) {
                        const int e = R.y + e0 + r * G + gl;
                        has[r] = act && e < R.z;
                        xa[r] = has[r] ? xh_s + 8u * (unsigned)code[e] : 0u;
                        v[r] = has[r] ? val[e] : 0.0;
                    }
#pragma unroll
                    for (int r = 0; r < RND; ++r) xv[r] = has[r] ? ld_vol_shared(xa[r]) : 0.0;
                    auto pending = [&] {
                        bool w = false;
#pragma unroll
                        for (int r = 0; r < RND; ++r) w |= has[r] && __double_as_longlong(xv[r]) == (long long)PU_SENT;
                        return w;
                    };
                    long long spins = 0;
                    while (__any_sync(0xffffffffu, pending())) {
#pragma unroll
                        for (int r = 0; r < RND; ++r)
                            if (has[r] && __double_as_longlong(xv[r]) == (long long)PU_SENT) xv[r] = ld_vol_shared(xa[r]);
                        if (++spins > (1ll << 28)) __trap();
                    }
#pragma unroll
                    for (int r = 0; r < RND; ++r)
                        if (has[r]) sum += v[r] * xv[r];
                }
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o, G);
                if (act) {
                    double xr = (bi - sum) * dq;   // dq = 1/t_ii (as SuperLU's pre-scaled solve)
                    if (__double_as_longlong(xr) == (long long)PU_SENT) xr = __longlong_as_double(0x7ff8000000000000ll);
                    if (gl == 0) st_vol_shared(xh_s + 8u * (unsigned)R.x, xr);
                    const int p0 = R.w >> 4, pc = R.w & 15;
                    for (int u = gl; u < pc; u += G) {
                        const int pe = pl[p0 + u];
                        st_remote(peer[(unsigned)pe >> 28] + 8u * ((unsigned)pe & 0x0fffffffu), xr);
                    }
                }
            }
            __syncwarp();
            if (dbg && lane == 0 && (wid * 32) / G < nr) {   // warps with rows: landed / done (ns)
                unsigned long long *o = dbg + ((size_t)blockIdx.x * smax + t) * 4;
                atomicMin(o + 0, t_land);
                atomicMax(o + 1, gtimer());
                o[2] = hd.w;
                o[3] = nr;
            }
          }
          __syncwarp();
          if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&mempty[sl])) : "memory");
          a = e_run;
        }
    }
    __syncthreads();
    pdl_trigger();
    for (int i = threadIdx.x; i < mine; i += blockDim.x) {
        const size_t g = (size_t)(base + i) * ncomp + comp;
        x[g] = xh[i];
        if (xout) xout[g] = xadd[g] + xh[i];
    }
}

// ----------------------------------------------------------------- setup
__global__ void k_pu_keys(int n, int chunk, int L, const int *lev, int *key, int *rows) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        key[r] = (r / chunk) * L + lev[r];
        rows[r] = r;
    }
}
__global__ void k_pu_key_ptr(int n, const int *skey, int nkeys, int *lp) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x) {
        const int v = i < n ? skey[i] : nkeys;
        const int prev = i ? skey[i - 1] : -1;
        for (int k = prev + 1; k <= v && k <= nkeys; ++k) lp[k] = i;
    }
}
__global__ void k_pu_cross_count(int n, int chunk, const int *ptr, const int *idx, int *cnt) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        int c = 0;
        for (int p = ptr[r]; p < ptr[r + 1]; ++p) c += (idx[p] / chunk) != (r / chunk);
        cnt[r] = c;
    }
}
__global__ void k_pu_cross_fill(int n, int chunk, const int *ptr, const int *idx, const int *xptr,
                                unsigned long long *keys) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        int w = xptr[r];
        const unsigned long long d = (unsigned long long)(r / chunk);
        for (int p = ptr[r]; p < ptr[r + 1]; ++p)
            if ((idx[p] / chunk) != (r / chunk)) keys[w++] = (d << 32) | (unsigned)idx[p];
    }
}
// hstart[d] = first halo pair of consumer d (pairs sorted by (d, j))
__global__ void k_pu_hstart(int nh, const unsigned long long *h, int C, int *hstart) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d > C) return;
    const unsigned long long key = (unsigned long long)d << 32;
    int lo = 0, hi = nh;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (h[mid] < key) lo = mid + 1; else hi = mid;
    }
    hstart[d] = lo;
}
// push pairs keyed by source row: (j << 4 | d) -> slot; byte counts per (consumer, level of j)
__global__ void k_pu_push_keys(int nh, const unsigned long long *h, const int *hstart, int L, const int *lev,
                               unsigned long long *k2, int *slot, int *tx) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nh; i += gridDim.x * blockDim.x) {
        const int d = (int)(h[i] >> 32), j = (int)(h[i] & 0xffffffffu);
        k2[i] = ((unsigned long long)j << 4) | (unsigned)d;
        slot[i] = i - hstart[d];
        atomicAdd(&tx[d * L + lev[j]], 8);
    }
}
// pptr[j] = first push pair of source row j
__global__ void k_pu_pptr(int nh, const unsigned long long *k2s, int n, int *pptr) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= nh; i += gridDim.x * blockDim.x) {
        const int v = i < nh ? (int)(k2s[i] >> 4) : n;
        const int prev = i ? (int)(k2s[i - 1] >> 4) : -1;
        for (int j = prev + 1; j <= v && j <= n; ++j) pptr[j] = i;
    }
}
__global__ void k_pu_lens(int n, const int *perm, const int *ptr, const int *pptr, int *len, int *plen) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        const int r = perm[q];
        len[q] = ptr[r + 1] - ptr[r];
        plen[q] = pptr[r + 1] - pptr[r];
    }
}
__global__ void k_pu_headers(int np_, const int *pstart, const int *plev, const int *rptr, const int *rpp,
                             unsigned char *blocks, const long long *boff) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < np_; i += gridDim.x * blockDim.x) {
        int *h = reinterpret_cast<int *>(blocks + boff[i]);
        h[0] = pstart[i + 1] - pstart[i];
        h[1] = rptr[pstart[i + 1]] - rptr[pstart[i]];
        h[2] = rpp[pstart[i + 1]] - rpp[pstart[i]];
        h[3] = plev[i];
    }
}
__global__ void k_pu_fill(int n, int chunk, int chunkp, int np_, const int *pstart, const int *perm,
                          const int *rptr, const int *rpp, const long long *boff, const int *ptr, const int *idx,
                          const double *val, const double *diag, const unsigned long long *h, const int *hstart,
                          const int *pptr, const unsigned long long *k2s, const int *slots, unsigned char *blocks) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        int lo = 0, hi = np_;   // part holding sorted row q: last part with pstart <= q
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (pstart[mid] <= q) lo = mid; else hi = mid;
        }
        const int blk = lo;
        const int q0 = pstart[blk], nr = pstart[blk + 1] - q0, i = q - q0;
        const int ne = rptr[pstart[blk + 1]] - rptr[q0];
        unsigned char *B = blocks + boff[blk];
        const int r = perm[q];
        const int owner = r / chunk;
        int4 *rows = reinterpret_cast<int4 *>(B + 16);
        double *dg = reinterpret_cast<double *>(B + 16 + 16LL * nr);
        int *code = reinterpret_cast<int *>(B + pu_off_code(nr));
        double *vv = reinterpret_cast<double *>(B + pu_off_val(nr, ne));
        int *pl = reinterpret_cast<int *>(vv + ne);
        const int e0 = rptr[q] - rptr[q0], e1 = rptr[q + 1] - rptr[q0];
        const int p0 = rpp[q] - rpp[q0], pc = rpp[q + 1] - rpp[q];
        rows[i] = make_int4(r - owner * chunk, e0, e1, (p0 << 4) | pc);
        dg[i] = diag ? 1.0 / diag[r] : 1.0;
        int w = e0;
        const int hs = hstart[owner], he = hstart[owner + 1];
        for (int p = ptr[r]; p < ptr[r + 1]; ++p, ++w) {
            const int j = idx[p];
            const int o = j / chunk;
            if (o == owner) {
                code[w] = j - o * chunk;
            } else {
                const unsigned long long key = ((unsigned long long)owner << 32) | (unsigned)j;
                int lo = hs, hi = he;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (h[mid] < key) lo = mid + 1; else hi = mid;
                }
                code[w] = chunkp + (lo - hs);
            }
            vv[w] = val[p];
        }
        int u = p0;
        for (int t = pptr[r]; t < pptr[r + 1]; ++t, ++u)
            pl[u] = (int)(((unsigned)(k2s[t] & 15u) << 28) | (unsigned)slots[t]);
    }
}

template <typename T>
void cub_sort_keys(Ctx *c, T *in, T *out, int n, int end_bit) {
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, in, out, n, 0, end_bit, c->s));
    DBuf<char> t(tb, c->s);
    CK(cub::DeviceRadixSort::SortKeys(t.p, tb, in, out, n, 0, end_bit, c->s));
    launched(c);
}

bool try_push(Ctx *c, Tri &T, const DBuf<int> &lev, int L, int C) {
    const int n = T.n;
    const int chunk = (n + C - 1) / C;
    const int nblk = C * L;
    const Csr &S = T.strict;
    // rows grouped by (owner CTA, level)
    DBuf<int> key(n, c->s), skey(n, c->s), rows(n, c->s), perm(n, c->s), lp((size_t)nblk + 1, c->s);
    k_pu_keys<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, chunk, L, lev.p, key.p, rows.p);
    launched(c);
    {
        int bits = 1;
        while (bits < 31 && (1 << bits) <= nblk) ++bits;
        size_t tb = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, skey.p, rows.p, perm.p, n, 0, bits, c->s));
        DBuf<char> t(tb, c->s);
        CK(cub::DeviceRadixSort::SortPairs(t.p, tb, key.p, skey.p, rows.p, perm.p, n, 0, bits, c->s));
        launched(c);
    }
    k_pu_key_ptr<<<grid_for(n + 1, 256, c->sms), 256, 0, c->s>>>(n, skey.p, nblk, lp.p);
    launched(c);
    // unique cross-CTA (consumer, source row) pairs -> halo slots
    DBuf<int> xcnt(n, c->s), xptr;
    k_pu_cross_count<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, chunk, S.ptr.p, S.idx.p, xcnt.p);
    launched(c);
    const int64_t X = counts_to_ptr(c, xcnt.p, n, xptr);
    int nh = 0;
    DBuf<unsigned long long> H;
    if (X > 0) {
        DBuf<unsigned long long> keys(X, c->s), skeys(X, c->s);
        k_pu_cross_fill<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, chunk, S.ptr.p, S.idx.p, xptr.p, keys.p);
        launched(c);
        int cb = 1;
        while ((1 << cb) <= C) ++cb;
        cub_sort_keys(c, keys.p, skeys.p, (int)X, 32 + cb);
        H.alloc(X, c->s);
        DBuf<int> nsel(1, c->s);
        size_t tb = 0;
        CK(cub::DeviceSelect::Unique(nullptr, tb, skeys.p, H.p, nsel.p, (int)X, c->s));
        DBuf<char> t(tb, c->s);
        CK(cub::DeviceSelect::Unique(t.p, tb, skeys.p, H.p, nsel.p, (int)X, c->s));
        launched(c);
        nh = nsel.to_host()[0];
    }
    DBuf<int> hstart(C + 1, c->s);
    k_pu_hstart<<<1, 32, 0, c->s>>>(nh, H.p, C, hstart.p);
    launched(c);
    std::vector<int> hh = hstart.to_host();
    int hmax = 0;
    for (int d = 0; d < C; ++d) hmax = std::max(hmax, hh[d + 1] - hh[d]);
    if (hmax >= (1 << 28)) return false;
    // push lists by source row, byte counts per (consumer, level)
    DBuf<unsigned long long> k2(std::max(nh, 1), c->s), k2s(std::max(nh, 1), c->s);
    DBuf<int> slot(std::max(nh, 1), c->s), slots(std::max(nh, 1), c->s), pptr(n + 1, c->s);
    auto P = std::make_unique<PushPlan>();
    P->tx.alloc((size_t)C * L, c->s);
    CK(cudaMemsetAsync(P->tx.p, 0, sizeof(int) * (size_t)C * L, c->s));
    if (nh > 0) {
        k_pu_push_keys<<<grid_for(nh, 256, c->sms), 256, 0, c->s>>>(nh, H.p, hstart.p, L, lev.p, k2.p, slot.p,
                                                                    P->tx.p);
        launched(c);
        int nb = 1;
        while (nb < 31 && (1LL << nb) <= n) ++nb;
        size_t tb = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, k2.p, k2s.p, slot.p, slots.p, nh, 0, 4 + nb, c->s));
        DBuf<char> t(tb, c->s);
        CK(cub::DeviceRadixSort::SortPairs(t.p, tb, k2.p, k2s.p, slot.p, slots.p, nh, 0, 4 + nb, c->s));
        launched(c);
    }
    k_pu_pptr<<<grid_for(nh + 1, 256, c->sms), 256, 0, c->s>>>(nh, k2s.p, n, pptr.p);
    launched(c);
    // block sizes
    DBuf<int> len(n, c->s), plen(n, c->s), rptr, rpp;
    k_pu_lens<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, perm.p, S.ptr.p, pptr.p, len.p, plen.p);
    launched(c);
    counts_to_ptr(c, len.p, n, rptr);
    counts_to_ptr(c, plen.p, n, rpp);
    // steps: the non-empty (CTA, level) blocks, each cut into parts of at most `cap` bytes
    std::vector<int> hlp = lp.to_host(), hr = rptr.to_host(), hp = rpp.to_host();
    auto part_bytes = [&](int q0, int q1) {
        return pu_block_bytes(q1 - q0, (long long)hr[q1] - hr[q0], (long long)hp[q1] - hp[q0]);
    };
    std::vector<int> pstart, plev, sstart(C + 1, 0);
    std::vector<long long> pboff;
    int smax = 0, widest = 1;
    long long mx = 16;
    bool ok = false;
    for (int tries = 0; tries < 4 && !ok; ++tries) {
        const int smax_est = tries == 0 ? L : smax;
        const size_t fixed = pu_fixed(chunk, L, hmax, smax_est);
        if (fixed + 2 * 16384 >= PU_SMEM_LIMIT) return false;
        long long cap = (long long)(PU_SMEM_LIMIT - fixed) / 3;
        if (cap < 16384) cap = (long long)(PU_SMEM_LIMIT - fixed) / 2;
        cap &= ~127LL;
        pstart.clear(); plev.clear(); pboff.assign(1, 0);
        smax = 0; mx = 16; widest = 1;
        bool fit = true;
        for (int d = 0; d < C && fit; ++d) {
            sstart[d] = (int)plev.size();
            for (int l = 0; l < L && fit; ++l) {
                const int a0 = hlp[d * L + l], a1 = hlp[d * L + l + 1];
                for (int q = a0; q < a1;) {
                    int e = q + 1;
                    if (part_bytes(q, e) > cap) { fit = false; break; }
                    while (e < a1 && part_bytes(q, e + 1) <= cap) ++e;
                    const long long by = part_bytes(q, e);
                    pstart.push_back(q); plev.push_back(l); pboff.push_back(pboff.back() + by);
                    mx = std::max(mx, by);
                    widest = std::max(widest, e - q);
                    q = e;
                }
            }
            smax = std::max(smax, (int)plev.size() - sstart[d]);
        }
        if (!fit) return false;
        sstart[C] = (int)plev.size();
        ok = smax <= smax_est;
    }
    if (!ok) return false;
    const int np_ = (int)plev.size();
    pstart.push_back(n);
    const size_t fixed = pu_fixed(chunk, L, hmax, smax);
    const long long stage = (mx + 127) & ~127LL;
    const int nst = (int)std::min<long long>(PU_NST_MAX, (long long)(PU_SMEM_LIMIT - fixed) / stage);
    if (nst < 2) return false;
    const long long total = pboff.back();
    DBuf<int> dpstart((size_t)np_ + 1, c->s), dplev((size_t)std::max(np_, 1), c->s);
    dpstart.upload(pstart.data(), pstart.size());
    dplev.upload(plev.data(), plev.size());
    P->sstart.alloc(C + 1, c->s);
    P->sstart.upload(sstart.data(), sstart.size());
    P->boff.alloc((size_t)np_ + 1, c->s);
    P->boff.upload(pboff.data(), pboff.size());
    P->C = C;
    P->chunk = chunk;
    P->L = L;
    P->smax = smax;
    P->hmax = hmax;
    P->stage = (int)stage;
    P->nst = nst;
    const double avg = (double)S.nnz / n;
    P->G = 2;
    while (P->G < 32 && P->G * 4 < avg) P->G *= 2;
    static const int force_g = [] { const char *e = std::getenv("DPP_PU_G"); return e ? std::atoi(e) : 0; }();
    if (force_g && P->G < force_g) P->G = force_g;   // experiment: wider lane groups for thin rows
    static const int set_g = [] { const char *e = std::getenv("DPP_PU_GSET"); return e ? std::atoi(e) : 0; }();
    if (set_g && n == set_g / 100) P->G = set_g % 100;   // experiment: G for one triangle size (n*100+G)
    int threads = 64;
    while (threads < PU_THREADS && (threads / P->G) < widest) threads *= 2;
    static const int force_thr = [] { const char *e = std::getenv("DPP_PU_THREADS"); return e ? std::atoi(e) : 0; }();
    if (force_thr) threads = std::min(threads, force_thr);
    P->threads = threads;
    P->blocks.alloc((size_t)total, c->s);
    if (np_) {
        k_pu_headers<<<grid_for(np_, 256, c->sms), 256, 0, c->s>>>(np_, dpstart.p, dplev.p, rptr.p, rpp.p,
                                                                   P->blocks.p, P->boff.p);
        launched(c);
        k_pu_fill<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, chunk, pu_chunkp(chunk), np_, dpstart.p, perm.p,
                                                              rptr.p, rpp.p, P->boff.p, S.ptr.p, S.idx.p, S.val.p,
                                                              T.diag.n ? T.diag.p : nullptr, H.p, hstart.p, pptr.p,
                                                              k2s.p, slots.p, P->blocks.p);
        launched(c);
    }
    CK(cudaStreamSynchronize(c->s));
    if (TraceScope::on())
        std::fprintf(stderr, "[dpp-trace]   push_plan n=%d C=%d L=%d steps max %d G=%d thr=%d halo max %d (pairs %d) stage=%lld nst=%d\n",
                     n, C, L, smax, P->G, threads, hmax, nh, stage, nst);
    T.pu = std::move(P);
    return true;
}

}  // namespace

bool push_plan(Ctx *c, Tri &T, const DBuf<int> &lev, int L) {
    const int n = T.n;
    if (n == 0 || L < 1 || L > PU_LMAX) return false;
    static bool attr = false;
    if (!attr) {
        auto setk = [](const void *f) {
            CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PU_SMEM_LIMIT));
            CK(cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        };
        setk((const void *)k_trsv_push<2>);
        setk((const void *)k_trsv_push<4>);
        setk((const void *)k_trsv_push<8>);
        setk((const void *)k_trsv_push<16>);
        setk((const void *)k_trsv_push<32>);
        setk((const void *)k_trsv_flow<2>);
        setk((const void *)k_trsv_flow<4>);
        setk((const void *)k_trsv_flow<8>);
        setk((const void *)k_trsv_flow<16>);
        setk((const void *)k_trsv_flow<32>);
        attr = true;
    }
    // as many CTAs as useful: each keeps >= ~2k rows of x
    const int C0 = std::max(2, std::min(PU_MAX, (n + 2047) / 2048));
    for (int C = C0; C <= PU_MAX; ++C)
        if (try_push(c, T, lev, L, C)) return true;
    return false;
}

void trsv_push(Ctx *c, const Tri &T, const double *b, double *x, const double *xadd, double *xout,
               cudaStream_t st) {
    const PushPlan &P = *T.pu;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P.C * T.ncomp, 1, 1);
    cfg.blockDim = dim3(P.threads, 1, 1);
    cfg.dynamicSmemBytes = pu_fixed(P.chunk, P.L, P.hmax, P.smax) + (size_t)P.nst * P.stage;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = P.C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_on() ? 2 : 1;
    const unsigned char *B = P.blocks.p;
    const long long *O = P.boff.p;
    static const int l2pf = [] { const char *e = std::getenv("DPP_PU_NOPF"); return e && *e == '1' ? 0 : 4; }();
    static const char *dbg_path = std::getenv("DPP_PU_DEBUG");
    const size_t nd = (size_t)P.C * T.ncomp * std::max(P.smax, 1) * 6;
    unsigned long long *dbg = nullptr;
    if (dbg_path && *dbg_path && !c->capturing) {
        CK(cudaMallocAsync((void **)&dbg, sizeof(unsigned long long) * nd, st));
        CK(cudaMemsetAsync(dbg, 0, sizeof(unsigned long long) * nd, st));
    }
    const int *wp = T.W.rows ? (const int *)T.W.ptr.p : nullptr, *wi = T.W.rows ? (const int *)T.W.idx.p : nullptr;
    const double *wv = T.W.rows ? (const double *)T.W.val.p : nullptr;
    cudaError_t e;
    static const bool flow = [] { const char *e = std::getenv("DPP_PU_FLOW"); return !(e && *e == '0'); }();
    const size_t fixed = pu_fixed(P.chunk, P.L, P.hmax, P.smax), flags = (size_t)p16(8LL * P.chunk);   // b slice
    const int nst_b = (int)std::min<size_t>(P.nst, (PU_SMEM_LIMIT - fixed - flags) / P.stage);
    // the ring's bytes regrouped into 2 large slots (runs of blocks per slot; 2 slots measured
    // best: 1.75 vs 1.82 / 1.84 / 1.89 ms per C2 PC apply for 3 / 4 / per-block slots)
    static const int flow_slots = [] { const char *e = std::getenv("DPP_FLOW_SLOTS"); return e ? std::atoi(e) : 2; }();
    const int nst_f = std::max(1, std::min(nst_b, flow_slots));
    const long long stage_f = nst_b >= 2 ? ((long long)nst_b * P.stage / nst_f) & ~15LL : P.stage;
    static const char *fdbg_path = std::getenv("DPP_FLOW_DEBUG");
    unsigned long long *fdbg = nullptr;
    const size_t nfd = (size_t)P.C * T.ncomp * std::max(P.smax, 1) * 4;
    if (fdbg_path && *fdbg_path && !c->capturing && flow) {
        CK(cudaMallocAsync((void **)&fdbg, sizeof(unsigned long long) * nfd, st));
        std::vector<unsigned long long> init(nfd, 0);
        for (size_t i = 0; i < nfd; i += 4) init[i] = ~0ull;
        CK(cudaMemcpyAsync(fdbg, init.data(), nfd * 8, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
    }
    // dataflow for thin rows (C2: G = 2 / 8); the level-synchronous kernel measured faster for
    // the 32-lane groups of the long-row triangles of configs 3/4 (34.0 vs 37.8 ms per PC apply at C3)
    static const int flow_gmax = [] { const char *e = std::getenv("DPP_FLOW_GMAX"); return e ? std::atoi(e) : 16; }();
    if (flow && P.G <= flow_gmax && !wp && !dbg && P.L >= nst_f && nst_b >= 2 && nst_f >= 2 &&
        fixed + flags + (size_t)nst_f * stage_f <= PU_SMEM_LIMIT) {
        cfg.blockDim = dim3(std::min(PU_THREADS, P.threads + 32), 1, 1);
        cfg.dynamicSmemBytes = fixed + (size_t)nst_f * stage_f + flags;
        switch (P.G) {
            case 2: e = cudaLaunchKernelEx(&cfg, k_trsv_flow<2>, T.n / T.ncomp, T.ncomp, P.chunk, P.L, P.smax, P.hmax, (int)stage_f, nst_f, B, O, (const int *)P.sstart.p, b, x, xadd, xout, l2pf, fdbg); break;
            case 4: e = cudaLaunchKernelEx(&cfg, k_trsv_flow<4>, T.n / T.ncomp, T.ncomp, P.chunk, P.L, P.smax, P.hmax, (int)stage_f, nst_f, B, O, (const int *)P.sstart.p, b, x, xadd, xout, l2pf, fdbg); break;
            case 8: e = cudaLaunchKernelEx(&cfg, k_trsv_flow<8>, T.n / T.ncomp, T.ncomp, P.chunk, P.L, P.smax, P.hmax, (int)stage_f, nst_f, B, O, (const int *)P.sstart.p, b, x, xadd, xout, l2pf, fdbg); break;
            case 16: e = cudaLaunchKernelEx(&cfg, k_trsv_flow<16>, T.n / T.ncomp, T.ncomp, P.chunk, P.L, P.smax, P.hmax, (int)stage_f, nst_f, B, O, (const int *)P.sstart.p, b, x, xadd, xout, l2pf, fdbg); break;
            default: e = cudaLaunchKernelEx(&cfg, k_trsv_flow<32>, T.n / T.ncomp, T.ncomp, P.chunk, P.L, P.smax, P.hmax, (int)stage_f, nst_f, B, O, (const int *)P.sstart.p, b, x, xadd, xout, l2pf, fdbg); break;
        }
        CK(e);
        launched(c);
        if (fdbg) {   // "# n C ncomp smax" then per (cta, step): cta step level rows t_land t_done
            std::vector<unsigned long long> h(nfd);
            CK(cudaMemcpyAsync(h.data(), fdbg, nfd * 8, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            cudaFreeAsync(fdbg, st);
            if (FILE *f = std::fopen(fdbg_path, "a")) {
                std::fprintf(f, "# n=%d C=%d ncomp=%d smax=%d L=%d G=%d\n", T.n, P.C, T.ncomp, P.smax, P.L, P.G);
                for (size_t i = 0; i < nfd / 4; ++i) {
                    const unsigned long long *o = &h[i * 4];
                    if (o[1]) std::fprintf(f, "%zu %zu %llu %llu %llu %llu\n", i / P.smax, i % P.smax, o[2], o[3], o[0], o[1]);
                }
                std::fclose(f);
            }
        }
        return;
    }
    switch (P.G) {
        case 2: e = cudaLaunchKernelEx(&cfg, k_trsv_push<2>, T.n / T.ncomp, T.ncomp, P.chunk, P.L, P.smax, P.hmax, P.stage, P.nst, B, O, (const int *)P.sstart.p, (const int *)P.tx.p, wp, wi, wv, b, x, xadd, xout, l2pf, dbg); break;
        case 4: e = cudaLaunchKernelEx(&cfg, k_trsv_push<4>, T.n / T.ncomp, T.ncomp, P.chunk, P.L, P.smax, P.hmax, P.stage, P.nst, B, O, (const int *)P.sstart.p, (const int *)P.tx.p, wp, wi, wv, b, x, xadd, xout, l2pf, dbg); break;
        case 8: e = cudaLaunchKernelEx(&cfg, k_trsv_push<8>, T.n / T.ncomp, T.ncomp, P.chunk, P.L, P.smax, P.hmax, P.stage, P.nst, B, O, (const int *)P.sstart.p, (const int *)P.tx.p, wp, wi, wv, b, x, xadd, xout, l2pf, dbg); break;
        case 16: e = cudaLaunchKernelEx(&cfg, k_trsv_push<16>, T.n / T.ncomp, T.ncomp, P.chunk, P.L, P.smax, P.hmax, P.stage, P.nst, B, O, (const int *)P.sstart.p, (const int *)P.tx.p, wp, wi, wv, b, x, xadd, xout, l2pf, dbg); break;
        default: e = cudaLaunchKernelEx(&cfg, k_trsv_push<32>, T.n / T.ncomp, T.ncomp, P.chunk, P.L, P.smax, P.hmax, P.stage, P.nst, B, O, (const int *)P.sstart.p, (const int *)P.tx.p, wp, wi, wv, b, x, xadd, xout, l2pf, dbg); break;
    }
    CK(e);
    launched(c);
    if (dbg) {   // append "n C ncomp smax" then one line per (cta, step)
        std::vector<unsigned long long> h(nd);
        CK(cudaMemcpyAsync(h.data(), dbg, nd * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        cudaFreeAsync(dbg, st);
        if (FILE *f = std::fopen(dbg_path, "a")) {
            std::fprintf(f, "# n=%d C=%d ncomp=%d smax=%d L=%d G=%d\n", T.n, P.C, T.ncomp, P.smax, P.L, P.G);
            for (size_t i = 0; i < nd / 6; ++i) {
                const unsigned long long *o = &h[i * 6];
                if (o[4]) std::fprintf(f, "%zu %zu %llu %llu %llu %llu %llu %llu\n", i / P.smax, i % P.smax, o[0], o[1], o[2], o[3], o[4], o[5]);
            }
            std::fclose(f);
        }
    }
}

}  // namespace dpp
