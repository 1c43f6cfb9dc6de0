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
#include <cstring>

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
#ifdef LV_BACKOFF
        __nanosleep(LV_BACKOFF);
#endif
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

// block layout of the level-mbarrier sweep (16-byte aligned), rows in 32-row chunks whose
// entries are stored column by column (SELL-32: entry k of the chunk's lane-l row at
// ebase + 32 k + l, so a warp's 32 lanes read 32 consecutive words -- no bank conflicts):
//   int4 {nr, nch, np, level} | int4 chunk[nch] {ebase, nE, nL, 0} | int2 row[nr] {local row,
//   p0 << 4 | npush} | double dq[nr] | int code[NE] | double val[NE] | int push[np]
// where a chunk holds nE early columns (sources of level <= l-2) then nL late ones (level
// l-1), padded with (zero slot, 0.0) entries.
__host__ __device__ inline long long lv_off_rw(long long nch) { return 16 + 16 * nch; }
__host__ __device__ inline long long lv_off_dq(long long nch, long long nr) { return p16(lv_off_rw(nch) + 8 * nr); }
__host__ __device__ inline long long lv_off_code(long long nch, long long nr) { return p16(lv_off_dq(nch, nr) + 8 * nr); }
__host__ __device__ inline long long lv_off_val(long long nch, long long nr, long long ne) {
    return p16(lv_off_code(nch, nr) + 2 * ne);
}
__host__ __device__ inline long long lv_block_bytes(long long nch, long long nr, long long ne, long long np) {
    return p16(lv_off_val(nch, nr, ne) + 8 * ne + 4 * np);
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
            const int rx = R.x & 0xffff;   // local row (upper bits: late-entry count, k_trsv_lvl)
            const double xr = (xh[rx] - sum) * dq;   // dq = 1/t_ii (as SuperLU's pre-scaled solve)
            __syncwarp(gmask);
            if (gl == 0) xh[rx] = xr;
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
#ifdef DPP_FLOW_PHASES
// per (CTA, warp): cycles in {ring wait, row header, loads+poll, fma+reduce, store+push, idle},
// row-group iterations, spin rounds (profiling build only: tools/flow_phases.sh)
__device__ unsigned long long *g_flow_phase = nullptr;
__device__ unsigned long long *g_flow_tl = nullptr;   // per (CTA, step): {level, min t late-wait done, max t arrive}
__device__ int g_flow_smax = 0;
__device__ int g_flow_nopush = 0;
__device__ int g_flow_rot = 0;
__device__ __forceinline__ long long clk() { long long t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)); return t; }
#define PH_T(v) const long long v = clk()
#define PH_ADD(i, d) ph[i] += (d)
#else
#define PH_T(v)
#define PH_ADD(i, d)
#endif
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
#ifdef DPP_FLOW_PHASES
        long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        long long t_last = clk();
#endif
        for (int a = 0, j = 0; a < S; ++j) {
          const int e_run = run_end(a), sl = j % nst;
          PH_T(tw0);
          mwait(su32(&mfull[sl]), (unsigned)((j / nst) & 1));
          PH_T(tw1);
          PH_ADD(0, tw1 - tw0);
          unsigned long long t_land = 0;
          if (dbg && lane == 0) t_land = gtimer();
          for (int t = a; t < e_run; ++t) {
            const unsigned char *blk = ring + (size_t)sl * stage + (boff_s[t] - boff_s[a]);
            DPP_DCHECK(boff_s[t + 1] - boff_s[a] <= stage);   // the block lies inside its ring slot
            const int4 hd = *reinterpret_cast<const int4 *>(blk);
            const int nr = hd.x, ne = hd.y;
            DPP_DCHECK(nr >= 0 && ne >= 0 && hd.w >= 0 && hd.w < L && pu_block_bytes(nr, ne, hd.z) <= boff_s[t + 1] - boff_s[t]);
            const int4 *rows = reinterpret_cast<const int4 *>(blk + 16);
            const double *dg = reinterpret_cast<const double *>(blk + 16 + 16LL * nr);
            const int *code = reinterpret_cast<const int *>(blk + pu_off_code(nr));
            const double *val = reinterpret_cast<const double *>(blk + pu_off_val(nr, ne));
            const int *pl = reinterpret_cast<const int *>(val + ne);
            // warp-uniform row loop and polling (a spinning lane group must not hold back
            // the other groups of its warp): the groups of a warp take consecutive rows
            const int g0 = (wid * 32) / G;   // first group of this warp
            for (int q0 = g0; q0 < nr; q0 += ngrp) {
                PH_T(t0);
#ifdef DPP_FLOW_PHASES
                PH_ADD(5, t0 - t_last);
#endif
                const int q = q0 + (grp - g0);
                const bool act = q < nr;
                int4 R = make_int4(0, 0, 0, 0);
                double dq = 0.0, bi = 0.0;
                if (act) {
                    R = rows[q];
                    dq = dg[q];
                    DPP_DCHECK((R.x & 0xffff) < mine && R.y >= 0 && R.y <= R.z && R.z <= ne);
                    bi = bsl[R.x & 0xffff];
                }
                int len = R.z - R.y;
                len = __reduce_max_sync(0xffffffffu, len);
                PH_T(t1);
                PH_ADD(1, t1 - t0);
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
                        DPP_DCHECK(!has[r] || (code[e] >= 0 && (code[e] < mine || (code[e] >= chunkp && code[e] < chunkp + hmax))));
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
                    PH_ADD(7, spins);
#pragma unroll
                    for (int r = 0; r < RND; ++r)
                        if (has[r]) sum += v[r] * xv[r];
                }
                PH_T(t2);
                PH_ADD(2, t2 - t1);
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o, G);
#ifdef DPP_FLOW_PHASES
                sum = __shfl_sync(0xffffffffu, sum, lane);   // materialise before the timestamp
#endif
                PH_T(t3);
                PH_ADD(3, t3 - t2);
                if (act) {
                    double xr = (bi - sum) * dq;   // dq = 1/t_ii (as SuperLU's pre-scaled solve)
                    if (__double_as_longlong(xr) == (long long)PU_SENT) xr = __longlong_as_double(0x7ff8000000000000ll);
                    if (gl == 0) st_vol_shared(xh_s + 8u * (unsigned)(R.x & 0xffff), xr);
                    const int p0 = R.w >> 4, pc = R.w & 15;
                    for (int u = gl; u < pc; u += G) {
                        const int pe = pl[p0 + u];
                        DPP_DCHECK((int)((unsigned)pe >> 28) < C && (int)((unsigned)pe & 0x0fffffffu) < hmax);
                        st_remote(peer[(unsigned)pe >> 28] + 8u * ((unsigned)pe & 0x0fffffffu), xr);
                    }
                }
                __syncwarp();
                PH_T(t4);
                PH_ADD(4, t4 - t3);
                PH_ADD(6, 1);
#ifdef DPP_FLOW_PHASES
                t_last = t4;
#endif
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
#ifdef DPP_FLOW_PHASES
        (void)t_last;
        if (lane == 0 && g_flow_phase)
            for (int i = 0; i < 8; ++i) g_flow_phase[((size_t)blockIdx.x * 32 + wid) * 8 + i] = ph[i];
#endif
    }
    __syncthreads();
    pdl_trigger();
    for (int i = threadIdx.x; i < mine; i += blockDim.x) {
        const size_t g = (size_t)(base + i) * ncomp + comp;
        x[g] = xh[i];
        if (xout) xout[g] = xadd[g] + xh[i];
    }
}

// ----------------------------------------------------------------- level-mbarrier variant
// Same plan and arithmetic again (so bit-for-bit the other two kernels), but readiness is
// tracked per level with one single-use mbarrier per (CTA, level), armed at launch with
//   count = local rows of the level + 1   and   tx = bytes pushed into this CTA from the level.
// A warp arrives once per step with the number of rows it solved (after its x stores: release),
// remote producers push with st.async + complete_tx, so a completed level mbarrier means every
// value of that level this CTA will read is in place.  Before its rows of level l a warp waits
// (hardware-suspended try_wait, no polling of x slots) on the levels from the CTA's previous
// step's level up to l-1; earlier levels are implied (the previous step's rows waited on them).
// Warps without rows in a step do nothing for it, so no warp spins on shared memory and the
// critical path per level is one wake-up + one row (measured phase breakdown: DESIGN.md §5).
constexpr int LV_THREADS = 512;
// Warp layout: warp w sits on SM sub-partition w % 4 and belongs to level team w % LV_TEAMS, so
// each team owns one sub-partition; there is no producer warp (the ring refills itself).
constexpr int LV_TEAMS = 4;   // level teams of k_trsv_lvl (and the plan's column classes)
constexpr int LV_NS_MAX = 16;  // ring slots (one block each)
// shared memory: ring mbarriers [2][LV_NS_MAX] | level mbarriers [L] | x slice | halo |
//                step offsets [smax+1] | step levels [smax] | peer addresses [32] | ring [ns][stage]
__host__ __device__ inline size_t lv_fixed(int chunk, int L, int hmax, int smax) {
    return 16 * LV_NS_MAX + p16(8LL * L) + p16(8LL * chunk) + p16(8LL * hmax) + p16(8LL * (smax + 1)) +
           p16(4LL * smax) + 128 + 4 * LV_NS_MAX + 16;
}
__device__ __forceinline__ bool mtest(unsigned a, unsigned parity) {
    unsigned ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(a), "r"(parity) : "memory");
    return ok;
}
__global__ void __launch_bounds__(LV_THREADS, 1)
    k_trsv_lvl(int n, int ncomp, int chunk, int L, int smax, int hmax, int stage, int ns,
               const unsigned char *__restrict__ blocks, const long long *__restrict__ boff,
               const int *__restrict__ tstart, const int *__restrict__ splev, const int *__restrict__ tx,
               const int *__restrict__ lrows, const double *__restrict__ b, double *__restrict__ x,
               const double *__restrict__ xadd, double *__restrict__ xout, int l2pf) {
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned long long *mfull = reinterpret_cast<unsigned long long *>(smem);
    unsigned long long *mempty = mfull + LV_NS_MAX;
    unsigned long long *mlev = mfull + 2 * LV_NS_MAX;
    double *xh = reinterpret_cast<double *>(smem + 16 * LV_NS_MAX + p16(8LL * L));
    const int chunkp = pu_chunkp(chunk);
    long long *boff_s = reinterpret_cast<long long *>(xh + chunkp + p16(8LL * hmax) / 8);
    int *slev = reinterpret_cast<int *>(boff_s + p16(8LL * (smax + 1)) / 8);
    unsigned *peer = reinterpret_cast<unsigned *>(slev + p16(4LL * smax) / 4);   // [0,16): halo, [16,32): mlev
    unsigned char *ring = smem + lv_fixed(chunk, L, hmax, smax);
    cg::cluster_group cl = cg::this_cluster();
    const int k = (int)cl.block_rank(), C = (int)cl.num_blocks();
    const int comp = blockIdx.x / C;
    const int s0 = tstart[k], S = tstart[k + 1] - s0;
    const int nw = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int base = k * chunk, mine = min(chunk, n - base);
    const int b0 = k * L;
    if (threadIdx.x < ns) {   // slot s: full when the block's bytes landed
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mfull[threadIdx.x])) : "memory");
        reinterpret_cast<int *>(peer + 32)[threadIdx.x] = 0;   // release counter
    }
    if (threadIdx.x == 0) reinterpret_cast<int *>(peer + 32)[LV_NS_MAX] = 0;   // completed-level prefix
#ifdef DPP_FLOW_PHASES
    const bool nopush = g_flow_nopush;   // timing experiment only: no remote pushes (results invalid)
#else
    constexpr bool nopush = false;
#endif
    for (int l = threadIdx.x; l < L; l += blockDim.x) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&mlev[l])), "r"(lrows[b0 + l] + 1) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mlev[l])), "r"(nopush ? 0 : tx[b0 + l])
                     : "memory");
    }
    if (threadIdx.x < C) {
        peer[threadIdx.x] = mapa_u32(su32(xh + chunkp), threadIdx.x);
        peer[16 + threadIdx.x] = mapa_u32(su32(mlev), threadIdx.x);
    }
    for (int i = threadIdx.x; i <= S; i += blockDim.x) boff_s[i] = boff[s0 + i];
    for (int i = threadIdx.x; i < S; i += blockDim.x) slev[i] = splev[s0 + i];
    pdl_wait();   // b is the previous kernel's output
    for (int i = threadIdx.x; i < mine; i += blockDim.x) xh[i] = b[(size_t)(base + i) * ncomp + comp];
    for (int i = threadIdx.x; i < hmax; i += blockDim.x) xh[chunkp + i] = 0.0;   // slot hmax-1: padding
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    // every CTA's level mbarriers are armed before the first push
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    // Ring of ns one-block slots in step order (step s in slot s % ns) without a producer warp:
    // every warp passes every step (the owning team after solving the block, the others as soon
    // as the block landed) and the LAST warp to release a slot issues the bulk copy of step
    // s + ns into it.  (A dedicated producer warp made the team sharing its SM sub-partition
    // 3-5x slower per level; the copy issue itself costs nothing measurable,
    // tools/micro/tma_interference.cu.)
    int *rel = reinterpret_cast<int *>(peer + 32);   // ns release counters
    auto issue = [&](int st) {
        const int sl = st % ns;
        const unsigned bytes = (unsigned)(boff_s[st + 1] - boff_s[st]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mfull[sl])), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(ring + (size_t)sl * stage)), "l"(blocks + boff_s[st]), "r"(bytes), "r"(su32(&mfull[sl]))
                     : "memory");
        const int pf = st + l2pf;
        if (l2pf && pf < S)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(blocks + boff_s[pf]),
                         "r"((unsigned)(boff_s[pf + 1] - boff_s[pf]))
                         : "memory");
    };
    auto release = [&](int st) {
        __syncwarp();
        if (lane == 0) {
            const int sl = st % ns;
            if (atomicAdd(&rel[sl], 1) == nw - 1) {   // every warp passed step st
                atomicExch(&rel[sl], 0);
                if (st + ns < S) issue(st + ns);
            }
        }
    };
    if (threadIdx.x == 0)
        for (int st = 0; st < min(ns, S); ++st) issue(st);
    {
        // warps in LV_TEAMS teams by level (team = wid % LV_TEAMS = level % LV_TEAMS), one team
        // per sub-partition.  A team's warps deal a block's 32-row chunks; for its level-l rows a
        // warp sums the early columns (sources of levels <= l-LV_TEAMS-1, complete before its
        // previous block ended) right away, the mid columns (levels l-LV_TEAMS .. l-2) once those
        // are complete, and only the late columns (level l-1) after the last wait -- the other
        // teams' rows run meanwhile, so a level's critical path is one wake-up plus the late
        // columns.  Index / value loads of the first mid / late group are issued before the
        // waits; partial sums regroup the row's dot product (exact-arithmetic equivalent).
#ifdef DPP_FLOW_PHASES
        const int team = (wid + g_flow_rot * k) % LV_TEAMS, wi = wid / LV_TEAMS;   // experiment: rotate by rank
#else
        const int team = wid % LV_TEAMS, wi = wid / LV_TEAMS;
#endif
        const int nteam = nw / LV_TEAMS;
        int waited = 0;   // levels [0, waited) known complete by this warp
        int part_of_lvl = 0;
        // levels [0, *lvdone) are known complete CTA-wide (the largest prefix any warp waited
        // through): a warp that skipped many levels starts its waits there instead of
        // re-checking every completed barrier (~100 cycles each)
        int *lvdone = rel + LV_NS_MAX;
        auto wait_levels = [&](int upto) {   // all levels < upto complete
            if (waited >= upto) return;
            waited = max(waited, *reinterpret_cast<volatile int *>(lvdone));
            if (waited >= upto) return;
            for (; waited < upto; ++waited) mwait(su32(&mlev[waited]), 0);
            if (lane == 0) atomicMax(lvdone, waited);
        };
#ifdef DPP_FLOW_PHASES
        long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        long long sink = 0;
#endif
        for (int st = 0; st < S; ++st) {
            const int sl = st % ns;
            const int lvl = slev[st];
            // the parts of a level (consecutive steps) are dealt to the team's warps in turn
            const int pidx = (st > 0 && slev[st - 1] == lvl) ? ++part_of_lvl : (part_of_lvl = 0);
            // every warp waits for the slot's fill before releasing it, so a release always
            // counts toward the slot's current use
            PH_T(cr0);
            mwait(su32(&mfull[sl]), (unsigned)((st / ns) & 1));
            PH_T(cr1);
            PH_ADD(0, cr1 - cr0);
            if (lvl % LV_TEAMS != team) {
                release(st);
                continue;
            }
            {
                const unsigned char *blk = ring + (size_t)sl * stage;
                const int4 hd = *reinterpret_cast<const int4 *>(blk);
                const int nr = hd.x, nch = hd.y;
                const int ci0 = ((wi - pidx) % nteam + nteam) % nteam;   // chunks ci = ci0 (mod nteam)
                if (ci0 >= nch) goto release;
                {
                const int4 *chs = reinterpret_cast<const int4 *>(blk + 16);
                const int2 *rw = reinterpret_cast<const int2 *>(blk + lv_off_rw(nch));
                const double *dg = reinterpret_cast<const double *>(blk + lv_off_dq(nch, nr));
                const unsigned short *code = reinterpret_cast<const unsigned short *>(blk + lv_off_code(nch, nr));
                int ne = 0;   // the last chunk's end (its width: the block's remaining rows)
                {
                    const int4 lc = chs[nch - 1];
                    ne = lc.x + (nr - 32 * (nch - 1)) * (lc.y + lc.z + lc.w);
                }
                const double *val = reinterpret_cast<const double *>(blk + lv_off_val(nch, nr, ne));
                const int *pl = reinterpret_cast<const int *>(val + ne);
                int done = 0;
#ifdef DPP_FLOW_PHASES
                long long c_late = 1ll << 62;
                const long long c_first = clk();
#endif
                for (int ci = ci0; ci < nch; ci += nteam) {
                    const int q = 32 * ci + lane;
                    const bool act = q < nr;
                    done += min(32, nr - 32 * ci);
                    const int4 ch = chs[ci];
                    int2 R = make_int2(0, 0);
                    double dq = 0.0;
                    if (act) {
                        R = rw[q];
                        dq = dg[q];
                    }
                    PH_T(c0);
                    wait_levels(lvl - LV_TEAMS);   // early levels
                    PH_T(c1);
                    PH_ADD(1, c1 - c0);
                    // early columns (a multiple of 4): two groups of 4 loads in flight, four partial sums
                    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
                    // a chunk's columns are w = its rows (<= 32) entries apart
                    const int w = min(32, nr - 32 * ci);
                    int e = ch.x + (act ? lane : 0);
#pragma unroll 2
                    for (int k = 0; k < ch.y; k += 4, e += 4 * w) {
                        int cd[4];
                        double v[4], xv[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) { cd[u] = code[e + w * u]; v[u] = val[e + w * u]; }
#pragma unroll
                        for (int u = 0; u < 4; ++u) xv[u] = xh[cd[u]];
                        s0 = fma(v[0], xv[0], s0); s1 = fma(v[1], xv[1], s1);
                        s2 = fma(v[2], xv[2], s2); s3 = fma(v[3], xv[3], s3);
                    }
                    // mid / late columns (multiples of 4): the first group's indices and values are
                    // fetched before the waits, only the x gathers follow them
                    const int em = e, el = e + w * ch.z;
                    int mc[4], lc[4];
                    double mv[4], lv[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        mc[u] = ch.z ? code[em + w * u] : 0;
                        mv[u] = ch.z ? val[em + w * u] : 0.0;
                        lc[u] = ch.w ? code[el + w * u] : 0;
                        lv[u] = ch.w ? val[el + w * u] : 0.0;
                    }
                    const double bq = act ? xh[R.x] : 0.0;
                    double sum = (s0 + s1) + (s2 + s3);
#ifdef DPP_FLOW_PHASES
                    sink ^= (long long)__double_as_longlong(sum);
#endif
                    PH_T(c2);
                    PH_ADD(2, c2 - c1);
                    wait_levels(lvl - 1);   // mid levels
                    auto group4 = [&](const int *gc, const double *gv, double &t0, double &t1) {
                        double gx[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) gx[u] = xh[gc[u]];
                        t0 = fma(gv[0], gx[0], t0); t1 = fma(gv[1], gx[1], t1);
                        t0 = fma(gv[2], gx[2], t0); t1 = fma(gv[3], gx[3], t1);
                    };
                    auto rest4 = [&](int e0, int n, double &t0, double &t1) {   // groups after the first
                        for (int k = 4; k < n; k += 4) {
                            int gc[4];
                            double gv[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) { gc[u] = code[e0 + w * (k + u)]; gv[u] = val[e0 + w * (k + u)]; }
                            group4(gc, gv, t0, t1);
                        }
                    };
                    if (ch.z) {
                        double t0 = 0.0, t1 = 0.0;
                        group4(mc, mv, t0, t1);
                        rest4(em, ch.z, t0, t1);
                        sum += t0 + t1;
                    }
                    PH_T(c3);
                    PH_ADD(3, c3 - c2);
                    wait_levels(lvl);   // level l-1
                    PH_T(c4);
                    PH_ADD(5, c4 - c3);
#ifdef DPP_FLOW_PHASES
                    c_late = min(c_late, c4);
#endif
                    if (ch.w) {
                        double t0 = 0.0, t1 = 0.0;
                        group4(lc, lv, t0, t1);
                        rest4(el, ch.w, t0, t1);
                        sum += t0 + t1;
                    }
#ifdef DPP_FLOW_PHASES
                    sink ^= (long long)__double_as_longlong(sum);
                    PH_T(c4a);
                    PH_ADD(4, c4a - c4);
#endif
                    if (act) {
                        const double xr = (bq - sum) * dq;   // dq = 1/t_ii
                        xh[R.x] = xr;
                        const int p0 = R.y >> 4, pc = nopush ? 0 : R.y & 15;
                        for (int u = 0; u < pc; ++u) {
                            const int pe = pl[p0 + u];
                            const int dst = (int)((unsigned)pe >> 28);
                            const unsigned slh = (unsigned)pe & 0x0fffffffu;
                            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
                                         ::"r"(peer[dst] + 8u * slh), "l"(__double_as_longlong(xr)),
                                         "r"(peer[16 + dst] + 8u * lvl)
                                         : "memory");
                        }
#ifdef DPP_FLOW_PHASES
                        sink ^= (long long)__double_as_longlong(xr);
#endif
                    }
                    __syncwarp();
                    PH_T(c5);
#ifdef DPP_FLOW_PHASES
                    PH_ADD(7, c5 - c4a);
#endif
                    PH_ADD(6, 1);
                }
                __syncwarp();
                PH_T(c6);
                if (lane == 0)   // release: this warp's x stores of the level precede the arrival
                    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mlev[lvl])),
                                 "r"(done)
                                 : "memory");
                PH_T(c7);
#ifdef DPP_FLOW_PHASES
                if (lane == 0 && g_flow_tl) {
                    unsigned long long *o = g_flow_tl + ((size_t)blockIdx.x * g_flow_smax + st) * 4;
                    o[0] = lvl;
                    atomicMin(o + 1, (unsigned long long)c_late);
                    atomicMax(o + 2, (unsigned long long)c7);
                    atomicMin(o + 3, (unsigned long long)c_first);
                }
#endif
                }
            }
        release:
            release(st);
        }
#ifdef DPP_FLOW_PHASES
        if (lane == 0 && g_flow_phase)
            for (int i = 0; i < 8; ++i) g_flow_phase[((size_t)blockIdx.x * 32 + wid) * 8 + i] = ph[i] + (sink == 0x1234567 ? 1 : 0);
#endif
    }
    __syncthreads();
    pdl_trigger();
    for (int i = threadIdx.x; i < mine; i += blockDim.x) {
        const size_t g = (size_t)(base + i) * ncomp + comp;
        x[g] = xh[i];
        if (xout) xout[g] = xadd[g] + xh[i];
    }
}


// ----------------------------------------------------------------- warp-stream dataflow variant
// Lane-per-row dataflow sweep (DPP_PU_MODE=ws).  Same partition and halo / push tables as the
// other kernels of this file, but:
//   * a CTA's rows of one level are cut into chunks of <= 32 rows, and chunk g of the CTA (in
//     level order) belongs to warp g % nw -- consecutive levels sit on different warps;
//   * lane l of the warp owns row l of the chunk and walks its entries four columns at a time
//     (SELL layout: column t of the chunk is w consecutive (code, value) pairs), the entries of
//     a row sorted by source level and right-aligned, so every lane meets its level l-1 sources
//     in the chunk's last group;
//   * readiness is the x slot itself (NaN sentinel until the value lands: own rows by a
//     volatile shared store, remote rows by a plain cluster store into the halo), polled
//     warp-uniformly -- the lanes of a chunk never depend on one another;
//   * every warp streams its own chunks through a private ring of TMA slots that it refills
//     itself (pieces of <= slot bytes, sizes in a per-warp offset table), so no warp waits for
//     another one's ring and there is no CTA-wide step;
//   * b is read and x written straight from / to global memory by the owning lane (loads issued
//     at the chunk's first piece, far ahead of their use).
// A level therefore costs one poll hit + one group of FMAs + the row's store on the critical
// path.  Arithmetic: four partial sums per row (exact-arithmetic regrouping of the dot product).
//
// piece (16-byte aligned): int4 {groups, w, flags (1 first piece of a chunk, 2 last), np} |
//   first: u16 local row[w] | groups x { u16 code[4][w] | f64 val[4][w] } |
//   last: f64 1/diag[w] | int (p0 << 4 | npush)[w] | int push[np]
constexpr int WS_NS_MAX = 8;
#ifdef DPP_WS_TL
// timeline build: per (CTA, warp, chunk ordinal) {t first piece landed, t last group entered, t inputs ready, t stored}
constexpr int WS_TL_MAXC = 1024;
__device__ unsigned long long *g_ws_tl = nullptr;
#endif
__host__ __device__ inline long long ws_group_bytes(int w) { return p16(8LL * w) + 32LL * w; }
__host__ __device__ inline long long ws_head_bytes(int w) { return 16 + p16(2LL * w); }
__host__ __device__ inline long long ws_tail_bytes(int w, int np) { return p16(8LL * w) + p16(4LL * w) + p16(4LL * np); }
__host__ __device__ inline size_t ws_fixed(int chunk, int hmax, int nw, int ns) {
    return (size_t)((p16(8LL * nw * ns) + p16(8LL * chunk) + p16(8LL * hmax) + 64 + 127) & ~127LL);
}
struct WsWalk {   // the pieces of one chunk (w rows, ngr column groups, np push entries), greedy in slot bytes
    int w, ngr, np, slot;
    long long off, bytes;   // the current piece: offset from the chunk's start, size
    int g0, ng, flags;
    __host__ __device__ void place(bool fst) {
        long long sz = fst ? ws_head_bytes(w) : 16;
        const long long gb = ws_group_bytes(w);
        ng = 0;
        while (g0 + ng < ngr && sz + gb <= slot) { sz += gb; ++ng; }
        flags = fst ? 1 : 0;
        if (g0 + ng == ngr && sz + ws_tail_bytes(w, np) <= slot) { flags |= 2; sz += ws_tail_bytes(w, np); }
        bytes = sz;
    }
    __host__ __device__ void first() { off = 0; g0 = 0; place(true); }
    __host__ __device__ bool next() {
        if (flags & 2) return false;
        off += bytes; g0 += ng;
        place(false);
        return true;
    }
    __host__ __device__ long long data() const { return off + ((flags & 1) ? ws_head_bytes(w) : 16); }   // first group
};

__global__ void __launch_bounds__(512, 1)
    k_trsv_ws(int n, int ncomp, int chunk, int hmax, int slot, int ns, const unsigned char *__restrict__ blocks,
              const long long *__restrict__ poff, const int *__restrict__ pidx, const double *__restrict__ b,
              double *__restrict__ x, const double *__restrict__ xadd, double *__restrict__ xout, int nap) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int nw = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long *mb = reinterpret_cast<unsigned long long *>(smem) + wid * ns;
    const int chunkp = pu_chunkp(chunk);
    double *xh = reinterpret_cast<double *>(smem + p16(8LL * nw * ns));
    unsigned *peer = reinterpret_cast<unsigned *>(xh + chunkp + p16(8LL * hmax) / 8);
    unsigned char *ring = smem + ws_fixed(chunk, hmax, nw, ns) + (size_t)wid * ns * slot;
    cg::cluster_group cl = cg::this_cluster();
    const int k = (int)cl.block_rank(), C = (int)cl.num_blocks();
    const int comp = blockIdx.x / C;
    const int base = k * chunk, mine = max(0, min(chunk, n - base));
    const int pi0 = pidx[k * nw + wid], NP = pidx[k * nw + wid + 1] - pi0 - 1;
    const long long *po = poff + pi0;
    auto issue = [&](int i, long long o0, long long o1) {
        const int sl = i % ns;
        const unsigned bytes = (unsigned)(o1 - o0);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mb[sl])), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(ring + (size_t)sl * slot)), "l"(blocks + o0), "r"(bytes), "r"(su32(&mb[sl]))
                     : "memory");
    };
    // the plan is static: the ring's first pieces are in flight before the predecessor ends
    if (lane == 0) {
        for (int s = 0; s < ns; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mb[s])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int i = 0; i < min(ns, NP); ++i) issue(i, po[i], po[i + 1]);
    }
    if (threadIdx.x < C) peer[threadIdx.x] = mapa_u32(su32(xh + chunkp), threadIdx.x);
    const double sent = __longlong_as_double((long long)PU_SENT);
    for (int i = threadIdx.x; i < mine; i += blockDim.x) xh[i] = sent;
    for (int i = threadIdx.x; i < hmax - 1; i += blockDim.x) xh[chunkp + i] = sent;
    if (threadIdx.x == 0) xh[chunkp + hmax - 1] = 0.0;   // the padding entries' source
    __syncthreads();
    // every CTA's slots hold the sentinel before anyone pushes
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    pdl_wait();   // b is the previous kernel's output
    const unsigned xh_s = su32(xh);
    const int zero_code = chunkp + hmax - 1;
    int row = 0;
    size_t g = 0;
    double bq = 0.0, xa = 0.0, s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#ifdef DPP_WS_TL
    int tl_ord = -1;
    unsigned long long tl0 = 0, tl1 = 0, tl2 = 0, tlw = 0, tlm = 0, tlq = 0;   // tlw: poll time of the earlier groups, tlm: mbarrier waits
#endif
    for (int pi = 0; pi < NP; ++pi) {
        const int sl = pi % ns;
        long long n0 = 0, n1 = 0;   // the refill's extent, fetched before it is needed
        if (pi + ns < NP) { n0 = po[pi + ns]; n1 = po[pi + ns + 1]; }
#ifdef DPP_WS_TL
        tlq = clock64();
#endif
        mwait(su32(&mb[sl]), (unsigned)((pi / ns) & 1));
        const unsigned char *pc = ring + (size_t)sl * slot;
        const int4 hd = *reinterpret_cast<const int4 *>(pc);
        const int ng = hd.x, w = hd.y, fl = hd.z;
        DPP_DCHECK(w >= 1 && w <= 32 && ng >= 0 && hd.w >= 0);
#ifdef DPP_WS_TL
        if (fl & 1) { tlw = 0; tlm = 0; }
        tlm += clock64() - tlq;
#endif
        const bool act = lane < w;
        int o = 16;
        if (fl & 1) {
#ifdef DPP_WS_TL
            ++tl_ord;
            tl0 = clock64();
#endif
            const unsigned short *rows = reinterpret_cast<const unsigned short *>(pc + 16);
            row = act ? rows[lane] : 0;
            DPP_DCHECK(row < mine);
            g = (size_t)(base + row) * ncomp + comp;
            bq = act ? b[g] : 0.0;
            xa = (act && xout) ? xadd[g] : 0.0;
            s0 = s1 = s2 = s3 = 0.0;
            o += (int)p16(2LL * w);
        }
        const int cb = (int)p16(8LL * w), gb = cb + 32 * w;
        DPP_DCHECK(o + (long long)ng * gb + ((fl & 2) ? ws_tail_bytes(w, hd.w) : 0) <= slot);
        double dq = 0.0;
        int pinf = 0;
        const int *pl = nullptr;
        if (fl & 2) {
            const unsigned char *t = pc + o + ng * gb;
            dq = act ? reinterpret_cast<const double *>(t)[lane] : 0.0;
            pinf = act ? reinterpret_cast<const int *>(t + cb)[lane] : 0;
            pl = reinterpret_cast<const int *>(t + cb + p16(4LL * w));
        }
        int cd[4];
        double v[4];
#define WS_LOAD_CV(gi)                                                                                  \
    {                                                                                                   \
        const unsigned short *code_ = reinterpret_cast<const unsigned short *>(pc + o + (gi) * gb);     \
        const double *val_ = reinterpret_cast<const double *>(pc + o + (gi) * gb + cb);                 \
        _Pragma("unroll") for (int u = 0; u < 4; ++u) {                                                 \
            cd[u] = act ? (int)code_[u * w + lane] : zero_code;                                         \
            v[u] = act ? val_[u * w + lane] : 0.0;                                                      \
        }                                                                                               \
    }
        if (ng) WS_LOAD_CV(0);
        for (int gi = 0; gi < ng; ++gi) {
            unsigned a[4];
            double cv[4], xv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                DPP_DCHECK(cd[u] >= 0 && (cd[u] < mine || (cd[u] >= chunkp && cd[u] < chunkp + hmax)));
                a[u] = xh_s + 8u * (unsigned)cd[u];
                cv[u] = v[u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) xv[u] = ld_vol_shared(a[u]);
            if (gi + 1 < ng) WS_LOAD_CV(gi + 1);
            long long spins = 0;
#ifdef DPP_WS_TL
            tlq = clock64();
            if ((fl & 2) && gi == ng - 1) tl1 = tlq;
#endif
            // the sentinel is the only stored value whose high word is all ones (a computed NaN is
            // stored as the canonical quiet NaN), and 8-byte shared accesses are single transactions
            while (true) {
                bool pend = false;
#pragma unroll
                for (int u = 0; u < 4; ++u) pend |= __double2hiint(xv[u]) == -1;
                if (!__any_sync(0xffffffffu, pend)) break;
                // far from the chunk's last groups the missing sources are levels away
                if (nap && (!(fl & 2) || gi + 2 < ng)) __nanosleep(nap);
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (__double2hiint(xv[u]) == -1) xv[u] = ld_vol_shared(a[u]);
                if (++spins > (1ll << 26)) __trap();
            }
#ifdef DPP_WS_TL
            if ((fl & 2) && gi == ng - 1) tl2 = clock64();
            else tlw += clock64() - tlq;
#endif
            s0 = fma(cv[0], xv[0], s0);
            s1 = fma(cv[1], xv[1], s1);
            s2 = fma(cv[2], xv[2], s2);
            s3 = fma(cv[3], xv[3], s3);
        }
#undef WS_LOAD_CV
        if ((fl & 2) && act) {
            double xr = (bq - ((s0 + s1) + (s2 + s3))) * dq;   // dq = 1/t_ii
            if (__double2hiint(xr) == -1) xr = __longlong_as_double(0x7ff8000000000000ll);   // a NaN that looks pending
            st_vol_shared(xh_s + 8u * (unsigned)row, xr);
            const int p0 = pinf >> 4, pn = pinf & 15;
            for (int u = 0; u < pn; ++u) {
                const int pe = pl[p0 + u];
                DPP_DCHECK((int)((unsigned)pe >> 28) < C && (int)((unsigned)pe & 0x0fffffffu) < hmax - 1);
                st_remote(peer[(unsigned)pe >> 28] + 8u * ((unsigned)pe & 0x0fffffffu), xr);
            }
            x[g] = xr;
            if (xout) xout[g] = xa + xr;
        }
        __syncwarp();
#ifdef DPP_WS_TL
        if (fl & 2) {
            const unsigned long long tl3 = clock64();
            if (lane == 0 && g_ws_tl && tl_ord < WS_TL_MAXC) {
                unsigned long long *o = g_ws_tl + (((size_t)blockIdx.x * nw + wid) * WS_TL_MAXC + tl_ord) * 6;
                o[0] = tl0; o[1] = tl1; o[2] = tl2; o[3] = tl3; o[4] = tlw; o[5] = tlm;
            }
        }
#endif
        if (lane == 0 && pi + ns < NP) issue(pi + ns, n0, n1);
    }
    pdl_trigger();
    // a CTA's shared memory must outlive the pushes aimed at it
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// ----------------------------------------------------------------- global-stream dataflow variant
// Lane-per-row dataflow sweep without a shared-memory ring (the default for thin rows).  The
// warp-stream kernel above was measured (-DDPP_WS_PH) to be bound by the SM's shared-memory
// pipe, not by the dependency chain: per chunk a warp spends ~3,800 cycles of which only ~800
// wait for inputs, and doubling the warps (shared ring) made every phase 4-5x slower -- the TMA
// writes, the code / value reads back out of the ring and the x-slot polls all go through the
// same banks.  Here only x lives in shared memory: every lane streams its own row's entries
// straight from global memory (coalesced SELL columns, whole batches of 4-column groups in
// flight in registers, the next chunk's header / rows and an L2 prefetch issued a chunk ahead),
// so the shared-memory traffic is the x gathers alone and 16+ warps hide the load latency.
// Same partition, halo / push tables, level-sorted right-aligned rows, NaN-sentinel readiness
// and arithmetic (four partial sums per row) as k_trsv_ws.
//
// chunk (16-byte aligned segments): int4 {groups, w, np, level} | u16 local row[w] | f64 1/diag[w] |
//   int (p0 << 4 | npush)[w] | int2 first two push entries[w] | int push[np] |
//   groups x { u16 code[w][4] | f64 val[4][w] }
#ifndef DPP_GS_WARPS_MAX
#define DPP_GS_WARPS_MAX 16   // 512 threads: up to 128 registers each (a batch of groups lives in registers)
#endif
#ifndef DPP_GS_GB
#define DPP_GS_GB 4
#endif
constexpr int GS_WARPS_MAX = DPP_GS_WARPS_MAX, GS_GB = DPP_GS_GB;
__host__ __device__ inline long long gs_group_bytes(int w) { return p16(8LL * w) + 32LL * w; }
__host__ __device__ inline long long gs_off_dq(int w) { return 16 + p16(2LL * w); }
__host__ __device__ inline long long gs_off_pinf(int w) { return gs_off_dq(w) + p16(8LL * w); }
__host__ __device__ inline long long gs_off_p2(int w) { return gs_off_pinf(w) + p16(4LL * w); }
__host__ __device__ inline long long gs_off_pl(int w) { return gs_off_p2(w) + p16(8LL * w); }
__host__ __device__ inline long long gs_off_groups(int w, int np) { return gs_off_pl(w) + p16(4LL * np); }
__host__ __device__ inline long long gs_chunk_bytes(int w, int ngr, int np) {
    return gs_off_groups(w, np) + (long long)ngr * gs_group_bytes(w);
}
__host__ __device__ inline size_t gs_smem(int chunk, int hmax) {   // x slice | halo | peers
    return (size_t)((p16(8LL * chunk) + p16(8LL * hmax) + 64 + 127) & ~127LL);
}
#ifdef DPP_WS_PH
// phase build: per (CTA, warp) cycles summed over its chunks {head, loads + groups, tail, -, -, polls, chunks, -}
__device__ unsigned long long *g_ws_ph = nullptr;
// CTA 0 only: per (warp, chunk) {level, t last group entered, t its inputs were there, t x stored} (clock64)
__device__ unsigned long long *g_ws_hop = nullptr;
constexpr int GS_HOP_MAX = 256;
#define GS_PH(i, t0_) { const unsigned long long t_ = clock64(); ph[i] += t_ - (t0_); (t0_) = t_; }
#else
#define GS_PH(i, t0_)
#endif
__device__ __forceinline__ unsigned long long ldg_u64(const void *p) {
    unsigned long long v;
    asm volatile("ld.global.nc.L1::no_allocate.b64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double ldg_f64(const void *p) { return __longlong_as_double((long long)ldg_u64(p)); }

__global__ void __launch_bounds__(32 * GS_WARPS_MAX, 1)
    k_trsv_gs(int n, int ncomp, int chunk, int hmax, int CT, int rev, const unsigned char *__restrict__ blocks,
              const long long *__restrict__ soff, const int *__restrict__ scnt,
              const unsigned long long *__restrict__ imp, const int *__restrict__ istart,
              const double *__restrict__ b, double *x, const double *__restrict__ xadd, double *__restrict__ xout,
              int nap) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int nw = (blockDim.x >> 5) - (imp ? 1 : 0), wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int chunkp = pu_chunkp(chunk);
    double *xh = reinterpret_cast<double *>(smem);
    unsigned *peer = reinterpret_cast<unsigned *>(xh + chunkp + p16(8LL * hmax) / 8);
    cg::cluster_group cl = cg::this_cluster();
    const int C = (int)cl.num_blocks();
    const int comp = blockIdx.x / CT;
    // CTA slice of this block.  With several clusters the one without cross-cluster sources gets the
    // lowest block index (a backward sweep's sources have higher rows), so a resident cluster only
    // ever waits for clusters that were dispatched before it.
    const int cid = (blockIdx.x % CT) / C, ncl = CT / C;
    const int k = (rev ? ncl - 1 - cid : cid) * C + (int)cl.block_rank();
    const int base = k * chunk, mine = max(0, min(chunk, n - base));
    // the plan is static: this warp's first header and rows are in flight before the predecessor ends
    const bool importer = imp && wid == nw;
    const unsigned char *pc = blocks + (importer ? 0 : soff[k * nw + wid]);
    const int NCH = importer ? 0 : scnt[k * nw + wid];
    int4 hd = make_int4(0, 0, 0, 0);
    int rown = 0;
    if (NCH) {
        hd = *reinterpret_cast<const int4 *>(pc);
        rown = reinterpret_cast<const unsigned short *>(pc + 16)[lane];
    }
    if (threadIdx.x < C) peer[threadIdx.x] = mapa_u32(su32(xh + chunkp), threadIdx.x);
    const double sent = __longlong_as_double((long long)PU_SENT);
    for (int i = threadIdx.x; i < mine; i += blockDim.x) xh[i] = sent;
    for (int i = threadIdx.x; i < hmax - 1; i += blockDim.x) xh[chunkp + i] = sent;
    if (threadIdx.x == 0) xh[chunkp + hmax - 1] = 0.0;   // the padding entries' source
    __syncthreads();
    // every CTA's slots hold the sentinel before anyone pushes
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    pdl_wait();   // b is the previous kernel's output
    const unsigned xh_s = su32(xh);
    if (importer) {
        // sources solved by another cluster: x in global memory (sentinel-filled before the launch,
        // written by the owning lane) is polled and copied into this CTA's halo slots, 64 entries in
        // flight, in the order of the sources' levels
        const int i0 = istart[k], i1 = istart[k + 1];
        for (int pos = i0; pos < i1; pos += 64) {
            unsigned long long e[2];
            bool done[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int i = pos + 32 * u + lane;
                e[u] = i < i1 ? imp[i] : 0ull;
                done[u] = i >= i1;
            }
            long long spins = 0;
            while (true) {
#pragma unroll
                for (int u = 0; u < 2; ++u)
                    if (!done[u]) {
                        unsigned long long v;
                        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];"
                                     : "=l"(v) : "l"(x + (size_t)(e[u] >> 32) * ncomp + comp) : "memory");
                        if ((int)(v >> 32) != -1) {
                            st_vol_shared(xh_s + 8u * (unsigned)(chunkp + (int)(e[u] & 0xffffffffu)),
                                          __longlong_as_double((long long)v));
                            done[u] = true;
                        }
                    }
                if (__all_sync(0xffffffffu, done[0] && done[1])) break;
                __nanosleep(100);
                if (++spins > (1ll << 24)) __trap();
            }
        }
        pdl_trigger();
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        return;
    }
    const unsigned long long zero4 = 0x0001000100010001ull * (unsigned long long)(chunkp + hmax - 1);
#ifdef DPP_WS_PH
    unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0}, pt = clock64(), pq = 0;
#endif
    for (int ci = 0; ci < NCH; ++ci) {
        const int ng = hd.x, w = hd.y, np = hd.z;
#ifdef DPP_WS_PH
        const int hd_lev = hd.w;
        unsigned long long hop1 = 0, hop2 = 0, hop3 = 0;
#endif
        DPP_DCHECK(w >= 1 && w <= 32 && ng >= 0 && np >= 0);
        const bool act = lane < w;
        const int row = act ? rown : 0;
        DPP_DCHECK(row < mine);
        const size_t g = (size_t)(base + row) * ncomp + comp;
        const double bq = act ? b[g] : 0.0;
        const double xa = (act && xout) ? xadd[g] : 0.0;
        const double dq = act ? ldg_f64(pc + gs_off_dq(w) + 8 * lane) : 0.0;
        const int pinf = act ? reinterpret_cast<const int *>(pc + gs_off_pinf(w))[lane] : 0;
        const unsigned long long p2 = act ? ldg_u64(pc + gs_off_p2(w) + 8 * lane) : 0ull;
        const int *pl = reinterpret_cast<const int *>(pc + gs_off_pl(w));
        const unsigned char *gp = pc + gs_off_groups(w, np);
        const long long cb = p16(8LL * w), gb = cb + 32LL * w;
        const unsigned char *pnx = gp + (long long)ng * gb;   // the next chunk of this warp's stream
        if (ci + 1 < NCH) {
            hd = *reinterpret_cast<const int4 *>(pnx);
            rown = reinterpret_cast<const unsigned short *>(pnx + 16)[lane];
            // and its entries on their way into L2 (128 B per lane and instruction)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pnx + 128 * lane));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pnx + 4096 + 128 * lane));
        }
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        GS_PH(0, pt);
        // batches of GS_GB groups: a batch's codes / values are all in flight before its first group is
        // polled (double-buffering the batches measured slower: 1.11 vs 1.07 ms per C2 PC apply -- the
        // sweep is bound by the ~300-cycle shared-memory hand-off between the warps of consecutive
        // levels, tools/micro/fp64lat.cu, not by load latency)
        for (int g0 = 0; g0 < ng; g0 += GS_GB) {
            unsigned long long c4[GS_GB];
            double v[GS_GB][4];
#pragma unroll
            for (int j = 0; j < GS_GB; ++j) {
                const unsigned char *q = gp + (long long)(g0 + j) * gb;
                const bool on = act && g0 + j < ng;
                c4[j] = on ? ldg_u64(q + 8 * lane) : zero4;
#pragma unroll
                for (int u = 0; u < 4; ++u) v[j][u] = on ? ldg_f64(q + cb + 8 * (u * w + lane)) : 0.0;
            }
#pragma unroll
            for (int j = 0; j < GS_GB; ++j) {
                if (g0 + j >= ng) break;
                unsigned a[4];
                double xv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int cd = (int)((c4[j] >> (16 * u)) & 0xffffu);
                    DPP_DCHECK(cd < mine || (cd >= chunkp && cd < chunkp + hmax));
                    a[u] = xh_s + 8u * (unsigned)cd;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) xv[u] = ld_vol_shared(a[u]);
                long long spins = 0;
#ifdef DPP_WS_PH
                pq = clock64();
                if (g0 + j == ng - 1) hop1 = pq;
#endif
                // the sentinel is the only stored value whose high word is all ones (a computed NaN is
                // stored as the canonical quiet NaN), and 8-byte shared accesses are single transactions
                while (true) {
                    bool pend = false;
#pragma unroll
                    for (int u = 0; u < 4; ++u) pend |= __double2hiint(xv[u]) == -1;
                    if (!__any_sync(0xffffffffu, pend)) break;
                    if (nap) __nanosleep(nap);
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (__double2hiint(xv[u]) == -1) xv[u] = ld_vol_shared(a[u]);
                    if (++spins > (1ll << 26)) __trap();
                }
#ifdef DPP_WS_PH
                {
                    const unsigned long long tq = clock64();
                    ph[5] += tq - pq;
                    if (g0 + j == ng - 1) hop2 = tq;
                }
#endif
                s0 = fma(v[j][0], xv[0], s0);
                s1 = fma(v[j][1], xv[1], s1);
                s2 = fma(v[j][2], xv[2], s2);
                s3 = fma(v[j][3], xv[3], s3);
            }
        }
        GS_PH(1, pt);
        if (act) {
            double xr = (bq - ((s0 + s1) + (s2 + s3))) * dq;   // dq = 1/t_ii
            if (__double2hiint(xr) == -1) xr = __longlong_as_double(0x7ff8000000000000ll);   // a NaN that looks pending
            st_vol_shared(xh_s + 8u * (unsigned)row, xr);
#ifdef DPP_WS_PH
            hop3 = clock64();
#endif
            const int p0 = pinf >> 4, pn = pinf & 15;
            for (int u = 0; u < pn; ++u) {
                const int pe = u < 2 ? (int)(p2 >> (32 * u)) : pl[p0 + u];
                DPP_DCHECK((int)((unsigned)pe >> 28) < C && (int)((unsigned)pe & 0x0fffffffu) < hmax - 1);
                st_remote(peer[(unsigned)pe >> 28] + 8u * ((unsigned)pe & 0x0fffffffu), xr);
            }
            x[g] = xr;
            if (xout) xout[g] = xa + xr;
        }
        __syncwarp();
        pc = pnx;
#ifdef DPP_WS_PH
        ph[6] += 1;
        if (lane == 0 && g_ws_hop && blockIdx.x == 0 && ci < GS_HOP_MAX) {
            unsigned long long *o = g_ws_hop + ((size_t)wid * GS_HOP_MAX + ci) * 4;
            o[0] = (unsigned long long)hd_lev; o[1] = hop1; o[2] = hop2; o[3] = hop3;
        }
        {
            unsigned long long gt;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
            if (ci == 0) ph[3] = gt;   // first chunk of this warp solved (ns)
            ph[4] = gt;                // last one
        }
#endif
        GS_PH(2, pt);
    }
#ifdef DPP_WS_PH
    if (lane == 0 && g_ws_ph)
        for (int i = 0; i < 8; ++i) g_ws_ph[((size_t)blockIdx.x * nw + wid) * 8 + i] = ph[i];
#endif
    pdl_trigger();
    // a CTA's shared memory must outlive the pushes aimed at it
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
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
    const int d = blockIdx.x * blockDim.x + threadIdx.x;   // one thread per CTA slice (+ the terminator)
    if (d > C) return;
    const unsigned long long key = (unsigned long long)d << 32;
    int lo = 0, hi = nh;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (h[mid] < key) lo = mid + 1; else hi = mid;
    }
    hstart[d] = lo;
}
// push pairs keyed by source row: (j << 8 | d) -> slot; byte counts per (consumer, level of j).
// A pair whose source row lives in another cluster (multi-cluster sweeps: CTA slices beyond 16)
// cannot be pushed through distributed shared memory: it leaves the push lists (key past every
// row) and goes to the consumer's import list (k_pu_import_keys).
__global__ void k_pu_push_keys(int nh, const unsigned long long *h, const int *hstart, int L, const int *lev, int n,
                               int chunk, unsigned long long *k2, int *slot, int *tx) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nh; i += gridDim.x * blockDim.x) {
        const int d = (int)(h[i] >> 32), j = (int)(h[i] & 0xffffffffu);
        const bool cross = (d >> 4) != ((j / chunk) >> 4);
        k2[i] = ((unsigned long long)(cross ? n : j) << 8) | (unsigned)d;   // cross-cluster pairs sort past every row
        slot[i] = i - hstart[d];
        if (!cross) atomicAdd(&tx[d * L + lev[j]], 8);
    }
}
// import pairs keyed by (consumer CTA, level of the source row) -> (source row << 32 | halo slot)
__global__ void k_pu_import_keys(int nh, const unsigned long long *h, const int *hstart, const int *lev, int chunk,
                                 unsigned long long *ik, unsigned long long *iv, int *ncross) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nh; i += gridDim.x * blockDim.x) {
        const int d = (int)(h[i] >> 32), j = (int)(h[i] & 0xffffffffu);
        const bool cross = (d >> 4) != ((j / chunk) >> 4);
        ik[i] = cross ? (((unsigned long long)d << 32) | (unsigned)lev[j]) : ~0ull;
        iv[i] = ((unsigned long long)j << 32) | (unsigned)(i - hstart[d]);
        if (cross) atomicAdd(ncross, 1);
    }
}
// pptr[j] = first push pair of source row j
__global__ void k_pu_pptr(int nh, const unsigned long long *k2s, int n, int *pptr) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= nh; i += gridDim.x * blockDim.x) {
        const int v = i < nh ? (int)(k2s[i] >> 8) : n;
        const int prev = i ? (int)(k2s[i - 1] >> 8) : -1;
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
// A row's entries are stored with the sources of levels <= l-2 first ("early") and those of
// level l-1 last ("late"; their count in R.x >> 16): k_trsv_lvl sums the early ones before it
// waits for level l-1.  Every kernel adds a lane's entries in storage order.
__global__ void k_pu_fill(int n, int chunk, int chunkp, int np_, const int *pstart, const int *perm,
                          const int *rptr, const int *rpp, const long long *boff, const int *ptr, const int *idx,
                          const double *val, const double *diag, const unsigned long long *h, const int *hstart,
                          const int *pptr, const unsigned long long *k2s, const int *slots, const int *lev,
                          unsigned char *blocks) {
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
        const int lr = lev[r];
        int nlate = 0;
        for (int p = ptr[r]; p < ptr[r + 1]; ++p) nlate += lev[idx[p]] >= lr - 1;
        rows[i] = make_int4((r - owner * chunk) | (nlate << 16), e0, e1, (p0 << 4) | pc);
        dg[i] = diag ? 1.0 / diag[r] : 1.0;
        int w = e0;
        const int hs = hstart[owner], he = hstart[owner + 1];
        for (int pass = 0; pass < 2; ++pass)
        for (int p = ptr[r]; p < ptr[r + 1]; ++p) {
            const int j = idx[p];
            if ((lev[j] >= lr - 1) != (pass == 1)) continue;
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
            ++w;
        }
        int u = p0;
        for (int t = pptr[r]; t < pptr[r + 1]; ++t, ++u)
            pl[u] = (int)(((unsigned)(k2s[t] & 15u) << 28 /* rank in the cluster */) | (unsigned)slots[t]);
    }
}

// ---- level-mbarrier (SELL chunk) format
__device__ __forceinline__ int pu_code(int j, int owner, int chunk, int chunkp, const unsigned long long *h, int hs,
                                       int he) {
    const int o = j / chunk;
    if (o == owner) return j - o * chunk;
    const unsigned long long key = ((unsigned long long)owner << 32) | (unsigned)j;
    int lo = hs, hi = he;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (h[mid] < key) lo = mid + 1; else hi = mid;
    }
    return chunkp + (lo - hs);
}
// entry class by source level distance: 0 early (<= l-LV_TEAMS-1), 1 mid (l-LV_TEAMS .. l-2), 2 late (l-1)
__device__ __forceinline__ int lv_class(int ls, int lr) { return ls >= lr - 1 ? 2 : ls >= lr - LV_TEAMS ? 1 : 0; }
__global__ void k_lv_counts(int n, const int *perm, const int *ptr, const int *idx, const int *lev, int *cnt) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        const int r = perm[q], lr = lev[r];
        int c3[3] = {0, 0, 0};
        for (int p = ptr[r]; p < ptr[r + 1]; ++p) ++c3[lv_class(lev[idx[p]], lr)];
        cnt[3 * q] = c3[0];
        cnt[3 * q + 1] = c3[1];
        cnt[3 * q + 2] = c3[2];
    }
}
// block headers and chunk tables; padding lanes of a partial last chunk get (zero slot, 0.0)
__global__ void k_lv_headers(int np_, const int *pstart, const int *pch, const int *plev, const int *rpp,
                             const int4 *ctab, int zero_code, const long long *boff, unsigned char *blocks) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < np_; i += gridDim.x * blockDim.x) {
        unsigned char *B = blocks + boff[i];
        const int nr = pstart[i + 1] - pstart[i], g0 = pch[i], nch = pch[i + 1] - g0;
        const int4 lc = ctab[pch[i + 1] - 1];
        const int ncol = lc.y + lc.z + lc.w;
        const int ne = lc.x + (nr - 32 * (nch - 1)) * ncol;
        int *h = reinterpret_cast<int *>(B);
        h[0] = nr;
        h[1] = nch;
        h[2] = rpp[pstart[i + 1]] - rpp[pstart[i]];
        h[3] = plev[i];
        int4 *chs = reinterpret_cast<int4 *>(B + 16);
        for (int c = 0; c < nch; ++c) chs[c] = ctab[g0 + c];
        unsigned short *code = reinterpret_cast<unsigned short *>(B + lv_off_code(nch, nr));
        double *vv = reinterpret_cast<double *>(B + lv_off_val(nch, nr, ne));
        (void)code; (void)vv; (void)zero_code;   // chunks are exactly as wide as their rows: no padding lanes
    }
}
__global__ void k_lv_fill(int n, int chunk, int chunkp, int zero_code, int np_, const int *pstart, const int *pch,
                          const int *perm, const int *rpp, const long long *boff, const int *ptr, const int *idx,
                          const double *val, const double *diag, const int *lev, const unsigned long long *h,
                          const int *hstart, const int *pptr, const unsigned long long *k2s, const int *slots,
                          const int4 *ctab, unsigned char *blocks) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        int lo = 0, hi = np_;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (pstart[mid] <= q) lo = mid; else hi = mid;
        }
        const int part = lo, q0 = pstart[part], nr = pstart[part + 1] - q0, i = q - q0;
        const int g0 = pch[part], nch = pch[part + 1] - g0;
        const int4 lc = ctab[pch[part + 1] - 1];
        const int ne = lc.x + (nr - 32 * (nch - 1)) * (lc.y + lc.z + lc.w);
        const int gc = g0 + i / 32, lane = i % 32, wch = min(32, nr - 32 * (i / 32));
        unsigned char *B = blocks + boff[part];
        int2 *rw = reinterpret_cast<int2 *>(B + lv_off_rw(nch));
        double *dq = reinterpret_cast<double *>(B + lv_off_dq(nch, nr));
        unsigned short *code = reinterpret_cast<unsigned short *>(B + lv_off_code(nch, nr));
        double *vv = reinterpret_cast<double *>(B + lv_off_val(nch, nr, ne));
        int *pl = reinterpret_cast<int *>(vv + ne);
        const int r = perm[q], owner = r / chunk, lr = lev[r];
        const int p0 = rpp[q] - rpp[q0], pc = rpp[q + 1] - rpp[q];
        rw[i] = make_int2(r - owner * chunk, (p0 << 4) | pc);
        dq[i] = diag ? 1.0 / diag[r] : 1.0;
        const int hs = hstart[owner], he = hstart[owner + 1];
        const int4 ch = ctab[gc];
        const int nc[3] = {ch.y, ch.z, ch.w};
        const int c0[3] = {0, ch.y, ch.y + ch.z};
        int kk[3] = {0, 0, 0};
        for (int p = ptr[r]; p < ptr[r + 1]; ++p) {
            const int j = idx[p];
            const int cl = lv_class(lev[j], lr);
            const int e = ch.x + wch * (c0[cl] + kk[cl]++) + lane;
            code[e] = pu_code(j, owner, chunk, chunkp, h, hs, he);
            vv[e] = val[p];
        }
        for (int cl = 0; cl < 3; ++cl)
            for (; kk[cl] < nc[cl]; ++kk[cl]) {
                const int e = ch.x + wch * (c0[cl] + kk[cl]) + lane;
                code[e] = zero_code;
                vv[e] = 0.0;
            }
        int u = p0;
        for (int t = pptr[r]; t < pptr[r + 1]; ++t, ++u)
            pl[u] = (int)(((unsigned)(k2s[t] & 15u) << 28 /* rank in the cluster */) | (unsigned)slots[t]);
    }
}


// ---- warp-stream format (k_trsv_ws): one thread per sorted row writes its lane of the chunk
// ctab[gc] = {first sorted row, rows, column groups, push entries}, cbase[gc] = the chunk's bytes
__device__ inline long long ws_group_off(int w, int ngr, int np, int slot, int gi) {   // from the chunk's start
    WsWalk wk{w, ngr, np, slot};
    wk.first();
    while (gi >= wk.g0 + wk.ng) wk.next();
    return wk.data() + (long long)(gi - wk.g0) * ws_group_bytes(w);
}
__global__ void k_ws_fill(int n, int chunk, int chunkp, int zero_code, int slot, int nchunks, const int4 *ctab,
                          const long long *cbase, const int *perm, const int *rpp, const int *ptr, const int *idx,
                          const double *val, const double *diag, const int *lev, const unsigned long long *h,
                          const int *hstart, const int *pptr, const unsigned long long *k2s, const int *slots,
                          unsigned char *blocks) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        int lo = 0, hi = nchunks;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (ctab[mid].x <= q) lo = mid; else hi = mid;
        }
        const int4 ct = ctab[lo];
        const int q0 = ct.x, w = ct.y, ngr = ct.z, np = ct.w, lane = q - q0;
        unsigned char *B = blocks + cbase[lo];
        const int r = perm[q], owner = r / chunk;
        const int a0 = ptr[r], len = ptr[r + 1] - a0, pad = 4 * ngr - len;
        const int hs = hstart[owner], he = hstart[owner + 1];
        const long long cb = p16(8LL * w);
        // pieces: headers (lane 0), local rows (first piece), 1/diag + push list (last piece)
        WsWalk wk{w, ngr, np, slot};
        wk.first();
        while (true) {
            unsigned char *pc = B + wk.off;
            if (lane == 0) *reinterpret_cast<int4 *>(pc) = make_int4(wk.ng, w, wk.flags, np);
            if (wk.flags & 1) reinterpret_cast<unsigned short *>(pc + 16)[lane] = (unsigned short)(r - owner * chunk);
            if (wk.flags & 2) {
                unsigned char *t = B + wk.data() + (long long)wk.ng * ws_group_bytes(w);
                const int p0 = rpp[q] - rpp[q0], pn = rpp[q + 1] - rpp[q];
                reinterpret_cast<double *>(t)[lane] = diag ? 1.0 / diag[r] : 1.0;
                reinterpret_cast<int *>(t + cb)[lane] = (p0 << 4) | pn;
                int *pl = reinterpret_cast<int *>(t + cb + p16(4LL * w));
                int u = p0;
                for (int tt = pptr[r]; tt < pptr[r + 1]; ++tt, ++u)
                    pl[u] = (int)(((unsigned)(k2s[tt] & 15u) << 28) | (unsigned)slots[tt]);
                break;
            }
            wk.next();
        }
        // entries by source level (ties in storage order), right-aligned in the chunk's columns
        auto put = [&](int col, int code, double vv) {
            unsigned char *gp = B + ws_group_off(w, ngr, np, slot, col >> 2);
            reinterpret_cast<unsigned short *>(gp)[(col & 3) * w + lane] = (unsigned short)code;
            reinterpret_cast<double *>(gp + cb)[(col & 3) * w + lane] = vv;
        };
        for (int col = 0; col < pad; ++col) put(col, zero_code, 0.0);
        for (int p = a0; p < a0 + len; ++p) {
            const int j = idx[p], lj = lev[j];
            int rank = 0;
            for (int t = a0; t < a0 + len; ++t) {
                const int lt = lev[idx[t]];
                rank += (lt < lj) || (lt == lj && t < p);
            }
            put(pad + rank, pu_code(j, owner, chunk, chunkp, h, hs, he), val[p]);
        }
    }
}

// ---- global-stream format (k_trsv_gs): one thread per sorted row writes its lane of the chunk
// ctab[gc] = {first sorted row, rows, column groups, push entries}, cbase[gc] = the chunk's bytes
__global__ void k_gs_fill(int n, int chunk, int chunkp, int zero_code, int nchunks, const int4 *ctab,
                          const long long *cbase, const int *perm, const int *rpp, const int *ptr, const int *idx,
                          const double *val, const double *diag, const int *lev, const unsigned long long *h,
                          const int *hstart, const int *pptr, const unsigned long long *k2s, const int *slots,
                          unsigned char *blocks) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        int lo = 0, hi = nchunks;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (ctab[mid].x <= q) lo = mid; else hi = mid;
        }
        const int4 ct = ctab[lo];
        const int q0 = ct.x, w = ct.y, ngr = ct.z, np = ct.w, lane = q - q0;
        unsigned char *B = blocks + cbase[lo];
        const int r = perm[q], owner = r / chunk;
        const int a0 = ptr[r], len = ptr[r + 1] - a0, pad = 4 * ngr - len;
        const int hs = hstart[owner], he = hstart[owner + 1];
        if (lane == 0) *reinterpret_cast<int4 *>(B) = make_int4(ngr, w, np, lev[r]);   // .w: the chunk's level (instrumented builds)
        reinterpret_cast<unsigned short *>(B + 16)[lane] = (unsigned short)(r - owner * chunk);
        reinterpret_cast<double *>(B + gs_off_dq(w))[lane] = diag ? 1.0 / diag[r] : 1.0;
        const int p0 = rpp[q] - rpp[q0], pn = rpp[q + 1] - rpp[q];
        reinterpret_cast<int *>(B + gs_off_pinf(w))[lane] = (p0 << 4) | pn;
        int *pl = reinterpret_cast<int *>(B + gs_off_pl(w));
        int first2[2] = {0, 0};
        int u = 0;
        for (int tt = pptr[r]; tt < pptr[r + 1]; ++tt, ++u) {
            const int pe = (int)(((unsigned)(k2s[tt] & 15u) << 28) | (unsigned)slots[tt]);
            pl[p0 + u] = pe;
            if (u < 2) first2[u] = pe;
        }
        reinterpret_cast<int2 *>(B + gs_off_p2(w))[lane] = make_int2(first2[0], first2[1]);
        // entries by source level (ties in storage order), right-aligned in the chunk's columns
        unsigned char *G = B + gs_off_groups(w, np);
        const long long cb = p16(8LL * w), gb = cb + 32LL * w;
        auto put = [&](int col, int code, double vv) {
            unsigned char *gq = G + (long long)(col >> 2) * gb;
            reinterpret_cast<unsigned short *>(gq)[4 * lane + (col & 3)] = (unsigned short)code;
            reinterpret_cast<double *>(gq + cb)[(col & 3) * w + lane] = vv;
        };
        for (int col = 0; col < pad; ++col) put(col, zero_code, 0.0);
        for (int p = a0; p < a0 + len; ++p) {
            const int j = idx[p], lj = lev[j];
            int rank = 0;
            for (int t = a0; t < a0 + len; ++t) {
                const int lt = lev[idx[t]];
                rank += (lt < lj) || (lt == lj && t < p);
            }
            put(pad + rank, pu_code(j, owner, chunk, chunkp, h, hs, he), val[p]);
        }
    }
}

// sweep kernel: 4 auto (default: global streams for thin rows, lane-group dataflow otherwise),
// 1 lane-group dataflow (DPP_PU_MODE=flow), 3 warp streams through TMA rings everywhere (ws),
// 5 global streams everywhere (gs), 0 level-mbarrier
// (lvl; own block format), 2 level-synchronous push (push or DPP_PU_FLOW=0)
int pu_mode() {
    static const int mode = [] {
        const char *e = std::getenv("DPP_PU_MODE");
        const char *f = std::getenv("DPP_PU_FLOW");
        if (f && *f == '0') return 2;
        if (e && !std::strcmp(e, "lvl")) return 0;
        if (e && !std::strcmp(e, "push")) return 2;
        if (e && !std::strcmp(e, "ws")) return 3;
        if (e && !std::strcmp(e, "gs")) return 5;
        if (e && !std::strcmp(e, "flow")) return 1;
        return 4;
    }();
    return mode;
}
// lane groups the row-major kernels would use for rows of this average length
inline int pu_lane_group(double avg) {
    int G = 2;
    while (G < 32 && G * 4 < avg) G *= 2;
    return G;
}
// a lane per row: measured on the global-stream kernel for every row length the configs have
// (C2: 7 / 26 entries per row; C3 level 0: 58, PC apply 18.7 -> 12.2 ms; C4 level 1: 74, 26.2 -> 25.5 ms).
// The TMA-ring warp streams were slower on the long rows (C4 PC apply 47 -> 68 ms): DPP_WS_GMAX caps
// the lane-group width (4 entries per lane) up to which a lane-per-row kernel is chosen.
inline bool pu_use_ws(double avg) {
    static const int gmax = [] { const char *e = std::getenv("DPP_WS_GMAX"); return e ? std::atoi(e) : 32; }();
    return pu_mode() == 3 || pu_mode() == 5 || (pu_mode() == 4 && pu_lane_group(avg) <= gmax);
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
    if (chunk >= (1 << 16)) return false;   // local row index in 16 bits of the row header
    if (p16(8LL * chunk) + 8192 > (long long)PU_SMEM_LIMIT) return false;   // before any work: the x slice alone is too large
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
    k_pu_hstart<<<(C + 32) / 32, 32, 0, c->s>>>(nh, H.p, C, hstart.p);
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
        k_pu_push_keys<<<grid_for(nh, 256, c->sms), 256, 0, c->s>>>(nh, H.p, hstart.p, L, lev.p, n, chunk, k2.p, slot.p,
                                                                    P->tx.p);
        launched(c);
        int nb = 1;
        while (nb < 31 && (1LL << nb) <= n) ++nb;
        size_t tb = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, k2.p, k2s.p, slot.p, slots.p, nh, 0, 8 + nb, c->s));
        DBuf<char> t(tb, c->s);
        CK(cub::DeviceRadixSort::SortPairs(t.p, tb, k2.p, k2s.p, slot.p, slots.p, nh, 0, 8 + nb, c->s));
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
    {
        std::vector<int> lr((size_t)C * L);
        for (size_t i = 0; i < lr.size(); ++i) lr[i] = hlp[i + 1] - hlp[i];
        P->lrows.alloc(lr.size(), c->s);
        P->lrows.upload(lr.data(), lr.size());
    }
    auto part_bytes = [&](int q0, int q1) {
        return pu_block_bytes(q1 - q0, (long long)hr[q1] - hr[q0], (long long)hp[q1] - hp[q0]);
    };
    int fmt = pu_mode() == 0 ? 1 : (pu_use_ws((double)S.nnz / n) && !T.W.rows) ? 2 : 0;
    auto ws_plan = [&]() -> bool {   // warp streams (k_trsv_ws)
        static const int nw_env = [] { const char *e = std::getenv("DPP_WS_WARPS"); return e ? std::atoi(e) : 8; }();
        static const int ns_env = [] { const char *e = std::getenv("DPP_WS_SLOTS"); return e ? std::atoi(e) : 2; }();
        const int NW = std::max(1, std::min(16, nw_env)), NS = std::max(2, std::min(WS_NS_MAX, ns_env));
        const size_t fixed = ws_fixed(chunk, hmax, NW, NS);
        if (fixed + (size_t)NW * NS * 2048 > PU_SMEM_LIMIT) return false;
        const int slot = (int)(((PU_SMEM_LIMIT - fixed) / ((size_t)NW * NS)) & ~(size_t)127);
        // chunks: the rows of a (CTA, level) cut evenly into ceil(rows / 32) chunks
        std::vector<int4> ctab;
        std::vector<int> cstart(C + 1, 0);
        for (int d = 0; d < C; ++d) {
            cstart[d] = (int)ctab.size();
            for (int l = 0; l < L; ++l) {
                const int a0 = hlp[d * L + l], nr = hlp[d * L + l + 1] - a0;
                const int nch = (nr + 31) / 32;
                for (int cc = 0; cc < nch; ++cc) {
                    const int q0 = a0 + (int)((long long)nr * cc / nch), q1 = a0 + (int)((long long)nr * (cc + 1) / nch);
                    int mxl = 0;
                    for (int q = q0; q < q1; ++q) mxl = std::max(mxl, hr[q + 1] - hr[q]);
                    const int w = q1 - q0, ngr = (mxl + 3) / 4, np = hp[q1] - hp[q0];
                    if (16 + ws_group_bytes(w) > slot || 16 + ws_tail_bytes(w, np) > slot || np >= (1 << 27)) return false;
                    ctab.push_back(make_int4(q0, w, ngr, np));
                }
            }
        }
        cstart[C] = (int)ctab.size();
        const int nchunks = (int)ctab.size();
        if (nchunks == 0) return false;
        // streams: chunk g of CTA d belongs to warp g % NW; a stream's pieces are contiguous
        std::vector<long long> cbase(nchunks), poffs;
        std::vector<int> pidx((size_t)C * NW + 1, 0);
        long long cur = 0;
        for (int d = 0; d < C; ++d)
            for (int wv = 0; wv < NW; ++wv) {
                pidx[(size_t)d * NW + wv] = (int)poffs.size();
                for (int gc = cstart[d] + wv; gc < cstart[d + 1]; gc += NW) {
                    cbase[gc] = cur;
                    WsWalk wk{ctab[gc].y, ctab[gc].z, ctab[gc].w, slot};
                    wk.first();
                    do poffs.push_back(cur + wk.off); while (wk.next());
                    cur += wk.off + wk.bytes;
                }
                poffs.push_back(cur);
            }
        pidx[(size_t)C * NW] = (int)poffs.size();
        P->C = C; P->chunk = chunk; P->L = L; P->hmax = hmax; P->smax = 0;
        P->stage = slot; P->nst = NS; P->threads = 32 * NW; P->fmt = 2; P->G = 1; P->widest = 1;
        P->blocks.alloc((size_t)std::max<long long>(cur, 16), c->s);
        P->boff.alloc(poffs.size(), c->s);
        P->boff.upload(poffs.data(), poffs.size());
        P->sstart.alloc(pidx.size(), c->s);
        P->sstart.upload(pidx.data(), pidx.size());
        DBuf<int4> dct(ctab.size(), c->s);
        DBuf<long long> dcb(cbase.size(), c->s);
        dct.upload(ctab.data(), ctab.size());
        dcb.upload(cbase.data(), cbase.size());
        k_ws_fill<<<grid_for(n, 128, c->sms), 128, 0, c->s>>>(n, chunk, pu_chunkp(chunk), pu_chunkp(chunk) + hmax - 1, slot,
                                                              nchunks, dct.p, dcb.p, perm.p, rpp.p, S.ptr.p, S.idx.p,
                                                              S.val.p, T.diag.n ? T.diag.p : nullptr, lev.p, H.p,
                                                              hstart.p, pptr.p, k2s.p, slots.p, P->blocks.p);
        launched(c);
        CK(cudaStreamSynchronize(c->s));
        if (TraceScope::on())
            std::fprintf(stderr, "[dpp-trace]   ws_plan n=%d C=%d L=%d chunks %d pieces %zu warps %d slots %d x %d B halo max %d bytes=%lld\n",
                         n, C, L, nchunks, poffs.size() - (size_t)C * NW, NW, NS, slot, hmax, cur);
        T.pu = std::move(P);
        return true;
    };
    auto gs_plan = [&]() -> bool {   // global streams (k_trsv_gs): no ring, x slice + halo in shared memory
        static const int nw_env = [] { const char *e = std::getenv("DPP_GS_WARPS"); return e ? std::atoi(e) : 16; }();
        const int NW = std::max(1, std::min(GS_WARPS_MAX - (C > 16 ? 1 : 0), nw_env));   // + an importer warp beyond one cluster
        if (gs_smem(chunk, hmax) > PU_SMEM_LIMIT) return false;
        // chunks: the rows of a (CTA, level) cut evenly into ceil(rows / 32) chunks
        std::vector<int4> ctab;
        std::vector<int> cstart(C + 1, 0);
        for (int d = 0; d < C; ++d) {
            cstart[d] = (int)ctab.size();
            for (int l = 0; l < L; ++l) {
                const int a0 = hlp[d * L + l], nr = hlp[d * L + l + 1] - a0;
                const int nch = (nr + 31) / 32;
                for (int cc = 0; cc < nch; ++cc) {
                    const int q0 = a0 + (int)((long long)nr * cc / nch), q1 = a0 + (int)((long long)nr * (cc + 1) / nch);
                    int mxl = 0;
                    for (int q = q0; q < q1; ++q) mxl = std::max(mxl, hr[q + 1] - hr[q]);
                    const int np = hp[q1] - hp[q0];
                    if (np >= (1 << 27)) return false;
                    ctab.push_back(make_int4(q0, q1 - q0, (mxl + 3) / 4, np));
                }
            }
        }
        cstart[C] = (int)ctab.size();
        const int nchunks = (int)ctab.size();
        if (nchunks == 0) return false;
        // streams: chunk g of CTA d belongs to warp g % NW; a stream's chunks are contiguous
        std::vector<long long> cbase(nchunks), soff((size_t)C * NW, 0);
        std::vector<int> scnt((size_t)C * NW, 0);
        long long cur = 0;
        for (int d = 0; d < C; ++d)
            for (int wv = 0; wv < NW; ++wv) {
                soff[(size_t)d * NW + wv] = cur;
                for (int gc = cstart[d] + wv; gc < cstart[d + 1]; gc += NW) {
                    cbase[gc] = cur;
                    cur += gs_chunk_bytes(ctab[gc].y, ctab[gc].z, ctab[gc].w);
                    ++scnt[(size_t)d * NW + wv];
                }
            }
        P->C = C; P->chunk = chunk; P->L = L; P->hmax = hmax; P->smax = 0;
        P->stage = 128; P->nst = 1;   // unused (no ring); kept non-zero for the shared launch arithmetic
        P->threads = 32 * NW; P->fmt = 3; P->G = 1; P->widest = 1;
        if (C > 16) {   // several clusters: the cross-cluster halo pairs, by consumer and source level
            if (nh == 0) return false;
            DBuf<unsigned long long> ik(nh, c->s), iks(nh, c->s), iv(nh, c->s);
            DBuf<int> ncross(1, c->s);
            CK(cudaMemsetAsync(ncross.p, 0, sizeof(int), c->s));
            P->imp.alloc(nh, c->s);
            k_pu_import_keys<<<grid_for(nh, 256, c->sms), 256, 0, c->s>>>(nh, H.p, hstart.p, lev.p, chunk, ik.p, iv.p,
                                                                          ncross.p);
            launched(c);
            size_t tb = 0;
            CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, ik.p, iks.p, iv.p, P->imp.p, nh, 0, 64, c->s));
            DBuf<char> t(tb, c->s);
            CK(cub::DeviceRadixSort::SortPairs(t.p, tb, ik.p, iks.p, iv.p, P->imp.p, nh, 0, 64, c->s));
            launched(c);
            P->istart.alloc(C + 1, c->s);
            k_pu_hstart<<<(C + 32) / 32, 32, 0, c->s>>>(nh, iks.p, C, P->istart.p);
            launched(c);
            CK(cudaStreamSynchronize(c->s));   // the key buffers are freed on return
            P->threads = 32 * (NW + 1);        // + the importer warp
        }
        P->blocks.alloc((size_t)cur + 8192 + 4096, c->s);   // slack: the L2 prefetch of a stream's last chunk
        P->boff.alloc(soff.size(), c->s);
        P->boff.upload(soff.data(), soff.size());
        P->sstart.alloc(scnt.size(), c->s);
        P->sstart.upload(scnt.data(), scnt.size());
        DBuf<int4> dct(ctab.size(), c->s);
        DBuf<long long> dcb(cbase.size(), c->s);
        dct.upload(ctab.data(), ctab.size());
        dcb.upload(cbase.data(), cbase.size());
        k_gs_fill<<<grid_for(n, 128, c->sms), 128, 0, c->s>>>(n, chunk, pu_chunkp(chunk), pu_chunkp(chunk) + hmax - 1,
                                                              nchunks, dct.p, dcb.p, perm.p, rpp.p, S.ptr.p, S.idx.p,
                                                              S.val.p, T.diag.n ? T.diag.p : nullptr, lev.p, H.p,
                                                              hstart.p, pptr.p, k2s.p, slots.p, P->blocks.p);
        launched(c);
        CK(cudaStreamSynchronize(c->s));
        if (TraceScope::on())
            std::fprintf(stderr, "[dpp-trace]   gs_plan n=%d C=%d (%d clusters) L=%d chunks %d warps %d halo max %d bytes=%lld\n",
                         n, C, (C + 15) / 16, L, nchunks, NW, hmax, cur);
        T.pu = std::move(P);
        return true;
    };
    if (C > 16 && (fmt != 2 || pu_mode() == 3)) return false;   // only the global-stream kernel spans clusters
    if (fmt == 2) {
        ++hmax;   // one zero slot after the halo: the padding entries' source
        if (pu_chunkp(chunk) + hmax < (1 << 16) && (pu_mode() == 3 ? ws_plan() : gs_plan())) return true;   // 16-bit column codes
        if (pu_mode() == 3 || pu_mode() == 5 || C > 16) return false;
        --hmax;   // auto: the row-major plan instead
        fmt = 0;
    }
    if (fmt) ++hmax;
    if (fmt && pu_chunkp(chunk) + hmax >= (1 << 16)) return false;
    std::vector<int> hcnt;   // lvl format: per sorted row, entries of class early / mid / late
    if (fmt == 1) {
        DBuf<int> dcnt(3 * (size_t)n, c->s);
        k_lv_counts<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, perm.p, S.ptr.p, S.idx.p, lev.p, dcnt.p);
        launched(c);
        hcnt = dcnt.to_host();
    }
    std::vector<int> pch;    // lvl format: chunks of part i are ctab[pch[i] .. pch[i+1])
    std::vector<int4> ctab;  //   {ebase, early, mid, late columns}
    std::vector<int> pstart, plev, sstart(C + 1, 0);
    std::vector<long long> pboff;
    int smax = 0, widest = 1;
    long long mx = 16;
    bool ok = false;
    for (int tries = 0; tries < 4 && !ok; ++tries) {
        const int smax_est = tries == 0 ? L : smax;
        const size_t fixed = fmt == 1 ? lv_fixed(chunk, L, hmax, smax_est) : pu_fixed(chunk, L, hmax, smax_est);
        if (fixed + 2 * 16384 >= PU_SMEM_LIMIT) return false;
        long long cap = (long long)(PU_SMEM_LIMIT - fixed) / 3;
        if (cap < 16384) cap = (long long)(PU_SMEM_LIMIT - fixed) / 2;
        // >= LV_TEAMS + 2 one-block ring slots (12 smaller slots measured slower: 2.69 vs 1.78 ms per
        // C2 PC apply); a level bigger than a slot becomes several parts, dealt to the team's warps
        if (fmt == 1) cap = (long long)(PU_SMEM_LIMIT - fixed) / (LV_TEAMS + 2);
        cap &= ~127LL;
        pstart.clear(); plev.clear(); pboff.assign(1, 0);
        pch.assign(1, 0); ctab.clear();
        smax = 0; mx = 16; widest = 1;
        bool fit = true;
        for (int d = 0; d < C && fit; ++d) {
            sstart[d] = (int)plev.size();
            for (int l = 0; l < L && fit; ++l) {
                const int a0 = hlp[d * L + l], a1 = hlp[d * L + l + 1];
                if (fmt == 1) {   // parts grown row by row; chunk maxima tracked incrementally
                    for (int q = a0; q < a1 && fit;) {
                        long long nr = 0, nch = 0, ne = 0, np = 0;
                        int cur[3] = {0, 0, 0}, inc = 0;
                        const int q0 = q;
                        while (q < a1) {
                            const int *rc = &hcnt[3 * (size_t)q];
                            const bool fresh = nch == 0 || inc == 32;
                            int nx[3];   // early columns padded to 8, mid / late to 4 (whole load groups)
                            for (int u = 0; u < 3; ++u) {
                                const int pad = 4;
                                const int want = (rc[u] + pad - 1) / pad * pad;
                                nx[u] = fresh ? want : std::max(cur[u], want);
                            }
                            const long long nch2 = nch + (fresh ? 1 : 0);
                            // a chunk occupies (its rows) x (its padded columns) entries
                            const long long ne2 = fresh ? ne + (nx[0] + nx[1] + nx[2])
                                                        : ne - (long long)inc * (cur[0] + cur[1] + cur[2]) +
                                                              (long long)(inc + 1) * (nx[0] + nx[1] + nx[2]);
                            const long long np2 = np + (hp[q + 1] - hp[q]);
                            if (lv_block_bytes(nch2, nr + 1, ne2, np2) > cap) break;
                            if (fresh) ctab.push_back(make_int4((int)ne, nx[0], nx[1], nx[2]));
                            else ctab.back() = make_int4(ctab.back().x, nx[0], nx[1], nx[2]);
                            nch = nch2; ne = ne2; np = np2; inc = fresh ? 1 : inc + 1; ++nr; ++q;
                            for (int u = 0; u < 3; ++u) cur[u] = nx[u];
                        }
                        if (nr == 0) { fit = false; break; }
                        const long long by = lv_block_bytes(nch, nr, ne, np);
                        pstart.push_back(q0); plev.push_back(l); pboff.push_back(pboff.back() + by);
                        pch.push_back((int)ctab.size());
                        mx = std::max(mx, by);
                        widest = std::max(widest, (int)nch);
                    }
                    continue;
                }
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
    const size_t fixed = fmt == 1 ? lv_fixed(chunk, L, hmax, smax) : pu_fixed(chunk, L, hmax, smax);
    const long long stage = (mx + 127) & ~127LL;
    const int nst = fmt == 1 ? (int)std::min<long long>(LV_NS_MAX, (long long)(PU_SMEM_LIMIT - fixed) / stage)
                             : (int)std::min<long long>(PU_NST_MAX, (long long)(PU_SMEM_LIMIT - fixed) / stage);
    if (nst < (fmt == 1 ? LV_TEAMS + 2 : 2)) return false;
    const long long total = pboff.back();
    DBuf<int> dpstart((size_t)np_ + 1, c->s), dplev((size_t)std::max(np_, 1), c->s);
    dpstart.upload(pstart.data(), pstart.size());
    dplev.upload(plev.data(), plev.size());
    P->sstart.alloc(C + 1, c->s);
    P->sstart.upload(sstart.data(), sstart.size());
    P->boff.alloc((size_t)np_ + 1, c->s);
    P->boff.upload(pboff.data(), pboff.size());
    if (fmt == 1) {
        P->slev.alloc(std::max(np_, 1), c->s);
        P->slev.upload(plev.data(), np_);
    }
    P->C = C;
    P->chunk = chunk;
    P->L = L;
    P->smax = smax;
    P->hmax = hmax;
    P->stage = (int)stage;
    P->nst = nst;
    P->G = pu_lane_group((double)S.nnz / n);
    static const int force_g = [] { const char *e = std::getenv("DPP_PU_G"); return e ? std::atoi(e) : 0; }();
    if (force_g && P->G < force_g) P->G = force_g;   // experiment: wider lane groups for thin rows
    static const int set_g = [] { const char *e = std::getenv("DPP_PU_GSET"); return e ? std::atoi(e) : 0; }();
    if (set_g && n == set_g / 100) P->G = set_g % 100;   // experiment: G for one triangle size (n*100+G)
    int threads = 64;
    while (threads < PU_THREADS && (threads / P->G) < widest) threads *= 2;
    static const int force_thr = [] { const char *e = std::getenv("DPP_PU_THREADS"); return e ? std::atoi(e) : 0; }();
    if (force_thr) threads = std::min(threads, force_thr);
    P->threads = threads;
    P->widest = widest;
    P->fmt = fmt;
    P->blocks.alloc((size_t)total, c->s);
    if (np_ && fmt == 1) {
        DBuf<int> dpch(pch.size(), c->s);
        DBuf<int4> dct(ctab.size(), c->s);
        dpch.upload(pch.data(), pch.size());
        dct.upload(ctab.data(), ctab.size());
        const int zero_code = pu_chunkp(chunk) + hmax - 1;
        k_lv_headers<<<grid_for(np_, 128, c->sms), 128, 0, c->s>>>(np_, dpstart.p, dpch.p, dplev.p, rpp.p, dct.p,
                                                                   zero_code, P->boff.p, P->blocks.p);
        launched(c);
        k_lv_fill<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, chunk, pu_chunkp(chunk), zero_code, np_, dpstart.p,
                                                              dpch.p, perm.p, rpp.p, P->boff.p, S.ptr.p, S.idx.p,
                                                              S.val.p, T.diag.n ? T.diag.p : nullptr, lev.p, H.p,
                                                              hstart.p, pptr.p, k2s.p, slots.p, dct.p, P->blocks.p);
        launched(c);
        CK(cudaStreamSynchronize(c->s));   // the chunk tables are freed on return
    } else if (np_) {
        k_pu_headers<<<grid_for(np_, 256, c->sms), 256, 0, c->s>>>(np_, dpstart.p, dplev.p, rptr.p, rpp.p,
                                                                   P->blocks.p, P->boff.p);
        launched(c);
        k_pu_fill<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, chunk, pu_chunkp(chunk), np_, dpstart.p, perm.p,
                                                              rptr.p, rpp.p, P->boff.p, S.ptr.p, S.idx.p, S.val.p,
                                                              T.diag.n ? T.diag.p : nullptr, H.p, hstart.p, pptr.p,
                                                              k2s.p, slots.p, lev.p, P->blocks.p);
        launched(c);
    }
    CK(cudaStreamSynchronize(c->s));
    if (TraceScope::on())
        std::fprintf(stderr, "[dpp-trace]   push_plan n=%d C=%d L=%d steps max %d G=%d thr=%d halo max %d (pairs %d) stage=%lld nst=%d fmt=%d bytes=%lld widest=%d\n",
                     n, C, L, smax, P->G, threads, hmax, nh, stage, nst, fmt, total, widest);
    T.pu = std::move(P);
    return true;
}

}  // namespace

bool push_plan(Ctx *c, Tri &T, const DBuf<int> &lev, int L) {
    DPP_TRACE_SCOPE(c, "tri.push_plan");
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
        setk((const void *)k_trsv_lvl);
        setk((const void *)k_trsv_ws);
        setk((const void *)k_trsv_gs);
        attr = true;
    }
    // as many CTAs as useful: each keeps >= ~2k rows of x
    const int C0 = std::max(2, std::min(PU_MAX, (n + 2047) / 2048));
    // DPP_GS_MIN_CLUSTERS > 1 (tests): skip the single-cluster plans
    static const int cl_min = [] { const char *e = std::getenv("DPP_GS_MIN_CLUSTERS"); return e ? std::atoi(e) : 1; }();
    for (int C = C0; C <= PU_MAX && cl_min <= 1; ++C)
        if (try_push(c, T, lev, L, C)) return true;
    // x too large for one cluster's shared memory: thin-row triangles spread over several clusters
    // of 16 (global-stream kernel, cross-cluster sources imported from global memory)
    static const int cl_max = [] { const char *e = std::getenv("DPP_GS_CLUSTERS"); return e ? std::atoi(e) : 9; }();
    if (pu_use_ws((double)T.strict.nnz / n) && pu_mode() != 3 && !T.W.rows)
        for (int ncl = std::max(2, cl_min); ncl <= cl_max; ++ncl) {
            if ((n + 16 * ncl - 1) / (16 * ncl) >= (1 << 16)) continue;   // slices still too long
            if (try_push(c, T, lev, L, 16 * ncl)) return true;
        }
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
    // level-mbarrier sweep (default): no polling; DPP_PU_MODE=flow|push selects the others
    const int mode = pu_mode();
    if (P.fmt == 3) {
        static const int nap = [] { const char *e = std::getenv("DPP_GS_NAP"); return e ? std::atoi(e) : 0; }();
        cfg.blockDim = dim3(P.threads, 1, 1);
        cfg.dynamicSmemBytes = gs_smem(P.chunk, P.hmax);
#ifdef DPP_WS_PH
        static const char *ph_pathw = std::getenv("DPP_WS_PH");
        unsigned long long *phw = nullptr, *hopb = nullptr;
        const size_t nphw = (size_t)P.C * T.ncomp * (P.threads / 32) * 8;
        cudaEvent_t pe0w = nullptr, pe1w = nullptr;
        if (ph_pathw && *ph_pathw && !c->capturing) {
            CK(cudaStreamSynchronize(st));
            CK(cudaMalloc((void **)&phw, nphw * 8));
            CK(cudaMemset(phw, 0, nphw * 8));
            CK(cudaMemcpyToSymbol(g_ws_ph, &phw, sizeof(phw)));
            CK(cudaMalloc((void **)&hopb, sizeof(unsigned long long) * 32 * GS_HOP_MAX * 4));
            CK(cudaMemset(hopb, 0, sizeof(unsigned long long) * 32 * GS_HOP_MAX * 4));
            CK(cudaMemcpyToSymbol(g_ws_hop, &hopb, sizeof(hopb)));
            cudaEventCreate(&pe0w); cudaEventCreate(&pe1w);
            cudaEventRecord(pe0w, st);
        }
#endif
        const bool multi = P.C > 16;
        if (multi) {   // the importers poll x: nothing of the previous sweep may look solved
            CK(cudaMemsetAsync(x, 0xFF, sizeof(double) * (size_t)T.n, st));
            cfg.gridDim = dim3(P.C * T.ncomp, 1, 1);
            at[0].val.clusterDim.x = 16;
            if (TraceScope::on() && !c->capturing) {
                int nact = -1;
                cudaOccupancyMaxActiveClusters(&nact, k_trsv_gs, &cfg);
                std::fprintf(stderr, "[dpp-trace]   gs launch n=%d: %d clusters of 16, %zu B shared per CTA, co-resident clusters %d\n",
                             T.n, P.C / 16, (size_t)cfg.dynamicSmemBytes, nact);
            }
        }
        CK(cudaLaunchKernelEx(&cfg, k_trsv_gs, T.n / T.ncomp, T.ncomp, P.chunk, P.hmax, P.C, (int)T.backward, B, O,
                              (const int *)P.sstart.p, multi ? (const unsigned long long *)P.imp.p : nullptr,
                              multi ? (const int *)P.istart.p : nullptr, b, x, xadd, xout, nap));
        launched(c);
#ifdef DPP_WS_PH
        if (phw) {
            cudaEventRecord(pe1w, st);
            CK(cudaStreamSynchronize(st));
            float ms = 0;
            cudaEventElapsedTime(&ms, pe0w, pe1w);
            std::vector<unsigned long long> h(nphw);
            CK(cudaMemcpy(h.data(), phw, nphw * 8, cudaMemcpyDeviceToHost));
            unsigned long long *z = nullptr;
            CK(cudaMemcpyToSymbol(g_ws_ph, &z, sizeof(z)));
            cudaFree(phw);
            if (FILE *f = std::fopen(ph_pathw, "a")) {
                const int nwv = P.threads / 32;
                {
                    std::vector<unsigned long long> hh((size_t)32 * GS_HOP_MAX * 4);
                    CK(cudaMemcpy(hh.data(), hopb, hh.size() * 8, cudaMemcpyDeviceToHost));
                    unsigned long long *zz = nullptr;
                    CK(cudaMemcpyToSymbol(g_ws_hop, &zz, sizeof(zz)));
                    cudaFree(hopb);
                    std::string hp = std::string(ph_pathw) + ".hop";
                    if (FILE *fh = std::fopen(hp.c_str(), "a")) {
                        std::fprintf(fh, "# gs n=%d C=%d ncomp=%d L=%d warps=%d\n", T.n, P.C, T.ncomp, P.L, nwv);
                        for (size_t i = 0; i < hh.size() / 4; ++i)
                            if (hh[i * 4 + 3])
                                std::fprintf(fh, "%zu %zu %llu %llu %llu %llu\n", i / GS_HOP_MAX, i % GS_HOP_MAX, hh[i * 4],
                                             hh[i * 4 + 1], hh[i * 4 + 2], hh[i * 4 + 3]);
                        std::fclose(fh);
                    }
                }
                std::fprintf(f, "# gs n=%d C=%d ncomp=%d L=%d warps=%d us=%.2f\n", T.n, P.C, T.ncomp, P.L, nwv, ms * 1e3);
                for (size_t i = 0; i < nphw / 8; ++i) {
                    const unsigned long long *o = &h[i * 8];
                    std::fprintf(f, "%zu %zu %llu %llu %llu %llu %llu %llu %llu %llu\n", i / nwv, i % nwv, o[0], o[1], o[2],
                                 o[3], o[4], o[5], o[6], o[7]);
                }
                std::fclose(f);
            }
        }
#endif
        return;
    }
    if (P.fmt == 2) {
        static const int nap = [] { const char *e = std::getenv("DPP_WS_NAP"); return e ? std::atoi(e) : 0; }();
        cfg.blockDim = dim3(P.threads, 1, 1);
        cfg.dynamicSmemBytes = ws_fixed(P.chunk, P.hmax, P.threads / 32, P.nst) + (size_t)(P.threads / 32) * P.nst * P.stage;
#ifdef DPP_WS_TL
        static const char *tl_path = std::getenv("DPP_WS_TL");
        unsigned long long *tlb = nullptr;
        const size_t ntl = (size_t)P.C * T.ncomp * (P.threads / 32) * WS_TL_MAXC * 6;
        cudaEvent_t te0 = nullptr, te1 = nullptr;
        if (tl_path && *tl_path && !c->capturing) {
            CK(cudaStreamSynchronize(st));
            CK(cudaMalloc((void **)&tlb, ntl * 8));
            CK(cudaMemset(tlb, 0, ntl * 8));
            CK(cudaMemcpyToSymbol(g_ws_tl, &tlb, sizeof(tlb)));
            cudaEventCreate(&te0); cudaEventCreate(&te1);
            cudaEventRecord(te0, st);
        }
#endif
        CK(cudaLaunchKernelEx(&cfg, k_trsv_ws, T.n / T.ncomp, T.ncomp, P.chunk, P.hmax, P.stage, P.nst, B, O,
                              (const int *)P.sstart.p, b, x, xadd, xout, nap));
        launched(c);
#ifdef DPP_WS_TL
        if (tlb) {
            cudaEventRecord(te1, st);
            CK(cudaStreamSynchronize(st));
            float ms = 0;
            cudaEventElapsedTime(&ms, te0, te1);
            std::vector<unsigned long long> h(ntl);
            CK(cudaMemcpy(h.data(), tlb, ntl * 8, cudaMemcpyDeviceToHost));
            unsigned long long *z = nullptr;
            CK(cudaMemcpyToSymbol(g_ws_tl, &z, sizeof(z)));
            cudaFree(tlb);
            if (FILE *f = std::fopen(tl_path, "a")) {
                std::fprintf(f, "# ws n=%d C=%d ncomp=%d L=%d warps=%d slots=%d slot=%d us=%.2f\n", T.n, P.C, T.ncomp, P.L,
                             P.threads / 32, P.nst, P.stage, ms * 1e3);
                const int nwv = P.threads / 32;
                for (size_t i = 0; i < ntl / 6; ++i) {
                    const unsigned long long *o = &h[i * 6];
                    if (o[3]) std::fprintf(f, "%zu %zu %zu %llu %llu %llu %llu %llu %llu\n", i / WS_TL_MAXC / nwv,
                                           (i / WS_TL_MAXC) % nwv, i % WS_TL_MAXC, o[0], o[1], o[2], o[3], o[4], o[5]);
                }
                std::fclose(f);
            }
        }
#endif
        return;
    }
    if (P.fmt == 1) {
        const size_t lfixed = lv_fixed(P.chunk, P.L, P.hmax, P.smax);
        if (wp || P.nst < LV_TEAMS + 2 || lfixed + (size_t)P.nst * P.stage > PU_SMEM_LIMIT)
            DPP_FAIL(DPP_ERR_RUNTIME, "level-mbarrier sweep: plan does not fit");
        // LV_TEAMS level teams, each wide enough for the widest block (in 32-row chunks) in one round
        static const int pt_env = [] { const char *e = std::getenv("DPP_LVL_PER_TEAM"); return e ? std::atoi(e) : 0; }();
        const int per_team = pt_env ? pt_env : std::max(1, std::min(P.widest, LV_THREADS / (32 * LV_TEAMS)));
        cfg.blockDim = dim3(32 * LV_TEAMS * per_team, 1, 1);   // per_team warps on each sub-partition
        cfg.dynamicSmemBytes = lfixed + (size_t)P.nst * P.stage;
        const int *lr = P.lrows.p, *txp = P.tx.p, *ss = P.sstart.p;
        const int nn = T.n / T.ncomp;
#ifdef DPP_FLOW_PHASES
        static const char *ph_path2 = std::getenv("DPP_FLOW_PHASES");
        unsigned long long *phb2 = nullptr;
        const size_t nph2 = (size_t)P.C * T.ncomp * 32 * 8;
        cudaEvent_t pe0 = nullptr, pe1 = nullptr;
        unsigned long long *tlb = nullptr;
        const size_t ntl = (size_t)P.C * T.ncomp * std::max(P.smax, 1) * 4;
        if (ph_path2 && *ph_path2 && !c->capturing) {
            CK(cudaStreamSynchronize(st));
            CK(cudaMalloc((void **)&phb2, nph2 * 8));
            CK(cudaMemset(phb2, 0, nph2 * 8));
            CK(cudaMemcpyToSymbol(g_flow_phase, &phb2, sizeof(phb2)));
            CK(cudaMalloc((void **)&tlb, ntl * 8));
            std::vector<unsigned long long> init(ntl, 0);
            for (size_t i = 0; i < ntl; i += 4) { init[i + 1] = ~0ull; init[i + 3] = ~0ull; }
            CK(cudaMemcpy(tlb, init.data(), ntl * 8, cudaMemcpyHostToDevice));
            CK(cudaMemcpyToSymbol(g_flow_tl, &tlb, sizeof(tlb)));
            const int sm_ = P.smax;
            CK(cudaMemcpyToSymbol(g_flow_smax, &sm_, sizeof(int)));
            const int np_env = std::getenv("DPP_LVL_NOPUSH") ? 1 : 0;
            CK(cudaMemcpyToSymbol(g_flow_nopush, &np_env, sizeof(int)));
            const int rot_env = std::getenv("DPP_LVL_ROT") ? std::atoi(std::getenv("DPP_LVL_ROT")) : 0;
            CK(cudaMemcpyToSymbol(g_flow_rot, &rot_env, sizeof(int)));
            cudaEventCreate(&pe0); cudaEventCreate(&pe1);
            cudaEventRecord(pe0, st);
        }
#endif
        e = cudaLaunchKernelEx(&cfg, k_trsv_lvl, nn, T.ncomp, P.chunk, P.L, P.smax, P.hmax, P.stage, P.nst, B, O, ss,
                               (const int *)P.slev.p, txp, lr, b, x, xadd, xout, l2pf);
#ifdef DPP_FLOW_PHASES
        if (phb2) {
            cudaEventRecord(pe1, st);
            CK(cudaStreamSynchronize(st));
            float ms = 0;
            cudaEventElapsedTime(&ms, pe0, pe1);
            std::vector<unsigned long long> h(nph2);
            CK(cudaMemcpy(h.data(), phb2, nph2 * 8, cudaMemcpyDeviceToHost));
            unsigned long long *z = nullptr;
            CK(cudaMemcpyToSymbol(g_flow_phase, &z, sizeof(z)));
            CK(cudaMemcpyToSymbol(g_flow_tl, &z, sizeof(z)));
            cudaFree(phb2);
            {
                std::vector<unsigned long long> tl(ntl);
                CK(cudaMemcpy(tl.data(), tlb, ntl * 8, cudaMemcpyDeviceToHost));
                cudaFree(tlb);
                std::string tp = std::string(ph_path2) + ".tl";
                if (FILE *f = std::fopen(tp.c_str(), "a")) {
                    std::fprintf(f, "# n=%d C=%d ncomp=%d smax=%d L=%d\n", T.n, P.C, T.ncomp, P.smax, P.L);
                    for (size_t i = 0; i < ntl / 4; ++i)
                        if (tl[i * 4 + 2]) std::fprintf(f, "%zu %zu %llu %llu %llu %llu\n", i / P.smax, i % P.smax, tl[i * 4], tl[i * 4 + 3], tl[i * 4 + 1], tl[i * 4 + 2]);
                    std::fclose(f);
                }
            }
            if (FILE *f = std::fopen(ph_path2, "a")) {
                std::fprintf(f, "# lvl n=%d C=%d ncomp=%d L=%d G=%d threads=%d us=%.2f\n", T.n, P.C, T.ncomp, P.L, 1, (int)cfg.blockDim.x, ms * 1e3);
                for (size_t i = 0; i < nph2 / 8; ++i) {
                    const unsigned long long *o = &h[i * 8];
                    if (o[6]) std::fprintf(f, "%zu %zu %llu %llu %llu %llu %llu %llu %llu %llu\n", i / 32, i % 32, o[0], o[1], o[2], o[3], o[4], o[5], o[6], o[7]);
                }
                std::fclose(f);
            }
        }
#endif
        CK(e);
        launched(c);
        return;
    }
    // dataflow for thin rows (C2: G = 2 / 8); the level-synchronous kernel measured faster for
    // the 32-lane groups of the long-row triangles of configs 3/4 (34.0 vs 37.8 ms per PC apply at C3)
    static const int flow_gmax = [] { const char *e = std::getenv("DPP_FLOW_GMAX"); return e ? std::atoi(e) : 16; }();
    if (flow && mode != 2 && P.G <= flow_gmax && !wp && !dbg && P.L >= nst_f && nst_b >= 2 && nst_f >= 2 &&
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
#ifdef DPP_FLOW_PHASES
        static const char *ph_path = std::getenv("DPP_FLOW_PHASES");
        unsigned long long *phb = nullptr;
        const size_t nph = (size_t)P.C * T.ncomp * 32 * 8;
        if (ph_path && *ph_path && !c->capturing) {
            CK(cudaStreamSynchronize(st));
            CK(cudaMalloc((void **)&phb, nph * 8));
            CK(cudaMemset(phb, 0, nph * 8));
            CK(cudaMemcpyToSymbol(g_flow_phase, &phb, sizeof(phb)));
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0, st);
            switch (P.G) {
                case 2: e = cudaLaunchKernelEx(&cfg, k_trsv_flow<2>, T.n / T.ncomp, T.ncomp, P.chunk, P.L, P.smax, P.hmax, (int)stage_f, nst_f, B, O, (const int *)P.sstart.p, b, x, xadd, xout, l2pf, fdbg); break;
                case 4: e = cudaLaunchKernelEx(&cfg, k_trsv_flow<4>, T.n / T.ncomp, T.ncomp, P.chunk, P.L, P.smax, P.hmax, (int)stage_f, nst_f, B, O, (const int *)P.sstart.p, b, x, xadd, xout, l2pf, fdbg); break;
                case 8: e = cudaLaunchKernelEx(&cfg, k_trsv_flow<8>, T.n / T.ncomp, T.ncomp, P.chunk, P.L, P.smax, P.hmax, (int)stage_f, nst_f, B, O, (const int *)P.sstart.p, b, x, xadd, xout, l2pf, fdbg); break;
                case 16: e = cudaLaunchKernelEx(&cfg, k_trsv_flow<16>, T.n / T.ncomp, T.ncomp, P.chunk, P.L, P.smax, P.hmax, (int)stage_f, nst_f, B, O, (const int *)P.sstart.p, b, x, xadd, xout, l2pf, fdbg); break;
                default: e = cudaLaunchKernelEx(&cfg, k_trsv_flow<32>, T.n / T.ncomp, T.ncomp, P.chunk, P.L, P.smax, P.hmax, (int)stage_f, nst_f, B, O, (const int *)P.sstart.p, b, x, xadd, xout, l2pf, fdbg); break;
            }
            cudaEventRecord(e1, st);
            CK(cudaStreamSynchronize(st));
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            std::vector<unsigned long long> h(nph);
            CK(cudaMemcpy(h.data(), phb, nph * 8, cudaMemcpyDeviceToHost));
            unsigned long long *z = nullptr;
            CK(cudaMemcpyToSymbol(g_flow_phase, &z, sizeof(z)));
            cudaFree(phb);
            if (FILE *f = std::fopen(ph_path, "a")) {
                std::fprintf(f, "# n=%d C=%d ncomp=%d L=%d G=%d threads=%d us=%.2f\n", T.n, P.C, T.ncomp, P.L, P.G, (int)cfg.blockDim.x, ms * 1e3);
                for (size_t i = 0; i < nph / 8; ++i) {
                    const unsigned long long *o = &h[i * 8];
                    if (o[6]) std::fprintf(f, "%zu %zu %llu %llu %llu %llu %llu %llu %llu %llu\n", i / 32, i % 32, o[0], o[1], o[2], o[3], o[4], o[5], o[6], o[7]);
                }
                std::fclose(f);
            }
        }
#endif
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
