// Sync-free sparse triangular solves and ILU(0) numeric factorisation.
//
// Reference: linalg.apply_ilu0 / _sgs_sweep (linalg.py:225-227, :383-385) call
// scipy spsolve_triangular (SuperLU gstrs), and linalg.ilu0 (linalg.py:178-222)
// factors with the IKJ loop.  Both are sequential in row order; the dependency
// depth is hundreds of levels, so instead of level sets each
// row is handled by one warp that takes rows in processing order from an
// atomic ticket and spins only on the rows it actually depends on.
//  * TRSV: the solution vector doubles as the ready flag (pre-filled with an
//    all-ones NaN sentinel; a row's value is published with one relaxed
//    store), so a dependency costs one L2 round trip.  Exact zeros are
//    dropped from the factors (exact: they never change a sum).
//  * ILU(0): per-row ready flags with release/acquire; a row skips (does not
//    wait for) pivot rows whose current multiplier numerator is exactly 0,
//    which is exact (l = 0 leaves every update unchanged) and removes the
//    cross-component dependencies of c*(M (x) I) velocity blocks.  The update
//    order per row is the reference's (k ascending, separate mul/sub), so the
//    factors are bitwise those of the reference.
// Deadlock freedom: a warp only waits on rows with an earlier ticket, which
// are owned by warps that are already running.
#include <cub/cub.cuh>

#include <cstdio>
#include <type_traits>
#include <cstdlib>

#include <cooperative_groups.h>

#include "dpp_internal.cuh"

namespace cg = cooperative_groups;

namespace dpp {

static constexpr unsigned long long SENT = 0xFFFFFFFFFFFFFFFFull;
// watchdog: a dependency that never resolves (malformed input) traps instead of hanging the GPU
static constexpr long long SPIN_LIMIT = 1ll << 26;

__device__ __forceinline__ double ld_relaxed(const double *p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(double *p, double v) {
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// level values are the only data exchanged by the level analysis: relaxed (L2) accesses suffice
__device__ __forceinline__ int ld_relaxed_i(const int *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_i(int *p, int v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release(int *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ------------------------------------------------------------------ TRSV
// ------------------------------------------------------------------ level analysis
// One thread per row, all threads resident, rows dealt round-robin across warps
// (consecutive rows land in different warps); a row's level is 1 + the max level
// of the rows it reads.  Smallest unfinished row is always runnable -> progress.
__global__ void __launch_bounds__(256) k_levels(int n, int backward, const int *__restrict__ ptr,
                                                const int *__restrict__ idx, int *level) {
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t W = T >> 5, w = g >> 5, lane = g & 31;
    for (int64_t base = 0; base < n; base += T) {
        const int64_t t = base + lane * W + w;
        if (t >= n) continue;
        const int row = backward ? n - 1 - (int)t : (int)t;
        // dependencies in batches of 8 loads in flight; spin only on the ones not ready.
        // Far dependencies first (CSR columns ascend: the nearest row is last for a
        // lower triangle, first for an upper one): while the nearest -- normally the
        // last to finish -- is pending, the others are already loaded.
        int lv = 0;
        const int rs = ptr[row], re = ptr[row + 1];
        for (int k0 = 0; k0 < re - rs; k0 += 8) {
            const int cnt = min(8, re - rs - k0);
            int lj[8], pj[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                pj[u] = backward ? re - 1 - (k0 + u) : rs + k0 + u;
                DPP_DCHECK(u >= cnt || (backward ? idx[pj[u]] > row : idx[pj[u]] < row));   // a strict triangle
                lj[u] = u < cnt ? ld_relaxed_i(level + idx[pj[u]]) : 0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                long long spins = 0;
                while (lj[u] < 0) {
                    __nanosleep(32);
                    lj[u] = ld_relaxed_i(level + idx[pj[u]]);
                    if (++spins > SPIN_LIMIT) __trap();
                }
                lv = max(lv, lj[u] + 1);
            }
        }
        st_relaxed_i(level + row, lv);
    }
}

// warp per row (small matrices with long rows: coarse AMG levels)
__global__ void __launch_bounds__(256) k_levels_warp(int n, int backward, const int *__restrict__ ptr,
                                                     const int *__restrict__ idx, int *level) {
    const int lane = threadIdx.x & 31;
    const int64_t W = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n; t += W) {
        const int row = backward ? n - 1 - (int)t : (int)t;
        int lv = 0;
        const int rs = ptr[row], re = ptr[row + 1];
        for (int k = lane; k < re - rs; k += 32) {   // far dependencies first (see k_levels)
            const int j = idx[backward ? re - 1 - k : rs + k];
            int lj = ld_relaxed_i(level + j);
            long long spins = 0;
            while (lj < 0) {
                __nanosleep(32);
                lj = ld_relaxed_i(level + j);
                if (++spins > SPIN_LIMIT) __trap();
            }
            lv = max(lv, lj + 1);
        }
        for (int o = 16; o > 0; o >>= 1) lv = max(lv, __shfl_xor_sync(0xffffffffu, lv, o));
        if (lane == 0) st_relaxed_i(level + row, lv);
    }
}

__global__ void k_iota(int n, int *a) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}
__global__ void k_maxlev(int n, const int *lv, int *mx) {
    int m = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) m = max(m, lv[i]);
    atomicMax(mx, m);
}

__global__ void k_levptr(int n, const int *sorted_lev, int nlev, int *levptr) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x) {
        if (i == n) { levptr[nlev] = n; continue; }
        const int l = sorted_lev[i];
        const int prev = i ? sorted_lev[i - 1] : -1;
        for (int k = prev + 1; k <= l; ++k) levptr[k] = i;
    }
}

int tri_levels(Ctx *c, const Csr &S, bool backward, DBuf<int> &order, DBuf<int> *levptr,
               DBuf<int> *lev_out) {
    DPP_TRACE_SCOPE(c, "tri_levels");
    const int n = S.rows;
    order.alloc(n, c->s);
    if (!n) return 0;
    DBuf<int> lev(n, c->s), lev2(n, c->s), rows(n, c->s), mx(1, c->s);
    CK(cudaMemsetAsync(lev.p, 0xFF, sizeof(int) * n, c->s));
    CK(cudaMemsetAsync(mx.p, 0, sizeof(int), c->s));
    // every thread of the grid must be resident (waits are on other threads' rows)
    const int block = 256;
    int per_sm = 0, per_sm_w = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_levels, block, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_w, k_levels_warp, block, 0));
    if (per_sm < 1 || per_sm_w < 1) DPP_FAIL(DPP_ERR_CUDA, "level analysis kernels cannot be resident");
    // the spinning analysis kernels take at most half of every SM, so setup work of
    // other fork_join branches (SpGEMM, other analyses) keeps running beside them
    static const int share = [] { const char *e = std::getenv("DPP_LEVELS_SHARE"); return e ? std::atoi(e) : 2; }();
    per_sm = std::max(1, per_sm / std::max(1, share));
    per_sm_w = std::max(1, per_sm_w / std::max(1, share));
    const int64_t warps_res = (int64_t)c->sms * per_sm_w * (block / 32);
    const double avg = n ? (double)S.nnz / n : 0.0;
    // cooperative launches: the grid is co-resident by construction, even while other
    // setup branches' kernels (or other spinning analyses) hold part of the device --
    // a plain launch could leave blocks whose rows others wait on unscheduled
    int nn = n, bw = backward ? 1 : 0;
    const int *pp = S.ptr.p, *ii = S.idx.p;
    int *lv = lev.p;
    void *args[] = {&nn, &bw, &pp, &ii, &lv};
    if (n <= warps_res && avg > 8.0) {
        const int grid = (int)(((int64_t)n * 32 + block - 1) / block);
        CK(cudaLaunchCooperativeKernel((const void *)k_levels_warp, grid, block, args, 0, c->s));
    } else {
        const int64_t need = ((int64_t)n + 31) / 32 * 32;
        const int64_t cap = (int64_t)c->sms * per_sm * block;
        const int grid = (int)((std::min(need, cap) + block - 1) / block);
        CK(cudaLaunchCooperativeKernel((const void *)k_levels, grid, block, args, 0, c->s));
    }
    launched(c);
    k_iota<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, rows.p);
    launched(c);
    k_maxlev<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, lev.p, mx.p);
    launched(c);
    int hmx = 0;
    CK(cudaMemcpyAsync(&hmx, mx.p, sizeof(int), cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    int bits = 1;
    while (bits < 31 && (1 << bits) <= hmx) ++bits;
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, lev.p, lev2.p, rows.p, order.p, n, 0, bits, c->s));
    DBuf<char> t(tb, c->s);
    CK(cub::DeviceRadixSort::SortPairs(t.p, tb, lev.p, lev2.p, rows.p, order.p, n, 0, bits, c->s));
    launched(c);
    if (lev_out) {
        lev_out->alloc(n, c->s);
        CK(cudaMemcpyAsync(lev_out->p, lev.p, sizeof(int) * n, cudaMemcpyDeviceToDevice, c->s));
    }
    if (levptr) {
        levptr->alloc((size_t)hmx + 2, c->s);
        k_levptr<<<grid_for(n + 1, 256, c->sms), 256, 0, c->s>>>(n, lev2.p, hmx + 1, levptr->p);
        launched(c);
    }
    CK(cudaStreamSynchronize(c->s));
    return hmx + 1;
}

// ------------------------------------------------------------------ dense inverses (small levels)
__global__ void k_tri_dense(int n, const int *ptr, const int *idx, const double *val, const double *diag,
                            double *T) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        for (int p = ptr[r]; p < ptr[r + 1]; ++p) T[(int64_t)r * n + idx[p]] += val[p];
        T[(int64_t)r * n + r] += diag ? diag[r] : 1.0;
    }
}
// column c of T^-1 by substitution: one warp per column, the column lives in
// shared memory, each step is a lane-parallel dot product over a row of T
constexpr int INV_WPB = 4;
__global__ void __launch_bounds__(32 * INV_WPB) k_tri_inverse(int n, int backward, const double *__restrict__ T,
                                                             double *Ti) {
    extern __shared__ double col[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *x = col + (size_t)w * n;
    for (int c = blockIdx.x * INV_WPB + w; c < n; c += gridDim.x * INV_WPB) {
        for (int i = lane; i < n; i += 32) x[i] = 0.0;
        __syncwarp();
        for (int s = 0; s < n; ++s) {
            const int i = backward ? c - s : c + s;
            if (i < 0 || i >= n) break;
            const int j0 = backward ? i + 1 : c, j1 = backward ? c + 1 : i;
            double acc = 0.0;
            for (int j = j0 + lane; j < j1; j += 32) acc += T[(int64_t)i * n + j] * x[j];
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) x[i] = ((i == c ? 1.0 : 0.0) - acc) / T[(int64_t)i * n + i];
            __syncwarp();
        }
        for (int i = lane; i < n; i += 32) Ti[(int64_t)i * n + c] = x[i];
        __syncwarp();
    }
}
// x = Ti b over the triangle's nonzero half; xout = xadd + x
__global__ void k_tri_gemv(int n, int backward, const double *__restrict__ Ti, const double *__restrict__ b,
                           double *x, const double *__restrict__ xadd, double *xout) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int j0 = backward ? (int)r : 0, j1 = backward ? n : (int)r + 1;
        double s = 0.0;
        for (int j = j0 + lane; j < j1; j += 32) s += Ti[r * n + j] * b[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
            x[r] = s;
            if (xout) xout[r] = xadd[r] + s;
        }
    }
    pdl_trigger();
}

__global__ void __launch_bounds__(128) k_trsv(int n, const int *__restrict__ order, const int *__restrict__ ptr,
                                              const int *__restrict__ idx,
                                              const double *__restrict__ val,
                                              const double *__restrict__ diag,
                                              const double *__restrict__ b, double *x, int *ticket,
                                              const double *__restrict__ xadd, double *xout) {
    const int lane = threadIdx.x & 31;
    while (true) {
        int t = 0;
        if (lane == 0) t = atomicAdd(ticket, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= n) return;
        const int row = order[t];
        const int s = ptr[row], e = ptr[row + 1];
        // per-row constants first: their latency must not follow the dependency wait
        double bi = 0.0, di = 1.0, ai = 0.0;
        if (lane == 0) {
            bi = b[row];
            if (diag) di = diag[row];
            if (xout) ai = xadd[row];
        }
        double sum = 0.0;
        for (int p = s + lane; p < e; p += 32) {
            const int j = idx[p];
            const double a = val[p];
            double v = ld_relaxed(x + j);
            long long spins = 0;
            while (__double_as_longlong(v) == (long long)SENT) {
                v = ld_relaxed(x + j);
                if (++spins > SPIN_LIMIT) __trap();
            }
            sum += a * v;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0) {
            double xi = bi - sum;
            if (diag) xi = xi / di;
            if (__double_as_longlong(xi) == (long long)SENT) xi = __longlong_as_double(0x7ff8000000000000ll);
            st_relaxed(x + row, xi);
            if (xout) xout[row] = ai + xi;
        }
    }
}

// ------------------------------------------------------------------ non-parity fast mode
// the exact substitution replaced by k Jacobi sweeps on the triangle,
//     x_0 = D^-1 b,   x_{s+1} = D^-1 (b - S x_s)      (S strict part, D = I for unit factors)
// -- a fixed linear operator, so GMRES stays valid, but iterates and iteration counts
// differ from the reference's (never used unless asked for).  Every sweep is one
// bandwidth-bound pass over S with no dependency chain.  G lanes per scalar row; the
// Kronecker form M (x) I_d is swept on M with d interleaved components per row.
template <int G, int D>
__global__ void __launch_bounds__(256) k_jacobi(int rows, int d, const int *__restrict__ ptr,
                                                const int *__restrict__ idx, const double *__restrict__ val,
                                                const double *__restrict__ diag, const double *__restrict__ b,
                                                const double *__restrict__ xin, double *__restrict__ xo,
                                                const double *__restrict__ xadd, double *__restrict__ xout) {
    pdl_wait();
    // every lane of a warp runs the same trip count (the width-G shuffles stay full)
    const int gl = threadIdx.x % G, gw = (threadIdx.x & 31) / G;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = warp * (32 / G); base < rows; base += nwarp * (32 / G)) {
        const int64_t r = base + gw;
        const bool act = r < rows;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        if (xin && act) {
            const int pe = ptr[r + 1];
            for (int p = ptr[r] + gl; p < pe; p += G) {
                const int j = idx[p];
                const double v = val[p];
                const double *xj = xin + (int64_t)j * d;
                s0 += v * xj[0];
                if (D > 1) s1 += v * xj[1];
                if (D > 2) s2 += v * xj[2];
                if (D > 3) s3 += v * xj[3];
            }
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
            s0 += __shfl_xor_sync(0xffffffffu, s0, o, G);
            if (D > 1) s1 += __shfl_xor_sync(0xffffffffu, s1, o, G);
            if (D > 2) s2 += __shfl_xor_sync(0xffffffffu, s2, o, G);
            if (D > 3) s3 += __shfl_xor_sync(0xffffffffu, s3, o, G);
        }
        if (act && gl < D) {
            const double sq = gl == 0 ? s0 : gl == 1 ? s1 : gl == 2 ? s2 : s3;
            const int64_t R = r * d + gl;
            double y = b[R] - sq;
            if (diag) y = y / diag[r];
            xo[R] = y;
            if (xout) xout[R] = xadd[R] + y;
        }
    }
}

// S' = D^-1 S (rows divided by the diagonal) and x0 = D^-1 b: the sweeps of a scalar
// triangle are then x <- x0 - S' x, plain planned SpMVs
__global__ void k_rowdiv(int rows, const int *__restrict__ ptr, double *val, const double *__restrict__ d) {
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const double dr = d[r];
        for (int p = ptr[r] + (threadIdx.x & 31); p < ptr[r + 1]; p += 32) val[p] = val[p] / dr;
    }
}
__global__ void k_vdiv(int64_t n, const double *__restrict__ b, const double *__restrict__ d, double *o) {
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        o[i] = b[i] / d[i];
    pdl_trigger();
}

Tri make_tri_jacobi(Ctx *c, const Csr &M, bool lower, bool unit, int d, int k) {
    if (d < 1 || d > 4) DPP_FAIL(DPP_ERR_VALUE, "Jacobi sweeps support up to 4 interleaved components");
    Tri T;
    T.backward = !lower;
    T.strict = csr_part(c, M, lower ? -1 : 1, true);
    if (!unit) {
        T.diag.alloc(M.rows, c->s);
        csr_diag(c, M, T.diag.p, nullptr);
    }
    T.ncomp = d;
    T.n = M.rows * d;
    T.nnz_alg = T.strict.nnz * d;
    T.jacobi = k;
    T.nlev = 1;
    T.wb.alloc(T.n, c->s);
    if (d == 1) {
        if (!unit) {
            k_rowdiv<<<grid_for((int64_t)M.rows * 32, 256, c->sms, 8), 256, 0, c->s>>>(M.rows, T.strict.ptr.p,
                                                                                      T.strict.val.p, T.diag.p);
            launched(c);
        }
        spmv_plan(c, T.strict);
        T.W.rows = 0;
        T.wb2.alloc(T.n, c->s);
    }
    return T;
}

static void trsv_jacobi(Ctx *c, const Tri &T, const double *b, double *x, const double *xadd, double *xout,
                        cudaStream_t st) {
    const int rows = T.strict.rows, d = T.ncomp, k = T.jacobi;
    const double *dg = T.diag.n ? T.diag.p : nullptr;
    // the last sweep lands in x: start in x when k is even, in the scratch when odd
    double *buf[2] = {x, T.wb.p};
    int cur = k % 2;
    if (d == 1) {   // x0 = D^-1 b (b itself when unit); sweeps x <- x0 - S' x as planned SpMVs
        const double *x0 = b;
        if (dg) {
            CK(launch_pdl(k_vdiv, dim3(grid_for(rows, 256, c->sms)), dim3(256), 0, st, (int64_t)rows, b, dg,
                          T.wb2.p));
            launched(c);
            x0 = T.wb2.p;
        }
        const double *xin = x0;
        for (int s = 0; s < k; ++s) {
            double *xo = buf[(k - 1 - s) % 2 == 0 ? 0 : 1];
            spmv(c, T.strict, xin, xo, x0, -1.0, st);
            xin = xo;
        }
        if (k == 0 && xin != x) CK(cudaMemcpyAsync(x, xin, sizeof(double) * rows, cudaMemcpyDeviceToDevice, st));
        if (xout) axpby_to(c, rows, xadd, 1.0, x, xout, st);
        return;
    }
    const double avg = rows ? (double)T.strict.nnz / rows : 0.0;
    auto sweep = [&](const double *xin, double *xo, bool last) {
        auto go = [&](auto kern, int G) {
            const int64_t thr = ((int64_t)rows * G + 255) / 256 * 256;
            const int grid = (int)std::min<int64_t>(thr / 256, (int64_t)c->sms * 8);
            CK(launch_pdl(kern, dim3(grid), dim3(256), 0, st, rows, d, (const int *)T.strict.ptr.p,
                          (const int *)T.strict.idx.p, (const double *)T.strict.val.p, dg, b, xin, xo,
                          last ? xadd : (const double *)nullptr, last ? xout : (double *)nullptr));
            launched(c);
        };
        auto pick = [&](auto dtag) {
            constexpr int DD = decltype(dtag)::value;
            if (avg > 24) go(k_jacobi<32, DD>, 32);
            else if (avg > 10) go(k_jacobi<16, DD>, 16);
            else go(k_jacobi<8, DD>, 8);
        };
        if (d == 2) pick(std::integral_constant<int, 2>{});
        else if (d == 3) pick(std::integral_constant<int, 3>{});
        else pick(std::integral_constant<int, 4>{});
    };
    sweep(nullptr, buf[cur], k == 0);
    for (int s = 0; s < k; ++s) {
        sweep(buf[cur], buf[cur ^ 1], s == k - 1);
        cur ^= 1;
    }
}

void trsv(Ctx *c, const Tri &T, const double *b, double *x, int *ticket, const double *xadd,
          double *xout, cudaStream_t st) {
    st = st ? st : c->s;
    if (T.n == 0) return;
    if (T.jacobi) {
        trsv_jacobi(c, T, b, x, xadd, xout, st);
        return;
    }
    if (T.W.rows && !T.pu) {   // level-merged form: sweep on W b (the push sweep folds W in)
        spmv(c, T.W, b, T.wb.p, nullptr, 1.0, st);
        b = T.wb.p;
    }
    if (T.dense.n) {
        CK(launch_pdl(k_tri_gemv, dim3(grid_for((int64_t)T.n * 32, 256, c->sms, 8)), dim3(256), 0, st, T.n,
                      (int)T.backward, (const double *)T.dense.p, b, x, xadd, xout));
        launched(c);
        return;
    }
    if (T.bd) {
        trsv_bd(c, T, b, x, xadd, xout, st);
        return;
    }
    if (T.gbd) {
        trsv_gbd(c, T, b, x, xadd, xout, st);
        return;
    }
    if (T.bl) {
        trsv_block(c, T, b, x, xadd, xout, st);
        return;
    }
    if (T.pu) {
        trsv_push(c, T, b, x, xadd, xout, st);
        return;
    }
    if (T.cl) {
        trsv_cluster(c, T, b, x, xadd, xout, st);
        return;
    }
    CK(cudaMemsetAsync(x, 0xFF, sizeof(double) * T.n, st));
    CK(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    const int warps = std::min<int64_t>(T.n, (int64_t)c->sms * 32);
    const int grid = (warps + 3) / 4;
    k_trsv<<<grid, 128, 0, st>>>(T.n, T.order.p, T.strict.ptr.p, T.strict.idx.p, T.strict.val.p,
                                 T.diag.n ? T.diag.p : nullptr, b, x, ticket, xadd, xout);
    launched(c);
}

// ------------------------------------------------------------------ level merging
// Exact-arithmetic rewrite of a level-scheduled sweep: consecutive
// dependency levels are grouped m at a time.  With T = D + L_in + L_out (L_in: entries
// inside a group, L_out: entries on earlier groups) and N = D^-1 L_in (nilpotent,
// N^m = 0 inside a group),
//     x = T^-1 b  <=>  x = W b - Z x,   W = (I + N)^-1 D^-1,   Z = (I + N)^-1 D^-1 L_out,
// with (I + N)^-1 = sum_{k<m} (-N)^k evaluated by Horner (Z <- Z0 - N Z).  Z only
// references earlier groups, so the sweep has at most ceil(levels / m) dependent
// steps at the price of a wider Z; W b is one parallel SpMV ahead of the sweep.
// Results differ from the sequential substitution by rounding only.
__global__ void k_group_count(int n, const int *__restrict__ ptr, const int *__restrict__ idx,
                              const int *__restrict__ lev, int m, int same, int *cnt) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const int g = lev[r] / m;
        int k = 0;
        for (int p = ptr[r]; p < ptr[r + 1]; ++p) k += ((lev[idx[p]] / m) == g) == (same != 0);
        cnt[r] = k;
    }
}
__global__ void k_group_fill(int n, const int *__restrict__ ptr, const int *__restrict__ idx,
                             const double *__restrict__ val, const int *__restrict__ lev, int m, int same,
                             const double *__restrict__ dinv, const int *__restrict__ optr, int *oidx,
                             double *oval) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const int g = lev[r] / m;
        const double s = dinv ? dinv[r] : 1.0;
        int w = optr[r];
        for (int p = ptr[r]; p < ptr[r + 1]; ++p)
            if (((lev[idx[p]] / m) == g) == (same != 0)) { oidx[w] = idx[p]; oval[w] = val[p] * s; ++w; }
    }
}
__global__ void k_diag_csr(int n, const double *__restrict__ d, int *ptr, int *idx, double *val) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r <= n; r += gridDim.x * blockDim.x) {
        ptr[r] = r;
        if (r < n) { idx[r] = r; val[r] = d ? 1.0 / d[r] : 1.0; }
    }
}

static Csr group_part(Ctx *c, const Csr &S, const int *lev, int m, bool same, const double *dinv) {
    const int n = S.rows;
    DBuf<int> cnt(n, c->s);
    k_group_count<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, S.ptr.p, S.idx.p, lev, m, same, cnt.p);
    launched(c);
    Csr B;
    B.rows = n;
    B.cols = S.cols;
    B.nnz = counts_to_ptr(c, cnt.p, n, B.ptr);
    B.idx.alloc(B.nnz, c->s);
    B.val.alloc(B.nnz, c->s);
    k_group_fill<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, S.ptr.p, S.idx.p, S.val.p, lev, m, same, dinv,
                                                             B.ptr.p, B.idx.p, B.val.p);
    launched(c);
    return B;
}

__global__ void k_recip_tri(int n, const double *d, double *o) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) o[r] = 1.0 / d[r];
}

static int merge_levels(Ctx *c, Tri &T, DBuf<int> &lev, int m) {
    const int n = T.n;
    DBuf<double> dinv;
    if (T.diag.n) {
        dinv.alloc(n, c->s);
        k_recip_tri<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, T.diag.p, dinv.p);
        launched(c);
    }
    const double *di = T.diag.n ? dinv.p : nullptr;
    Csr N = group_part(c, T.strict, lev.p, m, true, di);     // D^-1 L_in
    Csr Z0 = group_part(c, T.strict, lev.p, m, false, di);   // D^-1 L_out
    Csr W0;
    W0.alloc(n, n, n, c->s);
    k_diag_csr<<<grid_for(n + 1, 256, c->sms), 256, 0, c->s>>>(n, T.diag.n ? T.diag.p : nullptr, W0.ptr.p, W0.idx.p,
                                                               W0.val.p);
    launched(c);
    Csr Z = csr_copy(c, Z0), W = csr_copy(c, W0);
    if (N.nnz)
        for (int k = 1; k < m; ++k) {
            Z = spgemm(c, N, Z, nullptr, false, &Z0);
            W = spgemm(c, N, W, nullptr, false, &W0);
        }
    T.nnz_alg = T.strict.nnz;
    T.strict = std::move(Z);
    T.diag.release();
    T.W = std::move(W);
    spmv_plan(c, T.W);
    T.wb.alloc(n, c->s);
    return tri_levels(c, T.strict, T.backward, T.order, nullptr, &lev);
}

// ------------------------------------------------------------------ Kronecker triangles
// The velocity blocks of the VMS formulations are c M (x) I_dim with interleaved
// components (assembly.py:339); ILU(0) keeps the cross-component entries exactly zero,
// so each factor (zero-free) is T_s (x) I_dim with the same values in every component.
// Such a triangle is swept as dim independent copies of T_s -- one cluster each, one
// schedule, identical arithmetic per component.
__global__ void k_kron_check(int n, int d, const int *__restrict__ ptr, const int *__restrict__ idx,
                             const double *__restrict__ val, const double *__restrict__ diag, int *bad) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const int c = r % d, r0 = r - c;
        bool ok = true;
        if (c == 0) {
            for (int p = ptr[r]; p < ptr[r + 1]; ++p) ok &= idx[p] % d == 0;
        } else {
            const int a = ptr[r], a0 = ptr[r0], len = ptr[r + 1] - a;
            ok = len == ptr[r0 + 1] - a0;
            for (int k = 0; ok && k < len; ++k)
                ok = idx[a + k] == idx[a0 + k] + c && __double_as_longlong(val[a + k]) == __double_as_longlong(val[a0 + k]);
            if (diag) ok &= __double_as_longlong(diag[r]) == __double_as_longlong(diag[r0]);
        }
        if (!ok) atomicAdd(bad, 1);
    }
}
__global__ void k_kron_count(int ns, int d, const int *ptr, int *cnt) {
    for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < ns; a += gridDim.x * blockDim.x)
        cnt[a] = ptr[a * d + 1] - ptr[a * d];
}
__global__ void k_kron_fill(int ns, int d, const int *ptr, const int *idx, const double *val, const double *diag,
                            const int *optr, int *oidx, double *oval, double *odiag) {
    for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < ns; a += gridDim.x * blockDim.x) {
        int w = optr[a];
        for (int p = ptr[a * d]; p < ptr[a * d + 1]; ++p, ++w) { oidx[w] = idx[p] / d; oval[w] = val[p]; }
        if (diag) odiag[a] = diag[a * d];
    }
}
// largest d in {3, 2} with T = T_s (x) I_d, else 1
static int kron_detect(Ctx *c, const Tri &T) {
    for (int d = 3; d >= 2; --d) {
        if (T.n % d) continue;
        DBuf<int> bad(1, c->s);
        CK(cudaMemsetAsync(bad.p, 0, sizeof(int), c->s));
        k_kron_check<<<grid_for(T.n, 256, c->sms), 256, 0, c->s>>>(T.n, d, T.strict.ptr.p, T.strict.idx.p,
                                                                  T.strict.val.p, T.diag.n ? T.diag.p : nullptr, bad.p);
        launched(c);
        if (bad.to_host()[0] == 0) return d;
    }
    return 1;
}
static Tri kron_scalar(Ctx *c, const Tri &T, int d) {
    Tri S;
    const int ns = T.n / d;
    S.n = ns;
    S.backward = T.backward;
    DBuf<int> cnt(ns, c->s);
    k_kron_count<<<grid_for(ns, 256, c->sms), 256, 0, c->s>>>(ns, d, T.strict.ptr.p, cnt.p);
    launched(c);
    S.strict.rows = S.strict.cols = ns;
    S.strict.nnz = counts_to_ptr(c, cnt.p, ns, S.strict.ptr);
    S.strict.idx.alloc(S.strict.nnz, c->s);
    S.strict.val.alloc(S.strict.nnz, c->s);
    if (T.diag.n) S.diag.alloc(ns, c->s);
    k_kron_fill<<<grid_for(ns, 256, c->sms), 256, 0, c->s>>>(ns, d, T.strict.ptr.p, T.strict.idx.p, T.strict.val.p,
                                                            T.diag.n ? T.diag.p : nullptr, S.strict.ptr.p,
                                                            S.strict.idx.p, S.strict.val.p, S.diag.p);
    launched(c);
    return S;
}

static int merge_factor() {
    static const int m = [] { const char *e = std::getenv("DPP_MERGE"); return e ? std::atoi(e) : 1; }();
    return m;
}

Tri make_tri(Ctx *c, const Csr &A, bool lower, bool unit, bool allow_dense, DBuf<int> *pre_order,
             DBuf<int> *pre_lev, int pre_nlev) {
    // non-parity fast mode: Jacobi sweeps (small dense coarse levels stay exact)
    if (c->tri_jacobi > 0 && !(allow_dense && A.rows <= DENSE_TRI_MAX))
        return make_tri_jacobi(c, A, lower, unit, 1, c->tri_jacobi);
    Tri T;
    T.n = A.rows;
    T.backward = !lower;
    {
        DPP_TRACE_SCOPE(c, "tri.strict_part");
        T.strict = csr_part(c, A, lower ? -1 : 1, true);
    }
    if (!unit) {
        T.diag.alloc(A.rows, c->s);
        csr_diag(c, A, T.diag.p, nullptr);
    }
    if (allow_dense && T.n <= DENSE_TRI_MAX) {
        // exact-arithmetic rewrite for small, deep coarse levels: x = T^-1 b as a GEMV
        const int n = T.n;
        DPP_TRACE_SCOPE(c, "tri.dense_inverse");
        tri_dense_inverse(c, T);
        CK(cudaStreamSynchronize(c->s));
        T.nlev = n;
        return T;
    }
    // AMG smoother factors above the dense limit and up to DPP_BD_MAX rows: block-dense
    // sweep (no level analysis).  Measured on C2: the 5593-row level goes from 264 us
    // (block-sequential) to ~35 us per sweep; on the 68921-row level it only ties the
    // cluster sweep (468 us), so larger factors stay level-scheduled.
    static const int bd_max = [] { const char *e = std::getenv("DPP_BD_MAX"); return e ? std::atoi(e) : 8192; }();
    static const int bd_b = [] { const char *e = std::getenv("DPP_BD_B"); return e ? std::atoi(e) : 512; }();
    if (allow_dense && T.n <= bd_max && bd_plan(c, T, std::min(bd_b, 1024))) {
        T.nlev = T.bd->nb;
        return T;
    }
    // long-row smoother factors beyond that (deep coarse levels of configs 3/4: hundreds of entries
    // per row, thousands of levels): the block recurrence with two device-wide launches per block
    static const int gbd_max = [] { const char *e = std::getenv("DPP_GBD_MAX"); return e ? std::atoi(e) : 65536; }();
    static const int gbd_row = [] { const char *e = std::getenv("DPP_GBD_ROW"); return e ? std::atoi(e) : 128; }();
    if (allow_dense && T.n <= gbd_max && (double)T.strict.nnz >= (double)gbd_row * T.n && gbd_plan(c, T, 512)) {
        T.nlev = T.gbd->nb;
        return T;
    }
    static const bool kron_on = [] { const char *e = std::getenv("DPP_KRON"); return !(e && *e == '0'); }();
    if (kron_on && !pre_lev && T.n > 2 * 8192) {
        const int d = kron_detect(c, T);
        if (d > 1) {
            Tri S = kron_scalar(c, T, d);
            DBuf<int> slev;
            S.nlev = tri_levels(c, S.strict, S.backward, S.order, nullptr, &slev);
            const int before = S.nlev;
            const int m = merge_factor();
            if (m > 1 && S.nlev >= 4 * m) S.nlev = merge_levels(c, S, slev, m);
            if (push_plan(c, S, slev, S.nlev)) {
                if (TraceScope::on())
                    std::fprintf(stderr, "[dpp-trace]   make_tri kron d=%d n=%d levels %d -> %d strict nnz %lld (x%d)\n", d,
                                 S.n, before, S.nlev, (long long)S.strict.nnz, d);
                S.ncomp = d;
                S.n = T.n;
                S.nnz_alg = T.strict.nnz;
                return S;
            }
        }
    }
    DBuf<int> lev;
    if (pre_lev) {   // the caller's analysis covers every dependency of this triangle
        T.order = std::move(*pre_order);
        lev = std::move(*pre_lev);
        T.nlev = pre_nlev;
    } else {
        T.nlev = tri_levels(c, T.strict, T.backward, T.order, nullptr, &lev);
    }
    // wide, deep triangles (ILU factors, AMG level 0): merge levels m at a time
    const int merge = merge_factor();
    if (merge > 1 && T.n > 8192 && T.nlev >= 4 * merge) {
        const int before = T.nlev;
        T.nlev = merge_levels(c, T, lev, merge);
        if (TraceScope::on())
            std::fprintf(stderr, "[dpp-trace]   merge_levels m=%d levels %d -> %d, strict nnz %lld -> %lld, W nnz %lld\n",
                         merge, before, T.nlev, (long long)T.nnz_alg, (long long)T.strict.nnz, (long long)T.W.nnz);
    }
    // narrow, deep levels (coarse AMG): block-sequential sweep with dense block inverses
    static const bool no_block = [] { const char *e = std::getenv("DPP_NO_BLOCK"); return e && *e == '1'; }();
    if (TraceScope::on())
        std::fprintf(stderr, "[dpp-trace]   make_tri n=%d nnz=%lld levels=%d backward=%d\n", T.n,
                     (long long)T.strict.nnz, T.nlev, (int)T.backward);
    if (!no_block && T.n <= 8192 && (int64_t)T.nlev * 64 > T.n && block_plan(c, T)) return T;
    static const bool no_cluster = [] { const char *e = std::getenv("DPP_NO_CLUSTER"); return e && *e == '1'; }();
    static const bool no_push = [] { const char *e = std::getenv("DPP_NO_PUSH"); return e && *e == '1'; }();
    if (!no_cluster && !(!no_push && push_plan(c, T, lev, T.nlev))) cluster_plan(c, T, lev, T.nlev);
    return T;
}

// ------------------------------------------------------------------ ILU(0)
__global__ void k_diag_pos(int n, const int *ptr, const int *idx, int *dpos, int *missing) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        int d = -1;
        for (int p = ptr[r]; p < ptr[r + 1]; ++p)
            if (idx[p] == r) d = p;
        dpos[r] = d;
        if (d < 0) atomicAdd(missing, 1);
    }
}

constexpr int ILU_CAP = 256;
constexpr int ILU_WPB = 4;

__global__ void __launch_bounds__(32 * ILU_WPB) k_ilu0(int n, const int *__restrict__ ptr,
                                                       const int *__restrict__ idx, double *val,
                                                       const int *__restrict__ dpos, int *done,
                                                       int *ticket, int *err_row,
                                                       const int *__restrict__ order) {
    __shared__ double sv[ILU_WPB][ILU_CAP];
    __shared__ int sc[ILU_WPB][ILU_CAP];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    while (true) {
        int i = 0;
        if (lane == 0) i = atomicAdd(ticket, 1);
        i = __shfl_sync(0xffffffffu, i, 0);
        if (i >= n) return;
        i = order[i];
        const int s = ptr[i], e = ptr[i + 1], len = e - s;
        const bool big = len > ILU_CAP;
        double *v = big ? val + s : sv[w];
        const int *cols = big ? idx + s : sc[w];
        if (!big) {
            for (int q = lane; q < len; q += 32) { sv[w][q] = val[s + q]; sc[w][q] = idx[s + q]; }
        }
        __syncwarp();
        for (int q = 0; q < len; ++q) {
            const int k = cols[q];
            if (k >= i) break;
            DPP_DCHECK(k >= 0);
            const double a = v[q];
            if (a == 0.0) continue;   // l_ik = 0: no update, no dependency (exact)
            long long spins = 0;
            while (ld_acquire(done + k) == 0)
                if (++spins > SPIN_LIMIT) __trap();
            const int dk = dpos[k];
            DPP_DCHECK(dk >= ptr[k] && dk < ptr[k + 1] && idx[dk] == k);   // k's diagonal, k already factored
            const double piv = __ldcg(val + dk);
            if (piv == 0.0) {
                if (lane == 0) atomicMin(err_row, k);
                continue;
            }
            const double l = __ddiv_rn(a, piv);
            __syncwarp();
            if (lane == 0) v[q] = l;
            const int ke = ptr[k + 1];
            for (int p2 = dk + 1 + lane; p2 < ke; p2 += 32) {
                const int j = idx[p2];
                int lo = q + 1, hi = len - 1;   // binary search j in cols[q+1..len)
                while (lo <= hi) {
                    const int mid = (lo + hi) >> 1;
                    const int cm = cols[mid];
                    if (cm == j) { lo = mid; break; }
                    if (cm < j) lo = mid + 1; else hi = mid - 1;
                }
                if (lo < len && cols[lo] == j) v[lo] = __dsub_rn(v[lo], __dmul_rn(l, __ldcg(val + p2)));
            }
            __syncwarp();
        }
        const int dq = dpos[i] - s;
        if (v[dq] == 0.0 && lane == 0) atomicMin(err_row, i);
        if (!big)
            for (int q = lane; q < len; q += 32) val[s + q] = sv[w][q];
        __syncwarp();
        __threadfence();
        if (lane == 0) st_release(done + i, 1);
    }
}

// In-place ILU(0) of LU (IKJ order, linalg.py:178-222); returns the failing row or -1.
static int ilu_factor(Ctx *c, Csr &LU, DBuf<int> *order_out = nullptr, DBuf<int> *lev_out = nullptr,
                      int *nlev_out = nullptr) {
    const int n = LU.rows;
    DBuf<int> dpos(n, c->s), flags((size_t)n + 3, c->s);
    CK(cudaMemsetAsync(flags.p, 0, sizeof(int) * (n + 3), c->s));
    int *missing = flags.p + n, *ticket = flags.p + n + 1, *err = flags.p + n + 2;
    CK(cudaMemsetAsync(err, 0x7f, sizeof(int), c->s));
    if (n) {
        k_diag_pos<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, LU.ptr.p, LU.idx.p, dpos.p, missing);
        launched(c);
    }
    int hm = 0;
    CK(cudaMemcpyAsync(&hm, missing, sizeof(int), cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    if (hm) DPP_FAIL(DPP_ERR_ZERO_PIVOT, "missing diagonal entry in sparsity pattern");
    DBuf<int> order, lev;
    int nlev;
    {
        Csr lower = csr_part(c, LU, -1, false);   // stored pattern: every row the IKJ loop may read
        nlev = tri_levels(c, lower, false, order, nullptr, &lev);
    }
    DPP_TRACE_SCOPE(c, "ilu0.factor_kernel");
    if (n) {
        const int warps = std::min<int64_t>(n, (int64_t)c->sms * 8);
        k_ilu0<<<(warps + ILU_WPB - 1) / ILU_WPB, 32 * ILU_WPB, 0, c->s>>>(
            n, LU.ptr.p, LU.idx.p, LU.val.p, dpos.p, flags.p, ticket, err, order.p);
        launched(c);
    }
    int he = 0;
    CK(cudaMemcpyAsync(&he, err, sizeof(int), cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    if (order_out) {   // the stored lower pattern's schedule covers the factor's L sweep
        *order_out = std::move(order);
        *lev_out = std::move(lev);
        *nlev_out = nlev;
    }
    return he != 0x7f7f7f7f ? he : -1;
}

// Sweep of the Kronecker triangle T_s (x) I_d built from the scalar factor directly
// (ilu0's Kronecker path); ok = false when the push plan does not fit
static Tri make_tri_kron(Ctx *c, const Csr &M, bool lower, bool unit, int d, DBuf<int> *pre_order,
                         DBuf<int> *pre_lev, int pre_nlev, bool &ok) {
    Tri S;
    S.n = M.rows;
    S.backward = !lower;
    S.strict = csr_part(c, M, lower ? -1 : 1, true);
    if (!unit) {
        S.diag.alloc(M.rows, c->s);
        csr_diag(c, M, S.diag.p, nullptr);
    }
    DBuf<int> lev;
    if (pre_lev) {
        S.order = std::move(*pre_order);
        lev = std::move(*pre_lev);
        S.nlev = pre_nlev;
    } else {
        S.nlev = tri_levels(c, S.strict, S.backward, S.order, nullptr, &lev);
    }
    const int64_t snnz = S.strict.nnz;
    const int m = merge_factor();
    if (m > 1 && S.nlev >= 4 * m) S.nlev = merge_levels(c, S, lev, m);
    ok = push_plan(c, S, lev, S.nlev);
    if (!ok) return Tri{};
    S.ncomp = d;
    S.n = M.rows * d;
    S.nnz_alg = snnz * d;
    if (TraceScope::on())
        std::fprintf(stderr, "[dpp-trace]   make_tri_kron d=%d n=%d levels %d strict nnz %lld (x%d)\n", d, M.rows,
                     S.nlev, (long long)S.strict.nnz, d);
    return S;
}

// Kronecker ILU(0): when A = M (x) I_d on the node-blocked pattern (every cross-component
// entry stored as +0, assembly.py:339), the IKJ loop never updates across components
// (l_ik = 0 is skipped, a_kj = 0 leaves a_ij unchanged and +0), so the factor is the
// ILU(0) of M in every component and +0 on every cross entry: bitwise the full
// factorization at 1/d the rows and 1/d^2 the entries.
__device__ __forceinline__ int row_find(const int *idx, int a, int e, int j) {
    while (a < e) {
        const int m = (a + e) >> 1;
        if (idx[m] < j) a = m + 1; else e = m;
    }
    return a;
}
__global__ void k_ilu_kron_check(int n, int d, const int *__restrict__ ptr, const int *__restrict__ idx,
                                 const double *__restrict__ val, const int *__restrict__ mp, const int *__restrict__ mi,
                                 const double *__restrict__ mv, int *bad) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const int a = r / d, c = r % d, m0 = mp[a], m1 = mp[a + 1];
        int same = 0;
        bool ok = true;
        for (int p = ptr[r]; ok && p < ptr[r + 1]; ++p) {
            const int j = idx[p];
            if (j % d == c) {
                const int q = row_find(mi, m0, m1, j / d);
                ok = q < m1 && mi[q] == j / d && __double_as_longlong(mv[q]) == __double_as_longlong(val[p]);
                ++same;
            } else {
                ok = __double_as_longlong(val[p]) == 0;
            }
        }
        if (!ok || same != m1 - m0) atomicAdd(bad, 1);
    }
}
__global__ void k_ilu_kron_expand(int n, int d, const int *__restrict__ ptr, const int *__restrict__ idx,
                                  const int *__restrict__ mp, const int *__restrict__ mi, const double *__restrict__ mv,
                                  double *val) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const int a = r / d, c = r % d;
        for (int p = ptr[r]; p < ptr[r + 1]; ++p) {
            const int j = idx[p];
            val[p] = j % d == c ? mv[row_find(mi, mp[a], mp[a + 1], j / d)] : 0.0;
        }
    }
}
__global__ void k_comp0_count(int ns, int d, const int *ptr, const int *idx, int *cnt) {
    for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < ns; a += gridDim.x * blockDim.x) {
        int k = 0;
        for (int p = ptr[a * d]; p < ptr[a * d + 1]; ++p) k += idx[p] % d == 0;
        cnt[a] = k;
    }
}
__global__ void k_comp0_fill(int ns, int d, const int *ptr, const int *idx, const double *val, const int *optr,
                             int *oidx, double *oval) {
    for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < ns; a += gridDim.x * blockDim.x) {
        int w = optr[a];
        for (int p = ptr[a * d]; p < ptr[a * d + 1]; ++p)
            if (idx[p] % d == 0) { oidx[w] = idx[p] / d; oval[w] = val[p]; ++w; }
    }
}
// M from the component-0 rows / columns of A, if A = M (x) I_d (else M.rows = 0)
static Csr kron_block(Ctx *c, const Csr &A) {
    Csr M;
    static const bool on = [] { const char *e = std::getenv("DPP_KRON"); return !(e && *e == '0'); }();
    if (!on || A.rows < 2 * 8192) return M;
    for (int d = 3; d >= 2; --d) {
        if (A.rows % d) continue;
        const int ns = A.rows / d;
        DBuf<int> cnt(ns, c->s);
        k_comp0_count<<<grid_for(ns, 256, c->sms), 256, 0, c->s>>>(ns, d, A.ptr.p, A.idx.p, cnt.p);
        launched(c);
        Csr B;
        B.rows = B.cols = ns;
        B.nnz = counts_to_ptr(c, cnt.p, ns, B.ptr);
        B.idx.alloc(B.nnz, c->s);
        B.val.alloc(B.nnz, c->s);
        k_comp0_fill<<<grid_for(ns, 256, c->sms), 256, 0, c->s>>>(ns, d, A.ptr.p, A.idx.p, A.val.p, B.ptr.p, B.idx.p,
                                                                 B.val.p);
        launched(c);
        DBuf<int> bad(1, c->s);
        CK(cudaMemsetAsync(bad.p, 0, sizeof(int), c->s));
        k_ilu_kron_check<<<grid_for(A.rows, 256, c->sms), 256, 0, c->s>>>(A.rows, d, A.ptr.p, A.idx.p, A.val.p,
                                                                          B.ptr.p, B.idx.p, B.val.p, bad.p);
        launched(c);
        if (bad.to_host()[0] == 0) return B;
    }
    return M;
}

std::unique_ptr<Ilu> ilu0(Ctx *c, const Csr &A) {
    DPP_TRACE_SCOPE(c, "ilu0.total");
    if (A.rows != A.cols) DPP_FAIL(DPP_ERR_VALUE, "ilu0 requires a square matrix");
    auto f = std::make_unique<Ilu>();
    f->ctx = c;
    f->n = A.rows;
    f->LU = csr_copy(c, A);
    const int n = A.rows;
    Csr M = kron_block(c, A);
    if (M.rows) {
        const int d = n / M.rows;
        {   // a missing diagonal in any component is one in component 0 (same pattern)
            DBuf<int> dpos(n, c->s), missing(1, c->s);
            CK(cudaMemsetAsync(missing.p, 0, sizeof(int), c->s));
            k_diag_pos<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, A.ptr.p, A.idx.p, dpos.p, missing.p);
            launched(c);
            if (missing.to_host()[0]) DPP_FAIL(DPP_ERR_ZERO_PIVOT, "missing diagonal entry in sparsity pattern");
        }
        DBuf<int> order, lev;
        int nlev = 0;
        const int bad = ilu_factor(c, M, &order, &lev, &nlev);
        if (bad >= 0) DPP_FAIL(DPP_ERR_ZERO_PIVOT, "zero pivot at row " + std::to_string(bad * d));
        k_ilu_kron_expand<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, d, A.ptr.p, A.idx.p, M.ptr.p, M.idx.p,
                                                                      M.val.p, f->LU.val.p);
        launched(c);
        if (c->tri_jacobi > 0) {
            f->L = make_tri_jacobi(c, M, true, true, d, c->tri_jacobi);
            f->U = make_tri_jacobi(c, M, false, false, d, c->tri_jacobi);
            f->y.alloc(n, c->s);
            f->tmp.alloc(n, c->s);
            f->ticket.alloc(2, c->s);
            return f;
        }
        bool okl = false, oku = false;
        f->L = make_tri_kron(c, M, true, true, d, &order, &lev, nlev, okl);
        if (okl) f->U = make_tri_kron(c, M, false, false, d, nullptr, nullptr, 0, oku);
        if (okl && oku) {
            f->y.alloc(n, c->s);
            f->tmp.alloc(n, c->s);
            f->ticket.alloc(2, c->s);
            return f;
        }
    } else {
        const int bad = ilu_factor(c, f->LU);
        if (bad >= 0) DPP_FAIL(DPP_ERR_ZERO_PIVOT, "zero pivot at row " + std::to_string(bad));
    }
    // (the factorization's levels follow the STORED pattern, explicit zeros included:
    // 363 levels on C2 against 121 for L's zero-free pattern, so L gets its own analysis)
    f->L = make_tri(c, f->LU, true, true);
    f->U = make_tri(c, f->LU, false, false);
    f->y.alloc(n, c->s);
    f->tmp.alloc(n, c->s);
    f->ticket.alloc(2, c->s);
    return f;
}

void ilu_apply(Ctx *c, Ilu &f, const double *r, double *z, cudaStream_t st) {
    trsv(c, f.L, r, f.y.p, f.ticket.p, nullptr, nullptr, st);
    trsv(c, f.U, f.y.p, z, f.ticket.p + 1, nullptr, nullptr, st);
}

}  // namespace dpp
