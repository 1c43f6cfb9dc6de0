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
#include "dpp_internal.cuh"

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
__device__ __forceinline__ void st_release(int *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ------------------------------------------------------------------ TRSV
__global__ void __launch_bounds__(128) k_trsv(int n, int backward, const int *__restrict__ ptr,
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
        const int row = backward ? n - 1 - t : t;
        const int s = ptr[row], e = ptr[row + 1];
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
            double xi = b[row] - sum;
            if (diag) xi = xi / diag[row];
            if (__double_as_longlong(xi) == (long long)SENT) xi = __longlong_as_double(0x7ff8000000000000ll);
            st_relaxed(x + row, xi);
            if (xout) xout[row] = xadd[row] + xi;
        }
    }
}

void trsv(Ctx *c, const Tri &T, const double *b, double *x, int *ticket, const double *xadd,
          double *xout, cudaStream_t st) {
    st = st ? st : c->s;
    if (T.n == 0) return;
    CK(cudaMemsetAsync(x, 0xFF, sizeof(double) * T.n, st));
    CK(cudaMemsetAsync(ticket, 0, sizeof(int), st));
    const int warps = std::min<int64_t>(T.n, (int64_t)c->sms * 32);
    const int grid = (warps + 3) / 4;
    k_trsv<<<grid, 128, 0, st>>>(T.n, T.backward, T.strict.ptr.p, T.strict.idx.p, T.strict.val.p,
                                 T.diag.n ? T.diag.p : nullptr, b, x, ticket, xadd, xout);
    launched(c);
}

Tri make_tri(Ctx *c, const Csr &A, bool lower, bool unit) {
    Tri T;
    T.n = A.rows;
    T.backward = !lower;
    T.strict = csr_part(c, A, lower ? -1 : 1, true);
    if (!unit) {
        T.diag.alloc(A.rows, c->s);
        csr_diag(c, A, T.diag.p, nullptr);
    }
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
                                                       int *ticket, int *err_row) {
    __shared__ double sv[ILU_WPB][ILU_CAP];
    __shared__ int sc[ILU_WPB][ILU_CAP];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    while (true) {
        int i = 0;
        if (lane == 0) i = atomicAdd(ticket, 1);
        i = __shfl_sync(0xffffffffu, i, 0);
        if (i >= n) return;
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
            const double a = v[q];
            if (a == 0.0) continue;   // l_ik = 0: no update, no dependency (exact)
            long long spins = 0;
            while (ld_acquire(done + k) == 0)
                if (++spins > SPIN_LIMIT) __trap();
            const int dk = dpos[k];
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

std::unique_ptr<Ilu> ilu0(Ctx *c, const Csr &A) {
    if (A.rows != A.cols) DPP_FAIL(DPP_ERR_VALUE, "ilu0 requires a square matrix");
    auto f = std::make_unique<Ilu>();
    f->ctx = c;
    f->n = A.rows;
    f->LU = csr_copy(c, A);
    const int n = A.rows;
    DBuf<int> dpos(n, c->s), flags((size_t)n + 3, c->s);
    CK(cudaMemsetAsync(flags.p, 0, sizeof(int) * (n + 3), c->s));
    int *missing = flags.p + n, *ticket = flags.p + n + 1, *err = flags.p + n + 2;
    CK(cudaMemsetAsync(err, 0x7f, sizeof(int), c->s));
    if (n) {
        k_diag_pos<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, A.ptr.p, A.idx.p, dpos.p, missing);
        launched(c);
    }
    int hm = 0;
    CK(cudaMemcpyAsync(&hm, missing, sizeof(int), cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    if (hm) DPP_FAIL(DPP_ERR_ZERO_PIVOT, "missing diagonal entry in sparsity pattern");
    if (n) {
        const int warps = std::min<int64_t>(n, (int64_t)c->sms * 16);
        k_ilu0<<<(warps + ILU_WPB - 1) / ILU_WPB, 32 * ILU_WPB, 0, c->s>>>(
            n, f->LU.ptr.p, f->LU.idx.p, f->LU.val.p, dpos.p, flags.p, ticket, err);
        launched(c);
    }
    int he = 0;
    CK(cudaMemcpyAsync(&he, err, sizeof(int), cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    if (he != 0x7f7f7f7f) DPP_FAIL(DPP_ERR_ZERO_PIVOT, "zero pivot at row " + std::to_string(he));
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
