// Restarted, left-preconditioned GMRES(m) with modified Gram-Schmidt.
//
// Reference: linalg.gmres (linalg.py:65-165).  The control flow is the
// reference's, statement for statement: true-residual convergence test at
// each restart, stagnation when a cycle's true residual >= 0.9999 x the
// previous one, happy breakdown at H[j+1,j] <= 1e-14 beta, Givens rotations
// with hypot, inner exit on the preconditioned estimate |g_{j+1}| <= rtol*||Mb||,
// back substitution, final true residual.  Vectors (Krylov basis V, w, x, r)
// live in HBM; the (m+1) x m Hessenberg matrix and rotations live on the host,
// which reads one column (j+2 doubles) per Arnoldi step.
#include <chrono>
#include <cmath>

#include <cooperative_groups.h>

#include "system.cuh"

namespace cg = cooperative_groups;

namespace dpp {

// deterministic dot product: partials per block, then one ordered sum
__global__ void k_dot_partial(int64_t n, const double *x, const double *y, double *part) {
    __shared__ double sh[32];
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) s += x[i] * y[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) part[blockIdx.x] = s;
    }
}
__global__ void k_sum(int np, const double *part, double *out) {
    double s = 0.0;
    for (int i = threadIdx.x; i < np; i += 32) s += part[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *out = s;
}
// w -= h * v with h read from device memory
__global__ void k_axpy_neg_dev(int64_t n, const double *h, const double *v, double *w) {
    const double a = *h;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) w[i] -= a * v[i];
}
// One Arnoldi step's modified Gram-Schmidt in one cooperative kernel:
//   for i = 0..j: h_i = <V_i, w> ; w -= h_i V_i      then h_{j+1} = ||w||
// Bitwise the sequence k_dot_partial + k_sum + k_axpy_neg_dev (+ norm2_dev) computes:
// the same NRM_BLOCKS x 256 grid-stride partials and block reductions, every block
// forms the final 32-lane ordered sum itself, and each thread only touches its own
// elements of w between two dots, so one grid barrier per basis vector suffices
// (partials are double-buffered).
__device__ __forceinline__ double mgs_block_partial(double s, double *sh) {
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x < 32) {
        r = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
    }
    __syncthreads();
    return r;   // valid in thread 0
}
__device__ __forceinline__ double mgs_final_sum(const double *part, int np, double *sh) {
    if (threadIdx.x < 32) {
        double s = 0.0;
        for (int i = threadIdx.x; i < np; i += 32) s += __ldcg(part + i);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) sh[0] = s;
    }
    __syncthreads();
    const double s = sh[0];
    __syncthreads();
    return s;
}
__global__ void __launch_bounds__(256) k_mgs(int64_t n, int j, const double *V, double *w, double *hcol,
                                            double *part0, double *part1) {
    __shared__ double sh[32];
    cg::grid_group grid = cg::this_grid();
    const int64_t g0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
    for (int i = 0; i <= j + 1; ++i) {
        double *part = (i & 1) ? part1 : part0;
        const double *Vi = V + (size_t)i * n;
        double s = 0.0;
        if (i <= j)
            for (int64_t k = g0; k < n; k += gs) s += Vi[k] * w[k];
        else
            for (int64_t k = g0; k < n; k += gs) s += w[k] * w[k];
        const double bp = mgs_block_partial(s, sh);
        if (threadIdx.x == 0) part[blockIdx.x] = bp;
        grid.sync();
        const double h = mgs_final_sum(part, gridDim.x, sh);
        if (i <= j) {
            if (blockIdx.x == 0 && threadIdx.x == 0) hcol[i] = h;
            for (int64_t k = g0; k < n; k += gs) w[k] -= h * Vi[k];
        } else if (blockIdx.x == 0 && threadIdx.x == 0) {
            hcol[j + 1] = sqrt(h);
        }
    }
}

// x = x + V[:k]^T y
__global__ void k_update_x(int64_t n, int k, const double *V, const double *y, double *x) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int t = 0; t < k; ++t) s += V[(int64_t)t * n + i] * y[t];
        x[i] = x[i] + s;
    }
}

namespace {
struct Gm {
    Ctx *c;
    int64_t n;
    const Operator &A;
    const PcOp &M;
    std::vector<double> hin, hout;
    DBuf<double> part, part2;
    int mv = 0, pcs = 0;

    void host_apply(dpp_apply_fn cb, void *user, const double *in, double *out) {
        if (hin.empty()) { hin.resize(n); hout.resize(n); }
        CK(cudaMemcpyAsync(hin.data(), in, sizeof(double) * n, cudaMemcpyDeviceToHost, c->s));
        CK(cudaStreamSynchronize(c->s));
        cb(hin.data(), hout.data(), user);
        CK(cudaMemcpyAsync(out, hout.data(), sizeof(double) * n, cudaMemcpyHostToDevice, c->s));
    }
    // out = b - A x (b may be null => out = A x)
    void matvec(const double *x, double *out, const double *b = nullptr) {
        ++mv;
        if (A.A) { spmv(c, *A.A, x, out, b, b ? -1.0 : 1.0); return; }
        host_apply(A.cb, A.user, x, out);
        if (b) axpby_to(c, n, b, -1.0, out, out);
    }
    void pc(const double *r, double *z) {
        ++pcs;
        if (M.pc) pc_apply_dev(M.pc, r, z);
        else if (M.cb) host_apply(M.cb, M.user, r, z);
        else CK(cudaMemcpyAsync(z, r, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->s));
    }
    void dot_dev(const double *x, const double *y, double *out) {
        k_dot_partial<<<NRM_BLOCKS, 256, 0, c->s>>>(n, x, y, part.p);
        launched(c);
        k_sum<<<1, 32, 0, c->s>>>(NRM_BLOCKS, part.p, out);
        launched(c);
    }
    double fetch(const double *d) {
        double h;
        CK(cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, c->s));
        CK(cudaStreamSynchronize(c->s));
        return h;
    }
};
}  // namespace

void gmres_dev(Ctx *c, int64_t n, const Operator &A, const PcOp &M, const double *b, double *x,
               double rtol, int max_iter, int restart, dpp_krylov_stats *st,
               std::vector<double> *history, bool x_zero) {
    const auto t0 = std::chrono::steady_clock::now();
    Gm g{c, n, A, M};
    g.part.alloc(NRM_BLOCKS, c->s);
    g.part2.alloc(NRM_BLOCKS, c->s);
    *st = dpp_krylov_stats{};
    DBuf<double> sc(restart + 8, c->s), r(n, c->s), z(n, c->s), w(n, c->s), tmp(n, c->s);
    // H column read back through pinned memory + an event, so the host can wait for it alone
    PinnedBuf hbuf = pinned_acquire(sizeof(double) * (restart + 8));
    double *hpin = static_cast<double *>(hbuf.p);
    cudaEvent_t hev;
    CK(cudaEventCreateWithFlags(&hev, cudaEventDisableTiming));
    struct HRelease {
        PinnedBuf b;
        cudaEvent_t e;
        ~HRelease() { cudaEventDestroy(e); pinned_release(b); }
    } hrel{hbuf, hev};
    double *hcol = sc.p;                  // H[0..j+1, j]
    double *dnorm = sc.p + restart + 2;   // scratch scalars
    auto finish = [&](int its, double rel, bool conv, int reason) {
        st->iterations = its;
        st->relative_residual = rel;
        st->converged = conv;
        st->reason = reason;
        st->pc_applies = g.pcs;
        st->matvecs = g.mv;
        st->wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };
    norm2_dev(c, n, b, dnorm);
    const double norm_b = g.fetch(dnorm);
    if (norm_b == 0.0) {
        fill(c, x, n, 0.0);
        CK(cudaStreamSynchronize(c->s));
        finish(0, 0.0, true, 0);
        return;
    }
    g.pc(b, z.p);
    norm2_dev(c, n, z.p, dnorm);
    const double norm_mb = g.fetch(dnorm);

    const int m_max = restart;
    DBuf<double> V((size_t)(m_max + 1) * n, c->s);
    std::vector<double> H((size_t)(m_max + 1) * m_max), cs(m_max), sn(m_max), gg(m_max + 1);
    auto Hij = [&](int i, int j) -> double & { return H[(size_t)i * m_max + j]; };
    int total = 0, reason = 1, cycles = 0;
    bool converged = false;
    double last = -1.0;
    // x0 = 0 with the device CSR operator and a device (or identity) preconditioner:
    // the first cycle's r = b - A 0 is b bit for bit, so ||r|| = ||b|| and M r = M b,
    // which is already in z -- the same values the reference recomputes (linalg.py:94-108)
    bool first_is_b = x_zero && A.A && !M.cb;
    while (total < max_iter) {
        double rel, beta;
        if (first_is_b) {
            first_is_b = false;
            rel = norm_b / norm_b;
            if (rel <= rtol) { converged = true; reason = 0; break; }
            last = rel;
            beta = norm_mb;
            CK(cudaMemcpyAsync(dnorm, &norm_mb, sizeof(double), cudaMemcpyHostToDevice, c->s));
        } else {
            g.matvec(x, r.p, b);                   // r = b - A x
            norm2_dev(c, n, r.p, dnorm);
            rel = g.fetch(dnorm) / norm_b;
            if (rel <= rtol) { converged = true; reason = 0; break; }
            if (last >= 0.0 && rel >= last * 0.9999) { reason = 2; break; }
            last = rel;
            g.pc(r.p, z.p);
            norm2_dev(c, n, z.p, dnorm);
            beta = g.fetch(dnorm);
        }
        if (beta == 0.0) { converged = true; reason = 0; break; }
        ++cycles;
        const int m = std::min(restart, max_iter - total);
        std::fill(H.begin(), H.end(), 0.0);
        std::fill(cs.begin(), cs.end(), 0.0);
        std::fill(sn.begin(), sn.end(), 0.0);
        std::fill(gg.begin(), gg.end(), 0.0);
        gg[0] = beta;
        scale_by_dev(c, n, z.p, dnorm, V.p);       // V[0] = z / beta
        int k_used = 0;
        bool happy = false, ahead = false;   // ahead: V[j] and M^-1 A V[j] already enqueued
        for (int j = 0; j < m; ++j) {
            double *Vj = V.p + (size_t)j * n;
            if (!ahead) {
            DPP_TRACE_SCOPE(c, "gmres.matvec_pc");
            g.matvec(Vj, tmp.p);
            g.pc(tmp.p, w.p);                      // w = M^-1 A V[j]
            }
            ahead = false;
            DPP_TRACE_SCOPE(c, "gmres.mgs_givens");
            {   // modified Gram-Schmidt + ||w||, one cooperative kernel
                int64_t nn = n;
                int jj = j;
                const double *Vp = V.p;
                double *wp = w.p, *hp = hcol, *p0 = g.part.p, *p1 = g.part2.p;
                void *args[] = {&nn, &jj, &Vp, &wp, &hp, &p0, &p1};
                CK(cudaLaunchCooperativeKernel((const void *)k_mgs, NRM_BLOCKS, 256, args, 0, c->s));
                launched(c);
            }
            double *hc = hpin;
            CK(cudaMemcpyAsync(hc, hcol, sizeof(double) * (j + 2), cudaMemcpyDeviceToHost, c->s));
            CK(cudaEventRecord(hev, c->s));
            // while the host waits for H[:, j] and does the Givens algebra, the device already
            // forms V[j+1] = w / h_{j+1,j} and M^-1 A V[j+1] -- only when this iteration cannot
            // end the cycle (estimate far above the target, not the last column), so the
            // speculative work is always the next iteration's (a breakdown leaves it unused)
            static const bool spec_on = [] { const char *e = std::getenv("DPP_GMRES_AHEAD"); return !(e && *e == '0'); }();
            // (device operators only: a host callback would be called on a column that may be
            // thrown away, and its synchronous round trip gains no overlap)
            if (spec_on && A.A && M.pc && j + 1 < m && total + 1 < max_iter &&
                std::fabs(gg[j]) > 1e3 * rtol * norm_mb) {
                double *Vn = V.p + (size_t)(j + 1) * n;
                scale_by_dev(c, n, w.p, hcol + j + 1, Vn);
                g.matvec(Vn, tmp.p);
                g.pc(tmp.p, w.p);
                ahead = true;
            }
            CK(cudaEventSynchronize(hev));   // H[:, j] only (not the work enqueued after it)
            for (int i = 0; i <= j + 1; ++i) Hij(i, j) = hc[i];
            if (Hij(j + 1, j) > 1e-14 * beta) {
                if (!ahead) scale_by_dev(c, n, w.p, hcol + j + 1, V.p + (size_t)(j + 1) * n);
            } else {
                happy = true;
            }
            for (int i = 0; i < j; ++i) {
                const double t = cs[i] * Hij(i, j) + sn[i] * Hij(i + 1, j);
                Hij(i + 1, j) = -sn[i] * Hij(i, j) + cs[i] * Hij(i + 1, j);
                Hij(i, j) = t;
            }
            const double den = std::hypot(Hij(j, j), Hij(j + 1, j));
            if (den == 0) { cs[j] = 1.0; sn[j] = 0.0; }
            else { cs[j] = Hij(j, j) / den; sn[j] = Hij(j + 1, j) / den; }
            Hij(j, j) = cs[j] * Hij(j, j) + sn[j] * Hij(j + 1, j);
            Hij(j + 1, j) = 0.0;
            gg[j + 1] = -sn[j] * gg[j];
            gg[j] = cs[j] * gg[j];
            ++total;
            k_used = j + 1;
            if (history) history->push_back(std::fabs(gg[j + 1]) / norm_mb);
            if (happy || std::fabs(gg[j + 1]) <= rtol * norm_mb) {
                if (ahead) {   // the speculative column is discarded: it is not counted
                    --g.mv;
                    --g.pcs;
                    ahead = false;
                }
                break;
            }
        }
        // y = R^-1 g by column-oriented back substitution (LAPACK getrs on triu(R))
        std::vector<double> y(gg.begin(), gg.begin() + k_used);
        for (int j = k_used - 1; j >= 0; --j) {
            if (Hij(j, j) == 0.0) { y[j] = 0.0; continue; }   // singular: least-squares-like fallback
            y[j] /= Hij(j, j);
            for (int i = 0; i < j; ++i) y[i] -= y[j] * Hij(i, j);
        }
        DBuf<double> dy(std::max(k_used, 1), c->s);
        dy.upload(y.data(), k_used);
        k_update_x<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, k_used, V.p, dy.p, x);
        launched(c);
        if (happy) {
            g.matvec(x, r.p, b);
            norm2_dev(c, n, r.p, dnorm);
            const double rel2 = g.fetch(dnorm) / norm_b;
            if (rel2 <= rtol || rel2 < 1e-13) { converged = true; reason = 0; break; }
        }
    }
    g.matvec(x, r.p, b);
    norm2_dev(c, n, r.p, dnorm);
    const double fin = g.fetch(dnorm) / norm_b;
    if (fin <= rtol) { converged = true; reason = 0; }
    finish(total, fin, converged, reason);
    st->cycles = cycles;
}

}  // namespace dpp
