// Discrete fields on the device: evaluation at reference points of every cell and the L2 error
// against an exact field (reference assembly.py:591-644 DiscreteField.evaluate_all,
// spectrum.py:149-176 l2_error / field_errors).
//
// One thread per (cell, quadrature point): the field value from the cell's coefficients and the
// reference basis at the point -- P1 / Q1 nodal values for pressures and CG / DG velocities,
// the contravariant Piola map (J V_ref s_f c_f) / det of the RT facet-flux basis for H(div)
// velocities -- then |u_h - u|^2 w_q det_c, reduced per block and summed in a fixed order
// (deterministic).  The exact field is either a package manufactured solution evaluated on
// the device (kinds below) or values the caller computed at dpp_cell_points().
#include <cmath>

#include "abi_guard.cuh"
#include "devmesh.cuh"

namespace dpp {
namespace {

constexpr int FQ_MAX = 128;   // quadrature points per cell

struct RefPts {
    int nq = 0;
    double p[FQ_MAX][3] = {};
    double w[FQ_MAX] = {};
};

__device__ inline void cell_jacobian(int kind, int dim, int nn, const double *V, const int *cv, double J[3][3]) {
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) J[a][b] = 0.0;
    if (kind == DPP_TRI || kind == DPP_TET) {   // J[:, k] = v_{k+1} - v_0 (reference mesh.py:175-183)
        for (int k = 0; k < dim; ++k)
            for (int d = 0; d < dim; ++d) J[d][k] = V[(int64_t)cv[k + 1] * dim + d] - V[(int64_t)cv[0] * dim + d];
    } else {   // axis-aligned boxes: diag(v_last - v_0)
        for (int d = 0; d < dim; ++d) J[d][d] = V[(int64_t)cv[nn - 1] * dim + d] - V[(int64_t)cv[0] * dim + d];
    }
}

// reference scalar basis (elements.py eval_basis P1 / Q1)
__device__ inline void scalar_basis(int kind, int dim, const double *x, double *N) {
    if (kind == DPP_TRI || kind == DPP_TET) {
        double s = 0.0;
        for (int d = 0; d < dim; ++d) s += x[d];
        N[0] = 1.0 - s;
        for (int d = 0; d < dim; ++d) N[1 + d] = x[d];
        return;
    }
    const int nd = 1 << dim;
    for (int a = 0; a < nd; ++a) {
        double v = 1.0;
        for (int axis = 0; axis < dim; ++axis) v *= ((a >> axis) & 1) ? x[axis] : 1.0 - x[axis];
        N[a] = v;
    }
}

// reference RT facet-flux basis, facet order of LOCAL_FACETS (elements.py eval_basis RT_*)
__device__ inline void rt_basis(int kind, int dim, const double *x, double Vr[6][3]) {
    if (kind == DPP_TRI) {
        const double opp[3][2] = {{0.0, 1.0}, {1.0, 0.0}, {0.0, 0.0}};
        for (int f = 0; f < 3; ++f)
            for (int d = 0; d < 2; ++d) Vr[f][d] = x[d] - opp[f][d];
    } else if (kind == DPP_TET) {
        const double opp[4][3] = {{0, 0, 1}, {0, 1, 0}, {1, 0, 0}, {0, 0, 0}};
        for (int f = 0; f < 4; ++f)
            for (int d = 0; d < 3; ++d) Vr[f][d] = 2.0 * (x[d] - opp[f][d]);
    } else {
        for (int f = 0; f < 2 * dim; ++f)
            for (int d = 0; d < dim; ++d) Vr[f][d] = 0.0;
        for (int axis = 0; axis < dim; ++axis) {
            Vr[2 * axis][axis] = x[axis] - 1.0;
            Vr[2 * axis + 1][axis] = x[axis];
        }
    }
}

// package manufactured solutions (problem.py mms_2d / mms_3d): kinds 1 / 2 pressures
// a X S + c E; kinds 3 / 4 velocities -k [X S_x, X cos(pi y) + c e^{e y}, (X cos(pi z) + c e^{e z})]
__device__ inline void mms_value(int kind, const double *cf, const double *x, double *out) {
    const double X = exp(M_PI * x[0]);
    if (kind == 1 || kind == 2) {
        double s = sin(M_PI * x[1]), ee = exp(cf[2] * x[1]);
        if (kind == 2) { s += sin(M_PI * x[2]); ee += exp(cf[2] * x[2]); }
        out[0] = cf[0] * X * s + cf[1] * ee;
        return;
    }
    const double k = cf[0], c = cf[1], e = cf[2];
    const double sy = sin(M_PI * x[1]), cy = cos(M_PI * x[1]);
    if (kind == 3) {
        out[0] = -k * (X * sy);
        out[1] = -k * (X * cy + c * exp(e * x[1]));
    } else {
        const double sz = sin(M_PI * x[2]), cz = cos(M_PI * x[2]);
        out[0] = -k * (X * (sy + sz));
        out[1] = -k * (X * cy + c * exp(e * x[1]));
        out[2] = -k * (X * cz + c * exp(e * x[2]));
    }
}

struct FieldArgs {
    int form, vel, kind, dim, nn, nf;
    int64_t C;
    const double *V, *det, *coef;
    const int *cells, *cf;
    const signed char *cs;
};

// value of the field at reference point x of cell c (ncomp = dim for velocities, else 1)
__device__ inline void field_value(const FieldArgs &a, int64_t c, const double *x, double *out) {
    const int *cv = a.cells + c * a.nn;
    if (a.form == DPP_HDIV) {
        if (!a.vel) { out[0] = a.coef[c]; return; }
        double Vr[6][3], J[3][3], vr[3] = {0, 0, 0};
        rt_basis(a.kind, a.dim, x, Vr);
        cell_jacobian(a.kind, a.dim, a.nn, a.V, cv, J);
        for (int f = 0; f < a.nf; ++f) {
            const double w = (double)a.cs[c * a.nf + f] * a.coef[a.cf[c * a.nf + f]];
            for (int d = 0; d < a.dim; ++d) vr[d] += Vr[f][d] * w;
        }
        for (int i = 0; i < a.dim; ++i) {
            double s = 0.0;
            for (int j = 0; j < a.dim; ++j) s += J[i][j] * vr[j];
            out[i] = s / a.det[c];
        }
        return;
    }
    double N[8];
    scalar_basis(a.kind, a.dim, x, N);
    const int nc = a.vel ? a.dim : 1;
    for (int i = 0; i < nc; ++i) out[i] = 0.0;
    for (int n = 0; n < a.nn; ++n) {
        const int64_t node = a.form == DPP_CGVMS ? (int64_t)cv[n] : c * a.nn + n;
        for (int i = 0; i < nc; ++i) out[i] += N[n] * a.coef[node * nc + i];
    }
}

__global__ void k_field_eval(FieldArgs a, RefPts R, double *out) {
    const int nc = a.vel ? a.dim : 1;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < a.C * R.nq; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = t / R.nq;
        const int q = (int)(t % R.nq);
        double v[3];
        field_value(a, c, R.p[q], v);
        for (int i = 0; i < nc; ++i) out[t * nc + i] = v[i];
    }
}

__global__ void k_cell_points(FieldArgs a, RefPts R, double *X) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < a.C * R.nq; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = t / R.nq;
        const int q = (int)(t % R.nq);
        const int *cv = a.cells + c * a.nn;
        double J[3][3];
        cell_jacobian(a.kind, a.dim, a.nn, a.V, cv, J);
        for (int i = 0; i < a.dim; ++i) {   // origin + J x (reference spectrum.py:160-161)
            double s = 0.0;
            for (int j = 0; j < a.dim; ++j) s += J[i][j] * R.p[q][j];
            X[t * a.dim + i] = a.V[(int64_t)cv[0] * a.dim + i] + s;
        }
    }
}

constexpr int L2_BLOCKS = 296, L2_THREADS = 256;

__global__ void __launch_bounds__(L2_THREADS) k_l2_partial(FieldArgs a, RefPts R, int ekind, double e0, double e1,
                                                           double e2, const double *exact, double *part) {
    __shared__ double red[L2_THREADS];
    const int nc = a.vel ? a.dim : 1;
    const double ecf[3] = {e0, e1, e2};
    double acc = 0.0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < a.C * R.nq; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = t / R.nq;
        const int q = (int)(t % R.nq);
        double v[3], ex[3];
        field_value(a, c, R.p[q], v);
        if (ekind) {
            const int *cv = a.cells + c * a.nn;
            double J[3][3], X[3] = {0, 0, 0};
            cell_jacobian(a.kind, a.dim, a.nn, a.V, cv, J);
            for (int i = 0; i < a.dim; ++i) {
                double s = 0.0;
                for (int j = 0; j < a.dim; ++j) s += J[i][j] * R.p[q][j];
                X[i] = a.V[(int64_t)cv[0] * a.dim + i] + s;
            }
            mms_value(ekind, ecf, X, ex);
        } else {
            for (int i = 0; i < nc; ++i) ex[i] = exact[t * nc + i];
        }
        double d2 = 0.0;
        for (int i = 0; i < nc; ++i) d2 += (v[i] - ex[i]) * (v[i] - ex[i]);
        acc += R.w[q] * d2 * a.det[c];
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = L2_THREADS / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void k_l2_final(int n, const double *part, double *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += part[i];
        out[0] = sqrt(s);
    }
}

RefPts ref_points(int dim, int nq, const double *pts, const double *w) {
    if (nq < 1 || nq > FQ_MAX) DPP_FAIL(DPP_ERR_VALUE, "1..128 reference points per cell");
    RefPts R;
    R.nq = nq;
    for (int q = 0; q < nq; ++q) {
        for (int d = 0; d < dim; ++d) R.p[q][d] = pts[q * dim + d];
        R.w[q] = w ? w[q] : 0.0;
    }
    return R;
}

FieldArgs field_args(Ctx *c, HostMesh &hm, DevMesh &m, int form, int field, const double *coef_dev) {
    if (field < 0 || field > 3) DPP_FAIL(DPP_ERR_VALUE, "field must be 0..3 (u1, p1, u2, p2)");
    if (form != DPP_HDIV && form != DPP_CGVMS && form != DPP_DGVMS) DPP_FAIL(DPP_ERR_VALUE, "unknown formulation");
    FieldArgs a{};
    a.form = form;
    a.vel = field == 0 || field == 2;
    a.kind = m.kind;
    a.dim = m.dim;
    a.nn = m.nn;
    a.nf = m.nf;
    a.C = m.C;
    a.V = m.verts.p;
    a.det = m.det.p;
    a.cells = m.cells.p;
    a.coef = coef_dev;
    if (form == DPP_HDIV && a.vel) {
        ensure_facets(c, hm, m);
        a.cf = m.cf.p;
        a.cs = m.cs.p;
    }
    return a;
}

int64_t field_size(const DevMesh &m, int form, int field) {
    const bool vel = field == 0 || field == 2;
    if (form == DPP_HDIV) return vel ? m.F : m.C;
    const int64_t nodes = form == DPP_CGVMS ? m.V : m.C * m.nn;
    return vel ? nodes * m.dim : nodes;
}

}  // namespace
}  // namespace dpp

using namespace dpp;

extern "C" {

int dpp_field_evaluate(dpp_ctx *ctx, dpp_mesh *mm, int formulation, int field, const double *coeffs, int64_t ncoef,
                       int nq, const double *ref_points_host, double *out_host) {
    return guard([&] {
        Ctx *c = &ctx->c;
        DevMesh &m = dev_mesh(c, mm->m);
        if (ncoef != field_size(m, formulation, field)) DPP_FAIL(DPP_ERR_VALUE, "coefficient vector has the wrong size");
        RefPts R = ref_points(m.dim, nq, ref_points_host, nullptr);
        DBuf<double> cf(ncoef, c->s);
        cf.upload(coeffs, ncoef);
        FieldArgs a = field_args(c, mm->m, m, formulation, field, cf.p);
        const int nc = a.vel ? m.dim : 1;
        DBuf<double> out((size_t)m.C * nq * nc, c->s);
        k_field_eval<<<grid_for(m.C * nq, 256, c->sms), 256, 0, c->s>>>(a, R, out.p);
        launched(c);
        out.download(out_host, (size_t)m.C * nq * nc);
        CK(cudaStreamSynchronize(c->s));
    });
}

int dpp_cell_points(dpp_ctx *ctx, dpp_mesh *mm, int nq, const double *ref_points_host, double *X_host) {
    return guard([&] {
        Ctx *c = &ctx->c;
        DevMesh &m = dev_mesh(c, mm->m);
        RefPts R = ref_points(m.dim, nq, ref_points_host, nullptr);
        FieldArgs a{};
        a.kind = m.kind; a.dim = m.dim; a.nn = m.nn; a.C = m.C; a.V = m.verts.p; a.cells = m.cells.p;
        DBuf<double> X((size_t)m.C * nq * m.dim, c->s);
        k_cell_points<<<grid_for(m.C * nq, 256, c->sms), 256, 0, c->s>>>(a, R, X.p);
        launched(c);
        X.download(X_host, (size_t)m.C * nq * m.dim);
        CK(cudaStreamSynchronize(c->s));
    });
}

int dpp_field_l2_error(dpp_ctx *ctx, dpp_mesh *mm, int formulation, int field, const double *coeffs, int64_t ncoef,
                       int nq, const double *ref_points_host, const double *weights_host, int exact_kind,
                       const double exact_coef[3], const double *exact_values_host, double *l2) {
    return guard([&] {
        Ctx *c = &ctx->c;
        DevMesh &m = dev_mesh(c, mm->m);
        if (ncoef != field_size(m, formulation, field)) DPP_FAIL(DPP_ERR_VALUE, "coefficient vector has the wrong size");
        if (exact_kind < 0 || exact_kind > 4) DPP_FAIL(DPP_ERR_VALUE, "unknown exact-field kind");
        const bool vel = field == 0 || field == 2;
        if (exact_kind && ((exact_kind >= 3) != vel || (exact_kind == 1 || exact_kind == 3) != (m.dim == 2)))
            DPP_FAIL(DPP_ERR_VALUE, "exact-field kind does not match the field / dimension");
        if (!exact_kind && !exact_values_host) DPP_FAIL(DPP_ERR_VALUE, "exact values missing");
        RefPts R = ref_points(m.dim, nq, ref_points_host, weights_host);
        DBuf<double> cf(ncoef, c->s);
        cf.upload(coeffs, ncoef);
        FieldArgs a = field_args(c, mm->m, m, formulation, field, cf.p);
        const int nc = vel ? m.dim : 1;
        DBuf<double> ex;
        if (!exact_kind) {
            ex.alloc((size_t)m.C * nq * nc, c->s);
            ex.upload(exact_values_host, (size_t)m.C * nq * nc);
        }
        DBuf<double> part(L2_BLOCKS, c->s), res(1, c->s);
        const double e0 = exact_kind ? exact_coef[0] : 0.0, e1 = exact_kind ? exact_coef[1] : 0.0,
                     e2 = exact_kind ? exact_coef[2] : 0.0;
        k_l2_partial<<<L2_BLOCKS, L2_THREADS, 0, c->s>>>(a, R, exact_kind, e0, e1, e2, ex.p, part.p);
        launched(c);
        k_l2_final<<<1, 32, 0, c->s>>>(L2_BLOCKS, part.p, res.p);
        launched(c);
        res.download(l2, 1);
        CK(cudaStreamSynchronize(c->s));
    });
}

}  // extern "C"
