// Device assembly of the ten-block four-field DPP systems.
//
// Reference: assembly.assemble_hdiv / _vms_cell_blocks / assemble_cgvms /
// assemble_dgvms / _Coo (assembly.py:123-147, :233-557).
//
// Pattern: every formulation is a Kronecker expansion of a scalar "node graph"
// G (CG: vertices, DG: cell-local nodes, H(div): facets).  The local couplings
// (cell pairs (a,b), DG interior-facet side pairs) are emitted as 64-bit keys
// in the reference's COO insertion order and stably radix-sorted, so G (with
// explicit zeros, sorted columns) is bit-identical to scipy's pattern and each
// G entry owns its list of contributions in insertion order.
// Values: one thread per G entry walks its contribution list, recomputes each
// cell's (or facet's) local integral in FP64 and writes the entries of all
// blocks that the entry expands to (deterministic segmented sum, no atomics).
// H(div) follows the reference's einsum order bitwise (needed: its AMG setup is
// ulp-sensitive).
#include <cub/cub.cuh>

#include <chrono>
#include <cmath>
#include <cstring>

#include "abi_guard.cuh"
#include "devmesh.cuh"
#include "mesh.h"
#include "system.cuh"

namespace dpp {

// ------------------------------------------------------------------ rules
struct Rule {
    int nq = 0, rdim = 0;
    double p[27][3] = {};
    double w[27] = {};
};

static const double GL_T[5][4] = {
    {0}, {0x1.0000000000000p-1},
    {0x1.b0cb174df99c8p-3, 0x1.93cd3a2c8198ep-1},
    {0x1.cda042f0236e0p-4, 0x1.0000000000000p-1, 0x1.c64bf7a1fb924p-1},
    {0x1.1c6490c2719ecp-4, 0x1.51ee013116102p-2, 0x1.5708ff6774f7fp-1, 0x1.dc736de7b1cc2p-1}};
static const double GL_W[5][4] = {
    {0}, {0x1.0000000000000p+0},
    {0x1.0000000000000p-1, 0x1.0000000000000p-1},
    {0x1.1c71c71c71c73p-2, 0x1.c71c71c71c71cp-2, 0x1.1c71c71c71c73p-2},
    {0x1.64340f7e7b666p-3, 0x1.4de5f840c24cdp-2, 0x1.4de5f840c24cdp-2, 0x1.64340f7e7b666p-3}};

// elements.quadrature_rule (elements.py:175-221) for the degrees used here
static Rule cell_rule(int kind, int degree) {
    Rule r;
    degree = std::max(degree, 1);
    const int dim = kind_dim(kind);
    r.rdim = dim;
    if (kind == DPP_QUAD || kind == DPP_HEX) {
        const int n = (degree + 2) / 2;   // ceil((degree+1)/2)
        if (n > 4) throw Error(DPP_ERR_VALUE, "quadrature degree too high");
        int q = 0;
        if (dim == 2) {
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j, ++q) {
                    r.p[q][0] = GL_T[n][i]; r.p[q][1] = GL_T[n][j];
                    r.w[q] = 1.0 * GL_W[n][i] * GL_W[n][j];
                }
        } else {
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j)
                    for (int k = 0; k < n; ++k, ++q) {
                        r.p[q][0] = GL_T[n][i]; r.p[q][1] = GL_T[n][j]; r.p[q][2] = GL_T[n][k];
                        r.w[q] = 1.0 * GL_W[n][i] * GL_W[n][j] * GL_W[n][k];
                    }
        }
        r.nq = q;
        return r;
    }
    if (kind == DPP_TRI) {
        if (degree == 1) { r.nq = 1; r.p[0][0] = r.p[0][1] = 1.0 / 3; r.w[0] = 0.5; return r; }
        if (degree == 2) {
            const double pts[3][2] = {{1.0 / 6, 1.0 / 6}, {2.0 / 3, 1.0 / 6}, {1.0 / 6, 2.0 / 3}};
            r.nq = 3;
            for (int q = 0; q < 3; ++q) { r.p[q][0] = pts[q][0]; r.p[q][1] = pts[q][1]; r.w[q] = 1.0 / 6; }
            return r;
        }
        const int n = (degree + 3) / 2;   // ceil((degree+2)/2)
        int q = 0;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j, ++q) {
                const double u = GL_T[n][i], v = GL_T[n][j];
                r.p[q][0] = u;
                r.p[q][1] = v * (1 - u);
                r.w[q] = GL_W[n][i] * GL_W[n][j] * (1 - u);
            }
        r.nq = q;
        return r;
    }
    // TET
    if (degree == 1) { r.nq = 1; r.p[0][0] = r.p[0][1] = r.p[0][2] = 0.25; r.w[0] = 1.0 / 6; return r; }
    if (degree == 2) {
        const double a = (5.0 + 3.0 * std::sqrt(5.0)) / 20.0, b = (5.0 - std::sqrt(5.0)) / 20.0;
        const double pts[4][3] = {{a, b, b}, {b, a, b}, {b, b, a}, {b, b, b}};
        r.nq = 4;
        for (int q = 0; q < 4; ++q) {
            for (int d = 0; d < 3; ++d) r.p[q][d] = pts[q][d];
            r.w[q] = 1.0 / 24;
        }
        return r;
    }
    throw Error(DPP_ERR_VALUE, "TET cell rules above degree 2 are not needed on the hot path");
}

// facet reference rule (assembly.py:161-170): 2D Gauss on [0,1]; TET faces: TRI
// rule (ref measure 1/2); HEX faces: QUAD rule
static Rule facet_rule(int kind, int degree, double &ref_measure) {
    const int dim = kind_dim(kind);
    if (dim == 2) {
        Rule r;
        const int n = (degree + 2) / 2;   // ceil((degree+1)/2)
        r.nq = n;
        r.rdim = 1;
        for (int q = 0; q < n; ++q) { r.p[q][0] = GL_T[n][q]; r.w[q] = GL_W[n][q]; }
        ref_measure = 1.0;
        return r;
    }
    if (kind == DPP_TET) { ref_measure = 0.5; return cell_rule(DPP_TRI, degree); }
    ref_measure = 1.0;
    return cell_rule(DPP_QUAD, degree);
}

// ------------------------------------------------------------------ element tables
struct Elem {
    int kind, dim, nn, nq;
    double w[8];
    double N[8][8];       // [q][a]
    double G[8][8][3];    // [q][a][j] reference gradients
    double Mref[8][8];    // sum_q w N_a N_b
    double wsum;
};

__host__ __device__ inline void scalar_basis(int kind, int dim, const double *x, double *N, double *G) {
    if (kind == DPP_TRI || kind == DPP_TET) {
        double s = x[0];
        for (int d = 1; d < dim; ++d) s += x[d];
        N[0] = 1.0 - s;
        for (int d = 0; d < dim; ++d) N[d + 1] = x[d];
        if (G) {
            for (int j = 0; j < dim; ++j) G[j] = -1.0;
            for (int a = 1; a <= dim; ++a)
                for (int j = 0; j < dim; ++j) G[a * 3 + j] = (a - 1 == j) ? 1.0 : 0.0;
        }
        return;
    }
    const int nd = 1 << dim;
    for (int a = 0; a < nd; ++a) {
        double v = 1.0;
        double g[3] = {1.0, 1.0, 1.0};
        for (int ax = 0; ax < dim; ++ax) {
            const int s = (a >> ax) & 1;
            const double f = s ? x[ax] : 1.0 - x[ax];
            const double df = s ? 1.0 : -1.0;
            v *= f;
            for (int o = 0; o < dim; ++o) g[o] *= (o == ax) ? df : f;
        }
        N[a] = v;
        if (G)
            for (int o = 0; o < dim; ++o) G[a * 3 + o] = g[o];
    }
}

static Elem make_elem(int kind) {
    Elem e{};
    e.kind = kind;
    e.dim = kind_dim(kind);
    e.nn = kind_nodes(kind);
    Rule r = cell_rule(kind, 2);
    e.nq = r.nq;
    double ws = 0.0;
    for (int q = 0; q < r.nq; ++q) {
        e.w[q] = r.w[q];
        ws += r.w[q];
        scalar_basis(kind, e.dim, r.p[q], e.N[q], &e.G[q][0][0]);
    }
    e.wsum = ws;
    for (int a = 0; a < e.nn; ++a)
        for (int b = 0; b < e.nn; ++b) {
            double s = 0.0;
            for (int q = 0; q < e.nq; ++q) s += e.w[q] * e.N[q][a] * e.N[q][b];
            e.Mref[a][b] = s;
        }
    return e;
}

// ------------------------------------------------------------------ device mesh (devmesh.cuh)

// J (mesh.py:175-183) and J^-1 by LU with partial pivoting (numpy.linalg.inv)
__global__ void k_geom(int64_t C, int dim, int kind, int nn, const double *V, const int *cells,
                       double *Jinv) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C; c += (int64_t)gridDim.x * blockDim.x) {
        double a[9] = {0}, inv[9] = {0};
        const int *cv = cells + c * nn;
        if (kind == DPP_TRI || kind == DPP_TET) {
            for (int k = 0; k < dim; ++k)
                for (int d = 0; d < dim; ++d) a[d * dim + k] = V[(int64_t)cv[k + 1] * dim + d] - V[(int64_t)cv[0] * dim + d];
        } else {
            for (int d = 0; d < dim; ++d) a[d * dim + d] = V[(int64_t)cv[nn - 1] * dim + d] - V[(int64_t)cv[0] * dim + d];
        }
        int perm[3] = {0, 1, 2};
        for (int k = 0; k < dim; ++k) {
            int p = k;
            double best = fabs(a[k * dim + k]);
            for (int r = k + 1; r < dim; ++r)
                if (fabs(a[r * dim + k]) > best) { best = fabs(a[r * dim + k]); p = r; }
            if (p != k) {
                for (int cc = 0; cc < dim; ++cc) { double t = a[k * dim + cc]; a[k * dim + cc] = a[p * dim + cc]; a[p * dim + cc] = t; }
                int t = perm[k]; perm[k] = perm[p]; perm[p] = t;
            }
            const double rp = 1.0 / a[k * dim + k];
            for (int r = k + 1; r < dim; ++r) {
                const double l = __dmul_rn(a[r * dim + k], rp);
                a[r * dim + k] = l;
                for (int cc = k + 1; cc < dim; ++cc) a[r * dim + cc] = __dsub_rn(a[r * dim + cc], __dmul_rn(l, a[k * dim + cc]));
            }
        }
        for (int col = 0; col < dim; ++col) {
            double y[3];
            for (int i = 0; i < dim; ++i) {
                double s = perm[i] == col ? 1.0 : 0.0;
                for (int j = 0; j < i; ++j) s = __dsub_rn(s, __dmul_rn(a[i * dim + j], y[j]));
                y[i] = s;
            }
            for (int i = dim - 1; i >= 0; --i) {
                double s = y[i];
                for (int j = i + 1; j < dim; ++j) s = __dsub_rn(s, __dmul_rn(a[i * dim + j], y[j]));
                y[i] = s / a[i * dim + i];
            }
            for (int i = 0; i < dim; ++i) inv[i * dim + col] = y[i];
        }
        for (int k = 0; k < dim * dim; ++k) Jinv[c * dim * dim + k] = inv[k];
    }
}

DevMesh &dev_mesh(Ctx *c, HostMesh &m) {
    if (m.dev && m.dev->c == c) return *m.dev;
    auto d = std::make_shared<DevMesh>();
    d->c = c;
    d->dim = m.dim;
    d->kind = m.kind;
    d->nn = kind_nodes(m.kind);
    d->nf = kind_facets(m.kind);
    d->nvf = kind_facet_nodes(m.kind);
    d->V = m.n_vertices;
    d->C = m.n_cells;
    d->F = m.n_facets;
    // device-layout image (int32 ids) in pinned host memory, built once per mesh: every
    // upload is then asynchronous copies at full PCIe / C2C bandwidth
    struct Part { size_t off, bytes; };
    auto pad = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t nV = m.vertices.size(), nD = m.det.size(), nC = m.cells.size(), nCF = m.cell_facets.size(),
                 nFV = m.facet_vertex_ids.size(), nF = m.facet_plus.size(), nCS = m.cell_facet_signs.size(),
                 nFN = m.facet_normals.size(), nFM = m.facet_measures.size();
    Part pv{0, 8 * nV}, pd{0, 8 * nD}, pc{0, 4 * nC}, pcf{0, 4 * nCF}, pfv{0, 4 * nFV}, pfp{0, 4 * nF},
        pfm{0, 4 * nF}, pcs{0, nCS}, pfn{0, 8 * nFN}, pfs{0, 8 * nFM};
    size_t total = 0;
    for (Part *q : {&pv, &pd, &pc, &pcf, &pfv, &pfp, &pfm, &pcs, &pfn, &pfs}) { q->off = total; total += pad(q->bytes); }
    if (!m.pinned || m.pinned_bytes != total) {
        void *h = nullptr;
        CK(cudaMallocHost(&h, std::max<size_t>(total, 256)));
        m.pinned = std::shared_ptr<void>(h, [](void *q) { cudaFreeHost(q); });
        m.pinned_bytes = total;
        unsigned char *B = static_cast<unsigned char *>(h);
        std::memcpy(B + pv.off, m.vertices.data(), pv.bytes);
        std::memcpy(B + pd.off, m.det.data(), pd.bytes);
        auto narrow = [&](const Part &q, const std::vector<int64_t> &v) {
            int *o = reinterpret_cast<int *>(B + q.off);
            for (size_t i = 0; i < v.size(); ++i) o[i] = (int)v[i];
        };
        narrow(pc, m.cells);
        narrow(pcf, m.cell_facets);
        narrow(pfv, m.facet_vertex_ids);
        narrow(pfp, m.facet_plus);
        narrow(pfm, m.facet_minus);
        std::memcpy(B + pcs.off, m.cell_facet_signs.data(), pcs.bytes);
        std::memcpy(B + pfn.off, m.facet_normals.data(), pfn.bytes);
        std::memcpy(B + pfs.off, m.facet_measures.data(), pfs.bytes);
    }
    const unsigned char *B = static_cast<const unsigned char *>(m.pinned.get());
    auto up = [&](auto &buf, const Part &q, size_t count) {
        buf.alloc(count, c->s);
        if (count) CK(cudaMemcpyAsync(buf.p, B + q.off, q.bytes, cudaMemcpyHostToDevice, c->s));
    };
    up(d->verts, pv, nV);
    up(d->det, pd, nD);
    up(d->cells, pc, nC);
    m.dev_bytes = pv.bytes + pd.bytes + pc.bytes;
    m.bc_bytes = 0;
    // the facet arrays (80 % of the image for TET meshes) follow only when a formulation uses them
    const Part fparts[7] = {pcf, pfv, pfp, pfm, pcs, pfn, pfs};
    for (int q = 0; q < 7; ++q) { d->foff[q] = fparts[q].off; d->fbytes[q] = fparts[q].bytes; }
    // cell Jacobian inverses for the trace / field queries; every assembly recomputes them inside
    // its own timing, as the reference does (assembly.py:154-158)
    cell_jinv(c, *d);
    CK(cudaStreamSynchronize(c->s));
    m.dev = d;
    return *d;
}

void cell_jinv(Ctx *c, DevMesh &d) {
    if (d.Jinv.n != (size_t)d.C * d.dim * d.dim) d.Jinv.alloc((size_t)d.C * d.dim * d.dim, c->s);
    if (!d.C) return;
    k_geom<<<grid_for(d.C, 128, c->sms), 128, 0, c->s>>>(d.C, d.dim, d.kind, d.nn, d.verts.p, d.cells.p, d.Jinv.p);
    launched(c);
}

void ensure_facets(Ctx *c, HostMesh &hm, DevMesh &d) {
    if (d.facets) return;
    const unsigned char *B = static_cast<const unsigned char *>(hm.pinned.get());
    auto up = [&](auto &buf, int q, size_t count) {
        buf.alloc(count, c->s);
        if (count) CK(cudaMemcpyAsync(buf.p, B + d.foff[q], d.fbytes[q], cudaMemcpyHostToDevice, c->s));
        hm.dev_bytes += d.fbytes[q];
    };
    up(d.cf, 0, hm.cell_facets.size());
    up(d.fv, 1, hm.facet_vertex_ids.size());
    up(d.fplus, 2, hm.facet_plus.size());
    up(d.fminus, 3, hm.facet_minus.size());
    up(d.cs, 4, hm.cell_facet_signs.size());
    up(d.fn, 5, hm.facet_normals.size());
    up(d.fm, 6, hm.facet_measures.size());
    CK(cudaStreamSynchronize(c->s));
    d.facets = true;
}

__global__ void k_iota64(int64_t n, int64_t *o) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) o[i] = i;
}

// ------------------------------------------------------------------ facet points
struct FRule { int nq, rdim; double p[27][2]; double w[27]; double rm; };
static FRule frule(int kind, int degree) {
    double rm;
    Rule r = facet_rule(kind, degree, rm);
    FRule f{};
    f.nq = r.nq;
    f.rdim = r.rdim;
    f.rm = rm;
    for (int q = 0; q < r.nq; ++q) {
        f.p[q][0] = r.p[q][0];
        f.p[q][1] = r.p[q][1];
        f.w[q] = r.w[q];
    }
    return f;
}

// X = v0 + sum_k ref_qk (v_{k+1} - v0), W = w_q * (|f| / ref measure) (assembly.py:173-181)
__device__ inline void facet_point(const FRule &R, int dim, int nvf, const int *fv, const double *V,
                                   int64_t f, int q, double *X) {
    const int *vid = fv + f * nvf;
    for (int i = 0; i < dim; ++i) {
        const double v0 = V[(int64_t)vid[0] * dim + i];
        double s = 0.0;
        for (int k = 0; k < R.rdim; ++k) s += R.p[q][k] * (V[(int64_t)vid[k + 1] * dim + i] - v0);
        X[i] = v0 + s;
    }
}

__global__ void k_facet_points(int64_t nf, const int64_t *fids, FRule R, int dim, int nvf,
                               const int *fv, const double *V, const double *fm, double *X,
                               double *W) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nf * R.nq; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / R.nq;
        const int q = (int)(t % R.nq);
        const int64_t f = fids[i];
        double x[3];
        facet_point(R, dim, nvf, fv, V, f, q, x);
        for (int d = 0; d < dim; ++d) X[t * dim + d] = x[d];
        if (W) W[t] = R.w[q] * (fm[f] / R.rm);
    }
}

// trace of the nodal basis of cell c at physical point X (assembly.py:184-189)
__device__ inline void trace(int kind, int dim, int nn, const double *V, const int *cells,
                             const double *Jinv, int64_t c, const double *X, double *N) {
    const double *o = V + (int64_t)cells[c * nn] * dim;
    const double *Ji = Jinv + c * dim * dim;
    double xh[3];
    for (int i = 0; i < dim; ++i) {
        double s = 0.0;
        for (int j = 0; j < dim; ++j) s += Ji[i * dim + j] * (X[j] - o[j]);
        xh[i] = s;
    }
    scalar_basis(kind, dim, xh, N, nullptr);
}

// ------------------------------------------------------------------ node graph
struct Graph {
    int64_t n_nodes = 0, nnz = 0;
    DBuf<int> ptr, col, row;
    DBuf<int64_t> seg;      // contribution segment starts (nnz+1)
    DBuf<int> pay;          // sorted payloads
};

__global__ void k_flag_new(int64_t n, const uint64_t *k, int *flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = (i == 0 || k[i] != k[i - 1]) ? 1 : 0;
}
__global__ void k_segments(int64_t n, const uint64_t *k, const int *flag, const int64_t *eid,
                           int64_t nodes, int64_t *seg, int *col, int *row, int *rowcnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (!flag[i]) continue;
        const int64_t e = eid[i];
        seg[e] = i;
        const int64_t r = (int64_t)(k[i] / (uint64_t)nodes);
        col[e] = (int)(k[i] % (uint64_t)nodes);
        row[e] = (int)r;
        atomicAdd(&rowcnt[r], 1);
    }
}

// keys/payloads in insertion order -> G (stable sort keeps insertion order per key)
static Graph build_graph(Ctx *c, DBuf<uint64_t> &keys, DBuf<int> &pay, int64_t n, int64_t nodes) {
    Graph g;
    g.n_nodes = nodes;
    DBuf<uint64_t> k2(n, c->s);
    g.pay.alloc(n, c->s);
    int end_bit = 1;
    while (end_bit < 64 && ((uint64_t)1 << end_bit) < (uint64_t)nodes * (uint64_t)nodes) ++end_bit;
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, k2.p, pay.p, g.pay.p, n, 0, end_bit, c->s));
    {
        DBuf<char> t(tb, c->s);
        CK(cub::DeviceRadixSort::SortPairs(t.p, tb, keys.p, k2.p, pay.p, g.pay.p, n, 0, end_bit, c->s));
        launched(c);
    }
    DBuf<int> flag(n, c->s);
    DBuf<int64_t> eid(n, c->s);
    k_flag_new<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, k2.p, flag.p);
    launched(c);
    tb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, flag.p, eid.p, n, c->s));
    {
        DBuf<char> t(tb, c->s);
        CK(cub::DeviceScan::ExclusiveSum(t.p, tb, flag.p, eid.p, n, c->s));
        launched(c);
    }
    int64_t last_e = 0;
    int last_f = 0;
    CK(cudaMemcpyAsync(&last_e, eid.p + n - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, c->s));
    CK(cudaMemcpyAsync(&last_f, flag.p + n - 1, sizeof(int), cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    g.nnz = last_e + last_f;
    g.seg.alloc(g.nnz + 1, c->s);
    g.col.alloc(g.nnz, c->s);
    g.row.alloc(g.nnz, c->s);
    DBuf<int> rowcnt(nodes, c->s);
    CK(cudaMemsetAsync(rowcnt.p, 0, sizeof(int) * nodes, c->s));
    k_segments<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, k2.p, flag.p, eid.p, nodes, g.seg.p,
                                                           g.col.p, g.row.p, rowcnt.p);
    launched(c);
    CK(cudaMemcpyAsync(g.seg.p + g.nnz, &n, sizeof(int64_t), cudaMemcpyHostToDevice, c->s));
    counts_to_ptr(c, rowcnt.p, (int)nodes, g.ptr);
    CK(cudaStreamSynchronize(c->s));
    return g;
}

// cell pairs (a,b) of node ids nodes_of(c,a) -> keys, payload c*nn*nn + a*nn + b
__global__ void k_emit_cell_pairs(int64_t C, int nn, const int *cellnodes, int node_mode, int64_t nodes,
                                  uint64_t *keys, int *pay) {
    const int64_t per = (int64_t)nn * nn;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < C * per; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = t / per;
        const int a = (int)((t / nn) % nn), b = (int)(t % nn);
        int64_t na, nb;
        if (node_mode == 0) { na = cellnodes[c * nn + a]; nb = cellnodes[c * nn + b]; }   // CG: vertices / H(div): facets
        else { na = c * nn + a; nb = c * nn + b; }                                        // DG nodes
        keys[t] = (uint64_t)na * (uint64_t)nodes + (uint64_t)nb;
        pay[t] = (int)t;
    }
}
// DG interior facet side pairs in the reference insertion order: (s,t) major, facet, a, b
__global__ void k_emit_dg_facets(int64_t Fi, int nn, int64_t C, const int *interior, const int *fplus,
                                 const int *fminus, int64_t nodes, uint64_t *keys, int *pay) {
    const int64_t per = (int64_t)nn * nn;
    const int64_t base = C * per;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 4 * Fi * per; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = t / per;
        const int st = (int)(q / Fi);
        const int64_t fi = q % Fi;
        const int a = (int)((t / nn) % nn), b = (int)(t % nn);
        const int f = interior[fi];
        const int64_t cs = (st < 2) ? fplus[f] : fminus[f];
        const int64_t ct = (st % 2 == 0) ? fplus[f] : fminus[f];
        keys[t] = (uint64_t)(cs * nn + a) * (uint64_t)nodes + (uint64_t)(ct * nn + b);
        pay[t] = (int)(base + t);
    }
}

// ------------------------------------------------------------------ VMS values
struct VmsArgs {
    Elem E;
    int64_t C, Fi;
    int dg;
    const double *det, *Jinv;
    const int *gptr, *gcol, *grow;
    const int64_t *seg;
    const int *pay;
    int64_t nnz;
    double s_uu[2], s_pp_gg[2], s_pp_m, s_cross;
    const double *ck[2];         // per-cell k1 / k2 (config-3 extension) or null: s_uu, s_pp_gg per cell
    double mu;
    double c_uu[2], c_pp[2];     // DG facet coefficients (before side signs)
    // DG facet tables
    const int *interior;
    const double *fW, *fNp, *fNm, *fn;  // (Fi,nq), (Fi,nq,nn) x2, normals of all facets
    int fnq;
    // DG prescribed-flux facets: network 1's nv1 facets then network 2's
    int64_t nvt, nv1;
    const int *vfac;
    const double *vW, *vN;              // (nvt,nq), (nvt,nq,nn)
    // outputs (CSR idx/val) ; ptr arrays computed separately
    int *uu_i[2], *up_i[2], *pu_i[2], *pp_i[2], *cr_i;
    double *uu_v[2], *up_v[2], *pu_v[2], *pp_v[2], *cr_v;
};

// per-cell gradient of node a at quadrature point q: Gp_i = sum_j Gref_qaj Jinv_ji
__device__ inline void grad_phys(const Elem &E, const double *Ji, int q, int a, double *g) {
    for (int i = 0; i < E.dim; ++i) {
        double s = 0.0;
        for (int j = 0; j < E.dim; ++j) s += E.G[q][a][j] * Ji[j * E.dim + i];
        g[i] = s;
    }
}
template <int DIM>
__device__ inline void grad_phys(const Elem &E, const double *Ji, int q, int a, double *g) {
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < DIM; ++j) s += E.G[q][a][j] * Ji[j * DIM + i];
        g[i] = s;
    }
}

// One thread per node-graph entry, its contributions in insertion order (deterministic
// sums).  DIM is a template parameter so the per-entry block accumulators stay in
// registers, and the element tables are read from shared memory (per-thread a, b, q
// indices would serialise constant-bank reads).
template <int DIM>
__global__ void __launch_bounds__(128) k_vms_values(VmsArgs A) {
    __shared__ Elem E;
    {
        const double *src = reinterpret_cast<const double *>(&A.E);
        double *dst = reinterpret_cast<double *>(&E);
        for (int i = threadIdx.x; i < (int)(sizeof(Elem) / sizeof(double)); i += blockDim.x) dst[i] = src[i];
        __syncthreads();
    }
    constexpr int dim = DIM;
    const int nn = E.nn;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < A.nnz; e += (int64_t)gridDim.x * blockDim.x) {
        double uu[2][3][3] = {}, up[2][3] = {}, pu[2][3] = {}, pp[2] = {}, cr = 0.0;
        for (int64_t t = A.seg[e]; t < A.seg[e + 1]; ++t) {
            const int64_t p = A.pay[t];
            const int64_t per = (int64_t)nn * nn;
            if (p < A.C * per) {       // cell contribution (assembly.py:330-342)
                const int64_t c = p / per;
                const int a = (int)((p / nn) % nn), b = (int)(p % nn);
                const double det = A.det[c];
                const double *Ji = A.Jinv + c * dim * dim;
                const double mass = det * E.Mref[a][b];
                double gg = 0.0, gnab[3] = {0, 0, 0}, gnba[3] = {0, 0, 0};
                for (int q = 0; q < E.nq; ++q) {
                    double ga[3], gb[3];
                    grad_phys<DIM>(E, Ji, q, a, ga);
                    grad_phys<DIM>(E, Ji, q, b, gb);
                    #pragma unroll
                    for (int i = 0; i < dim; ++i) {
                        gg += E.w[q] * ga[i] * gb[i];
                        gnab[i] += E.w[q] * ga[i] * E.N[q][b];
                        gnba[i] += E.w[q] * gb[i] * E.N[q][a];
                    }
                }
                gg *= det;
                #pragma unroll
                for (int i = 0; i < dim; ++i) { gnab[i] *= det; gnba[i] *= det; }
                #pragma unroll
                for (int n = 0; n < 2; ++n) {
                    // per-cell k: (0.5 mu) / k_c and (0.5 k_c) / mu, the scalar path's operation order
                    const double suu = A.ck[n] ? 0.5 * A.mu / A.ck[n][c] : A.s_uu[n];
                    const double spp = A.ck[n] ? 0.5 * A.ck[n][c] / A.mu : A.s_pp_gg[n];
                    const double v = suu * mass;
                    #pragma unroll
                    for (int i = 0; i < dim; ++i) uu[n][i][i] += v;
                    pp[n] += spp * gg + A.s_pp_m * mass;
                }
                #pragma unroll
                for (int i = 0; i < dim; ++i) {
                    const double vu = -(gnab[i] + 0.5 * gnba[i]), vp = gnba[i] + 0.5 * gnab[i];
                    up[0][i] += vu; up[1][i] += vu;
                    pu[0][i] += vp; pu[1][i] += vp;
                }
                cr += A.s_cross * mass;
            } else if (p >= A.C * per + 4 * A.Fi * per) {   // DG prescribed-flux facet (assembly.py:521-531)
                const int64_t idx = p - A.C * per - 4 * A.Fi * per;
                const int64_t vi = idx / per;
                const int a = (int)((idx / nn) % nn), b = (int)(idx % nn);
                const int net = vi < A.nv1 ? 0 : 1;
                double F = 0.0;
                for (int q = 0; q < A.fnq; ++q)
                    F += A.vW[vi * A.fnq + q] * A.vN[(vi * A.fnq + q) * nn + a] * A.vN[(vi * A.fnq + q) * nn + b];
                const double *n = A.fn + (int64_t)A.vfac[vi] * dim;
                #pragma unroll
                for (int i = 0; i < dim; ++i) {   // (branches keep the accumulators in registers)
                    if (net == 0) { up[0][i] += F * n[i]; pu[0][i] += -(F * n[i]); }
                    else { up[1][i] += F * n[i]; pu[1][i] += -(F * n[i]); }
                }
            } else {                   // DG interior facet side pair (assembly.py:497-517)
                const int64_t idx = p - A.C * per;
                const int64_t q2 = idx / per;
                const int st = (int)(q2 / A.Fi);
                const int64_t fi = q2 % A.Fi;
                const int a = (int)((idx / nn) % nn), b = (int)(idx % nn);
                const double ss = st < 2 ? 1.0 : -1.0, tt = (st % 2 == 0) ? 1.0 : -1.0;
                const double *Ns = (st < 2 ? A.fNp : A.fNm) + fi * A.fnq * nn;
                const double *Nt = (st % 2 == 0 ? A.fNp : A.fNm) + fi * A.fnq * nn;
                double F = 0.0;
                for (int q = 0; q < A.fnq; ++q) F += A.fW[fi * A.fnq + q] * Ns[q * nn + a] * Nt[q * nn + b];
                const double *n = A.fn + (int64_t)A.interior[fi] * dim;
                #pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const double cu = A.c_uu[k] * ss * tt;
                    #pragma unroll
                    for (int i = 0; i < dim; ++i)
                        #pragma unroll
                        for (int j = 0; j < dim; ++j) uu[k][i][j] += cu * (F * n[i] * n[j]);
                    pp[k] += A.c_pp[k] * ss * tt * F;
                }
                #pragma unroll
                for (int i = 0; i < dim; ++i) {
                    const double vu = 0.5 * ss * (F * n[i]), vp = -0.5 * tt * (F * n[i]);
                    up[0][i] += vu; up[1][i] += vu;
                    pu[0][i] += vp; pu[1][i] += vp;
                }
            }
        }
        // Kronecker placement of entry e (row v, col v2) into the expanded blocks
        const int v = A.grow[e], v2 = A.gcol[e];
        const int64_t g0 = A.gptr[v], len = A.gptr[v + 1] - g0, o = e - g0;
        #pragma unroll
        for (int n = 0; n < 2; ++n) {
            #pragma unroll
            for (int i = 0; i < dim; ++i) {
                const int64_t rs = (int64_t)dim * dim * g0 + (int64_t)i * dim * len;
                #pragma unroll
                for (int j = 0; j < dim; ++j) {
                    const int64_t pos = rs + o * dim + j;
                    A.uu_i[n][pos] = v2 * dim + j;
                    A.uu_v[n][pos] = uu[n][i][j];
                }
                const int64_t ps = (int64_t)dim * g0 + (int64_t)i * len + o;
                A.up_i[n][ps] = v2;
                A.up_v[n][ps] = up[n][i];
            }
            #pragma unroll
            for (int j = 0; j < dim; ++j) {
                const int64_t pos = (int64_t)dim * g0 + o * dim + j;
                A.pu_i[n][pos] = v2 * dim + j;
                A.pu_v[n][pos] = pu[n][j];
            }
            A.pp_i[n][e] = v2;
            A.pp_v[n][e] = pp[n];
        }
        if (A.cr_i) {
            A.cr_i[e] = v2;
            A.cr_v[e] = cr;
        }
    }
}

// row pointers of the expanded blocks from G.ptr
__global__ void k_kron_ptr(int64_t nodes, int dim, const int *gptr, int *uu, int *up, int *pu) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= nodes; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g0 = gptr[v];
        if (v < nodes) {
            const int64_t len = gptr[v + 1] - g0;
            for (int i = 0; i < dim; ++i) {
                uu[v * dim + i] = (int)(dim * dim * g0 + i * dim * len);
                up[v * dim + i] = (int)(dim * g0 + i * len);
            }
        } else {
            uu[v * dim] = (int)(dim * dim * g0);
            up[v * dim] = (int)(dim * g0);
        }
        pu[v] = (int)(dim * g0);
    }
}

// DG cross blocks: cell-local mass (assembly.py:487-489)
__global__ void k_dg_cross(int64_t C, Elem E, const double *det, double s_cross, int *ptr, int *idx,
                           double *val) {
    const int nn = E.nn;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= C * nn; r += (int64_t)gridDim.x * blockDim.x) {
        ptr[r] = (int)(r * nn);
        if (r == C * nn) continue;
        const int64_t c = r / nn;
        const int a = (int)(r % nn);
        for (int b = 0; b < nn; ++b) {
            idx[r * nn + b] = (int)(c * nn + b);
            val[r * nn + b] = s_cross * (det[c] * E.Mref[a][b]);
        }
    }
}

// DG interior facet traces at the degree-2 facet rule
__global__ void k_dg_facet_tables(int64_t Fi, FRule R, int kind, int dim, int nn, int nvf,
                                  const int *interior, const int *fv, const int *fplus,
                                  const int *fminus, const double *V, const int *cells,
                                  const double *Jinv, const double *fm, double *W, double *Np,
                                  double *Nm) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < Fi * R.nq; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t fi = t / R.nq;
        const int q = (int)(t % R.nq);
        const int f = interior[fi];
        double X[3];
        facet_point(R, dim, nvf, fv, V, f, q, X);
        W[t] = R.w[q] * (fm[f] / R.rm);
        trace(kind, dim, nn, V, cells, Jinv, fplus[f], X, Np + t * nn);
        if (Nm) trace(kind, dim, nn, V, cells, Jinv, fminus[f], X, Nm + t * nn);
    }
}
// DG-VMS prescribed-flux facets (assembly.py:521-531): plus-cell pairs of every velocity
// facet, both networks' lists back to back (payloads after the interior-facet ones)
__global__ void k_emit_dg_vel(int64_t nvt, int nn, int64_t base, const int *vfac, const int *fplus, int64_t nodes,
                              uint64_t *keys, int *pay) {
    const int64_t per = (int64_t)nn * nn;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nvt * per; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t vi = t / per;
        const int a = (int)((t / nn) % nn), b = (int)(t % nn);
        const int64_t c = fplus[vfac[vi]];
        keys[t] = (uint64_t)(c * nn + a) * (uint64_t)nodes + (uint64_t)(c * nn + b);
        pay[t] = (int)(base + t);
    }
}
// f_p -= sum_q W_q (u.n)_q N_a on the velocity facets (assembly.py:532-535)
__global__ void k_rhs_dg_vel(int64_t nv, const int64_t *fids, FRule R, int kind, int dim, int nn, int nvf,
                             const int *fv, const int *fplus, const double *fm, const double *V, const int *cells,
                             const double *Jinv, const double *un, int64_t *dof, double *val) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = fids[i];
        const int64_t c = fplus[f];
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int q = 0; q < R.nq; ++q) {
            double X[3], N[8];
            facet_point(R, dim, nvf, fv, V, f, q, X);
            trace(kind, dim, nn, V, cells, Jinv, c, X, N);
            const double W = R.w[q] * (fm[f] / R.rm);
            const double wu = W * un[i * R.nq + q];
            for (int a = 0; a < nn; ++a) acc[a] += wu * N[a];
        }
        for (int a = 0; a < nn; ++a) {
            dof[i * nn + a] = c * nn + a;
            val[i * nn + a] = -acc[a];
        }
    }
}

// ------------------------------------------------------------------ H(div) values
struct HdivArgs {
    int dim, nf, nq;
    double w[8];
    double Vref[8][6][3];   // [q][f][j]
    double s_uu[2];
    const double *ck[2];   // per-cell k1 / k2 or null: mu / k_c
    double mu;
    const double *V, *det;
    const int *cells, *cf;
    const signed char *cs;
    int nn, kind;
    const int *gptr, *gcol, *grow;
    const int64_t *seg;
    const int *pay;
    int64_t nnz;
    int *uu_i[2];
    double *uu_v[2];
};

// local mass[f][g] of cell c, einsum order of assembly.py:262-264 (bitwise)
__device__ inline double hdiv_mass(const HdivArgs &A, int64_t c, int lf, int lg) {
    const int dim = A.dim;
    double J[9];
    const int *cv = A.cells + c * A.nn;
    if (A.kind == DPP_TRI || A.kind == DPP_TET) {
        for (int k = 0; k < dim; ++k)
            for (int d = 0; d < dim; ++d) J[d * dim + k] = __dsub_rn(A.V[(int64_t)cv[k + 1] * dim + d], A.V[(int64_t)cv[0] * dim + d]);
    } else {
        for (int k = 0; k < dim * dim; ++k) J[k] = 0.0;
        for (int d = 0; d < dim; ++d) J[d * dim + d] = __dsub_rn(A.V[(int64_t)cv[A.nn - 1] * dim + d], A.V[(int64_t)cv[0] * dim + d]);
    }
    const double det = A.det[c];
    double m = 0.0;
    for (int q = 0; q < A.nq; ++q) {
        double acc = 0.0;
        for (int i = 0; i < dim; ++i) {
            double vf = __dmul_rn(J[i * dim], A.Vref[q][lf][0]);
            double vg = __dmul_rn(J[i * dim], A.Vref[q][lg][0]);
            for (int j = 1; j < dim; ++j) {
                vf = __dadd_rn(vf, __dmul_rn(J[i * dim + j], A.Vref[q][lf][j]));
                vg = __dadd_rn(vg, __dmul_rn(J[i * dim + j], A.Vref[q][lg][j]));
            }
            vf = __ddiv_rn(vf, det);
            vg = __ddiv_rn(vg, det);
            acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(A.w[q], vf), vg));
        }
        m = __dadd_rn(m, acc);
    }
    m = __dmul_rn(m, det);
    const double sf = A.cs[c * A.nf + lf], sg = A.cs[c * A.nf + lg];
    return __dmul_rn(__dmul_rn(m, sf), sg);
}

__global__ void k_hdiv_uu(HdivArgs A) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < A.nnz; e += (int64_t)gridDim.x * blockDim.x) {
        double acc[2] = {0.0, 0.0};
        bool first = true;
        for (int64_t t = A.seg[e]; t < A.seg[e + 1]; ++t) {
            const int64_t p = A.pay[t];
            const int64_t per = (int64_t)A.nf * A.nf;
            const int64_t c = p / per;
            const int lf = (int)((p / A.nf) % A.nf), lg = (int)(p % A.nf);
            const double m = hdiv_mass(A, c, lf, lg);
            for (int n = 0; n < 2; ++n) {
                const double v = __dmul_rn(A.ck[n] ? __ddiv_rn(A.mu, A.ck[n][c]) : A.s_uu[n], m);
                acc[n] = first ? v : __dadd_rn(acc[n], v);
            }
            first = false;
        }
        for (int n = 0; n < 2; ++n) {
            A.uu_i[n][e] = A.gcol[e];
            A.uu_v[n][e] = acc[n];
        }
    }
}

// up (F x C): row f = [plus, minus]; pu (C x F): row c = its facets sorted by id;
// pp / cross diagonal (assembly.py:266-280)
__global__ void k_hdiv_rest(int64_t F, int64_t C, int nf, const int *fplus, const int *fminus,
                            const int *cf, const signed char *cs, const double *det, double wsum,
                            double bm, double nbm, int *up_p, int *up_i, double *up_v, int *pu_p,
                            int *pu_i, double *pu_v, int *pp_p, int *pp_i, double *pp_v,
                            double *cr_v) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= C; c += (int64_t)gridDim.x * blockDim.x) {
        pu_p[c] = (int)(c * nf);
        pp_p[c] = (int)c;
        if (c == C) continue;
        int ids[6];
        double sg[6];
        for (int k = 0; k < nf; ++k) { ids[k] = cf[c * nf + k]; sg[k] = cs[c * nf + k]; }
        for (int i = 1; i < nf; ++i)
            for (int j = i; j > 0 && ids[j - 1] > ids[j]; --j) {
                int t = ids[j]; ids[j] = ids[j - 1]; ids[j - 1] = t;
                double s = sg[j]; sg[j] = sg[j - 1]; sg[j - 1] = s;
            }
        for (int k = 0; k < nf; ++k) { pu_i[c * nf + k] = ids[k]; pu_v[c * nf + k] = sg[k]; }
        const double vol = det[c] * wsum;
        pp_i[c] = (int)c;
        pp_v[c] = bm * vol * 1.0;
        cr_v[c] = nbm * vol * 1.0;
    }
}
__global__ void k_hdiv_up(int64_t F, const int *fplus, const int *fminus, const int *upp, int *up_i,
                          double *up_v) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < F; f += (int64_t)gridDim.x * blockDim.x) {
        const int o = upp[f];
        up_i[o] = fplus[f];
        up_v[o] = -1.0;
        if (fminus[f] >= 0) { up_i[o + 1] = fminus[f]; up_v[o + 1] = 1.0; }
    }
}
__global__ void k_hdiv_up_cnt(int64_t F, const int *fminus, int *cnt) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < F; f += (int64_t)gridDim.x * blockDim.x)
        cnt[f] = fminus[f] >= 0 ? 2 : 1;
}

// ------------------------------------------------------------------ manufactured pressure on the device
// problem.py:100-144 in numpy's operation order: mu/pi * X * (sy [+ sz]) + c * (Y [+ Z])
__global__ void k_mms_p0(int64_t nf, const int64_t *fids, FRule R, int dim, int nvf, const int *fv, const double *V,
                         int kind, double mupi, double cc, double e, double *p0) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nf * R.nq; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / R.nq;
        const int q = (int)(t % R.nq);
        double X[3];
        facet_point(R, dim, nvf, fv, V, fids[i], q, X);
        const double Xe = exp(M_PI * X[0]);
        double s = sin(M_PI * X[1]), ee = exp(e * X[1]);
        if (kind == 2) {
            s = s + sin(M_PI * X[2]);
            ee = ee + exp(e * X[2]);
        }
        p0[t] = mupi * Xe * s + cc * ee;
    }
}

// ------------------------------------------------------------------ boundary RHS
// contributions of -(w.n, p0) on pressure facets (assembly.py:422-436, :291-300)
__global__ void k_rhs_nodal(int64_t nf, const int64_t *fids, FRule R, int kind, int dim, int nn,
                            int nvf, int dg, const int *fv, const int *fplus, const double *fn,
                            const double *fm, const double *V, const int *cells, const double *Jinv,
                            const double *p0, int64_t *dof, double *val) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nf; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = fids[i];
        const int64_t c = fplus[f];
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int q = 0; q < R.nq; ++q) {
            double X[3], N[8];
            facet_point(R, dim, nvf, fv, V, f, q, X);
            trace(kind, dim, nn, V, cells, Jinv, c, X, N);
            const double W = R.w[q] * (fm[f] / R.rm);
            const double wp = W * p0[i * R.nq + q];
            for (int a = 0; a < nn; ++a) acc[a] += wp * N[a];
        }
        for (int a = 0; a < nn; ++a)
            for (int d = 0; d < dim; ++d) {
                const int64_t k = (i * nn + a) * dim + d;
                const int64_t node = dg ? c * nn + a : cells[c * nn + a];
                dof[k] = node * dim + d;
                val[k] = -(acc[a] * fn[f * dim + d]);
            }
    }
}
__global__ void k_rhs_hdiv(int64_t nf, const int64_t *fids, FRule R, const double *fm,
                           const double *p0, int64_t *dof, double *val) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nf; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = fids[i];
        double s = 0.0;
        for (int q = 0; q < R.nq; ++q) s += (R.w[q] * (fm[f] / R.rm)) * p0[i * R.nq + q];
        dof[i] = f;
        val[i] = -s / fm[f];
    }
}
__global__ void k_seg_add(int64_t n, const int64_t *dof, const double *val, double *rhs) {
    // dof sorted (stable); one thread per run start sums the run in order
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (i > 0 && dof[i - 1] == dof[i]) continue;
        double s = rhs[dof[i]];
        for (int64_t j = i; j < n && dof[j] == dof[i]; ++j) s += val[j];
        rhs[dof[i]] = s;
    }
}
// np.add.at(rhs, dof, val) with the per-dof order of insertion
static void add_at(Ctx *c, int64_t n, DBuf<int64_t> &dof, DBuf<double> &val, double *rhs) {
    if (!n) return;
    DBuf<int64_t> d2(n, c->s);
    DBuf<double> v2(n, c->s);
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dof.p, d2.p, val.p, v2.p, n, 0, 64, c->s));
    DBuf<char> t(tb, c->s);
    CK(cub::DeviceRadixSort::SortPairs(t.p, tb, dof.p, d2.p, val.p, v2.p, n, 0, 64, c->s));
    launched(c);
    k_seg_add<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, d2.p, v2.p, rhs);
    launched(c);
    CK(cudaStreamSynchronize(c->s));
}

// ------------------------------------------------------------------ body force (gamma_b)
// VMS (assembly.py:352-356): fu[c,a,i] = 0.5 det intN_a g_i ; fp[c,a] = 0.5 k/mu det sum_q w_q (Gp_qa . g)
__global__ void k_body_vms(int64_t C, Elem E, const double *det, const double *Jinv, const int *cells, int dg,
                           double g0, double g1, double g2, double kmu, const double *ck, double mu, int64_t *du,
                           double *vu, int64_t *dp, double *vp) {
    const int dim = E.dim, nn = E.nn;
    const double gb[3] = {g0, g1, g2};
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C; c += (int64_t)gridDim.x * blockDim.x) {
        const double d = det[c];
        const double *Ji = Jinv + c * dim * dim;
        for (int a = 0; a < nn; ++a) {
            const int64_t node = dg ? c * nn + a : cells[c * nn + a];
            double intN = 0.0;
            for (int q = 0; q < E.nq; ++q) intN += E.w[q] * E.N[q][a];
            for (int i = 0; i < dim; ++i) {
                const int64_t k = (c * nn + a) * dim + i;
                du[k] = node * dim + i;
                vu[k] = 0.5 * d * intN * gb[i];
            }
            double s = 0.0;
            for (int q = 0; q < E.nq; ++q) {
                double ga[3];
                grad_phys(E, Ji, q, a, ga);
                double t = 0.0;
                for (int i = 0; i < dim; ++i) t += ga[i] * gb[i];
                s += E.w[q] * t;
            }
            dp[c * nn + a] = node;
            vp[c * nn + a] = (ck ? 0.5 * ck[c] / mu : kmu) * d * s;
        }
    }
}
// H(div) (assembly.py:274-276): fu[c,f] = (sum_q w_q Vphys_qf . g) det s_cf
struct HdivBody {
    int dim, nf, nq, nn, kind;
    double w[8];
    double Vref[8][6][3];
};
__global__ void k_body_hdiv(int64_t C, HdivBody B, const double *V, const double *det, const int *cells,
                            const int *cf, const signed char *cs, double g0, double g1, double g2, int64_t *du,
                            double *vu) {
    const int dim = B.dim;
    const double gb[3] = {g0, g1, g2};
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C; c += (int64_t)gridDim.x * blockDim.x) {
        double J[9];
        const int *cv = cells + c * B.nn;
        if (B.kind == DPP_TRI || B.kind == DPP_TET) {
            for (int k = 0; k < dim; ++k)
                for (int d = 0; d < dim; ++d) J[d * dim + k] = V[(int64_t)cv[k + 1] * dim + d] - V[(int64_t)cv[0] * dim + d];
        } else {
            for (int k = 0; k < dim * dim; ++k) J[k] = 0.0;
            for (int d = 0; d < dim; ++d) J[d * dim + d] = V[(int64_t)cv[B.nn - 1] * dim + d] - V[(int64_t)cv[0] * dim + d];
        }
        const double dt = det[c];
        for (int f = 0; f < B.nf; ++f) {
            double s = 0.0;
            for (int q = 0; q < B.nq; ++q) {
                double t = 0.0;
                for (int i = 0; i < dim; ++i) {
                    double v = 0.0;
                    for (int j = 0; j < dim; ++j) v += J[i * dim + j] * B.Vref[q][f][j];
                    t += (v / dt) * gb[i];
                }
                s += B.w[q] * t;
            }
            du[c * B.nf + f] = cf[c * B.nf + f];
            vu[c * B.nf + f] = s * dt * cs[c * B.nf + f];
        }
    }
}

// ------------------------------------------------------------------ strong elimination
// assembly._eliminate (assembly.py:200-226) on one block: B @ D_keep (columns of the
// pinned dofs and every exact zero dropped, as scipy's csr_matmat does), D_keep @ B
// (pinned rows dropped), and for the (field, field) block + D_pin (unit diagonal).
__global__ void k_elim_count(int rows, const int *ptr, const int *idx, const double *val, const unsigned char *pin,
                             int rowpin, int colpin, int diag, int *cnt) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
        if (rowpin && pin[r]) { cnt[r] = diag ? 1 : 0; continue; }
        int k = 0;
        for (int p = ptr[r]; p < ptr[r + 1]; ++p) k += val[p] != 0.0 && !(colpin && pin[idx[p]]);
        cnt[r] = k;
    }
}
__global__ void k_elim_fill(int rows, const int *ptr, const int *idx, const double *val, const unsigned char *pin,
                            int rowpin, int colpin, int diag, const int *optr, int *oidx, double *oval) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
        int w = optr[r];
        if (rowpin && pin[r]) {
            if (diag) { oidx[w] = r; oval[w] = 1.0; }
            continue;
        }
        for (int p = ptr[r]; p < ptr[r + 1]; ++p)
            if (val[p] != 0.0 && !(colpin && pin[idx[p]])) { oidx[w] = idx[p]; oval[w] = val[p]; ++w; }
    }
}
// rhs[r] -= B @ lift with scipy's csr_matvec order (sequential per row, no FMA), then
// numpy's elementwise subtraction: bitwise what the reference computes
__global__ void k_sub_matvec_seq(int rows, const int *ptr, const int *idx, const double *val, const double *x,
                                 double *rhs) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int p = ptr[r]; p < ptr[r + 1]; ++p) s = __dadd_rn(s, __dmul_rn(val[p], x[idx[p]]));
        rhs[r] = __dsub_rn(rhs[r], s);
    }
}
__global__ void k_scatter_vals(int64_t n, const int64_t *idx, const double *v, double *dst, unsigned char *pin) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (dst) dst[idx[i]] = v[i];
        if (pin) pin[idx[i]] = 1;
    }
}

// ------------------------------------------------------------------ drivers
static void alloc_blk(Ctx *c, Csr &B, int rows, int cols, int64_t nnz) { B.alloc(rows, cols, nnz, c->s); }

static void assemble_vms(Ctx *c, HostMesh &hm, DevMesh &m, const dpp_params &p, bool dg,
                         const dpp_bc *bc, dpp_system &S, const double *ck1 = nullptr, const double *ck2 = nullptr) {
    const Elem E = make_elem(m.kind);
    const int dim = m.dim, nn = m.nn;
    const int64_t C = m.C;
    const int64_t nodes = dg ? C * nn : m.V;
    // interior facets (DG)
    std::vector<int64_t> inter;
    if (dg)
        for (int64_t f = 0; f < hm.n_facets; ++f)
            if (hm.facet_minus[f] >= 0) inter.push_back(f);
    const int64_t Fi = (int64_t)inter.size();
    // DG prescribed-flux facets of both networks (assembly.py:519-535)
    std::vector<int> vfh;
    int64_t nv1 = 0;
    if (dg && bc) {
        for (int n = 0; n < 2; ++n) {
            for (int64_t i = 0; i < bc->n_vfacets[n]; ++i) vfh.push_back((int)bc->vfacets[n][i]);
            if (n == 0) nv1 = (int64_t)vfh.size();
        }
    }
    const int64_t nvt = (int64_t)vfh.size();
    const int64_t ncell = C * nn * nn, nfac = dg ? 4 * Fi * nn * nn : 0, nvel = nvt * nn * nn;
    const int64_t ntot = ncell + nfac + nvel;
    if (ntot > INT32_MAX) DPP_FAIL(DPP_ERR_VALUE, "mesh too large for 32-bit contribution ids");
    DBuf<uint64_t> keys(ntot, c->s);
    DBuf<int> pay(ntot, c->s);
    k_emit_cell_pairs<<<grid_for(ncell, 256, c->sms), 256, 0, c->s>>>(C, nn, m.cells.p, dg ? 1 : 0, nodes,
                                                                   keys.p, pay.p);
    launched(c);
    DBuf<int> dinter(Fi, c->s);
    DBuf<double> fW, fNp, fNm;
    FRule R2 = frule(m.kind, 2);
    if (dg && Fi) {
        std::vector<int> t(inter.begin(), inter.end());
        dinter.upload(t.data(), Fi);
        k_emit_dg_facets<<<grid_for(nfac, 256, c->sms), 256, 0, c->s>>>(Fi, nn, C, dinter.p, m.fplus.p,
                                                                     m.fminus.p, nodes, keys.p + ncell,
                                                                     pay.p + ncell);
        launched(c);
        fW.alloc(Fi * R2.nq, c->s);
        fNp.alloc(Fi * R2.nq * nn, c->s);
        fNm.alloc(Fi * R2.nq * nn, c->s);
        k_dg_facet_tables<<<grid_for(Fi * R2.nq, 128, c->sms), 128, 0, c->s>>>(
            Fi, R2, m.kind, dim, nn, m.nvf, dinter.p, m.fv.p, m.fplus.p, m.fminus.p, m.verts.p,
            m.cells.p, m.Jinv.p, m.fm.p, fW.p, fNp.p, fNm.p);
        launched(c);
        CK(cudaStreamSynchronize(c->s));
    }
    DBuf<int> dvfac(nvt, c->s);
    DBuf<double> vW, vN;
    if (nvt) {
        dvfac.upload(vfh.data(), nvt);
        k_emit_dg_vel<<<grid_for(nvel, 256, c->sms), 256, 0, c->s>>>(nvt, nn, ncell + nfac, dvfac.p, m.fplus.p, nodes,
                                                                   keys.p + ncell + nfac, pay.p + ncell + nfac);
        launched(c);
        vW.alloc(nvt * R2.nq, c->s);
        vN.alloc(nvt * R2.nq * nn, c->s);
        k_dg_facet_tables<<<grid_for(nvt * R2.nq, 128, c->sms), 128, 0, c->s>>>(
            nvt, R2, m.kind, dim, nn, m.nvf, dvfac.p, m.fv.p, m.fplus.p, m.fminus.p, m.verts.p, m.cells.p,
            m.Jinv.p, m.fm.p, vW.p, vN.p, nullptr);
        launched(c);
    }
    Graph G;
    {
        DPP_TRACE_SCOPE(c, "assemble.graph_sort");
        G = build_graph(c, keys, pay, ntot, nodes);
    }
    keys.release();
    pay.release();
    const int64_t g = G.nnz;
    const int nu = (int)(nodes * dim), np_ = (int)nodes;
    Csr *uu[2] = {&S.blk[DPP_K1_UU], &S.blk[DPP_K2_UU]}, *up[2] = {&S.blk[DPP_K1_UP], &S.blk[DPP_K2_UP]},
        *pu[2] = {&S.blk[DPP_K1_PU], &S.blk[DPP_K2_PU]}, *pp[2] = {&S.blk[DPP_K1_PP], &S.blk[DPP_K2_PP]};
    for (int n = 0; n < 2; ++n) {
        alloc_blk(c, *uu[n], nu, nu, g * dim * dim);
        alloc_blk(c, *up[n], nu, np_, g * dim);
        alloc_blk(c, *pu[n], np_, nu, g * dim);
        alloc_blk(c, *pp[n], np_, np_, g);
        k_kron_ptr<<<grid_for(nodes + 1, 256, c->sms), 256, 0, c->s>>>(nodes, dim, G.ptr.p, uu[n]->ptr.p,
                                                                     up[n]->ptr.p, pu[n]->ptr.p);
        launched(c);
        CK(cudaMemcpyAsync(pp[n]->ptr.p, G.ptr.p, sizeof(int) * (nodes + 1), cudaMemcpyDeviceToDevice, c->s));
    }
    VmsArgs A{};
    A.E = E;
    A.C = C;
    A.Fi = Fi;
    A.dg = dg;
    A.det = m.det.p;
    A.Jinv = m.Jinv.p;
    A.gptr = G.ptr.p;
    A.gcol = G.col.p;
    A.grow = G.row.p;
    A.seg = G.seg.p;
    A.pay = G.pay.p;
    A.nnz = g;
    const double ks[2] = {p.k1, p.k2};
    for (int n = 0; n < 2; ++n) {
        A.s_uu[n] = 0.5 * p.mu / ks[n];
        A.s_pp_gg[n] = 0.5 * ks[n] / p.mu;
        A.c_uu[n] = p.eta_u * (1.0 / hm.n_div) * p.mu / ks[n];
        A.c_pp[n] = p.eta_p / (1.0 / hm.n_div) * ks[n] / p.mu;
        A.uu_i[n] = uu[n]->idx.p; A.uu_v[n] = uu[n]->val.p;
        A.up_i[n] = up[n]->idx.p; A.up_v[n] = up[n]->val.p;
        A.pu_i[n] = pu[n]->idx.p; A.pu_v[n] = pu[n]->val.p;
        A.pp_i[n] = pp[n]->idx.p; A.pp_v[n] = pp[n]->val.p;
    }
    A.s_pp_m = p.beta / p.mu;
    A.s_cross = -p.beta / p.mu;
    A.mu = p.mu;
    A.ck[0] = ck1;
    A.ck[1] = ck2;
    A.interior = dinter.p;
    A.fW = fW.p;
    A.fNp = fNp.p;
    A.fNm = fNm.p;
    A.fn = m.fn.p;
    A.fnq = R2.nq;
    A.nvt = nvt;
    A.nv1 = nv1;
    A.vfac = dvfac.p;
    A.vW = vW.p;
    A.vN = vN.p;
    Csr &c12 = S.blk[DPP_K12_PP], &c21 = S.blk[DPP_K21_PP];
    if (!dg) {
        alloc_blk(c, c12, np_, np_, g);
        CK(cudaMemcpyAsync(c12.ptr.p, G.ptr.p, sizeof(int) * (nodes + 1), cudaMemcpyDeviceToDevice, c->s));
        A.cr_i = c12.idx.p;
        A.cr_v = c12.val.p;
    }
    if (E.dim == 2) k_vms_values<2><<<grid_for(g, 128, c->sms, 32), 128, 0, c->s>>>(A);
    else k_vms_values<3><<<grid_for(g, 128, c->sms, 32), 128, 0, c->s>>>(A);
    launched(c);
    if (dg) {
        alloc_blk(c, c12, np_, np_, C * nn * nn);
        k_dg_cross<<<grid_for(C * nn + 1, 128, c->sms), 128, 0, c->s>>>(C, E, m.det.p, -p.beta / p.mu,
                                                                      c12.ptr.p, c12.idx.p, c12.val.p);
        launched(c);
    }
    c21 = csr_copy(c, c12);
    if (p.gamma_b[0] != 0.0 || p.gamma_b[1] != 0.0 || (dim == 3 && p.gamma_b[2] != 0.0)) {
        // body force, np.add.at in cell order (assembly.py:395-399)
        const int64_t nu_c = C * nn * dim, np_c = C * nn;
        for (int n = 0; n < 2; ++n) {
            DBuf<int64_t> du(nu_c, c->s), dpi(np_c, c->s);
            DBuf<double> vu(nu_c, c->s), vp(np_c, c->s);
            k_body_vms<<<grid_for(C, 128, c->sms), 128, 0, c->s>>>(C, E, m.det.p, m.Jinv.p, m.cells.p, dg,
                                                                 p.gamma_b[0], p.gamma_b[1], p.gamma_b[2],
                                                                 0.5 * ks[n] / p.mu, n == 0 ? ck1 : ck2, p.mu,
                                                                 du.p, vu.p, dpi.p, vp.p);
            launched(c);
            add_at(c, nu_c, du, vu, S.rhs[n == 0 ? 0 : 2].p);
            add_at(c, np_c, dpi, vp, S.rhs[n == 0 ? 1 : 3].p);
        }
    }
    if (nvt) {   // f_p -= (u.n, q) on the prescribed-flux facets, after the body force (assembly.py:532-535)
        FRule R4 = frule(m.kind, 4);
        for (int n = 0; n < 2; ++n) {
            const int64_t nv = bc->n_vfacets[n];
            if (nv <= 0) continue;
            DBuf<int64_t> fids(nv, c->s), dof(nv * nn, c->s);
            DBuf<double> un(nv * R4.nq, c->s), val(nv * nn, c->s);
            fids.upload(bc->vfacets[n], nv);
            un.upload(bc->vdata[n], nv * R4.nq);
            k_rhs_dg_vel<<<grid_for(nv, 128, c->sms), 128, 0, c->s>>>(nv, fids.p, R4, m.kind, dim, nn, m.nvf, m.fv.p,
                                                                     m.fplus.p, m.fm.p, m.verts.p, m.cells.p, m.Jinv.p,
                                                                     un.p, dof.p, val.p);
            launched(c);
            add_at(c, nv * nn, dof, val, S.rhs[n == 0 ? 1 : 3].p);
        }
    }
    CK(cudaStreamSynchronize(c->s));
}

static void assemble_hdiv(Ctx *c, HostMesh &hm, DevMesh &m, const dpp_params &p, dpp_system &S,
                          const double *ck1 = nullptr, const double *ck2 = nullptr) {
    const int dim = m.dim, nf = m.nf;
    const int64_t C = m.C, F = m.F;
    Rule r = cell_rule(m.kind, 2);
    HdivArgs A{};
    A.dim = dim;
    A.nf = nf;
    A.nq = r.nq;
    for (int q = 0; q < r.nq; ++q) {
        A.w[q] = r.w[q];
        // elements.eval_basis flux families (elements.py:124-138)
        for (int f = 0; f < nf; ++f)
            for (int j = 0; j < dim; ++j) {
                double v;
                if (m.kind == DPP_TRI) {
                    static const double opp[3][2] = {{0.0, 1.0}, {1.0, 0.0}, {0.0, 0.0}};
                    v = r.p[q][j] - opp[f][j];
                } else if (m.kind == DPP_TET) {
                    static const double opp[4][3] = {{0, 0, 1}, {0, 1, 0}, {1, 0, 0}, {0, 0, 0}};
                    v = 2.0 * (r.p[q][j] - opp[f][j]);
                } else {
                    const int ax = f / 2;
                    v = (j != ax) ? 0.0 : ((f % 2 == 0) ? r.p[q][ax] - 1.0 : r.p[q][ax]);
                }
                A.Vref[q][f][j] = v;
            }
    }
    double ws = 0.0;
    for (int q = 0; q < r.nq; ++q) ws += r.w[q];
    A.s_uu[0] = p.mu / p.k1;
    A.s_uu[1] = p.mu / p.k2;
    A.ck[0] = ck1;
    A.ck[1] = ck2;
    A.mu = p.mu;
    A.V = m.verts.p;
    A.det = m.det.p;
    A.cells = m.cells.p;
    A.cf = m.cf.p;
    A.cs = m.cs.p;
    A.nn = m.nn;
    A.kind = m.kind;
    const int64_t ne = C * nf * nf;
    DBuf<uint64_t> keys(ne, c->s);
    DBuf<int> pay(ne, c->s);
    k_emit_cell_pairs<<<grid_for(ne, 256, c->sms), 256, 0, c->s>>>(C, nf, m.cf.p, 0, F, keys.p, pay.p);
    launched(c);
    Graph G = build_graph(c, keys, pay, ne, F);
    keys.release();
    pay.release();
    A.gptr = G.ptr.p;
    A.gcol = G.col.p;
    A.grow = G.row.p;
    A.seg = G.seg.p;
    A.pay = G.pay.p;
    A.nnz = G.nnz;
    Csr *uu[2] = {&S.blk[DPP_K1_UU], &S.blk[DPP_K2_UU]};
    for (int n = 0; n < 2; ++n) {
        alloc_blk(c, *uu[n], (int)F, (int)F, G.nnz);
        CK(cudaMemcpyAsync(uu[n]->ptr.p, G.ptr.p, sizeof(int) * (F + 1), cudaMemcpyDeviceToDevice, c->s));
        A.uu_i[n] = uu[n]->idx.p;
        A.uu_v[n] = uu[n]->val.p;
    }
    k_hdiv_uu<<<grid_for(G.nnz, 128, c->sms, 32), 128, 0, c->s>>>(A);
    launched(c);
    // up / pu / pp / cross
    Csr &up1 = S.blk[DPP_K1_UP], &pu1 = S.blk[DPP_K1_PU], &pp1 = S.blk[DPP_K1_PP], &c12 = S.blk[DPP_K12_PP];
    {
        DBuf<int> cnt(F, c->s);
        k_hdiv_up_cnt<<<grid_for(F, 256, c->sms), 256, 0, c->s>>>(F, m.fminus.p, cnt.p);
        launched(c);
        up1.rows = (int)F;
        up1.cols = (int)C;
        up1.nnz = counts_to_ptr(c, cnt.p, (int)F, up1.ptr);
        up1.idx.alloc(up1.nnz, c->s);
        up1.val.alloc(up1.nnz, c->s);
        k_hdiv_up<<<grid_for(F, 256, c->sms), 256, 0, c->s>>>(F, m.fplus.p, m.fminus.p, up1.ptr.p, up1.idx.p,
                                                           up1.val.p);
        launched(c);
    }
    alloc_blk(c, pu1, (int)C, (int)F, C * nf);
    alloc_blk(c, pp1, (int)C, (int)C, C);
    alloc_blk(c, c12, (int)C, (int)C, C);
    DBuf<double> crv(C, c->s);
    k_hdiv_rest<<<grid_for(C + 1, 256, c->sms), 256, 0, c->s>>>(
        F, C, nf, m.fplus.p, m.fminus.p, m.cf.p, m.cs.p, m.det.p, ws, p.beta / p.mu, -p.beta / p.mu,
        nullptr, nullptr, nullptr, pu1.ptr.p, pu1.idx.p, pu1.val.p, pp1.ptr.p, pp1.idx.p, pp1.val.p,
        c12.val.p);
    launched(c);
    CK(cudaMemcpyAsync(c12.ptr.p, pp1.ptr.p, sizeof(int) * (C + 1), cudaMemcpyDeviceToDevice, c->s));
    CK(cudaMemcpyAsync(c12.idx.p, pp1.idx.p, sizeof(int) * C, cudaMemcpyDeviceToDevice, c->s));
    S.blk[DPP_K2_UP] = csr_copy(c, up1);
    S.blk[DPP_K2_PU] = csr_copy(c, pu1);
    S.blk[DPP_K2_PP] = csr_copy(c, pp1);
    S.blk[DPP_K21_PP] = csr_copy(c, c12);
    if (p.gamma_b[0] != 0.0 || p.gamma_b[1] != 0.0 || (dim == 3 && p.gamma_b[2] != 0.0)) {
        // body force, np.add.at in cell order (assembly.py:274-277); same for both networks
        HdivBody B{};
        B.dim = dim; B.nf = nf; B.nq = A.nq; B.nn = m.nn; B.kind = m.kind;
        for (int q = 0; q < A.nq; ++q) {
            B.w[q] = A.w[q];
            for (int f = 0; f < nf; ++f)
                for (int j = 0; j < dim; ++j) B.Vref[q][f][j] = A.Vref[q][f][j];
        }
        for (int n = 0; n < 2; ++n) {
            DBuf<int64_t> du(C * nf, c->s);
            DBuf<double> vu(C * nf, c->s);
            k_body_hdiv<<<grid_for(C, 128, c->sms), 128, 0, c->s>>>(C, B, m.verts.p, m.det.p, m.cells.p, m.cf.p,
                                                                  m.cs.p, p.gamma_b[0], p.gamma_b[1], p.gamma_b[2],
                                                                  du.p, vu.p);
            launched(c);
            add_at(c, C * nf, du, vu, S.rhs[n == 0 ? 0 : 2].p);
        }
    }
    CK(cudaStreamSynchronize(c->s));
    (void)hm;
}

// field: 0 u1, 1 p1, 2 u2, 3 p2; idx/values host arrays (sorted dofs, as the reference's)
static const int BLK_RC[10][2] = {{0, 0}, {0, 1}, {1, 0}, {1, 1}, {2, 2}, {2, 3}, {3, 2}, {3, 3}, {1, 3}, {3, 1}};
void eliminate(Ctx *c, dpp_system &S, int field, int64_t n, const int64_t *idx_h, const double *vals_h) {
    if (n <= 0) return;
    const int64_t nf = S.sizes[field];
    for (int64_t i = 0; i < n; ++i)   // out-of-range ids would scatter out of bounds on the device
        if (idx_h[i] < 0 || idx_h[i] >= nf) DPP_FAIL(DPP_ERR_VALUE, "eliminated dof out of range");
    DBuf<int64_t> idx(n, c->s);
    DBuf<double> vals(n, c->s), lift(nf, c->s);
    DBuf<unsigned char> pin(nf, c->s);
    idx.upload(idx_h, n);
    vals.upload(vals_h, n);
    CK(cudaMemsetAsync(lift.p, 0, sizeof(double) * nf, c->s));
    CK(cudaMemsetAsync(pin.p, 0, nf, c->s));
    k_scatter_vals<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, idx.p, vals.p, lift.p, pin.p);
    launched(c);
    for (int b = 0; b < 10; ++b) {
        const int r = BLK_RC[b][0], cc = BLK_RC[b][1];
        if (r != field && cc != field) continue;
        Csr &B = S.blk[b];
        if (cc == field && B.rows) {   // rhs[r] -= B @ lift
            k_sub_matvec_seq<<<grid_for(B.rows, 256, c->sms), 256, 0, c->s>>>(B.rows, B.ptr.p, B.idx.p, B.val.p,
                                                                           lift.p, S.rhs[r].p);
            launched(c);
        }
        Csr O;
        O.rows = B.rows;
        O.cols = B.cols;
        DBuf<int> cnt(std::max(B.rows, 1), c->s);
        const int diag = r == field && cc == field;
        k_elim_count<<<grid_for(B.rows, 256, c->sms), 256, 0, c->s>>>(B.rows, B.ptr.p, B.idx.p, B.val.p, pin.p,
                                                                    r == field, cc == field, diag, cnt.p);
        launched(c);
        O.nnz = counts_to_ptr(c, cnt.p, B.rows, O.ptr);
        O.idx.alloc(std::max<int64_t>(O.nnz, 1), c->s);
        O.val.alloc(std::max<int64_t>(O.nnz, 1), c->s);
        k_elim_fill<<<grid_for(B.rows, 256, c->sms), 256, 0, c->s>>>(B.rows, B.ptr.p, B.idx.p, B.val.p, pin.p,
                                                                   r == field, cc == field, diag, O.ptr.p, O.idx.p,
                                                                   O.val.p);
        launched(c);
        B = std::move(O);
    }
    k_scatter_vals<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, idx.p, vals.p, S.rhs[field].p, nullptr);
    launched(c);
    S.hasK = false;   // the monolithic view is rebuilt from the new blocks
    CK(cudaStreamSynchronize(c->s));
}

static void boundary_rhs(Ctx *c, HostMesh &hm, DevMesh &m, int formulation, const dpp_bc *bc, dpp_system &S) {
    if (!bc) return;
    FRule R4 = frule(m.kind, 4);
    const bool dg = formulation == DPP_DGVMS;
    for (int net = 0; net < 2; ++net) {
        const int64_t nfp = bc->n_pfacets[net];
        if (nfp <= 0) continue;
        DBuf<int64_t> fids;
        if (m.facets) {
            fids.alloc(nfp, c->s);
            fids.upload(bc->pfacets[net], nfp);
            hm.bc_bytes += 8 * (size_t)nfp;
        }
        // without the mesh's facet arrays on the device (CG-VMS): the pressure facets' rows
        // (vertex ids, plus cell, normal, measure) gathered on the host, addressed 0..nfp-1
        const int *fv = m.fv.p, *fplus = m.fplus.p;
        const double *fn = m.fn.p, *fm = m.fm.p;
        const int64_t *ids = fids.p;
        DBuf<int> cfv, cfp;
        DBuf<double> cfn, cfm;
        DBuf<int64_t> iota;
        if (!m.facets) {
            const int64_t *f = bc->pfacets[net];
            const size_t bv = 4 * (size_t)nfp * m.nvf, bp = 4 * (size_t)nfp, bn = 8 * (size_t)nfp * m.dim, bm = 8 * (size_t)nfp;
            const size_t o_v = 0, o_p = (bv + 15) & ~(size_t)15, o_n = (o_p + bp + 15) & ~(size_t)15,
                         o_m = (o_n + bn + 15) & ~(size_t)15;
            // staging halves sized for the larger network's facet count
            const size_t nmax = (size_t)std::max<int64_t>(bc->n_pfacets[0], bc->n_pfacets[1]);
            const size_t tot = (16 * 4 + 4 * nmax * m.nvf + 4 * nmax + 8 * nmax * m.dim + 8 * nmax + 15) & ~(size_t)15;
            if (!hm.bc_pinned || hm.bc_pinned_bytes < 2 * tot + 64) {   // both networks' halves
                CK(cudaStreamSynchronize(c->s));   // the old staging may still be read
                void *h = nullptr;
                CK(cudaMallocHost(&h, 2 * tot + 64));
                hm.bc_pinned = std::shared_ptr<void>(h, [](void *q) { cudaFreeHost(q); });
                hm.bc_pinned_bytes = 2 * tot + 64;
            }
            // the staging may still feed a copy of an earlier assembly (one that failed before its
            // final synchronisation, or another context's): wait for its last recorded copies
            if (hm.bc_done) CK(cudaEventSynchronize(static_cast<cudaEvent_t>(hm.bc_done.get())));
            unsigned char *B = static_cast<unsigned char *>(hm.bc_pinned.get()) + (net ? hm.bc_pinned_bytes / 2 : 0);
            int *hv = reinterpret_cast<int *>(B + o_v), *hp = reinterpret_cast<int *>(B + o_p);
            double *hn = reinterpret_cast<double *>(B + o_n), *hmz = reinterpret_cast<double *>(B + o_m);
            for (int64_t i = 0; i < nfp; ++i) {
                const int64_t g = f[i];
                if (g < 0 || g >= m.F) DPP_FAIL(DPP_ERR_VALUE, "pressure facet id out of range");
                for (int k = 0; k < m.nvf; ++k) hv[(size_t)i * m.nvf + k] = (int)hm.facet_vertex_ids[(size_t)g * m.nvf + k];
                hp[i] = (int)hm.facet_plus[g];
                for (int k = 0; k < m.dim; ++k) hn[(size_t)i * m.dim + k] = hm.facet_normals[(size_t)g * m.dim + k];
                hmz[i] = hm.facet_measures[g];
            }
            // asynchronous copies; the next fill of the staging waits on bc_done
            cfv.alloc((size_t)nfp * m.nvf, c->s);
            cfp.alloc(nfp, c->s);
            cfn.alloc((size_t)nfp * m.dim, c->s);
            cfm.alloc(nfp, c->s);
            CK(cudaMemcpyAsync(cfv.p, hv, bv, cudaMemcpyHostToDevice, c->s));
            CK(cudaMemcpyAsync(cfp.p, hp, bp, cudaMemcpyHostToDevice, c->s));
            CK(cudaMemcpyAsync(cfn.p, hn, bn, cudaMemcpyHostToDevice, c->s));
            CK(cudaMemcpyAsync(cfm.p, hmz, bm, cudaMemcpyHostToDevice, c->s));
            if (!hm.bc_done) {
                cudaEvent_t ev;
                CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                hm.bc_done = std::shared_ptr<void>(ev, [](void *q) { cudaEventDestroy(static_cast<cudaEvent_t>(q)); });
            }
            CK(cudaEventRecord(static_cast<cudaEvent_t>(hm.bc_done.get()), c->s));
            hm.bc_bytes += bv + bp + bn + bm;
            iota.alloc(nfp, c->s);
            k_iota64<<<grid_for(nfp, 256, c->sms), 256, 0, c->s>>>(nfp, iota.p);
            launched(c);
            fv = cfv.p; fplus = cfp.p; fn = cfn.p; fm = cfm.p; ids = iota.p;
        }
        DBuf<double> p0(nfp * R4.nq, c->s);
        if (bc->p0_kind[net]) {
            const double *cf = bc->p0_coef[net];
            k_mms_p0<<<grid_for(nfp * R4.nq, 256, c->sms), 256, 0, c->s>>>(nfp, ids, R4, m.dim, m.nvf, fv, m.verts.p,
                                                                        bc->p0_kind[net], cf[0], cf[1], cf[2], p0.p);
            launched(c);
        } else {
            p0.upload(bc->p0[net], nfp * R4.nq);
            hm.bc_bytes += 8 * (size_t)nfp * R4.nq;
        }
        double *rhs = S.rhs[net == 0 ? 0 : 2].p;
        if (formulation == DPP_HDIV) {
            DBuf<int64_t> dof(nfp, c->s);
            DBuf<double> val(nfp, c->s);
            k_rhs_hdiv<<<grid_for(nfp, 256, c->sms), 256, 0, c->s>>>(nfp, ids, R4, fm, p0.p, dof.p, val.p);
            launched(c);
            add_at(c, nfp, dof, val, rhs);
        } else {
            const int64_t ne = nfp * m.nn * m.dim;
            DBuf<int64_t> dof(ne, c->s);
            DBuf<double> val(ne, c->s);
            k_rhs_nodal<<<grid_for(nfp, 128, c->sms), 128, 0, c->s>>>(
                nfp, ids, R4, m.kind, m.dim, m.nn, m.nvf, dg, fv, fplus, fn, fm,
                m.verts.p, m.cells.p, m.Jinv.p, p0.p, dof.p, val.p);
            launched(c);
            add_at(c, ne, dof, val, rhs);
        }
    }
}

}  // namespace dpp

// ------------------------------------------------------------------ C ABI
using namespace dpp;



extern "C" {

int dpp_mesh_generate(int dim, int kind, int n_div, dpp_mesh **out) {
    return guard([&] {
        try {
            auto *h = new dpp_mesh;
            h->m = generate(dim, kind, n_div);
            *out = h;
        } catch (const std::invalid_argument &e) {
            DPP_FAIL(DPP_ERR_VALUE, e.what());
        }
    });
}

int dpp_mesh_from_arrays(int dim, int kind, int n_div, int64_t nv, const double *vertices, int64_t nc,
                         const int64_t *cells, dpp_mesh **out) {
    return guard([&] {
        if (kind < 0 || kind > 3 || kind_dim(kind) != dim) DPP_FAIL(DPP_ERR_VALUE, "cell kind / dim mismatch");
        auto *h = new dpp_mesh;
        h->m.dim = dim;
        h->m.kind = kind;
        h->m.n_div = n_div;
        h->m.n_vertices = nv;
        h->m.n_cells = nc;
        h->m.vertices.assign(vertices, vertices + nv * dim);
        h->m.cells.assign(cells, cells + nc * kind_nodes(kind));
        for (int64_t v : h->m.cells)
            if (v < 0 || v >= nv) { delete h; DPP_FAIL(DPP_ERR_VALUE, "cell vertex id out of range"); }
        try {
            h->m.build();
        } catch (const std::runtime_error &e) {
            delete h;
            DPP_FAIL(DPP_ERR_VALUE, e.what());
        }
        *out = h;
    });
}

int dpp_mesh_counts(const dpp_mesh *m, int64_t *nv, int64_t *nc, int64_t *nf) {
    return guard([&] {
        if (nv) *nv = m->m.n_vertices;
        if (nc) *nc = m->m.n_cells;
        if (nf) *nf = m->m.n_facets;
    });
}

int dpp_mesh_export(const dpp_mesh *mm, double *vertices, int64_t *cells, int64_t *fvi, int64_t *cf,
                    int8_t *cs, int64_t *fp, int64_t *fmi, double *fn, double *fms, double *J, double *det) {
    return guard([&] {
        const HostMesh &m = mm->m;
        auto cp = [](auto *dst, const auto &v) {
            if (dst) std::copy(v.begin(), v.end(), dst);
        };
        cp(vertices, m.vertices);
        cp(cells, m.cells);
        cp(fvi, m.facet_vertex_ids);
        cp(cf, m.cell_facets);
        cp(cs, m.cell_facet_signs);
        cp(fp, m.facet_plus);
        cp(fmi, m.facet_minus);
        cp(fn, m.facet_normals);
        cp(fms, m.facet_measures);
        cp(J, m.J);
        cp(det, m.det);
    });
}

int dpp_mesh_destroy(dpp_mesh *m) {
    return guard([&] { delete m; });
}

int dpp_mesh_upload_bytes(dpp_mesh *m, int64_t *bytes) {
    return guard([&] {
        // what the current device image actually copied (the facet arrays only when a
        // formulation needed them) plus the last assembly's compact boundary-facet data
        const HostMesh &h = m->m;
        *bytes = (int64_t)(h.dev_bytes + h.bc_bytes);
    });
}

int dpp_mesh_release_device(dpp_mesh *m) {
    return guard([&] { m->m.dev.reset(); });
}

int dpp_facet_rule_size(int dim, int kind, int degree, int *nq) {
    return guard([&] {
        if (kind_dim(kind) != dim) DPP_FAIL(DPP_ERR_VALUE, "cell kind / dim mismatch");
        *nq = frule(kind, degree).nq;
    });
}

int dpp_facet_points(dpp_ctx *ctx, dpp_mesh *mm, int degree, int64_t nf, const int64_t *facets,
                     double *X, double *W) {
    return guard([&] {
        Ctx *c = &ctx->c;
        for (int64_t i = 0; i < nf; ++i)
            if (facets[i] < 0 || facets[i] >= mm->m.n_facets) DPP_FAIL(DPP_ERR_VALUE, "facet id out of range");
        DevMesh &m = dev_mesh(c, mm->m);
        ensure_facets(c, mm->m, m);
        FRule R = frule(m.kind, degree);
        if (nf <= 0) return;
        DBuf<int64_t> f(nf, c->s);
        f.upload(facets, nf);
        DBuf<double> dX(nf * R.nq * m.dim, c->s), dW(nf * R.nq, c->s);
        k_facet_points<<<grid_for(nf * R.nq, 256, c->sms), 256, 0, c->s>>>(nf, f.p, R, m.dim, m.nvf, m.fv.p,
                                                                        m.verts.p, m.fm.p, dX.p, dW.p);
        launched(c);
        if (X) dX.download(X, nf * R.nq * m.dim);
        if (W) dW.download(W, nf * R.nq);
        CK(cudaStreamSynchronize(c->s));
    });
}

int dpp_system_eliminate(dpp_system *s, int field, int64_t n, const int64_t *idx, const double *values) {
    return guard([&] {
        if (field < 0 || field > 3) DPP_FAIL(DPP_ERR_VALUE, "field must be 0..3 (u1, p1, u2, p2)");
        for (int64_t i = 0; i < n; ++i)
            if (idx[i] < 0 || idx[i] >= s->sizes[field]) DPP_FAIL(DPP_ERR_VALUE, "eliminated dof out of range");
        eliminate(s->ctx, *s, field, n, idx, values);
    });
}

int dpp_assemble(dpp_ctx *ctx, dpp_mesh *mm, int formulation, const dpp_params *p, const dpp_bc *bc,
                 dpp_system **out) {
    return dpp_assemble_ext(ctx, mm, formulation, p, nullptr, nullptr, bc, out);
}

int dpp_assemble_ext(dpp_ctx *ctx, dpp_mesh *mm, int formulation, const dpp_params *p, const double *cell_k1,
                     const double *cell_k2, const dpp_bc *bc, dpp_system **out) {
    return guard([&] {
        const auto t0 = std::chrono::steady_clock::now();
        Ctx *c = &ctx->c;
        HostMesh &hm = mm->m;
        if (p->mu <= 0 || p->k1 <= 0 || p->k2 <= 0) DPP_FAIL(DPP_ERR_VALUE, "mu, k1, k2 must be positive");
        if (bc)   // every boundary facet id is checked on the host before anything reaches the device
            for (int n = 0; n < 2; ++n) {
                if (bc->n_pfacets[n] < 0 || bc->n_vfacets[n] < 0) DPP_FAIL(DPP_ERR_VALUE, "negative facet count");
                if (bc->n_pfacets[n] && !bc->pfacets[n]) DPP_FAIL(DPP_ERR_VALUE, "pressure facets missing");
                if (bc->n_vfacets[n] && (!bc->vfacets[n] || !bc->vdata[n])) DPP_FAIL(DPP_ERR_VALUE, "velocity facets missing");
                for (int64_t i = 0; i < bc->n_pfacets[n]; ++i)
                    if (bc->pfacets[n][i] < 0 || bc->pfacets[n][i] >= hm.n_facets)
                        DPP_FAIL(DPP_ERR_VALUE, "pressure facet id out of range");
                for (int64_t i = 0; i < bc->n_vfacets[n]; ++i)
                    if (bc->vfacets[n][i] < 0 || bc->vfacets[n][i] >= hm.n_facets)
                        DPP_FAIL(DPP_ERR_VALUE, "velocity facet id out of range");
            }
        DPP_TRACE_SCOPE(c, "assemble.total");
        if ((cell_k1 == nullptr) != (cell_k2 == nullptr)) DPP_FAIL(DPP_ERR_VALUE, "give both cell_k1 and cell_k2 or neither");
        if (cell_k1 && formulation == DPP_DGVMS)
            DPP_FAIL(DPP_ERR_VALUE, "per-cell permeability is implemented for H(div) and CG-VMS");
        if (cell_k1)
            for (int64_t i = 0; i < hm.n_cells; ++i)
                if (!(cell_k1[i] > 0) || !(cell_k2[i] > 0)) DPP_FAIL(DPP_ERR_VALUE, "cell permeabilities must be positive");
        DevMesh *mp;
        {
            DPP_TRACE_SCOPE(c, "assemble.mesh_upload");
            mp = &dev_mesh(c, hm);
        }
        DevMesh &m = *mp;
        if (m.C) {   // cell geometry, inside the assembly's own timing
            k_geom<<<grid_for(m.C, 128, c->sms), 128, 0, c->s>>>(m.C, m.dim, m.kind, m.nn, m.verts.p, m.cells.p, m.Jinv.p);
            launched(c);
        }
        auto S = std::make_unique<dpp_system>();
        S->ctx = c;
        if (formulation == DPP_HDIV) {
            S->sizes[0] = S->sizes[2] = m.F;
            S->sizes[1] = S->sizes[3] = m.C;
        } else if (formulation == DPP_CGVMS) {
            S->sizes[0] = S->sizes[2] = m.V * m.dim;
            S->sizes[1] = S->sizes[3] = m.V;
        } else if (formulation == DPP_DGVMS) {
            S->sizes[1] = S->sizes[3] = m.C * m.nn;
            S->sizes[0] = S->sizes[2] = m.C * m.nn * m.dim;
        } else {
            DPP_FAIL(DPP_ERR_VALUE, "unknown formulation");
        }
        for (int k = 0; k < 4; ++k) {
            S->rhs[k].alloc(S->sizes[k], c->s);
            if (S->sizes[k]) CK(cudaMemsetAsync(S->rhs[k].p, 0, sizeof(double) * S->sizes[k], c->s));
        }
        hm.bc_bytes = 0;
        if (formulation != DPP_CGVMS || (bc && (bc->n_vfacets[0] > 0 || bc->n_vfacets[1] > 0)))
            ensure_facets(c, hm, m);
        {
            DPP_TRACE_SCOPE(c, "assemble.blocks");
            DBuf<double> ck1, ck2;   // per-cell permeabilities (config-3 extension)
            if (cell_k1) {
                ck1.alloc(hm.n_cells, c->s);
                ck2.alloc(hm.n_cells, c->s);
                ck1.upload(cell_k1, hm.n_cells);
                ck2.upload(cell_k2, hm.n_cells);
            }
            if (formulation == DPP_HDIV) assemble_hdiv(c, hm, m, *p, *S, ck1.p, ck2.p);
            else assemble_vms(c, hm, m, *p, formulation == DPP_DGVMS, bc, *S, ck1.p, ck2.p);
            CK(cudaStreamSynchronize(c->s));
        }
        {
            DPP_TRACE_SCOPE(c, "assemble.rhs");
            boundary_rhs(c, hm, m, formulation, bc, *S);
            // H(div) prescribed flux: strong elimination of the facet dofs (assembly.py:301-309);
            // CG-VMS velocity facets only drop the pressure functional (the caller's pfacets)
            if (bc && formulation == DPP_HDIV)
                for (int n = 0; n < 2; ++n)
                    if (bc->n_vfacets[n] > 0)
                        eliminate(c, *S, n == 0 ? 0 : 2, bc->n_vfacets[n], bc->vfacets[n], bc->vdata[n]);
        }
        CK(cudaStreamSynchronize(c->s));
        S->assembly_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        *out = S.release();
    });
}

}  // extern "C"
