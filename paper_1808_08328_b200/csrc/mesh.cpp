// Structured unit-square / unit-cube meshes with facet tables (host C++).
//
// Reference: mesh.generate_unit_mesh / Mesh._build_facets / _facet_geometry /
// jacobians (mesh.py:80-277).  Numbering contracts (bit-exact):
//   vertex id 2D j*(n+1)+i, 3D (k*(n+1)+j)*(n+1)+i, coordinates linspace(0,1,n+1)
//   (x_i = i*(1/n), last = 1.0); TRI cells (v00,v10,v11),(v00,v11,v01); QUAD/HEX
//   tensor order; TET = 6 Kuhn tets per cube from the axis permutations in
//   lexicographic order, v1<->v2 swapped for odd permutations;
//   facets = sorted unique sorted-vertex tuples, plus = lower cell id,
//   cell_facet_signs +1 for plus / -1 for minus, normal outward from plus.
// det J follows numpy.linalg.det (LAPACK getrf with reciprocal pivot scaling,
// then sign * exp(sum log|u_ii|)) so that it matches the reference bitwise on
// structured meshes; the facet sort is a plain std::sort (mesh generation is
// outside the reference's timed region, spectrum.py:224-242).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/dpp.h"
#include "mesh.h"

namespace dpp {

static const int LOCAL_FACETS_TRI[3][2] = {{0, 1}, {0, 2}, {1, 2}};
static const int LOCAL_FACETS_QUAD[4][2] = {{0, 2}, {1, 3}, {0, 1}, {2, 3}};
static const int LOCAL_FACETS_TET[4][3] = {{0, 1, 2}, {0, 1, 3}, {0, 2, 3}, {1, 2, 3}};
static const int LOCAL_FACETS_HEX[6][4] = {{0, 2, 4, 6}, {1, 3, 5, 7}, {0, 1, 4, 5},
                                           {2, 3, 6, 7}, {0, 1, 2, 3}, {4, 5, 6, 7}};

int kind_dim(int kind) { return kind == DPP_TRI || kind == DPP_QUAD ? 2 : 3; }
int kind_nodes(int kind) { return kind == DPP_TRI ? 3 : kind == DPP_HEX ? 8 : 4; }
int kind_facets(int kind) { return kind == DPP_TRI ? 3 : kind == DPP_HEX ? 6 : 4; }
int kind_facet_nodes(int kind) { return kind == DPP_TRI || kind == DPP_QUAD ? 2 : kind == DPP_TET ? 3 : 4; }
int local_facet(int kind, int f, int k) {
    switch (kind) {
        case DPP_TRI: return LOCAL_FACETS_TRI[f][k];
        case DPP_QUAD: return LOCAL_FACETS_QUAD[f][k];
        case DPP_TET: return LOCAL_FACETS_TET[f][k];
        default: return LOCAL_FACETS_HEX[f][k];
    }
}

// numpy.linalg.det of a small matrix (row-major, modified in place)
double np_det(double *a, int d) {
    double sign = 1.0;
    for (int k = 0; k < d; ++k) {
        int p = k;
        double best = std::fabs(a[k * d + k]);
        for (int r = k + 1; r < d; ++r)
            if (std::fabs(a[r * d + k]) > best) { best = std::fabs(a[r * d + k]); p = r; }
        if (p != k) {
            for (int c = 0; c < d; ++c) std::swap(a[k * d + c], a[p * d + c]);
            sign = -sign;
        }
        const double piv = a[k * d + k];
        if (piv == 0.0) return 0.0;
        const double rp = 1.0 / piv;
        for (int r = k + 1; r < d; ++r) {
            const double l = a[r * d + k] * rp;
            a[r * d + k] = l;
            for (int c = k + 1; c < d; ++c) a[r * d + c] = a[r * d + c] - l * a[k * d + c];
        }
    }
    double logdet = 0.0;
    for (int k = 0; k < d; ++k) {
        double u = a[k * d + k];
        if (u < 0) { sign = -sign; u = -u; }
        logdet += std::log(u);
    }
    return sign * std::exp(logdet);
}

void HostMesh::build() {
    const int nvf = kind_facet_nodes(kind), nf = kind_facets(kind), nv = kind_nodes(kind);
    const int64_t C = n_cells;
    // --- facets: sort (sorted vertex tuple, cell, local facet)
    struct Ent { int64_t k[4]; int64_t cell; int loc; };
    std::vector<Ent> ents((size_t)C * nf);
    for (int64_t c = 0; c < C; ++c)
        for (int f = 0; f < nf; ++f) {
            Ent &e = ents[(size_t)c * nf + f];
            for (int k = 0; k < 4; ++k) e.k[k] = k < nvf ? cells[c * nv + local_facet(kind, f, k)] : 0;
            std::sort(e.k, e.k + nvf);
            e.cell = c;
            e.loc = f;
        }
    std::vector<int64_t> order(ents.size());
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int64_t x, int64_t y) {
        const Ent &a = ents[x], &b = ents[y];
        for (int k = 0; k < nvf; ++k)
            if (a.k[k] != b.k[k]) return a.k[k] < b.k[k];
        if (a.cell != b.cell) return a.cell < b.cell;
        return a.loc < b.loc;
    });
    cell_facets.assign((size_t)C * nf, -1);
    cell_facet_signs.assign((size_t)C * nf, 0);
    facet_vertex_ids.clear();
    facet_plus.clear();
    facet_minus.clear();
    size_t i = 0;
    int64_t fid = 0;
    while (i < order.size()) {
        size_t j = i + 1;
        const Ent &a = ents[order[i]];
        while (j < order.size() && std::equal(a.k, a.k + nvf, ents[order[j]].k)) ++j;
        if (j - i > 2) throw std::runtime_error("facet shared by more than two cells");
        for (int k = 0; k < nvf; ++k) facet_vertex_ids.push_back(a.k[k]);
        facet_plus.push_back(a.cell);
        cell_facets[a.cell * nf + a.loc] = fid;
        cell_facet_signs[a.cell * nf + a.loc] = 1;
        if (j - i == 2) {
            const Ent &b = ents[order[i + 1]];
            facet_minus.push_back(b.cell);
            cell_facets[b.cell * nf + b.loc] = fid;
            cell_facet_signs[b.cell * nf + b.loc] = -1;
        } else {
            facet_minus.push_back(-1);
        }
        ++fid;
        i = j;
    }
    n_facets = fid;
    // --- facet geometry (mesh.py:145-167)
    facet_normals.assign((size_t)n_facets * dim, 0.0);
    facet_measures.assign((size_t)n_facets, 0.0);
    for (int64_t f = 0; f < n_facets; ++f) {
        const int64_t *vid = &facet_vertex_ids[(size_t)f * nvf];
        double p[4][3] = {};
        for (int k = 0; k < nvf; ++k)
            for (int d = 0; d < dim; ++d) p[k][d] = vertices[vid[k] * dim + d];
        double ctr[3] = {0, 0, 0}, cc[3] = {0, 0, 0}, nrm[3] = {0, 0, 0}, meas;
        for (int d = 0; d < dim; ++d) {
            double s = p[0][d];
            for (int k = 1; k < nvf; ++k) s += p[k][d];
            ctr[d] = s / nvf;
        }
        if (dim == 2) {
            const double t0 = p[1][0] - p[0][0], t1 = p[1][1] - p[0][1];
            meas = std::sqrt(t0 * t0 + t1 * t1);
            nrm[0] = t1 / meas;
            nrm[1] = -t0 / meas;
        } else {
            double a[3], b[3];
            for (int d = 0; d < 3; ++d) { a[d] = p[1][d] - p[0][d]; b[d] = p[2][d] - p[0][d]; }
            const double cr[3] = {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
            const double a2 = std::sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
            for (int d = 0; d < 3; ++d) nrm[d] = cr[d] / a2;
            meas = nvf == 3 ? 0.5 * a2 : a2;
        }
        const int64_t pc = facet_plus[f];
        for (int d = 0; d < dim; ++d) {
            double s = vertices[cells[pc * nv] * dim + d];
            for (int k = 1; k < nv; ++k) s += vertices[cells[pc * nv + k] * dim + d];
            cc[d] = s / nv;
        }
        double dot = 0;
        for (int d = 0; d < dim; ++d) dot += nrm[d] * (ctr[d] - cc[d]);
        if (dot < 0)
            for (int d = 0; d < dim; ++d) nrm[d] = -nrm[d];
        for (int d = 0; d < dim; ++d) facet_normals[f * dim + d] = nrm[d];
        facet_measures[f] = meas;
    }
    // --- Jacobians and numpy-faithful determinants (mesh.py:171-185)
    J.assign((size_t)C * dim * dim, 0.0);
    det.assign((size_t)C, 0.0);
    for (int64_t c = 0; c < C; ++c) {
        double *Jc = &J[(size_t)c * dim * dim];
        const int64_t *cv = &cells[c * nv];
        if (kind == DPP_TRI || kind == DPP_TET) {
            for (int k = 0; k < dim; ++k)
                for (int d = 0; d < dim; ++d)
                    Jc[d * dim + k] = vertices[cv[k + 1] * dim + d] - vertices[cv[0] * dim + d];
        } else {
            for (int d = 0; d < dim; ++d) Jc[d * dim + d] = vertices[cv[nv - 1] * dim + d] - vertices[cv[0] * dim + d];
        }
        double a[9];
        std::copy(Jc, Jc + dim * dim, a);
        det[c] = np_det(a, dim);
    }
}

HostMesh generate(int dim, int kind, int n) {
    if (n < 1) throw std::invalid_argument("n_div must be a positive integer");
    if (kind < 0 || kind > 3) throw std::invalid_argument("unknown cell kind");
    if (kind_dim(kind) != dim) throw std::invalid_argument("cell kind / dim mismatch");
    HostMesh m;
    m.dim = dim;
    m.kind = kind;
    m.n_div = n;
    const int64_t w = n + 1;
    const double step = 1.0 / n;
    std::vector<double> xs(w);
    for (int64_t i = 0; i < w; ++i) xs[i] = (double)i * step + 0.0;
    xs[n] = 1.0;
    const int nv = kind_nodes(kind);
    if (dim == 2) {
        m.n_vertices = w * w;
        m.vertices.resize((size_t)m.n_vertices * 2);
        for (int64_t j = 0; j < w; ++j)
            for (int64_t i = 0; i < w; ++i) {
                m.vertices[(j * w + i) * 2] = xs[i];
                m.vertices[(j * w + i) * 2 + 1] = xs[j];
            }
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < n; ++i) {
                const int64_t v00 = j * w + i, v10 = v00 + 1, v01 = v00 + w, v11 = v01 + 1;
                if (kind == DPP_QUAD) {
                    for (int64_t v : {v00, v10, v01, v11}) m.cells.push_back(v);
                } else {
                    for (int64_t v : {v00, v10, v11, v00, v11, v01}) m.cells.push_back(v);
                }
            }
    } else {
        m.n_vertices = w * w * w;
        m.vertices.resize((size_t)m.n_vertices * 3);
        for (int64_t k = 0; k < w; ++k)
            for (int64_t j = 0; j < w; ++j)
                for (int64_t i = 0; i < w; ++i) {
                    const int64_t v = (k * w + j) * w + i;
                    m.vertices[v * 3] = xs[i];
                    m.vertices[v * 3 + 1] = xs[j];
                    m.vertices[v * 3 + 2] = xs[k];
                }
        auto vid = [&](int64_t i, int64_t j, int64_t k) { return (k * w + j) * w + i; };
        static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
        static const int odd[6] = {0, 1, 1, 0, 0, 1};
        for (int64_t k = 0; k < n; ++k)
            for (int64_t j = 0; j < n; ++j)
                for (int64_t i = 0; i < n; ++i) {
                    if (kind == DPP_HEX) {
                        for (int dk = 0; dk < 2; ++dk)
                            for (int dj = 0; dj < 2; ++dj)
                                for (int di = 0; di < 2; ++di) m.cells.push_back(vid(i + di, j + dj, k + dk));
                        continue;
                    }
                    for (int p = 0; p < 6; ++p) {
                        int64_t pos[3] = {i, j, k};
                        int64_t t[4];
                        t[0] = vid(pos[0], pos[1], pos[2]);
                        for (int s = 0; s < 3; ++s) {
                            pos[perms[p][s]] += 1;
                            t[s + 1] = vid(pos[0], pos[1], pos[2]);
                        }
                        if (odd[p]) std::swap(t[1], t[2]);
                        for (int s = 0; s < 4; ++s) m.cells.push_back(t[s]);
                    }
                }
    }
    m.n_cells = (int64_t)m.cells.size() / nv;
    m.build();
    for (double d : m.det)
        if (d <= 0) throw std::runtime_error("mesh generation produced an inverted cell");
    return m;
}

}  // namespace dpp
