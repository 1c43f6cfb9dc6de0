// Structured unit-square / unit-cube meshes generated in HBM.
//
// Reference: mesh.generate_unit_mesh / Mesh._build_facets / _facet_geometry / jacobians
// (mesh.py:106-277); same numbering contracts as the host builder (mesh.cpp), bit for bit:
//   vertices    x_i = i * (1/n) with x_n = 1.0 (numpy.linspace), id (k*(n+1)+j)*(n+1)+i
//   cells       TRI (v00,v10,v11),(v00,v11,v01); QUAD / HEX tensor order; TET = 6 Kuhn
//               tetrahedra per cube, v1<->v2 swapped for odd axis permutations
//   facets      unique sorted-vertex tuples in lexicographic order: one or two stable radix
//               sorts of packed (vertex id) keys over the C*nf (cell, local facet) entries in
//               (cell, local) order, so the first entry of a group is the lower cell = plus
//   geometry    the host's expression order with explicit round-to-nearest operations (this
//               file is also compiled with --fmad=false)
//   det J       numpy.linalg.det goes through log / exp, whose device versions round differently
//               from glibc's: on a structured mesh J depends only on the cell's position in its
//               cube (p) and on the grid spacings h_i = x_{i+1} - x_i along its axes, which take
//               a handful of bit-distinct values; the host evaluates np_det once per
//               (p, class(h_i), class(h_j), class(h_k)) and the cells look their value up.
// The host arrays of the mesh object (dpp_mesh_export, boundary queries) are read back from the
// device image; no host numbering runs.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "devmesh.cuh"

namespace dpp {

struct MeshTab {
    int lf[6][4];      // local facet -> local vertices
    int perm[6][3];    // Kuhn axis permutations, lexicographic
    int odd[6];
};
static MeshTab mesh_tab(int kind) {
    MeshTab t{};
    const int nf = kind_facets(kind), nvf = kind_facet_nodes(kind);
    for (int f = 0; f < nf; ++f)
        for (int k = 0; k < nvf; ++k) t.lf[f][k] = local_facet(kind, f, k);
    const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    const int odd[6] = {0, 1, 1, 0, 0, 1};
    for (int p = 0; p < 6; ++p) {
        for (int s = 0; s < 3; ++s) t.perm[p][s] = perms[p][s];
        t.odd[p] = odd[p];
    }
    return t;
}

#define GRID_STRIDE(i, n) \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

__global__ void k_mesh_vertices(int64_t V, int dim, int n, double step, double *X) {
    const int64_t w = n + 1;
    GRID_STRIDE(v, V) {
        int64_t r = v;
        for (int d = 0; d < dim; ++d) {
            const int64_t i = r % w;
            r /= w;
            X[v * dim + d] = i == n ? 1.0 : __dmul_rn((double)i, step);
        }
    }
}

// the vertices of cell c (and its cube position / sub-cell index)
__device__ __forceinline__ void cell_vertices(int64_t c, int kind, int n, const MeshTab &T, int *v, int *ijk, int *sub) {
    const int64_t w = n + 1;
    if (kind == DPP_TRI || kind == DPP_QUAD) {
        const int per = kind == DPP_TRI ? 2 : 1;
        const int64_t q = c / per;
        const int t = (int)(c % per);
        const int i = (int)(q % n), j = (int)(q / n);
        const int v00 = (int)(j * w + i), v10 = v00 + 1, v01 = v00 + (int)w, v11 = v01 + 1;
        ijk[0] = i; ijk[1] = j; ijk[2] = 0;
        *sub = t;
        if (kind == DPP_QUAD) { v[0] = v00; v[1] = v10; v[2] = v01; v[3] = v11; }
        else if (t == 0) { v[0] = v00; v[1] = v10; v[2] = v11; }
        else { v[0] = v00; v[1] = v11; v[2] = v01; }
        return;
    }
    const int per = kind == DPP_TET ? 6 : 1;
    const int64_t q = c / per;
    const int p = (int)(c % per);
    const int i = (int)(q % n), j = (int)((q / n) % n), k = (int)(q / ((int64_t)n * n));
    ijk[0] = i; ijk[1] = j; ijk[2] = k;
    *sub = p;
    if (kind == DPP_HEX) {
        for (int a = 0; a < 8; ++a)
            v[a] = (int)(((k + (a >> 2)) * w + (j + ((a >> 1) & 1))) * w + (i + (a & 1)));
        return;
    }
    int pos[3] = {i, j, k};
    v[0] = (int)((pos[2] * w + pos[1]) * w + pos[0]);
    for (int s = 0; s < 3; ++s) {
        pos[T.perm[p][s]] += 1;
        v[s + 1] = (int)((pos[2] * w + pos[1]) * w + pos[0]);
    }
    if (T.odd[p]) { const int t = v[1]; v[1] = v[2]; v[2] = t; }
}

// cells, J (mesh.py:175-183) and det J (class table, see the header)
__global__ void k_mesh_cells(int64_t C, int kind, int dim, int nn, int n, MeshTab T, const double *X,
                             const int *cls, int ncls, const double *dettab, int *cells, double *J, double *det) {
    GRID_STRIDE(c, C) {
        int v[8], ijk[3], sub;
        cell_vertices(c, kind, n, T, v, ijk, &sub);
        for (int a = 0; a < nn; ++a) cells[c * nn + a] = v[a];
        double *Jc = J + c * dim * dim;
        for (int a = 0; a < dim * dim; ++a) Jc[a] = 0.0;
        if (kind == DPP_TRI || kind == DPP_TET) {
            for (int k = 0; k < dim; ++k)
                for (int d = 0; d < dim; ++d)
                    Jc[d * dim + k] = __dsub_rn(X[(int64_t)v[k + 1] * dim + d], X[(int64_t)v[0] * dim + d]);
        } else {
            for (int d = 0; d < dim; ++d)
                Jc[d * dim + d] = __dsub_rn(X[(int64_t)v[nn - 1] * dim + d], X[(int64_t)v[0] * dim + d]);
        }
        int64_t t = sub;
        for (int d = 0; d < dim; ++d) t = t * ncls + cls[ijk[d]];
        det[c] = dettab[t];
    }
}

// packed sorted-vertex keys of entry e = cell * nf + local facet: hi = the first two ids (or all
// of them when nvf * vb <= 64), lo = the rest
__global__ void k_facet_keys(int64_t E, int nf, int nvf, int nn, int vb, int single, MeshTab T, const int *cells,
                             uint64_t *hi, uint64_t *lo, int *ent) {
    GRID_STRIDE(e, E) {
        const int64_t c = e / nf;
        const int f = (int)(e % nf);
        uint64_t k[4];
        for (int a = 0; a < nvf; ++a) k[a] = (uint64_t)cells[c * nn + T.lf[f][a]];
        for (int a = 1; a < nvf; ++a)   // insertion sort of <= 4 ids
            for (int b = a; b > 0 && k[b - 1] > k[b]; --b) { const uint64_t t = k[b]; k[b] = k[b - 1]; k[b - 1] = t; }
        uint64_t h = 0, l = 0;
        if (single) {
            for (int a = 0; a < nvf; ++a) h = (h << vb) | k[a];
        } else {
            h = (k[0] << vb) | k[1];
            for (int a = 2; a < nvf; ++a) l = (l << vb) | k[a];
        }
        hi[e] = h;
        if (lo) lo[e] = l;
        ent[e] = (int)e;
    }
}

__global__ void k_gather_u64(int64_t n, const int *idx, const uint64_t *src, uint64_t *dst, int *iota) {
    GRID_STRIDE(i, n) { dst[i] = src[idx[i]]; iota[i] = (int)i; }
}
__global__ void k_gather_fin(int64_t n, const int *idx, const uint64_t *lo_s, const int *ent_s, uint64_t *lo, int *ent) {
    GRID_STRIDE(i, n) { lo[i] = lo_s[idx[i]]; ent[i] = ent_s[idx[i]]; }
}

// head[i] = 1 where a new facet starts; bad = 1 when three consecutive entries share a tuple
__global__ void k_facet_heads(int64_t E, const uint64_t *hi, const uint64_t *lo, int *head, int *bad) {
    GRID_STRIDE(i, E) {
        const bool same1 = i > 0 && hi[i] == hi[i - 1] && (!lo || lo[i] == lo[i - 1]);
        head[i] = same1 ? 0 : 1;
        if (same1 && i > 1 && hi[i] == hi[i - 2] && (!lo || lo[i] == lo[i - 2])) *bad = 1;
    }
}

__global__ void k_facet_scatter(int64_t E, int nf, int nvf, int vb, int single, const uint64_t *hi, const uint64_t *lo,
                                const int *ent, const int *head, const int *fid1, int *cf, signed char *cs,
                                int *fv, int *fplus, int *fminus) {
    const uint64_t mask = ((uint64_t)1 << vb) - 1;
    GRID_STRIDE(i, E) {
        const int e = ent[i];
        const int f = fid1[i] - 1;   // inclusive scan of the heads, minus one
        cf[e] = f;
        cs[e] = head[i] ? 1 : -1;
        if (!head[i]) continue;
        fplus[f] = e / nf;
        fminus[f] = (i + 1 < E && !head[i + 1]) ? ent[i + 1] / nf : -1;
        if (single) {
            for (int a = 0; a < nvf; ++a) fv[(int64_t)f * nvf + a] = (int)((hi[i] >> (vb * (nvf - 1 - a))) & mask);
        } else {
            fv[(int64_t)f * nvf] = (int)(hi[i] >> vb);
            fv[(int64_t)f * nvf + 1] = (int)(hi[i] & mask);
            for (int a = 2; a < nvf; ++a) fv[(int64_t)f * nvf + a] = (int)((lo[i] >> (vb * (nvf - 1 - a))) & mask);
        }
    }
}

// unit normals (outward from the plus cell) and measures (mesh.py:145-167), the host's operations
// in the host's order
__global__ void k_facet_geometry(int64_t F, int dim, int nvf, int nn, const double *X, const int *cells, const int *fv,
                                 const int *fplus, double *fn, double *fm) {
    GRID_STRIDE(f, F) {
        double p[4][3] = {};
        for (int k = 0; k < nvf; ++k)
            for (int d = 0; d < dim; ++d) p[k][d] = X[(int64_t)fv[f * nvf + k] * dim + d];
        double ctr[3] = {0, 0, 0}, cc[3] = {0, 0, 0}, nrm[3] = {0, 0, 0}, meas;
        for (int d = 0; d < dim; ++d) {
            double s = p[0][d];
            for (int k = 1; k < nvf; ++k) s = __dadd_rn(s, p[k][d]);
            ctr[d] = __ddiv_rn(s, (double)nvf);
        }
        if (dim == 2) {
            const double t0 = __dsub_rn(p[1][0], p[0][0]), t1 = __dsub_rn(p[1][1], p[0][1]);
            meas = __dsqrt_rn(__dadd_rn(__dmul_rn(t0, t0), __dmul_rn(t1, t1)));
            nrm[0] = __ddiv_rn(t1, meas);
            nrm[1] = __ddiv_rn(-t0, meas);
        } else {
            double a[3], b[3];
            for (int d = 0; d < 3; ++d) { a[d] = __dsub_rn(p[1][d], p[0][d]); b[d] = __dsub_rn(p[2][d], p[0][d]); }
            const double cr[3] = {__dsub_rn(__dmul_rn(a[1], b[2]), __dmul_rn(a[2], b[1])),
                                  __dsub_rn(__dmul_rn(a[2], b[0]), __dmul_rn(a[0], b[2])),
                                  __dsub_rn(__dmul_rn(a[0], b[1]), __dmul_rn(a[1], b[0]))};
            const double a2 = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(cr[0], cr[0]), __dmul_rn(cr[1], cr[1])),
                                                   __dmul_rn(cr[2], cr[2])));
            for (int d = 0; d < 3; ++d) nrm[d] = __ddiv_rn(cr[d], a2);
            meas = nvf == 3 ? __dmul_rn(0.5, a2) : a2;
        }
        const int64_t pc = fplus[f];
        for (int d = 0; d < dim; ++d) {
            double s = X[(int64_t)cells[pc * nn] * dim + d];
            for (int k = 1; k < nn; ++k) s = __dadd_rn(s, X[(int64_t)cells[pc * nn + k] * dim + d]);
            cc[d] = __ddiv_rn(s, (double)nn);
        }
        double dot = 0;
        for (int d = 0; d < dim; ++d) dot = __dadd_rn(dot, __dmul_rn(nrm[d], __dsub_rn(ctr[d], cc[d])));
        if (dot < 0)
            for (int d = 0; d < dim; ++d) nrm[d] = -nrm[d];
        for (int d = 0; d < dim; ++d) fn[f * dim + d] = nrm[d];
        fm[f] = meas;
    }
}

template <typename K>
static void sort_pairs(Ctx *c, const K *kin, K *kout, const int *vin, int *vout, int64_t n, int end_bit) {
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, n, 0, end_bit, c->s));
    DBuf<char> t(tb, c->s);
    CK(cub::DeviceRadixSort::SortPairs(t.p, tb, kin, kout, vin, vout, n, 0, end_bit, c->s));
    launched(c);
}

// det J per (sub-cell, spacing classes): the host's np_det on the J the cells of that class have
static std::vector<double> det_table(int kind, int dim, const std::vector<double> &hval) {
    const int ncls = (int)hval.size();
    const int P = kind == DPP_TET ? 6 : kind == DPP_TRI ? 2 : 1;
    const MeshTab T = mesh_tab(kind);
    size_t per = 1;
    for (int d = 0; d < dim; ++d) per *= ncls;
    std::vector<double> tab((size_t)P * per);
    for (size_t t = 0; t < tab.size(); ++t) {
        int cl[3] = {0, 0, 0};
        size_t r = t;
        for (int d = dim - 1; d >= 0; --d) { cl[d] = (int)(r % ncls); r /= ncls; }
        const int p = (int)r;
        double J[9] = {0};
        if (kind == DPP_QUAD || kind == DPP_HEX) {
            for (int d = 0; d < dim; ++d) J[d * dim + d] = hval[cl[d]];
        } else if (kind == DPP_TRI) {
            // (v00,v10,v11): columns (hx,0),(hx,hy); (v00,v11,v01): columns (hx,hy),(0,hy)
            const double hx = hval[cl[0]], hy = hval[cl[1]];
            if (p == 0) { J[0] = hx; J[1] = hx; J[2] = 0.0; J[3] = hy; }
            else { J[0] = hx; J[1] = 0.0; J[2] = hy; J[3] = hy; }
        } else {
            int stepped[4][3] = {};
            int pos[3] = {0, 0, 0};
            for (int s = 0; s < 3; ++s) {
                pos[T.perm[p][s]] = 1;
                for (int d = 0; d < 3; ++d) stepped[s + 1][d] = pos[d];
            }
            if (T.odd[p]) std::swap_ranges(stepped[1], stepped[1] + 3, stepped[2]);
            for (int k = 0; k < 3; ++k)
                for (int d = 0; d < 3; ++d) J[d * 3 + k] = stepped[k + 1][d] ? hval[cl[d]] : 0.0;
        }
        tab[t] = np_det(J, dim);
    }
    return tab;
}

template <typename T>
static void widen(const DBuf<T> &b, std::vector<int64_t> &out) {
    std::vector<T> h = b.to_host();
    out.assign(h.begin(), h.end());
}

void generate_on_device(Ctx *c, HostMesh &m, int dim, int kind, int n) {
    if (n < 1) DPP_FAIL(DPP_ERR_VALUE, "n_div must be a positive integer");
    if (kind < 0 || kind > 3) DPP_FAIL(DPP_ERR_VALUE, "unknown cell kind");
    if (kind_dim(kind) != dim) DPP_FAIL(DPP_ERR_VALUE, "cell kind / dim mismatch");
    DPP_TRACE_SCOPE(c, "mesh.generate_device");
    const int nn = kind_nodes(kind), nf = kind_facets(kind), nvf = kind_facet_nodes(kind);
    const int64_t w = n + 1;
    int64_t V = 1, cubes = 1;
    for (int d = 0; d < dim; ++d) { V *= w; cubes *= n; }
    const int64_t C = cubes * (kind == DPP_TET ? 6 : kind == DPP_TRI ? 2 : 1);
    const int64_t E = C * nf;
    if (V >= ((int64_t)1 << 31) || E >= ((int64_t)1 << 31)) DPP_FAIL(DPP_ERR_VALUE, "mesh too large for 32-bit device ids");
    int vb = 1;
    while (((int64_t)1 << vb) < V) ++vb;
    const int single = nvf * vb <= 64;

    // grid spacings and their bit-distinct classes (host, O(n))
    const double step = 1.0 / n;
    std::vector<double> xs(w);
    for (int64_t i = 0; i < w; ++i) xs[i] = (double)i * step + 0.0;
    xs[n] = 1.0;
    std::vector<double> hval;
    std::vector<int> cls(n);
    for (int i = 0; i < n; ++i) {
        const double h = xs[i + 1] - xs[i];
        size_t k = 0;
        while (k < hval.size() && std::memcmp(&hval[k], &h, 8) != 0) ++k;
        if (k == hval.size()) hval.push_back(h);
        cls[i] = (int)k;
    }
    const std::vector<double> tab = det_table(kind, dim, hval);
    for (double d : tab)
        if (!(d > 0)) DPP_FAIL(DPP_ERR_RUNTIME, "mesh generation produced an inverted cell");

    auto d = std::make_shared<DevMesh>();
    d->c = c;
    d->dim = dim; d->kind = kind; d->nn = nn; d->nf = nf; d->nvf = nvf;
    d->V = V; d->C = C;
    const MeshTab T = mesh_tab(kind);
    DBuf<int> dcls(cls.size(), c->s);
    DBuf<double> dtab(tab.size(), c->s), J((size_t)C * dim * dim, c->s);
    CK(cudaMemcpyAsync(dcls.p, cls.data(), 4 * cls.size(), cudaMemcpyHostToDevice, c->s));
    CK(cudaMemcpyAsync(dtab.p, tab.data(), 8 * tab.size(), cudaMemcpyHostToDevice, c->s));
    d->verts.alloc((size_t)V * dim, c->s);
    d->cells.alloc((size_t)C * nn, c->s);
    d->det.alloc((size_t)C, c->s);
    k_mesh_vertices<<<grid_for(V, 256, c->sms), 256, 0, c->s>>>(V, dim, n, step, d->verts.p);
    launched(c);
    k_mesh_cells<<<grid_for(C, 256, c->sms), 256, 0, c->s>>>(C, kind, dim, nn, n, T, d->verts.p, dcls.p,
                                                             (int)hval.size(), dtab.p, d->cells.p, J.p, d->det.p);
    launched(c);

    // facets: sort the (cell, local facet) entries by their sorted vertex tuples
    DBuf<uint64_t> hi(E, c->s), hi2(E, c->s), lo, lo2;
    DBuf<int> ent(E, c->s), ent2(E, c->s);
    if (!single) { lo.alloc(E, c->s); lo2.alloc(E, c->s); }
    k_facet_keys<<<grid_for(E, 256, c->sms), 256, 0, c->s>>>(E, nf, nvf, nn, vb, single, T, d->cells.p, hi.p,
                                                             single ? nullptr : lo.p, ent.p);
    launched(c);
    const uint64_t *shi, *slo = nullptr;
    const int *sent;
    DBuf<int> idx, idx2;
    if (single) {
        sort_pairs(c, hi.p, hi2.p, ent.p, ent2.p, E, nvf * vb);
        shi = hi2.p; sent = ent2.p;
    } else {
        // least-significant part first, then a stable sort on the leading two ids
        sort_pairs(c, lo.p, lo2.p, ent.p, ent2.p, E, (nvf - 2) * vb);
        idx.alloc(E, c->s); idx2.alloc(E, c->s);
        k_gather_u64<<<grid_for(E, 256, c->sms), 256, 0, c->s>>>(E, ent2.p, hi.p, hi2.p, idx.p);
        launched(c);
        sort_pairs(c, hi2.p, hi.p, idx.p, idx2.p, E, 2 * vb);
        k_gather_fin<<<grid_for(E, 256, c->sms), 256, 0, c->s>>>(E, idx2.p, lo2.p, ent2.p, lo.p, ent.p);
        launched(c);
        shi = hi.p; slo = lo.p; sent = ent.p;
    }
    DBuf<int> head(E, c->s), fid1(E, c->s), bad(1, c->s);
    CK(cudaMemsetAsync(bad.p, 0, 4, c->s));
    k_facet_heads<<<grid_for(E, 256, c->sms), 256, 0, c->s>>>(E, shi, slo, head.p, bad.p);
    launched(c);
    {
        size_t tb = 0;
        CK(cub::DeviceScan::InclusiveSum(nullptr, tb, head.p, fid1.p, E, c->s));
        DBuf<char> t(tb, c->s);
        CK(cub::DeviceScan::InclusiveSum(t.p, tb, head.p, fid1.p, E, c->s));
        launched(c);
    }
    int hF = 0, hbad = 0;
    CK(cudaMemcpyAsync(&hF, fid1.p + (E - 1), 4, cudaMemcpyDeviceToHost, c->s));
    CK(cudaMemcpyAsync(&hbad, bad.p, 4, cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    if (hbad) DPP_FAIL(DPP_ERR_VALUE, "facet shared by more than two cells");
    const int64_t F = hF;
    d->F = F;
    d->cf.alloc((size_t)E, c->s);
    d->cs.alloc((size_t)E, c->s);
    d->fv.alloc((size_t)F * nvf, c->s);
    d->fplus.alloc((size_t)F, c->s);
    d->fminus.alloc((size_t)F, c->s);
    d->fn.alloc((size_t)F * dim, c->s);
    d->fm.alloc((size_t)F, c->s);
    k_facet_scatter<<<grid_for(E, 256, c->sms), 256, 0, c->s>>>(E, nf, nvf, vb, single, shi, slo, sent, head.p, fid1.p,
                                                                d->cf.p, d->cs.p, d->fv.p, d->fplus.p, d->fminus.p);
    launched(c);
    k_facet_geometry<<<grid_for(F, 128, c->sms), 128, 0, c->s>>>(F, dim, nvf, nn, d->verts.p, d->cells.p, d->fv.p,
                                                                 d->fplus.p, d->fn.p, d->fm.p);
    launched(c);
    d->facets = true;
    cell_jinv(c, *d);

    // host arrays of the mesh object, read back from the device image
    m = HostMesh();
    m.dim = dim; m.kind = kind; m.n_div = n;
    m.n_vertices = V; m.n_cells = C; m.n_facets = F;
    m.vertices = d->verts.to_host();
    m.det = d->det.to_host();
    m.J = J.to_host();
    m.facet_normals = d->fn.to_host();
    m.facet_measures = d->fm.to_host();
    widen(d->cells, m.cells);
    widen(d->cf, m.cell_facets);
    widen(d->fv, m.facet_vertex_ids);
    widen(d->fplus, m.facet_plus);
    widen(d->fminus, m.facet_minus);
    {
        std::vector<signed char> h = d->cs.to_host();
        m.cell_facet_signs.assign(h.begin(), h.end());
    }
    m.dev = d;
    m.dev_bytes = 0;
    m.bc_bytes = 0;
}

}  // namespace dpp

using namespace dpp;
#include "abi_guard.cuh"

extern "C" int dpp_mesh_generate_device(dpp_ctx *ctx, int dim, int kind, int n_div, dpp_mesh **out) {
    return guard([&] {
        auto h = std::make_unique<dpp_mesh>();
        generate_on_device(&ctx->c, h->m, dim, kind, n_div);
        *out = h.release();
    });
}
