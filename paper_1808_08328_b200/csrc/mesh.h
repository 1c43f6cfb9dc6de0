// Host mesh representation shared by mesh.cpp (numbering) and assembly.cu.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

namespace dpp {

struct DevMesh;   // device copy (assembly.cu)

struct HostMesh {
    int dim = 2, kind = 0, n_div = 1;
    int64_t n_vertices = 0, n_cells = 0, n_facets = 0;
    std::vector<double> vertices;             // (V, dim)
    std::vector<int64_t> cells;               // (C, nv)
    std::vector<int64_t> facet_vertex_ids;    // (F, nvf)
    std::vector<int64_t> cell_facets;         // (C, nf)
    std::vector<int8_t> cell_facet_signs;     // (C, nf)
    std::vector<int64_t> facet_plus, facet_minus;
    std::vector<double> facet_normals, facet_measures;
    std::vector<double> J, det;               // (C, dim, dim), (C,)
    std::shared_ptr<DevMesh> dev;             // lazily uploaded
    std::shared_ptr<void> pinned;             // device-layout image in pinned host memory (built once)
    size_t pinned_bytes = 0;
    size_t dev_bytes = 0;                     // host->device bytes of the current device image
    size_t bc_bytes = 0;                      //   + the last assembly's compact boundary-facet data
    std::shared_ptr<void> bc_pinned;          // pinned staging of that data (reused)
    size_t bc_pinned_bytes = 0;
    std::shared_ptr<void> bc_done;            // event (cudaEvent_t) after the staging's last copies
    void build();
};

HostMesh generate(int dim, int kind, int n);
int kind_dim(int kind);
int kind_nodes(int kind);
int kind_facets(int kind);
int kind_facet_nodes(int kind);
int local_facet(int kind, int f, int k);
// numpy.linalg.det of a d x d matrix (row-major, destroyed): getrf + sign * exp(sum log|u_ii|)
double np_det(double *a, int d);

}  // namespace dpp
