// Device copy of a mesh (assembly.cu builds it from the host numbering; fields.cu reads it).
#pragma once

#include "dpp_internal.cuh"
#include "mesh.h"

namespace dpp {

struct DevMesh {
    Ctx *c = nullptr;
    int dim = 0, kind = 0, nn = 0, nf = 0, nvf = 0;
    int64_t V = 0, C = 0, F = 0;
    DBuf<double> verts, det, Jinv;
    DBuf<int> cells, cf, fv, fplus, fminus;
    DBuf<signed char> cs;
    DBuf<double> fn, fm;
    bool facets = false;   // facet arrays uploaded (H(div), DG-VMS, facet queries); CG-VMS needs none
    size_t foff[7] = {0}, fbytes[7] = {0};   // facet parts in the pinned image
};

// the mesh's device image for context c (uploaded on first use, cached in the host mesh)
DevMesh &dev_mesh(Ctx *c, HostMesh &m);
// facet arrays (H(div), DG-VMS, facet queries; CG-VMS assembly needs none)
void ensure_facets(Ctx *c, HostMesh &hm, DevMesh &d);
// cell Jacobian inverses (numpy.linalg.inv roundings) from the device vertices / cells
void cell_jinv(Ctx *c, DevMesh &d);
// the whole structured mesh built in HBM (devmesh.cu); the host arrays are read back from it
void generate_on_device(Ctx *c, HostMesh &m, int dim, int kind, int n);

}  // namespace dpp

struct dpp_mesh { dpp::HostMesh m; };
