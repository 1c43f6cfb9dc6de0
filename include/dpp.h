/*
 * dpp.h -- C ABI of libdpp, the B200-native (sm_100a, FP64) implementation of
 * the DPP (double porosity/permeability) assemble + field-split GMRES hot path
 * of arXiv 1808.08328's reference package `dppflow`.
 *
 * The reference is pure Python; it has no FFI.  Each entry point below
 * replaces one reference Python function on the hot path (file:line into
 * /root/reference/pkg/src/dppflow/), and the Python package
 * paper_1808_08328_b200 binds them with ctypes exactly as a maintainer would
 * (see INTEGRATION.md).  Conventions:
 *   - every function returns a status (DPP_OK = 0); on failure
 *     dpp_last_error() returns a thread-local message;
 *   - pointers named *_host are host memory, copied in/out synchronously;
 *   - handles own device memory (HBM) on the context's device and stream;
 *   - CSR index arrays are int32 (scipy's default), values are double;
 *   - a context is not thread-safe; distinct contexts are independent.
 */
#ifndef DPP_H
#define DPP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dpp_ctx dpp_ctx;
typedef struct dpp_csr dpp_csr;
typedef struct dpp_mesh dpp_mesh;
typedef struct dpp_system dpp_system;
typedef struct dpp_ilu dpp_ilu;
typedef struct dpp_amg dpp_amg;
typedef struct dpp_pc dpp_pc;

enum {
    DPP_OK = 0,
    DPP_ERR_CUDA = 1,       /* CUDA runtime failure (no device, launch error)   */
    DPP_ERR_VALUE = 2,      /* ValueError in the reference                     */
    DPP_ERR_ZERO_PIVOT = 3, /* linalg.ZeroPivotError (linalg.py:23)             */
    DPP_ERR_RUNTIME = 4,    /* RuntimeError (e.g. stalled aggregation, linalg.py:363-366) */
    DPP_ERR_ALLOC = 5
};

enum { DPP_TRI = 0, DPP_QUAD = 1, DPP_TET = 2, DPP_HEX = 3 };       /* mesh.py:24-28 */
enum { DPP_HDIV = 0, DPP_CGVMS = 1, DPP_DGVMS = 2 };                /* elements.py:34-37 */
/* block ids, in BlockSystem field order (assembly.py:55-64) */
enum { DPP_K1_UU = 0, DPP_K1_UP, DPP_K1_PU, DPP_K1_PP, DPP_K2_UU, DPP_K2_UP, DPP_K2_PU,
       DPP_K2_PP, DPP_K12_PP, DPP_K21_PP };

const char *dpp_last_error(void);
int dpp_version(void);

/* ---- context: one device, one stream, stream-ordered allocator ---------- */
int dpp_ctx_create(int device, dpp_ctx **out);
int dpp_ctx_destroy(dpp_ctx *ctx);
int dpp_ctx_sync(dpp_ctx *ctx);
/* CUDA-event timer on the context stream: start, then stop -> elapsed ms */
int dpp_timer_start(dpp_ctx *ctx);
int dpp_timer_stop(dpp_ctx *ctx, double *ms);
/* number of libdpp kernel launches issued on this context so far */
int dpp_ctx_launches(const dpp_ctx *ctx, int64_t *count);
/* NON-PARITY fast mode (no reference counterpart): triangular solves of
 * preconditioners built afterwards on this context become `sweeps` Jacobi sweeps
 * (x0 = D^-1 b, x <- D^-1 (b - S x)); 0 restores the reference's exact substitution */
int dpp_ctx_set_tri_jacobi(dpp_ctx *ctx, int sweeps);

/* ---- CSR matrices (scipy.sparse.csr_matrix on the device) --------------- */
int dpp_csr_create(dpp_ctx *ctx, int rows, int cols, int64_t nnz, const int32_t *indptr_host,
                   const int32_t *indices_host, const double *data_host, dpp_csr **out);
int dpp_csr_info(const dpp_csr *A, int *rows, int *cols, int64_t *nnz);
int dpp_csr_download(const dpp_csr *A, int32_t *indptr_host, int32_t *indices_host,
                     double *data_host);
int dpp_csr_destroy(dpp_csr *A);
/* linalg.spmv (linalg.py:27-32): y = A x */
int dpp_spmv(dpp_ctx *ctx, const dpp_csr *A, const double *x_host, double *y_host);
/* SpMV plan of a matrix applied repeatedly (the operators inside dpp_solve get one
 * automatically): 0 none (warp-per-row CSR), 1 CSR-stream row blocks, 2 SELL-32,
 * 3 automatic (SELL-32 when its zero padding stays under 25 %, else CSR-stream).
 * Replaces nothing in the reference (scipy's csr_matvec has one format); exposed so the
 * kernels can be checked against linalg.py:27-32 one by one. */
int dpp_csr_plan(dpp_csr *A, int kind);

/* ---- mesh (mesh.py:73-277): numbering is bit-exact with the reference ----- */
int dpp_mesh_generate(int dim, int kind, int n_div, dpp_mesh **out);
/* generate_unit_mesh (mesh.py:206-277) with _build_facets / _facet_geometry / jacobians
 * (mesh.py:106-185) run on the device: vertices, cells, the facet sort-unique (radix sorts of
 * packed sorted-vertex keys), cell / facet adjacency, normals, measures and J are built in HBM
 * (the mesh's device image) and the host arrays are read back from it; same arrays bit for bit
 * as dpp_mesh_generate.  The mesh is bound to ctx's device. */
int dpp_mesh_generate_device(dpp_ctx *ctx, int dim, int kind, int n_div, dpp_mesh **out);
int dpp_mesh_from_arrays(int dim, int kind, int n_div, int64_t n_vertices,
                         const double *vertices_host, int64_t n_cells, const int64_t *cells_host,
                         dpp_mesh **out);
int dpp_mesh_counts(const dpp_mesh *m, int64_t *n_vertices, int64_t *n_cells, int64_t *n_facets);
/* any output pointer may be NULL; shapes: vertices (V,dim), cells (C,k),
 * facet_vertex_ids (F,nv), cell_facets/signs (C,nf), facet_* (F[,dim]), J (C,dim,dim), det (C) */
int dpp_mesh_export(const dpp_mesh *m, double *vertices, int64_t *cells, int64_t *facet_vertex_ids,
                    int64_t *cell_facets, int8_t *cell_facet_signs, int64_t *facet_plus,
                    int64_t *facet_minus, double *facet_normals, double *facet_measures,
                    double *J, double *det);
int dpp_mesh_destroy(dpp_mesh *m);
/* drop the mesh's device copy (the next dpp_assemble re-uploads it) */
int dpp_mesh_release_device(dpp_mesh *m);

/* ---- assembly (assembly.py:233-584) ------------------------------------- */
typedef struct {
    double mu, beta, k1, k2, eta_u, eta_p;
    double gamma_b[3];
} dpp_params;                                          /* problem.py:26-45 */

/* boundary data, per network (index 0 = network 1).  p0 / un are the user's
 * boundary functions evaluated at the points returned by dpp_facet_points
 * (degree 4 facet rule, assembly.py:173-181, DATA_QUAD_DEGREE).  vfacets sorted; hdiv:
 * vdata = one prescribed flux integral per velocity facet (assembly.py:303-309);
 * dgvms: vdata = u.n at the degree-4 facet points, (n_vfacets, nq) (assembly.py:532-535);
 * cgvms: velocity facets only leave the pressure functional (pfacets exclude them). */
typedef struct {
    int64_t n_pfacets[2];
    const int64_t *pfacets[2];
    const double *p0[2];
    int64_t n_vfacets[2];
    const int64_t *vfacets[2];
    const double *vdata[2];
    /* p0_kind[k] != 0: p0[k] is not read; the device evaluates the reference's
     * manufactured pressure (problem.py:100-144) at the facet points itself:
     * 1 = 2-D (Eq. 44), 2 = 3-D (Eq. 46); p0_coef = {mu/pi, c, e} with
     * p = mu/pi * X * S + c * E (X = exp(pi x), S = sin(pi y) [+ sin(pi z)],
     * E = exp(e y) [+ exp(e z)]; c = -mu/(beta k1) for network 1, +mu/(beta k) for 2) */
    int32_t p0_kind[2];
    double p0_coef[2][4];
} dpp_bc;

int dpp_facet_rule_size(int dim, int kind, int degree, int *nq);
/* physical points (nf, nq, dim) and weights (nf, nq) of the facet rule */
int dpp_facet_points(dpp_ctx *ctx, dpp_mesh *m, int degree, int64_t nf, const int64_t *facets_host,
                     double *X_host, double *W_host);
/* bc may be NULL (bcs=None).  The mesh is uploaded on first use. */
int dpp_assemble(dpp_ctx *ctx, dpp_mesh *m, int formulation, const dpp_params *p,
                 const dpp_bc *bc, dpp_system **out);
/* Config-3 extension (the reference has scalar k only, problem.py:26-45):
 * per-cell permeabilities cell_k1 / cell_k2 (n_cells each, > 0; both or neither) replace
 * params.k1 / k2 cell by cell in the H(div) and CG-VMS cell integrals (assembly.py:274-276,
 * :338-342: mu/k in the velocity mass, k/mu in the pressure Laplacian and body force).
 * NULL -> dpp_assemble.  Parity for heterogeneous k is "unpinned" (no reference answer); with
 * every cell at params' k the system is bit-for-bit dpp_assemble's. */
int dpp_assemble_ext(dpp_ctx *ctx, dpp_mesh *m, int formulation, const dpp_params *p,
                     const double *cell_k1, const double *cell_k2, const dpp_bc *bc, dpp_system **out);
/* ---- discrete fields (assembly.py:591-644, spectrum.py:149-176) ----------
 * field 0..3 = u1, p1, u2, p2 of a formulation; coeffs = that field's segment of the
 * solution vector (ncoef checked).  ref_points: (nq, dim) reference coordinates, nq <= 128. */
/* values on every cell, (C, nq) for pressures, (C, nq, dim) for velocities
 * (DiscreteField.evaluate_all: nodal P1/Q1 sums, Piola map of the RT basis for H(div)) */
int dpp_field_evaluate(dpp_ctx *ctx, dpp_mesh *m, int formulation, int field, const double *coeffs_host,
                       int64_t ncoef, int nq, const double *ref_points_host, double *out_host);
/* physical points origin + J x_q of every cell, (C, nq, dim) (spectrum.py:159-161) */
int dpp_cell_points(dpp_ctx *ctx, dpp_mesh *m, int nq, const double *ref_points_host, double *X_host);
/* sqrt(sum_c sum_q w_q |u_h - u|^2 det_c) (spectrum.l2_error).  The exact field is either
 * exact_values_host (C, nq[, dim]) evaluated by the caller at dpp_cell_points, or, with
 * exact_kind != 0, the package manufactured solution evaluated on the device:
 * 1 / 2 = 2-D / 3-D pressure (exact_coef as dpp_bc.p0_coef), 3 / 4 = 2-D / 3-D velocity
 * -k [X S, X cos(pi y) + c e^{e y}, X cos(pi z) + c e^{e z}] with exact_coef = {k, c, e}. */
int dpp_field_l2_error(dpp_ctx *ctx, dpp_mesh *m, int formulation, int field, const double *coeffs_host,
                       int64_t ncoef, int nq, const double *ref_points_host, const double *weights_host,
                       int exact_kind, const double exact_coef[3], const double *exact_values_host,
                       double *l2);

/* a system from existing blocks (BlockSystem(...) constructed by the user):
 * blocks are copied; NULL block = empty matrix of the implied shape */
int dpp_system_from_blocks(dpp_ctx *ctx, const dpp_csr *const blocks[10],
                           const double *const rhs_host[4], const int64_t sizes[4],
                           dpp_system **out);
int dpp_system_sizes(const dpp_system *s, int64_t sizes[4]);
/* assembly._eliminate (assembly.py:200-226): symmetric strong elimination of dofs idx
 * (sorted, host) of field 0..3 = (u1, p1, u2, p2) with the given values; used for
 * CG-VMS pressure_dirichlet='strong' (assembly.py:410-415).  H(div) prescribed-flux
 * facets are eliminated inside dpp_assemble from dpp_bc.vfacets / vdata. */
int dpp_system_eliminate(dpp_system *s, int field, int64_t n, const int64_t *idx_host,
                         const double *values_host);
/* borrowed handle, valid while the system lives */
int dpp_system_block(dpp_system *s, int block, dpp_csr **out);
int dpp_system_rhs(const dpp_system *s, int field, double *out_host);
/* assembly.monolithic_view (assembly.py:102-108): borrowed K */
int dpp_system_monolithic(dpp_system *s, dpp_csr **out);
int dpp_system_timing(const dpp_system *s, double *assembly_ms);
int dpp_system_destroy(dpp_system *s);

/* ---- ILU(0) (linalg.py:178-227) ----------------------------------------- */
int dpp_ilu0_create(dpp_ctx *ctx, const dpp_csr *A, dpp_ilu **out);
int dpp_ilu0_apply(dpp_ilu *f, const double *r_host, double *z_host);
/* new handles with the reference's storage: L = tril(A,-1)+I (zero-free), U = triu(A) */
int dpp_ilu0_factors(dpp_ilu *f, dpp_csr **L, dpp_csr **U);
int dpp_ilu0_destroy(dpp_ilu *f);

/* ---- selfp Schur product (linalg.py:234-254) ------------------------------ */
int dpp_diag(dpp_ctx *ctx, const dpp_csr *A, double *out_host);
int dpp_schur_selfp(dpp_ctx *ctx, const dpp_csr *D, const dpp_csr *C, const double *diagA_host,
                    const dpp_csr *B, dpp_csr **out);

/* ---- smoothed-aggregation AMG (linalg.py:341-400) ------------------------ */
/* fills out[0..n) with the power-iteration start vector of linalg.py:330
 * (numpy default_rng(12345).standard_normal(n)); supplied by the binding */
typedef void (*dpp_randn_fn)(int64_t n, double *out, void *user);
int dpp_amg_create(dpp_ctx *ctx, const dpp_csr *A, double theta, double omega, int max_coarse,
                   int max_levels, dpp_randn_fn randn, void *user, dpp_amg **out);
int dpp_amg_levels(const dpp_amg *h, int *levels);
/* strength-graph greedy aggregation alone (linalg.py:279-324 _strength_aggregates): agg_host (n)
 * receives the aggregate id of every row, *n_agg their count; path 0 = automatic (device passes
 * from 32768 rows), 1 = host greedy over the device strength graph, 2 = device passes */
int dpp_strength_aggregates(dpp_ctx *ctx, const dpp_csr *A, double theta, int path, int64_t *agg_host,
                            int64_t *n_agg);
/* borrowed A_l and P_l (P NULL on the coarsest level); agg_host (n_l) may be NULL */
int dpp_amg_level(dpp_amg *h, int level, dpp_csr **A, dpp_csr **P, int64_t *agg_host,
                  double *rho);
int dpp_amg_vcycle(dpp_amg *h, const double *r_host, double *z_host);
int dpp_amg_destroy(dpp_amg *h);

/* ---- field-split preconditioner tree (blocksolve.py:217-294) -------------- */
enum { DPP_SPLIT_ADDITIVE = 0, DPP_SPLIT_SCHUR_FULL_SELFP = 1 };
enum { DPP_LEAF_BJACOBI_ILU0 = 0, DPP_LEAF_AMG = 1, DPP_LEAF_NESTED = 2 };
typedef struct {
    int split_type;
    int ngroup[2];
    int groups[2][2];     /* global field ids (0=u1,1=p1,2=u2,3=p2) */
    int child_type[2];
    int child_node[2];    /* index into the node array when DPP_LEAF_NESTED */
} dpp_split_node;
int dpp_pc_create(dpp_ctx *ctx, dpp_system *s, const dpp_split_node *nodes, int n_nodes,
                  dpp_randn_fn randn, void *user, dpp_pc **out);
/* build_preconditioner(bs, config, monolithic=K) (blocksolve.py:288-294): the split tree's
 * blocks are extracted from the caller's K (n x n, n = the system's total size) by the
 * system's field index sets instead of from the system's own blocks */
int dpp_pc_create_explicit(dpp_ctx *ctx, dpp_system *s, const dpp_csr *K, const dpp_split_node *nodes,
                           int n_nodes, dpp_randn_fn randn, void *user, dpp_pc **out);
int dpp_pc_apply(dpp_pc *pc, const double *r_host, double *z_host);
int dpp_pc_describe(const dpp_pc *pc, char *buf, int cap);
int dpp_pc_setup_ms(const dpp_pc *pc, double *ms);
int dpp_pc_destroy(dpp_pc *pc);

/* ---- restarted left-preconditioned GMRES (linalg.py:65-165) -------------- */
typedef void (*dpp_apply_fn)(const double *in_host, double *out_host, void *user);
typedef struct {
    int iterations, cycles, converged, reason; /* reason: 0 converged, 1 max_iter, 2 stagnation */
    int pc_applies, matvecs;
    double relative_residual, wall_time_s;
} dpp_krylov_stats;
/* operator: A (device CSR) or A_cb (host callback); preconditioner: pc, pc_cb or
 * neither (identity).  history_host receives |g_{j+1}|/||Mb|| per iteration. */
int dpp_gmres(dpp_ctx *ctx, const dpp_csr *A, dpp_apply_fn A_cb, void *A_user, dpp_pc *pc,
              dpp_apply_fn pc_cb, void *pc_user, int64_t n, const double *b_host,
              const double *x0_host, double *x_host, double rtol, int max_iter, int restart,
              dpp_krylov_stats *stats, double *history_host, int history_cap);
/* blocksolve.solve (blocksolve.py:346-360) GMRES part on the system's monolithic K */
int dpp_solve(dpp_ctx *ctx, dpp_system *s, dpp_pc *pc, double rtol, int max_iter, int restart,
              double *x_host, dpp_krylov_stats *stats, double *history_host, int history_cap);

/* ---- row-sharded SpMV over NVLink peer memory (NON-PARITY extension) ----
 * The reference's SpMV is scipy's csr_matvec on the whole matrix (linalg.py:27-32).  Here rank p
 * (one process per GPU) owns a contiguous row block of K and the matching slice of every vector;
 * slices live in IPC-exportable buffers that the other ranks map, and the SpMV kernel loads
 * off-rank entries of x directly through the peer mappings (no all-gather, no halo copy).
 * Columns are 32-bit codes: owner << 29 | offset in the owner's slice (<= 8 ranks).  Row sums are
 * lane-parallel: equal to csr_matvec up to the order of additions, so outside the parity contract. */
typedef struct dpp_peerbuf dpp_peerbuf;
typedef struct dpp_shard dpp_shard;
int dpp_peerbuf_create(dpp_ctx *ctx, int64_t n, dpp_peerbuf **out);
int dpp_peerbuf_export(const dpp_peerbuf *b, unsigned char *handle64);       /* cudaIpcMemHandle_t */
int dpp_peerbuf_open(dpp_ctx *ctx, const unsigned char *handle64, int64_t n, dpp_peerbuf **out);
int dpp_peerbuf_write(dpp_peerbuf *b, const double *host, int64_t n);
int dpp_peerbuf_read(const dpp_peerbuf *b, double *host, int64_t n);
int dpp_peerbuf_destroy(dpp_peerbuf *b);
int dpp_shard_create(dpp_ctx *ctx, int rows, int64_t nnz, const int32_t *indptr, const uint32_t *codes,
                     const double *values, int nseg, const int64_t *seg_len, dpp_shard **out);
/* y[0:rows] = K[rows of this rank, :] x, x given as nseg slices (own buffer or mapped peers) */
int dpp_shard_spmv(dpp_ctx *ctx, const dpp_shard *sh, dpp_peerbuf *const *xseg, dpp_peerbuf *y);
int dpp_shard_profile(dpp_ctx *ctx, const dpp_shard *sh, dpp_peerbuf *const *xseg, dpp_peerbuf *y, int reps,
                      double *ms_per_call, double *bytes_per_call);
int dpp_shard_destroy(dpp_shard *sh);

/* ---- measurement: CUDA-event timing of the Arnoldi-step kernels ----------- */
typedef struct {
    double spmv_ms, pc_ms;           /* mean per call over reps */
    double spmv_bytes, pc_bytes;     /* algorithmic bytes */
    double mgs_ms;
    int64_t pc_launches;
} dpp_step_profile;
int dpp_profile_step(dpp_ctx *ctx, dpp_system *s, dpp_pc *pc, int reps, int flush_l2,
                     dpp_step_profile *out);

#ifdef __cplusplus
}
#endif
#endif /* DPP_H */
