// Block system (ten CSR blocks + four RHS segments) and the cross-module API
// of the solver layers (pc.cu, gmres.cu, assembly.cu).
#pragma once

#include <string>

#include "dpp_internal.cuh"

// reference BlockSystem (assembly.py:48-99): blocks in the order of dpp.h's DPP_K*_*
struct dpp_system {
    dpp::Ctx *ctx = nullptr;
    dpp::Csr blk[10];
    dpp::DBuf<double> rhs[4];
    int64_t sizes[4] = {0, 0, 0, 0};   // u1, p1, u2, p2
    bool hasK = false;
    dpp::Csr K;                         // monolithic view, stored pattern (explicit zeros kept)
    dpp::Csr Kc;                        // zero-free compute copy used by SpMV
    dpp::DBuf<double> f;                // monolithic RHS
    double assembly_ms = 0.0;
};

namespace dpp {

void reciprocal(Ctx *c, int64_t n, const double *d, double *o);
const Csr &system_K(Ctx *c, dpp_system *s);
const Csr &system_Kc(Ctx *c, dpp_system *s);
const double *system_f(Ctx *c, dpp_system *s);

dpp_pc *pc_create(Ctx *c, dpp_system *s, const dpp_split_node *nodes, int n_nodes,
                  dpp_randn_fn randn, void *user, const Csr *K = nullptr);
void pc_apply_dev(dpp_pc *pc, const double *r_dev, double *z_dev);
std::string pc_desc(const dpp_pc *pc);
double pc_setup_ms(const dpp_pc *pc);
int pc_size(const dpp_pc *pc);
double *pc_in(dpp_pc *pc);
double *pc_out(dpp_pc *pc);
int64_t pc_kernels(const dpp_pc *pc);
Ctx *pc_ctx(dpp_pc *pc);
void pc_destroy(dpp_pc *pc);

// restarted left-preconditioned GMRES on device vectors (linalg.py:65-165)
struct Operator {
    const Csr *A = nullptr;            // device matrix, or
    dpp_apply_fn cb = nullptr;         // host callback
    void *user = nullptr;
};
struct PcOp {
    dpp_pc *pc = nullptr;
    dpp_apply_fn cb = nullptr;
    void *user = nullptr;
};
void gmres_dev(Ctx *c, int64_t n, const Operator &A, const PcOp &M, const double *b_dev,
               double *x_dev, double rtol, int max_iter, int restart, dpp_krylov_stats *st,
               std::vector<double> *history, bool x_zero = false);

}  // namespace dpp

namespace dpp {
double pc_bytes(const dpp_pc *pc);
double spmv_bytes(const Csr &A);
}  // namespace dpp
