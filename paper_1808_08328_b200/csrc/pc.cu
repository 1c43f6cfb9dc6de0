// Composable field-split preconditioner on the device.
//
// Reference: blocksolve._build_leaf / _build_node / build_preconditioner
// (blocksolve.py:227-294).  A node splits its index space into two field
// groups; "additive" applies the two children independently (here on two
// streams, so e.g. both pore networks of the scale split run concurrently),
// "schur" (full factorisation, selfp) applies
//     zA = pcA(rA); zB = pcS(rB - C zA); zA -= pcA(B zB)
// with S_p = D - C diag(A)^-1 B built by the ordered SpGEMM.  Leaves are
// bjacobi -> ILU(0) and hypre -> smoothed-aggregation AMG V-cycle.
// The whole apply is captured once into a CUDA graph and replayed.
#include <cstdlib>
#include <exception>
#include <string>
#include <thread>

#include "dpp_internal.cuh"
#include "system.cuh"

namespace dpp {

struct PcNode;

struct PcLeaf {
    int type = -1;
    std::unique_ptr<Ilu> ilu;
    std::unique_ptr<Amg> amg;
    std::unique_ptr<PcNode> node;
    std::string desc;
    void apply(Ctx *c, const double *r, double *z, cudaStream_t st);
};

struct PcNode {
    SideStream side_owner;
    int split = 0;
    int n = 0, nA = 0, nB = 0;
    std::vector<std::pair<int, int>> segA, segB;   // (offset, length) in the local space
    PcLeaf a, b;
    Csr Bc, Cc;                                    // zero-free B = M[A,B], C = M[B,A]
    DBuf<double> rA, rB, zA, zB, t, w, zA2;
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    std::string desc;
    ~PcNode() {
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
    }
    void apply(Ctx *c, const double *r, double *z, cudaStream_t st);
};

static void gather(Ctx *c, double *dst, const double *src, const std::vector<std::pair<int, int>> &seg,
                   cudaStream_t st) {
    int64_t d[4], s[4], l[4];
    int64_t off = 0;
    for (size_t k = 0; k < seg.size(); ++k) { d[k] = off; s[k] = seg[k].first; l[k] = seg[k].second; off += l[k]; }
    copy_segments(c, dst, src, (int)seg.size(), d, s, l, st);
}
static void scatter(Ctx *c, double *dst, const double *src, const std::vector<std::pair<int, int>> &seg,
                    cudaStream_t st) {
    int64_t d[4], s[4], l[4];
    int64_t off = 0;
    for (size_t k = 0; k < seg.size(); ++k) { s[k] = off; d[k] = seg[k].first; l[k] = seg[k].second; off += l[k]; }
    copy_segments(c, dst, src, (int)seg.size(), d, s, l, st);
}

void PcLeaf::apply(Ctx *c, const double *r, double *z, cudaStream_t st) {
    if (type == DPP_LEAF_BJACOBI_ILU0) ilu_apply(c, *ilu, r, z, st);
    else if (type == DPP_LEAF_AMG) amg_vcycle(c, *amg, r, z, st);
    else node->apply(c, r, z, st);
}

void PcNode::apply(Ctx *c, const double *r, double *z, cudaStream_t st) {
    gather(c, rA.p, r, segA, st);
    gather(c, rB.p, r, segB, st);
    if (split == DPP_SPLIT_ADDITIVE) {
        CK(cudaEventRecord(ev_fork, st));
        CK(cudaStreamWaitEvent(side, ev_fork, 0));
        b.apply(c, rB.p, zB.p, side);
        a.apply(c, rA.p, zA.p, st);
        CK(cudaEventRecord(ev_join, side));
        CK(cudaStreamWaitEvent(st, ev_join, 0));
        scatter(c, z, zA.p, segA, st);
        scatter(c, z, zB.p, segB, st);
        return;
    }
    a.apply(c, rA.p, zA.p, st);                       // zA = pcA(rA)
    spmv(c, Cc, zA.p, t.p, rB.p, -1.0, st);            // t = rB - C zA
    b.apply(c, t.p, zB.p, st);                        // zB = pcS(t)
    spmv(c, Bc, zB.p, w.p, nullptr, 1.0, st);          // w = B zB
    a.apply(c, w.p, zA2.p, st);                       // zA2 = pcA(w)
    axpby_to(c, nA, zA.p, -1.0, zA2.p, zA.p, st);     // zA = zA - zA2
    scatter(c, z, zA.p, segA, st);
    scatter(c, z, zB.p, segB, st);
}

struct Builder {
    Ctx *c;
    const dpp_split_node *nodes;
    int n_nodes;
    dpp_system *sys;       // field blocks (u1, p1, u2, p2)
    dpp_randn_fn randn;
    void *user;

    // The submatrix of the monolithic K on field lists (rows fr, cols fc): the reference
    // extracts it from K by index sets (blocksolve.py:227-228, order-preserving, stored
    // zeros kept), which is exactly the system's field block (borrowed, no copy), an
    // empty block for fields that do not couple, or sp.bmat of field blocks.
    const Csr &fmat(const std::vector<int> &fr, const std::vector<int> &fc, Csr &store) {
        static const int RC[10][2] = {{0, 0}, {0, 1}, {1, 0}, {1, 1}, {2, 2}, {2, 3}, {3, 2}, {3, 3}, {1, 3}, {3, 1}};
        auto block = [&](int r, int cc) -> const Csr * {
            for (int b = 0; b < 10; ++b)
                if (RC[b][0] == r && RC[b][1] == cc) return &sys->blk[b];
            return nullptr;
        };
        if (fr.size() == 1 && fc.size() == 1) {
            if (const Csr *B = block(fr[0], fc[0])) return *B;
            store = csr_empty(c, (int)sys->sizes[fr[0]], (int)sys->sizes[fc[0]]);
            return store;
        }
        std::vector<const Csr *> grid;
        std::vector<int> rsz, csz;
        for (int r : fr) rsz.push_back((int)sys->sizes[r]);
        for (int cc : fc) csz.push_back((int)sys->sizes[cc]);
        for (int r : fr)
            for (int cc : fc) grid.push_back(block(r, cc));
        store = csr_bmat(c, grid, (int)fr.size(), (int)fc.size(), rsz, csz);
        return store;
    }

    PcLeaf leaf_on(int type, const Csr &M) {
        PcLeaf L;
        L.type = type;
        if (type == DPP_LEAF_BJACOBI_ILU0) {
            L.ilu = ilu0(c, M);
            L.desc = "bjacobi/ilu0";
        } else if (type == DPP_LEAF_AMG) {
            L.amg = amg_setup(c, M, 0.5, 2.0 / 3.0, 64, 25, randn, user);
            L.desc = "amg[" + std::to_string(L.amg->lv.size()) + "]";
        } else {
            DPP_FAIL(DPP_ERR_VALUE, "unknown leaf type");
        }
        return L;
    }

    // Node on fields `fids`: M == nullptr -> the system's field blocks (fmat); otherwise M is
    // the node's explicit matrix (e.g. the Schur complement) and blocks are extracted from it
    // by index sets, as the reference does (blocksolve.py:241-256).
    std::unique_ptr<PcNode> node(int id, const std::vector<int> &fids, const Csr *M = nullptr) {
        const dpp_split_node &nd = nodes[id];
        auto N = std::make_unique<PcNode>();
        N->split = nd.split_type;
        std::vector<int> off(fids.size() + 1, 0);
        for (size_t i = 0; i < fids.size(); ++i) off[i + 1] = off[i] + (int)sys->sizes[fids[i]];
        N->n = off.back();
        if (M && N->n != M->rows) DPP_FAIL(DPP_ERR_VALUE, "split node: matrix does not match field sizes");
        std::vector<int> gA(nd.groups[0], nd.groups[0] + nd.ngroup[0]);
        std::vector<int> gB(nd.groups[1], nd.groups[1] + nd.ngroup[1]);
        auto segs = [&](const std::vector<int> &g) {
            std::vector<std::pair<int, int>> s;
            for (int f : g) {
                int pos = -1;
                for (size_t i = 0; i < fids.size(); ++i)
                    if (fids[i] == f) pos = (int)i;
                if (pos < 0) DPP_FAIL(DPP_ERR_VALUE, "split group field not in parent");
                s.push_back({off[pos], off[pos + 1] - off[pos]});
            }
            return s;
        };
        N->segA = segs(gA);
        N->segB = segs(gB);
        for (auto &s : N->segA) N->nA += s.second;
        for (auto &s : N->segB) N->nB += s.second;
        for (DBuf<double> *b : {&N->rA, &N->zA, &N->zA2, &N->w}) b->alloc(N->nA, c->s);
        for (DBuf<double> *b : {&N->rB, &N->zB, &N->t}) b->alloc(N->nB, c->s);
        // sub-block (rows g1, cols g2) of this node's matrix
        auto sub = [&](Builder &bb, const std::vector<int> &g1, const std::vector<std::pair<int, int>> &s1,
                       const std::vector<int> &g2, const std::vector<std::pair<int, int>> &s2,
                       Csr &store) -> const Csr & {
            if (!M) return bb.fmat(g1, g2, store);
            DPP_TRACE_SCOPE(bb.c, "pc.submatrix");
            store = csr_submatrix(bb.c, *M, s1, s2);
            return store;
        };
        // a child on group g of this node
        auto child = [&](Builder &bb, int type, int nested, const std::vector<int> &g,
                         const std::vector<std::pair<int, int>> &s) {
            Csr store;
            if (type == DPP_LEAF_NESTED) {
                if (nested < 0 || nested >= n_nodes) DPP_FAIL(DPP_ERR_VALUE, "bad nested split index");
                PcLeaf L;
                L.type = type;
                if (M) store = csr_submatrix(bb.c, *M, s, s);
                L.node = bb.node(nested, g, M ? &store : nullptr);
                L.desc = L.node->desc;
                return L;
            }
            return bb.leaf_on(type, sub(bb, g, s, g, s, store));
        };
        if (nd.split_type == DPP_SPLIT_ADDITIVE) {
            // the two children are independent: build B on the side stream from a
            // second host thread while A is built here (both pore networks of the
            // scale split, both AMG hierarchies of the field split's Schur leaf)
            N->side_owner.ensure(c);
            N->side = N->side_owner.s;
            fork_join(c, N->side_owner,
                      [&](Ctx *sc) {
                          Builder bb = *this;
                          bb.c = sc;
                          N->b = child(bb, nd.child_type[1], nd.child_node[1], gB, N->segB);
                      },
                      [&] { N->a = child(*this, nd.child_type[0], nd.child_node[0], gA, N->segA); }, FORK_ADDITIVE);
            CK(cudaEventCreateWithFlags(&N->ev_fork, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&N->ev_join, cudaEventDisableTiming));
            N->desc = "additive(" + N->a.desc + ", " + N->b.desc + ")";
            return N;
        }
        if (nd.split_type != DPP_SPLIT_SCHUR_FULL_SELFP) DPP_FAIL(DPP_ERR_VALUE, "unknown split type");
        Csr sA, sD, sB, sC;
        const Csr &A = sub(*this, gA, N->segA, gA, N->segA, sA);
        const Csr &D = sub(*this, gB, N->segB, gB, N->segB, sD);
        const Csr &B = sub(*this, gA, N->segA, gB, N->segB, sB);
        const Csr &C = sub(*this, gB, N->segB, gA, N->segA, sC);
        // diag_lump(A) (linalg.py:234-241) and selfp (linalg.py:244-254)
        DBuf<double> d(N->nA, c->s), dinv(N->nA, c->s);
        {
            DPP_TRACE_SCOPE(c, "pc.schur_diag");
            csr_diag(c, A, d.p, nullptr);
            if (any_zero_dev(c, N->nA, d.p)) DPP_FAIL(DPP_ERR_ZERO_PIVOT, "zero diagonal entry in diag_lump");
            reciprocal(c, N->nA, d.p, dinv.p);
        }
        Csr S;
        fork_join(c, N->side_owner,
                  [&](Ctx *sc) {   // the A-block leaf (ILU(0)) does not need S_p
                      Builder bb = *this;
                      bb.c = sc;
                      if (nd.child_type[0] == DPP_LEAF_NESTED) {
                          if (nd.child_node[0] < 0 || nd.child_node[0] >= n_nodes)
                              DPP_FAIL(DPP_ERR_VALUE, "bad nested split index");
                          N->a.type = DPP_LEAF_NESTED;
                          N->a.node = bb.node(nd.child_node[0], gA, &A);
                          N->a.desc = N->a.node->desc;
                      } else {
                          N->a = bb.leaf_on(nd.child_type[0], A);
                      }
                      // the coupling operators of the apply (zero-free copies + SpMV plans)
                      // are built here too, off the S_p -> AMG critical path
                      N->Bc = csr_drop_zeros(sc, B);
                      N->Cc = csr_drop_zeros(sc, C);
                      spmv_plan(sc, N->Bc);
                      spmv_plan(sc, N->Cc);
                  },
                  [&] {
                      {
                          DPP_TRACE_SCOPE(c, "pc.selfp_spgemm");
                          S = spgemm(c, C, B, dinv.p, true, &D);
                      }
                      if (nd.child_type[1] == DPP_LEAF_NESTED) {
                          if (nd.child_node[1] < 0 || nd.child_node[1] >= n_nodes)
                              DPP_FAIL(DPP_ERR_VALUE, "bad nested split index");
                          N->b.type = DPP_LEAF_NESTED;
                          N->b.node = node(nd.child_node[1], gB, &S);
                          N->b.desc = N->b.node->desc;
                      } else if (nd.child_type[1] == DPP_LEAF_AMG) {
                          // S_p is not needed after the hierarchy is built: it becomes level 0
                          N->b.type = DPP_LEAF_AMG;
                          N->b.amg = amg_setup(c, S, 0.5, 2.0 / 3.0, 64, 25, randn, user, &S);
                          N->b.desc = "amg[" + std::to_string(N->b.amg->lv.size()) + "]";
                      } else {
                          N->b = leaf_on(nd.child_type[1], S);
                      }
                  }, FORK_SCHUR);
        N->desc = "schur-full(" + N->a.desc + ", selfp->" + N->b.desc + ")";
        CK(cudaStreamSynchronize(c->s));
        return N;
    }
};

}  // namespace dpp

using namespace dpp;

struct dpp_pc {
    Ctx *ctx;
    std::unique_ptr<PcNode> root;
    int n = 0;
    DBuf<double> r, z;                 // fixed graph input / output
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int64_t kernels_per_apply = 0;
    double setup_ms = 0;
    ~dpp_pc() {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
    }
};

namespace dpp {

dpp_pc *pc_create(Ctx *c, dpp_system *s, const dpp_split_node *nodes, int n_nodes,
                  dpp_randn_fn randn, void *user, const Csr *K) {
    if (n_nodes < 1) DPP_FAIL(DPP_ERR_VALUE, "empty split tree");
    const int64_t ntot = s->sizes[0] + s->sizes[1] + s->sizes[2] + s->sizes[3];
    if (K && (K->rows != ntot || K->cols != ntot))
        DPP_FAIL(DPP_ERR_VALUE, "monolithic matrix does not match the system's field sizes");
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, c->s));
    auto pc = std::make_unique<dpp_pc>();
    pc->ctx = c;
    {
        DPP_TRACE_SCOPE(c, "pc.total");
        Builder b{c, nodes, n_nodes, s, randn, user};
        // K given: the tree's blocks are extracted from it by field index sets, as the reference
        // does with the matrix its caller passes (blocksolve.py:288-294); else from the system's blocks
        pc->root = b.node(0, {0, 1, 2, 3}, K);
    }
    pc->n = (int)(s->sizes[0] + s->sizes[1] + s->sizes[2] + s->sizes[3]);
    pc->r.alloc(pc->n, c->s);
    pc->z.alloc(pc->n, c->s);
    CK(cudaEventRecord(e1, c->s));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    pc->setup_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    TraceScope::ev_flush("pc_create");
    return pc.release();
}

// z_dev = M^-1 r_dev (device pointers; r_dev may be pc->r)
void pc_apply_dev(dpp_pc *pc, const double *r_dev, double *z_dev) {
    Ctx *c = pc->ctx;
    if (r_dev != pc->r.p)
        CK(cudaMemcpyAsync(pc->r.p, r_dev, sizeof(double) * pc->n, cudaMemcpyDeviceToDevice, c->s));
    static const bool nograph = [] { const char *e = std::getenv("DPP_PC_NOGRAPH"); return e && *e == '1'; }();
    if (nograph) {   // debugging / per-kernel instrumentation: plain stream launches
        const int64_t before = c->launches;
        pc->root->apply(c, pc->r.p, pc->z.p, c->s);
        pc->kernels_per_apply = c->launches - before;
        if (z_dev != pc->z.p)
            CK(cudaMemcpyAsync(z_dev, pc->z.p, sizeof(double) * pc->n, cudaMemcpyDeviceToDevice, c->s));
        return;
    }
    if (!pc->exec) {
        DPP_TRACE_SCOPE(c, "pc.capture_instantiate");
        const int64_t before = c->launches;
        CK(cudaStreamBeginCapture(c->s, cudaStreamCaptureModeThreadLocal));
        try {
            pc->root->apply(c, pc->r.p, pc->z.p, c->s);
        } catch (...) {
            cudaGraph_t g;
            cudaStreamEndCapture(c->s, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        CK(cudaStreamEndCapture(c->s, &pc->graph));
        CK(cudaGraphInstantiate(&pc->exec, pc->graph, 0));
        pc->kernels_per_apply = c->launches - before;
        c->launches = before;
    }
    if (TraceScope::on()) {   // device time of this apply (trace runs only)
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        CK(cudaEventRecord(e0, c->s));
        CK(cudaGraphLaunch(pc->exec, c->s));
        CK(cudaEventRecord(e1, c->s));
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        fprintf(stderr, "[dpp-trace]   pc apply graph %.3f ms (%lld kernels)\n", ms, (long long)pc->kernels_per_apply);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    } else
        CK(cudaGraphLaunch(pc->exec, c->s));
    c->launches += pc->kernels_per_apply;
    if (z_dev != pc->z.p)
        CK(cudaMemcpyAsync(z_dev, pc->z.p, sizeof(double) * pc->n, cudaMemcpyDeviceToDevice, c->s));
}

std::string pc_desc(const dpp_pc *pc) { return pc->root->desc; }
double pc_setup_ms(const dpp_pc *pc) { return pc->setup_ms; }
int pc_size(const dpp_pc *pc) { return pc->n; }
double *pc_in(dpp_pc *pc) { return pc->r.p; }
double *pc_out(dpp_pc *pc) { return pc->z.p; }
int64_t pc_kernels(const dpp_pc *pc) { return pc->kernels_per_apply; }
Ctx *pc_ctx(dpp_pc *pc) { return pc->ctx; }
void pc_destroy(dpp_pc *pc) { delete pc; }

}  // namespace dpp

// ---------------------------------------------------------------- algorithmic bytes
// B_spmv = 12 nnz_eff + 4 (r+1) + 8 c + 8 r ; B_tri = 12 nnz_eff(incl diag) + 4 (r+1) + 16 r
namespace dpp {
static double b_spmv(const Csr &A) { return 12.0 * A.nnz + 4.0 * (A.rows + 1) + 8.0 * A.cols + 8.0 * A.rows; }
static double b_tri(const Tri &T) {   // of the reference triangle, not of a merged form
    if (T.jacobi) {   // non-parity fast mode: init pass + k sweeps over the (scalar) strict part
        const double dg = T.diag.n ? 8.0 * T.strict.rows : 0.0;
        const double sweep = 12.0 * T.strict.nnz + 4.0 * (T.strict.rows + 1) + 24.0 * T.n + dg;
        return 16.0 * T.n + dg + T.jacobi * sweep;
    }
    const double nz = T.nnz_alg >= 0 ? (double)T.nnz_alg : (double)T.strict.nnz;
    return 12.0 * (nz + T.n) + 4.0 * (T.n + 1) + 16.0 * T.n;
}
static double leaf_bytes(const PcLeaf &L);
static double node_bytes(const PcNode &N) {
    if (N.split == DPP_SPLIT_ADDITIVE) return leaf_bytes(N.a) + leaf_bytes(N.b);
    return 2.0 * leaf_bytes(N.a) + leaf_bytes(N.b) + b_spmv(N.Bc) + b_spmv(N.Cc);
}
static double leaf_bytes(const PcLeaf &L) {
    if (L.type == DPP_LEAF_BJACOBI_ILU0) return b_tri(L.ilu->L) + b_tri(L.ilu->U);
    if (L.type == DPP_LEAF_AMG) {
        double b = 0;
        const Amg &h = *L.amg;
        for (size_t l = 0; l + 1 < h.lv.size(); ++l) {
            const AmgLevel &v = *h.lv[l];
            b += 4 * b_spmv(v.A) + 2 * (b_tri(v.lo) + b_tri(v.up)) + b_spmv(v.P) + b_spmv(v.R);
        }
        b += 8.0 * h.nc * h.nc + 16.0 * h.nc;
        return b;
    }
    return node_bytes(*L.node);
}
double pc_bytes(const dpp_pc *pc) { return node_bytes(*pc->root); }
double spmv_bytes(const Csr &A) { return b_spmv(A); }
}  // namespace dpp
