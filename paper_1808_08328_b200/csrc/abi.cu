// extern "C" entry points of libdpp (include/dpp.h).  Thin: validate, call
// the device layers, translate exceptions into status codes + dpp_last_error().
#include <chrono>
#include <climits>
#include <cstdio>

#include "abi_guard.cuh"
#include "system.cuh"

using namespace dpp;

std::string &dpp::last_error_ref() {
    static thread_local std::string e;
    return e;
}

struct dpp_ilu { Ctx *c; std::unique_ptr<Ilu> f; DBuf<double> r, z; };
struct dpp_amg { Ctx *c; std::unique_ptr<Amg> h; DBuf<double> r, z; };

// borrowed CSR views are plain dpp_csr objects whose matrix is referenced, not owned
struct CsrView { dpp_csr h; const Csr *ref; };
static const Csr &M(const dpp_csr *h) {
    if (!h) DPP_FAIL(DPP_ERR_VALUE, "null matrix handle");
    return h->m.rows < 0 ? *reinterpret_cast<const CsrView *>(h)->ref : h->m;
}
static dpp_csr *borrow(Ctx *c, const Csr &A) {
    auto *v = new CsrView;
    v->h.ctx = c;
    v->h.m.rows = -1;   // marks a view
    v->ref = &A;
    return &v->h;
}

// reads n 16-byte words and keeps the compiler from dropping the loads (the store never happens
// for a memset pattern): the read half of dpp_profile_step's L2 flush
__global__ void k_read_sink(const int4 *p, size_t n, int *sink) {
    int acc = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int4 v = p[i];
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x5a5a5a5b) *sink = acc;
}

extern "C" {

const char *dpp_last_error(void) { return last_error_ref().c_str(); }
int dpp_version(void) { return 1; }

int dpp_ctx_create(int device, dpp_ctx **out) {
    return guard([&] {
        int n = 0;
        CK(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) DPP_FAIL(DPP_ERR_CUDA, "no such CUDA device");
        CK(cudaSetDevice(device));
        auto *h = new dpp_ctx;
        h->c.device = device;
        CK(cudaDeviceGetAttribute(&h->c.sms, cudaDevAttrMultiProcessorCount, device));
        CK(cudaStreamCreateWithPriority(&h->c.s, cudaStreamNonBlocking, stream_priority(false)));
        CK(cudaStreamCreateWithPriority(&h->c.s2, cudaStreamNonBlocking, stream_priority(false)));
        CK(cudaMalloc(&h->c.nrm_part, sizeof(double) * NRM_BLOCKS));
        CK(cudaMalloc(&h->c.nrm_part2, sizeof(double) * NRM_BLOCKS));
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t thr = UINT64_MAX;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        *out = h;
    });
}

int dpp_ctx_destroy(dpp_ctx *ctx) {
    return guard([&] {
        if (!ctx) return;
        cudaStreamSynchronize(ctx->c.s);
        cudaFree(ctx->c.nrm_part);
        cudaFree(ctx->c.nrm_part2);
        cudaStreamDestroy(ctx->c.s);
        cudaStreamDestroy(ctx->c.s2);
        delete ctx;
    });
}

int dpp_timer_start(dpp_ctx *ctx) {
    return guard([&] {
        Ctx *c = &ctx->c;
        if (!c->t0) {
            CK(cudaEventCreate(&c->t0));
            CK(cudaEventCreate(&c->t1));
        }
        CK(cudaEventRecord(c->t0, c->s));
    });
}
int dpp_timer_stop(dpp_ctx *ctx, double *ms) {
    return guard([&] {
        Ctx *c = &ctx->c;
        if (!c->t0) DPP_FAIL(DPP_ERR_VALUE, "timer not started");
        CK(cudaEventRecord(c->t1, c->s));
        CK(cudaEventSynchronize(c->t1));
        float f = 0;
        CK(cudaEventElapsedTime(&f, c->t0, c->t1));
        *ms = f;
    });
}
int dpp_ctx_sync(dpp_ctx *ctx) { return guard([&] { CK(cudaStreamSynchronize(ctx->c.s)); }); }
int dpp_ctx_launches(const dpp_ctx *ctx, int64_t *count) {
    return guard([&] { *count = ctx->c.launches; });
}
int dpp_ctx_set_tri_jacobi(dpp_ctx *ctx, int sweeps) {
    return guard([&] {
        if (sweeps < 0 || sweeps > 64) DPP_FAIL(DPP_ERR_VALUE, "Jacobi sweep count must be in [0, 64]");
        ctx->c.tri_jacobi = sweeps;
    });
}

// ---------------------------------------------------------------- CSR
int dpp_csr_create(dpp_ctx *ctx, int rows, int cols, int64_t nnz, const int32_t *indptr,
                   const int32_t *indices, const double *data, dpp_csr **out) {
    return guard([&] {
        if (rows < 0 || cols < 0 || nnz < 0 || nnz > INT_MAX) DPP_FAIL(DPP_ERR_VALUE, "bad CSR shape");
        auto *h = new dpp_csr;
        h->ctx = &ctx->c;
        h->m = csr_from_host(&ctx->c, rows, cols, nnz, indptr, indices, data);
        CK(cudaStreamSynchronize(ctx->c.s));
        *out = h;
    });
}
int dpp_csr_info(const dpp_csr *A, int *rows, int *cols, int64_t *nnz) {
    return guard([&] {
        const Csr &m = M(A);
        if (rows) *rows = m.rows;
        if (cols) *cols = m.cols;
        if (nnz) *nnz = m.nnz;
    });
}
int dpp_csr_download(const dpp_csr *A, int32_t *indptr, int32_t *indices, double *data) {
    return guard([&] {
        const Csr &m = M(A);
        if (indptr) m.ptr.download(indptr, m.rows + 1);
        if (indices) m.idx.download(indices, m.nnz);
        if (data) m.val.download(data, m.nnz);
        CK(cudaStreamSynchronize(A->ctx->s));
    });
}
int dpp_csr_destroy(dpp_csr *A) {
    return guard([&] {
        if (!A) return;
        if (A->m.rows < 0) delete reinterpret_cast<CsrView *>(A);
        else delete A;
    });
}
int dpp_csr_plan(dpp_csr *A, int kind) {
    return guard([&] {
        if (!A || A->m.rows < 0) DPP_FAIL(DPP_ERR_VALUE, "dpp_csr_plan needs an owned matrix");
        if (kind < 0 || kind > 3) DPP_FAIL(DPP_ERR_VALUE, "unknown SpMV plan kind");
        spmv_plan(A->ctx, A->m, kind);
        CK(cudaStreamSynchronize(A->ctx->s));
    });
}
int dpp_spmv(dpp_ctx *ctx, const dpp_csr *A, const double *x, double *y) {
    return guard([&] {
        Ctx *c = &ctx->c;
        const Csr &m = M(A);
        DBuf<double> dx(m.cols, c->s), dy(m.rows, c->s);
        dx.upload(x, m.cols);
        if (m.rows) {
            if (m.nnz) spmv(c, m, dx.p, dy.p);
            else fill(c, dy.p, m.rows, 0.0);
        }
        dy.download(y, m.rows);
        CK(cudaStreamSynchronize(c->s));
    });
}

// ---------------------------------------------------------------- systems
int dpp_system_from_blocks(dpp_ctx *ctx, const dpp_csr *const blocks[10], const double *const rhs[4],
                           const int64_t sizes[4], dpp_system **out) {
    return guard([&] {
        Ctx *c = &ctx->c;
        auto s = std::make_unique<dpp_system>();
        s->ctx = c;
        for (int k = 0; k < 4; ++k) s->sizes[k] = sizes[k];
        // block (row field, col field) of each id
        static const int rf[10] = {0, 0, 1, 1, 2, 2, 3, 3, 1, 3};
        static const int cf[10] = {0, 1, 0, 1, 2, 3, 2, 3, 3, 1};
        for (int b = 0; b < 10; ++b) {
            if (blocks[b]) {
                const Csr &m = M(blocks[b]);
                if (m.rows != sizes[rf[b]] || m.cols != sizes[cf[b]])
                    DPP_FAIL(DPP_ERR_VALUE, "block shape does not match field sizes");
                s->blk[b] = csr_copy(c, m);
            } else {
                s->blk[b] = csr_empty(c, (int)sizes[rf[b]], (int)sizes[cf[b]]);
            }
        }
        for (int k = 0; k < 4; ++k) {
            s->rhs[k].alloc(sizes[k], c->s);
            if (rhs[k]) s->rhs[k].upload(rhs[k], sizes[k]);
            else if (sizes[k]) CK(cudaMemsetAsync(s->rhs[k].p, 0, sizeof(double) * sizes[k], c->s));
        }
        CK(cudaStreamSynchronize(c->s));
        *out = s.release();
    });
}
int dpp_system_sizes(const dpp_system *s, int64_t sizes[4]) {
    return guard([&] { for (int k = 0; k < 4; ++k) sizes[k] = s->sizes[k]; });
}
int dpp_system_block(dpp_system *s, int block, dpp_csr **out) {
    return guard([&] {
        if (block < 0 || block > 9) DPP_FAIL(DPP_ERR_VALUE, "block id");
        *out = borrow(s->ctx, s->blk[block]);
    });
}
int dpp_system_rhs(const dpp_system *s, int field, double *out) {
    return guard([&] {
        if (field < 0 || field > 3) DPP_FAIL(DPP_ERR_VALUE, "field id");
        s->rhs[field].download(out, s->sizes[field]);
        CK(cudaStreamSynchronize(s->ctx->s));
    });
}
int dpp_system_monolithic(dpp_system *s, dpp_csr **out) {
    return guard([&] {
        const Csr &K = system_K(s->ctx, s);
        CK(cudaStreamSynchronize(s->ctx->s));
        *out = borrow(s->ctx, K);
    });
}
int dpp_system_timing(const dpp_system *s, double *ms) { return guard([&] { *ms = s->assembly_ms; }); }
int dpp_system_destroy(dpp_system *s) {
    return guard([&] {
        if (!s) return;
        cudaStreamSynchronize(s->ctx->s);
        delete s;
    });
}

// ---------------------------------------------------------------- ILU(0)
int dpp_ilu0_create(dpp_ctx *ctx, const dpp_csr *A, dpp_ilu **out) {
    return guard([&] {
        auto h = std::make_unique<dpp_ilu>();
        h->c = &ctx->c;
        h->f = ilu0(&ctx->c, M(A));
        h->r.alloc(h->f->n, ctx->c.s);
        h->z.alloc(h->f->n, ctx->c.s);
        CK(cudaStreamSynchronize(ctx->c.s));
        *out = h.release();
    });
}
int dpp_ilu0_apply(dpp_ilu *f, const double *r, double *z) {
    return guard([&] {
        f->r.upload(r, f->f->n);
        ilu_apply(f->c, *f->f, f->r.p, f->z.p);
        f->z.download(z, f->f->n);
        CK(cudaStreamSynchronize(f->c->s));
    });
}
int dpp_ilu0_factors(dpp_ilu *f, dpp_csr **L, dpp_csr **U) {
    return guard([&] {
        Ctx *c = f->c;
        const int n = f->f->n;
        // U = triu(LU) keeps stored zeros; L = tril(LU,-1) + I drops them (scipy '+')
        auto *hu = new dpp_csr;
        hu->ctx = c;
        hu->m = csr_part(c, f->f->LU, 3, false);
        Csr Ls = csr_part(c, f->f->LU, -1, true);
        std::vector<int> p = Ls.ptr.to_host(), ix = Ls.idx.to_host();
        std::vector<double> v = Ls.val.to_host();
        std::vector<int> p2(n + 1), ix2;
        std::vector<double> v2;
        ix2.reserve(ix.size() + n);
        v2.reserve(ix.size() + n);
        p2[0] = 0;
        for (int i = 0; i < n; ++i) {
            for (int q = p[i]; q < p[i + 1]; ++q) { ix2.push_back(ix[q]); v2.push_back(v[q]); }
            ix2.push_back(i);
            v2.push_back(1.0);
            p2[i + 1] = (int)ix2.size();
        }
        auto *hl = new dpp_csr;
        hl->ctx = c;
        hl->m = csr_from_host(c, n, n, (int64_t)ix2.size(), p2.data(), ix2.data(), v2.data());
        CK(cudaStreamSynchronize(c->s));
        *L = hl;
        *U = hu;
    });
}
int dpp_ilu0_destroy(dpp_ilu *f) {
    return guard([&] {
        if (!f) return;
        cudaStreamSynchronize(f->c->s);
        delete f;
    });
}

// ---------------------------------------------------------------- selfp
int dpp_diag(dpp_ctx *ctx, const dpp_csr *A, double *out) {
    return guard([&] {
        const Csr &m = M(A);
        const int n = std::min(m.rows, m.cols);
        DBuf<double> d(n, ctx->c.s);
        csr_diag(&ctx->c, m, d.p, nullptr);
        d.download(out, n);
        CK(cudaStreamSynchronize(ctx->c.s));
    });
}
int dpp_schur_selfp(dpp_ctx *ctx, const dpp_csr *D, const dpp_csr *C, const double *diagA,
                    const dpp_csr *B, dpp_csr **out) {
    return guard([&] {
        Ctx *c = &ctx->c;
        const Csr &d = M(D), &cc = M(C), &b = M(B);
        const int n = cc.cols;
        for (int i = 0; i < n; ++i)
            if (diagA[i] == 0.0) DPP_FAIL(DPP_ERR_ZERO_PIVOT, "zero entry in diagA");
        if (b.rows != n || d.rows != cc.rows || d.cols != b.cols)
            DPP_FAIL(DPP_ERR_VALUE, "schur_selfp: non-conforming block dimensions");
        DBuf<double> da(n, c->s), dinv(n, c->s);
        da.upload(diagA, n);
        reciprocal(c, n, da.p, dinv.p);
        auto *h = new dpp_csr;
        h->ctx = c;
        h->m = spgemm(c, cc, b, dinv.p, true, &d);
        CK(cudaStreamSynchronize(c->s));
        *out = h;
    });
}

// ---------------------------------------------------------------- AMG
int dpp_amg_create(dpp_ctx *ctx, const dpp_csr *A, double theta, double omega, int max_coarse,
                   int max_levels, dpp_randn_fn randn, void *user, dpp_amg **out) {
    return guard([&] {
        auto h = std::make_unique<dpp_amg>();
        h->c = &ctx->c;
        h->h = amg_setup(&ctx->c, M(A), theta, omega, max_coarse, max_levels, randn, user);
        const int n = M(A).rows;
        h->r.alloc(n, ctx->c.s);
        h->z.alloc(n, ctx->c.s);
        CK(cudaStreamSynchronize(ctx->c.s));
        *out = h.release();
    });
}
int dpp_strength_aggregates(dpp_ctx *ctx, const dpp_csr *A, double theta, int path, int64_t *agg_host,
                            int64_t *n_agg) {
    return guard([&] {
        DBuf<int> agg;
        *n_agg = strength_aggregates(&ctx->c, M(A), theta, path, agg);
        TraceScope::ev_flush("strength_aggregates");
        std::vector<int> a = agg.to_host();
        std::copy(a.begin(), a.end(), agg_host);
    });
}
int dpp_amg_levels(const dpp_amg *h, int *levels) { return guard([&] { *levels = (int)h->h->lv.size(); }); }
int dpp_amg_level(dpp_amg *h, int level, dpp_csr **A, dpp_csr **P, int64_t *agg, double *rho) {
    return guard([&] {
        if (level < 0 || level >= (int)h->h->lv.size()) DPP_FAIL(DPP_ERR_VALUE, "level out of range");
        AmgLevel &L = *h->h->lv[level];
        const bool coarsest = level + 1 == (int)h->h->lv.size();
        if (A) *A = borrow(h->c, L.A);
        if (P) *P = coarsest ? nullptr : borrow(h->c, L.P);
        if (agg && !coarsest) {
            std::vector<int> a = L.agg.to_host();
            std::copy(a.begin(), a.end(), agg);
        }
        if (rho) *rho = L.rho;
    });
}
int dpp_amg_vcycle(dpp_amg *h, const double *r, double *z) {
    return guard([&] {
        const int n = h->h->lv[0]->A.rows;
        h->r.upload(r, n);
        amg_vcycle(h->c, *h->h, h->r.p, h->z.p);
        h->z.download(z, n);
        CK(cudaStreamSynchronize(h->c->s));
    });
}
int dpp_amg_destroy(dpp_amg *h) {
    return guard([&] {
        if (!h) return;
        cudaStreamSynchronize(h->c->s);
        delete h;
    });
}

// ---------------------------------------------------------------- preconditioner
int dpp_pc_create(dpp_ctx *ctx, dpp_system *s, const dpp_split_node *nodes, int n_nodes,
                  dpp_randn_fn randn, void *user, dpp_pc **out) {
    return guard([&] { *out = pc_create(&ctx->c, s, nodes, n_nodes, randn, user); });
}
int dpp_pc_create_explicit(dpp_ctx *ctx, dpp_system *s, const dpp_csr *K, const dpp_split_node *nodes,
                           int n_nodes, dpp_randn_fn randn, void *user, dpp_pc **out) {
    return guard([&] { *out = pc_create(&ctx->c, s, nodes, n_nodes, randn, user, &K->m); });
}
int dpp_pc_apply(dpp_pc *pc, const double *r, double *z) {
    return guard([&] {
        const int n = pc_size(pc);
        Ctx *c = pc_ctx(pc);
        CK(cudaMemcpyAsync(pc_in(pc), r, sizeof(double) * n, cudaMemcpyHostToDevice, c->s));
        pc_apply_dev(pc, pc_in(pc), pc_out(pc));
        CK(cudaMemcpyAsync(z, pc_out(pc), sizeof(double) * n, cudaMemcpyDeviceToHost, c->s));
        CK(cudaStreamSynchronize(c->s));
    });
}
int dpp_pc_describe(const dpp_pc *pc, char *buf, int cap) {
    return guard([&] {
        std::string d = pc_desc(pc);
        if (cap > 0) {
            std::snprintf(buf, (size_t)cap, "%s", d.c_str());
        }
    });
}
int dpp_pc_setup_ms(const dpp_pc *pc, double *ms) { return guard([&] { *ms = pc_setup_ms(pc); }); }
int dpp_pc_destroy(dpp_pc *pc) {
    return guard([&] {
        if (!pc) return;
        cudaDeviceSynchronize();
        pc_destroy(pc);
    });
}

// ---------------------------------------------------------------- GMRES
int dpp_gmres(dpp_ctx *ctx, const dpp_csr *A, dpp_apply_fn A_cb, void *A_user, dpp_pc *pc,
              dpp_apply_fn pc_cb, void *pc_user, int64_t n, const double *b, const double *x0,
              double *x, double rtol, int max_iter, int restart, dpp_krylov_stats *stats,
              double *history, int history_cap) {
    return guard([&] {
        Ctx *c = &ctx->c;
        if (restart < 1) DPP_FAIL(DPP_ERR_VALUE, "restart must be >= 1");
        Operator op;
        if (A) {
            op.A = &M(A);
            if (op.A->rows != n || op.A->cols != n) DPP_FAIL(DPP_ERR_VALUE, "operator shape mismatch");
        } else if (A_cb) {
            op.cb = A_cb;
            op.user = A_user;
        } else {
            DPP_FAIL(DPP_ERR_VALUE, "no operator");
        }
        PcOp pm;
        pm.pc = pc;
        pm.cb = pc ? nullptr : pc_cb;
        pm.user = pc_user;
        if (pc && pc_size(pc) != n) DPP_FAIL(DPP_ERR_VALUE, "preconditioner size mismatch");
        DBuf<double> db(n, c->s), dx(n, c->s);
        db.upload(b, n);
        if (x0) dx.upload(x0, n);
        else if (n) CK(cudaMemsetAsync(dx.p, 0, sizeof(double) * n, c->s));
        std::vector<double> hist;
        gmres_dev(c, n, op, pm, db.p, dx.p, rtol, max_iter, restart, stats, &hist, x0 == nullptr);
        dx.download(x, n);
        CK(cudaStreamSynchronize(c->s));
        for (int i = 0; i < (int)hist.size() && i < history_cap; ++i) history[i] = hist[i];
    });
}

int dpp_solve(dpp_ctx *ctx, dpp_system *s, dpp_pc *pc, double rtol, int max_iter, int restart,
              double *x, dpp_krylov_stats *stats, double *history, int history_cap) {
    return guard([&] {
        Ctx *c = &ctx->c;
        const Csr &Kc = system_Kc(c, s);
        const double *f = system_f(c, s);
        const int64_t n = Kc.rows;
        Operator op;
        op.A = &Kc;
        PcOp pm;
        pm.pc = pc;
        DBuf<double> dx(n, c->s);
        if (n) CK(cudaMemsetAsync(dx.p, 0, sizeof(double) * n, c->s));
        std::vector<double> hist;
        {
            DPP_TRACE_SCOPE(c, "solve.gmres");
            gmres_dev(c, n, op, pm, f, dx.p, rtol, max_iter, restart, stats, &hist, true);
        }
        if (x) dx.download(x, n);
        CK(cudaStreamSynchronize(c->s));
        for (int i = 0; i < (int)hist.size() && i < history_cap; ++i) history[i] = hist[i];
    });
}

// ---------------------------------------------------------------- measurement
int dpp_profile_step(dpp_ctx *ctx, dpp_system *s, dpp_pc *pc, int reps, int flush_l2,
                     dpp_step_profile *out) {
    return guard([&] {
        // L2 flush between timed launches: 256 MiB written, then read back -- the read pass evicts the
        // dirty lines the write left behind, so the timed kernel starts on a cold *and clean* L2 (with
        // only the write, ~120 MB of write-backs drained during the 50 us SpMV and inflated it by ~10 us)
        auto flush = [&](Ctx *c, char *junk, size_t fl, int v) {
            if (!fl) return;
            CK(cudaMemsetAsync(junk, v & 0xff, fl, c->s));
            k_read_sink<<<c->sms * 8, 256, 0, c->s>>>(reinterpret_cast<const int4 *>(junk), fl / 16, (int *)junk);
        };
        Ctx *c = &ctx->c;
        const Csr &Kc = system_Kc(c, s);
        const int64_t n = Kc.rows;
        DBuf<double> x(n, c->s), y(n, c->s);
        fill(c, x.p, n, 1.0);
        const size_t fl = flush_l2 ? (size_t)256 << 20 : 0;   // 256 MiB > 126 MB L2
        DBuf<char> junk(fl, c->s);
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        double t_spmv = 0, t_pc = 0;
        // warm-up (also captures the PC graph)
        spmv(c, Kc, x.p, pc_in(pc));
        pc_apply_dev(pc, pc_in(pc), pc_out(pc));
        CK(cudaStreamSynchronize(c->s));
        for (int r = 0; r < reps; ++r) {
            flush(c, junk.p, fl, r);
            CK(cudaEventRecord(a, c->s));
            spmv(c, Kc, x.p, pc_in(pc));
            CK(cudaEventRecord(b, c->s));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            t_spmv += ms;
            flush(c, junk.p, fl, r + 1);
            CK(cudaEventRecord(a, c->s));
            pc_apply_dev(pc, pc_in(pc), pc_out(pc));
            CK(cudaEventRecord(b, c->s));
            CK(cudaEventSynchronize(b));
            CK(cudaEventElapsedTime(&ms, a, b));
            t_pc += ms;
        }
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        out->spmv_ms = t_spmv / reps;
        out->pc_ms = t_pc / reps;
        out->spmv_bytes = spmv_bytes(Kc);
        out->pc_bytes = pc_bytes(pc);
        out->mgs_ms = 0;
        out->pc_launches = pc_kernels(pc);
    });
}

}  // extern "C"
