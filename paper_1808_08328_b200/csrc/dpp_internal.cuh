// libdpp internals: context, device buffers, device CSR, shared kernel helpers.
// sm_100a, FP64.  See DESIGN.md for the data layout in HBM.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/dpp.h"

namespace dpp {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

#define DPP_FAIL(code, msg) throw ::dpp::Error((code), (msg))
#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess)                                                                  \
            throw ::dpp::Error(DPP_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));  \
    } while (0)

struct Ctx {
    int device = 0;
    int sms = 148;
    cudaStream_t s = nullptr;    // main stream
    cudaStream_t s2 = nullptr;   // fork stream (concurrent branches of additive splits)
    int64_t launches = 0;        // libdpp kernels launched (incl. graph replays' kernels)
    int capturing = 0;
    double *nrm_part = nullptr;  // NRM_BLOCKS partial sums (norm reductions on s)
    double *nrm_part2 = nullptr; // same for s2
    cudaEvent_t t0 = nullptr, t1 = nullptr;   // dpp_timer_*
    int tri_jacobi = 0;          // non-parity fast mode: triangular solves built at setup become
                                 // this many Jacobi sweeps (0 = exact substitution, the reference)
};
constexpr int NRM_BLOCKS = 296;

// Optional phase tracer (DPP_TRACE=1): synchronises the stream at scope
// boundaries and prints wall-clock milliseconds per named phase to stderr.
struct TraceScope {
    Ctx *c;
    const char *name;
    double t0;
    static bool on();
    static double now();
    cudaEvent_t ev0 = nullptr;   // DPP_TRACE=ev: events on the scope's stream, no syncs
    static bool ev_on();
    static void ev_flush(const char *title);   // resolve + print every recorded scope (stream idle)
    TraceScope(Ctx *cc, const char *n) : c(cc), name(n), t0(0) {
        if (on()) { cudaStreamSynchronize(c->s); t0 = now(); }
        else if (ev_on()) ev_begin();
    }
    ~TraceScope();
    void ev_begin();
};
#define DPP_CAT2(a, b) a##b
#define DPP_CAT(a, b) DPP_CAT2(a, b)
#define DPP_TRACE_SCOPE(c, name) ::dpp::TraceScope DPP_CAT(dpp_trace_scope_, __LINE__)((c), (name))

// Programmatic dependent launch (PC-apply kernels): a kernel launched with
// launch_pdl may start while its predecessor in the stream runs; it triggers its own
// dependents at entry and waits (griddepcontrol.wait) before touching any data the
// predecessor produces or reads.  Both are no-ops for ordinary launches.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_on();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_on() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Checked build (-DDPP_CHECKED, tools/checked_build.sh): device-side bounds / invariant checks in
// the lock-free kernels (shared-memory slot ranges, push targets, ring offsets, dependency ids);
// a violated check traps.  Stands in for compute-sanitizer, which is closed on the GPU pool.
#ifdef DPP_CHECKED
#define DPP_DCHECK(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define DPP_DCHECK(cond) do { } while (0)
#endif

// record one kernel launch (checks launch errors outside graph capture)
inline void launched(Ctx *c) {
    c->launches++;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error(DPP_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
}

// Stream-ordered device buffer.
// process-wide pool of pinned host staging buffers (never freed; first fit)
struct PinnedBuf {
    void *p = nullptr;
    size_t cap = 0;
};
constexpr size_t PINNED_MIN = 64 * 1024;
PinnedBuf pinned_acquire(size_t bytes);
void pinned_release(PinnedBuf b);

template <typename T>
struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    DBuf() = default;
    DBuf(size_t count, cudaStream_t st) { alloc(count, st); }
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    DBuf(DBuf &&o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
    DBuf &operator=(DBuf &&o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; s = o.s; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(size_t count, cudaStream_t st) {
        release();
        s = st;
        n = count;
        if (count) {
            cudaError_t e = cudaMallocAsync((void **)&p, sizeof(T) * count, st);
            if (e != cudaSuccess)
                throw Error(DPP_ERR_ALLOC, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
        }
    }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
    // transfers >= PINNED_MIN bytes go through pinned staging buffers (pinned_acquire):
    // pageable copies are staged by the driver and serialise across the setup threads
    void upload(const T *h, size_t count) {
        if (!count) return;
        const size_t bytes = sizeof(T) * count;
        if (bytes < PINNED_MIN) {
            CK(cudaMemcpyAsync(p, h, bytes, cudaMemcpyHostToDevice, s));
            return;
        }
        PinnedBuf b = pinned_acquire(bytes);
        std::memcpy(b.p, h, bytes);
        CK(cudaMemcpyAsync(p, b.p, bytes, cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));   // the staging buffer is reused after this
        pinned_release(b);
    }
    void download(T *h, size_t count) const {
        if (!count) return;
        const size_t bytes = sizeof(T) * count;
        if (bytes < PINNED_MIN) {
            CK(cudaMemcpyAsync(h, p, bytes, cudaMemcpyDeviceToHost, s));
            return;
        }
        PinnedBuf b = pinned_acquire(bytes);
        CK(cudaMemcpyAsync(b.p, p, bytes, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        std::memcpy(h, b.p, bytes);
        pinned_release(b);
    }
    std::vector<T> to_host() const {
        std::vector<T> v(n);
        download(v.data(), n);
        CK(cudaStreamSynchronize(s));
        return v;
    }
};

// Device CSR (int32 indices, FP64 values), scipy storage semantics.
struct Csr {
    int rows = 0, cols = 0;
    int64_t nnz = 0;
    DBuf<int> ptr, idx;
    DBuf<double> val;
    // optional SpMV plans (spmv_plan), preferred in this order:
    DBuf<int> sp;         // SELL-32: slice k = rows [32k, 32k+32), entries sp[k] .. sp[k+1]
    DBuf<int> sc;         //   column of (slice k, column t, lane l) at sp[k] + 32 t + l
    DBuf<double> sv;      //   value (padding: 0.0 with a valid column)
    DBuf<uint16_t> sc16;  //   or 16-bit column codes (sc then empty): sel = code >> 14,
    DBuf<int4> sbase;     //   column = sbase[k][sel] + (code & 0x3fff)
    int nsl = 0;
    DBuf<int> rb;         // CSR-stream row blocks: block k = rows starting in [k*T, (k+1)*T)
    int nrb = 0;
    void alloc(int r, int c, int64_t z, cudaStream_t s) {
        rb.release(); nrb = 0;
        sp.release(); sc.release(); sv.release(); sc16.release(); sbase.release(); nsl = 0;
        rows = r; cols = c; nnz = z;
        ptr.alloc((size_t)r + 1, s);
        idx.alloc((size_t)z, s);
        val.alloc((size_t)z, s);
    }
};

// ---- host task parallelism for setup ----------------------------------------
// A side stream plus a context view bound to it.  Objects built through the
// view allocate (and later free) on the side stream, so the owner of those
// objects must also own the SideStream and destroy it last.
// stream priorities: setup work off the critical path (smoother plans, the ILU branch)
// runs on low-priority streams so the AMG level chain's small kernels are scheduled first
int stream_priority(bool low);
struct SideStream {
    cudaStream_t s = nullptr;
    int low = 0;
    Ctx ctx;
    void ensure(Ctx *parent, bool low_prio = false);
    ~SideStream();
};
// run side(view) on a host thread with the side stream while main_fn() runs here
// kind: FORK_ADDITIVE / FORK_SCHUR (DPP_FORK_MASK bits; DPP_SERIAL_SETUP=1 clears all)
constexpr int FORK_ADDITIVE = 1, FORK_SCHUR = 2, FORK_AMG_SMOOTHER = 4;
int fork_mask();
void fork_join(Ctx *c, SideStream &owner, const std::function<void(Ctx *)> &side,
               const std::function<void()> &main_fn, int kind);

int64_t counts_to_ptr(Ctx *c, const int *counts, int n, DBuf<int> &ptr);
// counts[n] -> ptr[n+1] without a read back (caller bounds the total below 2^31)
void scan_to_ptr32(Ctx *c, const int *counts, int n, int *ptr);

inline int grid_for(int64_t work, int block, int sms, int per_sm = 16) {
    int64_t g = (work + block - 1) / block;
    int64_t cap = (int64_t)sms * per_sm;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

// ---- core sparse / vector ops (core.cu) -----------------------------------
void spmv(Ctx *c, const Csr &A, const double *x, double *y, const double *b = nullptr,
          double alpha = 1.0, cudaStream_t st = nullptr);   // y = b + alpha*A x (b may be null)
// row-block partition for the nnz-streaming SpMV (operators applied many times)
// kind: 0 none (row kernel), 1 CSR-stream, 2 SELL-32 (any fill), 3 auto (SELL when the
// padding stays small, else CSR-stream; DPP_SPMV=row|stream overrides)
void spmv_plan(Ctx *c, Csr &A, int kind = 3);
void fill(Ctx *c, double *x, int64_t n, double v, cudaStream_t st = nullptr);
void axpy(Ctx *c, int64_t n, double a, const double *x, double *y, cudaStream_t st = nullptr);
void axpby_to(Ctx *c, int64_t n, const double *x, double a, const double *y, double *out,
              cudaStream_t st = nullptr);                    // out = x + a*y
void scale_by_dev(Ctx *c, int64_t n, const double *x, const double *num, double *out,
                  cudaStream_t st = nullptr);                // out = x / *num
void norm2_dev(Ctx *c, int64_t n, const double *x, double *out_dev, cudaStream_t st = nullptr);
double norm2(Ctx *c, int64_t n, const double *x);
void copy_segments(Ctx *c, double *dst, const double *src, int nseg, const int64_t *dst_off,
                   const int64_t *src_off, const int64_t *len, cudaStream_t st = nullptr);
Csr csr_from_host(Ctx *c, int rows, int cols, int64_t nnz, const int *ptr, const int *idx,
                  const double *val);
Csr csr_copy(Ctx *c, const Csr &A);
Csr csr_empty(Ctx *c, int rows, int cols);
Csr csr_drop_zeros(Ctx *c, const Csr &A);
// part: -1 strict lower, 0 diag only, +1 strict upper, 2 lower incl diag, 3 upper incl diag
Csr csr_part(Ctx *c, const Csr &A, int part, bool drop_zeros);
void csr_diag(Ctx *c, const Csr &A, double *d_out, int *missing_dev);
// any exact zero among d[0..n) (one 4-byte read back instead of the whole vector)
bool any_zero_dev(Ctx *c, int64_t n, const double *d);
Csr csr_transpose(Ctx *c, const Csr &A);
// rows/cols selected by segment lists of the parent index space (order preserving)
Csr csr_submatrix(Ctx *c, const Csr &M, const std::vector<std::pair<int, int>> &rowseg,
                  const std::vector<std::pair<int, int>> &colseg);
// block grid (4x4 of optional blocks) -> one CSR (sp.bmat semantics, sorted, zeros kept)
Csr csr_bmat(Ctx *c, const std::vector<const Csr *> &grid, int nbr, int nbc,
             const std::vector<int> &rsz, const std::vector<int> &csz);
int64_t csr_count_nonzero(Ctx *c, const Csr &A);

// ---- SpGEMM (spgemm.cu) ----------------------------------------------------
// C = D - (A*diag(s)) * B or C = A * B with the reference's accumulation order:
// for each output row, products are accumulated over A's row entries in storage
// order (descending when `reverse`), a'_ik = fl(a_ik * s_k) when s given,
// acc = fl(acc + fl(a' * b)), exact zeros dropped (scipy csr_matmat / csr_binop).
Csr spgemm(Ctx *c, const Csr &A, const Csr &B, const double *s_dev, bool reverse,
           const Csr *D, bool keep_zeros = false);

// ---- triangular solves and ILU(0) (trsv.cu) --------------------------------
struct ClusterPlan {      // level-ordered per-CTA blocks for the cluster sweep (tricluster.cu)
    int C = 0, chunk = 0, L = 0, G = 32, stage = 0, nst = 0, threads = 1024;
    DBuf<unsigned char> blocks;
    DBuf<long long> boff;
};
struct PushPlan {         // cluster sweep with st.async point-to-point x exchange (tripush.cu)
    int C = 0, chunk = 0, L = 0, G = 32, stage = 0, nst = 0, threads = 1024, hmax = 0, smax = 0;
    DBuf<unsigned char> blocks;
    DBuf<long long> boff; // per step (CTA-major)
    DBuf<int> sstart;     // first step of each CTA
    DBuf<int> tx;         // bytes each CTA receives per level
    DBuf<int> lrows;      // rows of each (CTA, level)
    DBuf<int> slev;       // fmt 1: level of each step
    int widest = 1;       // most rows (fmt 1: 32-row chunks) in one block (step)
    int fmt = 0;          // block format: 0 row-major (k_trsv_flow / k_trsv_push), 1 SELL chunks (k_trsv_lvl),
                          // 2 warp streams (k_trsv_ws), 3 global streams (k_trsv_gs)
    // multi-cluster global streams (C > 16 CTA slices in clusters of 16): sources in another cluster
    // are imported from x in global memory by an extra warp of the consumer CTA
    DBuf<unsigned long long> imp;   // (source row << 32 | halo slot), by consumer CTA and source level
    DBuf<int> istart;               // first import entry of each CTA slice (C + 1)
};
struct BlockPlan {        // block-sequential sweep with dense diagonal-block inverses (triblock.cu)
    int nblk = 0, stage = 0, nst = 0;
    DBuf<unsigned char> blocks;
    DBuf<long long> boff;
};
struct BdPlan {           // block-dense sweep: per-(block, CTA) segments of inverse rows + off-block CSR (tribd.cu)
    int B = 0, nb = 0, C = 0, W = 0, stage = 0, nst = 0;
    DBuf<unsigned char> segs;
    DBuf<long long> soff;
};
struct GbdPlan {          // global block-dense sweep: dense diagonal-block inverses + off-block CSR, two launches per block (tribd.cu)
    int B = 0, nb = 0;
    DBuf<double> dinv;    // nb x B x B, row-major, inverse of every diagonal block
    Csr off;              // strict entries outside the row's diagonal block
    DBuf<double> y;       // b - off x of the current block
};
struct Tri {              // one sweep: strict part (zero-free) + optional diagonal
    Csr strict;
    DBuf<double> diag;    // empty -> unit diagonal
    DBuf<int> order;      // rows in (dependency level, row) order: the sweep's ticket order
    DBuf<int> levptr;     // level l = order[levptr[l] .. levptr[l+1])
    std::unique_ptr<ClusterPlan> cl;   // cluster-resident sweep when x fits in one cluster
    std::unique_ptr<PushPlan> pu;      // cluster-resident sweep, push exchange (preferred)
    std::unique_ptr<BlockPlan> bl;     // block-sequential sweep (small n, narrow levels)
    std::unique_ptr<BdPlan> bd;        // block-dense sweep (AMG smoother factors)
    std::unique_ptr<GbdPlan> gbd;      // global block-dense sweep (long-row factors too large for one cluster's window)
    DBuf<double> dense;   // optional dense inverse (small coarse levels): sweep = triangular GEMV
    int ncomp = 1;        // Kronecker form: the triangle is this one (x) I_ncomp, rows interleaved
    Csr W;                // level-merged form (merge_levels): x = solve_unit(strict, W b)
    DBuf<double> wb;      //   scratch for W b
    DBuf<double> wb2;     // Jacobi mode: x0 = D^-1 b
    int64_t nnz_alg = -1; // stored entries of the original strict triangle (algorithmic bytes)
    int jacobi = 0;       // non-parity fast mode: x = k Jacobi sweeps on (strict, diag), ncomp-interleaved
    bool backward = false;
    int n = 0, nlev = 0;
};
// dependency levels of a strict triangle -> topological (level, row) order
int tri_levels(Ctx *c, const Csr &strict, bool backward, DBuf<int> &order, DBuf<int> *levptr = nullptr,
               DBuf<int> *lev_out = nullptr);
bool cluster_plan(Ctx *c, Tri &T, const DBuf<int> &lev, int L);
bool push_plan(Ctx *c, Tri &T, const DBuf<int> &lev, int L);
void trsv_push(Ctx *c, const Tri &T, const double *b, double *x, const double *xadd, double *xout,
               cudaStream_t st);
bool block_plan(Ctx *c, Tri &T);
bool bd_plan(Ctx *c, Tri &T, int B);
void tri_dense_inverse(Ctx *c, Tri &T);
void trsv_bd(Ctx *c, const Tri &T, const double *b, double *x, const double *xadd, double *xout,
             cudaStream_t st);
bool gbd_plan(Ctx *c, Tri &T, int B);
void trsv_gbd(Ctx *c, const Tri &T, const double *b, double *x, const double *xadd, double *xout,
              cudaStream_t st);
void trsv_block(Ctx *c, const Tri &T, const double *b, double *x, const double *xadd, double *xout,
                cudaStream_t st);
void trsv_cluster(Ctx *c, const Tri &T, const double *b, double *x, const double *xadd, double *xout,
                  cudaStream_t st);
constexpr int DENSE_TRI_MAX = 4096;   // dense inverse up to 134 MB per factor: a sweep is one GEMV
// pre_order / pre_lev: a level analysis of a superset pattern of this triangle
// (e.g. ILU(0)'s stored lower pattern for its L factor), reused as the schedule
Tri make_tri(Ctx *c, const Csr &A, bool lower, bool unit, bool allow_dense = false,
             DBuf<int> *pre_order = nullptr, DBuf<int> *pre_lev = nullptr, int pre_nlev = 0);
// non-parity fast mode (Ctx::tri_jacobi): the triangle M (x) I_d as k Jacobi sweeps
Tri make_tri_jacobi(Ctx *c, const Csr &M, bool lower, bool unit, int d, int k);
// x = T^{-1} b  (xout = xadd + x when xadd given); x/ticket are scratch of size n / 1
void trsv(Ctx *c, const Tri &T, const double *b, double *x, int *ticket, const double *xadd,
          double *xout, cudaStream_t st = nullptr);

struct Ilu {
    Ctx *ctx = nullptr;
    Csr LU;             // factored values on A's pattern (sorted)
    Tri L, U;
    DBuf<double> tmp, y;
    DBuf<int> ticket;
    int n = 0;
};
std::unique_ptr<Ilu> ilu0(Ctx *c, const Csr &A);
void ilu_apply(Ctx *c, Ilu &f, const double *r, double *z, cudaStream_t st = nullptr);

// ---- AMG (amg.cu) -----------------------------------------------------------
struct AmgLevel {
    Csr A, P, R;               // R = P^T
    Tri lo, up;                // D+L, D+U
    DBuf<int> agg;             // aggregates (device)
    double rho = 0;
    DBuf<double> b, x, r, t, y; // workspace
    DBuf<double> dg;           // diag(A): the Gauss-Seidel sweeps' shortcut residuals
    DBuf<int> ticket;
};
struct Amg {
    SideStream side;           // smoother setup of level l overlaps the Galerkin product of l+1
    SideStream side_rho;       // rho(D^-1 A) of a level, concurrent with its aggregation
    std::vector<std::unique_ptr<SideStream>> lvside;   // per level: (D+L) and (D+U) sweep setups
    Ctx *ctx = nullptr;
    std::vector<std::unique_ptr<AmgLevel>> lv;
    DBuf<double> coarse_inv;   // dense inverse of the coarsest operator (row-major)
    int nc = 0;
    // tail collapse: the V-cycle of levels >= tail_level as one dense operator (row-major);
    // exact-arithmetic rewrite of the small, launch-latency-bound tail of the hierarchy
    DBuf<double> tail_M;
    int tail_level = -1;
};
// A0_steal: optional; its storage becomes level 0 (no copy) when the caller is done with it
// greedy strength aggregation (path 0 auto, 1 host greedy, 2 device passes); returns the count
int64_t strength_aggregates(Ctx *c, const Csr &A, double theta, int path, DBuf<int> &agg);
std::unique_ptr<Amg> amg_setup(Ctx *c, const Csr &A, double theta, double omega, int max_coarse,
                               int max_levels, dpp_randn_fn randn, void *user, Csr *A0_steal = nullptr);
void amg_vcycle(Ctx *c, Amg &h, const double *r, double *z, cudaStream_t st = nullptr);

// ---- launch bookkeeping for graph capture ----------------------------------
struct Recorder { int64_t kernels = 0; };

}  // namespace dpp

// ---- opaque handles ----------------------------------------------------------
struct dpp_ctx { dpp::Ctx c; };
struct dpp_csr { dpp::Ctx *ctx; dpp::Csr m; };
