// Block-system helpers: monolithic view (assembly.monolithic_view,
// assembly.py:102-108) and small shared kernels.
#include "system.cuh"

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace dpp {

bool TraceScope::on() {
    static int v = -1;
    if (v < 0) { const char *e = std::getenv("DPP_TRACE"); v = e && *e && *e != '0' && std::string(e) != "ev"; }
    return v == 1;
}
bool TraceScope::ev_on() {
    static int v = -1;
    if (v < 0) { const char *e = std::getenv("DPP_TRACE"); v = e && std::string(e) == "ev"; }
    return v == 1;
}
namespace {
struct EvRec {
    std::string name;
    cudaEvent_t a, b;
    size_t tid;
};
std::mutex g_ev_mu;
std::vector<EvRec> g_ev;
cudaEvent_t g_ev_origin = nullptr;
}  // namespace
void TraceScope::ev_begin() {
    std::lock_guard<std::mutex> g(g_ev_mu);
    if (!g_ev_origin) {
        cudaEventCreate(&g_ev_origin);
        cudaEventRecord(g_ev_origin, c->s);
    }
    cudaEventCreate(&ev0);
    cudaEventRecord(ev0, c->s);
}
void TraceScope::ev_flush(const char *title) {
    std::lock_guard<std::mutex> g(g_ev_mu);
    if (!g_ev_origin) return;
    cudaDeviceSynchronize();
    std::fprintf(stderr, "[dpp-evtrace] == %s ==\n", title);
    for (auto &r : g_ev) {
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, g_ev_origin, r.a);
        cudaEventElapsedTime(&b, g_ev_origin, r.b);
        std::fprintf(stderr, "[dpp-evtrace] %9.3f %9.3f %8.3f t%03zu %s\n", a, b, b - a, r.tid, r.name.c_str());
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    g_ev.clear();
    cudaEventDestroy(g_ev_origin);
    g_ev_origin = nullptr;
}
double TraceScope::now() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
TraceScope::~TraceScope() {
    if (ev0) {
        cudaEvent_t e1;
        cudaEventCreate(&e1);
        cudaEventRecord(e1, c->s);
        std::lock_guard<std::mutex> g(g_ev_mu);
        g_ev.push_back({name, ev0, e1, std::hash<std::thread::id>{}(std::this_thread::get_id()) % 1000});
        return;
    }
    if (!on()) return;
    cudaStreamSynchronize(c->s);
    cudaMemPool_t pool;
    unsigned long long res = 0, used = 0;
    if (cudaDeviceGetDefaultMemPool(&pool, c->device) == cudaSuccess) {
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res);
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    }
    static const double origin = now();
    const size_t tid = std::hash<std::thread::id>{}(std::this_thread::get_id()) % 1000;
    std::fprintf(stderr, "[dpp-trace] %-28s %9.3f ms   pool reserved %7.1f MB used %7.1f MB  @%10.3f t%03zu\n", name,
                 now() - t0, res / 1048576.0, used / 1048576.0, t0 - origin, tid);
}

// Side streams come from a process-wide pool: creating a stream while the other setup
// branches have work in flight was measured at ~6 ms (at the head of every AMG setup)
namespace {
std::mutex g_pool_mu;
struct Pooled {
    int device, low;
    cudaStream_t s;
};
std::vector<Pooled> g_pool;   // idle streams
cudaStream_t pool_acquire(int device, int low) {
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        for (size_t i = 0; i < g_pool.size(); ++i)
            if (g_pool[i].device == device && g_pool[i].low == low) {
                cudaStream_t s = g_pool[i].s;
                g_pool.erase(g_pool.begin() + (long)i);
                return s;
            }
    }
    cudaStream_t s;
    CK(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, stream_priority(low != 0)));
    return s;
}
void pool_release(int device, int low, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_pool.push_back({device, low, s});
}
}  // namespace

namespace {
std::mutex g_pin_mu;
std::vector<PinnedBuf> g_pin_free;
}  // namespace
PinnedBuf pinned_acquire(size_t bytes) {
    {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        for (size_t i = 0; i < g_pin_free.size(); ++i)
            if (g_pin_free[i].cap >= bytes) {
                PinnedBuf b = g_pin_free[i];
                g_pin_free.erase(g_pin_free.begin() + (long)i);
                return b;
            }
    }
    PinnedBuf b;
    b.cap = 1 << 22;
    while (b.cap < bytes) b.cap <<= 1;
    CK(cudaMallocHost(&b.p, b.cap));
    return b;
}
void pinned_release(PinnedBuf b) {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_free.push_back(b);
}

int stream_priority(bool low) {
    static const bool off = [] { const char *e = std::getenv("DPP_NO_PRIO"); return e && *e == '1'; }();
    int least = 0, greatest = 0;
    if (off || cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) return 0;
    return low ? least : greatest;
}

void SideStream::ensure(Ctx *parent, bool low_prio) {
    if (s) return;
    low = low_prio;
    s = pool_acquire(parent->device, low);
    ctx = *parent;
    ctx.s = ctx.s2 = s;
    ctx.launches = 0;
    ctx.t0 = ctx.t1 = nullptr;
    // stream-ordered: a plain cudaMalloc here may wait for the kernels the other setup
    // branches have in flight (measured: ~7 ms at the head of every AMG setup)
    CK(cudaMallocAsync((void **)&ctx.nrm_part, sizeof(double) * NRM_BLOCKS, s));
    ctx.nrm_part2 = ctx.nrm_part;
}
SideStream::~SideStream() {
    if (!s) return;
    if (ctx.nrm_part) cudaFreeAsync(ctx.nrm_part, s);
    cudaStreamSynchronize(s);
    pool_release(ctx.device, low, s);
}

bool pdl_on() {
    static const bool on = [] { const char *e = std::getenv("DPP_NO_PDL"); return !(e && *e == '1'); }();
    return on;
}

int fork_mask() {
    static const int m = [] {
        const char *s = std::getenv("DPP_SERIAL_SETUP");
        if (s && *s == '1') return 0;
        const char *e = std::getenv("DPP_FORK_MASK");
        return e ? std::atoi(e) : 7;
    }();
    return m;
}

void fork_join(Ctx *c, SideStream &owner, const std::function<void(Ctx *)> &side,
               const std::function<void()> &main_fn, int kind) {
    owner.ensure(c, kind == FORK_SCHUR);   // the Schur fork's side branch (ILU setup) has slack
    CK(cudaStreamSynchronize(c->s));   // inputs produced on the parent stream are ready
    if (!(fork_mask() & kind)) {
        side(&owner.ctx);
        CK(cudaStreamSynchronize(owner.s));
        main_fn();
    } else {
        std::exception_ptr err;
        std::thread t([&] {
            try {
                CK(cudaSetDevice(owner.ctx.device));
                side(&owner.ctx);
                CK(cudaStreamSynchronize(owner.s));
            } catch (...) {
                err = std::current_exception();
            }
        });
        try {
            main_fn();
        } catch (...) {
            t.join();
            throw;
        }
        t.join();
        if (err) std::rethrow_exception(err);
    }
    c->launches += owner.ctx.launches;
    owner.ctx.launches = 0;
}

__global__ void k_reciprocal(int64_t n, const double *d, double *o) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        o[i] = 1.0 / d[i];
}
void reciprocal(Ctx *c, int64_t n, const double *d, double *o) {
    if (!n) return;
    k_reciprocal<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, d, o);
    launched(c);
}

static void build_K(Ctx *c, dpp_system *s) {
    if (s->hasK) return;
    // (u1,p1,u2,p2) x (u1,p1,u2,p2) grid of reference blocks (assembly.py:88-93)
    const Csr *g[16] = {nullptr};
    auto at = [&](int r, int cc) -> const Csr *& { return g[r * 4 + cc]; };
    at(0, 0) = &s->blk[DPP_K1_UU];
    at(0, 1) = &s->blk[DPP_K1_UP];
    at(1, 0) = &s->blk[DPP_K1_PU];
    at(1, 1) = &s->blk[DPP_K1_PP];
    at(1, 3) = &s->blk[DPP_K12_PP];
    at(3, 1) = &s->blk[DPP_K21_PP];
    at(2, 2) = &s->blk[DPP_K2_UU];
    at(2, 3) = &s->blk[DPP_K2_UP];
    at(3, 2) = &s->blk[DPP_K2_PU];
    at(3, 3) = &s->blk[DPP_K2_PP];
    std::vector<const Csr *> grid(g, g + 16);
    std::vector<int> sz = {(int)s->sizes[0], (int)s->sizes[1], (int)s->sizes[2], (int)s->sizes[3]};
    s->K = csr_bmat(c, grid, 4, 4, sz, sz);
    s->Kc = csr_drop_zeros(c, s->K);
    spmv_plan(c, s->Kc);
    int64_t tot = s->sizes[0] + s->sizes[1] + s->sizes[2] + s->sizes[3], off = 0;
    s->f.alloc(tot, c->s);
    for (int k = 0; k < 4; ++k) {
        if (s->sizes[k])
            CK(cudaMemcpyAsync(s->f.p + off, s->rhs[k].p, sizeof(double) * s->sizes[k],
                               cudaMemcpyDeviceToDevice, c->s));
        off += s->sizes[k];
    }
    s->hasK = true;
}

const Csr &system_K(Ctx *c, dpp_system *s) { build_K(c, s); return s->K; }
const Csr &system_Kc(Ctx *c, dpp_system *s) { build_K(c, s); return s->Kc; }
const double *system_f(Ctx *c, dpp_system *s) { build_K(c, s); return s->f.p; }

}  // namespace dpp
