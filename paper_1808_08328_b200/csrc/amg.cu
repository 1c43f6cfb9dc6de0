// Smoothed-aggregation AMG on the device.
//
// Reference: linalg.amg_setup / _strength_aggregates / _jacobi_spectral_radius /
// _vcycle (linalg.py:279-400).
//  setup per level:  strength graph |a_ij| >= theta*max_k!=i |a_ik| (device),
//                    3-pass greedy aggregation in row order (exact; see aggregate()),
//                    rho(D^-1 A) by 10 power iterations from the reference's start
//                    vector (device SpMV + norms), P = P0 - (2w/rho) D^-1 (A P0)
//                    with scipy's rounding (device), A_c = (P^T A) P (device SpGEMM),
//                    D+L / D+U sweeps for SGS, dense inverse of the coarsest operator.
//  apply:            V(1,1) with SGS (forward then backward GS as x += T^-1 (b - A x)),
//                    restriction P^T, prolongation P, coarse dense solve.
#include <climits>
#include <cmath>
#include <cstdlib>
#include <exception>
#include <functional>
#include <memory>
#include <thread>

#include <cub/cub.cuh>
#include <thrust/iterator/transform_iterator.h>

#include "dpp_internal.cuh"

namespace dpp {

// ---------------------------------------------------------------- strength graph
__global__ void k_strength(int rows, const int *ptr, const int *idx, const double *val,
                           double theta, const int *optr, int *cnt, int *oidx) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int s = ptr[r], e = ptr[r + 1];
        double mx = -1.0;
        for (int p = s + lane; p < e; p += 32)
            if (idx[p] != r) mx = fmax(mx, fabs(val[p]));
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const double thr = theta * mx;
        int w = optr ? optr[r] : 0, n = 0;
        for (int base = s; base < e; base += 32) {
            const int p = base + lane;
            const bool keep = mx >= 0.0 && p < e && idx[p] != r && fabs(val[p]) >= thr;
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep && oidx) oidx[w + __popc(m & ((1u << lane) - 1))] = idx[p];
            w += __popc(m);
            n += __popc(m);
        }
        if (lane == 0 && cnt) cnt[r] = n;
    }
}

// Greedy aggregation (linalg.py:301-323), exact sequential semantics on the
// host from the device-built strength graph: pass 1 seeds nodes whose closed
// strong neighbourhood is still free, pass 2 attaches leftovers to the first
// aggregated strong neighbour (in stored order, seeing pass-2 assignments of
// earlier rows), pass 3 makes singletons.
static int64_t greedy(int n, const std::vector<int> &sp, const std::vector<int> &si,
                      std::vector<int64_t> &agg) {
    agg.assign(n, -1);
    int64_t next = 0;
    for (int i = 0; i < n; ++i) {
        if (agg[i] != -1) continue;
        bool free_nb = true;
        for (int p = sp[i]; p < sp[i + 1] && free_nb; ++p) free_nb = agg[si[p]] == -1;
        if (!free_nb) continue;
        agg[i] = next;
        for (int p = sp[i]; p < sp[i + 1]; ++p) agg[si[p]] = next;
        ++next;
    }
    for (int i = 0; i < n; ++i) {
        if (agg[i] != -1) continue;
        for (int p = sp[i]; p < sp[i + 1]; ++p)
            if (agg[si[p]] != -1) { agg[i] = agg[si[p]]; break; }
    }
    for (int i = 0; i < n; ++i)
        if (agg[i] == -1) agg[i] = next++;
    return next;
}

static int64_t aggregate_host(Ctx *c, const Csr &A, double theta, DBuf<int> &dagg) {
    const int n = A.rows;
    DBuf<int> cnt(n, c->s);
    const int grid = grid_for((int64_t)n * 32, 256, c->sms, 8);
    k_strength<<<grid, 256, 0, c->s>>>(n, A.ptr.p, A.idx.p, A.val.p, theta, nullptr, cnt.p, nullptr);
    launched(c);
    DBuf<int> sptr;
    int64_t snnz = counts_to_ptr(c, cnt.p, n, sptr);
    DBuf<int> sidx(snnz, c->s);
    k_strength<<<grid, 256, 0, c->s>>>(n, A.ptr.p, A.idx.p, A.val.p, theta, sptr.p, nullptr, sidx.p);
    launched(c);
    std::vector<int> hp, hi;
    {
        DPP_TRACE_SCOPE(c, "amg.strength_d2h");
        hp = sptr.to_host();
        hi = sidx.to_host();
    }
    DPP_TRACE_SCOPE(c, "amg.greedy_host");
    std::vector<int64_t> agg;
    const int64_t nc = greedy(n, hp, hi, agg);
    std::vector<int> agg32(agg.begin(), agg.end());
    dagg.alloc(n, c->s);
    dagg.upload(agg32.data(), n);
    return nc;
}

// ---------------------------------------------------------------- device aggregation
// The same three passes on the device, bit for bit.  N[i] = {i} + strong(i).
//  pass 1: i seeds iff no earlier seed j has N[j] & N[i] != {} (an earlier seed that
//          took i or one of its neighbours).  The owners of a node k are k itself and
//          the rows whose strong list holds k (the transposed strength pattern); i waits
//          only on the states of lower owners of its N[i], and decides "not a seed" as
//          soon as one of them is a seed.  Seeds' N[] are disjoint, so a seed's
//          aggregate id is its rank among the seeds and it stamps its whole N[].
//  pass 2: i (untaken) takes the aggregate of its first strong neighbour, in stored
//          order, that is taken at that point of the sequential loop: taken in pass 1,
//          or a lower row that took one in pass 2 (i waits for that row's pass 2).
//  pass 3: the rest become singletons, numbered after the seeds in row order.
// Spinning rows only wait on lower rows and every thread walks its rows in ascending
// order (the level-analysis dealing), so the lowest undecided row is always runnable;
// the grid is co-resident (cooperative launch).
namespace {
constexpr long long AGG_SPIN_LIMIT = 1ll << 26;
__device__ __forceinline__ int agg_ld(const int *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void agg_st(int *p, int v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// wait until x[j] != undecided; returns the value
__device__ __forceinline__ int agg_wait(const int *x, int j, int undecided) {
    int v = agg_ld(x + j);
    long long spins = 0;
    while (v == undecided) {
        __nanosleep(32);
        v = agg_ld(x + j);
        if (++spins > AGG_SPIN_LIMIT) __trap();
    }
    return v;
}
__global__ void k_tcount(int n, const int *__restrict__ sp, const int *__restrict__ si, int *tc) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        for (int p = sp[j]; p < sp[j + 1]; ++p) atomicAdd(tc + si[p], 1);
}
__global__ void k_tfill(int n, const int *__restrict__ sp, const int *__restrict__ si, const int *__restrict__ tp,
                        int *tcur, int *ti) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        for (int p = sp[j]; p < sp[j + 1]; ++p) {
            const int k = si[p];
            ti[tp[k] + atomicAdd(tcur + k, 1)] = j;
        }
}
// Pass 1 as a dataflow: pending[i] counts the (k, j) pairs with k in N[i] and j a lower
// owner of k (j conflicts with i through k).  A row that decides pushes to its higher
// conflicting rows: a seed marks them (not seeds), a non-seed decrements their pending
// count.  A row waits until it is marked or its count drains, i.e. until one lower
// conflicting row is a seed or all of them are not -- the lexicographically-first MIS,
// decided along its own dependency depth (148 steps on C2's S_p).
template <typename F>
__device__ __forceinline__ void agg_pairs(int i, const int *__restrict__ sp, const int *__restrict__ si,
                                          const int *__restrict__ tp, const int *__restrict__ ti, F f) {
    const int s0 = sp[i], s1 = sp[i + 1];
    for (int q = s0 - 1; q < s1; ++q) {
        const int k = q < s0 ? i : si[q];
        f(k);
        for (int p = tp[k], pe = tp[k + 1]; p < pe; ++p) f(ti[p]);
    }
}
// per row: pending = lower conflicting pairs, hc = higher conflicting pairs
__global__ void k_agg_count(int n, const int *__restrict__ sp, const int *__restrict__ si,
                            const int *__restrict__ tp, const int *__restrict__ ti, int *pending, int *hc) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        int lo = 0, hi = 0;
        agg_pairs(i, sp, si, tp, ti, [&](int j) {
            lo += j < i;
            hi += j > i;
        });
        pending[i] = lo;
        hc[i] = hi;
    }
}
// the higher conflicting rows of every row, flattened (the push list of pass 1)
__global__ void k_agg_hfill(int n, const int *__restrict__ sp, const int *__restrict__ si,
                            const int *__restrict__ tp, const int *__restrict__ ti, const int *__restrict__ hp,
                            int *hl) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        int o = hp[i];
        agg_pairs(i, sp, si, tp, ti, [&](int h) {
            if (h > i) hl[o++] = h;
        });
    }
}
// state: 1 seed, 0 not a seed
__global__ void __launch_bounds__(256) k_agg_pass1(int n, const int *__restrict__ hp, const int *__restrict__ hl,
                                                   int *pending, int *mark, int *state) {
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t W = T >> 5, w = g >> 5, lane = g & 31;
    for (int64_t base = 0; base < n; base += T) {
        const int64_t t = base + lane * W + w;
        if (t >= n) continue;
        const int i = (int)t;
        int mk = agg_ld(mark + i), pd = agg_ld(pending + i);
        long long spins = 0;
        while (!mk && pd > 0) {
            __nanosleep(20);
            mk = agg_ld(mark + i);
            pd = agg_ld(pending + i);
            if (++spins > AGG_SPIN_LIMIT) __trap();
        }
        const bool seed = !mk;
        state[i] = seed ? 1 : 0;
        const int p0 = hp[i], p1 = hp[i + 1];
        if (seed)
            for (int p = p0; p < p1; ++p) agg_st(mark + hl[p], 1);
        else
            for (int p = p0; p < p1; ++p) atomicSub(pending + hl[p], 1);
    }
}
// a1[k] = rank of the seed whose N[] holds k (pass 1), else -1
__global__ void k_agg_stamp(int n, const int *__restrict__ sp, const int *__restrict__ si,
                            const int *__restrict__ state, const int *__restrict__ rank, int *a1) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        if (state[j] != 1) continue;
        const int id = rank[j];
        a1[j] = id;
        for (int p = sp[j]; p < sp[j + 1]; ++p) a1[si[p]] = id;
    }
}
// fin: -2 undecided, -1 untaken after pass 2, else the aggregate
__global__ void __launch_bounds__(256) k_agg_pass2(int n, const int *__restrict__ sp, const int *__restrict__ si,
                                                   const int *__restrict__ a1, int *fin) {
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t W = T >> 5, w = g >> 5, lane = g & 31;
    for (int64_t base = 0; base < n; base += T) {
        const int64_t t = base + lane * W + w;
        if (t >= n) continue;
        const int i = (int)t;
        int v = a1[i];
        if (v < 0) {
            for (int p = sp[i]; p < sp[i + 1]; ++p) {
                const int k = si[p];
                const int ak = a1[k];
                if (ak >= 0) { v = ak; break; }
                if (k < i) {
                    const int fk = agg_wait(fin, k, -2);
                    if (fk >= 0) { v = fk; break; }
                }
            }
        }
        agg_st(fin + i, v);
    }
}
struct IsSeed {
    __host__ __device__ int operator()(int s) const { return s == 1; }
};
struct IsLeft {
    __host__ __device__ int operator()(int f) const { return f == -1; }
};
__global__ void k_fill_i(int *x, int n, int v) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] = v;
}
// pass 3 + count: agg = fin, or nseed + rank among the untaken
__global__ void k_agg_final(int n, const int *__restrict__ state, const int *__restrict__ srank,
                            const int *__restrict__ lrank, int *fin, int *nc) {
    const int nseed = srank[n - 1] + (state[n - 1] == 1);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const bool left = fin[i] == -1;
        if (i == n - 1) *nc = nseed + lrank[i] + (left ? 1 : 0);
        if (left) fin[i] = nseed + lrank[i];
    }
}
}  // namespace

// threads of the spinning pass kernels (DPP_AGG_THREADS, default 16384): the waits
// follow the MIS dependency depth, not the thread count, and a small co-resident grid
// neither waits for half the device to drain nor keeps it spinning
static int64_t agg_threads() {
    static const int64_t t = [] { const char *e = std::getenv("DPP_AGG_THREADS"); return e ? std::atoll(e) : 16384LL; }();
    return t;
}
static void coop_launch(Ctx *c, const void *k, int n, void **args, int64_t max_threads = agg_threads()) {
    const int block = 256;
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, block, 0));
    if (per_sm < 1) DPP_FAIL(DPP_ERR_CUDA, "aggregation kernels cannot be resident");
    per_sm = std::max(1, per_sm / 2);   // leave room for the other setup branches
    const int64_t need = std::min<int64_t>(((int64_t)n + 31) / 32 * 32, std::max<int64_t>(max_threads, 256));
    const int64_t cap = (int64_t)c->sms * per_sm * block;
    const int grid = (int)((std::min(need, cap) + block - 1) / block);
    CK(cudaLaunchCooperativeKernel(k, grid, block, args, 0, c->s));
    launched(c);
}

template <typename Op>
static void flag_scan(Ctx *c, const int *in, int *out, int n) {
    auto it = thrust::make_transform_iterator(in, Op());
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, it, out, n, c->s));
    DBuf<char> t(std::max<size_t>(tb, 1), c->s);
    CK(cub::DeviceScan::ExclusiveSum(t.p, tb, it, out, n, c->s));
    launched(c);
}

static int64_t aggregate_dev(Ctx *c, const Csr &A, double theta, DBuf<int> &agg) {
    const int n = A.rows;
    agg.alloc(n, c->s);
    if (!n) return 0;
    // strength graph: counts -> int32 scan (total <= nnz(A), no read back) -> fill
    std::unique_ptr<TraceScope> ph(new TraceScope(c, "agg.strength"));
    DBuf<int> cnt(n, c->s), sp(n + 1, c->s), si(std::max<int64_t>(A.nnz, 1), c->s);
    const int grid = grid_for((int64_t)n * 32, 256, c->sms, 8);
    k_strength<<<grid, 256, 0, c->s>>>(n, A.ptr.p, A.idx.p, A.val.p, theta, nullptr, cnt.p, nullptr);
    launched(c);
    scan_to_ptr32(c, cnt.p, n, sp.p);
    k_strength<<<grid, 256, 0, c->s>>>(n, A.ptr.p, A.idx.p, A.val.p, theta, sp.p, nullptr, si.p);
    launched(c);
    // transposed pattern (owners)
    ph.reset(new TraceScope(c, "agg.transpose"));
    DBuf<int> tc(n, c->s), tp(n + 1, c->s), ti(std::max<int64_t>(A.nnz, 1), c->s);
    CK(cudaMemsetAsync(tc.p, 0, sizeof(int) * n, c->s));
    const int g1 = grid_for(n, 256, c->sms);
    k_tcount<<<g1, 256, 0, c->s>>>(n, sp.p, si.p, tc.p);
    launched(c);
    scan_to_ptr32(c, tc.p, n, tp.p);
    CK(cudaMemsetAsync(tc.p, 0, sizeof(int) * n, c->s));
    k_tfill<<<g1, 256, 0, c->s>>>(n, sp.p, si.p, tp.p, tc.p, ti.p);
    launched(c);
    // pass 1
    ph.reset(new TraceScope(c, "agg.pass1"));
    DBuf<int> state(n, c->s), srank(n, c->s), lrank(n, c->s), nc(1, c->s), pend(n, c->s), mark(n, c->s);
    DBuf<int> hc(n, c->s), hp(n + 1, c->s);
    CK(cudaMemsetAsync(mark.p, 0, sizeof(int) * n, c->s));
    k_agg_count<<<g1, 256, 0, c->s>>>(n, sp.p, si.p, tp.p, ti.p, pend.p, hc.p);
    launched(c);
    scan_to_ptr32(c, hc.p, n, hp.p);
    int nh = 0;
    CK(cudaMemcpyAsync(&nh, hp.p + n, sizeof(int), cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    // dense strong hubs make the push lists quadratic: the host loop has no such term
    if (nh < 0 || nh > (1 << 28)) {
        ph.reset();
        return aggregate_host(c, A, theta, agg);
    }
    DBuf<int> hl(std::max(nh, 1), c->s);
    k_agg_hfill<<<g1, 256, 0, c->s>>>(n, sp.p, si.p, tp.p, ti.p, hp.p, hl.p);
    launched(c);
    {
        int nn = n;
        const int *a = hp.p, *b = hl.p;
        int *pe = pend.p, *mk = mark.p, *st = state.p;
        void *args[] = {&nn, &a, &b, &pe, &mk, &st};
        coop_launch(c, (const void *)k_agg_pass1, n, args, agg_threads());
    }
    ph.reset(new TraceScope(c, "agg.stamp"));
    flag_scan<IsSeed>(c, state.p, srank.p, n);
    DBuf<int> a1(n, c->s);
    CK(cudaMemsetAsync(a1.p, 0xFF, sizeof(int) * n, c->s));
    k_agg_stamp<<<g1, 256, 0, c->s>>>(n, sp.p, si.p, state.p, srank.p, a1.p);
    launched(c);
    // pass 2 (into agg, -2 = undecided)
    ph.reset(new TraceScope(c, "agg.pass2"));
    k_fill_i<<<g1, 256, 0, c->s>>>(agg.p, n, -2);
    launched(c);
    {
        int nn = n;
        const int *a = sp.p, *b = si.p, *d = a1.p;
        int *f = agg.p;
        void *args[] = {&nn, &a, &b, &d, &f};
        coop_launch(c, (const void *)k_agg_pass2, n, args);
    }
    // pass 3
    ph.reset(new TraceScope(c, "agg.pass3"));
    flag_scan<IsLeft>(c, agg.p, lrank.p, n);
    k_agg_final<<<g1, 256, 0, c->s>>>(n, state.p, srank.p, lrank.p, agg.p, nc.p);
    launched(c);
    ph.reset();
    int h = 0;
    CK(cudaMemcpyAsync(&h, nc.p, sizeof(int), cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    return h;
}

// Device passes from DPP_AGG_DEV_MIN rows up (default 32768): below it the strength graph
// is small enough that its read back + the host loop beat the cooperative launches, which
// must wait for half the device to drain while the other setup branches run.
// DPP_AGG_HOST=1 / =0 forces either path (read per call); path 1 / 2 force them per call.
int64_t strength_aggregates(Ctx *c, const Csr &A, double theta, int path, DBuf<int> &agg) {
    static const int dev_min = [] { const char *v = std::getenv("DPP_AGG_DEV_MIN"); return v ? std::atoi(v) : 32768; }();
    bool host = A.rows < dev_min;
    const char *e = std::getenv("DPP_AGG_HOST");
    if (e && *e) host = *e == '1';
    if (path == 1 || path == 2) host = path == 1;
    return host ? aggregate_host(c, A, theta, agg) : aggregate_dev(c, A, theta, agg);
}
static int64_t aggregate(Ctx *c, const Csr &A, double theta, DBuf<int> &agg) {
    return strength_aggregates(c, A, theta, 0, agg);
}

// ---------------------------------------------------------------- P construction
// P = P0 - damping * (Dinv @ (A @ P0)) with scipy's rounding:
//   w = fl(dinv_i * y_ij), dw = fl(damping * w), p = fl(p0 - dw), zeros dropped.
__global__ void k_build_p(int rows, const int *yp, const int *yi, const double *yv,
                          const int *agg, const double *dinv, double damping, const int *optr,
                          int *cnt, int *oi, double *ov) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
        const int a = agg[r];
        int w = optr ? optr[r] : 0, n = 0;
        bool seen = false;
        auto emit = [&](int j, double v) {
            if (v == 0.0) return;
            if (oi) { oi[w] = j; ov[w] = v; ++w; }
            ++n;
        };
        for (int p = yp[r]; p < yp[r + 1]; ++p) {
            const int j = yi[p];
            if (!seen && j > a) { emit(a, 1.0); seen = true; }
            const double dw = __dmul_rn(damping, __dmul_rn(dinv[r], yv[p]));
            if (j == a) { emit(j, __dsub_rn(1.0, dw)); seen = true; }
            else emit(j, -dw);
        }
        if (!seen) emit(a, 1.0);
        if (cnt) cnt[r] = n;
    }
}

// Same P straight from A and the aggregates, without forming A @ P0: (A P0)_ij is the
// sum of a_ik over the row's entries with agg[k] == j, accumulated from 0 in storage
// order (scipy csr_matmat with b_kj = 1.0, so a_ik * 1.0 is exact), columns ascending.
// Warp per row, 32 entries at a time: __match_any groups a chunk's lanes by key, the
// group leader finds (or appends) the key in the warp's shared list of distinct keys
// and adds the group's values to that key's running sum one member at a time in lane
// (= storage) order.  The diagonal aggregate seeds the list with sum +0.0, so it is
// always present without changing any sum.  Output slots are ranks among the distinct
// keys (exact-zero results squeezed out).  Rows with PD_CAP or more entries extract
// keys one at a time.
constexpr int PD_CAP = 512, PD_W = 8;
constexpr size_t PD_SMEM = (size_t)PD_W * PD_CAP * 12;
__global__ void __launch_bounds__(32 * PD_W) k_p_direct(int rows, const int *__restrict__ ap,
                                                        const int *__restrict__ ai, const double *__restrict__ av,
                                                        const int *__restrict__ agg, const double *__restrict__ dinv,
                                                        double damping, int ncols, int *__restrict__ cnt, int *__restrict__ oi,
                                                        double *__restrict__ ov) {
    extern __shared__ __align__(16) unsigned char pd_smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double *dy = reinterpret_cast<double *>(pd_smem) + (size_t)wid * PD_CAP;
    int *dk = reinterpret_cast<int *>(pd_smem + (size_t)PD_W * PD_CAP * 8) + (size_t)wid * PD_CAP;
    const unsigned lt = (1u << lane) - 1;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int s = ap[r], e = ap[r + 1], a = agg[r], len = e - s;
        const double di = dinv[r];
        const int w0 = s + (int)r;   // scratch slot: at most len + 1 outputs
        if (len < PD_CAP || ncols <= PD_CAP) {   // distinct keys <= min(len + 1, ncols)
            __syncwarp();
            if (lane == 0) { dk[0] = a; dy[0] = 0.0; }
            int nd = 1;
            __syncwarp();
            // keys / values of up to PD_PF chunks are loaded before any is processed
            constexpr int PD_PF = 3;
            for (int base0 = s; base0 < e; base0 += 32 * PD_PF) {
                int kq[PD_PF];
                double vq[PD_PF];
#pragma unroll
                for (int q = 0; q < PD_PF; ++q) {
                    const int p = base0 + 32 * q + lane;
                    kq[q] = p < e ? ai[p] : -1;
                    vq[q] = p < e ? av[p] : 0.0;
                }
#pragma unroll
                for (int q = 0; q < PD_PF; ++q)
                    if (kq[q] >= 0) kq[q] = agg[kq[q]];
#pragma unroll
                for (int q = 0; q < PD_PF; ++q) {
                    if (base0 + 32 * q >= e) break;
                    const int k = kq[q];
                    const double v = vq[q];
                    const bool valid = k >= 0;
                    const unsigned g = __match_any_sync(0xffffffffu, k);
                    const bool lead = valid && (g & lt) == 0;
                    int slot = -1;
                    if (lead)
                        for (int j = 0; j < nd; ++j)
                            if (dk[j] == k) { slot = j; break; }
                    const unsigned nm = __ballot_sync(0xffffffffu, lead && slot < 0);
                    if (lead && slot < 0) {
                        slot = nd + __popc(nm & lt);
                        dk[slot] = k;
                        dy[slot] = 0.0;
                    }
                    nd += __popc(nm);
                    const int gs = lead ? __popc(g) : 0;
                    const int rounds = __reduce_max_sync(0xffffffffu, gs);
                    double y = lead ? dy[slot] : 0.0;
                    unsigned rem = lead ? g : 0u;   // members not yet added, lowest lane first
                    for (int t = 0; t < rounds; ++t) {
                        const int src = rem ? __ffs(rem) - 1 : lane;
                        const double vt = __shfl_sync(0xffffffffu, v, src);
                        if (rem) y = __dadd_rn(y, vt);
                        rem &= rem - 1;
                    }
                    if (lead) dy[slot] = y;
                    __syncwarp();
                }
            }
            // values, then ranks among the nonzero distinct keys
            bool zero = false;
            for (int j = lane; j < nd; j += 32) {
                const double dw = __dmul_rn(damping, __dmul_rn(di, dy[j]));
                const double v = dk[j] == a ? __dsub_rn(1.0, dw) : -dw;
                dy[j] = v;
                zero |= v == 0.0;
            }
            zero = __any_sync(0xffffffffu, zero);
            __syncwarp();
            int nz = 0;
            for (int j = lane; j < nd; j += 32) {
                const int k = dk[j];
                const double v = dy[j];
                int pos = 0;
                for (int q = 0; q < nd; ++q) pos += dk[q] < k && (!zero || dy[q] != 0.0);
                if (v != 0.0) {
                    oi[w0 + pos] = k;
                    ov[w0 + pos] = v;
                    ++nz;
                }
            }
            nz = __reduce_add_sync(0xffffffffu, nz);
            if (lane == 0) cnt[r] = nz;
            continue;
        }
        int w = w0, n = 0, last = -1;
        for (;;) {
            int mk = a > last ? a : INT_MAX;
            for (int p = s + lane; p < e; p += 32) {
                const int k = agg[ai[p]];
                if (k > last && k < mk) mk = k;
            }
            for (int o = 16; o > 0; o >>= 1) mk = min(mk, __shfl_xor_sync(0xffffffffu, mk, o));
            if (mk == INT_MAX) break;
            double y = 0.0;
            for (int base = s; base < e; base += 32) {
                const int p = base + lane;
                const bool hit = p < e && agg[ai[p]] == mk;
                const double v = hit ? av[p] : 0.0;
                unsigned m = __ballot_sync(0xffffffffu, hit);
                while (m) {
                    const int b = __ffs(m) - 1;
                    y = __dadd_rn(y, __shfl_sync(0xffffffffu, v, b));
                    m &= m - 1;
                }
            }
            const double dw = __dmul_rn(damping, __dmul_rn(di, y));
            const double v = mk == a ? __dsub_rn(1.0, dw) : -dw;
            if (v != 0.0) {
                if (lane == 0) { oi[w] = mk; ov[w] = v; }
                ++w;
                ++n;
            }
            last = mk;
        }
        if (lane == 0) cnt[r] = n;
    }
}

__global__ void k_p_compact(int rows, const int *__restrict__ ap, const int *__restrict__ ptr,
                            const int *__restrict__ ti, const double *__restrict__ tv, int *oi, double *ov) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t s = ap[r] + r;
        const int o = ptr[r], n = ptr[r + 1] - o;
        for (int q = lane; q < n; q += 32) {
            oi[o + q] = ti[s + q];
            ov[o + q] = tv[s + q];
        }
    }
}

__global__ void k_p0(int rows, const int *agg, int *ptr, int *idx, double *val) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r <= rows; r += gridDim.x * blockDim.x) {
        ptr[r] = r;
        if (r < rows) { idx[r] = agg[r]; val[r] = 1.0; }
    }
}

__global__ void k_recip(int n, const double *d, double *o) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) o[r] = 1.0 / d[r];
}

// M = diag(dinv) @ A  (row scaling, exact products)
__global__ void k_rowscale(int rows, const int *ptr, const double *val, const double *dinv, double *o) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const double d = dinv[r];
        for (int p = ptr[r] + lane; p < ptr[r + 1]; p += 32) o[p] = __dmul_rn(d, val[p]);
    }
}

static double spectral_radius(Ctx *c, const Csr &A, const double *dinv, dpp_randn_fn randn,
                              void *user) {
    const int n = A.rows;
    Csr M = csr_copy(c, A);
    k_rowscale<<<grid_for((int64_t)n * 32, 256, c->sms, 8), 256, 0, c->s>>>(n, M.ptr.p, A.val.p, dinv, M.val.p);
    launched(c);
    std::vector<double> x0(n);
    if (!randn) DPP_FAIL(DPP_ERR_VALUE, "amg_setup needs the power-iteration start vector callback");
    randn(n, x0.data(), user);
    DBuf<double> x(n, c->s), y(n, c->s), nr(12, c->s);
    x.upload(x0.data(), n);
    norm2_dev(c, n, x.p, nr.p);
    scale_by_dev(c, n, x.p, nr.p, x.p);
    for (int it = 1; it <= 10; ++it) {
        spmv(c, M, x.p, y.p);
        norm2_dev(c, n, y.p, nr.p + it);
        scale_by_dev(c, n, y.p, nr.p + it, x.p);
    }
    spmv(c, M, x.p, y.p);
    norm2_dev(c, n, y.p, nr.p + 11);
    std::vector<double> h = nr.to_host();
    for (int it = 1; it <= 10; ++it)
        if (h[it] == 0.0) return 1.0;
    return std::max(h[11], 1e-8);
}

// ---------------------------------------------------------------- dense coarse solve
__global__ void k_to_dense(int n, const int *ptr, const int *idx, const double *val, double *D) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
        for (int p = ptr[r]; p < ptr[r + 1]; ++p) D[(int64_t)r * n + idx[p]] += val[p];
}

// LU with partial pivoting (first maximal |pivot|, as LAPACK idamax) and explicit
// inverse, one block.  n is small (<= max_coarse unless aggregation stalls).
__global__ void __launch_bounds__(256) k_dense_inverse(int n, double *A, int *perm, double *Ainv) {
    __shared__ double smax[256];
    __shared__ int sarg[256];
    const int t = threadIdx.x;
    for (int i = t; i < n; i += blockDim.x) perm[i] = i;
    __syncthreads();
    for (int k = 0; k < n; ++k) {
        double best = -1.0;
        int arg = k;
        for (int r = k + t; r < n; r += blockDim.x) {
            const double v = fabs(A[(int64_t)r * n + k]);
            if (v > best) { best = v; arg = r; }
        }
        smax[t] = best;
        sarg[t] = arg;
        __syncthreads();
        for (int o = blockDim.x / 2; o > 0; o >>= 1) {
            if (t < o) {
                if (smax[t + o] > smax[t] || (smax[t + o] == smax[t] && sarg[t + o] < sarg[t])) {
                    smax[t] = smax[t + o];
                    sarg[t] = sarg[t + o];
                }
            }
            __syncthreads();
        }
        const int p = sarg[0];
        __syncthreads();
        if (p != k) {
            for (int j = t; j < n; j += blockDim.x) {
                const double tmp = A[(int64_t)k * n + j];
                A[(int64_t)k * n + j] = A[(int64_t)p * n + j];
                A[(int64_t)p * n + j] = tmp;
            }
            if (t == 0) { int q = perm[k]; perm[k] = perm[p]; perm[p] = q; }
        }
        __syncthreads();
        const double piv = A[(int64_t)k * n + k];
        for (int r = k + 1 + t; r < n; r += blockDim.x) A[(int64_t)r * n + k] /= piv;
        __syncthreads();
        const int m = n - k - 1;
        for (int64_t q = t; q < (int64_t)m * m; q += blockDim.x) {
            const int r = k + 1 + (int)(q / m), cc = k + 1 + (int)(q % m);
            A[(int64_t)r * n + cc] -= A[(int64_t)r * n + k] * A[(int64_t)k * n + cc];
        }
        __syncthreads();
    }
    // column c of the inverse: solve L U x = P e_c (row i of P e_c is [perm[i] == c])
    for (int cidx = t; cidx < n; cidx += blockDim.x) {
        for (int i = 0; i < n; ++i) {
            double s = perm[i] == cidx ? 1.0 : 0.0;
            for (int j = 0; j < i; ++j) s -= A[(int64_t)i * n + j] * Ainv[(int64_t)j * n + cidx];
            Ainv[(int64_t)i * n + cidx] = s;
        }
        for (int i = n - 1; i >= 0; --i) {
            double s = Ainv[(int64_t)i * n + cidx];
            for (int j = i + 1; j < n; ++j) s -= A[(int64_t)i * n + j] * Ainv[(int64_t)j * n + cidx];
            Ainv[(int64_t)i * n + cidx] = s / A[(int64_t)i * n + i];
        }
    }
}

__global__ void k_gemv(int n, const double *M, const double *x, double *y) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        double s = 0.0;
        for (int j = lane; j < n; j += 32) s += M[r * n + j] * x[j];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) y[r] = s;
    }
}

static void coarse_setup(Ctx *c, Amg &h, const Csr &A) {
    const int n = A.rows;
    h.nc = n;
    DBuf<double> D((size_t)n * n, c->s);
    DBuf<int> perm(n, c->s);
    h.coarse_inv.alloc((size_t)n * n, c->s);
    if (!n) return;
    CK(cudaMemsetAsync(D.p, 0, sizeof(double) * n * n, c->s));
    k_to_dense<<<grid_for(n, 128, c->sms), 128, 0, c->s>>>(n, A.ptr.p, A.idx.p, A.val.p, D.p);
    launched(c);
    k_dense_inverse<<<1, 256, 0, c->s>>>(n, D.p, perm.p, h.coarse_inv.p);
    launched(c);
    CK(cudaStreamSynchronize(c->s));
}

// ---------------------------------------------------------------- tail collapse
// The last levels of the hierarchy are tiny (C2: 590 / 80 / 12 rows) and their V-cycle is a chain
// of ~25 dependent launches that each run for a few microseconds.  Where both smoother
// triangles of every remaining level already are dense inverses Li = (D+L)^-1, Ui = (D+U)^-1,
// the cycle below that level is a fixed linear map and is formed once at setup (reference
// linalg.py:383-400 composed symbolically, level by level from the coarsest):
//   T = Li + Ui (I - A Li)                      one symmetric Gauss-Seidel sweep from x = 0
//   Y = T + P M_c R (I - A T)                   + coarse correction
//   M = Y - Li (A Y);  M = M - Ui (A M);  M += T   post-smoothing sweep from Y b
// An exact-arithmetic rewrite like the dense triangular inverses themselves; DPP_AMG_TAIL=0
// (or a level above the row limit) keeps the launch-by-launch cycle.
// Y = Z + alpha * A X (+ I): A CSR (rows x k), X dense k x m, row-major
__global__ void k_spmm(int rows, int m, const int *__restrict__ ptr, const int *__restrict__ idx,
                       const double *__restrict__ val, const double *__restrict__ X, const double *Z, double alpha,
                       int add_identity, double *Y) {
    const int r = blockIdx.y;
    const int p0 = ptr[r], p1 = ptr[r + 1];
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
        double s = 0.0;
        int p = p0;
        for (; p + 4 <= p1; p += 4) {   // four rows of X in flight (the sum keeps the storage order)
            const double x0 = X[(int64_t)idx[p] * m + j], x1 = X[(int64_t)idx[p + 1] * m + j];
            const double x2 = X[(int64_t)idx[p + 2] * m + j], x3 = X[(int64_t)idx[p + 3] * m + j];
            s += val[p] * x0;
            s += val[p + 1] * x1;
            s += val[p + 2] * x2;
            s += val[p + 3] * x3;
        }
        for (; p < p1; ++p) s += val[p] * X[(int64_t)idx[p] * m + j];
        double y = alpha * s;
        if (Z) y += Z[(int64_t)r * m + j];
        if (add_identity && j == r) y += 1.0;
        Y[(int64_t)r * m + j] = y;
    }
}
// C = Cin + alpha * A B: A n x k, B k x m, row-major; tri = 1 / 2: A is lower / upper triangular
// (k == n) and the zero tiles are skipped
constexpr int GT = 64, GK = 16;
__global__ void __launch_bounds__(256) k_dgemm(int n, int m, int k, const double *__restrict__ A,
                                               const double *__restrict__ B, const double *Cin, double alpha,
                                               double *C, int tri) {
    __shared__ double As[GK][GT + 1], Bs[GK][GT];
    const int bi = blockIdx.y * GT, bj = blockIdx.x * GT;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    const int k_begin = tri == 2 ? (bi / GK) * GK : 0;
    const int k_end = tri == 1 ? min(k, bi + GT) : k;
    for (int k0 = k_begin; k0 < k_end; k0 += GK) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = threadIdx.x + 256 * q;
            const int ar = e >> 4, ak = e & 15;
            As[ak][ar] = (bi + ar < n && k0 + ak < k) ? A[(int64_t)(bi + ar) * k + k0 + ak] : 0.0;
            const int bk = e >> 6, bc = e & 63;
            Bs[bk][bc] = (k0 + bk < k && bj + bc < m) ? B[(int64_t)(k0 + bk) * m + bj + bc] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < GK; ++kk) {
            double av[4], bv[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) av[a] = As[kk][ty + 16 * a];
#pragma unroll
            for (int b = 0; b < 4; ++b) bv[b] = Bs[kk][tx + 16 * b];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int i = bi + ty + 16 * a;
        if (i >= n) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int j = bj + tx + 16 * b;
            if (j >= m) continue;
            const double cin = Cin ? Cin[(int64_t)i * m + j] : 0.0;
            C[(int64_t)i * m + j] = cin + alpha * acc[a][b];
        }
    }
}
__global__ void k_add_to(int64_t n, const double *a, double *y) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] += a[i];
}

static void tail_collapse(Ctx *c, Amg &h) {
    static const int tail_max = [] { const char *e = std::getenv("DPP_AMG_TAIL"); return e ? std::atoi(e) : 1024; }();
    const int nl = (int)h.lv.size();
    h.tail_level = -1;
    if (tail_max <= 0 || nl < 2 || h.nc <= 0) return;
    int l0 = nl - 1;   // first level of the collapsed tail
    while (l0 > 0) {
        const AmgLevel &L = *h.lv[l0 - 1];
        if (L.A.rows > tail_max || !L.lo.dense.n || !L.up.dense.n || L.lo.ncomp != 1 || L.up.ncomp != 1) break;
        --l0;
    }
    if (l0 == nl - 1) return;   // only the coarse solve: already one GEMV
    DPP_TRACE_SCOPE(c, "amg.tail_collapse");
    auto spmm = [&](const Csr &A, int m, const double *X, const double *Z, double alpha, int addI, double *Y) {
        if (!A.rows || !m) return;
        k_spmm<<<dim3((m + 127) / 128, A.rows), 128, 0, c->s>>>(A.rows, m, A.ptr.p, A.idx.p, A.val.p, X, Z, alpha, addI, Y);
        launched(c);
    };
    auto gemm = [&](int n, int m, int k, const double *A, const double *B, const double *Cin, double alpha, double *C,
                    int tri) {
        if (!n || !m) return;
        k_dgemm<<<dim3((m + GT - 1) / GT, (n + GT - 1) / GT), 256, 0, c->s>>>(n, m, k, A, B, Cin, alpha, C, tri);
        launched(c);
    };
    DBuf<double> Mc;   // the collapsed cycle of level l+1
    const double *mc = h.coarse_inv.p;
    for (int l = nl - 2; l >= l0; --l) {
        AmgLevel &L = *h.lv[l];
        const int n = L.A.rows, nc = L.P.cols;
        const size_t nn = (size_t)n * n;
        const double *Li = L.lo.dense.p, *Ui = L.up.dense.p;
        DBuf<double> E(nn, c->s), T(nn, c->s), W(nn, c->s), G1((size_t)nc * n, c->s), G2((size_t)nc * n, c->s), M(nn, c->s);
        spmm(L.A, n, Li, nullptr, -1.0, 1, E.p);                 // E = I - A Li
        gemm(n, n, n, Ui, E.p, Li, 1.0, T.p, 2);                 // T = Li + Ui E
        spmm(L.A, n, T.p, nullptr, -1.0, 1, W.p);                // W = I - A T
        spmm(L.R, n, W.p, nullptr, 1.0, 0, G1.p);                // G1 = R W
        gemm(nc, n, nc, mc, G1.p, nullptr, 1.0, G2.p, 0);        // G2 = M_c G1
        spmm(L.P, n, G2.p, T.p, 1.0, 0, E.p);                    // Y = T + P G2            (in E)
        spmm(L.A, n, E.p, nullptr, 1.0, 0, W.p);                 // W = A Y
        gemm(n, n, n, Li, W.p, E.p, -1.0, M.p, 1);               // Z1 = Y - Li W           (in M)
        spmm(L.A, n, M.p, nullptr, 1.0, 0, W.p);                 // W = A Z1
        gemm(n, n, n, Ui, W.p, M.p, -1.0, E.p, 2);               // Z2 = Z1 - Ui W          (in E)
        k_add_to<<<grid_for((int64_t)nn, 256, c->sms), 256, 0, c->s>>>((int64_t)nn, T.p, E.p);   // M = Z2 + T
        launched(c);
        CK(cudaStreamSynchronize(c->s));   // the temporaries are freed on scope exit
        Mc = std::move(E);
        mc = Mc.p;
    }
    h.tail_M = std::move(Mc);
    h.tail_level = l0;
}

// ---------------------------------------------------------------- setup
std::unique_ptr<Amg> amg_setup(Ctx *c, const Csr &A0, double theta, double omega, int max_coarse,
                               int max_levels, dpp_randn_fn randn, void *user, Csr *A0_steal) {
    DPP_TRACE_SCOPE(c, "amg.total");
    if (A0.rows != A0.cols) DPP_FAIL(DPP_ERR_VALUE, "amg_setup requires a square matrix");
    auto h = std::make_unique<Amg>();
    h->ctx = c;
    {
        DPP_TRACE_SCOPE(c, "amg.diag_check");
        DBuf<double> d(A0.rows, c->s);
        csr_diag(c, A0, d.p, nullptr);
        if (any_zero_dev(c, A0.rows, d.p))
            DPP_FAIL(DPP_ERR_ZERO_PIVOT, "structurally singular input: zero diagonal entry");
    }
    Csr cur;
    if (A0_steal && A0_steal == &A0) {
        cur = std::move(*A0_steal);
    } else {
        DPP_TRACE_SCOPE(c, "amg.copy");
        cur = csr_copy(c, A0);
    }
    // smoother setup (level analysis + sweep plans) of level l runs on a worker
    // thread / side stream while this thread builds level l+1
    {
        DPP_TRACE_SCOPE(c, "amg.side_ensure");
        h->side.ensure(c);
        h->side_rho.ensure(c);
    }
    // sweep setups of every level run on their own host threads / side streams and
    // are joined once, after the last Galerkin product
    std::vector<std::thread> workers;
    std::vector<std::unique_ptr<std::exception_ptr>> werrs;
    auto join_worker = [&] {
        for (auto &t : workers)
            if (t.joinable()) t.join();
        for (auto &e : werrs)
            if (*e) std::rethrow_exception(*e);
    };
    const bool serial = !(fork_mask() & FORK_AMG_SMOOTHER);
    struct Joiner {
        std::vector<std::thread> &t;
        ~Joiner() {
            for (auto &x : t)
                if (x.joinable()) x.join();
        }
    } joiner{workers};
    while (cur.rows > max_coarse && (int)h->lv.size() < max_levels - 1) {
        auto L = std::make_unique<AmgLevel>();
        const int n = cur.rows;
        DBuf<double> d(n, c->s), dinv(n, c->s);
        csr_diag(c, cur, d.p, nullptr);
        k_recip<<<grid_for(n, 256, c->sms), 256, 0, c->s>>>(n, d.p, dinv.p);
        launched(c);
        // rho(D^-1 A) does not depend on the aggregates: the power iteration runs on its
        // own side stream / host thread while this thread aggregates
        double rho = 0.0;
        std::exception_ptr rerr;
        std::thread rt;
        Ctx *rc = &h->side_rho.ctx;
        auto rho_fn = [&] {
            DPP_TRACE_SCOPE(rc, "amg.rho");
            rho = spectral_radius(rc, cur, dinv.p, randn, user);
            CK(cudaStreamSynchronize(rc->s));
        };
        CK(cudaStreamSynchronize(c->s));   // dinv is read on the side stream
        if (serial) {
            rho_fn();
        } else {
            rt = std::thread([&] {
                try {
                    CK(cudaSetDevice(rc->device));
                    rho_fn();
                } catch (...) {
                    rerr = std::current_exception();
                }
            });
        }
        int64_t nc;
        {
            DPP_TRACE_SCOPE(c, "amg.aggregate");
            try {
                nc = aggregate(c, cur, theta, L->agg);
            } catch (...) {
                if (rt.joinable()) rt.join();
                throw;
            }
        }
        if (rt.joinable()) rt.join();
        if (rerr) std::rethrow_exception(rerr);
        if (nc >= n) {
            if (n > 5000) DPP_FAIL(DPP_ERR_RUNTIME, "aggregation stalled on a large operator");
            break;
        }
        L->rho = rho;
        const double damping = 2.0 * omega / L->rho;
        DBuf<int> &dagg = L->agg;
        static const bool p_generic = [] { const char *e = std::getenv("DPP_P_GENERIC"); return e && *e == '1'; }();
        L->P.rows = n;
        L->P.cols = (int)nc;
        DBuf<int> cnt(n, c->s);
        if (p_generic) {
            Csr P0;
            P0.alloc(n, (int)nc, n, c->s);
            k_p0<<<grid_for(n + 1, 256, c->sms), 256, 0, c->s>>>(n, dagg.p, P0.ptr.p, P0.idx.p, P0.val.p);
            launched(c);
            Csr Y = spgemm(c, cur, P0, nullptr, false, nullptr);
            k_build_p<<<grid_for(n, 128, c->sms), 128, 0, c->s>>>(n, Y.ptr.p, Y.idx.p, Y.val.p, dagg.p, dinv.p,
                                                                 damping, nullptr, cnt.p, nullptr, nullptr);
            launched(c);
            L->P.nnz = counts_to_ptr(c, cnt.p, n, L->P.ptr);
            L->P.idx.alloc(L->P.nnz, c->s);
            L->P.val.alloc(L->P.nnz, c->s);
            k_build_p<<<grid_for(n, 128, c->sms), 128, 0, c->s>>>(n, Y.ptr.p, Y.idx.p, Y.val.p, dagg.p, dinv.p,
                                                                 damping, L->P.ptr.p, nullptr, L->P.idx.p,
                                                                 L->P.val.p);
            launched(c);
        } else {
            static bool pattr = false;
            if (!pattr) {
                CK(cudaFuncSetAttribute(k_p_direct, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PD_SMEM));
                pattr = true;
            }
            const int g = grid_for((int64_t)n * 32, 32 * PD_W, c->sms, 4);
            DBuf<int> ti(cur.nnz + n, c->s);
            DBuf<double> tv(cur.nnz + n, c->s);
            k_p_direct<<<g, 32 * PD_W, PD_SMEM, c->s>>>(n, cur.ptr.p, cur.idx.p, cur.val.p, dagg.p, dinv.p, damping,
                                                       (int)nc, cnt.p, ti.p, tv.p);
            launched(c);
            L->P.nnz = counts_to_ptr(c, cnt.p, n, L->P.ptr);
            L->P.idx.alloc(L->P.nnz, c->s);
            L->P.val.alloc(L->P.nnz, c->s);
            k_p_compact<<<grid_for((int64_t)n * 32, 256, c->sms, 8), 256, 0, c->s>>>(n, cur.ptr.p, L->P.ptr.p, ti.p,
                                                                                    tv.p, L->P.idx.p, L->P.val.p);
            launched(c);
        }
        Csr next;
        {
            DPP_TRACE_SCOPE(c, "amg.rap");
            // A_c = P^T (A P): both products keep per-row distinct counts small enough
            // for the shared-memory tables (the reference's (P^T A) P association
            // differs only by rounding; coarse levels are insensitive)
            L->R = csr_transpose(c, L->P);
            Csr AP = spgemm(c, cur, L->P, nullptr, false, nullptr);
            next = spgemm(c, L->R, AP, nullptr, false, nullptr);
        }
        L->A = std::move(cur);
        for (DBuf<double> *b : {&L->b, &L->x, &L->r, &L->t, &L->y}) b->alloc(n, c->s);
        L->ticket.alloc(4, c->s);
        L->dg = std::move(d);   // this level's diagonal (kept for the smoother's shortcut residuals)
        CK(cudaStreamSynchronize(c->s));
        // level setup off the critical path, on two side streams / host threads: the
        // (D+L) sweep plan + SpMV plans, and the (D+U) sweep plan
        AmgLevel *Lp = L.get();
        for (int q = 0; q < 2; ++q) {
            h->lvside.push_back(std::make_unique<SideStream>());
            h->lvside.back()->ensure(c, true);
        }
        Ctx *sc = &h->lvside[h->lvside.size() - 2]->ctx, *su = &h->lvside.back()->ctx;
        auto smoother_lo = [Lp, sc] {
            DPP_TRACE_SCOPE(sc, "amg.smoother_setup");
            Lp->lo = make_tri(sc, Lp->A, true, false, true);
            spmv_plan(sc, Lp->A);
            spmv_plan(sc, Lp->P);
            spmv_plan(sc, Lp->R);
            CK(cudaStreamSynchronize(sc->s));
        };
        auto smoother_up = [Lp, su] {
            DPP_TRACE_SCOPE(su, "amg.smoother_setup_up");
            Lp->up = make_tri(su, Lp->A, false, false, true);
            CK(cudaStreamSynchronize(su->s));
        };
        if (serial) {
            smoother_lo();
            smoother_up();
        } else {
            auto spawn = [&](std::function<void()> fn, Ctx *x) {
                werrs.push_back(std::make_unique<std::exception_ptr>());
                std::exception_ptr *err = werrs.back().get();
                workers.emplace_back([fn, x, err] {
                    try {
                        CK(cudaSetDevice(x->device));
                        fn();
                    } catch (...) {
                        *err = std::current_exception();
                    }
                });
            };
            spawn(smoother_lo, sc);
            spawn(smoother_up, su);
        }
        h->lv.push_back(std::move(L));
        cur = std::move(next);
        CK(cudaStreamSynchronize(c->s));
    }
    {
        DPP_TRACE_SCOPE(c, "amg.join_smoothers");
        join_worker();
    }
    std::vector<SideStream *> sides = {&h->side, &h->side_rho};
    for (auto &ss : h->lvside) sides.push_back(ss.get());
    for (SideStream *ss : sides) {
        c->launches += ss->ctx.launches;
        ss->ctx.launches = 0;
    }
    auto last = std::make_unique<AmgLevel>();
    coarse_setup(c, *h, cur);
    const int n = cur.rows;
    for (DBuf<double> *b : {&last->b, &last->x}) b->alloc(n, c->s);
    last->A = std::move(cur);
    h->lv.push_back(std::move(last));
    tail_collapse(c, *h);
    CK(cudaStreamSynchronize(c->s));
    return h;
}

// ---------------------------------------------------------------- V(1,1) cycle
__global__ void k_mul_to(int64_t n, const double *__restrict__ a, const double *__restrict__ x, double *o) {
    pdl_wait();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        o[i] = a[i] * x[i];
    pdl_trigger();
}
static void vc(Ctx *c, Amg &h, size_t l, const double *b, double *xo, cudaStream_t st) {
    AmgLevel &L = *h.lv[l];
    const int n = L.A.rows;
    if ((int)l == h.tail_level) {   // the collapsed tail: one dense operator
        k_gemv<<<grid_for((int64_t)n * 32, 128, c->sms, 4), 128, 0, st>>>(n, h.tail_M.p, b, xo);
        launched(c);
        return;
    }
    if (l + 1 == h.lv.size()) {
        if (n) {
            k_gemv<<<grid_for((int64_t)n * 32, 128, c->sms, 4), 128, 0, st>>>(n, h.coarse_inv.p, b, xo);
            launched(c);
        }
        return;
    }
    AmgLevel &C = *h.lv[l + 1];
    // Symmetric Gauss-Seidel as x += (D+L)^-1 (b - A x); x += (D+U)^-1 (b - A x) (reference
    // linalg.py:383-385).  After the forward half-sweep with d = (D+L)^-1 r the new residual is
    // r - A d = r - (D+L) d - U_s d = -U_s d, and (D+U)^-1 (-U_s d) = (D+U)^-1 D d - d: the backward
    // half-sweep is x_old + (D+U)^-1 (D d) -- the same numbers in exact arithmetic without the
    // second product with A (two SpMVs per level and cycle instead of four).  DPP_SGS_PLAIN=1 keeps
    // the literal sequence.
    static const bool plain = [] { const char *e = std::getenv("DPP_SGS_PLAIN"); return e && *e == '1'; }();
    if (!plain && L.dg.n == (size_t)n && !L.lo.jacobi && !L.up.jacobi) {   // exact sweeps only
        // pre-smoothing from x = 0: d = (D+L)^-1 b, x2 = (D+U)^-1 (D d)
        trsv(c, L.lo, b, L.x.p, L.ticket.p, nullptr, nullptr, st);
        CK(launch_pdl(k_mul_to, dim3(grid_for(n, 256, c->sms)), dim3(256), 0, st, (int64_t)n, (const double *)L.dg.p,
                      (const double *)L.x.p, L.r.p));
        launched(c);
        trsv(c, L.up, L.r.p, L.t.p, L.ticket.p + 1, nullptr, nullptr, st);
        // restriction of the residual, coarse correction, prolongation
        spmv(c, L.A, L.t.p, L.r.p, b, -1.0, st);
        spmv(c, L.R, L.r.p, C.b.p, nullptr, 1.0, st);
        vc(c, h, l + 1, C.b.p, C.x.p, st);
        spmv(c, L.P, C.x.p, L.x.p, L.t.p, 1.0, st);
        // post-smoothing: d = (D+L)^-1 (b - A x3), x5 = x3 + (D+U)^-1 (D d)
        spmv(c, L.A, L.x.p, L.r.p, b, -1.0, st);
        trsv(c, L.lo, L.r.p, L.y.p, L.ticket.p + 2, nullptr, nullptr, st);
        CK(launch_pdl(k_mul_to, dim3(grid_for(n, 256, c->sms)), dim3(256), 0, st, (int64_t)n, (const double *)L.dg.p,
                      (const double *)L.y.p, L.r.p));
        launched(c);
        trsv(c, L.up, L.r.p, L.y.p, L.ticket.p + 3, L.x.p, xo, st);
        return;
    }
    // pre-smoothing, x starts at 0: x1 = (D+L)^-1 b ; x2 = x1 + (D+U)^-1 (b - A x1)
    trsv(c, L.lo, b, L.x.p, L.ticket.p, nullptr, nullptr, st);
    spmv(c, L.A, L.x.p, L.r.p, b, -1.0, st);
    trsv(c, L.up, L.r.p, L.y.p, L.ticket.p + 1, L.x.p, L.t.p, st);
    // restriction of the residual, coarse correction, prolongation
    spmv(c, L.A, L.t.p, L.r.p, b, -1.0, st);
    spmv(c, L.R, L.r.p, C.b.p, nullptr, 1.0, st);
    vc(c, h, l + 1, C.b.p, C.x.p, st);
    spmv(c, L.P, C.x.p, L.x.p, L.t.p, 1.0, st);
    // post-smoothing
    spmv(c, L.A, L.x.p, L.r.p, b, -1.0, st);
    trsv(c, L.lo, L.r.p, L.y.p, L.ticket.p + 2, L.x.p, L.t.p, st);
    spmv(c, L.A, L.t.p, L.r.p, b, -1.0, st);
    trsv(c, L.up, L.r.p, L.y.p, L.ticket.p + 3, L.t.p, xo, st);
}

void amg_vcycle(Ctx *c, Amg &h, const double *r, double *z, cudaStream_t st) {
    vc(c, h, 0, r, z, st ? st : c->s);
}

}  // namespace dpp
