// Core device sparse/vector kernels: CSR SpMV, vector ops, CSR restructuring.
// Reference semantics: scipy.sparse CSR as used by dppflow (linalg.py:27-32,
// blocksolve.py:227-228, assembly.py:102-108, linalg.py:218-219, :372-374).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>
#include <thrust/iterator/transform_output_iterator.h>

#include <climits>
#include <cstdlib>
#include <cstring>

#include "dpp_internal.cuh"

namespace dpp {

static inline cudaStream_t S(Ctx *c, cudaStream_t st) { return st ? st : c->s; }

// ---------------------------------------------------------------- scans
// One decoupled-look-back scan: counts widened to int64 on the fly (element n reads as
// 0), the running sum narrowed on the way out with saturation to -1, so a total of
// 2^31 or more shows up as a negative ptr[n] instead of wrapping silently.
namespace {
struct CountAt {
    const int *c;
    int n;
    __host__ __device__ long long operator()(int i) const { return i < n ? (long long)c[i] : 0LL; }
};
struct Narrow {
    __host__ __device__ int operator()(long long v) const { return v > INT_MAX ? -1 : (int)v; }
};
}  // namespace
void scan_to_ptr32(Ctx *c, const int *counts, int n, int *ptr) {
    auto in = thrust::make_transform_iterator(thrust::make_counting_iterator<int>(0), CountAt{counts, n});
    auto out = thrust::make_transform_output_iterator(ptr, Narrow{});
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n + 1, c->s));
    DBuf<char> t(std::max<size_t>(tb, 1), c->s);
    CK(cub::DeviceScan::ExclusiveSum(t.p, tb, in, out, n + 1, c->s));
    launched(c);
}
// counts[n] -> ptr[n+1] (int32), returns total; errors if total >= 2^31
int64_t counts_to_ptr(Ctx *c, const int *counts, int n, DBuf<int> &ptr) {
    ptr.alloc((size_t)n + 1, c->s);
    scan_to_ptr32(c, counts, n, ptr.p);
    int total = 0;
    CK(cudaMemcpyAsync(&total, ptr.p + n, sizeof(int), cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    if (total < 0) DPP_FAIL(DPP_ERR_VALUE, "CSR with more than 2^31-1 entries");
    return total;
}

// ---------------------------------------------------------------- SpMV
// G lanes per row; every lane of a warp runs the same number of iterations so
// the width-G shuffles are always fully populated.
template <int G>
__global__ void __launch_bounds__(256) k_spmv(int rows, const int *__restrict__ ptr,
                                              const int *__restrict__ idx,
                                              const double *__restrict__ val,
                                              const double *__restrict__ x, double *__restrict__ y,
                                              const double *__restrict__ b, double alpha) {
    pdl_wait();
    constexpr int RPW = 32 / G;
    const int lane = threadIdx.x & (G - 1);
    const int grp = (threadIdx.x & 31) / G;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t w = warp; w * RPW < rows; w += nwarp) {
        const int64_t r = w * RPW + grp;
        double sum = 0.0;
        if (r < rows) {
            const int s = __ldg(ptr + r), e = __ldg(ptr + r + 1);
            for (int p = s + lane; p < e; p += G) sum += __ldg(val + p) * __ldg(x + __ldg(idx + p));
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, o, G);
        if (r < rows && lane == 0) y[r] = b ? b[r] + alpha * sum : alpha * sum;
    }
    pdl_trigger();
}

// nnz-streaming SpMV (CSR-stream): one CTA per row block of <= SB_CAP entries.  All
// lanes load SB_E consecutive-strided (val, col) pairs up front -- 2*SB_E independent
// coalesced loads per thread keep enough bytes in flight to cover HBM latency, which
// the row-per-warp kernel above cannot at ~40 entries per row -- then gather x, park
// the products in shared memory and reduce each row with G lanes.
constexpr int SB_THREADS = 256, SB_E = 8, SB_CAP = SB_THREADS * SB_E, SB_T = SB_CAP - 256;

__global__ void k_spmv_plan(int rows, const int *__restrict__ ptr, int nb, int *rb) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k <= nb; k += gridDim.x * blockDim.x) {
        if (k == nb) { rb[k] = rows; continue; }
        // first row whose first entry is at or after k*T
        const int64_t key = (int64_t)k * SB_T;
        int lo = 0, hi = rows;
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if ((int64_t)ptr[mid] < key) lo = mid + 1; else hi = mid;
        }
        rb[k] = lo;
    }
}

// SELL-32 (sliced ELLPACK, slice height 32, rows kept in order): lane l of a warp owns
// row 32k + l and walks its entries in column order, so a warp's loads of one slice
// column are 256 B / 128 B coalesced and -- on the structured meshes of the DPP
// systems, where the t-th neighbour of consecutive nodes is a consecutive node --
// its x gathers hit a handful of lines instead of one line per couple of entries
// (the CSR kernels are L1-wavefront bound on those gathers).  Each row is summed
// sequentially in column order with separate multiply and add roundings: y = K x
// is bitwise scipy's csr_matvec (linalg.py:27-32) on the same entries; skipped
// exact zeros and the zero padding leave the sums unchanged.
__global__ void k_sell_width(int rows, const int *__restrict__ ptr, int nsl, int *wcnt) {
    const int lane = threadIdx.x & 31;
    for (int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < nsl;
         k += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t r = k * 32 + lane;
        int len = r < rows ? ptr[r + 1] - ptr[r] : 0;
        for (int o = 16; o > 0; o >>= 1) len = max(len, __shfl_xor_sync(0xffffffffu, len, o));
        if (lane == 0) wcnt[k] = len * 32;
    }
}
__global__ void k_sell_fill(int rows, const int *__restrict__ ptr, const int *__restrict__ idx,
                            const double *__restrict__ val, int nsl, const int *__restrict__ sp, int *sc,
                            double *sv) {
    const int lane = threadIdx.x & 31;
    for (int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < nsl;
         k += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t r = k * 32 + lane;
        const int a = r < rows ? ptr[r] : 0, len = r < rows ? ptr[r + 1] - a : 0;
        const int w = (sp[k + 1] - sp[k]) >> 5;
        int last = r < rows ? (int)r : 0;   // padding column: any valid index
        for (int t = 0; t < w; ++t) {
            const int64_t o = sp[k] + (int64_t)t * 32 + lane;
            if (t < len) { last = idx[a + t]; sc[o] = last; sv[o] = val[a + t]; }
            else { sc[o] = last; sv[o] = 0.0; }
        }
    }
}

// 16-bit column codes: a slice's columns fall in at most 4 windows of 2^14 columns
// (mesh operators: the node's neighbourhood in each field block the row couples to), so
// each entry stores a 2-bit window id and a 14-bit offset -- 10 bytes per entry instead
// of 12.  Windows start at the smallest column not yet covered (greedy); a slice that
// needs a fifth window fails the whole matrix back to 32-bit columns.
constexpr int SELL_WIN = 1 << 14;
__global__ void k_sell_bases(int rows, const int *__restrict__ ptr, const int *__restrict__ idx, int nsl,
                             int4 *base, int *fail) {
    const int lane = threadIdx.x & 31;
    for (int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < nsl;
         k += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t r = k * 32 + lane;
        const int a = r < rows ? ptr[r] : 0, e = r < rows ? ptr[r + 1] : 0;
        int b[4] = {0, 0, 0, 0}, nb = 0;
        auto covered = [&](int c) {
            bool cv = false;
#pragma unroll
            for (int s = 0; s < 4; ++s) cv |= s < nb && c >= b[s] && c - b[s] < SELL_WIN;
            return cv;
        };
        for (int s = 0; s < 4; ++s) {
            int m = INT_MAX;
            for (int p = a; p < e; ++p) {
                const int c = idx[p];
                if (!covered(c)) m = min(m, c);
            }
            for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (m == INT_MAX) break;
            b[nb++] = m;
        }
        bool bad = false;
        for (int p = a; p < e; ++p) bad |= !covered(idx[p]);
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(fail, 1);
        if (lane == 0) base[k] = make_int4(b[0], nb > 1 ? b[1] : b[0], nb > 2 ? b[2] : b[0], nb > 3 ? b[3] : b[0]);
    }
}
__global__ void k_sell_fill16(int rows, const int *__restrict__ ptr, const int *__restrict__ idx,
                              const double *__restrict__ val, int nsl, const int *__restrict__ sp,
                              const int4 *__restrict__ base, uint16_t *sc, double *sv) {
    const int lane = threadIdx.x & 31;
    for (int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < nsl;
         k += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t r = k * 32 + lane;
        const int a = r < rows ? ptr[r] : 0, len = r < rows ? ptr[r + 1] - a : 0;
        const int w = (sp[k + 1] - sp[k]) >> 5;
        const int4 B = base[k];
        const int bs[4] = {B.x, B.y, B.z, B.w};
        uint16_t last = 0;   // padding: window 0, offset 0 (a valid column: the slice's smallest)
        for (int t = 0; t < w; ++t) {
            const int64_t o = sp[k] + (int64_t)t * 32 + lane;
            if (t < len) {
                const int c = idx[a + t];
                int sel = 3;
#pragma unroll
                for (int s = 3; s >= 0; --s)
                    if (c >= bs[s] && c - bs[s] < SELL_WIN) sel = s;
                last = (uint16_t)((sel << 14) | (c - bs[sel]));
                sc[o] = last;
                sv[o] = val[a + t];
            } else {
                sc[o] = last;
                sv[o] = 0.0;
            }
        }
    }
}

// SELL-32 is used when padding stays under this factor of the stored entries
constexpr double SELL_MAX_FILL = 1.25;
// DPP_SPMV=row|stream|sell (default sell): kernel selection for A/B measurements
static int spmv_mode() {
    static const int m = [] {
        const char *e = std::getenv("DPP_SPMV");
        if (!e || !*e) return 2;
        return !strcmp(e, "row") ? 0 : !strcmp(e, "stream") ? 1 : 2;
    }();
    return m;
}

// DPP_SELL16=0 keeps 32-bit SELL columns (A/B); read per plan
static bool sell16_on() {
    const char *e = std::getenv("DPP_SELL16");
    return !(e && *e == '0');
}

void spmv_plan(Ctx *c, Csr &A, int kind) {
    A.rb.release(); A.nrb = 0;
    A.sp.release(); A.sc.release(); A.sv.release(); A.sc16.release(); A.sbase.release(); A.nsl = 0;
    if (kind == 3) kind = spmv_mode() == 0 ? 0 : spmv_mode() == 1 ? 1 : 3;
    if (A.rows == 0 || A.nnz == 0 || kind == 0) return;
    if (kind >= 2) {
        const int nsl = (A.rows + 31) / 32;
        DBuf<int> wcnt((size_t)nsl, c->s);
        const int grid = grid_for((int64_t)nsl * 32, 256, c->sms, 8);
        k_sell_width<<<grid, 256, 0, c->s>>>(A.rows, A.ptr.p, nsl, wcnt.p);
        launched(c);
        DBuf<int> sp;
        const int64_t tot = counts_to_ptr(c, wcnt.p, nsl, sp);
        if (kind == 2 || (double)tot <= SELL_MAX_FILL * (double)A.nnz) {
            A.sp = std::move(sp);
            A.sv.alloc((size_t)tot, c->s);
            bool narrow = sell16_on();
            if (narrow) {
                A.sbase.alloc((size_t)nsl, c->s);
                DBuf<int> fail(1, c->s);
                CK(cudaMemsetAsync(fail.p, 0, sizeof(int), c->s));
                k_sell_bases<<<grid, 256, 0, c->s>>>(A.rows, A.ptr.p, A.idx.p, nsl, A.sbase.p, fail.p);
                launched(c);
                narrow = fail.to_host()[0] == 0;
            }
            if (narrow) {
                A.sc16.alloc((size_t)tot, c->s);
                k_sell_fill16<<<grid, 256, 0, c->s>>>(A.rows, A.ptr.p, A.idx.p, A.val.p, nsl, A.sp.p, A.sbase.p,
                                                     A.sc16.p, A.sv.p);
            } else {
                A.sbase.release();
                A.sc.alloc((size_t)tot, c->s);
                k_sell_fill<<<grid, 256, 0, c->s>>>(A.rows, A.ptr.p, A.idx.p, A.val.p, nsl, A.sp.p, A.sc.p, A.sv.p);
            }
            launched(c);
            A.nsl = nsl;
            return;
        }
    }
    const int nb = (int)((A.nnz + SB_T - 1) / SB_T);
    A.rb.alloc((size_t)nb + 1, c->s);
    k_spmv_plan<<<grid_for(nb + 1, 256, c->sms), 256, 0, c->s>>>(A.rows, A.ptr.p, nb, A.rb.p);
    launched(c);
    A.nrb = nb;
}

__global__ void __launch_bounds__(SB_THREADS) k_spmv_stream(const int *__restrict__ rb,
                                                            const int *__restrict__ ptr,
                                                            const int *__restrict__ idx,
                                                            const double *__restrict__ val,
                                                            const double *__restrict__ x,
                                                            double *__restrict__ y,
                                                            const double *__restrict__ b, double alpha) {
    __shared__ double prod[SB_CAP];
    const int tid = threadIdx.x;
    pdl_wait();
    const int r0 = __ldg(rb + blockIdx.x), r1 = __ldg(rb + blockIdx.x + 1);
    if (r0 >= r1) { pdl_trigger(); return; }
    const int s = __ldg(ptr + r0), e = __ldg(ptr + r1), n = e - s, nr = r1 - r0;
    auto out = [&](int r, double sum) { y[r] = b ? b[r] + alpha * sum : alpha * sum; };
    if (n <= SB_CAP) {
        double v[SB_E];
        int j[SB_E];
#pragma unroll
        for (int k = 0; k < SB_E; ++k) {
            const int p = s + k * SB_THREADS + tid;
            v[k] = p < e ? __ldg(val + p) : 0.0;
            j[k] = p < e ? __ldg(idx + p) : -1;
        }
#pragma unroll
        for (int k = 0; k < SB_E; ++k)
            if (j[k] >= 0) prod[k * SB_THREADS + tid] = v[k] * __ldg(x + j[k]);
        __syncthreads();
        // G lanes per row, G ~ mean row length / 4 (power of two in [2, 32])
        const int avg = n / nr;
        const int G = avg <= 8 ? 2 : avg <= 16 ? 4 : avg <= 32 ? 8 : avg <= 64 ? 16 : 32;
        const int lane = tid & (G - 1), rpp = SB_THREADS / G;
        for (int base = 0; base < nr; base += rpp) {
            const int rr = base + tid / G;
            double sum = 0.0;
            if (rr < nr) {
                const int a = __ldg(ptr + r0 + rr) - s, z = __ldg(ptr + r0 + rr + 1) - s;
                for (int q = a + lane; q < z; q += G) sum += prod[q];
            }
            for (int o = G >> 1; o > 0; o >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, o, G);
            if (rr < nr && lane == 0) out(r0 + rr, sum);
        }
    } else {   // oversized block (rows longer than ~256 entries): warp per row
        const int lane = tid & 31;
        for (int r = r0 + (tid >> 5); r < r1; r += SB_THREADS / 32) {
            double sum = 0.0;
            for (int p = __ldg(ptr + r) + lane; p < __ldg(ptr + r + 1); p += 32)
                sum += __ldg(val + p) * __ldg(x + __ldg(idx + p));
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, o);
            if (lane == 0) out(r, sum);
        }
    }
    pdl_trigger();
}

// T warps share a slice: warp q of the slice sums columns q, q+T, ... of its lane's row
// sequentially; the T partial sums are added in q order (T = 1: one sequential sum
// per row in column order).  Up to SELL_U columns of a lane are in flight at once.
constexpr int SELL_U = 8;
template <int T, bool C16>
__global__ void __launch_bounds__(256) k_spmv_sell(int rows, int nsl, const int *__restrict__ sp,
                                                   const int *__restrict__ sc, const uint16_t *__restrict__ sc16,
                                                   const int4 *__restrict__ sbase, const double *__restrict__ sv,
                                                   const double *__restrict__ x, double *__restrict__ y,
                                                   const double *__restrict__ b, double alpha) {
    constexpr int SPB = 8 / T;   // slices per CTA
    __shared__ double part[T > 1 ? 8 : 1][32];
    __shared__ int sbw[8][4];    // 16-bit codes: the slice's column windows, per warp
    pdl_wait();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, q = warp % T;
    const int64_t k = (int64_t)blockIdx.x * SPB + warp / T;
    double sum = 0.0;
    if (k < nsl) {
        const int o0 = __ldg(sp + k), w = (__ldg(sp + k + 1) - o0) >> 5;
        if (C16 && lane < 4) sbw[warp][lane] = __ldg(reinterpret_cast<const int *>(sbase + k) + lane);
        if (C16) __syncwarp();
        const int *J = sc + o0 + lane;
        const uint16_t *J16 = sc16 + o0 + lane;
        const double *V = sv + o0 + lane;
        for (int t = q; t < w; t += T * SELL_U) {
            double v[SELL_U], xv[SELL_U];
            int j[SELL_U];
            if (C16) {   // all code loads in flight first, then the decode (window base from smem)
                unsigned cd[SELL_U];
#pragma unroll
                for (int u = 0; u < SELL_U; ++u) {
                    const int tt = t + u * T;
                    v[u] = tt < w ? __ldg(V + tt * 32) : 0.0;
                    cd[u] = tt < w ? (unsigned)__ldg(J16 + tt * 32) : 0xffffffffu;
                }
#pragma unroll
                for (int u = 0; u < SELL_U; ++u)
                    j[u] = cd[u] == 0xffffffffu ? -1 : sbw[warp][cd[u] >> 14] + (int)(cd[u] & 0x3fffu);
            } else {
#pragma unroll
                for (int u = 0; u < SELL_U; ++u) {
                    const int tt = t + u * T;
                    v[u] = tt < w ? __ldg(V + tt * 32) : 0.0;
                    j[u] = tt < w ? __ldg(J + tt * 32) : -1;
                }
            }
#pragma unroll
            for (int u = 0; u < SELL_U; ++u) xv[u] = j[u] >= 0 ? __ldg(x + j[u]) : 0.0;
#pragma unroll
            for (int u = 0; u < SELL_U; ++u)
                if (j[u] >= 0) sum = __dadd_rn(sum, __dmul_rn(v[u], xv[u]));
        }
    }
    if (T > 1) {
        part[warp][lane] = sum;
        __syncthreads();
        if (q != 0) { pdl_trigger(); return; }
#pragma unroll
        for (int qq = 1; qq < T; ++qq) sum = __dadd_rn(sum, part[warp + qq][lane]);
    }
    const int64_t r = k * 32 + lane;
    if (k < nsl && r < rows) y[r] = b ? __dadd_rn(b[r], __dmul_rn(alpha, sum)) : __dmul_rn(alpha, sum);
    pdl_trigger();
}

void spmv(Ctx *c, const Csr &A, const double *x, double *y, const double *b, double alpha,
          cudaStream_t st) {
    st = S(c, st);
    if (A.rows == 0) return;
    if (A.nsl > 0) {
        // warps per slice: about SELL_U columns per lane (one round of loads per row)
        static const int tenv = [] { const char *e = std::getenv("DPP_SELL_T"); return e && *e ? atoi(e) : 0; }();
        auto go = [&](auto kern, int spb) {
            CK(launch_pdl(kern, dim3((A.nsl + spb - 1) / spb), dim3(256), 0, st, A.rows, A.nsl, (const int *)A.sp.p,
                          (const int *)A.sc.p, (const uint16_t *)A.sc16.p, (const int4 *)A.sbase.p,
                          (const double *)A.sv.p, x, y, b, alpha));
        };
        const size_t ent = A.sc16.n ? A.sc16.n : A.sc.n;
        const int wavg = (int)(ent / ((size_t)A.nsl * 32));
        // warps per slice: about rpw rounds of SELL_U columns per warp (DPP_SELL_RPW; 3 measured
        // best on C2's K with 16-bit codes: 59.3 us against 69.8 at 1)
        static const int rpw = [] { const char *e = std::getenv("DPP_SELL_RPW"); return e && *e ? atoi(e) : 3; }();
        const int cpw = SELL_U * rpw;
        const int T = tenv ? tenv : wavg <= cpw ? 1 : wavg <= 2 * cpw ? 2 : wavg <= 4 * cpw ? 4 : 8;
        if (A.sc16.n) {
            if (T == 1) go(k_spmv_sell<1, true>, 8);
            else if (T == 2) go(k_spmv_sell<2, true>, 4);
            else if (T == 4) go(k_spmv_sell<4, true>, 2);
            else go(k_spmv_sell<8, true>, 1);
        } else {
            if (T == 1) go(k_spmv_sell<1, false>, 8);
            else if (T == 2) go(k_spmv_sell<2, false>, 4);
            else if (T == 4) go(k_spmv_sell<4, false>, 2);
            else go(k_spmv_sell<8, false>, 1);
        }
        launched(c);
        return;
    }
    if (A.nrb > 0) {
        CK(launch_pdl(k_spmv_stream, dim3(A.nrb), dim3(SB_THREADS), 0, st, (const int *)A.rb.p,
                      (const int *)A.ptr.p, (const int *)A.idx.p, (const double *)A.val.p, x, y, b, alpha));
        launched(c);
        return;
    }
    const double avg = A.rows ? (double)A.nnz / A.rows : 0.0;
    const int block = 256;
    auto launch = [&](auto kern, int G) {
        int64_t warps = ((int64_t)A.rows * G + 31) / 32;
        int grid = grid_for(warps * 32, block, c->sms, 8);
        CK(launch_pdl(kern, dim3(grid), dim3(block), 0, st, A.rows, (const int *)A.ptr.p, (const int *)A.idx.p,
                      (const double *)A.val.p, x, y, b, alpha));
    };
    if (avg <= 6) launch(k_spmv<4>, 4);
    else if (avg <= 12) launch(k_spmv<8>, 8);
    else if (avg <= 28) launch(k_spmv<16>, 16);
    else launch(k_spmv<32>, 32);
    launched(c);
}

// ---------------------------------------------------------------- vectors
__global__ void k_fill(double *x, int64_t n, double v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) x[i] = v;
}
__global__ void k_axpy(int64_t n, double a, const double *x, double *y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) y[i] += a * x[i];
}
__global__ void k_axpby_to(int64_t n, const double *x, double a, const double *y, double *o) {
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) o[i] = x[i] + a * y[i];
    pdl_trigger();
}
__global__ void k_div_dev(int64_t n, const double *x, const double *num, double *o) {
    const double d = *num;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) o[i] = x[i] / d;
}

void fill(Ctx *c, double *x, int64_t n, double v, cudaStream_t st) {
    if (!n) return;
    k_fill<<<grid_for(n, 256, c->sms), 256, 0, S(c, st)>>>(x, n, v);
    launched(c);
}
void axpy(Ctx *c, int64_t n, double a, const double *x, double *y, cudaStream_t st) {
    if (!n) return;
    k_axpy<<<grid_for(n, 256, c->sms), 256, 0, S(c, st)>>>(n, a, x, y);
    launched(c);
}
void axpby_to(Ctx *c, int64_t n, const double *x, double a, const double *y, double *o,
              cudaStream_t st) {
    if (!n) return;
    CK(launch_pdl(k_axpby_to, dim3(grid_for(n, 256, c->sms)), dim3(256), 0, S(c, st), n, x, a, y, o));
    launched(c);
}
void scale_by_dev(Ctx *c, int64_t n, const double *x, const double *num, double *o,
                  cudaStream_t st) {
    if (!n) return;
    k_div_dev<<<grid_for(n, 256, c->sms), 256, 0, S(c, st)>>>(n, x, num, o);
    launched(c);
}

// deterministic two-stage sum of squares -> sqrt
__global__ void k_sumsq_partial(int64_t n, const double *x, double *part) {
    __shared__ double sh[32];
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) s += x[i] * x[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) part[blockIdx.x] = s;
    }
}
__global__ void k_sum_sqrt(int np, const double *part, double *out) {
    double s = 0.0;
    for (int i = threadIdx.x; i < np; i += 32) s += part[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *out = sqrt(s);
}

void norm2_dev(Ctx *c, int64_t n, const double *x, double *out_dev, cudaStream_t st) {
    st = S(c, st);
    double *part = st == c->s2 ? c->nrm_part2 : c->nrm_part;
    k_sumsq_partial<<<NRM_BLOCKS, 256, 0, st>>>(n, x, part);
    launched(c);
    k_sum_sqrt<<<1, 32, 0, st>>>(NRM_BLOCKS, part, out_dev);
    launched(c);
}

double norm2(Ctx *c, int64_t n, const double *x) {
    DBuf<double> o(1, c->s);
    norm2_dev(c, n, x, o.p);
    double h = 0;
    CK(cudaMemcpyAsync(&h, o.p, sizeof(double), cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    return h;
}

struct Segs { int64_t d[4], s[4], l[4]; int n; };
__global__ void k_copy_segs(double *dst, const double *src, Segs g) {
    pdl_wait();
#pragma unroll
    for (int k = 0; k < 4; ++k) {   // constant indices: the segment table stays in the parameter bank
        if (k >= g.n) break;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.l[k]; i += (int64_t)gridDim.x * blockDim.x)
            dst[g.d[k] + i] = src[g.s[k] + i];
    }
    pdl_trigger();
}
void copy_segments(Ctx *c, double *dst, const double *src, int nseg, const int64_t *doff,
                   const int64_t *soff, const int64_t *len, cudaStream_t st) {
    Segs g{};
    int64_t tot = 0;
    if (nseg > 4) DPP_FAIL(DPP_ERR_VALUE, "copy_segments: too many segments");
    g.n = nseg;
    for (int k = 0; k < nseg; ++k) g.d[k] = doff[k], g.s[k] = soff[k], g.l[k] = len[k], tot = std::max(tot, len[k]);
    if (!tot) return;
    CK(launch_pdl(k_copy_segs, dim3(grid_for(tot, 256, c->sms)), dim3(256), 0, S(c, st), dst, src, g));
    launched(c);
}

// ---------------------------------------------------------------- CSR utilities
Csr csr_from_host(Ctx *c, int rows, int cols, int64_t nnz, const int *ptr, const int *idx,
                  const double *val) {
    Csr A;
    A.alloc(rows, cols, nnz, c->s);
    A.ptr.upload(ptr, (size_t)rows + 1);
    A.idx.upload(idx, (size_t)nnz);
    A.val.upload(val, (size_t)nnz);
    return A;
}

Csr csr_copy(Ctx *c, const Csr &A) {
    Csr B;
    B.alloc(A.rows, A.cols, A.nnz, c->s);
    CK(cudaMemcpyAsync(B.ptr.p, A.ptr.p, sizeof(int) * (A.rows + 1), cudaMemcpyDeviceToDevice, c->s));
    if (A.nnz) {
        CK(cudaMemcpyAsync(B.idx.p, A.idx.p, sizeof(int) * A.nnz, cudaMemcpyDeviceToDevice, c->s));
        CK(cudaMemcpyAsync(B.val.p, A.val.p, sizeof(double) * A.nnz, cudaMemcpyDeviceToDevice, c->s));
    }
    return B;
}

Csr csr_empty(Ctx *c, int rows, int cols) {
    Csr A;
    A.alloc(rows, cols, 0, c->s);
    CK(cudaMemsetAsync(A.ptr.p, 0, sizeof(int) * (rows + 1), c->s));
    return A;
}

// row filter: keep entry p of row r when pred(r, col, val); warp per row, ordered compaction
struct Pred {
    int part;      // -1 strict lower, 0 diag, 1 strict upper, 2 lower+diag, 3 upper+diag, 9 all
    bool nz;       // also require val != 0
    __device__ bool operator()(int r, int j, double v) const {
        bool ok;
        switch (part) {
            case -1: ok = j < r; break;
            case 0: ok = j == r; break;
            case 1: ok = j > r; break;
            case 2: ok = j <= r; break;
            case 3: ok = j >= r; break;
            default: ok = true;
        }
        return ok && (!nz || v != 0.0);
    }
};

__global__ void k_filter_count(int rows, const int *ptr, const int *idx, const double *val,
                               Pred pr, int *cnt) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        int s = ptr[r], e = ptr[r + 1], n = 0;
        for (int p = s + lane; p < e; p += 32) n += pr((int)r, idx[p], val[p]);
        for (int o = 16; o > 0; o >>= 1) n += __shfl_down_sync(0xffffffffu, n, o);
        if (lane == 0) cnt[r] = n;
    }
}
__global__ void k_filter_fill(int rows, const int *ptr, const int *idx, const double *val,
                              Pred pr, const int *optr, int *oidx, double *oval) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        int s = ptr[r], e = ptr[r + 1], w = optr[r];
        for (int base = s; base < e; base += 32) {
            int p = base + lane;
            bool keep = p < e && pr((int)r, idx[p], val[p]);
            unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                int pos = w + __popc(m & ((1u << lane) - 1));
                oidx[pos] = idx[p];
                oval[pos] = val[p];
            }
            w += __popc(m);
        }
    }
}

static Csr csr_filter(Ctx *c, const Csr &A, Pred pr) {
    DBuf<int> cnt((size_t)A.rows, c->s);
    int grid = grid_for((int64_t)A.rows * 32, 256, c->sms, 8);
    if (A.rows) {
        k_filter_count<<<grid, 256, 0, c->s>>>(A.rows, A.ptr.p, A.idx.p, A.val.p, pr, cnt.p);
        launched(c);
    }
    Csr B;
    B.rows = A.rows;
    B.cols = A.cols;
    B.nnz = counts_to_ptr(c, cnt.p, A.rows, B.ptr);
    B.idx.alloc((size_t)B.nnz, c->s);
    B.val.alloc((size_t)B.nnz, c->s);
    if (A.rows) {
        k_filter_fill<<<grid, 256, 0, c->s>>>(A.rows, A.ptr.p, A.idx.p, A.val.p, pr, B.ptr.p, B.idx.p,
                                              B.val.p);
        launched(c);
    }
    return B;
}

Csr csr_drop_zeros(Ctx *c, const Csr &A) { return csr_filter(c, A, Pred{9, true}); }
Csr csr_part(Ctx *c, const Csr &A, int part, bool dz) { return csr_filter(c, A, Pred{part, dz}); }

int64_t csr_count_nonzero(Ctx *c, const Csr &A) {
    Csr B = csr_drop_zeros(c, A);
    return B.nnz;
}

// rows are sorted and duplicate-free here (canonical CSR), so the diagonal is one
// entry: a warp per row finds it with one ballot
__global__ void k_diag(int rows, const int *ptr, const int *idx, const double *val, double *d,
                       int *missing) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        double v = 0.0;
        bool found = false;
        for (int p = ptr[r] + lane; p < ptr[r + 1]; p += 32)
            if (idx[p] == r) { v += val[p]; found = true; }
        for (int o = 16; o > 0; o >>= 1) {
            v += __shfl_xor_sync(0xffffffffu, v, o);
            found |= __shfl_xor_sync(0xffffffffu, (int)found, o);
        }
        if (lane == 0) {
            d[r] = v;
            if (!found && missing) atomicAdd(missing, 1);
        }
    }
}
__global__ void k_count_zero(int64_t n, const double *d, int *cnt) {
    int z = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        z += d[i] == 0.0;
    z = __reduce_add_sync(0xffffffffu, z);
    if ((threadIdx.x & 31) == 0 && z) atomicAdd(cnt, z);
}
bool any_zero_dev(Ctx *c, int64_t n, const double *d) {
    if (n <= 0) return false;
    DBuf<int> cnt(1, c->s);
    CK(cudaMemsetAsync(cnt.p, 0, sizeof(int), c->s));
    k_count_zero<<<grid_for(n, 256, c->sms, 4), 256, 0, c->s>>>(n, d, cnt.p);
    launched(c);
    int h = 0;
    CK(cudaMemcpyAsync(&h, cnt.p, sizeof(int), cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    return h != 0;
}
void csr_diag(Ctx *c, const Csr &A, double *d, int *missing) {
    int n = std::min(A.rows, A.cols);
    if (!n) return;
    k_diag<<<grid_for((int64_t)n * 32, 256, c->sms, 8), 256, 0, c->s>>>(n, A.ptr.p, A.idx.p, A.val.p, d, missing);
    launched(c);
}

// Transpose = stable radix sort of the column ids (entries enter in row-major order,
// so rows stay ascending inside every column): only ceil(log2(cols)) key bits.
__global__ void k_coo_keys(int rows, const int *ptr, const int *idx, unsigned *key, int *pos, int *rowof) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5)
        for (int p = ptr[r] + lane; p < ptr[r + 1]; p += 32) {
            key[p] = (unsigned)idx[p];
            pos[p] = p;
            rowof[p] = (int)r;
        }
}
__global__ void k_tr_fill(int64_t nnz, const unsigned *key, const int *pos, const int *rowof, const double *val,
                          int *oidx, double *oval, int *cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
        const int p = pos[i];
        oidx[i] = rowof[p];
        oval[i] = val[p];
        atomicAdd(&cnt[key[i]], 1);
    }
}
Csr csr_transpose(Ctx *c, const Csr &A) {
    Csr T;
    T.rows = A.cols;
    T.cols = A.rows;
    T.nnz = A.nnz;
    DBuf<int> cnt((size_t)A.cols + 1, c->s);
    CK(cudaMemsetAsync(cnt.p, 0, sizeof(int) * (A.cols + 1), c->s));
    T.idx.alloc((size_t)A.nnz, c->s);
    T.val.alloc((size_t)A.nnz, c->s);
    if (A.nnz) {
        DBuf<unsigned> k0(A.nnz, c->s), k1(A.nnz, c->s);
        DBuf<int> p0(A.nnz, c->s), p1(A.nnz, c->s), rowof(A.nnz, c->s);
        k_coo_keys<<<grid_for((int64_t)A.rows * 32, 256, c->sms, 8), 256, 0, c->s>>>(A.rows, A.ptr.p, A.idx.p, k0.p,
                                                                                   p0.p, rowof.p);
        launched(c);
        int bits = 1;
        while (bits < 32 && ((int64_t)1 << bits) < (int64_t)A.cols) ++bits;
        size_t tb = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0.p, k1.p, p0.p, p1.p, (int)A.nnz, 0, bits, c->s));
        DBuf<char> t(tb, c->s);
        CK(cub::DeviceRadixSort::SortPairs(t.p, tb, k0.p, k1.p, p0.p, p1.p, (int)A.nnz, 0, bits, c->s));
        launched(c);
        k_tr_fill<<<grid_for(A.nnz, 256, c->sms), 256, 0, c->s>>>(A.nnz, k1.p, p1.p, rowof.p, A.val.p, T.idx.p,
                                                                  T.val.p, cnt.p);
        launched(c);
    }
    counts_to_ptr(c, cnt.p, A.cols, T.ptr);
    return T;
}

// submatrix by segment lists (blocksolve._submatrix: M[rows][:, cols], order preserving)
__global__ void k_sub_count(int nr, const int *rowmap, const int *ptr, const int *idx,
                            const int *colmap, int *cnt) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nr;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        int src = rowmap[r], n = 0;
        for (int p = ptr[src] + lane; p < ptr[src + 1]; p += 32) n += colmap[idx[p]] >= 0;
        for (int o = 16; o > 0; o >>= 1) n += __shfl_down_sync(0xffffffffu, n, o);
        if (lane == 0) cnt[r] = n;
    }
}
__global__ void k_sub_fill(int nr, const int *rowmap, const int *ptr, const int *idx,
                           const double *val, const int *colmap, const int *optr, int *oidx,
                           double *oval) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nr;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        int src = rowmap[r], w = optr[r], s = ptr[src], e = ptr[src + 1];
        for (int base = s; base < e; base += 32) {
            int p = base + lane;
            int m = p < e ? colmap[idx[p]] : -1;
            unsigned b = __ballot_sync(0xffffffffu, m >= 0);
            if (m >= 0) {
                int pos = w + __popc(b & ((1u << lane) - 1));
                oidx[pos] = m;
                oval[pos] = val[p];
            }
            w += __popc(b);
        }
    }
}
Csr csr_submatrix(Ctx *c, const Csr &M, const std::vector<std::pair<int, int>> &rowseg,
                  const std::vector<std::pair<int, int>> &colseg) {
    std::vector<int> rmap, cmap(M.cols, -1);
    for (auto &s : rowseg)
        for (int i = 0; i < s.second; ++i) rmap.push_back(s.first + i);
    int nc = 0;
    for (auto &s : colseg)
        for (int i = 0; i < s.second; ++i) cmap[s.first + i] = nc++;
    int nr = (int)rmap.size();
    DBuf<int> drm(rmap.size(), c->s), dcm(cmap.size(), c->s), cnt(nr, c->s);
    drm.upload(rmap.data(), rmap.size());
    dcm.upload(cmap.data(), cmap.size());
    int grid = grid_for((int64_t)nr * 32, 256, c->sms, 8);
    if (nr) {
        k_sub_count<<<grid, 256, 0, c->s>>>(nr, drm.p, M.ptr.p, M.idx.p, dcm.p, cnt.p);
        launched(c);
    }
    Csr B;
    B.rows = nr;
    B.cols = nc;
    B.nnz = counts_to_ptr(c, cnt.p, nr, B.ptr);
    B.idx.alloc(B.nnz, c->s);
    B.val.alloc(B.nnz, c->s);
    if (nr) {
        k_sub_fill<<<grid, 256, 0, c->s>>>(nr, drm.p, M.ptr.p, M.idx.p, M.val.p, dcm.p, B.ptr.p,
                                           B.idx.p, B.val.p);
        launched(c);
    }
    CK(cudaStreamSynchronize(c->s));  // host vectors go out of scope
    return B;
}

// sp.bmat of a block grid: per output row concatenate the block rows left to right
struct BGrid {
    const int *ptr[16];
    const int *idx[16];
    const double *val[16];
    int roff[5], coff[5];
    int nbr, nbc;
};
__global__ void k_bmat_count(int rows, BGrid g, int *cnt) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
        int I = 0;
        while (r >= g.roff[I + 1]) ++I;
        int lr = r - g.roff[I], n = 0;
        for (int J = 0; J < g.nbc; ++J) {
            const int *p = g.ptr[I * g.nbc + J];
            if (p) n += p[lr + 1] - p[lr];
        }
        cnt[r] = n;
    }
}
__global__ void k_bmat_fill(int rows, BGrid g, const int *optr, int *oidx, double *oval) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        int I = 0;
        while (r >= g.roff[I + 1]) ++I;
        int lr = (int)r - g.roff[I], w = optr[r];
        for (int J = 0; J < g.nbc; ++J) {
            int b = I * g.nbc + J;
            const int *p = g.ptr[b];
            if (!p) continue;
            int s = p[lr], e = p[lr + 1];
            for (int q = s + lane; q < e; q += 32) {
                oidx[w + q - s] = g.idx[b][q] + g.coff[J];
                oval[w + q - s] = g.val[b][q];
            }
            w += e - s;
        }
    }
}
Csr csr_bmat(Ctx *c, const std::vector<const Csr *> &grid, int nbr, int nbc,
             const std::vector<int> &rsz, const std::vector<int> &csz) {
    BGrid g{};
    g.nbr = nbr;
    g.nbc = nbc;
    g.roff[0] = g.coff[0] = 0;
    for (int i = 0; i < nbr; ++i) g.roff[i + 1] = g.roff[i] + rsz[i];
    for (int j = 0; j < nbc; ++j) g.coff[j + 1] = g.coff[j] + csz[j];
    for (int b = 0; b < nbr * nbc; ++b) {
        const Csr *B = grid[b];
        if (B && B->nnz > 0) {
            g.ptr[b] = B->ptr.p;
            g.idx[b] = B->idx.p;
            g.val[b] = B->val.p;
        }
    }
    int rows = g.roff[nbr];
    DBuf<int> cnt(rows, c->s);
    k_bmat_count<<<grid_for(rows, 256, c->sms), 256, 0, c->s>>>(rows, g, cnt.p);
    launched(c);
    Csr K;
    K.rows = rows;
    K.cols = g.coff[nbc];
    K.nnz = counts_to_ptr(c, cnt.p, rows, K.ptr);
    K.idx.alloc(K.nnz, c->s);
    K.val.alloc(K.nnz, c->s);
    k_bmat_fill<<<grid_for((int64_t)rows * 32, 256, c->sms, 8), 256, 0, c->s>>>(rows, g, K.ptr.p,
                                                                                   K.idx.p, K.val.p);
    launched(c);
    return K;
}

}  // namespace dpp
