// Ordered row-merge SpGEMM with scipy's arithmetic (no FMA, zero dropping).
//
// Reference: linalg.schur_selfp (linalg.py:244-254) computes
//   S = D - (C @ diag(1/dA)) @ B
// through scipy's csr_matmat (per output row: sums[j] += a_ik*b_kj over the left
// operand's entries in storage order, starting from 0, exact zeros dropped) and
// csr_binop (d - x over the union, zeros dropped).  C @ diag(.) emits each row
// in reverse first-touch order, i.e. descending k, so the second product
// accumulates over k DESCENDING.  This kernel reproduces that bit-for-bit:
// one warp per output row, a shared-memory open-addressing table keyed by
// column, products accumulated k by k (__syncwarp between k) with separate
// __dmul_rn / __dadd_rn, survivors rank-sorted into canonical CSR order.
// Rows whose column bound exceeds the shared table use a per-row table in
// global memory (same code path through generic pointers).
#include <cstdio>
#include <new>

#include "dpp_internal.cuh"

namespace dpp {

namespace {

constexpr int SM_CAP = 512;     // slots per warp in shared memory (rows with <= 255 distinct columns)
constexpr int WPB = 2;          // warps per block
constexpr int SM_CAP_L = 4096;  // large rows (<= 2047 distinct columns): one warp per block

struct Table {
    int *key;
    unsigned char *has;   // bit0: x present, bit1: d present
    double *x, *d;
    int *lk;
    double *lv;
    int cap;
};

__device__ __forceinline__ unsigned hsh(int j) { return (unsigned)j * 2654435761u; }

__device__ __forceinline__ int tab_slot(Table &t, int j) {
    unsigned h = hsh(j) & (t.cap - 1);
    while (true) {
        int old = atomicCAS(&t.key[h], -1, j);
        if (old == -1 || old == j) return (int)h;
        h = (h + 1) & (t.cap - 1);
    }
}

struct Args {
    int rows;
    const int *ap, *ai;
    const double *av;
    const int *bp, *bi;
    const double *bv;
    const double *s;      // optional column scale of A
    const int *dp, *di;   // optional D
    const double *dv;
    int reverse, keep_zeros;
    const int64_t *goff;  // per-row global table offsets (or -1 => shared)
    const int *gcap;
    int *g_key;
    unsigned char *g_has;
    double *g_x, *g_d, *g_lv;
    int *g_lk;
    int *cnt;             // count pass output
    const int *optr;      // fill pass input
    int *oi;
    double *ov;
};

// CLS: -1 = the row's table is in shared memory of capacity CAP, class chosen
// by goff: -1 small rows (CAP = SM_CAP), -2 large rows (CAP = SM_CAP_L);
// goff >= 0 rows use a global table (processed by the small-row launch)
template <bool FILL, int CAP, int W>
__global__ void __launch_bounds__(32 * W) k_spgemm(Args a, int cls) {
    extern __shared__ unsigned char smem[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t per = (size_t)CAP * (4 + 1 + 8 + 8 + 4 + 8);
    unsigned char *base = smem + per * w;
    for (int64_t row = (int64_t)blockIdx.x * W + w; row < a.rows; row += (int64_t)gridDim.x * W) {
        Table t;
        const int64_t go = a.goff[row];
        if (cls == -1 ? go == -2 : go != -2) continue;   // not this launch's class
        if (go < 0) {
            t.cap = CAP;
            t.x = (double *)base;
            t.d = t.x + CAP;
            t.lv = t.d + CAP;
            t.key = (int *)(t.lv + CAP);
            t.lk = t.key + CAP;
            t.has = (unsigned char *)(t.lk + CAP);
        } else {
            t.cap = a.gcap[row];
            t.key = a.g_key + go;
            t.has = a.g_has + go;
            t.x = a.g_x + go;
            t.d = a.g_d + go;
            t.lk = a.g_lk + go;
            t.lv = a.g_lv + go;
        }
        for (int h = lane; h < t.cap; h += 32) { t.key[h] = -1; t.has[h] = 0; }
        __syncwarp();
        if (a.dp) {
            for (int p = a.dp[row] + lane; p < a.dp[row + 1]; p += 32) {
                int sl = tab_slot(t, a.di[p]);
                t.d[sl] = a.dv[p];
                t.has[sl] |= 2;
            }
            __syncwarp();
        }
        // A's row is fetched 32 entries at a time (k, scaled a_ik, B-row bounds in lane
        // registers); the next k's B entries are prefetched while the current k is
        // accumulated, so the k-ordered loop does not wait on global memory.
        const int s = a.ap[row], e = a.ap[row + 1], len = e - s;
        for (int q0 = 0; q0 < len; q0 += 32) {
            int bs = 0, be = 0;
            double aq = 0.0;
            if (q0 + lane < len) {
                const int p = a.reverse ? e - 1 - (q0 + lane) : s + q0 + lane;
                const int kq = a.ai[p];
                aq = a.av[p];
                if (a.s) aq = __dmul_rn(aq, a.s[kq]);
                bs = a.bp[kq];
                be = a.bp[kq + 1];
            }
            const int cnt = min(32, len - q0);
            int cj = -1;
            double cb = 0.0;
            {
                const int rs = __shfl_sync(0xffffffffu, bs, 0), re = __shfl_sync(0xffffffffu, be, 0);
                if (rs + lane < re) { cj = a.bi[rs + lane]; cb = a.bv[rs + lane]; }
            }
            for (int qq = 0; qq < cnt; ++qq) {
                const double av = __shfl_sync(0xffffffffu, aq, qq);
                const int rs = __shfl_sync(0xffffffffu, bs, qq), re = __shfl_sync(0xffffffffu, be, qq);
                const int ns = __shfl_sync(0xffffffffu, bs, (qq + 1) & 31), ne = __shfl_sync(0xffffffffu, be, (qq + 1) & 31);
                int nj = -1;
                double nbv = 0.0;
                if (qq + 1 < cnt && ns + lane < ne) { nj = a.bi[ns + lane]; nbv = a.bv[ns + lane]; }
                if (av != 0.0) {   // zero products never change a sum (scipy drops them)
                    auto acc = [&](int j, double bv) {
                        if (bv == 0.0) return;
                        const double pr = __dmul_rn(av, bv);
                        const int sl = tab_slot(t, j);
                        if (t.has[sl] & 1) t.x[sl] = __dadd_rn(t.x[sl], pr);
                        else { t.x[sl] = __dadd_rn(0.0, pr); t.has[sl] |= 1; }
                    };
                    if (cj >= 0) acc(cj, cb);
                    for (int r = rs + 32 + lane; r < re; r += 32) acc(a.bi[r], a.bv[r]);
                    __syncwarp();
                }
                cj = nj;
                cb = nbv;
            }
        }
        // survivors (slot order), then rank sort by column
        int nsurv = 0;
        for (int h0 = 0; h0 < t.cap; h0 += 32) {
            const int h = h0 + lane;
            bool keep = false;
            double v = 0.0;
            int j = -1;
            if (h < t.cap && t.key[h] >= 0) {
                const unsigned char f = t.has[h];
                j = t.key[h];
                if (!a.dp) v = t.x[h];                                   // C = A B
                else if (f & 1) v = (f & 2) ? __dsub_rn(t.d[h], t.x[h]) : -t.x[h];   // D - X
                else v = t.d[h];
                keep = a.keep_zeros || v != 0.0;
            }
            unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                int pos = nsurv + __popc(m & ((1u << lane) - 1));
                t.lk[pos] = j;
                t.lv[pos] = v;
            }
            nsurv += __popc(m);
        }
        __syncwarp();
        if (!FILL) {
            if (lane == 0) a.cnt[row] = nsurv;
        } else {
            const int o = a.optr[row];
            for (int u = lane; u < nsurv; u += 32) {
                const int j = t.lk[u];
                int rank = 0;
                for (int v = 0; v < nsurv; ++v) rank += t.lk[v] < j;
                a.oi[o + rank] = j;
                a.ov[o + rank] = t.lv[u];
            }
        }
        __syncwarp();
    }
}

// Dense-accumulator variant for products with a small column space (coarse AMG
// levels): each warp owns acc[ncols] + presence flags in shared memory, the
// k-ordered accumulation is the same as the hashed kernel, and survivors come
// out in column order (no sort).
template <bool FILL>
__global__ void k_spgemm_dense(Args a, int ncols, int W) {
    extern __shared__ unsigned char smem[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t per = (size_t)ncols * 8 * 2 + (size_t)((ncols + 15) & ~15);
    double *acc = reinterpret_cast<double *>(smem + per * w);
    double *dv = acc + ncols;
    unsigned char *has = reinterpret_cast<unsigned char *>(dv + ncols);
    for (int64_t row = (int64_t)blockIdx.x * W + w; row < a.rows; row += (int64_t)gridDim.x * W) {
        for (int j = lane; j < ncols; j += 32) has[j] = 0;
        __syncwarp();
        if (a.dp) {
            for (int p = a.dp[row] + lane; p < a.dp[row + 1]; p += 32) {
                dv[a.di[p]] = a.dv[p];
                has[a.di[p]] |= 2;
            }
            __syncwarp();
        }
        const int s = a.ap[row], e = a.ap[row + 1], len = e - s;
        for (int q0 = 0; q0 < len; q0 += 32) {
            int bs = 0, be = 0;
            double aq = 0.0;
            if (q0 + lane < len) {
                const int p = a.reverse ? e - 1 - (q0 + lane) : s + q0 + lane;
                const int kq = a.ai[p];
                aq = a.av[p];
                if (a.s) aq = __dmul_rn(aq, a.s[kq]);
                bs = a.bp[kq];
                be = a.bp[kq + 1];
            }
            const int cnt = min(32, len - q0);
            for (int qq = 0; qq < cnt; ++qq) {
                const double av = __shfl_sync(0xffffffffu, aq, qq);
                const int rs = __shfl_sync(0xffffffffu, bs, qq), re = __shfl_sync(0xffffffffu, be, qq);
                if (av == 0.0) continue;
                for (int r = rs + lane; r < re; r += 32) {
                    const double bv = a.bv[r];
                    if (bv == 0.0) continue;
                    const int j = a.bi[r];
                    const double pr = __dmul_rn(av, bv);
                    if (has[j] & 1) acc[j] = __dadd_rn(acc[j], pr);
                    else { acc[j] = __dadd_rn(0.0, pr); has[j] |= 1; }
                }
                __syncwarp();
            }
        }
        int w0 = FILL ? a.optr[row] : 0, nsurv = 0;
        for (int j0 = 0; j0 < ncols; j0 += 32) {
            const int j = j0 + lane;
            bool keep = false;
            double v = 0.0;
            if (j < ncols && has[j]) {
                const unsigned char f = has[j];
                if (!a.dp) v = acc[j];
                else if (f & 1) v = (f & 2) ? __dsub_rn(dv[j], acc[j]) : -acc[j];
                else v = dv[j];
                keep = a.keep_zeros || v != 0.0;
            }
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (FILL && keep) {
                const int pos = w0 + nsurv + __popc(m & ((1u << lane) - 1));
                a.oi[pos] = j;
                a.ov[pos] = v;
            }
            nsurv += __popc(m);
        }
        if (!FILL && lane == 0) a.cnt[row] = nsurv;
        __syncwarp();
    }
}

// upper bound of distinct columns per row -> table placement
__global__ void k_bound(int rows, const int *ap, const int *ai, const int *bp, const int *dp,
                        int bcols, int64_t *need) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
        int64_t ub = dp ? dp[r + 1] - dp[r] : 0;
        for (int p = ap[r]; p < ap[r + 1]; ++p) ub += bp[ai[p] + 1] - bp[ai[p]];
        if (ub > bcols) ub = bcols;
        need[r] = ub;
    }
}

constexpr int UCAP = 8192;   // key-only slots per warp for the symbolic pass
constexpr int UWPB = 1;

__global__ void __launch_bounds__(32 * UWPB) k_unique(int rows, const int *ap, const int *ai,
                                                      const int *bp, const int *bi, const int *dp,
                                                      const int *di, const int64_t *goff,
                                                      const int *gcap, int *gkey, int *uniq) {
    __shared__ int sk[UWPB][UCAP];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t row = (int64_t)blockIdx.x * UWPB + w; row < rows; row += (int64_t)gridDim.x * UWPB) {
        int *key;
        int cap;
        if (goff[row] < 0) { key = sk[w]; cap = UCAP; }
        else { key = gkey + goff[row]; cap = gcap[row]; }
        for (int h = lane; h < cap; h += 32) key[h] = -1;
        __syncwarp();
        int n = 0;
        auto ins = [&](int j) {
            unsigned h = hsh(j) & (cap - 1);
            while (true) {
                int old = atomicCAS(&key[h], -1, j);
                if (old == -1) { ++n; return; }
                if (old == j) return;
                h = (h + 1) & (cap - 1);
            }
        };
        if (dp)
            for (int p = dp[row] + lane; p < dp[row + 1]; p += 32) ins(di[p]);
        const int s = ap[row], len = ap[row + 1] - s;
        for (int q0 = 0; q0 < len; q0 += 32) {
            int bs = 0, be = 0;
            if (q0 + lane < len) {
                const int kq = ai[s + q0 + lane];
                bs = bp[kq];
                be = bp[kq + 1];
            }
            const int cnt = min(32, len - q0);
            for (int qq = 0; qq < cnt; ++qq) {
                const int rs = __shfl_sync(0xffffffffu, bs, qq), re = __shfl_sync(0xffffffffu, be, qq);
                for (int r = rs + lane; r < re; r += 32) ins(bi[r]);
            }
        }
        for (int o = 16; o > 0; o >>= 1) n += __shfl_down_sync(0xffffffffu, n, o);
        if (lane == 0) uniq[row] = n;
        __syncwarp();
    }
}

}  // namespace

Csr spgemm(Ctx *c, const Csr &A, const Csr &B, const double *s_dev, bool reverse, const Csr *D,
           bool keep_zeros) {
    if (A.cols != B.rows) DPP_FAIL(DPP_ERR_VALUE, "spgemm: dimension mismatch");
    if (D && (D->rows != A.rows || D->cols != B.cols)) DPP_FAIL(DPP_ERR_VALUE, "spgemm: D shape");
    const int rows = A.rows;
    Csr C;
    C.rows = rows;
    C.cols = B.cols;
    if (rows == 0) {
        C.ptr.alloc(1, c->s);
        CK(cudaMemsetAsync(C.ptr.p, 0, sizeof(int), c->s));
        return C;
    }
    DPP_TRACE_SCOPE(c, "spgemm");
    // small column space and dense-ish rows: dense accumulator, no hashing / sorting
    {
        const int ncols = B.cols;
        const size_t per = (size_t)ncols * 16 + (size_t)((ncols + 15) & ~15);
        const double avg_out = rows ? (double)std::min<int64_t>((int64_t)ncols, (int64_t)((double)A.nnz / rows * ((double)B.nnz / std::max(1, B.rows)))) : 0.0;
        if (ncols <= 4096 && avg_out * 8 >= ncols && per <= 200 * 1024) {
            const int W = (int)std::max<size_t>(1, std::min<size_t>(8, (200 * 1024) / per));
            const size_t smem_d = per * W;
            static bool dattr = false;
            if (!dattr) {
                CK(cudaFuncSetAttribute(k_spgemm_dense<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
                CK(cudaFuncSetAttribute(k_spgemm_dense<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
                dattr = true;
            }
            Args a{};
            a.rows = rows;
            a.ap = A.ptr.p; a.ai = A.idx.p; a.av = A.val.p;
            a.bp = B.ptr.p; a.bi = B.idx.p; a.bv = B.val.p;
            a.s = s_dev;
            if (D) { a.dp = D->ptr.p; a.di = D->idx.p; a.dv = D->val.p; }
            a.reverse = reverse;
            a.keep_zeros = keep_zeros;
            DBuf<int> cnt(rows, c->s);
            a.cnt = cnt.p;
            const int grid = std::max(1, std::min<int>((rows + W - 1) / W, c->sms * 4));
            k_spgemm_dense<false><<<grid, 32 * W, smem_d, c->s>>>(a, ncols, W);
            launched(c);
            C.nnz = counts_to_ptr(c, cnt.p, rows, C.ptr);
            C.idx.alloc(C.nnz, c->s);
            C.val.alloc(C.nnz, c->s);
            a.optr = C.ptr.p;
            a.oi = C.idx.p;
            a.ov = C.val.p;
            k_spgemm_dense<true><<<grid, 32 * W, smem_d, c->s>>>(a, ncols, W);
            launched(c);
            CK(cudaStreamSynchronize(c->s));
            return C;
        }
    }
    // 1) bound of distinct columns per row; 2) exact distinct count; 3) table placement
    DBuf<int64_t> need(rows, c->s);
    k_bound<<<grid_for(rows, 256, c->sms), 256, 0, c->s>>>(rows, A.ptr.p, A.idx.p, B.ptr.p,
                                                          D ? D->ptr.p : nullptr, B.cols, need.p);
    launched(c);
    std::vector<int64_t> h = need.to_host();
    DPP_TRACE_SCOPE(c, "spgemm.after_bound");
    std::vector<int64_t> uoff(rows, -1);
    std::vector<int> ucap(rows, 0);
    int64_t utot = 0;
    for (int r = 0; r < rows; ++r) {
        if (h[r] < UCAP - 1) continue;
        int cap = 64;
        while (cap < 2 * h[r] + 2) cap <<= 1;
        uoff[r] = utot;
        ucap[r] = cap;
        utot += cap;
    }
    std::vector<int> u(rows);
    {
        DPP_TRACE_SCOPE(c, "spgemm.unique");
        DBuf<int64_t> duoff(rows, c->s);
        DBuf<int> ducap(rows, c->s), dkey(utot, c->s), duniq(rows, c->s);
        duoff.upload(uoff.data(), rows);
        ducap.upload(ucap.data(), rows);
        k_unique<<<grid_for((int64_t)rows * 32, 32 * UWPB, c->sms, 12), 32 * UWPB, 0, c->s>>>(
            rows, A.ptr.p, A.idx.p, B.ptr.p, B.idx.p, D ? D->ptr.p : nullptr,
            D ? D->idx.p : nullptr, duoff.p, ducap.p, dkey.p, duniq.p);
        launched(c);
        duniq.download(u.data(), rows);
        CK(cudaStreamSynchronize(c->s));
    }
    std::vector<int64_t> goff(rows, -1);
    std::vector<int> gcap(rows, 0);
    int64_t gtot = 0;
    int nlarge = 0;
    for (int r = 0; r < rows; ++r) {
        if (2 * (int64_t)u[r] + 2 <= SM_CAP) continue;
        if (2 * (int64_t)u[r] + 2 <= SM_CAP_L) { goff[r] = -2; ++nlarge; continue; }
        int cap = 64;
        while (cap < 2 * (int64_t)u[r] + 2) cap <<= 1;
        goff[r] = gtot;
        gcap[r] = cap;
        gtot += cap;
    }
    DBuf<int64_t> dgoff(rows, c->s);
    DBuf<int> dgcap(rows, c->s);
    dgoff.upload(goff.data(), rows);
    dgcap.upload(gcap.data(), rows);
    DBuf<int> gk(gtot, c->s), glk(gtot, c->s);
    DBuf<unsigned char> ghas(gtot, c->s);
    DBuf<double> gx(gtot, c->s), gd(gtot, c->s), glv(gtot, c->s);
    DBuf<int> cnt(rows, c->s);

    Args a{};
    a.rows = rows;
    a.ap = A.ptr.p; a.ai = A.idx.p; a.av = A.val.p;
    a.bp = B.ptr.p; a.bi = B.idx.p; a.bv = B.val.p;
    a.s = s_dev;
    if (D) { a.dp = D->ptr.p; a.di = D->idx.p; a.dv = D->val.p; }
    a.reverse = reverse;
    a.keep_zeros = keep_zeros;
    a.goff = dgoff.p; a.gcap = dgcap.p;
    a.g_key = gk.p; a.g_has = ghas.p; a.g_x = gx.p; a.g_d = gd.p; a.g_lk = glk.p; a.g_lv = glv.p;
    a.cnt = cnt.p;
    const size_t smem = (size_t)WPB * SM_CAP * (4 + 1 + 8 + 8 + 4 + 8);
    const size_t smem_l = (size_t)SM_CAP_L * (4 + 1 + 8 + 8 + 4 + 8);
    static bool attr = false;
    if (!attr) {
        CK(cudaFuncSetAttribute(k_spgemm<false, SM_CAP, WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaFuncSetAttribute(k_spgemm<true, SM_CAP, WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaFuncSetAttribute(k_spgemm<false, SM_CAP_L, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_l));
        CK(cudaFuncSetAttribute(k_spgemm<true, SM_CAP_L, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_l));
        attr = true;
    }
    const int grid = grid_for((int64_t)rows * 32 * WPB / WPB, 32 * WPB, c->sms, 12);
    const int grid_l = std::max(1, std::min(nlarge, c->sms));
    if (TraceScope::on()) {
        int nglob = 0;
        for (int r = 0; r < rows; ++r) nglob += goff[r] >= 0;
        std::fprintf(stderr, "[dpp-trace]   spgemm %d x %d (A nnz %lld, B nnz %lld): %d large, %d global, gtot %lld\n",
                     rows, B.cols, (long long)A.nnz, (long long)B.nnz, nlarge, nglob, (long long)gtot);
    }
    TraceScope ts_count(c, "spgemm.count");
    k_spgemm<false, SM_CAP, WPB><<<grid, 32 * WPB, smem, c->s>>>(a, -1);
    launched(c);
    if (nlarge) {
        k_spgemm<false, SM_CAP_L, 1><<<grid_l, 32, smem_l, c->s>>>(a, -2);
        launched(c);
    }
    ts_count.~TraceScope();
    new (&ts_count) TraceScope(c, "spgemm.fill");
    C.nnz = counts_to_ptr(c, cnt.p, rows, C.ptr);
    C.idx.alloc(C.nnz, c->s);
    C.val.alloc(C.nnz, c->s);
    a.optr = C.ptr.p;
    a.oi = C.idx.p;
    a.ov = C.val.p;
    k_spgemm<true, SM_CAP, WPB><<<grid, 32 * WPB, smem, c->s>>>(a, -1);
    launched(c);
    if (nlarge) {
        k_spgemm<true, SM_CAP_L, 1><<<grid_l, 32, smem_l, c->s>>>(a, -2);
        launched(c);
    }
    CK(cudaStreamSynchronize(c->s));   // host vectors above go out of scope
    return C;
}

}  // namespace dpp
