// Ordered row-merge SpGEMM with scipy's arithmetic (no FMA, zero dropping).
//
// Reference: linalg.schur_selfp (linalg.py:244-254) computes
//   S = D - (C @ diag(1/dA)) @ B
// through scipy's csr_matmat (per output row: sums[j] += a_ik*b_kj over the left
// operand's entries in storage order, starting from 0, exact zeros dropped) and
// csr_binop (d - x over the union, zeros dropped).  C @ diag(.) emits each row
// in reverse first-touch order, i.e. descending k, so the second product
// accumulates over k DESCENDING.  The AMG Galerkin products (linalg.py:341-370)
// are plain csr_matmat products.  Every path below reproduces that bit-for-bit:
// one warp per output row, products accumulated k by k (__syncwarp between k)
// with separate __dmul_rn / __dadd_rn, survivors emitted in column order.
//
// Pipeline (hashed path):
//   1. symbolic: distinct columns per row in a 1024-key shared table (8 warps
//      per CTA); rows that overflow it are recounted with an 8192-key table or a
//      per-row global table sized from the row's product bound
//   2. numeric: ONE pass per size class (shared tables of 256 / 1024 / 4096
//      slots, or global), survivors rank-sorted by column and written to a
//      scratch at the row's symbolic offset, with the surviving count
//   3. compaction of the scratch into canonical CSR
// Small column spaces (coarse levels) use a dense per-warp accumulator instead,
// whose survivors come out in column order without sorting.
#include <cstdio>
#include <cstdlib>
#include <new>

#include <cub/cub.cuh>

#include "dpp_internal.cuh"

namespace dpp {

namespace {

__device__ __forceinline__ unsigned hsh(int j) { return (unsigned)j * 2654435761u; }

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
    int bmax;             // longest B row (host-side choice of the register prefetch depth)
    // numeric pass: rows of this launch and their global tables (if any)
    const int *rl;
    int nrl;
    const int64_t *goff;  // per list entry: global table offset (class G) or unused
    const int *gcap;
    int *g_key;
    unsigned char *g_has;
    double *g_x, *g_d;
    // output: sorted survivors at toff[row] in the scratch, count in cnt[row]
    const int64_t *toff;
    int *ti;
    double *tv;
    int *cnt;
};

// The k-ordered accumulation loop shared by the hashed and dense kernels: A's row
// is taken 32 entries at a time (k, scaled a_ik, B-row bounds in lane registers);
// each k's B row is held in registers (up to PF x 32 entries) and the NEXT k's
// row is loaded while the current one is accumulated.
constexpr int PF_HASH = 4;
template <int PF, typename Upd>
__device__ __forceinline__ void accumulate_row(const Args &a, int64_t row, int lane, Upd &&upd, int qb = 0,
                                               int qe = 0x7fffffff) {
    const int s = a.ap[row], e = a.ap[row + 1], len = min(e - s, qe);
    for (int q0 = qb; q0 < len; q0 += 32) {
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
        int cj[PF];
        double cb[PF];
        {
            const int rs = __shfl_sync(0xffffffffu, bs, 0), re = __shfl_sync(0xffffffffu, be, 0);
#pragma unroll
            for (int u = 0; u < PF; ++u) {
                const int r = rs + 32 * u + lane;
                cj[u] = r < re ? a.bi[r] : -1;
                cb[u] = r < re ? a.bv[r] : 0.0;
            }
        }
        for (int qq = 0; qq < cnt; ++qq) {
            const double av = __shfl_sync(0xffffffffu, aq, qq);
            const int rs = __shfl_sync(0xffffffffu, bs, qq), re = __shfl_sync(0xffffffffu, be, qq);
            const int ns = __shfl_sync(0xffffffffu, bs, (qq + 1) & 31), ne = __shfl_sync(0xffffffffu, be, (qq + 1) & 31);
            int nj[PF];
            double nb[PF];
#pragma unroll
            for (int u = 0; u < PF; ++u) {
                const int r = ns + 32 * u + lane;
                const bool ok = qq + 1 < cnt && r < ne;
                nj[u] = ok ? a.bi[r] : -1;
                nb[u] = ok ? a.bv[r] : 0.0;
            }
            if (av != 0.0) {   // zero products never change a sum (scipy drops them)
#pragma unroll
                for (int u = 0; u < PF; ++u)
                    if (cj[u] >= 0 && cb[u] != 0.0) upd(cj[u], __dmul_rn(av, cb[u]));
                // long B rows (dense coarse products): 4 x 32 entries in flight per batch;
                // every (k, j) pair is unique, so the per-j accumulation order stays k-ordered
                for (int r0 = rs + 32 * PF; r0 < re; r0 += 32 * 4) {
                    int bj[4];
                    double bb[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int r = r0 + 32 * u + lane;
                        bj[u] = r < re ? a.bi[r] : -1;
                        bb[u] = r < re ? a.bv[r] : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (bj[u] >= 0 && bb[u] != 0.0) upd(bj[u], __dmul_rn(av, bb[u]));
                }
                __syncwarp();
            }
#pragma unroll
            for (int u = 0; u < PF; ++u) { cj[u] = nj[u]; cb[u] = nb[u]; }
        }
    }
}

// ---------------------------------------------------------------- symbolic
constexpr int US_CAP = 1024;   // keys per warp, small symbolic table
constexpr int US_LIM = 768;    // distinct columns before a row is sent to the large path
constexpr int US_W = 8;

__global__ void __launch_bounds__(32 * US_W) k_unique_s(int rows, const int *ap, const int *ai, const int *bp,
                                                        const int *bi, const int *dp, const int *di, int *uniq) {
    __shared__ int sk[US_W][US_CAP];
    __shared__ int sn[US_W];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int *key = sk[w];
    for (int64_t row = (int64_t)blockIdx.x * US_W + w; row < rows; row += (int64_t)gridDim.x * US_W) {
        for (int h = lane; h < US_CAP; h += 32) key[h] = -1;
        if (lane == 0) sn[w] = 0;
        __syncwarp();
        bool over = false;
        auto ins = [&](int j) {
            if (over) return;
            unsigned h = hsh(j) & (US_CAP - 1);
            while (true) {
                const int old = atomicCAS(&key[h], -1, j);
                if (old == -1) {
                    if (atomicAdd(&sn[w], 1) >= US_LIM) over = true;
                    return;
                }
                if (old == j) return;
                h = (h + 1) & (US_CAP - 1);
            }
        };
        if (dp)
            for (int p = dp[row] + lane; p < dp[row + 1]; p += 32) ins(di[p]);
        // the symbolic pass needs no k order: each lane inserts its own k's B row, four
        // column ids loaded ahead of the inserts (the CAS loop would serialise them)
        for (int p0 = ap[row]; p0 < ap[row + 1]; p0 += 32) {
            const int p = p0 + lane;
            int rs = 0, re = 0;
            if (p < ap[row + 1]) {
                const int kq = ai[p];
                rs = bp[kq];
                re = bp[kq + 1];
            }
            const int mlen = __reduce_max_sync(0xffffffffu, re - rs);
            for (int u = 0; u < mlen; u += 4) {
                int j[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) j[q] = rs + u + q < re ? bi[rs + u + q] : -1;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (j[q] >= 0) ins(j[q]);
            }
        }
        over = __any_sync(0xffffffffu, over);
        __syncwarp();
        if (lane == 0) uniq[row] = over ? -1 : sn[w];
        __syncwarp();
    }
}

// rows of a list, table of up to UCAP keys in shared memory or per row in global memory
constexpr int UCAP = 8192;
__global__ void __launch_bounds__(32) k_unique_l(const int *rl, int nrl, const int *ap, const int *ai, const int *bp,
                                                 const int *bi, const int *dp, const int *di, const int64_t *goff,
                                                 const int *gcap, int *gkey, int *uniq) {
    __shared__ int sk[UCAP];
    const int lane = threadIdx.x;
    for (int li = blockIdx.x; li < nrl; li += gridDim.x) {
        const int row = rl[li];
        int *key;
        int cap;
        if (goff[li] < 0) { key = sk; cap = UCAP; }
        else { key = gkey + goff[li]; cap = gcap[li]; }
        for (int h = lane; h < cap; h += 32) key[h] = -1;
        __syncwarp();
        int n = 0;
        auto ins = [&](int j) {
            unsigned h = hsh(j) & (cap - 1);
            while (true) {
                const int old = atomicCAS(&key[h], -1, j);
                if (old == -1) { ++n; return; }
                if (old == j) return;
                h = (h + 1) & (cap - 1);
            }
        };
        if (dp)
            for (int p = dp[row] + lane; p < dp[row + 1]; p += 32) ins(di[p]);
        for (int p = ap[row] + lane; p < ap[row + 1]; p += 32) {
            const int kq = ai[p];
            for (int r = bp[kq]; r < bp[kq + 1]; ++r) ins(bi[r]);
        }
        for (int o = 16; o > 0; o >>= 1) n += __shfl_down_sync(0xffffffffu, n, o);
        if (lane == 0) uniq[row] = n;
        __syncwarp();
    }
}

// product bound per listed row (sizes the global symbolic tables)
__global__ void k_bound_list(const int *rl, int nrl, const int *ap, const int *ai, const int *bp, const int *dp,
                             int bcols, int64_t *need) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nrl; i += gridDim.x * blockDim.x) {
        const int r = rl[i];
        int64_t ub = dp ? dp[r + 1] - dp[r] : 0;
        for (int p = ap[r]; p < ap[r + 1]; ++p) ub += bp[ai[p] + 1] - bp[ai[p]];
        need[i] = ub < bcols ? ub : bcols;
    }
}

// ---------------------------------------------------------------- numeric
struct Table {
    int *key;
    unsigned char *has;   // bit0: x present, bit1: d present
    double *x, *d;
    int cap;
};
__device__ __forceinline__ int tab_slot(Table &t, int j) {
    unsigned h = hsh(j) & (t.cap - 1);
    while (true) {
        const int old = atomicCAS(&t.key[h], -1, j);
        if (old == -1 || old == j) return (int)h;
        h = (h + 1) & (t.cap - 1);
    }
}
// shared table per warp: x[CAP] | d[CAP] (only with a D operand) | key[CAP] | has[CAP];
// survivors are compacted in place (key -> column, x -> value)
__host__ __device__ constexpr int slot_bytes(bool has_d) { return 8 + (has_d ? 8 : 0) + 4 + 1; }

// CAP: shared table slots per warp (0 => global tables); K: survivor keys per
// lane held in registers for ranking (0 => rank loop over shared memory)
// TR (trial pass, no symbolic pass before it): every row, a budget of TR_LIM distinct
// columns per row, survivors at row * TR_LIM in the scratch; a row over budget is
// abandoned with cnt = -1 (the caller then runs the symbolic + sized passes instead)
constexpr int TR_LIM = 128;
template <int CAP, int W, int K, bool HD, int PF, bool TR = false>
__global__ void __launch_bounds__(32 * W) k_spgemm_num(Args a) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int tr_n[W];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char *base = smem + (size_t)CAP * slot_bytes(HD) * w;
    for (int li = blockIdx.x * W + w; li < a.nrl; li += gridDim.x * W) {
        const int row = TR ? li : a.rl[li];
        Table t;
        if (CAP > 0) {
            t.cap = CAP;
            t.x = (double *)base;
            t.d = HD ? t.x + CAP : t.x;
            t.key = (int *)(t.x + (HD ? 2 : 1) * CAP);
            t.has = (unsigned char *)(t.key + CAP);
        } else {
            const int64_t go = a.goff[li];
            t.cap = a.gcap[li];
            t.key = a.g_key + go;
            t.has = a.g_has + go;
            t.x = a.g_x + go;
            t.d = a.g_d + go;
        }
        for (int h = lane; h < t.cap; h += 32) { t.key[h] = -1; t.has[h] = 0; }
        if (TR && lane == 0) tr_n[w] = 0;
        __syncwarp();
        // slot of column j; in a trial pass -1 once the row is over budget (inserts stop,
        // so the table never fills: at most TR_LIM + 31 keys)
        auto slot = [&](int j) -> int {
            if (!TR) return tab_slot(t, j);
            unsigned h = hsh(j) & (t.cap - 1);
            while (true) {
                const int cur = t.key[h];
                if (cur == j) return (int)h;
                if (cur == -1) {
                    if (*(volatile int *)&tr_n[w] >= TR_LIM) return -1;
                    const int old = atomicCAS(&t.key[h], -1, j);
                    if (old == -1) { atomicAdd(&tr_n[w], 1); return (int)h; }
                    if (old == j) return (int)h;
                }
                h = (h + 1) & (t.cap - 1);
            }
        };
        if (HD) {
            for (int p = a.dp[row] + lane; p < a.dp[row + 1]; p += 32) {
                const int sl = slot(a.di[p]);
                if (TR && sl < 0) continue;
                t.d[sl] = a.dv[p];
                t.has[sl] |= 2;
            }
            __syncwarp();
        }
        accumulate_row<PF>(a, row, lane, [&](int j, double pr) {
            const int sl = slot(j);
            if (TR && sl < 0) return;
            if (t.has[sl] & 1) t.x[sl] = __dadd_rn(t.x[sl], pr);
            else { t.x[sl] = __dadd_rn(0.0, pr); t.has[sl] |= 1; }
        });
        if (TR) {
            __syncwarp();
            if (*(volatile int *)&tr_n[w] >= TR_LIM) {
                if (lane == 0) a.cnt[row] = -1;
                __syncwarp();
                continue;
            }
        }
        // survivors compacted in place, in slot order (a survivor's position never
        // exceeds its slot, so no unread slot is overwritten) ...
        int nsurv = 0;
        for (int h0 = 0; h0 < t.cap; h0 += 32) {
            const int h = h0 + lane;
            bool keep = false;
            double v = 0.0;
            int j = -1;
            if (h < t.cap && t.key[h] >= 0) {
                const unsigned char f = t.has[h];
                j = t.key[h];
                if (!HD) v = t.x[h];                                                 // C = A B
                else if (f & 1) v = (f & 2) ? __dsub_rn(t.d[h], t.x[h]) : -t.x[h];   // D - X
                else v = t.d[h];
                keep = a.keep_zeros || v != 0.0;
            }
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const int pos = nsurv + __popc(m & ((1u << lane) - 1));
                t.key[pos] = j;
                t.x[pos] = v;
            }
            nsurv += __popc(m);
            __syncwarp();
        }
        // ... ranked by column into the scratch
        const int64_t o = TR ? (int64_t)row * TR_LIM : a.toff[row];
        if (K > 0) {
            int mk[K > 0 ? K : 1], rk[K > 0 ? K : 1];
#pragma unroll
            for (int u = 0; u < K; ++u) {
                const int q = u * 32 + lane;
                mk[u] = q < nsurv ? t.key[q] : 0x7fffffff;
                rk[u] = 0;
            }
            for (int v = 0; v < nsurv; ++v) {
                const int kv = t.key[v];
#pragma unroll
                for (int u = 0; u < K; ++u) rk[u] += kv < mk[u];
            }
#pragma unroll
            for (int u = 0; u < K; ++u) {
                const int q = u * 32 + lane;
                if (q < nsurv) { a.ti[o + rk[u]] = mk[u]; a.tv[o + rk[u]] = t.x[q]; }
            }
        } else {
            for (int q = lane; q < nsurv; q += 32) {
                const int j = t.key[q];
                int rank = 0;
                for (int v = 0; v < nsurv; ++v) rank += t.key[v] < j;
                a.ti[o + rank] = j;
                a.tv[o + rank] = t.x[q];
            }
        }
        if (lane == 0) a.cnt[row] = nsurv;
        __syncwarp();
    }
}

// Dense-accumulator variant for products with a small column space (coarse AMG
// levels): each warp owns acc[ncols] + presence flags in shared memory; the
// survivors come out in column order (no sort), written to the scratch at
// toff[row] (= row * ncols).
template <int PFD>
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
        accumulate_row<PFD>(a, row, lane, [&](int j, double pr) {
            if (has[j] & 1) acc[j] = __dadd_rn(acc[j], pr);
            else { acc[j] = __dadd_rn(0.0, pr); has[j] |= 1; }
        });
        const int64_t o = a.toff[row];
        int nsurv = 0;
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
            if (keep) {
                const int64_t pos = o + nsurv + __popc(m & ((1u << lane) - 1));
                a.ti[pos] = j;
                a.tv[pos] = v;
            }
            nsurv += __popc(m);
        }
        if (lane == 0) a.cnt[row] = nsurv;
        __syncwarp();
    }
}

// Split-k dense variant for few long output rows (the Galerkin product R (A P) of a
// coarse level: ~600 rows of ~250 k-terms over ~500-entry B rows): one CTA per row,
// warp w accumulates the k-range w of the row in its own dense accumulator (k order
// inside the range), the 8 partials are added in warp order, survivors compacted in
// column order.  Differs from the k-sequential sum by rounding only (coarse levels
// are insensitive to it; the reference's association is (P^T A) P).
constexpr int SK_W = 8;
template <int PFD>
__global__ void __launch_bounds__(32 * SK_W) k_spgemm_dense_splitk(Args a, int ncols) {
    extern __shared__ unsigned char smem[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *accs = reinterpret_cast<double *>(smem);                       // [SK_W][ncols]
    double *dv = accs + (size_t)SK_W * ncols;                              // [ncols]
    unsigned char *has = reinterpret_cast<unsigned char *>(dv + ncols);    // [SK_W][ncols]
    __shared__ int wsum[SK_W];
    const int64_t row = blockIdx.x;
    for (int j = threadIdx.x; j < SK_W * ncols; j += blockDim.x) has[j] = 0;
    __syncthreads();
    if (a.dp) {
        for (int p = a.dp[row] + threadIdx.x; p < a.dp[row + 1]; p += blockDim.x) dv[a.di[p]] = a.dv[p];
    }
    const int len = a.ap[row + 1] - a.ap[row];
    const int per = (len + SK_W - 1) / SK_W;
    double *acc = accs + (size_t)w * ncols;
    unsigned char *hw = has + (size_t)w * ncols;
    accumulate_row<PFD>(a, row, lane, [&](int j, double pr) {
        if (hw[j]) acc[j] = __dadd_rn(acc[j], pr);
        else { acc[j] = __dadd_rn(0.0, pr); hw[j] = 1; }
    }, w * per, min(len, (w + 1) * per));
    __syncthreads();
    const int64_t o = a.toff[row];
    int base = 0;
    for (int j0 = 0; j0 < ncols; j0 += blockDim.x) {
        const int j = j0 + threadIdx.x;
        bool keep = false, any = false;
        double v = 0.0;
        if (j < ncols) {
            for (int q = 0; q < SK_W; ++q)
                if (has[(size_t)q * ncols + j]) {
                    v = any ? __dadd_rn(v, accs[(size_t)q * ncols + j]) : accs[(size_t)q * ncols + j];
                    any = true;
                }
            bool hd = false;
            if (a.dp) {   // D present at j?  (dv was only written where D has entries)
                const int p0 = a.dp[row], p1 = a.dp[row + 1];
                int lo = p0, hi = p1;
                while (lo < hi) { const int m = (lo + hi) >> 1; if (a.di[m] < j) lo = m + 1; else hi = m; }
                hd = lo < p1 && a.di[lo] == j;
            }
            if (any || hd) {
                if (!a.dp) v = v;
                else if (any) v = hd ? __dsub_rn(dv[j], v) : -v;
                else v = dv[j];
                keep = a.keep_zeros || v != 0.0;
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) wsum[w] = __popc(m);
        __syncthreads();
        int before = 0, tot = 0;
        for (int q = 0; q < SK_W; ++q) { before += q < w ? wsum[q] : 0; tot += wsum[q]; }
        if (keep) {
            const int64_t pos = o + base + before + __popc(m & ((1u << lane) - 1));
            a.ti[pos] = j;
            a.tv[pos] = v;
        }
        base += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) a.cnt[row] = base;
}

__global__ void k_toff_dense(int rows, int ncols, int64_t *toff) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x)
        toff[r] = (int64_t)r * ncols;
}

// scratch (row segments at toff, cnt entries) -> canonical CSR (warp per row)
__global__ void k_compact(int rows, const int64_t *toff, const int *ptr, const int *ti, const double *tv, int *oi,
                          double *ov) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t s = toff[r];
        const int o = ptr[r], n = ptr[r + 1] - o;
        for (int q = lane; q < n; q += 32) {
            oi[o + q] = ti[s + q];
            ov[o + q] = tv[s + q];
        }
    }
}

template <int CAP, int W, int K, bool HD, int PF>
void launch_num_pf(Ctx *c, const Args &a, int nrl) {
    const size_t smem = (size_t)CAP * slot_bytes(HD) * W;
    static bool attr = false;
    if (!attr && smem > 48 * 1024) {
        CK(cudaFuncSetAttribute(k_spgemm_num<CAP, W, K, HD, PF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
        attr = true;
    }
    const int grid = std::max(1, std::min<int>((nrl + W - 1) / W, c->sms * 32));
    k_spgemm_num<CAP, W, K, HD, PF><<<grid, 32 * W, smem, c->s>>>(a);
    launched(c);
}
// B rows held in registers PF x 32 entries at a time: short B rows (the velocity /
// pressure couplings, P) take one slot, so the per-k loop carries no idle slots
template <int CAP, int W, int K, bool HD>
void launch_num_t(Ctx *c, const Args &a, int nrl) {
    if (a.bmax <= 32) launch_num_pf<CAP, W, K, HD, 1>(c, a, nrl);
    else if (a.bmax <= 64) launch_num_pf<CAP, W, K, HD, 2>(c, a, nrl);
    else launch_num_pf<CAP, W, K, HD, PF_HASH>(c, a, nrl);
}
__global__ void k_count_neg(int rows, const int *cnt, int *out) {
    int z = 0;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) z += cnt[r] < 0;
    z = __reduce_add_sync(0xffffffffu, z);
    if ((threadIdx.x & 31) == 0 && z) atomicAdd(out, z);
}
__global__ void k_stride_off(int rows, int stride, int64_t *toff) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x)
        toff[r] = (int64_t)r * stride;
}
template <bool HD, int PF>
void launch_trial_pf(Ctx *c, const Args &a) {
    constexpr int CAP = 256, W = 8, K = 4;
    const size_t smem = (size_t)CAP * slot_bytes(HD) * W;
    const int grid = std::max(1, std::min<int>((a.nrl + W - 1) / W, c->sms * 32));
    k_spgemm_num<CAP, W, K, HD, PF, true><<<grid, 32 * W, smem, c->s>>>(a);
    launched(c);
}
template <bool HD>
void launch_trial(Ctx *c, const Args &a) {
    if (a.bmax <= 32) launch_trial_pf<HD, 1>(c, a);
    else if (a.bmax <= 64) launch_trial_pf<HD, 2>(c, a);
    else launch_trial_pf<HD, PF_HASH>(c, a);
}
__global__ void k_row_max(int rows, const int *ptr, int *out) {
    int m = 0;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x)
        m = max(m, ptr[r + 1] - ptr[r]);
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}
template <int CAP, int W, int K>
void launch_num_dev(Ctx *c, Args a, const int *rl, int nrl) {
    if (nrl <= 0) return;
    a.rl = rl;
    a.nrl = nrl;
    if (a.dp) launch_num_t<CAP, W, K, true>(c, a, a.nrl);
    else launch_num_t<CAP, W, K, false>(c, a, a.nrl);
}

// rows -> size-class lists (order inside a list is irrelevant: every row writes only
// its own scratch range), class counts in meta[0..2], overflow rows counted in meta[3]
__global__ void k_sp_classify(int rows, const int *u, int *lists, int *meta) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
        const int v = u[r];
        if (v < 0) { atomicAdd(&meta[3], 1); continue; }
        const int64_t need = 2 * (int64_t)v + 2;
        const int cls = need <= 256 ? 0 : need <= 1024 ? 1 : need <= 4096 ? 2 : 3;
        if (cls == 3) { atomicAdd(&meta[3], 1); continue; }
        lists[(size_t)cls * rows + atomicAdd(&meta[cls], 1)] = r;
    }
}
__global__ void k_sp_widen(const int *u, int64_t *o, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x)
        o[i] = i < n ? max(u[i], 0) : 0;
}

template <int CAP, int W, int K>
void launch_num(Ctx *c, Args a, const std::vector<int> &rows_h) {
    if (rows_h.empty()) return;
    DBuf<int> rl(rows_h.size(), c->s);
    rl.upload(rows_h.data(), rows_h.size());
    a.rl = rl.p;
    a.nrl = (int)rows_h.size();
    if (a.dp) launch_num_t<CAP, W, K, true>(c, a, a.nrl);
    else launch_num_t<CAP, W, K, false>(c, a, a.nrl);
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
    DBuf<int64_t> toff(rows, c->s);
    DBuf<int> ti;
    DBuf<double> tv;

    // small column space and dense-ish rows: dense accumulator, no hashing / sorting
    const int ncols = B.cols;
    const size_t per = (size_t)ncols * 16 + (size_t)((ncols + 15) & ~15);
    const double avg_out = std::min<double>(ncols, (double)A.nnz / rows * ((double)B.nnz / std::max(1, B.rows)));
    if (ncols <= 4096 && avg_out * 8 >= ncols && per <= 200 * 1024 && (int64_t)rows * ncols <= (int64_t)1 << 24) {
        const int W = (int)std::max<size_t>(1, std::min<size_t>(8, (200 * 1024) / per));
        static bool dattr = false;
        if (!dattr) {
            for (const void *f : {(const void *)k_spgemm_dense<4>, (const void *)k_spgemm_dense<8>,
                                  (const void *)k_spgemm_dense<16>})
                CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            dattr = true;
        }
        // B rows held in registers (and prefetched one k ahead): sized to ~1.5x the mean
        // B row so long coarse rows do not fall back to unprefetched batches
        const double bavg = (double)B.nnz / std::max(1, B.rows);
        const int pfd = bavg * 1.5 > 256 ? 16 : bavg * 1.5 > 128 ? 8 : 4;
        ti.alloc((size_t)rows * ncols, c->s);
        tv.alloc((size_t)rows * ncols, c->s);
        a.ti = ti.p;
        a.tv = tv.p;
        k_toff_dense<<<grid_for(rows, 256, c->sms), 256, 0, c->s>>>(rows, ncols, toff.p);
        launched(c);
        a.toff = toff.p;
        const int grid = std::max(1, std::min<int>((rows + W - 1) / W, c->sms * 4));
        const size_t sk_smem = (size_t)SK_W * ncols * 9 + (size_t)ncols * 8;
        const double alen = (double)A.nnz / rows;
        static const bool no_sk = [] { const char *e = std::getenv("DPP_NO_SPLITK"); return e && *e == '1'; }();
        if (!no_sk && rows < c->sms * 8 && alen >= 64 && sk_smem <= 200 * 1024) {
            static bool sattr = false;
            if (!sattr) {
                for (const void *f : {(const void *)k_spgemm_dense_splitk<4>, (const void *)k_spgemm_dense_splitk<8>,
                                      (const void *)k_spgemm_dense_splitk<16>})
                    CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
                sattr = true;
            }
            if (pfd == 16) k_spgemm_dense_splitk<16><<<rows, 32 * SK_W, sk_smem, c->s>>>(a, ncols);
            else if (pfd == 8) k_spgemm_dense_splitk<8><<<rows, 32 * SK_W, sk_smem, c->s>>>(a, ncols);
            else k_spgemm_dense_splitk<4><<<rows, 32 * SK_W, sk_smem, c->s>>>(a, ncols);
        } else if (pfd == 16) k_spgemm_dense<16><<<grid, 32 * W, per * W, c->s>>>(a, ncols, W);
        else if (pfd == 8) k_spgemm_dense<8><<<grid, 32 * W, per * W, c->s>>>(a, ncols, W);
        else k_spgemm_dense<4><<<grid, 32 * W, per * W, c->s>>>(a, ncols, W);
        launched(c);
    } else {
        // 0. trial pass for products whose rows are expected to be narrow: one numeric
        // pass without the symbolic pass; used only when no row went over budget
        static const bool no_trial = [] { const char *e = std::getenv("DPP_SPGEMM_NO_TRIAL"); return e && *e == '1'; }();
        const double prod = (double)A.nnz / rows * ((double)B.nnz / std::max(1, B.rows)) +
                            (D ? (double)D->nnz / rows : 0.0);
        static const double trial_max = [] { const char *e = std::getenv("DPP_SPGEMM_TRIAL_MAX"); return e ? std::atof(e) : 1024.0; }();
        if (!no_trial && rows >= 256 && prod <= trial_max) {
            DPP_TRACE_SCOPE(c, "spgemm.trial");
            DBuf<int> meta(2, c->s);
            CK(cudaMemsetAsync(meta.p, 0, 2 * sizeof(int), c->s));
            k_row_max<<<grid_for(B.rows, 256, c->sms, 4), 256, 0, c->s>>>(B.rows, B.ptr.p, meta.p + 1);
            launched(c);
            int hb[2] = {0, 0};
            CK(cudaMemcpyAsync(hb, meta.p, sizeof(hb), cudaMemcpyDeviceToHost, c->s));
            CK(cudaStreamSynchronize(c->s));
            a.bmax = hb[1];
            ti.alloc((size_t)rows * TR_LIM, c->s);
            tv.alloc((size_t)rows * TR_LIM, c->s);
            a.ti = ti.p;
            a.tv = tv.p;
            a.nrl = rows;
            if (D) launch_trial<true>(c, a);
            else launch_trial<false>(c, a);
            k_count_neg<<<grid_for(rows, 256, c->sms, 4), 256, 0, c->s>>>(rows, cnt.p, meta.p);
            launched(c);
            int nover = 0;
            CK(cudaMemcpyAsync(&nover, meta.p, sizeof(int), cudaMemcpyDeviceToHost, c->s));
            CK(cudaStreamSynchronize(c->s));
            if (nover == 0) {
                C.nnz = counts_to_ptr(c, cnt.p, rows, C.ptr);
                C.idx.alloc(std::max<int64_t>(C.nnz, 1), c->s);
                C.val.alloc(std::max<int64_t>(C.nnz, 1), c->s);
                k_stride_off<<<grid_for(rows, 256, c->sms, 4), 256, 0, c->s>>>(rows, TR_LIM, toff.p);
                launched(c);
                k_compact<<<grid_for((int64_t)rows * 32, 256, c->sms, 8), 256, 0, c->s>>>(rows, toff.p, C.ptr.p, ti.p,
                                                                                        tv.p, C.idx.p, C.val.p);
                launched(c);
                CK(cudaStreamSynchronize(c->s));
                return C;
            }
            ti.release();
            tv.release();
        }
        // 1. symbolic: distinct columns per row
        std::vector<int> u;
        DBuf<int> duniq(rows, c->s);
        k_unique_s<<<std::max(1, std::min<int>((rows + US_W - 1) / US_W, c->sms * 7)), 32 * US_W, 0, c->s>>>(
            rows, A.ptr.p, A.idx.p, B.ptr.p, B.idx.p, D ? D->ptr.p : nullptr, D ? D->idx.p : nullptr, duniq.p);
        launched(c);
        // common case (no row beyond the small symbolic table): scratch offsets and
        // size-class row lists are built on the device, one small read back
        DBuf<int> meta(5, c->s), lists((size_t)3 * rows, c->s);
        DBuf<int64_t> toff64((size_t)rows + 1, c->s), uw((size_t)rows + 1, c->s);
        int hm[5] = {0, 0, 0, 0, 0};
        int64_t ttot_d = 0;
        {
            DPP_TRACE_SCOPE(c, "spgemm.classify");
            CK(cudaMemsetAsync(meta.p, 0, 5 * sizeof(int), c->s));
            k_sp_classify<<<grid_for(rows, 256, c->sms, 4), 256, 0, c->s>>>(rows, duniq.p, lists.p, meta.p);
            launched(c);
            k_row_max<<<grid_for(B.rows, 256, c->sms, 4), 256, 0, c->s>>>(B.rows, B.ptr.p, meta.p + 4);
            launched(c);
            k_sp_widen<<<grid_for(rows + 1, 256, c->sms, 4), 256, 0, c->s>>>(duniq.p, uw.p, rows);
            launched(c);
            size_t tb = 0;
            CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, uw.p, toff64.p, rows + 1, c->s));
            DBuf<char> t(tb, c->s);
            CK(cub::DeviceScan::ExclusiveSum(t.p, tb, uw.p, toff64.p, rows + 1, c->s));
            launched(c);
            CK(cudaMemcpyAsync(hm, meta.p, sizeof(hm), cudaMemcpyDeviceToHost, c->s));
            CK(cudaMemcpyAsync(&ttot_d, toff64.p + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, c->s));
            CK(cudaStreamSynchronize(c->s));
        }
        static const bool host_lists = [] { const char *e = std::getenv("DPP_SPGEMM_HOSTLIST"); return e && *e == '1'; }();
        a.bmax = hm[4];
        if (hm[3] == 0 && !host_lists) {
            a.toff = toff64.p;
            ti.alloc(std::max<int64_t>(ttot_d, 1), c->s);
            tv.alloc(std::max<int64_t>(ttot_d, 1), c->s);
            a.ti = ti.p;
            a.tv = tv.p;
            if (TraceScope::on())
                std::fprintf(stderr, "[dpp-trace]   spgemm %d x %d (A nnz %lld, B nnz %lld): rows S %d M %d L %d (device lists)\n",
                             rows, B.cols, (long long)A.nnz, (long long)B.nnz, hm[0], hm[1], hm[2]);
            DPP_TRACE_SCOPE(c, "spgemm.numeric");
            launch_num_dev<256, 8, 4>(c, a, lists.p, hm[0]);
            launch_num_dev<1024, 4, 16>(c, a, lists.p + rows, hm[1]);
            launch_num_dev<4096, 2, 0>(c, a, lists.p + 2 * (size_t)rows, hm[2]);
            C.nnz = counts_to_ptr(c, cnt.p, rows, C.ptr);
            if (C.nnz == ttot_d) {   // no exact-zero sums: the scratch is the result
                C.idx = std::move(ti);
                C.val = std::move(tv);
            } else {
                C.idx.alloc(std::max<int64_t>(C.nnz, 1), c->s);
                C.val.alloc(std::max<int64_t>(C.nnz, 1), c->s);
                k_compact<<<grid_for((int64_t)rows * 32, 256, c->sms, 8), 256, 0, c->s>>>(
                    rows, toff64.p, C.ptr.p, ti.p, tv.p, C.idx.p, C.val.p);
                launched(c);
            }
            CK(cudaStreamSynchronize(c->s));
            return C;
        }
        u.resize(rows);
        {
            DPP_TRACE_SCOPE(c, "spgemm.unique");
            duniq.download(u.data(), rows);
            CK(cudaStreamSynchronize(c->s));
            std::vector<int> over;
            for (int r = 0; r < rows; ++r)
                if (u[r] < 0) over.push_back(r);
            if (!over.empty()) {
                const int no = (int)over.size();
                DBuf<int> drl(no, c->s);
                drl.upload(over.data(), no);
                DBuf<int64_t> need(no, c->s);
                k_bound_list<<<grid_for(no, 256, c->sms), 256, 0, c->s>>>(drl.p, no, A.ptr.p, A.idx.p, B.ptr.p,
                                                                          D ? D->ptr.p : nullptr, B.cols, need.p);
                launched(c);
                std::vector<int64_t> h = need.to_host();
                std::vector<int64_t> uoff(no, -1);
                std::vector<int> ucap(no, 0);
                int64_t utot = 0;
                for (int i = 0; i < no; ++i) {
                    if (h[i] < UCAP - 1) continue;
                    int cap = 64;
                    while (cap < 2 * h[i] + 2) cap <<= 1;
                    uoff[i] = utot;
                    ucap[i] = cap;
                    utot += cap;
                }
                DBuf<int64_t> duoff(no, c->s);
                DBuf<int> ducap(no, c->s), dkey(std::max<int64_t>(utot, 1), c->s);
                duoff.upload(uoff.data(), no);
                ducap.upload(ucap.data(), no);
                k_unique_l<<<std::min(no, c->sms * 6), 32, 0, c->s>>>(drl.p, no, A.ptr.p, A.idx.p, B.ptr.p, B.idx.p,
                                                                    D ? D->ptr.p : nullptr, D ? D->idx.p : nullptr,
                                                                    duoff.p, ducap.p, dkey.p, duniq.p);
                launched(c);
                duniq.download(u.data(), rows);
                CK(cudaStreamSynchronize(c->s));
            }
        }
        // 2. scratch offsets and size classes
        std::vector<int64_t> to(rows);
        int64_t ttot = 0;
        std::vector<int> rs_s, rs_m, rs_l, rs_g;
        std::vector<int64_t> goff;
        std::vector<int> gcap;
        int64_t gtot = 0;
        for (int r = 0; r < rows; ++r) {
            to[r] = ttot;
            ttot += u[r];
            const int64_t need = 2 * (int64_t)u[r] + 2;
            if (need <= 256) rs_s.push_back(r);
            else if (need <= 1024) rs_m.push_back(r);
            else if (need <= 4096) rs_l.push_back(r);
            else {
                int cap = 64;
                while (cap < need) cap <<= 1;
                rs_g.push_back(r);
                goff.push_back(gtot);
                gcap.push_back(cap);
                gtot += cap;
            }
        }
        toff.upload(to.data(), rows);
        a.toff = toff.p;
        ti.alloc(std::max<int64_t>(ttot, 1), c->s);
        tv.alloc(std::max<int64_t>(ttot, 1), c->s);
        a.ti = ti.p;
        a.tv = tv.p;
        if (TraceScope::on())
            std::fprintf(stderr, "[dpp-trace]   spgemm %d x %d (A nnz %lld, B nnz %lld): rows S %zu M %zu L %zu G %zu\n",
                         rows, B.cols, (long long)A.nnz, (long long)B.nnz, rs_s.size(), rs_m.size(), rs_l.size(),
                         rs_g.size());
        // 3. numeric, one pass per class
        DPP_TRACE_SCOPE(c, "spgemm.numeric");
        launch_num<256, 8, 4>(c, a, rs_s);
        launch_num<1024, 4, 16>(c, a, rs_m);
        launch_num<4096, 2, 0>(c, a, rs_l);
        if (!rs_g.empty()) {
            const int ng = (int)rs_g.size();
            DBuf<int64_t> dgoff(ng, c->s);
            DBuf<int> dgcap(ng, c->s);
            dgoff.upload(goff.data(), ng);
            dgcap.upload(gcap.data(), ng);
            DBuf<int> gk(gtot, c->s);
            DBuf<unsigned char> ghas(gtot, c->s);
            DBuf<double> gx(gtot, c->s), gd(gtot, c->s);
            Args g = a;
            g.goff = dgoff.p; g.gcap = dgcap.p;
            g.g_key = gk.p; g.g_has = ghas.p; g.g_x = gx.p; g.g_d = gd.p;
            launch_num<0, 1, 0>(c, g, rs_g);
            CK(cudaStreamSynchronize(c->s));   // global tables go out of scope
        }
    }
    // 4. compaction into canonical CSR
    C.nnz = counts_to_ptr(c, cnt.p, rows, C.ptr);
    C.idx.alloc(std::max<int64_t>(C.nnz, 1), c->s);
    C.val.alloc(std::max<int64_t>(C.nnz, 1), c->s);
    k_compact<<<grid_for((int64_t)rows * 32, 256, c->sms, 8), 256, 0, c->s>>>(rows, toff.p, C.ptr.p, ti.p, tv.p,
                                                                            C.idx.p, C.val.p);
    launched(c);
    CK(cudaStreamSynchronize(c->s));   // host vectors / scratch go out of scope
    return C;
}

}  // namespace dpp
