// Block-dense triangular sweep for AMG smoother factors (the Gauss-Seidel
// triangles of linalg.amg_vcycle, linalg.py:372-400).
//
// The level-scheduled sweep of a smoother triangle costs one cluster barrier
// plus a DSMEM round trip per dependency level (281 levels on the finest C2
// level, 691 on the next).  Here the rows are cut into consecutive blocks of B
// rows and the diagonal block inverses are formed once at setup, so a sweep is
// nb = ceil(n / B) dependent steps instead of nlev levels:
//
//     y     = b_blk - T[blk, outside] x     (off-block entries: rows already solved)
//     x_blk = inv(T[blk, blk]) y           (dense triangular GEMV)
//
// In exact arithmetic this is the same forward/backward substitution; the
// rounding is that of a dense inverse (as the small-level dense path,
// DENSE_TRI_MAX), which keeps V-cycle results within the parity tolerance.
//
// One thread-block cluster of C CTAs runs the whole sweep.  Block rows are dealt
// to the CTAs cyclically (row a -> CTA a % C, balancing the triangle), and
// everything a CTA needs for one step that does not depend on x -- its rows of
// the block inverse (packed triangle) and its off-block CSR rows -- is packed at
// setup into one contiguous segment per (block, CTA).  A TMA bulk-copy ring
// stages the segments NST-1 steps ahead, so the step's critical path is only
// the x gather (L2), one DSMEM exchange of y and two cluster barriers.
#include <cooperative_groups.h>

#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>

#include "dpp_internal.cuh"

namespace cg = cooperative_groups;

namespace dpp {

constexpr int BD_THREADS = 1024;
constexpr int BD_INV_WPB = 4;
constexpr int BD_NST_MAX = 8;
constexpr size_t BD_SMEM_LIMIT = 227 * 1024;

__host__ __device__ __forceinline__ long long bd_pad16(long long b) { return (b + 15) & ~15LL; }

__device__ __forceinline__ unsigned bd_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bd_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void bd_mbar_wait(unsigned long long *m, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(bd_u32(m)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bd_issue(unsigned char *dst, const unsigned char *src, unsigned bytes,
                                         unsigned long long *m) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bd_u32(m)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(bd_u32(dst)), "l"(src), "r"(bytes), "r"(bd_u32(m)) : "memory");
}

// ---------------------------------------------------------------- segment layout
// segment (blk, k), rows i = 0..nr-1 with block-local row a = k + C i:
//   int nr, int ne, int 0, int 0
//   int dofs[nr + 1]      packed-triangle row offsets (doubles)
//   int optr[nr + 1]      off-block CSR row pointers (local)
//   int oidx[ne]          global columns
//   (pad 16) double dinv[dofs[nr]]   row i = inv(T_blk)[a, j0:j1)
//   (pad 16) double oval[ne]
struct SegDims {
    int nr, nd, ne;
};
__host__ __device__ inline long long seg_bytes(int nr, long long nd, long long ne) {
    const long long ints = 16 + 4LL * (nr + 1) * 2 + 4LL * ne;
    return bd_pad16(bd_pad16(ints) + 8 * nd + 8 * ne);
}
__device__ __forceinline__ int row_len(int a, int m, int backward) { return backward ? m - a : a + 1; }

// warp per segment: lanes take the segment's rows
__global__ void k_bd_seg_size(int n, int B, int C, int nb, int backward, const int *__restrict__ ptr,
                              const int *__restrict__ idx, long long *bytes, int *maxback) {
    const int lane = threadIdx.x & 31;
    const int seg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (seg >= nb * C) return;
    const int blk = seg / C, k = seg % C, s = blk * B, m = min(B, n - s);
    long long nr = 0, nd = 0, ne = 0;
    int mb = 0;
    for (int a = k + C * lane; a < m; a += 32 * C) {
        ++nr;
        nd += row_len(a, m, backward);
        const int r = s + a;
        for (int p = ptr[r]; p < ptr[r + 1]; ++p) {
            const int bc = idx[p] / B;
            if (bc == blk) continue;
            ++ne;
            mb = max(mb, backward ? bc - blk : blk - bc);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        nr += __shfl_xor_sync(0xffffffffu, nr, o);
        nd += __shfl_xor_sync(0xffffffffu, nd, o);
        ne += __shfl_xor_sync(0xffffffffu, ne, o);
        mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, o));
    }
    if (lane == 0) {
        if (mb) atomicMax(maxback, mb);
        bytes[seg] = seg_bytes((int)nr, nd, ne);
    }
}

// one CTA per segment: dense block inverse rows + off-block CSR rows -> segment
// (row offsets from per-row counts; off-block entries keep their CSR order)
constexpr int BD_SEG_ROWS = 1024;
__global__ void k_bd_seg_fill(int n, int B, int C, int W, int backward, const int *__restrict__ ptr,
                              const int *__restrict__ idx, const double *__restrict__ val,
                              const double *__restrict__ dense, const long long *__restrict__ soff,
                              unsigned char *segs) {
    __shared__ int roff_d[BD_SEG_ROWS + 1], roff_e[BD_SEG_ROWS + 1];
    const int seg = blockIdx.x, blk = seg / C, k = seg % C, s = blk * B, m = min(B, n - s);
    unsigned char *S = segs + soff[seg];
    const int nr = m > k ? (m - k + C - 1) / C : 0;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    // per-row lengths
    for (int i = w; i < nr; i += nw) {
        const int a = k + C * i, r = s + a;
        int e = 0;
        for (int p = ptr[r] + lane; p < ptr[r + 1]; p += 32) e += (idx[p] / B) != blk;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
        if (lane == 0) { roff_d[i + 1] = row_len(a, m, backward); roff_e[i + 1] = e; }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        roff_d[0] = roff_e[0] = 0;
        for (int i = 0; i < nr; ++i) { roff_d[i + 1] += roff_d[i]; roff_e[i + 1] += roff_e[i]; }
    }
    __syncthreads();
    const int ne = roff_e[nr], nd = roff_d[nr];
    int *hdr = reinterpret_cast<int *>(S);
    int *dofs = hdr + 4;
    int *optr = dofs + nr + 1;
    int *oidx = optr + nr + 1;
    double *dv = reinterpret_cast<double *>(S + bd_pad16(16 + 4LL * (nr + 1) * 2 + 4LL * ne));
    double *ov = dv + nd;
    if (threadIdx.x == 0) { hdr[0] = nr; hdr[1] = ne; hdr[2] = 0; hdr[3] = 0; }
    for (int i = threadIdx.x; i <= nr; i += blockDim.x) { dofs[i] = roff_d[i]; optr[i] = roff_e[i]; }
    const double *Db = dense + (size_t)blk * B * B;
    for (int i = w; i < nr; i += nw) {
        const int a = k + C * i, r = s + a;
        const int j0 = backward ? a : 0, len = row_len(a, m, backward);
        for (int q = lane; q < len; q += 32) dv[roff_d[i] + q] = Db[(size_t)a * B + j0 + q];
        int o = roff_e[i];
        for (int p0 = ptr[r]; p0 < ptr[r + 1]; p0 += 32) {
            const int p = p0 + lane;
            const bool in = p < ptr[r + 1];
            const int j = in ? idx[p] : 0;
            const int bc = j / B;
            const bool keep = in && bc != blk;
            const unsigned msk = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const int q = o + __popc(msk & ((1u << lane) - 1));
                // every off-block column lies in the x window (W >= the largest block distance)
                oidx[q] = (bc % W) * B + (j - bc * B);
                ov[q] = val[p];
            }
            o += __popc(msk);
        }
    }
}

// Column c of inv(T[blk, blk]) by substitution over the strict CSR rows of the
// block (one warp per column, the column in shared memory); dense[blk] is B x B
// row-major with the block's rows/columns local.
__global__ void __launch_bounds__(32 * BD_INV_WPB)
    k_bd_inverse(int n, int B, int backward, const int *__restrict__ ptr, const int *__restrict__ idx,
                 const double *__restrict__ val, const double *__restrict__ diag, double *__restrict__ dense) {
    extern __shared__ double colbuf[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *xc = colbuf + (size_t)w * B;
    const int blk = blockIdx.y, s = blk * B, m = min(B, n - s);
    const int c = blockIdx.x * BD_INV_WPB + w;
    if (c >= m) return;
    for (int i = lane; i < m; i += 32) xc[i] = 0.0;
    __syncwarp();
    // forward: rows c, c+1, ..., m-1 ; backward: rows c, c-1, ..., 0.  Software
    // pipelined: row bounds two rows ahead, the first 32 entries and the diagonal
    // of the next row one row ahead, so a row costs shared-memory latency only.
    const int step = backward ? -1 : 1;
    auto valid = [&](int aa) { return backward ? aa >= 0 : aa < m; };
    int a = c;
    int pa0 = ptr[s + a], pa1 = ptr[s + a + 1];
    int pb0 = 0, pb1 = 0;
    if (valid(a + step)) { pb0 = ptr[s + a + step]; pb1 = ptr[s + a + step + 1]; }
    constexpr int IPF = 8;   // entries per lane held for the current / next row (whole coarse rows)
    int jc[IPF];
    double vc[IPF], dc = diag ? diag[s + a] : 1.0;
#pragma unroll
    for (int u = 0; u < IPF; ++u) {
        const int p = pa0 + 32 * u + lane;
        jc[u] = p < pa1 ? idx[p] - s : -1;
        vc[u] = p < pa1 ? val[p] : 0.0;
    }
    while (true) {
        const int an = a + step;
        int jn[IPF], pc0 = 0, pc1 = 0;
        double vn[IPF], dn = 1.0;
        const bool nv = valid(an);
#pragma unroll
        for (int u = 0; u < IPF; ++u) {
            const int p = pb0 + 32 * u + lane;
            jn[u] = nv && p < pb1 ? idx[p] - s : -1;
            vn[u] = nv && p < pb1 ? val[p] : 0.0;
        }
        if (nv) {
            if (diag) dn = diag[s + an];
            if (valid(an + step)) { pc0 = ptr[s + an + step]; pc1 = ptr[s + an + step + 1]; }
        }
        double acc = 0.0;
#pragma unroll
        for (int u = 0; u < IPF; ++u)
            if (jc[u] >= 0 && jc[u] < m) acc += vc[u] * xc[jc[u]];
        for (int p = pa0 + 32 * IPF + lane; p < pa1; p += 32) {
            const int j = idx[p] - s;
            if (j >= 0 && j < m) acc += val[p] * xc[j];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) xc[a] = ((a == c ? 1.0 : 0.0) - acc) / dc;
        __syncwarp();
        if (!nv) break;
        a = an;
        pa0 = pb0; pa1 = pb1; pb0 = pc0; pb1 = pc1;
#pragma unroll
        for (int u = 0; u < IPF; ++u) { jc[u] = jn[u]; vc[u] = vn[u]; }
        dc = dn;
    }
    double *D = dense + (size_t)blk * B * B;
    for (int i = lane; i < m; i += 32) D[(size_t)i * B + c] = xc[i];
}

// Same inverse, G columns per CTA at once: X[rows][G] lives in shared memory and the
// block's rows are dealt to G-lane workers in substitution order; a worker waits (on a
// per-row flag in shared memory) only for the rows its row reads, so independent rows of
// the block proceed in parallel instead of one warp walking every row of one column.
// Forward: column group [c0, c0+G) is zero above row c0; backward: zero below c0+G-1.
// Entries of a row are loaded G at a time by the worker's lanes and only the in-window
// ones are broadcast (ballot).  Rows outside the window are written as zeros.
constexpr int BDI_THREADS = 512;
template <int G>
__global__ void __launch_bounds__(BDI_THREADS)
    k_bd_inv_tile(int n, int B, int backward, const int *__restrict__ ptr, const int *__restrict__ idx,
                  const double *__restrict__ val, const double *__restrict__ diag, double *__restrict__ dense) {
    extern __shared__ double X[];
    const int blk = blockIdx.y, s = blk * B, m = min(B, n - s);
    const int c0 = blockIdx.x * G;
    if (c0 >= m) return;
    int *done = reinterpret_cast<int *>(X + (size_t)m * G);
    const int lo = backward ? 0 : c0, hi = backward ? min(m, c0 + G) : m;
    for (int i = threadIdx.x; i < hi - lo; i += blockDim.x) done[lo + i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, q = lane % G, sub = lane / G;
    const int wk = threadIdx.x / G, nwk = blockDim.x / G;
    const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (sub * G));
    const unsigned done_base = (unsigned)__cvta_generic_to_shared(done);
    for (int t = wk; t < hi - lo; t += nwk) {
        const int a = backward ? hi - 1 - t : lo + t, r = s + a;
        const int pe = ptr[r + 1];
        double acc = 0.0;
        for (int p0 = ptr[r]; p0 < pe; p0 += G) {
            const int p = p0 + q;
            int j = -1;
            double v = 0.0;
            if (p < pe) {
                j = idx[p] - s;
                v = val[p];
            }
            const bool keep = j >= lo && j < hi;
            unsigned km = (__ballot_sync(gmask, keep) & gmask) >> (sub * G);
            while (km) {
                const int e = __ffs(km) - 1;
                km &= km - 1;
                const int jj = __shfl_sync(gmask, j, e, G);
                const double vv = __shfl_sync(gmask, v, e, G);
                int f;
                long long spins = 0;
                do {
                    asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(f) : "r"(done_base + 4u * jj) : "memory");
                    if (++spins > (1ll << 28)) __trap();
                } while (!f);
                acc += vv * X[(size_t)jj * G + q];
            }
        }
        const double d = diag ? diag[r] : 1.0;
        X[(size_t)a * G + q] = ((a == c0 + q ? 1.0 : 0.0) - acc) / d;
        __syncwarp(gmask);
        if (q == 0) asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(done_base + 4u * a), "r"(1) : "memory");
    }
    __syncthreads();
    const int ncol = min(G, m - c0);
    double *D = dense + (size_t)blk * B * B;
    for (int i = threadIdx.x; i < m * G; i += blockDim.x) {
        const int row = i / G, cc = i % G;
        if (cc < ncol) D[(size_t)row * B + c0 + cc] = row >= lo && row < hi ? X[(size_t)row * G + cc] : 0.0;
    }
}

// ---------------------------------------------------------------- blocked dense inversion
// inv(T[blk, blk]) by recursive doubling on the densified block (the default; the sparse
// substitutions above cost ~0.4-0.55 ms per triangle, a third of the setup's kernel time at C2):
//   32 x 32 diagonal sub-blocks by substitution (one warp each), then for s = 32, 64, ...
//   [[A, 0], [C, B]]^-1 = [[A^-1, 0], [-B^-1 C A^-1, B^-1]]   (upper: [[A, C], [0, B]] -> -A^-1 C B^-1)
// as two batched tile GEMMs per size over every pair of every block, in place (C is untouched
// until its own size comes up).  Exact-arithmetic equal to the substitution; DPP_BD_INV=sparse
// selects the old kernels.
__global__ void k_ti_densify(int n, int B, const int *__restrict__ ptr, const int *__restrict__ idx,
                             const double *__restrict__ val, const double *__restrict__ diag, double *D) {
    const int lane = threadIdx.x & 31;
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += (gridDim.x * blockDim.x) >> 5) {
        const int blk = r / B, a = r - blk * B;
        double *row = D + ((size_t)blk * B + a) * B;
        for (int p = ptr[r] + lane; p < ptr[r + 1]; p += 32) {
            const int j = idx[p];
            if (j / B == blk) row[j - blk * B] = val[p];
        }
        if (lane == 0) row[a] = diag ? diag[r] : 1.0;
    }
}
__global__ void __launch_bounds__(32) k_ti_inv32(int n, int B, int backward, double *D) {
    __shared__ double Ts[32][33], Xs[32][33];
    const int blk = blockIdx.y, m = min(B, n - blk * B), r0 = blockIdx.x * 32;
    if (r0 >= m) return;
    const int sz = min(32, m - r0), c = threadIdx.x;
    double *Db = D + (size_t)blk * B * B + (size_t)r0 * B + r0;
    for (int i = 0; i < sz; ++i) Ts[i][c] = c < sz ? Db[(size_t)i * B + c] : 0.0;
    __syncwarp();
    if (c < sz) {
        if (!backward) {
            Xs[c][c] = 1.0 / Ts[c][c];
            for (int i = c + 1; i < sz; ++i) {
                double acc = 0.0;
                for (int j = c; j < i; ++j) acc += Ts[i][j] * Xs[j][c];
                Xs[i][c] = -acc / Ts[i][i];
            }
        } else {
            Xs[c][c] = 1.0 / Ts[c][c];
            for (int i = c - 1; i >= 0; --i) {
                double acc = 0.0;
                for (int j = i + 1; j <= c; ++j) acc += Ts[i][j] * Xs[j][c];
                Xs[i][c] = -acc / Ts[i][i];
            }
        }
    }
    __syncwarp();
    for (int i = 0; i < sz; ++i)
        if (c < sz) {
            const bool in = backward ? i <= c : i >= c;
            Db[(size_t)i * B + c] = in ? Xs[i][c] : 0.0;
        }
}
// one 64 x 64 output tile of out = alpha X Y for pair blockIdx.z of size s (phase 0: W = C A or C B,
// phase 1: C = -B W or -A W)
constexpr int TI_T = 64, TI_K = 16;
__global__ void __launch_bounds__(256) k_ti_gemm(int n, int B, int s, int phase, int backward, double *D, double *Wb) {
    __shared__ double Xs[TI_K][TI_T + 1], Ys[TI_K][TI_T];
    const int npairs = (B + 2 * s - 1) / (2 * s);
    const int blk = blockIdx.z / npairs, pr = blockIdx.z % npairs;
    const int m = min(B, n - blk * B), r0 = pr * 2 * s;
    const int s2 = min(s, m - r0 - s);
    if (s2 <= 0) return;
    double *Db = D + (size_t)blk * B * B;
    double *W = Wb + (size_t)blockIdx.z * s * s;
    double *Ab = Db + (size_t)r0 * B + r0, *Bb = Db + (size_t)(r0 + s) * B + r0 + s;
    double *Cb = backward ? Db + (size_t)r0 * B + r0 + s : Db + (size_t)(r0 + s) * B + r0;
    // out (on x om, ldo) = alpha X (on x ok, ldx) Y (ok x om, ldy)
    const double *X, *Y;
    double *O;
    int on, om, ok, ldx, ldy, ldo;
    double alpha;
    if (!backward) {
        on = s2; om = s;
        if (phase == 0) { X = Cb; ldx = B; Y = Ab; ldy = B; ok = s; O = W; ldo = s; alpha = 1.0; }
        else { X = Bb; ldx = B; Y = W; ldy = s; ok = s2; O = Cb; ldo = B; alpha = -1.0; }
    } else {
        on = s; om = s2;
        if (phase == 0) { X = Cb; ldx = B; Y = Bb; ldy = B; ok = s2; O = W; ldo = s; alpha = 1.0; }
        else { X = Ab; ldx = B; Y = W; ldy = s; ok = s; O = Cb; ldo = B; alpha = -1.0; }
    }
    const int bi = blockIdx.y * TI_T, bj = blockIdx.x * TI_T;
    if (bi >= on || bj >= om) return;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int k0 = 0; k0 < ok; k0 += TI_K) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = threadIdx.x + 256 * q;
            const int ar = e >> 4, ak = e & 15;
            Xs[ak][ar] = (bi + ar < on && k0 + ak < ok) ? X[(size_t)(bi + ar) * ldx + k0 + ak] : 0.0;
            const int bk = e >> 6, bc = e & 63;
            Ys[bk][bc] = (k0 + bk < ok && bj + bc < om) ? Y[(size_t)(k0 + bk) * ldy + bj + bc] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < TI_K; ++kk) {
            double av[4], bv[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) av[a] = Xs[kk][ty + 16 * a];
#pragma unroll
            for (int b = 0; b < 4; ++b) bv[b] = Ys[kk][tx + 16 * b];
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
        if (i >= on) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int j = bj + tx + 16 * b;
            if (j < om) O[(size_t)i * ldo + j] = alpha * acc[a][b];
        }
    }
}
// dense = inv of every diagonal block (nb blocks of B x B, row-major, zero outside the triangle)
static bool bd_inverse_gemm(Ctx *c, int n, int B, int nb, const Tri &T, double *dense) {
    static const bool off = [] { const char *e = std::getenv("DPP_BD_INV"); return e && !std::strcmp(e, "sparse"); }();
    if (off || T.ncomp != 1) return false;
    const int mmax = std::min(B, n);
    CK(cudaMemsetAsync(dense, 0, sizeof(double) * (size_t)nb * B * B, c->s));
    k_ti_densify<<<grid_for((int64_t)n * 32, 256, c->sms, 8), 256, 0, c->s>>>(n, B, T.strict.ptr.p, T.strict.idx.p,
                                                                            T.strict.val.p, T.diag.n ? T.diag.p : nullptr,
                                                                            dense);
    launched(c);
    k_ti_inv32<<<dim3((mmax + 31) / 32, nb), 32, 0, c->s>>>(n, B, (int)T.backward, dense);
    launched(c);
    if (mmax > 32) {
        size_t wmax = 0;
        for (int s = 32; s < mmax; s *= 2) wmax = std::max(wmax, (size_t)nb * ((B + 2 * s - 1) / (2 * s)) * s * s);
        DBuf<double> W(wmax, c->s);
        for (int s = 32; s < mmax; s *= 2) {
            const int npairs = (B + 2 * s - 1) / (2 * s), tiles = (s + TI_T - 1) / TI_T;
            for (int phase = 0; phase < 2; ++phase) {
                k_ti_gemm<<<dim3(tiles, tiles, nb * npairs), 256, 0, c->s>>>(n, B, s, phase, (int)T.backward, dense, W.p);
                launched(c);
            }
        }
        CK(cudaStreamSynchronize(c->s));   // W is freed on return
    }
    return true;
}

// G for an m-row block: the X tile plus flags within 200 KB
static int bd_inv_g(int m) {
    for (int g : {32, 16, 8, 4})
        if ((size_t)m * (8 * g + 4) <= 200 * 1024) return g;
    return 0;
}
static bool bd_inverse_tiles(Ctx *c, int n, int B, int nb, const Tri &T, double *dense) {
    // opt-in (DPP_BD_INV_TILE=1, read per call): measured slower than the column-per-warp
    // kernel on C2 (setup 24.9 vs 18.4 ms median): a row's entries stream in G-wide chunks
    // behind its dependency waits, so each row costs several L2 round trips on the chain
    const char *oe = std::getenv("DPP_BD_INV_TILE");
    const bool old = !(oe && *oe == '1');
    const int m = std::min(B, n);
    const int G = old ? 0 : bd_inv_g(m);
    if (!G) return false;
    const size_t sm = (size_t)m * (8 * G + 4);
    dim3 grid((m + G - 1) / G, nb);
    auto go = [&](auto gtag) {
        constexpr int GG = decltype(gtag)::value;
        static const bool attr = [] {   // thread-safe once per G (setups run on several host threads)
            CK(cudaFuncSetAttribute(k_bd_inv_tile<GG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            return true;
        }();
        (void)attr;
        k_bd_inv_tile<GG><<<grid, BDI_THREADS, sm, c->s>>>(n, B, T.backward, T.strict.ptr.p, T.strict.idx.p,
                                                          T.strict.val.p, T.diag.n ? T.diag.p : nullptr, dense);
    };
    switch (G) {
        case 32: go(std::integral_constant<int, 32>{}); break;
        case 16: go(std::integral_constant<int, 16>{}); break;
        case 8: go(std::integral_constant<int, 8>{}); break;
        default: go(std::integral_constant<int, 4>{}); break;
    }
    launched(c);
    return true;
}

// ---------------------------------------------------------------- sweep
// Values move between the cluster's CTAs only by st.async pushes that count
// their bytes on the receiving CTA's mbarrier (no cluster barrier, no fence):
//   y of step t  -> every CTA's yf[t & 1],       counted on mby[t & 1]
//   x of block t -> every CTA's x window slot,   counted on mbx[t & 1]
// Buffer reuse is safe by causality: a CTA can only produce step t+1 data after
// it received every CTA's step t data, and every CTA consumed its own step t
// buffers (CTA barrier) before producing step t+1 data.
//
// shared memory: mbarriers (ring NST, mby 2, mbx 2) | yf[2][B] | xw[W][B] | bst[2][B] | so[2 nb] | ring
__host__ __device__ inline size_t bd_fixed(int B, int nb, int W) {
    return 8 * (BD_NST_MAX + 4) + 8 * (size_t)B * (2 + W + 2) + (size_t)bd_pad16(16LL * nb);
}
__device__ __forceinline__ unsigned bd_mapa(unsigned a, int rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void bd_push(unsigned raddr, double v, unsigned rmbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
                 ::"r"(raddr), "l"(__double_as_longlong(v)), "r"(rmbar) : "memory");
}
__device__ __forceinline__ void bd_arm(unsigned long long *m, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bd_u32(m)), "r"(bytes) : "memory");
}

__global__ void __launch_bounds__(BD_THREADS, 1)
    k_trsv_bd(int n, int B, int nb, int W, int backward, int stage, int nst, const unsigned char *__restrict__ segs,
              const long long *__restrict__ soff, const double *__restrict__ b, double *x,
              const double *__restrict__ xadd, double *xout, unsigned long long *dbg) {
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned long long ph[6] = {0, 0, 0, 0, 0, 0}, tc = 0;
    unsigned long long *mbar = reinterpret_cast<unsigned long long *>(smem);
    unsigned long long *mby = mbar + BD_NST_MAX, *mbx = mby + 2;
    double *yf = reinterpret_cast<double *>(smem + 8 * (BD_NST_MAX + 4));
    double *xw = yf + 2 * (size_t)B;
    double *bst = xw + (size_t)W * B;
    long long *so = reinterpret_cast<long long *>(bst + 2 * (size_t)B);
    unsigned char *ring = smem + bd_fixed(B, nb, W);
    cg::cluster_group cl = cg::this_cluster();
    const int C = (int)cl.num_blocks(), k = (int)cl.block_rank();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    // push targets: lane l < C writes to CTA l
    const int peer = lane < C ? lane : 0;
    const unsigned yf_r = bd_mapa(bd_u32(yf), peer), xw_r = bd_mapa(bd_u32(xw), peer);
    const unsigned mby_r = bd_mapa(bd_u32(mby), peer), mbx_r = bd_mapa(bd_u32(mbx), peer);
    auto seg_of = [&](int t) { return (backward ? nb - 1 - t : t) * C + k; };
    auto rows_of = [&](int t) { const int blk = backward ? nb - 1 - t : t; return min(B, n - blk * B); };
    auto issue = [&](int t) {   // step t's segment -> ring slot t % nst
        bd_issue(ring + (size_t)(t % nst) * stage, segs + so[2 * t], (unsigned)so[2 * t + 1], &mbar[t % nst]);
    };
    auto fetch_b = [&](int t) {   // lane 0: b of this warp's rows of step t -> bst[t & 1] (async)
        if (lane != 0 || t >= nb) return;
        const int blk = backward ? nb - 1 - t : t;
        const int s = blk * B, m = min(B, n - s);
        double *dst = bst + (size_t)(t & 1) * B;
        for (int a = k + C * warp; a < m; a += C * nw)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(bd_u32(dst + a)), "l"(b + s + a) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (threadIdx.x < nst + 4)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bd_u32(&mbar[threadIdx.x < nst ? threadIdx.x : BD_NST_MAX + threadIdx.x - nst])) : "memory");
    for (int t = threadIdx.x; t < nb; t += blockDim.x) {
        const int sg = seg_of(t);
        so[2 * t] = soff[sg];
        so[2 * t + 1] = soff[sg + 1] - soff[sg];
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    // producer: lane 0 of the last warp (the TMA issue / mbarrier bookkeeping stays off
    // warp 0, whose row is the first of every block)
    const bool producer = threadIdx.x == blockDim.x - 32;
    if (producer) {
        for (int t = 0; t < min(nst - 1, nb); ++t) issue(t);
        bd_arm(&mby[0], 8u * rows_of(0));
        bd_arm(&mbx[0], 8u * rows_of(0));
        bd_mbar_wait(&mbar[0], 0);
    }
    fetch_b(0);
    // every CTA's mbarriers are initialised before the first remote push
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    for (int t = 0; t < nb; ++t) {
        const int blk = backward ? nb - 1 - t : t;
        const int s = blk * B, m = min(B, n - s);
        const unsigned par = (unsigned)((t >> 1) & 1);
        if (dbg) tc = clock64();
        if (producer) {
            if (t + nst - 1 < nb) issue(t + nst - 1);   // slot of step t-1 is free
            if (t + 1 < nb) bd_arm(&mby[(t + 1) & 1], 8u * rows_of(t + 1));   // its previous phase (t-1) completed
        }
        const double *bs = bst + (size_t)(t & 1) * B;
        if (lane == 0) asm volatile("cp.async.wait_all;" ::: "memory");   // this step's b
        __syncwarp();
        fetch_b(t + 1);
        const unsigned char *S = ring + (size_t)(t % nst) * stage;
        const int nr = reinterpret_cast<const int *>(S)[0], ne = reinterpret_cast<const int *>(S)[1];
        const int *dofs = reinterpret_cast<const int *>(S + 16);
        const int *optr = dofs + nr + 1;
        const int *oidx = optr + nr + 1;
        const double *dv = reinterpret_cast<const double *>(S + bd_pad16(16 + 4LL * (nr + 1) * 2 + 4LL * ne));
        const double *ov = dv + dofs[nr];
        // x of the previous block has landed in the window
        if (t > 0) bd_mbar_wait(&mbx[(t - 1) & 1], (unsigned)(((t - 1) >> 1) & 1));
        // mbx[(t+1) & 1] is re-armed only after its previous phase (block t-1) completed
        if (producer && t + 1 < nb) bd_arm(&mbx[(t + 1) & 1], 8u * rows_of(t + 1));
        if (dbg) { const unsigned long long u = clock64(); ph[0] += u - tc; tc = u; }
        // 1. y = b - T_off x over this CTA's rows (warp per row), pushed to every CTA
        for (int i = warp; i < nr; i += nw) {
            const int a = k + C * i;
            double acc = 0.0;
            for (int p = optr[i] + lane; p < optr[i + 1]; p += 32) acc += ov[p] * xw[oidx[p]];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane < C) bd_push(yf_r + 8u * ((t & 1) * B + a), bs[a] - acc, mby_r + 8u * (t & 1));
        }
        if (dbg) { const unsigned long long u = clock64(); ph[1] += u - tc; tc = u; }
        bd_mbar_wait(&mby[t & 1], par);
        if (dbg) { const unsigned long long u = clock64(); ph[2] += u - tc; tc = u; }
        // 2. x_blk = inv(T_blk) y, this CTA's rows (packed triangle rows in the segment)
        const double *y = yf + (size_t)(t & 1) * B;
        const unsigned slot = (unsigned)((blk % W) * B);
        for (int i = warp; i < nr; i += nw) {
            const int a = k + C * i;
            const int j0 = backward ? a : 0;
            const double *row = dv + dofs[i];
            const int len = dofs[i + 1] - dofs[i];
            double acc0 = 0.0, acc1 = 0.0;
            int q = lane;
            for (; q + 32 < len; q += 64) {
                acc0 += row[q] * y[j0 + q];
                acc1 += row[q + 32] * y[j0 + q + 32];
            }
            if (q < len) acc0 += row[q] * y[j0 + q];
            double acc = acc0 + acc1;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (dbg) { const unsigned long long u = clock64() + (unsigned long long)(acc != acc); ph[5] += u - tc; }
            if (lane < C) bd_push(xw_r + 8u * (slot + a), acc, mbx_r + 8u * (t & 1));
            if (lane == 31) {
                x[s + a] = acc;
                if (xout) xout[s + a] = xadd[s + a] + acc;
            }
        }
        if (dbg) { const unsigned long long u = clock64(); ph[3] += u - tc; tc = u; }
        // next step's segment landed; this step's ring slot and yf buffer are free
        if (producer && t + 1 < nb) bd_mbar_wait(&mbar[(t + 1) % nst], (unsigned)(((t + 1) / nst) & 1));
        if (dbg) { const unsigned long long u = clock64(); ph[4] += u - tc; tc = u; }
        __syncthreads();
    }
    // the last block's x pushes must land before this CTA's shared memory is released
    bd_mbar_wait(&mbx[(nb - 1) & 1], (unsigned)(((nb - 1) >> 1) & 1));
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (dbg && threadIdx.x == (int)(dbg[6 * 16] & 1023))
        for (int q = 0; q < 6; ++q) dbg[k * 6 + q] = ph[q];
}

static int bd_cluster_size() {
    static int C = -1;
    if (C < 0) {
        C = 16;
        if (cudaFuncSetAttribute(k_trsv_bd, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
            cudaGetLastError();
            C = 8;
        }
    }
    return C;
}

// dense inverse of a whole (small) triangle: T.dense = T^{-1}, n x n row-major
void tri_dense_inverse(Ctx *c, Tri &T) {
    const int n = T.n;
    T.dense.alloc((size_t)n * n, c->s);
    if (bd_inverse_gemm(c, n, n, 1, T, T.dense.p)) return;    // writes every entry
    if (bd_inverse_tiles(c, n, n, 1, T, T.dense.p)) return;   // writes every entry
    CK(cudaMemsetAsync(T.dense.p, 0, sizeof(double) * (size_t)n * n, c->s));
    const size_t sm = (size_t)BD_INV_WPB * n * sizeof(double);
    static bool attr = false;
    if (!attr) {
        CK(cudaFuncSetAttribute(k_bd_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(BD_INV_WPB * 4096 * sizeof(double))));
        attr = true;
    }
    dim3 grid((n + BD_INV_WPB - 1) / BD_INV_WPB, 1);
    k_bd_inverse<<<grid, 32 * BD_INV_WPB, sm, c->s>>>(n, n, T.backward, T.strict.ptr.p, T.strict.idx.p,
                                                       T.strict.val.p, T.diag.n ? T.diag.p : nullptr, T.dense.p);
    launched(c);
}

bool bd_plan(Ctx *c, Tri &T, int B) {
    DPP_TRACE_SCOPE(c, "tri.bd_plan");
    const int n = T.n;
    if (n == 0 || B <= 0) return false;
    auto P = std::make_unique<BdPlan>();
    P->B = B;
    P->nb = (n + B - 1) / B;
    P->C = bd_cluster_size();
    const int C = P->C, nseg = P->nb * C;
    // segment sizes -> offsets
    DBuf<long long> sz(nseg, c->s);
    DBuf<int> mb(1, c->s);
    CK(cudaMemsetAsync(mb.p, 0, sizeof(int), c->s));
    k_bd_seg_size<<<(nseg * 32 + 127) / 128, 128, 0, c->s>>>(n, B, C, P->nb, T.backward, T.strict.ptr.p,
                                                         T.strict.idx.p, sz.p, mb.p);
    launched(c);
    P->W = std::max(1, mb.to_host()[0] + 1);   // window slots: blocks back 1..maxback, plus the current
    std::vector<long long> hs = sz.to_host(), ho(nseg + 1, 0);
    long long mx = 0;
    for (int i = 0; i < nseg; ++i) {
        ho[i + 1] = ho[i] + hs[i];
        mx = std::max(mx, hs[i]);
    }
    const long long stage = (mx + 127) & ~127LL;
    const size_t fixed = bd_fixed(B, P->nb, P->W);
    if (fixed + 2 * (size_t)stage > BD_SMEM_LIMIT) return false;
    P->nst = (int)std::min<size_t>(BD_NST_MAX, (BD_SMEM_LIMIT - fixed) / stage);
    P->nst = std::min(P->nst, std::max(2, P->nb));
    P->stage = (int)stage;
    P->soff.alloc(nseg + 1, c->s);
    P->soff.upload(ho.data(), nseg + 1);
    P->segs.alloc((size_t)std::max<long long>(ho[nseg], 16), c->s);
    // dense diagonal-block inverses (temporary) -> packed segments
    {
        DBuf<double> dense((size_t)P->nb * B * B, c->s);
        const size_t sm = (size_t)BD_INV_WPB * B * sizeof(double);
        static bool attr = false;
        if (!attr) {
            CK(cudaFuncSetAttribute(k_bd_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(BD_INV_WPB * 4096 * sizeof(double))));
            CK(cudaFuncSetAttribute(k_trsv_bd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BD_SMEM_LIMIT));
            attr = true;
        }
        if (!bd_inverse_gemm(c, n, B, P->nb, T, dense.p) && !bd_inverse_tiles(c, n, B, P->nb, T, dense.p)) {
            dim3 grid((B + BD_INV_WPB - 1) / BD_INV_WPB, P->nb);
            k_bd_inverse<<<grid, 32 * BD_INV_WPB, sm, c->s>>>(n, B, T.backward, T.strict.ptr.p, T.strict.idx.p,
                                                               T.strict.val.p, T.diag.n ? T.diag.p : nullptr, dense.p);
            launched(c);
        }
        k_bd_seg_fill<<<nseg, 256, 0, c->s>>>(n, B, C, P->W, T.backward, T.strict.ptr.p, T.strict.idx.p,
                                               T.strict.val.p, dense.p, P->soff.p, P->segs.p);
        launched(c);
        CK(cudaStreamSynchronize(c->s));
    }
    if (TraceScope::on())
        std::fprintf(stderr, "[dpp-trace]   bd_plan n=%d B=%d nb=%d C=%d W=%d stage=%lld nst=%d segs %.1f MB\n", n, B,
                     P->nb, C, P->W, stage, P->nst, ho[nseg] / 1e6);
    T.bd = std::move(P);
    return true;
}

// ---------------------------------------------------------------- global block-dense sweep
// AMG smoother factors with long rows whose x window does not fit one cluster (C4: 16,604 rows,
// 485 entries per row, 2,524 levels; C3: 44,433 rows, 3,065 levels): the same block recurrence
// x_k = inv(T_kk) (b_k - sum_{j != k} T_kj x_j) as the cluster kernel above, but every block step
// is two ordinary launches over the whole device -- the off-block rows as a warp-per-row SpMV
// against x in global memory, then the block's rows of the dense inverse -- chained by
// programmatic dependent launches inside the preconditioner's CUDA graph.  ceil(n / B) dependent
// steps of a few microseconds each instead of thousands of levels.
__global__ void k_gbd_count(int n, int B, const int *__restrict__ ptr, const int *__restrict__ idx, int *cnt) {
    const int lane = threadIdx.x & 31;
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += (gridDim.x * blockDim.x) >> 5) {
        int e = 0;
        for (int p = ptr[r] + lane; p < ptr[r + 1]; p += 32) e += (idx[p] / B) != (r / B);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
        if (lane == 0) cnt[r] = e;
    }
}
__global__ void k_gbd_fill(int n, int B, const int *__restrict__ ptr, const int *__restrict__ idx,
                           const double *__restrict__ val, const int *__restrict__ optr, int *oidx, double *oval) {
    const int lane = threadIdx.x & 31;
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += (gridDim.x * blockDim.x) >> 5) {
        int w = optr[r];
        for (int base = ptr[r]; base < ptr[r + 1]; base += 32) {
            const int p = base + lane;
            const bool keep = p < ptr[r + 1] && (idx[p] / B) != (r / B);
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const int pos = w + __popc(m & ((1u << lane) - 1));
                oidx[pos] = idx[p];
                oval[pos] = val[p];
            }
            w += __popc(m);
        }
    }
}
// y[r] = b[r] - sum off[r, :] x for the rows [r0, r1) of one block (warp per row, entries in storage order per lane)
__global__ void __launch_bounds__(256) k_gbd_off(int r0, int r1, const int *__restrict__ ptr, const int *__restrict__ idx,
                                                 const double *__restrict__ val, const double *__restrict__ b,
                                                 const double *x, double *y) {
    const int lane = threadIdx.x & 31;
    const int r = r0 + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (r >= r1) return;
    const int p0 = ptr[r], p1 = ptr[r + 1];   // the plan is static: read before the predecessor ends
    pdl_wait();
    double acc = 0.0;
    for (int p = p0 + lane; p < p1; p += 32) acc = fma(val[p], __ldcg(x + idx[p]), acc);   // x: other launches' output
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) y[r] = b[r] - acc;
    pdl_trigger();
}
// x[r] = sum_j inv(T_kk)[a, j] y[s + j] over the triangle's half; xout = xadd + x
__global__ void __launch_bounds__(256) k_gbd_inv(int s, int m, int B, int backward, const double *__restrict__ Di,
                                                 const double *y, double *x, const double *xadd, double *xout) {
    const int lane = threadIdx.x & 31;
    const int a = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (a >= m) return;
    const int j0 = backward ? a : 0, j1 = backward ? m : a + 1;
    const double *row = Di + (size_t)a * B;
    double dv[4];   // the first entries of the inverse's row while the predecessor finishes
#pragma unroll
    for (int u = 0; u < 4; ++u) { const int j = j0 + lane + 32 * u; dv[u] = j < j1 ? row[j] : 0.0; }
    pdl_wait();
    double acc = 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u) { const int j = j0 + lane + 32 * u; if (j < j1) acc = fma(dv[u], __ldcg(y + s + j), acc); }
    for (int j = j0 + lane + 128; j < j1; j += 32) acc = fma(row[j], __ldcg(y + s + j), acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
        x[s + a] = acc;
        if (xout) xout[s + a] = xadd[s + a] + acc;
    }
    pdl_trigger();
}
bool gbd_plan(Ctx *c, Tri &T, int B) {
    DPP_TRACE_SCOPE(c, "tri.gbd_plan");
    const int n = T.n;
    if (n == 0 || B <= 0 || T.ncomp != 1) return false;
    auto P = std::make_unique<GbdPlan>();
    P->B = B;
    P->nb = (n + B - 1) / B;
    P->dinv.alloc((size_t)P->nb * B * B, c->s);
    if (!bd_inverse_gemm(c, n, B, P->nb, T, P->dinv.p)) return false;
    DBuf<int> cnt(n, c->s);
    const int grid = grid_for((int64_t)n * 32, 256, c->sms, 8);
    k_gbd_count<<<grid, 256, 0, c->s>>>(n, B, T.strict.ptr.p, T.strict.idx.p, cnt.p);
    launched(c);
    P->off.rows = n;
    P->off.cols = n;
    P->off.nnz = counts_to_ptr(c, cnt.p, n, P->off.ptr);
    P->off.idx.alloc((size_t)P->off.nnz, c->s);
    P->off.val.alloc((size_t)P->off.nnz, c->s);
    k_gbd_fill<<<grid, 256, 0, c->s>>>(n, B, T.strict.ptr.p, T.strict.idx.p, T.strict.val.p, P->off.ptr.p, P->off.idx.p,
                                       P->off.val.p);
    launched(c);
    P->y.alloc(n, c->s);
    CK(cudaStreamSynchronize(c->s));
    if (TraceScope::on())
        std::fprintf(stderr, "[dpp-trace]   gbd_plan n=%d B=%d nb=%d off-block nnz %lld of %lld\n", n, B, P->nb,
                     (long long)P->off.nnz, (long long)T.strict.nnz);
    T.gbd = std::move(P);
    return true;
}
void trsv_gbd(Ctx *c, const Tri &T, const double *b, double *x, const double *xadd, double *xout, cudaStream_t st) {
    const GbdPlan &P = *T.gbd;
    const int n = T.n, B = P.B;
    for (int t = 0; t < P.nb; ++t) {
        const int k = T.backward ? P.nb - 1 - t : t;
        const int s = k * B, m = std::min(B, n - s);
        CK(launch_pdl(k_gbd_off, dim3((m * 32 + 255) / 256), dim3(256), 0, st, s, s + m, (const int *)P.off.ptr.p,
                      (const int *)P.off.idx.p, (const double *)P.off.val.p, b, (const double *)x, P.y.p));
        launched(c);
        CK(launch_pdl(k_gbd_inv, dim3((m * 32 + 255) / 256), dim3(256), 0, st, s, m, B, (int)T.backward,
                      (const double *)(P.dinv.p + (size_t)k * B * B), (const double *)P.y.p, x, xadd, xout));
        launched(c);
    }
}

void trsv_bd(Ctx *c, const Tri &T, const double *b, double *x, const double *xadd, double *xout,
             cudaStream_t st) {
    const BdPlan &P = *T.bd;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P.C, 1, 1);
    cfg.blockDim = dim3(BD_THREADS, 1, 1);
    cfg.dynamicSmemBytes = bd_fixed(P.B, P.nb, P.W) + (size_t)P.nst * P.stage;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = P.C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    static const bool dbg_on = [] { const char *e = std::getenv("DPP_BD_DEBUG"); return e && *e == '1'; }();
    unsigned long long *dbg = nullptr;
    if (dbg_on && !c->capturing) {
        CK(cudaMallocAsync((void **)&dbg, sizeof(unsigned long long) * (6 * 16 + 1), st));
        static const unsigned long long who = [] { const char *e = std::getenv("DPP_BD_THREAD"); return e ? std::atoll(e) : 0ll; }();
        CK(cudaMemcpyAsync(dbg + 6 * 16, &who, 8, cudaMemcpyHostToDevice, st));
    }
    CK(cudaLaunchKernelEx(&cfg, k_trsv_bd, T.n, P.B, P.nb, P.W, (int)T.backward, P.stage, P.nst, P.segs.p, P.soff.p, b,
                          x, xadd, xout, dbg));
    launched(c);
    if (dbg) {
        std::vector<unsigned long long> h(6 * P.C);
        CK(cudaMemcpyAsync(h.data(), dbg, h.size() * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        cudaFreeAsync(dbg, st);
        std::fprintf(stderr, "[dpp-bd] n=%d nb=%d cycles/step (CTA0,1,15): top %.0f %.0f %.0f | gather %.0f | ywait %.0f | gemv %.0f | mbar %.0f | gemv-before-push %.0f\n",
                     T.n, P.nb, (double)h[0] / P.nb, (double)h[6] / P.nb, (double)h[6 * (P.C - 1)] / P.nb,
                     (double)h[1] / P.nb, (double)h[2] / P.nb, (double)h[3] / P.nb, (double)h[4] / P.nb, (double)h[5] / P.nb);
    }
}

}  // namespace dpp
