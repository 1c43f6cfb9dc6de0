// Row-sharded SpMV over NVLink peer memory (NON-PARITY extension).
//
// The reference has one SpMV, scipy's csr_matvec on the whole K (linalg.py:27-32).  For meshes
// beyond one GPU, K is cut into contiguous row blocks, one per rank (one process per GPU); rank p
// owns rows [r_p, r_{p+1}) of K and the same slice of every vector.  There is no halo exchange
// step: every rank keeps its slice of x in a cudaMalloc'd buffer exported over CUDA IPC, the
// other ranks map it (dpp_peerbuf_open), and the SpMV kernel loads the off-rank entries of x
// straight through those peer mappings -- NVLink 5 / NVSwitch loads issued from inside the row
// loop, overlapped with the streaming of the local values -- instead of an all-gather followed
// by a local SpMV.  A column is stored as a 32-bit code, owner << 29 | offset in the owner's
// slice (up to 8 ranks, 2^29 rows per rank), resolved at plan time on the host
// (paper_1808_08328_b200/sharded.py), so the kernel's only extra work per entry is a shift, a
// mask and an indexed pointer load from the kernel parameters.
//
// Each row's products are summed by G lanes and a shuffle tree: equal to csr_matvec up to the
// order of the additions (last-bit differences), hence outside the parity contract -- as is any
// sharded preconditioner.
#include <climits>
#include <cstdlib>
#include <memory>

#include "abi_guard.cuh"
#include "dpp_internal.cuh"

struct dpp_peerbuf {
    dpp::Ctx *ctx = nullptr;
    double *p = nullptr;
    int64_t n = 0;
    bool mapped = false;   // opened from another process' IPC handle (closed, not freed)
};

namespace dpp {

constexpr int SEG_MAX = 8;
constexpr int OFF_BITS = 29;
constexpr uint32_t OFF_MASK = (1u << OFF_BITS) - 1;

struct XSegs { const double *p[SEG_MAX]; };

template <int G>
__global__ void __launch_bounds__(256) k_shard_spmv(int rows, const int *__restrict__ ptr,
                                                    const uint32_t *__restrict__ code,
                                                    const double *__restrict__ val, const __grid_constant__ XSegs x,
                                                    double *__restrict__ y) {
    constexpr int RPW = 32 / G;
    const int lane = threadIdx.x & (G - 1);
    const int grp = (threadIdx.x & 31) / G;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t w = warp; w * RPW < rows; w += nwarp) {
        const int64_t r = w * RPW + grp;
        double s = 0.0;
        int b = 0, e = 0;
        if (r < rows) { b = ptr[r]; e = ptr[r + 1]; }
        // every lane of the warp runs the longest row's trip count (full shuffles below)
        int trips = (e - b + G - 1) / G;
#pragma unroll
        for (int o = 16; o >= G; o >>= 1) trips = max(trips, __shfl_xor_sync(0xffffffffu, trips, o));
        for (int t = 0; t < trips; ++t) {
            const int j = b + t * G + lane;
            if (j < e) {
                const uint32_t cd = __ldg(code + j);
                s = fma(__ldg(val + j), x.p[cd >> OFF_BITS][cd & OFF_MASK], s);
            }
        }
#pragma unroll
        for (int o = G >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0 && r < rows) y[r] = s;
    }
}

struct Shard {
    Ctx *ctx = nullptr;
    int rows = 0, nseg = 0, G = 8;
    int64_t nnz = 0;
    int64_t seg_len[SEG_MAX] = {0};
    DBuf<int> ptr;
    DBuf<uint32_t> code;
    DBuf<double> val;
};

static void shard_launch(Ctx *c, const Shard &S, const XSegs &x, double *y) {
    if (!S.rows) return;
    const int rpw = 32 / S.G;
    const int64_t warps = (S.rows + rpw - 1) / rpw;
    const int grid = grid_for(warps * 32, 256, c->sms, 8);
    switch (S.G) {
        case 2: k_shard_spmv<2><<<grid, 256, 0, c->s>>>(S.rows, S.ptr.p, S.code.p, S.val.p, x, y); break;
        case 4: k_shard_spmv<4><<<grid, 256, 0, c->s>>>(S.rows, S.ptr.p, S.code.p, S.val.p, x, y); break;
        case 8: k_shard_spmv<8><<<grid, 256, 0, c->s>>>(S.rows, S.ptr.p, S.code.p, S.val.p, x, y); break;
        case 16: k_shard_spmv<16><<<grid, 256, 0, c->s>>>(S.rows, S.ptr.p, S.code.p, S.val.p, x, y); break;
        default: k_shard_spmv<32><<<grid, 256, 0, c->s>>>(S.rows, S.ptr.p, S.code.p, S.val.p, x, y); break;
    }
    launched(c);
}

static XSegs bind(const Shard &S, dpp_peerbuf *const *xseg, const dpp_peerbuf *y) {
    XSegs x{};
    for (int p = 0; p < S.nseg; ++p) {
        if (!xseg[p] || xseg[p]->n < S.seg_len[p]) DPP_FAIL(DPP_ERR_VALUE, "x segment shorter than the plan's slice");
        if (xseg[p]->p == y->p) DPP_FAIL(DPP_ERR_VALUE, "y aliases an x segment");
        x.p[p] = xseg[p]->p;
    }
    if (y->n < S.rows) DPP_FAIL(DPP_ERR_VALUE, "y shorter than the shard's row count");
    return x;
}

}  // namespace dpp

struct dpp_shard { dpp::Shard s; };

using namespace dpp;

extern "C" {

int dpp_peerbuf_create(dpp_ctx *ctx, int64_t n, dpp_peerbuf **out) {
    return guard([&] {
        if (n < 0) DPP_FAIL(DPP_ERR_VALUE, "negative buffer length");
        auto h = std::make_unique<dpp_peerbuf>();
        h->ctx = &ctx->c;
        h->n = n;
        // cudaMalloc, not the stream-ordered pool: pool memory cannot be exported as a legacy IPC handle
        CK(cudaMalloc((void **)&h->p, sizeof(double) * (size_t)std::max<int64_t>(n, 1)));
        CK(cudaMemsetAsync(h->p, 0, sizeof(double) * (size_t)std::max<int64_t>(n, 1), ctx->c.s));
        CK(cudaStreamSynchronize(ctx->c.s));
        *out = h.release();
    });
}

int dpp_peerbuf_export(const dpp_peerbuf *b, unsigned char *handle64) {
    return guard([&] {
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
        if (b->mapped) DPP_FAIL(DPP_ERR_VALUE, "a mapped peer buffer cannot be re-exported");
        cudaIpcMemHandle_t h;
        CK(cudaIpcGetMemHandle(&h, b->p));
        std::memcpy(handle64, &h, 64);
    });
}

int dpp_peerbuf_open(dpp_ctx *ctx, const unsigned char *handle64, int64_t n, dpp_peerbuf **out) {
    return guard([&] {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle64, 64);
        auto b = std::make_unique<dpp_peerbuf>();
        b->ctx = &ctx->c;
        b->n = n;
        b->mapped = true;
        CK(cudaIpcOpenMemHandle((void **)&b->p, h, cudaIpcMemLazyEnablePeerAccess));
        *out = b.release();
    });
}

int dpp_peerbuf_write(dpp_peerbuf *b, const double *host, int64_t n) {
    return guard([&] {
        if (n < 0 || n > b->n) DPP_FAIL(DPP_ERR_VALUE, "write beyond the buffer");
        if (n) CK(cudaMemcpyAsync(b->p, host, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, b->ctx->s));
        CK(cudaStreamSynchronize(b->ctx->s));
    });
}

int dpp_peerbuf_read(const dpp_peerbuf *b, double *host, int64_t n) {
    return guard([&] {
        if (n < 0 || n > b->n) DPP_FAIL(DPP_ERR_VALUE, "read beyond the buffer");
        if (n) CK(cudaMemcpyAsync(host, b->p, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, b->ctx->s));
        CK(cudaStreamSynchronize(b->ctx->s));
    });
}

int dpp_peerbuf_destroy(dpp_peerbuf *b) {
    return guard([&] {
        if (!b) return;
        cudaStreamSynchronize(b->ctx->s);
        if (b->mapped) cudaIpcCloseMemHandle(b->p);
        else cudaFree(b->p);
        delete b;
    });
}

int dpp_shard_create(dpp_ctx *ctx, int rows, int64_t nnz, const int32_t *indptr, const uint32_t *codes,
                     const double *values, int nseg, const int64_t *seg_len, dpp_shard **out) {
    return guard([&] {
        if (rows < 0 || nnz < 0 || nnz > INT_MAX) DPP_FAIL(DPP_ERR_VALUE, "bad shard shape");
        if (nseg < 1 || nseg > SEG_MAX) DPP_FAIL(DPP_ERR_VALUE, "between 1 and 8 x segments (ranks)");
        for (int p = 0; p < nseg; ++p)
            if (seg_len[p] < 0 || seg_len[p] > (int64_t)OFF_MASK + 1) DPP_FAIL(DPP_ERR_VALUE, "x segment longer than 2^29");
        if (indptr[0] != 0 || indptr[rows] != nnz) DPP_FAIL(DPP_ERR_VALUE, "indptr does not span the entries");
        for (int r = 0; r < rows; ++r)
            if (indptr[r + 1] < indptr[r]) DPP_FAIL(DPP_ERR_VALUE, "indptr is not monotone");
        for (int64_t j = 0; j < nnz; ++j) {
            const uint32_t o = codes[j] >> OFF_BITS;
            if ((int)o >= nseg || (int64_t)(codes[j] & OFF_MASK) >= seg_len[o])
                DPP_FAIL(DPP_ERR_VALUE, "column code outside its owner's slice");
        }
        auto h = std::make_unique<dpp_shard>();
        Shard &S = h->s;
        Ctx *c = &ctx->c;
        S.ctx = c;
        S.rows = rows;
        S.nnz = nnz;
        S.nseg = nseg;
        for (int p = 0; p < nseg; ++p) S.seg_len[p] = seg_len[p];
        const double mean = rows ? (double)nnz / rows : 0.0;
        S.G = mean <= 3 ? 2 : mean <= 8 ? 4 : mean <= 64 ? 8 : mean <= 256 ? 16 : 32;   // measured on C2 K (40 per row): 8 lanes 4.5 TB/s, 16 lanes 3.8
        if (const char *e = std::getenv("DPP_SHARD_G")) {   // A/B of the lanes-per-row choice
            const int g = std::atoi(e);
            if (g == 2 || g == 4 || g == 8 || g == 16 || g == 32) S.G = g;
        }
        S.ptr.alloc((size_t)rows + 1, c->s);
        S.code.alloc((size_t)nnz, c->s);
        S.val.alloc((size_t)nnz, c->s);
        S.ptr.upload(indptr, (size_t)rows + 1);
        S.code.upload(codes, (size_t)nnz);
        S.val.upload(values, (size_t)nnz);
        CK(cudaStreamSynchronize(c->s));
        *out = h.release();
    });
}

int dpp_shard_spmv(dpp_ctx *ctx, const dpp_shard *sh, dpp_peerbuf *const *xseg, dpp_peerbuf *y) {
    return guard([&] {
        const XSegs x = bind(sh->s, xseg, y);
        shard_launch(&ctx->c, sh->s, x, y->p);
        CK(cudaStreamSynchronize(ctx->c.s));
    });
}

int dpp_shard_profile(dpp_ctx *ctx, const dpp_shard *sh, dpp_peerbuf *const *xseg, dpp_peerbuf *y, int reps,
                      double *ms_per_call, double *bytes_per_call) {
    return guard([&] {
        if (reps < 1) DPP_FAIL(DPP_ERR_VALUE, "reps must be positive");
        Ctx *c = &ctx->c;
        const Shard &S = sh->s;
        const XSegs x = bind(S, xseg, y);
        for (int i = 0; i < 3; ++i) shard_launch(c, S, x, y->p);
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, c->s));
        for (int i = 0; i < reps; ++i) shard_launch(c, S, x, y->p);
        CK(cudaEventRecord(e1, c->s));
        CK(cudaEventSynchronize(e1));
        float f = 0;
        CK(cudaEventElapsedTime(&f, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *ms_per_call = f / reps;
        // 12 B per entry + row pointers + one read of every x slice + the y rows
        double xb = 0;
        for (int p = 0; p < S.nseg; ++p) xb += 8.0 * S.seg_len[p];
        if (bytes_per_call) *bytes_per_call = 12.0 * S.nnz + 4.0 * (S.rows + 1) + xb + 8.0 * S.rows;
    });
}

int dpp_shard_destroy(dpp_shard *sh) {
    return guard([&] { delete sh; });
}

}  // extern "C"
