// mds_api.cu -- libmds: context, C-ABI entry points (include/mds.h), launch
// dispatch and the HMC driver.  One translation unit so the __constant__
// coefficient tables are visible to every kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mds.h"
#include "mds_kernels.cuh"

using namespace mdsk;

namespace {
const char* kVersion = "0.1.0";
}  // namespace

struct mds_ctx_s {
    int64_t n = 0;
    int d = 0;
    int prec = MDS_F64;
    int trunc = 1;
    int rank = 0, world = 1;
    int nb = 0;              // tile-rows/cols
    int64_t npad = 0;        // nb * B
    int ntl = 0;             // local tiles
    size_t elem = 8;         // bytes per stored y / x value

    std::vector<int> tiles;          // local tile codes (I << 16) | J, in storage order
    std::vector<int> row_local;      // [nb]: local index of tile (I, 0) or -1
    int* d_tiles = nullptr;
    int* d_row_local = nullptr;
    int* d_blk_ptr = nullptr;
    int* d_blk_ent = nullptr;

    void* d_y = nullptr;             // tiles
    double* d_x = nullptr;           // fp64 master X, npad x d
    float* d_xf = nullptr;           // fp32 copy (F32 only)
    double* d_part = nullptr;        // ntl x 2 x B x d
    double* d_likpart = nullptr;     // ntl
    double* d_grad = nullptr;        // n x d (internal result)
    double* d_lik = nullptr;         // [4]: loglik, scratch
    double* d_stage = nullptr;       // staging for packed rows
    size_t stage_elems = 0;
    int* d_bad = nullptr;
    unsigned long long* d_count = nullptr;

    // sharded exchange
    mds_allgather_fn ag_fn = nullptr;
    void* ag_user = nullptr;
    double* d_partial = nullptr;     // n*d + 1
    double* d_gathered = nullptr;    // world x (n*d + 1)

    // HMC
    double* d_p = nullptr;
    double* d_gl = nullptr;
    double* d_xsave = nullptr;
    double* d_glsave = nullptr;
    double* d_liksave = nullptr;
    double* d_H = nullptr;           // [3]
    double* d_H0 = nullptr;          // [3]

    uint64_t lf_version = 0;         // version the device-resident leapfrog state belongs to
    double lf_inv_tau2 = -1.0;

    SigmaParams P{};
    double sigma = 0.0;
    bool x_set = false, sigma_set = false;
    std::vector<uint8_t> row_supplied;
    int64_t rows_supplied = 0;
    int64_t rows_needed = 0;
    int64_t n_obs = -1;              // -1 = recount needed
    uint64_t version = 1, eval_version = 0;

    cudaStream_t stream = nullptr;
    bool timing = false;
    std::vector<cudaEvent_t> evpool;  // timing mode: 3 events per recorded pass
    size_t ev_used = 0;               // events recorded since the last mds_last_timing

    std::string err;
    mds_status sticky = MDS_OK;
};

namespace {

mds_status fail(mds_ctx c, mds_status s, const std::string& msg) {
    if (c) {
        c->err = msg;
        if (s == MDS_E_CUDA || s == MDS_E_COMM) c->sticky = s;
    }
    return s;
}

#define CK(call)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return fail(c, MDS_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define GUARD(c)                                          \
    do {                                                  \
        if (!(c)) return MDS_E_INVALID_ARG;               \
        if ((c)->sticky != MDS_OK) return (c)->sticky;    \
    } while (0)

mds_status check_device(mds_ctx c) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return fail(c, MDS_E_UNSUPPORTED, std::string("no CUDA device: ") + cudaGetErrorString(e));
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (major != 10)
        return fail(c, MDS_E_UNSUPPORTED, "libmds is built for sm_100a (B200); device has compute capability major " + std::to_string(major));
    return MDS_OK;
}

template <typename T>
mds_status dalloc(mds_ctx c, T** p, size_t count) {
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(c, MDS_E_OOM, "cudaMalloc of " + std::to_string(count * sizeof(T)) + " bytes failed");
    }
    return MDS_OK;
}

void free_all(mds_ctx c) {
    void* ps[] = {c->d_tiles, c->d_row_local, c->d_blk_ptr, c->d_blk_ent, c->d_y, c->d_x, c->d_xf,
                  c->d_part, c->d_likpart, c->d_grad, c->d_lik, c->d_stage, c->d_bad, c->d_count,
                  c->d_p, c->d_gl, c->d_xsave, c->d_glsave, c->d_liksave, c->d_H, c->d_H0,
                  c->d_partial, c->d_gathered};
    for (void* p : ps)
        if (p) cudaFree(p);
    for (auto& e : c->evpool)
        if (e) cudaEventDestroy(e);
}

inline int64_t packed_off(int64_t i) { return i * (i - 1) / 2; }

// ---------------------------------------------------------------- dispatch
template <typename T, bool TR>
void launch_tile_T(int d, int ntl, const TileArgs& a, cudaStream_t s) {
    switch (d) {
        case 1: tile_kernel<T, 1, TR><<<ntl, TILE_THREADS, 0, s>>>(a); break;
        case 2: tile_kernel<T, 2, TR><<<ntl, TILE_THREADS, 0, s>>>(a); break;
        case 3: tile_kernel<T, 3, TR><<<ntl, TILE_THREADS, 0, s>>>(a); break;
        case 4: tile_kernel<T, 4, TR><<<ntl, TILE_THREADS, 0, s>>>(a); break;
        case 5: tile_kernel<T, 5, TR><<<ntl, TILE_THREADS, 0, s>>>(a); break;
        case 6: tile_kernel<T, 6, TR><<<ntl, TILE_THREADS, 0, s>>>(a); break;
        case 7: tile_kernel<T, 7, TR><<<ntl, TILE_THREADS, 0, s>>>(a); break;
        case 8: tile_kernel<T, 8, TR><<<ntl, TILE_THREADS, 0, s>>>(a); break;
    }
}

void launch_tile(mds_ctx c, cudaStream_t s) {
    if (c->ntl == 0) return;   // a rank may own no tile-rows when world > nb
    TileArgs a;
    a.y = c->d_y;
    a.x = (c->prec == MDS_F64) ? (const void*)c->d_x : (const void*)c->d_xf;
    a.tiles = c->d_tiles;
    a.part = c->d_part;
    a.likpart = c->d_likpart;
    a.P = c->P;
    if (c->prec == MDS_F64) {
        if (c->trunc) launch_tile_T<double, true>(c->d, c->ntl, a, s);
        else launch_tile_T<double, false>(c->d, c->ntl, a, s);
    } else {
        if (c->trunc) launch_tile_T<float, true>(c->d, c->ntl, a, s);
        else launch_tile_T<float, false>(c->d, c->ntl, a, s);
    }
}

template <bool KICK>
void launch_reduce(mds_ctx c, double* grad_out, double* lik_out, const KickArgs& kk, cudaStream_t s) {
    const int64_t nd = c->n * c->d;
    const int64_t blocks = (nd + 31) / 32 + 1;
    reduce_kernel<KICK><<<(unsigned)blocks, 32 * RED_SEG, 0, s>>>(c->d_part, c->d_likpart, c->d_blk_ptr,
                                                                   c->d_blk_ent, c->n, c->d, c->ntl,
                                                                   grad_out, lik_out, kk);
}

void launch_x_convert(mds_ctx c, cudaStream_t s) {
    if (c->prec != MDS_F32) return;
    const int64_t m = c->npad * c->d;
    to_f32_kernel<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(c->d_x, c->d_xf, m);
}

// timing mode: the next event of the pool (grown on demand)
cudaEvent_t next_event(mds_ctx c) {
    if (c->ev_used == c->evpool.size()) {
        cudaEvent_t e = nullptr;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        c->evpool.push_back(e);
    }
    return c->evpool[c->ev_used++];
}

// One fused pass: [convert X] -> tile kernel -> fixed-order reduction
// [-> all-gather callback -> rank-ordered combine, when sharded] [-> kick].
// In timing mode three events bracket the pair kernel and the reduction.
template <bool KICK>
mds_status run_pass(mds_ctx c, double* grad_out, double* lik_out, const KickArgs& kk, cudaStream_t s, bool timed) {
    timed = timed && c->timing;
    launch_x_convert(c, s);
    if (timed) CK(cudaEventRecord(next_event(c), s));
    launch_tile(c, s);
    if (timed) CK(cudaEventRecord(next_event(c), s));
    if (c->world == 1) {
        launch_reduce<KICK>(c, grad_out, lik_out, kk, s);
    } else {
        if (!c->ag_fn) return fail(c, MDS_E_STATE, "sharded context: register the exchange with mds_set_allgather");
        const int64_t nd = c->n * c->d;
        launch_reduce<false>(c, c->d_partial, c->d_partial + nd, KickArgs{}, s);
        CK(cudaGetLastError());
        if (c->ag_fn(c->ag_user, c->d_partial, c->d_gathered, nd + 1, (void*)s) != 0)
            return fail(c, MDS_E_COMM, "all-gather callback failed");
        combine_kernel<<<(unsigned)((nd + 1 + 255) / 256), 256, 0, s>>>(c->d_gathered, c->world, nd + 1, grad_out, lik_out);
        if (KICK)
            kick_kernel<<<(unsigned)((nd + 255) / 256), 256, 0, s>>>(grad_out, kk.x, kk.gl, kk.p, nd, kk.half_eps, kk.inv_tau2);
    }
    if (timed) CK(cudaEventRecord(next_event(c), s));
    CK(cudaGetLastError());
    return MDS_OK;
}

mds_status ready(mds_ctx c) {
    if (c->rows_supplied < c->rows_needed)
        return fail(c, MDS_E_STATE, "dissimilarities not set (" + std::to_string(c->rows_supplied) + " of " +
                                        std::to_string(c->rows_needed) + " rows supplied)");
    if (!c->x_set) return fail(c, MDS_E_STATE, "locations not set");
    if (!c->sigma_set) return fail(c, MDS_E_STATE, "sigma not set");
    return MDS_OK;
}

// evaluate into the internal buffers if stale
mds_status eval_internal(mds_ctx c) {
    mds_status st = ready(c);
    if (st) return st;
    if (c->eval_version == c->version) return MDS_OK;
    KickArgs kk{};
    st = run_pass<false>(c, c->d_grad, c->d_lik, kk, c->stream, true);
    if (st) return st;
    c->eval_version = c->version;
    return MDS_OK;
}

mds_status create_impl(int64_t n, int32_t d, int32_t precision, int32_t truncation, int32_t rank,
                       int32_t world, mds_ctx* out) {
    if (!out) return MDS_E_INVALID_ARG;
    *out = nullptr;
    if (n < 2 || d < 1 || d > MDS_D_MAX || (precision != MDS_F64 && precision != MDS_F32) ||
        (truncation != 0 && truncation != 1) || world < 1 || rank < 0 || rank >= world)
        return MDS_E_INVALID_ARG;
    mds_ctx c = new (std::nothrow) mds_ctx_s();
    if (!c) return MDS_E_OOM;
    mds_status st = check_device(c);
    if (st) {
        delete c;
        return st;
    }
    c->n = n;
    c->d = d;
    c->prec = precision;
    c->trunc = truncation;
    c->rank = rank;
    c->world = world;
    c->elem = precision == MDS_F64 ? 8 : 4;
    c->nb = (int)((n + TB - 1) / TB);
    if (c->nb > 0xffff) {
        delete c;
        return MDS_E_INVALID_ARG;
    }
    c->npad = (int64_t)c->nb * TB;

    // tile-row ownership: cyclic (I mod world == rank), SURVEY 8(e)
    c->row_local.assign(c->nb, -1);
    for (int I = 0; I < c->nb; ++I) {
        if (I % world != rank) continue;
        c->row_local[I] = (int)c->tiles.size();
        for (int J = 0; J <= I; ++J) c->tiles.push_back((I << 16) | J);
    }
    c->ntl = (int)c->tiles.size();
    // rows this rank needs: all rows of its tile-rows
    c->row_supplied.assign(n, 0);
    for (int64_t i = 0; i < n; ++i)
        if (c->row_local[i / TB] >= 0) ++c->rows_needed;

    // per-block entry lists for the fixed-order reduction
    std::vector<int> ptr(c->nb + 1, 0), ent;
    for (int b = 0; b < c->nb; ++b) {
        ptr[b] = (int)ent.size();
        if (c->row_local[b] >= 0)
            for (int J = 0; J <= b; ++J) ent.push_back(2 * (c->row_local[b] + J) + 0);   // row role
        for (int I = b; I < c->nb; ++I)
            if (c->row_local[I] >= 0) ent.push_back(2 * (c->row_local[I] + b) + 1);      // column role
    }
    ptr[c->nb] = (int)ent.size();

    const size_t ntl = (size_t)std::max(c->ntl, 1);
#define AL(ptrv, cnt)                  \
    do {                               \
        st = dalloc(c, &ptrv, cnt);    \
        if (st) goto fail_alloc;       \
    } while (0)
    {
        AL(c->d_tiles, ntl);
        AL(c->d_row_local, (size_t)c->nb);
        AL(c->d_blk_ptr, (size_t)c->nb + 1);
        AL(c->d_blk_ent, std::max<size_t>(ent.size(), 1));
        char* yb = nullptr;
        AL(yb, ntl * TB * TB * c->elem);
        c->d_y = yb;
        AL(c->d_x, (size_t)c->npad * d);
        if (precision == MDS_F32) AL(c->d_xf, (size_t)c->npad * d);
        AL(c->d_part, ntl * 2 * TB * d);
        AL(c->d_likpart, ntl);
        AL(c->d_grad, (size_t)n * d);
        AL(c->d_lik, 4);
        AL(c->d_bad, 1);
        AL(c->d_count, 1);
        if (world > 1) {
            AL(c->d_partial, (size_t)n * d + 1);
            AL(c->d_gathered, ((size_t)n * d + 1) * world);
        }
        c->stage_elems = 0;
    }
#undef AL
    {
        cudaError_t e = cudaSuccess;
        if (c->ntl > 0) e = cudaMemcpy(c->d_tiles, c->tiles.data(), c->ntl * sizeof(int), cudaMemcpyHostToDevice);
        if (!e) e = cudaMemcpy(c->d_row_local, c->row_local.data(), c->nb * sizeof(int), cudaMemcpyHostToDevice);
        if (!e) e = cudaMemcpy(c->d_blk_ptr, ptr.data(), ptr.size() * sizeof(int), cudaMemcpyHostToDevice);
        if (!e && !ent.empty()) e = cudaMemcpy(c->d_blk_ent, ent.data(), ent.size() * sizeof(int), cudaMemcpyHostToDevice);
        if (!e) e = cudaMemset(c->d_x, 0, (size_t)c->npad * d * sizeof(double));
        if (!e && c->d_xf) e = cudaMemset(c->d_xf, 0, (size_t)c->npad * d * sizeof(float));
        if (!e) e = cudaMemset(c->d_part, 0, ntl * 2 * TB * d * sizeof(double));
        if (!e) e = cudaMemset(c->d_likpart, 0, ntl * sizeof(double));
        if (!e) {
            const size_t cnt = ntl * TB * TB;
            if (precision == MDS_F64) fill_nan_kernel<double><<<1184, 256>>>((double*)c->d_y, cnt);
            else fill_nan_kernel<float><<<1184, 256>>>((float*)c->d_y, cnt);
            e = cudaGetLastError();
        }
        if (!e) e = cudaDeviceSynchronize();
        if (e) {
            st = fail(c, MDS_E_CUDA, std::string("context setup: ") + cudaGetErrorString(e));
            goto fail_alloc;
        }
    }
    *out = c;
    return MDS_OK;
fail_alloc:
    free_all(c);
    delete c;
    return st;
}

// upload + pack rows [i0, i1) from a device pointer to fp64 packed rows
mds_status pack_rows_device(mds_ctx c, int64_t i0, int64_t i1, const double* src_dev, int64_t src_base) {
    CK(cudaMemsetAsync(c->d_bad, 0, sizeof(int), c->stream));
    PackArgs a;
    a.src = src_dev;
    a.i0 = i0;
    a.i1 = i1;
    a.src_base = src_base;
    a.row_local = c->d_row_local;
    a.dst = c->d_y;
    a.bad = c->d_bad;
    const unsigned blocks = (unsigned)(i1 - i0);
    if (blocks > 0) {
        if (c->prec == MDS_F64) pack_rows_kernel<double><<<blocks, 256, 0, c->stream>>>(a);
        else pack_rows_kernel<float><<<blocks, 256, 0, c->stream>>>(a);
        CK(cudaGetLastError());
    }
    int bad = 0;
    CK(cudaMemcpyAsync(&bad, c->d_bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (bad) {
        // the rows of this call now hold partial data: they count as not supplied
        for (int64_t i = i0; i < i1; ++i) {
            if (c->row_supplied[i]) {
                c->row_supplied[i] = 0;
                --c->rows_supplied;
            }
        }
        c->n_obs = -1;
        ++c->version;
        return fail(c, MDS_E_INVALID_ARG, "dissimilarities must be >= 0 and finite (NaN = missing)");
    }
    for (int64_t i = i0; i < i1; ++i) {
        if (c->row_local[i / TB] < 0) continue;
        if (!c->row_supplied[i]) {
            c->row_supplied[i] = 1;
            ++c->rows_supplied;
        }
    }
    c->n_obs = -1;
    ++c->version;
    return MDS_OK;
}

mds_status ensure_stage(mds_ctx c, size_t elems) {
    if (elems <= c->stage_elems) return MDS_OK;
    if (c->d_stage) cudaFree(c->d_stage);
    c->d_stage = nullptr;
    c->stage_elems = 0;
    mds_status st = dalloc(c, &c->d_stage, elems);
    if (st) return st;
    c->stage_elems = elems;
    return MDS_OK;
}

// host packed rows -> device, in chunks of at most ~32M values
mds_status set_rows_host(mds_ctx c, int64_t i0, int64_t i1, const double* y_lower) {
    const int64_t base0 = packed_off(std::max<int64_t>(i0, 1));
    const int64_t kChunk = 32LL << 20;
    int64_t r = std::max<int64_t>(i0, 1);
    while (r < i1) {
        int64_t r1 = r + 1;
        while (r1 < i1 && packed_off(r1 + 1) - packed_off(r) <= kChunk) ++r1;
        // skip chunks whose rows this rank does not own
        bool any = false;
        for (int64_t I = r / TB; I <= (r1 - 1) / TB; ++I) any = any || c->row_local[I] >= 0;
        if (any) {
            const int64_t cnt = packed_off(r1) - packed_off(r);
            mds_status st = ensure_stage(c, (size_t)cnt);
            if (st) return st;
            CK(cudaMemcpyAsync(c->d_stage, y_lower + (packed_off(r) - base0), cnt * sizeof(double),
                               cudaMemcpyHostToDevice, c->stream));
            st = pack_rows_device(c, r, r1, c->d_stage, packed_off(r));
            if (st) return st;
        }
        r = r1;
    }
    if (i0 == 0 && c->row_local[0] >= 0 && !c->row_supplied[0]) {   // row 0 has no entries
        c->row_supplied[0] = 1;
        ++c->rows_supplied;
    }
    return MDS_OK;
}

}  // namespace

// ======================================================================== ABI
extern "C" {

mds_status mds_create(int64_t n, int32_t d, int32_t precision, int32_t truncation, mds_ctx* out) {
    return create_impl(n, d, precision, truncation, 0, 1, out);
}

mds_status mds_create_sharded(int64_t n, int32_t d, int32_t precision, int32_t truncation, int32_t rank,
                              int32_t world, mds_ctx* out) {
    return create_impl(n, d, precision, truncation, rank, world, out);
}

void mds_destroy(mds_ctx c) {
    if (!c) return;
    if (c->stream) cudaStreamSynchronize(c->stream);
    else cudaDeviceSynchronize();
    free_all(c);
    delete c;
}

mds_status mds_set_stream(mds_ctx c, void* s) {
    GUARD(c);
    c->stream = (cudaStream_t)s;
    return MDS_OK;
}

mds_status mds_set_dissimilarity_rows(mds_ctx c, int64_t i0, int64_t i1, const double* y_lower) {
    GUARD(c);
    if (i0 < 0 || i1 > c->n || i0 > i1 || (!y_lower && packed_off(std::max<int64_t>(i1, 1)) > packed_off(std::max<int64_t>(i0, 1))))
        return fail(c, MDS_E_INVALID_ARG, "bad row range or NULL rows");
    return set_rows_host(c, i0, i1, y_lower);
}

mds_status mds_set_dissimilarity_rows_device(mds_ctx c, int64_t i0, int64_t i1, const double* y_dev) {
    GUARD(c);
    if (i0 < 0 || i1 > c->n || i0 > i1 || !y_dev) return fail(c, MDS_E_INVALID_ARG, "bad row range or NULL rows");
    const int64_t r0 = std::max<int64_t>(i0, 1);
    mds_status st = MDS_OK;
    if (i1 > r0) st = pack_rows_device(c, r0, i1, y_dev, packed_off(r0));
    if (st) return st;
    if (i0 == 0 && c->row_local[0] >= 0 && !c->row_supplied[0]) {
        c->row_supplied[0] = 1;
        ++c->rows_supplied;
    }
    return MDS_OK;
}

mds_status mds_set_dissimilarities(mds_ctx c, const double* y, int64_t ld) {
    GUARD(c);
    if (!y || ld < c->n) return fail(c, MDS_E_INVALID_ARG, "NULL matrix or ld < n");
    // pack the strict lower triangle row block by row block
    const int64_t kRows = 2048;
    std::vector<double> buf;
    for (int64_t r0 = 0; r0 < c->n; r0 += kRows) {
        const int64_t r1 = std::min<int64_t>(c->n, r0 + kRows);
        const int64_t lo = packed_off(std::max<int64_t>(r0, 1)), hi = packed_off(r1);
        buf.resize((size_t)std::max<int64_t>(hi - lo, 1));
        for (int64_t i = std::max<int64_t>(r0, 1); i < r1; ++i)
            std::memcpy(buf.data() + (packed_off(i) - lo), y + i * ld, i * sizeof(double));
        mds_status st = set_rows_host(c, r0, r1, buf.data());
        if (st) return st;
    }
    return MDS_OK;
}

mds_status mds_set_locations(mds_ctx c, const double* x) {
    GUARD(c);
    if (!x) return fail(c, MDS_E_INVALID_ARG, "NULL locations");
    const int64_t m = c->n * c->d;
    for (int64_t q = 0; q < m; ++q)
        if (!std::isfinite(x[q])) return fail(c, MDS_E_INVALID_ARG, "locations must be finite");
    CK(cudaMemcpyAsync(c->d_x, x, m * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->x_set = true;
    ++c->version;
    return MDS_OK;
}

mds_status mds_set_locations_device(mds_ctx c, const double* x_dev) {
    GUARD(c);
    if (!x_dev) return fail(c, MDS_E_INVALID_ARG, "NULL locations");
    CK(cudaMemcpyAsync(c->d_x, x_dev, c->n * c->d * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    c->x_set = true;
    ++c->version;
    return MDS_OK;
}

mds_status mds_set_sigma(mds_ctx c, double sigma) {
    GUARD(c);
    if (!(sigma > 0.0) || !std::isfinite(sigma)) return fail(c, MDS_E_INVALID_ARG, "sigma must be > 0 and finite");
    const double pi = 3.14159265358979323846;
    c->sigma = sigma;
    SigmaParams& P = c->P;
    P.inv_sigma = 1.0 / sigma;
    P.inv_sigma2 = 1.0 / (sigma * sigma);
    P.half_inv_sigma2 = 0.5 / (sigma * sigma);
    P.k0 = -0.5 * std::log(2.0 * pi * sigma * sigma);
    P.cg = 1.0 / (sigma * std::sqrt(2.0 * pi));
    P.inv_sigma_f = (float)P.inv_sigma;
    P.inv_sigma2_f = (float)P.inv_sigma2;
    P.half_inv_sigma2_f = (float)P.half_inv_sigma2;
    P.k0_f = (float)P.k0;
    P.cg_f = (float)P.cg;
    c->sigma_set = true;
    ++c->version;
    return MDS_OK;
}

mds_status mds_log_likelihood_and_gradient(mds_ctx c, double* loglik, double* grad) {
    GUARD(c);
    mds_status st = eval_internal(c);
    if (st) return st;
    if (loglik) CK(cudaMemcpyAsync(loglik, c->d_lik, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (grad) CK(cudaMemcpyAsync(grad, c->d_grad, c->n * c->d * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return MDS_OK;
}

mds_status mds_log_likelihood(mds_ctx c, double* loglik) {
    if (!loglik) return fail(c, MDS_E_INVALID_ARG, "NULL output");
    return mds_log_likelihood_and_gradient(c, loglik, nullptr);
}

mds_status mds_gradient(mds_ctx c, double* grad) {
    if (!grad) return fail(c, MDS_E_INVALID_ARG, "NULL output");
    return mds_log_likelihood_and_gradient(c, nullptr, grad);
}

mds_status mds_evaluate_device(mds_ctx c, double* loglik_dev, double* grad_dev) {
    GUARD(c);
    mds_status st = ready(c);
    if (st) return st;
    KickArgs kk{};
    st = run_pass<false>(c, grad_dev ? grad_dev : c->d_grad, loglik_dev ? loglik_dev : c->d_lik, kk, c->stream, true);
    if (st) return st;
    if (!grad_dev && !loglik_dev) c->eval_version = c->version;
    return MDS_OK;
}

mds_status mds_evaluate_partial_device(mds_ctx c, double* part_dev) {
    GUARD(c);
    if (!part_dev) return fail(c, MDS_E_INVALID_ARG, "NULL output");
    mds_status st = ready(c);
    if (st) return st;
    launch_x_convert(c, c->stream);
    launch_tile(c, c->stream);
    launch_reduce<false>(c, part_dev, part_dev + c->n * c->d, KickArgs{}, c->stream);
    CK(cudaGetLastError());
    return MDS_OK;
}

mds_status mds_set_allgather(mds_ctx c, mds_allgather_fn fn, void* user) {
    GUARD(c);
    c->ag_fn = fn;
    c->ag_user = user;
    return MDS_OK;
}

mds_status mds_get_locations(mds_ctx c, double* x) {
    GUARD(c);
    if (!x) return fail(c, MDS_E_INVALID_ARG, "NULL output");
    if (!c->x_set) return fail(c, MDS_E_STATE, "locations not set");
    CK(cudaMemcpyAsync(x, c->d_x, c->n * c->d * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return MDS_OK;
}

mds_status mds_get_momentum(mds_ctx c, double* p) {
    GUARD(c);
    if (!p) return fail(c, MDS_E_INVALID_ARG, "NULL output");
    if (!c->d_p) {
        std::memset(p, 0, c->n * c->d * sizeof(double));
        return MDS_OK;
    }
    CK(cudaMemcpyAsync(p, c->d_p, c->n * c->d * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return MDS_OK;
}

mds_status mds_combine_partials_device(mds_ctx c, const double* gathered_dev, int32_t world, double* loglik_dev,
                                       double* grad_dev) {
    GUARD(c);
    if (!gathered_dev || world < 1) return fail(c, MDS_E_INVALID_ARG, "bad gathered partials");
    const int64_t len = c->n * c->d + 1;
    combine_kernel<<<(unsigned)((len + 255) / 256), 256, 0, c->stream>>>(gathered_dev, world, len, grad_dev, loglik_dev);
    CK(cudaGetLastError());
    return MDS_OK;
}

mds_status mds_observed_pairs(mds_ctx c, int64_t* count) {
    GUARD(c);
    if (!count) return fail(c, MDS_E_INVALID_ARG, "NULL output");
    if (c->n_obs < 0) {
        CK(cudaMemsetAsync(c->d_count, 0, sizeof(unsigned long long), c->stream));
        const size_t cnt = (size_t)c->ntl * TB * TB;
        if (cnt) {
            if (c->prec == MDS_F64) count_obs_kernel<double><<<1184, 256, 0, c->stream>>>((const double*)c->d_y, cnt, c->d_count);
            else count_obs_kernel<float><<<1184, 256, 0, c->stream>>>((const float*)c->d_y, cnt, c->d_count);
            CK(cudaGetLastError());
        }
        unsigned long long h = 0;
        CK(cudaMemcpyAsync(&h, c->d_count, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        c->n_obs = (int64_t)h;
    }
    *count = c->n_obs;
    return MDS_OK;
}

mds_status mds_zero_distance_pairs(mds_ctx c, int64_t* count) {
    GUARD(c);
    if (!count) return fail(c, MDS_E_INVALID_ARG, "NULL output");
    mds_status st = ready(c);
    if (st) return st;
    CK(cudaMemsetAsync(c->d_count, 0, sizeof(unsigned long long), c->stream));
    if (c->ntl) {
        // fp64 X for both precisions: the diagnostic asks about the master X
        if (c->prec == MDS_F64) {
            switch (c->d) {
                case 1: zero_pairs_kernel<double, 1><<<c->ntl, 256, 0, c->stream>>>((const double*)c->d_y, c->d_x, c->d_tiles, c->d_count); break;
                case 2: zero_pairs_kernel<double, 2><<<c->ntl, 256, 0, c->stream>>>((const double*)c->d_y, c->d_x, c->d_tiles, c->d_count); break;
                case 3: zero_pairs_kernel<double, 3><<<c->ntl, 256, 0, c->stream>>>((const double*)c->d_y, c->d_x, c->d_tiles, c->d_count); break;
                case 4: zero_pairs_kernel<double, 4><<<c->ntl, 256, 0, c->stream>>>((const double*)c->d_y, c->d_x, c->d_tiles, c->d_count); break;
                case 5: zero_pairs_kernel<double, 5><<<c->ntl, 256, 0, c->stream>>>((const double*)c->d_y, c->d_x, c->d_tiles, c->d_count); break;
                case 6: zero_pairs_kernel<double, 6><<<c->ntl, 256, 0, c->stream>>>((const double*)c->d_y, c->d_x, c->d_tiles, c->d_count); break;
                case 7: zero_pairs_kernel<double, 7><<<c->ntl, 256, 0, c->stream>>>((const double*)c->d_y, c->d_x, c->d_tiles, c->d_count); break;
                default: zero_pairs_kernel<double, 8><<<c->ntl, 256, 0, c->stream>>>((const double*)c->d_y, c->d_x, c->d_tiles, c->d_count); break;
            }
        } else {
            launch_x_convert(c, c->stream);
            switch (c->d) {
                case 1: zero_pairs_kernel<float, 1><<<c->ntl, 256, 0, c->stream>>>((const float*)c->d_y, c->d_xf, c->d_tiles, c->d_count); break;
                case 2: zero_pairs_kernel<float, 2><<<c->ntl, 256, 0, c->stream>>>((const float*)c->d_y, c->d_xf, c->d_tiles, c->d_count); break;
                case 3: zero_pairs_kernel<float, 3><<<c->ntl, 256, 0, c->stream>>>((const float*)c->d_y, c->d_xf, c->d_tiles, c->d_count); break;
                case 4: zero_pairs_kernel<float, 4><<<c->ntl, 256, 0, c->stream>>>((const float*)c->d_y, c->d_xf, c->d_tiles, c->d_count); break;
                case 5: zero_pairs_kernel<float, 5><<<c->ntl, 256, 0, c->stream>>>((const float*)c->d_y, c->d_xf, c->d_tiles, c->d_count); break;
                case 6: zero_pairs_kernel<float, 6><<<c->ntl, 256, 0, c->stream>>>((const float*)c->d_y, c->d_xf, c->d_tiles, c->d_count); break;
                case 7: zero_pairs_kernel<float, 7><<<c->ntl, 256, 0, c->stream>>>((const float*)c->d_y, c->d_xf, c->d_tiles, c->d_count); break;
                default: zero_pairs_kernel<float, 8><<<c->ntl, 256, 0, c->stream>>>((const float*)c->d_y, c->d_xf, c->d_tiles, c->d_count); break;
            }
        }
        CK(cudaGetLastError());
    }
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, c->d_count, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    *count = (int64_t)h;
    return MDS_OK;
}

mds_status mds_set_timing(mds_ctx c, int32_t enable) {
    GUARD(c);
    c->timing = enable != 0;
    c->ev_used = 0;
    return MDS_OK;
}

mds_status mds_last_timing(mds_ctx c, float* pair_ms, float* reduce_ms) {
    GUARD(c);
    double sp = 0.0, sr = 0.0;
    const size_t passes = c->ev_used / 3;
    if (passes) CK(cudaEventSynchronize(c->evpool[3 * passes - 1]));
    for (size_t q = 0; q < passes; ++q) {
        float a = 0.f, b = 0.f;
        CK(cudaEventElapsedTime(&a, c->evpool[3 * q], c->evpool[3 * q + 1]));
        CK(cudaEventElapsedTime(&b, c->evpool[3 * q + 1], c->evpool[3 * q + 2]));
        sp += a;
        sr += b;
    }
    c->ev_used = 0;
    if (pair_ms) *pair_ms = passes ? (float)(sp / passes) : 0.f;
    if (reduce_ms) *reduce_ms = passes ? (float)(sr / passes) : 0.f;
    return MDS_OK;
}

const char* mds_last_error(mds_ctx c) { return c ? c->err.c_str() : ""; }

const char* mds_status_string(mds_status s) {
    switch (s) {
        case MDS_OK: return "ok";
        case MDS_E_INVALID_ARG: return "invalid argument";
        case MDS_E_STATE: return "invalid state";
        case MDS_E_OOM: return "out of device memory";
        case MDS_E_CUDA: return "CUDA error";
        case MDS_E_COMM: return "communication error";
        case MDS_E_UNSUPPORTED: return "unsupported";
    }
    return "unknown status";
}

const char* mds_version(void) { return kVersion; }

mds_status mds_device_info(int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return MDS_E_UNSUPPORTED;
    }
    int v = 0;
    if (sm_count && cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess) *sm_count = v;
    if (cc_major && cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMajor, dev) == cudaSuccess) *cc_major = v;
    if (cc_minor && cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMinor, dev) == cudaSuccess) *cc_minor = v;
    return MDS_OK;
}

mds_status mds_measure_fma_peaks(double* fp64, double* fp32) {
    mds_ctx c = nullptr;
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return MDS_E_UNSUPPORTED;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* d_out = nullptr;
    if (cudaMalloc(&d_out, 16) != cudaSuccess) return MDS_E_OOM;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int threads = 256, blocks = sms * 8, iters = 4096;
    float best64 = 1e30f, best32 = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(a);
        fma_peak_kernel<double><<<blocks, threads>>>(d_out, iters, 0.999999, 1e-9);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        if (rep) best64 = std::min(best64, ms);
        cudaEventRecord(a);
        fma_peak_kernel<float><<<blocks, threads>>>((float*)d_out, iters * 4, 0.999999f, 1e-9f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        if (rep) best32 = std::min(best32, ms);
    }
    cudaError_t e = cudaGetLastError();
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(d_out);
    if (e != cudaSuccess) return fail(c, MDS_E_CUDA, cudaGetErrorString(e));
    const double lanes = (double)blocks * threads * 64.0;
    if (fp64) *fp64 = lanes * iters / (best64 * 1e-3);
    if (fp32) *fp32 = lanes * iters * 4 / (best32 * 1e-3);
    return MDS_OK;
}

}  // extern "C"

#include "mds_hmc.inl"
