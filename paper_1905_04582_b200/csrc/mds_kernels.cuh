// mds_kernels.cuh -- sm_100a kernels of the fused MDS likelihood+gradient pass.
//
// Data layout in HBM:
//   Y  : the strict lower triangle cut into B x B tiles (I, J), I >= J, B = 64.
//        Only this rank's tiles are stored, back to back, tile-major; inside a
//        tile the layout is column-major, y(ii, jj) at [jj*B + ii], so a warp
//        whose lanes are consecutive rows ii reads one 256 B line per column.
//        Slots that are not an observed pair (missing y, i <= j in diagonal
//        tiles, padding rows/columns >= n) hold the canonical NaN, so the pair
//        loop has no bounds or i > j test.
//   X  : n_pad x D row-major, padding rows zero; fp64 master, fp32 copy for F32.
//   part: per local tile two B x D partial blocks (row role, column role), and
//        one log-likelihood partial per tile; a fixed-order reduction turns
//        them into g and log L (no atomics anywhere in the arithmetic).
//
// Pair kernel (one CTA = 4 warps per tile): warp (wr, wc) evaluates the 32 x 32
// sub-block rows wr*32.., columns wc*32..; lane = row.  Each lane keeps its
// row's gradient in registers (Alg. 2's per-row reduction),
// the column side of every pair (new: each unordered pair is computed once) is
// reduced across the 32 lanes with a 4-column reduce-scatter (2 halving steps
// + 3 butterflies), and the scalar log L is reduced warp -> CTA -> tile partial
// (Alg. 1's binary-tree reduction), all in a fixed order.
#pragma once
#include <cstdint>
#include "mds_math.cuh"

namespace mdsk {

constexpr int TB = 64;              // tile edge B
constexpr int TILE_THREADS = 128;   // 4 warps

template <typename T> struct Acc;   // accumulation type above the per-pair math
template <> struct Acc<double> { using type = double; };
template <> struct Acc<float> { using type = double; };

template <typename T>
__device__ __forceinline__ T ldg_nc(const T* p) { return __ldg(p); }

template <typename T, bool TRUNC> struct Pair;
template <bool TRUNC> struct Pair<double, TRUNC> {
    __device__ __forceinline__ static void eval(double s, double y, const SigmaParams& P, double& l, double& u) {
        pair_f64<TRUNC>(s, y, P, l, u);
    }
};
template <bool TRUNC> struct Pair<float, TRUNC> {
    __device__ __forceinline__ static void eval(float s, float y, const SigmaParams& P, float& l, float& u) {
        pair_f32<TRUNC>(s, y, P, l, u);
    }
};

template <typename T>
__device__ __forceinline__ T shfl_xor(T v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }

// Sum of 4 per-lane values a0..a3 over the 32 lanes; lane L ends with the total
// of column c = (L >> 3) & 3 (all 8 lanes of that group hold it).  Fixed order.
template <typename T>
__device__ __forceinline__ T reduce_scatter4(T a0, T a1, T a2, T a3, int lane) {
    const bool b4 = lane & 16, b3 = lane & 8;
    // xor 16: bit4 = 0 keeps columns {0,1}, bit4 = 1 keeps {2,3}
    T k0 = b4 ? a2 : a0, k1 = b4 ? a3 : a1;
    T s0 = b4 ? a0 : a2, s1 = b4 ? a1 : a3;
    k0 += shfl_xor(s0, 16);
    k1 += shfl_xor(s1, 16);
    // xor 8: bit3 = 0 keeps the first, bit3 = 1 the second
    T k = b3 ? k1 : k0;
    T sd = b3 ? k0 : k1;
    k += shfl_xor(sd, 8);
    k += shfl_xor(k, 4);
    k += shfl_xor(k, 2);
    k += shfl_xor(k, 1);
    return k;
}

struct TileArgs {
    const void* y;          // local tiles, [ntl][B][B] (column-major inside)
    const void* x;          // n_pad x D, compute precision
    const int* tiles;       // [ntl] (I << 16) | J
    double* part;           // [ntl][2][B][D]  (role 0 = rows I, role 1 = cols J)
    double* likpart;        // [ntl]
    SigmaParams P;
};

template <typename T, int D, bool TRUNC>
__global__ void __launch_bounds__(TILE_THREADS)
tile_kernel(TileArgs a) {
    using A = typename Acc<T>::type;
    __shared__ T xs[2][TB][D];
    __shared__ A rowacc[2][TB][D];   // [wc][row]
    __shared__ A colacc[2][TB][D];   // [wr][col]
    __shared__ A wlik[4];

    const int t = blockIdx.x;
    const int code = a.tiles[t];
    const int I = code >> 16, J = code & 0xffff;
    const T* __restrict__ X = static_cast<const T*>(a.x);
    for (int e = threadIdx.x; e < TB * D; e += TILE_THREADS) {
        xs[0][e / D][e % D] = X[(size_t)I * TB * D + e];
        xs[1][e / D][e % D] = X[(size_t)J * TB * D + e];
    }
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wr = warp & 1, wc = warp >> 1;
    const int ii = wr * 32 + lane;
    T xi[D];
#pragma unroll
    for (int k = 0; k < D; ++k) xi[k] = xs[0][ii][k];
    // per-sub-block accumulators (32 terms) in the compute precision; they are
    // widened to fp64 once per tile (reading R15 for the fp32 path)
    T gi[D];
#pragma unroll
    for (int k = 0; k < D; ++k) gi[k] = T(0);
    T lik = T(0);

    const T* __restrict__ ycol = static_cast<const T*>(a.y) + (size_t)t * TB * TB + (size_t)(wc * 32) * TB + ii;
    T ynext[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) ynext[q] = ldg_nc(ycol + q * TB);

#pragma unroll 1
    for (int g = 0; g < 8; ++g) {
        T yv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) yv[q] = ynext[q];
        if (g < 7) {
#pragma unroll
            for (int q = 0; q < 4; ++q) ynext[q] = ldg_nc(ycol + (4 * (g + 1) + q) * TB);
        }
        T v[4][D];
        T lsum = T(0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int jj = wc * 32 + 4 * g + q;
            T dl[D];
            T s = T(0);
#pragma unroll
            for (int k = 0; k < D; ++k) {
                dl[k] = xi[k] - xs[1][jj][k];
                s = fma(dl[k], dl[k], s);
            }
            T l, u;
            Pair<T, TRUNC>::eval(s, yv[q], a.P, l, u);
            const bool miss = is_missing(yv[q]);
            l = miss ? T(0) : l;
            u = miss ? T(0) : u;
            lsum += l;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                v[q][k] = u * dl[k];
                gi[k] -= v[q][k];
            }
        }
        lik += lsum;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            T cs = reduce_scatter4(v[0][k], v[1][k], v[2][k], v[3][k], lane);
            if ((lane & 7) == 0) colacc[wr][wc * 32 + 4 * g + (lane >> 3)][k] = A(cs);
        }
    }
#pragma unroll
    for (int k = 0; k < D; ++k) rowacc[wc][ii][k] = A(gi[k]);
    // warp-level tree for log L, fixed order
    A likw = A(lik);
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) likw += __shfl_xor_sync(0xffffffffu, likw, m);
    if (lane == 0) wlik[warp] = likw;
    __syncthreads();

    double* __restrict__ prow = a.part + (size_t)t * 2 * TB * D;
    double* __restrict__ pcol = prow + TB * D;
    for (int e = threadIdx.x; e < TB * D; e += TILE_THREADS) {
        const int r = e / D, k = e % D;
        prow[e] = rowacc[0][r][k] + rowacc[1][r][k];
        pcol[e] = colacc[0][r][k] + colacc[1][r][k];
    }
    if (threadIdx.x == 0) a.likpart[t] = (wlik[0] + wlik[1]) + (wlik[2] + wlik[3]);
}

// ------------------------------------------------------------ reduction
// g[i][k] = sum over this rank's entries touching block b = i / B, in the fixed
// order of blk_ent (row-role tiles by J, then column-role tiles by I').  A
// block of RED_SEG warps covers 32 consecutive (ii, k) elements; warp w sums
// entries w, w + RED_SEG, ...; the RED_SEG partials are added in warp order.
constexpr int RED_SEG = 8;

struct KickArgs {
    double* p;          // momentum n x D (updated: p += half_eps * (g + prior grad))
    double* gl;         // out: grad log pi (n x D)
    const double* x;    // positions (n_pad x D)
    double half_eps;
    double inv_tau2;    // 1/tau^2 or 0
};

template <bool KICK>
__global__ void __launch_bounds__(32 * RED_SEG)
reduce_kernel(const double* __restrict__ part, const double* __restrict__ likpart,
              const int* __restrict__ blk_ptr, const int* __restrict__ blk_ent,
              int64_t n, int D, int ntl, double* __restrict__ grad_out, double* __restrict__ lik_out,
              KickArgs kk) {
    __shared__ double red[RED_SEG][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t nd = n * D;
    const int64_t nelem_blocks = (nd + 31) / 32;
    if ((int64_t)blockIdx.x == nelem_blocks) {
        // log L: fixed-order strided partial sums + tree
        double s = 0.0;
        for (int q = threadIdx.x; q < ntl; q += blockDim.x) s += likpart[q];
        __shared__ double lr[32 * RED_SEG];
        lr[threadIdx.x] = s;
        __syncthreads();
        for (int m = blockDim.x / 2; m >= 1; m >>= 1) {
            if (threadIdx.x < m) lr[threadIdx.x] += lr[threadIdx.x + m];
            __syncthreads();
        }
        if (threadIdx.x == 0 && lik_out) *lik_out = lr[0];
        return;
    }
    const int64_t e = (int64_t)blockIdx.x * 32 + lane;
    double acc = 0.0;
    int64_t i = 0, b = 0, within = 0;
    if (e < nd) {
        i = e / D;
        b = i / TB;
        within = e - b * TB * D;          // (ii * D + k) inside the block's B x D slab
        const int e0 = blk_ptr[b], e1 = blk_ptr[b + 1];
        int q = e0 + w;
#pragma unroll 4
        for (; q < e1; q += RED_SEG) acc += part[(size_t)blk_ent[q] * TB * D + within];
    }
    red[w][lane] = acc;
    __syncthreads();
    if (w == 0 && e < nd) {
        double s = red[0][lane];
#pragma unroll
        for (int k = 1; k < RED_SEG; ++k) s += red[k][lane];
        if (grad_out) grad_out[e] = s;
        if (KICK) {
            const double gl = s - kk.x[e] * kk.inv_tau2;
            kk.gl[e] = gl;
            kk.p[e] += kk.half_eps * gl;
        }
    }
}

// ------------------------------------------------------------ Y packing
struct PackArgs {
    const double* src;      // packed rows [i0, i1), starting with y_{i0,0}
    int64_t i0, i1;
    int64_t src_base;       // packed offset of row i0
    const int* row_local;   // [nb] local tile-row start (tile index of (I, 0)) or -1
    void* dst;              // tiles
    int* bad;               // set to 1 on y < 0 or +-inf
};

template <typename T>
__global__ void pack_rows_kernel(PackArgs a) {
    const int64_t i = a.i0 + blockIdx.x;
    if (i >= a.i1 || i < 1) return;
    const int64_t I = i / TB, ii = i % TB;
    const int lt = a.row_local[I];
    if (lt < 0) return;                                   // tile-row not owned by this rank
    const double* row = a.src + (i * (i - 1) / 2 - a.src_base);
    T* dst = static_cast<T*>(a.dst);
    for (int64_t j = threadIdx.x; j < i; j += blockDim.x) {
        double y = row[j];
        T v;
        if (y != y) {
            if (sizeof(T) == 8) v = (T)__hiloint2double((int)CANON_NAN_HI64, 0);
            else v = (T)__int_as_float((int)CANON_NAN_F32);
        } else {
            if (y < 0.0 || y == __longlong_as_double(0x7ff0000000000000LL)) { *a.bad = 1; continue; }
            v = (T)y;
        }
        const int64_t J = j / TB, jj = j % TB;
        dst[(size_t)(lt + J) * TB * TB + jj * TB + ii] = v;
    }
}

template <typename T>
__global__ void fill_nan_kernel(T* p, size_t count) {
    size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    T nanv;
    if (sizeof(T) == 8) nanv = (T)__hiloint2double((int)CANON_NAN_HI64, 0);
    else nanv = (T)__int_as_float((int)CANON_NAN_F32);
    for (; k < count; k += stride) p[k] = nanv;
}

// count observed (non-canonical-NaN) slots of the local tiles
template <typename T>
__global__ void count_obs_kernel(const T* __restrict__ y, size_t count, unsigned long long* out) {
    size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    unsigned long long c = 0;
    for (; k < count; k += stride) c += is_missing(y[k]) ? 0 : 1;
    for (int m = 16; m >= 1; m >>= 1) c += __shfl_xor_sync(0xffffffffu, c, m);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// observed pairs at distance exactly 0 (diagnostic, reading R10)
template <typename T, int D>
__global__ void zero_pairs_kernel(const T* __restrict__ y, const T* __restrict__ X, const int* tiles,
                                  unsigned long long* out) {
    const int t = blockIdx.x;
    const int I = tiles[t] >> 16, J = tiles[t] & 0xffff;
    unsigned long long c = 0;
    for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) {
        const int jj = e / TB, ii = e % TB;
        const T yv = y[(size_t)t * TB * TB + e];
        if (is_missing(yv)) continue;
        T s = 0;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            T dl = X[((size_t)I * TB + ii) * D + k] - X[((size_t)J * TB + jj) * D + k];
            s += dl * dl;
        }
        c += (s == T(0)) ? 1 : 0;
    }
    for (int m = 16; m >= 1; m >>= 1) c += __shfl_xor_sync(0xffffffffu, c, m);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// ------------------------------------------------------------ X / HMC helpers
__global__ void to_f32_kernel(const double* __restrict__ x, float* __restrict__ xf, int64_t m) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < m) xf[k] = (float)x[k];
}

// leapfrog first half: p += half_eps * gl; x += eps * p   (rows < n only)
__global__ void kick_drift_kernel(double* __restrict__ x, double* __restrict__ p, const double* __restrict__ gl,
                                  int64_t m, double half_eps, double eps) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < m) {
        const double pk = p[k] + half_eps * gl[k];
        p[k] = pk;
        x[k] = x[k] + eps * pk;
    }
}

// sharded second half-kick: gl = g - x / tau^2; p += half_eps * gl
__global__ void kick_kernel(const double* __restrict__ g, const double* __restrict__ x, double* __restrict__ gl,
                            double* __restrict__ p, int64_t m, double half_eps, double inv_tau2) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < m) {
        const double v = g[k] - x[k] * inv_tau2;
        gl[k] = v;
        p[k] += half_eps * v;
    }
}

// gl = g - x / tau^2 (gradient of log pi) without a kick
__global__ void grad_logpi_kernel(const double* __restrict__ g, const double* __restrict__ x,
                                  double* __restrict__ gl, int64_t m, double inv_tau2) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < m) gl[k] = g[k] - x[k] * inv_tau2;
}

// H = -(loglik + prior(x)) + 1/2 p.p, fixed-order single-block reduction.
// out[0] = H, out[1] = loglik, out[2] = kinetic
__global__ void hamiltonian_kernel(const double* __restrict__ x, const double* __restrict__ p,
                                   const double* __restrict__ loglik, int64_t m, double inv_tau2,
                                   double* __restrict__ out) {
    __shared__ double sp[1024], sk[1024];
    double a = 0.0, kin = 0.0;
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
        a += x[k] * x[k];
        kin += p[k] * p[k];
    }
    sp[threadIdx.x] = a;
    sk[threadIdx.x] = kin;
    __syncthreads();
    for (int s = blockDim.x / 2; s >= 1; s >>= 1) {
        if (threadIdx.x < s) {
            sp[threadIdx.x] += sp[threadIdx.x + s];
            sk[threadIdx.x] += sk[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double prior = -0.5 * sp[0] * inv_tau2;
        const double K = 0.5 * sk[0];
        out[0] = -(loglik[0] + prior) + K;
        out[1] = loglik[0];
        out[2] = K;
    }
}

// rank-ordered sum of gathered partials: out[e] = sum_r gathered[r][e]
__global__ void combine_kernel(const double* __restrict__ gathered, int world, int64_t len,
                               double* __restrict__ grad_out, double* __restrict__ lik_out) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= len) return;
    double s = 0.0;
    for (int r = 0; r < world; ++r) s += gathered[(size_t)r * len + e];
    if (e < len - 1) { if (grad_out) grad_out[e] = s; }
    else if (lik_out) *lik_out = s;
}

// ------------------------------------------------------------ FMA peak probe
template <typename T>
__global__ void fma_peak_kernel(T* out, int iters, T a, T b) {
    T r0 = threadIdx.x * T(1e-7), r1 = r0 + T(1), r2 = r0 + T(2), r3 = r0 + T(3);
    T r4 = r0 + T(4), r5 = r0 + T(5), r6 = r0 + T(6), r7 = r0 + T(7);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            r0 = fma(r0, a, b); r1 = fma(r1, a, b); r2 = fma(r2, a, b); r3 = fma(r3, a, b);
            r4 = fma(r4, a, b); r5 = fma(r5, a, b); r6 = fma(r6, a, b); r7 = fma(r7, a, b);
        }
    }
    T s = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
    if (s == T(12345.678)) out[0] = s;   // keep the chains alive
}

}  // namespace mdsk
