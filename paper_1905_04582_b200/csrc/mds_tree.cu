// mds_tree.cu -- the Brownian-diffusion prior kernel (see mds_tree.cuh).
#include <cuda_runtime.h>
#include "mds_tree.cuh"

namespace mdsk {
namespace {

constexpr int TT = 512;
constexpr double LOG_2PI = 1.8378770664093454836;
constexpr int KP = 2;          // children whose static operands are prefetched (binary trees: all)

template <int D>
__device__ __forceinline__ double quad(const double* sinv, const double (&v)[D]) {
    double q = 0.0;
#pragma unroll
    for (int r = 0; r < D; ++r) {
        double w = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) w = fma(sinv[r * D + c], v[c], w);
        q = fma(v[r], w, q);
    }
    return q;
}

__device__ __forceinline__ void stamp(const TreeArgs& a, int slot) {
    if (a.prof && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        a.prof[slot] = t;
    }
}

template <int D>
__device__ __forceinline__ void level_sync(bool narrow) {
    if (narrow) __syncwarp();
    else __syncthreads();
}

template <int D>
__global__ void __launch_bounds__(TT, 1) tree_prior_kernel(TreeArgs a) {
    extern __shared__ __align__(16) double dyn[];
    __shared__ double red[TT / 32 + 1];
    const int tid = threadIdx.x;
    const int n = a.n_items;
    // internal-node messages: slot s = node - n; up pass (m[D], v), then down pass (m[D], 1/v)
    double* M = a.smem ? dyn : a.msg;
    stamp(a, 0);

    // ---- post-order (by height)
    auto up_level = [&](int L, bool narrow) {
        const int e0 = a.up_lvl_ptr[L], e1 = a.up_lvl_ptr[L + 1];
        const int stride = narrow ? 32 : TT;
        for (int eb = e0; eb < e1; eb += stride) {
            const int e = eb + tid;
            // static operands, before the barrier: ids, branch lengths, tip positions
            int nd = -1, c0 = 0, k = 0, kid[KP];
            double tk[KP], xk[KP][D];
            if (e < e1) {
                nd = a.up_lvl_nodes[e];
                c0 = a.ch_ptr[nd];
                k = a.ch_ptr[nd + 1] - c0;
#pragma unroll
                for (int i = 0; i < KP; ++i) {
                    kid[i] = i < k ? a.ch_idx[c0 + i] : 0;
                    tk[i] = i < k ? a.t[kid[i]] : 0.0;
#pragma unroll
                    for (int r = 0; r < D; ++r) xk[i][r] = (i < k && kid[i] < n) ? a.x[(int64_t)kid[i] * D + r] : 0.0;
                }
            }
            if (eb == e0) level_sync<D>(narrow);
            if (nd < 0) continue;
            // a child's up message: tips (x, 0) from the prefetch or x, internal nodes from M
            auto msg_of = [&](int c, const double* xpre, double (&am)[D], double& av) {
                if (c < n) {
#pragma unroll
                    for (int r = 0; r < D; ++r) am[r] = xpre ? xpre[r] : a.x[(int64_t)c * D + r];
                    av = 0.0;
                } else {
                    const double* mc = M + (size_t)(c - n) * (D + 1);
#pragma unroll
                    for (int r = 0; r < D; ++r) am[r] = mc[r];
                    av = mc[D];
                }
            };
            double A[D], W, q = 0.0, wp = 1.0, lw = 0.0;
            {
                double av;
                msg_of(kid[0], xk[0], A, av);
                W = av + tk[0];
            }
            for (int i = 1; i < k; ++i) {
                double am[D], av, tc;
                if (i == 1) {
                    msg_of(kid[1], xk[1], am, av);
                    tc = tk[1];
                } else {
                    const int c = a.ch_idx[c0 + i];
                    msg_of(c, nullptr, am, av);
                    tc = a.t[c];
                }
                const double wi = av + tc;
                const double w = W + wi;
                const double rw = 1.0 / w;
                double dl[D];
#pragma unroll
                for (int r = 0; r < D; ++r) dl[r] = am[r] - A[r];
                q = fma(quad<D>(a.sinv, dl), rw, q);
                wp *= w;
                if (!(wp > 1e-150 && wp < 1e150)) {     // many contrasts: fold the product into a log
                    lw += log(wp);
                    wp = 1.0;
                }
#pragma unroll
                for (int r = 0; r < D; ++r) A[r] = (wi * A[r] + W * am[r]) * rw;
                W = W * wi * rw;
            }
            double* mn = M + (size_t)(nd - n) * (D + 1);
#pragma unroll
            for (int r = 0; r < D; ++r) mn[r] = A[r];
            mn[D] = W;
            a.cq[nd] = -0.5 * q - 0.5 * (k - 1) * (D * LOG_2PI + a.logdet) - 0.5 * D * lw;
            a.cw[nd] = wp;
        }
    };
    for (int L = 0; L < a.up_narrow; ++L) {
        up_level(L, false);
        stamp(a, 1 + L);
    }
    __syncthreads();
    if (tid < 32)
        for (int L = a.up_narrow; L < a.n_up; ++L) {
            up_level(L, true);
            stamp(a, 1 + L);
        }
    __syncthreads();
    stamp(a, 100);

    // ---- between the passes (all nodes at once): global copy of the internal up
    // means, every up message's precision at its parent, tips' contributions
    const int nint = a.n_nodes - n;
    for (int s = tid; s < nint; s += TT) {
#pragma unroll
        for (int r = 0; r < D; ++r) a.up_m[(size_t)s * D + r] = M[(size_t)s * (D + 1) + r];
    }
    // (4 nodes per thread per round: independent loads and divisions in flight)
    for (int k0 = tid; k0 < a.n_nodes; k0 += 4 * TT) {
        double tt[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int k = k0 + u * TT;
            tt[u] = k < a.n_nodes ? a.t[k] : 1.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int k = k0 + u * TT;
            if (k >= a.n_nodes) break;
            const double v = k < n ? 0.0 : M[(size_t)(k - n) * (D + 1) + D];
            a.pw[k] = 1.0 / (v + tt[u]);
            if (k < n) {
                a.cq[k] = 0.0;
                a.cw[k] = 1.0;
            }
        }
    }
    __syncthreads();
    // roots: contrast against mu0 (variance v_root + tau_root); outside message (mu0, tau_root);
    // an unsequenced item (a root tip) gets its gradient here
    for (int e = tid; e < a.n_roots; e += TT) {
        const int r = a.roots[e];
        double um[D], dl[D];
        const double v = r < n ? 0.0 : M[(size_t)(r - n) * (D + 1) + D];
#pragma unroll
        for (int q = 0; q < D; ++q) {
            um[q] = r < n ? a.x[(int64_t)r * D + q] : a.up_m[(size_t)(r - n) * D + q];
            dl[q] = um[q] - a.mu0[q];
        }
        const double w = v + a.t[r];
        a.cq[r] += -0.5 * quad<D>(a.sinv, dl) / w - 0.5 * (D * LOG_2PI + a.logdet);
        a.cw[r] *= w;
        if (r < n) {
            const double iv = 1.0 / a.t[r];
#pragma unroll
            for (int q = 0; q < D; ++q) {
                double g = 0.0;
#pragma unroll
                for (int c = 0; c < D; ++c) g = fma(a.sinv[q * D + c], dl[c], g);
                a.grad[(int64_t)r * D + q] = -g * iv;
            }
        }
    }
    __syncthreads();   // the up messages in M are dead from here on: M now holds outside messages
    for (int e = tid; e < a.n_roots; e += TT) {
        const int r = a.roots[e];
        if (r < n) continue;
        double* mr = M + (size_t)(r - n) * (D + 1);
#pragma unroll
        for (int q = 0; q < D; ++q) mr[q] = a.mu0[q];
        mr[D] = 1.0 / a.t[r];
    }
    stamp(a, 101);

    // ---- pre-order (by depth): each child's outside message = the parent's outside
    // message combined with the siblings' up messages, moved down the child's branch
    auto dn_level = [&](int L, bool narrow) {
        const int e0 = a.dn_lvl_ptr[L], e1 = a.dn_lvl_ptr[L + 1];
        const int stride = narrow ? 32 : TT;
        for (int eb = e0; eb < e1; eb += stride) {
            const int e = eb + tid;
            // static operands: the children's ids, branch lengths, up means and precisions
            int nd = -1, c0 = 0, k = 0, kid[KP];
            double tk[KP], pk[KP], mk[KP][D];
            if (e < e1) {
                nd = a.dn_lvl_nodes[e];
                c0 = a.ch_ptr[nd];
                k = a.ch_ptr[nd + 1] - c0;
#pragma unroll
                for (int i = 0; i < KP; ++i) {
                    kid[i] = i < k ? a.ch_idx[c0 + i] : 0;
                    tk[i] = i < k ? a.t[kid[i]] : 0.0;
                    pk[i] = i < k ? a.pw[kid[i]] : 0.0;
#pragma unroll
                    for (int r = 0; r < D; ++r)
                        mk[i][r] = i >= k ? 0.0
                                          : (kid[i] < n ? a.x[(int64_t)kid[i] * D + r]
                                                        : a.up_m[(size_t)(kid[i] - n) * D + r]);
                }
            }
            level_sync<D>(narrow);    // the previous level's outside messages are published
            if (nd < 0) continue;
            const double* mo = M + (size_t)(nd - n) * (D + 1);
            const double ovi = mo[D];
            double base[D];
#pragma unroll
            for (int r = 0; r < D; ++r) base[r] = mo[r] * ovi;
            // child c's outside message from (P, Mm): the parent's outside plus its siblings
            auto emit = [&](int c, double tc, double P, const double (&Mm)[D]) {
                const double iv = 1.0 / P;
                const double ovc = 1.0 / (iv + tc);
                if (c < n) {
                    // tip: d log p / d x_c = -Sigma^-1 (x_c - m_c) / v_c
                    double rr[D];
#pragma unroll
                    for (int r = 0; r < D; ++r) rr[r] = a.x[(int64_t)c * D + r] - Mm[r] * iv;
#pragma unroll
                    for (int qq = 0; qq < D; ++qq) {
                        double g = 0.0;
#pragma unroll
                        for (int cc = 0; cc < D; ++cc) g = fma(a.sinv[qq * D + cc], rr[cc], g);
                        a.grad[(int64_t)c * D + qq] = -g * ovc;
                    }
                } else {
                    double* mc = M + (size_t)(c - n) * (D + 1);
#pragma unroll
                    for (int r = 0; r < D; ++r) mc[r] = Mm[r] * iv;
                    mc[D] = ovc;
                }
            };
            if (k == 2) {                       // binary node: siblings from the prefetch
                double M0[D], M1[D];
#pragma unroll
                for (int r = 0; r < D; ++r) {
                    M0[r] = fma(mk[1][r], pk[1], base[r]);
                    M1[r] = fma(mk[0][r], pk[0], base[r]);
                }
                emit(kid[0], tk[0], ovi + pk[1], M0);
                emit(kid[1], tk[1], ovi + pk[0], M1);
            } else {
                for (int i = 0; i < k; ++i) {
                    const int c = a.ch_idx[c0 + i];
                    double P = ovi, Mm[D];
#pragma unroll
                    for (int r = 0; r < D; ++r) Mm[r] = base[r];
                    for (int j = 0; j < k; ++j) {
                        if (j == i) continue;
                        const int sb = a.ch_idx[c0 + j];
                        const double ps = a.pw[sb];
                        P += ps;
#pragma unroll
                        for (int r = 0; r < D; ++r)
                            Mm[r] = fma(sb < n ? a.x[(int64_t)sb * D + r] : a.up_m[(size_t)(sb - n) * D + r], ps,
                                        Mm[r]);
                    }
                    emit(c, a.t[c], P, Mm);
                }
            }
        }
    };
    __syncthreads();
    if (tid < 32)
        for (int L = 0; L < a.dn_narrow; ++L) {
            dn_level(L, true);
            stamp(a, 102 + L);
        }
    __syncthreads();
    for (int L = a.dn_narrow; L < a.n_dn; ++L) {
        dn_level(L, false);
        stamp(a, 102 + L);
    }
    __syncthreads();
    stamp(a, 200);

    // log p: fixed-order sum of the node contributions (logs of the contrast variances here)
    // (8 nodes per thread per round: loads in flight, one log per product of 8
    // contrast variances when that product is representable)
    double acc = 0.0;
    for (int k0 = tid; k0 < a.n_nodes; k0 += 8 * TT) {
        double qv[8], wv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = k0 + u * TT;
            qv[u] = k < a.n_nodes ? a.cq[k] : 0.0;
            wv[u] = k < a.n_nodes ? a.cw[k] : 1.0;
        }
        double qs = 0.0, wpr = 1.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            qs += qv[u];
            wpr *= wv[u];
        }
        if (wpr > 1e-300 && wpr < 1e300) {
            acc += qs - 0.5 * D * log(wpr);
        } else {                      // high-arity nodes carry folded products: one log each
            double ls = 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u) ls += log(wv[u]);
            acc += qs - 0.5 * D * ls;
        }
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
    if ((tid & 31) == 0) red[tid >> 5] = acc;
    __syncthreads();
    if (tid < 32) {
        double s = tid < TT / 32 ? red[tid] : 0.0;
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
        if (tid == 0) *a.logp = s;
    }
    stamp(a, 201);
}

template <int D>
void launch(const TreeArgs& a, cudaStream_t s) {
    static size_t set = 0;
    if (a.smem > set) {
        cudaFuncSetAttribute(tree_prior_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)a.smem);
        set = a.smem;
    }
    tree_prior_kernel<D><<<1, TT, a.smem, s>>>(a);
}

}  // namespace

void tree_prior_launch(const TreeArgs& a, int d, cudaStream_t s) {
    switch (d) {
        case 1: launch<1>(a, s); break;
        case 2: launch<2>(a, s); break;
        case 3: launch<3>(a, s); break;
        case 4: launch<4>(a, s); break;
        case 5: launch<5>(a, s); break;
        case 6: launch<6>(a, s); break;
        case 7: launch<7>(a, s); break;
        default: launch<8>(a, s); break;
    }
}

}  // namespace mdsk
