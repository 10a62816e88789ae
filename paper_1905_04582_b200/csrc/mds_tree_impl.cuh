// mds_tree_impl.cuh -- device code of the tree-prior walk (see mds_tree.cuh),
// shared by the standalone kernel (mds_tree.cu) and the pass kernel, whose last
// CTA runs it during phase A when a tree prior is set (mds_pass.cuh).
#pragma once
#include <cuda_runtime.h>
#include "mds_tree.cuh"
#include "mds_math.cuh"

namespace mdsk {
namespace treek {


constexpr double LOG_2PI = 1.8378770664093454836;

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

// static operands of one post-order entry (one node): ids, branch lengths, tip x,
// the node's own branch length and its slot in its parent's pre-order entry
template <int D>
struct UpEnt {
    int4 e;
    double2 t;
    double tn;
    int pos;
    double x0[D], x1[D];
};
template <int D>
__device__ __forceinline__ void load_up(const TreeArgs& a, int e, UpEnt<D>& u) {
    // every operand indexed by the entry: one round of independent, coalesced loads
    u.e = a.up_e[e];
    u.t = a.up_t[e];
    u.tn = a.up_tn[e];
    u.pos = a.up_dpos[e];
    const double* xp = a.up_x + (size_t)e * 2 * D;
#pragma unroll
    for (int r = 0; r < D; ++r) {
        u.x0[r] = xp[r];
        u.x1[r] = xp[D + r];
    }
}

// static operands of one pre-order entry: ids, branch lengths, children's up messages
template <int D>
struct DnEnt {
    int4 e;
    double2 t;
    double s0[D + 1], s1[D + 1];   // (up mean, precision at the parent) of children 0 and 1
};
template <int D>
__device__ __forceinline__ void load_dn(const TreeArgs& a, int e, DnEnt<D>& u) {
    u.e = a.dn_e[e];
    u.t = a.dn_t[e];
    const double* sp = a.dn_sib + (size_t)e * 2 * (D + 1);
#pragma unroll
    for (int r = 0; r <= D; ++r) {
        u.s0[r] = sp[r];
        u.s1[r] = sp[D + 1 + r];
    }
}

// Post-order step: absorb the node's children contrast by contrast.
template <int D>
__device__ __forceinline__ void absorb(const TreeArgs& a, double* M, const UpEnt<D>& u) {
    const int n = a.n_items;
    const int slot = u.e.x, k = u.e.w;
    auto child = [&](int s, const double* xpre, double (&am)[D], double& av) {
        if (s < 0) {
#pragma unroll
            for (int r = 0; r < D; ++r) am[r] = xpre[r];
            av = 0.0;
        } else {
            const double* mc = M + (size_t)s * (D + 1);
#pragma unroll
            for (int r = 0; r < D; ++r) am[r] = mc[r];
            av = mc[D];
        }
    };
    double A[D], W, q = 0.0, wp = 1.0, lw = 0.0;
    {
        double av;
        child(u.e.y, u.x0, A, av);
        W = av + u.t.x;
    }
    for (int i = 1; i < k; ++i) {
        double am[D], av, tc;
        if (i == 1) {
            child(u.e.z, u.x1, am, av);
            tc = u.t.y;
        } else {
            const int c = a.ch_idx[a.ch_ptr[n + slot] + i];
            child(c < n ? -1 - c : c - n, a.x + (size_t)(c < n ? c : 0) * D, am, av);
            tc = a.t[c];
        }
        const double wi = av + tc;
        const double w = W + wi;
        const double rw = rcp_refined(w);
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
    double* mn = M + (size_t)slot * (D + 1);
#pragma unroll
    for (int r = 0; r < D; ++r) mn[r] = A[r];
    mn[D] = W;
    a.cq[n + slot] = -0.5 * q - 0.5 * (k - 1) * (D * LOG_2PI + a.logdet) - 0.5 * D * lw;
    a.cw[n + slot] = wp;
    // the node's up message as its parent's pre-order entry will read it
    const double p = rcp_refined(W + u.tn);
    a.pw[n + slot] = p;
#pragma unroll
    for (int r = 0; r < D; ++r) a.up_m[(size_t)slot * D + r] = A[r];
    if (u.pos >= 0) {
        double* sp = a.dn_sib + (size_t)u.pos * (D + 1);
#pragma unroll
        for (int r = 0; r < D; ++r) sp[r] = A[r];
        sp[D] = p;
    }
}

// child c's outside message from (P, Mm) -- the parent's outside message plus the
// siblings -- moved down c's branch; a tip gets its gradient
template <int D>
__device__ __forceinline__ void emit(const TreeArgs& a, double* M, int c, double tc, double P, const double (&Mm)[D]) {
    const int n = a.n_items;
    const double iv = rcp_refined(P);
    const double ovc = rcp_refined(iv + tc);
    if (c < n) {
        // d log p / d x_c = -Sigma^-1 (x_c - m_c) / v_c
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
}

// Pre-order step: every child's outside message
template <int D>
__device__ __forceinline__ void spread(const TreeArgs& a, double* M, const DnEnt<D>& u) {
    const int n = a.n_items;
    const int slot = u.e.x, k = u.e.w;
    const double* mo = M + (size_t)slot * (D + 1);
    const double ovi = mo[D];
    double base[D];
#pragma unroll
    for (int r = 0; r < D; ++r) base[r] = mo[r] * ovi;
    if (k == 2) {                       // binary node: each child's sibling from the entry
        double M0[D], M1[D];
#pragma unroll
        for (int r = 0; r < D; ++r) {
            M0[r] = fma(u.s1[r], u.s1[D], base[r]);
            M1[r] = fma(u.s0[r], u.s0[D], base[r]);
        }
        emit<D>(a, M, u.e.y, u.t.x, ovi + u.s1[D], M0);
        emit<D>(a, M, u.e.z, u.t.y, ovi + u.s0[D], M1);
    } else if (k == 1) {
        emit<D>(a, M, u.e.y, u.t.x, ovi, base);
    } else {
        const int c0 = a.ch_ptr[n + slot];
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
                    Mm[r] = fma(sb < n ? a.x[(int64_t)sb * D + r] : a.up_m[(size_t)(sb - n) * D + r], ps, Mm[r]);
            }
            emit<D>(a, M, c, a.t[c], P, Mm);
        }
    }
}


// Every tip-side operand, for items [i_lo, i_hi) (coalesced reads, scattered
// stores nothing waits on): x into the parent's post-order entry; (x, 1/t) into
// the parent's pre-order entry; the tip's precision and its (empty)
// contributions.  8 tips per thread per round: loads in flight first.
template <int D>
__device__ __forceinline__ void tips_pass(const TreeArgs& a, int i_lo, int i_hi, int tid, int nt) {
    for (int i0 = i_lo + tid; i0 < i_hi; i0 += 8 * nt) {
        int pos[8], dps[8];
        double xv[8][D], tv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * nt;
            pos[u] = i < i_hi ? a.tip_upos[i] : -1;
            dps[u] = i < i_hi ? a.dn_pos[i] : -1;
            tv[u] = i < i_hi ? a.t[i] : 1.0;
#pragma unroll
            for (int r = 0; r < D; ++r) xv[u][r] = i < i_hi ? a.x[(int64_t)i * D + r] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * nt;
            if (i >= i_hi) break;
            const double p = rcp_refined(tv[u]);
            a.pw[i] = p;
            a.cq[i] = 0.0;
            a.cw[i] = 1.0;
            if (pos[u] >= 0) {
#pragma unroll
                for (int r = 0; r < D; ++r) a.up_x[(size_t)pos[u] * D + r] = xv[u][r];
            }
            if (dps[u] >= 0) {
                double* sp = a.dn_sib + (size_t)dps[u] * (D + 1);
#pragma unroll
                for (int r = 0; r < D; ++r) sp[r] = xv[u][r];
                sp[D] = p;
            }
        }
    }
}

// The first post-order level (height 1: every child a tip) for entries
// [e_lo, e_hi), with the tips' x gathered straight from X, messages into the
// global buffer a.msg.  Inside the pass kernel the pair CTAs run one slice each
// at launch, so the walk starts at level 2.
template <int D>
__device__ __forceinline__ void level0_slice(const TreeArgs& a, int e_lo, int e_hi, int tid, int nt) {
    for (int e = e_lo + tid; e < e_hi; e += nt) {
        UpEnt<D> u;
        u.e = a.up_e[e];
        u.t = a.up_t[e];
        u.tn = a.up_tn[e];
        u.pos = a.up_dpos[e];
        const int s0 = u.e.y, s1 = u.e.z;
#pragma unroll
        for (int r = 0; r < D; ++r) {
            u.x0[r] = a.x[(int64_t)(-1 - s0) * D + r];
            u.x1[r] = u.e.w >= 2 ? a.x[(int64_t)(-1 - s1) * D + r] : 0.0;
        }
        absorb<D>(a, a.msg, u);
    }
}

// The whole walk on one CTA of NT threads.  dyn: the internal-node messages
// when a.smem != 0 (else a.msg is used); red: NT / 32 + 1 doubles of scratch.
template <int D, int NT>
__device__ __forceinline__ void tree_prior_block(const TreeArgs& a, double* dyn, double* red) {
    const int tid = threadIdx.x;
    const int n = a.n_items;
    // internal-node messages: slot s = node - n; up pass (m[D], v), then down pass (m[D], 1/v)
    double* M = a.smem ? dyn : a.msg;
    stamp(a, 0);
    // The level walk is a chain of dependent loads: pull every static array into
    // L2 up front (one TMA bulk prefetch each), so the chain runs at L2 latency.
    if (tid == 0 && !(a.prof && a.prof[255] == 1)) {   // (profiling switch: prof[255] = 1 skips the prefetch)
        auto pf = [](const void* p, size_t bytes) {
            bytes &= ~(size_t)15;
            if (bytes)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"((unsigned)bytes) : "memory");
        };
        const int eu = a.up_lvl_ptr[a.n_up], ed = a.dn_lvl_ptr[a.n_dn];
        pf(a.up_e, (size_t)eu * sizeof(int4));
        pf(a.up_t, (size_t)eu * sizeof(double2));
        pf(a.dn_e, (size_t)ed * sizeof(int4));
        pf(a.dn_t, (size_t)ed * sizeof(double2));
        pf(a.up_tn, (size_t)eu * sizeof(double));
        pf(a.up_dpos, (size_t)eu * sizeof(int));
        pf(a.tip_upos, (size_t)n * sizeof(int));
        pf(a.t, (size_t)a.n_nodes * sizeof(double));
        pf(a.dn_pos, (size_t)a.n_nodes * sizeof(int));
        pf(a.x, (size_t)n * D * sizeof(double));
    }
    stamp(a, 98);
    if (!a.ext_tips) tips_pass<D>(a, 0, n, tid, NT);
    else {
        // the pass kernel's pair CTAs did the tips pass (one slice each) at launch:
        // wait until all have published theirs, then re-arm the counter
        if (tid == 0) {
            const unsigned want = (unsigned)a.ext_tips;
            while (atomicAdd(a.tips_done, 0u) < want) __nanosleep(200);
            __threadfence();
            atomicExch(a.tips_done, 0u);
        }
        __syncthreads();
        // ... and the first level (into a.msg): bring those messages into M
        if (M != a.msg && a.n_up > 0) {
            const int e0 = a.up_lvl_ptr[1];
            for (int e = tid; e < e0; e += NT) {
                const int sl = a.up_e[e].x;
#pragma unroll
                for (int r = 0; r <= D; ++r) M[(size_t)sl * (D + 1) + r] = __ldcg(a.msg + (size_t)sl * (D + 1) + r);
            }
        }
    }
    __syncthreads();
    stamp(a, 99);
    // Level loop with a one-ahead pipeline: the static operands of the next chunk
    // (same level, or the next level's first chunk) are loaded before working on
    // the current one; `sync` publishes the previous level's writes.
    auto run_levels = [&](auto ent, auto load, auto work, const int* ptr, int L0, int L1, int stride, int lane,
                          auto sync, int sbase) {
        if (L0 >= L1) return;
        auto nxt = ent;
        bool hn = ptr[L0] + lane < ptr[L0 + 1];
        if (hn) load(ptr[L0] + lane, nxt);
        for (int L = L0; L < L1; ++L) {
            const int e0 = ptr[L], e1 = ptr[L + 1];
            for (int eb = e0; eb < e1; eb += stride) {
                const auto cur = nxt;
                const bool hc = hn;
                if (eb + stride < e1) {
                    hn = eb + stride + lane < e1;
                    if (hn) load(eb + stride + lane, nxt);
                } else if (L + 1 < L1) {
                    hn = ptr[L + 1] + lane < ptr[L + 2];
                    if (hn) load(ptr[L + 1] + lane, nxt);
                }
                if (eb == e0) sync();
                if (hc) work(cur);
            }
            if (sbase >= 0 && sbase + L < 256) stamp(a, sbase + L);
        }
    };
    auto ld_up = [&](int e, UpEnt<D>& u) { load_up<D>(a, e, u); };
    auto wk_up = [&](const UpEnt<D>& u) { absorb<D>(a, M, u); };
    auto bar_cta = [] { __syncthreads(); };
    auto bar_warp = [] { __syncwarp(); };

    // ---- post-order (by height): wide levels on the CTA, narrow ones on warp 0
    const int L0 = a.ext_tips ? 1 : 0;      // level 0 came from the pair CTAs
    run_levels(UpEnt<D>{}, ld_up, wk_up, a.up_lvl_ptr, L0, a.up_narrow, NT, tid, bar_cta, 3);
    __syncthreads();
    stamp(a, 2);
    if (tid < 32)
        run_levels(UpEnt<D>{}, ld_up, wk_up, a.up_lvl_ptr, max(L0, a.up_narrow), a.n_up, 32, tid, bar_warp, 3);
    __syncthreads();
    stamp(a, 100);
    // roots: contrast against mu0 (variance v_root + tau_root); an unsequenced item
    // (a root tip) gets its gradient here
    for (int e = tid; e < a.n_roots; e += NT) {
        const int r = a.roots[e];
        double dl[D];
        const double v = r < n ? 0.0 : M[(size_t)(r - n) * (D + 1) + D];
#pragma unroll
        for (int q = 0; q < D; ++q)
            dl[q] = (r < n ? a.x[(int64_t)r * D + q] : a.up_m[(size_t)(r - n) * D + q]) - a.mu0[q];
        const double w = v + a.t[r];
        a.cq[r] += -0.5 * quad<D>(a.sinv, dl) / w - 0.5 * (D * LOG_2PI + a.logdet);
        a.cw[r] *= w;
        if (r < n) {
            const double iv = rcp_refined(a.t[r]);
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
    for (int e = tid; e < a.n_roots; e += NT) {
        const int r = a.roots[e];
        if (r < n) continue;
        double* mr = M + (size_t)(r - n) * (D + 1);
#pragma unroll
        for (int q = 0; q < D; ++q) mr[q] = a.mu0[q];
        mr[D] = rcp_refined(a.t[r]);
    }
    __syncthreads();
    stamp(a, 101);

    // ---- pre-order (by depth): narrow head levels on warp 0, then the wide ones
    auto ld_dn = [&](int e, DnEnt<D>& u) { load_dn<D>(a, e, u); };
    auto wk_dn = [&](const DnEnt<D>& u) { spread<D>(a, M, u); };
    if (tid < 32) run_levels(DnEnt<D>{}, ld_dn, wk_dn, a.dn_lvl_ptr, 0, a.dn_narrow, 32, tid, bar_warp, 102);
    __syncthreads();
    run_levels(DnEnt<D>{}, ld_dn, wk_dn, a.dn_lvl_ptr, a.dn_narrow, a.n_dn, NT, tid, bar_cta, 102);
    __syncthreads();
    stamp(a, 200);

    // log p: fixed-order sum of the node contributions (8 nodes per thread per
    // round: loads in flight, one log per product of 8 contrast variances when
    // that product is representable)
    double acc = 0.0;
    for (int k0 = tid; k0 < a.n_nodes; k0 += 8 * NT) {
        double qv[8], wv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = k0 + u * NT;
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
        double s = tid < NT / 32 ? red[tid] : 0.0;
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
        if (tid == 0) *a.logp = s;
    }
    stamp(a, 201);
}

}  // namespace treek
}  // namespace mdsk
