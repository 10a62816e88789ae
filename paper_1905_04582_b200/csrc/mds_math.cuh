// mds_math.cuh -- per-pair arithmetic of the fused MDS likelihood+gradient pass.
//
// For one unordered pair (i > j) with squared latent distance s = ||x_i-x_j||^2
// and observation y this computes
//   ell = -1/2 log(2 pi sigma^2) - (y - d)^2/(2 sigma^2) - T log Phi(t)   (Eq. 2)
//   u   = [ (d - y)/sigma^2 + T phi(t)/(sigma Phi(t)) ] / d               (Eq. 6)
// with d = sqrt(s), t = d/sigma, so that the pair adds -u (x_i - x_j) to g_i and
// +u (x_i - x_j) to g_j.  The pair's v = u (x_i - x_j) is formed by the caller.
//
// Device math, t >= 0 always on this path:
//   E'     = cg exp(-t^2/2), cg = 1/(sigma sqrt(2 pi)) -- one exp, argument from s
//            directly: 2^n [cg 2^(j/256)] p(r), 256-entry table in shared memory
//            (scaled by cg per launch), degree-4 p
//   Q      = 1 - Phi(t) = E' P'(d)/R'(d): erfcx(t/sqrt2)/2 as a weighted-minimax rational
//            of degree (6, 7) (positive coefficients; absolute error of Q <= 2e-17 + rounding)
//   1/Phi, Q/(2-Q) from ONE reciprocal of (R - EP)(2R - EP), EP = E' P' = Q R
//   log Phi = log1p(-Q) = -2 atanh(Q/(2-Q))        -- degree-6 polynomial in z = (Q/(2-Q))^2
//            <= 1/9; absolute error <= 1.8e-12 (log Phi enters log L only: DESIGN.md R32)
//   phi/(sigma Phi) = E' / Phi                     -- shares E' with Q
// The reciprocal and rsqrt seeds come from MUFU (rcp/rsqrt.approx) refined by one
// cubic Newton step.  About 65 FP64 instructions per pair of math (+ ~8 for the
// distance and the sums, D = 2) instead of ~160 for libdevice erfc/log1p/exp/div.
#pragma once
#include <cstdint>
#include "mds_coeffs.h"

namespace mdsk {

// Per-sigma constants, passed by value as kernel parameters (constant bank).
struct SigmaParams {
    double inv_sigma;        // 1/sigma
    double inv_sigma2;       // 1/sigma^2
    double half_inv_sigma2;  // 1/(2 sigma^2)
    double k0;               // -1/2 log(2 pi sigma^2)
    double cg;               // 1/(sigma sqrt(2 pi))
    double qp[QP64_DEG + 1]; // P_j / (cg sigma^j): Q = E' P'(d) / R'(d) with E' = cg E (exp table scaled
    double qr[QR64_DEG + 1]; // R_j / sigma^j      by cg), in d directly: no t = d/sigma multiply
    int dclamp_hi;           // high word of TCLAMP64 sigma: d clamped there before P', R'
    int pad_;
    float inv_sigma_f, inv_sigma2_f, half_inv_sigma2_f, k0_f, cg_f;
    float ex2_slope_f;               // -log2(e) / (2 sigma^2): e^{-t^2/2} = 2^(s ex2_slope)
};

// Canonical NaN marks every non-pair slot of the tiled triangle (missing y,
// i <= j in diagonal tiles, padding).  Tested by its high word only.
constexpr uint32_t CANON_NAN_HI64 = 0x7FF80000u;
constexpr uint32_t CANON_NAN_F32 = 0x7FC00000u;

__device__ __forceinline__ double rsqrt_seed(double x) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    return r;
}
__device__ __forceinline__ double rcp_seed(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    return r;
}
__device__ __forceinline__ float rsqrt_f(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float rcp_f(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float ex2_f(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float lg2_f(float x) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// 1/x to ~1 ulp: MUFU seed (~20 bits) + one cubic Newton step (3 DFMA).
__device__ __forceinline__ double rcp_refined(double x) {
    double y0 = rcp_seed(x);
    double e = fma(-x, y0, 1.0);
    double ee = fma(e, e, e);
    return fma(ee, y0, y0);
}

template <int DEG, typename T>
__device__ __forceinline__ T horner(const T* c, T x) {
    T p = c[DEG];
#pragma unroll
    for (int k = DEG - 1; k >= 0; --k) p = fma(p, x, c[k]);
    return p;
}

// the per-launch exp table of pair_f64_n: cg 2^(j/256), j < EXPT64_N (call with
// every thread of the block, then __syncthreads)
__device__ __forceinline__ void build_exptab(double* tab, const SigmaParams& P) {
    for (int j = threadIdx.x; j < EXPT64_N; j += blockDim.x) tab[j] = EXPT64_TAB[j] * P.cg;
}

__device__ __forceinline__ bool is_missing(double y) {
    return (uint32_t)__double2hiint(y) == CANON_NAN_HI64;
}
__device__ __forceinline__ bool is_missing(float y) {
    return (uint32_t)__float_as_uint(y) == CANON_NAN_F32;
}

// ---------------------------------------------------------------- fp64 pairs
// NP independent pairs in lock-step: every step is issued for all NP pairs
// before the next, so the FP64 dependency chains (Horner steps, Newton steps)
// of different pairs interleave in the instruction stream and hide the DFMA
// latency (a single pair is one long dependent chain).
// WL: form ell (the Eq. 2 term); WG: form u (the Eq. 6 coefficient / d).  The
// pass variants that need only one of them (gradient-only leapfrog steps,
// likelihood-only sigma sweeps) drop the other's work:
//   WL && WG : one reciprocal of Phi (2 - Q) gives 1/Phi and 1/(2 - Q)
//   WG only  : 1/Phi alone (no atanh series)
//   WL only  : 1/(2 - Q) alone (no phi/Phi)
// ACC: ell is in/out -- the term WITHOUT the constant -1/2 log(2 pi sigma^2) is
// added to the incoming value (the caller's running sum), the constant being
// added once per observed pair count at the end (one FP64 add per pair less).
template <bool TRUNC, int NP, bool WL = true, bool WG = true, bool ACC = false>
__device__ __forceinline__ void pair_f64_n(const double (&s)[NP], const double (&y)[NP], const SigmaParams& P,
                                           const double* __restrict__ exptab, double (&ell)[NP], double (&u)[NP]) {
    double rs[NP], d[NP], res[NP], l[NP];
#pragma unroll
    for (int i = 0; i < NP; ++i) {
#ifndef MDS_NO_TRIM
        // the MUFU seed reads the high word only: clamp just that (s = 0, a coincident
        // pair, then gives a finite rs and d = s rs = 0 exactly; reading R10), and run
        // the Newton step on s itself (no register pair to rebuild)
        rs[i] = rsqrt_seed(__hiloint2double(max(__double2hiint(s[i]), 0x01000000), 0));
        const double sc = s[i];
#else
        const double sc = __hiloint2double(max(__double2hiint(s[i]), 0x01000000), __double2loint(s[i]));
        rs[i] = rsqrt_seed(sc);
#endif
        const double h = sc * rs[i];
        const double e = fma(-h, rs[i], 1.0);
        const double c = fma(e, 0.375, 0.5);
        const double re = rs[i] * e;
        rs[i] = fma(re, c, rs[i]);
    }
#pragma unroll
    for (int i = 0; i < NP; ++i) {
        d[i] = s[i] * rs[i];
        res[i] = y[i] - d[i];
        if (WL) l[i] = fma(-(res[i] * P.half_inv_sigma2), res[i], ACC ? ell[i] : P.k0);
    }
    if (TRUNC) {
        // E' = cg exp(-a), a = t^2/2 = s/(2 sigma^2): k = rint(-256 a / ln2),
        // E' = 2^(k>>8) [cg 2^((k&255)/256)] p(r), |r| <= ln2/512 (cg-scaled table in
        // shared memory, built per launch; degree-4 polynomial)
        double r[NP], E[NP];
        int k[NP];
        const double MAGIC = 6755399441055744.0;   // 1.5 * 2^52
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            double a = s[i] * P.half_inv_sigma2;
            a = __hiloint2double(min(__double2hiint(a), 0x4085E000), __double2loint(a));   // a <= ~700
            const double kd = fma(a, -EXPT64_INV_STEP, MAGIC);                           // 256 / ln2
            k[i] = __double2loint(kd);
            const double fk = kd - MAGIC;
#ifndef MDS_NO_TRIM
            // one fused step with ln2/256 rounded to double (no Cody-Waite split): r is
            // off by |k| 9.1e-20, i.e. E' by |k| 9.1e-20 relative -- 1.5e-16 at t = 3,
            // 1.2e-15 at t = 8.3 where E' ~ 1e-15 cg (reading R35)
            r[i] = fma(fk, -EXPT64_STEP, -a);
#else
            r[i] = fma(fk, -EXPT64_STEP_HI, -a);                                          // ln2/256 hi
            r[i] = fma(fk, -EXPT64_STEP_LO, r[i]);                                        // ln2/256 lo
#endif
        }
        // Q = 1 - Phi(t) = E q(t), q = P/R a rational of degree (6, 7) in t with positive
        // coefficients (tools/gen_coeffs.py), evaluated in d with the 1/sigma^j folded
        // into the coefficients; d clamped at 38 sigma (beyond, E' underflows).  Two
        // independent Horner chains, no reciprocal for a transformed variable.
        double pp[NP], rr[NP], dc[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            dc[i] = __hiloint2double(min(__double2hiint(d[i]), P.dclamp_hi), __double2loint(d[i]));
            pp[i] = fma(P.qp[QP64_DEG], dc[i], P.qp[QP64_DEG - 1]);
            rr[i] = fma(P.qr[QR64_DEG], dc[i], P.qr[QR64_DEG - 1]);
        }
#pragma unroll
        for (int j = QR64_DEG - 2; j >= 0; --j)
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                rr[i] = fma(rr[i], dc[i], P.qr[j]);
                if (j <= QP64_DEG - 2) pp[i] = fma(pp[i], dc[i], P.qp[j]);
            }
        double p[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) p[i] = EXPT64_C[EXPT64_DEG];
#pragma unroll
        for (int j = EXPT64_DEG - 1; j >= 0; --j)
#pragma unroll
            for (int i = 0; i < NP; ++i) p[i] = fma(p[i], r[i], EXPT64_C[j]);
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            const double pt = p[i] * exptab[k[i] & (EXPT64_N - 1)];
            // 2^(k>>8) spliced into the exponent field.  pt carries cg, so for large
            // sigma (cg < 2^-13, sigma > ~3.3e3) and a near the clamp the biased
            // exponent would go <= 0 and wrap into the sign bit: clamp the high word
            // at 0 instead (one IMNMX), i.e. E' < 2^-1022 where the true E' is below
            // the normal range (reading R33: absolute error < 2^-1022 in E', and
            // < 2^-1023 sigma sqrt(2 pi) in Q, both far inside the tolerances)
            const int ehi = __double2hiint(pt) + (int)((unsigned)(k[i] >> 8) << 20);
            E[i] = __hiloint2double(max(ehi, 0), __double2loint(pt));
        }
        // With EP = E' P' = Q R:  1 - Q = (R - EP)/R,  2 - Q = (2R - EP)/R, so
        //   1/Phi = R / (R - EP),   Q/(2 - Q) = EP / (2R - EP)
        // and one refined reciprocal of their product gives both (no cancellation:
        // R - EP = R Phi >= R/2).  phi/(sigma Phi) = E'/Phi = E' R / (R - EP).
        double EP[NP], D1[NP], D2[NP], prod[NP], z0[NP], nG[NP], nS[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            EP[i] = E[i] * pp[i];
            D1[i] = rr[i] - EP[i];
            D2[i] = fma(2.0, rr[i], -EP[i]);
            prod[i] = (WL && WG) ? D1[i] * D2[i] : (WG ? D1[i] : D2[i]);
            z0[i] = rcp_seed(prod[i]);
            // numerators, formed while the reciprocal is in flight
            if (WG) nG[i] = WL ? (E[i] * rr[i]) * D2[i] : E[i] * rr[i];
            if (WL) nS[i] = WG ? EP[i] * D1[i] : EP[i];
        }
        double sa[NP], zz[NP], G[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            const double f1 = fma(-prod[i], z0[i], 1.0);
            const double f2 = fma(f1, f1, f1);
            const double rp = fma(f2, z0[i], z0[i]);
            if (WG) G[i] = nG[i] * rp;            // E'/Phi (E' carries cg)
            if (WL) {
                sa[i] = nS[i] * rp;               // Q/(2 - Q)
                zz[i] = sa[i] * sa[i];
            }
        }
        if (WL) {
            double at[NP];
#pragma unroll
            for (int i = 0; i < NP; ++i) at[i] = ATANH64_C[ATANH64_DEG];
#pragma unroll
            for (int j = ATANH64_DEG - 1; j >= 0; --j)
#pragma unroll
                for (int i = 0; i < NP; ++i) at[i] = fma(at[i], zz[i], ATANH64_C[j]);
#pragma unroll
            for (int i = 0; i < NP; ++i) ell[i] = fma(sa[i], at[i], l[i]);
        }
        if (WG) {
#pragma unroll
            for (int i = 0; i < NP; ++i) u[i] = fma(-res[i], P.inv_sigma2, G[i]) * rs[i];
        }
    } else {
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            if (WL) ell[i] = l[i];
            if (WG) u[i] = (-res[i] * P.inv_sigma2) * rs[i];
        }
    }
}

// ---------------------------------------------------------------- fp32 pair
// fp32 storage and per-pair math (reading R15); MUFU rsqrt/ex2/rcp/lg2.
template <bool TRUNC, bool WL = true, bool WG = true>
__device__ __forceinline__ void pair_f32(float s, float y, const SigmaParams& P,
                                         float& ell, float& u) {
    const float sc = fmaxf(s, 1e-30f);
    const float rs = rsqrt_f(sc);
    const float d = s * rs;
    const float res = y - d;
    float l = fmaf(-(res * P.half_inv_sigma2_f), res, P.k0_f);
    if (TRUNC) {
        // E = e^{-t^2/2} straight from s (the -log2(e)/(2 sigma^2) folded into one
        // multiplier), 1/(t + kappa) with t + kappa as one FFMA from d (N = 30000, D = 6
        // A/B: 319.5 -> 322.2 G pair-evals/s; also folding cg into the exponent and 1/cg
        // into per-sigma q coefficients cut one FMUL more but spilled at 128 registers:
        // 306 G)
        const float E = ex2_f(s * P.ex2_slope_f);
        const float rden = rcp_f(fmaf(d, P.inv_sigma_f, KAPPA32));
        const float w = fmaf(-2.0f * KAPPA32, rden, 1.0f);
        const float q = horner<Q32_DEG>(Q32_C, w);
        const float Q = E * q;
        const float Phi = 1.0f - Q;
        const float invPhi = rcp_f(Phi);
        const float G = (E * P.cg_f) * invPhi;
        if (WL) l = fmaf(-0.693147181f, lg2_f(Phi), l);      // - log Phi
        if (WG) u = fmaf(-res, P.inv_sigma2_f, G) * rs;
    } else {
        if (WG) u = (-res * P.inv_sigma2_f) * rs;
    }
    if (WL) ell = l;
}

}  // namespace mdsk
