#!/usr/bin/env python
"""Generate the polynomial coefficients of the device special functions.

Product-side tool (never imports oracle/).  Writes
paper_1905_04582_b200/csrc/mds_coeffs.h.  Each table is a weighted minimax
fit (Lawson iteratively-reweighted least squares at 50 digits) of:

  EXP_C   : e^r on r in [-ln2/2, ln2/2], relative error            (fp64, deg 10)
  Q_C     : q(t) = Q(t) e^{t^2/2} = erfcx(t/sqrt2)/2 as a polynomial in
            w = (t - KAPPA)/(t + KAPPA), weighted by E(t) = e^{-t^2/2} so the
            fitted quantity is the ABSOLUTE error of Q(t) = 1 - Phi(t)      (fp64)
  ATANH_C : 2 atanh(sqrt z)/sqrt z on z in [0, 1/9], relative error     (fp64)
  and fp32 counterparts (lower degree).

Why these functions: for t = d/sigma >= 0 the truncation term needs
Phi(t) = 1 - E q, phi(t) = E/sqrt(2 pi) and log Phi(t) = -2 atanh(Q/(2-Q))
(PAPER.md:108 and Eq. 6).  See DESIGN.md "Device math".
"""
import os
import sys

import mpmath as mp

mp.mp.dps = 50
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_1905_04582_b200", "csrc", "mds_coeffs.h")


def lawson(xs, fs, ws, deg, iters=60):
    """min_c max_k ws[k] |fs[k] - sum_j c_j xs[k]^j| via Lawson's algorithm."""
    n = len(xs)
    lam = [mp.mpf(1) / n] * n
    best = None
    for it in range(iters):
        # weighted normal equations with weights lam * ws^2
        A = mp.matrix(deg + 1, deg + 1)
        b = mp.matrix(deg + 1, 1)
        pw = [[x ** j for j in range(deg + 1)] for x in xs]
        for k in range(n):
            wk = lam[k] * ws[k] ** 2
            for i in range(deg + 1):
                b[i] += wk * pw[k][i] * fs[k]
                for j in range(deg + 1):
                    A[i, j] += wk * pw[k][i] * pw[k][j]
        c = mp.lu_solve(A, b)
        errs = [abs(ws[k] * (fs[k] - sum(c[j] * pw[k][j] for j in range(deg + 1)))) for k in range(n)]
        m = max(errs)
        if best is None or m < best[0]:
            best = (m, [c[j] for j in range(deg + 1)])
        s = sum(lam[k] * errs[k] for k in range(n))
        lam = [lam[k] * errs[k] / s for k in range(n)]
    return best


def cheb_nodes(a, b, n):
    return [(a + b) / 2 + (b - a) / 2 * mp.cos(mp.pi * (k + mp.mpf(0.5)) / n) for k in range(n)]


def horner_double(c, x, single=False):
    import numpy as np
    t = np.float32 if single else np.float64
    x = t(x)
    p = t(c[-1])
    for a in reversed(c[:-1]):
        p = t(p * x + t(a))
    return float(p)


def fit_exp(deg, single=False):
    a = mp.log(2) / 2
    xs = cheb_nodes(-a, a, 200)
    fs = [mp.exp(x) for x in xs]
    ws = [1 / f for f in fs]
    return lawson(xs, fs, ws, deg)


def fit_exp_table(deg):
    """e^r on |r| <= ln2/512 (table-driven exp: e^x = 2^n 2^(j/256) e^r)."""
    a = mp.log(2) / 512
    xs = cheb_nodes(-a, a, 120)
    fs = [mp.exp(x) for x in xs]
    ws = [1 / f for f in fs]
    return lawson(xs, fs, ws, deg)


def Qf(t):
    return mp.erfc(t / mp.sqrt(2)) / 2


def fit_q(deg, kappa, tmax=12):
    kappa = mp.mpf(kappa)
    wmax = (tmax - kappa) / (tmax + kappa)
    ws_ = cheb_nodes(mp.mpf(-1), wmax, 260)
    xs, fs, wts = [], [], []
    for w in ws_:
        t = kappa * (1 + w) / (1 - w)
        E = mp.exp(-t * t / 2)
        xs.append(w)
        fs.append(Qf(t) / E)
        wts.append(E)
    return lawson(xs, fs, wts, deg)


def fit_q_rational(m, n, tmax=14, npts=300, iters=40):
    """q(t) = erfcx(t/sqrt2)/2 = P(t)/R(t), deg P = m, deg R = n, R(0) = 1, on t in
    [0, tmax] (Chebyshev nodes in w = (t-4)/(t+4)), weighted by E(t) = e^{-t^2/2} so
    the fitted quantity is the ABSOLUTE error of Q(t) = E P/R.  Sanathanan-Koerner
    iteration (linearised P - q R, reweighted by 1/R_prev) with Lawson weights for
    the minimax.  Beyond tmax E < 1e-42: the rational only has to stay positive
    and bounded there (every coefficient of this fit is positive)."""
    K = mp.mpf(4)
    wmax = (tmax - K) / (tmax + K)
    ts = [K * (1 + w) / (1 - w) for w in cheb_nodes(mp.mpf(-1), wmax, npts)]
    fs = [Qf(t) * mp.exp(t * t / 2) for t in ts]
    W = [mp.exp(-t * t / 2) for t in ts]
    Rprev = [mp.mpf(1)] * npts
    lam = [mp.mpf(1)] * npts
    best = None

    def ev(cs, t):
        acc = mp.mpf(0)
        for a in reversed(cs):
            acc = acc * t + a
        return acc

    for it in range(iters):
        nu = m + 1 + n
        A = mp.matrix(nu, nu)
        b = mp.matrix(nu, 1)
        for k, t in enumerate(ts):
            wk = lam[k] * (W[k] / Rprev[k]) ** 2
            row = [t ** j for j in range(m + 1)] + [-fs[k] * t ** j for j in range(1, n + 1)]
            for i in range(nu):
                b[i] += wk * row[i] * fs[k]
                for j in range(nu):
                    A[i, j] += wk * row[i] * row[j]
        c = mp.lu_solve(A, b)
        P = [c[j] for j in range(m + 1)]
        R = [mp.mpf(1)] + [c[m + 1 + j] for j in range(n)]
        Rv = [ev(R, t) for t in ts]
        errs = [abs(W[k] * (fs[k] - ev(P, t) / Rv[k])) for k, t in enumerate(ts)]
        mx = max(errs) if min(Rv) > 0 else mp.inf
        if best is None or mx < best[0]:
            best = (mx, P, R)
        Rprev = Rv
        if it >= 8:
            s = sum(lam[k] * errs[k] for k in range(npts))
            lam = [lam[k] * errs[k] / s * npts for k in range(npts)]
    return best


def fit_atanh(deg):
    xs = cheb_nodes(mp.mpf(0), mp.mpf(1) / 9, 120)
    fs = []
    for z in xs:
        s = mp.sqrt(z)
        fs.append(2 * mp.atanh(s) / s if z > 0 else mp.mpf(2))
    ws = [1 / f for f in fs]
    return lawson(xs, fs, ws, deg)


def fmt(c, single=False):
    if single:
        return ", ".join("%.9ef" % float(x) for x in c)
    return ", ".join(mp.nstr(x, 20, min_fixed=0, max_fixed=0) if False else repr(float(x)) for x in c)


def main():
    kappa64, kappa32 = 4.0, 2.5
    exp64 = fit_exp(10)
    expt64 = fit_exp_table(4)
    table = [mp.power(2, mp.mpf(j) / 256) for j in range(256)]
    # Cody-Waite split of ln2/256: hi keeps 32 significant bits, so fk * hi is exact for |fk| < 2^21
    l256 = mp.log(2) / 256
    e = mp.floor(mp.log(l256, 2))
    hi = mp.floor(l256 / mp.power(2, e - 31)) * mp.power(2, e - 31)
    lo = l256 - hi
    q64 = fit_q(13, kappa64)
    qr64 = fit_q_rational(6, 7)
    assert all(x > 0 for x in qr64[1]) and all(x > 0 for x in qr64[2]), "rational q: coefficient sign"
    at64 = fit_atanh(6)
    exp32 = fit_exp(5)
    q32 = fit_q(6, kappa32, tmax=7)
    at32 = fit_atanh(3)
    print("qr64     deg (6,7)  weighted max err %.3e" % float(qr64[0]), file=sys.stderr)
    for name, r in [("exp64", exp64), ("expt64", expt64), ("q64", q64), ("atanh64", at64),
                    ("exp32", exp32), ("q32", q32), ("atanh32", at32)]:
        print("%-8s deg %2d  weighted max err %.3e" % (name, len(r[1]) - 1, float(r[0])), file=sys.stderr)
    lines = [
        "// GENERATED by tools/gen_coeffs.py -- do not edit.",
        "// Weighted minimax fits (Lawson IRLS, 50 digits); see tools/gen_coeffs.py and DESIGN.md 'Device math'.",
        "#pragma once",
        "namespace mdsk {",
        "constexpr double KAPPA64 = %r;" % kappa64,
        "constexpr float KAPPA32 = %rf;" % kappa32,
        "// e^r, r in [-ln2/2, ln2/2]; ascending powers; max rel err %.2e" % float(exp64[0]),
        "constexpr int EXP64_DEG = %d;" % (len(exp64[1]) - 1),
        "static __constant__ double EXP64_C[] = {%s};" % fmt(exp64[1]),
        "// table-driven exp: e^r on |r| <= ln2/512, max rel err %.2e; EXPT64_TAB[j] = 2^(j/256)" % float(expt64[0]),
        "constexpr int EXPT64_DEG = %d;" % (len(expt64[1]) - 1),
        "constexpr int EXPT64_N = 256;",
        "constexpr double EXPT64_INV_STEP = %r;   // 256 / ln2" % float(256 / mp.log(2)),
        "constexpr double EXPT64_STEP_HI = %r;    // ln2/256, 32 significant bits" % float(hi),
        "constexpr double EXPT64_STEP_LO = %r;" % float(lo),
        "constexpr double EXPT64_STEP = %r;    // ln2/256 rounded to double (error %.1e)" % (
            float(mp.log(2) / 256), float(abs(mp.mpf(float(mp.log(2) / 256)) - mp.log(2) / 256))),
        "static __constant__ double EXPT64_C[] = {%s};" % fmt(expt64[1]),
        "static __device__ const double EXPT64_TAB[256] = {%s};   // global: the per-launch table build reads it coalesced" % fmt(table),
        "// q(w) = erfcx(t/sqrt2)/2, w = (t-K)/(t+K); max |E(t)(q - p)| = %.2e" % float(q64[0]),
        "// (host copy Q64_CH: the kernels take these scaled by 1/cg per sigma, SigmaParams::qc)",
        "constexpr int Q64_DEG = %d;" % (len(q64[1]) - 1),
        "static __constant__ double Q64_C[] = {%s};" % fmt(q64[1]),
        "constexpr double Q64_CH[] = {%s};" % fmt(q64[1]),
        "// q(t) = erfcx(t/sqrt2)/2 = P(t)/R(t), deg (6, 7), R(0) = 1, all coefficients > 0 (no pole on t >= 0);",
        "// max |E(t)(q - P/R)| = %.2e on [0, 14] (E = e^{-t^2/2}: the absolute error of Q = 1 - Phi)." % float(qr64[0]),
        "// One reciprocal of R(1-Q) R(2-Q) then gives 1/Phi and Q/(2-Q) (no reciprocal for a variable).",
        "// Host copies: the kernels take P / (cg sigma^j) and R / sigma^j per sigma (SigmaParams::qp, qr)",
        "constexpr int QP64_DEG = %d;" % (len(qr64[1]) - 1),
        "constexpr int QR64_DEG = %d;" % (len(qr64[2]) - 1),
        "constexpr double QP64_CH[] = {%s};" % fmt(qr64[1]),
        "constexpr double QR64_CH[] = {%s};" % fmt(qr64[2]),
        "constexpr double TCLAMP64 = 38.0;   // t = d/sigma clamped here (E' < 1e-313 cg beyond)",
        "// 2 atanh(sqrt z)/sqrt z, z in [0,1/9]; max rel err %.2e (log Phi only enters log L: DESIGN.md R32)" % float(at64[0]),
        "constexpr int ATANH64_DEG = %d;" % (len(at64[1]) - 1),
        "static __constant__ double ATANH64_C[] = {%s};" % fmt(at64[1]),
        "// fp32 variants",
        "constexpr int EXP32_DEG = %d;  // max rel err %.2e" % (len(exp32[1]) - 1, float(exp32[0])),
        "static __constant__ float EXP32_C[] = {%s};" % fmt(exp32[1], True),
        "constexpr int Q32_DEG = %d;  // max abs err of Q %.2e" % (len(q32[1]) - 1, float(q32[0])),
        "static __constant__ float Q32_C[] = {%s};" % fmt(q32[1], True),
        "constexpr int ATANH32_DEG = %d;  // max rel err %.2e" % (len(at32[1]) - 1, float(at32[0])),
        "static __constant__ float ATANH32_C[] = {%s};" % fmt(at32[1], True),
        "}  // namespace mdsk",
        "",
    ]
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        f.write("\n".join(lines))
    print("wrote", OUT, file=sys.stderr)


if __name__ == "__main__":
    main()
