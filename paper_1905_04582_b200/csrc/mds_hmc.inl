// mds_hmc.inl -- thin HMC driver (Eq. 5; readings R19, R20).
// Included at the end of mds_api.cu (same translation unit).
//
// Target log pi(x) = log L(x) - |x|^2/(2 tau^2) (iid N(0, tau^2) prior, Eq. 3 with
// V_G = tau I, Sigma = I; R20), mass M = I, leapfrog
//   p += eps/2 grad log pi;  x += eps p;  p += eps/2 grad log pi     (L times)
// State on the device: x, p, gl = grad log pi(x), log L(x) and
// xnext = x + eps (p + eps/2 gl), the position the next step evaluates at.
// One leapfrog step is ONE persistent kernel launch (unsharded): phase A
// evaluates every pair at xnext, phase B reduces the gradient in fixed order
// and applies the second half-kick and the next drift.  The L steps of an HMC
// transition are captured once into a CUDA graph; the only per-transition host
// sync reads H0 and H1 for the accept/reject.

namespace {

inline uint64_t hmc_mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
inline double hmc_u01(uint64_t h) { return ((double)(h >> 11) + 1.0) * (1.0 / 9007199254740992.0); }
inline double hmc_normal(uint64_t seed, uint64_t it, uint64_t q) {
    const uint64_t h1 = hmc_mix(seed ^ hmc_mix(it ^ hmc_mix(2 * q)));
    const uint64_t h2 = hmc_mix(seed ^ hmc_mix(it ^ hmc_mix(2 * q + 1)));
    return std::sqrt(-2.0 * std::log(hmc_u01(h1))) * std::cos(6.283185307179586 * hmc_u01(h2));
}

mds_status hmc_alloc(mds_ctx c) {
    const size_t m = (size_t)c->npad * c->d;
    mds_status st = MDS_OK;
    if (!c->d_xsave) st = dalloc(c, &c->d_xsave, m);
    if (!st && !c->d_glsave) st = dalloc(c, &c->d_glsave, m);
    if (!st && !c->d_liksave) st = dalloc(c, &c->d_liksave, 1);
    if (!st && !c->d_H) st = dalloc(c, &c->d_H, 3);
    if (!st && !c->d_H0) st = dalloc(c, &c->d_H0, 3);
    return st;
}

mds_status check_hmc_cfg(mds_ctx c, const mds_hmc_config* cfg) {
    if (!cfg || cfg->n_leapfrog < 1 || !(cfg->step_size > 0.0) || !std::isfinite(cfg->step_size) ||
        cfg->n_iter < 0 || !std::isfinite(cfg->prior_sd))
        return fail(c, MDS_E_INVALID_ARG, "bad HMC config (need n_leapfrog >= 1, step_size > 0, n_iter >= 0)");
    return MDS_OK;
}

// iid prior precision; 0 (unused) when a tree prior is set
inline double inv_tau2_of(mds_ctx c, const mds_hmc_config* cfg) {
    if (c->tree) return 0.0;
    return cfg->prior_sd > 0.0 ? 1.0 / (cfg->prior_sd * cfg->prior_sd) : 0.0;
}

// evaluate at x; gl = grad log pi(x); xnext = x + eps (p + eps/2 gl)
mds_status hmc_prime(mds_ctx c, double eps, double inv_tau2, cudaStream_t s) {
    mds_status st = run_pass(c, c->d_x, c->d_grad, c->d_lik, false, 0.0, 0.0, s, false);
    if (st) return st;
    if (c->tree) {                   // log prior and its gradient at x (tree prior)
        TreeArgs ta = c->ta;
        ta.x = c->d_x;
        tree_prior_launch(ta, c->d, s);
    }
    const int64_t m = c->n * c->d;
    prime_kernel<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(c->d_grad, c->d_x, c->d_p, c->d_gl, c->d_xnext, m,
                                                              inv_tau2, c->tree ? c->d_gprior : nullptr, eps,
                                                              0.5 * eps);
    CK(cudaGetLastError());
    c->lf_eps = eps;
    c->lf_inv_tau2 = inv_tau2;
    return MDS_OK;
}

mds_status hmc_redrift(mds_ctx c, double eps, cudaStream_t s) {
    const int64_t m = c->n * c->d;
    redrift_kernel<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(c->d_x, c->d_p, c->d_gl, c->d_xnext, m, eps, 0.5 * eps);
    CK(cudaGetLastError());
    c->lf_eps = eps;
    return MDS_OK;
}

// L leapfrog steps; only the last one forms log L (steps 1..L-1 run the
// gradient-only pass: nobody reads their log L)
mds_status hmc_enqueue_steps(mds_ctx c, int L, double eps, double inv_tau2, cudaStream_t s, bool timed) {
    for (int step = 0; step < L; ++step) {
        // steps after the first: programmatic dependent launch on the previous step's pass
        mds_status st = run_pass(c, c->d_xnext, c->d_grad, c->d_lik, true, eps, inv_tau2, s, timed, step == L - 1,
                                 step > 0);
        if (st) return st;
    }
    return MDS_OK;
}

mds_status hmc_energy(mds_ctx c, double* out, double inv_tau2, cudaStream_t s) {
    hamiltonian_kernel<<<1, 1024, 0, s>>>(c->d_x, c->d_p, c->d_lik, c->n * c->d, inv_tau2,
                                          c->tree ? c->d_logprior : nullptr, out);
    CK(cudaGetLastError());
    return MDS_OK;
}

// One HMC chain's launch state, kept across transitions (mds_hmc_run and the
// PAPER.md:672 sampler mds_mcmc_run): the CUDA graph of the L fused leapfrog
// steps (captured once; updated in place when sigma moves, since the sigma
// constants are kernel parameters), the pinned momentum buffer and the timing
// events.  Per transition: momentum upload (drawn on the host during the previous
// transition), one launch for save + redrift + H0, graph, H1, one
// host sync for the accept/reject.
struct HmcSession {
    cudaStream_t s = nullptr;
    bool owned = false;                 // stream created here (the context had the legacy stream)
    cudaGraphExec_t exec = nullptr;
    double* pbuf = nullptr;             // pinned momentum staging, two halves of n*d (or the vector below)
    bool pinned = false;
    int64_t ready_it = -1;              // transition whose momenta already sit in pbuf[ready_it & 1]
    std::vector<double> pvec;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    int L = 1;
    double eps = 0.0, it2 = 0.0;
    int64_t accepted = 0;
    double sum_abs_dh = 0.0;
    float elapsed_ms() const {
        float ms = 0.f;
        if (e0 && e1) cudaEventElapsedTime(&ms, e0, e1);
        return ms;
    }
};

void hmc_session_end(HmcSession& S) {
    if (S.exec) cudaGraphExecDestroy(S.exec);
    // (the pinned momentum buffer belongs to the context: cudaFreeHost would wait for
    // the whole device, e.g. for a peer rank's pass kernel sharing this GPU)
    if (S.e0) cudaEventDestroy(S.e0);
    if (S.e1) cudaEventDestroy(S.e1);
    if (S.owned && S.s) cudaStreamDestroy(S.s);
    S = HmcSession();
}

// (re)capture the L-step trajectory at the context's current sigma constants;
// an existing executable graph is updated in place (same topology)
mds_status hmc_session_capture(mds_ctx c, HmcSession& S) {
    NvtxRange nv("mds_hmc_capture");
    if (!graph_capturable(c)) return MDS_OK;      // host-callback exchange: direct launches
    if (std::getenv("MDS_NO_HMC_GRAPH")) return MDS_OK;   // (A/B: direct launches)
    cudaGraph_t graph = nullptr;
    CK(cudaStreamBeginCapture(S.s, cudaStreamCaptureModeThreadLocal));
    mds_status st = hmc_enqueue_steps(c, S.L, S.eps, S.it2, S.s, false);
    cudaError_t ce = cudaStreamEndCapture(S.s, &graph);
    if (st) {
        if (graph) cudaGraphDestroy(graph);
        return st;
    }
    if (ce) return fail(c, MDS_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    if (S.exec) {
        cudaGraphExecUpdateResultInfo info{};
        ce = cudaGraphExecUpdate(S.exec, graph, &info);
        if (ce) {                                  // topology changed: instantiate anew
            cudaGetLastError();
            cudaGraphExecDestroy(S.exec);
            S.exec = nullptr;
        }
    }
    if (!S.exec) ce = cudaGraphInstantiate(&S.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ce) return fail(c, MDS_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ce));
    return MDS_OK;
}

mds_status hmc_session_begin(mds_ctx c, const mds_hmc_config* cfg, HmcSession& S) {
    mds_status st = hmc_alloc(c);
    if (st) return st;
    S.s = c->stream;
    if (!S.s) {                                    // graph capture needs a non-legacy stream
        CK(cudaStreamCreateWithFlags(&S.s, cudaStreamNonBlocking));
        S.owned = true;
        CK(cudaDeviceSynchronize());
    }
    S.L = cfg->n_leapfrog;
    S.eps = cfg->step_size;
    S.it2 = inv_tau2_of(c, cfg);
    const size_t m = (size_t)(c->n * c->d);
    // two momentum halves + H0, H1 (pinned: the D2H copies of the energies must not
    // block the host, which draws the next transition's momenta meanwhile)
    if (!c->h_pbuf && cudaMallocHost(&c->h_pbuf, (2 * m + 2) * sizeof(double)) != cudaSuccess) c->h_pbuf = nullptr;
    if (c->h_pbuf) {
        S.pbuf = c->h_pbuf;
        S.pinned = true;
    } else {
        cudaGetLastError();
        S.pvec.assign(2 * m + 2, 0.0);
        S.pbuf = S.pvec.data();
    }
    CK(cudaEventCreate(&S.e0));
    CK(cudaEventCreate(&S.e1));
    return hmc_session_capture(c, S);
}

// gl and log L at the current X (after a start or a sigma move)
mds_status hmc_session_prime(mds_ctx c, HmcSession& S) { return hmc_prime(c, S.eps, S.it2, S.s); }

mds_status hmc_session_mark(mds_ctx c, HmcSession& S, cudaEvent_t e) {
    CK(cudaEventRecord(e, S.s));
    return MDS_OK;
}

void hmc_fill_momenta(double* pb, int64_t m, uint64_t seed, uint64_t it) {
    for (int64_t q = 0; q < m; ++q) pb[q] = hmc_normal(seed, it, (uint64_t)q);
}

// one HMC transition with momentum stream (seed, it): Metropolis accept on dH.
// more: another transition (it + 1, same seed) follows -- its momenta are drawn on
// the host while this one runs on the device (double-buffered staging: half it & 1
// was last uploaded by transition it - 2, complete at transition it - 1's sync)
mds_status hmc_session_transition(mds_ctx c, HmcSession& S, uint64_t seed, uint64_t it, bool more) {
    NvtxRange nv("mds_hmc_transition");
    cudaStream_t s = S.s;
    const int64_t m = c->n * c->d;
    const size_t mbytes = (size_t)c->npad * c->d * sizeof(double);
    double* pb = S.pbuf + (size_t)(it & 1) * m;
    if (S.ready_it != (int64_t)it) hmc_fill_momenta(pb, m, seed, it);
    CK(cudaMemcpyAsync(c->d_p, pb, m * sizeof(double), cudaMemcpyHostToDevice, s));
    // save for a rejection, xnext for the new momentum, H0: one launch
    const int64_t mpad = (int64_t)(mbytes / sizeof(double));
    transition_begin_kernel<<<1, 1024, 0, s>>>(c->d_x, c->d_p, c->d_gl, c->d_xsave, c->d_glsave, c->d_xnext, m, mpad,
                                               S.eps, 0.5 * S.eps, c->d_lik, c->d_liksave,
                                               c->tree ? c->d_logprior : nullptr, S.it2, c->d_H0);
    CK(cudaGetLastError());
    c->lf_eps = S.eps;
    mds_status st = MDS_OK;
    if (S.exec) {
        CK(cudaGraphLaunch(S.exec, s));
    } else if ((st = hmc_enqueue_steps(c, S.L, S.eps, S.it2, s, false))) {
        return st;
    }
    if ((st = hmc_energy(c, c->d_H, S.it2, s))) return st;
    double* hh = S.pbuf + 2 * (size_t)m;       // pinned: asynchronous
    CK(cudaMemcpyAsync(&hh[0], c->d_H0, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&hh[1], c->d_H, sizeof(double), cudaMemcpyDeviceToHost, s));
    S.ready_it = -1;
    if (more) {
        hmc_fill_momenta(S.pbuf + (size_t)((it + 1) & 1) * m, m, seed, it + 1);
        S.ready_it = (int64_t)it + 1;
    }
    CKS(s);
    const double dH = hh[1] - hh[0];
    const double u = hmc_u01(hmc_mix(seed ^ hmc_mix(0xACCE97ull ^ hmc_mix(it))));
    const bool ok = std::isfinite(dH) && std::log(u) < -dH;
    S.sum_abs_dh += std::isfinite(dH) ? std::fabs(dH) : 0.0;
    if (ok) {
        ++S.accepted;
    } else {
        const int64_t mpad = (int64_t)(mbytes / sizeof(double));
        transition_restore_kernel<<<(unsigned)((mpad + 255) / 256), 256, 0, s>>>(
            c->d_x, c->d_xsave, c->d_gl, c->d_glsave, m, mpad, c->d_lik, c->d_liksave,
            c->tree ? c->d_logprior : nullptr);
        CK(cudaGetLastError());
    }
    return MDS_OK;
}

// final log L (d_lik: the accepted state's) and X to the host
mds_status hmc_session_finish(mds_ctx c, HmcSession& S, double* x_out, double* final_ll) {
    CK(cudaMemcpyAsync(final_ll, c->d_lik, sizeof(double), cudaMemcpyDeviceToHost, S.s));
    if (x_out) CK(cudaMemcpyAsync(x_out, c->d_x, (size_t)(c->n * c->d) * sizeof(double), cudaMemcpyDeviceToHost, S.s));
    CKS(S.s);
    return MDS_OK;
}

}  // namespace

extern "C" {

mds_status mds_hmc_trajectory(mds_ctx c, const mds_hmc_config* cfg, const double* p0, double* x_out, double* p_out,
                              double* H0, double* H1) {
    GUARD(c);
    mds_status st = check_hmc_cfg(c, cfg);
    if (st) return st;
    if (!p0) return fail(c, MDS_E_INVALID_ARG, "NULL momentum");
    st = ready(c);
    if (st) return st;
    st = hmc_alloc(c);
    if (st) return st;
    cudaStream_t s = c->stream;
    const int64_t m = c->n * c->d;
    const size_t mbytes = (size_t)c->npad * c->d * sizeof(double);
    const double it2 = inv_tau2_of(c, cfg);
    CK(cudaMemcpyAsync(c->d_xsave, c->d_x, mbytes, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(c->d_p, p0, m * sizeof(double), cudaMemcpyHostToDevice, s));
    st = hmc_prime(c, cfg->step_size, it2, s);
    if (st) return st;
    st = hmc_energy(c, c->d_H0, it2, s);
    if (st) return st;
    st = hmc_enqueue_steps(c, cfg->n_leapfrog, cfg->step_size, it2, s, false);
    if (st) return st;
    st = hmc_energy(c, c->d_H, it2, s);
    if (st) return st;
    double h0 = 0, h1 = 0;
    CK(cudaMemcpyAsync(&h0, c->d_H0, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&h1, c->d_H, sizeof(double), cudaMemcpyDeviceToHost, s));
    if (x_out) CK(cudaMemcpyAsync(x_out, c->d_x, m * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (p_out) CK(cudaMemcpyAsync(p_out, c->d_p, m * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(c->d_x, c->d_xsave, mbytes, cudaMemcpyDeviceToDevice, s));
    CKS(s);
    c->eval_version = 0;   // internal results now belong to the proposal, not X
    c->lf_version = 0;
    if (H0) *H0 = h0;
    if (H1) *H1 = h1;
    return MDS_OK;
}

mds_status mds_leapfrog_device(mds_ctx c, const mds_hmc_config* cfg, const double* p0_dev) {
    GUARD(c);
    mds_status st = check_hmc_cfg(c, cfg);
    if (st) return st;
    st = ready(c);
    if (st) return st;
    cudaStream_t s = c->stream;
    const int64_t m = c->n * c->d;
    const double it2 = inv_tau2_of(c, cfg);
    if (p0_dev) CK(cudaMemcpyAsync(c->d_p, p0_dev, m * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (p0_dev || c->lf_version != c->version || c->lf_inv_tau2 != it2) {
        st = hmc_prime(c, cfg->step_size, it2, s);      // gl, log L at x; first drift
        if (st) return st;
    } else if (c->lf_eps != cfg->step_size) {
        st = hmc_redrift(c, cfg->step_size, s);          // same state, new step size
        if (st) return st;
    }
    st = hmc_enqueue_steps(c, cfg->n_leapfrog, cfg->step_size, it2, s, true);
    if (st) return st;
    ++c->version;                    // X moved
    c->lf_version = c->version;
    c->eval_version = c->version;    // d_grad / d_lik hold the pass at the new X
    return MDS_OK;
}

mds_status mds_hmc_run(mds_ctx c, const mds_hmc_config* cfg, double* x_inout, mds_hmc_stats* stats) {
    GUARD(c);
    mds_status st = check_hmc_cfg(c, cfg);
    if (st) return st;
    if (x_inout) {
        st = mds_set_locations(c, x_inout);
        if (st) return st;
    }
    st = ready(c);
    if (st) return st;
    HmcSession S;
    st = hmc_session_begin(c, cfg, S);
    if (!st) st = hmc_session_prime(c, S);
    if (!st) st = hmc_session_mark(c, S, S.e0);
    for (int it = 0; it < cfg->n_iter && !st; ++it)
        st = hmc_session_transition(c, S, cfg->seed, (uint64_t)it, it + 1 < cfg->n_iter);
    if (!st) st = hmc_session_mark(c, S, S.e1);
    double final_ll = 0.0;
    if (!st) st = hmc_session_finish(c, S, x_inout, &final_ll);
    const float ms = st ? 0.f : S.elapsed_ms();
    const int64_t accepted = S.accepted;
    const double sum_abs_dh = S.sum_abs_dh;
    hmc_session_end(S);
    if (st) return st;
    ++c->version;          // X moved
    c->eval_version = 0;
    c->lf_version = 0;
    if (stats) {
        stats->accepted = accepted;
        stats->grad_evals = (int64_t)cfg->n_iter * cfg->n_leapfrog;
        stats->mean_abs_dH = cfg->n_iter ? sum_abs_dh / cfg->n_iter : 0.0;
        stats->seconds = ms * 1e-3;
        stats->final_loglik = final_ll;
    }
    return MDS_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- MCMC driver
// The sampler structure of PAPER.md:672 on the path's pieces: each iteration one
// HMC transition of X (mds_hmc_run, L fused leapfrog steps) followed by one
// Metropolis-Hastings update of sigma^2 (mds_sigma_mh_step, reading R27).  The
// random numbers come from the same counter-based generator as mds_hmc_run,
// on streams distinct per iteration and per use.
extern "C" mds_status mds_mcmc_run(mds_ctx c, const mds_hmc_config* cfg, const mds_sigma_prior* prior,
                                   double sigma_step, double* x_inout, mds_mcmc_stats* stats) {
    GUARD(c);
    mds_status st = check_hmc_cfg(c, cfg);
    if (st) return st;
    if (!prior || !(prior->shape > 0.0) || !(prior->rate > 0.0) || !(sigma_step > 0.0) || !std::isfinite(sigma_step))
        return fail(c, MDS_E_INVALID_ARG, "mcmc: need a sigma prior with shape, rate > 0 and sigma_step > 0");
    if (x_inout) {
        st = mds_set_locations(c, x_inout);
        if (st) return st;
    }
    st = ready(c);
    if (st) return st;
    // one session for the whole chain: the trajectory graph is captured once and
    // updated in place only when sigma moves; the sigma proposal's likelihood-only
    // pass reuses the transition's log L at the current sigma (d_lik), so an
    // iteration costs L passes + 1 (+ 1 re-prime of grad log pi when sigma moved)
    HmcSession S;
    st = hmc_session_begin(c, cfg, S);
    if (!st) st = hmc_session_prime(c, S);
    if (!st) st = hmc_session_mark(c, S, S.e0);
    int64_t acc_s = 0;
    const uint64_t xseed = hmc_mix(cfg->seed ^ 0x3C3Cull);
    for (int it = 0; it < cfg->n_iter && !st; ++it) {
        if ((st = hmc_session_transition(c, S, xseed, (uint64_t)it, it + 1 < cfg->n_iter))) break;
        const double z = hmc_normal(cfg->seed ^ 0x5167A5ull, (uint64_t)it, 0);
        const double u = hmc_u01(hmc_mix(cfg->seed ^ hmc_mix(0x5167A6ull ^ hmc_mix((uint64_t)it))));
        int32_t a = 0;
        if ((st = sigma_mh_impl(c, S.s, prior, sigma_step, z, u, &a, nullptr, c->d_lik))) break;
        acc_s += a;
        if (a) {         // the sigma constants are kernel parameters; grad log pi depends on sigma
            if ((st = hmc_session_capture(c, S))) break;
            if ((st = hmc_session_prime(c, S))) break;
        }
    }
    if (!st) st = hmc_session_mark(c, S, S.e1);
    double ll = 0.0;
    if (!st) st = hmc_session_finish(c, S, x_inout, &ll);
    const float ms = st ? 0.f : S.elapsed_ms();
    const int64_t acc_x = S.accepted;
    hmc_session_end(S);
    if (st) return st;
    ++c->version;          // X moved
    c->eval_version = 0;
    c->lf_version = 0;
    if (stats) {
        stats->accepted_x = acc_x;
        stats->accepted_sigma = acc_s;
        stats->grad_evals = (int64_t)cfg->n_iter * cfg->n_leapfrog;
        stats->seconds = ms * 1e-3;
        stats->final_loglik = ll;
        stats->final_sigma = c->sigma;
    }
    return MDS_OK;
}
