/*
 * mds.h -- C-ABI of libmds, the B200 (sm_100a) hot path of Bayesian
 * multidimensional scaling (Holbrook et al., arXiv 1905.04582).
 *
 * What the library computes (PAPER.md = /root/reference/PAPER.md):
 *
 *   log L(X) = sum over observed i > j of
 *                 -1/2 log(2 pi sigma^2) - (y_ij - delta_ij)^2 / (2 sigma^2)
 *                 - T log Phi(delta_ij / sigma)                     PAPER.md:84-112 (Eq. 2)
 *   d log L / d x_i = - sum_{j != i} [ (delta_ij - y_ij)/sigma^2
 *                 + T phi(delta_ij/sigma) / (sigma Phi(delta_ij/sigma)) ] (x_i - x_j)/delta_ij
 *                                                                    PAPER.md:338-348 (Eq. 6)
 *   with delta_ij = ||x_i - x_j||, the truncated-normal model
 *   y_ij ~ N(delta_ij, sigma^2) I(y_ij > 0) of PAPER.md:78-83 (Eq. 1), and T the
 *   truncation flag of the App. B ablation.  The sum is one
 *   fused transformation-reduction over the strict lower
 *   triangle, each unordered pair evaluated once.
 *
 * Readings of the paper (full list in DESIGN.md): y is the observed
 * dissimilarity, delta the latent distance (R1); the normalising constant is
 * the full density per OBSERVED pair (R2); log L carries -log Phi (R3); NaN in
 * Y means missing (R7); only the strict lower triangle of Y is read (R4, R9);
 * y >= 0 accepted, y < 0 or +-inf rejected (R8); an observed pair with
 * delta = 0 contributes its likelihood term and a zero gradient (R10); sigma
 * is the standard deviation (R13); precision selects fp64 / fp32 storage and
 * per-pair arithmetic (R14, R15).
 *
 * Conventions for every entry point:
 *   - Return value: MDS_OK or an error status; mds_last_error() gives text.
 *   - Argument errors (MDS_E_INVALID_ARG) leave the context usable.  A CUDA
 *     error poisons the context: every later call returns MDS_E_CUDA.
 *   - Host arrays are owned by the caller; setters copy them, getters write
 *     into caller buffers; no caller pointer is retained after a call returns.
 *   - "_device" variants take device pointers and are stream-ordered on the
 *     context's stream (mds_set_stream); they do not synchronise the host.
 *   - One context may be used by one host thread at a time; distinct contexts
 *     are independent.
 *   - Arrays are row-major: X is n x d (x_ik at [i*d + k]); the packed lower
 *     triangle stores row i (i >= 1) as y_i0 .. y_i,i-1 at offset i(i-1)/2.
 *   - The library needs an sm_100 device; otherwise creation fails with
 *     MDS_E_UNSUPPORTED.  There is no CPU fallback.
 */
#ifndef MDS_H
#define MDS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mds_ctx_s *mds_ctx;

typedef enum { MDS_F64 = 0, MDS_F32 = 1 } mds_precision;

typedef enum {
    MDS_OK = 0,
    MDS_E_INVALID_ARG = 1,
    MDS_E_STATE = 2,       /* evaluation before Y, X and sigma are all set */
    MDS_E_OOM = 3,
    MDS_E_CUDA = 4,        /* sticky: the context is poisoned */
    MDS_E_COMM = 5,
    MDS_E_UNSUPPORTED = 6  /* no sm_100 device, or an option not built */
} mds_status;

#define MDS_D_MAX 8

/* ---- lifetime ---------------------------------------------------------- */

/* Create a context for n items in d latent dimensions on the current CUDA
 * device.  n >= 2; 1 <= d <= MDS_D_MAX; precision MDS_F64 or MDS_F32;
 * truncation 0 or 1 (T above).  Allocates the tile-packed triangle of Y
 * (about n^2/2 values of the chosen precision) and O(n d) side buffers.
 * Errors: MDS_E_INVALID_ARG, MDS_E_OOM, MDS_E_UNSUPPORTED, MDS_E_CUDA. */
mds_status mds_create(int64_t n, int32_t d, int32_t precision, int32_t truncation, mds_ctx *out);

/* As mds_create, but this rank owns only the tile-rows r with
 * r mod world == rank of the tiled triangle (the row-sharding
 * of the paper's multi-device cost model c0/S + c1): it
 * stores and evaluates only its share of the pairs, and each evaluation ends
 * with ONE exchange of this rank's partial (n*d gradient values + log L)
 * followed by a rank-ordered combine, so every rank holds the FULL result,
 * bitwise identical across ranks.
 *
 * nccl_unique_id: MDS_NCCL_ID_BYTES bytes from mds_nccl_unique_id() on one
 * rank, shared with all ranks (e.g. torch.distributed.broadcast_object_list).
 * Then this call is COLLECTIVE (every rank calls it with the same id, on its
 * own GPU): the context creates and owns an NCCL communicator, and the
 * exchange is ncclAllGather on the context's stream (NVLink/NVSwitch within a
 * node), so sharded leapfrog steps and HMC transitions are captured in CUDA
 * graphs like unsharded ones.  A world == 1 context with an id runs the same
 * partial -> all-gather -> combine sequence (plumbing check on one GPU).
 * nccl_unique_id == NULL: no communicator; register the exchange with
 * mds_set_allgather, or drive mds_evaluate_partial_device /
 * mds_combine_partials_device yourself.
 * Errors as mds_create, plus rank/world out of range (MDS_E_INVALID_ARG) and
 * NCCL load/initialisation failures (MDS_E_COMM). */
#define MDS_NCCL_ID_BYTES 128
mds_status mds_create_sharded(int64_t n, int32_t d, int32_t precision, int32_t truncation,
                              int32_t rank, int32_t world, const void *nccl_unique_id, mds_ctx *out);

/* A fresh NCCL unique id (MDS_NCCL_ID_BYTES bytes into id_out) for
 * mds_create_sharded; call on one rank only.  NCCL is loaded on first use
 * (the copy already in the process, e.g. torch's, else libnccl.so.2).
 * Errors: MDS_E_INVALID_ARG (NULL), MDS_E_COMM (NCCL unavailable). */
mds_status mds_nccl_unique_id(void *id_out);

/* *has = 1 if ctx owns an NCCL communicator (created with a unique id). */
mds_status mds_has_communicator(mds_ctx ctx, int32_t *has);

/* Free every device and host resource of ctx (NULL is ignored). */
void mds_destroy(mds_ctx ctx);

/* Use the given cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream)
 * for all later work.  NULL selects the legacy default stream.  Work queued on
 * the previous stream is waited for first. */
mds_status mds_set_stream(mds_ctx ctx, void *cuda_stream);

/* ---- inputs ------------------------------------------------------------ */

/* Observed dissimilarities from a host n x n matrix with leading dimension
 * ld >= n (row-major).  Only the strict lower triangle (i > j) is read.
 * NaN = missing.  Any y < 0 or +-inf -> MDS_E_INVALID_ARG (then Y counts as
 * not set).  Under sharding only this rank's tile-rows are stored. */
mds_status mds_set_dissimilarities(mds_ctx ctx, const double *y, int64_t ld);

/* Rows [i0, i1) of the packed strict lower triangle (row i holds its i
 * entries y_i0..y_i,i-1 back to back; the first value is y_{i0,0}).  Lets
 * callers stream Y without an n x n host matrix.  Same validation as above.
 * Under sharding, rows outside this rank's tile-rows are ignored, so every
 * rank may be fed the same stream.  Evaluation requires every row to have
 * been supplied once (else MDS_E_STATE). */
mds_status mds_set_dissimilarity_rows(mds_ctx ctx, int64_t i0, int64_t i1, const double *y_lower);

/* Device-pointer variant of mds_set_dissimilarity_rows (y_lower_dev is fp64
 * device memory, read on the ctx stream before the call returns). */
mds_status mds_set_dissimilarity_rows_device(mds_ctx ctx, int64_t i0, int64_t i1,
                                             const double *y_lower_dev);

/* Latent locations X (host, n x d row-major).  Non-finite -> INVALID_ARG (X
 * unchanged).  The values are copied into a context-owned pinned buffer and
 * uploaded stream-ordered on the context's stream, so x is free when the call
 * returns and a following evaluation queues right behind the upload. */
mds_status mds_set_locations(mds_ctx ctx, const double *x);

/* Latent locations from device memory (fp64, n x d), stream-ordered.  Not
 * validated (the caller owns finiteness of device data). */
mds_status mds_set_locations_device(mds_ctx ctx, const double *x_dev);

/* The standard deviation sigma (not sigma^2; R13), 1e-30 <= sigma <= 1e30
 * (the per-sigma device constants hold sigma^-7 .. sigma^2; reading R33).
 * Outside -> MDS_E_INVALID_ARG. */
mds_status mds_set_sigma(mds_ctx ctx, double sigma);

/* ---- evaluation (one fused pass computes both) ------------------------- */

/* log L into *loglik (host).  Synchronises.  A following mds_gradient with
 * no setter in between reuses the same pass. */
mds_status mds_log_likelihood(mds_ctx ctx, double *loglik);

/* d log L / dX into grad (host, n x d).  Synchronises. */
mds_status mds_gradient(mds_ctx ctx, double *grad);

/* Both from one pass; either pointer may be NULL.  Synchronises. */
mds_status mds_log_likelihood_and_gradient(mds_ctx ctx, double *loglik, double *grad);

/* Stream-ordered evaluation into device memory: *loglik_dev (1 double) and
 * grad_dev (n x d doubles); either may be NULL.  Does not synchronise. */
mds_status mds_evaluate_device(mds_ctx ctx, double *loglik_dev, double *grad_dev);

/* Sharded contexts: this rank's partial result into part_dev, laid out as
 * n*d gradient values followed by 1 log L value (n*d + 1 doubles). */
mds_status mds_evaluate_partial_device(mds_ctx ctx, double *part_dev);

/* Exchange used by sharded contexts WITHOUT a communicator (created with a
 * NULL unique id; a context that owns one ignores fn).  fn must all-gather `count` doubles
 * from every rank's send_dev into recv_dev[world][count] in rank order,
 * stream-ordered on cuda_stream (e.g. NCCL all-gather over NVLink through
 * torch.distributed), and return 0 on success.  Once registered, sharded
 * contexts run the whole pass themselves: local pair kernel -> fixed-order
 * local reduction -> fn -> rank-ordered combine, so mds_evaluate_device,
 * mds_log_likelihood_and_gradient, mds_leapfrog_device and the HMC driver
 * return the FULL result on every rank (bitwise identical across ranks).
 * Without fn, sharded evaluations fail with MDS_E_STATE.  A non-zero return
 * from fn fails the call with MDS_E_COMM. */
typedef int (*mds_allgather_fn)(void *user, const double *send_dev, double *recv_dev, int64_t count,
                                void *cuda_stream);
mds_status mds_set_allgather(mds_ctx ctx, mds_allgather_fn fn, void *user);

/* Combine world partials gathered_dev[world][n*d + 1] (rank order) into the
 * full result by a fixed rank-ordered sum (bitwise identical on every rank).
 * Either output may be NULL. */
mds_status mds_combine_partials_device(mds_ctx ctx, const double *gathered_dev, int32_t world,
                                       double *loglik_dev, double *grad_dev);

/* ---- fused peer-memory exchange (SURVEY.md 8(e) "stage 2") ---------------- */
/* The exchange of the paper's multi-device cost model c0/S + c1
 * done by the pass kernel itself over NVLink peer memory instead of a separate
 * collective: in phase B every CTA stores the fixed-order sums of its row blocks
 * (this rank's partial gradient) straight into a receive slot of EVERY rank's
 * window (remote stores through NVLink/NVSwitch), the last CTA adds this rank's
 * log L partial and raises this rank's arrival flag on every peer
 * (release, system scope); each CTA then waits for all ranks' flags (acquire)
 * and combines its row blocks from the local window in rank order, fused with
 * the leapfrog update.  One launch per step, no host or NCCL call, so sharded
 * steps are graph-capturable; results are bitwise identical to the all-gather
 * path (same rank-ordered sum).  Other sharded exchanges (likelihood-only
 * passes, single-location updates) go through the same windows with a one-CTA
 * push/flag/wait kernel.  Receive slots are double-buffered by exchange count,
 * so a fast rank never overwrites a slot a slower rank is still reading.
 *
 * Requirements: every rank's pass kernel must be co-resident with its peers'
 * (one process per GPU, or contexts sharing one GPU whose grids together fit
 * it: mds_set_grid_limit); ranks issue the same sequence of sharded calls.  A
 * rank that waits more than 60 s for a peer abandons the step and the context
 * is poisoned with MDS_E_COMM at its next synchronising call.
 *
 * Window: ((2 world (n d + 1)) doubles + 256 bytes of flags), allocated by the
 * first mds_p2p_window call, owned and freed by the context. */
#define MDS_IPC_HANDLE_BYTES 64
/* This context's window: *window_dev (may be NULL) receives its device address
 * (for contexts of one process), ipc_handle_out (may be NULL) receives
 * MDS_IPC_HANDLE_BYTES bytes of cudaIpcMemHandle_t for other processes.
 * A world-1 context connected to its own window runs the same push -> flag ->
 * wait -> combine sequence (plumbing check on one GPU). */
mds_status mds_p2p_window(mds_ctx ctx, void **window_dev, void *ipc_handle_out);
/* Connect the exchange: peer_window_dev[r] is rank r's window (r = 0..world-1,
 * this rank's own included) as a device address this context's device can
 * store to (the same process; peer access is enabled when the windows live on
 * other devices).  From then on every sharded exchange of the context goes
 * through peer memory.  Collective in effect: all ranks must connect before
 * any of them evaluates.  Ends with a handshake (one peer all-gather of the rank
 * ids, at most 30 s): MDS_E_COMM if it fails, the context then stays on its other
 * exchange. */
mds_status mds_p2p_connect(mds_ctx ctx, void *const *peer_window_dev);
/* The same from ipc_handles[world][MDS_IPC_HANDLE_BYTES] (rank order, e.g.
 * all-gathered through torch.distributed): peers' handles are opened
 * (cudaIpcOpenMemHandle, lazy peer access) and closed by mds_destroy. */
mds_status mds_p2p_connect_ipc(mds_ctx ctx, const void *ipc_handles);
/* Leave the peer-memory exchange (the context's NCCL communicator or callback,
 * if any, is used again).  All ranks must do the same, e.g. when one rank's
 * mds_p2p_connect failed. */
mds_status mds_p2p_disconnect(mds_ctx ctx);
/* *connected = 1 when the context exchanges through peer memory. */
mds_status mds_p2p_connected(mds_ctx ctx, int32_t *connected);

/* Cap the pass kernel's grid at `ctas` CTAs (0 = all SMs; the schedule is
 * rebuilt).  Leaves SMs to other work, e.g. the other ranks of a world that
 * shares one GPU through the peer-memory exchange.  Errors: MDS_E_INVALID_ARG
 * (ctas < 0). */
mds_status mds_set_grid_limit(mds_ctx ctx, int32_t ctas);

/* ---- sigma side ------------------------------------ */

/* log L (Eq. 2) at the context's X and Y for another sigma
 * (in [1e-30, 1e30]), into *loglik (host).  The context's sigma and cached results
 * are unchanged.  One likelihood-only pass: the per-pair Eq. 2 term without
 * the Eq. 6 coefficient, no gradient reduction.  Synchronises.  Errors:
 * MDS_E_INVALID_ARG, MDS_E_STATE (inputs not set), MDS_E_CUDA, MDS_E_COMM. */
mds_status mds_log_likelihood_at_sigma(mds_ctx ctx, double sigma, double *loglik);

/* Prior of the MDS error variance: sigma^-2 ~ Gamma(shape, rate). */
typedef struct {
    double shape;   /* s_0 > 0 */
    double rate;    /* r_0 > 0 */
} mds_sigma_prior;

/* One Metropolis-Hastings update of sigma^2 given X (the per-iteration
 * sigma^2 update of PAPER.md:672; under truncation its full conditional is not
 * of standard form, so a random walk on phi = log sigma^2 replaces Gibbs):
 *   phi' = phi + step * z,
 *   log r = [log L(sigma') - log L(sigma)] + [lp(phi') - lp(phi)],
 *   lp(phi) = -shape * phi - rate * e^-phi   (Gamma density of tau = e^-phi
 *                                             times the Jacobian tau),
 *   accept iff log(u) < log r; then sigma <- sigma' exactly as mds_set_sigma.
 * z ~ N(0, 1) and u ~ U(0, 1] are drawn by the caller and passed in.  Both log
 * L values come from likelihood-only passes (log L at the current sigma is
 * reused from the previous call while neither X, Y nor sigma changed).
 * Outputs (either may be NULL): *accepted (0/1), *log_ratio (log r).
 * Errors: MDS_E_INVALID_ARG (shape/rate/step <= 0, non-finite z, u outside
 * (0, 1]), MDS_E_STATE, MDS_E_CUDA, MDS_E_COMM. */
mds_status mds_sigma_mh_step(mds_ctx ctx, const mds_sigma_prior *prior, double step, double z, double u,
                             int32_t *accepted, double *log_ratio);

/* ---- single-location updates ---------------------- */

/* Change of log L when x_i alone moves to x_new_i (host, d values), with X, Y
 * and sigma otherwise as set ("changing the value of a
 * single x_i invalidates only N - 1 terms"):
 *   *delta = sum_{j != i, y_ij observed} [ ell(y_ij, ||x_new_i - x_j||) - ell(y_ij, ||x_i - x_j||) ]
 * with ell the Eq. 2 term.  O(N d), one 8-CTA cluster; the context is
 * unchanged.  Sharded contexts: each rank sums the pairs of its own tile-rows,
 * one exchange of 1 double per rank, rank-ordered sum (identical on every
 * rank; the call is collective).  Synchronises.  Errors: MDS_E_INVALID_ARG
 * (i outside [0, n), non-finite x_new_i, NULL), MDS_E_STATE, MDS_E_COMM, MDS_E_CUDA. */
mds_status mds_row_loglik_delta(mds_ctx ctx, int64_t i, const double *x_new_i, double *delta);

/* k sequential single-location random-walk Metropolis updates (the sampler of
 * Bedford et al. the paper compares HMC against), all in one
 * device launch (sharded contexts, collective: per update one propose kernel,
 * this rank's share of Delta_i, one exchange of 1 double per rank and one
 * decide kernel, stream-ordered, the same decision on every rank).
 * Update q: i = rows[q]; x' = x_i + step * z[q*d .. q*d+d-1];
 * log r = Delta_i(x') - (|x'|^2 - |x_i|^2) / (2 prior_sd^2) (iid N(0, prior_sd^2)
 * prior, reading R20; prior_sd <= 0: flat); accept iff log(u[q]) < log r, then
 * x_i <- x'.  rows (int64), z (k x d) and u (k, in (0, 1]) are host arrays of
 * the caller's random numbers.  X moves in place; *accepted (may be NULL)
 * counts acceptances.  Synchronises.  Errors: MDS_E_INVALID_ARG, MDS_E_STATE,
 * MDS_E_OOM, MDS_E_COMM, MDS_E_CUDA. */
mds_status mds_rw_sweep(mds_ctx ctx, int64_t k, const int64_t *rows, const double *z, const double *u,
                        double step, double prior_sd, int64_t *accepted);

/* ---- phylogenetic prior --------------------------- */

/* Set the Brownian-diffusion prior of X (Eq. 3):
 * X ~ MN(mu0, V_G, Sigma).  The forest has n_nodes nodes; node k < n is item k
 * (a tip), nodes >= n are internal.  parent[k] is the parent node, or -1 for a
 * root; t[k] > 0 is the branch length to the parent (x_k = x_parent +
 * N(0, t[k] Sigma)), or for a root its prior variance factor (x_root ~
 * N(mu0, t[k] Sigma): tau_0 for a tree root, tau_e for an unsequenced item,
 * which is a root without children).  Trees may be
 * multifurcating; items must be tips and internal nodes must have children.
 * mu0: d values (NULL = 0).  sigma_cov: d x d symmetric positive definite
 * (row-major; NULL = identity).  All host arrays, copied.  Once set, the HMC
 * calls (mds_hmc_trajectory, mds_leapfrog_device, mds_hmc_run) target
 * log L + log p(X) under this prior and ignore cfg->prior_sd; the prior and
 * its gradient come from an O(n d^2) post-order / pre-order pass over the
 * forest (the dynamic program of PAPER.md:243-246), never from V_G^-1.
 * n_nodes == 0 removes the tree prior (back to the iid prior).  Errors:
 * MDS_E_INVALID_ARG (bad forest: cycle, out-of-range parent, an item with
 * children, a childless internal node, t <= 0; Sigma not SPD), MDS_E_OOM,
 * MDS_E_CUDA. */
mds_status mds_set_tree_prior(mds_ctx ctx, int64_t n_nodes, const int64_t *parent, const double *t,
                              const double *mu0, const double *sigma_cov);

/* log p(X) under the tree prior at the context's X, and d log p / dX (host,
 * n x d); either may be NULL.  Synchronises.  Errors: MDS_E_STATE (no tree
 * prior or X not set), MDS_E_CUDA. */
mds_status mds_tree_prior(mds_ctx ctx, double *logp, double *grad);

/* ---- cross-validation ----------------------------- */

/* The held-out observations of one cross-validation fold:
 * m pairs (i[q], j[q], y[q]) with 0 <= i, j < n, i != j, y finite and >= 0
 * (host arrays; order is kept).  Replaces any previous fold and resets the
 * accumulator.  The caller trains on the complement: the Y given to
 * mds_set_dissimilarities* should hold NaN (missing, R7) at these pairs; this
 * is not checked.  Held-out terms are evaluated in fp64 whatever the context
 * precision, with the context's truncation flag.  Errors: MDS_E_INVALID_ARG,
 * MDS_E_OOM, MDS_E_CUDA. */
mds_status mds_cv_set_heldout(mds_ctx ctx, int64_t m, const int64_t *i, const int64_t *j, const double *y);

/* Add one posterior draw: at the context's current X and sigma, ell_q = log
 * p(y_q | X, sigma) (the Eq. 1 density = the Eq. 2 term) of every held-out
 * pair goes into that pair's running log-sum-exp.  Stream-ordered, no sync.
 * Errors: MDS_E_STATE (no fold, X or sigma not set), MDS_E_CUDA. */
mds_status mds_cv_accumulate(mds_ctx ctx);

/* The fold's log pointwise predictive density over the S draws accumulated:
 *   *lpd = sum_q log( (1/S) sum_s exp(ell_q^(s)) )
 * (PAPER.md:389-393 without the posterior-density factor, reading R29), a
 * fixed-order reduction; *draws (may be NULL) = S.  Synchronises.  Errors:
 * MDS_E_INVALID_ARG (NULL lpd), MDS_E_STATE (no fold / no draw), MDS_E_CUDA. */
mds_status mds_cv_lpd(mds_ctx ctx, double *lpd, int64_t *draws);

/* ---- diagnostics ------------------------------------------------------- */

/* Number of observed pairs stored by this context (this rank's share). */
mds_status mds_observed_pairs(mds_ctx ctx, int64_t *count);

/* Number of observed pairs with delta_ij == 0 at the current X (R10). */
mds_status mds_zero_distance_pairs(mds_ctx ctx, int64_t *count);

/* Timing mode (mds_set_timing(ctx, 1)): every fused pass outside a CUDA graph
 * records CUDA events on the ctx stream around the pair kernel and around the
 * reduction (+ exchange when sharded), without any host sync.
 * mds_last_timing synchronises on the last event and returns the MEAN
 * per-launch device time, in ms, of the pair kernel and of the reduction over
 * all passes recorded since the previous mds_last_timing / mds_set_timing
 * call (0 when none). */
mds_status mds_set_timing(mds_ctx ctx, int32_t enable);
mds_status mds_last_timing(mds_ctx ctx, float *pair_kernel_ms, float *reduce_ms);

/* ---- HMC driver (Eq. 5; readings R19, R20) ------------ */

typedef struct {
    int32_t n_iter;      /* HMC transitions */
    int32_t n_leapfrog;  /* L, leapfrog steps per transition (>= 1) */
    double step_size;    /* epsilon > 0 */
    double prior_sd;     /* tau: iid N(0, tau^2) prior per coordinate; <= 0 -> none */
    uint64_t seed;       /* momentum / accept-reject stream */
} mds_hmc_config;

typedef struct {
    int64_t accepted;
    int64_t grad_evals;
    double mean_abs_dH;
    double seconds;       /* device time of the chain (CUDA events) */
    double final_loglik;
} mds_hmc_stats;

/* One leapfrog trajectory from the current X with caller-supplied momentum
 * p0 (host, n x d): L steps of p += eps/2 grad; x += eps p; p += eps/2 grad
 * of log pi = log L + log prior.  Writes the end point to x_out / p_out
 * (host, either may be NULL) and the Hamiltonians H0, H1 (Eq. 5 with M = I).
 * The context's X is NOT changed (pure proposal). */
mds_status mds_hmc_trajectory(mds_ctx ctx, const mds_hmc_config *cfg, const double *p0,
                              double *x_out, double *p_out, double *H0, double *H1);

/* Device-resident leapfrog (the per-step hot path of HMC): enqueue
 * cfg->n_leapfrog steps that move the context's X in place, stream-ordered,
 * no host sync.  If p0_dev != NULL the momentum is (re)initialised from it
 * (device, n x d fp64) and grad log pi is primed at the current X; otherwise
 * the steps continue from the momentum and gradient the previous call left.
 * cfg->n_iter and cfg->seed are ignored.  Each step is one fused likelihood+
 * gradient pass (plus the exchange when sharded). */
mds_status mds_leapfrog_device(mds_ctx ctx, const mds_hmc_config *cfg, const double *p0_dev);

/* Current X (host, n x d) / momentum of the device-resident leapfrog (host,
 * n x d; zeros before any leapfrog call).  Synchronise. */
mds_status mds_get_locations(mds_ctx ctx, double *x);
mds_status mds_get_momentum(mds_ctx ctx, double *p);

/* Run cfg->n_iter HMC transitions (momentum ~ N(0, I) from a counter-based
 * generator seeded by cfg->seed; Metropolis accept with min(1, e^{-dH})),
 * starting from x_inout (host, n x d; NULL = the context's current X) and
 * writing the final state back to it.  One CUDA graph replays the L fused
 * leapfrog steps of a transition (unsharded contexts; sharded ones launch
 * directly since the exchange callback runs on the host); the only
 * per-transition host sync is the accept/reject.  The context's X is left at
 * the final state. */
mds_status mds_hmc_run(mds_ctx ctx, const mds_hmc_config *cfg, double *x_inout, mds_hmc_stats *stats);

/* The sampler of PAPER.md:672 on this library's pieces: cfg->n_iter
 * iterations of { one HMC transition of X (as mds_hmc_run with n_iter = 1:
 * cfg->n_leapfrog fused leapfrog steps, Metropolis accept), then one
 * Metropolis-Hastings update of sigma^2 (as mds_sigma_mh_step with prior and
 * random-walk scale sigma_step on log sigma^2) }.  Momenta and the sigma
 * proposals / uniforms come from the counter-based generator seeded by
 * cfg->seed.  x_inout (host, n x d, may be NULL = current X) is the start and
 * receives the final state; the context's X and sigma are left at the final
 * state.  Errors: as mds_hmc_run and mds_sigma_mh_step. */
typedef struct {
    int64_t accepted_x;      /* HMC transitions accepted */
    int64_t accepted_sigma;  /* sigma^2 updates accepted */
    int64_t grad_evals;
    double seconds;          /* device time (CUDA events) */
    double final_loglik;     /* log L at the final X and sigma */
    double final_sigma;
} mds_mcmc_stats;
mds_status mds_mcmc_run(mds_ctx ctx, const mds_hmc_config *cfg, const mds_sigma_prior *prior, double sigma_step,
                        double *x_inout, mds_mcmc_stats *stats);


/* ---- misc -------------------------------------------------------------- */

/* Text of the last error on ctx (never NULL; "" when none). */
const char *mds_last_error(mds_ctx ctx);

/* Static text for a status code. */
const char *mds_status_string(mds_status s);

/* Host-only work plan (no device needed): how a context with these
 * arguments splits the triangle for a pass kernel of ctas x warps_per_cta
 * warps.  Validates the plan's invariants (the warps' unit ranges tile the
 * local units in order without crossing tile-rows; every partial slab is in
 * exactly one row block's reduction list).  owned_rows (n bytes, nullable)
 * gets 1 for rows whose tile-row this rank owns.  Errors: MDS_E_INVALID_ARG,
 * MDS_E_UNSUPPORTED (too many segments per warp), MDS_E_STATE (a violated
 * invariant: a bug). */
typedef struct {
    int64_t tile_rows;            /* tile-rows owned */
    int64_t tiles;                /* 64x64 tiles stored */
    int64_t pair_slots;           /* tiles * 4096 (computed slots incl. padding) */
    int64_t pairs;                /* real unordered pairs (i > j, i < n) owned */
    int64_t segments;             /* row-partial slabs */
    int64_t slabs;                /* segments + tiles */
    int64_t max_slabs_per_block;  /* longest reduction list */
    int64_t min_units_per_warp, max_units_per_warp;
    int64_t ranges_per_warp;      /* a warp's range is split into this many segment tables */
} mds_plan_info;
mds_status mds_plan(int64_t n, int32_t rank, int32_t world, int32_t ctas, int32_t warps_per_cta,
                    mds_plan_info *info, uint8_t *owned_rows);

/* Library version "major.minor.patch". */
const char *mds_version(void);

/* SM count and compute capability of the current device (MDS_E_UNSUPPORTED
 * if there is no device). */
mds_status mds_device_info(int32_t *sm_count, int32_t *cc_major, int32_t *cc_minor);

/* Measurement utilities (L2 flush, FMA peak probe) are declared in
 * include/mds_bench.h: they are not part of the method. */

#ifdef __cplusplus
}
#endif
#endif /* MDS_H */
