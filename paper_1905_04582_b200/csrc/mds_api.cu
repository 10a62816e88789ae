// mds_api.cu -- libmds: context, C-ABI entry points (include/mds.h), the pass
// schedule, launch dispatch and (mds_hmc.inl) the HMC driver.  One translation
// unit so the __constant__ coefficient tables are visible to every kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <climits>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges cost nothing unless a profiler attaches
#include <nccl.h>   // types and enum values only: the entry points are resolved at run time (nccl_api)

#include "../../include/mds.h"
#include "../../include/mds_bench.h"
#include "mds_kernels.cuh"
#include "mds_row.cuh"
#include "mds_cv.cuh"
#include "mds_tree.cuh"

using namespace mdsk;

namespace {
const char* kVersion = "0.3.0";

// NVTX range for the lifetime of a scope (nsys / ncu --nvtx timelines of the host
// orchestration: passes, exchanges, HMC transitions, sigma updates, uploads)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// NCCL, loaded on first use.  In a process that already holds libnccl.so.2
// (torch's bundled copy), RTLD_NOLOAD reuses that one, so the library and
// torch.distributed share one NCCL; otherwise the system libnccl.so.2 is opened.
// Only sharded contexts created with a unique id need it.
struct NcclApi {
    bool tried = false, ok = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl_api() {
    static NcclApi a;
    if (a.tried) return a;
    a.tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
        const char* e = dlerror();
        a.err = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
        return a;
    }
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
    a.AllGather = (decltype(a.AllGather))dlsym(h, "ncclAllGather");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
    a.ok = a.GetUniqueId && a.CommInitRank && a.AllGather && a.CommDestroy && a.GetErrorString;
    if (!a.ok) a.err = "libnccl.so.2 lacks an entry point";
    return a;
}
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
    size_t elem = 8;         // bytes per stored y value

    std::vector<int> tiles;          // local tile codes (I << 16) | J, in storage order
    std::vector<int> row_local;      // [nb]: local index of tile (I, 0) or -1
    int* d_tiles = nullptr;
    int* d_row_local = nullptr;

    // persistent-pass schedule
    int grid = 0;                    // resident CTAs of the pass kernel
    int pair_ctas = 0;               // of which run phase A (grid - 1 with a tree prior: the last walks the tree)
    int wpc = 0;                     // its warps per CTA
    size_t smem = 0;                 // its dynamic shared memory
    int nseg = 0;
    int vpw = 1;
    int epl = 1;                     // phase B elements per lane
    int* d_warp_seg = nullptr;
    int4* d_segs = nullptr;
    int* d_blk_ptr = nullptr;
    int* d_slab_pos = nullptr;       // storage row of each logical slab (block-contiguous)
    double* d_slabs = nullptr;       // (nseg + ntl) x B x d
    double* d_likpart = nullptr;     // [wpc * grid] (one per warp)

    void* d_y = nullptr;             // tiles
    double* d_x = nullptr;           // fp64 master X, npad x d
    double* d_grad = nullptr;        // npad x d (internal result)
    double* d_lik = nullptr;         // [4]: loglik, scratch
    double* d_stage = nullptr;       // staging for packed rows
    size_t stage_elems = 0;
    int* d_bad = nullptr;
    unsigned long long* d_count = nullptr;

    // sharded exchange: the library's own NCCL communicator (mds_create_sharded
    // with a unique id; graph-capturable) or the caller's callback (mds_set_allgather)
    ncclComm_t comm = nullptr;
    mds_allgather_fn ag_fn = nullptr;
    void* ag_user = nullptr;
    double* d_partial = nullptr;     // n*d + 1
    double* d_gathered = nullptr;    // world x (n*d + 1)
    // fused peer-memory exchange (mds_p2p_window / mds_p2p_connect): this rank's
    // window, the world's window addresses, local counters, a host-mapped error word
    char* d_win = nullptr;
    size_t win_bytes = 0;
    char** d_peer_win = nullptr;     // [world]
    std::vector<void*> ipc_opened;   // peers' windows opened from IPC handles (closed on destroy)
    unsigned long long* d_p2p_state = nullptr;   // [4]
    int* h_p2p_err = nullptr;        // pinned, mapped: set by a kernel that timed out waiting for a peer
    int* d_p2p_err = nullptr;
    bool p2p = false;
    unsigned long long p2p_timeout_ns = 60000000000ull;   // MDS_P2P_TIMEOUT_S overrides (tests)
    int grid_limit = 0;              // mds_set_grid_limit (0 = all SMs)
    bool pdl_ok = std::getenv("MDS_NO_PDL") == nullptr;   // programmatic dependent launch of leapfrog steps
    unsigned* d_gbar = nullptr;      // [2] the pass kernel's software grid barrier

    // leapfrog / HMC state
    double* d_p = nullptr;
    double* d_gl = nullptr;
    double* d_xnext = nullptr;
    double* d_xsave = nullptr;
    double* d_glsave = nullptr;
    double* d_liksave = nullptr;
    double* d_H = nullptr;           // [3]
    double* d_H0 = nullptr;          // [3]
    uint64_t lf_version = 0;         // version the leapfrog state (gl, lik) belongs to
    double lf_inv_tau2 = -1.0;
    double lf_eps = -1.0;            // step size xnext was drifted with

    SigmaParams P{};
    double sigma = 0.0;
    bool x_set = false, sigma_set = false;
    std::vector<uint8_t> row_supplied;
    int64_t rows_supplied = 0;
    int64_t rows_needed = 0;
    int64_t n_obs = -1;              // -1 = recount needed
    uint64_t version = 1, eval_version = 0;
    uint64_t mh_version = 0;         // version mh_ll (log L from a MODE_LIK pass) belongs to
    double mh_ll = 0.0;

    cudaStream_t stream = nullptr;
    bool timing = false;
    std::vector<cudaEvent_t> evpool;  // timing mode: 3 events per recorded pass
    size_t ev_used = 0;               // events recorded since the last mds_last_timing

    // cross-validation fold (held-out pairs, per-pair running log-sum-exp)
    int2* d_cv_ij = nullptr;
    double* d_cv_y = nullptr;
    double* d_cv_max = nullptr;
    double* d_cv_sum = nullptr;
    double* d_cv_out = nullptr;
    int64_t cv_m = -1;               // -1: no fold set
    int64_t cv_draws = 0;

    // phylogenetic Brownian-diffusion prior (mds_set_tree_prior); replaces the
    // iid prior of the HMC driver when set
    bool tree = false;
    TreeArgs ta{};                   // device pointers + parameters of the forest
    int* d_tree_int = nullptr;       // CSR, levels, roots (one allocation)
    double* d_tree_dbl = nullptr;    // t, messages, contributions (one allocation)
    double* d_gprior = nullptr;      // [npad][d] d log prior / dX at the last evaluated point
    double* d_logprior = nullptr;    // [2]: log prior there, saved copy
    unsigned int* d_tips_done = nullptr;   // pass kernel: pair CTAs that finished their tips slice

    double* h_pbuf = nullptr;        // pinned momentum staging of the HMC driver (2 x n*d + H0, H1; allocated once)
    double* h_xstage = nullptr;      // pinned staging of mds_set_locations (asynchronous upload)
    double* h_ostage = nullptr;      // pinned staging of the host outputs (n*d gradient + log L)
    cudaEvent_t xstage_done = nullptr;

    void* d_rwbuf = nullptr;         // single-location sweeps: rows, z, u, outputs
    size_t rwbuf_bytes = 0;

    unsigned long long* d_prof = nullptr;   // MDS_PROFILE_PHASES=1: globaltimer stamps [grid][4]

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

// MDS_TRACE=1: host-side progress lines (rank, wall clock) at the points below
void trace(mds_ctx c, const char* what) {
    static const bool on = std::getenv("MDS_TRACE") != nullptr;
    if (!on) return;
    timespec ts;
    clock_gettime(CLOCK_REALTIME, &ts);
    std::fprintf(stderr, "[mds trace r%d %.6f] %s\n", c ? c->rank : -1, (ts.tv_sec % 1000) + ts.tv_nsec * 1e-9, what);
}

#define CK(call)                                                                            \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return fail(c, MDS_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// stream synchronisation that also reports a peer-memory exchange which timed out
#define CKS(stream)                                                                                       \
    do {                                                                                                  \
        CK(cudaStreamSynchronize(stream));                                                                \
        if (c->h_p2p_err && *(volatile int*)c->h_p2p_err)                                                 \
            return fail(c, MDS_E_COMM, "peer-memory exchange: a peer did not arrive in time (MDS_P2P_TIMEOUT_S, default 60 s)");       \
    } while (0)

#define GUARD(c)                                       \
    do {                                               \
        if (!(c)) return MDS_E_INVALID_ARG;            \
        if ((c)->sticky != MDS_OK) return (c)->sticky; \
    } while (0)

mds_status check_device(mds_ctx c) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(c, MDS_E_UNSUPPORTED, std::string("no CUDA device: ") + cudaGetErrorString(e));
    }
    int major = 0, coop = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    if (major != 10)
        return fail(c, MDS_E_UNSUPPORTED,
                    "libmds is built for sm_100a (B200); device has compute capability major " + std::to_string(major));
    if (!coop) return fail(c, MDS_E_UNSUPPORTED, "device does not support cooperative launch");
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
    void* ps[] = {c->d_tiles, c->d_row_local, c->d_warp_seg, c->d_segs, c->d_blk_ptr,
                  c->d_slab_pos, c->d_slabs, c->d_likpart, c->d_y, c->d_x, c->d_grad, c->d_lik, c->d_stage,
                  c->d_bad, c->d_count, c->d_partial, c->d_gathered, c->d_p, c->d_gl, c->d_xnext, c->d_xsave,
                  c->d_glsave, c->d_liksave, c->d_H, c->d_H0, c->d_prof, c->d_rwbuf,
                  c->d_cv_ij, c->d_cv_y, c->d_cv_max, c->d_cv_sum, c->d_cv_out,
                  c->d_tree_int, c->d_tree_dbl, c->d_gprior, c->d_logprior, c->d_tips_done, c->d_gbar};
    for (void* p : ps)
        if (p) cudaFree(p);
    for (auto& e : c->evpool)
        if (e) cudaEventDestroy(e);
    if (c->h_xstage) cudaFreeHost(c->h_xstage);
    if (c->h_ostage) cudaFreeHost(c->h_ostage);
    if (c->h_pbuf) cudaFreeHost(c->h_pbuf);
    if (c->xstage_done) cudaEventDestroy(c->xstage_done);
    if (c->comm) nccl_api().CommDestroy(c->comm);
    c->comm = nullptr;
    for (void* q : c->ipc_opened) cudaIpcCloseMemHandle(q);
    c->ipc_opened.clear();
    for (void* q : {(void*)c->d_win, (void*)c->d_peer_win, (void*)c->d_p2p_state})
        if (q) cudaFree(q);
    if (c->h_p2p_err) cudaFreeHost(c->h_p2p_err);
}

inline int64_t packed_off(int64_t i) { return i * (i - 1) / 2; }

// ---------------------------------------------------------------- dispatch
// pass kernel for (MODE, precision, truncation, D); instantiated in pass_m*_*.cu
PassKernel pass_fn_mode(int mode, int prec, int trunc, int d) {
    const bool f = prec == MDS_F64;
    switch (mode) {
        case MODE_EVAL: return f ? pass_m0_f64(trunc, d) : pass_m0_f32(trunc, d);
        case MODE_EVAL_NOLIK: return f ? pass_m1_f64(trunc, d) : pass_m1_f32(trunc, d);
        case MODE_LEAPFROG: return f ? pass_m2_f64(trunc, d) : pass_m2_f32(trunc, d);
        case MODE_LEAPFROG_NOLIK: return f ? pass_m3_f64(trunc, d) : pass_m3_f32(trunc, d);
        case MODE_LIK: return f ? pass_m4_f64(trunc, d) : pass_m4_f32(trunc, d);
        case MODE_LEAPFROG_TREE: return f ? pass_m5_f64(trunc, d) : pass_m5_f32(trunc, d);
        case MODE_LEAPFROG_NOLIK_TREE: return f ? pass_m6_f64(trunc, d) : pass_m6_f32(trunc, d);
        case MODE_EVAL_TREE: return f ? pass_m7_f64(trunc, d) : pass_m7_f32(trunc, d);
        default: return f ? pass_m8_f64(trunc, d) : pass_m8_f32(trunc, d);
    }
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

P2PArgs p2p_args(mds_ctx c) {
    P2PArgs q{};
    if (!c->p2p) return q;
    q.win = c->d_peer_win;
    q.state = c->d_p2p_state;
    q.err = c->d_p2p_err;
    q.rank = c->rank;
    q.world = c->world;
    q.m1 = c->n * c->d + 1;
    q.timeout_ns = c->p2p_timeout_ns;
    return q;
}

PassArgs base_args(mds_ctx c, const double* xeval) {
    PassArgs a{};
    a.y = c->d_y;
    a.xeval = xeval;
    a.warp_seg = c->d_warp_seg;
    a.segs = c->d_segs;
    a.blk_ptr = c->d_blk_ptr;
    a.slab_pos = c->d_slab_pos;
    a.nseg = c->nseg;
    a.vpw = c->vpw;
    a.epl = c->epl;
    a.nb = c->nb;
    a.n = c->n;
    a.slabs = c->d_slabs;
    a.likpart = c->d_likpart;
    a.pair_ctas = c->pair_ctas;
    a.P = c->P;
    a.prof = c->d_prof;
    a.p2p = p2p_args(c);
    a.p2p_lf = 0;
    a.gbar = c->d_gbar;
    return a;
}

mds_status launch_coop(mds_ctx c, PassKernel k, PassArgs& a, cudaStream_t s, bool pdl = false) {
    // the fp64 pass leaves the per-pair constant of Eq. 2 out of its sums (n_obs is
    // counted by ready() whenever Y changed)
    a.lik_const = c->prec == MDS_F64 ? (double)c->n_obs * a.P.k0 : 0.0;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[2];
    int na = 0;
    // Contexts on the peer-memory exchange launch WITHOUT the cooperative attribute:
    // with it, a launch blocks the host while another rank's cooperative pass kernel
    // (same process, sharing the GPU) is running -- which waits for this very launch
    // (measured: tools/p2p_dbg.py, 3 ranks).  The grid is still sized by the occupancy
    // API (one CTA per SM), so all CTAs are resident; the kernel then syncs through
    // its own grid barrier (1.5 us slower than grid.sync at C2, so only here).
    if (!c->p2p) {
        attr[na].id = cudaLaunchAttributeCooperative;
        attr[na].val.cooperative = 1;
        ++na;
    }
    a.soft_sync = c->p2p ? 1 : 0;
    // pdl: programmatic dependent launch after the previous leapfrog step's pass on
    // this stream (its prologue -- barriers, exp table, the first y copies -- overlaps
    // that grid's phase B; the kernel waits in pdl_wait before touching its results)
    const bool use_pdl = pdl && c->pdl_ok;
    if (use_pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.gridDim = dim3((unsigned)c->grid);
    cfg.blockDim = dim3(32 * k.wpc);
    cfg.dynamicSmemBytes = k.smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = na;
    trace(c, "pass launch");
    if (use_pdl) {
        const cudaError_t e = cudaLaunchKernelEx(&cfg, k.fn, a);
        if (e == cudaSuccess) {
            trace(c, "pass launched");
            return MDS_OK;
        }
        // not supported with this launch configuration: plain stream order from now on
        cudaGetLastError();
        c->pdl_ok = false;
        cfg.numAttrs = na - 1;
    }
    CK(cudaLaunchKernelEx(&cfg, k.fn, a));
    trace(c, "pass launched");
    return MDS_OK;
}

// The sharded exchange: every rank's count doubles at send into recv[world][count]
// in rank order, stream-ordered on s (NCCL all-gather over NVLink, or the caller's
// callback)
mds_status exchange(mds_ctx c, const double* send, double* recv, int64_t count, cudaStream_t s) {
    NvtxRange nv("mds_exchange");
    if (c->p2p) {       // peer-memory windows: one CTA pushes, flags, waits, gathers
        p2p_allgather_kernel<<<1, 256, 0, s>>>(p2p_args(c), send, count, recv);
        CK(cudaGetLastError());
        return MDS_OK;
    }
    if (c->comm) {
        const ncclResult_t r = nccl_api().AllGather(send, recv, (size_t)count, ncclFloat64, c->comm, s);
        if (r != ncclSuccess)
            return fail(c, MDS_E_COMM, std::string("ncclAllGather: ") + nccl_api().GetErrorString(r));
        return MDS_OK;
    }
    if (!c->ag_fn)
        return fail(c, MDS_E_STATE, "sharded context: create it with an NCCL unique id or register mds_set_allgather");
    if (c->ag_fn(c->ag_user, send, recv, count, (void*)s) != 0) return fail(c, MDS_E_COMM, "all-gather callback failed");
    return MDS_OK;
}

// unsharded: one pass kernel does everything; sharded (or a world-1 context with
// a communicator): local partial -> exchange -> rank-ordered combine
inline bool direct(mds_ctx c) { return c->world == 1 && !c->comm && !c->p2p; }

// A fused pass at xeval.  EVAL: (grad_out, lik_out) <- full result.  With a
// leapfrog state (lf = true): the pass runs at xnext and applies the leapfrog
// update (x, p, gl, xnext, grad, lik).  want_lik = false skips log L (the
// gradient-only variant; *lik_out is then NaN).  Sharded contexts go through
// the local partial, the exchange callback and the rank-ordered combine.  In
// timing mode three events bracket the pass kernel and the post-kernel work.
mds_status run_pass(mds_ctx c, const double* xeval, double* grad_out, double* lik_out, bool lf, double eps,
                    double inv_tau2, cudaStream_t s, bool timed, bool want_lik = true, bool pdl = false) {
    NvtxRange nv(lf ? "mds_leapfrog_step" : "mds_pass");
    timed = timed && c->timing;
    const int64_t nd = c->n * c->d;
    PassArgs a = base_args(c, xeval);
    a.eps = eps;
    a.heps = 0.5 * eps;
    a.inv_tau2 = inv_tau2;
    a.x = c->d_x;
    a.p = c->d_p;
    a.gl = c->d_gl;
    a.xnext = c->d_xnext;
    if (lf && c->tree) {
        // d log prior / dX at the point this pass evaluates, walked by the pass
        // kernel's last CTA during phase A (consumed by the leapfrog update)
        a.tree = c->ta;
        a.tree.x = xeval;
        const size_t need = (size_t)(c->ta.n_nodes - c->n) * (c->d + 1) * sizeof(double);
        a.tree.smem = need <= c->smem ? std::max<size_t>(need, 16) : 0;   // else the global message buffer
        a.tree.prof = nullptr;
        a.tree.ext_tips = c->pair_ctas;          // the pair CTAs run the tips pass
        a.tree.tips_done = c->d_tips_done;
        a.gprior = c->d_gprior;
    }
    if (timed) CK(cudaEventRecord(next_event(c), s));
    mds_status st;
    if (direct(c)) {
        a.grad = grad_out;
        a.lik = lik_out;
        const int mode = lf ? (c->tree ? (want_lik ? MODE_LEAPFROG_TREE : MODE_LEAPFROG_NOLIK_TREE)
                                       : (want_lik ? MODE_LEAPFROG : MODE_LEAPFROG_NOLIK))
                            : (want_lik ? MODE_EVAL : MODE_EVAL_NOLIK);
        st = launch_coop(c, pass_fn_mode(mode, c->prec, c->trunc, c->d), a, s, pdl && !timed);
        if (st) return st;
        if (timed) CK(cudaEventRecord(next_event(c), s));
    } else if (c->p2p) {
        // fused peer-memory exchange: the pass pushes its partial into every rank's
        // window, waits for all ranks and combines (+ leapfrog update) itself
        a.grad = grad_out;
        a.lik = lik_out;
        a.p2p_lf = lf ? 1 : 0;
        const int mode = (lf && c->tree) ? (want_lik ? MODE_EVAL_TREE : MODE_EVAL_NOLIK_TREE)
                                         : (want_lik ? MODE_EVAL : MODE_EVAL_NOLIK);
        st = launch_coop(c, pass_fn_mode(mode, c->prec, c->trunc, c->d), a, s, pdl && !timed);
        if (st) return st;
        if (timed) CK(cudaEventRecord(next_event(c), s));
    } else {
        // local partial; with a tree prior the pass kernel's last CTA walks the tree
        // at xeval during phase A (EVAL_TREE modes: d log prior / dX into gprior)
        a.grad = c->d_partial;
        a.lik = c->d_partial + nd;
        const int mode = (lf && c->tree) ? (want_lik ? MODE_EVAL_TREE : MODE_EVAL_NOLIK_TREE)
                                         : (want_lik ? MODE_EVAL : MODE_EVAL_NOLIK);
        st = launch_coop(c, pass_fn_mode(mode, c->prec, c->trunc, c->d), a, s);
        if (st) return st;
        if (timed) CK(cudaEventRecord(next_event(c), s));
        if ((st = exchange(c, c->d_partial, c->d_gathered, nd + 1, s))) return st;
        const unsigned blocks = (unsigned)((nd + 1 + 255) / 256);
        if (lf)      // rank-ordered combine fused with the leapfrog update
            combine_update_kernel<<<blocks, 256, 0, s>>>(c->d_gathered, c->world, nd, grad_out, lik_out, xeval, c->d_x,
                                                         c->d_p, c->d_gl, c->d_xnext, eps, 0.5 * eps, inv_tau2,
                                                         c->tree ? c->d_gprior : nullptr);
        else
            combine_kernel<<<blocks, 256, 0, s>>>(c->d_gathered, c->world, nd + 1, grad_out, lik_out);
    }
    if (timed) CK(cudaEventRecord(next_event(c), s));
    CK(cudaGetLastError());
    return MDS_OK;
}

SigmaParams sigma_params(double sigma);
// the sigma range of the device constants (sigma^+-7 normal, sigma^2 finite)
inline bool sigma_ok(double sigma) { return sigma >= 1e-30 && sigma <= 1e30; }
mds_status sigma_mh_impl(mds_ctx c, cudaStream_t s, const mds_sigma_prior* prior, double step, double z, double u,
                         int32_t* accepted, double* log_ratio, const double* cur_ll_dev);

// a pass sequence can be captured in a CUDA graph unless the exchange runs on
// the host (the mds_set_allgather callback of a sharded context)
bool graph_capturable(mds_ctx c) { return c->world == 1 || c->comm || c->p2p; }

// log L only (MODE_LIK) at the context's X for the SigmaParams given, into the
// device double lik_out; sharded: local partial -> exchange -> rank-ordered sum
mds_status run_lik_pass(mds_ctx c, const SigmaParams& P, double* lik_out, cudaStream_t s) {
    NvtxRange nv("mds_lik_pass");
    PassArgs a = base_args(c, c->d_x);
    a.P = P;
    const PassKernel k = pass_fn_mode(MODE_LIK, c->prec, c->trunc, c->d);
    if (direct(c) || c->p2p) {      // (peer-memory exchange fused into the pass)
        a.lik = lik_out;
        return launch_coop(c, k, a, s);
    }
    double* part = c->d_partial + c->n * c->d;
    a.lik = part;
    mds_status st = launch_coop(c, k, a, s);
    if (st) return st;
    if ((st = exchange(c, part, c->d_gathered, 1, s))) return st;
    combine_kernel<<<1, 32, 0, s>>>(c->d_gathered, c->world, 1, nullptr, lik_out);
    CK(cudaGetLastError());
    return MDS_OK;
}

// (stream-ordered: cudaFree would wait for the whole device, e.g. for a peer rank's
// pass kernel sharing this GPU through the peer-memory exchange)
mds_status rw_scratch(mds_ctx c, size_t bytes) {
    if (c->rwbuf_bytes >= bytes) return MDS_OK;
    if (c->d_rwbuf) cudaFreeAsync(c->d_rwbuf, c->stream);
    c->d_rwbuf = nullptr;
    c->rwbuf_bytes = 0;
    cudaError_t e = cudaMallocAsync(&c->d_rwbuf, bytes, c->stream);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(c, MDS_E_OOM, "cudaMalloc of sweep scratch failed");
    }
    c->rwbuf_bytes = bytes;
    return MDS_OK;
}

// one thread-block cluster of ROW_CLUSTER CTAs (mds_row.cuh)
mds_status launch_row(mds_ctx c, RowArgs& a) {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = ROW_CLUSTER;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(ROW_CLUSTER);
    cfg.blockDim = dim3(ROW_THREADS);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = c->stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, row_fn(c->prec == MDS_F64, c->trunc, c->d), a));
    return MDS_OK;
}

RowArgs row_args(mds_ctx c) {
    RowArgs a{};
    a.y = c->d_y;
    a.row_local = c->d_row_local;
    a.x = c->d_x;
    a.n = c->n;
    a.P = c->P;
    return a;
}

// observed pairs stored by this context (cached until Y changes; one count kernel)
mds_status count_obs(mds_ctx c) {
    if (c->n_obs >= 0) return MDS_OK;
    trace(c, "count_obs");
    CK(cudaMemsetAsync(c->d_count, 0, sizeof(unsigned long long), c->stream));
    const size_t cnt = (size_t)c->ntl * TB * TB;
    if (cnt) {
        if (c->prec == MDS_F64)
            count_obs_kernel<double><<<1184, 256, 0, c->stream>>>((const double*)c->d_y, cnt, c->d_count);
        else
            count_obs_kernel<float><<<1184, 256, 0, c->stream>>>((const float*)c->d_y, cnt, c->d_count);
        CK(cudaGetLastError());
    }
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, c->d_count, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    CKS(c->stream);
    c->n_obs = (int64_t)h;
    trace(c, "count_obs done");
    return MDS_OK;
}

mds_status ready(mds_ctx c) {
    if (c->rows_supplied < c->rows_needed)
        return fail(c, MDS_E_STATE, "dissimilarities not set (" + std::to_string(c->rows_supplied) + " of " +
                                        std::to_string(c->rows_needed) + " rows supplied)");
    if (!c->x_set) return fail(c, MDS_E_STATE, "locations not set");
    if (!c->sigma_set) return fail(c, MDS_E_STATE, "sigma not set");
    return count_obs(c);     // the fp64 pass adds n_obs x (-1/2 log(2 pi sigma^2)) once
}

// evaluate into the internal buffers if stale
mds_status eval_internal(mds_ctx c) {
    mds_status st = ready(c);
    if (st) return st;
    if (c->eval_version == c->version) return MDS_OK;
    st = run_pass(c, c->d_x, c->d_grad, c->d_lik, false, 0.0, 0.0, c->stream, true);
    if (st) return st;
    c->eval_version = c->version;
    return MDS_OK;
}

// ---------------------------------------------------------------- the plan
// Host-only description of a context's work split (no device needed; also
// exported through mds_plan for CPU tests).  Tile-rows are owned cyclically
// (I mod world == rank).  The local tiles' column-group units (16 per tile, in
// tile order) are cut into GW = ctas * wpc equal contiguous ranges, one per
// warp; each range is cut at tile-row boundaries into segments (I, u0, u1,
// tbase).  The CSR lists, for each row block b, its row slabs (the segments of
// tile-row b, in order) and then the column slabs of the local tiles (I, b),
// I ascending: the fixed order of the reduction.
struct Plan {
    int nb = 0;
    int vpw = 1;                      // virtual ranges per warp
    std::vector<int> tiles, row_local;
    std::vector<int> warp_seg;
    std::vector<int4> segs;
    std::vector<int> ptr, slab;
};

// segments per virtual range: MAXSEG_W, or less for tests (MDS_DEBUG_MAXSEG)
int max_segments() {
    const char* e = std::getenv("MDS_DEBUG_MAXSEG");
    const int v = e ? std::atoi(e) : 0;
    return (v >= 1 && v < MAXSEG_W) ? v : MAXSEG_W;
}

bool make_plan(int64_t n, int rank, int world, int64_t ctas, int wpc, Plan& P, std::string* why) {
    P = Plan();
    const int maxseg = max_segments();
    P.nb = (int)((n + TB - 1) / TB);
    P.row_local.assign(P.nb, -1);
    for (int I = 0; I < P.nb; ++I) {
        if (I % world != rank) continue;
        P.row_local[I] = (int)P.tiles.size();
        for (int J = 0; J <= I; ++J) P.tiles.push_back((I << 16) | J);
    }
    const int64_t ntl = (int64_t)P.tiles.size();
    const int64_t U = (int64_t)GROUPS_PER_TILE * ntl;
    const int64_t GW = (int64_t)wpc * ctas;
    // each warp's contiguous range is split into vpw virtual ranges; grow vpw
    // until no virtual range spans more than MAXSEG_W tile-row segments
    for (P.vpw = 1;; P.vpw *= 2) {
        const int64_t V = GW * P.vpw;
        P.warp_seg.assign(V + 1, 0);
        P.segs.clear();
        bool fits = true;
        for (int64_t w = 0; w < V && fits; ++w) {
            int64_t u = (U * w) / V, u1 = (U * (w + 1)) / V;
            int nsw = 0;
            while (u < u1) {
                const int t = (int)(u / GROUPS_PER_TILE);
                const int I = P.tiles[t] >> 16;
                const int64_t row_end = (int64_t)GROUPS_PER_TILE * (P.row_local[I] + I + 1);
                const int64_t e = std::min(u1, row_end);
                P.segs.push_back(make_int4(I, (int)u, (int)e, P.row_local[I]));
                u = e;
                ++nsw;
            }
            fits = nsw <= maxseg;
            P.warp_seg[w + 1] = (int)P.segs.size();
        }
        if (fits) break;
        if (P.vpw > (1 << 20)) {
            if (why) *why = "schedule: cannot bound segments per warp";
            return false;
        }
    }
    const int nseg = (int)P.segs.size();
    P.ptr.assign(P.nb + 1, 0);
    std::vector<std::vector<int>> rows_of(P.nb);
    for (int s2 = 0; s2 < nseg; ++s2) rows_of[P.segs[s2].x].push_back(s2);
    for (int b = 0; b < P.nb; ++b) {
        P.ptr[b] = (int)P.slab.size();
        for (int s2 : rows_of[b]) P.slab.push_back(s2);
        for (int I = b; I < P.nb; ++I)
            if (P.row_local[I] >= 0) P.slab.push_back(nseg + P.row_local[I] + b);
    }
    P.ptr[P.nb] = (int)P.slab.size();
    return true;
}

// Invariants of a plan (used by mds_plan; a failure is a bug).
bool check_plan(const Plan& P, std::string* why) {
    const int64_t U = (int64_t)GROUPS_PER_TILE * (int64_t)P.tiles.size();
    int64_t next = 0;
    for (const int4& sg : P.segs) {           // segments tile the unit range in order
        if (sg.y != next || sg.z <= sg.y) { if (why) *why = "segments not contiguous"; return false; }
        const int t0 = sg.y / GROUPS_PER_TILE, t1 = (sg.z - 1) / GROUPS_PER_TILE;
        if ((P.tiles[t0] >> 16) != sg.x || (P.tiles[t1] >> 16) != sg.x || P.row_local[sg.x] != sg.w) {
            if (why) *why = "segment crosses a tile-row";
            return false;
        }
        next = sg.z;
    }
    if (next != U) { if (why) *why = "units not covered"; return false; }
    std::vector<int> seen(P.segs.size() + P.tiles.size(), 0);
    for (int v : P.slab) {
        if (v < 0 || v >= (int)seen.size()) { if (why) *why = "slab index out of range"; return false; }
        ++seen[v];
    }
    for (size_t k = 0; k < seen.size(); ++k)
        if (seen[k] != 1) { if (why) *why = "slab not listed exactly once"; return false; }
    return true;
}

mds_status build_schedule(mds_ctx c) {
    int dev = 0, sms = 0, occ = 1 << 30;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    PassKernel ks[N_MODES];
    for (int m = 0; m < N_MODES; ++m) ks[m] = pass_fn_mode(m, c->prec, c->trunc, c->d);
    for (PassKernel k : ks) {
        CK(cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k.smem));
        int o = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k.fn, 32 * k.wpc, k.smem));
        occ = std::min(occ, o);
    }
    if (occ < 1) return fail(c, MDS_E_UNSUPPORTED, "pass kernel cannot be resident");
    c->smem = ks[0].smem;
    c->wpc = ks[0].wpc;
    const int64_t U = (int64_t)GROUPS_PER_TILE * c->ntl;
    int64_t G = (int64_t)sms * occ;
    if (c->grid_limit > 0) G = std::min<int64_t>(G, c->grid_limit);
    G = std::max<int64_t>(std::min<int64_t>(G, (U + c->wpc - 1) / c->wpc), 1);
    // with a tree prior one more CTA walks the tree during phase A
    const int64_t Gp = G;
    if (c->tree) G = Gp + 1 <= (int64_t)sms * occ ? Gp + 1 : Gp;
    const int64_t GA = c->tree ? G - 1 : G;
    if (GA < 1) return fail(c, MDS_E_UNSUPPORTED, "no CTA left for the pair phase");
    c->grid = (int)G;
    c->pair_ctas = (int)GA;
    const int64_t GW = (int64_t)c->wpc * G;
    {
        void* old[] = {c->d_warp_seg, c->d_segs, c->d_blk_ptr, c->d_slab_pos, c->d_slabs, c->d_likpart};
        for (void* p : old)
            if (p) cudaFree(p);
        c->d_warp_seg = nullptr;
        c->d_segs = nullptr;
        c->d_blk_ptr = nullptr;
        c->d_slab_pos = nullptr;
        c->d_slabs = nullptr;
        c->d_likpart = nullptr;
    }

    Plan P;
    std::string why;
    if (!make_plan(c->n, c->rank, c->world, GA, c->wpc, P, &why)) return fail(c, MDS_E_UNSUPPORTED, why);
    const std::vector<int>& warp_seg = P.warp_seg;
    const std::vector<int4>& segs = P.segs;
    const std::vector<int>& ptr = P.ptr;
    const std::vector<int>& slab = P.slab;
    c->nseg = (int)segs.size();
    c->vpw = P.vpw;
    // phase B: smallest elements-per-lane that fits the jobs in one grid round
    for (c->epl = 1; c->epl < 4; c->epl *= 2) {
        const int64_t chunks = (TB * c->d + 32 * c->epl - 1) / (32 * c->epl);
        if (chunks * c->nb <= G - 1) break;
    }

    mds_status st;
    const size_t nslab = (size_t)(c->nseg + std::max(c->ntl, 1));
    if ((st = dalloc(c, &c->d_warp_seg, warp_seg.size()))) return st;
    if ((st = dalloc(c, &c->d_segs, std::max<size_t>(segs.size(), 1)))) return st;
    if ((st = dalloc(c, &c->d_blk_ptr, ptr.size()))) return st;
    // storage row of each logical slab = its position in the CSR order, so that
    // every row block's slabs are contiguous for phase B
    std::vector<int> pos(slab.size());
    for (size_t q = 0; q < slab.size(); ++q) pos[slab[q]] = (int)q;
    if ((st = dalloc(c, &c->d_slab_pos, std::max<size_t>(pos.size(), 1)))) return st;
    if ((st = dalloc(c, &c->d_slabs, nslab * TB * c->d))) return st;
    if ((st = dalloc(c, &c->d_likpart, (size_t)GW))) return st;
    CK(cudaMemcpyAsync(c->d_warp_seg, warp_seg.data(), warp_seg.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
    if (!segs.empty()) CK(cudaMemcpyAsync(c->d_segs, segs.data(), segs.size() * sizeof(int4), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_blk_ptr, ptr.data(), ptr.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
    if (!pos.empty()) CK(cudaMemcpyAsync(c->d_slab_pos, pos.data(), pos.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(c->d_slabs, 0, nslab * TB * c->d * sizeof(double), c->stream));
    const char* pe = std::getenv("MDS_PROFILE_PHASES");
    if (pe && (pe[0] == '1' || pe[0] == '2')) {
        if (c->d_prof) cudaFree(c->d_prof);
        c->d_prof = nullptr;
        if ((st = dalloc(c, &c->d_prof, (size_t)G * 9))) return st;
        CK(cudaMemsetAsync(c->d_prof, 0, (size_t)G * 9 * sizeof(unsigned long long), c->stream));
    }
    // the host vectors above die on return and the uploads are stream-ordered on
    // the context's stream (possibly a non-blocking one): complete them here
    CKS(c->stream);
    return MDS_OK;
}

// MDS_PROFILE_PHASES=1: per-CTA phase times of the last pass, printed to stderr
void report_phases(mds_ctx c) {
    if (!c->d_prof) return;
    std::vector<unsigned long long> h((size_t)c->grid * 9);
    if (cudaMemcpy(h.data(), c->d_prof, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost)) return;
    unsigned long long t0 = ~0ull, t3 = 0;
    std::vector<double> a, w, b, s0, f0;
    for (int g = 0; g < c->grid; ++g) {
        t0 = std::min(t0, h[4 * g]);
        t3 = std::max(t3, h[4 * g + 3]);
    }
    for (int g = 0; g < c->grid; ++g) {
        a.push_back((h[4 * g + 1] - t0) * 1e-3);
        w.push_back((h[4 * g + 2] - h[4 * g + 1]) * 1e-3);
        b.push_back((h[4 * g + 3] - h[4 * g + 2]) * 1e-3);
        s0.push_back((h[4 * g] - t0) * 1e-3);
        if (h[(size_t)c->grid * 6 + g]) f0.push_back((h[(size_t)c->grid * 6 + g] - t0) * 1e-3);
    }
    auto st = [](std::vector<double> v) {
        std::sort(v.begin(), v.end());
        char buf[128];
        std::snprintf(buf, sizeof buf, "min %.2f med %.2f max %.2f", v.front(), v[v.size() / 2], v.back());
        return std::string(buf);
    };
    std::fprintf(stderr, "[mds phases] rank %d of %d: grid %d, first CTA start at globaltimer %llu ns, last end %llu\n",
                 c->rank, c->world, c->grid, t0, t3);
    std::fprintf(stderr, "[mds phases us] span %.2f | A end: %s | sync wait: %s | B: %s\n", (t3 - t0) * 1e-3,
                 st(a).c_str(), st(w).c_str(), st(b).c_str());
    {   // phase B of the job CTAs: slab loads, CTA reduction, final (update + stores)
        std::vector<double> l1, l2, l3;
        for (int g = 0; g < c->grid; ++g) {
            const unsigned long long s7 = h[(size_t)c->grid * 7 + g], s8 = h[(size_t)c->grid * 8 + g];
            if (!s7 || !s8 || s7 < h[4 * g + 2]) continue;
            l1.push_back((s7 - h[4 * g + 2]) * 1e-3);
            l2.push_back((s8 - s7) * 1e-3);
            l3.push_back((h[4 * g + 3] - s8) * 1e-3);
        }
        if (!l1.empty())
            std::fprintf(stderr, "[mds phases us] B jobs: slab loads %s | CTA sum %s | update+stores %s\n",
                         st(l1).c_str(), st(l2).c_str(), st(l3).c_str());
    }
    if (!f0.empty())
        std::fprintf(stderr, "[mds phases us] CTA start: %s | warp 0 first unit landed: %s\n", st(s0).c_str(),
                     st(f0).c_str());
    // slowest CTAs: SM id, phase-A end, units whose TMA data had not landed (cumulative)
    std::vector<int> idx(c->grid);
    for (int g = 0; g < c->grid; ++g) idx[g] = g;
    std::sort(idx.begin(), idx.end(), [&](int x, int y) { return a[x] > a[y]; });
    std::fprintf(stderr, "[mds phases] slowest (cta sm A_end not_ready):");
    for (int q = 0; q < std::min(8, c->grid); ++q)
        std::fprintf(stderr, " (%d %llu %.1f %llu)", idx[q], h[(size_t)c->grid * 5 + idx[q]], a[idx[q]],
                     h[(size_t)c->grid * 4 + idx[q]]);
    std::fprintf(stderr, "\n[mds phases] fastest:");
    for (int q = c->grid - 1; q >= std::max(0, c->grid - 8); --q)
        std::fprintf(stderr, " (%d %llu %.1f %llu)", idx[q], h[(size_t)c->grid * 5 + idx[q]], a[idx[q]],
                     h[(size_t)c->grid * 4 + idx[q]]);
    std::fprintf(stderr, "\n");
    const char* pe = std::getenv("MDS_PROFILE_PHASES");
    if (pe && pe[0] == '2') {      // every CTA's phase-A end, in CTA order
        std::fprintf(stderr, "[mds phases] A end by cta:");
        for (int g = 0; g < c->grid; ++g) std::fprintf(stderr, " %.1f", a[g]);
        std::fprintf(stderr, "\n[mds phases] sm by cta:");
        for (int g = 0; g < c->grid; ++g) std::fprintf(stderr, " %llu", h[(size_t)c->grid * 5 + g]);
        std::fprintf(stderr, "\n");
    }
}

mds_status create_impl(int64_t n, int32_t d, int32_t precision, int32_t truncation, int32_t rank, int32_t world,
                       const void* nccl_id, mds_ctx* out) {
    if (!out) return MDS_E_INVALID_ARG;
    *out = nullptr;
    if (n < 2 || d < 1 || d > MDS_D_MAX || (precision != MDS_F64 && precision != MDS_F32) ||
        (truncation != 0 && truncation != 1) || world < 1 || rank < 0 || rank >= world)
        return MDS_E_INVALID_ARG;
    {   // tile codes hold I, J in 16 bits; unit and slab indices are int32
        const int64_t nb = (n + TB - 1) / TB;
        if (nb > 0xffff || (nb * (nb + 1) / 2) * GROUPS_PER_TILE > 0x7fffffffLL) return MDS_E_INVALID_ARG;
    }
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
    c->npad = (int64_t)c->nb * TB;

    {   // tile-row ownership: cyclic (I mod world == rank), SURVEY 8(e)
        Plan P;
        make_plan(n, rank, world, 0, 1, P, nullptr);
        c->tiles = P.tiles;
        c->row_local = P.row_local;
    }
    c->ntl = (int)c->tiles.size();
    c->row_supplied.assign(n, 0);
    for (int64_t i = 0; i < n; ++i)
        if (c->row_local[i / TB] >= 0) ++c->rows_needed;

    const size_t ntl = (size_t)std::max(c->ntl, 1);
    const size_t m = (size_t)c->npad * d;
    char* yb = nullptr;
    if ((st = dalloc(c, &c->d_tiles, ntl)) || (st = dalloc(c, &c->d_row_local, (size_t)c->nb)) ||
        (st = dalloc(c, &yb, ntl * TB * TB * c->elem)) || (st = dalloc(c, &c->d_x, m)) ||
        (st = dalloc(c, &c->d_grad, m)) || (st = dalloc(c, &c->d_lik, 4)) || (st = dalloc(c, &c->d_bad, 1)) ||
        (st = dalloc(c, &c->d_count, 1)) || (st = dalloc(c, &c->d_p, m)) || (st = dalloc(c, &c->d_gl, m)) ||
        (st = dalloc(c, &c->d_xnext, m)) || (st = dalloc(c, &c->d_gbar, 2)))
        goto fail_alloc;
    c->d_y = yb;
    if ((world > 1 || nccl_id) && ((st = dalloc(c, &c->d_partial, (size_t)n * d + 1)) ||
                      (st = dalloc(c, &c->d_gathered, ((size_t)n * d + 1) * world))))
        goto fail_alloc;
    {
        cudaError_t e = cudaSuccess;
        if (c->ntl > 0) e = cudaMemcpy(c->d_tiles, c->tiles.data(), c->ntl * sizeof(int), cudaMemcpyHostToDevice);
        if (!e) e = cudaMemcpy(c->d_row_local, c->row_local.data(), c->nb * sizeof(int), cudaMemcpyHostToDevice);
        for (double* p : {c->d_x, c->d_grad, c->d_p, c->d_gl, c->d_xnext})
            if (!e) e = cudaMemset(p, 0, m * sizeof(double));
        if (!e) e = cudaMemset(c->d_lik, 0, 4 * sizeof(double));
        if (!e) e = cudaMemset(c->d_gbar, 0, 2 * sizeof(unsigned));
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
    st = build_schedule(c);
    if (st) goto fail_alloc;
    if (nccl_id) {
        // the context's own communicator (collective: every rank of the world calls
        // this with the same id); the exchange is then ncclAllGather on the context's
        // stream, so sharded passes can be captured in CUDA graphs
        NcclApi& api = nccl_api();
        if (!api.ok) {
            st = fail(c, MDS_E_COMM, api.err);
            goto fail_alloc;
        }
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        const ncclResult_t r = api.CommInitRank(&c->comm, world, id, rank);
        if (r != ncclSuccess) {
            c->comm = nullptr;
            st = fail(c, MDS_E_COMM, std::string("ncclCommInitRank: ") + api.GetErrorString(r));
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

// pack rows [i0, i1) from fp64 packed rows in device memory into the tiles
mds_status pack_rows_device(mds_ctx c, int64_t i0, int64_t i1, const double* src_dev, int64_t src_base) {
    NvtxRange nv("mds_pack_rows");
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
    CKS(c->stream);
    c->n_obs = -1;
    ++c->version;
    if (bad) {
        // the rows of this call now hold partial data: they count as not supplied
        for (int64_t i = i0; i < i1; ++i) {
            if (c->row_supplied[i]) {
                c->row_supplied[i] = 0;
                --c->rows_supplied;
            }
        }
        return fail(c, MDS_E_INVALID_ARG, "dissimilarities must be >= 0 and finite (NaN = missing)");
    }
    for (int64_t i = i0; i < i1; ++i) {
        if (c->row_local[i / TB] < 0) continue;
        if (!c->row_supplied[i]) {
            c->row_supplied[i] = 1;
            ++c->rows_supplied;
        }
    }
    return MDS_OK;
}

mds_status ensure_stage(mds_ctx c, size_t elems) {
    if (elems <= c->stage_elems) return MDS_OK;
    // stream-ordered (the rows are packed on c->stream; cudaFree would wait for the device)
    if (c->d_stage) cudaFreeAsync(c->d_stage, c->stream);
    c->d_stage = nullptr;
    c->stage_elems = 0;
    if (cudaMallocAsync((void**)&c->d_stage, elems * sizeof(double), c->stream) != cudaSuccess) {
        cudaGetLastError();
        c->d_stage = nullptr;
        return fail(c, MDS_E_OOM, "cudaMallocAsync of " + std::to_string(elems * sizeof(double)) + " bytes failed");
    }
    c->stage_elems = elems;
    return MDS_OK;
}

void mark_row0(mds_ctx c, int64_t i0) {
    if (i0 == 0 && c->row_local[0] >= 0 && !c->row_supplied[0]) {   // row 0 has no entries
        c->row_supplied[0] = 1;
        ++c->rows_supplied;
    }
}

// host packed rows -> device, in chunks of at most ~32M values
mds_status set_rows_host(mds_ctx c, int64_t i0, int64_t i1, const double* y_lower) {
    const int64_t base0 = packed_off(std::max<int64_t>(i0, 1));
    const int64_t kChunk = 32LL << 20;
    int64_t r = std::max<int64_t>(i0, 1);
    while (r < i1) {
        int64_t r1 = r + 1;
        while (r1 < i1 && packed_off(r1 + 1) - packed_off(r) <= kChunk) ++r1;
        bool any = false;   // skip chunks whose rows this rank does not own
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
    mark_row0(c, i0);
    return MDS_OK;
}

}  // namespace

// ======================================================================== ABI
extern "C" {

mds_status mds_create(int64_t n, int32_t d, int32_t precision, int32_t truncation, mds_ctx* out) {
    return create_impl(n, d, precision, truncation, 0, 1, nullptr, out);
}

mds_status mds_create_sharded(int64_t n, int32_t d, int32_t precision, int32_t truncation, int32_t rank,
                              int32_t world, const void* nccl_unique_id, mds_ctx* out) {
    return create_impl(n, d, precision, truncation, rank, world, nccl_unique_id, out);
}

mds_status mds_nccl_unique_id(void* id_out) {
    if (!id_out) return MDS_E_INVALID_ARG;
    NcclApi& api = nccl_api();
    if (!api.ok) return MDS_E_COMM;
    ncclUniqueId id;
    if (api.GetUniqueId(&id) != ncclSuccess) return MDS_E_COMM;
    std::memcpy(id_out, &id, sizeof(id));
    return MDS_OK;
}

mds_status mds_has_communicator(mds_ctx c, int32_t* has) {
    GUARD(c);
    if (!has) return fail(c, MDS_E_INVALID_ARG, "NULL output");
    *has = c->comm ? 1 : 0;
    return MDS_OK;
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
    // work already queued on the old stream (e.g. an asynchronous X upload) must
    // not race with what the new stream runs next
    if ((cudaStream_t)s != c->stream) CKS(c->stream);
    c->stream = (cudaStream_t)s;
    return MDS_OK;
}

mds_status mds_set_dissimilarity_rows(mds_ctx c, int64_t i0, int64_t i1, const double* y_lower) {
    GUARD(c);
    if (i0 < 0 || i1 > c->n || i0 > i1 ||
        (!y_lower && packed_off(std::max<int64_t>(i1, 1)) > packed_off(std::max<int64_t>(i0, 1))))
        return fail(c, MDS_E_INVALID_ARG, "bad row range or NULL rows");
    return set_rows_host(c, i0, i1, y_lower);
}

mds_status mds_set_dissimilarity_rows_device(mds_ctx c, int64_t i0, int64_t i1, const double* y_dev) {
    GUARD(c);
    if (i0 < 0 || i1 > c->n || i0 > i1 || !y_dev) return fail(c, MDS_E_INVALID_ARG, "bad row range or NULL rows");
    const int64_t r0 = std::max<int64_t>(i0, 1);
    if (i1 > r0) {
        mds_status st = pack_rows_device(c, r0, i1, y_dev, packed_off(r0));
        if (st) return st;
    }
    mark_row0(c, i0);
    return MDS_OK;
}

mds_status mds_set_dissimilarities(mds_ctx c, const double* y, int64_t ld) {
    GUARD(c);
    if (!y || ld < c->n) return fail(c, MDS_E_INVALID_ARG, "NULL matrix or ld < n");
    const int64_t kRows = 2048;   // pack the strict lower triangle block by block
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
    // validate while copying into a pinned staging buffer owned by the context, so
    // the upload is asynchronous (the caller's array is free when we return) and
    // the next evaluation queues right behind it with no host round trip
    if (!c->h_xstage) {
        if (cudaMallocHost(&c->h_xstage, (size_t)m * sizeof(double)) != cudaSuccess) {
            cudaGetLastError();
            c->h_xstage = nullptr;
        }
        if (c->h_xstage) CK(cudaEventCreateWithFlags(&c->xstage_done, cudaEventDisableTiming));
    }
    if (!c->h_xstage) {    // no pinned memory: synchronous upload from the caller's array
        for (int64_t q = 0; q < m; ++q)
            if (!std::isfinite(x[q])) return fail(c, MDS_E_INVALID_ARG, "locations must be finite");
        CK(cudaMemcpyAsync(c->d_x, x, m * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        CKS(c->stream);
    } else {
        CK(cudaEventSynchronize(c->xstage_done));      // the previous upload has left the buffer
        bool ok = true;
        for (int64_t q = 0; q < m; ++q) {
            const double v = x[q];
            ok &= std::isfinite(v);
            c->h_xstage[q] = v;
        }
        if (!ok) return fail(c, MDS_E_INVALID_ARG, "locations must be finite");
        CK(cudaMemcpyAsync(c->d_x, c->h_xstage, m * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        CK(cudaEventRecord(c->xstage_done, c->stream));
    }
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
    if (!sigma_ok(sigma)) return fail(c, MDS_E_INVALID_ARG, "sigma must lie in [1e-30, 1e30]");
    c->sigma = sigma;
    c->P = sigma_params(sigma);
    c->sigma_set = true;
    ++c->version;
    return MDS_OK;
}

mds_status mds_log_likelihood_at_sigma(mds_ctx c, double sigma, double* loglik) {
    GUARD(c);
    if (!loglik) return fail(c, MDS_E_INVALID_ARG, "NULL output");
    if (!sigma_ok(sigma)) return fail(c, MDS_E_INVALID_ARG, "sigma must lie in [1e-30, 1e30]");
    mds_status st = ready(c);
    if (st) return st;
    st = run_lik_pass(c, sigma_params(sigma), c->d_lik + 2, c->stream);
    if (st) return st;
    CK(cudaMemcpyAsync(loglik, c->d_lik + 2, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CKS(c->stream);
    return MDS_OK;
}

mds_status mds_row_loglik_delta(mds_ctx c, int64_t i, const double* x_new_i, double* delta) {
    GUARD(c);
    if (!x_new_i || !delta) return fail(c, MDS_E_INVALID_ARG, "NULL argument");
    if (i < 0 || i >= c->n) return fail(c, MDS_E_INVALID_ARG, "row index out of range");
    for (int k = 0; k < c->d; ++k)
        if (!std::isfinite(x_new_i[k])) return fail(c, MDS_E_INVALID_ARG, "non-finite location");
    mds_status st = ready(c);
    if (st) return st;
    if ((st = rw_scratch(c, 3 * sizeof(double) * 8))) return st;
    double* dx = static_cast<double*>(c->d_rwbuf);
    CK(cudaMemcpyAsync(dx, x_new_i, c->d * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    RowArgs a = row_args(c);
    a.i0 = i;
    a.xnew = dx;
    a.delta = dx + 8;
    a.K = 0;
    if ((st = launch_row(c, a))) return st;
    const double* out = dx + 8;
    if (!direct(c)) {
        // sharded: this rank's share (the pairs of its tile-rows), then the
        // rank-ordered sum of every rank's share
        if ((st = exchange(c, dx + 8, c->d_gathered, 1, c->stream))) return st;
        combine_kernel<<<1, 32, 0, c->stream>>>(c->d_gathered, c->world, 1, nullptr, dx + 16);
        CK(cudaGetLastError());
        out = dx + 16;
    }
    CK(cudaMemcpyAsync(delta, out, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CKS(c->stream);
    return MDS_OK;
}

mds_status mds_rw_sweep(mds_ctx c, int64_t k, const int64_t* rows, const double* z, const double* u, double step,
                        double prior_sd, int64_t* accepted) {
    GUARD(c);
    if (k < 0 || (k > 0 && (!rows || !z || !u))) return fail(c, MDS_E_INVALID_ARG, "bad sweep arrays");
    if (!(step > 0.0) || !std::isfinite(step) || !std::isfinite(prior_sd))
        return fail(c, MDS_E_INVALID_ARG, "need step > 0 and finite prior_sd");
    for (int64_t q = 0; q < k; ++q) {
        if (rows[q] < 0 || rows[q] >= c->n) return fail(c, MDS_E_INVALID_ARG, "row index out of range");
        if (!(u[q] > 0.0) || !(u[q] <= 1.0)) return fail(c, MDS_E_INVALID_ARG, "u must lie in (0, 1]");
        for (int j = 0; j < c->d; ++j)
            if (!std::isfinite(z[q * c->d + j])) return fail(c, MDS_E_INVALID_ARG, "non-finite z");
    }
    mds_status st = ready(c);
    if (st) return st;
    if (k == 0) {
        if (accepted) *accepted = 0;
        return MDS_OK;
    }
    const size_t zb = (size_t)k * c->d * sizeof(double), rb = (size_t)k * sizeof(int64_t), ub = (size_t)k * 8;
    const size_t hdr = 256;   // accepted count (8 B), sharded: proposal (64 B) and partial delta (8 B)
    if ((st = rw_scratch(c, hdr + rb + zb + ub))) return st;
    char* base = static_cast<char*>(c->d_rwbuf);
    unsigned long long* dacc = reinterpret_cast<unsigned long long*>(base);
    double* dxnew = reinterpret_cast<double*>(base + 64);
    double* dpart = reinterpret_cast<double*>(base + 128);
    int64_t* drows = reinterpret_cast<int64_t*>(base + hdr);
    double* dz = reinterpret_cast<double*>(base + hdr + rb);
    double* du = reinterpret_cast<double*>(base + hdr + rb + zb);
    CK(cudaMemcpyAsync(drows, rows, rb, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dz, z, zb, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(du, u, ub, cudaMemcpyHostToDevice, c->stream));
    const double inv_tau2 = prior_sd > 0.0 ? 1.0 / (prior_sd * prior_sd) : 0.0;
    if (direct(c)) {
        RowArgs a = row_args(c);
        a.K = k;
        a.rows = drows;
        a.z = dz;
        a.u = du;
        a.step = step;
        a.inv_tau2 = inv_tau2;
        a.accepted = dacc;
        if ((st = launch_row(c, a))) return st;
    } else {
        // sharded: every update needs all ranks' shares of Delta_i before its
        // decision, so each one is propose -> row share -> exchange -> decide
        // (stream-ordered; the decision and the move of x_i are identical on every rank)
        CK(cudaMemsetAsync(dacc, 0, sizeof(unsigned long long), c->stream));
        for (int64_t q = 0; q < k; ++q) {
            rw_propose_launch(c->d_x, drows, dz, q, step, c->d, dxnew, c->stream);
            RowArgs a = row_args(c);
            a.K = 0;
            a.i0 = rows[q];
            a.xnew = dxnew;
            a.delta = dpart;
            if ((st = launch_row(c, a))) return st;
            if ((st = exchange(c, dpart, c->d_gathered, 1, c->stream))) return st;
            rw_decide_launch(c->d_gathered, c->world, 1, c->d_x, drows, du, q, dxnew, inv_tau2, c->d, dacc,
                             c->stream);
        }
        CK(cudaGetLastError());
    }
    unsigned long long na = 0;
    CK(cudaMemcpyAsync(&na, dacc, sizeof(na), cudaMemcpyDeviceToHost, c->stream));
    CKS(c->stream);
    if (accepted) *accepted = (int64_t)na;
    ++c->version;      // X moved (possibly)
    return MDS_OK;
}

mds_status mds_set_tree_prior(mds_ctx c, int64_t n_nodes, const int64_t* parent, const double* t,
                              const double* mu0, const double* sigma_cov) {
    GUARD(c);
    if (n_nodes == 0) {             // back to the iid prior
        const bool was = c->tree;
        c->tree = false;
        c->lf_version = 0;
        return was ? build_schedule(c) : MDS_OK;   // phase A gets the tree CTA back
    }
    const int64_t n = c->n;
    const int d = c->d;
    if (n_nodes < n || n_nodes > INT_MAX / 2 || !parent || !t)
        return fail(c, MDS_E_INVALID_ARG, "tree prior: need n_nodes >= n and parent/t arrays");
    std::vector<int> nch((size_t)n_nodes, 0);
    for (int64_t k = 0; k < n_nodes; ++k) {
        if (parent[k] < -1 || parent[k] >= n_nodes || parent[k] == k)
            return fail(c, MDS_E_INVALID_ARG, "tree prior: parent of node " + std::to_string(k) + " out of range");
        if (parent[k] >= 0 && parent[k] < n)
            return fail(c, MDS_E_INVALID_ARG, "tree prior: item " + std::to_string(parent[k]) + " has a child (items are tips)");
        if (!(t[k] > 0.0) || !std::isfinite(t[k]))
            return fail(c, MDS_E_INVALID_ARG, "tree prior: branch lengths / root variances must be finite and > 0");
        if (parent[k] >= 0) ++nch[(size_t)parent[k]];
    }
    for (int64_t k = n; k < n_nodes; ++k)
        if (nch[(size_t)k] == 0) return fail(c, MDS_E_INVALID_ARG, "tree prior: internal node without children");
    // children CSR (ascending child index), depth from the roots, height from the tips
    std::vector<int> ch_ptr((size_t)n_nodes + 1, 0), ch_idx((size_t)std::max<int64_t>(n_nodes, 1)), fill;
    for (int64_t k = 0; k < n_nodes; ++k) ch_ptr[(size_t)k + 1] = ch_ptr[(size_t)k] + nch[(size_t)k];
    fill.assign(ch_ptr.begin(), ch_ptr.end() - 1);
    for (int64_t k = 0; k < n_nodes; ++k)
        if (parent[k] >= 0) ch_idx[(size_t)fill[(size_t)parent[k]]++] = (int)k;
    std::vector<int> roots, depth((size_t)n_nodes, -1), height((size_t)n_nodes, 0), order;
    order.reserve((size_t)n_nodes);
    for (int64_t k = 0; k < n_nodes; ++k)
        if (parent[k] < 0) {
            roots.push_back((int)k);
            depth[(size_t)k] = 0;
            order.push_back((int)k);
        }
    for (size_t q = 0; q < order.size(); ++q) {          // breadth-first from the roots
        const int v = order[q];
        for (int e = ch_ptr[(size_t)v]; e < ch_ptr[(size_t)v + 1]; ++e) {
            depth[(size_t)ch_idx[(size_t)e]] = depth[(size_t)v] + 1;
            order.push_back(ch_idx[(size_t)e]);
        }
    }
    if ((int64_t)order.size() != n_nodes) return fail(c, MDS_E_INVALID_ARG, "tree prior: parent array has a cycle");
    for (size_t q = order.size(); q-- > 0;) {             // reverse BFS: children before parents
        const int v = order[q];
        if (parent[v] >= 0) height[(size_t)parent[v]] = std::max(height[(size_t)parent[v]], height[(size_t)v] + 1);
    }
    int hmax = 0, dmax = 0;
    for (int64_t k = 0; k < n_nodes; ++k) {
        hmax = std::max(hmax, height[(size_t)k]);
        if (nch[(size_t)k]) dmax = std::max(dmax, depth[(size_t)k]);
    }
    // levels by counting sort (ascending node index inside a level)
    std::vector<int> up_ptr((size_t)hmax + 1, 0), up_nodes, dn_ptr((size_t)dmax + 2, 0), dn_nodes;
    for (int64_t k = n; k < n_nodes; ++k) ++up_ptr[(size_t)height[(size_t)k]];       // height >= 1
    for (int64_t k = 0; k < n_nodes; ++k)
        if (nch[(size_t)k]) ++dn_ptr[(size_t)depth[(size_t)k] + 1];
    up_ptr[0] = 0;
    for (int h = 1; h <= hmax; ++h) up_ptr[(size_t)h] += up_ptr[(size_t)h - 1];
    for (int dd = 1; dd <= dmax + 1; ++dd) dn_ptr[(size_t)dd] += dn_ptr[(size_t)dd - 1];
    up_nodes.assign((size_t)up_ptr[(size_t)hmax], 0);
    dn_nodes.assign((size_t)dn_ptr[(size_t)dmax + 1], 0);
    {
        std::vector<int> fu(up_ptr.begin(), up_ptr.end() - 1), fd(dn_ptr.begin(), dn_ptr.end() - 1);
        for (int64_t k = n; k < n_nodes; ++k) up_nodes[(size_t)fu[(size_t)height[(size_t)k] - 1]++] = (int)k;
        for (int64_t k = 0; k < n_nodes; ++k)
            if (nch[(size_t)k]) dn_nodes[(size_t)fd[(size_t)depth[(size_t)k]]++] = (int)k;
    }
    const int n_dn = dn_nodes.empty() ? 0 : dmax + 1;
    // narrow levels (<= 32 nodes) near the roots run on one warp
    int up_narrow = hmax;
    while (up_narrow > 0 && up_ptr[(size_t)up_narrow] - up_ptr[(size_t)up_narrow - 1] <= 32) --up_narrow;
    int dn_narrow = 0;
    while (dn_narrow < n_dn && dn_ptr[(size_t)dn_narrow + 1] - dn_ptr[(size_t)dn_narrow] <= 32) ++dn_narrow;
    // Sigma^-1 and log|Sigma| by Cholesky (d <= 8; parameter preprocessing, like SigmaParams)
    double S[TREE_DMAX * TREE_DMAX], Lc[TREE_DMAX * TREE_DMAX] = {0}, Si[TREE_DMAX * TREE_DMAX] = {0};
    for (int r = 0; r < d; ++r)
        for (int q = 0; q < d; ++q) S[r * d + q] = sigma_cov ? sigma_cov[r * d + q] : (r == q ? 1.0 : 0.0);
    double logdet = 0.0;
    for (int r = 0; r < d; ++r) {
        for (int q = 0; q <= r; ++q) {
            if (!std::isfinite(S[r * d + q]) || S[r * d + q] != S[q * d + r])
                return fail(c, MDS_E_INVALID_ARG, "tree prior: Sigma must be finite and symmetric");
            double v = S[r * d + q];
            for (int k = 0; k < q; ++k) v -= Lc[r * d + k] * Lc[q * d + k];
            if (r == q) {
                if (!(v > 0.0)) return fail(c, MDS_E_INVALID_ARG, "tree prior: Sigma is not positive definite");
                Lc[r * d + r] = std::sqrt(v);
                logdet += 2.0 * std::log(Lc[r * d + r]);
            } else {
                Lc[r * d + q] = v / Lc[q * d + q];
            }
        }
    }
    for (int col = 0; col < d; ++col) {                    // Sigma^-1 e_col by two triangular solves
        double z[TREE_DMAX];
        for (int r = 0; r < d; ++r) {
            double v = (r == col) ? 1.0 : 0.0;
            for (int k = 0; k < r; ++k) v -= Lc[r * d + k] * z[k];
            z[r] = v / Lc[r * d + r];
        }
        for (int r = d - 1; r >= 0; --r) {
            double v = z[r];
            for (int k = r + 1; k < d; ++k) v -= Lc[k * d + r] * Si[k * d + col];
            Si[r * d + col] = v / Lc[r * d + r];
        }
    }
    for (int q = 0; q < d; ++q)
        if (mu0 && !std::isfinite(mu0[q])) return fail(c, MDS_E_INVALID_ARG, "tree prior: non-finite mu0");
    // device buffers
    if (c->d_tree_int) cudaFree(c->d_tree_int);
    if (c->d_tree_dbl) cudaFree(c->d_tree_dbl);
    c->d_tree_int = nullptr;
    c->d_tree_dbl = nullptr;
    c->tree = false;
    // level-ordered entries: post-order (internal nodes by height), pre-order
    // (nodes with children by depth), and each child's slot in its parent's
    // pre-order entry
    const size_t nn = (size_t)n_nodes;
    const size_t E_up = up_nodes.size(), E_dn = dn_nodes.size();
    std::vector<int> up_e(4 * E_up), dn_e(4 * E_dn), dn_pos(nn, -1), up_dpos(E_up, -1), tip_upos((size_t)n, -1);
    std::vector<double> up_t(2 * E_up, 0.0), dn_t(2 * E_dn, 0.0), up_tn(E_up, 0.0);
    for (size_t e = 0; e < E_up; ++e) {
        const int v = up_nodes[e], c0 = ch_ptr[(size_t)v], k = ch_ptr[(size_t)v + 1] - c0;
        up_e[4 * e] = v - (int)n;
        for (int i = 0; i < 2; ++i) {
            const int ch = i < k ? ch_idx[(size_t)c0 + i] : -1;
            up_e[4 * e + 1 + i] = ch < 0 ? 0 : (ch < n ? -1 - ch : ch - (int)n);
            up_t[2 * e + i] = ch < 0 ? 0.0 : t[ch];
            if (ch >= 0 && ch < n) tip_upos[(size_t)ch] = (int)(2 * e + i);
        }
        up_e[4 * e + 3] = k;
        up_tn[e] = t[v];
    }
    for (size_t e = 0; e < E_dn; ++e) {
        const int v = dn_nodes[e], c0 = ch_ptr[(size_t)v], k = ch_ptr[(size_t)v + 1] - c0;
        dn_e[4 * e] = v - (int)n;
        for (int i = 0; i < 2; ++i) {
            const int ch = i < k ? ch_idx[(size_t)c0 + i] : -1;
            dn_e[4 * e + 1 + i] = ch < 0 ? 0 : ch;
            dn_t[2 * e + i] = ch < 0 ? 0.0 : t[ch];
            if (ch >= 0) dn_pos[(size_t)ch] = (int)(2 * e + i);
        }
        dn_e[4 * e + 3] = k;
    }
    for (size_t e = 0; e < E_up; ++e) up_dpos[e] = dn_pos[(size_t)up_nodes[e]];
    std::vector<int> ints;
    auto put = [&](const std::vector<int>& v) {     // 16-byte aligned offsets (int4 views)
        while (ints.size() % 4) ints.push_back(0);
        const size_t off = ints.size();
        ints.insert(ints.end(), v.begin(), v.end());
        return off;
    };
    const size_t o_upe = put(up_e), o_dne = put(dn_e), o_chp = put(ch_ptr), o_chi = put(ch_idx), o_upp = put(up_ptr),
                 o_dnp = put(dn_ptr), o_rt = put(roots), o_pos = put(dn_pos), o_udp = put(up_dpos),
                 o_tup = put(tip_upos);
    // doubles: t | pw | cq | cw | up_t | dn_t | up_m | dn_sib | msg   (16-byte aligned pieces)
    auto al2 = [](size_t v) { return (v + 1) & ~(size_t)1; };
    const size_t o_t = 0, o_pw = al2(o_t + nn), o_cq = al2(o_pw + nn), o_cw = al2(o_cq + nn), o_upt = al2(o_cw + nn),
                 o_dnt = al2(o_upt + 2 * E_up), o_utn = al2(o_dnt + 2 * E_dn), o_upx = al2(o_utn + E_up),
                 o_upm = al2(o_upx + 2 * E_up * d), o_sib = al2(o_upm + (nn - n) * d), o_msg = al2(o_sib + 2 * E_dn * (d + 1)),
                 n_dbl = al2(o_msg + (nn - n) * (d + 1));
    mds_status st;
    if ((st = dalloc(c, &c->d_tree_int, std::max<size_t>(ints.size(), 1))) ||
        (st = dalloc(c, &c->d_tree_dbl, n_dbl)) ||
        (!c->d_gprior && (st = dalloc(c, &c->d_gprior, (size_t)c->npad * d))) ||
        (!c->d_logprior && (st = dalloc(c, &c->d_logprior, 2))) ||
        (!c->d_tips_done && (st = dalloc(c, &c->d_tips_done, 1))))
        return st;
    CK(cudaMemsetAsync(c->d_tips_done, 0, sizeof(unsigned int), c->stream));
    CK(cudaMemcpyAsync(c->d_tree_int, ints.data(), ints.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(c->d_tree_dbl, 0, n_dbl * sizeof(double), c->stream));
    CK(cudaMemcpyAsync(c->d_tree_dbl + o_t, t, nn * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    if (E_up) CK(cudaMemcpyAsync(c->d_tree_dbl + o_upt, up_t.data(), up_t.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    if (E_dn) CK(cudaMemcpyAsync(c->d_tree_dbl + o_dnt, dn_t.data(), dn_t.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    if (E_up) CK(cudaMemcpyAsync(c->d_tree_dbl + o_utn, up_tn.data(), up_tn.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(c->d_gprior, 0, (size_t)c->npad * d * sizeof(double), c->stream));
    TreeArgs& A = c->ta;
    A = TreeArgs{};
    A.n_nodes = (int)n_nodes;
    A.n_items = (int)n;
    A.ch_ptr = c->d_tree_int + o_chp;
    A.ch_idx = c->d_tree_int + o_chi;
    A.t = c->d_tree_dbl + o_t;
    A.up_lvl_ptr = c->d_tree_int + o_upp;
    A.up_e = reinterpret_cast<const int4*>(c->d_tree_int + o_upe);
    A.up_t = reinterpret_cast<const double2*>(c->d_tree_dbl + o_upt);
    A.up_tn = c->d_tree_dbl + o_utn;
    A.up_dpos = c->d_tree_int + o_udp;
    A.tip_upos = c->d_tree_int + o_tup;
    A.up_x = c->d_tree_dbl + o_upx;
    A.n_up = hmax;
    A.up_narrow = up_narrow;
    A.dn_lvl_ptr = c->d_tree_int + o_dnp;
    A.dn_e = reinterpret_cast<const int4*>(c->d_tree_int + o_dne);
    A.dn_t = reinterpret_cast<const double2*>(c->d_tree_dbl + o_dnt);
    A.dn_sib = c->d_tree_dbl + o_sib;
    A.dn_pos = c->d_tree_int + o_pos;
    A.n_dn = n_dn;
    A.dn_narrow = dn_narrow;
    A.roots = c->d_tree_int + o_rt;
    A.n_roots = (int)roots.size();
    for (int q = 0; q < d; ++q) A.mu0[q] = mu0 ? mu0[q] : 0.0;
    for (int q = 0; q < d * d; ++q) A.sinv[q] = Si[q];
    A.logdet = logdet;
    A.pw = c->d_tree_dbl + o_pw;
    A.cq = c->d_tree_dbl + o_cq;
    A.cw = c->d_tree_dbl + o_cw;
    A.up_m = c->d_tree_dbl + o_upm;
    A.msg = c->d_tree_dbl + o_msg;
    {
        const size_t need = (nn - (size_t)n) * (d + 1) * sizeof(double);
        A.smem = need <= TREE_SMEM_MAX ? std::max<size_t>(need, 16) : 0;
    }
    A.grad = c->d_gprior;
    A.logp = c->d_logprior;
    CKS(c->stream);   // the uploads above read host vectors that die on return
    const char* pe = std::getenv("MDS_PROFILE_TREE");
    if (pe && pe[0] == '1') {
        static unsigned long long* prof = nullptr;
        if (!prof) cudaMalloc(&prof, 256 * sizeof(unsigned long long));
        cudaMemset(prof, 0, 256 * sizeof(unsigned long long));
        if (std::getenv("MDS_TREE_NO_PREFETCH")) {
            const unsigned long long one = 1;
            cudaMemcpy(prof + 255, &one, sizeof(one), cudaMemcpyHostToDevice);
        }
        A.prof = prof;
        fprintf(stderr, "tree levels: up %d (narrow from %d), dn %d (narrow below %d)\n", hmax, up_narrow, n_dn,
                dn_narrow);
    }
    c->tree = true;
    c->lf_version = 0;               // leapfrog state must be re-primed under the new prior
    return build_schedule(c);        // one CTA of the pass kernel walks the tree during phase A
}

void report_tree_profile(mds_ctx c) {
    if (!c->ta.prof) return;
    unsigned long long h[256];
    cudaMemcpy(h, c->ta.prof, sizeof(h), cudaMemcpyDeviceToHost);
    fprintf(stderr, "tree us:");
    for (int k = 1; k < 255; ++k)
        if (h[k]) fprintf(stderr, " %d:%.2f", k, (h[k] - h[0]) * 1e-3);
    fprintf(stderr, "\n");
}

mds_status mds_tree_prior(mds_ctx c, double* logp, double* grad) {
    GUARD(c);
    if (!c->tree) return fail(c, MDS_E_STATE, "no tree prior set (mds_set_tree_prior)");
    if (!c->x_set) return fail(c, MDS_E_STATE, "locations not set");
    TreeArgs ta = c->ta;
    ta.x = c->d_x;
    tree_prior_launch(ta, c->d, c->stream);
    CK(cudaGetLastError());
    if (logp) CK(cudaMemcpyAsync(logp, c->d_logprior, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (grad)
        CK(cudaMemcpyAsync(grad, c->d_gprior, (size_t)c->n * c->d * sizeof(double), cudaMemcpyDeviceToHost,
                           c->stream));
    CKS(c->stream);
    report_tree_profile(c);
    c->lf_version = 0;     // d_gprior / d_logprior now belong to X, not to the leapfrog state
    return MDS_OK;
}

mds_status mds_cv_set_heldout(mds_ctx c, int64_t m, const int64_t* i, const int64_t* j, const double* y) {
    GUARD(c);
    if (m < 0 || (m > 0 && (!i || !j || !y))) return fail(c, MDS_E_INVALID_ARG, "bad held-out arrays");
    if (m > INT_MAX) return fail(c, MDS_E_INVALID_ARG, "too many held-out pairs");
    std::vector<int2> ij((size_t)m);
    for (int64_t q = 0; q < m; ++q) {
        if (i[q] < 0 || i[q] >= c->n || j[q] < 0 || j[q] >= c->n || i[q] == j[q])
            return fail(c, MDS_E_INVALID_ARG, "held-out pair " + std::to_string(q) + " out of range or diagonal");
        if (!(y[q] >= 0.0) || !std::isfinite(y[q]))
            return fail(c, MDS_E_INVALID_ARG, "held-out y must be finite and >= 0");
        ij[(size_t)q] = make_int2((int)i[q], (int)j[q]);
    }
    void* ps[] = {c->d_cv_ij, c->d_cv_y, c->d_cv_max, c->d_cv_sum};
    for (void* p : ps)
        if (p) cudaFree(p);
    c->d_cv_ij = nullptr;
    c->d_cv_y = c->d_cv_max = c->d_cv_sum = nullptr;
    c->cv_m = -1;
    c->cv_draws = 0;
    mds_status st;
    if ((st = dalloc(c, &c->d_cv_ij, (size_t)m)) || (st = dalloc(c, &c->d_cv_y, (size_t)m)) ||
        (st = dalloc(c, &c->d_cv_max, (size_t)m)) || (st = dalloc(c, &c->d_cv_sum, (size_t)m)) ||
        (!c->d_cv_out && (st = dalloc(c, &c->d_cv_out, 1))))
        return st;
    if (m > 0) {
        CK(cudaMemcpyAsync(c->d_cv_ij, ij.data(), (size_t)m * sizeof(int2), cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(c->d_cv_y, y, (size_t)m * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        CKS(c->stream);   // ij dies on return; y belongs to the caller
    }
    c->cv_m = m;
    return MDS_OK;
}

mds_status mds_cv_accumulate(mds_ctx c) {
    GUARD(c);
    if (c->cv_m < 0) return fail(c, MDS_E_STATE, "no held-out fold set (mds_cv_set_heldout)");
    if (!c->x_set) return fail(c, MDS_E_STATE, "locations not set");
    if (!c->sigma_set) return fail(c, MDS_E_STATE, "sigma not set");
    if (c->cv_m > 0) {
        CvArgs a{};
        a.ij = c->d_cv_ij;
        a.y = c->d_cv_y;
        a.x = c->d_x;
        a.lmax = c->d_cv_max;
        a.lsum = c->d_cv_sum;
        a.m = c->cv_m;
        a.d = c->d;
        a.trunc = c->trunc;
        a.first = c->cv_draws == 0;
        a.P = c->P;
        int sms = 148;
        int dev = 0;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const int64_t want = (c->cv_m + 255) / 256;
        cv_accumulate_launch(a, (int)std::min<int64_t>(want, (int64_t)sms * 8), c->stream);
        CK(cudaGetLastError());
    }
    ++c->cv_draws;
    return MDS_OK;
}

mds_status mds_cv_lpd(mds_ctx c, double* lpd, int64_t* draws) {
    GUARD(c);
    if (!lpd) return fail(c, MDS_E_INVALID_ARG, "NULL output");
    if (c->cv_m < 0) return fail(c, MDS_E_STATE, "no held-out fold set (mds_cv_set_heldout)");
    if (c->cv_draws == 0) return fail(c, MDS_E_STATE, "no posterior draw accumulated (mds_cv_accumulate)");
    if (draws) *draws = c->cv_draws;
    if (c->cv_m == 0) {
        *lpd = 0.0;
        return MDS_OK;
    }
    cv_finalize_launch(c->d_cv_max, c->d_cv_sum, c->cv_m, c->cv_draws, c->d_cv_out, c->stream);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(lpd, c->d_cv_out, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CKS(c->stream);
    return MDS_OK;
}

mds_status mds_sigma_mh_step(mds_ctx c, const mds_sigma_prior* prior, double step, double z, double u,
                             int32_t* accepted, double* log_ratio) {
    GUARD(c);
    return sigma_mh_impl(c, c->stream, prior, step, z, u, accepted, log_ratio, nullptr);
}

}  // extern "C"

namespace {
// One MH update of sigma^2 on stream s.  cur_ll_dev (nullable): a device double
// holding log L at the current X and sigma (the HMC driver's d_lik), which then
// replaces the likelihood-only pass at the current sigma.
mds_status sigma_mh_impl(mds_ctx c, cudaStream_t s, const mds_sigma_prior* prior, double step, double z, double u,
                         int32_t* accepted, double* log_ratio, const double* cur_ll_dev) {
    NvtxRange nv("mds_sigma_mh_step");
    if (!prior || !(prior->shape > 0.0) || !(prior->rate > 0.0) || !std::isfinite(prior->shape) ||
        !std::isfinite(prior->rate))
        return fail(c, MDS_E_INVALID_ARG, "sigma prior needs shape > 0 and rate > 0");
    if (!(step > 0.0) || !std::isfinite(step) || !std::isfinite(z) || !(u > 0.0) || !(u <= 1.0))
        return fail(c, MDS_E_INVALID_ARG, "need step > 0, finite z and u in (0, 1]");
    mds_status st = ready(c);
    if (st) return st;
    const double phi0 = 2.0 * std::log(c->sigma);          // phi = log sigma^2
    const double phi1 = phi0 + step * z;
    const double sigma1 = std::exp(0.5 * phi1);
    if (!sigma_ok(sigma1)) return fail(c, MDS_E_INVALID_ARG, "proposal sigma outside [1e-30, 1e30]");
    // log L at the current sigma: cached from the previous step when nothing changed,
    // or handed in by the HMC driver
    const bool need_cur = !cur_ll_dev && c->mh_version != c->version;
    if (need_cur) {
        st = run_lik_pass(c, c->P, c->d_lik + 2, s);
        if (st) return st;
    }
    st = run_lik_pass(c, sigma_params(sigma1), c->d_lik + 3, s);
    if (st) return st;
    double ll[2] = {c->mh_ll, 0.0};
    if (cur_ll_dev) CK(cudaMemcpyAsync(&ll[0], cur_ll_dev, sizeof(double), cudaMemcpyDeviceToHost, s));
    else if (need_cur) CK(cudaMemcpyAsync(&ll[0], c->d_lik + 2, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&ll[1], c->d_lik + 3, sizeof(double), cudaMemcpyDeviceToHost, s));
    CKS(s);
    // log prior of phi: tau = 1/sigma^2 = e^-phi ~ Gamma(shape, rate), Jacobian |dtau/dphi| = tau
    auto lp = [&](double phi) { return -prior->shape * phi - prior->rate * std::exp(-phi); };
    const double lr = (ll[1] - ll[0]) + (lp(phi1) - lp(phi0));
    const bool ok = std::isfinite(lr) && std::log(u) < lr;
    if (log_ratio) *log_ratio = lr;
    if (accepted) *accepted = ok ? 1 : 0;
    if (ok) {
        st = mds_set_sigma(c, sigma1);
        if (st) return st;
        c->mh_ll = ll[1];
    } else {
        c->mh_ll = ll[0];
    }
    c->mh_version = c->version;
    return MDS_OK;
}

SigmaParams sigma_params(double sigma) {
    const double pi = 3.14159265358979323846;
    SigmaParams P{};
    P.inv_sigma = 1.0 / sigma;
    P.inv_sigma2 = 1.0 / (sigma * sigma);
    P.half_inv_sigma2 = 0.5 / (sigma * sigma);
    P.k0 = -0.5 * std::log(2.0 * pi * sigma * sigma);
    P.cg = 1.0 / (sigma * std::sqrt(2.0 * pi));
    // the rational q = P/R in d: P_j / (cg sigma^j), R_j / sigma^j (sigma in [1e-30, 1e30]:
    // sigma^-7 stays normal); d clamped at TCLAMP64 sigma (high word, rounded up)
    {
        double sj = 1.0;
        for (int j = 0; j <= QR64_DEG; ++j) {
            if (j <= QP64_DEG) P.qp[j] = QP64_CH[j] / (P.cg * sj);
            P.qr[j] = QR64_CH[j] / sj;
            sj *= sigma;
        }
        const double dcl = TCLAMP64 * sigma;
        uint64_t bits;
        std::memcpy(&bits, &dcl, sizeof(bits));
        P.dclamp_hi = (int)(bits >> 32) + 1;
    }
    P.inv_sigma_f = (float)P.inv_sigma;
    P.inv_sigma2_f = (float)P.inv_sigma2;
    P.half_inv_sigma2_f = (float)P.half_inv_sigma2;
    P.k0_f = (float)P.k0;
    P.cg_f = (float)P.cg;
    P.ex2_slope_f = (float)(-1.4426950408889634 * P.half_inv_sigma2);
    return P;
}
}  // namespace

extern "C" {

mds_status mds_log_likelihood_and_gradient(mds_ctx c, double* loglik, double* grad) {
    GUARD(c);
    trace(c, "log_likelihood_and_gradient");
    mds_status st = eval_internal(c);
    if (st) return st;
    trace(c, "results copy");
    const size_t m = (size_t)(c->n * c->d);
    if (!c->h_ostage && cudaMallocHost(&c->h_ostage, (m + 1) * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        c->h_ostage = nullptr;
    }
    if (c->h_ostage) {   // device -> pinned at full PCIe rate, then one host copy (C5: 1.6 MB)
        if (loglik) CK(cudaMemcpyAsync(c->h_ostage + m, c->d_lik, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        if (grad) CK(cudaMemcpyAsync(c->h_ostage, c->d_grad, m * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CKS(c->stream);
        if (loglik) *loglik = c->h_ostage[m];
        if (grad) std::memcpy(grad, c->h_ostage, m * sizeof(double));
        return MDS_OK;
    }
    if (loglik) CK(cudaMemcpyAsync(loglik, c->d_lik, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (grad) CK(cudaMemcpyAsync(grad, c->d_grad, m * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CKS(c->stream);
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
    st = run_pass(c, c->d_x, grad_dev ? grad_dev : c->d_grad, loglik_dev ? loglik_dev : c->d_lik, false, 0.0, 0.0,
                  c->stream, true);
    if (st) return st;
    if (!grad_dev && !loglik_dev) c->eval_version = c->version;
    return MDS_OK;
}

mds_status mds_evaluate_partial_device(mds_ctx c, double* part_dev) {
    GUARD(c);
    if (!part_dev) return fail(c, MDS_E_INVALID_ARG, "NULL output");
    mds_status st = ready(c);
    if (st) return st;
    PassArgs a = base_args(c, c->d_x);
    a.grad = part_dev;
    a.lik = part_dev + c->n * c->d;
    return launch_coop(c, pass_fn_mode(MODE_EVAL, c->prec, c->trunc, c->d), a, c->stream);
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
    CKS(c->stream);
    return MDS_OK;
}

mds_status mds_get_momentum(mds_ctx c, double* p) {
    GUARD(c);
    if (!p) return fail(c, MDS_E_INVALID_ARG, "NULL output");
    CK(cudaMemcpyAsync(p, c->d_p, c->n * c->d * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CKS(c->stream);
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

// ---- fused peer-memory exchange (SURVEY 8(e) stage 2; include/mds.h)
namespace {
mds_status hmc_alloc(mds_ctx c);     // mds_hmc.inl
// Load every kernel a sharded context may launch.  With CUDA's lazy module loading
// the first launch of a kernel loads it, and loading waits for the device to go idle
// (measured: tools/lock_probe.cu) -- while a rank's pass kernel waits in the
// peer-memory exchange for a rank whose host thread is in exactly such a first
// launch (ranks sharing one GPU in one process), that is a deadlock.
void preload_kernels(mds_ctx c) {
    cudaFuncAttributes fa;
    const void* fs[] = {(const void*)prime_kernel, (const void*)redrift_kernel, (const void*)leapfrog_update_kernel,
                        (const void*)hamiltonian_kernel, (const void*)combine_update_kernel,
                        (const void*)combine_kernel, (const void*)p2p_allgather_kernel,
                        (const void*)count_obs_kernel<double>, (const void*)count_obs_kernel<float>,
                        (const void*)zero_pairs_kernel<double>, (const void*)zero_pairs_kernel<float>,
                        (const void*)row_fn(c->prec == MDS_F64, c->trunc, c->d)};
    for (const void* f : fs) cudaFuncGetAttributes(&fa, f);
    for (int m = 0; m < N_MODES; ++m) cudaFuncGetAttributes(&fa, (const void*)pass_fn_mode(m, c->prec, c->trunc, c->d).fn);
    rw_preload();
    tree_preload(c->d);
    cudaGetLastError();
}
}  // namespace

mds_status mds_p2p_window(mds_ctx c, void** window_dev, void* ipc_handle_out) {
    GUARD(c);
    if (c->world > P2P_MAX_WORLD) return fail(c, MDS_E_UNSUPPORTED, "mds_p2p_window: world > 32");
    if (!c->d_win) {
        const size_t m1 = (size_t)(c->n * c->d + 1);
        c->win_bytes = P2P_FLAG_BYTES + 2 * (size_t)c->world * m1 * sizeof(double);
        mds_status st;
        if ((st = dalloc(c, &c->d_win, c->win_bytes))) return st;
        if ((st = dalloc(c, &c->d_p2p_state, 4))) return st;
        if (!c->d_gathered && ((st = dalloc(c, &c->d_partial, m1)) || (st = dalloc(c, &c->d_gathered, m1 * c->world))))
            return st;      // (a world-1 context: the small exchanges gather here)
        CK(cudaMemsetAsync(c->d_win, 0, c->win_bytes, c->stream));
        CK(cudaMemsetAsync(c->d_p2p_state, 0, 4 * sizeof(unsigned long long), c->stream));
        CK(cudaHostAlloc((void**)&c->h_p2p_err, sizeof(int), cudaHostAllocMapped));
        *c->h_p2p_err = 0;
        CK(cudaHostGetDevicePointer((void**)&c->d_p2p_err, c->h_p2p_err, 0));
        // everything a sharded call would load or allocate lazily, now, before any rank
        // can be waiting in an exchange: a kernel's first launch (lazy module loading)
        // and a first cudaMalloc can wait for the whole device (ranks sharing one GPU
        // would deadlock; profiles/r02/p2p_probes.md)
        preload_kernels(c);
        if (const char* e = std::getenv("MDS_P2P_TIMEOUT_S")) {
            const double v = std::atof(e);
            if (v > 0) c->p2p_timeout_ns = (unsigned long long)(v * 1e9);
        }
        if ((st = rw_scratch(c, 3 * sizeof(double) * 8)) || (st = hmc_alloc(c)) ||
            (st = dalloc(c, &c->d_peer_win, (size_t)c->world)))
            return st;
        if (!c->h_pbuf && cudaMallocHost(&c->h_pbuf, (2 * (size_t)(c->n * c->d) + 2) * sizeof(double)) != cudaSuccess) {
            cudaGetLastError();
            c->h_pbuf = nullptr;
        }
        CKS(c->stream);
    }
    if (window_dev) *window_dev = c->d_win;
    if (ipc_handle_out) {
        cudaIpcMemHandle_t h;
        CK(cudaIpcGetMemHandle(&h, c->d_win));
        static_assert(sizeof(h) == MDS_IPC_HANDLE_BYTES, "cudaIpcMemHandle_t size");
        std::memcpy(ipc_handle_out, &h, sizeof(h));
    }
    return MDS_OK;
}

mds_status mds_p2p_connect(mds_ctx c, void* const* peer_window_dev) {
    GUARD(c);
    if (!peer_window_dev) return fail(c, MDS_E_INVALID_ARG, "mds_p2p_connect: NULL");
    if (!c->d_win) return fail(c, MDS_E_STATE, "mds_p2p_connect: call mds_p2p_window first");
    if (peer_window_dev[c->rank] != c->d_win)
        return fail(c, MDS_E_INVALID_ARG, "mds_p2p_connect: entry [rank] is not this context's window");
    int dev = 0;
    CK(cudaGetDevice(&dev));
    for (int r = 0; r < c->world; ++r) {
        if (!peer_window_dev[r]) return fail(c, MDS_E_INVALID_ARG, "mds_p2p_connect: NULL window");
        cudaPointerAttributes at{};
        CK(cudaPointerGetAttributes(&at, peer_window_dev[r]));
        if (at.type == cudaMemoryTypeDevice && at.device != dev) {      // a window on another GPU
            int ok = 0;
            CK(cudaDeviceCanAccessPeer(&ok, dev, at.device));
            if (!ok) return fail(c, MDS_E_UNSUPPORTED, "mds_p2p_connect: no peer access to device " +
                                                           std::to_string(at.device));
            const cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else CK(e);
        }
    }
    if (!c->d_peer_win) return fail(c, MDS_E_STATE, "mds_p2p_connect: call mds_p2p_window first");
    CK(cudaMemcpyAsync(c->d_peer_win, peer_window_dev, c->world * sizeof(char*), cudaMemcpyHostToDevice, c->stream));
    CKS(c->stream);
    c->p2p = true;
    // handshake: one peer all-gather of (rank + 1) through the windows, checked on the
    // host, with a 30 s wait at most -- a broken path (IPC mapping, peer access) fails
    // here with MDS_E_COMM instead of inside a pass
    {
        const unsigned long long keep = c->p2p_timeout_ns;
        c->p2p_timeout_ns = std::min<unsigned long long>(keep, 30000000000ull);
        double* send = c->d_partial;
        double* recv = c->d_gathered;
        const double me = (double)(c->rank + 1);
        CK(cudaMemcpyAsync(send, &me, sizeof(double), cudaMemcpyHostToDevice, c->stream));
        p2p_allgather_kernel<<<1, 32, 0, c->stream>>>(p2p_args(c), send, 1, recv);
        CK(cudaGetLastError());
        std::vector<double> got(c->world, 0.0);
        CK(cudaMemcpyAsync(got.data(), recv, c->world * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        const cudaError_t e = cudaStreamSynchronize(c->stream);
        c->p2p_timeout_ns = keep;
        const bool timed_out = *(volatile int*)c->h_p2p_err != 0;
        bool ok = e == cudaSuccess && !timed_out;
        std::string seen;
        for (int r = 0; r < c->world; ++r) {
            ok = ok && got[r] == (double)(r + 1);
            seen += (r ? " " : "") + std::to_string(got[r]);
        }
        if (!ok) {
            c->p2p = false;
            *c->h_p2p_err = 0;
            if (e != cudaSuccess) return fail(c, MDS_E_CUDA, std::string("peer handshake: ") + cudaGetErrorString(e));
            return fail(c, MDS_E_COMM, std::string("peer-memory handshake failed (") +
                                           (timed_out ? "a peer did not answer in time" : "wrong values") +
                                           "; rank slots read: " + seen + "); the context keeps its other exchange");
        }
    }
    return MDS_OK;
}

mds_status mds_p2p_disconnect(mds_ctx c) {
    GUARD(c);
    CKS(c->stream);
    c->p2p = false;
    return MDS_OK;
}

mds_status mds_p2p_connect_ipc(mds_ctx c, const void* ipc_handles) {
    GUARD(c);
    if (!ipc_handles) return fail(c, MDS_E_INVALID_ARG, "mds_p2p_connect_ipc: NULL");
    if (!c->d_win) return fail(c, MDS_E_STATE, "mds_p2p_connect_ipc: call mds_p2p_window first");
    std::vector<void*> w(c->world, nullptr);
    for (int r = 0; r < c->world; ++r) {
        if (r == c->rank) {
            w[r] = c->d_win;
            continue;
        }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const char*>(ipc_handles) + (size_t)r * MDS_IPC_HANDLE_BYTES, sizeof(h));
        void* q = nullptr;
        CK(cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess));
        c->ipc_opened.push_back(q);
        w[r] = q;
    }
    return mds_p2p_connect(c, w.data());
}

mds_status mds_p2p_connected(mds_ctx c, int32_t* connected) {
    GUARD(c);
    if (!connected) return MDS_E_INVALID_ARG;
    *connected = c->p2p ? 1 : 0;
    return MDS_OK;
}

mds_status mds_set_grid_limit(mds_ctx c, int32_t ctas) {
    GUARD(c);
    if (ctas < 0) return fail(c, MDS_E_INVALID_ARG, "mds_set_grid_limit: ctas < 0");
    CKS(c->stream);                      // the old schedule may still be in use
    c->grid_limit = ctas;
    return build_schedule(c);
}

mds_status mds_observed_pairs(mds_ctx c, int64_t* count) {
    GUARD(c);
    if (!count) return fail(c, MDS_E_INVALID_ARG, "NULL output");
    mds_status st = count_obs(c);
    if (st) return st;
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
        if (c->prec == MDS_F64)
            zero_pairs_kernel<double><<<c->ntl, 256, 0, c->stream>>>((const double*)c->d_y, c->d_x, c->d_tiles, c->d,
                                                                     c->d_count);
        else
            zero_pairs_kernel<float><<<c->ntl, 256, 0, c->stream>>>((const float*)c->d_y, c->d_x, c->d_tiles, c->d,
                                                                    c->d_count);
        CK(cudaGetLastError());
    }
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, c->d_count, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    CKS(c->stream);
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
    report_phases(c);
    if (pair_ms) *pair_ms = passes ? (float)(sp / passes) : 0.f;
    if (reduce_ms) *reduce_ms = passes ? (float)(sr / passes) : 0.f;
    return MDS_OK;
}

mds_status mds_plan(int64_t n, int32_t rank, int32_t world, int32_t ctas, int32_t warps_per_cta, mds_plan_info* info,
                    uint8_t* owned_rows) {
    if (n < 2 || world < 1 || rank < 0 || rank >= world || ctas < 1 || warps_per_cta < 1 || !info ||
        (n + TB - 1) / TB > 0xffff)
        return MDS_E_INVALID_ARG;
    Plan P;
    std::string why;
    if (!make_plan(n, rank, world, ctas, warps_per_cta, P, &why)) return MDS_E_UNSUPPORTED;
    if (!check_plan(P, &why)) return MDS_E_STATE;
    mds_plan_info r{};
    int64_t pairs = 0;
    for (int I = 0; I < P.nb; ++I) {
        if (P.row_local[I] < 0) continue;
        ++r.tile_rows;
        for (int64_t i = (int64_t)I * TB; i < std::min<int64_t>(n, (int64_t)(I + 1) * TB); ++i) pairs += i;
    }
    if (owned_rows)
        for (int64_t i = 0; i < n; ++i) owned_rows[i] = P.row_local[i / TB] >= 0 ? 1 : 0;
    r.tiles = (int64_t)P.tiles.size();
    r.pair_slots = r.tiles * TB * TB;
    r.pairs = pairs;
    r.segments = (int64_t)P.segs.size();
    r.slabs = r.segments + r.tiles;
    int64_t mx = 0, umin = INT64_MAX, umax = 0;
    for (int b = 0; b < P.nb; ++b) mx = std::max<int64_t>(mx, P.ptr[b + 1] - P.ptr[b]);
    const int64_t GW = (int64_t)ctas * warps_per_cta, U = (int64_t)GROUPS_PER_TILE * r.tiles;
    const int64_t V = GW * P.vpw;
    for (int64_t w = 0; w < GW; ++w) {
        const int64_t u = (U * (w + 1) * P.vpw) / V - (U * w * P.vpw) / V;
        umin = std::min(umin, u);
        umax = std::max(umax, u);
    }
    r.max_slabs_per_block = mx;
    r.min_units_per_warp = umin;
    r.max_units_per_warp = umax;
    r.ranges_per_warp = P.vpw;
    *info = r;
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

mds_status mds_l2_flush(mds_ctx c, void* dev_buf, size_t bytes) {
    if (!c || !dev_buf || bytes < 16) return MDS_E_INVALID_ARG;
    static size_t attr_set = 0;      // largest dynamic shared memory enabled so far (contexts differ)
    if (c->smem > attr_set) {
        if (cudaFuncSetAttribute(l2_flush_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem))
            return fail(c, MDS_E_CUDA, "l2_flush attribute");
        attr_set = c->smem;
    }
    l2_flush_kernel<<<c->grid, 32 * c->wpc, c->smem, c->stream>>>((uint4*)dev_buf, bytes / 16, 0x3c3c3c3cu);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? MDS_OK : fail(c, MDS_E_CUDA, cudaGetErrorString(e));
}

mds_status mds_l2_flush_clean(mds_ctx c, void* dev_buf, size_t bytes) {
    if (!c || !dev_buf || bytes < 32) return MDS_E_INVALID_ARG;
    const size_t half = (bytes / 2) & ~(size_t)15;
    mds_status st = mds_l2_flush(c, dev_buf, half);
    if (st) return st;
    static size_t attr_set = 0;
    if (c->smem > attr_set) {
        if (cudaFuncSetAttribute(l2_read_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->smem))
            return fail(c, MDS_E_CUDA, "l2_flush attribute");
        attr_set = c->smem;
    }
    l2_read_kernel<<<c->grid, 32 * c->wpc, c->smem, c->stream>>>((const uint4*)((char*)dev_buf + half), half / 16,
                                                                   (unsigned*)dev_buf);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? MDS_OK : fail(c, MDS_E_CUDA, cudaGetErrorString(e));
}

mds_status mds_measure_fma_peaks(double* fp64, double* fp32) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return MDS_E_UNSUPPORTED;
    }
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* d_out = nullptr;
    if (cudaMalloc(&d_out, 16) != cudaSuccess) return MDS_E_OOM;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int threads = 256, blocks = sms * 8, iters = 4096;
    float best64 = 1e30f, best32 = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        float ms = 0.f;
        cudaEventRecord(a);
        fma_peak_kernel<double><<<blocks, threads>>>(d_out, iters, 0.999999, 1e-9);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
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
    if (e != cudaSuccess) return MDS_E_CUDA;
    const double lanes = (double)blocks * threads * 64.0;
    if (fp64) *fp64 = lanes * iters / (best64 * 1e-3);
    if (fp32) *fp32 = lanes * iters * 4 / (best32 * 1e-3);
    return MDS_OK;
}

}  // extern "C"

#include "mds_hmc.inl"
