// mds_pass.cuh -- the sm_100a pass kernel of the fused MDS likelihood+gradient pass.
// (Instantiated per mode and precision in pass_m<MODE>_<prec>.cu; the helper
// kernels live in mds_kernels.cuh.)
//
// Data layout in HBM:
//   Y   : the strict lower triangle cut into B x B tiles (I, J), I >= J, B = 64.
//         Only this rank's tile-rows are stored, tile-major in (I, J) order;
//         inside a tile the layout is column-major, y(ii, jj) at [jj*B + ii], so
//         the 32 lanes of a warp (consecutive rows) read one 256 B line per column.
//         Slots that are not an observed pair (missing y, i <= j in diagonal
//         tiles, padding rows/columns >= n) hold the canonical NaN, so the pair
//         loop has no bounds or i > j test.
//   X   : fp64 master, n_pad x D row-major, padding rows zero (plus p, grad log pi
//         and the drifted X of the next leapfrog step, same layout).
//   slab: B x D fp64 partial sums. Slabs [0, S) are row-segment partials, slabs
//         [S, S + ntl) the column partials of each local tile.
//
// ONE persistent cooperative kernel per pass:
//   phase A  grid = resident CTAs; CTA c owns the column-group units
//            [c U/G, (c+1) U/G) of the tile list (U = 16 column-groups x tiles),
//            cut into tile-row segments.  Warp w of the CTA takes units w, w+4, ..
//            of a segment; lane l evaluates rows l and l+32 against the 4 columns
//            of a unit: 8 pairs, Eq. 2 term and Eq. 6 coefficient each.  Row sums
//            stay in registers for the whole segment (Alg. 2's per-row reduction,
//            PAPER.md:786-805); the column side (each unordered pair is computed
//            once, so it is new) is summed over the 64 rows by a 2-row add + a
//            4-column reduce-scatter and stored once per column; log L partials
//            per CTA (Alg. 1's binary tree).  No atomics.
//   barrier  cooperative grid sync.
//   phase B  fixed-order reduction: g_i = sum of the row-segment slabs and column
//            slabs touching row block i/B (CSR built on the host), then either
//            the result (EVAL), the sharded partial (PARTIAL), or the leapfrog
//            update (LEAPFROG: second half-kick, next drift).  CTA 0 sums log L.
#pragma once
#include <cooperative_groups.h>
#include <cstdint>
#include <type_traits>
#include "mds_math.cuh"
#include "mds_tree_impl.cuh"

namespace mdsk {
namespace cg = cooperative_groups;

constexpr int TB = 64;              // tile edge B
constexpr int GROUPS_PER_TILE = TB / 4;     // 4-column groups per tile: the schedule's granule
constexpr int PT = 128;             // threads per CTA of the small helper kernels

// What one pass computes (template parameter MODE of pass_kernel):
//   EVAL            log L and gradient (Eq. 2 + Eq. 6)
//   EVAL_NOLIK      gradient only (sharded leapfrog steps that need no log L)
//   LEAPFROG        log L, gradient and the leapfrog update (Eq. 5)
//   LEAPFROG_NOLIK  gradient + leapfrog update: steps 1..L-1 of a trajectory,
//                   whose log L nobody reads
//   LIK             log L only, at the SigmaParams passed (sigma-side sweep for
//                   the MH update of sigma^2; no gradient, no slabs)
//   LEAPFROG_TREE, LEAPFROG_NOLIK_TREE
//                   the leapfrog modes under the phylogenetic prior: the grid's
//                   last CTA walks the tree during phase A
//   EVAL_TREE, EVAL_NOLIK_TREE
//                   sharded leapfrog steps under the phylogenetic prior: the rank's
//                   partial (EVAL) while the last CTA walks the tree into gprior; the
//                   leapfrog update follows the exchange (combine_update_kernel)
enum Mode {
    MODE_EVAL = 0, MODE_EVAL_NOLIK = 1, MODE_LEAPFROG = 2, MODE_LEAPFROG_NOLIK = 3, MODE_LIK = 4,
    MODE_LEAPFROG_TREE = 5, MODE_LEAPFROG_NOLIK_TREE = 6, MODE_EVAL_TREE = 7, MODE_EVAL_NOLIK_TREE = 8
};
constexpr int N_MODES = 9;
template <int MODE> struct ModeTraits {
    static constexpr bool TREE = MODE == MODE_LEAPFROG_TREE || MODE == MODE_LEAPFROG_NOLIK_TREE ||
                                 MODE == MODE_EVAL_TREE || MODE == MODE_EVAL_NOLIK_TREE;
    static constexpr bool LF = MODE == MODE_LEAPFROG || MODE == MODE_LEAPFROG_NOLIK ||
                               MODE == MODE_LEAPFROG_TREE || MODE == MODE_LEAPFROG_NOLIK_TREE;   // leapfrog update
    static constexpr bool WL = !(MODE == MODE_EVAL_NOLIK || MODE == MODE_LEAPFROG_NOLIK ||
                                 MODE == MODE_LEAPFROG_NOLIK_TREE || MODE == MODE_EVAL_NOLIK_TREE);   // log L wanted
    static constexpr bool WG = MODE != MODE_LIK;                                            // gradient wanted
};

template <typename T, bool TRUNC> struct Pair;
template <bool TRUNC> struct Pair<double, TRUNC> {
    // l is in/out: the caller's running sums; each gets its pair's Eq. 2 term
    // without the constant -1/2 log(2 pi sigma^2) (added as n_obs k0 at the end)
    template <bool WL, bool WG>
    __device__ __forceinline__ static void eval4(const double (&s)[4], const double (&y)[4], const SigmaParams& P,
                                                 const double* exptab, double (&l)[4], double (&u)[4]) {
        pair_f64_n<TRUNC, 4, WL, WG, true>(s, y, P, exptab, l, u);
    }
};
template <bool TRUNC> struct Pair<float, TRUNC> {
    template <bool WL, bool WG>
    __device__ __forceinline__ static void eval4(const float (&s)[4], const float (&y)[4], const SigmaParams& P,
                                                 const double*, float (&l)[4], float (&u)[4]) {
#pragma unroll
        for (int i = 0; i < 4; ++i) pair_f32<TRUNC, WL, WG>(s[i], y[i], P, l[i], u[i]);
    }
};

template <typename T>
__device__ __forceinline__ T shfl_xor(T v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }

// Sum over the 32 lanes of 4 per-lane column values stored in the per-lane
// order v[p] = column p ^ m, m = (L >> 3) & 3 (see the unit loop): every
// exchange then sends a fixed register, so no selects are needed.  Lane L ends
// with the total of column m (all 8 lanes with the same m hold it).  Fixed order.
template <typename T>
__device__ __forceinline__ T reduce_scatter4_perm(T v0, T v1, T v2, T v3) {
    T k0 = v0 + shfl_xor(v2, 16);     // partner L^16 holds my columns 0,1 at its positions 2,3
    T k1 = v1 + shfl_xor(v3, 16);
    T k = k0 + shfl_xor(k1, 8);       // partner L^8 holds my column 0 at its position 1
    k += shfl_xor(k, 4);
    k += shfl_xor(k, 2);
    k += shfl_xor(k, 1);
    return k;
}

// leapfrog drift of one coordinate: x + eps (p + eps/2 gl); the same expression
// (and rounding) wherever it is evaluated
__device__ __forceinline__ double drift(double x, double p, double gl, double eps, double heps) {
    return __fma_rn(eps, __fma_rn(heps, gl, p), x);
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// ------------------------------------------------------------ peer-memory exchange
// Window of every rank (device memory, mds_p2p_window): 32 arrival flags (uint64,
// flag r = the number of exchanges rank r has pushed into this window), then
// recv[2][world][m + 1] doubles (m = n d; slot parity = exchange count & 1).
// state (local, not in the window): [0] exchanges done, [1] CTAs done pushing,
// [2] CTAs done combining.  err: host-mapped word, set to 1 on a 60 s timeout.
constexpr int P2P_MAX_WORLD = 32;
constexpr size_t P2P_FLAG_BYTES = P2P_MAX_WORLD * sizeof(unsigned long long);
struct P2PArgs {
    char* const* win;               // [world] window base addresses (device array); NULL = no P2P
    unsigned long long* state;      // local counters
    int* err;                       // host-mapped error word
    int rank, world;
    int64_t m1;                     // slot length m + 1
    unsigned long long timeout_ns;  // give up waiting for a peer after this long
};
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long p2p_epoch(const P2PArgs& q) {
    return *reinterpret_cast<volatile unsigned long long*>(q.state);
}
// receive area of window w for the exchange ep: [world][m1]
__device__ __forceinline__ double* p2p_recv(const P2PArgs& q, char* w, unsigned long long ep) {
    return reinterpret_cast<double*>(w + P2P_FLAG_BYTES) + (size_t)(ep & 1) * q.world * q.m1;
}
// value e of this rank's partial -> slot [rank][e] of every rank's window (remote stores)
__device__ __forceinline__ void p2p_push(const P2PArgs& q, unsigned long long ep, int64_t e, double v) {
    for (int r = 0; r < q.world; ++r) p2p_recv(q, q.win[r], ep)[(size_t)q.rank * q.m1 + e] = v;
}
// thread 0 of each of `ctas` CTAs, after the CTA's pushes: count the CTA in; the
// last raises this rank's flag in every window; then wait for every rank's flag
__device__ __forceinline__ void p2p_arrive_and_wait(const P2PArgs& q, unsigned long long ep, unsigned ctas) {
    __threadfence_system();                                // this CTA's remote stores, system-wide
    if (atomicAdd(&q.state[1], 1ull) == ctas - 1) {
        q.state[1] = 0;                                    // (reset for the next exchange)
        __threadfence_system();
        for (int r = 0; r < q.world; ++r)
            st_release_sys(reinterpret_cast<unsigned long long*>(q.win[r]) + q.rank, ep + 1);
    }
    const unsigned long long* fl = reinterpret_cast<const unsigned long long*>(q.win[q.rank]);
    const unsigned long long t0 = gtimer();
    for (int r = 0; r < q.world; ++r) {
        while (ld_acquire_sys(fl + r) < ep + 1) {
            if (gtimer() - t0 > q.timeout_ns) {           // a peer never arrived: give up, report
                *reinterpret_cast<volatile int*>(q.err) = 1;
                return;
            }
        }
    }
}
// thread 0 of each CTA at the end of the combine: the last advances the exchange count
__device__ __forceinline__ void p2p_finish(const P2PArgs& q, unsigned long long ep, unsigned ctas) {
    if (atomicAdd(&q.state[2], 1ull) == ctas - 1) {
        q.state[2] = 0;
        q.state[0] = ep + 1;
    }
}

// grid-wide barrier of a co-resident grid (thread 0 of each CTA between two
// __syncthreads): the last arriving CTA resets the count and advances the generation
__device__ __forceinline__ void grid_barrier(unsigned* b, unsigned ctas) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = b + 1;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(b, 1u) == ctas - 1) {
            b[0] = 0;
            __threadfence();
            atomicExch(b + 1, g + 1);
        } else {
            while (*gen == g) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

struct PassArgs {
    // inputs
    const void* y;               // local tiles [ntl][B][B]
    const double* xeval;         // positions the pass evaluates at (n_pad x D)
    // schedule (per global warp gw = blockIdx.x * 4 + warp)
    const int* warp_seg;         // [GW + 1] segment range per warp
    const int4* segs;            // [S] (I, u0, u1, tbase): tile-row, unit range, local index of tile (I, 0)
    const int* blk_ptr;          // [nb + 1] slabs of row block b: storage rows [blk_ptr[b], blk_ptr[b+1])
    const int* slab_pos;         // [S + ntl] storage row of segment s's row slab (s) and of
                                 // local tile t's column slab (S + t): block-contiguous order
    int nseg;                    // S
    int nb;
    int64_t n;
    // scratch
    double* slabs;               // (S + ntl) x B x D
    double* likpart;             // [GW]
    // outputs
    double* grad;                // EVAL: d log L / dX (n x D)      (sharded: this rank's partial)
    double* lik;                 // log L                           (sharded: partial)
    // leapfrog state (MODE_LEAPFROG): x <- xeval, p, gl updated, xnext written
    double* x;
    double* p;
    double* gl;
    double* xnext;
    double eps, heps, inv_tau2;
    const double* gprior;        // LEAPFROG: d log prior / dX at xeval (tree prior), or NULL = iid N(0, 1/inv_tau2)
    int pair_ctas;               // CTAs [0, pair_ctas) run phase A (the plan's CTA count)
    TreeArgs tree;               // *_TREE modes: the tree prior walked by CTA gridDim.x - 1 during phase A
                                 //   (its x = xeval, its grad = gprior)
    int vpw;                     // virtual unit ranges per warp (warp_seg has GW * vpw + 1 entries)
    int epl;                     // phase B: slab elements per lane (1, 2 or 4)
    SigmaParams P;
    double lik_const;            // added to log L: n_obs x P.k0 (fp64 pass), 0 (fp32 pass)
    unsigned long long* prof;    // optional [G][4] globaltimer stamps (start, end A, after sync, end)
    // fused peer-memory exchange (sharded contexts after mds_p2p_connect; EVAL* / LIK modes):
    // phase B pushes this rank's partial into every rank's window, then phase C combines
    // the world partials in rank order into grad / lik (and, p2p_lf, the leapfrog update)
    P2PArgs p2p;
    int p2p_lf;
    unsigned* gbar;              // [2] software grid barrier: arrivals, generation
    int soft_sync;               // 1: launched without the cooperative attribute -> gbar, not grid.sync
};


constexpr int MAXSEG_W = 32;    // segments per warp (host checks)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
// TMA bulk copy global -> shared (SASS UBLKCP), completion counted on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(b))
                 : "memory");
}
// the same with an L2 cache-policy hint (Y is streamed once per pass: evict-first
// keeps X and the partial-sum slabs resident in L2 for phase B)
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* b, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
            smem_u32(b)),
        "r"(parity)
        : "memory");
}
// one try_wait probe (profiling: was the stage already complete?)
__device__ __forceinline__ bool mbar_ready(uint64_t* b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// programmatic dependent launch: wait for the preceding grid of the stream (a no-op
// when the launch was not programmatic), and let the next grid be scheduled
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// per-warp staging area (dynamic shared memory).  One TMA bulk copy per unit
// brings its UCOLS tile columns of y (NSTAGE-deep ring); x of the tile's 64
// columns is copied once per tile into xcol[t & 1].  x of the segment's 64
// rows is read straight into registers at the segment start.
constexpr int NSTAGE = 2;        // y stages per warp (the next unit is in flight)

// Warps per CTA and tile columns per unit (one bulk copy each; a multiple of
// the 4-column reduce group).  ONE CTA per SM with as many warps as the register
// file holds: warps of one CTA progress evenly, while several CTAs per SM drift
// apart by up to ~1.6x (issue arbitration; measured with MDS_PROFILE_PHASES),
// which a grid barrier turns into idle time.  Warps per CTA bound the registers
// per thread (ptxas budgets blocks in 4-warp granules: 16 warps -> 128 regs,
// 12 -> 168, 8 -> 255); fp64 needs ~128-150 for 4 interleaved pairs
// (tools/pair_probe.cu), more at larger D.  Wider units halve the per-unit
// issue/wait overhead where the 2-stage ring still fits shared memory.
template <typename T, int D> struct KernelShape {
    // fp64: 16-column units (8 KB copies) wherever 2 stages fit: D <= 2 at 12
    // warps (A/B on one box vs 8-column units at 16 warps: 150.0 vs 144.6 G
    // pair-evals/s on C2), D >= 4 at 8 warps; D = 3 keeps 8-column units
    static constexpr int wpc = sizeof(T) == 8 ? (D <= 3 ? 12 : 8) : (D <= 2 ? 24 : (D <= 6 ? 16 : 12));
    static constexpr int ucols = (sizeof(T) == 8 && D != 3) ? 16 : 8;
};
template <typename T, int D> struct WarpsPerCTA { static constexpr int value = KernelShape<T, D>::wpc; };

template <typename T, int D>
struct alignas(16) WarpStage {
    static constexpr int UC = KernelShape<T, D>::ucols;
    uint64_t bar[NSTAGE];
    uint64_t bar0[4];                       // the kernel's first unit: one barrier per 4-column group
    alignas(16) double xcol[2][TB * D];     // bulk-copy destinations: 16-byte aligned
    alignas(16) T y[NSTAGE][UC * TB];
    // fp32 pass: the tile's column x converted once per tile (not per pair)
    alignas(16) std::conditional_t<sizeof(T) == 4, float[2][TB * D], float[1]> xcolf;
    int4 seg[MAXSEG_W];
    int spos[MAXSEG_W];                     // storage rows of the segments' row slabs
};

template <typename T, int D>
constexpr size_t pass_smem_bytes() { return WarpsPerCTA<T, D>::value * sizeof(WarpStage<T, D>); }
// dynamic staging + the static reduction buffers must fit the 227 KB of one CTA
// (phase B reuses the staging area for its 4 x warps x 32 partial sums)
static_assert(pass_smem_bytes<double, 8>() + EXPT64_N * 8 + 512 <= 227 * 1024, "smem");
static_assert(pass_smem_bytes<double, 4>() + EXPT64_N * 8 + 512 <= 227 * 1024, "smem");
static_assert(pass_smem_bytes<float, 8>() + EXPT64_N * 8 + 512 <= 227 * 1024, "smem");
static_assert(pass_smem_bytes<float, 6>() + EXPT64_N * 8 + 512 <= 227 * 1024, "smem");
static_assert(pass_smem_bytes<float, 2>() + EXPT64_N * 8 + 512 <= 227 * 1024, "smem");
static_assert(pass_smem_bytes<double, 3>() + EXPT64_N * 8 + 512 <= 227 * 1024, "smem");
static_assert(pass_smem_bytes<double, 2>() + EXPT64_N * 8 + 512 <= 227 * 1024, "smem");
static_assert(pass_smem_bytes<double, 1>() + EXPT64_N * 8 + 512 <= 227 * 1024, "smem");
static_assert(pass_smem_bytes<float, 1>() + EXPT64_N * 8 + 512 <= 227 * 1024, "smem");
static_assert(sizeof(WarpStage<float, 1>) >= 4 * 32 * sizeof(double), "phase B buffer");

template <typename T, int D, bool TRUNC, int MODE>
__global__ void __launch_bounds__(WarpsPerCTA<T, D>::value * 32, 1)
pass_kernel(PassArgs a) {
    using A = double;
    constexpr bool LF = ModeTraits<MODE>::LF, WL = ModeTraits<MODE>::WL, WG = ModeTraits<MODE>::WG;
    constexpr bool TREE = ModeTraits<MODE>::TREE;
    constexpr int WPC = WarpsPerCTA<T, D>::value;
    constexpr int UCOLS = KernelShape<T, D>::ucols;     // tile columns per unit
    constexpr int GPU = UCOLS / 4;                      // 4-column groups per unit
    constexpr int UNITS_PER_TILE = TB / UCOLS;
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ double exptab[EXPT64_N];
    __shared__ uint64_t pb_bar;              // phase B: one bulk copy of a block's slabs
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gw = blockIdx.x * WPC + warp;
    WarpStage<T, D>& W = reinterpret_cast<WarpStage<T, D>*>(dsm)[warp];
    const T* __restrict__ Y = static_cast<const T*>(a.y);
    const double* __restrict__ X = a.xeval;
    constexpr uint32_t YB = UCOLS * TB * sizeof(T), XB = TB * D * sizeof(double);

    // ------------------------------------------------------------ phase A (per warp)
    // a warp's contiguous unit range is processed as vpw consecutive virtual
    // ranges of at most MAXSEG_W segments each (their segment table fits smem).
    // (Issuing the first unit's copy from the range bounds before the segment
    // tables arrive measured 1.4% slower: A/B on one box, 146.9 vs 148.4.)
    if (lane == 0) {
#pragma unroll
        for (int b = 0; b < NSTAGE; ++b) mbar_init(&W.bar[b], 1);
#pragma unroll
        for (int b = 0; b < 4; ++b) mbar_init(&W.bar0[b], 1);
        if (warp == 0) mbar_init(&pb_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_async_smem();
    }
    // The exp table (cg 2^(j/256), built per launch) is only needed once compute
    // starts: pair CTAs build it after their first TMA copies are in flight (the
    // first data lands ~2 us after issue); the tree CTA and the tree modes' pair
    // CTAs (tips pass first) build it here.
    const bool skip_a = blockIdx.x >= a.pair_ctas;
    const bool early_tab = TREE || skip_a || a.vpw < 1;
    if (early_tab) {
        build_exptab(exptab, a.P);
        __syncthreads();
        pdl_wait();      // (everything below may read the previous step's results)
    }
    if (a.prof && threadIdx.x == 0) a.prof[blockIdx.x * 4 + 0] = gtimer();
    const bool p2p = !LF && a.p2p.win != nullptr;
    A lik_w = A(0);
    A lacc[4] = {A(0), A(0), A(0), A(0)};   // fp64: running log L sums by lock-step position

#ifndef MDS_Y_NO_EVICT_FIRST
    const uint64_t ypol = policy_evict_first();
#endif
    // With a tree prior, the last CTA walks the tree (d log prior / dX at xeval,
    // PAPER.md:243-246) while the others run phase A; the grid barrier below
    // orders phase B's leapfrog update after both.
    if (TREE && !skip_a) {
        // this CTA's slice of the tree walk's tips pass (a few tips per CTA), then check in
        const int per = (a.tree.n_items + a.pair_ctas - 1) / a.pair_ctas;
        const int lo = min(a.tree.n_items, (int)blockIdx.x * per), hi = min(a.tree.n_items, lo + per);
        treek::tips_pass<D>(a.tree, lo, hi, threadIdx.x, WPC * 32);
        // ... and this CTA's slice of the walk's first level (cherries: tip children only)
        const int e_all = a.tree.n_up > 0 ? __ldg(a.tree.up_lvl_ptr + 1) : 0;
        const int pe = (e_all + a.pair_ctas - 1) / a.pair_ctas;
        const int elo = min(e_all, (int)blockIdx.x * pe), ehi = min(e_all, elo + pe);
        treek::level0_slice<D>(a.tree, elo, ehi, threadIdx.x, WPC * 32);
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(a.tree.tips_done, 1u);
        }
    }
    if (TREE && blockIdx.x == gridDim.x - 1)
        treek::tree_prior_block<D, WPC * 32>(a.tree, reinterpret_cast<double*>(dsm), exptab);
    unsigned not_ready = 0;                  // profiling: units whose data had not landed yet
    uint32_t phase = 0;                      // bit b: parity of stage b (persists across ranges)
    int cst = 0;                             // stage of the next unit to compute
#pragma unroll 1
    for (int vv = 0; vv < (skip_a ? 0 : a.vpw); ++vv) {
    const int vw = gw * a.vpw + vv;
    const int ws0 = a.warp_seg[vw], ws1 = a.warp_seg[vw + 1];
    const int nsw = ws1 - ws0;
    __syncwarp();
    if (lane < nsw) {
        W.seg[lane] = a.segs[ws0 + lane];
        W.spos[lane] = __ldg(a.slab_pos + ws0 + lane);
    }
    __syncwarp();
    {
        // segments are in 4-column groups (g); the warp works in UCOLS-column units
        // u = g / GPU, whose first/last may be partly outside the warp's range
        // (an empty range, nsw == 0, reads stale table entries that are never used)
        const int ub = W.seg[0].y / GPU, ue = (W.seg[max(nsw, 1) - 1].z + GPU - 1) / GPU;
        // the lane index from a volatile read: ptxas cannot rematerialise it (it re-read
        // SR_TID.X at the top of every group, a short-scoreboard wait in front of the
        // column-x loads: +0.7% pair throughput, A/B at N = 30000)
        int lane_v;
        asm volatile("mov.u32 %0, %%laneid;" : "=r"(lane_v));
        const int m = (lane_v >> 3) & 3;         // this lane's column order: position p <-> column p ^ m
        // issue cursor: units are staged in order, NSTAGE - 1 ahead of compute; tile t's
        // column x goes to xcol[t & 1] (consecutive tiles alternate)
        int iu = ub, isi = 0, iend = (W.seg[0].z + GPU - 1) / GPU, itb = W.seg[0].w, ist = cst;
        auto issue_one = [&]() {
            if (iu >= iend) {
                ++isi;
                iend = (W.seg[isi].z + GPU - 1) / GPU;
                itb = W.seg[isi].w;
            }
            const int t = iu / UNITS_PER_TILE, jj0 = (iu % UNITS_PER_TILE) * UCOLS;
            const bool nt = (iu % UNITS_PER_TILE == 0) || iu == ub;
            if (lane == 0) {
                // WAR on the stage (generic LDS reads of the unit before, async-proxy
                // writes now) is ordered by the __syncwarp after the wait below, as in
                // an mbarrier consumer-release / producer-acquire pipeline: no proxy
                // fence (it compiles to MEMBAR.ALL.CTA, which waits for this lane's
                // outstanding column-slab stores)
                mbar_arrive_tx(&W.bar[ist], YB + (nt ? XB : 0));
#ifndef MDS_Y_NO_EVICT_FIRST
                bulk_g2s_hint(W.y[ist], Y + (size_t)t * TB * TB + (size_t)jj0 * TB, YB, &W.bar[ist], ypol);
#else
                bulk_g2s(W.y[ist], Y + (size_t)t * TB * TB + (size_t)jj0 * TB, YB, &W.bar[ist]);
#endif
                if (nt) bulk_g2s(W.xcol[t & 1], X + (size_t)(t - itb) * TB * D, XB, &W.bar[ist]);
            }
            ++iu;
            ist = (ist + 1 == NSTAGE) ? 0 : ist + 1;
        };
        // Staggered start: at launch every warp's first copy competes for HBM, so the
        // kernel's first unit is fetched group by group -- the first 4-column group
        // alone (2 KB + the tile's x), the rest once it has landed -- and compute
        // starts on ~1/4 of the start-up traffic.
#ifdef MDS_NO_STAGGER
        bool first_pending = false;
#else
        bool first_pending = vv == 0;
#endif
        const int fc4b = max(W.seg[0].y - GPU * ub, 0), fc4e = min(W.seg[0].z - GPU * ub, GPU);
        const int fst = ist;                     // the first unit's stage
        // xmode: 0 = y only, 1 = y and the tile's x, 2 = y now, x later (counted now)
        auto issue_group = [&](int g, int xmode) {
            const bool with_x = xmode == 1;
            const int t = ub / UNITS_PER_TILE, jj0 = (ub % UNITS_PER_TILE) * UCOLS;
            constexpr uint32_t GB = 4 * TB * sizeof(T);
            mbar_arrive_tx(&W.bar0[g], GB + (xmode ? XB : 0));
#ifndef MDS_Y_NO_EVICT_FIRST
            bulk_g2s_hint(W.y[fst] + 4 * g * TB, Y + (size_t)t * TB * TB + (size_t)(jj0 + 4 * g) * TB, GB,
                          &W.bar0[g], ypol);
#else
            bulk_g2s(W.y[fst] + 4 * g * TB, Y + (size_t)t * TB * TB + (size_t)(jj0 + 4 * g) * TB, GB, &W.bar0[g]);
#endif
            if (with_x) bulk_g2s(W.xcol[t & 1], X + (size_t)(t - itb) * TB * D, XB, &W.bar0[g]);
        };
#ifndef MDS_EXP_NO_TMA
        // the first group's x (the previous step's drift) is issued after pdl_wait below;
        // its y (constant) goes out now, overlapping the previous grid's tail
        const bool defer_x = first_pending && !early_tab && vv == 0;
        if (nsw > 0) {
            if (first_pending) {
                if (lane == 0) issue_group(fc4b, defer_x ? 2 : 1);
                ++iu;
                ist = (ist + 1 == NSTAGE) ? 0 : ist + 1;
            } else {
                issue_one();
            }
            if (NSTAGE > 2 && iu < ue) issue_one();
        }
#endif
        if (!early_tab && vv == 0) {          // (uniform: every warp runs range 0)
            build_exptab(exptab, a.P);
            __syncthreads();
            pdl_wait();
            if (defer_x && nsw > 0 && lane == 0)
                bulk_g2s(W.xcol[(ub / UNITS_PER_TILE) & 1], X + (size_t)(ub / UNITS_PER_TILE - W.seg[0].w) * TB * D,
                         XB, &W.bar0[fc4b]);
        }
#pragma unroll 1
        for (int si = 0; si < nsw; ++si) {
            const int4 sg = W.seg[si];
            T xi0[D], xi1[D];
            A g0[D], g1[D];
#pragma unroll
            for (int k = 0; k < D; ++k) {          // the segment's 64 rows (2 per lane)
                xi0[k] = (T)X[((size_t)sg.x * TB + lane) * D + k];
                xi1[k] = (T)X[((size_t)sg.x * TB + lane + 32) * D + k];
                g0[k] = g1[k] = A(0);
            }
#pragma unroll 1
            for (int u = sg.y / GPU; u < (sg.z + GPU - 1) / GPU; ++u) {
                // the unit's 4-column groups inside this segment: [c4b, c4e)
                const int c4b = max(sg.y - GPU * u, 0), c4e = min(sg.z - GPU * u, GPU);
                const bool fu = first_pending;        // the staggered first unit (per-group barriers)
                first_pending = false;
                // fp32: this unit brought tile t's column x (first unit of the tile, or of the
                // range): convert it to fp32 once, right after it has landed
                const bool new_x = (u % UNITS_PER_TILE == 0) || u == ub;
                auto cvt_xcol = [&]() {
                    if constexpr (sizeof(T) == 4) {
                        const int tb = (u / UNITS_PER_TILE) & 1;
                        for (int e = lane; e < TB * D; e += 32) W.xcolf[tb][e] = (float)W.xcol[tb][e];
                        __syncwarp();
                    }
                };
                T gf0[D], gf1[D];                     // fp32: the unit's row sums (fp64 above the unit)
                T lsu = T(0);
                if constexpr (sizeof(T) == 4) {
#pragma unroll
                    for (int k = 0; k < D; ++k) gf0[k] = gf1[k] = T(0);
                }
#ifndef MDS_EXP_NO_TMA
                if (!fu) {
                    if (a.prof && lane == 0 && !mbar_ready(&W.bar[cst], (phase >> cst) & 1)) ++not_ready;
                    mbar_wait(&W.bar[cst], (phase >> cst) & 1);
                    if (a.prof && threadIdx.x == 0 && not_ready < 0x80000000u) {   // first unit of warp 0 landed
                        a.prof[gridDim.x * 6 + blockIdx.x] = gtimer();
                        not_ready |= 0x80000000u;
                    }
                    phase ^= 1u << cst;
                    __syncwarp();                     // all lanes are done with the stage being refilled
                    if (iu < ue) issue_one();
                    if (new_x) cvt_xcol();
                }
#endif
                const int t = u / UNITS_PER_TILE, jb = (u % UNITS_PER_TILE) * UCOLS;
                const int cpos = __ldg(a.slab_pos + a.nseg + t);    // used after the groups' math
                // One lock-step block: 4 pairs per lane -- rows lane and lane+32 against the
                // columns qa and qb of yb/xb (per-lane column indices) -- with the Eq. 2 terms
                // into the running sums, the row sums by fused multiply-adds, and the column
                // side added to the accumulators ca (column qa) and cb (column qb).
                auto block4 = [&](const T* __restrict__ yb, const T* __restrict__ xb, int qa, int qb,
                                  T (&ca)[D], T (&cb)[D]) {
                    T ys[4], ss[4], dd[4][D];
#pragma unroll
                    for (int qq = 0; qq < 2; ++qq) {
                        const int q = qq ? qb : qa;
                        ys[2 * qq] = yb[q * TB + lane_v];
                        ys[2 * qq + 1] = yb[q * TB + lane_v + 32];
                        T xj[D];
                        if constexpr (D == 2 && sizeof(T) == 8) {
                            // per-lane columns: one 16-byte load (conflict-free per quarter warp)
                            const double2 v = *reinterpret_cast<const double2*>(xb + q * 2);
                            xj[0] = v.x;
                            xj[1] = v.y;
                        } else {
#pragma unroll
                            for (int k = 0; k < D; ++k) xj[k] = (T)xb[q * D + k];
                        }
                        T sa = T(0), sb = T(0);
#pragma unroll
                        for (int k = 0; k < D; ++k) {
                            dd[2 * qq][k] = xi0[k] - xj[k];
                            dd[2 * qq + 1][k] = xi1[k] - xj[k];
                            sa = fma(dd[2 * qq][k], dd[2 * qq][k], sa);
                            sb = fma(dd[2 * qq + 1][k], dd[2 * qq + 1][k], sb);
                        }
                        ss[2 * qq] = sa;
                        ss[2 * qq + 1] = sb;
                    }
                    T ll[4], uu[4];
                    if constexpr (sizeof(T) == 8) {
                        // fp64: the log L terms go straight into the 4 running sums
                        // (missing pairs keep the old sum: a select, not an FP64 add)
#pragma unroll
                        for (int i = 0; i < 4; ++i) ll[i] = lacc[i];
                        Pair<T, TRUNC>::template eval4<WL, WG>(ss, ys, a.P, exptab, ll, uu);
                        bool mi[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) mi[i] = is_missing(ys[i]);
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            if (WL) lacc[i] = mi[i] ? lacc[i] : ll[i];
                            if (WG) uu[i] = mi[i] ? T(0) : uu[i];
                        }
                        if (WG) {
                            // pair (row r, column c) adds -u (x_r - x_c) to row r and +u (x_r - x_c)
                            // to column c: rows by fused multiply-adds
#pragma unroll
                            for (int k = 0; k < D; ++k) {
                                g0[k] = fma(-uu[0], dd[0][k], g0[k]);
                                g0[k] = fma(-uu[2], dd[2][k], g0[k]);
                                g1[k] = fma(-uu[1], dd[1][k], g1[k]);
                                g1[k] = fma(-uu[3], dd[3][k], g1[k]);
                            }
                        }
                    } else {
                        Pair<T, TRUNC>::template eval4<WL, WG>(ss, ys, a.P, exptab, ll, uu);
                        T lsum = T(0);
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const bool mi = is_missing(ys[i]);
                            if (WL && !mi) lsum += ll[i];         // predicated, no select
                            if (WG) uu[i] = mi ? T(0) : uu[i];
                        }
                        if (WG) {
#pragma unroll
                            for (int k = 0; k < D; ++k) {
                                gf0[k] = fmaf(-uu[0], dd[0][k], gf0[k]);
                                gf0[k] = fmaf(-uu[2], dd[2][k], gf0[k]);
                                gf1[k] = fmaf(-uu[1], dd[1][k], gf1[k]);
                                gf1[k] = fmaf(-uu[3], dd[3][k], gf1[k]);
                            }
                        }
                        if (WL) lsu += lsum;
                    }
                    if (WG) {
#pragma unroll
                        for (int k = 0; k < D; ++k) {
                            ca[k] = fma(uu[1], dd[1][k], fma(uu[0], dd[0][k], ca[k]));
                            cb[k] = fma(uu[3], dd[3][k], fma(uu[2], dd[2][k], cb[k]));
                        }
                    }
                };
                // Two ways through a unit:
                //  * rotation (every whole unit but the warp's staggered first one): rotating
                //    column accumulators.  Lanes form groups of UCOLS; at step s lane L takes
                //    column (L + s) mod UCOLS of the unit (rows L and L+32), two steps per
                //    lock-step block, one accumulator for the even and one for the odd
                //    steps; after every block both move 2 lanes down the lane group, so each
                //    follows its column across the group.  A column's sum is then one fused
                //    multiply-add per pair plus, once per unit, 1 + log2(32 / UCOLS) adds,
                //    instead of a 2-row sum and a reduce-scatter (6 adds per 8 pairs) per 4
                //    columns.  Lane L ends with column (L - 2) mod UCOLS.
                //  * group mode (a warp range's partial first / last unit, the staggered first
                //    unit): per 4-column group a 2-row sum per column and a select-free
                //    reduce-scatter over the 32 lanes (the column order p ^ m, see m).
                // Fixed order either way: deterministic.  (N = 30000 A/B, G pair-evals/s,
                // group mode only -> rotation: fp64 D = 2 216.8 -> 227.0, D = 3 191.6 -> 200.7,
                // D = 4 173.0 -> 189.4, D = 6 155.4 -> 171.3; fp32 D = 2 508.2 -> 526.4, D = 6
                // 322.4 -> 344.0.  Four accumulators moved 4 lanes at the end of each 4-step
                // trip were slower: fp64 D = 2 223.4, D = 4 178.0, D = 3 186.0, D = 6 154.0,
                // and spilled the fp32 pass.)
                const int lr = lane_v & (UCOLS - 1);
                const T* __restrict__ yu = W.y[cst];
                const T* __restrict__ xu;
                if constexpr (sizeof(T) == 4) xu = &W.xcolf[t & 1][jb * D];
                else xu = W.xcol[t & 1] + jb * D;
                bool unit_done = false;
#ifndef MDS_NO_ROT
                if (WG && __all_sync(0xffffffffu, !fu && c4b == 0 && c4e == GPU)) {   // (a vote: warp-uniform)
                    T ce[D], co[D];
#pragma unroll
                    for (int k = 0; k < D; ++k) ce[k] = co[k] = T(0);
                    // trips unrolled: fp32 all of the unit's (N = 30000 D = 6 A/B 343.9 -> 353.9 G),
                    // fp64 two (D = 2 227.2 -> 229.9 G, D = 6 171.6 -> 175.6 G); fp64's four trips
                    // unrolled do not fit the instruction cache (D = 2 156.2 G, D = 6 80.6 G)
#ifndef MDS_F64_ROT_UNROLL
                    constexpr int ROT_UNROLL = sizeof(T) == 4 ? UCOLS / 4 : 2;
#else
                    constexpr int ROT_UNROLL = sizeof(T) == 4 ? UCOLS / 4 : MDS_F64_ROT_UNROLL;
#endif
#pragma unroll (ROT_UNROLL)
                    for (int s4 = 0; s4 < UCOLS; s4 += 4) {
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int k0 = s4 + 2 * h;
                            block4(yu, xu, (lr + k0) & (UCOLS - 1), (lr + k0 + 1) & (UCOLS - 1), ce, co);
                            if (k0 + 2 < UCOLS) {
#pragma unroll
                                for (int k = 0; k < D; ++k) {
                                    ce[k] = __shfl_sync(0xffffffffu, ce[k], lane_v + 2, UCOLS);
                                    co[k] = __shfl_sync(0xffffffffu, co[k], lane_v + 2, UCOLS);
                                }
                            }
                        }
                    }
                    double* __restrict__ cslab = a.slabs + (size_t)cpos * TB * D + (size_t)jb * D;
                    const int cc = (lr + UCOLS - 2) & (UCOLS - 1);
#pragma unroll
                    for (int k = 0; k < D; ++k) {
                        T cs = ce[k] + __shfl_sync(0xffffffffu, co[k], lane_v + UCOLS - 1, UCOLS);
#pragma unroll
                        for (int o = UCOLS; o < 32; o <<= 1) cs += shfl_xor(cs, o);
                        if (lane_v < UCOLS) cslab[cc * D + k] = A(cs);
                    }
                    unit_done = true;
                }
#endif
#ifdef MDS_ROT_COUNT
                unit_done = true;     // (count_sass.py: a build whose only pair loop is the rotation's)
#endif
                const int it_b = c4b, it_e = unit_done ? c4b : c4e;
                T cv[4][D];           // group mode: the 4 columns' 2-row sums (accumulated from zero)
#pragma unroll
                for (int p = 0; p < 4; ++p)
#pragma unroll
                    for (int k = 0; k < D; ++k) cv[p][k] = T(0);
#pragma unroll 1      // (unroll 2 measured: 168 regs + spills, 219 -> 154 G pair-evals/s)
                for (int c4 = it_b; c4 < it_e; ++c4) {     // 8 pairs per lane: a 4-column group / 4 steps
#ifndef MDS_EXP_NO_TMA
                if (fu) {
                    mbar_wait(&W.bar0[c4], 0);
                    if (c4 == c4b) {
                        if (a.prof && threadIdx.x == 0) {
                            a.prof[gridDim.x * 6 + blockIdx.x] = gtimer();
                            not_ready |= 0x80000000u;
                        }
                        __syncwarp();
                        // the first group has landed: fetch the rest of the unit and the next unit
                        if (lane == 0)
                            for (int g = c4b + 1; g < c4e; ++g) issue_group(g, 0);
                        if (iu < ue) issue_one();
                        cvt_xcol();                   // the tile's x came with the first group
                    }
                }
#endif
#pragma unroll
                for (int h = 0; h < 2; ++h) {         // positions 2h, 2h+1: 4 pairs per lane in lock-step
                    block4(yu, xu, 4 * c4 + ((2 * h) ^ m), 4 * c4 + ((2 * h + 1) ^ m), cv[2 * h], cv[2 * h + 1]);
                }
                {
                    double* __restrict__ cslab = a.slabs + (size_t)cpos * TB * D + (size_t)(jb + 4 * c4) * D;
#pragma unroll
                    for (int k = 0; k < (WG ? D : 0); ++k) {
                        const T cs = reduce_scatter4_perm(cv[0][k], cv[1][k], cv[2][k], cv[3][k]);
                        if ((lane & 7) == 0) cslab[m * D + k] = A(cs);
                    }
#pragma unroll
                    for (int p = 0; p < 4; ++p)
#pragma unroll
                        for (int k = 0; k < D; ++k) cv[p][k] = T(0);
                }
                }   // 4-column groups / steps
                if constexpr (sizeof(T) == 4) {       // at most 16 columns x 2 terms in fp32 (reading R15)
                    if (WG) {
#pragma unroll
                        for (int k = 0; k < D; ++k) {
                            g0[k] += A(gf0[k]);
                            g1[k] += A(gf1[k]);
                        }
                    }
                    if (WL) lik_w += A(lsu);
                }
                cst = (cst + 1 == NSTAGE) ? 0 : cst + 1;
            }
            // the segment's row partial
            double* __restrict__ rslab = a.slabs + (size_t)W.spos[si] * TB * D;
            if (WG) {
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    rslab[lane * D + k] = g0[k];
                    rslab[(lane + 32) * D + k] = g1[k];
                }
            }
        }
    }
    }   // virtual ranges
    lik_w += (lacc[0] + lacc[1]) + (lacc[2] + lacc[3]);
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) lik_w += __shfl_xor_sync(0xffffffffu, lik_w, m);
    if (lane == 0) a.likpart[gw] = lik_w;

    // ------------------------------------------------------------ barrier
    if (a.prof) {
        if (lane == 0) atomicAdd(&a.prof[gridDim.x * 4 + blockIdx.x], (unsigned long long)(not_ready & 0x7fffffffu));
        __syncthreads();
        if (threadIdx.x == 0) {
            a.prof[blockIdx.x * 4 + 1] = gtimer();
            unsigned smid;
            asm("mov.u32 %0, %%smid;" : "=r"(smid));
            a.prof[gridDim.x * 5 + blockIdx.x] = smid;
        }
    }
    // (Loading phase B's static inputs -- block pointers, leapfrog state -- before
    // the barrier measured 0.4% slower: A/B on one box.)
    constexpr int EPLMAX = 4;
    const int epl = a.epl;
    const int CH = 32 * epl;
    const int chunks = (TB * D + CH - 1) / CH;
    const int jobs = a.nb * chunks;
    __threadfence();
    if (a.soft_sync) grid_barrier(a.gbar, gridDim.x);   // plain launch (peer-memory exchange)
    else cg::this_grid().sync();
    pdl_launch_dependents();     // the next leapfrog step's grid may be scheduled (it waits in pdl_wait)
    // the exchange this pass is: read after pdl_wait (the previous pass advances it at
    // its very end) and before any CTA can advance it (at the end of this one)
    const unsigned long long p2p_ep = p2p ? p2p_epoch(a.p2p) : 0ull;
    if (a.prof && threadIdx.x == 0) a.prof[blockIdx.x * 4 + 2] = gtimer();

    // ------------------------------------------------------------ phase B
    // job = (row block b, chunk of 32 * epl slab elements, epl per lane; the host
    // picks epl in {1, 2, 4} so that the jobs fit the grid in one round); warp w
    // sums slabs w, w + WPC, ... in order with 8 slab indices in flight
    // the staging area is free after the grid barrier: reuse it for the sums
    A (*red)[WPC][32] = reinterpret_cast<A (*)[WPC][32]>(dsm);
    uint32_t pb_phase = 0;
    for (int job = blockIdx.x; WG && job < jobs; job += gridDim.x) {
        const int b = job / chunks, ch = job % chunks;
        const int q0 = a.blk_ptr[b], nq = a.blk_ptr[b + 1] - q0;
        A acc[EPLMAX];
        int el[EPLMAX];
#pragma unroll
        for (int ee = 0; ee < EPLMAX; ++ee) {
            acc[ee] = A(0);
            el[ee] = ch * CH + ee * 32 + lane;
        }
        // leapfrog state of the element this warp updates below (independent of the sums)
        double pre_xe = 0, pre_p = 0, pre_gl = 0;
        const int e_up = ch * CH + warp * 32 + lane;
        const int64_t e_glb = (int64_t)b * TB * D + e_up;
        if (LF && warp < epl && e_up < TB * D && e_glb < a.n * D) {
            pre_xe = a.xeval[e_glb];
            pre_p = a.p[e_glb];
            pre_gl = a.gl[e_glb];
        }
        // block b's slabs are contiguous: warp w sums rows w, w + WPC, ... in order,
        // 8 rows in flight (rows past the end add exact zeros).  When the job covers
        // whole slabs and they fit the (now free) staging area, ONE bulk copy brings
        // them into shared memory first: the sums then read shared memory, same order.
        const double* __restrict__ sb = a.slabs + (size_t)q0 * TB * D;
#ifndef MDS_NO_PHASEB_TMA
        constexpr size_t PB_OFF = ((sizeof(A) * EPLMAX * WPC * 32) + 127) & ~(size_t)127;   // past red[][][]
        const uint32_t pb_bytes = (uint32_t)nq * TB * D * sizeof(A);
        if (chunks == 1 && PB_OFF + pb_bytes <= (size_t)WPC * sizeof(WarpStage<T, D>) && nq > 0) {
            double* sm = reinterpret_cast<double*>(dsm + PB_OFF);
            if (threadIdx.x == 0) {
                fence_async_smem();
                mbar_arrive_tx(&pb_bar, pb_bytes);
                bulk_g2s(sm, sb, pb_bytes, &pb_bar);
            }
            mbar_wait(&pb_bar, pb_phase);
            pb_phase ^= 1u;
            sb = sm;
        }
#endif
        for (int k0 = warp; k0 < nq; k0 += 8 * WPC) {
            // all (element, slab) loads of the round first, then the adds in order:
            // one L2 round trip per round instead of one per element
            A x[EPLMAX][8];
#pragma unroll
            for (int ee = 0; ee < EPLMAX; ++ee) {
                const bool on = ee < epl && el[ee] < TB * D;
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const int k = k0 + r * WPC;
                    x[ee][r] = (on && k < nq) ? sb[(size_t)k * TB * D + el[ee]] : A(0);
                }
            }
#pragma unroll
            for (int ee = 0; ee < EPLMAX; ++ee)
#pragma unroll
                for (int r = 0; r < 8; ++r) acc[ee] += x[ee][r];
        }
        if (a.prof && threadIdx.x == 0) a.prof[gridDim.x * 7 + blockIdx.x] = gtimer();   // slab sums loaded
#pragma unroll
        for (int ee = 0; ee < EPLMAX; ++ee)
            if (ee < epl) red[ee][warp][lane] = acc[ee];
        __syncthreads();
        if (a.prof && threadIdx.x == 0) a.prof[gridDim.x * 8 + blockIdx.x] = gtimer();   // CTA partials in smem
        if (warp < epl) {
            const int ee = warp;
            const int e_in = ch * CH + ee * 32 + lane;
            if (e_in < TB * D) {
                A g = red[ee][0][lane];
#pragma unroll
                for (int w = 1; w < WPC; ++w) g += red[ee][w][lane];
                const int64_t e = (int64_t)b * TB * D + e_in;
                if (e < a.n * D) {
                    if (!LF) {
                        if (p2p) p2p_push(a.p2p, p2p_ep, e, g);   // this rank's partial -> every rank's window
                        else a.grad[e] = g;
                    } else {
                        // leapfrog: the pass ran at xnext = x + eps (p + eps/2 gl)
                        const double xe = pre_xe;
                        const double ph = __fma_rn(a.heps, pre_gl, pre_p);    // first half-kick
                        const double gn = a.gprior ? g + a.gprior[e] : g - xe * a.inv_tau2;   // grad log pi at xnext
                        const double pn = __fma_rn(a.heps, gn, ph);             // second half-kick
                        a.grad[e] = g;
                        a.x[e] = xe;
                        a.p[e] = pn;
                        a.gl[e] = gn;
                        a.xnext[e] = drift(xe, pn, gn, a.eps, a.heps);           // next step's drift
                    }
                }
            }
        }
        __syncthreads();
    }
    // log L on the last CTA (job-free when jobs < grid): fixed-order strided
    // partial sums over the warp partials, then warps in order
    if (!WL) {
        // nobody reads log L of this pass: mark it as not computed
        if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
            const double nan = __longlong_as_double(0x7ff8000000000000LL);
            if (p2p) p2p_push(a.p2p, p2p_ep, a.n * D, nan);
            else *a.lik = nan;
        }
    } else if (blockIdx.x == gridDim.x - 1) {
        const int GW = gridDim.x * WPC;
        // 4 partials per thread per round: the loads are in flight together
        A s = A(0);
        for (int q0 = threadIdx.x; q0 < GW; q0 += 4 * WPC * 32) {
            A v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = q0 + u * WPC * 32 < GW ? a.likpart[q0 + u * WPC * 32] : A(0);
#pragma unroll
            for (int u = 0; u < 4; ++u) s += v[u];
        }
        red[0][warp][lane] = s;
        __syncthreads();
        if (threadIdx.x < 32) {
            A t = A(0);
            for (int w = 0; w < WPC; ++w) t += red[0][w][threadIdx.x];
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) t += __shfl_xor_sync(0xffffffffu, t, m);
            // the per-pair constant -1/2 log(2 pi sigma^2) of the fp64 path, once:
            // n_obs (this context's observed pairs) x k0
            if (threadIdx.x == 0) {
                if (p2p) p2p_push(a.p2p, p2p_ep, a.n * D, t + a.lik_const);
                else *a.lik = t + a.lik_const;
            }
        }
    }
    // ------------------------------------------------------------ exchange + phase C
    // (fused peer-memory exchange, SURVEY 8(e) stage 2) every CTA's pushes are
    // fenced system-wide and counted; the last CTA raises this rank's flag on every
    // rank; all CTAs wait for every rank's flag, then combine in rank order
    if (p2p) {
        __syncthreads();
        if (threadIdx.x == 0) p2p_arrive_and_wait(a.p2p, p2p_ep, gridDim.x);
        __syncthreads();
        const int64_t m = a.n * D;
        const double* __restrict__ rv = p2p_recv(a.p2p, a.p2p.win[a.p2p.rank], p2p_ep);   // own window
        auto combine_one = [&](int64_t e) {
            double g = 0.0;                      // the rank-ordered sum of combine_kernel
            for (int r = 0; r < a.p2p.world; ++r) g += rv[(size_t)r * (m + 1) + e];
            if (e == m) {
                if (a.lik) *a.lik = g;
            } else if (!a.p2p_lf) {
                if (a.grad) a.grad[e] = g;
            } else {
                // combine_update_kernel's leapfrog update (the pass ran at xnext)
                const double xv = a.xeval[e];
                const double ph = __fma_rn(a.heps, a.gl[e], a.p[e]);
                const double gn = a.gprior ? g + a.gprior[e] : g - xv * a.inv_tau2;
                const double pn = __fma_rn(a.heps, gn, ph);
                a.grad[e] = g;
                a.x[e] = xv;
                a.p[e] = pn;
                a.gl[e] = gn;
                a.xnext[e] = drift(xv, pn, gn, a.eps, a.heps);
            }
        };
        if (WG) {
            const int64_t stride = (int64_t)gridDim.x * blockDim.x;
            for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e <= m; e += stride) combine_one(e);
        } else if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
            combine_one(m);                      // likelihood-only pass: log L alone
        }
        __syncthreads();
        if (threadIdx.x == 0) p2p_finish(a.p2p, p2p_ep, gridDim.x);
    }
    if (a.prof) {
        __syncthreads();
        if (threadIdx.x == 0) a.prof[blockIdx.x * 4 + 3] = gtimer();
    }
}

// ------------------------------------------------------------ dispatch
typedef void (*PassFn)(PassArgs);
struct PassKernel {
    PassFn fn;
    size_t smem;
    int wpc;   // warps per CTA
};
// pass_m<MODE>_<prec>(trunc, d): the instantiation for one (MODE, precision),
// defined in csrc/pass_m<MODE>_<prec>.cu (one translation unit each)
#define MDS_DECLARE_PASS(M)                       \
    PassKernel pass_m##M##_f64(int trunc, int d); \
    PassKernel pass_m##M##_f32(int trunc, int d);
MDS_DECLARE_PASS(0)
MDS_DECLARE_PASS(1)
MDS_DECLARE_PASS(2)
MDS_DECLARE_PASS(3)
MDS_DECLARE_PASS(4)
MDS_DECLARE_PASS(5)
MDS_DECLARE_PASS(6)
MDS_DECLARE_PASS(7)
MDS_DECLARE_PASS(8)
#undef MDS_DECLARE_PASS

}  // namespace mdsk

