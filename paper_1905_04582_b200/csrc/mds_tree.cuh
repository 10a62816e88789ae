// mds_tree.cuh -- phylogenetic Brownian-diffusion prior of X (SURVEY 8(f)
// NEXT-2; Eq. 3) and its gradient, in O(N D^2).
//
// X ~ MN(mu0, V_G, Sigma): tips of a forest evolve by Brownian motion with
// covariance t_c Sigma along each branch; tree roots are N(mu0, tau0 Sigma),
// unsequenced items are single-node trees N(mu0, tau_e Sigma).  Instead of
// forming V_G^-1 (O(N^3)) the prior follows the dynamic program the paper
// cites: a post-order pass absorbs the children's messages
// (m, v) -- "the tips below are N(m; x_node, v Sigma)" -- contrast by contrast,
//   delta = a_i - A, w = W + w_i:  log p += -1/2 delta' Sigma^-1 delta / w
//                                          - D/2 log(2 pi w) - 1/2 log|Sigma|
//   A <- (w_i A + W a_i)/w,  W <- W w_i / w,
// and a root contrast against mu0 with variance v_root + tau_root (N contrasts
// in all).  A pre-order pass forms each node's outside message (the law of
// x_node given every tip NOT below it); for tip i that is the conditional law
// N(m_i, v_i Sigma) of x_i given all other tips, so
//   d log p / d x_i = - Sigma^-1 (x_i - m_i) / v_i        ([V^-1 (X - mu0) Sigma^-1]_i).
//
// One CTA walks the levels (nodes of equal height / depth in parallel).  The
// pass is latency-bound (26 + 26 levels at C2), so the level critical path is
// kept on chip: the messages of INTERNAL nodes (the only dynamic state) live in
// shared memory when they fit ((n_nodes - n) (D + 1) doubles; else a global
// buffer); the static operands of every level are laid out level by level
// (one int4 + one double2 per node, the tip children's x and, for the
// pre-order, the children's up messages gathered by wide parallel passes), so
// a level's operands are one coalesced round of loads issued before the
// barrier that publishes the previous level -- and one level ahead on the
// narrow levels near the roots, which run on warp 0 alone with __syncwarp;
// reciprocals from the MUFU seed + one cubic Newton step (no IEEE division
// subroutine on the level chain); the logs of the contrast variances are deferred to the
// final parallel reduction.  Tip
// gradients are written as the pre-order reaches them.  Node contributions are
// summed in a fixed order: deterministic, no atomics.
#pragma once
#include <cstdint>
#include <cstddef>

namespace mdsk {

constexpr int TREE_DMAX = 8;

struct TreeArgs {
    // forest (device): node k < n is item k; internal node k has slot k - n
    int n_nodes;
    int n_items;
    const int* ch_ptr;        // [n_nodes + 1] children CSR (ascending child index; arity > 2 only)
    const int* ch_idx;
    const double* t;          // [n_nodes] branch length (roots: prior variance factor)
    // post-order entries (internal nodes by height), level L = [up_lvl_ptr[L], up_lvl_ptr[L+1])
    const int* up_lvl_ptr;    // [n_up + 1]
    const int4* up_e;         // {slot, src0, src1, k}; src = internal slot, or -1 - item for a tip
    const double2* up_t;      // {t(child 0), t(child 1)}
    const double* up_tn;      // [E_up] the node's own branch length (root: prior variance)
    const int* up_dpos;       // [E_up] the node's slot in its parent's pre-order entry (dn_pos of the node)
    const int* tip_upos;      // [n] 2 e + i if item i is child i < 2 of post-order entry e, else -1
    double* up_x;             // [E_up][2][D] x of tip children 0/1, scattered from X at the start of a walk
    int n_up;
    int up_narrow;            // first post-order level from which every level has <= 32 nodes
    // pre-order entries (nodes with children by depth)
    const int* dn_lvl_ptr;    // [n_dn + 1]
    const int4* dn_e;         // {slot, child 0, child 1, k} (children as node ids)
    const double2* dn_t;      // {t(child 0), t(child 1)}
    double* dn_sib;           // [E_dn][2][D + 1] up message (mean, precision at the parent) of children 0/1
    const int* dn_pos;        // [n_nodes] 2 e + i for child i < 2 of pre-order entry e, else -1
    int n_dn;
    int dn_narrow;            // pre-order levels [0, dn_narrow) all have <= 32 nodes
    const int* roots;         // [n_roots]
    int n_roots;
    // parameters
    double mu0[TREE_DMAX];
    double sinv[TREE_DMAX * TREE_DMAX];   // Sigma^-1 (row-major)
    double logdet;                        // log |Sigma|
    // state / scratch
    const double* x;          // positions (n_pad x D)
    double* up_m;             // [n_nodes - n][D]  up message means of internal nodes (global copy)
    double* pw;               // [n_nodes]         1 / (up_v + t): each up message's precision at its parent
    double* msg;              // [(n_nodes - n) (D + 1)] internal-node messages when they do not fit smem
    size_t smem;              // dynamic shared memory for the messages (0 = use msg)
    double* cq;               // [n_nodes] -1/2 sum delta' Sigma^-1 delta / w - (#contrasts)(D log 2pi + log|Sigma|)/2
    double* cw;               // [n_nodes] product of the node's contrast variances w (log taken at the end)
    // outputs
    double* grad;             // [n_items][D]  d log p / d X
    double* logp;             // [1]
    unsigned long long* prof; // optional (MDS_PROFILE_TREE=1): globaltimer stamps per level
    // inside the pass kernel: the tips pass is split over the pair CTAs, which
    // count themselves in tips_done; the walk waits for ext_tips arrivals (0 = the
    // walk does the tips pass itself)
    int ext_tips;
    unsigned int* tips_done;
};

constexpr size_t TREE_SMEM_MAX = 200 * 1024;
void tree_prior_launch(const TreeArgs& a, int d, cudaStream_t s);
void tree_preload(int d);   // load the standalone walk kernel now (see preload_kernels)

}  // namespace mdsk
