/*
 * msp_b200.h -- C ABI of the B200-native PEGP/MSP graph-Laplacian solver
 * (arxiv 2207.07847, "PEGP / MSP").  Shared library:
 * paper_2207_07847_b200/libmsp_b200.so (sm_100a).
 *
 * The calls follow the problem statement of the paper: solve L_G x = b for a
 * weighted graph Laplacian (§2.1, Eq. eqn:originalsys, l.97-100) with
 * b orthogonal to the ones vector, by conjugate gradient preconditioned with
 * R = P(mu) L_X^+ P(mu)^T (Eq. graphL_precsys l.26-32 applied to the expanded
 * system of Eq. def:L_ell; reading R9), X = T~ (MSP, §3.3) or
 * X = H~ (PEGP, §3.2).
 *
 * Conventions shared by every call
 *  - Return value: MSP_OK (0) on success, a negative MSP_ERR_* code on
 *    failure; msp_last_error() then returns a thread-local message.  No call
 *    aborts the process; on error the output buffers are unspecified.
 *  - Vectors are fp64, length n, in the ORIGINAL vertex numbering of the graph
 *    passed to msp_setup.  `mem` says where every pointer argument of the call
 *    lives: MSP_MEM_DEVICE (CUDA device pointers, no host<->device copies) or
 *    MSP_MEM_HOST (host pointers; the call copies in and out itself).
 *  - `stream` is a cudaStream_t (may be NULL = legacy default stream).  Device
 *    calls are asynchronous with respect to the host when mem ==
 *    MSP_MEM_DEVICE, except msp_setup and msp_pcg_solve which synchronise the
 *    stream before returning (setup builds host-side sizes; pcg reads the
 *    convergence flag).
 *  - The caller owns every buffer it passes; the handle owns its device
 *    memory until msp_destroy.  A handle may be used by one host thread at a
 *    time.
 */
#ifndef MSP_B200_H
#define MSP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSP_OK 0
#define MSP_ERR_ARG (-1)          /* bad argument (null, size, enum)            */
#define MSP_ERR_CUDA (-2)         /* CUDA runtime failure                       */
#define MSP_ERR_GRAPH (-3)        /* graph not usable: isolated vertex, bad CSR */
#define MSP_ERR_UNSUPPORTED (-4)  /* valid request outside this build's scope  */

#define MSP_MEM_DEVICE 0
#define MSP_MEM_HOST 1

#define MSP_PRECOND_NONE 0        /* plain CG (R = I)                           */
#define MSP_PRECOND_MSP 1         /* R = P(mu) L_T~^+ P(mu)^T   (§3.3)          */
#define MSP_PRECOND_PEGP 2        /* R = P(mu) L_H~^+ P(mu)^T   (§3.2), inner CG */

typedef struct msp_handle msp_handle;

typedef struct msp_params {
  double mu;            /* scaling parameter of {P(mu)}^l, 0 < mu;
                           <= 0 selects the paper's practical default 0.8 (l.1004) */
  int32_t max_levels;   /* number of levels l; 0 = "level = max" (l.681):
                           coarsen while a level has > 2 nodes and >= 2 aggregates */
  int32_t top_max;      /* largest top level accepted for the dense top solve;
                           0 = default 256 (larger => MSP_ERR_UNSUPPORTED)        */
  uint64_t seed;        /* seed of the MWM visit order (reading R1) */
} msp_params;

typedef struct msp_info_t {
  int64_t n;            /* vertices of G                                        */
  int64_t nnz;          /* 2m + n: nonzeros of L_G                              */
  int64_t n_tilde;      /* sum of level sizes (size of the expanded graph)      */
  int32_t levels;       /* l                                                    */
  int32_t mwm_rounds;   /* parallel matching rounds used over all levels        */
  double mu;            /* mu actually used                                     */
  double setup_ms;      /* GPU setup time (hierarchy + expansion + MSP), device */
  /* solve schedule: levels 1..coarse_level run
     as ntiers tiers of tile kernels (the first covers levels 1..tile_level
     with ntiles CTAs), levels coarse_level..l in one single-CTA kernel */
  int32_t tile_level;
  int32_t coarse_level;
  int64_t ntiles;       /* tiles (CTAs) of the first tier                       */
  int32_t ntiers;
  int32_t spmv_grid;    /* CTAs of the L_G product                              */
  int32_t merged_coarse;  /* 1: the coarse levels run inside the last tier's down
                             kernel (one copy per CTA), 0: their own kernel   */
} msp_info_t;

typedef struct msp_report {
  int32_t iterations;   /* PCG iterations = number of L_G products performed    */
  int32_t converged;    /* 1 if ||r_k|| <= rtol ||b||                            */
  double relres;        /* final ||r_k|| / ||b|| (recursive residual)           */
  double solve_ms;      /* device time of the solve (CUDA events on `stream`)   */
  int64_t kernel_launches; /* kernels this library launched inside the solve    */
} msp_report;

/*
 * msp_setup -- build everything the solve needs, on the GPU.
 *   PAPER.md §2.2 (MWM aggregation l.61/l.70, prolongations Eq. def:P),
 *   §3.1 Eq. def:L_ell (expanded graph), §3.2 (positive subgraph H~ =
 *   negative-edge elimination), §3.3 (MSP T~).
 * n              number of vertices (>= 2).
 * rowptr,col,w   symmetric CSR of the weighted adjacency (no diagonal, no
 *                self loops, columns strictly increasing per row, w > 0);
 *                int64 row offsets [n+1], int32 columns [nnz], fp64 weights.
 *                Read during the call only (in `mem`).
 * params         may be NULL (defaults).
 * out            receives a new handle (caller frees with msp_destroy).
 * Errors: MSP_ERR_ARG (n < 2, null pointers), MSP_ERR_GRAPH (isolated
 * vertex or unsorted/out-of-range columns), MSP_ERR_UNSUPPORTED (top level
 * larger than top_max), MSP_ERR_CUDA.
 */
int msp_setup(int64_t n, const int64_t* rowptr, const int32_t* col, const double* w,
              int mem, const msp_params* params, void* stream, msp_handle** out);

/* msp_destroy -- free all device memory of the handle (NULL is a no-op). */
int msp_destroy(msp_handle* h);

/* msp_info -- sizes and timings of the built hierarchy (host struct). */
int msp_info(const msp_handle* h, msp_info_t* out);

/*
 * msp_level_sizes -- n_k for k = 1..l into host array sizes[l].
 * msp_get_aggregates -- for level k in 1..l-1, agg[i] = index of the
 *   level-(k+1) aggregate containing level-k node i, both in the canonical
 *   numbering of reading R3 (aggregates ordered by the smaller vertex of their
 *   matched pair).  Host array of n_k entries.  Used for the bit-exact
 *   hierarchy parity check.
 */
int msp_level_sizes(const msp_handle* h, int64_t* sizes);
int msp_get_aggregates(const msp_handle* h, int32_t level, int32_t* agg);

/*
 * msp_get_msp_edges -- the MSP T~ as an edge list (i < j, weight > 0) in the
 * canonical expanded numbering (level-k node a -> sum_{j<k} n_j + a).
 * Call with i = j = w = NULL to get *count; then with arrays of *count
 * entries (host).  Parity/inspection helper, not on the hot path.
 */
int msp_get_msp_edges(const msp_handle* h, int64_t* count, int64_t* i, int64_t* j, double* w);

/*
 * msp_apply_L -- y = L_G x  (§2.1 L_G = B^T W B), evaluated as
 * y_i = sum_j w_ij (x_i - x_j).  x, y: n entries in `mem`; may not alias.
 */
int msp_apply_L(msp_handle* h, const double* x, double* y, int mem, void* stream);

/*
 * msp_apply_R -- z = R r with R = P(mu) L_X^+ P(mu)^T (reading R9):
 *   precond = MSP_PRECOND_MSP  : X = T~, exact (block-tree elimination sweeps)
 *   precond = MSP_PRECOND_PEGP : X = H~ (§3.2, the positive subgraph of G~),
 *                                L_H~^+ by MSP-preconditioned CG in the
 *                                expanded space to the relative residual of
 *                                msp_pegp_params (reading R13)
 *   precond = MSP_PRECOND_NONE : z = r
 * r, z: n entries in `mem`; may alias.
 */
int msp_apply_R(msp_handle* h, int precond, const double* r, double* z, int mem, void* stream);

/*
 * Expanded-space calls (PEGP support and parity checks).  Vectors have n~
 * entries in the canonical expanded numbering (level-k node a at
 * sum_{j<k} n_j + a, as msp_get_msp_edges), in `mem`.
 *   msp_apply_LH : y~ = L_H~ x~, the Laplacian of the PEGP H~ (§3.2,
 *                  positive edges of Eq. def:L_ell), in the difference form
 *                  sum_j w_ij (x_i - x_j) over an explicit CSR of the H~ edge
 *                  weights assembled on the GPU at the first PEGP call.
 *   msp_solve_LH : z~ = L_H~^+ r~ (minimum norm) by CG preconditioned with the
 *                  exact L_T~^+ (§3.3); *inner_iterations receives the count
 *                  (may be NULL; refinement steps included).  Inexact:
 *                  relative residual <= inner_rtol, then refine_steps steps
 *                  of iterative refinement (residual in double-double).
 *   msp_pegp_params : inner_rtol in (0, 1) (default 1e-13), inner_maxit
 *                  (default 5000) of that CG, refine_steps in [0, 16]
 *                  (default 0).  Applies to msp_apply_R / msp_pcg_solve with
 *                  MSP_PRECOND_PEGP as well.
 * x and y (r and z) may not alias.  Errors: MSP_ERR_ARG, MSP_ERR_CUDA.
 */
int msp_apply_LH(msp_handle* h, const double* x, double* y, int mem, void* stream);
int msp_solve_LH(msp_handle* h, const double* r, double* z, int mem, void* stream, int32_t* inner_iterations);
int msp_pegp_params(msp_handle* h, double inner_rtol, int32_t inner_maxit, int32_t refine_steps);
/*
 * msp_pegp_info -- builds H~ if needed (on `stream`), then writes out5[5]
 * (host): [0] nnz of the H~ edge-weight CSR (both directions), [1] inner CG
 * iterations of the last PEGP apply / solve_LH (refinement included), [2]
 * the level above which the inner CG's sweeps run in one CTA, [3] H~ build
 * time in microseconds (device, CUDA events), [4] inner CG iterations of the
 * last PCG-PEGP solve (all its applies).  Errors: MSP_ERR_ARG, MSP_ERR_CUDA.
 */
int msp_pegp_info(msp_handle* h, void* stream, int64_t* out5);

/*
 * msp_pcg_solve -- preconditioned CG for L_G x = b, x0 = 0, stopping at the
 * first k with ||r_k||_2 <= rtol ||b||_2 or k = maxit (reading R10).
 * b, x: n entries in `mem` (x is overwritten).  report may be NULL.
 * b should be orthogonal to the ones vector (the compatible case of
 * Eq. eqn:originalsys); otherwise the residual stalls at its mean part.
 */
int msp_pcg_solve(msp_handle* h, int precond, const double* b, double* x, double rtol,
                  int32_t maxit, int mem, void* stream, msp_report* report);

/*
 * Kernel-level profiling of msp_pcg_solve (measurement support, DESIGN.md
 * "Measurement").  When enabled, every launch of the solve is bracketed by
 * CUDA events on the solve's stream (the iterations then run without the
 * captured CUDA graph) and its device time is accumulated per category:
 * 0 p = z + beta p fused with q = L_G p and (p, q);  1 tile up-sweep fused
 * with x/r update and (r, r);  2 per-level up-sweeps;  3 single-CTA coarse
 * kernel (coarse up-sweep, top solve, coarse down-sweep);  4 per-level
 * down-sweeps;  5 tile down-sweep with the output R r and (r, R r);  6 the
 * PEGP inner CG's fused p update + L_H~ p + (p, q) (k_h_spmv);  7 its
 * expanded-space MSP sweeps with the x / r updates and dots.  msp_get_profile copies ms[MSP_PROF_NCAT] and launch counts
 * counts[MSP_PROF_NCAT] (host arrays) and resets them.
 */
#define MSP_PROF_NCAT 8
int msp_set_profiling(msp_handle* h, int on);
int msp_get_profile(msp_handle* h, double* ms, int64_t* counts);

/*
 * Multi-GPU solve (row 6 of DESIGN.md §8).  One process
 * per GPU; every rank calls msp_setup on the full graph (same seed: the same
 * hierarchy, bit for bit), then msp_dist_init, then the ranks solve ONE
 * system together.  Partition: the nodes of a partition level kp (the top of
 * the highest solve tier with >= 32 nodes per rank) are split into
 * contiguous ranges balanced by the rows' work (adjacency entries + 8 per
 * row); by the nested numbering rank r then owns a contiguous range of every
 * level k <= kp, down to its level-1 rows; levels above kp are replicated.
 * Per PCG iteration (all stream-ordered, no host synchronisation): halo
 * exchange of p (NCCL send/recv), all-reduce of (p, q), all-gather of
 * [y_kp own range, (r, r), gdot], all-reduce of (r, R r).  Iterations run in
 * captured CUDA graphs; the host reads the done flag once per 64.
 *
 * msp_dist_unique_id -- fills id128 (128 bytes, an NCCL unique id); rank 0
 *   calls it and the caller broadcasts the bytes (e.g. torch.distributed).
 * msp_dist_init -- the partition, halo plan and NCCL communicator of `rank`
 *   (1 <= world <= 16); collective over the ranks (NCCL init).  Errors:
 *   MSP_ERR_UNSUPPORTED when the graph is too small for `world` ranks.
 * msp_dist_range -- out[8] = (row0, row1, kp, tp, nsend, nrecv, world, rank)
 *   of the handle's rank; rows in the nested numbering.
 * msp_dist_solve -- PCG-MSP (reading R10) on the partitioned system.  b: the
 *   FULL rhs in the original numbering (host or device per `mem`, the same
 *   on every rank); x receives the solution on the rank's own rows and 0
 *   elsewhere (a sum over ranks assembles it).  report as msp_pcg_solve
 *   (identical on every rank).  MSP_ERR_UNSUPPORTED for graphs whose SELL
 *   slices are wider than 16 (the pair SpMV).
 * msp_dist_group_solve -- the same decomposition for `world` ranks driven by
 *   ONE process on one device (handles hs[0..world), each set up on the same
 *   graph): the collectives become device copies and fixed-order sums on one
 *   stream, nothing waits on anything.  For tests of the partitioned
 *   arithmetic on a single GPU; x is the assembled solution.
 * msp_dist_boundaries / msp_halo_plan -- host-only (no GPU calls) parts of
 *   the plan: quantile boundaries of a non-decreasing prefix cost[m+1] into
 *   bnd[world+1] (MSP_ERR_UNSUPPORTED if a rank would own nothing); the halo
 *   of `rank` given level-1 row boundaries row_bnd[world+1] and the nested
 *   CSR (host): rows received from / sent to each peer (counts, and the
 *   sorted rows if the buffers are non-NULL).
 */
int msp_dist_unique_id(void* id128);
int msp_dist_init(msp_handle* h, int32_t world, int32_t rank, const void* id128, void* stream);
int msp_dist_range(msp_handle* h, int64_t* out8);
int msp_dist_solve(msp_handle* h, const double* b, double* x, double rtol, int32_t maxit, int mem, void* stream,
                   msp_report* report);
int msp_dist_group_solve(msp_handle** hs, int32_t world, const double* b, double* x, double rtol, int32_t maxit,
                         int mem, void* stream, msp_report* report);
int msp_dist_boundaries(int64_t m, const int64_t* cost, int32_t world, int64_t* bnd);
int msp_halo_plan(int64_t n, const int32_t* rowptr, const int32_t* col, int32_t world, const int64_t* row_bnd,
                  int32_t rank, int64_t* recv_counts, int64_t* send_counts, int64_t* recv_rows, int64_t recv_cap,
                  int64_t* send_rows, int64_t send_cap);

/* Thread-local description of the last error (never NULL). */
const char* msp_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* MSP_B200_H */
