/*
 * stokes_er.h -- C ABI of the B200 (sm_100a) hot path of the localized
 * extrapolated-regularization method for nearly singular Stokes layer
 * potentials (PAPER.md = arXiv 2507.00156, LaTeX source).
 *
 * One call evaluates, for M targets y near a closed surface discretized by N
 * quadrature nodes x (weights w, unit outward normals n), the subtracted,
 * regularized single layer (Stokeslet, eq. (10) `Stokes_SL2`)
 * and double layer (stresslet, eq. (11) `Stokes_DL2`)
 *
 *   u^d_i(y) = 1/(8pi) sum_x S^d_ij(y,x) [f_j(x) - (f(x0).n0) n_j(x)] w(x)
 *   v^d_i(y) = 1/(8pi) sum_x T^d_ijk(y,x) [q_j(x) - q_j(x0)] n_k(x) w(x) + chi(y) q_i(x0)
 *
 * with S^d, T^d of eqs. (12)-(13) (split of eq. (7),
 * PAPER.md:59-69) and smoothing factors s1, s2, s3 of eqs. (14)-(16)
 * (PAPER.md:90-102), for delta_k = rho_k h, k = 1..3, and
 * returns the extrapolated value: the u of the 3x3 system eq. (17)
 * with I0, I2 of eqs. (18)-(19),
 * lambda_k = b/delta_k; the same system for v.
 *
 * The regularization is localized: a pair (y, x) is NEAR
 * iff |y - x|^2 <= (STOKES_ER_CUTOFF * max_k delta_k)^2; near pairs use
 * s_i(r/delta_k) for all three delta_k, far pairs use the unregularized S
 * (eq. 3) and T (eq. 4) once, shared by the three sums (eq. (26) `near_far`).
 *
 * Conventions for every entry point below
 *  - All arrays are FP64, "SoA row-major": a [R][C] array stores row r at
 *    offset r*C.  Pointers are DEVICE pointers unless the name says _host.
 *    8-byte alignment is required.  The library never frees or keeps them.
 *  - Targets: y = x0 + b n0 with |n0| = 1, b the signed distance (> 0
 *    outside), x0 the closest surface point.  The library trusts
 *    this consistency; it does no projection.  chi = 1, 1/2, 0 for b < 0,
 *    b == 0, b > 0.
 *  - Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy
 *    default stream).  Device entry points only ENQUEUE work and return; the
 *    caller synchronizes.  No global mutable state: calls on different
 *    streams with different workspaces may run concurrently.
 *  - Workspace: caller-owned device memory of at least
 *    stokes_er_workspace_bytes(M, N, mode) bytes, 256-byte aligned; its
 *    contents need no initialization and are garbage afterwards.
 *  - Errors: a non-zero stokes_er_status is returned and NOTHING is enqueued
 *    when host-side validation fails (EINVAL, EWORKSPACE, EARCH).  ECUDA is
 *    returned if a CUDA call or launch fails (outputs then undefined).
 */
#ifndef STOKES_ER_H
#define STOKES_ER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STOKES_ER_ABI_VERSION 4  /* 4: options.shard_index/shard_count; 3: node-target entry points; 2: options.schedule, NEXT-2, NEXT-3 */
/* c: near iff r <= c * max(delta_k)  ("s1=s2=s3=1 for t > 6") */
#define STOKES_ER_CUTOFF 6.0
/* c for the on-surface s# variant: 1 - s2#(6) = 2.45e-12, 1 - s_i#(7) < 1e-16 (R15) */
#define STOKES_ER_CUTOFF_SURFACE 7.0

typedef enum {
  STOKES_ER_SL = 1,   /* single layer only: f required, out_u written            */
  STOKES_ER_DL = 2,   /* double layer only: q required, out_v written            */
  STOKES_ER_BOTH = 3  /* both                                                    */
} stokes_er_mode;

typedef enum {
  STOKES_ER_OK = 0,
  STOKES_ER_EINVAL = 1,     /* NULL pointer required by mode, M < 0, N < 1, h <= 0 or not
                               finite, rho not positive strictly increasing, bad mode   */
  STOKES_ER_ECUDA = 2,      /* a CUDA runtime call or kernel launch failed              */
  STOKES_ER_EWORKSPACE = 3, /* workspace NULL or smaller than stokes_er_workspace_bytes */
  STOKES_ER_EARCH = 4,      /* current device is not compute capability 10.x (sm_100)   */
  STOKES_ER_ENOCONV = 5     /* stokes_er_twodrop_solve: max_iter reached above tol      */
} stokes_er_status;

/* Bytes of device workspace needed by stokes_er_eval / stokes_er_eval_deltas. */
size_t stokes_er_workspace_bytes(int64_t M, int64_t N, int mode);

/*
 * The hot path.  Inputs (device, FP64):
 *   src_xyz        [3][N]  quadrature nodes x
 *   src_normal     [3][N]  unit outward normals n(x)
 *   src_weight     [N]     quadrature weights w(x) >= 0          (eq. (23))
 *   f              [3][N]  SL density at the nodes   (may be NULL if mode == DL)
 *   q              [3][N]  DL density at the nodes   (may be NULL if mode == SL)
 *   tgt_xyz        [3][M]  targets y
 *   tgt_b          [M]     signed distance b
 *   tgt_x0_density [9][M]  rows 0-2: n0 = n(x0); rows 3-5: f(x0); rows 6-8: q(x0)
 *                          (f/q rows ignored when the mode does not use them)
 *   M >= 0 (M == 0: returns OK, enqueues nothing), N >= 1, h > 0,
 *   rho[3] HOST array, 0 < rho_1 < rho_2 < rho_3 (equal rho make eq. (17) singular)
 * Outputs (device, FP64, fully overwritten):
 *   out_u [3][M] extrapolated SL velocity u (with the 1/(8pi))   (NULL if mode == DL)
 *   out_v [3][M] extrapolated DL velocity v incl. chi q(x0)       (NULL if mode == SL)
 */
int stokes_er_eval(const double* src_xyz, const double* src_normal, const double* src_weight,
                   const double* f, const double* q, const double* tgt_xyz, const double* tgt_b,
                   const double* tgt_x0_density, int64_t M, int64_t N, double h, const double rho[3],
                   int mode, double* out_u, double* out_v, void* workspace, size_t workspace_bytes,
                   void* stream);

/*
 * Same as stokes_er_eval with HOST input/output buffers (pinned memory
 * recommended): enqueues the host->device copies of the inputs into the
 * workspace, the evaluation, and the device->host copies of out_u / out_v,
 * then SYNCHRONIZES `stream` (the host outputs are valid on return).
 * Workspace: stokes_er_host_workspace_bytes(M, N, mode) device bytes.
 */
size_t stokes_er_host_workspace_bytes(int64_t M, int64_t N, int mode);
int stokes_er_eval_host(const double* src_xyz_host, const double* src_normal_host,
                        const double* src_weight_host, const double* f_host, const double* q_host,
                        const double* tgt_xyz_host, const double* tgt_b_host,
                        const double* tgt_x0_density_host, int64_t M, int64_t N, double h,
                        const double rho[3], int mode, double* out_u_host, double* out_v_host,
                        void* workspace, size_t workspace_bytes, void* stream);

/*
 * Debug / test entry point: the three per-delta values u^{delta_k}, v^{delta_k}
 * of eqs. (10)-(11) (incl. 1/(8pi) and chi q(x0)), same localized near/far
 * rule, no extrapolation.  out_udelta, out_vdelta: [3][3][M] = [k][i][m].
 * A simple one-target-per-thread kernel (not the tuned path).
 */
int stokes_er_eval_deltas(const double* src_xyz, const double* src_normal, const double* src_weight,
                          const double* f, const double* q, const double* tgt_xyz, const double* tgt_b,
                          const double* tgt_x0_density, int64_t M, int64_t N, double h,
                          const double rho[3], int mode, double* out_udelta, double* out_vdelta,
                          void* workspace, size_t workspace_bytes, void* stream);

/*
 * The extrapolation solve alone (eq. (17)): for each target m and column c,
 * out[c][m] = u solving  u + c1 rho_k I0(b/delta_k) + c2 rho_k^3 I2(b/delta_k) = in[k][c][m].
 * in_delta [3][C][M] device, out [C][M] device, tgt_b [M] device, 1 <= C <= 64.
 * Targets with |b| > STOKES_ER_CUTOFF * delta_3 (no near pairs, all u^{delta_k}
 * equal) and numerically singular systems return in[0][c][m] (R7).
 */
int stokes_er_extrapolate(const double* tgt_b, int64_t M, double h, const double rho[3],
                          const double* in_delta, int C, double* out, void* stream);

/*
 * NEXT-1: on-surface evaluation with the modified factors s1#, s2#, s3# of
 * PAPER.md Sec. 2.1 (lines 126-139) at ONE smoothing length delta (the
 * paper uses delta = 3h for self-surface integrals), no
 * extrapolation.  SL: S^delta of eq. (12) with s1#, s2#; DL: the unsplit
 * stresslet eq. (4) times s3# (R16) plus chi q(x0).  Near iff
 * r <= STOKES_ER_CUTOFF_SURFACE * delta.  Same arrays, workspace
 * (stokes_er_workspace_bytes) and error behaviour as stokes_er_eval;
 * intended for targets on the surface (b = 0, chi = 1/2).
 */
int stokes_er_eval_onsurface(const double* src_xyz, const double* src_normal, const double* src_weight,
                             const double* f, const double* q, const double* tgt_xyz, const double* tgt_b,
                             const double* tgt_x0_density, int64_t M, int64_t N, double delta, int mode,
                             double* out_u, double* out_v, void* workspace, size_t workspace_bytes,
                             void* stream);

/* Number of kernel launches one stokes_er_eval(M, N, mode) enqueues (ours; 4 when N, M <= 8192: the
 * counting-rank Morton prologue in one launch, no memset; 7 otherwise, plus the CUB radix-sort launches). */
int stokes_er_launch_count(int64_t M, int64_t N, int mode);

/* Optional profiling hooks for bench.py: if non-NULL, cudaEvent_t handles
 * (as void*) recorded on `stream` immediately before / after the far-field
 * pair-sum kernel (the dominant kernel) of this stokes_er_eval_ex call.  While
 * `stream` is being captured into a CUDA graph they are captured as external
 * event-record nodes (cudaEventRecordExternal), so each replay records them. */
typedef struct {
  void* pair_kernel_start_event;
  void* pair_kernel_end_event;
  int targets_per_thread; /* 0 = default (2); 1..4 (tuning/tests)         */
  int source_chunk_tiles; /* 0 = automatic; work item = chunk * 128 sources */
  int64_t stats[4];       /* out: [0] work items, [1] grid CTAs, [2] chunk tiles, [3] targets/thread */
  void* near_kernel_start_event; /* optional events around the near-field kernel */
  void* near_kernel_end_event;
  int near_phases;               /* 0 = automatic; near work units per 32-target group (1..128; node path 1..64) */
  int schedule;                  /* STOKES_ER_SCHEDULE_FUSED (0, default): one persistent kernel whose
                                    CTAs take far items (a target block x a source chunk) and near
                                    items (one near unit per warp) from one queue that interleaves
                                    them, so far and near work share every SM's FP64 pipe;
                                    STOKES_ER_SCHEDULE_SEPARATE (1): far kernel, then near kernel.
                                    Both give the same sums (same per-slot partials, same fixed-order
                                    finalize).  FUSED records only the pair_kernel events (around
                                    the one pair kernel). */
  int shard_index;               /* node path (stokes_er_eval_nodes_ex) only: with shard_count > 1 this call */
  int shard_count;               /* computes shard shard_index of the evaluation -- a contiguous 1/shard_count
                                    of the symmetric kernel's block-pair items and of the neighbour units'
                                    target groups -- and returns PARTIAL out_u, out_v (chi q0 only in shard
                                    0) whose sum over the shards is the evaluation (one all-reduce across
                                    GPUs).  0 / 0 or 0 / 1: the whole evaluation. */
} stokes_er_options;

#define STOKES_ER_SCHEDULE_FUSED 0
#define STOKES_ER_SCHEDULE_SEPARATE 1

/* Workspace for stokes_er_eval_ex with these tuning options (>= stokes_er_workspace_bytes
 * when the options force a finer source chunking). */
size_t stokes_er_workspace_bytes_ex(int64_t M, int64_t N, int mode, const stokes_er_options* options);

int stokes_er_eval_ex(const double* src_xyz, const double* src_normal, const double* src_weight,
                      const double* f, const double* q, const double* tgt_xyz, const double* tgt_b,
                      const double* tgt_x0_density, int64_t M, int64_t N, double h, const double rho[3],
                      int mode, double* out_u, double* out_v, void* workspace, size_t workspace_bytes,
                      void* stream, stokes_er_options* options);

/* ================================================================ node targets
 * Evaluation AT THE QUADRATURE NODES: the targets are the N nodes themselves,
 * on the surface (b = 0, chi = 1/2), with x0 = the node, n0 = its
 * normal, f(x0) = f and q(x0) = q at the node.  The result is exactly that of
 * stokes_er_eval with M = N, tgt_xyz = src_xyz, tgt_b = 0 and tgt_x0_density =
 * [src_normal; f; q] (same formulas, same localization and extrapolation; the
 * paper's on-surface targets, PAPER.md:249 with b = 0, and BASELINE.json
 * config 5).  Out: out_u, out_v [3][N] in the caller's node order.
 *
 * Node targets make the far-field pair sum symmetric: S(d) is even and T(d)
 * odd in d = x_i - x_j (eqs. (3)-(4)), and q0 = q at a node
 * makes the stresslet's d.(q_j - q_i) shared as well, so ONE evaluation of a
 * far pair's geometry (d, r^2, 1/r, 1/r^2, 1/r^5) and of d.(q_j - q_i) serves
 * both directed pairs (i <- j) and (j <- i).  Results are deterministic (no
 * data atomics; fixed summation order) and equal stokes_er_eval's to rounding.
 *
 * Arrays, errors and streams as stokes_er_eval (N >= 1; mode, h, rho alike).
 * Workspace: stokes_er_nodes_workspace_bytes(N, mode) device bytes -- it holds
 * one accumulator slice of 48 N bytes per persistent CTA (148), i.e. ~7.1 KB
 * per node (7.8 GB at N = 1.09e6), sized for the B200's 180 GB of HBM.
 * stokes_er_eval_nodes_ex takes the same options struct as stokes_er_eval_ex:
 * the pair_kernel events bracket the symmetric far kernel, the near_kernel
 * events the neighbour kernel (near pairs + the far pairs of the blocks the
 * symmetric kernel leaves out); near_phases is honoured; stats[0..3] = items,
 * CTAs, R blocks per item, I nodes per lane (3).
 */
size_t stokes_er_nodes_workspace_bytes(int64_t N, int mode);
size_t stokes_er_nodes_workspace_bytes_ex(int64_t N, int mode, const stokes_er_options* options);
int stokes_er_eval_nodes(const double* src_xyz, const double* src_normal, const double* src_weight,
                         const double* f, const double* q, int64_t N, double h, const double rho[3], int mode,
                         double* out_u, double* out_v, void* workspace, size_t workspace_bytes, void* stream);
int stokes_er_eval_nodes_ex(const double* src_xyz, const double* src_normal, const double* src_weight,
                            const double* f, const double* q, int64_t N, double h, const double rho[3], int mode,
                            double* out_u, double* out_v, void* workspace, size_t workspace_bytes, void* stream,
                            stokes_er_options* options);
/* NEXT-1 at the nodes: stokes_er_eval_onsurface (s# factors of PAPER.md:126-139, one delta,
 * cutoff STOKES_ER_CUTOFF_SURFACE, no extrapolation) with the targets = the N nodes, through
 * the same symmetric far kernel.  Workspace: stokes_er_nodes_workspace_bytes(N, mode).  The
 * two-drop solver's self blocks are exactly this call. */
int stokes_er_eval_nodes_onsurface(const double* src_xyz, const double* src_normal, const double* src_weight,
                                   const double* f, const double* q, int64_t N, double delta, int mode,
                                   double* out_u, double* out_v, void* workspace, size_t workspace_bytes,
                                   void* stream);
/* HOST buffers (pinned recommended): H2D, evaluation, D2H, then synchronizes `stream`.
 * Workspace: stokes_er_nodes_host_workspace_bytes(N, mode) device bytes. */
size_t stokes_er_nodes_host_workspace_bytes(int64_t N, int mode);
int stokes_er_eval_nodes_host(const double* src_xyz_host, const double* src_normal_host,
                              const double* src_weight_host, const double* f_host, const double* q_host, int64_t N,
                              double h, const double rho[3], int mode, double* out_u_host, double* out_v_host,
                              void* workspace, size_t workspace_bytes, void* stream);
/* Statistics for benchmarks (synchronizes `stream`; not for the hot path): after a
 * stokes_er_eval_nodes call with this workspace (same N, mode, h, rho), counts_host[0] =
 * directed pairs of real nodes summed by the symmetric far kernel (2 per shared pair),
 * counts_host[1] = N^2 - counts_host[0], the pairs the neighbour kernel owns. */
int stokes_er_nodes_pair_counts(int64_t N, int mode, double h, const double rho[3], void* workspace,
                                size_t workspace_bytes, int64_t* counts_host, void* stream);
/* Kernel launches one stokes_er_eval_nodes enqueues (ours; CUB's sort launches excluded). */
int stokes_er_nodes_launch_count(int64_t N, int mode);

/* Treecode parameters (NEXT-3, Sec. 3.4; section below). */
typedef struct {
  int leaf_size;          /* N0: at most N0 points per leaf                          */
  int degree;             /* p: Chebyshev degree per axis, 1..16                     */
  double theta;           /* MAC parameter (0: never approximate = direct sum)       */
} stokes_er_tree_params;

/* ===================================================================== NEXT-2
 * Two-drop interfacial Stokes flow (Sec. 4.3): the
 * interface velocity u on two drops solves the integral equation (35)
 * (`IE-2Surf`), for x0 on drop b, m != b:
 *
 *   (lambda_b + 1) u(x0) = -(1/(4 pi mu0)) sum_m int_m S [f] dS + sum_m (lambda_m - 1)/(4 pi) int_m T u n dS
 *
 * written with this library's evaluators (which carry 1/(8 pi)) as
 *
 *   A u|_b = (lambda_b + 1) u_b - 2 (lambda_b - 1) DL_bb[u_b] - 2 (lambda_m - 1) DL_bm[u_m]
 *   rhs_b  = -(2/mu0) (SL_bb[[f]_b] + SL_bm[[f]_m])
 *
 * Self blocks (bb) are stokes_er_eval_onsurface at delta_self (paper: 3h;
 * DL_bb is the principal value, chi = 1/2); cross blocks (bm) are
 * stokes_er_eval with rho (paper: 3,4,5) and targets = drop b's nodes whose
 * closest point x0 on drop m the caller supplies (b', n0, [f]_m(x0)).  The
 * cross DL subtracts u_m(x0), which is not a node value: it is the value at
 * x0 of the least-squares polynomial of total degree <= 4 in tangent-plane
 * coordinates over drop m's nodes within 3.5 h of x0 (R20).  The
 * solve is full GMRES (modified Gram-Schmidt, no restart) from u = 0 until
 * ||rhs - A u|| <= tol ||rhs|| (R21).
 *
 * Vectors u, rhs, A u: [3 N_1 + 3 N_2] device, drop 1 then drop 2, each [3][N_b].
 * Workspace: caller-owned device memory of stokes_er_twodrop_workspace_bytes;
 * stokes_er_twodrop_setup writes the interpolation stencils into it, and the
 * other calls read them (same drops, cross, params and workspace).
 * rhs/apply only enqueue on `stream`; setup and solve synchronize `stream`.
 * Errors as above; EINVAL also when a stencil finds fewer than 15 or more
 * than STOKES_ER_INTERP_KMAX nodes (setup), ENOCONV (5) when solve reaches
 * max_iter above tol (out_u then holds the last iterate).
 */
#define STOKES_ER_INTERP_KMAX 192

typedef struct {
  int64_t N;              /* quadrature nodes of the drop                          */
  const double* xyz;      /* [3][N] nodes                                          */
  const double* normal;   /* [3][N] outward unit normals                           */
  const double* weight;   /* [N]    quadrature weights                             */
  const double* f;        /* [3][N] interface force jump [f] at the nodes          */
  double lambda;          /* viscosity ratio mu_drop / mu0                         */
} stokes_er_drop;

typedef struct {          /* cross[b]: targets = nodes of drop b, sources = drop 1-b */
  const double* b;        /* [N_b] signed distance of the node to drop 1-b (> 0)    */
  const double* x0d;      /* [6][N_b]: n0 at the closest point x0 on drop 1-b (3),
                                       [f]_{1-b}(x0) (3); x0 = y - b n0              */
} stokes_er_cross;

typedef struct {
  double h;               /* grid spacing of both drops                            */
  double rho[3];          /* cross blocks: delta_k = rho_k h, strictly increasing  */
  double delta_self;      /* self blocks: the s# smoothing length                  */
  double mu0;             /* exterior viscosity                                    */
  double tol;             /* GMRES relative residual                               */
  int max_iter;           /* Krylov dimension cap, 1..512                          */
  int use_tree;           /* 0: direct sums; 1: every block through the treecode
                             (NEXT-3, "We apply ... the treecode to all
                             the integrals") with the plans below                 */
  const void* tree_plan[2]; /* host plans (stokes_er_tree_build) over each drop's
                             nodes, built with the same stokes_er_tree_params      */
  const stokes_er_tree_params* tree; /* treecode parameters (use_tree = 1)        */
} stokes_er_twodrop_params;

/* Workspace for max_iter Krylov steps with direct sums (use_tree = 0). */
size_t stokes_er_twodrop_workspace_bytes(int64_t N1, int64_t N2, int max_iter);
/* Workspace for these parameters (either mode). */
size_t stokes_er_twodrop_workspace_bytes_ex(int64_t N1, int64_t N2, const stokes_er_twodrop_params* params);
int stokes_er_twodrop_setup(const stokes_er_drop drops[2], const stokes_er_cross cross[2],
                            const stokes_er_twodrop_params* params, void* workspace, size_t workspace_bytes,
                            void* stream);
int stokes_er_twodrop_rhs(const stokes_er_drop drops[2], const stokes_er_cross cross[2],
                          const stokes_er_twodrop_params* params, double* out_rhs, void* workspace,
                          size_t workspace_bytes, void* stream);
int stokes_er_twodrop_apply(const stokes_er_drop drops[2], const stokes_er_cross cross[2],
                            const stokes_er_twodrop_params* params, const double* u, double* out_Au,
                            void* workspace, size_t workspace_bytes, void* stream);
/* out_iters: Arnoldi steps taken; out_res_host: [max_iter] relative residual
 * estimate after each step (host, may be NULL). */
int stokes_er_twodrop_solve(const stokes_er_drop drops[2], const stokes_er_cross cross[2],
                            const stokes_er_twodrop_params* params, double* out_u, int* out_iters,
                            double* out_res_host, void* workspace, size_t workspace_bytes, void* stream);

/* ===================================================================== NEXT-3
 * The kernel-independent treecode of PAPER.md Sec. 3.4 (lines 194-233) for the
 * far part of the localized sums: sources partitioned into an octree with at
 * most leaf_size (N0) points per leaf (host, stokes_er_tree_build; readings
 * R22-R25 in DESIGN.md); modified weights (eq. (32)) at the (degree+1)^3
 * second-kind Chebyshev points of every cluster; per target, a cluster is
 * approximated by eq. (31) with the unregularized S, T when the MAC
 * r_c / R <= theta (eq. (28)) holds AND its box lies beyond the cutoff
 * (gap > STOKES_ER_CUTOFF max delta_k, so no near pair is approximated), else
 * its children are checked; a leaf that fails is summed directly with the
 * localized 3-delta regularization.  The extrapolation is as in stokes_er_eval.
 * The paper's parameter policy (eq. (33)): theta = 0.6,
 * N0 = 2000 and p = 6 at h = 1/64, N0 doubling and p + 2 per halving of h.
 *
 * Plan: HOST memory of stokes_er_tree_plan_bytes(N, params) bytes, written by
 * stokes_er_tree_build from HOST node positions [3][N]; reusable for every
 * evaluation on the same nodes (densities may change).  stokes_er_eval_tree
 * copies it to the device workspace (stokes_er_tree_workspace_bytes) on
 * `stream`; other arguments and errors as stokes_er_eval.  EINVAL also for a
 * plan built for another N, degree > 16, or a tree over 8 N/N0 + 4096 nodes or
 * 63 levels.
 */
/* stokes_er_tree_params: see the NEXT-3 section below (declared here for NEXT-2). */

size_t stokes_er_tree_plan_bytes(int64_t N, const stokes_er_tree_params* params);
int stokes_er_tree_build(const double* src_xyz_host, int64_t N, const stokes_er_tree_params* params, void* plan,
                         size_t plan_bytes);
int stokes_er_tree_info(const void* plan, int64_t N, int64_t* out_nodes, int64_t* out_depth);
size_t stokes_er_tree_workspace_bytes(int64_t M, int64_t N, int mode, const stokes_er_tree_params* params,
                                      const void* plan);
int stokes_er_eval_tree(const double* src_xyz, const double* src_normal, const double* src_weight, const double* f,
                        const double* q, const double* tgt_xyz, const double* tgt_b, const double* tgt_x0_density,
                        int64_t M, int64_t N, double h, const double rho[3], int mode,
                        const stokes_er_tree_params* params, const void* plan, double* out_u, double* out_v,
                        void* workspace, size_t workspace_bytes, void* stream);

/* NEXT-1 with the treecode: the on-surface s# evaluation of
 * stokes_er_eval_onsurface (one delta, cutoff STOKES_ER_CUTOFF_SURFACE * delta)
 * with the far part from the treecode (guard distance 7 delta).  Workspace:
 * stokes_er_tree_workspace_bytes. */
int stokes_er_eval_tree_onsurface(const double* src_xyz, const double* src_normal, const double* src_weight,
                                  const double* f, const double* q, const double* tgt_xyz, const double* tgt_b,
                                  const double* tgt_x0_density, int64_t M, int64_t N, double delta, int mode,
                                  const stokes_er_tree_params* params, const void* plan, double* out_u,
                                  double* out_v, void* workspace, size_t workspace_bytes, void* stream);

const char* stokes_er_status_string(int status);
int stokes_er_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* STOKES_ER_H */
