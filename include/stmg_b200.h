/*
 * stmg_b200 — C ABI of the B200-native hp space-time multigrid hot path
 * (arXiv 2502.09159): matrix-free space-time operator, additive Vanka
 * smoothers, hp transfers, V-cycle, right-preconditioned GMRES and time
 * marching for 2D instationary Stokes, Q_{r+1}/P_r^disc x DG(k), FP64.
 *
 * Every entry point replaces one interface of the reference C++ library
 * (/root/reference/proj, cited per function). The reference binds these as
 * std::function callbacks (ApplyFn / PrecondFn, include/stmg/solver.hpp:70-71)
 * consumed by gmres() and time_march(); INTEGRATION.md shows the adapter.
 *
 * Conventions
 *  - Plain pointers and sizes only. Functions without a `_host` suffix take
 *    DEVICE pointers and are ordered on the context's CUDA stream
 *    (stmg_ctx_set_stream); `_host` variants take host pointers and block.
 *  - Vectors use the reference BlockVector layout (block_vector.hpp:13-45):
 *    one interval = [V^1..V^{k+1}, P^1..P^{k+1}], V^a = [comp 0 | comp 1] on
 *    the global GLL grid (node id iy*grid_x + ix), P^a cell-blocked
 *    (cell*n_p + mode). N intervals are stored interval-major.
 *  - Status codes (no exceptions cross the ABI):
 *      0 STMG_OK, 1 STMG_EINVAL  (reference: std::invalid_argument),
 *      2 STMG_ERUNTIME (reference: std::runtime_error — singular matrix,
 *        caps, GMRES non-convergence), 3 STMG_ECUDA.
 *    stmg_last_error() returns the message of the calling thread's last
 *    failure.
 */
#ifndef STMG_B200_H
#define STMG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STMG_OK 0
#define STMG_EINVAL 1
#define STMG_ERUNTIME 2
#define STMG_ECUDA 3

#define STMG_SMOOTHER_NONE (-1)
#define STMG_SMOOTHER_CELL 0        /* SmootherKind::cell        (vanka.hpp:15-19) */
#define STMG_SMOOTHER_VERTEX_STAR 1 /* SmootherKind::vertex_star (vanka.hpp:15-19) */

typedef struct stmg_ctx stmg_ctx;
typedef struct stmg_level stmg_level;
typedef struct stmg_solver stmg_solver;

const char *stmg_last_error(void);
/* Library version string, e.g. "stmg_b200 0.1 sm_100a". */
const char *stmg_version(void);

/* Tuning hooks (process-wide; 0 restores the default heuristic). No
 * reference counterpart: they fix launch shapes the library otherwise derives
 * from the level size, so tests can reach every packing of the kernels.
 *   "vanka_group"     intervals per block of the DMMA item kernels (n_T <= 176)
 *   "vanka_big_group" intervals per block of the big-patch kernel (n_T > 176)
 * Unknown keys or values outside [0, 1024]: STMG_EINVAL. */
int stmg_set_tuning(const char *key, int64_t value);

/* ------------------------------------------------------------ context */
int stmg_ctx_create(int device, stmg_ctx **out);
int stmg_ctx_destroy(stmg_ctx *ctx);
/* cudaStream_t passed as void*; NULL selects the legacy default stream. */
int stmg_ctx_set_stream(stmg_ctx *ctx, void *cuda_stream);
int stmg_ctx_synchronize(stmg_ctx *ctx);
/* Number of kernels this context has launched so far (evidence counter). */
int64_t stmg_ctx_launch_count(const stmg_ctx *ctx);

/* ------------------------------------------------------------ one level
 * SpaceTimeBlockOperator (st_operator.hpp:94-165) + VankaSmoother
 * (vanka.hpp:45-89) on an nx x ny Cartesian mesh of the unit square, with
 * Q_{r+1}/P_r^disc in space, DG(k) on intervals of length tau, viscosity nu
 * and grad-div coefficient gamma. smoother_kind: STMG_SMOOTHER_*.
 * r in 1..4, k in 0..4. */
int stmg_level_create(stmg_ctx *ctx, int nx, int ny, int r, int k, double tau, double nu, double gamma,
                      int smoother_kind, stmg_level **out);
int stmg_level_destroy(stmg_level *level);
/* out[0..9] = n_slots, M^v, M^p, interval size, n_scalar, grid_x,
 * n_patch_classes, sum over patches of n_T^2 (total_matrix_elements,
 * vanka.cpp:235-243), 1 if the smoother applies the time-diagonalised
 * (factored) patch inverses, and their multiply-adds per interval. */
int stmg_level_sizes(const stmg_level *level, int64_t *out);

/* y_n = D x_n for each of n_intervals independent intervals
 * (apply_block, raw=0: Dirichlet elimination, st_operator.cpp:397-401;
 *  apply_block_raw, raw=1: st_operator.cpp:403-407). */
int stmg_apply_block(stmg_level *level, const double *x, double *y, int n_intervals, int raw);

/* All-at-once operator of Eq. GloSys:
 *   y_n = D x_n - Z C x_{n-1}[slot k]        n = 0..n_intervals-1
 * with C the DG jump coupling (coupling_rhs, st_operator.cpp:409-421) and Z
 * zeroing constrained rows. x_prev_slot (M^v doubles, may be NULL) is the
 * velocity of slot k of the interval preceding x (the time-slab halo). */
int stmg_vmult(stmg_level *level, const double *x, double *y, int n_intervals, const double *x_prev_slot);

/* r = b - A x with A = stmg_vmult's operator (coupled=1) or the per-interval
 * apply_block (coupled=0). */
int stmg_residual(stmg_level *level, const double *b, const double *x, double *r, int n_intervals,
                  const double *x_prev_slot, int coupled);

/* Saddle-point health of converged steps (solver.cpp:286-299): per interval
 * out[2n] = max over slots of ||B v|| / sqrt(v^T M v), out[2n+1] = max over
 * slots of |<mean, p>| / ||p|| (the StepRecord fields of time_march). */
int stmg_step_health(stmg_level *level, const double *X, int n_intervals, double *out);

/* out = coupling_rhs(v_prev) for one interval (st_operator.cpp:409-421). */
int stmg_coupling_rhs(stmg_level *level, const double *v_prev, double *out);

/* out = sum_T R_T^T w_T (R_T S R_T^T)^{-1} R_T r per interval
 * (VankaSmoother::apply_additive, vanka.cpp:196-215). */
int stmg_apply_additive(stmg_level *level, const double *r, double *out, int n_intervals);

/* u <- u + omega * apply_additive(b - A u) (VankaSmoother::smooth_step,
 * vanka.cpp:217-233); A as in stmg_residual. omega must lie in (0, 1]
 * (else STMG_EINVAL, vanka.cpp:223-224). `work` is a caller buffer of
 * n_intervals interval sizes (may be NULL: the level allocates one). */
int stmg_smooth_step(stmg_level *level, const double *b, double *u, double omega, int n_intervals,
                     const double *x_prev_slot, int coupled, double *work);

/* u += omega * apply_additive(r): the patch-solve half of smooth_step
 * (vanka.cpp:229-232) for a precomputed residual r. */
int stmg_vanka_update(stmg_level *level, const double *r, double *u, double omega, int n_intervals);

/* Host-buffer variants of stmg_vmult / stmg_smooth_step: copy in, run,
 * copy out, synchronise (the end-to-end path a CPU caller binds). Pipelined
 * over 4-interval chunks on separate H2D / D2H streams; pinned host memory
 * lets the copies overlap the kernels. */
int stmg_vmult_host(stmg_level *level, const double *x, double *y, int n_intervals, const double *x_prev_slot);
int stmg_smooth_step_host(stmg_level *level, const double *b, double *u, double omega, int n_intervals,
                          const double *x_prev_slot, int coupled);
/* Non-blocking variants: enqueue the copies and kernels on the context's
 * streams and return; the host buffers must stay valid and untouched until
 * stmg_ctx_synchronize. Consecutive calls overlap (the next call's H2D copies
 * run while the previous call computes and copies back); a call waits only
 * for the previous call of the same kind to release its device staging. */
int stmg_vmult_host_async(stmg_level *level, const double *x, double *y, int n_intervals, const double *x_prev_slot);
int stmg_smooth_step_host_async(stmg_level *level, const double *b, double *u, double omega, int n_intervals,
                                const double *x_prev_slot, int coupled);

/* ------------------------------------------------------------ built-in problems
 * The reference's manufactured problem (problems.cpp:13-62): its load vector
 * via SpaceTimeBlockOperator::assemble_rhs (st_operator.cpp:423-467) and its
 * space-time error norms via compute_errors (harness.cpp:72-183), on the
 * device. F / X hold n_intervals consecutive intervals of this level, interval
 * i covering [t_start + i tau, t_start + (i+1) tau]. The force uses the
 * level's nu (the reference problem has nu = 0.1). assemble_rhs writes the
 * velocity rows (pressure rows 0, constrained rows 0). compute_errors writes
 * out[0..4] = e_v L2(L2), e_p L2(L2), e_v L2(H1-seminorm), ||div v|| L2(L2),
 * e_v max over quadrature points (host array). r <= 4, k <= 4. */
#define STMG_PROBLEM_MANUFACTURED 0
#define STMG_PROBLEM_CAVITY 1 /* lid-driven cavity (problems.cpp:64-78): boundary data only */
int stmg_assemble_rhs(stmg_level *level, int problem, double t_start, double *F, int n_intervals);
int stmg_compute_errors(stmg_level *level, int problem, double t_start, const double *X, int n_intervals,
                        double *out);
/* interpolate_exact (harness.cpp:185-239): the built-in exact solution as a
 * trajectory X (nodal velocity at the GLL grid, per-cell L2-projected
 * pressure), n_intervals intervals from t_start. */
int stmg_interpolate_exact(stmg_level *level, int problem, double t_start, double *X, int n_intervals);

/* ------------------------------------------------------------ solver
 * build_setup + VCycle + gmres + time_march (harness.cpp:26-70,
 * solver.cpp:56-325) on the 2^refinements x 2^refinements unit-square mesh:
 * hp hierarchy (spatial p-halving then h-doubling to 1x1; temporal k -> 1),
 * or h-only when h_only != 0. k < 0 selects k = r; n_steps <= 0 selects
 * tau = t_end / 2^(refinements+1) (harness.cpp:16-24). The coarse level is
 * solved on the GPU with a dense inverse of the pinned operator. */
int stmg_solver_create(stmg_ctx *ctx, int refinements, int r, int k, int n_steps, double t_end, double nu,
                       double gamma, int smoother_kind, int nu1, int nu2, double omega, int h_only, double rtol,
                       double atol, int max_iterations, stmg_solver **out);
int stmg_solver_destroy(stmg_solver *solver);
/* out[0] = n_levels, out[1] = n_steps, then per level l (coarse first):
 * out[2+5l..] = nx, r, k, kind_to_coarser (TransferKind, transfer.hpp:15-23),
 * interval size. */
int stmg_solver_info(const stmg_solver *solver, int64_t *out);
/* Borrowed handle of level l (0 = coarsest); owned by the solver. */
stmg_level *stmg_solver_level(stmg_solver *solver, int l);

/* TransferPair::restrict_residual / prolongate_correction between level l
 * and l-1 (transfer.cpp:102-132), one interval. prolongate writes
 * (accumulate=0) or adds (accumulate=1) into fine. */
int stmg_restrict_residual(stmg_solver *solver, int l, const double *fine, double *coarse, int project_pressure);
int stmg_prolongate_correction(stmg_solver *solver, int l, const double *coarse, double *fine,
                               int project_pressure, int accumulate);
/* CoarseSolver::solve (solver.cpp:43-54) on level 0. */
int stmg_coarse_solve(stmg_solver *solver, const double *b, double *x);
/* x = VCycle::apply(b) (solver.cpp:63-93), finest level, one interval. */
int stmg_vcycle(stmg_solver *solver, const double *b, double *x);
/* Right-preconditioned GMRES (solver.cpp:95-202) of apply_block x = b with
 * the V-cycle, x0 = 0. iterations/converged/residual history as GmresResult.
 * Returns STMG_ERUNTIME if not converged. */
int stmg_gmres(stmg_solver *solver, const double *b, double *x, int *iterations, double *residual_history,
               int history_cap);
/* time_march (solver.cpp:204-325) with zero initial velocity, homogeneous
 * Dirichlet data and a per-step load vector F_n (n_steps intervals,
 * interval-major) added to the right-hand side; writes the trajectory X
 * (n_steps intervals, pressure projected mean-zero per slot) and the GMRES
 * iterations of each step. */
int stmg_time_march(stmg_solver *solver, const double *F, double *X, int *iterations);
int stmg_time_march_host(stmg_solver *solver, const double *F, double *X, int *iterations);
/* time_march (solver.cpp:204-325) of a built-in problem with the solver's nu:
 * STMG_PROBLEM_MANUFACTURED assembles its force every step (assemble_rhs);
 * STMG_PROBLEM_CAVITY has no force and inhomogeneous Dirichlet data, applied
 * by the reference's lift: rhs -= A_raw lift, solve, x += lift
 * (solver.cpp:251-283). Zero initial velocity. */
int stmg_time_march_problem(stmg_solver *solver, int problem, double *X, int *iterations);
/* time_march with all of the reference's problem data as vectors; every
 * pointer may be NULL:
 *  - F: per-step load vectors (n_steps intervals);
 *  - lifts: general inhomogeneous Dirichlet data. n_steps interval vectors
 *    hold the boundary values g(x, y, t_a) of every slot on the constrained
 *    velocity nodes and zero elsewhere (set_boundary_values,
 *    dof_space.cpp:71-81). Step n solves with rhs -= A_raw lift_n and
 *    returns x + lift_n (solver.cpp:251-283);
 *  - v_init: the initial velocity at the nodes (M^v doubles,
 *    solver.cpp:229-236). */
int stmg_time_march_ex(stmg_solver *solver, const double *F, const double *lifts, const double *v_init, double *X,
                       int *iterations);

/* ------------------------------------------------------------ all-at-once
 * The global space-time system of Eq. GloSys: the block
 * lower-bidiagonal operator (A X)_n = D X_n - C X_{n-1} over a slab of
 * n_intervals intervals. It is solved by right-preconditioned FGMRES (the
 * reference's gmres, solver.cpp:95-202) with an all-at-once V-cycle:
 *  - Vanka smoothing of all intervals at once, residuals carrying the jump
 *    coupling;
 *  - the reference's spatial / temporal-p transfers per interval;
 *  - an exact coarse solve by block forward substitution in time.
 * The reference only time-marches (solver.cpp:204-325), so this path is
 * pinned by the identity "all-at-once solution = time-marched solution"
 * (SURVEY §8c).
 *
 * Time-slab partition: with a communicator installed, rank p owns
 * intervals [p*n_intervals, (p+1)*n_intervals) of a world*n_intervals system
 * (equal slabs). The library calls back for the only three exchanges the path
 * has. Every buffer is device memory, and every call is stream-ordered on
 * `stream` (the context's stream):
 *  - exchange_halo: send n doubles (slot-k velocity of this rank's last
 *    interval) to rank+1 and receive rank-1's into recv. The first rank
 *    receives nothing; the last rank sends nothing.
 *  - allreduce_sum: in-place sum over ranks of n doubles (Krylov dots).
 *  - allgather: recv[r*n .. (r+1)*n) = send of rank r (coarse right-hand sides).
 * Callbacks return 0 on success. */
typedef struct stmg_comm_ops {
    void *user;
    int rank;
    int world;
    int (*exchange_halo)(void *user, const double *send, double *recv, int64_t n, void *stream);
    int (*allreduce_sum)(void *user, double *buf, int64_t n, void *stream);
    int (*allgather)(void *user, const double *send, double *recv, int64_t n, void *stream);
} stmg_comm_ops;
/* Install (ops != NULL, copied) or remove (NULL) the communicator. */
int stmg_solver_set_comm(stmg_solver *solver, const stmg_comm_ops *ops);

/* Arnoldi orthogonalization of gmres / the all-at-once FGMRES:
 * STMG_ORTHO_MGS (default) is the reference's modified Gram-Schmidt
 * (solver.cpp:146-152): j+1 all-reduces in iteration j under a time-slab
 * partition. STMG_ORTHO_CGS2 is classical Gram-Schmidt applied twice with
 * batched inner products: two all-reduces per iteration. Same Krylov space;
 * iteration counts agree within +-1. */
#define STMG_ORTHO_MGS 0
#define STMG_ORTHO_CGS2 1
int stmg_solver_set_krylov(stmg_solver *solver, int orthogonalization);

/* NCCL time-slab communicator inside the library (no caller callbacks in the
 * per-iteration path): NCCL is loaded at run time (libnccl.so.2), so the
 * library itself has no link-time NCCL dependency.
 *  - stmg_comm_nccl_unique_id: rank 0 creates the 128-byte ncclUniqueId, the
 *    caller broadcasts it (any channel) to every rank;
 *  - stmg_comm_nccl_create: one communicator per rank on `device`;
 *  - stmg_comm_nccl_ops: fills an stmg_comm_ops whose callbacks run NCCL
 *    (send/recv for the halo, all-reduce, all-gather) on the given stream;
 *    pass it to stmg_solver_set_comm / stmg3_solver_set_comm. The ops stay
 *    valid until stmg_comm_destroy. */
typedef struct stmg_comm stmg_comm;
int stmg_comm_nccl_unique_id(void *unique_id_out /* 128 bytes */);
int stmg_comm_nccl_create(const void *unique_id, int rank, int world, int device, stmg_comm **out);
int stmg_comm_nccl_ops(stmg_comm *comm, stmg_comm_ops *ops_out);
int stmg_comm_destroy(stmg_comm *comm);
/* One all-at-once V-cycle x = V(b) on the finest level, n_intervals intervals. */
int stmg_vcycle_all_at_once(stmg_solver *solver, const double *b, double *x, int n_intervals);
/* Solve A X = F on the slab. v_init (nullable, M^v doubles) is the slot-k
 * velocity entering the slab's first interval: the hand-off between
 * consecutive macro steps. Only the first rank reads it.
 * X is projected mean-zero per slot. iterations receives the FGMRES
 * iteration count. */
int stmg_solve_all_at_once(stmg_solver *solver, const double *F, double *X, int n_intervals, const double *v_init,
                           int *iterations, double *residual_history, int history_cap);

/* ------------------------------------------------------------ host-only
 * Setup queries that need no GPU (used by the CPU test tier).
 * stmg_plan_levels: the level table of plan_hierarchy/combine_hierarchies
 * (harness.cpp:26-42, hierarchy.cpp:9-97) in the stmg_solver_info layout.
 * stmg_patch_info: Vanka patches of one level: out[0] n_patches, out[1]
 * n_classes, out[2] sum n_T^2, out[3] n_colours, out[4+c] n_T of class c
 * (c < 56), out[60] 1 if the level uses the factored (time-diagonalised)
 * patch inverses, out[61] their padded spatial size, out[62] their
 * multiply-adds per interval (middle blocks + temporal transforms). out must
 * hold 64 entries. If inverse_out is non-NULL, the dense (pseudo-)inverse of
 * class `class_index` (n_T x n_T, row-major) is written there. */
int stmg_plan_levels(int refinements, int r, int k, int n_steps, double t_end, int h_only, int64_t *out);
int stmg_patch_info(int nx, int ny, int r, int k, double tau, double nu, double gamma, int smoother_kind,
                    int64_t *out, double *inverse_out, int class_index);


/* ------------------------------------------------------------ 3D (BASELINE C3 / C5)
 * The reference is 2D only (dof_space.hpp:30); SURVEY.md §9 extends the same
 * interfaces to 3D by tensor product: Q_{r+1}^3 / P_r^disc on the unit cube
 * with a trilinear cell map, DG(k) in time. Layout:
 * BlockVector (block_vector.hpp:13-45) with three velocity components;
 * scalar node (Z*gy + Y)*gx + X, pressure cell ((cz*ny + cy)*nx + cx)*np + m.
 * `vertices` (nullable = Cartesian) is host memory, (nx+1)(ny+1)(nz+1) x 3
 * coordinates, vertex ((vz*(ny+1) + vy)*(nx+1) + vx). Parity is against the
 * oracle's 3D restatement (oracle/src/st3d.cpp); the reference does not pin 3D.
 * Instantiated for r in {1, 2} and k in {0, 1, 2}; cell Vanka only. */
typedef struct stmg3_level stmg3_level;
typedef struct stmg3_solver stmg3_solver;

/* SpaceTimeBlockOperator + VankaSmoother::build (st_operator.hpp:94-165,
 * vanka.cpp:30-194) of a 3D level. smoother_kind: STMG_SMOOTHER_NONE or
 * STMG_SMOOTHER_CELL. */
int stmg3_level_create(stmg_ctx *ctx, int nx, int ny, int nz, int r, int k, double tau, double nu, double gamma,
                       int smoother_kind, const double *vertices, stmg3_level **out);
int stmg3_level_destroy(stmg3_level *level);
/* out[0..11] = n_slots, M^v, M^p, interval size, n_scalar, gx, gy, gz, n_p,
 * max patch size n_T, patch classes, sum of n_T^2 over the patches. */
int stmg3_level_sizes(const stmg3_level *level, int64_t *out);
/* Vanka patch setup of the level: out[0] seconds, out[1] 1 if the exact
 * per-cell inverses were built on the GPU (deformed levels: element matrices,
 * R_T S R_T^T and batched Gauss-Jordan inverses on the device), 2 if they were
 * built there in the time-diagonalised form (DG(2): one real and one
 * complex-pair block per cell), out[2] 1 if the undeformed class inverses
 * stand in (affine_patches), out[3] classes; for the time-diagonalised form
 * out[4] = doubles one sweep streams from HBM per interval group (the real
 * block and the u-columns [P; Q] of the pair block of every patch), out[5] =
 * its multiply-adds per (patch, interval) column summed over the patches;
 * both 0 otherwise. out must hold 6 doubles. */
int stmg3_level_patch_info(const stmg3_level *level, double *out);
/* apply_block / apply_block_raw (st_operator.cpp:397-407) per interval. */
int stmg3_apply_block(stmg3_level *level, const double *x, double *y, int n_intervals, int raw);
/* All-at-once operator y_n = D x_n - Z C x_{n-1} (Eq. GloSys, st_operator.cpp:321-421). */
int stmg3_vmult(stmg3_level *level, const double *x, double *y, int n_intervals, const double *x_prev_slot);
int stmg3_residual(stmg3_level *level, const double *b, const double *x, double *r, int n_intervals,
                   const double *x_prev_slot, int coupled);
/* VankaSmoother::apply_additive / smooth_step (vanka.cpp:196-233), cell patches. */
int stmg3_apply_additive(stmg3_level *level, const double *r, double *out, int n_intervals);
int stmg3_smooth_step(stmg3_level *level, const double *b, double *u, double omega, int n_intervals,
                      const double *x_prev_slot, int coupled, double *work);
int stmg3_vanka_update(stmg3_level *level, const double *r, double *u, double omega, int n_intervals);
/* PressureSpace::project_mean_zero (dof_space.cpp:110-119) per slot, mapped basis. */
int stmg3_project_mean_zero(stmg3_level *level, double *x, int n_intervals);

/* hp-STMG hierarchy for the all-at-once system: p-coarsening k -> k/2 -> ... -> k_min,
 * r -> r/2 -> ... -> 1 (hierarchy.cpp:9-97 extended to k = 0), then n_hcoarse
 * h-steps in space, each also halving the time grid when time_coarsen != 0
 * (PAPER.md Eq. DeftPrRe). The coarsest level is solved exactly by forward
 * substitution in time on the GPU. tau = finest interval length. affine_patches != 0
 * (deformed meshes only): the Vanka patch inverses of the undeformed mesh stand in
 * for the per-cell ones (approximate local solves; the per-cell inverses of C5 are
 * 96 GB and 1.5e13 flop of setup). */
int stmg3_solver_create(stmg_ctx *ctx, int nx, int ny, int nz, int r, int k, double tau, double nu, double gamma,
                        int n_hcoarse, int time_coarsen, int k_min, int affine_patches, const double *vertices, int nu1,
                        int nu2, double omega,
                        double rtol, double atol, int max_iterations, stmg3_solver **out);
int stmg3_solver_destroy(stmg3_solver *solver);
/* Host-only: the level plan of stmg3_solver_create, in stmg3_solver_info's format. */
int stmg3_plan_levels(int nx, int ny, int nz, int r, int k, int n_hcoarse, int time_coarsen, int k_min, int64_t *out);
/* out[0] = n_levels; per level l (coarse first) out[1+7l..]: nx, ny, nz, r, k,
 * time shift (log2 of the time coarsening), interval size. */
int stmg3_solver_info(const stmg3_solver *solver, int64_t *out);
stmg3_level *stmg3_solver_level(stmg3_solver *solver, int l);
int stmg3_solver_set_comm(stmg3_solver *solver, const stmg_comm_ops *ops);
int stmg3_solver_set_krylov(stmg3_solver *solver, int orthogonalization); /* as stmg_solver_set_krylov */
/* TransferPair::restrict_residual / prolongate_correction (transfer.cpp:102-132)
 * between level l and l-1 on nc coarse intervals (2 nc fine ones when the
 * pair coarsens time). */
int stmg3_restrict_residual(stmg3_solver *solver, int l, const double *fine, double *coarse, int nc,
                            int project_pressure);
int stmg3_prolongate_correction(stmg3_solver *solver, int l, const double *coarse, double *fine, int nc,
                                int project_pressure, int accumulate);
/* Exact all-at-once solve on level 0: x_t = CoarseSolve(b_t + C x_{t-1}) (solver.cpp:43-54). */
int stmg3_coarse_forward(stmg3_solver *solver, const double *b, double *x, int n_intervals);
int stmg3_vcycle_all_at_once(stmg3_solver *solver, const double *b, double *x, int n_intervals);
/* FGMRES (solver.cpp:95-202) + all-at-once V-cycle on the slab (see stmg_solve_all_at_once). */
int stmg3_solve_all_at_once(stmg3_solver *solver, const double *F, double *X, int n_intervals, const double *v_init,
                            int *iterations, double *residual_history, int history_cap);

/* ------------------------------------------------------------ C5 hybrid split
 * Spatial partition of the 3D all-at-once solve into z_parts slabs of cells
 * along z (BASELINE C5: 2 spatial x 4 temporal on 8 GPUs; SURVEY.md §8e,
 * PAPER.md:1013-1014 runs the reference's method under MPI). Part p owns the
 * cells cz in [p nz/z_parts, (p+1) nz/z_parts) of every level and stores its
 * own sub-mesh as a complete level: velocity nodes of the interface plane it
 * shares with a neighbour are stored by both parts and kept equal.
 *   - vmult / residual: each part applies its cells, then the parts sum the
 *     interface planes (owner-accumulate; residual r = r_own + r_nb - b);
 *   - Vanka: patches of owned cells; their matrices include the neighbour's
 *     cells across the interface (ghost cell layer, setup only) and interface
 *     weights count the patches of both parts; the interface increments of
 *     both parts are exchanged and added to the pre-sweep values;
 *   - restriction: interface residuals are halved, restricted and the coarse
 *     interface planes summed; prolongation is local;
 *   - per-slot pressure means and Krylov inner products are summed over the
 *     parts (the shared plane counted once);
 *   - the coarsest level gathers its parts and solves globally.
 * Needs deformed-geometry levels (`vertices`, the GLOBAL (nx+1)(ny+1)(nz+1) x 3
 * array) with exact GPU-built patches, nz divisible by z_parts at every level
 * and >= 2 local cells per direction on smoothed levels. Time slabs still go
 * through stmg3_solver_set_comm (the communicator of the ranks holding the
 * same part); the part's neighbours through stmg3_solver_set_space_comm. */
typedef struct stmg_comm_space_ops {
    void *user;
    int part;  /* this rank's z part */
    int parts; /* z parts */
    /* Send the interface plane shared with part-1 (send_lo) and part+1
     * (send_hi), receive theirs (recv_lo / recv_hi); absent sides are NULL.
     * n doubles per plane, stream-ordered on `stream`. */
    int (*exchange_planes)(void *user, const double *send_lo, double *recv_lo, const double *send_hi,
                           double *recv_hi, int64_t n, void *stream);
    int (*allreduce_sum)(void *user, double *buf, int64_t n, void *stream); /* over the parts */
    int (*allgather)(void *user, const double *send, double *recv, int64_t n, void *stream); /* part order */
} stmg_comm_space_ops;
int stmg3_solver_create_split(stmg_ctx *ctx, int nx, int ny, int nz, int r, int k, double tau, double nu, double gamma,
                              int n_hcoarse, int time_coarsen, int k_min, const double *vertices, int z_parts,
                              int z_part, int nu1, int nu2, double omega, double rtol, double atol, int max_iterations,
                              stmg3_solver **out);
int stmg3_solver_set_space_comm(stmg3_solver *solver, const stmg_comm_space_ops *ops);
/* Space ops over an NCCL communicator of the z parts (rank = part). */
int stmg_comm_nccl_space_ops(stmg_comm *comm, stmg_comm_space_ops *ops_out);

#ifdef __cplusplus
}
#endif

#endif /* STMG_B200_H */
