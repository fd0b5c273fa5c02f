// Device-side data views and kernel launchers of the B200 hp-STMG path.
#pragma once

#include "level_consts.cuh"

#include <algorithm>
#include <cuda_runtime.h>

namespace stmg_b200
{

/// Geometry of one level as the auxiliary kernels see it.
struct DevGeom
{
  int nx, ny, gx, gy, S, np;
  long long nsc, mv, mp, isz;
  double hx, hy;
};

struct DevCsr
{
  const int *ptr;
  const int *col;
  const double *val;
};

/// One TransferPair on the device (transfer.hpp:33-96).
struct DevTransfer
{
  int spatial, temporal, pmode, zero_constrained;
  DevCsr px, py, rx, ry;
  const double *child; // pmode 1: 4 blocks np x np
  const int *embed;    // pmode 2
  double E[kMaxS * kMaxS]; // E[a*kMaxS+b], fine slot a, coarse slot b
  DevGeom f, c;
};

/// Device view of one Vanka patch class (setup.hpp PatchClass).
struct DevPatchClass
{
  int n_t, n_vel;
  const long long *rel;  // n_t offsets from the velocity / pressure anchor
  const double *weight;  // n_t valence weights
  const double *inverse; // n_t x n_t row-major
  // factored form (vanka_fac_kernel): spatial dofs n_s (n_vs velocity) and
  // the middle-block inverses, (S * n_sp) x (2 * n_sp) block-local columns
  int n_s, n_vs;
  const double *fac_inv;
};

/// Time-diagonalised Vanka (setup.hpp TemporalEigen): per level.
struct FacParams
{
  int S, nsp;
  double V[kMaxS * kMaxS], W[kMaxS * kMaxS]; // row-major
  int kbase[16], ksteps[16];                 // per warp (8-row tile): K range of its block
};

/// One Vanka block's work item: a run of same-class patches of one colour.
struct VankaBatch
{
  int cls;   // class index
  int first; // index into the anchor arrays
  int count; // <= vanka_cols_per_batch()
};

/// One tile of the pipelined tensor-core Vanka: <= 32 columns (patch,
/// interval) of one class; column data in parallel arrays at tile*32 + c.
/// <= 32 columns (patch, interval) of one class: column j is entry c0 + j
/// of the patch-major / interval-minor enumeration of the item whose patches
/// start at pfirst in the velocity / pressure anchor arrays (ncols == 0:
/// stage padding).
struct VankaTile
{
  int cls;
  int ncols;
  int pfirst;
  int c0;
  int phase; // colour sub-phase within the block (same-phase tiles share no dof)
};
cudaError_t launch_vanka_tc(const DevPatchClass *classes, const VankaTile *tiles, const long long *va,
                            const long long *pa, const int *tile_ptr, int n_blocks, int ng_full,
                            int max_nt, const double *r, double *u, long long isz, int n_intervals, double omega,
                            cudaStream_t stream);
cudaError_t launch_vanka_fac(const DevPatchClass *classes, const VankaTile *tiles, const long long *va,
                             const long long *pa, const int *tile_ptr, int n_blocks, int ng_full, const FacParams &F,
                             const double *r, double *u, long long isz, int n_intervals, double omega,
                             cudaStream_t stream);
/// Deferred-scatter DMMA sweep of one colour for 128 < n_T <= 176 (3D Q2 cells), batches of one class.
cudaError_t launch_vanka_dfr176(const DevPatchClass *classes, const VankaBatch *batches, int n_batches, int max_nt,
                                const long long *vel_anchor, const long long *pre_anchor, const double *r, double *u,
                                long long isz, int n_intervals, double omega, int group, cudaStream_t stream);
int vanka_tc_cols();
int vanka_tc_max_tiles();
bool vanka_fac_supported(int S, int nsp); // instantiated (S, n_sp) shapes of vanka_fac_kernel

cudaError_t launch_vmult(int r, int S, const LevelConsts &P, const double *x, const double *b, double *y,
                         int n_intervals, const double *xprev0, int coupled, int mode, cudaStream_t stream);
/// One Vanka launch. item_ptr == nullptr: block b runs item b (one colour
/// batch); otherwise block b runs items [item_ptr[b], item_ptr[b+1]) in
/// order (super-cell sub-phases). The non-DMMA fallback (n_T > 128) requires
/// item_ptr == nullptr.
cudaError_t launch_vanka_colour(const DevPatchClass *classes, const VankaBatch *batches, const int *item_ptr,
                                int n_batches, int max_nt, const long long *vel_anchor, const long long *pre_anchor,
                                const double *r, double *u, long long isz, int n_intervals, double omega,
                                cudaStream_t stream);
int vanka_cols_per_batch();
/// Intervals per block of the DMMA / big-patch item kernels (0 = the size
/// heuristic); the tuning hook behind stmg_set_tuning.
void set_vanka_group_override(int dmma_group, int big_group);
/// Multiprocessor count of the current device (cached per device).
int device_sm_count();
cudaError_t launch_prolongate(const DevTransfer &T, const double *coarse, double *fine, int n_intervals,
                              int accumulate, cudaStream_t st);
cudaError_t launch_restrict(const DevTransfer &T, const double *fine, double *coarse, int n_intervals,
                            cudaStream_t st);
/// Per-slot mean-zero projection of the pressure (two deterministic passes);
/// `scratch` holds project_scratch_doubles(G, n_intervals) doubles.
int project_scratch_doubles(const DevGeom &G, int n_intervals);
cudaError_t launch_project_mean_zero(const DevGeom &G, double *x, int n_intervals, double *scratch, cudaStream_t st);
cudaError_t launch_zero_constrained(const DevGeom &G, double *x, int n_intervals, cudaStream_t st);
cudaError_t launch_coarse_solve(const double *inv, const long long *pinned, int n_pinned, int nrows, const double *b,
                                double *x, cudaStream_t st);
// All-at-once coarse solve by block forward substitution in time:
// x_t = G b_t + H v_{t-1}, v_{t-1} = slot-k velocity of x_{t-1}, v_{-1} = 0.
// B holds n_all intervals; intervals [n_begin, n_begin + n_own) go to X.
cudaError_t launch_coarse_forward(const double *G, const double *H, int n, int mv, long long v_off, const double *B,
                                  int n_all, int n_begin, int n_own, double *X, cudaStream_t st);
// Built-in problems (problems.cu): manufactured force load vector and error norms.
cudaError_t launch_assemble_manufactured(const DevGeom &G, int r, const ProblemTables &T, double nu, double t_start,
                                         double tau, double *F, int n_intervals, cudaStream_t st);
long long errors_partials(const DevGeom &G, int n_intervals);
cudaError_t launch_lift_cavity(const DevGeom &G, int r, const ProblemTables &T, double t_start, double tau,
                               double *L, int n_intervals, cudaStream_t st);
cudaError_t launch_interpolate_manufactured(const DevGeom &G, int r, const ProblemTables &T, double t_start,
                                            double tau, double *X, int n_intervals, cudaStream_t st);
cudaError_t launch_errors_manufactured(const DevGeom &G, int r, const ProblemTables &T, double t_start, double tau,
                                       const double *X, int n_intervals, double *part, double *out, cudaStream_t st);
/// Saddle-point health sums per (interval, slot) of y = [M v ; B v]: 4 doubles each.
cudaError_t launch_health(const DevGeom &G, double cell_area, const double *X, const double *Y, double *out,
                          int n_intervals, cudaStream_t st);
int dot_partials();
/// Batched Krylov kernels (classical Gram-Schmidt, final update): up to
/// kMultiMax basis vectors per pass, chunked beyond.
constexpr int kMultiMax = 16;
struct MultiVec
{
  const double *p[kMultiMax];
};
struct MultiCoef
{
  double c[kMultiMax];
};
/// out[i] = <w, V_i> for i < m; out[m] = <w, w> when with_norm. `part`
/// holds (kMultiMax + 1) * dot_partials() doubles. Deterministic.
cudaError_t launch_multidot(const double *const *V, int m, bool with_norm, const double *w, long long n, double *part,
                            double *out, cudaStream_t st);
/// w += sign * sum_i c_i V_i with c on the device (c_dev) or host (c_host).
cudaError_t launch_multi_axpy(const double *const *V, int m, const double *c_dev, const double *c_host, double sign,
                              double *w, long long n, cudaStream_t st);
cudaError_t launch_dot(const double *x, const double *y, long long n, double *part, double *out, cudaStream_t st);
/// y += a x with a = alpha_dev ? sign * (*alpha_dev) : alpha (sign applies to
/// the device-resident coefficient only).
cudaError_t launch_axpy(long long n, double alpha, const double *alpha_dev, double sign, const double *x, double *y,
                        cudaStream_t st);
cudaError_t launch_scale(long long n, double alpha, double *y, cudaStream_t st);
cudaError_t launch_xpby(long long n, const double *x, double beta, double *y, cudaStream_t st);

} // namespace stmg_b200
