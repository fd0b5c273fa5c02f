// 3D hp-STMG path (BASELINE configs C3 and C5): level description, device
// constants, host setup and kernel launchers.
//
// The reference is 2D only (dof_space.hpp:30); SURVEY.md §9 extends it to 3D
// by tensor product with the trilinear (Q1) cell map of PAPER.md:205-218
// (mapped Q_{r+1}^3 velocity, mapped P_r^disc pressure). The data layout is
// the reference BlockVector (block_vector.hpp:13-45) with three velocity
// components:
//   interval n            : base n * isz, isz = S * (mv + mp)
//   velocity slot a       : a * mv;   component c : + c * nsc, mv = 3 * nsc
//   scalar node (X, Y, Z) : (Z * gy + Y) * gx + X
//   pressure slot a       : S * mv + a * mp; cell (cx, cy, cz), mode m :
//                           ((cz * ny + cy) * nx + cx) * NP + m
// Vertex coordinates (deformed meshes): ((vz * (ny+1) + vy) * (nx+1) + vx) * 3 + d.
#pragma once

#include "kernels.hpp"
#include "setup.hpp"

#include <cstdint>
#include <vector>

namespace stmg_b200
{

constexpr int kMaxNP3 = 35; // dim P_r^disc(3D), r <= 4

/// Device constants of one 3D level (kernel parameter, constant bank).
/// N = r + 2 GLL nodes = Gauss points per direction (st_operator.cpp:167).
struct Level3Consts
{
  int nx, ny, nz, gx, gy, gz, np;
  int zlo, zhi; // constrained z node planes (-1: interface face, Level3Spec::zlo/zhi)
  long long nsc, mv, mp, isz;
  double phi[kMaxN1 * kMaxN1];  // phi(q, i) = l_i(x_q), row-major [q * N + i]
  double dphi[kMaxN1 * kMaxN1]; // l_i'(x_q)
  double w[kMaxN1];             // Gauss weights
  double xq[kMaxN1];            // Gauss points on [-1, 1]
  double leg[kMaxP * kMaxN1];   // Legendre P_a(x_q) [a * N + q]
  int ex[kMaxNP3][3];           // P_r^disc mode exponents (pdisc.cpp:41-55, dim 3)
  double Kt[kMaxS * kMaxS], Mt[kMaxS * kMaxS], lv[kMaxS];
  double nu, gamma, hx, hy, hz;
  const double *verts; // nullptr: Cartesian unit-cube mesh
  const double *gemmE; // Cartesian r = 1: dense element operator (88 x 168), vmult3_gemm_kernel; else nullptr
  // reference-cell 1D node matrices (exact Gauss): M1(i,k) = int phi_i phi_k, K1 = int phi_i' phi_k',
  // C1(i,k) = int phi_i phi_k' (test i, trial derivative k); Legendre moments Lm(a,i) = int L_a phi_i,
  // Lc(a,i) = int L_a phi_i' (Cartesian 1D-factor kernel vmult3c_kernel)
  double m1[kMaxN1 * kMaxN1], k1[kMaxN1 * kMaxN1], c1[kMaxN1 * kMaxN1];
  double lm[kMaxP * kMaxN1], lc[kMaxP * kMaxN1];
};

struct Level3Spec
{
  int nx = 1, ny = 1, nz = 1, r = 1, k = 1;
  double tau = 1.0, nu = 1.0, gamma = 0.0;
  // spatial partition in z (C5 hybrid split, stmg3_solver_create_split):
  // a face is either the domain boundary (Dirichlet, *_bc = 1) or an
  // interface to the neighbouring part (0: its nodes are unconstrained and
  // shared with the neighbour). nz_glob: cells of the whole mesh in z
  // (0: this level is the whole mesh).
  int zlo_bc = 1, zhi_bc = 1, nz_glob = 0;
  bool split() const { return !zlo_bc || !zhi_bc; }
  /// Node plane index of the constrained z faces (-1: interface, none).
  int zlo() const { return zlo_bc ? 0 : -1; }
  int zhi() const { return zhi_bc ? gz() - 1 : -1; }
  double hz() const { return 1.0 / (nz_glob > 0 ? nz_glob : nz); }
  int n1() const { return r + 2; }
  int p() const { return r + 1; }
  int np() const { return (r + 1) * (r + 2) * (r + 3) / 6; }
  int S() const { return k + 1; }
  int gx() const { return nx * p() + 1; }
  int gy() const { return ny * p() + 1; }
  int gz() const { return nz * p() + 1; }
  long long nsc() const { return static_cast<long long>(gx()) * gy() * gz(); }
  long long mv() const { return 3 * nsc(); }
  long long ncells() const { return static_cast<long long>(nx) * ny * nz; }
  long long mp() const { return ncells() * np(); }
  long long isz() const { return S() * (mv() + mp()); }
  long long nverts() const { return static_cast<long long>(nx + 1) * (ny + 1) * (nz + 1); }
};

Level3Consts make_level3_consts(const Level3Spec &L, const double *dev_verts);

/// Cartesian unit-cube vertex coordinates, optionally with the interior
/// vertices displaced by a seeded uniform perturbation of at most
/// `amp` * h per coordinate (BASELINE C5).
std::vector<double> cartesian_vertices(const Level3Spec &L, double amp, unsigned seed);

/// Per-cell dense element matrices (quadrature, trilinear geometry):
/// local velocity dofs [comp][node (k*N + j)*N + i], pressure modes.
struct Cell3Matrices
{
  int nv = 0, np = 0;
  std::vector<double> mass; // nv x nv (scalar)
  std::vector<double> a;    // 3nv x 3nv: nu grad:grad + gamma div div
  std::vector<double> b;    // np x 3nv: int psi_l div u
  std::vector<double> pmean; // np: int psi_l
};
Cell3Matrices cell3_matrices(const Level3Spec &L, const double X8[8][3]);
/// Dense spatial element operator of a Cartesian r = 1 cell for vmult3_gemm_kernel:
/// rows [y_v (3 x 27) ; y_p (4)], columns [UK (81) ; UM (81) ; PM (4)], padded to 88 x 168.
std::vector<double> gemm_element_operator(const Level3Spec &L);
void cell_vertices(const Level3Spec &L, const std::vector<double> &verts, int cx, int cy, int cz, double X8[8][3]);

/// Cell-Vanka patch set of a 3D level: classes (Cartesian: by boundary
/// status per direction, <= 27) or one class per cell (deformed meshes).
struct Patch3Set
{
  std::vector<PatchClass> classes;
  std::vector<int> cell_class; // per cell
  std::uint64_t total_matrix_elements = 0;
  int max_nt = 0;
};
Patch3Set build_patches3(const Level3Spec &L, const std::vector<double> *verts);

/// Dof layout of every cell patch (one class per cell), without matrices:
/// the host half of the GPU patch setup (patch3_gpu.cu). rel / weight are
/// concatenated per cell (rel_off[c] .. rel_off[c] + nt[c]); the inverses go
/// to inv_off[c] (sum of the previous nt^2).
struct Patch3Layout
{
  std::vector<int> nt, nvel;
  std::vector<long long> rel_off, inv_off;
  std::vector<long long> rel;
  std::vector<double> weight;
  std::uint64_t total_matrix_elements = 0;
  int max_nt = 0;
};
Patch3Layout cell_patch_layouts3(const Level3Spec &L);

/// GPU setup of the exact per-cell patch inverses (patch3_gpu.cu): element
/// matrices into E (ncells x elem3_stride(r) doubles), patch matrices and
/// their in-place Gauss-Jordan inverses into Aall. *status (device) stays 0
/// on success; 1 = vanishing pivot, 2 = inverted cell, 3 = layout mismatch.
long long elem3_stride(int r);
/// Split levels: P is the level extended by a ghost cell layer across each
/// interface (ncells_elem element matrices); owned patch c is cell cell0 + c.
cudaError_t launch_patch3_setup(const Level3Consts &P, int r, int S, double *E, double *Aall, const long long *aoff,
                                const int *ntv, int max_nt, long long ncells, int *status, cudaStream_t st,
                                long long ncells_elem = -1, long long cell0 = 0);
/// Time-diagonalised cell patches (DG(k) with a Kronecker patch matrix
/// A_T = K_t (x) M^ + M_t (x) A^): A_T^{-1} = (V (x) I) blockdiag(B_b^{-1})
/// (W (x) I) with M_t^{-1} K_t = V Lambda V^{-1} in real block form, W =
/// V^{-1} M_t^{-1} (setup.cpp temporal_eigen), B_b = alpha M^ + A^ for a
/// real eigenvalue, [[alpha M^ + A^, beta M^], [-beta M^, alpha M^ + A^]]
/// for a pair. Block rows in "factored order": velocity of each coordinate
/// of the block, then pressure of each (all velocity first: pivot-free
/// Gauss-Jordan, the velocity block has a positive definite symmetric part).
struct Fac3Params
{
  int S = 0, nb = 0;
  int c0[kMaxS] = {}, sz[kMaxS] = {};
  double alpha[kMaxS] = {}, beta[kMaxS] = {};
  double V[kMaxS * kMaxS] = {}, W[kMaxS * kMaxS] = {}; // row-major S x S
};
/// Element matrices (as launch_patch3_setup) and the factored blocks of
/// every owned cell patch: matrix 2c + b of Aall (offsets aoff, sizes ntv)
/// is block b of cell c (nb == 2 for DG(2): a real and a pair block).
cudaError_t launch_patch3_fac_setup(const Level3Consts &P, int r, int S, const Fac3Params &F, double *E, double *Aall,
                                    const long long *aoff, const int *ntv, const int *cell_nt, int max_m,
                                    long long ncells, int *status, cudaStream_t st, long long ncells_elem = -1,
                                    long long cell0 = 0);
/// Batched in-place inverse of `count` dense row-major matrices (sizes ntv,
/// offsets aoff), pivot-free blocked Gauss-Jordan on the FP64 tensor path.
cudaError_t launch_gj_inverse(double *Aall, const long long *aoff, const int *ntv, int count, int max_nt, int *status,
                              cudaStream_t st);

/// Transfer between 3D levels: spatial h (1D stencils per direction and
/// pressure child blocks), spatial p (interpolation + modal embedding), none;
/// temporal p (E) and/or temporal h (E_left / E_right, PAPER.md Eq. DeftPrRe).
struct Transfer3Tables
{
  int spatial = 0, pmode = 0, h_time = 0;
  Csr1D px, py, pz, rx, ry, rz;
  std::vector<double> child; // h: 8 blocks (cz*4+cy*2+cx) of np_f x np_c row-major; p: 1 block
  std::vector<double> E;     // [half][a][b], (h_time ? 2 : 1) x S_f x S_c
};
Transfer3Tables build_transfer3(const Level3Spec &coarse, const Level3Spec &fine, bool h_time);

/// Exact all-at-once coarse solve by forward substitution in time,
/// x_t = G b_t + H v_{t-1}: G = P A^+ is the pinned inverse (solver.cpp:10-54)
/// followed by the per-slot mean-zero projection, H = G C with the jump
/// coupling C (isz x mv). Row-major; `verts` may be null (Cartesian).
void coarse3_tables(const Level3Spec &L, const std::vector<double> *verts, std::vector<double> &G,
                    std::vector<double> &H, std::vector<double> &pmean);

/// Pressure mean vector int_K psi_l for every cell (mp doubles) and |Omega|.
std::vector<double> pressure_mean3(const Level3Spec &L, const std::vector<double> *verts, double *volume);

// ---------------------------------------------------------------- device
struct DevGeom3
{
  int nx, ny, nz, gx, gy, gz, S, np;
  int zlo, zhi; // constrained z node planes (-1: interface face)
  long long nsc, mv, mp, isz;
};
DevGeom3 geom3(const Level3Spec &L);

struct DevTransfer3
{
  int spatial, pmode, h_time;
  DevCsr px, py, pz, rx, ry, rz;
  const double *child;
  double E[2 * kMaxS * kMaxS]; // [half][a * kMaxS + b]
  DevGeom3 f, c;
};

/// Additive Vanka sweep (one colour) with the time-diagonalised cell
/// inverses: per block one cell patch x <= 16 intervals; gather R, mix the
/// slots by W, block-diagonal DMMA with the cell's blocks streamed from HBM,
/// mix by V, weights, scatter (red.add; a colour's patches share no dof).
cudaError_t launch_vanka_big_fac(const DevPatchClass *classes, const VankaBatch *batches, int n_batches, int max_nt,
                                 const long long *vel_anchor, const long long *pre_anchor, const Fac3Params &F,
                                 const double *r, double *u, long long isz, int n_intervals, double omega,
                                 cudaStream_t st);
cudaError_t launch_vmult3(int r, int S, const Level3Consts &P, const double *x, const double *b, double *y,
                          int n_intervals, const double *xprev0, int coupled, int mode, cudaStream_t st);
bool vmult3_supported(int r, int S);
/// Kernel launches of one launch_vmult3 (an init and a cell pass per L2-sized interval chunk).
int vmult3_launch_count(const Level3Consts &P, int S, int nI);
cudaError_t launch_zero_constrained3(const DevGeom3 &G, double *x, int n_intervals, cudaStream_t st);
/// p -= (<pmean, p> / vol) on the constant mode, per (interval, slot);
/// deterministic single-block reductions.
cudaError_t launch_project3(const DevGeom3 &G, const double *pmean, double inv_vol, double *x, int n_intervals,
                            cudaStream_t st);
/// z-split interface planes (side 0: Z = 0, side 1: Z = gz - 1), packed
/// [n][a][c][gx * gy] (plane3_doubles). op: 0 pack x -> buf; 1 x += other
/// (owner-accumulate, Dirichlet edge rows skipped); 2 x = x + other - b
/// (residual, b the full vector); 3 x *= 1/2; 4 buf = x - saved;
/// 5 x = saved + (buf + other); 6 x = buf (unpack).
long long plane3_doubles(const DevGeom3 &G, int nI);
cudaError_t launch_plane_op3(const DevGeom3 &G, int side, int op, int nI, double *x, double *buf, const double *other,
                             const double *b, const double *saved, cudaStream_t st);
/// Split mean-zero projection: per (interval, slot) partial sums <pmean, p>
/// (sums[n * S + a]), summed over the parts by the caller, then applied.
cudaError_t launch_project3_sums(const DevGeom3 &G, const double *pmean, const double *x, int nI, double *sums,
                                 cudaStream_t st);
cudaError_t launch_project3_apply(const DevGeom3 &G, const double *sums, double inv_vol, double *x, int nI,
                                  cudaStream_t st);
/// out[i] -= plane part of <w, V_i> (and out[m] -= plane part of <w, w>):
/// the interface plane a part shares with its lower neighbour is counted
/// once in the Krylov inner products. part: plane_multidot_part_doubles().
long long plane_multidot_part_doubles();
cudaError_t launch_plane_multidot_sub(const DevGeom3 &G, int side, int nI, const double *const *V, int m,
                                      bool with_norm, const double *w, double *part, double *out, cudaStream_t st);
/// nc coarse intervals -> (h_time ? 2 nc : nc) fine intervals. With `work`
/// (transfer3_work_doubles) spatial transfers run as separable 1D passes.
long long transfer3_work_doubles(const DevTransfer3 &T, int nc);
cudaError_t launch_prolongate3(const DevTransfer3 &T, const double *coarse, double *fine, int nc, cudaStream_t st,
                               double *work = nullptr);
cudaError_t launch_restrict3(const DevTransfer3 &T, const double *fine, double *coarse, int nc, cudaStream_t st,
                             double *work = nullptr);

} // namespace stmg_b200
