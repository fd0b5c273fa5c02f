// Host-side setup of the B200 hp-STMG path: 1D numerics, per-level operator
// constants, Vanka patch classes with their dense local inverses, transfer
// stencils and the coarse-level inverse. Everything here runs once per
// hierarchy; the per-iteration work is in the .cu kernels.
//
// This is product code: it shares no source with oracle/ (an independent
// implementation -- Legendre root bracketing instead of Golub-Welsch -- so
// the parity tests compare two different derivations of the same tables).
#pragma once

#include "level_consts.cuh"

#include <cstdint>
#include <string>
#include <vector>

namespace stmg_b200
{

// ---------------------------------------------------------------- 1D numerics
struct Rule1D
{
  std::vector<double> x, w;
};
Rule1D gauss_legendre(int n);            // cf. quadrature.cpp:54-66
Rule1D gauss_radau_right(int n);         // cf. quadrature.cpp:68-101 (+1 included)
std::vector<double> gauss_lobatto(int n); // cf. quadrature.cpp:103-134
double legendre(int n, double x);
double legendre_deriv(int n, double x);
double lagrange(const std::vector<double> &nodes, int i, double x);
double lagrange_deriv(const std::vector<double> &nodes, int i, double x);

/// DG(k) temporal matrices on the right-Radau nodal basis (time_basis.cpp:8-59),
/// row-major s x s.
struct TimeTables
{
  int k = 0;
  double tau = 0;
  std::vector<double> Kt, Mt, lv, nodes, weights;
};
TimeTables time_tables(int k, double tau);

/// Real block-diagonalisation of the DG(k) time step, M_t^{-1} K_t =
/// V Lambda V^{-1}: Lambda has 1x1 blocks (real eigenvalue alpha) and 2x2
/// blocks [[alpha, beta], [-beta, alpha]] (pair alpha +- i beta, columns
/// Re v, Im v of V). With it, a space-time patch matrix K_t (x) M_s +
/// M_t (x) A_s factors as (M_t V (x) I) (Lambda (x) M_s + I (x) A_s)
/// (V^{-1} (x) I): the middle is block diagonal in time (Vanka factored form).
struct TemporalEigen
{
  int S = 0;
  std::vector<double> V, W;         // S x S row-major; W = V^{-1} M_t^{-1}
  std::vector<int> blk_c0, blk_sz;  // per block: first coordinate, size (1 or 2)
  std::vector<double> alpha, beta;  // per block (beta = 0 for a real eigenvalue)
  bool ok = false;
};
TemporalEigen temporal_eigen(const TimeTables &T);

/// Reference-cell 1D factors for Q_{r+1} (GLL nodes) / Legendre pressure.
struct Factors1D
{
  int r = 0, n1 = 0, P = 0;
  std::vector<double> nodes;      // GLL nodes
  std::vector<double> M1, K1, C1; // n1 x n1, row-major (i,k)
  std::vector<double> Lm, Lc;     // P x n1, row-major (a,k)
};
Factors1D factors_1d(int r);

/// Geometry/discretisation of one level of the hierarchy.
struct LevelSpec
{
  int nx = 1, ny = 1, r = 1, k = 1;
  double hx = 1.0, hy = 1.0, tau = 1.0, nu = 1.0, gamma = 0.0;
  int n1() const { return r + 2; }
  int p() const { return r + 1; }
  int np() const { return (r + 1) * (r + 2) / 2; }
  int S() const { return k + 1; }
  int gx() const { return nx * p() + 1; }
  int gy() const { return ny * p() + 1; }
  long long nsc() const { return static_cast<long long>(gx()) * gy(); }
  long long mv() const { return 2 * nsc(); }
  long long mp() const { return static_cast<long long>(nx) * ny * np(); }
  long long isz() const { return S() * (mv() + mp()); }
};

LevelConsts make_level_consts(const LevelSpec &L);

/// Dense element matrices of one cell, local dofs ordered
/// [comp 0 nodes (iy*n1+ix), comp 1 nodes, pressure modes].
struct CellMatrices
{
  int nv = 0, np = 0;
  std::vector<double> mass, lap; // nv x nv
  std::vector<double> gd;        // 2nv x 2nv
  std::vector<double> div;       // np x 2nv
};
CellMatrices cell_matrices(const LevelSpec &L);

// ---------------------------------------------------------------- Vanka
enum class PatchKind
{
  cell = 0,
  vertex_star = 1,
};

/// One class of congruent Vanka patches: identical dof pattern relative to
/// the patch anchor and therefore identical local matrix R_T S R_T^T
/// (vanka.cpp:92-176). Cartesian levels have at most 16 (cell) or 25
/// (vertex-star) classes, so inverses are stored per class, not per patch.
struct PatchClass
{
  int n_t = 0;
  int n_vel = 0;                      // first n_vel dofs are velocity
  std::vector<long long> rel;         // offset from the velocity / pressure anchor
  std::vector<double> weight;         // 1/valence (vanka.cpp:182-192)
  std::vector<double> inverse;        // n_t x n_t row-major (pseudo-inverse if singular)
  bool singular = false;
  // spatial factors of the patch matrix (k = 0 copy of the patch: velocity
  // mass M_s and Stokes block A_s on the n_s spatial dofs, n_vs velocity)
  int n_s = 0, n_vs = 0;
  std::vector<double> Ms, As;
  // factored inverse (fac_ok): the middle block inverses of TemporalEigen,
  // (S * n_sp) rows x (2 * n_sp) block-local columns, row = coord * n_sp + j
  bool fac_ok = false;
  std::vector<double> fac_inv;
};

struct PatchSet
{
  PatchKind kind = PatchKind::cell;
  std::vector<PatchClass> classes;
  /// Patches grouped by colour (no two patches of one colour share a dof),
  /// then by class: entries (class, ax, ay) with the anchor cell/vertex.
  struct Entry
  {
    int cls, ax, ay;
  };
  std::vector<std::vector<Entry>> colours;
  std::uint64_t total_matrix_elements = 0; // sum n_T^2 over all patches
  // factored form (all classes non-singular, k >= 2): padded spatial size
  bool factored = false;
  int n_sp = 0;
  TemporalEigen eig;
  std::uint64_t factored_matrix_elements = 0; // sum over patches of the middle-block MACs
};
PatchSet build_patches(const LevelSpec &L, PatchKind kind);

/// Velocity / pressure anchors of a patch in one interval.
inline long long
patch_vel_anchor(const LevelSpec &L, PatchKind kind, int ax, int ay)
{
  const int ox = kind == PatchKind::cell ? ax : ax - 1;
  const int oy = kind == PatchKind::cell ? ay : ay - 1;
  return static_cast<long long>(oy) * L.p() * L.gx() + static_cast<long long>(ox) * L.p();
}
inline long long
patch_pre_anchor(const LevelSpec &L, PatchKind kind, int ax, int ay)
{
  const int ox = kind == PatchKind::cell ? ax : ax - 1;
  const int oy = kind == PatchKind::cell ? ay : ay - 1;
  return L.S() * L.mv() + (static_cast<long long>(oy) * L.nx + ox) * L.np();
}

// ---------------------------------------------------------------- transfers
enum class TransferKind
{
  identity = 0,
  h_space = 1,
  p_space = 2,
  p_time = 3,
  h_space_p_time = 4,
  p_space_p_time = 5,
};

/// 1D interpolation stencil in CSR form (rows = output grid points).
struct Csr1D
{
  int rows = 0, cols = 0;
  std::vector<int> ptr, col;
  std::vector<double> val;
};

struct TransferTables
{
  TransferKind kind = TransferKind::identity;
  bool spatial = false, temporal = false;
  Csr1D px, py;   // prolongation, fine grid x coarse grid (per direction)
  Csr1D rx, ry;   // restriction = transposes
  int pmode = 0;  // 0 none, 1 h (child blocks), 2 p (embedding)
  std::vector<double> child; // h: 4 blocks (cy*2+cx) of np_f x np_c, row-major
  std::vector<int> embed;    // p: coarse mode l -> fine mode
  std::vector<double> e_time; // (k_f+1) x (k_c+1) row-major
};
TransferTables build_transfer(const LevelSpec &coarse, const LevelSpec &fine, TransferKind kind);
Csr1D transpose_csr(const Csr1D &a);
/// 1D interpolation from the coarse Q_{rc+1} grid to the fine grid points
/// (h_step: fine cells are the halves of the coarse cells).
Csr1D interp_1d(int nc_cells, int rc, int nf_cells, int rf, bool h_step);

// ---------------------------------------------------------------- coarse level
/// Dense constrained operator of a (small) level with the first pressure dof
/// of every slot pinned (solver.cpp:10-41), inverted. Row-major.
std::vector<double> coarse_inverse(const LevelSpec &L, std::vector<long long> &pinned);

/// Quadrature and basis tables of the built-in problem kernels (problems.cu).
ProblemTables problem_tables(const LevelSpec &L);

// ---------------------------------------------------------------- hierarchy
struct HierarchyConfig
{
  int refinements = 2;  // finest mesh 2^c x 2^c cells
  int r = 2, k = -1;    // k < 0: k = r
  int n_steps = 0;      // 0: tau = 2^-(c+1) * t_end
  double t_end = 1.0;
  double nu = 0.1, gamma = 1.0;
  int h_only = 0;
  PatchKind smoother = PatchKind::cell;
};
struct LevelPlan
{
  LevelSpec spec;
  TransferKind kind_to_coarser = TransferKind::identity;
};
/// plan_hierarchy + combine_hierarchies (harness.cpp:26-42,
/// hierarchy.cpp:9-97), coarse first.
std::vector<LevelPlan> plan_levels(const HierarchyConfig &cfg, int *n_steps_out);

// ---------------------------------------------------------------- dense helpers
/// In-place inverse via LU with partial pivoting; returns false if singular.
bool invert_dense(std::vector<double> &a, int n, double *rcond_out);
/// Moore-Penrose pseudo-inverse (one-sided Jacobi SVD).
std::vector<double> pseudo_inverse(const std::vector<double> &a, int n, int *rank_out);

} // namespace stmg_b200
