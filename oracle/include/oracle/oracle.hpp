// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference hp space-time multigrid path
// (/root/reference/proj, C++20 + Eigen3). The reference cannot be built in
// this image (Eigen3 and the vendored doctest/CLI11 are absent, see
// DESIGN.md "Oracle"), so this file restates its algorithms without Eigen,
// module by module, citing the reference file:line each piece follows.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference leg may load this code, and only as the checker or the
// CPU baseline. The product (paper_2502_09159_b200/) never links it.
//
// Pinning: the restatement is checked against every known-answer test of
// the reference suites that touches this path (oracle/tests/oracle_tests.cpp
// ports them with the reference's own tolerances, including the Table-1
// error values of tests/acceptance.cpp:394-420).
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

namespace oracle
{

using Vec = std::vector<double>;
using Index = std::int64_t;

// ---------------------------------------------------------------- dense LA
/// Column-major dense matrix (same storage order as Eigen::MatrixXd, which
/// the reference's local cell kernels rely on: local index iy*n1+ix is the
/// column-major linear index of an (n1 x n1) matrix with x the row).
struct Mat
{
  int r = 0, c = 0;
  Vec d;
  Mat() = default;
  Mat(int rows, int cols) : r(rows), c(cols), d(static_cast<size_t>(rows) * cols, 0.0) {}
  double &operator()(int i, int j) { return d[static_cast<size_t>(j) * r + i]; }
  double operator()(int i, int j) const { return d[static_cast<size_t>(j) * r + i]; }
  double *data() { return d.data(); }
  const double *data() const { return d.data(); }
  void setZero() { std::fill(d.begin(), d.end(), 0.0); }
};

Mat matmul(const Mat &a, const Mat &b);
Mat transpose(const Mat &a);

/// LU with partial pivoting (stands in for Eigen::PartialPivLU,
/// vanka.cpp:167, and FullPivLU/SparseLU at the call sites that only need a
/// direct solve: time_basis.cpp:70, solver.cpp:38).
struct LU
{
  int n = 0;
  Mat lu;
  std::vector<int> piv;
  bool singular = false;
  LU() = default;
  explicit LU(const Mat &a);
  void solve_inplace(double *x) const;
  Vec solve(const Vec &b) const;
  /// Reciprocal 1-norm condition number, computed exactly from the inverse
  /// (Eigen's rcond() estimates the same quantity; used only against the
  /// 1e-12 degeneracy threshold of vanka.cpp:168).
  double rcond(const Mat &a) const;
  Mat inverse() const;
};

/// Minimum-norm solver for rank-deficient square systems (stands in for
/// Eigen::CompleteOrthogonalDecomposition, vanka.cpp:172-174). Implemented
/// as a pseudo-inverse from a one-sided Jacobi SVD with Eigen's default rank
/// threshold eps * n relative to the largest singular value.
struct MinNormSolver
{
  int n = 0;
  int rank = 0;
  Mat pinv;
  MinNormSolver() = default;
  explicit MinNormSolver(const Mat &a);
  Vec solve(const Vec &b) const;
};

/// Eigen-decomposition of a symmetric tridiagonal matrix: ascending
/// eigenvalues and the first component of each unit eigenvector
/// (Golub-Welsch needs only those; quadrature.cpp:19-39).
void tridiag_eigen(const Vec &diag, const Vec &offdiag, Vec &evals, Vec &first_comp);

// ---------------------------------------------------------------- 1D numerics
struct QuadratureRule
{
  Vec points, weights;
  int size() const { return static_cast<int>(points.size()); }
};
QuadratureRule gauss_rule(int n);        // quadrature.cpp:54-66
QuadratureRule gauss_radau_right(int n); // quadrature.cpp:68-101
Vec gauss_lobatto_points(int n);         // quadrature.cpp:103-134

class NodalBasis1D // basis1d.cpp:8-81
{
public:
  explicit NodalBasis1D(Vec nodes);
  int size() const { return static_cast<int>(nodes_.size()); }
  const Vec &nodes() const { return nodes_; }
  double value(int i, double x) const;
  double derivative(int i, double x) const;
  Vec values(double x) const;
  Vec derivatives(double x) const;
  Mat value_table(const Vec &pts) const;
  Mat derivative_table(const Vec &pts) const;

private:
  Vec nodes_;
};

Vec legendre_values(int n, double x);      // pdisc.cpp:8-17
Vec legendre_derivatives(int n, double x); // pdisc.cpp:19-30

class PDiscBasis // pdisc.cpp:32-98
{
public:
  PDiscBasis(int r, int dim);
  int degree() const { return r_; }
  int size() const { return static_cast<int>(exps_.size()); }
  const std::array<int, 3> &exponents(int l) const { return exps_[l]; }
  double value(int l, const double *xi) const;
  void gradient(int l, const double *xi, double *g) const;
  double gram_diagonal(int l) const;

private:
  int r_, dim_;
  std::vector<std::array<int, 3>> exps_;
};

struct TemporalMatrices // time_basis.hpp:17-35, time_basis.cpp:8-59
{
  int k = 0;
  double tau = 0;
  Mat dt_plus_jump, mass, coupling;
  Vec nodes, weights, left_values;
  int n_dofs() const { return k + 1; }
};
TemporalMatrices temporal_matrices(int k, double tau);
double dg_ode_step(int k, double tau, double lambda, double y_prev); // time_basis.cpp:61-75

// ---------------------------------------------------------------- mesh / spaces
struct Box
{
  double x0, y0, x1, y1;
  double width() const { return x1 - x0; }
  double height() const { return y1 - y0; }
  double volume() const { return width() * height(); }
};

class Mesh // mesh.hpp:30-88, mesh.cpp
{
public:
  static Mesh build_cartesian(const Box &domain, int base_nx, int base_ny, int levels);
  int n_levels() const { return levels_; }
  int finest_level() const { return levels_ - 1; }
  const Box &domain() const { return domain_; }
  int cells_x(int l) const { return base_nx_ << l; }
  int cells_y(int l) const { return base_ny_ << l; }
  int n_cells(int l) const { return cells_x(l) * cells_y(l); }
  int n_vertices(int l) const { return (cells_x(l) + 1) * (cells_y(l) + 1); }
  double hx(int l) const { return domain_.width() / cells_x(l); }
  double hy(int l) const { return domain_.height() / cells_y(l); }
  int cell_index(int l, int ix, int iy) const { return iy * cells_x(l) + ix; }
  std::array<int, 2> cell_coords(int l, int cell) const { return {cell % cells_x(l), cell / cells_x(l)}; }
  Box cell_box(int l, int cell) const;
  int vertex_index(int l, int ix, int iy) const { return iy * (cells_x(l) + 1) + ix; }
  std::array<int, 2> vertex_coords(int l, int v) const { return {v % (cells_x(l) + 1), v / (cells_x(l) + 1)}; }
  std::array<int, 4> children(int l, int cell) const;
  int parent(int l, int cell) const;
  std::vector<int> cells_of_vertex(int l, int v) const;
  std::vector<int> vertex_neighbors(int l, int cell) const;

private:
  Mesh(const Box &d, int bx, int by, int lv) : domain_(d), base_nx_(bx), base_ny_(by), levels_(lv) {}
  void check_level(int l) const;
  Box domain_;
  int base_nx_, base_ny_, levels_;
};

class VelocitySpace // dof_space.cpp:10-81
{
public:
  VelocitySpace(const Mesh &mesh, int level, int r);
  int level() const { return level_; }
  int r() const { return r_; }
  int nodes_per_dir() const { return r_ + 2; }
  int n_scalar_dofs() const { return n_scalar_; }
  Index n_dofs() const { return 2 * static_cast<Index>(n_scalar_); }
  int grid_x() const { return grid_x_; }
  int grid_y() const { return grid_y_; }
  const Mesh &mesh() const { return *mesh_; }
  const NodalBasis1D &basis_1d() const { return basis_; }
  const std::vector<int> &cell_scalar_dofs(int cell) const { return cell_dofs_[cell]; }
  Index global_dof(int comp, int s) const { return static_cast<Index>(comp) * n_scalar_ + s; }
  double node_x(int s) const { return coord_x_[s % grid_x_]; }
  double node_y(int s) const { return coord_y_[s / grid_x_]; }
  bool scalar_on_boundary(int s) const { return boundary_[s] != 0; }
  const std::vector<int> &boundary_scalar_dofs() const { return boundary_list_; }
  void zero_constrained(double *v) const;
  void set_boundary_values(double *v, const std::function<double(double, double, double, int)> &g, double t) const;

private:
  const Mesh *mesh_;
  int level_, r_, grid_x_, grid_y_, n_scalar_;
  NodalBasis1D basis_;
  std::vector<std::vector<int>> cell_dofs_;
  Vec coord_x_, coord_y_;
  std::vector<char> boundary_;
  std::vector<int> boundary_list_;
};

class PressureSpace // dof_space.cpp:83-119
{
public:
  PressureSpace(const Mesh &mesh, int level, int r);
  int level() const { return level_; }
  int r() const { return r_; }
  int dofs_per_cell() const { return basis_.size(); }
  Index n_dofs() const { return n_dofs_; }
  const Mesh &mesh() const { return *mesh_; }
  const PDiscBasis &basis() const { return basis_; }
  Index cell_dof(int cell, int l) const { return static_cast<Index>(cell) * basis_.size() + l; }
  const Vec &mass_diagonal() const { return mass_diag_; }
  const Vec &one_coefficients() const { return one_; }
  const Vec &mean_vector() const { return mean_; }
  double domain_volume() const { return volume_; }
  void project_mean_zero(double *p) const;
  double mean_integral(const double *p) const;

private:
  const Mesh *mesh_;
  int level_, r_;
  Index n_dofs_;
  PDiscBasis basis_;
  Vec mass_diag_, one_, mean_;
  double volume_;
};

/// block_vector.hpp:13-87: (V^1..V^s, P^1..P^s), one contiguous vector.
struct BlockVector
{
  int ns = 0;
  Index nv = 0, np = 0;
  Vec data;
  BlockVector() = default;
  BlockVector(int s, Index v, Index p) : ns(s), nv(v), np(p), data(static_cast<size_t>(s) * (v + p), 0.0) {}
  Index size() const { return static_cast<Index>(data.size()); }
  double *velocity(int a) { return data.data() + a * nv; }
  const double *velocity(int a) const { return data.data() + a * nv; }
  double *pressure(int a) { return data.data() + ns * nv + a * np; }
  const double *pressure(int a) const { return data.data() + ns * nv + a * np; }
  void setZero() { std::fill(data.begin(), data.end(), 0.0); }
  double norm() const;
  double dot(const BlockVector &o) const;
  bool same_shape(const BlockVector &o) const { return ns == o.ns && nv == o.nv && np == o.np; }
  BlockVector &operator+=(const BlockVector &o);
  BlockVector &operator-=(const BlockVector &o);
  BlockVector &operator*=(double s);
};
void require_same_shape(const BlockVector &a, const BlockVector &b, const char *where);

// ---------------------------------------------------------------- operator
using ForceFn = std::function<double(double, double, double, int)>;

class CellKernels // st_operator.cpp:11-98
{
public:
  CellKernels(const VelocitySpace &vs, const PressureSpace &ps, int nq);
  int n_nodes_1d() const { return n1_; }
  int n_q_1d() const { return nq_; }
  int n_pressure() const { return np_; }
  double jdet() const { return jdet_; }
  void mass_local(const Mat &u, Mat &out) const;
  void laplace_local(const Mat &u, Mat &out) const;
  void div_local(const Mat &ux, const Mat &uy, double *p_out) const;
  void div_transpose_local(const double *p, Mat &ux_out, Mat &uy_out) const;
  void grad_div_local(const Mat &ux, const Mat &uy, Mat &ux_out, Mat &uy_out) const;
  const Mat &phi() const { return phi_; }
  const Mat &dphi() const { return dphi_; }
  const Mat &psi() const { return psi_; }
  const Vec &qpoints() const { return qp_; }
  const Vec &qweights() const { return qw_; }
  double dxi_dx() const { return 2.0 / hx_; }
  double deta_dy() const { return 2.0 / hy_; }

private:
  int n1_, nq_, np_;
  double hx_, hy_, jdet_;
  Mat phi_, dphi_, psi_, w2d_;
  Vec qp_, qw_;
};

struct ElementMatrices // st_operator.hpp:77-83
{
  Mat mass, laplace, div, grad_div;
};
ElementMatrices extract_element_matrices(const CellKernels &k); // st_operator.cpp:100-155

/// Triplet-assembled sparse matrix (CSR after assembly; duplicates summed
/// like Eigen::SparseMatrix::setFromTriplets).
struct SparseMatrix
{
  Index rows = 0, cols = 0;
  std::vector<Index> rowptr;
  std::vector<Index> col;
  Vec val;
  static SparseMatrix from_triplets(Index rows, Index cols, std::vector<std::tuple<Index, Index, double>> &trips);
  void multiply(const double *x, double *y) const; // y = A x
  void multiply_transpose(const double *x, double *y) const; // y = A^T x
  Mat to_dense() const;
};

class SpaceTimeBlockOperator // st_operator.hpp:94-165
{
public:
  SpaceTimeBlockOperator(const VelocitySpace &vs, const PressureSpace &ps, const TemporalMatrices &tm,
                         double nu, double grad_div = 0.0);
  const VelocitySpace &velocity_space() const { return *vs_; }
  const PressureSpace &pressure_space() const { return *ps_; }
  const TemporalMatrices &temporal() const { return *tm_; }
  double viscosity() const { return nu_; }
  double grad_div_coefficient() const { return gd_; }
  int n_slots() const { return tm_->n_dofs(); }
  BlockVector make_vector() const { return BlockVector(n_slots(), vs_->n_dofs(), ps_->n_dofs()); }
  void apply_velocity_mass(const double *v, double *y) const;
  void apply_laplace(const double *v, double *y) const;
  void apply_div(const double *v, double *p) const;
  void apply_div_transpose(const double *p, double *v) const;
  void apply_pressure_mass(const double *p, double *y) const;
  void apply_grad_div(const double *v, double *y) const;
  void apply_block(const BlockVector &x, BlockVector &y) const;
  void apply_block_raw(const BlockVector &x, BlockVector &y) const;
  BlockVector coupling_rhs(const double *v_prev) const;
  BlockVector assemble_rhs(const ForceFn &f, double t_start) const;
  SparseMatrix assemble_sparse_oracle() const;
  const ElementMatrices &element_matrices() const { return elem_; }
  const CellKernels &kernels() const { return kernels_; }

private:
  void apply_block_impl(const BlockVector &x, BlockVector &y, bool constrain) const;
  const VelocitySpace *vs_;
  const PressureSpace *ps_;
  const TemporalMatrices *tm_;
  double nu_, gd_;
  CellKernels kernels_;
  ElementMatrices elem_;
};

// ---------------------------------------------------------------- smoother
enum class SmootherKind
{
  cell = 0,
  vertex_star = 1,
};

struct PatchFactorization // vanka.hpp:24-39
{
  std::vector<Index> dofs;
  LU lu;
  std::unique_ptr<MinNormSolver> cod;
  Vec weights;
  bool factored = false;
  int size() const { return static_cast<int>(dofs.size()); }
  Vec solve(const Vec &rhs) const { return cod ? cod->solve(rhs) : lu.solve(rhs); }
};

class VankaSmoother // vanka.hpp:45-89, vanka.cpp
{
public:
  static VankaSmoother build(const SpaceTimeBlockOperator &op, SmootherKind kind, bool factor = true);
  /// R_T S R_T^T of patch ip (vanka.cpp:92-165) and its factorization
  /// (vanka.cpp:167-176), for smoothers built with factor == false.
  Mat local_matrix(const SpaceTimeBlockOperator &op, size_t ip) const;
  Mat factor_patch(const SpaceTimeBlockOperator &op, size_t ip); // returns R_T S R_T^T
  SmootherKind kind() const { return kind_; }
  const std::vector<PatchFactorization> &patches() const { return patches_; }
  void apply_additive(const BlockVector &residual, BlockVector &out) const;
  void smooth_step(const SpaceTimeBlockOperator &op, const BlockVector &b, BlockVector &u, double omega) const;
  std::uint64_t total_matrix_elements() const;
  static std::uint64_t nominal_block_size(int k, int r, int d);
  std::uint64_t mult_adds() const { return mult_adds_; }
  void reset_mult_adds() const { mult_adds_ = 0; }
  /// The assembled local matrices (kept for tests).
  std::vector<Mat> local_matrices;

private:
  SmootherKind kind_ = SmootherKind::cell;
  std::vector<PatchFactorization> patches_;
  mutable std::uint64_t mult_adds_ = 0;
};

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
std::string to_string(TransferKind k);

class TransferPair // transfer.hpp:33-96
{
public:
  TransferKind kind() const { return kind_; }
  BlockVector prolongate(const BlockVector &coarse) const;
  BlockVector restrict_(const BlockVector &fine) const;
  BlockVector prolongate_correction(const BlockVector &coarse, bool project_pressure) const;
  BlockVector restrict_residual(const BlockVector &fine, bool project_pressure) const;
  const SparseMatrix &velocity_matrix() const { return p_vel_; }
  const SparseMatrix &pressure_matrix() const { return p_pre_; }
  bool has_spatial() const { return has_spatial_; }
  bool has_temporal() const { return has_temporal_; }
  const Mat &temporal_matrix() const { return e_time_; }
  static TransferPair identity(const VelocitySpace &vs, const PressureSpace &ps, int k);

  friend TransferPair build_h_space_transfer(const VelocitySpace &, const PressureSpace &, const VelocitySpace &,
                                             const PressureSpace &, int);
  friend TransferPair build_p_space_transfer(const VelocitySpace &, const PressureSpace &, const VelocitySpace &,
                                             const PressureSpace &, int);
  friend TransferPair build_p_time_transfer(int, int, const VelocitySpace &, const PressureSpace &);
  friend TransferPair combine_space_time_transfer(TransferPair, TransferPair);

private:
  TransferKind kind_ = TransferKind::identity;
  bool has_spatial_ = false, has_temporal_ = false;
  SparseMatrix p_vel_, p_pre_;
  Mat e_time_;
  int k_coarse_ = 0, k_fine_ = 0;
  const VelocitySpace *vc_ = nullptr, *vf_ = nullptr;
  const PressureSpace *pc_ = nullptr, *pf_ = nullptr;
};
TransferPair build_h_space_transfer(const VelocitySpace &vc, const PressureSpace &pc, const VelocitySpace &vf,
                                    const PressureSpace &pf, int k);
TransferPair build_p_space_transfer(const VelocitySpace &vc, const PressureSpace &pc, const VelocitySpace &vf,
                                    const PressureSpace &pf, int k);
TransferPair build_p_time_transfer(int k_coarse, int k_fine, const VelocitySpace &vs, const PressureSpace &ps);
TransferPair combine_space_time_transfer(TransferPair spatial, TransferPair temporal);

// ---------------------------------------------------------------- hierarchy
struct HpEntry
{
  double h;
  int p;
  bool operator==(const HpEntry &o) const { return h == o.h && p == o.p; }
};
std::vector<HpEntry> construct_hierarchy(double h_fine, double h_coarse, int p_fine, int p_coarse);

struct LevelDescriptor
{
  int index, mesh_coarsening, time_coarsening, r, k;
  double h, tau;
  TransferKind kind_to_coarser;
};
std::vector<LevelDescriptor> combine_hierarchies(const std::vector<HpEntry> &spatial,
                                                 const std::vector<HpEntry> &temporal);

struct MultigridLevel
{
  LevelDescriptor desc;
  std::unique_ptr<VelocitySpace> vspace;
  std::unique_ptr<PressureSpace> pspace;
  std::unique_ptr<TemporalMatrices> tmat;
  std::unique_ptr<SpaceTimeBlockOperator> op;
  std::unique_ptr<VankaSmoother> smoother;
  std::unique_ptr<TransferPair> to_coarser;
  bool coarse_direct = false;
};

struct HierarchyParams
{
  double nu;
  double tau;
  double grad_div = 0.0;
  SmootherKind smoother = SmootherKind::cell;
  std::uint64_t patch_memory_cap = 8ull << 30;
};

class LevelHierarchy
{
public:
  int n_levels() const { return static_cast<int>(levels_.size()); }
  MultigridLevel &level(int l) { return *levels_[l]; }
  const MultigridLevel &level(int l) const { return *levels_[l]; }
  const MultigridLevel &finest() const { return *levels_.back(); }
  std::vector<std::unique_ptr<MultigridLevel>> levels_;
};
LevelHierarchy instantiate_levels(const Mesh &mesh, const std::vector<LevelDescriptor> &desc,
                                  const HierarchyParams &params);

// ---------------------------------------------------------------- solver
struct VCycleConfig // solver.hpp:15-22
{
  int nu1 = 1, nu2 = 1;
  double omega = 0.8;
  bool project_pressure = true;
  int coarse_dof_cap = 50000;
};
struct KrylovConfig // solver.hpp:24-30
{
  double rtol = 1e-8, atol = 1e-14;
  int max_iterations = 200, max_basis = 200;
};

class CoarseSolver // solver.cpp:10-54
{
public:
  CoarseSolver(const SpaceTimeBlockOperator &op, int dof_cap);
  BlockVector solve(const BlockVector &b) const;
  const Mat &pinned_matrix() const { return matrix_; }

private:
  const SpaceTimeBlockOperator *op_;
  Mat matrix_;
  LU lu_;
  std::vector<Index> pinned_;
};

class VCycle // solver.cpp:56-93
{
public:
  VCycle(const LevelHierarchy &levels, const VCycleConfig &config);
  BlockVector apply(const BlockVector &b) const;

private:
  BlockVector cycle(int l, const BlockVector &b) const;
  const LevelHierarchy *levels_;
  VCycleConfig config_;
  std::unique_ptr<CoarseSolver> coarse_;
};

using ApplyFn = std::function<void(const BlockVector &, BlockVector &)>;
using PrecondFn = std::function<BlockVector(const BlockVector &)>;
struct GmresResult
{
  BlockVector x;
  int iterations = 0;
  bool converged = false;
  Vec residual_history;
};
GmresResult gmres(const ApplyFn &apply, const PrecondFn &precondition, const BlockVector &b, const BlockVector &x0,
                  const KrylovConfig &config); // solver.cpp:95-202

struct StepRecord
{
  int step, iterations;
  double residual, seconds, max_divergence, max_pressure_mean;
};
struct TimeMarchResult
{
  std::vector<BlockVector> trajectory;
  std::vector<StepRecord> steps;
  double avg_iterations = 0.0, total_seconds = 0.0;
  std::uint64_t dofs_processed = 0;
  double throughput = 0.0;
  bool converged = true;
};
struct TimeMarchProblem
{
  ForceFn force;
  std::function<double(double, double, double, int)> boundary;
  std::function<double(double, double, int)> initial_velocity;
  /// Extension used by the seeded-RHS harness (not in the reference): a
  /// per-step load vector added to the right-hand side before the coupling.
  std::function<void(int step, BlockVector &rhs)> extra_rhs;
};
TimeMarchResult time_march(const LevelHierarchy &levels, const TimeMarchProblem &problem, int n_steps,
                           const VCycleConfig &mg, const KrylovConfig &kr, bool keep_trajectory = true);

// ---------------------------------------------------------------- problems / harness
struct ExactSolution
{
  std::function<double(double, double, double, int)> velocity;
  std::function<double(double, double, double, int, int)> velocity_gradient;
  std::function<double(double, double, double)> pressure;
};
struct StokesProblem
{
  double nu = 0.1, t_end = 1.0;
  TimeMarchProblem data;
  ExactSolution exact;
  bool has_exact = false;
};
StokesProblem manufactured_problem(); // problems.cpp:13-62
StokesProblem cavity_problem(double nu); // problems.cpp:64-78

struct ErrorReport
{
  double e_v_l2 = 0, e_p_l2 = 0, e_v_h1 = 0, e_div = 0, e_v_linf = 0;
};
struct RunConfig // harness.hpp:30-45
{
  int r = 2, k = -1, refinements = 2, n_steps = 0;
  double nu = 0.1, grad_div = 1.0;
  SmootherKind smoother = SmootherKind::cell;
  bool h_only = false, allow_large = false;
  VCycleConfig mg;
  KrylovConfig krylov;
  int time_degree() const { return k < 0 ? r : k; }
};
struct Setup
{
  std::unique_ptr<Mesh> mesh;
  std::vector<LevelDescriptor> descriptors;
  LevelHierarchy levels;
};
std::vector<LevelDescriptor> plan_hierarchy(const RunConfig &config, double t_end); // harness.cpp:26-42
Setup build_setup(const StokesProblem &problem, const RunConfig &config);          // harness.cpp:51-70
int step_count(const StokesProblem &problem, const RunConfig &config);
ErrorReport compute_errors(const Setup &setup, const TimeMarchResult &march, const ExactSolution &exact);
TimeMarchResult interpolate_exact(const Setup &setup, const ExactSolution &exact, int n_steps); // harness.cpp:185-239
double evaluate_pressure(const PressureSpace &ps, const double *coeffs, double x, double y);
double evaluate_velocity(const VelocitySpace &vs, const double *coeffs, double x, double y, int comp);

} // namespace oracle
