// ORACLE PIN — ports the reference suites' known-answer and oracle-equivalence
// tests onto the restatement, with the reference's own tolerances. Each case
// cites the reference test it follows (/root/reference/proj/tests/...).
//
//   oracle_tests [suite ...]     suites: quadrature time_basis mesh dof_space
//                                st_operator vanka transfer hierarchy solver
//                                acceptance_table1 (slow)
// Prints one "[PASS]/[FAIL] suite: case (detail)" line per check group and
// exits non-zero on any failure.
#include "oracle/oracle.hpp"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <sstream>

using namespace oracle;

namespace
{
int g_failures = 0;
std::string g_suite;

struct Case
{
  std::string name;
  bool ok = true;
  std::string detail;
  explicit Case(std::string n) : name(std::move(n)) {}
  void check(bool cond, const std::string &what)
  {
    if (!cond)
      {
        ok = false;
        if (detail.size() < 400)
          detail += what + "; ";
      }
  }
  ~Case()
  {
    std::printf("[%s] %s: %s %s\n", ok ? "PASS" : "FAIL", g_suite.c_str(), name.c_str(),
                detail.empty() ? "" : ("(" + detail + ")").c_str());
    if (!ok)
      ++g_failures;
  }
};

std::string
num(double v)
{
  char b[64];
  std::snprintf(b, sizeof b, "%.3g", v);
  return b;
}

bool
approx(double a, double b, double eps)
{ // doctest::Approx with epsilon, scale 1
  return std::abs(a - b) <= eps * (1.0 + std::max(std::abs(a), std::abs(b)));
}

template <class F>
bool
throws(F &&f)
{
  try
    {
      f();
    }
  catch (const std::exception &)
    {
      return true;
    }
  return false;
}

const Box unit{0.0, 0.0, 1.0, 1.0};

Vec
random_vector(Index n, std::mt19937 &rng)
{
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  Vec v(n);
  for (Index i = 0; i < n; ++i)
    v[i] = dist(rng);
  return v;
}

double
norm(const Vec &v)
{
  double s = 0;
  for (double x : v)
    s += x * x;
  return std::sqrt(s);
}

double
diffnorm(const double *a, const double *b, Index n)
{
  double s = 0;
  for (Index i = 0; i < n; ++i)
    s += (a[i] - b[i]) * (a[i] - b[i]);
  return std::sqrt(s);
}

double
dotp(const double *a, const double *b, Index n)
{
  double s = 0;
  for (Index i = 0; i < n; ++i)
    s += a[i] * b[i];
  return s;
}

double
moment(const QuadratureRule &r, int d)
{
  double s = 0;
  for (int q = 0; q < r.size(); ++q)
    s += r.weights[q] * std::pow(r.points[q], d);
  return s;
}

double
exact_moment(int d)
{
  return d % 2 == 0 ? 2.0 / (d + 1) : 0.0;
}

// ------------------------------------------------------------ quadrature
// tests/test_quadrature.cpp
void
suite_quadrature()
{
  {
    Case c("gauss_rule small cases (test_quadrature.cpp:32-46)");
    const auto g1 = gauss_rule(1);
    c.check(std::abs(g1.points[0]) < 1e-15 && approx(g1.weights[0], 2.0, 1e-14), "g1");
    const auto g2 = gauss_rule(2);
    c.check(approx(g2.points[0], -1.0 / std::sqrt(3.0), 1e-14) && approx(g2.points[1], 1.0 / std::sqrt(3.0), 1e-14),
            "g2 nodes");
    c.check(approx(g2.weights[0], 1.0, 1e-14) && approx(g2.weights[1], 1.0, 1e-14), "g2 weights");
    c.check(throws([] { gauss_rule(0); }), "n=0 throws");
  }
  {
    Case c("gauss_rule exactness n<=8 (test_quadrature.cpp:48-61)");
    for (int n = 1; n <= 8; ++n)
      {
        const auto r = gauss_rule(n);
        double s = 0;
        for (double w : r.weights)
          s += w;
        c.check(approx(s, 2.0, 1e-14), "weight sum n=" + std::to_string(n));
        for (int d = 0; d <= 2 * n - 1; ++d)
          c.check(approx(moment(r, d), exact_moment(d), 1e-13), "moment n=" + std::to_string(n));
      }
  }
  {
    Case c("gauss_radau_right small cases (test_quadrature.cpp:63-79)");
    const auto r1 = gauss_radau_right(1);
    c.check(r1.points[0] == 1.0 && approx(r1.weights[0], 2.0, 1e-14), "r1");
    const auto r2 = gauss_radau_right(2);
    c.check(std::abs(r2.points[0] + 1.0 / 3.0) < 1e-14 && r2.points[1] == 1.0, "r2 nodes " + num(r2.points[0]));
    c.check(std::abs(r2.weights[0] - 1.5) < 1e-14 && std::abs(r2.weights[1] - 0.5) < 1e-14, "r2 weights");
    c.check(approx(moment(gauss_radau_right(3), 4), 0.4, 1e-14), "r3 x^4");
    c.check(throws([] { gauss_radau_right(0); }), "n=0 throws");
  }
  {
    Case c("gauss_radau_right exactness/positivity (test_quadrature.cpp:81-94; acceptance.cpp:48-72)");
    double worst = 0;
    for (int n = 1; n <= 8; ++n)
      {
        const auto r = gauss_radau_right(n);
        c.check(r.points[n - 1] == 1.0, "endpoint");
        for (double w : r.weights)
          c.check(w > 0.0, "positive");
        for (int d = 0; d <= 2 * n - 2; ++d)
          worst = std::max(worst, std::abs(moment(r, d) - exact_moment(d)));
      }
    c.check(worst < 1e-13, "moment err " + num(worst));
  }
  {
    Case c("gauss_lobatto_points (test_quadrature.cpp:96-113)");
    const Vec gl3 = gauss_lobatto_points(3);
    c.check(gl3[0] == -1.0 && gl3[1] == 0.0 && gl3[2] == 1.0, "gl3");
    c.check(approx(gauss_lobatto_points(4)[1], -1.0 / std::sqrt(5.0), 1e-14), "gl4");
    for (int n = 2; n <= 9; ++n)
      {
        const Vec v = gauss_lobatto_points(n);
        c.check(v[0] == -1.0 && v[n - 1] == 1.0, "endpoints");
        for (int i = 0; i + 1 < n; ++i)
          c.check(v[i] < v[i + 1], "increasing");
      }
  }
  {
    Case c("lagrange basis properties (test_quadrature.cpp:115-137)");
    const NodalBasis1D lin(Vec{-1.0, 1.0});
    c.check(approx(lin.value(0, 0.0), 0.5, 1e-14) && approx(lin.derivative(1, -0.3), 0.5, 1e-14), "linear");
    const NodalBasis1D b(gauss_lobatto_points(5));
    for (int i = 0; i < b.size(); ++i)
      for (int j = 0; j < b.size(); ++j)
        c.check(approx(b.value(i, b.nodes()[j]), i == j ? 1.0 : 0.0, 1e-13), "lagrange");
    double s = 0, ds = 0;
    for (double v : b.values(0.37))
      s += v;
    for (double v : b.derivatives(0.37))
      ds += v;
    c.check(approx(s, 1.0, 1e-13) && std::abs(ds) < 1e-12, "partition of unity");
    c.check(throws([] { NodalBasis1D(Vec{0.5, 0.5}); }), "duplicate nodes throw");
  }
  {
    Case c("pdisc basis dimensions and orthogonality (test_quadrature.cpp:139-191)");
    c.check(PDiscBasis(1, 2).size() == 3 && PDiscBasis(2, 2).size() == 6 && PDiscBasis(4, 2).size() == 15, "2d sizes");
    c.check(PDiscBasis(1, 3).size() == 4 && PDiscBasis(2, 3).size() == 10, "3d sizes");
    c.check(throws([] { PDiscBasis(0, 2); }), "r=0 throws");
    for (int r : {1, 2, 3, 4})
      {
        const PDiscBasis basis(r, 2);
        const auto g = gauss_rule(r + 1);
        Mat gram(basis.size(), basis.size());
        double xi[2];
        for (int qy = 0; qy < g.size(); ++qy)
          for (int qx = 0; qx < g.size(); ++qx)
            {
              xi[0] = g.points[qx];
              xi[1] = g.points[qy];
              const double w = g.weights[qx] * g.weights[qy];
              for (int a = 0; a < basis.size(); ++a)
                for (int b = 0; b < basis.size(); ++b)
                  gram(a, b) += w * basis.value(a, xi) * basis.value(b, xi);
            }
        for (int a = 0; a < basis.size(); ++a)
          {
            c.check(approx(gram(a, a), basis.gram_diagonal(a), 1e-13), "gram diag");
            for (int b = 0; b < basis.size(); ++b)
              if (a != b)
                c.check(std::abs(gram(a, b)) < 1e-12 * gram(a, a), "orthogonal");
          }
        xi[0] = 0.123;
        xi[1] = -0.777;
        c.check(approx(basis.value(0, xi), 1.0, 1e-14), "constant first");
      }
  }
}

// ------------------------------------------------------------ time basis
double
radau_iia_stability(int s, double z) // tests/test_time_basis.cpp:15-33
{
  const int m = s - 1, n = s;
  const auto fact = [](int v) {
    double f = 1.0;
    for (int i = 2; i <= v; ++i)
      f *= i;
    return f;
  };
  double numr = 0.0, den = 0.0;
  for (int j = 0; j <= m; ++j)
    numr += fact(m) * fact(m + n - j) / (fact(m + n) * fact(j) * fact(m - j)) * std::pow(z, j);
  for (int j = 0; j <= n; ++j)
    den += fact(n) * fact(m + n - j) / (fact(m + n) * fact(j) * fact(n - j)) * std::pow(-z, j);
  return numr / den;
}

void
suite_time_basis()
{
  {
    Case c("k=0 reduces to backward Euler (test_time_basis.cpp:36-43)");
    const auto tm = temporal_matrices(0, 0.37);
    c.check(approx(tm.dt_plus_jump(0, 0), 1.0, 1e-14) && approx(tm.mass(0, 0), 0.37, 1e-14) &&
              approx(tm.coupling(0, 0), 1.0, 1e-14),
            "values");
  }
  {
    Case c("temporal matrix invariants (test_time_basis.cpp:45-76)");
    for (int k : {1, 2, 3})
      for (double tau : {0.3, 2.2})
        {
          const auto tm = temporal_matrices(k, tau);
          const auto ref = temporal_matrices(k, 1.0);
          double msum = 0, ksum = 0, asym = 0, dk = 0;
          for (int a = 0; a <= k; ++a)
            for (int b = 0; b <= k; ++b)
              {
                msum += tm.mass(a, b);
                ksum += tm.dt_plus_jump(a, b);
                asym = std::max(asym, std::abs(tm.mass(a, b) - tm.mass(b, a)));
                dk = std::max(dk, std::abs(tm.dt_plus_jump(a, b) - ref.dt_plus_jump(a, b)));
              }
          c.check(asym < 1e-14 * tau, "mass symmetric");
          c.check(approx(msum, tau, 1e-13), "mass sum");
          c.check(dk < 1e-13, "K tau-free");
          c.check(approx(ksum, 1.0, 1e-12), "K sum");
          const LU lu(tm.mass);
          c.check(!lu.singular, "mass nonsingular");
          for (int a = 0; a <= k; ++a)
            {
              for (int b = 0; b < k; ++b)
                c.check(tm.coupling(a, b) == 0.0, "coupling rank one");
              c.check(approx(tm.coupling(a, k), tm.left_values[a], 1e-14), "coupling last column");
            }
        }
    c.check(throws([] { temporal_matrices(1, 0.0); }) && throws([] { temporal_matrices(1, -1.0); }), "tau<=0 throws");
  }
  {
    Case c("dg_ode_step small cases (test_time_basis.cpp:78-94)");
    c.check(approx(dg_ode_step(0, 0.1, -1.0, 1.0), 1.0 / 1.1, 1e-14), "k=0");
    const double z = -0.1;
    const double r2 = (1.0 + z / 3.0) / (1.0 - 2.0 * z / 3.0 + z * z / 6.0);
    c.check(approx(dg_ode_step(1, 0.1, -1.0, 1.0), r2, 1e-13), "k=1");
    for (int k = 0; k <= 4; ++k)
      c.check(approx(dg_ode_step(k, 0.5, 0.0, 1.0), 1.0, 1e-13), "lambda=0");
    c.check(throws([] { dg_ode_step(0, 1.0, 1.0, 1.0); }), "pole throws");
  }
  {
    Case c("DG(k) endpoint = Radau IIA (test_time_basis.cpp:96-107; acceptance.cpp:95-107 gate 1e-12)");
    double worst = 0;
    for (int k = 0; k <= 3; ++k)
      for (double z : {-0.1, -0.5, -1.0, -4.0})
        worst = std::max(worst, std::abs(dg_ode_step(k, 1.0, z, 1.0) - radau_iia_stability(k + 1, z)));
    c.check(worst < 1e-12, "worst " + num(worst));
  }
  {
    Case c("DG(k) endpoint superconvergence 2k+1 (test_time_basis.cpp:109-126)");
    for (int k : {1, 2})
      {
        double e[3];
        int idx = 0;
        for (int n : {2, 4, 8})
          {
            double y = 1.0;
            for (int i = 0; i < n; ++i)
              y = dg_ode_step(k, 1.0 / n, -1.0, y);
            e[idx++] = std::abs(y - std::exp(-1.0));
          }
        const double eoc1 = std::log2(e[0] / e[1]), eoc2 = std::log2(e[1] / e[2]);
        c.check(std::abs(eoc1 - (2 * k + 1)) < 0.3 * (1 + 2 * k + 1) / (2 * k + 1), "eoc1 " + num(eoc1));
        c.check(std::abs(eoc2 - (2 * k + 1)) < 0.3 * (1 + 2 * k + 1) / (2 * k + 1), "eoc2 " + num(eoc2));
      }
  }
}

// ------------------------------------------------------------ mesh / dof space
void
suite_mesh()
{
  Case c("mesh hierarchy (test_mesh.cpp:15-114)");
  const Mesh m = Mesh::build_cartesian(unit, 1, 1, 3);
  c.check(m.n_levels() == 3 && m.n_cells(0) == 1 && m.n_cells(1) == 4 && m.n_cells(2) == 16, "counts");
  c.check(approx(m.hx(2), 0.25, 1e-15), "hx");
  c.check(throws([] { Mesh::build_cartesian(unit, 0, 1, 1); }) && throws([] { Mesh::build_cartesian(unit, 1, 1, 0); }),
          "bad args");
  for (int s = 0; s < 2; ++s)
    for (int cell = 0; cell < m.n_cells(s); ++cell)
      for (int ch : m.children(s, cell))
        c.check(m.parent(s + 1, ch) == cell, "parent/children");
  c.check(m.cells_of_vertex(2, m.vertex_index(2, 2, 2)).size() == 4, "interior vertex");
  c.check(m.cells_of_vertex(2, m.vertex_index(2, 0, 0)).size() == 1, "corner vertex");
  c.check(m.cells_of_vertex(2, m.vertex_index(2, 2, 0)).size() == 2, "edge vertex");
  c.check(throws([&] { m.cells_of_vertex(2, m.n_vertices(2)); }), "bad vertex");
  c.check(m.vertex_neighbors(2, m.cell_index(2, 1, 1)).size() == 9, "nbr 9");
  c.check(m.vertex_neighbors(2, m.cell_index(2, 0, 0)).size() == 4, "nbr 4");
  c.check(m.vertex_neighbors(2, m.cell_index(2, 0, 1)).size() == 6, "nbr 6");
}

void
suite_dof_space()
{
  const Mesh mesh = Mesh::build_cartesian(unit, 1, 1, 4);
  {
    Case c("dof counts (test_dof_space.cpp:16-34, 77-96)");
    const VelocitySpace v22(mesh, 1, 1);
    c.check(v22.n_scalar_dofs() == 25 && v22.n_dofs() == 50, "v22");
    const VelocitySpace v11(mesh, 0, 1);
    c.check(v11.n_dofs() == 18, "v11");
    const PressureSpace p22(mesh, 1, 1);
    c.check(p22.n_dofs() == 12, "p22");
    const PressureSpace p88(mesh, 3, 4);
    c.check(p88.n_dofs() == 960, "p88");
    c.check(approx(dotp(p22.one_coefficients().data(), p22.mean_vector().data(), p22.n_dofs()), 1.0, 1e-14),
            "<1,m>=|Omega|");
  }
  {
    Case c("project_mean_zero idempotent (test_dof_space.cpp:98-119)");
    const PressureSpace ps(mesh, 2, 2);
    std::mt19937 rng(3);
    Vec q = random_vector(ps.n_dofs(), rng);
    ps.project_mean_zero(q.data());
    c.check(std::abs(ps.mean_integral(q.data())) < 1e-13 * norm(q), "mean zero");
    Vec q2 = q;
    ps.project_mean_zero(q2.data());
    c.check(diffnorm(q.data(), q2.data(), ps.n_dofs()) < 1e-14 * norm(q), "idempotent");
    Vec one = ps.one_coefficients();
    ps.project_mean_zero(one.data());
    c.check(norm(one) < 1e-14, "constant projects to zero");
  }
}

// ------------------------------------------------------------ st_operator
// Dense quadrature assembly without sum factorisation (test_st_operator.cpp:27-102).
struct DenseOracle
{
  Mat mass, laplace, div, pmass, grad_div;
};

DenseOracle
assemble_dense(const VelocitySpace &vs, const PressureSpace &ps)
{
  const Mesh &mesh = vs.mesh();
  const int level = vs.level(), n1 = vs.nodes_per_dir(), np = ps.dofs_per_cell(), nsc = vs.n_scalar_dofs();
  DenseOracle o;
  o.mass = Mat(nsc, nsc);
  o.laplace = Mat(nsc, nsc);
  o.div = Mat(static_cast<int>(ps.n_dofs()), static_cast<int>(vs.n_dofs()));
  o.pmass = Mat(static_cast<int>(ps.n_dofs()), static_cast<int>(ps.n_dofs()));
  o.grad_div = Mat(static_cast<int>(vs.n_dofs()), static_cast<int>(vs.n_dofs()));
  const auto g = gauss_rule(n1 + 1);
  const double hx = mesh.hx(level), hy = mesh.hy(level), jdet = 0.25 * hx * hy;
  double xi[2];
  Vec val(n1 * n1), gx(n1 * n1), gy(n1 * n1);
  for (int cell = 0; cell < mesh.n_cells(level); ++cell)
    {
      const auto &dofs = vs.cell_scalar_dofs(cell);
      const int pb = static_cast<int>(ps.cell_dof(cell, 0));
      for (int qy = 0; qy < g.size(); ++qy)
        for (int qx = 0; qx < g.size(); ++qx)
          {
            const double w = g.weights[qx] * g.weights[qy] * jdet;
            xi[0] = g.points[qx];
            xi[1] = g.points[qy];
            for (int jy = 0; jy < n1; ++jy)
              for (int jx = 0; jx < n1; ++jx)
                {
                  const double vx = vs.basis_1d().value(jx, xi[0]), vy = vs.basis_1d().value(jy, xi[1]);
                  const double dx = vs.basis_1d().derivative(jx, xi[0]), dy = vs.basis_1d().derivative(jy, xi[1]);
                  val[jy * n1 + jx] = vx * vy;
                  gx[jy * n1 + jx] = (2.0 / hx) * dx * vy;
                  gy[jy * n1 + jx] = (2.0 / hy) * vx * dy;
                }
            for (int i = 0; i < n1 * n1; ++i)
              for (int j = 0; j < n1 * n1; ++j)
                {
                  o.mass(dofs[i], dofs[j]) += w * val[i] * val[j];
                  o.laplace(dofs[i], dofs[j]) += w * (gx[i] * gx[j] + gy[i] * gy[j]);
                  const int i0 = dofs[i], i1 = nsc + dofs[i], j0 = dofs[j], j1 = nsc + dofs[j];
                  o.grad_div(i0, j0) += w * gx[i] * gx[j];
                  o.grad_div(i0, j1) += w * gx[i] * gy[j];
                  o.grad_div(i1, j0) += w * gy[i] * gx[j];
                  o.grad_div(i1, j1) += w * gy[i] * gy[j];
                }
            for (int l = 0; l < np; ++l)
              {
                const double psi = ps.basis().value(l, xi);
                for (int j = 0; j < n1 * n1; ++j)
                  {
                    o.div(pb + l, dofs[j]) += w * psi * gx[j];
                    o.div(pb + l, nsc + dofs[j]) += w * psi * gy[j];
                  }
                for (int m = 0; m < np; ++m)
                  o.pmass(pb + l, pb + m) += w * psi * ps.basis().value(m, xi);
              }
          }
    }
  return o;
}

Vec
matvec(const Mat &m, const Vec &x)
{
  Vec y(m.r, 0.0);
  for (int j = 0; j < m.c; ++j)
    for (int i = 0; i < m.r; ++i)
      y[i] += m(i, j) * x[j];
  return y;
}

Vec
matvec_expand(const Mat &scalar, const Vec &x)
{ // vector_expand (test_st_operator.cpp:115-124)
  const int n = scalar.r;
  Vec y(2 * n, 0.0);
  for (int comp = 0; comp < 2; ++comp)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i)
        y[comp * n + i] += scalar(i, j) * x[comp * n + j];
  return y;
}

void
suite_st_operator()
{
  {
    Case c("velocity mass: constants, zero, dense oracle 1e-13 (test_st_operator.cpp:127-152)");
    const Mesh mesh = Mesh::build_cartesian(unit, 1, 1, 2);
    const VelocitySpace vs(mesh, 1, 1);
    const PressureSpace ps(mesh, 1, 1);
    const auto tm = temporal_matrices(1, 0.5);
    const SpaceTimeBlockOperator op(vs, ps, tm, 0.1);
    Vec ones(vs.n_dofs(), 1.0), y(vs.n_dofs());
    op.apply_velocity_mass(ones.data(), y.data());
    c.check(approx(dotp(ones.data(), y.data(), vs.n_dofs()), 2.0, 1e-14), "1^T M 1 = 2");
    const auto o = assemble_dense(vs, ps);
    std::mt19937 rng(11);
    for (int t = 0; t < 3; ++t)
      {
        const Vec v = random_vector(vs.n_dofs(), rng);
        op.apply_velocity_mass(v.data(), y.data());
        const Vec ref = matvec_expand(o.mass, v);
        c.check(diffnorm(y.data(), ref.data(), vs.n_dofs()) < 1e-13 * norm(ref), "dense oracle");
      }
  }
  {
    Case c("laplace: constants, <x,Ax>=1, dense oracle (test_st_operator.cpp:154-179)");
    const Mesh mesh = Mesh::build_cartesian(unit, 1, 1, 2);
    const VelocitySpace vs(mesh, 1, 2);
    const PressureSpace ps(mesh, 1, 2);
    const auto tm = temporal_matrices(1, 0.5);
    const SpaceTimeBlockOperator op(vs, ps, tm, 0.1);
    Vec y(vs.n_dofs()), ones(vs.n_dofs(), 1.0);
    op.apply_laplace(ones.data(), y.data());
    c.check(norm(y) < 1e-13, "constants");
    Vec vx(vs.n_dofs(), 0.0);
    for (int s = 0; s < vs.n_scalar_dofs(); ++s)
      vx[vs.global_dof(0, s)] = vs.node_x(s);
    op.apply_laplace(vx.data(), y.data());
    c.check(approx(dotp(vx.data(), y.data(), vs.n_dofs()), 1.0, 1e-13), "<x,Ax>=1");
    const auto o = assemble_dense(vs, ps);
    std::mt19937 rng(13);
    const Vec v = random_vector(vs.n_dofs(), rng);
    op.apply_laplace(v.data(), y.data());
    const Vec ref = matvec_expand(o.laplace, v);
    c.check(diffnorm(y.data(), ref.data(), vs.n_dofs()) < 1e-13 * norm(ref), "dense oracle");
  }
  {
    Case c("divergence pair: div-free, adjoint, dense oracle (test_st_operator.cpp:181-214)");
    const Mesh mesh = Mesh::build_cartesian(unit, 1, 1, 3);
    const VelocitySpace vs(mesh, 1, 1);
    const PressureSpace ps(mesh, 1, 1);
    const auto tm = temporal_matrices(1, 0.5);
    const SpaceTimeBlockOperator op(vs, ps, tm, 0.1);
    Vec v(vs.n_dofs(), 0.0), p(ps.n_dofs());
    for (int s = 0; s < vs.n_scalar_dofs(); ++s)
      {
        v[vs.global_dof(0, s)] = vs.node_x(s);
        v[vs.global_dof(1, s)] = -vs.node_y(s);
      }
    op.apply_div(v.data(), p.data());
    c.check(norm(p) < 1e-13, "B(x,-y)=0");
    std::mt19937 rng(17);
    const Vec w = random_vector(vs.n_dofs(), rng), q = random_vector(ps.n_dofs(), rng);
    Vec bw(ps.n_dofs()), btq(vs.n_dofs());
    op.apply_div(w.data(), bw.data());
    op.apply_div_transpose(q.data(), btq.data());
    c.check(approx(dotp(bw.data(), q.data(), ps.n_dofs()), dotp(w.data(), btq.data(), vs.n_dofs()), 1e-13),
            "adjoint");
    const auto o = assemble_dense(vs, ps);
    const Vec ref = matvec(o.div, w);
    c.check(diffnorm(bw.data(), ref.data(), ps.n_dofs()) < 1e-13 * norm(bw), "B oracle");
    const Vec reft = matvec(transpose(o.div), q);
    c.check(diffnorm(btq.data(), reft.data(), vs.n_dofs()) < 1e-13 * norm(btq), "B^T oracle");
  }
  {
    Case c("pressure mass: 1^T M_p 1 = 1, diagonal, oracle (test_st_operator.cpp:245-274)");
    const Mesh mesh = Mesh::build_cartesian(unit, 1, 1, 2);
    const VelocitySpace vs(mesh, 1, 3);
    const PressureSpace ps(mesh, 1, 3);
    const auto tm = temporal_matrices(1, 0.5);
    const SpaceTimeBlockOperator op(vs, ps, tm, 0.1);
    Vec y(ps.n_dofs());
    op.apply_pressure_mass(ps.one_coefficients().data(), y.data());
    c.check(approx(dotp(ps.one_coefficients().data(), y.data(), ps.n_dofs()), 1.0, 1e-14), "1^T Mp 1");
    const auto o = assemble_dense(vs, ps);
    std::mt19937 rng(19);
    const Vec q = random_vector(ps.n_dofs(), rng);
    op.apply_pressure_mass(q.data(), y.data());
    const Vec ref = matvec(o.pmass, q);
    c.check(diffnorm(y.data(), ref.data(), ps.n_dofs()) < 1e-13 * norm(y), "oracle");
  }
  {
    Case c("grad-div: constants, div-free, <v,Gv>=4, oracle (test_st_operator.cpp:276-313)");
    const Mesh mesh = Mesh::build_cartesian(unit, 1, 1, 2);
    const VelocitySpace vs(mesh, 1, 2);
    const PressureSpace ps(mesh, 1, 2);
    const auto tm = temporal_matrices(1, 0.5);
    const SpaceTimeBlockOperator op(vs, ps, tm, 0.1);
    Vec y(vs.n_dofs()), ones(vs.n_dofs(), 1.0);
    op.apply_grad_div(ones.data(), y.data());
    c.check(norm(y) < 1e-13, "constants");
    Vec v(vs.n_dofs(), 0.0);
    for (int s = 0; s < vs.n_scalar_dofs(); ++s)
      {
        v[vs.global_dof(0, s)] = vs.node_x(s);
        v[vs.global_dof(1, s)] = -vs.node_y(s);
      }
    op.apply_grad_div(v.data(), y.data());
    c.check(norm(y) < 1e-13, "div-free");
    for (int s = 0; s < vs.n_scalar_dofs(); ++s)
      v[vs.global_dof(1, s)] = vs.node_y(s);
    op.apply_grad_div(v.data(), y.data());
    c.check(approx(dotp(v.data(), y.data(), vs.n_dofs()), 4.0, 1e-13), "<v,Gv>=4");
    const auto o = assemble_dense(vs, ps);
    std::mt19937 rng(43);
    const Vec w = random_vector(vs.n_dofs(), rng);
    op.apply_grad_div(w.data(), y.data());
    const Vec ref = matvec(o.grad_div, w);
    c.check(diffnorm(y.data(), ref.data(), vs.n_dofs()) < 1e-13 * norm(ref), "oracle");
  }
  {
    Case c("apply_block vs sparse oracle r,k in {1,2} and gamma=0.7 (test_st_operator.cpp:315-417)");
    const Mesh mesh = Mesh::build_cartesian(unit, 1, 1, 2);
    std::mt19937 rng(29);
    for (int r : {1, 2})
      for (int k : {1, 2})
        for (double gd : {0.0, 0.7})
          {
            const VelocitySpace vs(mesh, 1, r);
            const PressureSpace ps(mesh, 1, r);
            const auto tm = temporal_matrices(k, 0.5);
            const SpaceTimeBlockOperator op(vs, ps, tm, 0.1, gd);
            const SparseMatrix oracle = op.assemble_sparse_oracle();
            BlockVector x = op.make_vector(), y = op.make_vector();
            for (int t = 0; t < 3; ++t)
              {
                x.data = random_vector(x.size(), rng);
                op.apply_block(x, y);
                Vec ref(x.size());
                oracle.multiply(x.data.data(), ref.data());
                c.check(diffnorm(y.data.data(), ref.data(), x.size()) < 1e-12 * norm(ref), "oracle");
              }
            x.setZero();
            op.apply_block(x, y);
            c.check(y.norm() == 0.0, "zero maps to zero");
          }
  }
  {
    Case c("k=0 one-stage reduction (test_st_operator.cpp:358-387)");
    const Mesh mesh = Mesh::build_cartesian(unit, 1, 1, 2);
    const VelocitySpace vs(mesh, 1, 1);
    const PressureSpace ps(mesh, 1, 1);
    const double tau = 0.25, nu = 0.1;
    const auto tm = temporal_matrices(0, tau);
    const SpaceTimeBlockOperator op(vs, ps, tm, nu);
    std::mt19937 rng(23);
    BlockVector x = op.make_vector();
    x.data = random_vector(x.size(), rng);
    vs.zero_constrained(x.velocity(0));
    BlockVector y = op.make_vector();
    op.apply_block(x, y);
    Vec mv(vs.n_dofs()), av(vs.n_dofs()), btp(vs.n_dofs()), bv(ps.n_dofs());
    op.apply_velocity_mass(x.velocity(0), mv.data());
    op.apply_laplace(x.velocity(0), av.data());
    op.apply_div_transpose(x.pressure(0), btp.data());
    op.apply_div(x.velocity(0), bv.data());
    Vec ev(vs.n_dofs());
    for (Index i = 0; i < vs.n_dofs(); ++i)
      ev[i] = mv[i] + tau * nu * av[i] - tau * btp[i];
    vs.zero_constrained(ev.data());
    Vec av2(y.velocity(0), y.velocity(0) + vs.n_dofs());
    vs.zero_constrained(av2.data());
    c.check(diffnorm(av2.data(), ev.data(), vs.n_dofs()) < 1e-13 * norm(ev), "velocity");
    Vec tbv(ps.n_dofs());
    for (Index i = 0; i < ps.n_dofs(); ++i)
      tbv[i] = tau * bv[i];
    c.check(diffnorm(y.pressure(0), tbv.data(), ps.n_dofs()) < 1e-13 * norm(bv), "pressure");
  }
  {
    Case c("coupling rhs (test_st_operator.cpp:404-439)");
    const Mesh mesh = Mesh::build_cartesian(unit, 1, 1, 2);
    const VelocitySpace vs(mesh, 1, 1);
    const PressureSpace ps(mesh, 1, 1);
    std::mt19937 rng(31);
    const auto tm = temporal_matrices(2, 0.25);
    const SpaceTimeBlockOperator op(vs, ps, tm, 0.1);
    const Vec vp = random_vector(vs.n_dofs(), rng);
    const BlockVector out = op.coupling_rhs(vp.data());
    Vec mv(vs.n_dofs());
    op.apply_velocity_mass(vp.data(), mv.data());
    for (int a = 0; a <= 2; ++a)
      {
        Vec e(vs.n_dofs());
        for (Index i = 0; i < vs.n_dofs(); ++i)
          e[i] = tm.left_values[a] * mv[i];
        c.check(diffnorm(out.velocity(a), e.data(), vs.n_dofs()) < 1e-13 * norm(mv), "slot");
        c.check(norm(Vec(out.pressure(a), out.pressure(a) + ps.n_dofs())) == 0.0, "pressure zero");
      }
  }
  {
    Case c("Kronecker rank-1 identity (test_st_operator.cpp:497-528)");
    const Mesh mesh = Mesh::build_cartesian(unit, 1, 1, 2);
    const VelocitySpace vs(mesh, 1, 1);
    const PressureSpace ps(mesh, 1, 1);
    const auto tm = temporal_matrices(2, 0.4);
    const SpaceTimeBlockOperator op(vs, ps, tm, 0.0);
    std::mt19937 rng(37);
    Vec w = random_vector(vs.n_dofs(), rng);
    vs.zero_constrained(w.data());
    const double cc[3] = {0.3, -1.1, 0.7};
    BlockVector x = op.make_vector();
    for (int a = 0; a < 3; ++a)
      for (Index i = 0; i < vs.n_dofs(); ++i)
        x.velocity(a)[i] = cc[a] * w[i];
    BlockVector y = op.make_vector();
    op.apply_block(x, y);
    Vec mw(vs.n_dofs());
    op.apply_velocity_mass(w.data(), mw.data());
    vs.zero_constrained(mw.data());
    for (int a = 0; a < 3; ++a)
      {
        double kc = 0;
        for (int b = 0; b < 3; ++b)
          kc += tm.dt_plus_jump(a, b) * cc[b];
        Vec e(vs.n_dofs()), act(y.velocity(a), y.velocity(a) + vs.n_dofs());
        vs.zero_constrained(act.data());
        for (Index i = 0; i < vs.n_dofs(); ++i)
          e[i] = kc * mw[i];
        c.check(diffnorm(act.data(), e.data(), vs.n_dofs()) < 1e-12 * norm(e), "slot");
      }
  }
  {
    Case c("matrix-free D vs oracle, meshes 2x2/4x4, r<=3, k<=2 (acceptance.cpp:127-152, gate 1e-12)");
    const Mesh mesh = Mesh::build_cartesian(unit, 1, 1, 3);
    std::mt19937 rng(101);
    double worst = 0;
    for (int level : {1, 2})
      for (int r : {1, 2, 3})
        for (int k : {1, 2})
          {
            const VelocitySpace vs(mesh, level, r);
            const PressureSpace ps(mesh, level, r);
            const auto tm = temporal_matrices(k, 0.25);
            const SpaceTimeBlockOperator op(vs, ps, tm, 0.1, level == 1 ? 0.0 : 1.0);
            const SparseMatrix oracle = op.assemble_sparse_oracle();
            for (int t = 0; t < 10; ++t)
              {
                BlockVector x = op.make_vector(), y = op.make_vector();
                x.data = random_vector(x.size(), rng);
                op.apply_block(x, y);
                Vec ref(x.size());
                oracle.multiply(x.data.data(), ref.data());
                worst = std::max(worst, diffnorm(y.data.data(), ref.data(), x.size()) / norm(ref));
              }
          }
    c.check(worst < 1e-12, "worst " + num(worst));
  }
  {
    Case c("oracle guard rejects large assemblies (test_st_operator.cpp:554-562)");
    const Mesh mesh = Mesh::build_cartesian(unit, 1, 1, 7);
    const VelocitySpace vs(mesh, 6, 2);
    const PressureSpace ps(mesh, 6, 2);
    const auto tm = temporal_matrices(2, 0.5);
    const SpaceTimeBlockOperator op(vs, ps, tm, 0.1);
    c.check(throws([&] { op.assemble_sparse_oracle(); }), "throws");
  }
}

// ------------------------------------------------------------ vanka
BlockVector
random_interior(const SpaceTimeBlockOperator &op, std::mt19937 &rng)
{
  BlockVector x = op.make_vector();
  x.data = random_vector(x.size(), rng);
  for (int a = 0; a < x.ns; ++a)
    op.velocity_space().zero_constrained(x.velocity(a));
  return x;
}

void
suite_vanka()
{
  {
    Case c("cell patch block sizes 42/44, sorted dof lists (test_vanka.cpp:28-51)");
    const Mesh mesh = Mesh::build_cartesian(unit, 1, 1, 3);
    const VelocitySpace vs(mesh, 2, 1);
    const PressureSpace ps(mesh, 2, 1);
    const auto tm = temporal_matrices(1, 0.25);
    const SpaceTimeBlockOperator op(vs, ps, tm, 0.1);
    const auto sm = VankaSmoother::build(op, SmootherKind::cell);
    c.check(sm.patches().size() == 16, "16 patches");
    c.check(sm.patches()[mesh.cell_index(2, 1, 1)].size() == 42, "interior 42");
    c.check(VankaSmoother::nominal_block_size(1, 1, 2) == 44, "nominal 44");
    for (const auto &p : sm.patches())
      c.check(std::is_sorted(p.dofs.begin(), p.dofs.end()) &&
                std::adjacent_find(p.dofs.begin(), p.dofs.end()) == p.dofs.end(),
              "sorted unique");
  }
  {
    Case c("vertex star patch sizes 124, corner = cell patch (test_vanka.cpp:53-74)");
    const Mesh mesh = Mesh::build_cartesian(unit, 1, 1, 4);
    const VelocitySpace vs(mesh, 3, 1);
    const PressureSpace ps(mesh, 3, 1);
    const auto tm = temporal_matrices(1, 0.25);
    const SpaceTimeBlockOperator op(vs, ps, tm, 0.1);
    const auto sm = VankaSmoother::build(op, SmootherKind::vertex_star);
    c.check(sm.patches().size() == 81, "81 patches");
    c.check(sm.patches()[mesh.vertex_index(3, 4, 4)].size() == 124, "124");
    const auto cells = VankaSmoother::build(op, SmootherKind::cell);
    c.check(sm.patches()[mesh.vertex_index(3, 0, 0)].dofs == cells.patches()[mesh.cell_index(3, 0, 0)].dofs,
            "corner");
  }
  {
    Case c("patch union covers every unconstrained dof (test_vanka.cpp:76-108)");
    const Mesh mesh = Mesh::build_cartesian(unit, 1, 1, 3);
    const VelocitySpace vs(mesh, 2, 2);
    const PressureSpace ps(mesh, 2, 2);
    const auto tm = temporal_matrices(2, 0.25);
    const SpaceTimeBlockOperator op(vs, ps, tm, 0.1);
    for (auto kind : {SmootherKind::cell, SmootherKind::vertex_star})
      {
        const auto sm = VankaSmoother::build(op, kind);
        std::vector<char> cov(op.make_vector().size(), 0);
        for (const auto &p : sm.patches())
          for (Index d : p.dofs)
            cov[d] = 1;
        for (int a = 0; a < 3; ++a)
          {
            for (int comp = 0; comp < 2; ++comp)
              for (int s = 0; s < vs.n_scalar_dofs(); ++s)
                c.check(static_cast<bool>(cov[a * vs.n_dofs() + comp * vs.n_scalar_dofs() + s]) ==
                          !vs.scalar_on_boundary(s),
                        "velocity cover");
            for (Index l = 0; l < ps.n_dofs(); ++l)
              c.check(cov[3 * vs.n_dofs() + a * ps.n_dofs() + l] == 1, "pressure cover");
          }
      }
  }
  {
    Case c("additive sweep vs dense oracle (test_vanka.cpp:110-150 1e-11; acceptance.cpp:178-204 1e-12)");
    std::mt19937 rng(3);
    double worst = 0;
    const Mesh mesh = Mesh::build_cartesian(unit, 1, 1, 3);
    for (auto kind : {SmootherKind::cell, SmootherKind::vertex_star})
      for (int level : {1, 2})
        for (int r : {1, 2})
          for (int k : {1, 2})
            {
              if (level == 2 && kind == SmootherKind::vertex_star && r == 2 && k == 2)
                continue;
              const VelocitySpace vs(mesh, level, r);
              const PressureSpace ps(mesh, level, r);
              const auto tm = temporal_matrices(k, 0.25);
              const SpaceTimeBlockOperator op(vs, ps, tm, 0.1, level == 2 ? 1.0 : 0.0);
              const auto sm = VankaSmoother::build(op, kind);
              const Mat dense = op.assemble_sparse_oracle().to_dense();
              const BlockVector b = random_interior(op, rng);
              BlockVector swept = op.make_vector();
              sm.apply_additive(b, swept);
              Vec ref(b.size(), 0.0);
              for (const auto &p : sm.patches())
                {
                  const int n = p.size();
                  Mat local(n, n);
                  Vec rl(n);
                  for (int i = 0; i < n; ++i)
                    {
                      rl[i] = b.data[p.dofs[i]];
                      for (int j = 0; j < n; ++j)
                        local(i, j) = dense(static_cast<int>(p.dofs[i]), static_cast<int>(p.dofs[j]));
                    }
                  const Vec sol = MinNormSolver(local).solve(rl);
                  for (int i = 0; i < n; ++i)
                    ref[p.dofs[i]] += p.weights[i] * sol[i];
                }
              worst = std::max(worst, diffnorm(swept.data.data(), ref.data(), b.size()) / norm(ref));
            }
    c.check(worst < 1e-11, "worst " + num(worst));
  }
  {
    Case c("single-patch problem: sweep is the exact solve (test_vanka.cpp:152-181)");
    const Mesh mesh = Mesh::build_cartesian(unit, 1, 1, 1);
    const VelocitySpace vs(mesh, 0, 2);
    const PressureSpace ps(mesh, 0, 2);
    const auto tm = temporal_matrices(1, 0.25);
    const SpaceTimeBlockOperator op(vs, ps, tm, 0.1);
    const auto sm = VankaSmoother::build(op, SmootherKind::cell);
    c.check(sm.patches().size() == 1, "one patch");
    std::mt19937 rng(5);
    BlockVector x = random_interior(op, rng);
    for (int a = 0; a < x.ns; ++a)
      ps.project_mean_zero(x.pressure(a));
    BlockVector b = op.make_vector(), solved = op.make_vector();
    op.apply_block(x, b);
    sm.apply_additive(b, solved);
    c.check(diffnorm(solved.data.data(), x.data.data(), x.size()) < 1e-10 * x.norm(), "exact solve");
    BlockVector zero = op.make_vector(), out = op.make_vector();
    sm.apply_additive(zero, out);
    c.check(out.norm() == 0.0, "zero stays zero");
  }
  {
    Case c("smooth_step fixed point; omega validation (test_vanka.cpp:183-202)");
    const Mesh mesh = Mesh::build_cartesian(unit, 1, 1, 2);
    const VelocitySpace vs(mesh, 1, 1);
    const PressureSpace ps(mesh, 1, 1);
    const auto tm = temporal_matrices(1, 0.25);
    const SpaceTimeBlockOperator op(vs, ps, tm, 0.1);
    const auto sm = VankaSmoother::build(op, SmootherKind::cell);
    std::mt19937 rng(7);
    BlockVector u = random_interior(op, rng), b = op.make_vector();
    op.apply_block(u, b);
    BlockVector u2 = u;
    sm.smooth_step(op, b, u2, 0.8);
    c.check(diffnorm(u2.data.data(), u.data.data(), u.size()) < 1e-12 * u.norm(), "fixed point");
    c.check(throws([&] { sm.smooth_step(op, b, u2, 0.0); }) && throws([&] { sm.smooth_step(op, b, u2, 1.5); }),
            "omega");
  }
  {
    Case c("mult-add accounting near sum n_T^2 (test_vanka.cpp:249-266)");
    const Mesh mesh = Mesh::build_cartesian(unit, 1, 1, 2);
    const VelocitySpace vs(mesh, 1, 2);
    const PressureSpace ps(mesh, 1, 2);
    const auto tm = temporal_matrices(1, 0.25);
    const SpaceTimeBlockOperator op(vs, ps, tm, 0.1);
    const auto sm = VankaSmoother::build(op, SmootherKind::cell);
    sm.reset_mult_adds();
    BlockVector b = op.make_vector(), out = op.make_vector();
    std::fill(b.data.begin(), b.data.end(), 1.0);
    sm.apply_additive(b, out);
    const auto nt2 = sm.total_matrix_elements();
    c.check(sm.mult_adds() >= nt2 / 2 && sm.mult_adds() <= 2 * nt2, "range");
  }
}

// ------------------------------------------------------------ transfer
void
suite_transfer()
{
  const Mesh mesh = Mesh::build_cartesian(unit, 1, 1, 3);
  {
    Case c("h transfer: constants, exactness, adjoint (test_transfer.cpp:26-70)");
    const VelocitySpace vc(mesh, 1, 2), vf(mesh, 2, 2);
    const PressureSpace pc(mesh, 1, 2), pf(mesh, 2, 2);
    const auto t = build_h_space_transfer(vc, pc, vf, pf, 1);
    BlockVector xc(2, vc.n_dofs(), pc.n_dofs());
    for (int a = 0; a < 2; ++a)
      std::fill(xc.velocity(a), xc.velocity(a) + vc.n_dofs(), 3.25);
    const BlockVector xf = t.prolongate(xc);
    for (int a = 0; a < 2; ++a)
      for (Index i = 0; i < vf.n_dofs(); ++i)
        c.check(approx(xf.velocity(a)[i], 3.25, 1e-14), "constant");
    std::mt19937 rng(5);
    BlockVector yc(2, vc.n_dofs(), pc.n_dofs());
    yc.data = random_vector(yc.size(), rng);
    const BlockVector yf = t.prolongate(yc);
    std::uniform_real_distribution<double> dist(0.0, 1.0);
    for (int tr = 0; tr < 50; ++tr)
      {
        const double x = dist(rng), y = dist(rng);
        c.check(approx(evaluate_pressure(pf, yf.pressure(0), x, y), evaluate_pressure(pc, yc.pressure(0), x, y),
                       1e-12),
                "pressure exact");
        c.check(approx(evaluate_velocity(vf, yf.velocity(1), x, y, 1), evaluate_velocity(vc, yc.velocity(1), x, y, 1),
                       1e-12),
                "velocity exact");
      }
    BlockVector zf(2, vf.n_dofs(), pf.n_dofs());
    zf.data = random_vector(zf.size(), rng);
    c.check(approx(t.prolongate(yc).dot(zf), yc.dot(t.restrict_(zf)), 1e-13), "adjoint");
  }
  {
    Case c("restriction equals assembled transpose entrywise (test_transfer.cpp:72-99)");
    const VelocitySpace vc(mesh, 0, 1), vf(mesh, 1, 1);
    const PressureSpace pc(mesh, 0, 1), pf(mesh, 1, 1);
    const auto t = build_h_space_transfer(vc, pc, vf, pf, 0);
    const Index nc = vc.n_dofs() + pc.n_dofs(), nf = vf.n_dofs() + pf.n_dofs();
    Mat pm(static_cast<int>(nf), static_cast<int>(nc)), rm(static_cast<int>(nc), static_cast<int>(nf));
    for (Index j = 0; j < nc; ++j)
      {
        BlockVector e(1, vc.n_dofs(), pc.n_dofs());
        e.data[j] = 1.0;
        const auto o = t.prolongate(e);
        for (Index i = 0; i < nf; ++i)
          pm(static_cast<int>(i), static_cast<int>(j)) = o.data[i];
      }
    for (Index j = 0; j < nf; ++j)
      {
        BlockVector e(1, vf.n_dofs(), pf.n_dofs());
        e.data[j] = 1.0;
        const auto o = t.restrict_(e);
        for (Index i = 0; i < nc; ++i)
          rm(static_cast<int>(i), static_cast<int>(j)) = o.data[i];
      }
    double d = 0;
    for (Index i = 0; i < nc; ++i)
      for (Index j = 0; j < nf; ++j)
        d = std::max(d, std::abs(rm(static_cast<int>(i), static_cast<int>(j)) -
                                 pm(static_cast<int>(j), static_cast<int>(i))));
    c.check(d == 0.0, "R == P^T");
  }
  {
    Case c("pressure mean preservation; restrict_residual projects (test_transfer.cpp:122-146)");
    const VelocitySpace vc(mesh, 1, 1), vf(mesh, 2, 1);
    const PressureSpace pc(mesh, 1, 1), pf(mesh, 2, 1);
    const auto t = build_h_space_transfer(vc, pc, vf, pf, 1);
    std::mt19937 rng(7);
    BlockVector xc(2, vc.n_dofs(), pc.n_dofs());
    xc.data = random_vector(xc.size(), rng);
    const auto xf = t.prolongate(xc);
    for (int a = 0; a < 2; ++a)
      c.check(approx(pf.mean_integral(xf.pressure(a)), pc.mean_integral(xc.pressure(a)), 1e-13), "mean");
    BlockVector rf(2, vf.n_dofs(), pf.n_dofs());
    rf.data = random_vector(rf.size(), rng);
    const auto rc = t.restrict_residual(rf, true);
    for (int a = 0; a < 2; ++a)
      c.check(std::abs(pc.mean_integral(rc.pressure(a))) <
                1e-13 * norm(Vec(rc.pressure(a), rc.pressure(a) + pc.n_dofs())),
              "projected");
  }
  {
    Case c("p_space transfer exact, zero padding, degree check (test_transfer.cpp:148-188)");
    const VelocitySpace vc(mesh, 1, 1), vf(mesh, 1, 2);
    const PressureSpace pc(mesh, 1, 1), pf(mesh, 1, 2);
    const auto t = build_p_space_transfer(vc, pc, vf, pf, 1);
    std::mt19937 rng(9);
    BlockVector xc(2, vc.n_dofs(), pc.n_dofs());
    xc.data = random_vector(xc.size(), rng);
    const auto xf = t.prolongate(xc);
    std::uniform_real_distribution<double> dist(0.0, 1.0);
    for (int tr = 0; tr < 50; ++tr)
      {
        const double x = dist(rng), y = dist(rng);
        c.check(approx(evaluate_velocity(vf, xf.velocity(0), x, y, 0), evaluate_velocity(vc, xc.velocity(0), x, y, 0),
                       1e-12),
                "velocity");
        c.check(approx(evaluate_pressure(pf, xf.pressure(1), x, y), evaluate_pressure(pc, xc.pressure(1), x, y),
                       1e-12),
                "pressure");
      }
    int nz = 0;
    for (int cell = 0; cell < mesh.n_cells(1); ++cell)
      for (int l = 0; l < pf.dofs_per_cell(); ++l)
        {
          const auto &e = pf.basis().exponents(l);
          if (e[0] + e[1] > 1 && xf.pressure(0)[pf.cell_dof(cell, l)] != 0.0)
            ++nz;
        }
    c.check(nz == 0, "padding");
    c.check(throws([&] { build_p_space_transfer(vf, pf, vf, pf, 1); }), "degree check");
  }
  {
    Case c("p_time transfer reproduction and block structure (test_transfer.cpp:190-219)");
    const VelocitySpace vs(mesh, 1, 1);
    const PressureSpace ps(mesh, 1, 1);
    const auto t = build_p_time_transfer(1, 2, vs, ps);
    std::mt19937 rng(11);
    const Vec w = random_vector(vs.n_dofs(), rng);
    BlockVector xc(2, vs.n_dofs(), ps.n_dofs());
    std::copy(w.begin(), w.end(), xc.velocity(0));
    std::copy(w.begin(), w.end(), xc.velocity(1));
    const auto xf = t.prolongate(xc);
    for (int a = 0; a < 3; ++a)
      c.check(diffnorm(xf.velocity(a), w.data(), vs.n_dofs()) < 1e-13 * norm(w), "constant in time");
    const Vec cn = gauss_radau_right(2).points, fn = gauss_radau_right(3).points;
    BlockVector lin(2, vs.n_dofs(), ps.n_dofs());
    for (int b = 0; b < 2; ++b)
      for (Index i = 0; i < vs.n_dofs(); ++i)
        lin.velocity(b)[i] = cn[b] * w[i];
    const auto lf = t.prolongate(lin);
    for (int a = 0; a < 3; ++a)
      {
        Vec e(vs.n_dofs());
        for (Index i = 0; i < vs.n_dofs(); ++i)
          e[i] = fn[a] * w[i];
        c.check(diffnorm(lf.velocity(a), e.data(), vs.n_dofs()) < 1e-12 * norm(w), "linear in time");
      }
  }
  {
    Case c("identity transfer (test_transfer.cpp:221-229)");
    const VelocitySpace vs(mesh, 1, 1);
    const PressureSpace ps(mesh, 1, 1);
    const auto t = TransferPair::identity(vs, ps, 1);
    std::mt19937 rng(13);
    BlockVector x(2, vs.n_dofs(), ps.n_dofs());
    x.data = random_vector(x.size(), rng);
    c.check(t.prolongate(x).data == x.data && t.restrict_(x).data == x.data &&
              t.prolongate_correction(x, true).data == x.data,
            "unchanged");
  }
}

// ------------------------------------------------------------ hierarchy
void
suite_hierarchy()
{
  Case c("construct/combine hierarchies (test_hierarchy.cpp:9-80; acceptance.cpp:339-351)");
  const auto list = construct_hierarchy(0.125, 0.5, 2, 1);
  c.check(list.size() == 4 && list[0] == HpEntry{0.5, 1} && list[1] == HpEntry{0.25, 1} &&
            list[2] == HpEntry{0.125, 1} && list[3] == HpEntry{0.125, 2},
          "construct");
  const auto single = construct_hierarchy(0.125, 0.125, 1, 1);
  c.check(single.size() == 1, "single");
  const auto deg = construct_hierarchy(1.0, 1.0, 4, 1);
  c.check(deg.size() == 3 && deg[0] == HpEntry{1.0, 1} && deg[1] == HpEntry{1.0, 2} && deg[2] == HpEntry{1.0, 4},
          "degrees");
  c.check(throws([] { construct_hierarchy(1.0, 0.5, 2, 1); }) && throws([] { construct_hierarchy(0.5, 1.0, 1, 2); }),
          "throws");
  const auto lv = combine_hierarchies(list, construct_hierarchy(0.25, 0.25, 2, 1));
  c.check(lv.size() == 4 && lv[0].h == 0.5 && lv[0].r == 1 && lv[0].k == 1 && lv[1].h == 0.25 && lv[1].k == 2 &&
            lv[3].r == 2 && lv[3].k == 2,
          "combine");
  c.check(lv[1].kind_to_coarser == TransferKind::h_space_p_time && lv[2].kind_to_coarser == TransferKind::h_space &&
            lv[3].kind_to_coarser == TransferKind::p_space,
          "kinds");
}

// ------------------------------------------------------------ solver
Mat
random_matrix(int n, std::mt19937 &rng, double shift)
{
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  Mat m(n, n);
  for (int i = 0; i < n; ++i) // row-major draw order as Eigen loops in the test
    for (int j = 0; j < n; ++j)
      m(i, j) = dist(rng);
  for (int i = 0; i < n; ++i)
    m(i, i) += shift;
  return m;
}

BlockVector
wrap(const Vec &v)
{
  BlockVector b(1, static_cast<Index>(v.size()), 0);
  b.data = v;
  return b;
}

void
suite_solver()
{
  {
    Case c("gmres Krylov exactness + monotone history (test_solver.cpp:33-63)");
    std::mt19937 rng(3);
    const int n = 24;
    const Mat m = random_matrix(n, rng, 5.0);
    const Vec rhs = random_vector(n, rng);
    KrylovConfig cfg;
    cfg.rtol = 1e-12;
    const ApplyFn ap = [&](const BlockVector &x, BlockVector &y) { y.data = matvec(m, x.data); };
    const PrecondFn id = [](const BlockVector &r) { return r; };
    const auto res = gmres(ap, id, wrap(rhs), wrap(Vec(n, 0.0)), cfg);
    c.check(res.converged && res.iterations <= n, "converged");
    const Vec ax = matvec(m, res.x.data);
    c.check(diffnorm(ax.data(), rhs.data(), n) < 1e-11 * norm(rhs), "solution");
    for (size_t i = 1; i < res.residual_history.size(); ++i)
      c.check(res.residual_history[i] <= res.residual_history[i - 1] * (1 + 1e-12), "monotone");
  }
  {
    Case c("gmres exact-inverse preconditioner: 1 iteration (test_solver.cpp:65-87)");
    std::mt19937 rng(5);
    const int n = 17;
    const Mat m = random_matrix(n, rng, 4.0);
    const Mat inv = LU(m).inverse();
    const Vec rhs = random_vector(n, rng);
    KrylovConfig cfg;
    cfg.rtol = 1e-10;
    const ApplyFn ap = [&](const BlockVector &x, BlockVector &y) { y.data = matvec(m, x.data); };
    const PrecondFn pc = [&](const BlockVector &r) { return wrap(matvec(inv, r.data)); };
    const auto res = gmres(ap, pc, wrap(rhs), wrap(Vec(n, 0.0)), cfg);
    c.check(res.converged && res.iterations == 1, "iters " + std::to_string(res.iterations));
  }
  {
    Case c("coarse solver residual 1e-11 and mean zero (test_solver.cpp:118-150)");
    const Mesh mesh = Mesh::build_cartesian(unit, 1, 1, 2);
    const VelocitySpace vs(mesh, 0, 1);
    const PressureSpace ps(mesh, 0, 1);
    const auto tm = temporal_matrices(1, 0.25);
    const SpaceTimeBlockOperator op(vs, ps, tm, 0.1);
    const CoarseSolver coarse(op, 50000);
    std::mt19937 rng(11);
    BlockVector xt = op.make_vector();
    xt.data = random_vector(xt.size(), rng);
    for (int a = 0; a < 2; ++a)
      {
        vs.zero_constrained(xt.velocity(a));
        ps.project_mean_zero(xt.pressure(a));
      }
    BlockVector b = op.make_vector();
    op.apply_block(xt, b);
    const BlockVector x = coarse.solve(b);
    BlockVector res = op.make_vector();
    op.apply_block(x, res);
    res -= b;
    c.check(res.norm() < 1e-11 * b.norm(), "residual " + num(res.norm() / b.norm()));
    for (int a = 0; a < 2; ++a)
      c.check(std::abs(ps.mean_integral(x.pressure(a))) <
                1e-12 * (1.0 + norm(Vec(x.pressure(a), x.pressure(a) + ps.n_dofs()))),
              "mean");
  }
  {
    Case c("v_cycle single level = direct solve; zero->zero (test_solver.cpp:152-184)");
    const StokesProblem problem = manufactured_problem();
    RunConfig cfg;
    cfg.r = 1;
    cfg.refinements = 0;
    cfg.n_steps = 2;
    Setup setup = build_setup(problem, cfg);
    c.check(setup.levels.n_levels() == 1, "one level");
    const VCycle vc(setup.levels, cfg.mg);
    const auto &op = *setup.levels.finest().op;
    std::mt19937 rng(13);
    BlockVector b = op.make_vector();
    b.data = random_vector(b.size(), rng);
    for (int a = 0; a < b.ns; ++a)
      {
        setup.levels.finest().vspace->zero_constrained(b.velocity(a));
        setup.levels.finest().pspace->project_mean_zero(b.pressure(a));
      }
    const BlockVector x = vc.apply(b);
    BlockVector res = op.make_vector();
    op.apply_block(x, res);
    res -= b;
    c.check(res.norm() <= 1e-12 * b.norm(), "direct");
    c.check(vc.apply(op.make_vector()).norm() == 0.0, "zero");
  }
  {
    Case c("v_cycle linearity 1e-12 and contraction rho<1 (test_solver.cpp:186-245)");
    const StokesProblem problem = manufactured_problem();
    RunConfig cfg;
    cfg.r = 1;
    cfg.refinements = 2;
    cfg.n_steps = 4;
    Setup setup = build_setup(problem, cfg);
    const VCycle vc(setup.levels, cfg.mg);
    const auto &op = *setup.levels.finest().op;
    const auto &vs = *setup.levels.finest().vspace;
    std::mt19937 rng(17);
    const auto rnd = [&]() {
      BlockVector b = op.make_vector();
      b.data = random_vector(b.size(), rng);
      for (int a = 0; a < b.ns; ++a)
        vs.zero_constrained(b.velocity(a));
      return b;
    };
    const BlockVector a = rnd(), cc = rnd();
    BlockVector combo = a;
    combo *= 0.4;
    {
      BlockVector t = cc;
      t *= -2.3;
      combo += t;
    }
    BlockVector lhs = vc.apply(combo), va = vc.apply(a), vcc = vc.apply(cc);
    va *= 0.4;
    vcc *= -2.3;
    va += vcc;
    c.check(diffnorm(lhs.data.data(), va.data.data(), va.size()) < 1e-12 * va.norm(), "linearity");
    BlockVector e = rnd();
    for (int s = 0; s < e.ns; ++s)
      setup.levels.finest().pspace->project_mean_zero(e.pressure(s));
    double rho = 0;
    for (int it = 0; it < 30; ++it)
      {
        e *= 1.0 / e.norm();
        BlockVector se = op.make_vector();
        op.apply_block(e, se);
        BlockVector ce = vc.apply(se);
        BlockVector nx = e;
        nx -= ce;
        for (int s = 0; s < nx.ns; ++s)
          setup.levels.finest().pspace->project_mean_zero(nx.pressure(s));
        rho = nx.norm();
        e = nx;
      }
    c.check(rho < 1.0, "rho " + num(rho));
  }
  {
    Case c("time_march zero data: zero solution, zero iterations (test_solver.cpp:247-262)");
    const StokesProblem problem = manufactured_problem();
    RunConfig cfg;
    cfg.r = 1;
    cfg.refinements = 1;
    Setup setup = build_setup(problem, cfg);
    TimeMarchProblem zero;
    const auto res = time_march(setup.levels, zero, 4, cfg.mg, cfg.krylov);
    c.check(res.converged, "converged");
    for (const auto &x : res.trajectory)
      c.check(x.norm() == 0.0, "zero");
    for (const auto &s : res.steps)
      c.check(s.iterations == 0, "iters");
  }
  {
    Case c("time_march manufactured r=2 c=2: saddle-point health (test_solver.cpp:306-336)");
    const StokesProblem problem = manufactured_problem();
    RunConfig cfg;
    cfg.r = 2;
    cfg.refinements = 2;
    Setup setup = build_setup(problem, cfg);
    const auto res = time_march(setup.levels, problem.data, step_count(problem, cfg), cfg.mg, cfg.krylov);
    c.check(res.converged && res.avg_iterations > 0.0 && res.avg_iterations < 40.0,
            "avg iters " + num(res.avg_iterations));
    for (const auto &s : res.steps)
      {
        c.check(s.max_divergence <= 10.0 * cfg.krylov.rtol, "divergence " + num(s.max_divergence));
        c.check(s.max_pressure_mean <= 1e-10, "mean");
      }
  }
  {
    Case c("h-robustness r=2, c=1..3: avg iterations in [8,22] (acceptance.cpp:461-490)");
    const StokesProblem problem = manufactured_problem();
    double prev = 1e300;
    std::string iters;
    for (int cc = 1; cc <= 3; ++cc)
      {
        RunConfig cfg;
        cfg.r = 2;
        cfg.refinements = cc;
        Setup setup = build_setup(problem, cfg);
        const auto res =
          time_march(setup.levels, problem.data, step_count(problem, cfg), cfg.mg, cfg.krylov, false);
        iters += num(res.avg_iterations) + " ";
        c.check(res.avg_iterations >= 8.0 && res.avg_iterations <= 22.0, "band");
        c.check(res.avg_iterations <= prev + 2.0, "monotone");
        prev = res.avg_iterations;
      }
    c.detail += "iters " + iters;
  }
}

// ------------------------------------------------------------ acceptance Table 1
void
suite_acceptance_table1()
{
  Case c("Table 1 r=4, c=1..3 within factor 2, EOC +-0.3 (acceptance.cpp:383-420, PAPER.md:1033-1035)");
  const double ref_v[3] = {1.00279e-04, 2.32706e-06, 3.98114e-08};
  const double ref_p[3] = {1.14907e-03, 1.11534e-04, 3.58645e-06};
  const double ref_eoc[2] = {5.43, 5.87};
  const StokesProblem problem = manufactured_problem();
  double ev[3], ep[3];
  for (int cc = 1; cc <= 3; ++cc)
    {
      RunConfig cfg;
      cfg.r = 4;
      cfg.refinements = cc;
      cfg.krylov.rtol = 1e-10;
      cfg.krylov.max_iterations = 400;
      cfg.krylov.max_basis = 400;
      Setup setup = build_setup(problem, cfg);
      const auto march = time_march(setup.levels, problem.data, step_count(problem, cfg), cfg.mg, cfg.krylov);
      const auto err = compute_errors(setup, march, problem.exact);
      ev[cc - 1] = err.e_v_l2;
      ep[cc - 1] = err.e_p_l2;
      const double fv = err.e_v_l2 / ref_v[cc - 1], fp = err.e_p_l2 / ref_p[cc - 1];
      c.detail += "c" + std::to_string(cc) + ": e_v=" + num(err.e_v_l2) + " e_p=" + num(err.e_p_l2) +
                  " iters=" + num(march.avg_iterations) + "; ";
      c.check(fv > 0.5 && fv < 2.0 && fp > 0.5 && fp < 2.0, "value factor");
    }
  for (int cc = 2; cc <= 3; ++cc)
    {
      const double eo = std::log2(ev[cc - 2] / ev[cc - 1]);
      c.check(std::abs(eo - ref_eoc[cc - 2]) <= 0.3, "eoc " + num(eo));
    }
  (void)ep;
}

} // namespace

int
main(int argc, char **argv)
{
  const std::vector<std::pair<std::string, void (*)()>> suites = {
    {"quadrature", suite_quadrature}, {"time_basis", suite_time_basis}, {"mesh", suite_mesh},
    {"dof_space", suite_dof_space},   {"st_operator", suite_st_operator}, {"vanka", suite_vanka},
    {"transfer", suite_transfer},     {"hierarchy", suite_hierarchy},   {"solver", suite_solver},
    {"acceptance_table1", suite_acceptance_table1},
  };
  std::vector<std::string> want;
  for (int i = 1; i < argc; ++i)
    want.push_back(argv[i]);
  for (const auto &[name, fn] : suites)
    {
      const bool selected =
        want.empty() ? name != "acceptance_table1" : std::find(want.begin(), want.end(), name) != want.end();
      if (!selected)
        continue;
      g_suite = name;
      try
        {
          fn();
        }
      catch (const std::exception &e)
        {
          std::printf("[FAIL] %s: uncaught exception %s\n", name.c_str(), e.what());
          ++g_failures;
        }
    }
  std::printf("== %d failures ==\n", g_failures);
  return g_failures == 0 ? 0 : 1;
}
