// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Restates quadrature.cpp, basis1d.cpp, pdisc.cpp and time_basis.cpp.
#include "oracle/oracle.hpp"

#include <cmath>

namespace oracle
{

namespace
{
  // quadrature.cpp:16-39 (Golub-Welsch).
  QuadratureRule
  golub_welsch(const Vec &diag, const Vec &offdiag, double mu0)
  {
    QuadratureRule rule;
    Vec first;
    tridiag_eigen(diag, offdiag, rule.points, first);
    rule.weights.resize(rule.points.size());
    for (size_t i = 0; i < first.size(); ++i)
      rule.weights[i] = mu0 * first[i] * first[i];
    return rule;
  }

  // quadrature.cpp:41-50: beta_k = k^2/(4k^2-1), k = 1..n-1.
  Vec
  legendre_beta(int n)
  {
    Vec beta(std::max(n - 1, 0));
    for (int k = 1; k < n; ++k)
      beta[k - 1] = static_cast<double>(k) * k / (4.0 * k * k - 1.0);
    return beta;
  }

  Vec
  sqrt_all(Vec v)
  {
    for (double &x : v)
      x = std::sqrt(x);
    return v;
  }
} // namespace

QuadratureRule
gauss_rule(int n)
{
  if (n < 1)
    throw std::invalid_argument("gauss_rule: n must be >= 1");
  if (n == 1)
    return QuadratureRule{{0.0}, {2.0}};
  return golub_welsch(Vec(n, 0.0), sqrt_all(legendre_beta(n)), 2.0);
}

QuadratureRule
gauss_radau_right(int n)
{
  if (n < 1)
    throw std::invalid_argument("gauss_radau_right: n must be >= 1");
  if (n == 1)
    return QuadratureRule{{1.0}, {2.0}};
  // quadrature.cpp:81-92: modified last diagonal entry puts +1 in the spectrum.
  const Vec beta = legendre_beta(n);
  double pi_prev = 1.0, pi_cur = 1.0;
  for (int k = 1; k < n - 1; ++k)
    {
      const double pi_next = pi_cur - beta[k - 1] * pi_prev;
      pi_prev = pi_cur;
      pi_cur = pi_next;
    }
  Vec diag(n, 0.0);
  diag[n - 1] = 1.0 - beta[n - 2] * pi_prev / pi_cur;
  QuadratureRule rule = golub_welsch(diag, sqrt_all(beta), 2.0);
  rule.points[n - 1] = 1.0; // quadrature.cpp:97-98
  return rule;
}

Vec
gauss_lobatto_points(int n)
{
  if (n < 2)
    throw std::invalid_argument("gauss_lobatto_points: n must be >= 2");
  Vec nodes(n);
  nodes[0] = -1.0;
  nodes[n - 1] = 1.0;
  const int n_int = n - 2;
  if (n_int > 0)
    {
      // Jacobi(1,1) Gauss nodes, quadrature.cpp:112-123.
      Vec beta(std::max(n_int - 1, 0));
      for (int k = 1; k < n_int; ++k)
        beta[k - 1] = static_cast<double>(k) * (k + 2) / ((2.0 * k + 1) * (2.0 * k + 3));
      const QuadratureRule interior = golub_welsch(Vec(n_int, 0.0), sqrt_all(beta), 4.0 / 3.0);
      for (int i = 0; i < n_int; ++i)
        nodes[1 + i] = interior.points[i];
    }
  for (int i = 0; i < n / 2; ++i) // quadrature.cpp:125-131
    {
      const double v = 0.5 * (nodes[i] - nodes[n - 1 - i]);
      nodes[i] = v;
      nodes[n - 1 - i] = -v;
    }
  if (n % 2 == 1)
    nodes[n / 2] = 0.0;
  return nodes;
}

// ---------------------------------------------------------------- basis1d.cpp
NodalBasis1D::NodalBasis1D(Vec nodes) : nodes_(std::move(nodes))
{
  if (nodes_.empty())
    throw std::invalid_argument("NodalBasis1D: empty node set");
  for (size_t i = 0; i + 1 < nodes_.size(); ++i)
    if (!(nodes_[i] < nodes_[i + 1]))
      throw std::invalid_argument("NodalBasis1D: nodes must be strictly increasing");
}

double
NodalBasis1D::value(int i, double x) const
{
  double v = 1.0;
  for (int j = 0; j < size(); ++j)
    if (j != i)
      v *= (x - nodes_[j]) / (nodes_[i] - nodes_[j]);
  return v;
}

double
NodalBasis1D::derivative(int i, double x) const
{
  double d = 0.0;
  for (int m = 0; m < size(); ++m)
    {
      if (m == i)
        continue;
      double term = 1.0 / (nodes_[i] - nodes_[m]);
      for (int j = 0; j < size(); ++j)
        if (j != i && j != m)
          term *= (x - nodes_[j]) / (nodes_[i] - nodes_[j]);
      d += term;
    }
  return d;
}

Vec
NodalBasis1D::values(double x) const
{
  Vec v(size());
  for (int i = 0; i < size(); ++i)
    v[i] = value(i, x);
  return v;
}

Vec
NodalBasis1D::derivatives(double x) const
{
  Vec v(size());
  for (int i = 0; i < size(); ++i)
    v[i] = derivative(i, x);
  return v;
}

Mat
NodalBasis1D::value_table(const Vec &pts) const
{
  Mat t(static_cast<int>(pts.size()), size());
  for (size_t q = 0; q < pts.size(); ++q)
    for (int i = 0; i < size(); ++i)
      t(static_cast<int>(q), i) = value(i, pts[q]);
  return t;
}

Mat
NodalBasis1D::derivative_table(const Vec &pts) const
{
  Mat t(static_cast<int>(pts.size()), size());
  for (size_t q = 0; q < pts.size(); ++q)
    for (int i = 0; i < size(); ++i)
      t(static_cast<int>(q), i) = derivative(i, pts[q]);
  return t;
}

// ---------------------------------------------------------------- pdisc.cpp
Vec
legendre_values(int n, double x)
{
  Vec v(n + 1);
  v[0] = 1.0;
  if (n >= 1)
    v[1] = x;
  for (int k = 1; k < n; ++k)
    v[k + 1] = ((2.0 * k + 1) * x * v[k] - k * v[k - 1]) / (k + 1);
  return v;
}

Vec
legendre_derivatives(int n, double x)
{
  const Vec v = legendre_values(n, x);
  Vec d(n + 1);
  d[0] = 0.0;
  if (n >= 1)
    d[1] = 1.0;
  for (int k = 1; k < n; ++k)
    d[k + 1] = (2.0 * k + 1) * v[k] + d[k - 1];
  return d;
}

PDiscBasis::PDiscBasis(int r, int dim) : r_(r), dim_(dim)
{
  if (r < 1)
    throw std::invalid_argument("PDiscBasis: degree r must be >= 1");
  if (dim != 2 && dim != 3)
    throw std::invalid_argument("PDiscBasis: dim must be 2 or 3");
  for (int deg = 0; deg <= r; ++deg) // degree-major, pdisc.cpp:41-55
    {
      if (dim == 2)
        for (int a = deg; a >= 0; --a)
          exps_.push_back({a, deg - a, 0});
      else
        for (int a = deg; a >= 0; --a)
          for (int b = deg - a; b >= 0; --b)
            exps_.push_back({a, b, deg - a - b});
    }
}

double
PDiscBasis::value(int l, const double *xi) const
{
  const auto &e = exps_[l];
  double v = 1.0;
  for (int d = 0; d < dim_; ++d)
    v *= legendre_values(e[d], xi[d])[e[d]];
  return v;
}

void
PDiscBasis::gradient(int l, const double *xi, double *g) const
{
  const auto &e = exps_[l];
  double vals[3], ders[3];
  for (int d = 0; d < dim_; ++d)
    {
      vals[d] = legendre_values(e[d], xi[d])[e[d]];
      ders[d] = legendre_derivatives(e[d], xi[d])[e[d]];
    }
  for (int d = 0; d < dim_; ++d)
    {
      double v = ders[d];
      for (int c = 0; c < dim_; ++c)
        if (c != d)
          v *= vals[c];
      g[d] = v;
    }
}

double
PDiscBasis::gram_diagonal(int l) const
{
  const auto &e = exps_[l];
  double v = 1.0;
  for (int d = 0; d < dim_; ++d)
    v *= 2.0 / (2.0 * e[d] + 1.0);
  return v;
}

// ---------------------------------------------------------------- time_basis.cpp
TemporalMatrices
temporal_matrices(int k, double tau)
{
  if (k < 0)
    throw std::invalid_argument("temporal_matrices: k must be >= 0");
  if (!(tau > 0.0))
    throw std::invalid_argument("temporal_matrices: tau must be positive");
  const int n = k + 1;
  const QuadratureRule radau = gauss_radau_right(n);
  const NodalBasis1D basis(radau.points);
  TemporalMatrices tm;
  tm.k = k;
  tm.tau = tau;
  tm.nodes = radau.points;
  tm.weights = radau.weights;
  const Mat phi = basis.value_table(radau.points);
  const Mat dphi = basis.derivative_table(radau.points);
  tm.mass = Mat(n, n);
  tm.dt_plus_jump = Mat(n, n);
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < n; ++b)
      {
        double m = 0.0, kd = 0.0;
        for (int q = 0; q < n; ++q)
          {
            m += radau.weights[q] * phi(q, b) * phi(q, a);
            kd += radau.weights[q] * dphi(q, b) * phi(q, a);
          }
        tm.mass(a, b) = 0.5 * tau * m;
        tm.dt_plus_jump(a, b) = kd;
      }
  tm.left_values = basis.values(-1.0);
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < n; ++b)
      tm.dt_plus_jump(a, b) += tm.left_values[b] * tm.left_values[a];
  tm.coupling = Mat(n, n);
  for (int a = 0; a < n; ++a)
    tm.coupling(a, n - 1) = tm.left_values[a];
  return tm;
}

double
dg_ode_step(int k, double tau, double lambda, double y_prev)
{
  const TemporalMatrices tm = temporal_matrices(k, tau);
  const int n = k + 1;
  Mat sys(n, n);
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < n; ++b)
      sys(a, b) = tm.dt_plus_jump(a, b) - lambda * tm.mass(a, b);
  Vec rhs(n);
  for (int a = 0; a < n; ++a)
    rhs[a] = tm.coupling(a, n - 1) * y_prev;
  const LU lu(sys);
  if (lu.singular)
    throw std::runtime_error("dg_ode_step: singular temporal system");
  return lu.solve(rhs)[n - 1];
}

} // namespace oracle
