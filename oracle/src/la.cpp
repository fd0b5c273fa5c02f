// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Dense linear algebra standing in for the Eigen calls of the reference.
#include "oracle/oracle.hpp"

#include <cmath>
#include <limits>

namespace oracle
{

Mat
matmul(const Mat &a, const Mat &b)
{
  if (a.c != b.r)
    throw std::invalid_argument("matmul: shape mismatch");
  Mat out(a.r, b.c);
  for (int j = 0; j < b.c; ++j)
    for (int k = 0; k < a.c; ++k)
      {
        const double bkj = b(k, j);
        for (int i = 0; i < a.r; ++i)
          out(i, j) += a(i, k) * bkj;
      }
  return out;
}

Mat
transpose(const Mat &a)
{
  Mat t(a.c, a.r);
  for (int j = 0; j < a.c; ++j)
    for (int i = 0; i < a.r; ++i)
      t(j, i) = a(i, j);
  return t;
}

LU::LU(const Mat &a) : n(a.r), lu(a), piv(a.r)
{
  if (a.r != a.c)
    throw std::invalid_argument("LU: matrix not square");
  for (int i = 0; i < n; ++i)
    piv[i] = i;
  for (int k = 0; k < n; ++k)
    {
      int p = k;
      double best = std::abs(lu(k, k));
      for (int i = k + 1; i < n; ++i)
        if (std::abs(lu(i, k)) > best)
          {
            best = std::abs(lu(i, k));
            p = i;
          }
      if (p != k)
        {
          for (int j = 0; j < n; ++j)
            std::swap(lu(k, j), lu(p, j));
          std::swap(piv[k], piv[p]);
        }
      const double pivot = lu(k, k);
      if (pivot == 0.0)
        {
          singular = true;
          continue;
        }
      for (int i = k + 1; i < n; ++i)
        lu(i, k) /= pivot;
      for (int j = k + 1; j < n; ++j)
        {
          const double ukj = lu(k, j);
          if (ukj == 0.0)
            continue;
          for (int i = k + 1; i < n; ++i)
            lu(i, j) -= lu(i, k) * ukj;
        }
    }
}

void
LU::solve_inplace(double *x) const
{
  Vec tmp(n);
  for (int i = 0; i < n; ++i)
    tmp[i] = x[piv[i]];
  for (int j = 0; j < n; ++j) // forward, unit lower
    {
      const double v = tmp[j];
      if (v != 0.0)
        for (int i = j + 1; i < n; ++i)
          tmp[i] -= lu(i, j) * v;
    }
  for (int j = n - 1; j >= 0; --j) // backward, upper
    {
      tmp[j] /= lu(j, j);
      const double v = tmp[j];
      if (v != 0.0)
        for (int i = 0; i < j; ++i)
          tmp[i] -= lu(i, j) * v;
    }
  for (int i = 0; i < n; ++i)
    x[i] = tmp[i];
}

Vec
LU::solve(const Vec &b) const
{
  Vec x = b;
  solve_inplace(x.data());
  return x;
}

Mat
LU::inverse() const
{
  Mat inv(n, n);
  Vec col(n);
  for (int j = 0; j < n; ++j)
    {
      std::fill(col.begin(), col.end(), 0.0);
      col[j] = 1.0;
      solve_inplace(col.data());
      for (int i = 0; i < n; ++i)
        inv(i, j) = col[i];
    }
  return inv;
}

double
LU::rcond(const Mat &a) const
{
  if (singular)
    return 0.0;
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(lu(i, i)))
      return 0.0;
  const auto norm1 = [](const Mat &m) {
    double best = 0.0;
    for (int j = 0; j < m.c; ++j)
      {
        double s = 0.0;
        for (int i = 0; i < m.r; ++i)
          s += std::abs(m(i, j));
        best = std::max(best, s);
      }
    return best;
  };
  const Mat inv = inverse();
  const double ni = norm1(inv);
  if (!std::isfinite(ni) || ni == 0.0)
    return 0.0;
  return 1.0 / (norm1(a) * ni);
}

// One-sided Jacobi SVD: A V = U S. Returns the pseudo-inverse V S^+ U^T.
MinNormSolver::MinNormSolver(const Mat &a) : n(a.c)
{
  const int m = a.r;
  Mat u = a;
  Mat v(n, n);
  for (int i = 0; i < n; ++i)
    v(i, i) = 1.0;
  const double eps = std::numeric_limits<double>::epsilon();
  for (int sweep = 0; sweep < 60; ++sweep)
    {
      double off = 0.0;
      for (int p = 0; p < n - 1; ++p)
        for (int q = p + 1; q < n; ++q)
          {
            double alpha = 0.0, beta = 0.0, gamma = 0.0;
            for (int i = 0; i < m; ++i)
              {
                alpha += u(i, p) * u(i, p);
                beta += u(i, q) * u(i, q);
                gamma += u(i, p) * u(i, q);
              }
            if (gamma == 0.0)
              continue;
            const double conv = std::abs(gamma) / std::sqrt(alpha * beta);
            if (!(conv > eps))
              continue;
            off = std::max(off, conv);
            const double zeta = (beta - alpha) / (2.0 * gamma);
            const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
            const double c = 1.0 / std::sqrt(1.0 + t * t);
            const double s = c * t;
            for (int i = 0; i < m; ++i)
              {
                const double up = u(i, p), uq = u(i, q);
                u(i, p) = c * up - s * uq;
                u(i, q) = s * up + c * uq;
              }
            for (int i = 0; i < n; ++i)
              {
                const double vp = v(i, p), vq = v(i, q);
                v(i, p) = c * vp - s * vq;
                v(i, q) = s * vp + c * vq;
              }
          }
      if (off <= eps)
        break;
    }
  Vec sigma(n);
  double smax = 0.0;
  for (int j = 0; j < n; ++j)
    {
      double s = 0.0;
      for (int i = 0; i < m; ++i)
        s += u(i, j) * u(i, j);
      sigma[j] = std::sqrt(s);
      smax = std::max(smax, sigma[j]);
    }
  const double thresh = smax * eps * std::max(m, n);
  pinv = Mat(n, m);
  rank = 0;
  for (int j = 0; j < n; ++j)
    {
      if (!(sigma[j] > thresh))
        continue;
      ++rank;
      const double inv_s2 = 1.0 / (sigma[j] * sigma[j]); // u(:,j) = sigma_j * U_j
      for (int col = 0; col < m; ++col)
        {
          const double ucj = u(col, j) * inv_s2;
          for (int row = 0; row < n; ++row)
            pinv(row, col) += v(row, j) * ucj;
        }
    }
}

Vec
MinNormSolver::solve(const Vec &b) const
{
  Vec x(n, 0.0);
  for (int j = 0; j < pinv.c; ++j)
    for (int i = 0; i < n; ++i)
      x[i] += pinv(i, j) * b[j];
  return x;
}

// Implicit symmetric QL with Wilkinson shifts on a tridiagonal matrix,
// accumulating the full eigenvector matrix (n is tiny here).
void
tridiag_eigen(const Vec &diag, const Vec &offdiag, Vec &evals, Vec &first_comp)
{
  const int n = static_cast<int>(diag.size());
  Vec d = diag, e(n, 0.0);
  for (int i = 0; i + 1 < n; ++i)
    e[i] = offdiag[i];
  Mat z(n, n);
  for (int i = 0; i < n; ++i)
    z(i, i) = 1.0;
  for (int l = 0; l < n; ++l)
    {
      int iter = 0;
      int m;
      do
        {
          for (m = l; m < n - 1; ++m)
            {
              const double dd = std::abs(d[m]) + std::abs(d[m + 1]);
              if (std::abs(e[m]) <= std::numeric_limits<double>::epsilon() * dd)
                break;
            }
          if (m != l)
            {
              if (++iter > 200)
                throw std::runtime_error("tridiag_eigen: no convergence");
              double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
              double r = std::hypot(g, 1.0);
              g = d[m] - d[l] + e[l] / (g + (g >= 0 ? std::abs(r) : -std::abs(r)));
              double s = 1.0, c = 1.0, p = 0.0;
              int i;
              for (i = m - 1; i >= l; --i)
                {
                  double f = s * e[i];
                  const double b = c * e[i];
                  r = std::hypot(f, g);
                  e[i + 1] = r;
                  if (r == 0.0)
                    {
                      d[i + 1] -= p;
                      e[m] = 0.0;
                      break;
                    }
                  s = f / r;
                  c = g / r;
                  g = d[i + 1] - p;
                  r = (d[i] - g) * s + 2.0 * c * b;
                  p = s * r;
                  d[i + 1] = g + p;
                  g = c * r - b;
                  for (int k = 0; k < n; ++k)
                    {
                      f = z(k, i + 1);
                      z(k, i + 1) = s * z(k, i) + c * f;
                      z(k, i) = c * z(k, i) - s * f;
                    }
                }
              if (r == 0.0 && i >= l)
                continue;
              d[l] -= p;
              e[l] = g;
              e[m] = 0.0;
            }
        }
      while (m != l);
    }
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i)
    order[i] = i;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return d[a] < d[b]; });
  evals.resize(n);
  first_comp.resize(n);
  for (int i = 0; i < n; ++i)
    {
      evals[i] = d[order[i]];
      first_comp[i] = z(0, order[i]);
    }
}

} // namespace oracle
