// Host setup for the B200 hp-STMG path (see setup.hpp).
#include "setup.hpp"

#include <algorithm>
#include <cmath>
#include <complex>
#include <limits>
#include <map>
#include <stdexcept>
#include <unordered_map>

namespace stmg_b200
{

// ================================================================ 1D numerics
double
legendre(int n, double x)
{
  if (n == 0)
    return 1.0;
  double p0 = 1.0, p1 = x;
  for (int k = 1; k < n; ++k)
    {
      const double p2 = ((2.0 * k + 1.0) * x * p1 - k * p0) / (k + 1.0);
      p0 = p1;
      p1 = p2;
    }
  return p1;
}

double
legendre_deriv(int n, double x)
{
  // P'_n = sum_{j = n-1, n-3, ...} (2j+1) P_j
  double d = 0.0;
  for (int j = n - 1; j >= 0; j -= 2)
    d += (2.0 * j + 1.0) * legendre(j, x);
  return d;
}

namespace
{
  // All simple roots of f in the open interval (lo, hi): sign-change scan on
  // a fine grid, then bisection to machine precision.
  template <class F>
  std::vector<double>
  bracket_roots(F &&f, double lo, double hi, int expected)
  {
    std::vector<double> roots;
    const int grid = 4000;
    double xa = lo, fa = f(lo);
    for (int i = 1; i <= grid; ++i)
      {
        const double xb = lo + (hi - lo) * i / grid;
        const double fb = f(xb);
        if (fa == 0.0 && xa > lo)
          roots.push_back(xa);
        else if ((fa < 0.0 && fb > 0.0) || (fa > 0.0 && fb < 0.0))
          {
            double a = xa, b = xb, fA = fa;
            for (int it = 0; it < 200; ++it)
              {
                const double m = 0.5 * (a + b);
                if (m <= a || m >= b)
                  break;
                const double fm = f(m);
                if (fm == 0.0)
                  {
                    a = b = m;
                    break;
                  }
                if ((fm < 0.0) == (fA < 0.0))
                  {
                    a = m;
                    fA = fm;
                  }
                else
                  b = m;
              }
            roots.push_back(0.5 * (a + b));
          }
        xa = xb;
        fa = fb;
      }
    if (static_cast<int>(roots.size()) != expected)
      throw std::runtime_error("bracket_roots: unexpected root count");
    return roots;
  }

  void
  symmetrize(std::vector<double> &x)
  {
    const int n = static_cast<int>(x.size());
    for (int i = 0; i < n / 2; ++i)
      {
        const double v = 0.5 * (x[i] - x[n - 1 - i]);
        x[i] = v;
        x[n - 1 - i] = -v;
      }
    if (n % 2 == 1)
      x[n / 2] = 0.0;
  }
} // namespace

Rule1D
gauss_legendre(int n)
{
  if (n < 1)
    throw std::invalid_argument("gauss_legendre: n must be >= 1");
  Rule1D r;
  r.x = bracket_roots([n](double x) { return legendre(n, x); }, -1.0, 1.0, n);
  symmetrize(r.x);
  for (double x : r.x)
    {
      const double d = legendre_deriv(n, x);
      r.w.push_back(2.0 / ((1.0 - x * x) * d * d));
    }
  return r;
}

Rule1D
gauss_radau_right(int n)
{
  if (n < 1)
    throw std::invalid_argument("gauss_radau_right: n must be >= 1");
  Rule1D r;
  if (n == 1)
    {
      r.x = {1.0};
      r.w = {2.0};
      return r;
    }
  // Interior nodes: roots of P_{n-1} - P_n in (-1, 1); the endpoint +1 is a root too.
  r.x = bracket_roots([n](double x) { return legendre(n - 1, x) - legendre(n, x); }, -1.0, 1.0 - 1e-12, n - 1);
  for (double x : r.x)
    {
      const double p = legendre(n - 1, x);
      r.w.push_back((1.0 + x) / (static_cast<double>(n) * n * p * p));
    }
  r.x.push_back(1.0);
  r.w.push_back(2.0 / (static_cast<double>(n) * n));
  return r;
}

std::vector<double>
gauss_lobatto(int n)
{
  if (n < 2)
    throw std::invalid_argument("gauss_lobatto: n must be >= 2");
  std::vector<double> x{-1.0};
  if (n > 2)
    {
      const auto in = bracket_roots([n](double t) { return legendre_deriv(n - 1, t); }, -1.0 + 1e-14, 1.0 - 1e-14, n - 2);
      x.insert(x.end(), in.begin(), in.end());
    }
  x.push_back(1.0);
  symmetrize(x);
  return x;
}

double
lagrange(const std::vector<double> &nodes, int i, double x)
{
  double v = 1.0;
  for (int j = 0; j < static_cast<int>(nodes.size()); ++j)
    if (j != i)
      v *= (x - nodes[j]) / (nodes[i] - nodes[j]);
  return v;
}

double
lagrange_deriv(const std::vector<double> &nodes, int i, double x)
{
  double d = 0.0;
  const int n = static_cast<int>(nodes.size());
  for (int m = 0; m < n; ++m)
    {
      if (m == i)
        continue;
      double t = 1.0 / (nodes[i] - nodes[m]);
      for (int j = 0; j < n; ++j)
        if (j != i && j != m)
          t *= (x - nodes[j]) / (nodes[i] - nodes[j]);
      d += t;
    }
  return d;
}

TimeTables
time_tables(int k, double tau)
{
  if (k < 0 || k >= kMaxS)
    throw std::invalid_argument("time_tables: k out of range");
  if (!(tau > 0.0))
    throw std::invalid_argument("time_tables: tau must be positive");
  const int s = k + 1;
  const Rule1D rad = gauss_radau_right(s);
  TimeTables t;
  t.k = k;
  t.tau = tau;
  t.nodes = rad.x;
  t.weights = rad.w;
  t.Kt.assign(s * s, 0.0);
  t.Mt.assign(s * s, 0.0);
  t.lv.resize(s);
  for (int a = 0; a < s; ++a)
    t.lv[a] = lagrange(rad.x, a, -1.0);
  for (int a = 0; a < s; ++a)
    for (int b = 0; b < s; ++b)
      {
        double m = 0.0, kd = 0.0;
        for (int q = 0; q < s; ++q)
          {
            const double pa = lagrange(rad.x, a, rad.x[q]);
            m += rad.w[q] * lagrange(rad.x, b, rad.x[q]) * pa;
            kd += rad.w[q] * lagrange_deriv(rad.x, b, rad.x[q]) * pa;
          }
        t.Mt[a * s + b] = 0.5 * tau * m;
        t.Kt[a * s + b] = kd + t.lv[b] * t.lv[a];
      }
  return t;
}

// ---------------------------------------------------------------- temporal eigen
namespace
{
  using cplx = std::complex<double>;

  // null vector of the complex S x S matrix A (rank S-1), full pivoting
  std::vector<cplx>
  null_vector(std::vector<cplx> A, int n)
  {
    std::vector<int> colp(n);
    for (int j = 0; j < n; ++j)
      colp[j] = j;
    int rank = 0;
    for (int k = 0; k < n; ++k)
      {
        int pi = -1, pj = -1;
        double best = 0.0;
        for (int i = k; i < n; ++i)
          for (int j = k; j < n; ++j)
            if (std::abs(A[i * n + j]) > best)
              {
                best = std::abs(A[i * n + j]);
                pi = i;
                pj = j;
              }
        if (best < 1e-11)
          break;
        for (int j = 0; j < n; ++j)
          std::swap(A[k * n + j], A[pi * n + j]);
        for (int i = 0; i < n; ++i)
          std::swap(A[i * n + k], A[i * n + pj]);
        std::swap(colp[k], colp[pj]);
        for (int i = k + 1; i < n; ++i)
          {
            const cplx f = A[i * n + k] / A[k * n + k];
            for (int j = k; j < n; ++j)
              A[i * n + j] -= f * A[k * n + j];
          }
        ++rank;
      }
    // back substitution with the free variables rank..n-1 = (1, 0, ...)
    std::vector<cplx> y(n, 0.0);
    if (rank < n)
      y[rank] = 1.0;
    for (int k = rank - 1; k >= 0; --k)
      {
        cplx t = 0.0;
        for (int j = k + 1; j < n; ++j)
          t += A[k * n + j] * y[j];
        y[k] = -t / A[k * n + k];
      }
    std::vector<cplx> v(n);
    for (int j = 0; j < n; ++j)
      v[colp[j]] = y[j];
    return v;
  }
} // namespace

TemporalEigen
temporal_eigen(const TimeTables &T)
{
  TemporalEigen e;
  const int S = T.k + 1;
  e.S = S;
  // Q = M_t^{-1} K_t
  std::vector<double> Minv = T.Mt;
  double rc = 0.0;
  if (!invert_dense(Minv, S, &rc))
    return e;
  std::vector<double> Q(S * S, 0.0);
  for (int i = 0; i < S; ++i)
    for (int j = 0; j < S; ++j)
      for (int l = 0; l < S; ++l)
        Q[i * S + j] += Minv[i * S + l] * T.Kt[l * S + j];
  // characteristic polynomial (Faddeev-LeVerrier): p(x) = sum_j c[j] x^j
  std::vector<double> c(S + 1, 0.0), Mk(S * S, 0.0), QM(S * S);
  c[S] = 1.0;
  for (int k = 1; k <= S; ++k)
    {
      for (int i = 0; i < S; ++i)
        for (int j = 0; j < S; ++j)
          {
            double t = 0.0;
            for (int l = 0; l < S; ++l)
              t += Q[i * S + l] * Mk[l * S + j];
            QM[i * S + j] = t;
          }
      for (int i = 0; i < S; ++i)
        for (int j = 0; j < S; ++j)
          Mk[i * S + j] = QM[i * S + j] + (i == j ? c[S - k + 1] : 0.0);
      double tr = 0.0;
      for (int i = 0; i < S; ++i)
        for (int l = 0; l < S; ++l)
          tr += Q[i * S + l] * Mk[l * S + i];
      c[S - k] = -tr / k;
    }
  const auto poly = [&](cplx x) {
    cplx r = c[S];
    for (int j = S - 1; j >= 0; --j)
      r = r * x + c[j];
    return r;
  };
  const auto dpoly = [&](cplx x) {
    cplx r = S * c[S];
    for (int j = S - 1; j >= 1; --j)
      r = r * x + static_cast<double>(j) * c[j];
    return r;
  };
  // roots: Durand-Kerner, then Newton polishing
  double scale = 0.0;
  for (int j = 0; j < S; ++j)
    scale = std::max(scale, std::abs(c[j]));
  std::vector<cplx> z(S);
  for (int i = 0; i < S; ++i)
    z[i] = std::pow(cplx(0.4, 0.9), i) * (1.0 + scale);
  for (int it = 0; it < 2000; ++it)
    {
      double moved = 0.0;
      for (int i = 0; i < S; ++i)
        {
          cplx den = 1.0;
          for (int j = 0; j < S; ++j)
            if (j != i)
              den *= z[i] - z[j];
          const cplx dz = poly(z[i]) / den;
          z[i] -= dz;
          moved = std::max(moved, std::abs(dz));
        }
      if (moved < 1e-15 * (1.0 + scale))
        break;
    }
  for (auto &x : z)
    for (int it = 0; it < 3; ++it)
      {
        const cplx d = dpoly(x);
        if (std::abs(d) > 0.0)
          x -= poly(x) / d;
      }
  // group: real roots, and pairs (one representative with Im > 0)
  std::vector<cplx> reps;
  std::vector<bool> used(S, false);
  for (int i = 0; i < S; ++i)
    {
      if (used[i])
        continue;
      used[i] = true;
      if (std::abs(z[i].imag()) <= 1e-9 * (1.0 + std::abs(z[i])))
        {
          reps.push_back(cplx(z[i].real(), 0.0));
          continue;
        }
      int partner = -1;
      for (int j = 0; j < S; ++j)
        if (!used[j] && std::abs(z[j] - std::conj(z[i])) <= 1e-7 * (1.0 + std::abs(z[i])))
          partner = j;
      if (partner < 0)
        return e; // not a real matrix spectrum: leave e.ok = false
      used[partner] = true;
      reps.push_back(z[i].imag() > 0 ? z[i] : std::conj(z[i]));
    }
  e.V.assign(S * S, 0.0);
  int col = 0;
  for (const cplx lam : reps)
    {
      std::vector<cplx> A(S * S);
      for (int i = 0; i < S; ++i)
        for (int j = 0; j < S; ++j)
          A[i * S + j] = Q[i * S + j] - (i == j ? lam : cplx(0.0));
      std::vector<cplx> v = null_vector(A, S);
      double nrm = 0.0;
      for (const auto &x : v)
        nrm = std::max(nrm, std::abs(x));
      for (auto &x : v)
        x /= nrm;
      e.blk_c0.push_back(col);
      e.alpha.push_back(lam.real());
      if (lam.imag() == 0.0)
        {
          e.blk_sz.push_back(1);
          e.beta.push_back(0.0);
          for (int i = 0; i < S; ++i)
            e.V[i * S + col] = v[i].real();
          col += 1;
        }
      else
        {
          e.blk_sz.push_back(2);
          e.beta.push_back(lam.imag());
          for (int i = 0; i < S; ++i)
            {
              e.V[i * S + col] = v[i].real();
              e.V[i * S + col + 1] = v[i].imag();
            }
          col += 2;
        }
    }
  if (col != S)
    return e;
  // verify Q V = V Lambda, then W = V^{-1} M_t^{-1}
  double res = 0.0, qn = 0.0;
  for (int i = 0; i < S * S; ++i)
    qn = std::max(qn, std::abs(Q[i]));
  for (size_t b = 0; b < e.blk_c0.size(); ++b)
    {
      const int c0 = e.blk_c0[b];
      for (int i = 0; i < S; ++i)
        for (int cc = 0; cc < e.blk_sz[b]; ++cc)
          {
            double qv = 0.0;
            for (int l = 0; l < S; ++l)
              qv += Q[i * S + l] * e.V[l * S + c0 + cc];
            double vl;
            if (e.blk_sz[b] == 1)
              vl = e.V[i * S + c0] * e.alpha[b];
            else if (cc == 0) // Q x = alpha x - beta y
              vl = e.alpha[b] * e.V[i * S + c0] - e.beta[b] * e.V[i * S + c0 + 1];
            else // Q y = beta x + alpha y
              vl = e.beta[b] * e.V[i * S + c0] + e.alpha[b] * e.V[i * S + c0 + 1];
            res = std::max(res, std::abs(qv - vl));
          }
    }
  if (res > 1e-10 * (1.0 + qn))
    return e;
  std::vector<double> Vinv = e.V;
  if (!invert_dense(Vinv, S, &rc) || rc < 1e-10)
    return e;
  e.W.assign(S * S, 0.0);
  for (int i = 0; i < S; ++i)
    for (int j = 0; j < S; ++j)
      for (int l = 0; l < S; ++l)
        e.W[i * S + j] += Vinv[i * S + l] * Minv[l * S + j];
  e.ok = true;
  return e;
}

Factors1D
factors_1d(int r)
{
  if (r < 1 || r + 2 > kMaxN1)
    throw std::invalid_argument("factors_1d: r out of supported range 1..4");
  Factors1D f;
  f.r = r;
  f.n1 = r + 2;
  f.P = r + 1;
  f.nodes = gauss_lobatto(f.n1);
  const Rule1D g = gauss_legendre(f.n1 + 1); // exact for all products below
  const int n = f.n1;
  f.M1.assign(n * n, 0.0);
  f.K1.assign(n * n, 0.0);
  f.C1.assign(n * n, 0.0);
  f.Lm.assign(f.P * n, 0.0);
  f.Lc.assign(f.P * n, 0.0);
  for (size_t q = 0; q < g.x.size(); ++q)
    {
      std::vector<double> v(n), d(n);
      for (int i = 0; i < n; ++i)
        {
          v[i] = lagrange(f.nodes, i, g.x[q]);
          d[i] = lagrange_deriv(f.nodes, i, g.x[q]);
        }
      for (int i = 0; i < n; ++i)
        for (int k = 0; k < n; ++k)
          {
            f.M1[i * n + k] += g.w[q] * v[i] * v[k];
            f.K1[i * n + k] += g.w[q] * d[i] * d[k];
            f.C1[i * n + k] += g.w[q] * d[i] * v[k];
          }
      for (int a = 0; a < f.P; ++a)
        {
          const double la = legendre(a, g.x[q]);
          for (int k = 0; k < n; ++k)
            {
              f.Lm[a * n + k] += g.w[q] * la * v[k];
              f.Lc[a * n + k] += g.w[q] * la * d[k];
            }
        }
    }
  return f;
}

LevelConsts
make_level_consts(const LevelSpec &L)
{
  if (L.S() > kMaxS)
    throw std::invalid_argument("make_level_consts: k too large");
  const Factors1D f = factors_1d(L.r);
  const TimeTables t = time_tables(L.k, L.tau);
  LevelConsts c{};
  c.nx = L.nx;
  c.ny = L.ny;
  c.gx = L.gx();
  c.gy = L.gy();
  c.nsc = L.nsc();
  c.mv = L.mv();
  c.mp = L.mp();
  c.isz = L.isz();
  const int n = f.n1;
  const double J = 0.25 * L.hx * L.hy, cx = 2.0 / L.hx, cy = 2.0 / L.hy;
  const double nu = L.nu, gm = L.gamma;
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k)
      {
        const int o = i * n + k;
        c.xM[o] = f.M1[o];
        c.xKa[o] = (nu + gm) * cx * cx * f.K1[o];
        c.xKb[o] = nu * cx * cx * f.K1[o];
        c.xC[o] = f.C1[o];
        c.xCt[o] = f.C1[k * n + i];
        // y-direction: index (j = i, l = k)
        c.yM[o] = J * f.M1[o];
        c.yKa[o] = J * nu * cy * cy * f.K1[o];
        c.yKb[o] = J * (nu + gm) * cy * cy * f.K1[o];
        c.yCx[o] = J * gm * cx * cy * f.C1[k * n + i];
        c.yCy[o] = J * gm * cx * cy * f.C1[o];
      }
  for (int a = 0; a < f.P; ++a)
    for (int k = 0; k < n; ++k)
      {
        const int o = a * n + k;
        c.xLc[o] = f.Lc[o];
        c.xLm[o] = f.Lm[o];
        c.yLm[o] = J * cx * f.Lm[o];
        c.yLc[o] = J * cy * f.Lc[o];
      }
  // compact, exactly symmetrised factors (canonical representative wins)
  const auto csym = [n](int i, int k) {
    const int a = i * n + k, b = k * n + i, cc = (n - 1 - i) * n + (n - 1 - k), d = (n - 1 - k) * n + (n - 1 - i);
    return std::min(std::min(a, b), std::min(cc, d));
  };
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k)
      {
        c.cM1[i * n + k] = f.M1[csym(i, k)];
        c.cK1[i * n + k] = f.K1[csym(i, k)];
        c.cC1[i * n + k] = f.C1[i * n + k];
      }
  for (int a = 0; a < f.P; ++a)
    for (int k = 0; k < n; ++k)
      {
        c.cLm[a * n + k] = f.Lm[a * n + k];
        c.cLc[a * n + k] = f.Lc[a * n + k];
      }
  c.sax = (nu + gm) * cx * cx;
  c.say = nu * cx * cx;
  c.sbx = nu * cy * cy;
  c.sby = (nu + gm) * cy * cy;
  c.sg = gm * cx * cy;
  c.scx = cx;
  c.scy = cy;
  const int s = L.S();
  for (int a = 0; a < s; ++a)
    {
      c.lvJ[a] = J * t.lv[a];
      for (int b = 0; b < s; ++b)
        {
          c.KtJ[a * s + b] = J * t.Kt[a * s + b];
          c.MtJ[a * s + b] = J * t.Mt[a * s + b];
        }
    }
  for (int a = 0; a < s; ++a)
    {
      c.lv[a] = t.lv[a];
      for (int b = 0; b < s; ++b)
        {
          c.Kt[a * s + b] = t.Kt[a * s + b];
          c.Mt[a * s + b] = t.Mt[a * s + b];
        }
    }
  return c;
}

CellMatrices
cell_matrices(const LevelSpec &L)
{
  const Factors1D f = factors_1d(L.r);
  const int n = f.n1, nv = n * n, np = L.np();
  const double J = 0.25 * L.hx * L.hy, cx = 2.0 / L.hx, cy = 2.0 / L.hy;
  CellMatrices e;
  e.nv = nv;
  e.np = np;
  e.mass.assign(nv * nv, 0.0);
  e.lap.assign(nv * nv, 0.0);
  e.gd.assign(4 * nv * nv, 0.0);
  e.div.assign(np * 2 * nv, 0.0);
  const auto M = [&](int i, int k) { return f.M1[i * n + k]; };
  const auto K = [&](int i, int k) { return f.K1[i * n + k]; };
  const auto C = [&](int i, int k) { return f.C1[i * n + k]; };
  for (int iy = 0; iy < n; ++iy)
    for (int ix = 0; ix < n; ++ix)
      for (int jy = 0; jy < n; ++jy)
        for (int jx = 0; jx < n; ++jx)
          {
            const int i = iy * n + ix, j = jy * n + jx;
            e.mass[i * nv + j] = J * M(ix, jx) * M(iy, jy);
            e.lap[i * nv + j] = J * (cx * cx * K(ix, jx) * M(iy, jy) + cy * cy * M(ix, jx) * K(iy, jy));
            const int w = 2 * nv;
            e.gd[i * w + j] = J * cx * cx * K(ix, jx) * M(iy, jy);
            e.gd[i * w + nv + j] = J * cx * cy * C(ix, jx) * C(jy, iy);
            e.gd[(nv + i) * w + j] = J * cx * cy * C(jx, ix) * C(iy, jy);
            e.gd[(nv + i) * w + nv + j] = J * cy * cy * M(ix, jx) * K(iy, jy);
          }
  for (int m = 0; m < np; ++m)
    {
      const int am = pdisc_mode_ax(L.r, m), bm = pdisc_mode_ay(L.r, m);
      for (int jy = 0; jy < n; ++jy)
        for (int jx = 0; jx < n; ++jx)
          {
            const int j = jy * n + jx;
            e.div[m * 2 * nv + j] = J * cx * f.Lc[am * n + jx] * f.Lm[bm * n + jy];
            e.div[m * 2 * nv + nv + j] = J * cy * f.Lm[am * n + jx] * f.Lc[bm * n + jy];
          }
    }
  return e;
}

// ================================================================ dense LA
bool
invert_dense(std::vector<double> &a, int n, double *rcond_out)
{
  std::vector<double> lu = a;
  std::vector<int> piv(n);
  double anorm = 0.0;
  for (int j = 0; j < n; ++j)
    {
      double s = 0.0;
      for (int i = 0; i < n; ++i)
        s += std::abs(a[i * n + j]);
      anorm = std::max(anorm, s);
    }
  for (int i = 0; i < n; ++i)
    piv[i] = i;
  for (int k = 0; k < n; ++k)
    {
      int p = k;
      for (int i = k + 1; i < n; ++i)
        if (std::abs(lu[i * n + k]) > std::abs(lu[p * n + k]))
          p = i;
      if (lu[p * n + k] == 0.0)
        {
          if (rcond_out)
            *rcond_out = 0.0;
          return false;
        }
      if (p != k)
        {
          for (int j = 0; j < n; ++j)
            std::swap(lu[k * n + j], lu[p * n + j]);
          std::swap(piv[k], piv[p]);
        }
      const double inv = 1.0 / lu[k * n + k];
      for (int i = k + 1; i < n; ++i)
        {
          const double l = lu[i * n + k] * inv;
          lu[i * n + k] = l;
          if (l != 0.0)
            for (int j = k + 1; j < n; ++j)
              lu[i * n + j] -= l * lu[k * n + j];
        }
    }
  std::vector<double> col(n);
  for (int c = 0; c < n; ++c)
    {
      for (int i = 0; i < n; ++i)
        col[i] = piv[i] == c ? 1.0 : 0.0;
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < i; ++j)
          col[i] -= lu[i * n + j] * col[j];
      for (int i = n - 1; i >= 0; --i)
        {
          for (int j = i + 1; j < n; ++j)
            col[i] -= lu[i * n + j] * col[j];
          col[i] /= lu[i * n + i];
        }
      for (int i = 0; i < n; ++i)
        a[i * n + c] = col[i];
    }
  double inorm = 0.0;
  for (int j = 0; j < n; ++j)
    {
      double s = 0.0;
      for (int i = 0; i < n; ++i)
        s += std::abs(a[i * n + j]);
      inorm = std::max(inorm, s);
    }
  const double rc = (std::isfinite(inorm) && inorm > 0.0) ? 1.0 / (anorm * inorm) : 0.0;
  if (rcond_out)
    *rcond_out = rc;
  return std::isfinite(inorm);
}

std::vector<double>
pseudo_inverse(const std::vector<double> &a, int n, int *rank_out)
{
  // One-sided Jacobi on the columns of A (row-major input).
  std::vector<double> u(n * n), v(n * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      u[j * n + i] = a[i * n + j]; // column j contiguous
  for (int i = 0; i < n; ++i)
    v[i * n + i] = 1.0;            // column i contiguous
  const double eps = std::numeric_limits<double>::epsilon();
  for (int sweep = 0; sweep < 80; ++sweep)
    {
      double off = 0.0;
      for (int p = 0; p < n - 1; ++p)
        for (int q = p + 1; q < n; ++q)
          {
            double al = 0, be = 0, ga = 0;
            for (int i = 0; i < n; ++i)
              {
                al += u[p * n + i] * u[p * n + i];
                be += u[q * n + i] * u[q * n + i];
                ga += u[p * n + i] * u[q * n + i];
              }
            if (ga == 0.0 || al == 0.0 || be == 0.0)
              continue;
            const double conv = std::abs(ga) / std::sqrt(al * be);
            if (!(conv > eps))
              continue;
            off = std::max(off, conv);
            const double zeta = (be - al) / (2.0 * ga);
            const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
            const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
            for (int i = 0; i < n; ++i)
              {
                const double up = u[p * n + i], uq = u[q * n + i];
                u[p * n + i] = c * up - s * uq;
                u[q * n + i] = s * up + c * uq;
                const double vp = v[p * n + i], vq = v[q * n + i];
                v[p * n + i] = c * vp - s * vq;
                v[q * n + i] = s * vp + c * vq;
              }
          }
      if (off <= eps)
        break;
    }
  std::vector<double> sig(n);
  double smax = 0.0;
  for (int j = 0; j < n; ++j)
    {
      double s = 0;
      for (int i = 0; i < n; ++i)
        s += u[j * n + i] * u[j * n + i];
      sig[j] = std::sqrt(s);
      smax = std::max(smax, sig[j]);
    }
  const double thresh = smax * eps * n;
  std::vector<double> pinv(n * n, 0.0);
  int rank = 0;
  for (int j = 0; j < n; ++j)
    {
      if (!(sig[j] > thresh))
        continue;
      ++rank;
      const double is2 = 1.0 / (sig[j] * sig[j]);
      for (int row = 0; row < n; ++row)
        for (int col = 0; col < n; ++col)
          pinv[row * n + col] += v[j * n + row] * u[j * n + col] * is2;
    }
  if (rank_out)
    *rank_out = rank;
  return pinv;
}

// ================================================================ Vanka patches
namespace
{
  struct PatchGeom
  {
    std::vector<std::pair<int, int>> cells;           // sorted by cell index
    std::vector<long long> dofs;                       // flat offsets within one interval, sorted
  };

  PatchGeom
  patch_geometry(const LevelSpec &L, PatchKind kind, int ax, int ay)
  {
    PatchGeom g;
    if (kind == PatchKind::cell)
      g.cells.push_back({ax, ay});
    else
      for (int cy = ay - 1; cy <= ay; ++cy)
        for (int cx = ax - 1; cx <= ax; ++cx)
          if (cx >= 0 && cx < L.nx && cy >= 0 && cy < L.ny)
            g.cells.push_back({cx, cy});
    const int p = L.p(), n1 = L.n1(), gx = L.gx(), gy = L.gy();
    std::vector<long long> nodes;
    for (auto [cx, cy] : g.cells)
      for (int iy = 0; iy < n1; ++iy)
        for (int ix = 0; ix < n1; ++ix)
          {
            const int X = cx * p + ix, Y = cy * p + iy;
            if (X == 0 || X == gx - 1 || Y == 0 || Y == gy - 1)
              continue; // constrained (dof_space.cpp:52-59)
            nodes.push_back(static_cast<long long>(Y) * gx + X);
          }
    std::sort(nodes.begin(), nodes.end());
    nodes.erase(std::unique(nodes.begin(), nodes.end()), nodes.end());
    const int S = L.S();
    for (int a = 0; a < S; ++a)
      for (int c = 0; c < 2; ++c)
        for (long long s : nodes)
          g.dofs.push_back(a * L.mv() + c * L.nsc() + s);
    for (int a = 0; a < S; ++a)
      for (auto [cx, cy] : g.cells)
        for (int m = 0; m < L.np(); ++m)
          g.dofs.push_back(S * L.mv() + a * L.mp() + (static_cast<long long>(cy) * L.nx + cx) * L.np() + m);
    return g;
  }

  // Number of patches (in 1D) covering a grid node / a cell.
  int
  cover_node(PatchKind kind, int ncell, int p, int X)
  {
    int count = 0;
    const int nanch = kind == PatchKind::cell ? ncell : ncell + 1;
    for (int a = 0; a < nanch; ++a)
      {
        const int c0 = kind == PatchKind::cell ? a : std::max(a - 1, 0);
        const int c1 = kind == PatchKind::cell ? a : std::min(a, ncell - 1);
        bool hit = false;
        for (int c = c0; c <= c1 && !hit; ++c)
          hit = c * p <= X && X <= (c + 1) * p;
        count += hit;
      }
    return count;
  }
  int
  cover_cell(PatchKind kind, int ncell, int C)
  {
    if (kind == PatchKind::cell)
      return 1;
    int count = 0;
    for (int a = 0; a <= ncell; ++a)
      count += (C == a - 1 || C == a);
    return count;
  }

  int
  class_key(const LevelSpec &L, PatchKind kind, int ax, int ay)
  {
    const auto bits = [&](int a, int n) {
      if (kind == PatchKind::cell)
        return (a == 0 ? 1 : 0) | (a == n - 1 ? 2 : 0);
      return (a == 0 ? 1 : 0) | (a == 1 ? 2 : 0) | (a == n - 1 ? 4 : 0) | (a == n ? 8 : 0);
    };
    return bits(ax, L.nx) | (bits(ay, L.ny) << 4);
  }

  PatchClass
  build_class(const LevelSpec &L, PatchKind kind, int ax, int ay, const CellMatrices &E, const TimeTables &T,
              bool invert = true)
  {
    const PatchGeom g = patch_geometry(L, kind, ax, ay);
    PatchClass pc;
    pc.n_t = static_cast<int>(g.dofs.size());
    const int S = L.S(), n1 = L.n1(), p = L.p(), nv = E.nv, np = E.np;
    const long long va = patch_vel_anchor(L, kind, ax, ay), pa = patch_pre_anchor(L, kind, ax, ay);
    std::unordered_map<long long, int> pos;
    for (int i = 0; i < pc.n_t; ++i)
      {
        const long long d = g.dofs[i];
        pos[d] = i;
        const bool vel = d < S * L.mv();
        if (vel)
          {
            pc.n_vel = i + 1;
            const long long a = d / L.mv(), rem = d % L.mv(), c = rem / L.nsc(), s = rem % L.nsc();
            pc.rel.push_back(a * L.mv() + c * L.nsc() + (s - va));
            const int X = static_cast<int>(s % L.gx()), Y = static_cast<int>(s / L.gx());
            pc.weight.push_back(1.0 / (cover_node(kind, L.nx, p, X) * cover_node(kind, L.ny, p, Y)));
          }
        else
          {
            const long long q = d - S * L.mv(), a = q / L.mp(), cm = q % L.mp();
            const long long cell = cm / L.np();
            pc.rel.push_back(a * L.mp() + (cm - (pa - S * L.mv())));
            const int CX = static_cast<int>(cell % L.nx), CY = static_cast<int>(cell / L.nx);
            pc.weight.push_back(1.0 / (cover_cell(kind, L.nx, CX) * cover_cell(kind, L.ny, CY)));
          }
      }
    // Assemble R_T S R_T^T over every cell touching the patch (vanka.cpp:88-165).
    std::vector<double> A(static_cast<size_t>(pc.n_t) * pc.n_t, 0.0);
    std::vector<std::pair<int, int>> contrib;
    for (auto [cx, cy] : g.cells)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx)
          {
            const int X = cx + dx, Y = cy + dy;
            if (X >= 0 && X < L.nx && Y >= 0 && Y < L.ny)
              contrib.push_back({X, Y});
          }
    std::sort(contrib.begin(), contrib.end());
    contrib.erase(std::unique(contrib.begin(), contrib.end()), contrib.end());
    std::vector<int> vpos(S * 2 * nv), ppos(S * np);
    for (auto [cx, cy] : contrib)
      {
        for (int a = 0; a < S; ++a)
          {
            for (int c = 0; c < 2; ++c)
              for (int iy = 0; iy < n1; ++iy)
                for (int ix = 0; ix < n1; ++ix)
                  {
                    const long long s = static_cast<long long>(cy * p + iy) * L.gx() + cx * p + ix;
                    const auto it = pos.find(a * L.mv() + c * L.nsc() + s);
                    vpos[(a * 2 + c) * nv + iy * n1 + ix] = it == pos.end() ? -1 : it->second;
                  }
            for (int m = 0; m < np; ++m)
              {
                const auto it =
                  pos.find(S * L.mv() + a * L.mp() + (static_cast<long long>(cy) * L.nx + cx) * np + m);
                ppos[a * np + m] = it == pos.end() ? -1 : it->second;
              }
          }
        for (int a = 0; a < S; ++a)
          for (int b = 0; b < S; ++b)
            {
              const double ck = T.Kt[a * S + b], cb = T.Mt[a * S + b];
              const double cm = L.nu * cb, cg = L.gamma * cb;
              for (int ci = 0; ci < 2; ++ci)
                for (int i = 0; i < nv; ++i)
                  {
                    const int row = vpos[(a * 2 + ci) * nv + i];
                    if (row < 0)
                      continue;
                    for (int cj = 0; cj < 2; ++cj)
                      for (int j = 0; j < nv; ++j)
                        {
                          const int col = vpos[(b * 2 + cj) * nv + j];
                          if (col < 0)
                            continue;
                          double val = cg * E.gd[(ci * nv + i) * 2 * nv + cj * nv + j];
                          if (ci == cj)
                            val += ck * E.mass[i * nv + j] + cm * E.lap[i * nv + j];
                          A[static_cast<size_t>(row) * pc.n_t + col] += val;
                        }
                  }
              for (int m = 0; m < np; ++m)
                {
                  const int prow = ppos[a * np + m], pcol = ppos[b * np + m];
                  for (int c = 0; c < 2; ++c)
                    for (int j = 0; j < nv; ++j)
                      {
                        const double bv = E.div[m * 2 * nv + c * nv + j];
                        const int vr = vpos[(a * 2 + c) * nv + j], vc = vpos[(b * 2 + c) * nv + j];
                        if (prow >= 0 && vc >= 0)
                          A[static_cast<size_t>(prow) * pc.n_t + vc] += cb * bv;
                        if (vr >= 0 && pcol >= 0)
                          A[static_cast<size_t>(vr) * pc.n_t + pcol] -= cb * bv;
                      }
                }
            }
      }
    if (!invert)
      {
        pc.inverse = std::move(A); // the assembled matrix itself
        return pc;
      }
    if (L.k >= 2)
      {
        // spatial factors: the same assembly on a single-slot copy with unit
        // temporal coefficients, (K, M) = (1, 0) -> M_s and (0, 1) -> A_s
        LevelSpec L0 = L;
        L0.k = 0;
        TimeTables t0;
        t0.k = 0;
        t0.tau = L.tau;
        t0.Kt = {1.0};
        t0.Mt = {0.0};
        PatchClass ms = build_class(L0, kind, ax, ay, E, t0, false);
        t0.Kt = {0.0};
        t0.Mt = {1.0};
        PatchClass as = build_class(L0, kind, ax, ay, E, t0, false);
        pc.n_s = ms.n_t;
        pc.n_vs = ms.n_vel;
        pc.Ms = std::move(ms.inverse);
        pc.As = std::move(as.inverse);
        // A_T must equal K_t (x) M_s + M_t (x) A_s in the patch ordering
        // (velocity of all slots, then pressure of all slots)
        const int ns = pc.n_s, nvs = pc.n_vs, nps = ns - nvs;
        const auto prow = [&](int a, int j) { return j < nvs ? a * nvs + j : S * nvs + a * nps + (j - nvs); };
        double err = 0.0, amax = 0.0;
        for (int a = 0; a < S; ++a)
          for (int b = 0; b < S; ++b)
            for (int i = 0; i < ns; ++i)
              for (int j = 0; j < ns; ++j)
                {
                  const double want = T.Kt[a * S + b] * pc.Ms[i * ns + j] + T.Mt[a * S + b] * pc.As[i * ns + j];
                  const double got = A[static_cast<size_t>(prow(a, i)) * pc.n_t + prow(b, j)];
                  err = std::max(err, std::abs(want - got));
                  amax = std::max(amax, std::abs(got));
                }
        if (pc.n_t != S * ns || err > 1e-12 * amax)
          {
            pc.n_s = 0; // no Kronecker structure: dense path only
            pc.Ms.clear();
            pc.As.clear();
          }
      }
    std::vector<double> inv = A;
    double rc = 0.0;
    const bool ok = invert_dense(inv, pc.n_t, &rc);
    if (!ok || rc < 1e-12)
      {
        // Whole-domain patch: constant-pressure null space per slot; the
        // min-norm solve of vanka.cpp:167-176 is the pseudo-inverse.
        int rank = 0;
        inv = pseudo_inverse(A, pc.n_t, &rank);
        if (rank + S < pc.n_t)
          throw std::runtime_error("build_patches: singular local patch matrix");
        pc.singular = true;
      }
    pc.inverse = std::move(inv);
    return pc;
  }
} // namespace

PatchSet
build_patches(const LevelSpec &L, PatchKind kind)
{
  PatchSet ps;
  ps.kind = kind;
  const CellMatrices E = cell_matrices(L);
  const TimeTables T = time_tables(L.k, L.tau);
  const int nax = kind == PatchKind::cell ? L.nx : L.nx + 1;
  const int nay = kind == PatchKind::cell ? L.ny : L.ny + 1;
  const int period = kind == PatchKind::cell ? 2 : 3;
  ps.colours.resize(period * period);
  std::map<int, int> key_to_class;
  for (int ay = 0; ay < nay; ++ay)
    for (int ax = 0; ax < nax; ++ax)
      {
        const int key = class_key(L, kind, ax, ay);
        auto it = key_to_class.find(key);
        if (it == key_to_class.end())
          {
            ps.classes.push_back(build_class(L, kind, ax, ay, E, T));
            it = key_to_class.emplace(key, static_cast<int>(ps.classes.size()) - 1).first;
          }
        const int cls = it->second;
        ps.total_matrix_elements += static_cast<std::uint64_t>(ps.classes[cls].n_t) * ps.classes[cls].n_t;
        ps.colours[(ay % period) * period + (ax % period)].push_back({cls, ax, ay});
      }
  for (auto &col : ps.colours)
    std::stable_sort(col.begin(), col.end(), [](const auto &a, const auto &b) { return a.cls < b.cls; });

  // Factored inverses (k >= 2, every class regular with Kronecker structure):
  // A_T^{-1} = (V (x) I) blockdiag(B_b^{-1}) (W (x) I), middle blocks
  //   real eigenvalue:  B = alpha M_s + A_s                      (n_s)
  //   pair:             B = [[alpha M_s + A_s, beta M_s],
  //                          [-beta M_s, alpha M_s + A_s]]      (2 n_s)
  bool all_ok = L.k >= 2 && !ps.classes.empty();
  int max_ns = 0;
  for (const auto &pc : ps.classes)
    {
      all_ok = all_ok && !pc.singular && pc.n_s > 0;
      max_ns = std::max(max_ns, pc.n_s);
    }
  if (all_ok)
    {
      ps.eig = temporal_eigen(T);
      const int S = L.S(), nsp = (max_ns + 7) / 8 * 8;
      if (ps.eig.ok && S * nsp <= 128)
        {
          ps.n_sp = nsp;
          bool inv_ok = true;
          for (auto &pc : ps.classes)
            {
              const int ns = pc.n_s;
              pc.fac_inv.assign(static_cast<size_t>(S * nsp) * 2 * nsp, 0.0);
              for (size_t b = 0; b < ps.eig.blk_c0.size() && inv_ok; ++b)
                {
                  const int c0 = ps.eig.blk_c0[b], sz = ps.eig.blk_sz[b], m = sz * ns;
                  const double al = ps.eig.alpha[b], be = ps.eig.beta[b];
                  std::vector<double> B(static_cast<size_t>(m) * m, 0.0);
                  for (int bi = 0; bi < sz; ++bi)
                    for (int bj = 0; bj < sz; ++bj)
                      {
                        // block (bi, bj): diagonal alpha Ms + As; off-diagonal +-beta Ms
                        const double cm = bi == bj ? al : (bi == 0 ? be : -be), ca = bi == bj ? 1.0 : 0.0;
                        for (int i = 0; i < ns; ++i)
                          for (int j = 0; j < ns; ++j)
                            B[static_cast<size_t>(bi * ns + i) * m + bj * ns + j] =
                              cm * pc.Ms[i * ns + j] + ca * pc.As[i * ns + j];
                      }
                  double rc = 0.0;
                  if (!invert_dense(B, m, &rc) || rc < 1e-14)
                    {
                      inv_ok = false;
                      break;
                    }
                  for (int bi = 0; bi < sz; ++bi)
                    for (int i = 0; i < ns; ++i)
                      for (int bj = 0; bj < sz; ++bj)
                        for (int j = 0; j < ns; ++j)
                          pc.fac_inv[static_cast<size_t>((c0 + bi) * nsp + i) * 2 * nsp + bj * nsp + j] =
                            B[static_cast<size_t>(bi * ns + i) * m + bj * ns + j];
                }
              pc.fac_ok = inv_ok;
            }
          ps.factored = inv_ok;
          // safety net: the factored inverse must reproduce the dense one
          for (size_t ci = 0; ci < ps.classes.size() && ps.factored; ++ci)
            {
              const PatchClass &pc = ps.classes[ci];
              const int ns = pc.n_s, nvs = pc.n_vs, nps = ns - nvs, nt = pc.n_t;
              const auto prow = [&](int a, int j) { return j < nvs ? a * nvs + j : S * nvs + a * nps + (j - nvs); };
              std::vector<double> r(nt), t(S * nsp, 0.0), y(S * nsp, 0.0), z(nt, 0.0), zd(nt, 0.0);
              for (int i = 0; i < nt; ++i)
                r[i] = std::sin(1.0 + 3.7 * i) + 0.3 * std::cos(0.9 * i * i);
              for (int i = 0; i < S; ++i)
                for (int j = 0; j < ns; ++j)
                  for (int b = 0; b < S; ++b)
                    t[i * nsp + j] += ps.eig.W[i * S + b] * r[prow(b, j)];
              for (size_t b = 0; b < ps.eig.blk_c0.size(); ++b)
                {
                  const int c0 = ps.eig.blk_c0[b], sz = ps.eig.blk_sz[b];
                  for (int bi = 0; bi < sz; ++bi)
                    for (int i = 0; i < ns; ++i)
                      for (int bj = 0; bj < sz; ++bj)
                        for (int j = 0; j < ns; ++j)
                          y[(c0 + bi) * nsp + i] +=
                            pc.fac_inv[static_cast<size_t>((c0 + bi) * nsp + i) * 2 * nsp + bj * nsp + j] *
                            t[(c0 + bj) * nsp + j];
                }
              for (int a = 0; a < S; ++a)
                for (int j = 0; j < ns; ++j)
                  for (int i = 0; i < S; ++i)
                    z[prow(a, j)] += ps.eig.V[a * S + i] * y[i * nsp + j];
              double err = 0.0, zmax = 0.0;
              for (int i = 0; i < nt; ++i)
                {
                  for (int j = 0; j < nt; ++j)
                    zd[i] += pc.inverse[static_cast<size_t>(i) * nt + j] * r[j];
                  zmax = std::max(zmax, std::abs(zd[i]));
                }
              for (int i = 0; i < nt; ++i)
                err = std::max(err, std::abs(z[i] - zd[i]));
              if (!(err <= 1e-10 * zmax))
                ps.factored = false;
            }
        }
    }
  if (ps.factored)
    for (int ay = 0; ay < nay; ++ay)
      for (int ax = 0; ax < nax; ++ax)
        {
          const int cls = key_to_class[class_key(L, kind, ax, ay)];
          std::uint64_t e = 0;
          for (size_t b = 0; b < ps.eig.blk_sz.size(); ++b)
            e += static_cast<std::uint64_t>(ps.eig.blk_sz[b] * ps.classes[cls].n_s) * ps.eig.blk_sz[b] *
                 ps.classes[cls].n_s;
          ps.factored_matrix_elements += e + 2ull * L.S() * L.S() * ps.classes[cls].n_s;
        }
  for (auto &pc : ps.classes)
    {
      pc.Ms.clear();
      pc.As.clear();
    }
  return ps;
}

// ================================================================ transfers
  Csr1D
  transpose_csr(const Csr1D &a)
  {
    Csr1D t;
    t.rows = a.cols;
    t.cols = a.rows;
    t.ptr.assign(t.rows + 1, 0);
    for (int c : a.col)
      t.ptr[c + 1]++;
    for (int i = 0; i < t.rows; ++i)
      t.ptr[i + 1] += t.ptr[i];
    t.col.resize(a.col.size());
    t.val.resize(a.val.size());
    std::vector<int> fill(t.ptr.begin(), t.ptr.end() - 1);
    for (int r = 0; r < a.rows; ++r)
      for (int k = a.ptr[r]; k < a.ptr[r + 1]; ++k)
        {
          const int dst = fill[a.col[k]]++;
          t.col[dst] = r;
          t.val[dst] = a.val[k];
        }
    return t;
  }

  // 1D interpolation from the coarse Q_{rc+1} grid to the fine grid points.
  Csr1D
  interp_1d(int nc_cells, int rc, int nf_cells, int rf, bool h_step)
  {
    const auto cnodes = gauss_lobatto(rc + 2), fnodes = gauss_lobatto(rf + 2);
    const int pc = rc + 1, pf = rf + 1;
    Csr1D m;
    m.rows = nf_cells * pf + 1;
    m.cols = nc_cells * pc + 1;
    m.ptr.push_back(0);
    for (int X = 0; X < m.rows; ++X)
      {
        const int fc = std::min(X / pf, nf_cells - 1);
        const int ix = X - fc * pf;
        int cc;
        double xi;
        if (h_step)
          {
            cc = fc / 2;
            const int child = fc % 2;
            xi = 0.5 * (fnodes[ix] + 2.0 * child - 1.0); // transfer.cpp:168-175
          }
        else
          {
            cc = fc;
            xi = fnodes[ix]; // transfer.cpp:295-298
          }
        for (int jx = 0; jx < rc + 2; ++jx)
          {
            const double v = lagrange(cnodes, jx, xi);
            if (v != 0.0)
              {
                m.col.push_back(cc * pc + jx);
                m.val.push_back(v);
              }
          }
        m.ptr.push_back(static_cast<int>(m.col.size()));
      }
    return m;
  }

  double
  pdisc_value(int r, int m, double x, double y)
  {
    return legendre(pdisc_mode_ax(r, m), x) * legendre(pdisc_mode_ay(r, m), y);
  }

TransferTables
build_transfer(const LevelSpec &c, const LevelSpec &f, TransferKind kind)
{
  TransferTables t;
  t.kind = kind;
  const bool h = kind == TransferKind::h_space || kind == TransferKind::h_space_p_time;
  const bool p = kind == TransferKind::p_space || kind == TransferKind::p_space_p_time;
  t.spatial = h || p;
  t.temporal = kind == TransferKind::p_time || kind == TransferKind::h_space_p_time ||
               kind == TransferKind::p_space_p_time;
  if (h)
    {
      if (f.nx != 2 * c.nx || f.ny != 2 * c.ny || f.r != c.r)
        throw std::invalid_argument("build_transfer: levels not nested for h_space");
      t.px = interp_1d(c.nx, c.r, f.nx, f.r, true);
      t.py = interp_1d(c.ny, c.r, f.ny, f.r, true);
      t.pmode = 1;
      // Pressure: L2 re-expansion of the parent polynomial on each child
      // (transfer.cpp:225-253), exact Gauss rule with r+1 points.
      const int np = c.np();
      const Rule1D g = gauss_legendre(c.r + 1);
      t.child.assign(4 * np * np, 0.0);
      for (int cy = 0; cy < 2; ++cy)
        for (int cx = 0; cx < 2; ++cx)
          for (int m = 0; m < np; ++m)
            {
              const int am = pdisc_mode_ax(c.r, m), bm = pdisc_mode_ay(c.r, m);
              const double gram = (2.0 / (2 * am + 1)) * (2.0 / (2 * bm + 1));
              for (int l = 0; l < np; ++l)
                {
                  double s = 0.0;
                  for (size_t qy = 0; qy < g.x.size(); ++qy)
                    for (size_t qx = 0; qx < g.x.size(); ++qx)
                      {
                        const double xc = g.x[qx], yc = g.x[qy];
                        const double xp = 0.5 * (xc + 2.0 * cx - 1.0), yp = 0.5 * (yc + 2.0 * cy - 1.0);
                        s += g.w[qx] * g.w[qy] * pdisc_value(c.r, m, xc, yc) * pdisc_value(c.r, l, xp, yp);
                      }
                  t.child[(cy * 2 + cx) * np * np + m * np + l] = s / gram;
                }
            }
    }
  else if (p)
    {
      if (f.nx != c.nx || f.ny != c.ny || c.r != f.r / 2)
        throw std::invalid_argument("build_transfer: degrees not related by bisection");
      t.px = interp_1d(c.nx, c.r, f.nx, f.r, false);
      t.py = interp_1d(c.ny, c.r, f.ny, f.r, false);
      t.pmode = 2;
      t.embed.resize(c.np());
      for (int l = 0; l < c.np(); ++l)
        for (int m = 0; m < f.np(); ++m)
          if (pdisc_mode_ax(f.r, m) == pdisc_mode_ax(c.r, l) && pdisc_mode_ay(f.r, m) == pdisc_mode_ay(c.r, l))
            {
              t.embed[l] = m;
              break;
            }
    }
  else if (kind == TransferKind::identity || kind == TransferKind::p_time)
    {
      if (f.nx != c.nx || f.r != c.r)
        throw std::invalid_argument("build_transfer: spatial mismatch for a temporal-only transfer");
    }
  if (t.spatial)
    {
      t.rx = transpose_csr(t.px);
      t.ry = transpose_csr(t.py);
    }
  if (t.temporal)
    {
      const Rule1D rc = gauss_radau_right(c.k + 1), rf = gauss_radau_right(f.k + 1);
      t.e_time.assign((f.k + 1) * (c.k + 1), 0.0);
      for (int a = 0; a <= f.k; ++a)
        for (int b = 0; b <= c.k; ++b)
          t.e_time[a * (c.k + 1) + b] = lagrange(rc.x, b, rf.x[a]);
    }
  return t;
}

// ================================================================ coarse level
std::vector<double>
coarse_inverse(const LevelSpec &L, std::vector<long long> &pinned)
{
  const long long N = L.isz();
  if (N > 20000)
    throw std::runtime_error("coarse_inverse: coarse level too large for a dense direct solve");
  const int n = static_cast<int>(N), S = L.S(), n1 = L.n1(), p = L.p(), nv = n1 * n1, np = L.np();
  const CellMatrices E = cell_matrices(L);
  const TimeTables T = time_tables(L.k, L.tau);
  std::vector<double> A(static_cast<size_t>(n) * n, 0.0);
  const auto constrained = [&](long long s) {
    const int X = static_cast<int>(s % L.gx()), Y = static_cast<int>(s / L.gx());
    return X == 0 || X == L.gx() - 1 || Y == 0 || Y == L.gy() - 1;
  };
  // st_operator.cpp:469-554 on the level's own element matrices
  for (int cy = 0; cy < L.ny; ++cy)
    for (int cx = 0; cx < L.nx; ++cx)
      {
        std::vector<long long> node(nv);
        for (int iy = 0; iy < n1; ++iy)
          for (int ix = 0; ix < n1; ++ix)
            node[iy * n1 + ix] = static_cast<long long>(cy * p + iy) * L.gx() + cx * p + ix;
        const long long pb = (static_cast<long long>(cy) * L.nx + cx) * np;
        for (int a = 0; a < S; ++a)
          for (int b = 0; b < S; ++b)
            {
              const double ck = T.Kt[a * S + b], cb = T.Mt[a * S + b];
              for (int ci = 0; ci < 2; ++ci)
                for (int i = 0; i < nv; ++i)
                  {
                    if (constrained(node[i]))
                      continue;
                    const long long row = a * L.mv() + ci * L.nsc() + node[i];
                    for (int cj = 0; cj < 2; ++cj)
                      for (int j = 0; j < nv; ++j)
                        {
                          if (constrained(node[j]))
                            continue;
                          double v = L.gamma * cb * E.gd[(ci * nv + i) * 2 * nv + cj * nv + j];
                          if (ci == cj)
                            v += ck * E.mass[i * nv + j] + L.nu * cb * E.lap[i * nv + j];
                          A[row * n + b * L.mv() + cj * L.nsc() + node[j]] += v;
                        }
                  }
              for (int m = 0; m < np; ++m)
                for (int c = 0; c < 2; ++c)
                  for (int j = 0; j < nv; ++j)
                    {
                      if (constrained(node[j]))
                        continue;
                      const double bv = E.div[m * 2 * nv + c * nv + j];
                      const long long vrow = a * L.mv() + c * L.nsc() + node[j];
                      const long long pcol = S * L.mv() + b * L.mp() + pb + m;
                      const long long prow = S * L.mv() + a * L.mp() + pb + m;
                      const long long vcol = b * L.mv() + c * L.nsc() + node[j];
                      A[vrow * n + pcol] -= cb * bv;
                      A[prow * n + vcol] += cb * bv;
                    }
            }
      }
  for (int a = 0; a < S; ++a)
    for (int c = 0; c < 2; ++c)
      for (long long s = 0; s < L.nsc(); ++s)
        if (constrained(s))
          {
            const long long g = a * L.mv() + c * L.nsc() + s;
            A[g * n + g] = 1.0;
          }
  pinned.clear();
  for (int a = 0; a < S; ++a) // solver.cpp:20-36
    {
      const long long pr = S * L.mv() + a * L.mp();
      pinned.push_back(pr);
      for (int j = 0; j < n; ++j)
        A[pr * n + j] = 0.0;
      A[pr * n + pr] = 1.0;
    }
  double rc = 0.0;
  if (!invert_dense(A, n, &rc) || rc < 1e-14)
    throw std::runtime_error("coarse_inverse: singular coarse matrix");
  return A;
}

// ================================================================ problem tables
ProblemTables
problem_tables(const LevelSpec &L)
{
  if (L.r > 4 || L.k > 4)
    throw std::invalid_argument("problem_tables: r and k must be <= 4");
  ProblemTables T{};
  const int n1 = L.n1();
  const std::vector<double> gll = gauss_lobatto(n1);
  for (int i = 0; i < n1; ++i)
    T.gll[i] = gll[i];
  const Rule1D ga = gauss_legendre(L.r + 2); // st_operator.cpp:167
  for (int q = 0; q < L.r + 2; ++q)
    {
      T.ax[q] = ga.x[q];
      T.aw[q] = ga.w[q];
      for (int i = 0; i < n1; ++i)
        T.aphi[q * n1 + i] = lagrange(gll, i, ga.x[q]);
    }
  const TimeTables tt = time_tables(L.k, L.tau);
  for (int a = 0; a <= L.k; ++a)
    {
      T.tn[a] = tt.nodes[a];
      T.tw[a] = tt.weights[a];
    }
  const Rule1D ge = gauss_legendre(L.r + 3); // harness.cpp:85 (CellKernels eval(vs, ps, r + 3))
  for (int q = 0; q < L.r + 3; ++q)
    {
      T.ex[q] = ge.x[q];
      T.ew[q] = ge.w[q];
      for (int i = 0; i < n1; ++i)
        {
          T.ephi[q * n1 + i] = lagrange(gll, i, ge.x[q]);
          T.edphi[q * n1 + i] = lagrange_deriv(gll, i, ge.x[q]);
        }
      for (int a = 0; a <= L.r; ++a)
        T.eleg[q * (L.r + 1) + a] = legendre(a, ge.x[q]);
    }
  const Rule1D gt = gauss_legendre(L.k + 2); // harness.cpp:81
  for (int q = 0; q < L.k + 2; ++q)
    {
      T.tq[q] = gt.x[q];
      T.tqw[q] = gt.w[q];
      for (int a = 0; a <= L.k; ++a)
        T.tval[q * (L.k + 1) + a] = lagrange(tt.nodes, a, gt.x[q]);
    }
  return T;
}

// ================================================================ hierarchy plan
std::vector<LevelPlan>
plan_levels(const HierarchyConfig &cfg, int *n_steps_out)
{
  struct Entry
  {
    double h;
    int p;
  };
  const auto construct = [](double h_fine, double h_coarse, int p_fine, int p_coarse) {
    if (!(h_fine <= h_coarse) || !(p_fine >= p_coarse && p_coarse >= 1))
      throw std::invalid_argument("plan_levels: invalid coarsening bounds");
    std::vector<Entry> list; // hierarchy.cpp:9-35
    double h = h_fine;
    int p = p_fine;
    while (p > p_coarse)
      {
        list.insert(list.begin(), Entry{h, p});
        p = std::max(p / 2, p_coarse);
      }
    while (h <= h_coarse * (1.0 + 1e-12))
      {
        list.insert(list.begin(), Entry{h, p});
        h *= 2.0;
      }
    return list;
  };
  const int c = cfg.refinements;
  const int k = cfg.k < 0 ? cfg.r : cfg.k;
  const double h = std::pow(0.5, c);
  const int n = cfg.n_steps > 0 ? cfg.n_steps : static_cast<int>(std::lround(cfg.t_end * (1 << (c + 1))));
  const double tau = cfg.t_end / n;
  if (n_steps_out)
    *n_steps_out = n;
  std::vector<Entry> sp = cfg.h_only ? construct(h, 1.0, cfg.r, cfg.r) : construct(h, 1.0, cfg.r, 1);
  std::vector<Entry> tm = cfg.h_only ? construct(tau, tau, k, k) : construct(tau, tau, k, 1);
  const size_t L = std::max(sp.size(), tm.size()); // hierarchy.cpp:45-52
  while (sp.size() < L)
    sp.push_back(sp.back());
  while (tm.size() < L)
    tm.push_back(tm.back());
  std::vector<LevelPlan> out(L);
  const double h_finest = sp.back().h;
  for (size_t l = 0; l < L; ++l)
    {
      const int mc = static_cast<int>(std::lround(std::log2(sp[l].h / h_finest)));
      LevelSpec &s = out[l].spec;
      s.nx = s.ny = 1 << (c - mc);
      s.hx = s.hy = 1.0 / s.nx;
      s.r = sp[l].p;
      s.k = tm[l].p;
      s.tau = tm[l].h;
      s.nu = cfg.nu;
      s.gamma = cfg.gamma;
      if (l == 0)
        continue;
      const LevelSpec &co = out[l - 1].spec;
      const bool hs = s.nx != co.nx, ps = s.r != co.r, ks = s.k != co.k;
      if (hs && ps)
        throw std::invalid_argument("plan_levels: spatial h- and p-step on one level");
      out[l].kind_to_coarser = hs   ? (ks ? TransferKind::h_space_p_time : TransferKind::h_space)
                               : ps ? (ks ? TransferKind::p_space_p_time : TransferKind::p_space)
                               : ks ? TransferKind::p_time
                                    : TransferKind::identity;
    }
  return out;
}

} // namespace stmg_b200
