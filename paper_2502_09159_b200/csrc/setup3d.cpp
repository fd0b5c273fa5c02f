// Host setup of the 3D hp-STMG path (BASELINE C3 / C5): device constants,
// element matrices on trilinear cells, cell-Vanka patch classes and their
// inverses, transfer tables (spatial h / p, temporal p / h) and the coarse
// level's pinned inverse. Product code, independent of oracle/.
#include "st3d.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <map>
#include <random>
#include <stdexcept>

namespace stmg_b200
{

namespace
{
std::vector<std::array<int, 3>>
modes3(int r) // pdisc.cpp:41-55 (dim 3), degree-major
{
  std::vector<std::array<int, 3>> e;
  for (int deg = 0; deg <= r; ++deg)
    for (int a = deg; a >= 0; --a)
      for (int b = deg - a; b >= 0; --b)
        e.push_back({a, b, deg - a - b});
  return e;
}
} // namespace

Level3Consts
make_level3_consts(const Level3Spec &L, const double *dev_verts)
{
  if (L.r < 1 || L.r > 4 || L.k < 0 || L.k > 4)
    throw std::invalid_argument("3D level: need 1 <= r <= 4, 0 <= k <= 4");
  Level3Consts P{};
  P.nx = L.nx;
  P.ny = L.ny;
  P.nz = L.nz;
  P.gx = L.gx();
  P.gy = L.gy();
  P.gz = L.gz();
  P.zlo = L.zlo();
  P.zhi = L.zhi();
  P.np = L.np();
  P.nsc = L.nsc();
  P.mv = L.mv();
  P.mp = L.mp();
  P.isz = L.isz();
  const int N = L.n1();
  const auto gll = gauss_lobatto(N);
  const Rule1D g = gauss_legendre(N);
  for (int q = 0; q < N; ++q)
    {
      P.w[q] = g.w[q];
      P.xq[q] = g.x[q];
      for (int i = 0; i < N; ++i)
        {
          P.phi[q * N + i] = lagrange(gll, i, g.x[q]);
          P.dphi[q * N + i] = lagrange_deriv(gll, i, g.x[q]);
        }
      for (int a = 0; a <= L.r; ++a)
        P.leg[a * N + q] = legendre(a, g.x[q]);
    }
  const auto ex = modes3(L.r);
  for (size_t m = 0; m < ex.size(); ++m)
    for (int d = 0; d < 3; ++d)
      P.ex[m][d] = ex[m][d];
  const TimeTables T = time_tables(L.k, L.tau);
  const int S = L.S();
  for (int a = 0; a < S; ++a)
    {
      P.lv[a] = T.lv[a];
      for (int b = 0; b < S; ++b)
        {
          P.Kt[a * S + b] = T.Kt[a * S + b];
          P.Mt[a * S + b] = T.Mt[a * S + b];
        }
    }
  P.nu = L.nu;
  P.gamma = L.gamma;
  P.hx = 1.0 / L.nx;
  P.hy = 1.0 / L.ny;
  P.hz = L.hz();
  P.verts = dev_verts;
  P.gemmE = nullptr;
  for (int i = 0; i < N; ++i)
    for (int k = 0; k < N; ++k)
      {
        double m = 0.0, kk = 0.0, c = 0.0;
        for (int q = 0; q < N; ++q)
          {
            m += g.w[q] * P.phi[q * N + i] * P.phi[q * N + k];
            kk += g.w[q] * P.dphi[q * N + i] * P.dphi[q * N + k];
            c += g.w[q] * P.phi[q * N + i] * P.dphi[q * N + k];
          }
        P.m1[i * N + k] = m;
        P.k1[i * N + k] = kk;
        P.c1[i * N + k] = c;
      }
  for (int a = 0; a <= L.r; ++a)
    for (int i = 0; i < N; ++i)
      {
        double sm = 0.0, sc = 0.0;
        for (int q = 0; q < N; ++q)
          {
            sm += g.w[q] * P.leg[a * N + q] * P.phi[q * N + i];
            sc += g.w[q] * P.leg[a * N + q] * P.dphi[q * N + i];
          }
        P.lm[a * N + i] = sm;
        P.lc[a * N + i] = sc;
      }
  return P;
}

std::vector<double>
cartesian_vertices(const Level3Spec &L, double amp, unsigned seed)
{
  std::vector<double> v(static_cast<size_t>(L.nverts()) * 3);
  std::mt19937 gen(seed);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  const double h[3] = {1.0 / L.nx, 1.0 / L.ny, 1.0 / L.nz};
  for (int vz = 0; vz <= L.nz; ++vz)
    for (int vy = 0; vy <= L.ny; ++vy)
      for (int vx = 0; vx <= L.nx; ++vx)
        {
          const size_t i = ((static_cast<size_t>(vz) * (L.ny + 1) + vy) * (L.nx + 1) + vx) * 3;
          const int c[3] = {vx, vy, vz}, n[3] = {L.nx, L.ny, L.nz};
          const bool interior = vx > 0 && vy > 0 && vz > 0 && vx < L.nx && vy < L.ny && vz < L.nz;
          for (int d = 0; d < 3; ++d)
            {
              double x = static_cast<double>(c[d]) / n[d];
              if (amp > 0.0 && interior)
                x += amp * h[d] * U(gen);
              v[i + d] = x;
            }
        }
  return v;
}

void
cell_vertices(const Level3Spec &L, const std::vector<double> &verts, int cx, int cy, int cz, double X8[8][3])
{
  for (int c = 0; c < 8; ++c)
    {
      const int vx = cx + (c & 1), vy = cy + ((c >> 1) & 1), vz = cz + (c >> 2);
      const size_t i = ((static_cast<size_t>(vz) * (L.ny + 1) + vy) * (L.nx + 1) + vx) * 3;
      for (int d = 0; d < 3; ++d)
        X8[c][d] = verts[i + d];
    }
}

Cell3Matrices
cell3_matrices(const Level3Spec &L, const double X8[8][3])
{
  const int N = L.n1(), nv = N * N * N, np = L.np();
  const auto gll = gauss_lobatto(N);
  const Rule1D g = gauss_legendre(N);
  const auto ex = modes3(L.r);
  Cell3Matrices M;
  M.nv = nv;
  M.np = np;
  M.mass.assign(static_cast<size_t>(nv) * nv, 0.0);
  M.a.assign(static_cast<size_t>(9) * nv * nv, 0.0);
  M.b.assign(static_cast<size_t>(np) * 3 * nv, 0.0);
  M.pmean.assign(np, 0.0);
  std::vector<double> val(nv), gp(3 * nv), psi(np);
  for (int qz = 0; qz < N; ++qz)
    for (int qy = 0; qy < N; ++qy)
      for (int qx = 0; qx < N; ++qx)
        {
          const double xi[3] = {g.x[qx], g.x[qy], g.x[qz]};
          double J[3][3] = {};
          for (int c = 0; c < 8; ++c)
            {
              const int s[3] = {c & 1, (c >> 1) & 1, c >> 2};
              double nvl[3], nd[3];
              for (int e = 0; e < 3; ++e)
                {
                  nvl[e] = s[e] ? 0.5 * (1 + xi[e]) : 0.5 * (1 - xi[e]);
                  nd[e] = s[e] ? 0.5 : -0.5;
                }
              const double dN[3] = {nd[0] * nvl[1] * nvl[2], nvl[0] * nd[1] * nvl[2], nvl[0] * nvl[1] * nd[2]};
              for (int d = 0; d < 3; ++d)
                for (int e = 0; e < 3; ++e)
                  J[d][e] += X8[c][d] * dN[e];
            }
          const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                             J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                             J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
          if (!(det > 0.0))
            throw std::runtime_error("3D level: inverted cell");
          double Ji[3][3]; // dxi_e / dX_d = Ji[e][d]
          Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
          Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
          Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
          Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
          Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
          Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
          Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
          Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
          Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
          const double wd = g.w[qx] * g.w[qy] * g.w[qz] * det;
          for (int k = 0; k < N; ++k)
            for (int j = 0; j < N; ++j)
              for (int i = 0; i < N; ++i)
                {
                  const int t = (k * N + j) * N + i;
                  const double v0 = lagrange(gll, i, xi[0]), v1 = lagrange(gll, j, xi[1]), v2 = lagrange(gll, k, xi[2]);
                  const double gr[3] = {lagrange_deriv(gll, i, xi[0]) * v1 * v2, v0 * lagrange_deriv(gll, j, xi[1]) * v2,
                                        v0 * v1 * lagrange_deriv(gll, k, xi[2])};
                  val[t] = v0 * v1 * v2;
                  for (int d = 0; d < 3; ++d)
                    gp[3 * t + d] = gr[0] * Ji[0][d] + gr[1] * Ji[1][d] + gr[2] * Ji[2][d];
                }
          for (int l = 0; l < np; ++l)
            {
              psi[l] = legendre(ex[l][0], xi[0]) * legendre(ex[l][1], xi[1]) * legendre(ex[l][2], xi[2]);
              M.pmean[l] += wd * psi[l];
            }
          for (int a = 0; a < nv; ++a)
            for (int b = 0; b < nv; ++b)
              {
                M.mass[static_cast<size_t>(a) * nv + b] += wd * val[a] * val[b];
                const double gg = gp[3 * a] * gp[3 * b] + gp[3 * a + 1] * gp[3 * b + 1] + gp[3 * a + 2] * gp[3 * b + 2];
                for (int c = 0; c < 3; ++c)
                  for (int c2 = 0; c2 < 3; ++c2)
                    M.a[(static_cast<size_t>(c) * nv + a) * 3 * nv + c2 * nv + b] +=
                      wd * (L.gamma * gp[3 * a + c] * gp[3 * b + c2] + (c == c2 ? L.nu * gg : 0.0));
              }
          for (int l = 0; l < np; ++l)
            for (int c = 0; c < 3; ++c)
              for (int b = 0; b < nv; ++b)
                M.b[static_cast<size_t>(l) * 3 * nv + c * nv + b] += wd * psi[l] * gp[3 * b + c];
        }
  return M;
}

std::vector<double>
gemm_element_operator(const Level3Spec &L)
{
  if (L.r != 1)
    throw std::invalid_argument("gemm_element_operator: r = 1 only");
  double X8[8][3];
  for (int c = 0; c < 8; ++c)
    {
      X8[c][0] = (c & 1) * (1.0 / L.nx);
      X8[c][1] = ((c >> 1) & 1) * (1.0 / L.ny);
      X8[c][2] = (c >> 2) * (1.0 / L.nz);
    }
  const Cell3Matrices M = cell3_matrices(L, X8);
  const int nv = 27, np = 4, R = 88, K = 168;
  std::vector<double> E(static_cast<size_t>(R) * K, 0.0);
  for (int c = 0; c < 3; ++c)
    for (int i = 0; i < nv; ++i)
      {
        double *row = &E[static_cast<size_t>(c * nv + i) * K];
        for (int j = 0; j < nv; ++j)
          row[c * nv + j] = M.mass[i * nv + j]; // M UK
        for (int c2 = 0; c2 < 3; ++c2)
          for (int j = 0; j < nv; ++j)
            row[81 + c2 * nv + j] = M.a[(static_cast<size_t>(c) * nv + i) * 3 * nv + c2 * nv + j]; // A UM
        for (int l = 0; l < np; ++l)
          row[162 + l] = -M.b[static_cast<size_t>(l) * 3 * nv + c * nv + i]; // -B^T PM
      }
  for (int l = 0; l < np; ++l)
    for (int c2 = 0; c2 < 3; ++c2)
      for (int j = 0; j < nv; ++j)
        E[static_cast<size_t>(81 + l) * K + 81 + c2 * nv + j] = M.b[static_cast<size_t>(l) * 3 * nv + c2 * nv + j];
  return E;
}

std::vector<double>
pressure_mean3(const Level3Spec &L, const std::vector<double> *verts, double *volume)
{
  const int np = L.np();
  std::vector<double> m(static_cast<size_t>(L.mp()), 0.0);
  double vol = 0.0;
  if (!verts)
    {
      const double cellvol = 1.0 / static_cast<double>(L.ncells());
      for (long long c = 0; c < L.ncells(); ++c)
        m[c * np] = cellvol * 8.0 / 8.0; // int_K psi_0 = |K| (Legendre orthogonality kills the rest)
      *volume = 1.0;
      return m;
    }
  // int_K psi_l on trilinear cells: Gauss rule of the operator
  const int N = L.n1();
  const Rule1D g = gauss_legendre(N);
  const auto ex = modes3(L.r);
  for (int cz = 0; cz < L.nz; ++cz)
    for (int cy = 0; cy < L.ny; ++cy)
      for (int cx = 0; cx < L.nx; ++cx)
        {
          double X8[8][3];
          cell_vertices(L, *verts, cx, cy, cz, X8);
          const long long cell = (static_cast<long long>(cz) * L.ny + cy) * L.nx + cx;
          for (int qz = 0; qz < N; ++qz)
            for (int qy = 0; qy < N; ++qy)
              for (int qx = 0; qx < N; ++qx)
                {
                  const double xi[3] = {g.x[qx], g.x[qy], g.x[qz]};
                  double J[3][3] = {};
                  for (int c = 0; c < 8; ++c)
                    {
                      const int s[3] = {c & 1, (c >> 1) & 1, c >> 2};
                      double nvl[3], nd[3];
                      for (int e = 0; e < 3; ++e)
                        {
                          nvl[e] = s[e] ? 0.5 * (1 + xi[e]) : 0.5 * (1 - xi[e]);
                          nd[e] = s[e] ? 0.5 : -0.5;
                        }
                      const double dN[3] = {nd[0] * nvl[1] * nvl[2], nvl[0] * nd[1] * nvl[2], nvl[0] * nvl[1] * nd[2]};
                      for (int d = 0; d < 3; ++d)
                        for (int e = 0; e < 3; ++e)
                          J[d][e] += X8[c][d] * dN[e];
                    }
                  const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                                     J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                                     J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
                  const double wd = g.w[qx] * g.w[qy] * g.w[qz] * det;
                  vol += wd;
                  for (int l = 0; l < np; ++l)
                    m[cell * np + l] +=
                      wd * legendre(ex[l][0], xi[0]) * legendre(ex[l][1], xi[1]) * legendre(ex[l][2], xi[2]);
                }
        }
  *volume = vol;
  return m;
}

// ================================================================ Vanka
namespace
{
/// Local matrix R_T S R_T^T of the cell patch at (cx, cy, cz) (vanka.cpp:92-165):
/// all cells whose shape functions overlap the patch contribute; dofs are the
/// patch cell's unconstrained velocity nodes (sorted = lexicographic (k,j,i)),
/// velocity for all slots and components, then the cell's pressure modes.
PatchClass
cell_patch(const Level3Spec &L, const std::vector<double> *verts, int cx, int cy, int cz,
           const std::vector<int> &valence, const Cell3Matrices *cart)
{
  const int N = L.n1(), p = L.p(), nv = N * N * N, np = L.np(), S = L.S();
  const TimeTables T = time_tables(L.k, L.tau);
  const int gx = L.gx(), gy = L.gy(), gz = L.gz();
  auto on_bnd = [&](int X, int Y, int Z) {
    return X == 0 || Y == 0 || Z == L.zlo() || X == gx - 1 || Y == gy - 1 || Z == L.zhi();
  };
  std::vector<int> loc; // local node index of the patch's unconstrained nodes
  for (int k = 0; k < N; ++k)
    for (int j = 0; j < N; ++j)
      for (int i = 0; i < N; ++i)
        if (!on_bnd(cx * p + i, cy * p + j, cz * p + k))
          loc.push_back((k * N + j) * N + i);
  const int nl = static_cast<int>(loc.size());
  std::vector<int> pos(nv, -1);
  for (int t = 0; t < nl; ++t)
    pos[loc[t]] = t;
  // spatial matrices on the patch nodes: Ms (nl x nl), As (3nl x 3nl), Bs (np x 3nl)
  std::vector<double> Ms(static_cast<size_t>(nl) * nl, 0.0), As(static_cast<size_t>(9) * nl * nl, 0.0),
    Bs(static_cast<size_t>(np) * 3 * nl, 0.0);
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx)
        {
          const int ox = cx + dx, oy = cy + dy, oz = cz + dz;
          if (ox < 0 || oy < 0 || oz < 0 || ox >= L.nx || oy >= L.ny || oz >= L.nz)
            continue;
          Cell3Matrices own;
          const Cell3Matrices *E = cart;
          if (!E)
            {
              double X8[8][3];
              cell_vertices(L, *verts, ox, oy, oz, X8);
              own = cell3_matrices(L, X8);
              E = &own;
            }
          // local node of neighbour cell -> patch position (or -1)
          std::vector<int> map(nv, -1);
          for (int k = 0; k < N; ++k)
            for (int j = 0; j < N; ++j)
              for (int i = 0; i < N; ++i)
                {
                  const int pi = i + dx * p, pj = j + dy * p, pk = k + dz * p;
                  if (pi < 0 || pj < 0 || pk < 0 || pi >= N || pj >= N || pk >= N)
                    continue;
                  map[(k * N + j) * N + i] = pos[(pk * N + pj) * N + pi];
                }
          for (int a = 0; a < nv; ++a)
            {
              if (map[a] < 0)
                continue;
              for (int b = 0; b < nv; ++b)
                {
                  if (map[b] < 0)
                    continue;
                  Ms[static_cast<size_t>(map[a]) * nl + map[b]] += E->mass[static_cast<size_t>(a) * nv + b];
                  for (int c = 0; c < 3; ++c)
                    for (int c2 = 0; c2 < 3; ++c2)
                      As[(static_cast<size_t>(c) * nl + map[a]) * 3 * nl + c2 * nl + map[b]] +=
                        E->a[(static_cast<size_t>(c) * nv + a) * 3 * nv + c2 * nv + b];
                }
            }
          if (dx == 0 && dy == 0 && dz == 0)
            for (int l = 0; l < np; ++l)
              for (int c = 0; c < 3; ++c)
                for (int b = 0; b < nv; ++b)
                  if (map[b] >= 0)
                    Bs[static_cast<size_t>(l) * 3 * nl + c * nl + map[b]] +=
                      E->b[static_cast<size_t>(l) * 3 * nv + c * nv + b];
        }
  PatchClass pc;
  const int nvel = S * 3 * nl;
  pc.n_t = nvel + S * np;
  pc.n_vel = nvel;
  const long long nsc = L.nsc(), mv = L.mv(), mp = L.mp();
  for (int a = 0; a < S; ++a)
    for (int c = 0; c < 3; ++c)
      for (int t = 0; t < nl; ++t)
        {
          const int i = loc[t] % N, j = (loc[t] / N) % N, k = loc[t] / (N * N);
          pc.rel.push_back(a * mv + c * nsc + (static_cast<long long>(k) * gy + j) * gx + i);
          const long long s = (static_cast<long long>(cz * p + k) * gy + cy * p + j) * gx + cx * p + i;
          pc.weight.push_back(1.0 / valence[s]);
        }
  for (int a = 0; a < S; ++a)
    for (int l = 0; l < np; ++l)
      {
        pc.rel.push_back(a * mp + l);
        pc.weight.push_back(1.0);
      }
  const int n = pc.n_t;
  std::vector<double> A(static_cast<size_t>(n) * n, 0.0);
  for (int a = 0; a < S; ++a)
    for (int b = 0; b < S; ++b)
      {
        const double kt = T.Kt[a * S + b], mt = T.Mt[a * S + b];
        for (int c = 0; c < 3; ++c)
          for (int c2 = 0; c2 < 3; ++c2)
            for (int t = 0; t < nl; ++t)
              for (int u = 0; u < nl; ++u)
                {
                  double v = mt * As[(static_cast<size_t>(c) * nl + t) * 3 * nl + c2 * nl + u];
                  if (c == c2)
                    v += kt * Ms[static_cast<size_t>(t) * nl + u];
                  A[static_cast<size_t>((a * 3 + c) * nl + t) * n + (b * 3 + c2) * nl + u] = v;
                }
        for (int l = 0; l < np; ++l)
          for (int c = 0; c < 3; ++c)
            for (int t = 0; t < nl; ++t)
              {
                const double bv = Bs[static_cast<size_t>(l) * 3 * nl + c * nl + t];
                // velocity row (a, c, t), pressure column (b, l): -Mt(a,b) B^T
                A[static_cast<size_t>((a * 3 + c) * nl + t) * n + nvel + b * np + l] = -mt * bv;
                // pressure row (a, l), velocity column (b, c, t): Mt(a,b) B
                A[static_cast<size_t>(nvel + a * np + l) * n + (b * 3 + c) * nl + t] = mt * bv;
              }
      }
  std::vector<double> inv = A;
  double rc = 0.0;
  const bool ok = invert_dense(inv, n, &rc);
  if (ok && rc >= 1e-12)
    pc.inverse = std::move(inv);
  else
    {
      int rank = 0;
      pc.inverse = pseudo_inverse(A, n, &rank);
      pc.singular = true;
    }
  return pc;
}
} // namespace

namespace
{
/// Nodes on an interface plane also belong to the neighbour part's cells
/// across it: their valence (vanka.cpp:182-192, counted over the whole
/// mesh) is twice the local count.
void
interface_valence(const Level3Spec &L, std::vector<int> &valence)
{
  const long long plane = static_cast<long long>(L.gx()) * L.gy();
  for (int side = 0; side < 2; ++side)
    if (side == 0 ? !L.zlo_bc : !L.zhi_bc)
      {
        const long long z0 = side == 0 ? 0 : static_cast<long long>(L.gz() - 1) * plane;
        for (long long i = 0; i < plane; ++i)
          valence[z0 + i] *= 2;
      }
}
} // namespace

Patch3Set
build_patches3(const Level3Spec &L, const std::vector<double> *verts)
{
  if (L.split())
    throw std::invalid_argument("3D level: patches of a z-split level are set up on the GPU (nx, ny, nz >= 2, "
                                "r <= 2, deformed geometry)");
  const int N = L.n1(), p = L.p();
  std::vector<int> valence(static_cast<size_t>(L.nsc()), 0);
  for (int cz = 0; cz < L.nz; ++cz)
    for (int cy = 0; cy < L.ny; ++cy)
      for (int cx = 0; cx < L.nx; ++cx)
        for (int k = 0; k < N; ++k)
          for (int j = 0; j < N; ++j)
            for (int i = 0; i < N; ++i)
              valence[(static_cast<size_t>(cz * p + k) * L.gy() + cy * p + j) * L.gx() + cx * p + i]++;
  Patch3Set ps;
  ps.cell_class.assign(static_cast<size_t>(L.ncells()), -1);
  if (!verts)
    {
      // Cartesian: the patch depends only on the boundary status per
      // direction (0 low, 1 interior, 2 high, 3 both)
      double X8[8][3];
      const double h[3] = {1.0 / L.nx, 1.0 / L.ny, 1.0 / L.nz};
      for (int c = 0; c < 8; ++c)
        {
          X8[c][0] = (c & 1) * h[0];
          X8[c][1] = ((c >> 1) & 1) * h[1];
          X8[c][2] = (c >> 2) * h[2];
        }
      const Cell3Matrices E = cell3_matrices(L, X8);
      std::map<int, int> key_to_class;
      auto status = [](int c, int n) { return n == 1 ? 3 : (c == 0 ? 0 : (c == n - 1 ? 2 : 1)); };
      for (int cz = 0; cz < L.nz; ++cz)
        for (int cy = 0; cy < L.ny; ++cy)
          for (int cx = 0; cx < L.nx; ++cx)
            {
              const int key = (status(cz, L.nz) * 4 + status(cy, L.ny)) * 4 + status(cx, L.nx);
              auto it = key_to_class.find(key);
              int cls;
              if (it == key_to_class.end())
                {
                  cls = static_cast<int>(ps.classes.size());
                  key_to_class[key] = cls;
                  ps.classes.push_back(cell_patch(L, nullptr, cx, cy, cz, valence, &E));
                }
              else
                cls = it->second;
              ps.cell_class[(static_cast<size_t>(cz) * L.ny + cy) * L.nx + cx] = cls;
            }
    }
  else
    {
      for (int cz = 0; cz < L.nz; ++cz)
        for (int cy = 0; cy < L.ny; ++cy)
          for (int cx = 0; cx < L.nx; ++cx)
            {
              ps.cell_class[(static_cast<size_t>(cz) * L.ny + cy) * L.nx + cx] = static_cast<int>(ps.classes.size());
              ps.classes.push_back(cell_patch(L, verts, cx, cy, cz, valence, nullptr));
            }
    }
  for (size_t c = 0; c < ps.cell_class.size(); ++c)
    {
      const int n = ps.classes[ps.cell_class[c]].n_t;
      ps.total_matrix_elements += static_cast<std::uint64_t>(n) * n;
      ps.max_nt = std::max(ps.max_nt, n);
    }
  return ps;
}

Patch3Layout
cell_patch_layouts3(const Level3Spec &L)
{
  const int N = L.n1(), p = L.p(), np = L.np(), S = L.S();
  const int gx = L.gx(), gy = L.gy(), gz = L.gz();
  const long long nsc = L.nsc(), mv = L.mv(), mp = L.mp();
  std::vector<int> valence(static_cast<size_t>(nsc), 0);
  for (int cz = 0; cz < L.nz; ++cz)
    for (int cy = 0; cy < L.ny; ++cy)
      for (int cx = 0; cx < L.nx; ++cx)
        for (int k = 0; k < N; ++k)
          for (int j = 0; j < N; ++j)
            for (int i = 0; i < N; ++i)
              valence[(static_cast<size_t>(cz * p + k) * gy + cy * p + j) * gx + cx * p + i]++;
  interface_valence(L, valence);
  auto on_bnd = [&](int X, int Y, int Z) {
    return X == 0 || Y == 0 || Z == L.zlo() || X == gx - 1 || Y == gy - 1 || Z == L.zhi();
  };
  Patch3Layout Lo;
  const long long nc = L.ncells();
  Lo.nt.resize(nc);
  Lo.nvel.resize(nc);
  Lo.rel_off.resize(nc + 1);
  Lo.inv_off.resize(nc + 1);
  Lo.rel_off[0] = Lo.inv_off[0] = 0;
  std::vector<int> loc;
  for (int cz = 0; cz < L.nz; ++cz)
    for (int cy = 0; cy < L.ny; ++cy)
      for (int cx = 0; cx < L.nx; ++cx)
        {
          const long long c = (static_cast<long long>(cz) * L.ny + cy) * L.nx + cx;
          loc.clear();
          for (int k = 0; k < N; ++k) // cell_patch: unconstrained nodes, lexicographic
            for (int j = 0; j < N; ++j)
              for (int i = 0; i < N; ++i)
                if (!on_bnd(cx * p + i, cy * p + j, cz * p + k))
                  loc.push_back((k * N + j) * N + i);
          const int nl = static_cast<int>(loc.size());
          for (int a = 0; a < S; ++a)
            for (int comp = 0; comp < 3; ++comp)
              for (int t = 0; t < nl; ++t)
                {
                  const int i = loc[t] % N, j = (loc[t] / N) % N, k = loc[t] / (N * N);
                  Lo.rel.push_back(a * mv + comp * nsc + (static_cast<long long>(k) * gy + j) * gx + i);
                  const long long sn = (static_cast<long long>(cz * p + k) * gy + cy * p + j) * gx + cx * p + i;
                  Lo.weight.push_back(1.0 / valence[sn]);
                }
          for (int a = 0; a < S; ++a)
            for (int l = 0; l < np; ++l)
              {
                Lo.rel.push_back(a * mp + l);
                Lo.weight.push_back(1.0);
              }
          const int n = S * (3 * nl + np);
          Lo.nt[c] = n;
          Lo.nvel[c] = S * 3 * nl;
          Lo.rel_off[c + 1] = Lo.rel_off[c] + n;
          Lo.inv_off[c + 1] = Lo.inv_off[c] + static_cast<long long>(n) * n;
          Lo.total_matrix_elements += static_cast<std::uint64_t>(n) * n;
          Lo.max_nt = std::max(Lo.max_nt, n);
        }
  return Lo;
}

// ================================================================ transfers
Transfer3Tables
build_transfer3(const Level3Spec &c, const Level3Spec &f, bool h_time)
{
  Transfer3Tables t;
  t.h_time = h_time ? 1 : 0;
  const bool h = f.nx == 2 * c.nx && f.ny == 2 * c.ny && f.nz == 2 * c.nz && f.r == c.r;
  const bool same_mesh = f.nx == c.nx && f.ny == c.ny && f.nz == c.nz;
  const bool p = same_mesh && f.r != c.r;
  if (!(h || (same_mesh && (p || f.r == c.r))))
    throw std::invalid_argument("build_transfer3: unsupported level pair");
  if (p && c.r != f.r / 2)
    throw std::invalid_argument("build_transfer3: degrees not related by bisection");
  t.spatial = (h || p) ? 1 : 0;
  if (t.spatial)
    {
      t.px = interp_1d(c.nx, c.r, f.nx, f.r, h);
      t.py = interp_1d(c.ny, c.r, f.ny, f.r, h);
      t.pz = interp_1d(c.nz, c.r, f.nz, f.r, h);
      t.rx = transpose_csr(t.px);
      t.ry = transpose_csr(t.py);
      t.rz = transpose_csr(t.pz);
      // pressure: L2 re-expansion of the coarse cell polynomial on each fine
      // cell in reference coordinates (transfer.cpp:225-253; for p this is
      // the modal embedding of transfer.cpp:338-359)
      t.pmode = h ? 1 : 2;
      const auto ef = modes3(f.r), ec = modes3(c.r);
      const int npf = f.np(), npc = c.np();
      const Rule1D g = gauss_legendre(f.r + 2);
      const int nch = h ? 8 : 1;
      t.child.assign(static_cast<size_t>(nch) * npf * npc, 0.0);
      for (int ch = 0; ch < nch; ++ch)
        {
          const int o[3] = {ch & 1, (ch >> 1) & 1, ch >> 2};
          for (int m = 0; m < npf; ++m)
            for (int l = 0; l < npc; ++l)
              {
                double s = 1.0;
                // separable: product over directions of 1D integrals
                for (int d = 0; d < 3; ++d)
                  {
                    double sd = 0.0;
                    for (size_t q = 0; q < g.x.size(); ++q)
                      {
                        const double xf = g.x[q];
                        const double xc = h ? 0.5 * (xf + 2.0 * o[d] - 1.0) : xf;
                        sd += g.w[q] * legendre(ef[m][d], xf) * legendre(ec[l][d], xc);
                      }
                    s *= sd / (2.0 / (2.0 * ef[m][d] + 1.0));
                  }
                t.child[(static_cast<size_t>(ch) * npf + m) * npc + l] = std::abs(s) < 1e-15 ? 0.0 : s;
              }
        }
    }
  // temporal: E(a, b) = coarse Radau-Lagrange basis b at fine node a, the
  // fine node mapped into the coarse interval for h in time (Eq. DeftPrRe)
  const Rule1D rc = gauss_radau_right(c.k + 1), rf = gauss_radau_right(f.k + 1);
  const int Sf = f.S(), Sc = c.S();
  t.E.assign(static_cast<size_t>(2) * Sf * Sc, 0.0);
  for (int half = 0; half < (h_time ? 2 : 1); ++half)
    for (int a = 0; a < Sf; ++a)
      {
        double tt = rf.x[a];
        if (h_time)
          tt = half == 0 ? 0.5 * (tt - 1.0) : 0.5 * (tt + 1.0);
        for (int b = 0; b < Sc; ++b)
          t.E[(static_cast<size_t>(half) * Sf + a) * Sc + b] = Sc == 1 ? 1.0 : lagrange(rc.x, b, tt);
      }
  return t;
}

// ================================================================ coarse level
void
coarse3_tables(const Level3Spec &L, const std::vector<double> *verts, std::vector<double> &Ginv,
               std::vector<double> &H, std::vector<double> &pmean)
{
  const int N = L.n1(), p = L.p(), nv = N * N * N, np = L.np(), S = L.S();
  const long long nsc = L.nsc(), mv = L.mv(), mp = L.mp(), isz = L.isz();
  if (isz > 20000)
    throw std::invalid_argument("coarse3: coarse level too large for a dense solve");
  const int n = static_cast<int>(isz);
  const TimeTables T = time_tables(L.k, L.tau);
  const int gx = L.gx(), gy = L.gy(), gz = L.gz();
  std::vector<char> bnd(nsc, 0);
  for (int Z = 0; Z < gz; ++Z)
    for (int Y = 0; Y < gy; ++Y)
      for (int X = 0; X < gx; ++X)
        if (X == 0 || Y == 0 || Z == 0 || X == gx - 1 || Y == gy - 1 || Z == gz - 1)
          bnd[(static_cast<long long>(Z) * gy + Y) * gx + X] = 1;
  // assembled spatial matrices (dense: the coarse level is small)
  std::vector<double> Ms(static_cast<size_t>(nsc) * nsc, 0.0), As(static_cast<size_t>(mv) * mv, 0.0),
    Bs(static_cast<size_t>(mp) * mv, 0.0);
  double vol = 0.0;
  pmean = pressure_mean3(L, verts, &vol);
  Cell3Matrices cart;
  if (!verts)
    {
      double X8[8][3];
      for (int c = 0; c < 8; ++c)
        {
          X8[c][0] = (c & 1) * (1.0 / L.nx);
          X8[c][1] = ((c >> 1) & 1) * (1.0 / L.ny);
          X8[c][2] = (c >> 2) * (1.0 / L.nz);
        }
      cart = cell3_matrices(L, X8);
    }
  for (int cz = 0; cz < L.nz; ++cz)
    for (int cy = 0; cy < L.ny; ++cy)
      for (int cx = 0; cx < L.nx; ++cx)
        {
          Cell3Matrices own;
          const Cell3Matrices *E = &cart;
          if (verts)
            {
              double X8[8][3];
              cell_vertices(L, *verts, cx, cy, cz, X8);
              own = cell3_matrices(L, X8);
              E = &own;
            }
          std::vector<long long> sid(nv);
          for (int k = 0; k < N; ++k)
            for (int j = 0; j < N; ++j)
              for (int i = 0; i < N; ++i)
                sid[(k * N + j) * N + i] = (static_cast<long long>(cz * p + k) * gy + cy * p + j) * gx + cx * p + i;
          const long long cell = (static_cast<long long>(cz) * L.ny + cy) * L.nx + cx;
          for (int a = 0; a < nv; ++a)
            for (int b = 0; b < nv; ++b)
              {
                Ms[sid[a] * nsc + sid[b]] += E->mass[static_cast<size_t>(a) * nv + b];
                for (int c = 0; c < 3; ++c)
                  for (int c2 = 0; c2 < 3; ++c2)
                    As[(c * nsc + sid[a]) * mv + c2 * nsc + sid[b]] +=
                      E->a[(static_cast<size_t>(c) * nv + a) * 3 * nv + c2 * nv + b];
              }
          for (int l = 0; l < np; ++l)
            for (int c = 0; c < 3; ++c)
              for (int b = 0; b < nv; ++b)
                Bs[(cell * np + l) * mv + c * nsc + sid[b]] += E->b[static_cast<size_t>(l) * 3 * nv + c * nv + b];
        }
  auto vbnd = [&](long long i) { return bnd[i % nsc] != 0; };
  // constrained interval operator (apply_block: zeroed constrained inputs,
  // identity rows), first pressure dof of each slot pinned
  std::vector<double> D(static_cast<size_t>(n) * n, 0.0);
  for (int a = 0; a < S; ++a)
    for (int b = 0; b < S; ++b)
      {
        const double kt = T.Kt[a * S + b], mt = T.Mt[a * S + b];
        for (long long i = 0; i < mv; ++i)
          {
            if (vbnd(i))
              continue;
            double *row = &D[static_cast<size_t>(a * mv + i) * n];
            for (long long j = 0; j < mv; ++j)
              {
                if (vbnd(j))
                  continue;
                double v = mt * As[i * mv + j];
                if (i / nsc == j / nsc)
                  v += kt * Ms[(i % nsc) * nsc + (j % nsc)];
                row[b * mv + j] += v;
              }
            for (long long q = 0; q < mp; ++q)
              row[S * mv + b * mp + q] += -mt * Bs[q * mv + i];
          }
        for (long long q = 0; q < mp; ++q)
          {
            double *row = &D[static_cast<size_t>(S * mv + a * mp + q) * n];
            for (long long j = 0; j < mv; ++j)
              if (!vbnd(j))
                row[b * mv + j] += mt * Bs[q * mv + j];
          }
      }
  for (int a = 0; a < S; ++a)
    for (long long i = 0; i < mv; ++i)
      if (vbnd(i))
        D[static_cast<size_t>(a * mv + i) * n + a * mv + i] = 1.0;
  for (int a = 0; a < S; ++a)
    {
      const long long pin = S * mv + a * mp;
      std::fill(D.begin() + pin * n, D.begin() + (pin + 1) * n, 0.0);
      D[static_cast<size_t>(pin) * n + pin] = 1.0;
    }
  double rc = 0.0;
  if (!invert_dense(D, n, &rc))
    throw std::runtime_error("coarse3: singular coarse matrix");
  // G = P D^{-1} with pinned rhs entries ignored and the per-slot mean-zero
  // projection P applied (solver.cpp:43-54)
  for (int a = 0; a < S; ++a)
    {
      const long long pin = S * mv + a * mp;
      for (int i = 0; i < n; ++i)
        D[static_cast<size_t>(i) * n + pin] = 0.0;
    }
  Ginv = D;
  for (int a = 0; a < S; ++a)
    {
      const long long base = S * mv + a * mp;
      for (int j = 0; j < n; ++j)
        {
          double mean = 0.0;
          for (long long q = 0; q < mp; ++q)
            mean += pmean[q] * D[static_cast<size_t>(base + q) * n + j];
          mean /= vol;
          for (long long c = 0; c < L.ncells(); ++c)
            Ginv[static_cast<size_t>(base + c * np) * n + j] -= mean;
        }
    }
  // H = G C with the jump coupling C: rhs_{a, v} += lv_a (M_h v_prev),
  // constrained rows zero (coupling_rhs, st_operator.cpp:409-421); C is
  // sparse, so H accumulates G's columns over C's nonzeros
  H.assign(static_cast<size_t>(n) * mv, 0.0);
  for (int a = 0; a < S; ++a)
    for (long long i = 0; i < mv; ++i)
      {
        if (vbnd(i))
          continue;
        const long long c = i / nsc, s = i % nsc, q = a * mv + i;
        for (long long s2 = 0; s2 < nsc; ++s2)
          {
            const double cv = T.lv[a] * Ms[s * nsc + s2];
            if (cv == 0.0)
              continue;
            const long long j = c * nsc + s2;
            for (int r = 0; r < n; ++r)
              H[static_cast<size_t>(r) * mv + j] += Ginv[static_cast<size_t>(r) * n + q] * cv;
          }
      }
}

DevGeom3
geom3(const Level3Spec &L)
{
  DevGeom3 g{};
  g.nx = L.nx;
  g.ny = L.ny;
  g.nz = L.nz;
  g.gx = L.gx();
  g.gy = L.gy();
  g.gz = L.gz();
  g.zlo = L.zlo();
  g.zhi = L.zhi();
  g.S = L.S();
  g.np = L.np();
  g.nsc = L.nsc();
  g.mv = L.mv();
  g.mp = L.mp();
  g.isz = L.isz();
  return g;
}

} // namespace stmg_b200
