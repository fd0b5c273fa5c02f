// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/include/oracle/oracle.hpp).
//
// 3D extension of the CPU restatement (BASELINE configs C3 and C5). The
// reference is 2D only (dof_space.hpp:30, mesh.hpp:30-33); SURVEY.md §9
// prescribes extending it "by tensor product" and marks 3D parity as
// UNPINNED by the reference. This file therefore restates the reference's
// algorithms in 3D as directly as possible and computes everything in the
// plainest form available, independent of the GPU's sum factorisation:
//
//  * element matrices by full Gauss quadrature (r+2 points per direction,
//    st_operator.cpp:167) on each cell, with the trilinear (Q1) geometry map
//    of the cell (mapped Q_{r+1}^d / mapped P_r^disc;
//    Cartesian cells are the special case of undeformed vertices);
//  * the spatial operators assembled into sparse matrices
//    (assemble_sparse_oracle, st_operator.cpp:469-554) and applied as SpMV
//    inside the reference's apply_block_impl (st_operator.cpp:321-407) and
//    coupling_rhs (st_operator.cpp:409-421);
//  * cell Vanka (vanka.cpp:30-233): patch dofs as in vanka.cpp:69-86, local
//    matrices R_T S R_T^T read out of the assembled operator, LU with the
//    rcond < 1e-12 fall-back to the minimum-norm solve (vanka.cpp:167-176);
//  * transfers (transfer.cpp:36-132, 148-402) in 3D: GLL interpolation of the
//    coarse cell polynomial, L2 re-expansion of the pressure on children,
//    modal embedding for p, Radau-node evaluation for p in time, and the
//    temporal h-transfer of PAPER.md Eq. DeftPrRe (coarse interval = two fine
//    intervals, canonical injection; restriction = transpose);
//  * pinned direct coarse solve (solver.cpp:10-54) and an exact "time-marched"
//    solve of the all-at-once system by the same pinned direct solve per
//    interval, which pins the all-at-once FGMRES solution;
//  * the all-at-once V-cycle (solver.cpp:69-93 with Eq. GloSys residuals and
//    exact forward substitution on the coarse time grid) and the reference's
//    GMRES (solver.cpp:95-202) around it.
#include "oracle/oracle.hpp"

#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <string>

namespace oracle
{
namespace o3
{
namespace
{
struct Csr
{
  Index rows = 0, cols = 0;
  std::vector<Index> ptr, col;
  Vec val;
  void
  mult_add(const double *x, double *y, double s = 1.0) const
  {
    for (Index i = 0; i < rows; ++i)
      {
        double acc = 0.0;
        for (Index e = ptr[i]; e < ptr[i + 1]; ++e)
          acc += val[e] * x[col[e]];
        y[i] += s * acc;
      }
  }
  void
  mult_t_add(const double *x, double *y, double s = 1.0) const
  {
    for (Index i = 0; i < rows; ++i)
      for (Index e = ptr[i]; e < ptr[i + 1]; ++e)
        y[col[e]] += s * val[e] * x[i];
  }
  double
  at(Index i, Index j) const
  {
    auto b = col.begin() + ptr[i], e = col.begin() + ptr[i + 1];
    auto it = std::lower_bound(b, e, j);
    return (it != e && *it == j) ? val[it - col.begin()] : 0.0;
  }
};

struct Builder
{
  Index rows, cols;
  std::vector<std::map<Index, double>> r;
  Builder(Index nr, Index nc) : rows(nr), cols(nc), r(nr) {}
  void add(Index i, Index j, double v) { r[i][j] += v; }
  Csr
  done()
  {
    Csr m;
    m.rows = rows;
    m.cols = cols;
    m.ptr.assign(rows + 1, 0);
    for (Index i = 0; i < rows; ++i)
      {
        for (auto &kv : r[i])
          {
            m.col.push_back(kv.first);
            m.val.push_back(kv.second);
          }
        m.ptr[i + 1] = static_cast<Index>(m.col.size());
      }
    return m;
  }
};

/// 3D P_r^disc mode exponents, degree-major (pdisc.cpp:41-55, dim = 3).
std::vector<std::array<int, 3>>
pdisc3(int r)
{
  std::vector<std::array<int, 3>> e;
  for (int deg = 0; deg <= r; ++deg)
    for (int a = deg; a >= 0; --a)
      for (int b = deg - a; b >= 0; --b)
        e.push_back({a, b, deg - a - b});
  return e;
}
double
leg(int n, double x)
{
  return legendre_values(n, x)[n];
}
} // namespace

/// One level: mesh (nx, ny, nz) cells on the unit cube with optional vertex
/// coordinates (deformed Q1 geometry), Q_{r+1}^3 / P_r^disc, DG(k) in time.
struct Level3
{
  int nx, ny, nz, r, k, n1, p, np, S;
  double tau, nu, gamma;
  int gx, gy, gz;
  Index nsc, mv, mp, isz;
  Vec verts; // (nx+1)(ny+1)(nz+1) x 3
  TemporalMatrices tm;
  std::vector<char> bnd;
  Csr Ms, A, B; // scalar mass (nsc x nsc), velocity stiffness (mv x mv), divergence (mp x mv)
  Vec pmean;    // int_K psi_l (mp)
  double vol = 0.0;
  // Vanka (cell patches)
  struct Patch
  {
    std::vector<Index> dofs;
    Vec weights;
    Mat inv; // dense inverse or pseudo-inverse
  };
  std::vector<Patch> patches;
  bool has_smoother = false;

  Index vid(int comp, int X, int Y, int Z) const { return comp * nsc + (static_cast<Index>(Z) * gy + Y) * gx + X; }
  Index cell_id(int cx, int cy, int cz) const { return (static_cast<Index>(cz) * ny + cy) * nx + cx; }
  double vtx(int vx, int vy, int vz, int d) const
  {
    return verts[((static_cast<Index>(vz) * (ny + 1) + vy) * (nx + 1) + vx) * 3 + d];
  }

  Level3(int nx_, int ny_, int nz_, int r_, int k_, double tau_, double nu_, double gamma_, const double *v)
    : nx(nx_), ny(ny_), nz(nz_), r(r_), k(k_), tau(tau_), nu(nu_), gamma(gamma_)
  {
    if (nx < 1 || ny < 1 || nz < 1 || r < 1 || r > 4 || k < 0 || k > 4 || !(tau > 0.0))
      throw std::invalid_argument("Level3: bad parameters");
    n1 = r + 2;
    p = r + 1;
    S = k + 1;
    np = static_cast<int>(pdisc3(r).size());
    gx = nx * p + 1;
    gy = ny * p + 1;
    gz = nz * p + 1;
    nsc = static_cast<Index>(gx) * gy * gz;
    mv = 3 * nsc;
    mp = static_cast<Index>(nx) * ny * nz * np;
    isz = S * (mv + mp);
    const Index nvert = static_cast<Index>(nx + 1) * (ny + 1) * (nz + 1);
    verts.resize(nvert * 3);
    if (v)
      std::copy(v, v + nvert * 3, verts.begin());
    else
      for (int vz = 0; vz <= nz; ++vz)
        for (int vy = 0; vy <= ny; ++vy)
          for (int vx = 0; vx <= nx; ++vx)
            {
              const Index i = ((static_cast<Index>(vz) * (ny + 1) + vy) * (nx + 1) + vx) * 3;
              verts[i] = static_cast<double>(vx) / nx;
              verts[i + 1] = static_cast<double>(vy) / ny;
              verts[i + 2] = static_cast<double>(vz) / nz;
            }
    tm = temporal_matrices(k, tau);
    bnd.assign(nsc, 0);
    for (int Z = 0; Z < gz; ++Z)
      for (int Y = 0; Y < gy; ++Y)
        for (int X = 0; X < gx; ++X)
          if (X == 0 || Y == 0 || Z == 0 || X == gx - 1 || Y == gy - 1 || Z == gz - 1)
            bnd[(static_cast<Index>(Z) * gy + Y) * gx + X] = 1;
    assemble();
  }

  void
  assemble()
  {
    const Vec gll = gauss_lobatto_points(n1);
    const NodalBasis1D b1(gll);
    const QuadratureRule q = gauss_rule(n1);
    const int nq = q.size();
    const auto ex = pdisc3(r);
    const int nv = n1 * n1 * n1;
    Builder bm(nsc, nsc), ba(mv, mv), bb(mp, mv);
    pmean.assign(mp, 0.0);
    vol = 0.0;
    std::vector<double> phi(nv), g(3 * nv), gp(3 * nv), psi(np);
    for (int cz = 0; cz < nz; ++cz)
      for (int cy = 0; cy < ny; ++cy)
        for (int cx = 0; cx < nx; ++cx)
          {
            const Index cell = cell_id(cx, cy, cz);
            double X8[8][3];
            for (int c = 0; c < 8; ++c)
              for (int d = 0; d < 3; ++d)
                X8[c][d] = vtx(cx + (c & 1), cy + ((c >> 1) & 1), cz + (c >> 2), d);
            std::vector<Index> sid(nv);
            for (int kk = 0; kk < n1; ++kk)
              for (int j = 0; j < n1; ++j)
                for (int i = 0; i < n1; ++i)
                  sid[(kk * n1 + j) * n1 + i] =
                    (static_cast<Index>(cz * p + kk) * gy + (cy * p + j)) * gx + (cx * p + i);
            std::vector<double> Me(nv * nv, 0.0), Ae(9 * nv * nv, 0.0), Be(np * 3 * nv, 0.0);
            for (int qz = 0; qz < nq; ++qz)
              for (int qy = 0; qy < nq; ++qy)
                for (int qx = 0; qx < nq; ++qx)
                  {
                    const double xi[3] = {q.points[qx], q.points[qy], q.points[qz]};
                    const double w = q.weights[qx] * q.weights[qy] * q.weights[qz];
                    // trilinear Jacobian J(d, e) = dX_d / dxi_e
                    double J[3][3] = {};
                    for (int c = 0; c < 8; ++c)
                      {
                        const int s[3] = {c & 1, (c >> 1) & 1, c >> 2};
                        double nval[3], nder[3];
                        for (int e = 0; e < 3; ++e)
                          {
                            nval[e] = s[e] ? 0.5 * (1 + xi[e]) : 0.5 * (1 - xi[e]);
                            nder[e] = s[e] ? 0.5 : -0.5;
                          }
                        const double dN[3] = {nder[0] * nval[1] * nval[2], nval[0] * nder[1] * nval[2],
                                              nval[0] * nval[1] * nder[2]};
                        for (int d = 0; d < 3; ++d)
                          for (int e = 0; e < 3; ++e)
                            J[d][e] += X8[c][d] * dN[e];
                      }
                    const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                                       J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                                       J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
                    if (!(det > 0.0))
                      throw std::runtime_error("Level3: inverted cell");
                    double Ji[3][3]; // Ji(e, d) = dxi_e / dX_d
                    Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
                    Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
                    Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
                    Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
                    Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
                    Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
                    Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
                    Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
                    Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
                    const double wd = w * det;
                    for (int kk = 0; kk < n1; ++kk)
                      for (int j = 0; j < n1; ++j)
                        for (int i = 0; i < n1; ++i)
                          {
                            const int t = (kk * n1 + j) * n1 + i;
                            const double v0 = b1.value(i, xi[0]), v1 = b1.value(j, xi[1]), v2 = b1.value(kk, xi[2]);
                            const double d0 = b1.derivative(i, xi[0]), d1 = b1.derivative(j, xi[1]),
                                         d2 = b1.derivative(kk, xi[2]);
                            phi[t] = v0 * v1 * v2;
                            const double gr[3] = {d0 * v1 * v2, v0 * d1 * v2, v0 * v1 * d2};
                            for (int d = 0; d < 3; ++d)
                              gp[3 * t + d] = gr[0] * Ji[0][d] + gr[1] * Ji[1][d] + gr[2] * Ji[2][d];
                          }
                    for (int l = 0; l < np; ++l)
                      psi[l] = leg(ex[l][0], xi[0]) * leg(ex[l][1], xi[1]) * leg(ex[l][2], xi[2]);
                    for (int l = 0; l < np; ++l)
                      pmean[cell * np + l] += wd * psi[l];
                    vol += wd;
                    for (int a = 0; a < nv; ++a)
                      for (int b = 0; b < nv; ++b)
                        {
                          Me[a * nv + b] += wd * phi[a] * phi[b];
                          const double gg = gp[3 * a] * gp[3 * b] + gp[3 * a + 1] * gp[3 * b + 1] +
                                            gp[3 * a + 2] * gp[3 * b + 2];
                          for (int c = 0; c < 3; ++c)
                            for (int c2 = 0; c2 < 3; ++c2)
                              {
                                double v = gamma * gp[3 * a + c] * gp[3 * b + c2];
                                if (c == c2)
                                  v += nu * gg;
                                Ae[(c * nv + a) * 3 * nv + c2 * nv + b] += wd * v;
                              }
                        }
                    for (int l = 0; l < np; ++l)
                      for (int c = 0; c < 3; ++c)
                        for (int b = 0; b < nv; ++b)
                          Be[l * 3 * nv + c * nv + b] += wd * psi[l] * gp[3 * b + c];
                  }
            for (int a = 0; a < nv; ++a)
              for (int b = 0; b < nv; ++b)
                bm.add(sid[a], sid[b], Me[a * nv + b]);
            for (int c = 0; c < 3; ++c)
              for (int a = 0; a < nv; ++a)
                for (int c2 = 0; c2 < 3; ++c2)
                  for (int b = 0; b < nv; ++b)
                    ba.add(c * nsc + sid[a], c2 * nsc + sid[b], Ae[(c * nv + a) * 3 * nv + c2 * nv + b]);
            for (int l = 0; l < np; ++l)
              for (int c = 0; c < 3; ++c)
                for (int b = 0; b < nv; ++b)
                  bb.add(cell * np + l, c * nsc + sid[b], Be[l * 3 * nv + c * nv + b]);
          }
    Ms = bm.done();
    A = ba.done();
    B = bb.done();
  }

  void
  zero_constrained(double *v) const
  {
    for (int c = 0; c < 3; ++c)
      for (Index s = 0; s < nsc; ++s)
        if (bnd[s])
          v[c * nsc + s] = 0.0;
  }
  /// PressureSpace::project_mean_zero (dof_space.cpp:110-119) with the mapped
  /// basis: mean = <int psi, p> / |Omega|, subtracted from the coefficient of
  /// the constant mode (psi_0 = 1) of every cell.
  void
  project_mean_zero(double *pr) const
  {
    double m = 0.0;
    for (Index i = 0; i < mp; ++i)
      m += pmean[i] * pr[i];
    m /= vol;
    for (Index c = 0; c < mp / np; ++c)
      pr[c * np] -= m;
  }
  /// Residual (dual) vectors: remove the component along the left null
  /// vector of the pressure rows, the constant-mode coefficients
  /// (one_coefficients). On Cartesian meshes this is project_mean_zero
  /// (|K| is uniform); on deformed meshes the |K|-weighted mean would leave
  /// the restricted residual inconsistent.
  void
  project_residual(double *pr) const
  {
    const Index nc = mp / np;
    double m = 0.0;
    for (Index c = 0; c < nc; ++c)
      m += pr[c * np];
    m /= static_cast<double>(nc);
    for (Index c = 0; c < nc; ++c)
      pr[c * np] -= m;
  }
  void
  mass_apply(const double *v, double *y) const // y = M_h v (three components), overwrite
  {
    std::fill(y, y + mv, 0.0);
    for (int c = 0; c < 3; ++c)
      Ms.mult_add(v + c * nsc, y + c * nsc);
  }

  /// apply_block_impl (st_operator.cpp:321-407).
  void
  apply_block(const double *x, double *y, bool constrain) const
  {
    Vec xc(x, x + isz);
    if (constrain)
      for (int a = 0; a < S; ++a)
        zero_constrained(xc.data() + a * mv);
    std::vector<Vec> mvs(S, Vec(mv)), avs(S, Vec(mv, 0.0)), bvs(S, Vec(mp, 0.0)), btp(S, Vec(mv, 0.0));
    for (int b = 0; b < S; ++b)
      {
        const double *u = xc.data() + b * mv;
        const double *pr = xc.data() + S * mv + b * mp;
        mass_apply(u, mvs[b].data());
        A.mult_add(u, avs[b].data());
        B.mult_add(u, bvs[b].data());
        B.mult_t_add(pr, btp[b].data());
      }
    std::fill(y, y + isz, 0.0);
    for (int a = 0; a < S; ++a)
      for (int b = 0; b < S; ++b)
        {
          const double kt = tm.dt_plus_jump(a, b), mt = tm.mass(a, b);
          double *yv = y + a * mv;
          for (Index i = 0; i < mv; ++i)
            yv[i] += kt * mvs[b][i] + mt * avs[b][i] - mt * btp[b][i];
          double *yp = y + S * mv + a * mp;
          for (Index i = 0; i < mp; ++i)
            yp[i] += mt * bvs[b][i];
        }
    if (constrain)
      for (int a = 0; a < S; ++a)
        for (int c = 0; c < 3; ++c)
          for (Index s = 0; s < nsc; ++s)
            if (bnd[s])
              y[a * mv + c * nsc + s] = x[a * mv + c * nsc + s];
  }

  /// y = D x - Z C v_prev (capi vmult_interval; coupling_rhs st_operator.cpp:409-421
  /// with constrained rows zeroed as time_march does, solver.cpp:267-268).
  void
  vmult_interval(const double *x, const double *vprev, double *y) const
  {
    apply_block(x, y, true);
    if (vprev)
      {
        Vec mw(mv);
        mass_apply(vprev, mw.data());
        zero_constrained(mw.data());
        for (int a = 0; a < S; ++a)
          for (Index i = 0; i < mv; ++i)
            y[a * mv + i] -= tm.left_values[a] * mw[i];
      }
  }

  double
  op_entry(Index i, Index j) const // entry of the (raw) interval operator S
  {
    const Index V = S * mv;
    if (i < V && j < V)
      {
        const int a = static_cast<int>(i / mv), b = static_cast<int>(j / mv);
        const Index li = i % mv, lj = j % mv;
        double v = tm.mass(a, b) * A.at(li, lj);
        if (li / nsc == lj / nsc)
          v += tm.dt_plus_jump(a, b) * Ms.at(li % nsc, lj % nsc);
        return v;
      }
    if (i < V && j >= V)
      {
        const int a = static_cast<int>(i / mv), b = static_cast<int>((j - V) / mp);
        return -tm.mass(a, b) * B.at((j - V) % mp, i % mv);
      }
    if (i >= V && j < V)
      {
        const int a = static_cast<int>((i - V) / mp), b = static_cast<int>(j / mv);
        return tm.mass(a, b) * B.at((i - V) % mp, j % mv);
      }
    return 0.0;
  }

  /// VankaSmoother::build for cell patches (vanka.cpp:30-194).
  void
  build_cell_vanka()
  {
    patches.clear();
    std::vector<int> valence(nsc, 0);
    for (int cz = 0; cz < nz; ++cz)
      for (int cy = 0; cy < ny; ++cy)
        for (int cx = 0; cx < nx; ++cx)
          for (int kk = 0; kk < n1; ++kk)
            for (int j = 0; j < n1; ++j)
              for (int i = 0; i < n1; ++i)
                valence[(static_cast<Index>(cz * p + kk) * gy + cy * p + j) * gx + cx * p + i]++;
    for (int cz = 0; cz < nz; ++cz)
      for (int cy = 0; cy < ny; ++cy)
        for (int cx = 0; cx < nx; ++cx)
          {
            std::vector<Index> sc;
            for (int kk = 0; kk < n1; ++kk)
              for (int j = 0; j < n1; ++j)
                for (int i = 0; i < n1; ++i)
                  {
                    const Index s = (static_cast<Index>(cz * p + kk) * gy + cy * p + j) * gx + cx * p + i;
                    if (!bnd[s])
                      sc.push_back(s);
                  }
            std::sort(sc.begin(), sc.end());
            Patch P;
            for (int a = 0; a < S; ++a)
              for (int c = 0; c < 3; ++c)
                for (Index s : sc)
                  {
                    P.dofs.push_back(a * mv + c * nsc + s);
                    P.weights.push_back(1.0 / valence[s]);
                  }
            const Index cell = cell_id(cx, cy, cz);
            for (int a = 0; a < S; ++a)
              for (int l = 0; l < np; ++l)
                {
                  P.dofs.push_back(S * mv + a * mp + cell * np + l);
                  P.weights.push_back(1.0);
                }
            const int n = static_cast<int>(P.dofs.size());
            Mat Al(n, n);
            for (int i = 0; i < n; ++i)
              for (int j = 0; j < n; ++j)
                Al(i, j) = op_entry(P.dofs[i], P.dofs[j]);
            LU lu(Al);
            if (!lu.singular && lu.rcond(Al) >= 1e-12)
              P.inv = lu.inverse();
            else
              P.inv = MinNormSolver(Al).pinv;
            patches.push_back(std::move(P));
          }
    has_smoother = true;
  }

  void
  apply_additive(const double *res, double *out) const
  {
    std::fill(out, out + isz, 0.0);
    for (const Patch &P : patches)
      {
        const int n = static_cast<int>(P.dofs.size());
        Vec rl(n), z(n, 0.0);
        for (int i = 0; i < n; ++i)
          rl[i] = res[P.dofs[i]];
        for (int i = 0; i < n; ++i)
          {
            double acc = 0.0;
            for (int j = 0; j < n; ++j)
              acc += P.inv(i, j) * rl[j];
            z[i] = acc;
          }
        for (int i = 0; i < n; ++i)
          out[P.dofs[i]] += P.weights[i] * z[i];
      }
  }

  /// Dense interval operator with the first pressure dof of each slot pinned
  /// (CoarseSolver, solver.cpp:10-41), constrained rows identity.
  Mat
  pinned_dense() const
  {
    Mat D(static_cast<int>(isz), static_cast<int>(isz));
    Vec e(isz, 0.0), col(isz);
    for (Index j = 0; j < isz; ++j)
      {
        e[j] = 1.0;
        apply_block(e.data(), col.data(), true);
        e[j] = 0.0;
        for (Index i = 0; i < isz; ++i)
          D(static_cast<int>(i), static_cast<int>(j)) = col[i];
      }
    for (int a = 0; a < S; ++a)
      {
        const Index pin = S * mv + a * mp;
        for (Index j = 0; j < isz; ++j)
          D(static_cast<int>(pin), static_cast<int>(j)) = 0.0;
        D(static_cast<int>(pin), static_cast<int>(pin)) = 1.0;
      }
    return D;
  }
};

/// Transfer between two levels (coarse c, fine f); spatial part (h: nx_f =
/// 2 nx_c, or p: r_c = r_f / 2 on the same mesh, or none) and temporal part
/// (p: k_c < k_f, and/or h: N_f = 2 N_c).
struct Transfer3
{
  const Level3 *c, *f;
  bool spatial = false, h_time = false;
  Csr Pv, Pp;           // scalar velocity (nsc_f x nsc_c), pressure (mp_f x mp_c)
  Mat E[2];             // fine slot x coarse slot, for the left / right half (h_time) or E[0]
  Transfer3(const Level3 &cl, const Level3 &fl, bool htime) : c(&cl), f(&fl), h_time(htime)
  {
    const bool h_sp = fl.nx == 2 * cl.nx && fl.ny == 2 * cl.ny && fl.nz == 2 * cl.nz && fl.r == cl.r;
    const bool p_sp = fl.nx == cl.nx && fl.ny == cl.ny && fl.nz == cl.nz && fl.r != cl.r;
    const bool none = fl.nx == cl.nx && fl.ny == cl.ny && fl.nz == cl.nz && fl.r == cl.r;
    if (!(h_sp || p_sp || none))
      throw std::invalid_argument("Transfer3: unsupported level pair");
    spatial = !none;
    if (spatial)
      build_spatial(h_sp);
    // temporal: E(a, b) = coarse Lagrange basis b (Radau nodes) at fine node a
    const NodalBasis1D bc(cl.tm.nodes);
    for (int half = 0; half < (h_time ? 2 : 1); ++half)
      {
        E[half] = Mat(fl.S, cl.S);
        for (int a = 0; a < fl.S; ++a)
          {
            double t = fl.tm.nodes[a];
            if (h_time)
              t = half == 0 ? 0.5 * (t - 1.0) : 0.5 * (t + 1.0);
            for (int b = 0; b < cl.S; ++b)
              E[half](a, b) = cl.S == 1 ? 1.0 : bc.value(b, t);
          }
      }
  }

  void
  build_spatial(bool h)
  {
    const Level3 &C = *c, &F = *f;
    const NodalBasis1D bcv(gauss_lobatto_points(C.n1));
    const Vec gf = gauss_lobatto_points(F.n1);
    Builder bv(F.nsc, C.nsc), bp(F.mp, C.mp);
    const int ratio = h ? 2 : 1;
    // velocity: every fine node takes the coarse cell polynomial of (one of)
    // its coarse cells at its reference position (transfer.cpp:168-175)
    std::vector<char> done(F.nsc, 0);
    for (int fz = 0; fz < F.nz; ++fz)
      for (int fy = 0; fy < F.ny; ++fy)
        for (int fx = 0; fx < F.nx; ++fx)
          {
            const int ccx = fx / ratio, ccy = fy / ratio, ccz = fz / ratio;
            const int off[3] = {fx % ratio, fy % ratio, fz % ratio};
            for (int kk = 0; kk < F.n1; ++kk)
              for (int j = 0; j < F.n1; ++j)
                for (int i = 0; i < F.n1; ++i)
                  {
                    const Index s = (static_cast<Index>(fz * F.p + kk) * F.gy + fy * F.p + j) * F.gx + fx * F.p + i;
                    if (done[s])
                      continue;
                    done[s] = 1;
                    const int li[3] = {i, j, kk};
                    double xc[3];
                    for (int d = 0; d < 3; ++d)
                      xc[d] = h ? 0.5 * (gf[li[d]] + (off[d] == 0 ? -1.0 : 1.0)) : gf[li[d]];
                    for (int c2 = 0; c2 < C.n1; ++c2)
                      for (int b2 = 0; b2 < C.n1; ++b2)
                        for (int a2 = 0; a2 < C.n1; ++a2)
                          {
                            const double v = bcv.value(a2, xc[0]) * bcv.value(b2, xc[1]) * bcv.value(c2, xc[2]);
                            if (v != 0.0)
                              bv.add(s, (static_cast<Index>(ccz * C.p + c2) * C.gy + ccy * C.p + b2) * C.gx +
                                          ccx * C.p + a2,
                                     v);
                          }
                  }
          }
    // pressure: L2 re-expansion of the coarse modes on each fine cell in
    // reference coordinates (transfer.cpp:225-253); for p the coarse modes
    // embed into the fine ones (transfer.cpp:338-359) -- the same formula.
    const auto exc = pdisc3(C.r), exf = pdisc3(F.r);
    const QuadratureRule q = gauss_rule(F.r + 2);
    for (int fz = 0; fz < F.nz; ++fz)
      for (int fy = 0; fy < F.ny; ++fy)
        for (int fx = 0; fx < F.nx; ++fx)
          {
            const int off[3] = {fx % ratio, fy % ratio, fz % ratio};
            const Index fc = F.cell_id(fx, fy, fz), cc = C.cell_id(fx / ratio, fy / ratio, fz / ratio);
            for (int lf = 0; lf < F.np; ++lf)
              for (int lc = 0; lc < C.np; ++lc)
                {
                  double acc = 0.0;
                  for (int qz = 0; qz < q.size(); ++qz)
                    for (int qy = 0; qy < q.size(); ++qy)
                      for (int qx = 0; qx < q.size(); ++qx)
                        {
                          const double xf[3] = {q.points[qx], q.points[qy], q.points[qz]};
                          double xcp[3];
                          for (int d = 0; d < 3; ++d)
                            xcp[d] = h ? 0.5 * (xf[d] + (off[d] == 0 ? -1.0 : 1.0)) : xf[d];
                          acc += q.weights[qx] * q.weights[qy] * q.weights[qz] * leg(exf[lf][0], xf[0]) *
                                 leg(exf[lf][1], xf[1]) * leg(exf[lf][2], xf[2]) * leg(exc[lc][0], xcp[0]) *
                                 leg(exc[lc][1], xcp[1]) * leg(exc[lc][2], xcp[2]);
                        }
                  double gram = 1.0;
                  for (int d = 0; d < 3; ++d)
                    gram *= 2.0 / (2.0 * exf[lf][d] + 1.0);
                  acc /= gram;
                  if (std::abs(acc) > 1e-14)
                    bp.add(fc * F.np + lf, cc * C.np + lc, acc);
                }
          }
    Pv = bv.done();
    Pp = bp.done();
  }

  int n_fine(int nc) const { return h_time ? 2 * nc : nc; }

  /// Prolongation of nc coarse intervals (transfer.cpp:51-75 + Eq. DeftPrRe).
  void
  prolongate(const double *xc, double *xf, int nc) const
  {
    const Level3 &C = *c, &F = *f;
    const int nf = n_fine(nc);
    std::fill(xf, xf + F.isz * nf, 0.0);
    Vec sv(F.mv), sp(F.mp);
    for (int n = 0; n < nf; ++n)
      {
        const int m = h_time ? n / 2 : n;
        const Mat &Em = E[h_time ? (n & 1) : 0];
        for (int b = 0; b < C.S; ++b)
          {
            const double *cv = xc + m * C.isz + b * C.mv;
            const double *cp = xc + m * C.isz + C.S * C.mv + b * C.mp;
            if (spatial)
              {
                std::fill(sv.begin(), sv.end(), 0.0);
                std::fill(sp.begin(), sp.end(), 0.0);
                for (int comp = 0; comp < 3; ++comp)
                  Pv.mult_add(cv + comp * C.nsc, sv.data() + comp * F.nsc);
                Pp.mult_add(cp, sp.data());
              }
            else
              {
                std::copy(cv, cv + C.mv, sv.begin());
                std::copy(cp, cp + C.mp, sp.begin());
              }
            for (int a = 0; a < F.S; ++a)
              {
                const double e = Em(a, b);
                double *fv = xf + n * F.isz + a * F.mv;
                double *fp = xf + n * F.isz + F.S * F.mv + a * F.mp;
                for (Index i = 0; i < F.mv; ++i)
                  fv[i] += e * sv[i];
                for (Index i = 0; i < F.mp; ++i)
                  fp[i] += e * sp[i];
              }
          }
      }
  }

  /// Restriction = transpose of the prolongation (transfer.cpp:77-100).
  void
  restrict_(const double *xf, double *xc, int nc) const
  {
    const Level3 &C = *c, &F = *f;
    const int nf = n_fine(nc);
    std::fill(xc, xc + C.isz * nc, 0.0);
    Vec tv(F.mv), tp(F.mp);
    for (int n = 0; n < nf; ++n)
      {
        const int m = h_time ? n / 2 : n;
        const Mat &Em = E[h_time ? (n & 1) : 0];
        for (int b = 0; b < C.S; ++b)
          {
            std::fill(tv.begin(), tv.end(), 0.0);
            std::fill(tp.begin(), tp.end(), 0.0);
            for (int a = 0; a < F.S; ++a)
              {
                const double e = Em(a, b);
                const double *fv = xf + n * F.isz + a * F.mv;
                const double *fp = xf + n * F.isz + F.S * F.mv + a * F.mp;
                for (Index i = 0; i < F.mv; ++i)
                  tv[i] += e * fv[i];
                for (Index i = 0; i < F.mp; ++i)
                  tp[i] += e * fp[i];
              }
            double *cv = xc + m * C.isz + b * C.mv;
            double *cp = xc + m * C.isz + C.S * C.mv + b * C.mp;
            if (spatial)
              {
                for (int comp = 0; comp < 3; ++comp)
                  Pv.mult_t_add(tv.data() + comp * F.nsc, cv + comp * C.nsc);
                Pp.mult_t_add(tp.data(), cp);
              }
            else
              {
                for (Index i = 0; i < C.mv; ++i)
                  cv[i] += tv[i];
                for (Index i = 0; i < C.mp; ++i)
                  cp[i] += tp[i];
              }
          }
      }
  }
};

/// hp-STMG hierarchy for the all-at-once system (C3/C5 plan):
/// coarse first. Each level: mesh, r, k, number of intervals relative to
/// the finest (time coarsening), tau.
struct Hier3
{
  std::vector<std::unique_ptr<Level3>> L;
  std::vector<int> tshift; // log2(N_fine / N_l)
  std::vector<std::unique_ptr<Transfer3>> T; // T[l]: l-1 <- l (T[0] unused)
  Mat coarse_inv;                            // pinned inverse of level 0
  Mat coarse_C;                              // level-0 coupling: rows isz, cols mv (D x_t -= C v)
  int nu1 = 2, nu2 = 2;
  double omega = 0.8;

  void
  finish()
  {
    T.clear();
    T.push_back(nullptr);
    for (size_t l = 1; l < L.size(); ++l)
      T.push_back(std::make_unique<Transfer3>(*L[l - 1], *L[l], tshift[l - 1] > tshift[l]));
    for (size_t l = 1; l < L.size(); ++l)
      L[l]->build_cell_vanka();
    const Level3 &c = *L[0];
    Mat D = c.pinned_dense();
    LU lu(D);
    if (lu.singular)
      throw std::runtime_error("Hier3: singular coarse matrix");
    coarse_inv = lu.inverse();
  }

  /// CoarseSolver::solve for one interval of level 0 (solver.cpp:43-54).
  void
  coarse_solve(const double *b, double *x) const
  {
    const Level3 &c = *L[0];
    Vec rhs(b, b + c.isz);
    for (int a = 0; a < c.S; ++a)
      rhs[c.S * c.mv + a * c.mp] = 0.0;
    for (Index i = 0; i < c.isz; ++i)
      {
        double acc = 0.0;
        for (Index j = 0; j < c.isz; ++j)
          acc += coarse_inv(static_cast<int>(i), static_cast<int>(j)) * rhs[j];
        x[i] = acc;
      }
    for (int a = 0; a < c.S; ++a)
      c.project_mean_zero(x + c.S * c.mv + a * c.mp);
  }

  /// Exact all-at-once solve on level 0 by forward substitution in time:
  /// x_t = CoarseSolve(b_t + Z C v_{t-1}).
  void
  coarse_forward(const double *b, double *x, int n) const
  {
    const Level3 &c = *L[0];
    Vec rhs(c.isz), mw(c.mv);
    for (int t = 0; t < n; ++t)
      {
        std::copy(b + t * c.isz, b + (t + 1) * c.isz, rhs.begin());
        if (t > 0)
          {
            c.mass_apply(x + (t - 1) * c.isz + (c.S - 1) * c.mv, mw.data());
            c.zero_constrained(mw.data());
            for (int a = 0; a < c.S; ++a)
              for (Index i = 0; i < c.mv; ++i)
                rhs[a * c.mv + i] += c.tm.left_values[a] * mw[i];
          }
        coarse_solve(rhs.data(), x + t * c.isz);
      }
  }

  void
  residual(int l, const double *b, const double *x, double *res, int n) const
  {
    const Level3 &lv = *L[l];
    for (int t = 0; t < n; ++t)
      {
        lv.vmult_interval(x + t * lv.isz, t > 0 ? x + (t - 1) * lv.isz + (lv.S - 1) * lv.mv : nullptr,
                          res + t * lv.isz);
        for (Index i = 0; i < lv.isz; ++i)
          res[t * lv.isz + i] = b[t * lv.isz + i] - res[t * lv.isz + i];
      }
  }

  void
  smooth(int l, const double *b, double *x, int n) const
  {
    const Level3 &lv = *L[l];
    Vec res(lv.isz * n), z(lv.isz);
    residual(l, b, x, res.data(), n);
    for (int t = 0; t < n; ++t)
      {
        lv.apply_additive(res.data() + t * lv.isz, z.data());
        for (Index i = 0; i < lv.isz; ++i)
          x[t * lv.isz + i] += omega * z[i];
      }
  }

  void
  project_slots(const Level3 &lv, double *x, int n, bool residual) const
  {
    for (int t = 0; t < n; ++t)
      for (int a = 0; a < lv.S; ++a)
        {
          lv.zero_constrained(x + t * lv.isz + a * lv.mv);
          if (residual)
            lv.project_residual(x + t * lv.isz + lv.S * lv.mv + a * lv.mp);
          else
            lv.project_mean_zero(x + t * lv.isz + lv.S * lv.mv + a * lv.mp);
        }
  }

  /// All-at-once VCycle::cycle (solver.cpp:69-93), n = intervals on level l.
  void
  cycle(int l, const double *b, double *x, int n) const
  {
    const Level3 &lv = *L[l];
    if (l == 0)
      {
        coarse_forward(b, x, n);
        return;
      }
    std::fill(x, x + lv.isz * n, 0.0);
    for (int s = 0; s < nu1; ++s)
      smooth(l, b, x, n);
    Vec res(lv.isz * n);
    residual(l, b, x, res.data(), n);
    const Transfer3 &tr = *T[l];
    const int nc = tr.h_time ? n / 2 : n;
    const Level3 &cl = *L[l - 1];
    Vec bc(cl.isz * nc), xc(cl.isz * nc), corr(lv.isz * n);
    tr.restrict_(res.data(), bc.data(), nc);
    project_slots(cl, bc.data(), nc, true);
    cycle(l - 1, bc.data(), xc.data(), nc);
    tr.prolongate(xc.data(), corr.data(), nc);
    project_slots(lv, corr.data(), n, false);
    for (Index i = 0; i < lv.isz * n; ++i)
      x[i] += corr[i];
    for (int s = 0; s < nu2; ++s)
      smooth(l, b, x, n);
  }
};

int g_kmin = 0; // lowest temporal degree of the p-coarsening (0: k -> ... -> 0)

/// Default C3-type plan: finest (nx,ny,nz, r, k, N); p-coarsen k -> 0 (via
/// k/2 steps), then h-coarsen space and time together while the mesh and N
/// stay even and above (cmin, nmin).
std::unique_ptr<Hier3>
plan(int nx, int ny, int nz, int r, int k, int N, double t_end, double nu, double gamma, int n_hcoarse,
     int time_coarsen, const double *verts)
{
  struct Desc
  {
    int nx, ny, nz, r, k, tsh;
  };
  // combine_hierarchies (hierarchy.cpp:9-97, harness.cpp:26-42) in 3D: the
  // spatial list (fine first: p-halving of r, then h-steps, each h-step also
  // halving the time grid when time_coarsen) and the temporal list (k, k/2,
  // ..., k_min) are aligned at the COARSE end, so the temporal p-steps sit on
  // the coarsest levels (as the reference's C2 plan: L1 = h_space + p_time).
  std::vector<Desc> sp; // spatial, fine first (k filled below)
  sp.push_back({nx, ny, nz, r, 0, 0});
  while (sp.back().r > 1)
    {
      Desc e = sp.back();
      e.r = e.r / 2;
      sp.push_back(e);
    }
  for (int i = 0; i < n_hcoarse; ++i)
    {
      Desc e = sp.back();
      if (e.nx % 2 || e.ny % 2 || e.nz % 2)
        throw std::invalid_argument("plan: mesh not divisible");
      e.nx /= 2;
      e.ny /= 2;
      e.nz /= 2;
      if (time_coarsen)
        e.tsh += 1;
      sp.push_back(e);
    }
  std::vector<int> tk{k}; // temporal, fine first
  while (tk.back() > g_kmin)
    tk.push_back(tk.back() / 2);
  const size_t L = std::max(sp.size(), tk.size());
  std::vector<Desc> d(L); // fine first
  for (size_t i = 0; i < L; ++i)
    {
      // index from the coarse end: c = L - 1 - i
      const size_t c = L - 1 - i;
      Desc e = sp[std::min(sp.size() - 1, i)];
      e.k = tk[tk.size() - 1 - std::min(c, tk.size() - 1)];
      d[i] = e;
    }
  auto H = std::make_unique<Hier3>();
  const double tau = t_end / N;
  for (auto it = d.rbegin(); it != d.rend(); ++it)
    {
      const bool finest = (it == d.rend() - 1);
      H->L.push_back(std::make_unique<Level3>(it->nx, it->ny, it->nz, it->r, it->k, tau * (1 << it->tsh), nu, gamma,
                                              finest ? verts : nullptr));
      H->tshift.push_back(it->tsh);
    }
  // coarser geometry: the fine vertices restricted to the coarse vertex set
  for (size_t l = H->L.size() - 1; l-- > 0;)
    {
      Level3 &c = *H->L[l];
      const Level3 &f = *H->L[l + 1];
      const int ratio = f.nx / c.nx;
      for (int vz = 0; vz <= c.nz; ++vz)
        for (int vy = 0; vy <= c.ny; ++vy)
          for (int vx = 0; vx <= c.nx; ++vx)
            for (int dd = 0; dd < 3; ++dd)
              c.verts[((static_cast<Index>(vz) * (c.ny + 1) + vy) * (c.nx + 1) + vx) * 3 + dd] =
                f.vtx(vx * ratio, vy * ratio, vz * ratio, dd);
      c.assemble();
    }
  H->finish();
  return H;
}

} // namespace o3
} // namespace oracle

// ---------------------------------------------------------------- C API
using oracle::Index;
using oracle::Vec;
using oracle::o3::Hier3;
using oracle::o3::Level3;

namespace
{
std::string g_err3;
template <class F>
int
guard3(F &&f)
{
  try
    {
      f();
      return 0;
    }
  catch (const std::invalid_argument &e)
    {
      g_err3 = e.what();
      return 1;
    }
  catch (const std::exception &e)
    {
      g_err3 = e.what();
      return 2;
    }
}
} // namespace

extern "C" {

const char *
o3_last_error()
{
  return g_err3.c_str();
}

int
o3_level_create(int nx, int ny, int nz, int r, int k, double tau, double nu, double gamma, const double *verts,
                int smoother, void **out)
{
  return guard3([&] {
    auto *L = new Level3(nx, ny, nz, r, k, tau, nu, gamma, verts);
    if (smoother >= 0)
      L->build_cell_vanka();
    *out = L;
  });
}

void
o3_level_destroy(void *h)
{
  delete static_cast<Level3 *>(h);
}

/// out: S, mv, mp, isz, nsc, gx, gy, gz, np
int
o3_level_sizes(void *h, long *out)
{
  const auto *L = static_cast<Level3 *>(h);
  const long v[9] = {L->S, L->mv, L->mp, L->isz, L->nsc, L->gx, L->gy, L->gz, L->np};
  std::memcpy(out, v, sizeof(v));
  return 0;
}

int
o3_apply_block(void *h, const double *x, double *y, int raw)
{
  return guard3([&] { static_cast<Level3 *>(h)->apply_block(x, y, raw == 0); });
}

int
o3_vmult_all(void *h, const double *x, double *y, int n, const double *xprev)
{
  return guard3([&] {
    const auto *L = static_cast<Level3 *>(h);
#pragma omp parallel for schedule(dynamic, 1)
    for (int t = 0; t < n; ++t)
      L->vmult_interval(x + t * L->isz, t == 0 ? xprev : x + (t - 1) * L->isz + (L->S - 1) * L->mv,
                        y + t * L->isz);
  });
}

int
o3_smooth_step_all(void *h, const double *b, double *u, double omega, int n, const double *xprev)
{
  return guard3([&] {
    const auto *L = static_cast<Level3 *>(h);
    if (!L->has_smoother)
      throw std::invalid_argument("no smoother");
    Vec uo(u, u + L->isz * n);
#pragma omp parallel for schedule(dynamic, 1)
    for (int t = 0; t < n; ++t)
      {
        Vec res(L->isz), z(L->isz);
        L->vmult_interval(uo.data() + t * L->isz, t == 0 ? xprev : uo.data() + (t - 1) * L->isz + (L->S - 1) * L->mv,
                          res.data());
        for (Index i = 0; i < L->isz; ++i)
          res[i] = b[t * L->isz + i] - res[i];
        L->apply_additive(res.data(), z.data());
        for (Index i = 0; i < L->isz; ++i)
          u[t * L->isz + i] += omega * z[i];
      }
  });
}

/// Patch info for the GPU class check: number of patches; patch i's dofs,
/// weights and inverse.
long
o3_patch_count(void *h)
{
  return static_cast<long>(static_cast<Level3 *>(h)->patches.size());
}

int
o3_project_mean_zero(void *h, double *p)
{
  return guard3([&] { static_cast<Level3 *>(h)->project_mean_zero(p); });
}

void
o3_set_kmin(int kmin)
{
  oracle::o3::g_kmin = kmin;
}

int
o3_project_residual(void *h, double *p)
{
  return guard3([&] { static_cast<Level3 *>(h)->project_residual(p); });
}

int
o3_hier_create(int nx, int ny, int nz, int r, int k, int N, double t_end, double nu, double gamma, int n_hcoarse,
               int time_coarsen, const double *verts, int nu1, int nu2, double omega, void **out)
{
  return guard3([&] {
    auto H = oracle::o3::plan(nx, ny, nz, r, k, N, t_end, nu, gamma, n_hcoarse, time_coarsen, verts);
    H->nu1 = nu1;
    H->nu2 = nu2;
    H->omega = omega;
    *out = H.release();
  });
}

void
o3_hier_destroy(void *h)
{
  delete static_cast<Hier3 *>(h);
}

/// out[0] = levels; per level: nx, ny, nz, r, k, tshift, isz
int
o3_hier_info(void *h, long *out)
{
  const auto *H = static_cast<Hier3 *>(h);
  out[0] = static_cast<long>(H->L.size());
  for (size_t l = 0; l < H->L.size(); ++l)
    {
      const Level3 &L = *H->L[l];
      long *o = out + 1 + 7 * l;
      o[0] = L.nx;
      o[1] = L.ny;
      o[2] = L.nz;
      o[3] = L.r;
      o[4] = L.k;
      o[5] = H->tshift[l];
      o[6] = L.isz;
    }
  return 0;
}

void *
o3_hier_level(void *h, int l)
{
  return static_cast<Hier3 *>(h)->L[l].get();
}

int
o3_hier_prolongate(void *h, int l, const double *xc, double *xf, int nc)
{
  return guard3([&] { static_cast<Hier3 *>(h)->T[l]->prolongate(xc, xf, nc); });
}

int
o3_hier_restrict(void *h, int l, const double *xf, double *xc, int nc)
{
  return guard3([&] { static_cast<Hier3 *>(h)->T[l]->restrict_(xf, xc, nc); });
}

int
o3_hier_coarse_forward(void *h, const double *b, double *x, int n)
{
  return guard3([&] { static_cast<Hier3 *>(h)->coarse_forward(b, x, n); });
}

/// One all-at-once V-cycle on the finest level with n intervals.
int
o3_hier_vcycle(void *h, const double *b, double *x, int n)
{
  return guard3([&] {
    const auto *H = static_cast<Hier3 *>(h);
    H->cycle(static_cast<int>(H->L.size()) - 1, b, x, n);
  });
}

/// FGMRES (solver.cpp:95-202) on the all-at-once system of n intervals,
/// preconditioned by the all-at-once V-cycle.
int
o3_hier_fgmres(void *h, const double *b, double *x, int n, double rtol, int maxit, int *iterations)
{
  return guard3([&] {
    const auto *H = static_cast<Hier3 *>(h);
    const Level3 &F = *H->L.back();
    const Index N = F.isz * n;
    oracle::BlockVector bv(1, N, 0), x0(1, N, 0);
    std::copy(b, b + N, bv.data.begin());
    oracle::KrylovConfig kc;
    kc.rtol = rtol;
    kc.max_iterations = maxit;
    kc.max_basis = maxit;
    auto apply = [&](const oracle::BlockVector &in, oracle::BlockVector &out) {
      out = oracle::BlockVector(1, N, 0);
      for (int t = 0; t < n; ++t)
        F.vmult_interval(in.data.data() + t * F.isz,
                         t > 0 ? in.data.data() + (t - 1) * F.isz + (F.S - 1) * F.mv : nullptr,
                         out.data.data() + t * F.isz);
    };
    auto pre = [&](const oracle::BlockVector &in) {
      oracle::BlockVector out(1, N, 0);
      H->cycle(static_cast<int>(H->L.size()) - 1, in.data.data(), out.data.data(), n);
      return out;
    };
    oracle::GmresResult res = oracle::gmres(apply, pre, bv, x0, kc);
    std::copy(res.x.data.begin(), res.x.data.end(), x);
    *iterations = res.iterations;
    if (!res.converged)
      throw std::runtime_error("fgmres: not converged");
  });
}

/// Exact "time-marched" solution of the all-at-once system on a single level
/// (pinned direct solve per interval with the jump coupling), pressure mean
/// zero per slot: the pin of the all-at-once solve.
int
o3_direct_time_march(void *h, const double *b, double *x, int n)
{
  return guard3([&] {
    const auto *L = static_cast<Level3 *>(h);
    oracle::Mat D = L->pinned_dense();
    oracle::LU lu(D);
    if (lu.singular)
      throw std::runtime_error("direct: singular");
    Vec rhs(L->isz), mw(L->mv);
    for (int t = 0; t < n; ++t)
      {
        std::copy(b + t * L->isz, b + (t + 1) * L->isz, rhs.begin());
        if (t > 0)
          {
            L->mass_apply(x + (t - 1) * L->isz + (L->S - 1) * L->mv, mw.data());
            L->zero_constrained(mw.data());
            for (int a = 0; a < L->S; ++a)
              for (Index i = 0; i < L->mv; ++i)
                rhs[a * L->mv + i] += L->tm.left_values[a] * mw[i];
          }
        for (int a = 0; a < L->S; ++a)
          rhs[L->S * L->mv + a * L->mp] = 0.0;
        Vec sol = lu.solve(rhs);
        for (int a = 0; a < L->S; ++a)
          L->project_mean_zero(sol.data() + L->S * L->mv + a * L->mp);
        std::copy(sol.begin(), sol.end(), x + t * L->isz);
      }
  });
}

} // extern "C"
