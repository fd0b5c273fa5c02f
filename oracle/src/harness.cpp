// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Restates problems.cpp and the planning / error-norm parts of harness.cpp.
#include "oracle/oracle.hpp"

#include <cmath>

namespace oracle
{

namespace
{
  constexpr double PI = 3.14159265358979323846;

  // harness.cpp:16-24
  int
  default_steps(double t_end, int refinements)
  {
    return static_cast<int>(std::lround(t_end * (1 << (refinements + 1))));
  }
} // namespace

// problems.cpp:13-62
StokesProblem
manufactured_problem()
{
  StokesProblem p;
  p.nu = 0.1;
  p.t_end = 1.0;
  p.has_exact = true;
  const double nu = p.nu;
  p.exact.velocity = [](double x, double y, double t, int comp) {
    const double cx = std::cos(2 * PI * x), sx = std::sin(2 * PI * x);
    const double cy = std::cos(2 * PI * y), sy = std::sin(2 * PI * y);
    const double s = 0.25 * std::sin(t);
    return comp == 0 ? s * (1.0 - cx) * sy : -s * sx * (1.0 - cy);
  };
  p.exact.velocity_gradient = [](double x, double y, double t, int comp, int deriv) {
    const double cx = std::cos(2 * PI * x), sx = std::sin(2 * PI * x);
    const double cy = std::cos(2 * PI * y), sy = std::sin(2 * PI * y);
    const double s = 0.5 * PI * std::sin(t);
    if (comp == 0)
      return deriv == 0 ? s * sx * sy : s * (1.0 - cx) * cy;
    return deriv == 0 ? -s * cx * (1.0 - cy) : -s * sx * sy;
  };
  p.exact.pressure = [](double x, double y, double t) {
    return 0.25 * std::sin(t) * std::sin(2 * PI * x) * std::sin(2 * PI * y);
  };
  p.data.force = [nu](double x, double y, double t, int comp) {
    const double cx = std::cos(2 * PI * x), sx = std::sin(2 * PI * x);
    const double cy = std::cos(2 * PI * y), sy = std::sin(2 * PI * y);
    const double st = std::sin(t), ct = std::cos(t);
    if (comp == 0)
      return 0.25 * ct * (1.0 - cx) * sy - nu * st * PI * PI * sy * (2.0 * cx - 1.0) + 0.5 * PI * st * cx * sy;
    return -0.25 * ct * sx * (1.0 - cy) - nu * st * PI * PI * sx * (1.0 - 2.0 * cy) + 0.5 * PI * st * sx * cy;
  };
  return p;
}

// problems.cpp:64-78
StokesProblem
cavity_problem(double nu)
{
  StokesProblem p;
  p.nu = nu;
  p.t_end = 8.0;
  p.has_exact = false;
  p.data.boundary = [](double x, double y, double t, int comp) {
    if (comp == 0 && y >= 1.0 && x > 0.0 && x < 1.0)
      return std::sin(0.25 * PI * t);
    return 0.0;
  };
  return p;
}

// harness.cpp:26-42
std::vector<LevelDescriptor>
plan_hierarchy(const RunConfig &config, double t_end)
{
  const int c = config.refinements;
  const int k = config.time_degree();
  const double h = std::pow(0.5, c);
  const int n = config.n_steps > 0 ? config.n_steps : default_steps(t_end, c);
  const double tau = t_end / n;
  const std::vector<HpEntry> spatial =
    config.h_only ? construct_hierarchy(h, 1.0, config.r, config.r) : construct_hierarchy(h, 1.0, config.r, 1);
  const std::vector<HpEntry> temporal =
    config.h_only ? construct_hierarchy(tau, tau, k, k) : construct_hierarchy(tau, tau, k, 1);
  return combine_hierarchies(spatial, temporal);
}

int
step_count(const StokesProblem &problem, const RunConfig &config)
{
  return config.n_steps > 0 ? config.n_steps : default_steps(problem.t_end, config.refinements);
}

// harness.cpp:51-70
Setup
build_setup(const StokesProblem &problem, const RunConfig &config)
{
  if (!config.allow_large && (config.r > 5 || config.refinements > 5))
    throw std::invalid_argument("build_setup: r > 5 or refinements > 5 need allow_large");
  Setup s;
  s.mesh = std::make_unique<Mesh>(Mesh::build_cartesian(Box{0.0, 0.0, 1.0, 1.0}, 1, 1, config.refinements + 1));
  s.descriptors = plan_hierarchy(config, problem.t_end);
  HierarchyParams params;
  params.nu = config.nu;
  params.tau = problem.t_end / step_count(problem, config);
  params.grad_div = config.grad_div;
  params.smoother = config.smoother;
  s.levels = instantiate_levels(*s.mesh, s.descriptors, params);
  return s;
}

// harness.cpp:72-183
ErrorReport
compute_errors(const Setup &setup, const TimeMarchResult &march, const ExactSolution &exact)
{
  const MultigridLevel &fine = setup.levels.finest();
  const VelocitySpace &vs = *fine.vspace;
  const PressureSpace &ps = *fine.pspace;
  const TemporalMatrices &tm = *fine.tmat;
  const int ns = tm.n_dofs();
  const int r = vs.r();
  const double tau = tm.tau;
  const NodalBasis1D time_basis(tm.nodes);
  const QuadratureRule tq_rule = gauss_rule(tm.k + 2);
  const Mat time_values = time_basis.value_table(tq_rule.points);
  const CellKernels eval(vs, ps, r + 3);
  const int nq = eval.n_q_1d(), n1 = eval.n_nodes_1d(), np = ps.dofs_per_cell();
  const Mesh &mesh = vs.mesh();
  const int level = vs.level();
  double sum_v = 0, sum_p = 0, sum_h1 = 0, sum_div = 0, linf = 0;
  Vec vbar(vs.n_dofs()), pbar(ps.n_dofs());
  Mat ux(n1, n1), uy(n1, n1);
  const Mat &phi = eval.phi(), &dphi = eval.dphi();
  // (A u B^T)(qx, qy) for 1D tables A, B (nq x n1).
  const auto interp = [&](const Mat &a, const Mat &u, const Mat &b) {
    Mat out(nq, nq);
    for (int qy = 0; qy < nq; ++qy)
      for (int qx = 0; qx < nq; ++qx)
        {
          double s = 0.0;
          for (int iy = 0; iy < n1; ++iy)
            {
              double t = 0.0;
              for (int ix = 0; ix < n1; ++ix)
                t += a(qx, ix) * u(ix, iy);
              s += t * b(qy, iy);
            }
          out(qx, qy) = s;
        }
    return out;
  };
  for (size_t step = 0; step < march.trajectory.size(); ++step)
    {
      const BlockVector &x = march.trajectory[step];
      const double t0 = static_cast<double>(step) * tau;
      for (int tq = 0; tq < tq_rule.size(); ++tq)
        {
          const double t = t0 + 0.5 * tau * (tq_rule.points[tq] + 1.0);
          const double wt = 0.5 * tau * tq_rule.weights[tq];
          std::fill(vbar.begin(), vbar.end(), 0.0);
          std::fill(pbar.begin(), pbar.end(), 0.0);
          for (int a = 0; a < ns; ++a)
            {
              const double c = time_values(tq, a);
              for (Index i = 0; i < vs.n_dofs(); ++i)
                vbar[i] += c * x.velocity(a)[i];
              for (Index i = 0; i < ps.n_dofs(); ++i)
                pbar[i] += c * x.pressure(a)[i];
            }
          for (int cell = 0; cell < mesh.n_cells(level); ++cell)
            {
              const Box box = mesh.cell_box(level, cell);
              const auto &dofs = vs.cell_scalar_dofs(cell);
              for (size_t loc = 0; loc < dofs.size(); ++loc)
                {
                  ux.d[loc] = vbar[vs.global_dof(0, dofs[loc])];
                  uy.d[loc] = vbar[vs.global_dof(1, dofs[loc])];
                }
              const Mat vxq = interp(phi, ux, phi), vyq = interp(phi, uy, phi);
              const Mat dvxdx = interp(dphi, ux, phi), dvxdy = interp(phi, ux, dphi);
              const Mat dvydx = interp(dphi, uy, phi), dvydy = interp(phi, uy, dphi);
              for (int qy = 0; qy < nq; ++qy)
                for (int qx = 0; qx < nq; ++qx)
                  {
                    const double xp = box.x0 + 0.5 * box.width() * (eval.qpoints()[qx] + 1.0);
                    const double yp = box.y0 + 0.5 * box.height() * (eval.qpoints()[qy] + 1.0);
                    const double wq = wt * eval.qweights()[qx] * eval.qweights()[qy] * eval.jdet();
                    const double ex0 = vxq(qx, qy) - exact.velocity(xp, yp, t, 0);
                    const double ex1 = vyq(qx, qy) - exact.velocity(xp, yp, t, 1);
                    sum_v += wq * (ex0 * ex0 + ex1 * ex1);
                    linf = std::max({linf, std::abs(ex0), std::abs(ex1)});
                    const double cx = eval.dxi_dx(), cy = eval.deta_dy();
                    const double g00 = cx * dvxdx(qx, qy) - exact.velocity_gradient(xp, yp, t, 0, 0);
                    const double g01 = cy * dvxdy(qx, qy) - exact.velocity_gradient(xp, yp, t, 0, 1);
                    const double g10 = cx * dvydx(qx, qy) - exact.velocity_gradient(xp, yp, t, 1, 0);
                    const double g11 = cy * dvydy(qx, qy) - exact.velocity_gradient(xp, yp, t, 1, 1);
                    sum_h1 += wq * (g00 * g00 + g01 * g01 + g10 * g10 + g11 * g11);
                    const double divh = cx * dvxdx(qx, qy) + cy * dvydy(qx, qy);
                    sum_div += wq * divh * divh;
                    double pq = 0.0;
                    for (int l = 0; l < np; ++l)
                      pq += eval.psi()(qy * nq + qx, l) * pbar[ps.cell_dof(cell, l)];
                    const double ep = pq - exact.pressure(xp, yp, t);
                    sum_p += wq * ep * ep;
                  }
            }
        }
    }
  ErrorReport rep;
  rep.e_v_l2 = std::sqrt(sum_v);
  rep.e_p_l2 = std::sqrt(sum_p);
  rep.e_v_h1 = std::sqrt(sum_h1);
  rep.e_div = std::sqrt(sum_div);
  rep.e_v_linf = linf;
  return rep;
}

// harness.cpp:185-239: nodal velocity at the GLL grid, pressure by the
// per-cell L2 projection onto the orthogonal P_r^disc basis (Gauss(r+3)).
TimeMarchResult
interpolate_exact(const Setup &setup, const ExactSolution &exact, int n_steps)
{
  const MultigridLevel &fine = setup.levels.finest();
  const VelocitySpace &vs = *fine.vspace;
  const PressureSpace &ps = *fine.pspace;
  const TemporalMatrices &tm = *fine.tmat;
  const int ns = tm.n_dofs();
  const int np = ps.dofs_per_cell();
  const CellKernels eval(vs, ps, vs.r() + 3);
  const int nq = eval.n_q_1d();
  const Mesh &mesh = vs.mesh();
  TimeMarchResult result;
  for (int n = 1; n <= n_steps; ++n)
    {
      BlockVector x = fine.op->make_vector();
      for (int a = 0; a < ns; ++a)
        {
          const double t = (n - 1) * tm.tau + 0.5 * tm.tau * (tm.nodes[a] + 1.0);
          double *v = x.velocity(a);
          for (int s = 0; s < vs.n_scalar_dofs(); ++s)
            for (int comp = 0; comp < 2; ++comp)
              v[vs.global_dof(comp, s)] = exact.velocity(vs.node_x(s), vs.node_y(s), t, comp);
          double *p = x.pressure(a);
          for (int cell = 0; cell < mesh.n_cells(vs.level()); ++cell)
            {
              const Box box = mesh.cell_box(vs.level(), cell);
              std::vector<double> rhs(np, 0.0);
              for (int qy = 0; qy < nq; ++qy)
                for (int qx = 0; qx < nq; ++qx)
                  {
                    const double xp = box.x0 + 0.5 * box.width() * (eval.qpoints()[qx] + 1.0);
                    const double yp = box.y0 + 0.5 * box.height() * (eval.qpoints()[qy] + 1.0);
                    const double wq = eval.qweights()[qx] * eval.qweights()[qy] * eval.jdet() * exact.pressure(xp, yp, t);
                    for (int l = 0; l < np; ++l)
                      rhs[l] += wq * eval.psi()(qy * nq + qx, l);
                  }
              for (int l = 0; l < np; ++l)
                p[ps.cell_dof(cell, l)] = rhs[l] / (eval.jdet() * ps.basis().gram_diagonal(l));
            }
        }
      result.trajectory.push_back(std::move(x));
    }
  return result;
}

// harness.cpp:325-346
double
evaluate_pressure(const PressureSpace &ps, const double *coeffs, double x, double y)
{
  const Mesh &mesh = ps.mesh();
  const int level = ps.level();
  const Box dom = mesh.domain();
  const int nx = mesh.cells_x(level), ny = mesh.cells_y(level);
  const int ix = std::min(static_cast<int>((x - dom.x0) / mesh.hx(level)), nx - 1);
  const int iy = std::min(static_cast<int>((y - dom.y0) / mesh.hy(level)), ny - 1);
  const int cell = mesh.cell_index(level, ix, iy);
  const Box box = mesh.cell_box(level, cell);
  const double xi[2] = {2.0 * (x - box.x0) / box.width() - 1.0, 2.0 * (y - box.y0) / box.height() - 1.0};
  double v = 0.0;
  for (int l = 0; l < ps.dofs_per_cell(); ++l)
    v += coeffs[ps.cell_dof(cell, l)] * ps.basis().value(l, xi);
  return v;
}

// harness.cpp:348-373
double
evaluate_velocity(const VelocitySpace &vs, const double *coeffs, double x, double y, int comp)
{
  const Mesh &mesh = vs.mesh();
  const int level = vs.level();
  const Box dom = mesh.domain();
  const int nx = mesh.cells_x(level), ny = mesh.cells_y(level);
  const int ix = std::min(static_cast<int>((x - dom.x0) / mesh.hx(level)), nx - 1);
  const int iy = std::min(static_cast<int>((y - dom.y0) / mesh.hy(level)), ny - 1);
  const int cell = mesh.cell_index(level, ix, iy);
  const Box box = mesh.cell_box(level, cell);
  const double xi = 2.0 * (x - box.x0) / box.width() - 1.0;
  const double eta = 2.0 * (y - box.y0) / box.height() - 1.0;
  const auto &b = vs.basis_1d();
  const int n1 = vs.nodes_per_dir();
  const auto &dofs = vs.cell_scalar_dofs(cell);
  double v = 0.0;
  for (int jy = 0; jy < n1; ++jy)
    for (int jx = 0; jx < n1; ++jx)
      v += coeffs[vs.global_dof(comp, dofs[jy * n1 + jx])] * b.value(jx, xi) * b.value(jy, eta);
  return v;
}

} // namespace oracle
