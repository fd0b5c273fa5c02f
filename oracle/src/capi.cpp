// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// extern "C" surface of the restatement for the Python tests and the CPU
// baseline leg of bench.py (ctypes). Not part of the product.
#include "oracle/oracle.hpp"

#include <cmath>
#include <cstring>
#include <random>

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace oracle;

namespace
{
thread_local std::string g_err;

template <class F>
int
guard(F &&f)
{
  try
    {
      f();
      return 0;
    }
  catch (const std::invalid_argument &e)
    {
      g_err = e.what();
      return 1;
    }
  catch (const std::exception &e)
    {
      g_err = e.what();
      return 2;
    }
}

/// One operator level on a (nc x nc) unit-square mesh (the shape every
/// BASELINE configuration uses): spaces, temporal matrices, operator and
/// optionally the smoother, as instantiate_levels builds them per level
/// (hierarchy.cpp:99-176).
struct LevelHandle
{
  std::unique_ptr<Mesh> mesh;
  std::unique_ptr<VelocitySpace> vs;
  std::unique_ptr<PressureSpace> ps;
  std::unique_ptr<TemporalMatrices> tm;
  std::unique_ptr<SpaceTimeBlockOperator> op;
  std::unique_ptr<VankaSmoother> sm;
};

struct SolverHandle
{
  StokesProblem problem;
  RunConfig config;
  Setup setup;
  std::unique_ptr<VCycle> vcycle;
  int n_steps = 0;
};

BlockVector
view_copy(const SpaceTimeBlockOperator &op, const double *p)
{
  BlockVector v = op.make_vector();
  std::memcpy(v.data.data(), p, sizeof(double) * v.size());
  return v;
}

// All-at-once residual of interval n: r_n = b_n - (D x_n - Z C x_{n-1}).
void
vmult_interval(const LevelHandle &h, const double *x, const double *x_prev_slot, double *y)
{
  const BlockVector xv = view_copy(*h.op, x);
  BlockVector yv = h.op->make_vector();
  h.op->apply_block(xv, yv);
  if (x_prev_slot)
    {
      BlockVector c = h.op->coupling_rhs(x_prev_slot);
      for (int a = 0; a < c.ns; ++a)
        h.vs->zero_constrained(c.velocity(a));
      yv -= c;
    }
  std::memcpy(y, yv.data.data(), sizeof(double) * yv.size());
}
} // namespace

extern "C" {

const char *
oracle_last_error()
{
  return g_err.c_str();
}

void
oracle_seeded_uniform(unsigned seed, double *out, long n)
{
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (long i = 0; i < n; ++i)
    out[i] = dist(rng);
}

int
oracle_level_create(int nc, int r, int k, double tau, double nu, double gamma, int smoother_kind,
                    int build_smoother, void **out)
{
  return guard([&] {
    int levels = 1;
    while ((1 << (levels - 1)) < nc)
      ++levels;
    if ((1 << (levels - 1)) != nc)
      throw std::invalid_argument("oracle_level_create: nc must be a power of two");
    auto h = std::make_unique<LevelHandle>();
    h->mesh = std::make_unique<Mesh>(Mesh::build_cartesian(Box{0, 0, 1, 1}, 1, 1, levels));
    h->vs = std::make_unique<VelocitySpace>(*h->mesh, levels - 1, r);
    h->ps = std::make_unique<PressureSpace>(*h->mesh, levels - 1, r);
    h->tm = std::make_unique<TemporalMatrices>(temporal_matrices(k, tau));
    h->op = std::make_unique<SpaceTimeBlockOperator>(*h->vs, *h->ps, *h->tm, nu, gamma);
    // build_smoother: 0 none, 1 full (every patch factored), 2 patch lists and
    // weights only (patches factored on demand by oracle_smooth_step_rows)
    if (build_smoother)
      h->sm = std::make_unique<VankaSmoother>(VankaSmoother::build(
        *h->op, smoother_kind == 1 ? SmootherKind::vertex_star : SmootherKind::cell, build_smoother != 2));
    *out = h.release();
  });
}

void
oracle_level_destroy(void *h)
{
  delete static_cast<LevelHandle *>(h);
}

/// sizes: [n_slots, n_velocity(M^v), n_pressure(M^p), interval size, n_scalar, grid_x, n_patches]
void
oracle_level_sizes(void *hp, long *out)
{
  const auto *h = static_cast<LevelHandle *>(hp);
  out[0] = h->op->n_slots();
  out[1] = h->vs->n_dofs();
  out[2] = h->ps->n_dofs();
  out[3] = h->op->make_vector().size();
  out[4] = h->vs->n_scalar_dofs();
  out[5] = h->vs->grid_x();
  out[6] = h->sm ? static_cast<long>(h->sm->patches().size()) : 0;
}

/// Saddle-point health of a converged step (solver.cpp:286-299): per slot
/// ||B v|| / sqrt(v^T M v) and |<mean, p>| / ||p||, maximised over the slots.
int
oracle_step_health(void *hp, const double *x, double *out)
{
  return guard([&] {
    const auto *h = static_cast<LevelHandle *>(hp);
    const BlockVector xv = view_copy(*h->op, x);
    const Index mv = h->vs->n_dofs(), mp = h->ps->n_dofs();
    Vec work_p(mp), work_v(mv);
    double max_div = 0.0, max_mean = 0.0;
    for (int a = 0; a < xv.ns; ++a)
      {
        std::fill(work_p.begin(), work_p.end(), 0.0);
        std::fill(work_v.begin(), work_v.end(), 0.0);
        h->op->apply_div(xv.velocity(a), work_p.data());
        h->op->apply_velocity_mass(xv.velocity(a), work_v.data());
        double vmv = 0.0, pn = 0.0, bn = 0.0, mdot = 0.0;
        for (Index i = 0; i < mv; ++i)
          vmv += xv.velocity(a)[i] * work_v[i];
        for (Index i = 0; i < mp; ++i)
          {
            bn += work_p[i] * work_p[i];
            pn += xv.pressure(a)[i] * xv.pressure(a)[i];
            mdot += h->ps->mean_vector()[i] * xv.pressure(a)[i];
          }
        const double vnorm = std::sqrt(std::abs(vmv));
        if (vnorm > 0.0)
          max_div = std::max(max_div, std::sqrt(bn) / vnorm);
        if (pn > 0.0)
          max_mean = std::max(max_mean, std::abs(mdot) / std::sqrt(pn));
      }
    out[0] = max_div;
    out[1] = max_mean;
  });
}

int
oracle_apply_block(void *hp, const double *x, double *y, int raw)
{
  return guard([&] {
    const auto *h = static_cast<LevelHandle *>(hp);
    const BlockVector xv = view_copy(*h->op, x);
    BlockVector yv = h->op->make_vector();
    if (raw)
      h->op->apply_block_raw(xv, yv);
    else
      h->op->apply_block(xv, yv);
    std::memcpy(y, yv.data.data(), sizeof(double) * yv.size());
  });
}

int
oracle_coupling_rhs(void *hp, const double *v_prev, double *out)
{
  return guard([&] {
    const auto *h = static_cast<LevelHandle *>(hp);
    const BlockVector c = h->op->coupling_rhs(v_prev);
    std::memcpy(out, c.data.data(), sizeof(double) * c.size());
  });
}

/// All-at-once vmult over n intervals (interval-major): y_n = D x_n - Z C
/// x_{n-1}[slot k], with x_prev_slot (may be null) feeding interval 0.
int
oracle_vmult_all(void *hp, const double *x, double *y, int n_intervals, const double *x_prev_slot, int threads)
{
  return guard([&] {
    const auto *h = static_cast<LevelHandle *>(hp);
    const Index sz = h->op->make_vector().size();
    const Index mv = h->vs->n_dofs();
    const int ns = h->op->n_slots();
#ifdef _OPENMP
    if (threads > 0)
      omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 1) if (threads != 1)
#endif
    for (int n = 0; n < n_intervals; ++n)
      {
        const double *prev = n == 0 ? x_prev_slot : x + (n - 1) * sz + (ns - 1) * mv;
        vmult_interval(*h, x + n * sz, prev, y + n * sz);
      }
  });
}

int
oracle_apply_additive(void *hp, const double *r, double *out)
{
  return guard([&] {
    const auto *h = static_cast<LevelHandle *>(hp);
    if (!h->sm)
      throw std::invalid_argument("no smoother built");
    const BlockVector rv = view_copy(*h->op, r);
    BlockVector o = h->op->make_vector();
    h->sm->apply_additive(rv, o);
    std::memcpy(out, o.data.data(), sizeof(double) * o.size());
  });
}

/// One smoother step per interval on the all-at-once system:
/// u_n <- u_n + omega * apply_additive(b_n - (D u_n - Z C u_{n-1}^{old})).
/// The coupling uses the pre-step iterate of the previous interval (Jacobi
/// in time, block-diagonal smoother).
int
oracle_smooth_step_all(void *hp, const double *b, double *u, double omega, int n_intervals,
                       const double *x_prev_slot, int threads)
{
  return guard([&] {
    const auto *h = static_cast<LevelHandle *>(hp);
    if (!h->sm)
      throw std::invalid_argument("no smoother built");
    if (!(omega > 0.0 && omega <= 1.0))
      throw std::invalid_argument("smooth_step: omega must be in (0, 1]");
    const Index sz = h->op->make_vector().size();
    const Index mv = h->vs->n_dofs();
    const int ns = h->op->n_slots();
    std::vector<double> u_old(u, u + sz * n_intervals);
#ifdef _OPENMP
    if (threads > 0)
      omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 1) if (threads != 1)
#endif
    for (int n = 0; n < n_intervals; ++n)
      {
        const double *prev = n == 0 ? x_prev_slot : u_old.data() + (n - 1) * sz + (ns - 1) * mv;
        Vec au(sz);
        vmult_interval(*h, u_old.data() + n * sz, prev, au.data());
        BlockVector res = h->op->make_vector();
        for (Index i = 0; i < sz; ++i)
          res.data[i] = b[n * sz + i] - au[i];
        BlockVector corr = h->op->make_vector();
        h->sm->apply_additive(res, corr);
        for (Index i = 0; i < sz; ++i)
          u[n * sz + i] = u_old[n * sz + i] + omega * corr.data[i];
      }
  });
}

/// smooth_step_all (above) evaluated at a subset of rows, for meshes whose
/// full set of patch factorizations does not fit (BASELINE-size parity):
/// out[n * nrows + i] = u_new[n][rows[i]]. Only the patches containing a
/// requested row are factored; they are applied in patch order, so every
/// requested row receives exactly the additions of the full sweep, in the
/// same order (vanka.cpp:196-215).
int
oracle_smooth_step_rows(void *hp, const double *b, const double *u, double omega, int n_intervals,
                        const double *x_prev_slot, const long *rows, long nrows, double *out, int threads)
{
  return guard([&] {
    auto *h = static_cast<LevelHandle *>(hp);
    if (!h->sm)
      throw std::invalid_argument("no smoother built");
    if (!(omega > 0.0 && omega <= 1.0))
      throw std::invalid_argument("smooth_step: omega must be in (0, 1]");
    const Index sz = h->op->make_vector().size();
    const Index mv = h->vs->n_dofs();
    const int ns = h->op->n_slots();
    std::vector<int> idx(static_cast<size_t>(sz), -1);
    for (long i = 0; i < nrows; ++i)
      {
        if (rows[i] < 0 || rows[i] >= sz)
          throw std::invalid_argument("oracle_smooth_step_rows: row out of range");
        idx[rows[i]] = static_cast<int>(i);
      }
    auto &patches = h->sm->patches();
    std::vector<size_t> need;
    for (size_t ip = 0; ip < patches.size(); ++ip)
      for (const Index d : patches[ip].dofs)
        if (idx[d] >= 0)
          {
            need.push_back(ip);
            break;
          }
#ifdef _OPENMP
    if (threads > 0)
      omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 4) if (threads != 1)
#endif
    for (long q = 0; q < static_cast<long>(need.size()); ++q)
      if (!patches[need[q]].factored)
        h->sm->factor_patch(*h->op, need[q]);
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1) if (threads != 1)
#endif
    for (int n = 0; n < n_intervals; ++n)
      {
        const double *prev = n == 0 ? x_prev_slot : u + (n - 1) * sz + (ns - 1) * mv;
        Vec au(sz);
        vmult_interval(*h, u + n * sz, prev, au.data());
        for (Index i = 0; i < sz; ++i)
          au[i] = b[n * sz + i] - au[i];
        std::vector<double> corr(static_cast<size_t>(nrows), 0.0);
        Vec loc;
        for (const size_t ip : need)
          {
            const auto &patch = patches[ip];
            const int n_t = patch.size();
            loc.resize(n_t);
            for (int i = 0; i < n_t; ++i)
              loc[i] = au[patch.dofs[i]];
            loc = patch.solve(loc);
            for (int i = 0; i < n_t; ++i)
              if (idx[patch.dofs[i]] >= 0)
                corr[idx[patch.dofs[i]]] += patch.weights[i] * loc[i];
          }
        for (long i = 0; i < nrows; ++i)
          out[n * nrows + i] = u[n * sz + rows[i]] + omega * corr[i];
      }
  });
}

/// Number of patches, their sizes, flattened dof lists and weights.
long
oracle_patch_count(void *hp)
{
  const auto *h = static_cast<LevelHandle *>(hp);
  return h->sm ? static_cast<long>(h->sm->patches().size()) : 0;
}

int
oracle_patch(void *hp, long i, long *dofs, double *weights, double *local_matrix)
{
  return guard([&] {
    const auto *h = static_cast<LevelHandle *>(hp);
    const auto &p = h->sm->patches().at(i);
    for (int j = 0; j < p.size(); ++j)
      {
        if (dofs)
          dofs[j] = p.dofs[j];
        if (weights)
          weights[j] = p.weights[j];
      }
    if (local_matrix)
      std::memcpy(local_matrix, h->sm->local_matrices.at(i).data(), sizeof(double) * p.size() * p.size());
  });
}

long
oracle_patch_size(void *hp, long i)
{
  const auto *h = static_cast<LevelHandle *>(hp);
  return h->sm->patches().at(i).size();
}

// ---------------------------------------------------------------- solver handle
int
oracle_solver_create(int refinements, int r, int k, int n_steps, double t_end, double nu, double gamma,
                     int smoother_kind, int nu1, int nu2, double omega, int h_only, double rtol, double atol,
                     int maxit, void **out)
{
  return guard([&] {
    auto h = std::make_unique<SolverHandle>();
    h->problem.nu = nu;
    h->problem.t_end = t_end;
    h->config.r = r;
    h->config.k = k;
    h->config.refinements = refinements;
    h->config.n_steps = n_steps;
    h->config.nu = nu;
    h->config.grad_div = gamma;
    h->config.smoother = smoother_kind == 1 ? SmootherKind::vertex_star : SmootherKind::cell;
    h->config.h_only = h_only != 0;
    h->config.allow_large = true;
    h->config.mg.nu1 = nu1;
    h->config.mg.nu2 = nu2;
    h->config.mg.omega = omega;
    h->config.krylov.rtol = rtol;
    h->config.krylov.atol = atol;
    h->config.krylov.max_iterations = maxit;
    h->config.krylov.max_basis = maxit;
    h->setup = build_setup(h->problem, h->config);
    h->n_steps = step_count(h->problem, h->config);
    h->vcycle = std::make_unique<VCycle>(h->setup.levels, h->config.mg);
    *out = h.release();
  });
}

void
oracle_solver_destroy(void *h)
{
  delete static_cast<SolverHandle *>(h);
}

/// level info: [n_levels, then per level: nc, r, k, kind_to_coarser, interval size]
void
oracle_solver_info(void *hp, long *out)
{
  const auto *h = static_cast<SolverHandle *>(hp);
  const auto &lv = h->setup.levels;
  out[0] = lv.n_levels();
  for (int l = 0; l < lv.n_levels(); ++l)
    {
      const auto &L = lv.level(l);
      out[1 + 5 * l + 0] = L.vspace->mesh().cells_x(L.vspace->level());
      out[1 + 5 * l + 1] = L.desc.r;
      out[1 + 5 * l + 2] = L.desc.k;
      out[1 + 5 * l + 3] = static_cast<long>(L.desc.kind_to_coarser);
      out[1 + 5 * l + 4] = L.op->make_vector().size();
    }
}

double
oracle_solver_tau(void *hp)
{
  return static_cast<SolverHandle *>(hp)->setup.levels.finest().desc.tau;
}

int
oracle_solver_n_steps(void *hp)
{
  return static_cast<SolverHandle *>(hp)->n_steps;
}

int
oracle_level_apply_block(void *hp, int l, const double *x, double *y)
{
  return guard([&] {
    const auto *h = static_cast<SolverHandle *>(hp);
    const auto &op = *h->setup.levels.level(l).op;
    const BlockVector xv = view_copy(op, x);
    BlockVector yv = op.make_vector();
    op.apply_block(xv, yv);
    std::memcpy(y, yv.data.data(), sizeof(double) * yv.size());
  });
}

int
oracle_level_smooth_step(void *hp, int l, const double *b, double *u, double omega)
{
  return guard([&] {
    const auto *h = static_cast<SolverHandle *>(hp);
    const auto &L = h->setup.levels.level(l);
    if (!L.smoother)
      throw std::invalid_argument("level has no smoother");
    const BlockVector bv = view_copy(*L.op, b);
    BlockVector uv = view_copy(*L.op, u);
    L.smoother->smooth_step(*L.op, bv, uv, omega);
    std::memcpy(u, uv.data.data(), sizeof(double) * uv.size());
  });
}

int
oracle_level_restrict_residual(void *hp, int l, const double *fine, double *coarse, int project)
{
  return guard([&] {
    const auto *h = static_cast<SolverHandle *>(hp);
    const auto &L = h->setup.levels.level(l);
    const BlockVector f = view_copy(*L.op, fine);
    const BlockVector c = L.to_coarser->restrict_residual(f, project != 0);
    std::memcpy(coarse, c.data.data(), sizeof(double) * c.size());
  });
}

int
oracle_level_prolongate_correction(void *hp, int l, const double *coarse, double *fine, int project)
{
  return guard([&] {
    const auto *h = static_cast<SolverHandle *>(hp);
    const auto &L = h->setup.levels.level(l);
    const auto &C = h->setup.levels.level(l - 1);
    const BlockVector c = view_copy(*C.op, coarse);
    const BlockVector f = L.to_coarser->prolongate_correction(c, project != 0);
    std::memcpy(fine, f.data.data(), sizeof(double) * f.size());
  });
}

int
oracle_vcycle(void *hp, const double *b, double *x)
{
  return guard([&] {
    const auto *h = static_cast<SolverHandle *>(hp);
    const auto &op = *h->setup.levels.finest().op;
    const BlockVector bv = view_copy(op, b);
    const BlockVector xv = h->vcycle->apply(bv);
    std::memcpy(x, xv.data.data(), sizeof(double) * xv.size());
  });
}

/// One preconditioned GMRES solve of D x = b on the finest level.
int
oracle_gmres(void *hp, const double *b, double *x, int *iterations, double *history, int history_cap)
{
  return guard([&] {
    const auto *h = static_cast<SolverHandle *>(hp);
    const auto &op = *h->setup.levels.finest().op;
    const ApplyFn apply = [&op](const BlockVector &xx, BlockVector &yy) { op.apply_block(xx, yy); };
    const PrecondFn pre = [h](const BlockVector &r) { return h->vcycle->apply(r); };
    const GmresResult res = gmres(apply, pre, view_copy(op, b), op.make_vector(), h->config.krylov);
    std::memcpy(x, res.x.data.data(), sizeof(double) * res.x.size());
    *iterations = res.iterations;
    for (int i = 0; i < history_cap && i < static_cast<int>(res.residual_history.size()); ++i)
      history[i] = res.residual_history[i];
    if (!res.converged)
      throw std::runtime_error("gmres: not converged");
  });
}

/// Time marching (solver.cpp:204-325) with a seeded per-step load vector F_n
/// (interval-major, n_steps intervals) added to the right-hand side in place
/// of the force; zero initial velocity, homogeneous Dirichlet data. Writes
/// the trajectory X and the iteration count per step; returns throughput.
int
oracle_time_march_seeded(void *hp, const double *F, double *X, int *iterations, double *throughput)
{
  return guard([&] {
    auto *h = static_cast<SolverHandle *>(hp);
    const auto &op = *h->setup.levels.finest().op;
    const Index sz = op.make_vector().size();
    TimeMarchProblem prob;
    prob.extra_rhs = [&](int step, BlockVector &rhs) {
      for (Index i = 0; i < sz; ++i)
        rhs.data[i] += F[(step - 1) * sz + i];
    };
    const TimeMarchResult res =
      time_march(h->setup.levels, prob, h->n_steps, h->config.mg, h->config.krylov, true);
    for (int n = 0; n < h->n_steps; ++n)
      {
        std::memcpy(X + n * sz, res.trajectory[n].data.data(), sizeof(double) * sz);
        iterations[n] = res.steps[n].iterations;
      }
    if (throughput)
      *throughput = res.throughput;
  });
}

/// Manufactured problem (problems.cpp:13-62; its force uses nu = 0.1):
/// assemble_rhs (st_operator.cpp:423-467) on the finest level at t_start.
int
oracle_assemble_rhs_manufactured(void *hp, double t_start, double *out)
{
  return guard([&] {
    auto *h = static_cast<SolverHandle *>(hp);
    const StokesProblem mp = manufactured_problem();
    const BlockVector v = h->setup.levels.finest().op->assemble_rhs(mp.data.force, t_start);
    std::memcpy(out, v.data.data(), sizeof(double) * v.data.size());
  });
}

/// time_march (solver.cpp:204-325) of the manufactured problem: trajectory X
/// (n_steps intervals) and GMRES iterations per step.
int
oracle_time_march_manufactured(void *hp, double *X, int *iterations)
{
  return guard([&] {
    auto *h = static_cast<SolverHandle *>(hp);
    const StokesProblem mp = manufactured_problem();
    const TimeMarchResult res = time_march(h->setup.levels, mp.data, h->n_steps, h->config.mg, h->config.krylov, true);
    const size_t sz = res.trajectory.empty() ? 0 : res.trajectory[0].data.size();
    for (int n = 0; n < h->n_steps; ++n)
      {
        std::memcpy(X + n * sz, res.trajectory[n].data.data(), sizeof(double) * sz);
        iterations[n] = res.steps[n].iterations;
      }
  });
}

/// compute_errors (harness.cpp:72-183) of a trajectory X (n_steps intervals)
/// against the manufactured exact solution: out = e_v, e_p, e_h1, e_div, linf.
int
oracle_manufactured_errors(void *hp, const double *X, double *out)
{
  return guard([&] {
    auto *h = static_cast<SolverHandle *>(hp);
    const auto &op = *h->setup.levels.finest().op;
    const size_t sz = op.make_vector().data.size();
    TimeMarchResult m;
    for (int n = 0; n < h->n_steps; ++n)
      m.trajectory.push_back(view_copy(op, X + n * sz));
    const ErrorReport e = compute_errors(h->setup, m, manufactured_problem().exact);
    out[0] = e.e_v_l2;
    out[1] = e.e_p_l2;
    out[2] = e.e_v_h1;
    out[3] = e.e_div;
    out[4] = e.e_v_linf;
  });
}

/// interpolate_exact (harness.cpp:185-239) of the manufactured solution on
/// the finest level: X (n_steps intervals).
int
oracle_interpolate_manufactured(void *hp, double *X)
{
  return guard([&] {
    auto *h = static_cast<SolverHandle *>(hp);
    const TimeMarchResult m = interpolate_exact(h->setup, manufactured_problem().exact, h->n_steps);
    const size_t sz = m.trajectory[0].data.size();
    for (int n = 0; n < h->n_steps; ++n)
      std::memcpy(X + n * sz, m.trajectory[n].data.data(), sizeof(double) * sz);
  });
}

/// time_march of the lid-driven cavity (problems.cpp:64-78) with the
/// solver's nu: inhomogeneous Dirichlet data by lifting (solver.cpp:251-283).
int
oracle_time_march_cavity(void *hp, double *X, int *iterations)
{
  return guard([&] {
    auto *h = static_cast<SolverHandle *>(hp);
    const StokesProblem cp = cavity_problem(h->config.nu);
    const TimeMarchResult res = time_march(h->setup.levels, cp.data, h->n_steps, h->config.mg, h->config.krylov, true);
    const size_t sz = res.trajectory[0].data.size();
    for (int n = 0; n < h->n_steps; ++n)
      {
        std::memcpy(X + n * sz, res.trajectory[n].data.data(), sizeof(double) * sz);
        iterations[n] = res.steps[n].iterations;
      }
  });
}

} // extern "C"
