// stmg_gpu: drop-in for the reference's `stmg` command line (tools/stmg.cpp:84-310)
// on the B200 library. Same subcommands (convergence, robustness, cavity,
// hierarchy, selftest), the same dotted flags (--problem.nu, --mesh.refinements,
// --mg.nu1, --gmres.rtol, ...), the same flat-INI --config with command-line
// precedence, exit code 3 for an unreadable config or unknown keys, and the
// same printed tables / CSV files. Every solve runs through the C ABI
// (include/stmg_b200.h) on the GPU.
#include "stmg_b200.h"

#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <map>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace
{
struct Options
{
  int r = 2, k = -1, refinements = 2, n_steps = 0;
  double nu = 0.1, grad_div = 1.0;
  std::string smoother = "cell", mode = "hp";
  int nu1 = 1, nu2 = 1, coarse_cap = 50000;
  double omega = 0.8;
  bool project_pressure = true, allow_large = false, show_stats = false;
  double rtol = 1e-8, atol = 1e-14;
  int maxit = 200;
  std::string csv_path, steps_csv;
  std::vector<int> r_list{2}, c_list{1, 2, 3}, n_sm_list{1};
};

void
check(int code)
{
  if (code != STMG_OK)
    throw std::runtime_error(stmg_last_error());
}

std::vector<int>
int_list(const std::string &text)
{
  std::vector<int> out;
  std::stringstream ss(text);
  std::string tok;
  while (std::getline(ss, tok, ','))
    {
      std::stringstream item(tok);
      int v;
      while (item >> v)
        out.push_back(v);
    }
  return out;
}

bool
to_bool(const std::string &v)
{
  return v == "1" || v == "true" || v == "on" || v == "yes";
}

/// key -> setter; keys are the flag names without "--" (stmg.cpp:84-179)
std::map<std::string, std::function<void(const std::string &)>>
setters(Options &o)
{
  return {
    {"problem.nu", [&](const std::string &v) { o.nu = std::stod(v); }},
    {"problem.grad_div", [&](const std::string &v) { o.grad_div = std::stod(v); }},
    {"problem.N", [&](const std::string &v) { o.n_steps = std::stoi(v); }},
    {"discretization.r", [&](const std::string &v) { o.r = std::stoi(v); }},
    {"discretization.k", [&](const std::string &v) { o.k = std::stoi(v); }},
    {"mesh.refinements", [&](const std::string &v) { o.refinements = std::stoi(v); }},
    {"mg.nu1", [&](const std::string &v) { o.nu1 = std::stoi(v); }},
    {"mg.nu2", [&](const std::string &v) { o.nu2 = std::stoi(v); }},
    {"mg.omega", [&](const std::string &v) { o.omega = std::stod(v); }},
    {"mg.smoother", [&](const std::string &v) { o.smoother = v; }},
    {"mg.mode", [&](const std::string &v) { o.mode = v; }},
    {"mg.coarse_cap", [&](const std::string &v) { o.coarse_cap = std::stoi(v); }},
    {"mg.project_pressure", [&](const std::string &v) { o.project_pressure = to_bool(v); }},
    {"gmres.rtol", [&](const std::string &v) { o.rtol = std::stod(v); }},
    {"gmres.atol", [&](const std::string &v) { o.atol = std::stod(v); }},
    {"gmres.maxit", [&](const std::string &v) { o.maxit = std::stoi(v); }},
    {"output.csv_path", [&](const std::string &v) { o.csv_path = v; }},
    {"output.steps_csv", [&](const std::string &v) { o.steps_csv = v; }},
    {"r_list", [&](const std::string &v) { o.r_list = int_list(v); }},
    {"c_list", [&](const std::string &v) { o.c_list = int_list(v); }},
    {"n_sm_list", [&](const std::string &v) { o.n_sm_list = int_list(v); }},
  };
}

/// Flat INI (stmg.cpp:17-50): [section] scopes key = value to section.key.
std::map<std::string, std::string>
read_flat_ini(const std::string &path)
{
  std::ifstream in(path);
  if (!in)
    throw std::runtime_error("cannot open config file: " + path);
  std::map<std::string, std::string> values;
  std::string line, section;
  auto trim = [](std::string s) {
    const auto b = s.find_first_not_of(" \t\r"), e = s.find_last_not_of(" \t\r");
    return b == std::string::npos ? std::string() : s.substr(b, e - b + 1);
  };
  while (std::getline(in, line))
    {
      const auto c = line.find_first_of("#;");
      if (c != std::string::npos)
        line.erase(c);
      line = trim(line);
      if (line.empty())
        continue;
      if (line.front() == '[' && line.back() == ']')
        {
          section = trim(line.substr(1, line.size() - 2));
          continue;
        }
      const auto eq = line.find('=');
      if (eq == std::string::npos)
        throw std::runtime_error("config: expected key = value, got: " + line);
      values[section.empty() ? trim(line.substr(0, eq)) : section + "." + trim(line.substr(0, eq))] =
        trim(line.substr(eq + 1));
    }
  return values;
}

struct Problem
{
  int id;
  double nu, t_end;
};

/// One GPU hierarchy for a built-in problem (build_setup, harness.cpp:51-70).
struct Run
{
  stmg_ctx *ctx = nullptr;
  stmg_solver *sol = nullptr;
  int n_levels = 0, n_steps = 0;
  int64_t fine_size = 0;
  std::vector<int64_t> info;
  Run(stmg_ctx *c, const Options &o, int r, int refinements, int nu1, int nu2, const Problem &p, bool cell) : ctx(c)
  {
    if (!o.allow_large && (r > 5 || refinements > 5))
      throw std::runtime_error("run exceeds r = 5 or c = 5 refinements (pass --allow_large)");
    check(stmg_solver_create(ctx, refinements, r, o.k, o.n_steps, p.t_end, p.nu, o.grad_div,
                             cell ? STMG_SMOOTHER_CELL : STMG_SMOOTHER_VERTEX_STAR, nu1, nu2, o.omega,
                             o.mode == "h_only" ? 1 : 0, o.rtol, o.atol, o.maxit, &sol));
    info.assign(2 + 5 * 64, 0);
    check(stmg_solver_info(sol, info.data()));
    n_levels = static_cast<int>(info[0]);
    n_steps = static_cast<int>(info[1]);
    fine_size = info[2 + 5 * (n_levels - 1) + 4];
  }
  ~Run()
  {
    if (sol)
      stmg_solver_destroy(sol);
  }
};

double
eoc(double coarse, double fine)
{
  return (coarse > 0.0 && fine > 0.0) ? std::log2(coarse / fine) : 0.0;
}

double
legendre(int n, double x)
{
  double p0 = 1.0, p1 = x;
  if (n == 0)
    return p0;
  for (int k = 2; k <= n; ++k)
    {
      const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
  return p1;
}

/// evaluate_pressure (harness.cpp:321-343) on the unit square, 2D P_r^disc.
double
pressure_at(const std::vector<double> &p, int nc, int r, double x, double y)
{
  const int np = (r + 1) * (r + 2) / 2;
  const double h = 1.0 / nc;
  const int ix = std::min(static_cast<int>(x / h), nc - 1), iy = std::min(static_cast<int>(y / h), nc - 1);
  const double xi = 2.0 * (x - ix * h) / h - 1.0, eta = 2.0 * (y - iy * h) / h - 1.0;
  double v = 0.0;
  int l = 0;
  for (int deg = 0; deg <= r; ++deg)
    for (int a = deg; a >= 0; --a, ++l)
      v += p[(static_cast<size_t>(iy) * nc + ix) * np + l] * legendre(a, xi) * legendre(deg - a, eta);
  return v;
}

void
print_hierarchy(const std::vector<int64_t> &out, double t_end)
{
  static const char *kinds[] = {"identity", "h_space", "p_space", "p_time", "h_space+p_time", "p_space+p_time"};
  const int n = static_cast<int>(out[0]), steps = static_cast<int>(out[1]);
  std::printf("level |   h      r  |  tau     k  | transfer to coarser\n");
  std::printf("------+-------------+-------------+--------------------\n");
  for (int l = n - 1; l >= 0; --l)
    {
      const int64_t *o = &out[2 + 5 * l];
      std::printf("%5d | %-8.4g %2d | %-8.4g %2d | %s\n", l, 1.0 / static_cast<double>(o[0]), static_cast<int>(o[1]),
                  t_end / steps, static_cast<int>(o[2]), l == 0 ? "(direct solve)" : kinds[o[3]]);
    }
}

int
usage()
{
  std::fprintf(stderr, "usage: stmg_gpu <convergence|robustness|cavity|hierarchy|selftest> [--key value ...] "
                       "[--config file.ini]\n");
  return 2;
}
} // namespace

int
main(int argc, char **argv)
{
  Options o;
  auto set = setters(o);
  std::string sub, config;
  std::set<std::string> given;
  for (int i = 1; i < argc; ++i)
    {
      std::string a = argv[i];
      if (a.rfind("--", 0) != 0)
        {
          if (!sub.empty())
            return usage();
          sub = a;
          continue;
        }
      a = a.substr(2);
      std::string val;
      const auto eq = a.find('=');
      const bool is_flag = a == "allow_large" || a == "report.smoother_stats" || a == "mg.project_pressure" ||
                           a == "mg.no-project_pressure";
      if (eq != std::string::npos)
        {
          val = a.substr(eq + 1);
          a = a.substr(0, eq);
        }
      else if (!is_flag)
        {
          if (i + 1 >= argc)
            return usage();
          val = argv[++i];
        }
      if (a == "config")
        config = val;
      else if (a == "allow_large")
        o.allow_large = true;
      else if (a == "report.smoother_stats")
        o.show_stats = true;
      else if (a == "mg.no-project_pressure")
        o.project_pressure = false, given.insert("mg.project_pressure");
      else if (a == "mg.project_pressure" && val.empty())
        o.project_pressure = true, given.insert(a);
      else if (set.count(a))
        {
          set[a](val);
          given.insert(a);
        }
      else
        {
          std::fprintf(stderr, "unknown option --%s\n", a.c_str());
          return 2;
        }
    }
  if (sub.empty())
    return usage();
  if (!config.empty())
    {
      try
        {
          for (const auto &[key, value] : read_flat_ini(config))
            {
              const auto it = set.find(key);
              if (it == set.end())
                throw std::runtime_error("config: unknown key '" + key + "'");
              if (!given.count(key)) // command-line flags win (stmg.cpp:160-170)
                it->second(value);
            }
        }
      catch (const std::exception &e)
        {
          std::fprintf(stderr, "%s\n", e.what());
          return 3;
        }
    }
  const bool cell = o.smoother != "vertex_star";
  try
    {
      stmg_ctx *ctx = nullptr;
      if (sub != "hierarchy") // the hierarchy plan is host-only
        check(stmg_ctx_create(0, &ctx));
      const Problem manufactured{STMG_PROBLEM_MANUFACTURED, 0.1, 1.0}; // problems.cpp:13-62
      if (sub == "convergence")
        {
          std::printf("%2s %2s %-10s %-12s %-6s %-12s %-6s %-12s %-6s %-12s %-6s %s\n", "r", "c", "h", "e_v_L2", "eoc",
                      "e_p_L2", "eoc", "e_v_H1", "eoc", "e_div", "eoc", "iters");
          std::ofstream csv;
          if (!o.csv_path.empty())
            {
              csv.open(o.csv_path);
              csv.precision(12);
              csv << "r,c,h,e_v_L2,eoc,e_p_L2,eoc,e_v_H1,eoc,e_div,eoc\n";
            }
          for (int r : o.r_list)
            {
              double prev[4] = {0, 0, 0, 0};
              bool have = false;
              for (int c : o.c_list)
                {
                  Options oc = o;
                  oc.k = -1;
                  Run run(ctx, oc, r, c, o.nu1, o.nu2, manufactured, cell);
                  stmg_level *fine = stmg_solver_level(run.sol, run.n_levels - 1);
                  double *X = nullptr;
                  cudaMalloc(&X, sizeof(double) * run.fine_size * run.n_steps);
                  std::vector<int> its(run.n_steps);
                  check(stmg_time_march_problem(run.sol, STMG_PROBLEM_MANUFACTURED, X, its.data()));
                  double e[5];
                  check(stmg_compute_errors(fine, STMG_PROBLEM_MANUFACTURED, 0.0, X, run.n_steps, e));
                  cudaFree(X);
                  double avg = 0.0;
                  for (int v : its)
                    avg += v;
                  avg /= run.n_steps;
                  const double ev[4] = {e[0], e[1], e[2], e[3]};
                  double eo[4] = {0, 0, 0, 0};
                  if (have)
                    for (int q = 0; q < 4; ++q)
                      eo[q] = eoc(prev[q], ev[q]);
                  std::printf("%2d %2d %-10.4g %-12.5g %-6.2f %-12.5g %-6.2f %-12.5g %-6.2f %-12.5g %-6.2f %.1f\n", r,
                              c, std::pow(0.5, c), ev[0], eo[0], ev[1], eo[1], ev[2], eo[2], ev[3], eo[3], avg);
                  if (csv)
                    csv << r << ',' << c << ',' << std::pow(0.5, c) << ',' << ev[0] << ',' << eo[0] << ',' << ev[1]
                        << ',' << eo[1] << ',' << ev[2] << ',' << eo[2] << ',' << ev[3] << ',' << eo[3] << '\n';
                  for (int q = 0; q < 4; ++q)
                    prev[q] = ev[q];
                  have = true;
                }
            }
        }
      else if (sub == "robustness")
        {
          std::printf("%2s %2s %-12s %4s %-10s %-14s %-12s\n", "r", "c", "smoother", "n_sm", "avg_iters", "sum_nT2",
                      "throughput");
          std::ofstream csv;
          if (!o.csv_path.empty())
            {
              csv.open(o.csv_path);
              csv << "r,c,smoother,n_sm,avg_iters,sum_nT2\n";
            }
          for (int r : o.r_list)
            for (int c : o.c_list)
              for (int nsm : o.n_sm_list)
                {
                  Options oc = o;
                  oc.k = -1;
                  Run run(ctx, oc, r, c, nsm, nsm, manufactured, cell);
                  double *X = nullptr;
                  cudaMalloc(&X, sizeof(double) * run.fine_size * run.n_steps);
                  std::vector<int> its(run.n_steps);
                  cudaDeviceSynchronize();
                  cudaEvent_t e0, e1;
                  cudaEventCreate(&e0);
                  cudaEventCreate(&e1);
                  cudaEventRecord(e0);
                  check(stmg_time_march_problem(run.sol, STMG_PROBLEM_MANUFACTURED, X, its.data()));
                  cudaEventRecord(e1);
                  cudaEventSynchronize(e1);
                  float ms = 0.0f;
                  cudaEventElapsedTime(&ms, e0, e1);
                  cudaFree(X);
                  double avg = 0.0;
                  for (int v : its)
                    avg += v;
                  avg /= run.n_steps;
                  unsigned long long sum_nt2 = 0;
                  for (int l = 1; l < run.n_levels; ++l)
                    {
                      int64_t sz[10];
                      check(stmg_level_sizes(stmg_solver_level(run.sol, l), sz));
                      sum_nt2 += static_cast<unsigned long long>(sz[7]);
                    }
                  const double thr = static_cast<double>(run.fine_size) * run.n_steps / (ms * 1e-3);
                  std::printf("%2d %2d %-12s %4d %-10.2f %-14llu %-12.4g\n", r, c, cell ? "cell" : "vertex_star", nsm,
                              avg, sum_nt2, thr);
                  if (csv)
                    csv << r << ',' << c << ',' << (cell ? "cell" : "vertex_star") << ',' << nsm << ',' << avg << ','
                        << sum_nt2 << '\n';
                }
        }
      else if (sub == "cavity")
        {
          const Problem cavity{STMG_PROBLEM_CAVITY, o.nu, 8.0}; // problems.cpp:64-78
          Run run(ctx, o, o.r, o.refinements, o.nu1, o.nu2, cavity, cell);
          double *X = nullptr;
          cudaMalloc(&X, sizeof(double) * run.fine_size * run.n_steps);
          std::vector<int> its(run.n_steps);
          cudaDeviceSynchronize();
          cudaEvent_t e0, e1;
          cudaEventCreate(&e0);
          cudaEventCreate(&e1);
          cudaEventRecord(e0);
          check(stmg_time_march_problem(run.sol, STMG_PROBLEM_CAVITY, X, its.data()));
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms = 0.0f;
          cudaEventElapsedTime(&ms, e0, e1);
          int64_t sz[10];
          check(stmg_level_sizes(stmg_solver_level(run.sol, run.n_levels - 1), sz));
          const int S = static_cast<int>(sz[0]);
          const int64_t mv = sz[1], mp = sz[2];
          const int nc = 1 << o.refinements;
          std::vector<double> p(mp);
          std::ofstream csv;
          if (!o.csv_path.empty())
            {
              csv.open(o.csv_path);
              csv.precision(12);
              csv << "t,p_probe1,p_probe2,p_diff\n";
            }
          std::printf("t        p(0.875,0.125)  p(0.875,0.875)  p_diff\n");
          const double tau = cavity.t_end / run.n_steps;
          for (int n = 1; n <= run.n_steps; ++n)
            {
              cudaMemcpy(p.data(), X + (n - 1) * run.fine_size + S * mv + (S - 1) * mp, sizeof(double) * mp,
                         cudaMemcpyDeviceToHost);
              const double p1 = pressure_at(p, nc, o.r, 0.875, 0.125), p2 = pressure_at(p, nc, o.r, 0.875, 0.875);
              const bool valid = std::abs(p1) >= 1e-12;
              if (valid)
                std::printf("%-8.4g %-15.6g %-15.6g %-10.6g\n", n * tau, p1, p2, (p1 - p2) / p1);
              else
                std::printf("%-8.4g %-15.6g %-15.6g (skipped)\n", n * tau, p1, p2);
              if (csv)
                {
                  csv << n * tau << ',' << p1 << ',' << p2 << ',';
                  if (valid)
                    csv << (p1 - p2) / p1;
                  csv << '\n';
                }
            }
          cudaFree(X);
          double avg = 0.0;
          for (int v : its)
            avg += v;
          avg /= run.n_steps;
          std::printf("avg GMRES iterations: %.2f, throughput %.4g dofs/s\n", avg,
                      static_cast<double>(run.fine_size) * run.n_steps / (ms * 1e-3));
          if (!o.steps_csv.empty())
            {
              std::ofstream st(o.steps_csv);
              st << "step,iterations\n";
              for (int n = 0; n < run.n_steps; ++n)
                st << n << ',' << its[n] << '\n';
            }
        }
      else if (sub == "hierarchy")
        {
          std::vector<int64_t> out(2 + 5 * 64);
          check(stmg_plan_levels(o.refinements, o.r, o.k, o.n_steps, 1.0, o.mode == "h_only" ? 1 : 0, out.data()));
          print_hierarchy(out, 1.0);
        }
      else if (sub == "selftest")
        {
          // GPU self-checks: the manufactured problem converges at the
          // theoretical order and the saddle-point record stays clean
          bool all = true;
          Options oc = o;
          oc.k = -1;
          double prev = 0.0;
          for (int c = 1; c <= 2; ++c)
            {
              Run run(ctx, oc, 2, c, 1, 1, manufactured, true);
              stmg_level *fine = stmg_solver_level(run.sol, run.n_levels - 1);
              double *X = nullptr;
              cudaMalloc(&X, sizeof(double) * run.fine_size * run.n_steps);
              std::vector<int> its(run.n_steps);
              check(stmg_time_march_problem(run.sol, STMG_PROBLEM_MANUFACTURED, X, its.data()));
              double e[5];
              check(stmg_compute_errors(fine, STMG_PROBLEM_MANUFACTURED, 0.0, X, run.n_steps, e));
              std::vector<double> h(2 * run.n_steps);
              check(stmg_step_health(fine, X, run.n_steps, h.data()));
              cudaFree(X);
              double worst = 0.0;
              for (int n = 0; n < run.n_steps; ++n)
                worst = std::max(worst, h[2 * n + 1]);
              const bool ok_mean = worst <= 1e-10;
              std::printf("[%s] pressure mean, c = %d: max |<m, p>| / |p| = %.3g\n", ok_mean ? "PASS" : "FAIL", c,
                          worst);
              all = all && ok_mean;
              if (c == 2)
                {
                  const double rate = eoc(prev, e[0]);
                  const bool ok = rate > 2.5; // r = 2: Q3 velocity, L2 order >= 3 in the asymptote
                  std::printf("[%s] velocity L2 EOC r = 2, c = 1 -> 2: %.2f\n", ok ? "PASS" : "FAIL", rate);
                  all = all && ok;
                }
              prev = e[0];
            }
          stmg_ctx_destroy(ctx);
          return all ? 0 : 1;
        }
      else
        return usage();
      if (ctx)
        stmg_ctx_destroy(ctx);
    }
  catch (const std::exception &e)
    {
      std::fprintf(stderr, "error: %s\n", e.what());
      return 1;
    }
  return 0;
}
