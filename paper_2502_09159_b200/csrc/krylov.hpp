// Arnoldi orthogonalization of the FGMRES solvers (2D stmg.cu, 3D stmg3d.cu).
//
// The reference orthogonalizes by modified Gram-Schmidt (solver.cpp:146-152):
// j+1 inner products and updates per iteration, each inner product summed
// over the ranks of a time-slab partition (one all-reduce each). Classical
// Gram-Schmidt with re-orthogonalization (CGS2) computes the same Hessenberg
// column with two batched passes over the basis and two all-reduces per
// iteration, whatever j is:
//   pass 1: h = V^T w (one all-reduce), w -= V h
//   pass 2: c = V^T w and <w, w> (one all-reduce), w -= V c, h += c,
//           ||w||^2 = <w, w> - ||c||^2 (V orthonormal; c is O(eps) small
//           after pass 1, so the difference does not cancel).
// Both are deterministic (fixed-order reductions).
#pragma once

#include "kernels.hpp"
#include "runtime.hpp"

#include <cmath>
#include <memory>
#include <vector>

namespace stmg_krylov
{
using stmg_rt::check;
using stmg_rt::DevArray;

enum Ortho
{
  kMGS = 0,  // modified Gram-Schmidt, the reference's (solver.cpp:146-152)
  kCGS2 = 1, // classical Gram-Schmidt, twice; two all-reduces per iteration
};

/// No correction of the local inner products (unpartitioned vectors).
struct NoFix
{
  void operator()(const double *const *, int, bool, const double *, double *) const {}
};

/// Orthogonalize w against V[0..j]; hcol[0..j] receives the Hessenberg
/// column, the return value is ||w|| after orthogonalization. `part` must
/// hold part_doubles() doubles, `scal` 2 * (j + 2) or more. fix(V, m,
/// with_norm, w, out) runs after every local batch of inner products
/// (out[i] = <w, V_i>, out[m] = <w, w>) and before its all-reduce: a z-split
/// solver removes there the interface plane a part shares with its lower
/// neighbour, so every dof is counted once.
template <class Allreduce, class Fix = NoFix>
double
orthogonalize(int ortho, const std::vector<std::unique_ptr<DevArray<double>>> &V, int j, double *w, long long n,
              double *part, double *scal, std::vector<double> &hcol, Allreduce &&allreduce, stmg_ctx *ctx,
              Fix &&fix = Fix{})
{
  using namespace stmg_b200;
  cudaStream_t st = ctx->stream;
  hcol.resize(j + 2);
  if (ortho == kMGS)
    {
      for (int i = 0; i <= j; ++i)
        {
          check(launch_dot(w, V[i]->p, n, part, scal + i, st), "dot");
          const double *vi = V[i]->p;
          fix(&vi, 1, false, w, scal + i);
          allreduce(scal + i, 1);
          check(launch_axpy(n, 0.0, scal + i, -1.0, V[i]->p, w, st), "axpy");
          ctx->count(3);
        }
      check(launch_dot(w, w, n, part, scal + j + 1, st), "dot");
      fix(nullptr, 0, true, w, scal + j + 1);
      allreduce(scal + j + 1, 1);
      ctx->count(2);
      check(cudaMemcpyAsync(hcol.data(), scal, sizeof(double) * (j + 2), cudaMemcpyDeviceToHost, st), "d2h");
      check(cudaStreamSynchronize(st), "sync");
      return std::sqrt(hcol[j + 1]);
    }
  std::vector<const double *> ptr(j + 1);
  for (int i = 0; i <= j; ++i)
    ptr[i] = V[i]->p;
  const int chunks = (j + 1 + kMultiMax - 1) / kMultiMax;
  double *h1 = scal, *h2 = scal + (j + 1);
  check(launch_multidot(ptr.data(), j + 1, false, w, n, part, h1, st), "multidot");
  fix(ptr.data(), j + 1, false, w, h1);
  allreduce(h1, j + 1);
  check(launch_multi_axpy(ptr.data(), j + 1, h1, nullptr, -1.0, w, n, st), "multi_axpy");
  check(launch_multidot(ptr.data(), j + 1, true, w, n, part, h2, st), "multidot");
  fix(ptr.data(), j + 1, true, w, h2);
  allreduce(h2, j + 2);
  check(launch_multi_axpy(ptr.data(), j + 1, h2, nullptr, -1.0, w, n, st), "multi_axpy");
  ctx->count(6 * chunks);
  std::vector<double> hh(2 * j + 3);
  check(cudaMemcpyAsync(hh.data(), scal, sizeof(double) * (2 * j + 3), cudaMemcpyDeviceToHost, st), "d2h");
  check(cudaStreamSynchronize(st), "sync");
  double cc = 0.0;
  for (int i = 0; i <= j; ++i)
    {
      const double c = hh[j + 1 + i];
      hcol[i] = hh[i] + c;
      cc += c * c;
    }
  const double ww = hh[2 * j + 2] - cc;
  hcol[j + 1] = ww > 0.0 ? ww : 0.0;
  return std::sqrt(hcol[j + 1]);
}

/// x += sum_i y_i Z_i in batched passes (the solution update, solver.cpp:187-200).
inline void
update_solution(const std::vector<std::unique_ptr<DevArray<double>>> &Z, const std::vector<double> &y, double *x,
                long long n, stmg_ctx *ctx)
{
  using namespace stmg_b200;
  const int m = static_cast<int>(y.size());
  if (m == 0)
    return;
  std::vector<const double *> ptr(m);
  for (int i = 0; i < m; ++i)
    ptr[i] = Z[i]->p;
  check(launch_multi_axpy(ptr.data(), m, nullptr, y.data(), 1.0, x, n, ctx->stream), "multi_axpy");
  ctx->count((m + kMultiMax - 1) / kMultiMax);
}

/// Scratch doubles for `part` of orthogonalize().
inline int
part_doubles()
{
  return (stmg_b200::kMultiMax + 1) * stmg_b200::dot_partials();
}
} // namespace stmg_krylov
