// Built-in problem data on the GPU: the load vector of SpaceTimeBlockOperator::
// assemble_rhs (st_operator.cpp:423-467) for the reference's manufactured
// problem (problems.cpp:13-62), its interpolant (interpolate_exact,
// harness.cpp:185-239) and the space-time error norms of compute_errors
// (harness.cpp:72-183). These close the loop of acceptance Table 1
// on the device: assemble -> time_march -> errors, with
// no host round trip of the trajectory.
#include "kernels.hpp"

#include <cuda_runtime.h>

namespace stmg_b200
{

namespace
{
constexpr double kPi = 3.14159265358979323846;

// problems.cpp:13-62 (sign-corrected manufactured solution, nu enters the force)
__device__ __forceinline__ double
mf_force(double sx, double cx, double sy, double cy, double st, double ct, double nu, int comp)
{
  if (comp == 0)
    return 0.25 * ct * (1.0 - cx) * sy - nu * st * kPi * kPi * sy * (2.0 * cx - 1.0) + 0.5 * kPi * st * cx * sy;
  return -0.25 * ct * sx * (1.0 - cy) - nu * st * kPi * kPi * sx * (1.0 - 2.0 * cy) + 0.5 * kPi * st * sx * cy;
}

// 2x2-coloured cell pass: cells of one colour share no velocity node, so the
// scatter is a plain read-modify-write (deterministic).
template <int R>
__global__ void
assemble_manufactured_kernel(DevGeom G, ProblemTables T, double nu, double t_start, double tau, double *F, int colour)
{
  constexpr int N1 = R + 2, NQ = R + 2, p = R + 1;
  const int ox = colour & 1, oy = colour >> 1;
  const int ncx = (G.nx - ox + 1) / 2, ncy = (G.ny - oy + 1) / 2;
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long long>(ncx) * ncy)
    return;
  const int n = blockIdx.y;
  const int cx = 2 * static_cast<int>(idx % ncx) + ox, cy = 2 * static_cast<int>(idx / ncx) + oy;
  const double x0 = cx * G.hx, y0 = cy * G.hy, jdet = 0.25 * G.hx * G.hy;
  double sxq[NQ], cxq[NQ], syq[NQ], cyq[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q)
    {
      sincos(2.0 * kPi * (x0 + 0.5 * G.hx * (T.ax[q] + 1.0)), &sxq[q], &cxq[q]);
      sincos(2.0 * kPi * (y0 + 0.5 * G.hy * (T.ax[q] + 1.0)), &syq[q], &cyq[q]);
    }
  double *Fn = F + n * G.isz;
  for (int a = 0; a < G.S; ++a)
    {
      const double t = t_start + n * tau + 0.5 * tau * (T.tn[a] + 1.0);
      const double wt = 0.5 * tau * T.tw[a];
      double st, ct;
      sincos(t, &st, &ct);
#pragma unroll
      for (int comp = 0; comp < 2; ++comp)
        {
          // (phi^T fq)(i, qy), then * phi -> loc(i, j)
          double A[N1][NQ];
#pragma unroll
          for (int i = 0; i < N1; ++i)
#pragma unroll
            for (int qy = 0; qy < NQ; ++qy)
              A[i][qy] = 0.0;
#pragma unroll
          for (int qx = 0; qx < NQ; ++qx)
#pragma unroll
            for (int qy = 0; qy < NQ; ++qy)
              {
                const double f = mf_force(sxq[qx], cxq[qx], syq[qy], cyq[qy], st, ct, nu, comp) * T.aw[qx] *
                                 T.aw[qy] * jdet * wt;
#pragma unroll
                for (int i = 0; i < N1; ++i)
                  A[i][qy] = fma(T.aphi[qx * N1 + i], f, A[i][qy]);
              }
          double *out = Fn + a * G.mv + comp * G.nsc;
#pragma unroll
          for (int j = 0; j < N1; ++j)
#pragma unroll
            for (int i = 0; i < N1; ++i)
              {
                double s = 0.0;
#pragma unroll
                for (int qy = 0; qy < NQ; ++qy)
                  s = fma(A[i][qy], T.aphi[qy * N1 + j], s);
                out[static_cast<long long>(cy * p + j) * G.gx + cx * p + i] += s;
              }
        }
    }
}

// exact solution of the manufactured problem
__device__ __forceinline__ void
mf_exact(double xp, double yp, double t, double &u0, double &u1, double g[4], double &pr)
{
  double sx, cx, sy, cy;
  sincos(2.0 * kPi * xp, &sx, &cx);
  sincos(2.0 * kPi * yp, &sy, &cy);
  const double stt = sin(t);
  const double s = 0.25 * stt, sg = 0.5 * kPi * stt;
  u0 = s * (1.0 - cx) * sy;
  u1 = -s * sx * (1.0 - cy);
  g[0] = sg * sx * sy;           // d u0 / dx
  g[1] = sg * (1.0 - cx) * cy;   // d u0 / dy
  g[2] = -sg * cx * (1.0 - cy);  // d u1 / dx
  g[3] = -sg * sx * sy;          // d u1 / dy
  pr = 0.25 * stt * sx * sy;
}

// interpolate_exact (harness.cpp:185-239), velocity: nodal values at the GLL
// grid, one thread per (scalar node, interval).
__global__ void
interp_velocity_kernel(DevGeom G, int p, ProblemTables T, double t_start, double tau, double *X)
{
  const long long s = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (s >= G.nsc)
    return;
  const int n = blockIdx.y;
  const int ix = static_cast<int>(s % G.gx), iy = static_cast<int>(s / G.gx);
  const int cx = min(ix / p, G.nx - 1), cy = min(iy / p, G.ny - 1);
  const double xp = cx * G.hx + 0.5 * G.hx * (T.gll[ix - cx * p] + 1.0);
  const double yp = cy * G.hy + 0.5 * G.hy * (T.gll[iy - cy * p] + 1.0);
  for (int a = 0; a < G.S; ++a)
    {
      const double t = t_start + n * tau + 0.5 * tau * (T.tn[a] + 1.0);
      double u0, u1, g[4], pr;
      mf_exact(xp, yp, t, u0, u1, g, pr);
      X[n * G.isz + a * G.mv + s] = u0;
      X[n * G.isz + a * G.mv + G.nsc + s] = u1;
    }
}

// pressure: per-cell L2 projection onto the orthogonal tensor-Legendre
// P_r^disc basis with Gauss(r+3), one thread per (cell, interval)
template <int R>
__global__ void
interp_pressure_kernel(DevGeom G, ProblemTables T, double t_start, double tau, double *X)
{
  constexpr int NQ = R + 3, NP = (R + 1) * (R + 2) / 2;
  const long long cell = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (cell >= static_cast<long long>(G.nx) * G.ny)
    return;
  const int n = blockIdx.y;
  const int cx = static_cast<int>(cell % G.nx), cy = static_cast<int>(cell / G.nx);
  const double x0 = cx * G.hx, y0 = cy * G.hy;
  for (int a = 0; a < G.S; ++a)
    {
      const double t = t_start + n * tau + 0.5 * tau * (T.tn[a] + 1.0);
      double rhs[NP];
#pragma unroll
      for (int l = 0; l < NP; ++l)
        rhs[l] = 0.0;
      for (int qy = 0; qy < NQ; ++qy)
        for (int qx = 0; qx < NQ; ++qx)
          {
            double u0, u1, g[4], pr;
            mf_exact(x0 + 0.5 * G.hx * (T.ex[qx] + 1.0), y0 + 0.5 * G.hy * (T.ex[qy] + 1.0), t, u0, u1, g, pr);
            const double wq = T.ew[qx] * T.ew[qy] * pr; // jdet cancels against the Gram scaling
#pragma unroll
            for (int l = 0; l < NP; ++l)
              rhs[l] = fma(wq, T.eleg[qx * (R + 1) + pdisc_mode_ax(R, l)] * T.eleg[qy * (R + 1) + pdisc_mode_ay(R, l)],
                           rhs[l]);
          }
#pragma unroll
      for (int l = 0; l < NP; ++l)
        {
          const int ax = pdisc_mode_ax(R, l), ay = pdisc_mode_ay(R, l);
          const double gram = (2.0 / (2 * ax + 1)) * (2.0 / (2 * ay + 1)); // pdisc.cpp gram_diagonal
          X[n * G.isz + G.S * G.mv + a * G.mp + cell * NP + l] = rhs[l] / gram;
        }
    }
}

// Lid-driven cavity boundary data (problems.cpp:64-78): u_x = sin(pi t / 4)
// on the open lid y = 1, 0 < x < 1; zero elsewhere. Writes the lift vector of
// time_march (solver.cpp:251-262): boundary values on the constrained nodes
// at the slot times (VelocitySpace::set_boundary_values, dof_space.cpp:71-81),
// zero everywhere else. Node coordinates follow dof_space.cpp:40-50 exactly
// (last grid line forced to the domain edge), so the y >= 1 test matches.
__global__ void
lift_cavity_kernel(DevGeom G, int p, ProblemTables T, double t_start, double tau, double *L)
{
  const long long s = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (s >= G.nsc)
    return;
  const int n = blockIdx.y;
  const int ix = static_cast<int>(s % G.gx), iy = static_cast<int>(s / G.gx);
  const bool bnd = ix == 0 || ix == G.gx - 1 || iy == 0 || iy == G.gy - 1;
  const auto coord = [&](int i, int g, double h) {
    if (i == g - 1)
      return 1.0;
    const int c = i / p;
    return h * (c + 0.5 * (T.gll[i - c * p] + 1.0));
  };
  const double xp = coord(ix, G.gx, G.hx), yp = coord(iy, G.gy, G.hy);
  for (int a = 0; a < G.S; ++a)
    {
      const double t = t_start + n * tau + 0.5 * tau * (T.tn[a] + 1.0);
      const double ux = (bnd && yp >= 1.0 && xp > 0.0 && xp < 1.0) ? sin(0.25 * kPi * t) : 0.0;
      L[n * G.isz + a * G.mv + s] = ux;
      L[n * G.isz + a * G.mv + G.nsc + s] = 0.0;
    }
}

constexpr int kErrThreads = 128;

// compute_errors (harness.cpp:72-183): one thread per (cell, interval);
// Gauss(k+2) in time, Gauss(r+3) in space; block partial sums, then a
// fixed-order final reduction (deterministic).
template <int R, int S>
__global__ void __launch_bounds__(kErrThreads)
errors_manufactured_kernel(DevGeom G, ProblemTables T, double t_start, double tau, const double *__restrict__ X,
                           int n_intervals, double *__restrict__ part)
{
  constexpr int N1 = R + 2, NQ = R + 3, p = R + 1, NP = (R + 1) * (R + 2) / 2, KQ = S + 1;
  const long long ncell = static_cast<long long>(G.nx) * G.ny;
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  double sv = 0.0, sp = 0.0, sh = 0.0, sd = 0.0, li = 0.0;
  if (idx < ncell * n_intervals)
    {
      const int n = static_cast<int>(idx / ncell);
      const long long cell = idx % ncell;
      const int cx = static_cast<int>(cell % G.nx), cy = static_cast<int>(cell / G.nx);
      const double x0 = cx * G.hx, y0 = cy * G.hy, jdet = 0.25 * G.hx * G.hy;
      const double dxi = 2.0 / G.hx, deta = 2.0 / G.hy;
      const double *Xn = X + n * G.isz;
      for (int tq = 0; tq < KQ; ++tq)
        {
          const double t = t_start + n * tau + 0.5 * tau * (T.tq[tq] + 1.0);
          const double wt = 0.5 * tau * T.tqw[tq];
          double ux[N1][N1], uy[N1][N1], pb[NP];
#pragma unroll
          for (int j = 0; j < N1; ++j)
#pragma unroll
            for (int i = 0; i < N1; ++i)
              ux[i][j] = uy[i][j] = 0.0;
#pragma unroll
          for (int l = 0; l < NP; ++l)
            pb[l] = 0.0;
#pragma unroll
          for (int a = 0; a < S; ++a)
            {
              const double c = T.tval[tq * S + a];
#pragma unroll
              for (int j = 0; j < N1; ++j)
#pragma unroll
                for (int i = 0; i < N1; ++i)
                  {
                    const long long node = static_cast<long long>(cy * p + j) * G.gx + cx * p + i;
                    ux[i][j] = fma(c, Xn[a * G.mv + node], ux[i][j]);
                    uy[i][j] = fma(c, Xn[a * G.mv + G.nsc + node], uy[i][j]);
                  }
#pragma unroll
              for (int l = 0; l < NP; ++l)
                pb[l] = fma(c, Xn[S * G.mv + a * G.mp + cell * NP + l], pb[l]);
            }
          for (int qx = 0; qx < NQ; ++qx)
            {
              // x-contractions at qx: value and x-derivative tables
              double Ax[N1], Bx[N1], Ay[N1], By[N1];
#pragma unroll
              for (int j = 0; j < N1; ++j)
                {
                  double a0 = 0, b0 = 0, a1 = 0, b1 = 0;
#pragma unroll
                  for (int i = 0; i < N1; ++i)
                    {
                      a0 = fma(T.ephi[qx * N1 + i], ux[i][j], a0);
                      b0 = fma(T.edphi[qx * N1 + i], ux[i][j], b0);
                      a1 = fma(T.ephi[qx * N1 + i], uy[i][j], a1);
                      b1 = fma(T.edphi[qx * N1 + i], uy[i][j], b1);
                    }
                  Ax[j] = a0;
                  Bx[j] = b0;
                  Ay[j] = a1;
                  By[j] = b1;
                }
              const double xp = x0 + 0.5 * G.hx * (T.ex[qx] + 1.0);
              for (int qy = 0; qy < NQ; ++qy)
                {
                  double vx = 0, vy = 0, dxx = 0, dxy = 0, dyx = 0, dyy = 0;
#pragma unroll
                  for (int j = 0; j < N1; ++j)
                    {
                      const double ph = T.ephi[qy * N1 + j], dph = T.edphi[qy * N1 + j];
                      vx = fma(Ax[j], ph, vx);
                      vy = fma(Ay[j], ph, vy);
                      dxx = fma(Bx[j], ph, dxx);
                      dxy = fma(Ax[j], dph, dxy);
                      dyx = fma(By[j], ph, dyx);
                      dyy = fma(Ay[j], dph, dyy);
                    }
                  const double yp = y0 + 0.5 * G.hy * (T.ex[qy] + 1.0);
                  const double wq = wt * T.ew[qx] * T.ew[qy] * jdet;
                  double u0, u1, g[4], pr;
                  mf_exact(xp, yp, t, u0, u1, g, pr);
                  const double e0 = vx - u0, e1 = vy - u1;
                  sv += wq * (e0 * e0 + e1 * e1);
                  li = fmax(li, fmax(fabs(e0), fabs(e1)));
                  const double g00 = dxi * dxx - g[0], g01 = deta * dxy - g[1];
                  const double g10 = dxi * dyx - g[2], g11 = deta * dyy - g[3];
                  sh += wq * (g00 * g00 + g01 * g01 + g10 * g10 + g11 * g11);
                  const double dv = dxi * dxx + deta * dyy;
                  sd += wq * dv * dv;
                  double pq = 0.0;
#pragma unroll
                  for (int l = 0; l < NP; ++l)
                    pq = fma(T.eleg[qx * (R + 1) + pdisc_mode_ax(R, l)] * T.eleg[qy * (R + 1) + pdisc_mode_ay(R, l)],
                             pb[l], pq);
                  const double ep = pq - pr;
                  sp += wq * ep * ep;
                }
            }
        }
    }
  __shared__ double red[5][kErrThreads];
  red[0][threadIdx.x] = sv;
  red[1][threadIdx.x] = sp;
  red[2][threadIdx.x] = sh;
  red[3][threadIdx.x] = sd;
  red[4][threadIdx.x] = li;
  __syncthreads();
  for (int s = kErrThreads / 2; s > 0; s >>= 1)
    {
      if (threadIdx.x < s)
        {
#pragma unroll
          for (int v = 0; v < 4; ++v)
            red[v][threadIdx.x] += red[v][threadIdx.x + s];
          red[4][threadIdx.x] = fmax(red[4][threadIdx.x], red[4][threadIdx.x + s]);
        }
      __syncthreads();
    }
  if (threadIdx.x < 5)
    part[blockIdx.x * 5 + threadIdx.x] = red[threadIdx.x][0];
}

__global__ void
errors_final_kernel(const double *__restrict__ part, int nblocks, double *__restrict__ out)
{
  // one thread per norm, fixed order over the blocks
  const int v = threadIdx.x;
  if (v >= 5)
    return;
  double s = 0.0;
  for (int b = 0; b < nblocks; ++b)
    s = v == 4 ? fmax(s, part[b * 5 + 4]) : s + part[b * 5 + v];
  out[v] = v == 4 ? s : sqrt(s);
}

template <int R>
cudaError_t
launch_errors_r(const DevGeom &G, const ProblemTables &T, double t_start, double tau, const double *X, int n,
                double *part, double *out, cudaStream_t st)
{
  const long long items = static_cast<long long>(G.nx) * G.ny * n;
  const int blocks = static_cast<int>((items + kErrThreads - 1) / kErrThreads);
  switch (G.S)
    {
      case 1: errors_manufactured_kernel<R, 1><<<blocks, kErrThreads, 0, st>>>(G, T, t_start, tau, X, n, part); break;
      case 2: errors_manufactured_kernel<R, 2><<<blocks, kErrThreads, 0, st>>>(G, T, t_start, tau, X, n, part); break;
      case 3: errors_manufactured_kernel<R, 3><<<blocks, kErrThreads, 0, st>>>(G, T, t_start, tau, X, n, part); break;
      case 4: errors_manufactured_kernel<R, 4><<<blocks, kErrThreads, 0, st>>>(G, T, t_start, tau, X, n, part); break;
      default: errors_manufactured_kernel<R, 5><<<blocks, kErrThreads, 0, st>>>(G, T, t_start, tau, X, n, part); break;
    }
  errors_final_kernel<<<1, 32, 0, st>>>(part, blocks, out);
  return cudaGetLastError();
}
} // namespace

long long
errors_partials(const DevGeom &G, int n_intervals)
{
  return 5 * ((static_cast<long long>(G.nx) * G.ny * n_intervals + kErrThreads - 1) / kErrThreads);
}

cudaError_t
launch_assemble_manufactured(const DevGeom &G, int r, const ProblemTables &T, double nu, double t_start, double tau,
                             double *F, int n_intervals, cudaStream_t st)
{
  if (n_intervals <= 0)
    return cudaSuccess;
  cudaMemsetAsync(F, 0, sizeof(double) * G.isz * n_intervals, st);
  for (int colour = 0; colour < 4; ++colour)
    {
      const long long ncells = static_cast<long long>((G.nx - (colour & 1) + 1) / 2) * ((G.ny - (colour >> 1) + 1) / 2);
      if (ncells == 0)
        continue;
      dim3 grid(static_cast<unsigned>((ncells + 127) / 128), n_intervals);
      switch (r)
        {
          case 1: assemble_manufactured_kernel<1><<<grid, 128, 0, st>>>(G, T, nu, t_start, tau, F, colour); break;
          case 2: assemble_manufactured_kernel<2><<<grid, 128, 0, st>>>(G, T, nu, t_start, tau, F, colour); break;
          case 3: assemble_manufactured_kernel<3><<<grid, 128, 0, st>>>(G, T, nu, t_start, tau, F, colour); break;
          default: assemble_manufactured_kernel<4><<<grid, 128, 0, st>>>(G, T, nu, t_start, tau, F, colour); break;
        }
    }
  return launch_zero_constrained(G, F, n_intervals, st); // st_operator.cpp:465
}

cudaError_t
launch_interpolate_manufactured(const DevGeom &G, int r, const ProblemTables &T, double t_start, double tau,
                                double *X, int n_intervals, cudaStream_t st)
{
  if (n_intervals <= 0)
    return cudaSuccess;
  dim3 gv(static_cast<unsigned>((G.nsc + 127) / 128), n_intervals);
  interp_velocity_kernel<<<gv, 128, 0, st>>>(G, r + 1, T, t_start, tau, X);
  const long long ncell = static_cast<long long>(G.nx) * G.ny;
  dim3 gp(static_cast<unsigned>((ncell + 127) / 128), n_intervals);
  switch (r)
    {
      case 1: interp_pressure_kernel<1><<<gp, 128, 0, st>>>(G, T, t_start, tau, X); break;
      case 2: interp_pressure_kernel<2><<<gp, 128, 0, st>>>(G, T, t_start, tau, X); break;
      case 3: interp_pressure_kernel<3><<<gp, 128, 0, st>>>(G, T, t_start, tau, X); break;
      default: interp_pressure_kernel<4><<<gp, 128, 0, st>>>(G, T, t_start, tau, X); break;
    }
  return cudaGetLastError();
}

cudaError_t
launch_lift_cavity(const DevGeom &G, int r, const ProblemTables &T, double t_start, double tau, double *L,
                   int n_intervals, cudaStream_t st)
{
  if (n_intervals <= 0)
    return cudaSuccess;
  cudaMemsetAsync(L, 0, sizeof(double) * G.isz * n_intervals, st);
  dim3 g(static_cast<unsigned>((G.nsc + 127) / 128), n_intervals);
  lift_cavity_kernel<<<g, 128, 0, st>>>(G, r + 1, T, t_start, tau, L);
  return cudaGetLastError();
}

cudaError_t
launch_errors_manufactured(const DevGeom &G, int r, const ProblemTables &T, double t_start, double tau,
                           const double *X, int n_intervals, double *part, double *out, cudaStream_t st)
{
  switch (r)
    {
      case 1: return launch_errors_r<1>(G, T, t_start, tau, X, n_intervals, part, out, st);
      case 2: return launch_errors_r<2>(G, T, t_start, tau, X, n_intervals, part, out, st);
      case 3: return launch_errors_r<3>(G, T, t_start, tau, X, n_intervals, part, out, st);
      default: return launch_errors_r<4>(G, T, t_start, tau, X, n_intervals, part, out, st);
    }
}

} // namespace stmg_b200
