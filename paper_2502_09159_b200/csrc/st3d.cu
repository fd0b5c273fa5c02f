// 3D kernels of the B200 hp-STMG path (BASELINE C3 / C5), sm_100a, FP64.
//
// vmult3: the space-time operator of one interval or the all-at-once system
//   y_n = D x_n - Z C x_{n-1}[slot k]       (Eq. GloSys)
// composed exactly as SpaceTimeBlockOperator::apply_block_impl
// (st_operator.cpp:321-407, here with three velocity components) plus
// coupling_rhs (st_operator.cpp:409-421). Per output slot a the temporal
// Kronecker combination is done first on nodal values (UK = sum_b Kt(a,b) u^b
// - lv_a v_prev, UM = sum_b Mt(a,b) u^b, PM = sum_b Mt(a,b) p^b), so each
// slot costs one spatial Stokes cell operator:
//   y_v^a = M UK + (nu A + gamma G) UM - B^T PM,   y_p^a = B UM.
// The cell operator is evaluated by sum factorisation through the Gauss
// points (r+2 per direction, st_operator.cpp:167) with the trilinear cell map
// evaluated on the fly: Cartesian cells use the constant Jacobian, deformed
// cells (C5) read their 8 vertices (24 doubles) instead of precomputed
// per-point geometry.
//
// Mapping: a thread block holds CB cells; each cell is worked by N*N threads,
// one per 1D line of its N^3 node / quadrature-point tile. Every
// sum-factorisation pass loads a line into registers, applies the 1D matrix
// (constant bank, compile-time indices) and writes the line back in place,
// so passes need no scratch beyond 13 fields per cell in shared memory.
// Velocity contributions are scattered with red.global.add.f64 into y, which
// a first kernel initialises (0, b, or the identity rows of constrained
// dofs); cell-owned pressure rows are written directly.
#include "st3d.hpp"

#include <algorithm>
#include <cstdlib>
#include <cuda_runtime.h>

namespace stmg_b200
{

namespace
{
template <int R, int MAP = 0, bool DEF = false>
struct V3
{
  static constexpr int N = R + 2, NN = N * N, NNN = N * N * N, p = R + 1;
  static constexpr int NP = (R + 1) * (R + 2) * (R + 3) / 6;
  // MAP 0, lane = cell: a warp works one line of CW cells (two lines per
  // warp), so a warp's shared accesses hit CW different cells at the same
  // offset (odd cell stride: conflict-free) and its global gathers walk
  // consecutive cells along x. MAP 1, line = thread: N*N consecutive threads
  // work the lines of one cell (fewer registers per resident cell; used at
  // r = 1, where more cells in flight beat conflict-free banks).
  static constexpr int CW = 16;
  static constexpr int LPW = 32 / CW;
  static constexpr int NWARP = (NN + LPW - 1) / LPW;
  static constexpr int THREADS = MAP == 0 ? 32 * NWARP : NN * CW;
  static constexpr int NF = 13; // in-place fields per cell
  // deformed cells cache J^{-1} (9) and det (1) per Gauss point: computed in
  // the first output slot, reused by the others
  static constexpr int GC = DEF ? 10 * NNN : 0;
  static constexpr int CELL = NF * NNN + NP + 24 + GC + 1 - (NF * NNN + NP + 24 + GC) % 2; // odd
  static constexpr size_t smem() { return sizeof(double) * (CW * CELL + NP * NNN + 2 * N); }
};

#ifndef STMG_V3_MAP1_MINB
#define STMG_V3_MAP1_MINB 3
#endif
#ifndef STMG_V3_MAP1_CELLMINOR
#define STMG_V3_MAP1_CELLMINOR 1
#endif
// Forward 1D contraction of a line: o[q] = sum_m M(q, m) in[m] (M = phi /
// dphi, constant bank, compile-time indices).
#define V3_FWD(M, in, o)                                                                                             \
  _Pragma("unroll") for (int q_ = 0; q_ < N; ++q_)                                                                   \
  {                                                                                                                  \
    double s_ = 0.0;                                                                                                 \
    _Pragma("unroll") for (int m_ = 0; m_ < N; ++m_) s_ = fma(P.M[q_ * N + m_], in[m_], s_);                         \
    o[q_] = s_;                                                                                                      \
  }

template <int R, int S, int MODE, int MAP = 0, bool DEF = true>
__global__ void __launch_bounds__(V3<R, MAP, DEF>::THREADS, MAP == 0 ? 1 : (DEF ? 2 : STMG_V3_MAP1_MINB))
vmult3_kernel(const Level3Consts P, const double *__restrict__ x, const double *__restrict__ b,
              double *__restrict__ y, const double *__restrict__ xprev0, int coupled, long long n_cells_total)
{
  using C = V3<R, MAP, DEF>;
  constexpr int N = C::N, NN = C::NN, NNN = C::NNN, p = C::p, NP = C::NP, CW = C::CW;
  extern __shared__ __align__(16) double sm3[];
  double *const psi = sm3 + CW * C::CELL; // psi[m * NNN + q]: P_r^disc mode m at Gauss point q
  double *const tw = psi + NP * NNN;      // Gauss weights, points
  double *const txq = tw + N;
  for (int e = threadIdx.x; e < NP * NNN; e += C::THREADS)
    {
      const int m = e / NNN, q = e - m * NNN;
      const int qx = q % N, qy = (q / N) % N, qz = q / NN;
      double v = 1.0;
#pragma unroll
      for (int mm = 0; mm < NP; ++mm)
        if (mm == m)
          v = P.leg[P.ex[mm][0] * N + qx] * P.leg[P.ex[mm][1] * N + qy] * P.leg[P.ex[mm][2] * N + qz];
      psi[e] = v;
    }
#pragma unroll
  for (int q = 0; q < N; ++q)
    if (threadIdx.x == q)
      {
        tw[q] = P.w[q];
        txq[q] = P.xq[q];
      }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#if STMG_V3_MAP1_CELLMINOR
  // MAP 1 cell-minor: a half-warp = one line of CW cells (conflict-free, as MAP 0), fewer registers per thread
  const int cl = MAP == 0 ? lane % CW : static_cast<int>(threadIdx.x) % CW;             // cell in block
  const int t = MAP == 0 ? warp * C::LPW + lane / CW : static_cast<int>(threadIdx.x) / CW; // line index
#else
  const int cl = MAP == 0 ? lane % CW : static_cast<int>(threadIdx.x) / NN;             // cell in block
  const int t = MAP == 0 ? warp * C::LPW + lane / CW : static_cast<int>(threadIdx.x) % NN; // line index
#endif
  const long long gc = static_cast<long long>(blockIdx.x) * CW + cl;
  const bool active = gc < n_cells_total && t < NN;
  const long long ncells = static_cast<long long>(P.nx) * P.ny * P.nz;
  const int n = gc < n_cells_total ? static_cast<int>(gc / ncells) : 0;
  const long long cell = gc < n_cells_total ? gc - n * ncells : 0;
  const int cx = static_cast<int>(cell % P.nx), cy = static_cast<int>((cell / P.nx) % P.ny),
            cz = static_cast<int>(cell / (static_cast<long long>(P.nx) * P.ny));
  double *const F = sm3 + cl * C::CELL;
  double *const PM = F + C::NF * NNN;
  double *const X8 = PM + NP;
  double *const GCa = X8 + 24; // deformed: [point][10] J^{-1}, det
  const int tA = t % N, tB = t / N; // line coordinates
  const long long isz = P.isz, mv = P.mv, mp = P.mp, nsc = P.nsc;
  const int gx = P.gx, gy = P.gy;
  constexpr bool deformed = DEF; // Cartesian instantiations use the diagonal Jacobian
  const double *__restrict__ xn = x + n * isz;
  const double *__restrict__ vprev = nullptr;
  if (coupled)
    vprev = n > 0 ? x + (n - 1) * isz + (S - 1) * mv : xprev0;
  if (active && deformed)
    for (int q = t; q < 24; q += NN)
      {
        const int c = q / 3, d = q % 3;
        const int vx = cx + (c & 1), vy = cy + ((c >> 1) & 1), vz = cz + (c >> 2);
        X8[q] = __ldg(P.verts + ((static_cast<long long>(vz) * (P.ny + 1) + vy) * (P.nx + 1) + vx) * 3 + d);
      }
  // fields (in place): F[c] VK_c, F[3+c] Ax/AA/T0/Yb, F[6+c] Dx/DA/T1, F[9+c] AD, F[12] QP
  auto fld = [&](int f) { return F + f * NNN; };
  // line bases: x-line (j = tA, k = tB), y-line (i = tA, k = tB), z-line (i = tA, j = tB)
  const int bx = (tB * N + tA) * N, by = tB * NN + tA, bz = tB * N + tA;
  __syncthreads(); // tables

  for (int a = 0; a < S; ++a)
    {
      double kt[S], mt[S], lva = 0.0;
#pragma unroll
      for (int aa = 0; aa < S; ++aa)
        if (a == aa)
          {
#pragma unroll
            for (int bs = 0; bs < S; ++bs)
              {
                kt[bs] = P.Kt[aa * S + bs];
                mt[bs] = P.Mt[aa * S + bs];
              }
            lva = P.lv[aa];
          }
      // ---- phase 1 (x-lines): gather, temporal combination, x-contraction
      if (active)
        {
          const int Y = cy * p + tA, Z = cz * p + tB;
          const bool yzb = MODE != 2 && (Y == 0 || Z == P.zlo || Y == gy - 1 || Z == P.zhi);
          const long long row = (static_cast<long long>(Z) * gy + Y) * gx + cx * p;
#pragma unroll
          for (int c = 0; c < 3; ++c)
            {
              double uk[N], um[N], o[N];
#pragma unroll
              for (int i = 0; i < N; ++i)
                {
                  const int X = cx * p + i;
                  const bool bnd = yzb || (MODE != 2 && (X == 0 || X == gx - 1));
                  double k_ = 0.0, m_ = 0.0;
                  if (!bnd)
#pragma unroll
                    for (int bs = 0; bs < S; ++bs)
                      {
                        const double v = __ldg(xn + bs * mv + c * nsc + row + i);
                        k_ = fma(kt[bs], v, k_);
                        m_ = fma(mt[bs], v, m_);
                      }
                  if (vprev != nullptr)
                    k_ = fma(-lva, __ldg(vprev + c * nsc + row + i), k_);
                  uk[i] = k_;
                  um[i] = m_;
                }
              V3_FWD(phi, uk, o)
#pragma unroll
              for (int q = 0; q < N; ++q)
                fld(c)[bx + q] = o[q];
              V3_FWD(phi, um, o)
#pragma unroll
              for (int q = 0; q < N; ++q)
                fld(3 + c)[bx + q] = o[q];
              V3_FWD(dphi, um, o)
#pragma unroll
              for (int q = 0; q < N; ++q)
                fld(6 + c)[bx + q] = o[q];
            }
          if (t < NP)
            {
              double s = 0.0;
#pragma unroll
              for (int bs = 0; bs < S; ++bs)
                s = fma(mt[bs], __ldg(xn + S * mv + bs * mp + cell * NP + t), s);
              PM[t] = s;
            }
        }
      __syncthreads();
      // ---- phase 2 (y-lines, in place): VK; Ax -> AA (phi_y), AD (dphi_y, F[9+c]); Dx -> DA
      if (active)
        {
#pragma unroll
          for (int c = 0; c < 3; ++c)
            {
              double in[N], o[N];
#pragma unroll
              for (int m = 0; m < N; ++m)
                in[m] = fld(c)[by + m * N];
              V3_FWD(phi, in, o)
#pragma unroll
              for (int q = 0; q < N; ++q)
                fld(c)[by + q * N] = o[q];
#pragma unroll
              for (int m = 0; m < N; ++m)
                in[m] = fld(3 + c)[by + m * N];
              V3_FWD(phi, in, o)
#pragma unroll
              for (int q = 0; q < N; ++q)
                fld(3 + c)[by + q * N] = o[q];
              V3_FWD(dphi, in, o)
#pragma unroll
              for (int q = 0; q < N; ++q)
                fld(9 + c)[by + q * N] = o[q];
#pragma unroll
              for (int m = 0; m < N; ++m)
                in[m] = fld(6 + c)[by + m * N];
              V3_FWD(phi, in, o)
#pragma unroll
              for (int q = 0; q < N; ++q)
                fld(6 + c)[by + q * N] = o[q];
            }
        }
      __syncthreads();
      // ---- phase 3 (z-lines, in place): z-contraction, fluxes at the Gauss
      // points, transposed z-contraction, all in registers:
      // Sv_c = phi_z^T Fval_c + dphi_z^T Fref_c2 (F[c]), T0_c = phi_z^T Fref_c0
      // (F[3+c]), T1_c = phi_z^T Fref_c1 (F[6+c]); QP = w det div (F[12])
      if (active)
        {
          double vk[3][N], g[3][3][N];
#pragma unroll
          for (int c = 0; c < 3; ++c)
            {
              double in[N];
#pragma unroll
              for (int m = 0; m < N; ++m)
                in[m] = fld(c)[bz + m * NN];
              V3_FWD(phi, in, vk[c])
#pragma unroll
              for (int m = 0; m < N; ++m)
                in[m] = fld(6 + c)[bz + m * NN];
              V3_FWD(phi, in, g[c][0])
#pragma unroll
              for (int m = 0; m < N; ++m)
                in[m] = fld(9 + c)[bz + m * NN];
              V3_FWD(phi, in, g[c][1])
#pragma unroll
              for (int m = 0; m < N; ++m)
                in[m] = fld(3 + c)[bz + m * NN];
              V3_FWD(dphi, in, g[c][2])
            }
          double sv[3][N], t0[3][N], t1[3][N];
#pragma unroll
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int i = 0; i < N; ++i)
              sv[c][i] = t0[c][i] = t1[c][i] = 0.0;
          const double wxy = tw[tA] * tw[tB];
#pragma unroll
          for (int qz = 0; qz < N; ++qz)
            {
              double Ji[3][3], det, jd[3];
              if constexpr (!deformed)
                {
                  jd[0] = 2.0 / P.hx;
                  jd[1] = 2.0 / P.hy;
                  jd[2] = 2.0 / P.hz;
                  det = 0.125 * P.hx * P.hy * P.hz;
                }
              else if (a > 0)
                {
                  const double *gp = GCa + (qz * NN + bz) * 10;
#pragma unroll
                  for (int e = 0; e < 9; ++e)
                    Ji[e / 3][e % 3] = gp[e];
                  det = gp[9];
                }
              else
                {
                  const double xi[3] = {txq[tA], txq[tB], P.xq[qz]};
                  double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
                  for (int v = 0; v < 8; ++v)
                    {
                      const double n0 = (v & 1) ? 0.5 * (1 + xi[0]) : 0.5 * (1 - xi[0]);
                      const double n1 = ((v >> 1) & 1) ? 0.5 * (1 + xi[1]) : 0.5 * (1 - xi[1]);
                      const double n2 = (v >> 2) ? 0.5 * (1 + xi[2]) : 0.5 * (1 - xi[2]);
                      const double d0 = (v & 1) ? 0.5 : -0.5, d1 = ((v >> 1) & 1) ? 0.5 : -0.5,
                                   d2 = (v >> 2) ? 0.5 : -0.5;
                      const double dN[3] = {d0 * n1 * n2, n0 * d1 * n2, n0 * n1 * d2};
#pragma unroll
                      for (int d = 0; d < 3; ++d)
#pragma unroll
                        for (int e = 0; e < 3; ++e)
                          J[d][e] = fma(X8[3 * v + d], dN[e], J[d][e]);
                    }
                  det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                        J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                        J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
                  const double id = 1.0 / det;
                  Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) * id;
                  Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * id;
                  Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * id;
                  Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) * id;
                  Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * id;
                  Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * id;
                  Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) * id;
                  Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * id;
                  Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * id;
                  if (S > 1)
                    {
                      double *gp = GCa + (qz * NN + bz) * 10;
#pragma unroll
                      for (int e = 0; e < 9; ++e)
                        gp[e] = Ji[e / 3][e % 3];
                      gp[9] = det;
                    }
                }
              const double wd = P.w[qz] * wxy * det;
              double G[3][3];
#pragma unroll
              for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int d = 0; d < 3; ++d)
                  if constexpr (deformed)
                    G[c][d] = g[c][0][qz] * Ji[0][d] + g[c][1][qz] * Ji[1][d] + g[c][2][qz] * Ji[2][d];
                  else
                    G[c][d] = g[c][d][qz] * jd[d];
              const double div = G[0][0] + G[1][1] + G[2][2];
              const int q = qz * NN + bz;
              double pq = 0.0;
#pragma unroll
              for (int m = 0; m < NP; ++m)
                pq = fma(psi[m * NNN + q], PM[m], pq);
              const double diag = P.gamma * div - pq;
              fld(12)[q] = wd * div;
#pragma unroll
              for (int c = 0; c < 3; ++c)
                {
                  double Fp[3];
#pragma unroll
                  for (int d = 0; d < 3; ++d)
                    Fp[d] = wd * (P.nu * G[c][d] + (c == d ? diag : 0.0));
                  double Fr[3];
#pragma unroll
                  for (int e = 0; e < 3; ++e)
                    if constexpr (deformed)
                      Fr[e] = Fp[0] * Ji[e][0] + Fp[1] * Ji[e][1] + Fp[2] * Ji[e][2];
                    else
                      Fr[e] = Fp[e] * jd[e];
                  const double fv = wd * vk[c][qz];
#pragma unroll
                  for (int i = 0; i < N; ++i)
                    {
                      sv[c][i] = fma(P.phi[qz * N + i], fv, sv[c][i]);
                      sv[c][i] = fma(P.dphi[qz * N + i], Fr[2], sv[c][i]);
                      t0[c][i] = fma(P.phi[qz * N + i], Fr[0], t0[c][i]);
                      t1[c][i] = fma(P.phi[qz * N + i], Fr[1], t1[c][i]);
                    }
                }
            }
#pragma unroll
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int i = 0; i < N; ++i)
              {
                fld(c)[bz + i * NN] = sv[c][i];
                fld(3 + c)[bz + i * NN] = t0[c][i];
                fld(6 + c)[bz + i * NN] = t1[c][i];
              }
        }
      __syncthreads();
      // ---- phase 4 (y-lines, in place): Ya_c = phi_y^T Sv_c + dphi_y^T T1_c (F[c]),
      // Yb_c = phi_y^T T0_c (F[3+c]); pressure rows from QP
      if (active)
        {
#pragma unroll
          for (int c = 0; c < 3; ++c)
            {
              double in[N], in2[N], in3[N];
#pragma unroll
              for (int m = 0; m < N; ++m)
                {
                  in[m] = fld(c)[by + m * N];
                  in2[m] = fld(6 + c)[by + m * N];
                  in3[m] = fld(3 + c)[by + m * N];
                }
#pragma unroll
              for (int i = 0; i < N; ++i)
                {
                  double s1 = 0.0, s2 = 0.0;
#pragma unroll
                  for (int q = 0; q < N; ++q)
                    {
                      s1 = fma(P.phi[q * N + i], in[q], s1);
                      s1 = fma(P.dphi[q * N + i], in2[q], s1);
                      s2 = fma(P.phi[q * N + i], in3[q], s2);
                    }
                  fld(c)[by + i * N] = s1;
                  fld(3 + c)[by + i * N] = s2;
                }
            }
          if (t < NP)
            {
              const double *qp = fld(12);
              const double *ps = psi + t * NNN;
              double s = 0.0;
#pragma unroll
              for (int q = 0; q < NNN; ++q)
                s = fma(ps[q], qp[q], s);
              const long long o = n * isz + S * mv + a * mp + cell * NP + t;
              y[o] = MODE == 1 ? __ldg(b + o) - s : s;
            }
        }
      __syncthreads();
      // ---- phase 5 (x-lines): y = phi_x^T Ya + dphi_x^T Yb, scattered from registers
      if (active)
        {
          const int Y = cy * p + tA, Z = cz * p + tB;
          const bool yzb = Y == 0 || Z == P.zlo || Y == gy - 1 || Z == P.zhi;
#pragma unroll
          for (int c = 0; c < 3; ++c)
            {
              double in[N], in2[N];
#pragma unroll
              for (int m = 0; m < N; ++m)
                {
                  in[m] = fld(c)[bx + m];
                  in2[m] = fld(3 + c)[bx + m];
                }
              double *yv = y + n * isz + a * mv + c * nsc + (static_cast<long long>(Z) * gy + Y) * gx + cx * p;
#pragma unroll
              for (int i = 0; i < N; ++i)
                {
                  double s = 0.0;
#pragma unroll
                  for (int q = 0; q < N; ++q)
                    {
                      s = fma(P.phi[q * N + i], in[q], s);
                      s = fma(P.dphi[q * N + i], in2[q], s);
                    }
                  const int X = cx * p + i;
                  const bool bnd = MODE != 2 && (yzb || X == 0 || X == gx - 1);
                  if (!bnd)
                    atomicAdd(yv + i, MODE == 1 ? -s : s);
                }
            }
        }
      // the next slot's phase 1 rewrites this thread's own x-line (fields
      // 0..8) and nothing another thread still reads: no barrier here
    }
}
#undef V3_FWD

// ---------------------------------------------------------------------------
// Deformed cells, two blocks per SM (vmult3d_kernel, default for r >= 2 on
// deformed levels). Same lane = cell map, passes and fields as vmult3_kernel,
// but phase 3 runs in three thread-local steps on the thread's own z-line
// (which no other thread touches between the surrounding barriers), with the
// shared-memory fields as the staging space instead of registers:
//   3a z-contraction of the four y-pass fields, in place;
//   3b point loop: geometry, gradients, fluxes, written back in place;
//   3c transposed z-contraction, in place.
// No per-point J^{-1}/det cache: the trilinear map is kept as its 8 monomial
// coefficients per cell (X(xi) = sum_S c_S prod_{i in S} xi_i), so along a
// z-line each Jacobian column is affine in zeta and costs 2 FMAs per entry.
// 12 fields per cell (the divergence moments reuse field 9 once the z-flux
// is consumed): 105 KB per 16-cell block at r = 2, two blocks (16 warps) per
// SM, against one block (8 warps, 255 registers) for vmult3_kernel.
template <int R>
struct V3D
{
  static constexpr int N = R + 2, NN = N * N, NNN = N * N * N, p = R + 1;
  static constexpr int NP = (R + 1) * (R + 2) * (R + 3) / 6;
  static constexpr int CW = 16, LPW = 2, NWARP = (NN + 1) / 2, THREADS = 32 * NWARP;
  static constexpr int NF = 12;
  static constexpr int CELL = NF * NNN + NP + 24 + 1 - (NF * NNN + NP + 24) % 2; // odd
  static constexpr size_t smem() { return sizeof(double) * (CW * CELL + (R + 1) * N + 2 * N); }
#ifndef STMG_V3D_MINB_R1
#define STMG_V3D_MINB_R1 3 // 2 / 3 / 4 blocks per SM: 2.66 / 2.39 / 2.46 ms (4 spills)
#endif
  static constexpr int MINB = R == 1 ? STMG_V3D_MINB_R1 : (smem() <= 112 * 1024 ? 2 : 1);
};

/// Exponent d of P_r^disc mode m in 3D, in the order of modes3() (setup3d.cpp,
/// pdisc.cpp:41-55): degree-major, then descending x, then descending y.
/// Called with unrolled (constant) m, so it folds to a constant.
__host__ __device__ constexpr int
mode3_ex(int r, int m, int d)
{
  int i = 0;
  for (int deg = 0; deg <= r; ++deg)
    for (int a = deg; a >= 0; --a)
      for (int b = deg - a; b >= 0; --b, ++i)
        if (i == m)
          return d == 0 ? a : (d == 1 ? b : deg - a - b);
  return 0;
}

#define V3_FWD(M, in, o)                                                                                             \
  _Pragma("unroll") for (int q_ = 0; q_ < N; ++q_)                                                                   \
  {                                                                                                                  \
    double s_ = 0.0;                                                                                                 \
    _Pragma("unroll") for (int m_ = 0; m_ < N; ++m_) s_ = fma(P.M[q_ * N + m_], in[m_], s_);                         \
    o[q_] = s_;                                                                                                      \
  }

template <int R, int S, int MODE>
__global__ void __launch_bounds__(V3D<R>::THREADS, V3D<R>::MINB)
vmult3d_kernel(const Level3Consts P, const double *__restrict__ x, const double *__restrict__ b,
               double *__restrict__ y, const double *__restrict__ xprev0, int coupled, long long n_cells_total)
{
  using C = V3D<R>;
  constexpr int N = C::N, NN = C::NN, NNN = C::NNN, p = C::p, NP = C::NP, CW = C::CW;
  extern __shared__ __align__(16) double sm3[];
  double *const lg = sm3 + CW * C::CELL; // Legendre L_e(x_q) at [e * N + q]
  double *const tw = lg + (R + 1) * N;
  double *const txq = tw + N;
  for (int e = threadIdx.x; e < (R + 1) * N; e += C::THREADS)
    lg[e] = P.leg[e];
#pragma unroll
  for (int q = 0; q < N; ++q)
    if (threadIdx.x == q)
      {
        tw[q] = P.w[q];
        txq[q] = P.xq[q];
      }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cl = lane % CW, t = warp * C::LPW + lane / CW; // cell in block, line index
  const long long gc = static_cast<long long>(blockIdx.x) * CW + cl;
  const bool active = gc < n_cells_total && t < NN;
  const long long ncells = static_cast<long long>(P.nx) * P.ny * P.nz;
  const int n = gc < n_cells_total ? static_cast<int>(gc / ncells) : 0;
  const long long cell = gc < n_cells_total ? gc - n * ncells : 0;
  const int cx = static_cast<int>(cell % P.nx), cy = static_cast<int>((cell / P.nx) % P.ny),
            cz = static_cast<int>(cell / (static_cast<long long>(P.nx) * P.ny));
  double *const F = sm3 + cl * C::CELL;
  double *const PM = F + C::NF * NNN;
  double *const CF = PM + NP; // trilinear map coefficients c_S[d] at CF[3 * S + d]
  const int tA = t % N, tB = t / N;
  const long long isz = P.isz, mv = P.mv, mp = P.mp, nsc = P.nsc;
  const int gx = P.gx, gy = P.gy;
  const double *__restrict__ xn = x + n * isz;
  const double *__restrict__ vprev = nullptr;
  if (coupled)
    vprev = n > 0 ? x + (n - 1) * isz + (S - 1) * mv : xprev0;
  if (active)
    for (int u = t; u < 24; u += NN)
    {
      // c_S[d] = 1/8 sum_v X_v[d] prod_{i in S} s_{v,i}, s_{v,i} = +-1 by vertex bit i
      const int Sm = u / 3, d = u % 3;
      double c = 0.0;
#pragma unroll
      for (int v = 0; v < 8; ++v)
        {
          const int vx = cx + (v & 1), vy = cy + ((v >> 1) & 1), vz = cz + (v >> 2);
          const double X = __ldg(P.verts + ((static_cast<long long>(vz) * (P.ny + 1) + vy) * (P.nx + 1) + vx) * 3 + d);
          c += (__popc(v & Sm) & 1) ? -X : X;
        }
      // the sign above is prod_{i in S} s_{v,i} with s = -1 where bit i of v is 0: flip for |S| odd
      CF[u] = 0.125 * ((__popc(Sm) & 1) ? -c : c);
    }
  auto fld = [&](int f) { return F + f * NNN; };
  const int bx = (tB * N + tA) * N, by = tB * NN + tA, bz = tB * N + tA;
  __syncthreads();

  for (int a = 0; a < S; ++a)
    {
      double kt[S], mt[S], lva = 0.0;
#pragma unroll
      for (int aa = 0; aa < S; ++aa)
        if (a == aa)
          {
#pragma unroll
            for (int bs = 0; bs < S; ++bs)
              {
                kt[bs] = P.Kt[aa * S + bs];
                mt[bs] = P.Mt[aa * S + bs];
              }
            lva = P.lv[aa];
          }
      // ---- phase 1 (x-lines): gather, temporal combination, x-contraction
      if (active)
        {
          const int Y = cy * p + tA, Z = cz * p + tB;
          const bool yzb = MODE != 2 && (Y == 0 || Z == P.zlo || Y == gy - 1 || Z == P.zhi);
          const long long row = (static_cast<long long>(Z) * gy + Y) * gx + cx * p;
#pragma unroll
          for (int c = 0; c < 3; ++c)
            {
              double uk[N], um[N], o[N];
#pragma unroll
              for (int i = 0; i < N; ++i)
                {
                  const int X = cx * p + i;
                  const bool bnd = yzb || (MODE != 2 && (X == 0 || X == gx - 1));
                  double k_ = 0.0, m_ = 0.0;
                  if (!bnd)
#pragma unroll
                    for (int bs = 0; bs < S; ++bs)
                      {
                        const double v = __ldg(xn + bs * mv + c * nsc + row + i);
                        k_ = fma(kt[bs], v, k_);
                        m_ = fma(mt[bs], v, m_);
                      }
                  if (vprev != nullptr)
                    k_ = fma(-lva, __ldg(vprev + c * nsc + row + i), k_);
                  uk[i] = k_;
                  um[i] = m_;
                }
              V3_FWD(phi, uk, o)
#pragma unroll
              for (int q = 0; q < N; ++q)
                fld(c)[bx + q] = o[q];
              V3_FWD(phi, um, o)
#pragma unroll
              for (int q = 0; q < N; ++q)
                fld(3 + c)[bx + q] = o[q];
              V3_FWD(dphi, um, o)
#pragma unroll
              for (int q = 0; q < N; ++q)
                fld(6 + c)[bx + q] = o[q];
            }
          if (t < NP)
            {
              double s = 0.0;
#pragma unroll
              for (int bs = 0; bs < S; ++bs)
                s = fma(mt[bs], __ldg(xn + S * mv + bs * mp + cell * NP + t), s);
              PM[t] = s;
            }
        }
      __syncthreads();
      // ---- phase 2 (y-lines, in place): VK; Ax -> AA (phi_y), AD (dphi_y, F[9+c]); Dx -> DA
      if (active)
        {
#pragma unroll
          for (int c = 0; c < 3; ++c)
            {
              double in[N], o[N];
#pragma unroll
              for (int m = 0; m < N; ++m)
                in[m] = fld(c)[by + m * N];
              V3_FWD(phi, in, o)
#pragma unroll
              for (int q = 0; q < N; ++q)
                fld(c)[by + q * N] = o[q];
#pragma unroll
              for (int m = 0; m < N; ++m)
                in[m] = fld(3 + c)[by + m * N];
              V3_FWD(phi, in, o)
#pragma unroll
              for (int q = 0; q < N; ++q)
                fld(3 + c)[by + q * N] = o[q];
              V3_FWD(dphi, in, o)
#pragma unroll
              for (int q = 0; q < N; ++q)
                fld(9 + c)[by + q * N] = o[q];
#pragma unroll
              for (int m = 0; m < N; ++m)
                in[m] = fld(6 + c)[by + m * N];
              V3_FWD(phi, in, o)
#pragma unroll
              for (int q = 0; q < N; ++q)
                fld(6 + c)[by + q * N] = o[q];
            }
        }
      __syncthreads();
      // ---- phase 3 (z-lines, thread-local: no barrier between 3a, 3b, 3c)
      if (active)
        {
          // 3a: F[c] -> vk_c, F[6+c] -> g_c0, F[9+c] -> g_c1 (phi_z); F[3+c] -> g_c2 (dphi_z).
          // Rolled loops: unrolled, ptxas hoists every field's loads and spills.
#pragma unroll 1
          for (int f = 0; f < 12; ++f)
            {
              double in[N], o[N];
              double *const fz = fld(f) + bz;
#pragma unroll
              for (int m = 0; m < N; ++m)
                in[m] = fz[m * NN];
              if (f >= 3 && f < 6)
                {
                  V3_FWD(dphi, in, o)
#pragma unroll
                  for (int q = 0; q < N; ++q)
                    fz[q * NN] = o[q];
                }
              else
                {
                  V3_FWD(phi, in, o)
#pragma unroll
                  for (int q = 0; q < N; ++q)
                    fz[q * NN] = o[q];
                }
            }
          // 3b: per Gauss point (vk_c stays in F[c], its weight w det in wdq): Fr_c0 -> F[3+c], Fr_c1 -> F[6+c], Fr_c2 -> F[9+c]
          const double xi = txq[tA], eta = txq[tB], wxy = tw[tA] * tw[tB];
          double j0a[3], j0b[3], j1a[3], j1b[3], j2[3]; // J[:,0] = j0a + j0b zeta, J[:,1] = j1a + j1b zeta
#pragma unroll
          for (int d = 0; d < 3; ++d)
            {
              j0a[d] = fma(CF[3 * 3 + d], eta, CF[3 * 1 + d]);
              j0b[d] = fma(CF[3 * 7 + d], eta, CF[3 * 5 + d]);
              j1a[d] = fma(CF[3 * 3 + d], xi, CF[3 * 2 + d]);
              j1b[d] = fma(CF[3 * 7 + d], xi, CF[3 * 6 + d]);
              j2[d] = fma(CF[3 * 7 + d], xi * eta, fma(CF[3 * 6 + d], eta, fma(CF[3 * 5 + d], xi, CF[3 * 4 + d])));
            }
          // pressure at the line's Gauss points: p(qz) = sum_e2 L_e2(z_qz) w2[e2],
          // w2[e2] = sum over modes of z-degree e2 of L_e0(x_tA) L_e1(y_tB) PM[m]
          double w2[R + 1], lx[R + 1], ly[R + 1];
#pragma unroll
          for (int e = 0; e <= R; ++e)
            {
              w2[e] = 0.0;
              lx[e] = lg[e * N + tA];
              ly[e] = lg[e * N + tB];
            }
#pragma unroll
          for (int m = 0; m < NP; ++m)
            {
              double fx = 0.0, fy = 0.0; // selects, not indices: the arrays stay in registers
#pragma unroll
              for (int e = 0; e <= R; ++e)
                {
                  fx = mode3_ex(R, m, 0) == e ? lx[e] : fx;
                  fy = mode3_ex(R, m, 1) == e ? ly[e] : fy;
                }
              const double v = fx * fy * PM[m];
#pragma unroll
              for (int e = 0; e <= R; ++e)
                w2[e] += mode3_ex(R, m, 2) == e ? v : 0.0;
            }
          double qp[N], wdq[N];
#pragma unroll 1
          for (int qz = 0; qz < N; ++qz)
            {
              const int q = qz * NN + bz;
              const double ze = P.xq[qz];
              double J[3][3];
#pragma unroll
              for (int d = 0; d < 3; ++d)
                {
                  J[d][0] = fma(j0b[d], ze, j0a[d]);
                  J[d][1] = fma(j1b[d], ze, j1a[d]);
                  J[d][2] = j2[d];
                }
              const double a00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
              const double a10 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
              const double a20 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
              const double det = J[0][0] * a00 + J[0][1] * a10 + J[0][2] * a20;
              const double id = 1.0 / det;
              double Ji[3][3];
              Ji[0][0] = a00 * id;
              Ji[1][0] = a10 * id;
              Ji[2][0] = a20 * id;
              Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * id;
              Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * id;
              Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * id;
              Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * id;
              Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * id;
              Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * id;
              const double wd = P.w[qz] * wxy * det;
              double G[3][3];
#pragma unroll
              for (int c = 0; c < 3; ++c)
                {
                  const double g0 = fld(6 + c)[q], g1 = fld(9 + c)[q], g2 = fld(3 + c)[q];
#pragma unroll
                  for (int d = 0; d < 3; ++d)
                    G[c][d] = g0 * Ji[0][d] + g1 * Ji[1][d] + g2 * Ji[2][d];
                }
              const double div = G[0][0] + G[1][1] + G[2][2];
              double pq = 0.0;
#pragma unroll
              for (int e = 0; e <= R; ++e)
                pq = fma(P.leg[e * N + qz], w2[e], pq);
              const double diag = P.gamma * div - pq;
#pragma unroll
              for (int i = 0; i < N; ++i) // register-resident: select, no dynamic index
                if (i == qz)
                  {
                    qp[i] = wd * div;
                    wdq[i] = wd;
                  }
#pragma unroll
              for (int c = 0; c < 3; ++c)
                {
                  double Fp[3];
#pragma unroll
                  for (int d = 0; d < 3; ++d)
                    Fp[d] = wd * (P.nu * G[c][d] + (c == d ? diag : 0.0));
#pragma unroll
                  for (int e = 0; e < 3; ++e)
                    fld(3 * (e + 1) + c)[q] = Fp[0] * Ji[e][0] + Fp[1] * Ji[e][1] + Fp[2] * Ji[e][2];
                }
            }
          // 3c: Sv_c = phi_z^T (w det vk_c) + dphi_z^T Fr_c2 -> F[c]; T0_c = phi_z^T Fr_c0 -> F[3+c];
          // T1_c = phi_z^T Fr_c1 -> F[6+c]; then QP -> F[9]
#pragma unroll 1
          for (int c = 0; c < 3; ++c)
            {
              double fv[N], f2[N], o[N];
#pragma unroll
              for (int m = 0; m < N; ++m)
                {
                  fv[m] = wdq[m] * fld(c)[bz + m * NN];
                  f2[m] = fld(9 + c)[bz + m * NN];
                }
#pragma unroll
              for (int i = 0; i < N; ++i)
                {
                  double s = 0.0;
#pragma unroll
                  for (int q = 0; q < N; ++q)
                    {
                      s = fma(P.phi[q * N + i], fv[q], s);
                      s = fma(P.dphi[q * N + i], f2[q], s);
                    }
                  o[i] = s;
                }
#pragma unroll
              for (int i = 0; i < N; ++i)
                fld(c)[bz + i * NN] = o[i];
#pragma unroll
              for (int e = 0; e < 2; ++e)
                {
                  double in[N];
#pragma unroll
                  for (int m = 0; m < N; ++m)
                    in[m] = fld(3 * (e + 1) + c)[bz + m * NN];
#pragma unroll
                  for (int i = 0; i < N; ++i)
                    {
                      double s = 0.0;
#pragma unroll
                      for (int q = 0; q < N; ++q)
                        s = fma(P.phi[q * N + i], in[q], s);
                      o[i] = s;
                    }
#pragma unroll
                  for (int i = 0; i < N; ++i)
                    fld(3 * (e + 1) + c)[bz + i * NN] = o[i];
                }
            }
#pragma unroll
          for (int i = 0; i < N; ++i)
            fld(9)[bz + i * NN] = qp[i];
        }
      __syncthreads();
      // ---- phase 4 (y-lines, in place): Ya_c = phi_y^T Sv_c + dphi_y^T T1_c (F[c]),
      // Yb_c = phi_y^T T0_c (F[3+c]); pressure rows from QP (F[9])
      if (active)
        {
#pragma unroll
          for (int c = 0; c < 3; ++c)
            {
              double in[N], in2[N], in3[N];
#pragma unroll
              for (int m = 0; m < N; ++m)
                {
                  in[m] = fld(c)[by + m * N];
                  in2[m] = fld(6 + c)[by + m * N];
                  in3[m] = fld(3 + c)[by + m * N];
                }
#pragma unroll
              for (int i = 0; i < N; ++i)
                {
                  double s1 = 0.0, s2 = 0.0;
#pragma unroll
                  for (int q = 0; q < N; ++q)
                    {
                      s1 = fma(P.phi[q * N + i], in[q], s1);
                      s1 = fma(P.dphi[q * N + i], in2[q], s1);
                      s2 = fma(P.phi[q * N + i], in3[q], s2);
                    }
                  fld(c)[by + i * N] = s1;
                  fld(3 + c)[by + i * N] = s2;
                }
            }
          if (t < NP)
            {
              // separable: s = sum_qz L_e2(z) sum_qy L_e1(y) sum_qx L_e0(x) QP
              const double *qpf = fld(9);
              int e0 = 0, e1 = 0, e2 = 0;
#pragma unroll
              for (int m = 0; m < NP; ++m)
                if (m == t)
                  {
                    e0 = mode3_ex(R, m, 0);
                    e1 = mode3_ex(R, m, 1);
                    e2 = mode3_ex(R, m, 2);
                  }
              double lxq[N];
#pragma unroll
              for (int q = 0; q < N; ++q)
                lxq[q] = lg[e0 * N + q];
              double s = 0.0;
#pragma unroll
              for (int qz = 0; qz < N; ++qz)
                {
                  double sy = 0.0;
#pragma unroll
                  for (int qy = 0; qy < N; ++qy)
                    {
                      double sx = 0.0;
#pragma unroll
                      for (int qx = 0; qx < N; ++qx)
                        sx = fma(lxq[qx], qpf[(qz * N + qy) * N + qx], sx);
                      sy = fma(lg[e1 * N + qy], sx, sy);
                    }
                  s = fma(lg[e2 * N + qz], sy, s);
                }
              const long long o = n * isz + S * mv + a * mp + cell * NP + t;
              y[o] = MODE == 1 ? __ldg(b + o) - s : s;
            }
        }
      __syncthreads();
      // ---- phase 5 (x-lines): y = phi_x^T Ya + dphi_x^T Yb, scattered from registers
      if (active)
        {
          const int Y = cy * p + tA, Z = cz * p + tB;
          const bool yzb = Y == 0 || Z == P.zlo || Y == gy - 1 || Z == P.zhi;
#pragma unroll
          for (int c = 0; c < 3; ++c)
            {
              double in[N], in2[N];
#pragma unroll
              for (int m = 0; m < N; ++m)
                {
                  in[m] = fld(c)[bx + m];
                  in2[m] = fld(3 + c)[bx + m];
                }
              double *yv = y + n * isz + a * mv + c * nsc + (static_cast<long long>(Z) * gy + Y) * gx + cx * p;
#pragma unroll
              for (int i = 0; i < N; ++i)
                {
                  double s = 0.0;
#pragma unroll
                  for (int q = 0; q < N; ++q)
                    {
                      s = fma(P.phi[q * N + i], in[q], s);
                      s = fma(P.dphi[q * N + i], in2[q], s);
                    }
                  const int X = cx * p + i;
                  const bool bnd = MODE != 2 && (yzb || X == 0 || X == gx - 1);
                  if (!bnd)
                    atomicAdd(yv + i, MODE == 1 ? -s : s);
                }
            }
        }
      // the next slot's phase 1 rewrites only this thread's own x-line of
      // fields 0..8, which phase 5 alone read: no barrier here
    }
}
#undef V3_FWD

// ---------------------------------------------------------------------------
// Line-per-thread variant (r = 1): N*N threads per cell, 16 cells per block,
// 13 in-place fields; every pass reads / writes shared memory. At r = 1 it
// keeps more warps resident than the lane-per-cell kernel below
// (C3 vmult 8.9 ms vs 11.3 ms measured on the B200).
template <int R>
struct V3L
{
  static constexpr int N = R + 2, NN = N * N, NNN = N * N * N, p = R + 1;
  static constexpr int NP = (R + 1) * (R + 2) * (R + 3) / 6;
  static constexpr int CB = R == 1 ? 16 : (R == 2 ? 8 : 4); // cells per block
  static constexpr int NF = 13;                             // fields per cell
  static constexpr int CELL = NF * NNN + NP + 24;           // doubles per cell
  // block-wide tables (dynamic indexing): w, xq, leg, ex
  static constexpr int TAB = 2 * N + (R + 1) * N;
  static constexpr size_t smem() { return sizeof(double) * (CB * CELL + TAB) + sizeof(int) * 3 * NP; }
};


template <int R, int S, int MODE>
__global__ void __launch_bounds__(V3L<R>::NN *V3L<R>::CB)
vmult3l_kernel(const Level3Consts P, const double *__restrict__ x, const double *__restrict__ b,
              double *__restrict__ y, const double *__restrict__ xprev0, int coupled, long long n_cells_total)
{
  using C = V3L<R>;
  constexpr int N = C::N, NN = C::NN, NNN = C::NNN, p = C::p, NP = C::NP;
  extern __shared__ __align__(16) double sm3[];
  double *const tw = sm3 + C::CB * C::CELL; // w[N], xq[N], leg[(R+1) * N]
  double *const txq = tw + N;
  double *const tleg = txq + N;
  int *const tex = reinterpret_cast<int *>(tleg + (R + 1) * N);
  const int tid = threadIdx.y * NN + threadIdx.x;
  if (tid < N)
    {
      tw[tid] = P.w[0];
#pragma unroll
      for (int q = 0; q < N; ++q)
        if (tid == q)
          {
            tw[q] = P.w[q];
            txq[q] = P.xq[q];
#pragma unroll
            for (int a = 0; a <= R; ++a)
              tleg[a * N + q] = P.leg[a * N + q];
          }
    }
#pragma unroll
  for (int m = 0; m < NP; ++m)
    if (tid == m)
      {
        tex[3 * m] = P.ex[m][0];
        tex[3 * m + 1] = P.ex[m][1];
        tex[3 * m + 2] = P.ex[m][2];
      }

  const long long gc = static_cast<long long>(blockIdx.x) * C::CB + threadIdx.y;
  const bool active = gc < n_cells_total;
  const long long ncells = static_cast<long long>(P.nx) * P.ny * P.nz;
  const int n = active ? static_cast<int>(gc / ncells) : 0;
  const long long cell = active ? gc - n * ncells : 0;
  const int cx = static_cast<int>(cell % P.nx), cy = static_cast<int>((cell / P.nx) % P.ny),
            cz = static_cast<int>(cell / (static_cast<long long>(P.nx) * P.ny));
  double *const F = sm3 + threadIdx.y * C::CELL;
  double *const PM = F + C::NF * NNN;
  double *const X8 = PM + NP;
  const int t = threadIdx.x;
  const int tA = t % N, tB = t / N; // line coordinates
  const long long isz = P.isz, mv = P.mv, mp = P.mp, nsc = P.nsc;
  const int gx = P.gx, gy = P.gy;
  const bool deformed = P.verts != nullptr;
  const double *__restrict__ xn = x + n * isz;
  const double *__restrict__ vprev = nullptr;
  if (coupled)
    vprev = n > 0 ? x + (n - 1) * isz + (S - 1) * mv : xprev0;
  if (active && deformed)
    for (int q = t; q < 24; q += NN)
      {
        const int c = q / 3, d = q % 3;
        const int vx = cx + (c & 1), vy = cy + ((c >> 1) & 1), vz = cz + (c >> 2);
        X8[q] = __ldg(P.verts + ((static_cast<long long>(vz) * (P.ny + 1) + vy) * (P.nx + 1) + vx) * 3 + d);
      }
  // field indices: VK[c] = c, G[c][e] = 3 + 3c + e, QP = 12
  auto fld = [&](int f) { return F + f * NNN; };

  for (int a = 0; a < S; ++a)
    {
      double kt[S], mt[S], lva = 0.0;
#pragma unroll
      for (int aa = 0; aa < S; ++aa)
        if (a == aa)
          {
#pragma unroll
            for (int bs = 0; bs < S; ++bs)
              {
                kt[bs] = P.Kt[aa * S + bs];
                mt[bs] = P.Mt[aa * S + bs];
              }
            lva = P.lv[aa];
          }
      __syncthreads(); // tables ready; previous slot's fields consumed
      // ---- gather: x-line (j = tA, k = tB)
      if (active)
        {
          const int Y = cy * p + tA, Z = cz * p + tB;
#pragma unroll
          for (int i = 0; i < N; ++i)
            {
              const int X = cx * p + i;
              const long long node = (static_cast<long long>(Z) * gy + Y) * gx + X;
              const bool bnd = MODE != 2 && (X == 0 || Y == 0 || Z == P.zlo || X == gx - 1 || Y == gy - 1 || Z == P.zhi);
              const int li = (tB * N + tA) * N + i;
#pragma unroll
              for (int c = 0; c < 3; ++c)
                {
                  double uk = 0.0, um = 0.0;
                  if (!bnd)
#pragma unroll
                    for (int bs = 0; bs < S; ++bs)
                      {
                        const double v = __ldg(xn + bs * mv + c * nsc + node);
                        uk = fma(kt[bs], v, uk);
                        um = fma(mt[bs], v, um);
                      }
                  if (vprev != nullptr)
                    uk = fma(-lva, __ldg(vprev + c * nsc + node), uk);
                  fld(c)[li] = uk;
                  fld(3 + 3 * c)[li] = um;
                }
            }
          if (t < NP)
            {
              double s = 0.0;
#pragma unroll
              for (int bs = 0; bs < S; ++bs)
                s = fma(mt[bs], __ldg(xn + S * mv + bs * mp + cell * NP + t), s);
              PM[t] = s;
            }
        }
      __syncthreads();
      // ---- forward passes (nodes -> Gauss points)
      // x: VK value; UM -> A = phi_x UM (into G[c][2]), D = dphi_x UM (into G[c][0])
      if (active)
        {
          const int base = (tB * N + tA) * N; // x-line
#pragma unroll
          for (int c = 0; c < 3; ++c)
            {
              double in[N], o1[N], o2[N];
              double *vk = fld(c) + base;
#pragma unroll
              for (int m = 0; m < N; ++m)
                in[m] = vk[m];
#pragma unroll
              for (int q = 0; q < N; ++q)
                {
                  double s = 0.0;
#pragma unroll
                  for (int m = 0; m < N; ++m)
                    s = fma(P.phi[q * N + m], in[m], s);
                  o1[q] = s;
                }
#pragma unroll
              for (int q = 0; q < N; ++q)
                vk[q] = o1[q];
              double *g0 = fld(3 + 3 * c) + base, *g2 = fld(5 + 3 * c) + base;
#pragma unroll
              for (int m = 0; m < N; ++m)
                in[m] = g0[m];
#pragma unroll
              for (int q = 0; q < N; ++q)
                {
                  double s1 = 0.0, s2 = 0.0;
#pragma unroll
                  for (int m = 0; m < N; ++m)
                    {
                      s1 = fma(P.phi[q * N + m], in[m], s1);
                      s2 = fma(P.dphi[q * N + m], in[m], s2);
                    }
                  o1[q] = s1;
                  o2[q] = s2;
                }
#pragma unroll
              for (int q = 0; q < N; ++q)
                {
                  g2[q] = o1[q];
                  g0[q] = o2[q];
                }
            }
        }
      __syncthreads();
      // y: VK value; A -> AA (phi_y, in G[c][2]), AD (dphi_y, into G[c][1]); D -> DA (phi_y, in G[c][0])
      if (active)
        {
          const int base = tB * NN + tA; // y-line (i = tA, k = tB), stride N
#pragma unroll
          for (int c = 0; c < 3; ++c)
            {
              double in[N], o1[N], o2[N];
              double *vk = fld(c) + base;
#pragma unroll
              for (int m = 0; m < N; ++m)
                in[m] = vk[m * N];
#pragma unroll
              for (int q = 0; q < N; ++q)
                {
                  double s = 0.0;
#pragma unroll
                  for (int m = 0; m < N; ++m)
                    s = fma(P.phi[q * N + m], in[m], s);
                  o1[q] = s;
                }
#pragma unroll
              for (int q = 0; q < N; ++q)
                vk[q * N] = o1[q];
              double *g0 = fld(3 + 3 * c) + base, *g1 = fld(4 + 3 * c) + base, *g2 = fld(5 + 3 * c) + base;
#pragma unroll
              for (int m = 0; m < N; ++m)
                in[m] = g2[m * N];
#pragma unroll
              for (int q = 0; q < N; ++q)
                {
                  double s1 = 0.0, s2 = 0.0;
#pragma unroll
                  for (int m = 0; m < N; ++m)
                    {
                      s1 = fma(P.phi[q * N + m], in[m], s1);
                      s2 = fma(P.dphi[q * N + m], in[m], s2);
                    }
                  o1[q] = s1;
                  o2[q] = s2;
                }
#pragma unroll
              for (int q = 0; q < N; ++q)
                {
                  g2[q * N] = o1[q];
                  g1[q * N] = o2[q];
                }
#pragma unroll
              for (int m = 0; m < N; ++m)
                in[m] = g0[m * N];
#pragma unroll
              for (int q = 0; q < N; ++q)
                {
                  double s = 0.0;
#pragma unroll
                  for (int m = 0; m < N; ++m)
                    s = fma(P.phi[q * N + m], in[m], s);
                  o1[q] = s;
                }
#pragma unroll
              for (int q = 0; q < N; ++q)
                g0[q * N] = o1[q];
            }
        }
      __syncthreads();
      // z: VK value; DA -> d/dxi (phi_z); AD -> d/deta (phi_z); AA -> d/dzeta (dphi_z)
      if (active)
        {
          const int base = tB * N + tA; // z-line (i = tA, j = tB), stride NN
#pragma unroll
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int f = 0; f < 4; ++f)
              {
                double *fp = f == 0 ? fld(c) + base : fld(3 + 3 * c + (f - 1)) + base;
                const bool der = f == 3;
                double in[N], o1[N];
#pragma unroll
                for (int m = 0; m < N; ++m)
                  in[m] = fp[m * NN];
#pragma unroll
                for (int q = 0; q < N; ++q)
                  {
                    double s = 0.0;
#pragma unroll
                    for (int m = 0; m < N; ++m)
                      s = fma(der ? P.dphi[q * N + m] : P.phi[q * N + m], in[m], s);
                    o1[q] = s;
                  }
#pragma unroll
                for (int q = 0; q < N; ++q)
                  fp[q * NN] = o1[q];
              }
        }
      __syncthreads();
      // ---- quadrature points: x-line (qy = tA, qz = tB)
      if (active)
        {
          const double wyz = tw[tA] * tw[tB];
#pragma unroll
          for (int qx = 0; qx < N; ++qx)
            {
              const int li = (tB * N + tA) * N + qx;
              double Ji[3][3], det;
              if (!deformed)
                {
                  Ji[0][0] = 2.0 / P.hx;
                  Ji[1][1] = 2.0 / P.hy;
                  Ji[2][2] = 2.0 / P.hz;
                  Ji[0][1] = Ji[0][2] = Ji[1][0] = Ji[1][2] = Ji[2][0] = Ji[2][1] = 0.0;
                  det = 0.125 * P.hx * P.hy * P.hz;
                }
              else
                {
                  const double xi[3] = {P.xq[qx], txq[tA], txq[tB]};
                  double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
                  for (int v = 0; v < 8; ++v)
                    {
                      const double n0 = (v & 1) ? 0.5 * (1 + xi[0]) : 0.5 * (1 - xi[0]);
                      const double n1 = ((v >> 1) & 1) ? 0.5 * (1 + xi[1]) : 0.5 * (1 - xi[1]);
                      const double n2 = (v >> 2) ? 0.5 * (1 + xi[2]) : 0.5 * (1 - xi[2]);
                      const double d0 = (v & 1) ? 0.5 : -0.5, d1 = ((v >> 1) & 1) ? 0.5 : -0.5,
                                   d2 = (v >> 2) ? 0.5 : -0.5;
                      const double dN[3] = {d0 * n1 * n2, n0 * d1 * n2, n0 * n1 * d2};
#pragma unroll
                      for (int d = 0; d < 3; ++d)
#pragma unroll
                        for (int e = 0; e < 3; ++e)
                          J[d][e] = fma(X8[3 * v + d], dN[e], J[d][e]);
                    }
                  det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                        J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                        J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
                  const double id = 1.0 / det;
                  Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) * id;
                  Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * id;
                  Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * id;
                  Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) * id;
                  Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * id;
                  Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * id;
                  Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) * id;
                  Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * id;
                  Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * id;
                }
              const double wd = P.w[qx] * wyz * det;
              // physical gradient G(c, d) = sum_e dUM_c/dxi_e Ji(e, d)
              double G[3][3];
#pragma unroll
              for (int c = 0; c < 3; ++c)
                {
                  const double g0 = fld(3 + 3 * c)[li], g1 = fld(4 + 3 * c)[li], g2 = fld(5 + 3 * c)[li];
#pragma unroll
                  for (int d = 0; d < 3; ++d)
                    G[c][d] = g0 * Ji[0][d] + g1 * Ji[1][d] + g2 * Ji[2][d];
                }
              const double div = G[0][0] + G[1][1] + G[2][2];
              double pq = 0.0;
              for (int m = 0; m < NP; ++m)
                pq = fma(tleg[tex[3 * m] * N + qx] * tleg[tex[3 * m + 1] * N + tA] * tleg[tex[3 * m + 2] * N + tB],
                         PM[m], pq);
              const double diag = P.gamma * div - pq;
#pragma unroll
              for (int c = 0; c < 3; ++c)
                {
                  double Fp[3];
#pragma unroll
                  for (int d = 0; d < 3; ++d)
                    Fp[d] = wd * (P.nu * G[c][d] + (c == d ? diag : 0.0));
#pragma unroll
                  for (int e = 0; e < 3; ++e)
                    fld(3 + 3 * c + e)[li] = Fp[0] * Ji[e][0] + Fp[1] * Ji[e][1] + Fp[2] * Ji[e][2];
                  fld(c)[li] *= wd;
                }
              fld(12)[li] = wd * div;
            }
        }
      __syncthreads();
      // ---- pressure rows: y_p(l) = sum_q psi_l(q) wd div(q)
      if (active && t < NP)
        {
          const int e0 = tex[3 * t], e1 = tex[3 * t + 1], e2 = tex[3 * t + 2];
          double s = 0.0;
          for (int qz = 0; qz < N; ++qz)
            for (int qy = 0; qy < N; ++qy)
              {
                const double lyz = tleg[e1 * N + qy] * tleg[e2 * N + qz];
#pragma unroll
                for (int qx = 0; qx < N; ++qx)
                  s = fma(tleg[e0 * N + qx] * lyz, fld(12)[(qz * N + qy) * N + qx], s);
              }
          const long long o = n * isz + S * mv + a * mp + cell * NP + t;
          y[o] = MODE == 1 ? __ldg(b + o) - s : s;
        }
      // ---- transpose passes (Gauss points -> nodes)
      // z: VK <- phi_z^T VK + dphi_z^T G2; G0 <- phi_z^T G0; G1 <- phi_z^T G1
      if (active)
        {
          const int base = tB * N + tA;
#pragma unroll
          for (int c = 0; c < 3; ++c)
            {
              double in[N], in2[N], o1[N];
              double *vk = fld(c) + base, *g2 = fld(5 + 3 * c) + base;
#pragma unroll
              for (int m = 0; m < N; ++m)
                {
                  in[m] = vk[m * NN];
                  in2[m] = g2[m * NN];
                }
#pragma unroll
              for (int i = 0; i < N; ++i)
                {
                  double s = 0.0;
#pragma unroll
                  for (int q = 0; q < N; ++q)
                    {
                      s = fma(P.phi[q * N + i], in[q], s);
                      s = fma(P.dphi[q * N + i], in2[q], s);
                    }
                  o1[i] = s;
                }
#pragma unroll
              for (int i = 0; i < N; ++i)
                vk[i * NN] = o1[i];
#pragma unroll
              for (int f = 0; f < 2; ++f)
                {
                  double *fp = fld(3 + 3 * c + f) + base;
#pragma unroll
                  for (int m = 0; m < N; ++m)
                    in[m] = fp[m * NN];
#pragma unroll
                  for (int i = 0; i < N; ++i)
                    {
                      double s = 0.0;
#pragma unroll
                      for (int q = 0; q < N; ++q)
                        s = fma(P.phi[q * N + i], in[q], s);
                      o1[i] = s;
                    }
#pragma unroll
                  for (int i = 0; i < N; ++i)
                    fp[i * NN] = o1[i];
                }
            }
        }
      __syncthreads();
      // y: VK <- phi_y^T VK + dphi_y^T G1; G0 <- phi_y^T G0
      if (active)
        {
          const int base = tB * NN + tA;
#pragma unroll
          for (int c = 0; c < 3; ++c)
            {
              double in[N], in2[N], o1[N];
              double *vk = fld(c) + base, *g1 = fld(4 + 3 * c) + base, *g0 = fld(3 + 3 * c) + base;
#pragma unroll
              for (int m = 0; m < N; ++m)
                {
                  in[m] = vk[m * N];
                  in2[m] = g1[m * N];
                }
#pragma unroll
              for (int i = 0; i < N; ++i)
                {
                  double s = 0.0;
#pragma unroll
                  for (int q = 0; q < N; ++q)
                    {
                      s = fma(P.phi[q * N + i], in[q], s);
                      s = fma(P.dphi[q * N + i], in2[q], s);
                    }
                  o1[i] = s;
                }
#pragma unroll
              for (int i = 0; i < N; ++i)
                vk[i * N] = o1[i];
#pragma unroll
              for (int m = 0; m < N; ++m)
                in[m] = g0[m * N];
#pragma unroll
              for (int i = 0; i < N; ++i)
                {
                  double s = 0.0;
#pragma unroll
                  for (int q = 0; q < N; ++q)
                    s = fma(P.phi[q * N + i], in[q], s);
                  o1[i] = s;
                }
#pragma unroll
              for (int i = 0; i < N; ++i)
                g0[i * N] = o1[i];
            }
        }
      __syncthreads();
      // x: y = phi_x^T VK + dphi_x^T G0, scattered straight from registers
      if (active)
        {
          const int base = (tB * N + tA) * N;
          const int Y = cy * p + tA, Z = cz * p + tB;
          const bool yzb = Y == 0 || Z == P.zlo || Y == gy - 1 || Z == P.zhi;
#pragma unroll
          for (int c = 0; c < 3; ++c)
            {
              double in[N], in2[N];
              const double *vk = fld(c) + base, *g0 = fld(3 + 3 * c) + base;
#pragma unroll
              for (int m = 0; m < N; ++m)
                {
                  in[m] = vk[m];
                  in2[m] = g0[m];
                }
              double *yv = y + n * isz + a * mv + c * nsc + (static_cast<long long>(Z) * gy + Y) * gx + cx * p;
#pragma unroll
              for (int i = 0; i < N; ++i)
                {
                  double s = 0.0;
#pragma unroll
                  for (int q = 0; q < N; ++q)
                    {
                      s = fma(P.phi[q * N + i], in[q], s);
                      s = fma(P.dphi[q * N + i], in2[q], s);
                    }
                  const int X = cx * p + i;
                  const bool bnd = MODE != 2 && (yzb || X == 0 || X == gx - 1);
                  if (!bnd)
                    atomicAdd(yv + i, MODE == 1 ? -s : s);
                }
            }
        }
    }
}


// ---------------------------------------------------------------------------
// Cartesian r = 1 (C3): every cell has the same spatial element operator, so
// one output slot of one cell is a dense product
//   [y_v ; y_p] (85) = E (85 x 166) [UK ; UM ; PM]  (UK, UM: 81 nodal values,
//   PM: 4 modes, temporally combined as in vmult3_kernel).
// Batched over all (cell, slot) columns it is a GEMM with a shared A = E.
// vmult3_gemm_kernel keeps E in shared memory (88 x 168 padded, loaded once by
// a persistent block), gathers 32 columns at a time and runs the product on
// the FP64 tensor path (mma.m8n8k4); the velocity rows are scattered with
// red.global.add from the accumulators, the cell-owned pressure rows stored.
// This trades ~2x more flops than sum factorisation for DMMA issue density.
// Measured on C3 (B200): 9.95 ms against 8.91 ms for the line kernel; ncu:
// DMMA pipe 36% active, stalls on the accumulator chains (wait), the gather
// (long scoreboard) and the tile barriers. Opt-in (STMG_V3_GEMM=1) until the
// gather overlaps the MMA (double-buffered B, more columns per warp).
constexpr int kGK = 168, kGBP = 36, kGCols = 32, kGThreads = 352; // 11 warps = 11 row tiles

__device__ __forceinline__ void
dmma3(double (&d)[2], double a, double b)
{
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

#ifndef STMG_GEMM_MINB
#define STMG_GEMM_MINB 2
#endif
template <int S, int MODE>
__global__ void __launch_bounds__(kGThreads, STMG_GEMM_MINB)
vmult3_gemm_kernel(const Level3Consts P, const double *__restrict__ E, const double *__restrict__ x,
                   const double *__restrict__ b, double *__restrict__ y, const double *__restrict__ xprev0,
                   int coupled, long long n_cols)
{
  extern __shared__ __align__(16) double gsm[];
  double *Bs = gsm;                        // kGK x kGBP
  long long *cbase = reinterpret_cast<long long *>(Bs + kGK * kGBP); // [kGCols] node base of the column's cell
  long long *cpre = cbase + kGCols;        // [kGCols] pressure base (interval + cell)
  long long *cx_ = cpre + kGCols;          // [kGCols] x of the interval base
  int *cflag = reinterpret_cast<int *>(cx_ + kGCols); // [kGCols] boundary bits | slot << 8 | valid << 16
  int *roff = cflag + kGCols;              // [27] local node offset per velocity node
  double *ck = reinterpret_cast<double *>(roff + 32); // [kGCols][S] K_t(a, b) of the column's slot a
  double *cm = ck + kGCols * S;                       // [kGCols][S] M_t(a, b)
  double *clv = cm + kGCols * S;                      // [kGCols] lv(a)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long nsc = P.nsc, mv = P.mv, mp = P.mp, isz = P.isz;
  const int gx = P.gx, gy = P.gy;
  // warp w owns row tile w of E: its A-fragments stay in registers
  double afr[kGK / 4];
#pragma unroll
  for (int kk = 0; kk < kGK / 4; ++kk)
    afr[kk] = __ldg(E + (8 * warp + (lane >> 2)) * kGK + 4 * kk + (lane & 3));
  for (int i = tid; i < 27; i += kGThreads)
    roff[i] = ((i / 9) * gy + (i / 3) % 3) * gx + i % 3;
  const long long ncells = static_cast<long long>(P.nx) * P.ny * P.nz;
  const long long ntiles = (n_cols + kGCols - 1) / kGCols;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
    {
      if (tid < kGCols)
        {
          const long long j = tile * kGCols + tid;
          int flag = 0;
          long long nb = 0, pb = 0, xb = 0;
          if (j < n_cols)
            {
              const long long cg = j / S;
              const int a = static_cast<int>(j - cg * S);
              const long long n = cg / ncells, cell = cg - n * ncells;
              const int cx = static_cast<int>(cell % P.nx), cy = static_cast<int>((cell / P.nx) % P.ny),
                        cz = static_cast<int>(cell / (static_cast<long long>(P.nx) * P.ny));
              nb = (static_cast<long long>(2 * cz) * gy + 2 * cy) * gx + 2 * cx;
              pb = n * isz + S * mv + cell * 4;
              xb = n * isz;
              flag = (cx == 0) | ((cx == P.nx - 1) << 1) | ((cy == 0) << 2) | ((cy == P.ny - 1) << 3) |
                     ((cz == 0) << 4) | ((cz == P.nz - 1) << 5) | (a << 8) | (1 << 16) | (n > 0 ? (1 << 17) : 0);
            }
          cbase[tid] = nb;
          cpre[tid] = pb;
          cx_[tid] = xb;
          cflag[tid] = flag;
          const int a = (flag >> 8) & 0xff;
#pragma unroll
          for (int bs = 0; bs < S; ++bs)
            {
              ck[tid * S + bs] = P.Kt[a * S + bs];
              cm[tid * S + bs] = P.Mt[a * S + bs];
            }
          clv[tid] = P.lv[a];
        }
      __syncthreads();
      // ---- gather B (kGK x 32): UK (81), UM (81), PM (4), zero padding
      for (int e = tid; e < kGK * kGCols; e += kGThreads)
        {
          const int kr = e / kGCols, c = e - kr * kGCols;
          const int flag = cflag[c];
          double v = 0.0;
          if ((flag >> 16) & 1 && kr < 166)
            {
              const long long xb = cx_[c];
              if (kr < 162)
                {
                  const int q = kr < 81 ? kr : kr - 81;
                  const int comp = q / 27, i = q - comp * 27;
                  const int lx = i % 3, ly = (i / 3) % 3, lz = i / 9;
                  const bool bnd = MODE != 2 && (((flag & 1) && lx == 0) || ((flag & 2) && lx == 2) ||
                                                 ((flag & 4) && ly == 0) || ((flag & 8) && ly == 2) ||
                                                 ((flag & 16) && lz == 0) || ((flag & 32) && lz == 2));
                  const long long node = cbase[c] + roff[i] + comp * nsc;
                  if (kr < 81)
                    {
                      if (!bnd)
#pragma unroll
                        for (int bs = 0; bs < S; ++bs)
                          v = fma(ck[c * S + bs], __ldg(x + xb + bs * mv + node), v);
                      if (coupled)
                        {
                          const double *vp = (flag >> 17) & 1 ? x + xb - isz + (S - 1) * mv : xprev0;
                          if (vp != nullptr)
                            v = fma(-clv[c], __ldg(vp + node), v);
                        }
                    }
                  else if (!bnd)
#pragma unroll
                    for (int bs = 0; bs < S; ++bs)
                      v = fma(cm[c * S + bs], __ldg(x + xb + bs * mv + node), v);
                }
              else
                {
                  const int l = kr - 162;
#pragma unroll
                  for (int bs = 0; bs < S; ++bs)
                    v = fma(cm[c * S + bs], __ldg(x + cpre[c] + bs * mp + l), v);
                }
            }
          Bs[kr * kGBP + c] = v;
        }
      __syncthreads();
      // ---- DMMA: warp w = row tile w, all 4 column tiles
      {
        double acc[4][2];
#pragma unroll
        for (int ct = 0; ct < 4; ++ct)
          acc[ct][0] = acc[ct][1] = 0.0;
        const double *bp = Bs + (lane & 3) * kGBP + (lane >> 2);
#pragma unroll
        for (int kk = 0; kk < kGK / 4; ++kk)
#pragma unroll
          for (int ct = 0; ct < 4; ++ct)
            dmma3(acc[ct], afr[kk], bp[4 * kk * kGBP + 8 * ct]);
        const int row = 8 * warp + (lane >> 2);
#pragma unroll
        for (int ct = 0; ct < 4; ++ct)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            {
              const int c = 8 * ct + 2 * (lane & 3) + h;
              const int flag = cflag[c];
              if (!((flag >> 16) & 1) || row >= 85)
                continue;
              const double val = acc[ct][h];
              const int a = (flag >> 8) & 0xff;
              if (row < 81)
                {
                  const int comp = row / 27, i = row - comp * 27;
                  const int lx = i % 3, ly = (i / 3) % 3, lz = i / 9;
                  const bool bnd = MODE != 2 && (((flag & 1) && lx == 0) || ((flag & 2) && lx == 2) ||
                                                 ((flag & 4) && ly == 0) || ((flag & 8) && ly == 2) ||
                                                 ((flag & 16) && lz == 0) || ((flag & 32) && lz == 2));
                  if (!bnd)
                    atomicAdd(y + cx_[c] + a * mv + comp * nsc + cbase[c] + roff[i], MODE == 1 ? -val : val);
                }
              else
                {
                  const long long o = cpre[c] + a * mp + (row - 81);
                  y[o] = MODE == 1 ? __ldg(b + o) - val : val;
                }
            }
      }
      __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Cartesian r = 1 (C3), 1D-factor form: on congruent rectangular cells every
// term of the spatial Stokes operator is a tensor product of exact 1D node
// matrices (M1, K1, C1 and the Legendre moments Lm, Lc), as in the 2D
// kernel, so no Gauss points are visited:
//   y_c = J M(x)M(x)M UK_c + sum_e nu_e s_e K_e (x) M (x) M UM_c
//         + gamma sum_{d != c} (2/h_c)(2/h_d) J  Ct_c (x) C_d (x) M  UM_d - B_c^T PM,
//   y_p = sum_c B_c UM_c.
// Three phases (x, y, z lines, 2 barriers per slot): the x pass forms the
// 12 x-contracted fields, the y pass combines them into 3 groups per output
// component by their z factor (M, K, C or C^T), the z pass finishes and
// scatters from registers. ~40% fewer line passes and no point fluxes.
#ifndef STMG_V3C_MINB
#define STMG_V3C_MINB 4
#endif
// Thread map: cell-minor (thread = t * 16 + cell), so a half-warp holds the
// same line t of 16 cells. With an odd cell stride its 64-bit shared-memory
// accesses hit 16 distinct bank pairs in every phase (conflict-free), and
// its global loads / scatters walk 16 neighbouring cells along x. The
// cell-major map (thread = cell * 9 + t, STMG_V3C_CELLMINOR=0) spans 3.5
// cells per warp; padding its slot from 365 to 379 doubles (= 11 mod 16)
// takes a bank model of the three line patterns from 2268 to 1944
// wavefronts per block slot (ideal 1134).
#ifndef STMG_V3C_CB
#define STMG_V3C_CB 16 // cells per block (9 threads each); 12 or 14 cells with 6 / 5 blocks per SM spill
#endif
#ifndef STMG_V3C_CELLMINOR
#define STMG_V3C_CELLMINOR 1
#endif
#ifndef STMG_V3C_CELL
#if STMG_V3C_CELLMINOR
#define STMG_V3C_CELL 365 // 12 x 27 x-fields + 36 pressure partials + 4 PM, made odd
#else
#define STMG_V3C_CELL 379
#endif
#endif
template <int S, int MODE>
__global__ void __launch_bounds__(9 * STMG_V3C_CB, STMG_V3C_MINB)
vmult3c_kernel(const Level3Consts P, const double *__restrict__ x, const double *__restrict__ b,
               double *__restrict__ y, const double *__restrict__ xprev0, int coupled, long long n_cells_total)
{
  constexpr int N = 3, NN = 9, NNN = 27, p = 2, NP = 4, CB = STMG_V3C_CB;
  constexpr int CELL = STMG_V3C_CELL; // the y groups overwrite x fields 0..8 in place
  static_assert(CELL >= 12 * NNN + NP * NN + NP, "cell slot too small");
  extern __shared__ __align__(16) double smc[];
  double *const tab = smc + CB * CELL; // lm[2][3], lc[2][3]
  if (threadIdx.x < 6)
    {
      tab[threadIdx.x] = P.lm[threadIdx.x];
      tab[6 + threadIdx.x] = P.lc[threadIdx.x];
    }
#if STMG_V3C_CELLMINOR
  const int t = threadIdx.x / CB, cl = threadIdx.x % CB;
#else
  const int t = threadIdx.x % NN, cl = threadIdx.x / NN;
#endif
  const long long gc = static_cast<long long>(blockIdx.x) * CB + cl;
  const bool active = gc < n_cells_total;
  const long long ncells = static_cast<long long>(P.nx) * P.ny * P.nz;
  const int n = active ? static_cast<int>(gc / ncells) : 0;
  const long long cell = active ? gc - n * ncells : 0;
  const int cx = static_cast<int>(cell % P.nx), cy = static_cast<int>((cell / P.nx) % P.ny),
            cz = static_cast<int>(cell / (static_cast<long long>(P.nx) * P.ny));
  double *const XF = smc + cl * CELL; // 12 fields
  double *const YF = XF;             // 9 fields, written in place over the y-line of XF
  double *const PP = XF + 12 * NNN;  // [NP][NN] pressure-row partials
  double *const PM = PP + NP * NN;
  const int tA = t % N, tB = t / N;
  const long long isz = P.isz, mv = P.mv, mp = P.mp, nsc = P.nsc;
  const int gx = P.gx, gy = P.gy;
  const double *__restrict__ xn = x + n * isz;
  const double *__restrict__ vprev = nullptr;
  if (coupled)
    vprev = n > 0 ? x + (n - 1) * isz + (S - 1) * mv : xprev0;
  const double ix2[3] = {2.0 / P.hx, 2.0 / P.hy, 2.0 / P.hz};
  const double Jm = 0.125 * P.hx * P.hy * P.hz;
  double se[3];
#pragma unroll
  for (int e = 0; e < 3; ++e)
    se[e] = ix2[e] * ix2[e] * Jm;
  const double nu = P.nu, ga = P.gamma;
  auto lmv = [&](int a, int i) { return tab[a * N + i]; };
  auto lcv = [&](int a, int i) { return tab[6 + a * N + i]; };
  // mode exponents of P_1^disc (pdisc.cpp:41-55): (0,0,0), (1,0,0), (0,1,0), (0,0,1)
  auto ex = [](int m, int d) { return (m > 0 && m - 1 == d) ? 1 : 0; };
  __syncthreads();

  for (int a = 0; a < S; ++a)
    {
      double kt[S], mt[S], lva = 0.0;
#pragma unroll
      for (int aa = 0; aa < S; ++aa)
        if (a == aa)
          {
#pragma unroll
            for (int bs = 0; bs < S; ++bs)
              {
                kt[bs] = P.Kt[aa * S + bs];
                mt[bs] = P.Mt[aa * S + bs];
              }
            lva = P.lv[aa];
          }
      // ---- x phase (j = tA, k = tB)
      if (active)
        {
          const int Y = cy * p + tA, Z = cz * p + tB;
          const bool yzb = MODE != 2 && (Y == 0 || Z == P.zlo || Y == gy - 1 || Z == P.zhi);
          const long long row = (static_cast<long long>(Z) * gy + Y) * gx + cx * p;
          double uk[3][N], um[3][N];
#pragma unroll
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int i = 0; i < N; ++i)
              {
                const int X = cx * p + i;
                const bool bnd = yzb || (MODE != 2 && (X == 0 || X == gx - 1));
                double k_ = 0.0, m_ = 0.0;
                if (!bnd)
#pragma unroll
                  for (int bs = 0; bs < S; ++bs)
                    {
                      const double v = __ldg(xn + bs * mv + c * nsc + row + i);
                      k_ = fma(kt[bs], v, k_);
                      m_ = fma(mt[bs], v, m_);
                    }
                if (vprev != nullptr)
                  k_ = fma(-lva, __ldg(vprev + c * nsc + row + i), k_);
                uk[c][i] = k_;
                um[c][i] = m_;
              }
          const int base = (tB * N + tA) * N;
          // out[o] = sum_i A(o, i) in[i]; C: A(o,i) = C1(o,i); C^T: A(o,i) = C1(i,o)
#pragma unroll
          for (int o = 0; o < N; ++o)
            {
              double f[12];
#pragma unroll
              for (int q = 0; q < 12; ++q)
                f[q] = 0.0;
#pragma unroll
              for (int i = 0; i < N; ++i)
                {
                  const double m = P.m1[o * N + i], k = P.k1[o * N + i], c = P.c1[o * N + i], ct = P.c1[i * N + o];
#pragma unroll
                  for (int cc = 0; cc < 3; ++cc)
                    f[cc] = fma(m, uk[cc][i], f[cc]);
                  f[3] = fma(m, um[0][i], f[3]);
                  f[4] = fma(k, um[0][i], f[4]);
                  f[5] = fma(c, um[0][i], f[5]);
                  f[6] = fma(m, um[1][i], f[6]);
                  f[7] = fma(k, um[1][i], f[7]);
                  f[8] = fma(ct, um[1][i], f[8]);
                  f[9] = fma(m, um[2][i], f[9]);
                  f[10] = fma(k, um[2][i], f[10]);
                  f[11] = fma(ct, um[2][i], f[11]);
                }
#pragma unroll
              for (int q = 0; q < 12; ++q)
                XF[q * NNN + base + o] = f[q];
            }
          // pressure rows: partial sums of y_p(l) = sum_c (2/h_c) J [L^c_x (x) L^c_y (x) L^c_z](l) UM_c over this x-line
#pragma unroll
          for (int l = 0; l < NP; ++l)
            {
              double s = 0.0;
#pragma unroll
              for (int c = 0; c < 3; ++c)
                {
                  double sx = 0.0;
#pragma unroll
                  for (int i = 0; i < N; ++i)
                    sx = fma(c == 0 ? lcv(ex(l, 0), i) : lmv(ex(l, 0), i), um[c][i], sx);
                  const double wy = c == 1 ? lcv(ex(l, 1), tA) : lmv(ex(l, 1), tA);
                  const double wz = c == 2 ? lcv(ex(l, 2), tB) : lmv(ex(l, 2), tB);
                  s = fma(ix2[c] * Jm * wy * wz, sx, s);
                }
              PP[l * NN + t] = s;
            }
          if (t < NP)
            {
              double s = 0.0;
#pragma unroll
              for (int bs = 0; bs < S; ++bs)
                s = fma(mt[bs], __ldg(xn + S * mv + bs * mp + cell * NP + t), s);
              PM[t] = s;
            }
        }
      __syncthreads();
      // ---- y phase (i = tA, k = tB): groups by z factor
      if (active)
        {
          const int base = tB * NN + tA; // + j * N
          double in[12][N];
#pragma unroll
          for (int q = 0; q < 12; ++q)
#pragma unroll
            for (int j = 0; j < N; ++j)
              in[q][j] = XF[q * NNN + base + j * N];
          const double gxy = ga * ix2[0] * ix2[1] * Jm, gxz = ga * ix2[0] * ix2[2] * Jm, gyz = ga * ix2[1] * ix2[2] * Jm;
#pragma unroll
          for (int o = 0; o < N; ++o)
            {
              // only the combinations the three outputs use
              double My[12], Ky3 = 0.0, Ky6 = 0.0, Ky9 = 0.0, Cy6 = 0.0, Cy8 = 0.0, Cty5 = 0.0, Cty9 = 0.0;
#pragma unroll
              for (int q = 0; q < 12; ++q)
                My[q] = 0.0;
#pragma unroll
              for (int j = 0; j < N; ++j)
                {
                  const double m = P.m1[o * N + j], k = P.k1[o * N + j], c = P.c1[o * N + j], ct = P.c1[j * N + o];
#pragma unroll
                  for (int q = 0; q < 12; ++q)
                    if (q != 8)
                      My[q] = fma(m, in[q][j], My[q]);
                  Ky3 = fma(k, in[3][j], Ky3);
                  Ky6 = fma(k, in[6][j], Ky6);
                  Ky9 = fma(k, in[9][j], Ky9);
                  Cy6 = fma(c, in[6][j], Cy6);
                  Cy8 = fma(c, in[8][j], Cy8);
                  Cty5 = fma(ct, in[5][j], Cty5);
                  Cty9 = fma(ct, in[9][j], Cty9);
                }
              const int yo = base + o * N;
              // output x
              YF[0 * NNN + yo] = Jm * My[0] + (nu + ga) * se[0] * My[4] + nu * se[1] * Ky3 + gxy * Cy8;
              YF[1 * NNN + yo] = nu * se[2] * My[3];
              YF[2 * NNN + yo] = gxz * My[11];
              // output y
              YF[3 * NNN + yo] = Jm * My[1] + nu * se[0] * My[7] + (nu + ga) * se[1] * Ky6 + gxy * Cty5;
              YF[4 * NNN + yo] = nu * se[2] * My[6];
              YF[5 * NNN + yo] = gyz * Cty9;
              // output z
              YF[6 * NNN + yo] = Jm * My[2] + nu * se[0] * My[10] + nu * se[1] * Ky9;
              YF[7 * NNN + yo] = (nu + ga) * se[2] * My[9];
              YF[8 * NNN + yo] = gxz * My[5] + gyz * Cy6;
            }
          if (t < NP)
            {
              double s = 0.0;
#pragma unroll
              for (int q = 0; q < NN; ++q)
                s += PP[t * NN + q];
              const long long o = n * isz + S * mv + a * mp + cell * NP + t;
              y[o] = MODE == 1 ? __ldg(b + o) - s : s;
            }
        }
      __syncthreads();
      // ---- z phase (i = tA, j = tB): finish, subtract B^T PM, scatter
      if (active)
        {
          const int base = tB * N + tA; // + k * NN
          const int X = cx * p + tA, Y = cy * p + tB;
          const bool xyb = X == 0 || Y == 0 || X == gx - 1 || Y == gy - 1;
#pragma unroll
          for (int c = 0; c < 3; ++c)
            {
              double gm[N], gk[N], g3[N];
#pragma unroll
              for (int k = 0; k < N; ++k)
                {
                  gm[k] = YF[(3 * c) * NNN + base + k * NN];
                  gk[k] = YF[(3 * c + 1) * NNN + base + k * NN];
                  g3[k] = YF[(3 * c + 2) * NNN + base + k * NN];
                }
              double *yv = y + n * isz + a * mv + c * nsc + static_cast<long long>(Y) * gx + X;
#pragma unroll
              for (int o = 0; o < N; ++o)
                {
                  double s = 0.0;
#pragma unroll
                  for (int k = 0; k < N; ++k)
                    {
                      s = fma(P.m1[o * N + k], gm[k], s);
                      s = fma(P.k1[o * N + k], gk[k], s);
                      // z factor of group 3: C (trial derivative in z) for outputs x, y; C^T for output z
                      s = fma(c == 2 ? P.c1[k * N + o] : P.c1[o * N + k], g3[k], s);
                    }
                  // - B_c^T PM: sum_l PM_l (2/h_c) J [L^c_x (x) L^c_y (x) L^c_z](l; tA, tB, o)
#pragma unroll
                  for (int l = 0; l < NP; ++l)
                    {
                      const double wx = c == 0 ? lcv(ex(l, 0), tA) : lmv(ex(l, 0), tA);
                      const double wy = c == 1 ? lcv(ex(l, 1), tB) : lmv(ex(l, 1), tB);
                      const double wz = c == 2 ? lcv(ex(l, 2), o) : lmv(ex(l, 2), o);
                      s = fma(-ix2[c] * Jm * wx * wy * wz, PM[l], s);
                    }
                  const int Z = cz * p + o;
                  const bool bnd = MODE != 2 && (xyb || Z == P.zlo || Z == P.zhi);
                  if (!bnd)
                    atomicAdd(yv + static_cast<long long>(Z) * gy * gx, MODE == 1 ? -s : s);
                }
            }
        }
      __syncthreads(); // the next slot's x phase overwrites the groups the z phase reads
    }
}
/// y's velocity rows before the scatter: 0 (plain / raw), b (residual); the
/// constrained rows get the identity x (plain) or b - x (residual),
/// st_operator.cpp:383-394.
template <int MODE>
__global__ void __launch_bounds__(128)
vmult3_init_kernel(DevGeom3 G, const double *__restrict__ x, const double *__restrict__ b, double *__restrict__ y,
                   long long total)
{
  // grid: (X*Y blocks, Z, interval * slot * component); 32-bit index math
  const int xy = blockIdx.x * 128 + threadIdx.x;
  if (xy >= G.gx * G.gy)
    return;
  const int X = xy % G.gx, Y = xy / G.gx, Z = blockIdx.y;
  const int q = blockIdx.z, comp = q % 3, a = (q / 3) % G.S, n = q / (3 * G.S);
  const long long o = n * G.isz + a * G.mv + comp * G.nsc + (static_cast<long long>(Z) * G.gy + Y) * G.gx + X;
  const bool bnd = X == 0 || Y == 0 || Z == G.zlo || X == G.gx - 1 || Y == G.gy - 1 || Z == G.zhi;
  double v = 0.0;
  if (MODE != 2 && bnd)
    v = x[o];
  if (MODE == 1)
    v = __ldg(b + o) - v;
  y[o] = v;
  (void)total;
}

template <int R, int S>
cudaError_t
launch_rs3_chunk(const Level3Consts &P, const double *x, const double *b, double *y, int nI, const double *xprev0,
                 int coupled, int mode, cudaStream_t st)
{
  DevGeom3 G{};
  G.nx = P.nx;
  G.ny = P.ny;
  G.nz = P.nz;
  G.gx = P.gx;
  G.gy = P.gy;
  G.gz = P.gz;
  G.zlo = P.zlo;
  G.zhi = P.zhi;
  G.S = S;
  G.np = P.np;
  G.nsc = P.nsc;
  G.mv = P.mv;
  G.mp = P.mp;
  G.isz = P.isz;
  const long long total_v = static_cast<long long>(nI) * S * P.mv;
  const dim3 igrid((P.gx * P.gy + 127) / 128, P.gz, nI * S * 3);
  const long long cells = static_cast<long long>(nI) * P.nx * P.ny * P.nz;
  auto go = [&](auto init, auto kern, dim3 block, unsigned grid, size_t smem) {
    init<<<igrid, 128, 0, st>>>(G, x, b, y, total_v);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kern<<<grid, block, smem, st>>>(P, x, b, y, xprev0, coupled, cells);
  };
  if constexpr (R == 1)
    if (P.gemmE != nullptr && std::getenv("STMG_V3_GEMM") != nullptr) // opt-in: measured slower
      {
        const long long ncols = cells * S;
        const size_t smem = sizeof(double) * (kGK * kGBP) + sizeof(long long) * 3 * kGCols +
                            sizeof(int) * (kGCols + 32) + sizeof(double) * (2 * S + 1) * kGCols;
        const unsigned grid = static_cast<unsigned>(std::min<long long>(2 * device_sm_count(), (ncols + kGCols - 1) / kGCols));
        auto gg = [&](auto init, auto kern) {
          init<<<igrid, 128, 0, st>>>(G, x, b, y, total_v);
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
          kern<<<grid, kGThreads, smem, st>>>(P, P.gemmE, x, b, y, xprev0, coupled, ncols);
        };
        switch (mode)
          {
            case 0: gg(vmult3_init_kernel<0>, vmult3_gemm_kernel<S, 0>); break;
            case 1: gg(vmult3_init_kernel<1>, vmult3_gemm_kernel<S, 1>); break;
            default: gg(vmult3_init_kernel<2>, vmult3_gemm_kernel<S, 2>); break;
          }
        return cudaGetLastError();
      }
  if constexpr (R == 1)
    if (P.verts == nullptr && std::getenv("STMG_V3_QUAD") == nullptr)
      {
        constexpr int CB = STMG_V3C_CB;
        const size_t smem = sizeof(double) * (CB * STMG_V3C_CELL + 12);
        const unsigned grid = static_cast<unsigned>((cells + CB - 1) / CB);
        auto gc = [&](auto init, auto kern) {
          init<<<igrid, 128, 0, st>>>(G, x, b, y, total_v);
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
          kern<<<grid, 9 * CB, smem, st>>>(P, x, b, y, xprev0, coupled, cells);
        };
        switch (mode)
          {
            case 0: gc(vmult3_init_kernel<0>, vmult3c_kernel<S, 0>); break;
            case 1: gc(vmult3_init_kernel<1>, vmult3c_kernel<S, 1>); break;
            default: gc(vmult3_init_kernel<2>, vmult3c_kernel<S, 2>); break;
          }
        return cudaGetLastError();
      }
  if constexpr (R == 1)
    if (std::getenv("STMG_V3_LINE") == nullptr)
      {
        // fused in-place pipeline (4 barriers per slot), N*N threads per cell
        using C = V3<R, 1, false>;
        using CD = V3<R, 1, true>;
        const dim3 block(C::THREADS);
        const unsigned grid = static_cast<unsigned>((cells + C::CW - 1) / C::CW);
        const bool def = P.verts != nullptr;
        if (def && std::getenv("STMG_V3_R1_DEF_OLD") == nullptr)
          { // the r >= 2 deformed kernel (no J^-1 cache, thread-local z-lines) also on deformed r = 1 levels,
            // three blocks per SM: 32^3 x 16 intervals, DG(2): residual 3.00 -> 2.39 ms
            using D = V3D<R>;
            const unsigned gridd = static_cast<unsigned>((cells + D::CW - 1) / D::CW);
            switch (mode)
              {
                case 0: go(vmult3_init_kernel<0>, vmult3d_kernel<R, S, 0>, dim3(D::THREADS), gridd, D::smem()); break;
                case 1: go(vmult3_init_kernel<1>, vmult3d_kernel<R, S, 1>, dim3(D::THREADS), gridd, D::smem()); break;
                default: go(vmult3_init_kernel<2>, vmult3d_kernel<R, S, 2>, dim3(D::THREADS), gridd, D::smem()); break;
              }
            return cudaGetLastError();
          }
        switch (mode)
          {
            case 0:
              def ? go(vmult3_init_kernel<0>, vmult3_kernel<R, S, 0, 1, true>, block, grid, CD::smem())
                  : go(vmult3_init_kernel<0>, vmult3_kernel<R, S, 0, 1, false>, block, grid, C::smem());
              break;
            case 1:
              def ? go(vmult3_init_kernel<1>, vmult3_kernel<R, S, 1, 1, true>, block, grid, CD::smem())
                  : go(vmult3_init_kernel<1>, vmult3_kernel<R, S, 1, 1, false>, block, grid, C::smem());
              break;
            default:
              def ? go(vmult3_init_kernel<2>, vmult3_kernel<R, S, 2, 1, true>, block, grid, CD::smem())
                  : go(vmult3_init_kernel<2>, vmult3_kernel<R, S, 2, 1, false>, block, grid, C::smem());
              break;
          }
        return cudaGetLastError();
      }
  if constexpr (R == 1)
    {
      using C = V3L<R>;
      const dim3 block(C::NN, C::CB);
      const unsigned grid = static_cast<unsigned>((cells + C::CB - 1) / C::CB);
      switch (mode)
        {
          case 0: go(vmult3_init_kernel<0>, vmult3l_kernel<R, S, 0>, block, grid, C::smem()); break;
          case 1: go(vmult3_init_kernel<1>, vmult3l_kernel<R, S, 1>, block, grid, C::smem()); break;
          default: go(vmult3_init_kernel<2>, vmult3l_kernel<R, S, 2>, block, grid, C::smem()); break;
        }
    }
  else
    {
      using C = V3<R, 0, false>;
      using CD = V3<R, 0, true>;
      const dim3 block(C::THREADS);
      const unsigned grid = static_cast<unsigned>((cells + C::CW - 1) / C::CW);
      const bool def = P.verts != nullptr;
      if (def && std::getenv("STMG_V3_DEF_OLD") == nullptr)
        {
          using D = V3D<R>;
          const unsigned gridd = static_cast<unsigned>((cells + D::CW - 1) / D::CW);
          switch (mode)
            {
              case 0: go(vmult3_init_kernel<0>, vmult3d_kernel<R, S, 0>, dim3(D::THREADS), gridd, D::smem()); break;
              case 1: go(vmult3_init_kernel<1>, vmult3d_kernel<R, S, 1>, dim3(D::THREADS), gridd, D::smem()); break;
              default: go(vmult3_init_kernel<2>, vmult3d_kernel<R, S, 2>, dim3(D::THREADS), gridd, D::smem()); break;
            }
          return cudaGetLastError();
        }
      switch (mode)
        {
          case 0:
            def ? go(vmult3_init_kernel<0>, vmult3_kernel<R, S, 0, 0, true>, block, grid, CD::smem())
                : go(vmult3_init_kernel<0>, vmult3_kernel<R, S, 0, 0, false>, block, grid, C::smem());
            break;
          case 1:
            def ? go(vmult3_init_kernel<1>, vmult3_kernel<R, S, 1, 0, true>, block, grid, CD::smem())
                : go(vmult3_init_kernel<1>, vmult3_kernel<R, S, 1, 0, false>, block, grid, C::smem());
            break;
          default:
            def ? go(vmult3_init_kernel<2>, vmult3_kernel<R, S, 2, 0, true>, block, grid, CD::smem())
                : go(vmult3_init_kernel<2>, vmult3_kernel<R, S, 2, 0, false>, block, grid, C::smem());
            break;
        }
    }
  return cudaGetLastError();
}

/// Intervals per init + scatter pass: the velocity rows the pass's red.adds
/// hit stay L2-resident between the init kernel and the cell kernel (on
/// C5's fine level one interval is 66 MB), so y is written to DRAM once
/// instead of written, re-read and re-written.
int
vmult3_chunk(const Level3Consts &P, int S)
{
  const long long bytes = static_cast<long long>(S) * P.mv * sizeof(double);
  return static_cast<int>(std::max<long long>(1, (64ll << 20) / std::max<long long>(1, bytes)));
}

template <int R, int S>
cudaError_t
launch_rs3(const Level3Consts &P, const double *x, const double *b, double *y, int nI, const double *xprev0,
           int coupled, int mode, cudaStream_t st)
{
  const int chunk = vmult3_chunk(P, S);
  for (int c0 = 0; c0 < nI; c0 += chunk)
    {
      const int nc = std::min(chunk, nI - c0);
      const long long off = static_cast<long long>(c0) * P.isz;
      const double *xp = c0 == 0 ? xprev0 : x + off - P.isz + (S - 1) * P.mv;
      const cudaError_t e =
        launch_rs3_chunk<R, S>(P, x + off, b ? b + off : nullptr, y + off, nc, xp, coupled, mode, st);
      if (e != cudaSuccess)
        return e;
    }
  return cudaSuccess;
}

// ---------------------------------------------------------------- aux
__global__ void __launch_bounds__(128)
zero_constrained3_kernel(DevGeom3 G, double *__restrict__ x)
{
  // grid: (X*Y blocks, Z, interval * slot * component); only boundary nodes are written
  const int xy = blockIdx.x * 128 + threadIdx.x;
  if (xy >= G.gx * G.gy)
    return;
  const int X = xy % G.gx, Y = xy / G.gx, Z = blockIdx.y;
  if (!(X == 0 || Y == 0 || Z == G.zlo || X == G.gx - 1 || Y == G.gy - 1 || Z == G.zhi))
    return;
  const int q = blockIdx.z, comp = q % 3, a = (q / 3) % G.S, n = q / (3 * G.S);
  x[n * G.isz + a * G.mv + comp * G.nsc + (static_cast<long long>(Z) * G.gy + Y) * G.gx + X] = 0.0;
}

constexpr int kProjThreads = 512;
__global__ void __launch_bounds__(kProjThreads)
project3_kernel(DevGeom3 G, const double *__restrict__ pmean, double inv_vol, double *__restrict__ x)
{
  __shared__ double red[kProjThreads];
  const int n = blockIdx.y, a = blockIdx.x;
  double *pr = x + n * G.isz + G.S * G.mv + a * G.mp;
  double s = 0.0;
  for (long long i = threadIdx.x; i < G.mp; i += kProjThreads)
    s = fma(pmean[i], pr[i], s);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = kProjThreads / 2; w > 0; w >>= 1)
    {
      if (threadIdx.x < w)
        red[threadIdx.x] += red[threadIdx.x + w];
      __syncthreads();
    }
  const double mean = red[0] * inv_vol;
  const long long ncell = G.mp / G.np;
  for (long long c = threadIdx.x; c < ncell; c += kProjThreads)
    pr[c * G.np] -= mean;
}

// Transfers: velocity rows on a (X-block, Y*Z, interval*slot*component)
// grid and pressure rows on a (cell-mode block, interval*slot) grid, so the
// index math is 32-bit and per block instead of 64-bit divisions per element.
constexpr int kTrX = 64;

__global__ void __launch_bounds__(kTrX)
prolongate3_vel_kernel(DevTransfer3 T, const double *__restrict__ coarse, double *__restrict__ fine)
{
  const DevGeom3 &F = T.f, &Cg = T.c;
  const int X = blockIdx.x * kTrX + threadIdx.x;
  if (X >= F.gx)
    return;
  const int Y = blockIdx.y % F.gy, Z = blockIdx.y / F.gy;
  const int q = blockIdx.z; // (n * S_f + a) * 3 + comp
  const int comp = q % 3, a = (q / 3) % F.S, n = q / (3 * F.S);
  const int m = T.h_time ? n / 2 : n, half = T.h_time ? (n & 1) : 0;
  const double *E = T.E + half * kMaxS * kMaxS + a * kMaxS;
  const long long s = (static_cast<long long>(Z) * F.gy + Y) * F.gx + X;
  double v = 0.0;
  for (int bs = 0; bs < Cg.S; ++bs)
    {
      const double *cv = coarse + m * Cg.isz + bs * Cg.mv + comp * Cg.nsc;
      double sv;
      if (T.spatial)
        {
          sv = 0.0;
          for (int kz = T.pz.ptr[Z]; kz < T.pz.ptr[Z + 1]; ++kz)
            for (int ky = T.py.ptr[Y]; ky < T.py.ptr[Y + 1]; ++ky)
              {
                const double wyz = T.pz.val[kz] * T.py.val[ky];
                const double *row = cv + (static_cast<long long>(T.pz.col[kz]) * Cg.gy + T.py.col[ky]) * Cg.gx;
                for (int kx = T.px.ptr[X]; kx < T.px.ptr[X + 1]; ++kx)
                  sv = fma(wyz * T.px.val[kx], __ldg(row + T.px.col[kx]), sv);
              }
        }
      else
        sv = __ldg(cv + s);
      v = fma(E[bs], sv, v);
    }
  fine[n * F.isz + a * F.mv + comp * F.nsc + s] = v;
}

__global__ void
prolongate3_pre_kernel(DevTransfer3 T, const double *__restrict__ coarse, double *__restrict__ fine)
{
  const DevGeom3 &F = T.f, &Cg = T.c;
  const int e = blockIdx.x * blockDim.x + threadIdx.x; // cell * np + mode
  const int ncm = F.nx * F.ny * F.nz * F.np;
  if (e >= ncm)
    return;
  const int q = blockIdx.y; // n * S_f + a
  const int a = q % F.S, n = q / F.S;
  const int m = T.h_time ? n / 2 : n, half = T.h_time ? (n & 1) : 0;
  const double *E = T.E + half * kMaxS * kMaxS + a * kMaxS;
  const int cell = e / F.np, mf = e - cell * F.np;
  int ccell = cell, ch = 0;
  if (T.pmode == 1)
    {
      const int fx = cell % F.nx, fy = (cell / F.nx) % F.ny, fz = cell / (F.nx * F.ny);
      ch = (fz & 1) * 4 + (fy & 1) * 2 + (fx & 1);
      ccell = ((fz >> 1) * Cg.ny + (fy >> 1)) * Cg.nx + (fx >> 1);
    }
  double v = 0.0;
  for (int bs = 0; bs < Cg.S; ++bs)
    {
      const double *cp = coarse + m * Cg.isz + Cg.S * Cg.mv + bs * Cg.mp + static_cast<long long>(ccell) * Cg.np;
      double sv = 0.0;
      if (T.spatial)
        {
          const double *blk = T.child + (ch * F.np + mf) * Cg.np;
          for (int l = 0; l < Cg.np; ++l)
            sv = fma(blk[l], cp[l], sv);
        }
      else
        sv = cp[mf];
      v = fma(E[bs], sv, v);
    }
  fine[n * F.isz + F.S * F.mv + a * F.mp + e] = v;
}

__global__ void __launch_bounds__(kTrX)
restrict3_vel_kernel(DevTransfer3 T, const double *__restrict__ fine, double *__restrict__ coarse)
{
  const DevGeom3 &F = T.f, &Cg = T.c;
  const int X = blockIdx.x * kTrX + threadIdx.x;
  if (X >= Cg.gx)
    return;
  const int Y = blockIdx.y % Cg.gy, Z = blockIdx.y / Cg.gy;
  const int q = blockIdx.z; // (m * S_c + b) * 3 + comp
  const int comp = q % 3, bs = (q / 3) % Cg.S, m = q / (3 * Cg.S);
  const long long s = (static_cast<long long>(Z) * Cg.gy + Y) * Cg.gx + X;
  const int nh = T.h_time ? 2 : 1;
  double v = 0.0;
  for (int h = 0; h < nh; ++h)
    {
      const int n = T.h_time ? 2 * m + h : m;
      const double *E = T.E + h * kMaxS * kMaxS;
      for (int a = 0; a < F.S; ++a)
        {
          const double *fv = fine + n * F.isz + a * F.mv + comp * F.nsc;
          double sv;
          if (T.spatial)
            {
              sv = 0.0;
              for (int kz = T.rz.ptr[Z]; kz < T.rz.ptr[Z + 1]; ++kz)
                for (int ky = T.ry.ptr[Y]; ky < T.ry.ptr[Y + 1]; ++ky)
                  {
                    const double wyz = T.rz.val[kz] * T.ry.val[ky];
                    const double *row = fv + (static_cast<long long>(T.rz.col[kz]) * F.gy + T.ry.col[ky]) * F.gx;
                    for (int kx = T.rx.ptr[X]; kx < T.rx.ptr[X + 1]; ++kx)
                      sv = fma(wyz * T.rx.val[kx], __ldg(row + T.rx.col[kx]), sv);
                  }
            }
          else
            sv = __ldg(fv + s);
          v = fma(E[a * kMaxS + bs], sv, v);
        }
    }
  coarse[m * Cg.isz + bs * Cg.mv + comp * Cg.nsc + s] = v;
}

__global__ void
restrict3_pre_kernel(DevTransfer3 T, const double *__restrict__ fine, double *__restrict__ coarse)
{
  const DevGeom3 &F = T.f, &Cg = T.c;
  const int e = blockIdx.x * blockDim.x + threadIdx.x; // coarse cell * np + mode
  const int ncm = Cg.nx * Cg.ny * Cg.nz * Cg.np;
  if (e >= ncm)
    return;
  const int q = blockIdx.y; // m * S_c + b
  const int bs = q % Cg.S, m = q / Cg.S;
  const int ccell = e / Cg.np, l = e - ccell * Cg.np;
  const int ccx = ccell % Cg.nx, ccy = (ccell / Cg.nx) % Cg.ny, ccz = ccell / (Cg.nx * Cg.ny);
  const int nch = T.pmode == 1 ? 8 : 1, nh = T.h_time ? 2 : 1;
  double v = 0.0;
  for (int h = 0; h < nh; ++h)
    {
      const int n = T.h_time ? 2 * m + h : m;
      const double *E = T.E + h * kMaxS * kMaxS;
      for (int a = 0; a < F.S; ++a)
        {
          double sv = 0.0;
          for (int ch = 0; ch < nch; ++ch)
            {
              int fcell = ccell;
              if (T.pmode == 1)
                fcell = ((2 * ccz + (ch >> 2)) * F.ny + 2 * ccy + ((ch >> 1) & 1)) * F.nx + 2 * ccx + (ch & 1);
              const double *fp = fine + n * F.isz + F.S * F.mv + a * F.mp + static_cast<long long>(fcell) * F.np;
              if (T.spatial)
                {
                  const double *blk = T.child + ch * F.np * Cg.np;
                  for (int mf = 0; mf < F.np; ++mf)
                    sv = fma(blk[mf * Cg.np + l], fp[mf], sv);
                }
              else
                sv += fp[l];
            }
          v = fma(E[a * kMaxS + bs], sv, v);
        }
    }
  coarse[m * Cg.isz + Cg.S * Cg.mv + bs * Cg.mp + e] = v;
}


// Separable spatial transfers: the velocity prolongation / restriction is a
// tensor product of 1D stencils, applied as three 1D passes through two
// scratch arrays instead of one gather over the product stencil (r 2 -> 1:
// up to 7^3 = 343 terms per coarse node against 3 x 7). The temporal E
// matrices (p and h in time) are folded into the x pass.
struct SepDims
{
  int ix, iy, iz, ox, oy, oz;
};

__global__ void __launch_bounds__(kTrX)
sep1d_kernel(DevCsr A, int axis, const double *__restrict__ in, long long ism, long long isb, long long isc,
             double *__restrict__ out, long long osm, long long osb, long long osc, SepDims D, int S)
{
  const int xy = blockIdx.x * kTrX + threadIdx.x;
  if (xy >= D.ox * D.oy)
    return;
  const int X = xy % D.ox, Y = xy / D.ox, Z = blockIdx.y;
  const int q = blockIdx.z, comp = q % 3, b = (q / 3) % S, m = q / (3 * S);
  const double *ib = in + m * ism + b * isb + comp * isc;
  const int r = axis == 0 ? X : (axis == 1 ? Y : Z);
  double s = 0.0;
  for (int e = A.ptr[r]; e < A.ptr[r + 1]; ++e)
    {
      const int c = A.col[e];
      const long long idx = axis == 0 ? (static_cast<long long>(Z) * D.iy + Y) * D.ix + c
                                      : (axis == 1 ? (static_cast<long long>(Z) * D.iy + c) * D.ix + X
                                                   : (static_cast<long long>(c) * D.iy + Y) * D.ix + X);
      s = fma(A.val[e], __ldg(ib + idx), s);
    }
  out[m * osm + b * osb + comp * osc + (static_cast<long long>(Z) * D.oy + Y) * D.ox + X] = s;
}

/// prolongation, last pass: fine[n][a][comp](Z, Y, X) = sum_b E_h(a, b) sum_i px(X, i) T2[(m, b, comp)](Z, Y, i)
__global__ void __launch_bounds__(kTrX)
sep_prolong_x_kernel(DevTransfer3 T, const double *__restrict__ T2, double *__restrict__ fine, int gxc)
{
  const DevGeom3 &F = T.f, &Cg = T.c;
  const int xy = blockIdx.x * kTrX + threadIdx.x;
  if (xy >= F.gx * F.gy)
    return;
  const int X = xy % F.gx, Y = xy / F.gx, Z = blockIdx.y;
  const int q = blockIdx.z, comp = q % 3, a = (q / 3) % F.S, n = q / (3 * F.S);
  const int m = T.h_time ? n / 2 : n, half = T.h_time ? (n & 1) : 0;
  const double *E = T.E + half * kMaxS * kMaxS + a * kMaxS;
  const long long plane = static_cast<long long>(F.gz) * F.gy * gxc;
  const long long row = (static_cast<long long>(Z) * F.gy + Y) * gxc;
  double v = 0.0;
  for (int bs = 0; bs < Cg.S; ++bs)
    {
      const double *t = T2 + ((static_cast<long long>(m) * Cg.S + bs) * 3 + comp) * plane + row;
      double sv = 0.0;
      for (int e = T.px.ptr[X]; e < T.px.ptr[X + 1]; ++e)
        sv = fma(T.px.val[e], __ldg(t + T.px.col[e]), sv);
      v = fma(E[bs], sv, v);
    }
  fine[n * F.isz + a * F.mv + comp * F.nsc + (static_cast<long long>(Z) * F.gy + Y) * F.gx + X] = v;
}

/// restriction, first pass: T1[(m, b, comp)](Zf, Yf, i) = sum_h sum_a E_h(a, b) sum_X rx(i, X) fine[n(m, h)][a][comp](Zf, Yf, X)
__global__ void __launch_bounds__(kTrX)
sep_restrict_x_kernel(DevTransfer3 T, const double *__restrict__ fine, double *__restrict__ T1)
{
  const DevGeom3 &F = T.f, &Cg = T.c;
  const int xy = blockIdx.x * kTrX + threadIdx.x;
  if (xy >= Cg.gx * F.gy)
    return;
  const int i = xy % Cg.gx, Y = xy / Cg.gx, Z = blockIdx.y;
  const int q = blockIdx.z, comp = q % 3, bs = (q / 3) % Cg.S, m = q / (3 * Cg.S);
  const long long row = (static_cast<long long>(Z) * F.gy + Y) * F.gx;
  const int nh = T.h_time ? 2 : 1;
  double v = 0.0;
  for (int h = 0; h < nh; ++h)
    {
      const int n = T.h_time ? 2 * m + h : m;
      const double *E = T.E + h * kMaxS * kMaxS;
      for (int a = 0; a < F.S; ++a)
        {
          const double *f = fine + n * F.isz + a * F.mv + comp * F.nsc + row;
          double sv = 0.0;
          for (int e = T.rx.ptr[i]; e < T.rx.ptr[i + 1]; ++e)
            sv = fma(T.rx.val[e], __ldg(f + T.rx.col[e]), sv);
          v = fma(E[a * kMaxS + bs], sv, v);
        }
    }
  const long long plane = static_cast<long long>(F.gz) * F.gy * Cg.gx;
  T1[((static_cast<long long>(m) * Cg.S + bs) * 3 + comp) * plane + (static_cast<long long>(Z) * F.gy + Y) * Cg.gx + i] =
    v;
}
} // namespace

bool
vmult3_supported(int r, int S)
{
  return r >= 1 && r <= 2 && S >= 1 && S <= 3;
}

int
vmult3_launch_count(const Level3Consts &P, int S, int nI)
{
  const int chunk = vmult3_chunk(P, S);
  return 2 * ((nI + chunk - 1) / chunk);
}

cudaError_t
launch_vmult3(int r, int S, const Level3Consts &P, const double *x, const double *b, double *y, int nI,
              const double *xprev0, int coupled, int mode, cudaStream_t st)
{
  if (nI <= 0)
    return cudaSuccess;
#define STMG_V3(RR, SS)                                                                                              \
  if (r == RR && S == SS)                                                                                            \
    return launch_rs3<RR, SS>(P, x, b, y, nI, xprev0, coupled, mode, st);
  STMG_V3(1, 1)
  STMG_V3(1, 2)
  STMG_V3(1, 3)
  STMG_V3(2, 1)
  STMG_V3(2, 2)
  STMG_V3(2, 3)
#undef STMG_V3
  return cudaErrorInvalidValue;
}

cudaError_t
launch_zero_constrained3(const DevGeom3 &G, double *x, int nI, cudaStream_t st)
{
  const long long total = static_cast<long long>(nI) * G.S * G.mv;
  if (total == 0)
    return cudaSuccess;
  const dim3 grid((G.gx * G.gy + 127) / 128, G.gz, nI * G.S * 3);
  zero_constrained3_kernel<<<grid, 128, 0, st>>>(G, x);
  return cudaGetLastError();
}

cudaError_t
launch_project3(const DevGeom3 &G, const double *pmean, double inv_vol, double *x, int nI, cudaStream_t st)
{
  if (nI == 0)
    return cudaSuccess;
  dim3 grid(G.S, nI);
  project3_kernel<<<grid, kProjThreads, 0, st>>>(G, pmean, inv_vol, x);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- z-split
// Interface planes of a z-split level (stmg3_solver_create_split): the
// velocity nodes of the node plane Z = 0 (side 0) or Z = gz - 1 (side 1), for
// every interval, slot and component, packed as [n][a][c][gx * gy].
namespace
{
__device__ __forceinline__ long long
plane_index(const DevGeom3 &G, int side, long long e)
{
  const long long L = static_cast<long long>(G.gx) * G.gy;
  const long long seg = e / L, off = e - seg * L;
  const long long c = seg % 3, a = (seg / 3) % G.S, n = seg / (3 * G.S);
  return n * G.isz + a * G.mv + c * G.nsc + (side ? static_cast<long long>(G.gz - 1) * L : 0) + off;
}
__device__ __forceinline__ bool
plane_edge(const DevGeom3 &G, long long e)
{
  const long long off = e % (static_cast<long long>(G.gx) * G.gy);
  const int X = static_cast<int>(off % G.gx), Y = static_cast<int>(off / G.gx);
  return X == 0 || Y == 0 || X == G.gx - 1 || Y == G.gy - 1; // Dirichlet rows of the plane
}

__global__ void
plane_op3_kernel(DevGeom3 G, int side, int op, long long n, double *__restrict__ x, double *__restrict__ buf,
                 const double *__restrict__ other, const double *__restrict__ b, const double *__restrict__ saved)
{
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<long long>(gridDim.x) * blockDim.x)
    {
      const long long i = plane_index(G, side, e);
      switch (op)
        {
        case 0: // pack
          buf[e] = x[i];
          break;
        case 1: // owner-accumulate: x += partner's partial sums (plain application)
          if (!plane_edge(G, e))
            x[i] += other[e];
          break;
        case 2: // residual: r = r_own + r_partner - b (both are b - partial; b: full vector)
          if (!plane_edge(G, e))
            x[i] = (x[i] + other[e]) - b[i];
          break;
        case 3: // scale by 1/2 (fine residual before a restriction)
          x[i] *= 0.5;
          break;
        case 4: // Vanka delta of this part: buf = x - saved
          buf[e] = x[i] - saved[e];
          break;
        case 5: // x = saved + (own delta + partner delta): the same sum on both parts
          x[i] = saved[e] + (buf[e] + other[e]);
          break;
        case 6: // unpack
          x[i] = buf[e];
          break;
        }
    }
}

__global__ void __launch_bounds__(kProjThreads)
project3_sums_kernel(DevGeom3 G, const double *__restrict__ pmean, const double *__restrict__ x,
                     double *__restrict__ sums)
{
  __shared__ double red[kProjThreads];
  const int n = blockIdx.y, a = blockIdx.x;
  const double *pr = x + n * G.isz + G.S * G.mv + a * G.mp;
  double s = 0.0;
  for (long long i = threadIdx.x; i < G.mp; i += kProjThreads)
    s = fma(pmean[i], pr[i], s);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = kProjThreads / 2; w > 0; w >>= 1)
    {
      if (threadIdx.x < w)
        red[threadIdx.x] += red[threadIdx.x + w];
      __syncthreads();
    }
  if (threadIdx.x == 0)
    sums[n * G.S + a] = red[0];
}

__global__ void __launch_bounds__(kProjThreads)
project3_apply_kernel(DevGeom3 G, const double *__restrict__ sums, double inv_vol, double *__restrict__ x)
{
  const int n = blockIdx.y, a = blockIdx.x;
  double *pr = x + n * G.isz + G.S * G.mv + a * G.mp;
  const double mean = sums[n * G.S + a] * inv_vol;
  const long long ncell = G.mp / G.np;
  for (long long c = threadIdx.x; c < ncell; c += kProjThreads)
    pr[c * G.np] -= mean;
}

constexpr int kPlaneDotBlocks = 64;
__global__ void __launch_bounds__(256)
plane_multidot_kernel(DevGeom3 G, int side, long long n, MultiVec V, int m, int with_norm, const double *__restrict__ w,
                      double *__restrict__ part)
{
  __shared__ double red[256];
  for (int i = 0; i < m + with_norm; ++i)
    {
      const double *v = i < m ? V.p[i] : w;
      double s = 0.0;
      for (long long e = blockIdx.x * 256ll + threadIdx.x; e < n; e += 256ll * gridDim.x)
        {
          const long long k = plane_index(G, side, e);
          s = fma(v[k], w[k], s);
        }
      red[threadIdx.x] = s;
      __syncthreads();
      for (int h = 128; h > 0; h >>= 1)
        {
          if (threadIdx.x < h)
            red[threadIdx.x] += red[threadIdx.x + h];
          __syncthreads();
        }
      if (threadIdx.x == 0)
        part[i * kPlaneDotBlocks + blockIdx.x] = red[0];
      __syncthreads();
    }
}

__global__ void
plane_multidot_sub_kernel(const double *__restrict__ part, int count, double *__restrict__ out)
{
  const int i = threadIdx.x;
  if (i >= count)
    return;
  double s = 0.0;
  for (int b = 0; b < kPlaneDotBlocks; ++b)
    s += part[i * kPlaneDotBlocks + b];
  out[i] -= s;
}
} // namespace

long long
plane3_doubles(const DevGeom3 &G, int nI)
{
  return static_cast<long long>(nI) * G.S * 3 * G.gx * G.gy;
}

cudaError_t
launch_plane_op3(const DevGeom3 &G, int side, int op, int nI, double *x, double *buf, const double *other,
                 const double *b, const double *saved, cudaStream_t st)
{
  const long long n = plane3_doubles(G, nI);
  if (n == 0)
    return cudaSuccess;
  const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 4 * 148));
  plane_op3_kernel<<<blocks, 256, 0, st>>>(G, side, op, n, x, buf, other, b, saved);
  return cudaGetLastError();
}

cudaError_t
launch_project3_sums(const DevGeom3 &G, const double *pmean, const double *x, int nI, double *sums, cudaStream_t st)
{
  if (nI == 0)
    return cudaSuccess;
  project3_sums_kernel<<<dim3(G.S, nI), kProjThreads, 0, st>>>(G, pmean, x, sums);
  return cudaGetLastError();
}

cudaError_t
launch_project3_apply(const DevGeom3 &G, const double *sums, double inv_vol, double *x, int nI, cudaStream_t st)
{
  if (nI == 0)
    return cudaSuccess;
  project3_apply_kernel<<<dim3(G.S, nI), kProjThreads, 0, st>>>(G, sums, inv_vol, x);
  return cudaGetLastError();
}

long long
plane_multidot_part_doubles()
{
  return static_cast<long long>(kMultiMax + 1) * kPlaneDotBlocks;
}

cudaError_t
launch_plane_multidot_sub(const DevGeom3 &G, int side, int nI, const double *const *V, int m, bool with_norm,
                          const double *w, double *part, double *out, cudaStream_t st)
{
  const long long n = plane3_doubles(G, nI);
  for (int i0 = 0;; i0 += kMultiMax)
    {
      const int mm = std::min(kMultiMax, m - i0);
      const bool last = i0 + kMultiMax >= m;
      const int wn = last && with_norm ? 1 : 0;
      MultiVec mv{};
      for (int i = 0; i < mm; ++i)
        mv.p[i] = V[i0 + i];
      if (mm + wn > 0)
        {
          plane_multidot_kernel<<<kPlaneDotBlocks, 256, 0, st>>>(G, side, n, mv, mm, wn, w, part);
          plane_multidot_sub_kernel<<<1, 32, 0, st>>>(part, mm + wn, out + i0);
        }
      if (last)
        break;
    }
  return cudaGetLastError();
}

long long
transfer3_work_doubles(const DevTransfer3 &T, int nc)
{
  if (!T.spatial)
    return 0;
  return 2ll * nc * T.c.S * 3 * T.f.gz * T.f.gy * static_cast<long long>(T.c.gx);
}

cudaError_t
launch_prolongate3(const DevTransfer3 &T, const double *coarse, double *fine, int nc, cudaStream_t st, double *work)
{
  const int nf = T.h_time ? 2 * nc : nc;
  if (nf == 0)
    return cudaSuccess;
  const DevGeom3 &F = T.f, &C = T.c;
  if (T.spatial && work)
    {
      // z: T1(i, j, Z) over the coarse (i, j); y: T2(i, Y, Z); x + time: fine
      const long long p1 = static_cast<long long>(F.gz) * C.gy * C.gx, p2 = static_cast<long long>(F.gz) * F.gy * C.gx;
      double *T1 = work, *T2 = work + static_cast<long long>(nc) * C.S * 3 * p2;
      const int nb = nc * C.S * 3;
      SepDims dz{C.gx, C.gy, C.gz, C.gx, C.gy, F.gz};
      sep1d_kernel<<<dim3((C.gx * C.gy + kTrX - 1) / kTrX, F.gz, nb), kTrX, 0, st>>>(
        T.pz, 2, coarse, C.isz, C.mv, C.nsc, T1, 3ll * C.S * p1, 3 * p1, p1, dz, C.S);
      SepDims dy{C.gx, C.gy, F.gz, C.gx, F.gy, F.gz};
      sep1d_kernel<<<dim3((C.gx * F.gy + kTrX - 1) / kTrX, F.gz, nb), kTrX, 0, st>>>(
        T.py, 1, T1, 3ll * C.S * p1, 3 * p1, p1, T2, 3ll * C.S * p2, 3 * p2, p2, dy, C.S);
      sep_prolong_x_kernel<<<dim3((F.gx * F.gy + kTrX - 1) / kTrX, F.gz, nf * F.S * 3), kTrX, 0, st>>>(T, T2, fine,
                                                                                                      C.gx);
    }
  else
    {
      dim3 gv((F.gx + kTrX - 1) / kTrX, F.gy * F.gz, nf * F.S * 3);
      prolongate3_vel_kernel<<<gv, kTrX, 0, st>>>(T, coarse, fine);
    }
  const int ncm = F.nx * F.ny * F.nz * F.np;
  dim3 gp((ncm + 255) / 256, nf * F.S);
  prolongate3_pre_kernel<<<gp, 256, 0, st>>>(T, coarse, fine);
  return cudaGetLastError();
}

cudaError_t
launch_restrict3(const DevTransfer3 &T, const double *fine, double *coarse, int nc, cudaStream_t st, double *work)
{
  if (nc == 0)
    return cudaSuccess;
  const DevGeom3 &F = T.f, &C = T.c;
  if (T.spatial && work)
    {
      // x + time: T1(i, Yf, Zf); y: T2(i, j, Zf); z: coarse
      const long long p1 = static_cast<long long>(F.gz) * F.gy * C.gx, p2 = static_cast<long long>(F.gz) * C.gy * C.gx;
      double *T1 = work, *T2 = work + static_cast<long long>(nc) * C.S * 3 * p1;
      const int nb = nc * C.S * 3;
      sep_restrict_x_kernel<<<dim3((C.gx * F.gy + kTrX - 1) / kTrX, F.gz, nb), kTrX, 0, st>>>(T, fine, T1);
      SepDims dy{C.gx, F.gy, F.gz, C.gx, C.gy, F.gz};
      sep1d_kernel<<<dim3((C.gx * C.gy + kTrX - 1) / kTrX, F.gz, nb), kTrX, 0, st>>>(
        T.ry, 1, T1, 3ll * C.S * p1, 3 * p1, p1, T2, 3ll * C.S * p2, 3 * p2, p2, dy, C.S);
      SepDims dz{C.gx, C.gy, F.gz, C.gx, C.gy, C.gz};
      sep1d_kernel<<<dim3((C.gx * C.gy + kTrX - 1) / kTrX, C.gz, nb), kTrX, 0, st>>>(
        T.rz, 2, T2, 3ll * C.S * p2, 3 * p2, p2, coarse, C.isz, C.mv, C.nsc, dz, C.S);
    }
  else
    {
      dim3 gv((C.gx + kTrX - 1) / kTrX, C.gy * C.gz, nc * C.S * 3);
      restrict3_vel_kernel<<<gv, kTrX, 0, st>>>(T, fine, coarse);
    }
  const int ncm = C.nx * C.ny * C.nz * C.np;
  dim3 gp((ncm + 255) / 256, nc * C.S);
  restrict3_pre_kernel<<<gp, 256, 0, st>>>(T, fine, coarse);
  return cudaGetLastError();
}

} // namespace stmg_b200
