// Per-level constants of the B200 space-time operator, shared by host setup
// and the device kernels. Passed BY VALUE as a kernel parameter, so every
// coefficient below lives in the constant bank and feeds DFMA directly.
//
// Layout of the data the kernels address (identical to the reference's
// BlockVector, block_vector.hpp:13-45, so host buffers cross the C-ABI
// unchanged):
//   interval n            : base n * isz, isz = S * (mv + mp)
//   velocity slot a       : a * mv;   component c : + c * nsc
//   scalar node (gx,gy)   : gy * grid_x + gx      (dof_space.cpp:33)
//   pressure slot a       : S * mv + a * mp; cell (cx,cy), mode m :
//                           (cy * nx + cx) * NP + m  (dof_space.hpp:101-104)
#pragma once

#ifndef __CUDACC__
#ifndef __host__
#define __host__
#endif
#ifndef __device__
#define __device__
#endif
#endif

namespace stmg_b200
{

constexpr int kMaxN1 = 6;  // r <= 4
constexpr int kMaxP = 5;   // Legendre degrees 0..r
constexpr int kMaxS = 5;   // k <= 4
constexpr int kMaxNP = 15; // dim P_r^disc(2D), r <= 4

/// Sum-factorised 1D operator factors of one level (Cartesian cells are
/// congruent, so one set serves every cell; cf. st_operator.hpp:18-19).
/// Index convention: x-contractions are out[i] = sum_k X[i*N1+k] in[k];
/// y-accumulations are Y(i,j) += T[j*N1+l] t_l[i] (T indexed by output j and
/// input row l). J = hx*hy/4, cx = 2/hx, cy = 2/hy.
struct LevelConsts
{
  int nx, ny;            // cells per direction
  int gx, gy;            // scalar grid points per direction
  long long nsc;         // scalar nodes = gx*gy
  long long mv, mp;      // velocity dofs (2*nsc), pressure dofs
  long long isz;         // one interval: S*(mv+mp)
  // x-direction (reference-cell) factors
  double xM[kMaxN1 * kMaxN1];  // M1(i,k) = int phi_i phi_k
  double xKa[kMaxN1 * kMaxN1]; // (nu+gamma) cx^2 K1(i,k)
  double xKb[kMaxN1 * kMaxN1]; // nu cx^2 K1(i,k)
  double xC[kMaxN1 * kMaxN1];  // C1(i,k) = int phi_i' phi_k
  double xCt[kMaxN1 * kMaxN1]; // C1(k,i)
  double xLc[kMaxP * kMaxN1];  // Lc(a,k) = int L_a phi_k'
  double xLm[kMaxP * kMaxN1];  // Lm(a,k) = int L_a phi_k
  // y-direction factors, J and the physical coefficients folded in
  double yM[kMaxN1 * kMaxN1];  // J M1(j,l)
  double yKa[kMaxN1 * kMaxN1]; // J nu cy^2 K1(j,l)
  double yKb[kMaxN1 * kMaxN1]; // J (nu+gamma) cy^2 K1(j,l)
  double yCx[kMaxN1 * kMaxN1]; // J gamma cx cy C1(l,j)
  double yCy[kMaxN1 * kMaxN1]; // J gamma cx cy C1(j,l)
  double yLm[kMaxP * kMaxN1];  // J cx Lm(b,l)
  double yLc[kMaxP * kMaxN1];  // J cy Lc(b,l)
  // compact form used by the fused kernel: exactly symmetrised reference
  // factors, scalar coefficients, and temporal matrices scaled by J
  double cM1[kMaxN1 * kMaxN1], cK1[kMaxN1 * kMaxN1], cC1[kMaxN1 * kMaxN1];
  double cLm[kMaxP * kMaxN1], cLc[kMaxP * kMaxN1];
  double sax, say, sbx, sby, sg, scx, scy; // (nu+g)cx^2, nu cx^2, nu cy^2, (nu+g)cy^2, g cx cy, cx, cy
  double KtJ[kMaxS * kMaxS], MtJ[kMaxS * kMaxS], lvJ[kMaxS];
  // DG(k) temporal matrices (time_basis.cpp:8-59)
  double Kt[kMaxS * kMaxS]; // dt_plus_jump(a,b)
  double Mt[kMaxS * kMaxS]; // mass(a,b)
  double lv[kMaxS];         // left_values(a)
};

/// 1D tables of the built-in problem kernels (problems.cu), r <= 4, k <= 4:
/// assemble_rhs quadrature (st_operator.cpp:423-467) and compute_errors
/// quadrature (harness.cpp:72-183). Passed by value as a kernel parameter.
struct ProblemTables
{
  // assemble: Gauss(r+2) points/weights, GLL Lagrange basis phi(q, i)
  double ax[8], aw[8], aphi[8 * 8];
  // temporal right-Radau nodes / weights (time_basis.cpp:8-59)
  double tn[6], tw[6];
  // errors: Gauss(r+3) in space, phi / dphi(q, i), Legendre P_a(x_q)
  double ex[9], ew[9], ephi[9 * 8], edphi[9 * 8], eleg[9 * 6];
  // errors: Gauss(k+2) in time, Radau-node Lagrange values tval(q, a)
  double tq[8], tqw[8], tval[8 * 6];
  // GLL nodes of the velocity basis (interpolate_exact)
  double gll[8];
};

/// Degree-major P_r^disc mode list (pdisc.cpp:41-55): mode m has Legendre
/// degrees (ax(m), ay(m)).
__host__ __device__ constexpr int
pdisc_mode_ax(int r, int m)
{
  int idx = 0;
  for (int deg = 0; deg <= r; ++deg)
    for (int a = deg; a >= 0; --a)
      {
        if (idx == m)
          return a;
        ++idx;
      }
  return -1;
}

__host__ __device__ constexpr int
pdisc_mode_ay(int r, int m)
{
  int idx = 0;
  for (int deg = 0; deg <= r; ++deg)
    for (int a = deg; a >= 0; --a)
      {
        if (idx == m)
          return deg - a;
        ++idx;
      }
  return -1;
}

} // namespace stmg_b200
