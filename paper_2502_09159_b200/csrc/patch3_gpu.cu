// GPU setup of the exact cell-Vanka patch inverses on deformed 3D levels
// (BASELINE C5: 32^3 cells, Q3/P2disc x DG(2), n_T = 606 per interior cell).
//
// Replaces, for one-class-per-cell levels, the host loop of
// VankaSmoother::build (vanka.cpp:30-194): patch dof lists (host, cheap),
// local matrices R_T S R_T^T (vanka.cpp:92-165) and their factorizations
// (vanka.cpp:167-176), here as explicit inverses:
//   1. elem3_kernel        per-cell element matrices on the trilinear cell
//                          (mass, nu grad:grad + gamma div div, B), Gauss
//                          quadrature, the same formulas as setup3d.cpp
//                          cell3_matrices;
//   2. patch3_assemble     R_T S R_T^T of every cell patch from the element
//                          matrices of the <= 8 cells sharing each node pair,
//                          combined with the DG(k) time matrices
//                          (K_t (x) M + M_t (x) A, -+ M_t (x) B), written in
//                          place into the inverse storage;
//   3. gj_inverse_kernel   batched blocked Gauss-Jordan inversion in place,
//                          one CTA per patch, 32-column pivot blocks: the
//                          trailing rank-32 updates run on the FP64 tensor
//                          path (DMMA m8n8k4) with the pivot row panel in
//                          shared memory. No pivoting: the velocity block
//                          K_t (x) M + M_t (x) (nu A + gamma G) has a positive
//                          definite symmetric part (DG upwind K_t + K_t^T >= 0,
//                          M_t > 0, A on the patch's interior nodes > 0) and
//                          the pressure Schur complement B K^{-1} B^T is
//                          nonsingular for patches with >= 2 cells per mesh
//                          direction; a vanishing pivot is reported per patch
//                          (status) and the level falls back to the host
//                          path (LU with partial pivoting).
#include "st3d.hpp"

#include <cuda_runtime.h>

namespace stmg_b200
{
namespace
{
__device__ __forceinline__ void
dmma(double (&d)[2], double a, double b)
{
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------- element matrices
// E layout per cell (stride elem3_stride): mass [NV x NV], a [3NV x 3NV]
// (row (c, node), column (c2, node)), b [np x 3NV], as Cell3Matrices.
template <int N>
__global__ void __launch_bounds__(256)
elem3_kernel(Level3Consts P, double *__restrict__ E, long long stride, int *__restrict__ status)
{
  constexpr int NV = N * N * N, NQ = N * N * N;
  const int np = P.np;
  extern __shared__ double sm[];
  double *val = sm;                 // [NQ][NV]
  double *gp = val + NQ * NV;       // [NQ][NV][3]
  double *wd = gp + NQ * NV * 3;    // [NQ]
  double *Ji = wd + NQ;             // [NQ][9], Ji[e*3 + d] = dxi_e / dX_d
  double *psi = Ji + NQ * 9;        // [NQ][np]
  __shared__ double X8[8][3];
  const int tid = threadIdx.x;
  const long long cell = blockIdx.x;
  const int cx = static_cast<int>(cell % P.nx), cy = static_cast<int>((cell / P.nx) % P.ny),
            cz = static_cast<int>(cell / (static_cast<long long>(P.nx) * P.ny));
  if (tid < 24)
    {
      const int c = tid / 3, d = tid % 3;
      const int vx = cx + (c & 1), vy = cy + ((c >> 1) & 1), vz = cz + (c >> 2);
      X8[c][d] = P.verts[((static_cast<long long>(vz) * (P.ny + 1) + vy) * (P.nx + 1) + vx) * 3 + d];
    }
  __syncthreads();
  for (int q = tid; q < NQ; q += blockDim.x)
    {
      const int qx = q % N, qy = (q / N) % N, qz = q / (N * N);
      const double xi[3] = {P.xq[qx], P.xq[qy], P.xq[qz]};
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
        atomicExch(status, 2); // inverted cell
      double *ji = Ji + q * 9;
      ji[0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
      ji[1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
      ji[2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
      ji[3] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
      ji[4] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
      ji[5] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
      ji[6] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
      ji[7] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
      ji[8] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
      wd[q] = P.w[qx] * P.w[qy] * P.w[qz] * det;
    }
  __syncthreads();
  for (int e = tid; e < NQ * NV; e += blockDim.x)
    {
      const int q = e / NV, t = e % NV;
      const int qx = q % N, qy = (q / N) % N, qz = q / (N * N);
      const int i = t % N, j = (t / N) % N, k = t / (N * N);
      const double v0 = P.phi[qx * N + i], v1 = P.phi[qy * N + j], v2 = P.phi[qz * N + k];
      const double gr[3] = {P.dphi[qx * N + i] * v1 * v2, v0 * P.dphi[qy * N + j] * v2, v0 * v1 * P.dphi[qz * N + k]};
      val[e] = v0 * v1 * v2;
      const double *ji = Ji + q * 9;
      for (int d = 0; d < 3; ++d)
        gp[e * 3 + d] = gr[0] * ji[d] + gr[1] * ji[3 + d] + gr[2] * ji[6 + d];
    }
  for (int e = tid; e < NQ * np; e += blockDim.x)
    {
      const int q = e / np, l = e % np;
      const int qx = q % N, qy = (q / N) % N, qz = q / (N * N);
      psi[e] = P.leg[P.ex[l][0] * N + qx] * P.leg[P.ex[l][1] * N + qy] * P.leg[P.ex[l][2] * N + qz];
    }
  __syncthreads();
  double *Ec = E + cell * stride;
  double *Em = Ec, *Ea = Ec + NV * NV, *Eb = Ea + 9 * NV * NV;
  for (int pr = tid; pr < NV * NV; pr += blockDim.x)
    {
      const int a = pr / NV, b = pr % NV;
      double m = 0.0, s[3][3] = {};
      for (int q = 0; q < NQ; ++q)
        {
          const double w = wd[q];
          const double *ga = gp + (q * NV + a) * 3, *gb = gp + (q * NV + b) * 3;
          m += w * val[q * NV + a] * val[q * NV + b];
          const double gg = ga[0] * gb[0] + ga[1] * gb[1] + ga[2] * gb[2];
          for (int c = 0; c < 3; ++c)
            for (int c2 = 0; c2 < 3; ++c2)
              s[c][c2] += w * (P.gamma * ga[c] * gb[c2] + (c == c2 ? P.nu * gg : 0.0));
        }
      Em[pr] = m;
      for (int c = 0; c < 3; ++c)
        for (int c2 = 0; c2 < 3; ++c2)
          Ea[(static_cast<long long>(c) * NV + a) * 3 * NV + c2 * NV + b] = s[c][c2];
    }
  for (int pr = tid; pr < np * NV; pr += blockDim.x)
    {
      const int l = pr / NV, t = pr % NV;
      double s[3] = {};
      for (int q = 0; q < NQ; ++q)
        {
          const double w = wd[q] * psi[q * np + l];
          for (int c = 0; c < 3; ++c)
            s[c] += w * gp[(q * NV + t) * 3 + c];
        }
      for (int c = 0; c < 3; ++c)
        Eb[static_cast<long long>(l) * 3 * NV + c * NV + t] = s[c];
    }
}

// ---------------------------------------------------------------- patch assembly
// Patch dof order (setup3d.cpp cell_patch, vanka.cpp:69-86): velocity rows
// (a, c, t) -> (a * 3 + c) * nl + t over the patch's unconstrained nodes t
// (lexicographic k, j, i), then pressure (a, l) -> S * 3 * nl + a * np + l.
template <int N>
__global__ void __launch_bounds__(256)
patch3_assemble_kernel(Level3Consts P, int S, const double *__restrict__ E, long long estride,
                       double *__restrict__ Aall, const long long *__restrict__ aoff, const int *__restrict__ ntv,
                       long long cell0, int *__restrict__ status)
{
  // P describes the element-matrix mesh: the level itself, or for a z-split
  // level the level plus one ghost cell layer across each interface; patch
  // oc (layouts, inverses) belongs to its cell cell0 + oc
  constexpr int NV = N * N * N, p = N - 1;
  const int np = P.np;
  __shared__ int loc[NV];
  __shared__ int s_nl;
  const int tid = threadIdx.x;
  const long long oc = blockIdx.x, cell = cell0 + oc;
  const int cx = static_cast<int>(cell % P.nx), cy = static_cast<int>((cell / P.nx) % P.ny),
            cz = static_cast<int>(cell / (static_cast<long long>(P.nx) * P.ny));
  if (tid == 0)
    {
      int nl = 0;
      for (int t = 0; t < NV; ++t)
        {
          const int i = t % N, j = (t / N) % N, k = t / (N * N);
          const int X = cx * p + i, Y = cy * p + j, Z = cz * p + k;
          const bool bnd = X == 0 || Y == 0 || Z == P.zlo || X == P.gx - 1 || Y == P.gy - 1 || Z == P.zhi;
          if (!bnd)
            loc[nl++] = t;
        }
      s_nl = nl;
    }
  __syncthreads();
  const int nl = s_nl;
  const int nvel = S * 3 * nl, nt = nvel + S * np;
  if (nt != ntv[oc])
    {
      if (tid == 0)
        atomicExch(status, 3); // host / device patch layouts disagree
      return;
    }
  double *A = Aall + aoff[oc];
  __shared__ double kt[kMaxS * kMaxS], mt[kMaxS * kMaxS];
  if (tid < S * S)
    {
      kt[tid] = P.Kt[tid];
      mt[tid] = P.Mt[tid];
    }
  __syncthreads();
  const long long cstride = 1, ystride = P.nx, zstride = static_cast<long long>(P.nx) * P.ny;
  auto range = [&](int x, int &lo, int &hi) {
    lo = x == 0 ? -1 : 0;
    hi = x == p ? 1 : 0;
  };
  // velocity-velocity: sum over the cells sharing both nodes (vanka.cpp:92-143)
  for (int pr = tid; pr < nl * nl; pr += blockDim.x)
    {
      const int t = pr / nl, u = pr % nl;
      const int lt = loc[t], lu = loc[u];
      const int ti = lt % N, tj = (lt / N) % N, tk = lt / (N * N);
      const int ui = lu % N, uj = (lu / N) % N, uk = lu / (N * N);
      int lx0, lx1, ly0, ly1, lz0, lz1, a0, a1;
      range(ti, lx0, lx1);
      range(ui, a0, a1);
      lx0 = max(lx0, a0);
      lx1 = min(lx1, a1);
      range(tj, ly0, ly1);
      range(uj, a0, a1);
      ly0 = max(ly0, a0);
      ly1 = min(ly1, a1);
      range(tk, lz0, lz1);
      range(uk, a0, a1);
      lz0 = max(lz0, a0);
      lz1 = min(lz1, a1);
      double ms = 0.0, as[3][3] = {};
      for (int dz = lz0; dz <= lz1; ++dz)
        for (int dy = ly0; dy <= ly1; ++dy)
          for (int dx = lx0; dx <= lx1; ++dx)
            {
              const long long e = cell + dx * cstride + dy * ystride + dz * zstride;
              const double *Ee = E + e * estride;
              const int at = ((tk - dz * p) * N + (tj - dy * p)) * N + (ti - dx * p);
              const int au = ((uk - dz * p) * N + (uj - dy * p)) * N + (ui - dx * p);
              ms += Ee[at * NV + au];
              const double *Ea = Ee + NV * NV;
              for (int c = 0; c < 3; ++c)
                for (int c2 = 0; c2 < 3; ++c2)
                  as[c][c2] += Ea[(static_cast<long long>(c) * NV + at) * 3 * NV + c2 * NV + au];
            }
      for (int a = 0; a < S; ++a)
        for (int c = 0; c < 3; ++c)
          {
            double *row = A + static_cast<long long>((a * 3 + c) * nl + t) * nt;
            for (int b = 0; b < S; ++b)
              for (int c2 = 0; c2 < 3; ++c2)
                {
                  double v = mt[a * S + b] * as[c][c2];
                  if (c == c2)
                    v += kt[a * S + b] * ms;
                  row[(b * 3 + c2) * nl + u] = v;
                }
          }
    }
  // velocity-pressure / pressure-velocity: the patch cell's B (vanka.cpp:124-140)
  const double *Eb = E + cell * estride + 10 * NV * NV;
  for (int pr = tid; pr < np * 3 * nl; pr += blockDim.x)
    {
      const int l = pr / (3 * nl), c = (pr / nl) % 3, u = pr % nl;
      const double bv = Eb[static_cast<long long>(l) * 3 * NV + c * NV + loc[u]];
      for (int a = 0; a < S; ++a)
        for (int b = 0; b < S; ++b)
          {
            A[static_cast<long long>((a * 3 + c) * nl + u) * nt + nvel + b * np + l] = -mt[a * S + b] * bv;
            A[static_cast<long long>(nvel + a * np + l) * nt + (b * 3 + c) * nl + u] = mt[a * S + b] * bv;
          }
    }
  for (int pr = tid; pr < S * np * S * np; pr += blockDim.x)
    {
      const int r = pr / (S * np), c = pr % (S * np);
      A[static_cast<long long>(nvel + r) * nt + nvel + c] = 0.0;
    }
}

// ---------------------------------------------------------------- factored blocks
// The time-diagonalised patch blocks (st3d.hpp Fac3Params) of every owned
// cell: B_b = alpha_b M^ + A^ (real eigenvalue) or the 2 x 2 block form of a
// complex pair, from the same spatial patch matrices as patch3_assemble:
// M^ (velocity mass per component), A^ = [[A, -B^T], [B, 0]].
template <int N>
__global__ void __launch_bounds__(256)
patch3_fac_assemble_kernel(Level3Consts P, int S, Fac3Params F, const double *__restrict__ E, long long estride,
                           double *__restrict__ Aall, const long long *__restrict__ aoff,
                           const int *__restrict__ cell_nt, long long cell0, int *__restrict__ status)
{
  constexpr int NV = N * N * N, p = N - 1;
  const int np = P.np;
  __shared__ int loc[NV];
  __shared__ int s_nl;
  const int tid = threadIdx.x;
  const long long oc = blockIdx.x, cell = cell0 + oc;
  const int cx = static_cast<int>(cell % P.nx), cy = static_cast<int>((cell / P.nx) % P.ny),
            cz = static_cast<int>(cell / (static_cast<long long>(P.nx) * P.ny));
  if (tid == 0)
    {
      int nl = 0;
      for (int t = 0; t < NV; ++t)
        {
          const int i = t % N, j = (t / N) % N, k = t / (N * N);
          const int X = cx * p + i, Y = cy * p + j, Z = cz * p + k;
          const bool bnd = X == 0 || Y == 0 || Z == P.zlo || X == P.gx - 1 || Y == P.gy - 1 || Z == P.zhi;
          if (!bnd)
            loc[nl++] = t;
        }
      s_nl = nl;
    }
  __syncthreads();
  const int nl = s_nl, nvs = 3 * nl, ns = nvs + np;
  if (S * ns != cell_nt[oc])
    {
      if (tid == 0)
        atomicExch(status, 3); // host / device patch layouts disagree
      return;
    }
  for (int b = 0; b < F.nb; ++b)
    {
      double *A = Aall + aoff[2 * oc + b];
      const long long m = static_cast<long long>(F.sz[b]) * ns;
      for (long long e = tid; e < m * m; e += blockDim.x)
        A[e] = 0.0;
    }
  __syncthreads();
  const long long cstride = 1, ystride = P.nx, zstride = static_cast<long long>(P.nx) * P.ny;
  auto range = [&](int x, int &lo, int &hi) {
    lo = x == 0 ? -1 : 0;
    hi = x == p ? 1 : 0;
  };
  for (int pr = tid; pr < nl * nl; pr += blockDim.x)
    {
      const int t = pr / nl, u = pr % nl;
      const int lt = loc[t], lu = loc[u];
      const int ti = lt % N, tj = (lt / N) % N, tk = lt / (N * N);
      const int ui = lu % N, uj = (lu / N) % N, uk = lu / (N * N);
      int lx0, lx1, ly0, ly1, lz0, lz1, a0, a1;
      range(ti, lx0, lx1);
      range(ui, a0, a1);
      lx0 = max(lx0, a0);
      lx1 = min(lx1, a1);
      range(tj, ly0, ly1);
      range(uj, a0, a1);
      ly0 = max(ly0, a0);
      ly1 = min(ly1, a1);
      range(tk, lz0, lz1);
      range(uk, a0, a1);
      lz0 = max(lz0, a0);
      lz1 = min(lz1, a1);
      double ms = 0.0, as[3][3] = {};
      for (int dz = lz0; dz <= lz1; ++dz)
        for (int dy = ly0; dy <= ly1; ++dy)
          for (int dx = lx0; dx <= lx1; ++dx)
            {
              const long long e = cell + dx * cstride + dy * ystride + dz * zstride;
              const double *Ee = E + e * estride;
              const int at = ((tk - dz * p) * N + (tj - dy * p)) * N + (ti - dx * p);
              const int au = ((uk - dz * p) * N + (uj - dy * p)) * N + (ui - dx * p);
              ms += Ee[at * NV + au];
              const double *Ea = Ee + NV * NV;
              for (int c = 0; c < 3; ++c)
                for (int c2 = 0; c2 < 3; ++c2)
                  as[c][c2] += Ea[(static_cast<long long>(c) * NV + at) * 3 * NV + c2 * NV + au];
            }
      for (int b = 0; b < F.nb; ++b)
        {
          const int sz = F.sz[b];
          const long long m = static_cast<long long>(sz) * ns;
          double *A = Aall + aoff[2 * oc + b];
          for (int bi = 0; bi < sz; ++bi)
            for (int bj = 0; bj < sz; ++bj)
              {
                const double cm = bi == bj ? F.alpha[b] : (bi == 0 ? F.beta[b] : -F.beta[b]);
                const double ca = bi == bj ? 1.0 : 0.0;
                for (int c = 0; c < 3; ++c)
                  for (int c2 = 0; c2 < 3; ++c2) // transposed: (row, col) at col * m + row
                    A[static_cast<long long>(bj * nvs + c2 * nl + u) * m + bi * nvs + c * nl + t] =
                      ca * as[c][c2] + (c == c2 ? cm * ms : 0.0);
              }
        }
    }
  // B and -B^T: the patch cell's own B (vanka.cpp:124-140), diagonal blocks only
  const double *Eb = E + cell * estride + 10 * NV * NV;
  for (int pr = tid; pr < np * 3 * nl; pr += blockDim.x)
    {
      const int l = pr / (3 * nl), c = (pr / nl) % 3, u = pr % nl;
      const double bv = Eb[static_cast<long long>(l) * 3 * NV + c * NV + loc[u]];
      for (int b = 0; b < F.nb; ++b)
        {
          const int sz = F.sz[b];
          const long long m = static_cast<long long>(sz) * ns;
          double *A = Aall + aoff[2 * oc + b];
          for (int bi = 0; bi < sz; ++bi)
            {
              const long long vr = bi * nvs + c * nl + u, pc = sz * nvs + bi * np + l;
              A[pc * m + vr] = -bv; // transposed
              A[vr * m + pc] = bv;
            }
        }
    }
}

// ---------------------------------------------------------------- batched inverse
constexpr int kGJB = 32;       // pivot block
constexpr int kGJThreads = 512; // 16 warps
constexpr int kGJDLd = kGJB + 1;

__host__ __device__ constexpr int
gj_ldr(int n)
{
  return (n + 15) / 16 * 16 + 8; // == 8 mod 16 doubles: conflict-free B-fragment loads
}

__global__ void __launch_bounds__(kGJThreads, 1)
gj_inverse_kernel(double *__restrict__ Aall, const long long *__restrict__ aoff, const int *__restrict__ ntv,
                  int *__restrict__ status)
{
  extern __shared__ double sm[];
  double *Dinv = sm;                 // kGJB x kGJDLd
  double *Rp = sm + kGJB * kGJDLd;   // kGJB x ldr: pivot row panel D^{-1} A[K, :]
  const int mat = blockIdx.x;
  const int n = ntv[mat];
  const int ldr = gj_ldr(n);
  double *A = Aall + aoff[mat];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  bool bad = false;
  for (int k0 = 0; k0 < n; k0 += kGJB)
    {
      const int kb = min(kGJB, n - k0);
      // (1) pivot block, identity-padded to 32 x 32
      for (int e = tid; e < kGJB * kGJB; e += kGJThreads)
        {
          const int r = e / kGJB, c = e % kGJB;
          Dinv[r * kGJDLd + c] = (r < kb && c < kb) ? A[static_cast<long long>(k0 + r) * n + k0 + c] : (r == c ? 1.0 : 0.0);
        }
      __syncthreads();
      if (warp == 0)
        {
          // unblocked in-place Gauss-Jordan, lane j owns column j
          for (int pv = 0; pv < kGJB; ++pv)
            {
              double colp[kGJB];
#pragma unroll
              for (int i = 0; i < kGJB; ++i)
                colp[i] = Dinv[i * kGJDLd + pv];
              const double piv = Dinv[pv * kGJDLd + pv];
              __syncwarp();
              if (!(fabs(piv) > 1e-280) || !isfinite(piv))
                bad = true;
              const double inv = 1.0 / piv;
              const double mpj = (lane == pv ? 1.0 : Dinv[pv * kGJDLd + lane]) * inv;
              Dinv[pv * kGJDLd + lane] = mpj;
#pragma unroll
              for (int i = 0; i < kGJB; ++i)
                if (i != pv)
                  {
                    const double mij = lane == pv ? 0.0 : Dinv[i * kGJDLd + lane];
                    Dinv[i * kGJDLd + lane] = mij - colp[i] * mpj;
                  }
              __syncwarp();
            }
        }
      __syncthreads();
      // (2) row panel R' = D^{-1} A[K, j], j outside K: shared copy and global write-back
      for (int j = tid; j < n; j += kGJThreads)
        {
          if (j >= k0 && j < k0 + kb)
            continue;
          double col[kGJB];
#pragma unroll
          for (int q = 0; q < kGJB; ++q)
            col[q] = q < kb ? A[static_cast<long long>(k0 + q) * n + j] : 0.0;
#pragma unroll 4
          for (int r = 0; r < kGJB; ++r)
            {
              double s = 0.0;
#pragma unroll
              for (int q = 0; q < kGJB; ++q)
                s = fma(Dinv[r * kGJDLd + q], col[q], s);
              Rp[r * ldr + j] = r < kb ? s : 0.0;
              if (r < kb)
                A[static_cast<long long>(k0 + r) * n + j] = s;
            }
        }
      for (int e = tid; e < kGJB * kGJB; e += kGJThreads) // K columns of the panel: unused, keep finite
        {
          const int r = e / kGJB, c = k0 + e % kGJB;
          if (c < ldr)
            Rp[r * ldr + c] = 0.0;
        }
      __syncthreads();
      // (3) rows outside K: A[i, j] -= A[i, K] R'[:, j] (DMMA), then A[i, K] = -A[i, K] D^{-1}
      const int nrt = (n + 7) / 8;
      for (int rt = warp; rt < nrt; rt += kGJThreads / 32)
        {
          const int i0 = rt * 8;
          if (i0 >= k0 && i0 < k0 + kb)
            continue;
          const int row = i0 + lr;
          double af[kGJB / 4];
#pragma unroll
          for (int kk = 0; kk < kGJB / 4; ++kk)
            {
              const int c = 4 * kk + lc;
              af[kk] = (row < n && c < kb) ? -A[static_cast<long long>(row) * n + k0 + c] : 0.0;
            }
          for (int j0 = 0; j0 < n; j0 += 8)
            {
              if (j0 >= k0 && j0 < k0 + kb)
                continue;
              const int col = j0 + 2 * lc;
              double acc[2];
              acc[0] = (row < n && col < n) ? A[static_cast<long long>(row) * n + col] : 0.0;
              acc[1] = (row < n && col + 1 < n) ? A[static_cast<long long>(row) * n + col + 1] : 0.0;
              const double *bb = Rp + lc * ldr + j0 + lr;
#pragma unroll
              for (int kk = 0; kk < kGJB / 4; ++kk)
                dmma(acc, af[kk], bb[4 * kk * ldr]);
              if (row < n && col < n)
                A[static_cast<long long>(row) * n + col] = acc[0];
              if (row < n && col + 1 < n)
                A[static_cast<long long>(row) * n + col + 1] = acc[1];
            }
#pragma unroll
          for (int ct = 0; ct < kGJB / 8; ++ct)
            {
              double acc[2] = {0.0, 0.0};
#pragma unroll
              for (int kk = 0; kk < kGJB / 4; ++kk)
                dmma(acc, af[kk], Dinv[(4 * kk + lc) * kGJDLd + 8 * ct + lr]);
              const int col = 8 * ct + 2 * lc;
              if (row < n && col < kb)
                A[static_cast<long long>(row) * n + k0 + col] = acc[0];
              if (row < n && col + 1 < kb)
                A[static_cast<long long>(row) * n + k0 + col + 1] = acc[1];
            }
        }
      // (4) the pivot block itself
      for (int e = tid; e < kb * kb; e += kGJThreads)
        {
          const int r = e / kb, c = e % kb;
          A[static_cast<long long>(k0 + r) * n + k0 + c] = Dinv[r * kGJDLd + c];
        }
      __syncthreads();
    }
  if (warp == 0 && __any_sync(0xffffffffu, bad) && lane == 0)
    atomicExch(status, 1); // vanishing pivot: the host path (partial pivoting) takes over
}
} // namespace

long long
elem3_stride(int r)
{
  const int N = r + 2, nv = N * N * N, np = (r + 1) * (r + 2) * (r + 3) / 6;
  return 10LL * nv * nv + static_cast<long long>(np) * 3 * nv;
}

cudaError_t
launch_patch3_setup(const Level3Consts &P, int r, int S, double *E, double *Aall, const long long *aoff,
                    const int *ntv, int max_nt, long long ncells, int *status, cudaStream_t st, long long ncells_elem,
                    long long cell0)
{
  if (ncells_elem < 0)
    ncells_elem = ncells;
  const long long es = elem3_stride(r);
  const int N = r + 2, nv = N * N * N, nq = nv;
  const size_t esmem = sizeof(double) * (static_cast<size_t>(nq) * nv * 4 + nq * 10 + static_cast<size_t>(nq) * P.np);
  auto go = [&](auto elem, auto asm_) {
    cudaFuncSetAttribute(elem, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(esmem));
    elem<<<static_cast<unsigned>(ncells_elem), 256, esmem, st>>>(P, E, es, status);
    asm_<<<static_cast<unsigned>(ncells), 256, 0, st>>>(P, S, E, es, Aall, aoff, ntv, cell0, status);
  };
  if (r == 1)
    go(elem3_kernel<3>, patch3_assemble_kernel<3>);
  else if (r == 2)
    go(elem3_kernel<4>, patch3_assemble_kernel<4>);
  else
    return cudaErrorInvalidValue;
  const size_t gsmem = sizeof(double) * (kGJB * kGJDLd + static_cast<size_t>(kGJB) * gj_ldr(max_nt));
  cudaFuncSetAttribute(gj_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(gsmem));
  gj_inverse_kernel<<<static_cast<unsigned>(ncells), kGJThreads, gsmem, st>>>(Aall, aoff, ntv, status);
  return cudaGetLastError();
}

cudaError_t
launch_patch3_fac_setup(const Level3Consts &P, int r, int S, const Fac3Params &F, double *E, double *Aall,
                        const long long *aoff, const int *ntv, const int *cell_nt, int max_m, long long ncells,
                        int *status, cudaStream_t st, long long ncells_elem, long long cell0)
{
  if (ncells_elem < 0)
    ncells_elem = ncells;
  if (F.nb < 1 || F.nb > 2)
    return cudaErrorInvalidValue; // matrices 2c, 2c + 1 per cell
  const long long es = elem3_stride(r);
  const int N = r + 2, nv = N * N * N, nq = nv;
  const size_t esmem = sizeof(double) * (static_cast<size_t>(nq) * nv * 4 + nq * 10 + static_cast<size_t>(nq) * P.np);
  auto go = [&](auto elem, auto asm_) {
    cudaFuncSetAttribute(elem, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(esmem));
    elem<<<static_cast<unsigned>(ncells_elem), 256, esmem, st>>>(P, E, es, status);
    asm_<<<static_cast<unsigned>(ncells), 256, 0, st>>>(P, S, F, E, es, Aall, aoff, cell_nt, cell0, status);
  };
  if (r == 1)
    go(elem3_kernel<3>, patch3_fac_assemble_kernel<3>);
  else if (r == 2)
    go(elem3_kernel<4>, patch3_fac_assemble_kernel<4>);
  else
    return cudaErrorInvalidValue;
  // the 1-block case (nb == 1) leaves matrix 2c + 1 empty (size 0)
  const size_t gsmem = sizeof(double) * (kGJB * kGJDLd + static_cast<size_t>(kGJB) * gj_ldr(max_m));
  cudaFuncSetAttribute(gj_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(gsmem));
  gj_inverse_kernel<<<static_cast<unsigned>(2 * ncells), kGJThreads, gsmem, st>>>(Aall, aoff, ntv, status);
  return cudaGetLastError();
}

cudaError_t
launch_gj_inverse(double *Aall, const long long *aoff, const int *ntv, int count, int max_nt, int *status,
                  cudaStream_t st)
{
  const size_t gsmem = sizeof(double) * (kGJB * kGJDLd + static_cast<size_t>(kGJB) * gj_ldr(max_nt));
  cudaFuncSetAttribute(gj_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(gsmem));
  gj_inverse_kernel<<<static_cast<unsigned>(count), kGJThreads, gsmem, st>>>(Aall, aoff, ntv, status);
  return cudaGetLastError();
}

} // namespace stmg_b200
