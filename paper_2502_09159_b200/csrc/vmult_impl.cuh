// Fused matrix-free space-time operator on B200 (sm_100a), FP64.
//
// Replaces SpaceTimeBlockOperator::apply_block / apply_block_raw /
// coupling_rhs (st_operator.cpp:321-421) and the residual b - D x of
// VankaSmoother::smooth_step (vanka.cpp:225-228), for one interval or the
// all-at-once system of N intervals with the DG jump coupling
//   y_n = D x_n - Z C x_{n-1}[slot k]      (Eq. GloSys).
//
// Design:
//  * One pass over memory: all k+1 temporal slots and all five spatial
//    operators (mass, Laplacian, grad-div, B, B^T) of a cell are evaluated in
//    registers. The temporal Kronecker combination is done on nodal values
//    (UK = sum_b K_ab u^b - lv_a v_prev, UM = sum_b M_ab u^b), so each output
//    slot costs one spatial Stokes cell operator.
//  * Cartesian cells are congruent: the element operator factorises into 1D
//    matrices (M1, K1, C1, Legendre moments) that sit in the kernel parameter
//    constant bank (LevelConsts) and feed DFMA directly.
//  * Thread mapping: warp = one (output slot a, velocity component) pair
//    (pressure rides with the x component), lane = one cell of a strip of
//    31 owned cells (+1 halo cell on the left). Slot and component are
//    compile-time per warp (dispatch switch), so every coefficient is a
//    uniform-register DFMA operand and only one component's accumulators are
//    live.
//  * The block stages the node rows of its strip (all slots, both
//    components, the coupling slot of the previous interval) and the cell
//    pressures in shared memory with fully coalesced loads, as a ring buffer
//    of n1 node rows over the y-march: every input is read from HBM once per
//    block and shared by the 2S warps. A block marches upward through
//    a segment of cell rows. Contributions to shared nodes are summed with
//    __shfl_up_sync across the strip (x) and a register carry (y): no atomics,
//    no zero-fill pass, every output written exactly once. Halo work: 1/31 in
//    x, 1/rows_per_seg in y.
#pragma once
#include "level_consts.cuh"

#include <cuda_runtime.h>

namespace stmg_b200
{

namespace vmult_detail
{
constexpr int kStrip = 31; // owned cells per warp strip
constexpr int kMinBlocksR2 = 1;
#ifndef STMG_VMULT_SPLIT
#define STMG_VMULT_SPLIT 0
#endif
constexpr bool kSplitComps = STMG_VMULT_SPLIT != 0;

__device__ __forceinline__ void
cp_async8(double *dst, const double *src)
{
  const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(saddr), "l"(src));
}
__device__ __forceinline__ void
cp_async_commit()
{
  asm volatile("cp.async.commit_group;\n" ::);
}
template <int N>
__device__ __forceinline__ void
cp_async_wait()
{
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}



template <int R, int S>
struct StripLayout
{
  static constexpr int N1 = R + 2, p = R + 1, NPM = (R + 1) * (R + 2) / 2;
  static constexpr int RL = 32 * p + 1;          // nodes per staged row
  static constexpr int NR = 2 * p + 1;           // ring: rows of the current cell row + the prefetched next
  static constexpr int NARR = 2 * S + 2;         // (slot, comp) arrays + coupling slot
  static constexpr int VEL = NARR * NR * RL;     // doubles
  static constexpr int PRE = S * 32 * NPM;       // doubles per pressure buffer (double-buffered)
  static constexpr int BYTES = 8 * (VEL + 2 * PRE);
  __device__ static int vidx(int arr, int row_slot, int xloc) { return (arr * NR + row_slot) * RL + xloc; }
};

/// One warp's share of one cell row: output slot A, component COMP
/// (0: x-velocity + pressure, 1: y-velocity, 2: everything).
template <int R, int S, int COMP, bool RESID, bool RAW>
__device__ __forceinline__ void
vmult_row(const LevelConsts &P, const double *__restrict__ sm, const double *__restrict__ x,
          const double *__restrict__ b, double *__restrict__ y, int n, int cx0, int cy, bool write_row,
          bool add_carry, bool coupled_here, double (&carx)[R + 2], double (&cary)[R + 2], const int A,
          const double (&kt)[S], const double (&mt)[S], const double lva)
{
  using L = StripLayout<R, S>;
  constexpr int N1 = R + 2, p = R + 1, NPM = (R + 1) * (R + 2) / 2, PL = R + 1;
  constexpr bool DOX = COMP != 1, DOY = COMP != 0;
  const int lane = threadIdx.x & 31;
  const int cx = cx0 + lane;
  const bool active = cx >= 0 && cx < P.nx;
  const bool owner = lane >= 1 && active;
  const long long isz = P.isz, mv = P.mv, mp = P.mp, nsc = P.nsc;
  const int gx = P.gx, gy = P.gy;
  const double *sp = sm + L::VEL + (cy & 1) * L::PRE;

  double Yx[DOX ? N1 : 1][N1], Yy[DOY ? N1 : 1][N1], Yp[DOX ? NPM : 1];
#pragma unroll
  for (int i = 0; i < N1; ++i)
#pragma unroll
    for (int j = 0; j < N1; ++j)
      {
        if constexpr (DOX)
          Yx[i][j] = 0.0;
        if constexpr (DOY)
          Yy[i][j] = 0.0;
      }
  if constexpr (DOX)
#pragma unroll
    for (int m = 0; m < NPM; ++m)
      Yp[m] = 0.0;

  if (active)
    {
      // ---- pressure: PM = sum_b Mt(A,b) p^b; B^T init of Yx / Yy
      {
        double PM[NPM];
#pragma unroll
        for (int m = 0; m < NPM; ++m)
          PM[m] = 0.0;
#pragma unroll
        for (int bs = 0; bs < S; ++bs)
#pragma unroll
          for (int m = 0; m < NPM; ++m)
            PM[m] = fma(mt[bs], sp[(bs * 32 + lane) * NPM + m], PM[m]);
#pragma unroll
        for (int bb = 0; bb < PL; ++bb)
          {
            double Q[N1], Qy[N1];
#pragma unroll
            for (int i = 0; i < N1; ++i)
              Q[i] = Qy[i] = 0.0;
#pragma unroll
            for (int m = 0; m < NPM; ++m)
              {
                if (pdisc_mode_ay(R, m) != bb)
                  continue;
                const int am = pdisc_mode_ax(R, m);
#pragma unroll
                for (int i = 0; i < N1; ++i)
                  {
                    if constexpr (DOX)
                      Q[i] = fma(P.xLc[am * N1 + i], PM[m], Q[i]);
                    if constexpr (DOY)
                      Qy[i] = fma(P.xLm[am * N1 + i], PM[m], Qy[i]);
                  }
              }
#pragma unroll
            for (int i = 0; i < N1; ++i)
#pragma unroll
              for (int j = 0; j < N1; ++j)
                {
                  if constexpr (DOX)
                    Yx[i][j] = fma(-Q[i], P.yLm[bb * N1 + j], Yx[i][j]);
                  if constexpr (DOY)
                    Yy[i][j] = fma(-Qy[i], P.yLc[bb * N1 + j], Yy[i][j]);
                }
          }
      }

      // ---- velocity rows of the cell (from the staged strip)
#pragma unroll
      for (int l = 0; l < N1; ++l)
        {
          const int Yr = cy * p + l;
          const int rs = Yr % L::NR;
          const bool yb = !RAW && (Yr == 0 || Yr == gy - 1);
          double UKx[N1], UMx[N1], UKy[N1], UMy[N1];
#pragma unroll
          for (int k = 0; k < N1; ++k)
            {
              const int xl = lane * p + k;
              const int Xn = cx * p + k;
              // constrained inputs are zeroed on read (apply_block, st_operator.cpp:333-341)
              const bool bnd = yb || (!RAW && (Xn == 0 || Xn == gx - 1));
              double ukx = 0.0, umx = 0.0, uky = 0.0, umy = 0.0;
#pragma unroll
              for (int bs = 0; bs < S; ++bs)
                {
                  const double vx = bnd ? 0.0 : sm[L::vidx(2 * bs, rs, xl)];
                  const double vy = bnd ? 0.0 : sm[L::vidx(2 * bs + 1, rs, xl)];
                  if constexpr (DOX)
                    ukx = fma(kt[bs], vx, ukx);
                  umx = fma(mt[bs], vx, umx);
                  if constexpr (DOY)
                    uky = fma(kt[bs], vy, uky);
                  umy = fma(mt[bs], vy, umy);
                }
              if (coupled_here)
                {
                  if constexpr (DOX)
                    ukx = fma(-lva, sm[L::vidx(2 * S, rs, xl)], ukx);
                  if constexpr (DOY)
                    uky = fma(-lva, sm[L::vidx(2 * S + 1, rs, xl)], uky);
                }
              UKx[k] = ukx;
              UMx[k] = umx;
              UKy[k] = uky;
              UMy[k] = umy;
            }
#pragma unroll
          for (int i = 0; i < N1; ++i)
            {
              if constexpr (DOX)
                {
                  double s0 = 0, s1 = 0, s2 = 0;
#pragma unroll
                  for (int k = 0; k < N1; ++k)
                    {
                      const int o = i * N1 + k;
                      s0 = fma(P.xM[o], UKx[k], s0);
                      s0 = fma(P.xKa[o], UMx[k], s0);
                      s1 = fma(P.xM[o], UMx[k], s1);
                      s2 = fma(P.xC[o], UMy[k], s2);
                    }
#pragma unroll
                  for (int j = 0; j < N1; ++j)
                    {
                      const int o = j * N1 + l;
                      double v = Yx[i][j];
                      v = fma(P.yM[o], s0, v);
                      v = fma(P.yKa[o], s1, v);
                      v = fma(P.yCx[o], s2, v);
                      Yx[i][j] = v;
                    }
                }
              if constexpr (DOY)
                {
                  double s3 = 0, s4 = 0, s5 = 0;
#pragma unroll
                  for (int k = 0; k < N1; ++k)
                    {
                      const int o = i * N1 + k;
                      s3 = fma(P.xM[o], UKy[k], s3);
                      s3 = fma(P.xKb[o], UMy[k], s3);
                      s4 = fma(P.xM[o], UMy[k], s4);
                      s5 = fma(P.xCt[o], UMx[k], s5);
                    }
#pragma unroll
                  for (int j = 0; j < N1; ++j)
                    {
                      const int o = j * N1 + l;
                      double v = Yy[i][j];
                      v = fma(P.yM[o], s3, v);
                      v = fma(P.yKb[o], s4, v);
                      v = fma(P.yCy[o], s5, v);
                      Yy[i][j] = v;
                    }
                }
            }
          if constexpr (DOX)
            {
#pragma unroll
              for (int aa = 0; aa < PL; ++aa)
                {
                  double dp = 0, ep = 0;
#pragma unroll
                  for (int k = 0; k < N1; ++k)
                    {
                      dp = fma(P.xLc[aa * N1 + k], UMx[k], dp);
                      ep = fma(P.xLm[aa * N1 + k], UMy[k], ep);
                    }
#pragma unroll
                  for (int m = 0; m < NPM; ++m)
                    {
                      if (pdisc_mode_ax(R, m) != aa)
                        continue;
                      const int bm = pdisc_mode_ay(R, m);
                      Yp[m] = fma(P.yLm[bm * N1 + l], dp, Yp[m]);
                      Yp[m] = fma(P.yLc[bm * N1 + l], ep, Yp[m]);
                    }
                }
            }
        }
    }

  // ---- assemble shared nodes: x across lanes, y through the carry
#pragma unroll
  for (int j = 0; j < N1; ++j)
    {
      if constexpr (DOX)
        {
          const double lx = __shfl_up_sync(0xffffffffu, Yx[N1 - 1][j], 1);
          if (lane > 0)
            Yx[0][j] += lx;
        }
      if constexpr (DOY)
        {
          const double ly = __shfl_up_sync(0xffffffffu, Yy[N1 - 1][j], 1);
          if (lane > 0)
            Yy[0][j] += ly;
        }
    }
  if (add_carry)
#pragma unroll
    for (int i = 0; i < N1; ++i)
      {
        if constexpr (DOX)
          Yx[i][0] += carx[i];
        if constexpr (DOY)
          Yy[i][0] += cary[i];
      }
#pragma unroll
  for (int i = 0; i < N1; ++i)
    {
      if constexpr (DOX)
        carx[i] = Yx[i][N1 - 1];
      if constexpr (DOY)
        cary[i] = Yy[i][N1 - 1];
    }

  // ---- write owned outputs
  if (owner && write_row)
    {
      const int ixmax = (cx == P.nx - 1) ? p : p - 1;
      const int iymax = (cy == P.ny - 1) ? p : p - 1;
      const long long obase = n * isz + A * mv;
#pragma unroll
      for (int j = 0; j < N1; ++j)
        {
          if (j > iymax)
            continue;
          const int Yr = cy * p + j;
          const bool yb = (Yr == 0) || (Yr == gy - 1);
#pragma unroll
          for (int i = 0; i < N1; ++i)
            {
              if (i > ixmax)
                continue;
              const int X = cx * p + i;
              const long long node = static_cast<long long>(Yr) * gx + X;
              const bool cons = !RAW && (yb || X == 0 || X == gx - 1);
              if constexpr (DOX)
                {
                  // identity rows on constrained velocity dofs (st_operator.cpp:383-394)
                  double v = cons ? __ldg(x + obase + node) : Yx[i][j];
                  if (RESID)
                    v = __ldg(b + obase + node) - v;
                  y[obase + node] = v;
                }
              if constexpr (DOY)
                {
                  double v = cons ? __ldg(x + obase + nsc + node) : Yy[i][j];
                  if (RESID)
                    v = __ldg(b + obase + nsc + node) - v;
                  y[obase + nsc + node] = v;
                }
            }
        }
      if constexpr (DOX)
        {
          const long long pbase = n * isz + S * mv + A * mp + (static_cast<long long>(cy) * P.nx + cx) * NPM;
#pragma unroll
          for (int m = 0; m < NPM; ++m)
            y[pbase + m] = RESID ? __ldg(b + pbase + m) - Yp[m] : Yp[m];
        }
    }
}

/// COMPS = 2: 2S warps per block, one per (slot, component); COMPS = 1: S
/// warps, one per slot computing both components (large r).
template <int R, int S, int COMPS, bool RESID, bool RAW>
__global__ void __launch_bounds__(32 * S * COMPS, R == 2 ? kMinBlocksR2 : 1)
vmult_kernel(const LevelConsts P, const double *__restrict__ x, const double *__restrict__ b,
             double *__restrict__ y, const double *__restrict__ xprev0, int rows_per_seg, int coupled)
{
  using L = StripLayout<R, S>;
  constexpr int N1 = R + 2, p = R + 1, NPM = L::NPM;
  extern __shared__ __align__(16) double sm[];
  const int n = blockIdx.z;
  const int cx0 = blockIdx.x * kStrip - 1; // halo cell
  const long long isz = P.isz, mv = P.mv, mp = P.mp, nsc = P.nsc;
  const int gx = P.gx, gy = P.gy;
  const double *__restrict__ xn = x + n * isz;
  const double *__restrict__ vprev = nullptr;
  if (coupled)
    vprev = n > 0 ? x + (n - 1) * isz + (S - 1) * mv : xprev0;
  const bool coupled_here = vprev != nullptr;
  const int narr = coupled_here ? L::NARR : 2 * S;

  const int cy_begin = blockIdx.y * rows_per_seg;
  const int cy_end = min(P.ny, cy_begin + rows_per_seg);
  const int cy_first = max(cy_begin - 1, 0);
  const int X0 = cx0 * p;

  double carx[N1], cary[N1];
#pragma unroll
  for (int i = 0; i < N1; ++i)
    carx[i] = cary[i] = 0.0;

  // this warp's output slot / component (runtime: one shared code stream)
  const int wid = threadIdx.x >> 5;
  const int slot = COMPS == 2 ? wid >> 1 : wid;
  const int comp = COMPS == 2 ? wid & 1 : 2;
  double kt[S], mt[S], lva = 0.0;
#pragma unroll
  for (int bs = 0; bs < S; ++bs)
    kt[bs] = mt[bs] = 0.0;
#pragma unroll
  for (int aa = 0; aa < S; ++aa)
    if (slot == aa)
      {
#pragma unroll
        for (int bs = 0; bs < S; ++bs)
          {
            kt[bs] = P.Kt[aa * S + bs];
            mt[bs] = P.Mt[aa * S + bs];
          }
        lva = P.lv[aa];
      }

  // async staging of cell row `cyr` (rows r0..cy*p+p of every array, plus
  // the row's pressures) into the ring / pressure buffer
  auto stage = [&](int cyr, bool full) {
    const int r0 = full ? cyr * p : cyr * p + 1;
    const int nrows = cyr * p + p - r0 + 1;
    const int total = narr * nrows * L::RL;
    for (int e = threadIdx.x; e < total; e += blockDim.x)
      {
        const int xl = e % L::RL;
        const int t = e / L::RL;
        const int rr = t % nrows, arr = t / nrows;
        const int Yr = r0 + rr, X = X0 + xl;
        double *dst = sm + L::vidx(arr, Yr % L::NR, xl);
        if (X >= 0 && X < gx && Yr < gy)
          {
            const long long node = static_cast<long long>(Yr) * gx + X;
            const double *src = arr < 2 * S ? xn + (arr >> 1) * mv + (arr & 1) * nsc + node
                                            : vprev + (arr - 2 * S) * nsc + node;
            cp_async8(dst, src);
          }
        else
          *dst = 0.0;
      }
    double *pb = sm + L::VEL + (cyr & 1) * L::PRE;
    for (int e = threadIdx.x; e < S * 32 * NPM; e += blockDim.x)
      {
        const int m = e % NPM, t = e / NPM, c = t % 32, bs = t / 32;
        const int cx = cx0 + c;
        if (cx >= 0 && cx < P.nx)
          cp_async8(pb + e, xn + S * mv + bs * mp + (static_cast<long long>(cyr) * P.nx + cx) * NPM + m);
        else
          pb[e] = 0.0;
      }
    cp_async_commit();
  };

  stage(cy_first, true);
  for (int cy = cy_first; cy < cy_end; ++cy)
    {
      if (cy + 1 < cy_end)
        {
          stage(cy + 1, false);
          cp_async_wait<1>(); // row cy landed, row cy+1 in flight
        }
      else
        cp_async_wait<0>();
      __syncthreads();
      if (COMPS == 1)
        vmult_row<R, S, 2, RESID, RAW>(P, sm, x, b, y, n, cx0, cy, cy >= cy_begin, cy > cy_first, coupled_here,
                                       carx, cary, slot, kt, mt, lva);
      else if (comp == 0)
        vmult_row<R, S, 0, RESID, RAW>(P, sm, x, b, y, n, cx0, cy, cy >= cy_begin, cy > cy_first, coupled_here,
                                       carx, cary, slot, kt, mt, lva);
      else
        vmult_row<R, S, 1, RESID, RAW>(P, sm, x, b, y, n, cx0, cy, cy >= cy_begin, cy > cy_first, coupled_here,
                                       carx, cary, slot, kt, mt, lva);
      __syncthreads();
    }
}

template <int R, int S>
cudaError_t
launch_rs(const LevelConsts &P, const double *x, const double *b, double *y, int n_intervals, const double *xprev0,
          int coupled, int mode, cudaStream_t stream)
{
  constexpr int COMPS = kSplitComps && R <= 2 ? 2 : 1;
  using L = StripLayout<R, S>;
  static bool attr = false;
  if (!attr)
    {
      cudaFuncSetAttribute(vmult_kernel<R, S, COMPS, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           L::BYTES);
      cudaFuncSetAttribute(vmult_kernel<R, S, COMPS, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           L::BYTES);
      cudaFuncSetAttribute(vmult_kernel<R, S, COMPS, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           L::BYTES);
      attr = true;
    }
  const int strips = (P.nx + kStrip - 1) / kStrip;
  // Row segments: enough blocks to fill 148 SMs several times, >= 8 rows
  // each so the recomputed halo row stays small.
  int segs = 1;
  const long long base_blocks = static_cast<long long>(strips) * n_intervals;
  while (base_blocks * segs < 148 * 8 && P.ny / (segs * 2) >= 8)
    segs *= 2;
  const int rows = (P.ny + segs - 1) / segs;
  dim3 grid(strips, (P.ny + rows - 1) / rows, n_intervals);
  dim3 block(32 * S * COMPS);
  switch (mode)
    {
      case 0:
        vmult_kernel<R, S, COMPS, false, false><<<grid, block, L::BYTES, stream>>>(P, x, b, y, xprev0, rows, coupled);
        break;
      case 1:
        vmult_kernel<R, S, COMPS, true, false><<<grid, block, L::BYTES, stream>>>(P, x, b, y, xprev0, rows, coupled);
        break;
      default:
        vmult_kernel<R, S, COMPS, false, true><<<grid, block, L::BYTES, stream>>>(P, x, b, y, xprev0, rows, coupled);
        break;
    }
  return cudaGetLastError();
}

} // namespace vmult_detail
} // namespace stmg_b200
