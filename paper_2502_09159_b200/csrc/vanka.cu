// Additive space-time Vanka smoother on B200 (sm_100a), FP64.
//
// Replaces VankaSmoother::apply_additive / smooth_step (vanka.cpp:196-233):
//   u <- u + omega * sum_T R_T^T w_T (R_T S R_T^T)^{-1} R_T r
// for cell or vertex-star patches, over one interval or N intervals at once
// (the local inverses are shared by all intervals: uniform tau).
//
// Design:
//  * Patches of a Cartesian level fall into <= 25 congruence classes; the
//    dense inverse of each class is computed once at setup (host) and staged
//    in shared memory by every block that works on that class.
//  * The patch solves of a block form a small GEMM: Z = A^{-1} [r_T1 ... r_TC]
//    over C columns = (patch, interval) pairs, evaluated from shared memory
//    with double2 loads along the contraction.
//  * Scatter: patches are coloured (2x2 colours for cells, 3x3 for vertex
//    stars) so that one launch never touches a dof twice: read-modify-write
//    of u with no atomics, deterministic results.
#include <algorithm>
#include <cstdlib>
#include "kernels.hpp"
#include "st3d.hpp"

#include <cooperative_groups.h>
#include <cuda_runtime.h>

namespace stmg_b200
{

namespace
{
constexpr int kVankaCols = 32;
constexpr int kVankaThreads = 256;

__global__ void __launch_bounds__(kVankaThreads)
vanka_kernel(const DevPatchClass *__restrict__ classes, const VankaBatch *__restrict__ batches,
             const long long *__restrict__ vel_anchor, const long long *__restrict__ pre_anchor,
             const double *__restrict__ r, double *__restrict__ u, long long isz, double omega,
             int inverse_in_smem)
{
  extern __shared__ __align__(16) double smem[];
  const VankaBatch bt = batches[blockIdx.x];
  const DevPatchClass pc = classes[bt.cls];
  const int n = blockIdx.y;
  const int nt = pc.n_t;
  const int ntp = (nt + 1) & ~1; // even row pitch for double2 loads
  double *Ainv = smem;                                            // nt x ntp
  double *Rt = smem + (inverse_in_smem ? nt * ntp : 0);           // ntp x kVankaCols
  const int tid = threadIdx.x;

  if (inverse_in_smem)
    for (int idx = tid; idx < nt * ntp; idx += blockDim.x)
      {
        const int i = idx / ntp, j = idx - i * ntp;
        Ainv[idx] = j < nt ? __ldg(pc.inverse + i * nt + j) : 0.0;
      }
  // gather R_T r for the batch's patches (column c = patch)
  const long long ibase = n * isz;
  for (int idx = tid; idx < ntp * kVankaCols; idx += blockDim.x)
    {
      const int j = idx / kVankaCols, c = idx - j * kVankaCols;
      double v = 0.0;
      if (j < nt && c < bt.count)
        {
          const long long anchor = j < pc.n_vel ? vel_anchor[bt.first + c] : pre_anchor[bt.first + c];
          v = __ldg(r + ibase + anchor + pc.rel[j]);
        }
      Rt[idx] = v;
    }
  __syncthreads();

  // Z = Ainv * Rt: lane = column, warp strides over rows.
  const int c = tid & 31;
  const int warp = tid >> 5, nwarps = blockDim.x >> 5;
  if (c < bt.count)
    {
      const long long va = vel_anchor[bt.first + c], pa = pre_anchor[bt.first + c];
      for (int i0 = warp; i0 < nt; i0 += 2 * nwarps)
        {
          const int i1 = i0 + nwarps;
          const bool two = i1 < nt;
          double z0 = 0.0, z1 = 0.0;
          if (inverse_in_smem)
            {
              const double2 *a0 = reinterpret_cast<const double2 *>(Ainv + i0 * ntp);
              const double2 *a1 = reinterpret_cast<const double2 *>(Ainv + (two ? i1 : i0) * ntp);
#pragma unroll 4
              for (int jj = 0; jj < ntp / 2; ++jj)
                {
                  const double r0 = Rt[(2 * jj) * kVankaCols + c], r1 = Rt[(2 * jj + 1) * kVankaCols + c];
                  const double2 x0 = a0[jj], x1 = a1[jj];
                  z0 = fma(x0.x, r0, z0);
                  z0 = fma(x0.y, r1, z0);
                  z1 = fma(x1.x, r0, z1);
                  z1 = fma(x1.y, r1, z1);
                }
            }
          else
            {
              const double *a0 = pc.inverse + static_cast<long long>(i0) * nt;
              const double *a1 = pc.inverse + static_cast<long long>(two ? i1 : i0) * nt;
              for (int j = 0; j < nt; ++j)
                {
                  const double rj = Rt[j * kVankaCols + c];
                  z0 = fma(__ldg(a0 + j), rj, z0);
                  z1 = fma(__ldg(a1 + j), rj, z1);
                }
            }
          {
            const long long addr = ibase + (i0 < pc.n_vel ? va : pa) + pc.rel[i0];
            u[addr] += omega * pc.weight[i0] * z0;
          }
          if (two)
            {
              const long long addr = ibase + (i1 < pc.n_vel ? va : pa) + pc.rel[i1];
              u[addr] += omega * pc.weight[i1] * z1;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// DMMA path (n_T <= 128): the class inverse lives in registers as FP64 tensor
// core A-fragments (warp w owns rows 8w..8w+7), residual columns are staged
// in shared memory as B-fragments, Z = A^{-1} R runs on mma.m8n8k4.f64.
// Gather of tile t+1 and the read half of the scatter of tile t are issued
// before the MMAs of tile t (register prefetch), so their latency overlaps
// the tensor-core work.
constexpr int kDThreads = 512;            // 16 warps
constexpr int kDRows = 128;               // max n_T
#ifndef STMG_VANKA_COLS
#define STMG_VANKA_COLS 16
#endif
constexpr int kDCols = STMG_VANKA_COLS;   // columns per tile
constexpr int kDRLd = 36;                 // R tile pitch (doubles): conflict-free B-fragment loads
constexpr int kDZLd = 33;                 // Z tile pitch
constexpr int kDPer = kDRows * kDCols / kDThreads; // elements per thread per tile (8)
constexpr int kDGroup = 16;               // intervals per block
constexpr long long kNoCol = -(1ll << 62); // column-base sentinel (anchors may be negative)

__device__ __forceinline__ void
dmma_8x8x4(double (&d)[2], double a, double b)
{
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

#ifndef STMG_SPLIT_MINB
#define STMG_SPLIT_MINB 1
#endif
#ifndef STMG_V176_COLS
#define STMG_V176_COLS 16
#endif
// 176-row split, opt-in: the 2 CTAs of a row split form a cluster and each
// gathers half of the R rows into both CTAs' tiles (distributed shared
// memory). No spills, but the two cluster barriers per tile cost more than
// the halved gather saves (C3: 10.8 vs 13.1 TF/s), so it is off.
#ifndef STMG_V176_CLUSTER
#define STMG_V176_CLUSTER 0
#endif
template <int KS, int ROWS = kDRows, int TPW = 1, int COLS = kDCols, int SPLIT = 1>
__global__ void __launch_bounds__(ROWS / SPLIT / 8 / TPW * 32, SPLIT == 1 ? 1 : STMG_SPLIT_MINB)
vanka_dmma_kernel(const DevPatchClass *__restrict__ classes, const VankaBatch *__restrict__ items,
                  const int *__restrict__ item_ptr, const long long *__restrict__ vel_anchor,
                  const long long *__restrict__ pre_anchor, const double *__restrict__ r, double *__restrict__ u,
                  long long isz, int n_intervals, double omega, int group)
{
  // ROWS rows of the patch matrix, split over SPLIT CTAs (blockIdx.z): a CTA
  // computes and scatters OROWS rows but gathers all ROWS rows of R (the
  // contraction dimension); warp w owns the TPW 8-row tiles w + j * NW
  constexpr int kDCols = COLS;
  static_assert(COLS <= kDZLd && COLS <= kDRLd, "tile columns must fit the R / Z pitches");
  constexpr int OROWS = ROWS / SPLIT;
  constexpr bool CL = SPLIT > 1 && STMG_V176_CLUSTER; // cluster of the SPLIT CTAs shares the R gather
  constexpr int kDRows = ROWS, kDThreads = OROWS / 8 / TPW * 32;
  constexpr int kDPer = (CL ? OROWS : kDRows) * kDCols / kDThreads; // R rows gathered per thread
  constexpr int kDPerS = OROWS * kDCols / kDThreads;
  constexpr int NW = kDThreads / 32;
  const int row0 = SPLIT > 1 ? static_cast<int>(blockIdx.z) * OROWS : 0;
  extern __shared__ __align__(16) double dsm[];
  double *Rs = dsm;                                                 // kDRows x kDRLd
  double *Rp = Rs; // the peer CTA's tile (CL)
  if constexpr (CL)
    Rp = cooperative_groups::this_cluster().map_shared_rank(Rs, static_cast<int>(blockIdx.z) ^ 1);
  const int grow0 = CL ? row0 : 0; // first R row this CTA gathers
  auto bar = [&]() {
    if constexpr (CL)
      cooperative_groups::this_cluster().sync();
    else
      __syncthreads();
  };
  double *Zs = Rs + kDRows * kDRLd;                                 // OROWS x kDZLd
  double *w_s = Zs + OROWS * kDZLd;                                 // OROWS
  long long *cb = reinterpret_cast<long long *>(w_s + OROWS);      // [3][2][kDCols] column bases

  const int n0 = blockIdx.y * group;
  const int ng = min(group, n_intervals - n0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = tid % kDCols;        // column of this thread in every tile
  const int ibase = tid / kDCols;    // first row of this thread (rows ibase + q * kDThreads / kDCols)
  const int it0 = item_ptr ? item_ptr[blockIdx.x] : blockIdx.x;
  const int it1 = item_ptr ? item_ptr[blockIdx.x + 1] : blockIdx.x + 1;

  int loaded = -1, nt = 0, nvel = 0;
  double afr[TPW][KS];
  long long relq[kDPer], relS[kDPerS];
  bool velq[kDPer], validq[kDPer], velS[kDPerS], validS[kDPerS];

  // Items run in order; consecutive items of one block are separated by
  // block barriers (every tile ends with one), which is what makes the
  // super-cell sub-phases conflict-free.
  for (int it = it0; it < it1; ++it)
    {
      const VankaBatch bt = items[it];
      if (bt.cls != loaded)
        {
          const DevPatchClass pc = classes[bt.cls];
          nt = pc.n_t;
          nvel = pc.n_vel;
          for (int i = tid; i < OROWS; i += kDThreads)
            w_s[i] = row0 + i < nt ? omega * pc.weight[row0 + i] : 0.0;
#pragma unroll
          for (int tw = 0; tw < TPW; ++tw)
            {
              const int arow = row0 + 8 * (warp + tw * NW) + (lane >> 2);
              // unpredicated clamped loads first (all in flight), mask after
              const double *ap = pc.inverse + (arow < nt ? arow : 0) * nt;
#pragma unroll
              for (int kk = 0; kk < KS; ++kk)
                afr[tw][kk] = __ldg(ap + min(4 * kk + (lane & 3), nt - 1));
#pragma unroll
              for (int kk = 0; kk < KS; ++kk)
                if (!(arow < nt && 4 * kk + (lane & 3) < nt))
                  afr[tw][kk] = 0.0;
            }
#pragma unroll
          for (int q = 0; q < kDPer; ++q)
            {
              const int i = grow0 + ibase + q * (kDThreads / kDCols);
              validq[q] = i < nt;
              velq[q] = i < nvel;
              relq[q] = i < nt ? pc.rel[i] : 0;
            }
#pragma unroll
          for (int q = 0; q < kDPerS; ++q)
            {
              const int i = row0 + ibase + q * (kDThreads / kDCols);
              validS[q] = i < nt;
              velS[q] = i < nvel;
              relS[q] = i < nt ? pc.rel[i] : 0;
            }
          loaded = bt.cls;
        }
      const int ncols = bt.count * ng;
      const int ntiles = (ncols + kDCols - 1) / kDCols;

      // column bases of tile t: interval base + velocity / pressure anchor
      auto column_bases = [&](int t) {
        if (tid < kDCols && t < ntiles)
          {
            const int j = t * kDCols + tid;
            long long vb = kNoCol, pb = kNoCol;
            if (j < ncols)
              {
                const int patch = j / ng, n = n0 + j - patch * ng;
                vb = n * isz + __ldg(vel_anchor + bt.first + patch);
                pb = n * isz + __ldg(pre_anchor + bt.first + patch);
              }
            cb[(t % 3) * 2 * kDCols + tid] = vb;
            cb[(t % 3) * 2 * kDCols + kDCols + tid] = pb;
          }
      };
      column_bases(0);
      column_bases(1);
      __syncthreads();

      double g[kDPer];
      {
        const long long vb = cb[c], pb = cb[kDCols + c];
#pragma unroll
        for (int q = 0; q < kDPer; ++q)
          {
            const long long base = velq[q] ? vb : pb;
            g[q] = (validq[q] && base != kNoCol) ? __ldg(r + base + relq[q]) : 0.0;
          }
#pragma unroll
        for (int q = 0; q < kDPer; ++q)
          {
            const int i = (grow0 + ibase + q * (kDThreads / kDCols)) * kDRLd + c;
            Rs[i] = g[q];
            if constexpr (CL)
              Rp[i] = g[q];
          }
      }
      bar();

      for (int t = 0; t < ntiles; ++t)
        {
          const long long *cbt = cb + (t % 3) * 2 * kDCols;
          const long long vb = cbt[c], pb = cbt[kDCols + c];
          // prefetch: old u of this tile and the residual of the next tile
          double uo[kDPerS];
#pragma unroll
          for (int q = 0; q < kDPerS; ++q)
            {
              const long long base = velS[q] ? vb : pb;
              uo[q] = (validS[q] && base != kNoCol) ? u[base + relS[q]] : 0.0;
            }
          if (t + 1 < ntiles)
            {
              const long long *cbn = cb + ((t + 1) % 3) * 2 * kDCols;
              const long long nvb = cbn[c], npb = cbn[kDCols + c];
#pragma unroll
              for (int q = 0; q < kDPer; ++q)
                {
                  const long long base = velq[q] ? nvb : npb;
                  g[q] = (validq[q] && base != kNoCol) ? __ldg(r + base + relq[q]) : 0.0;
                }
            }
          // Z = A^{-1} R on the FP64 tensor path
#pragma unroll
          for (int tw = 0; tw < TPW; ++tw)
            if (row0 + 8 * (warp + tw * NW) < nt)
              {
                double acc[kDCols / 8][2];
#pragma unroll
                for (int ct = 0; ct < kDCols / 8; ++ct)
                  acc[ct][0] = acc[ct][1] = 0.0;
                const double *bbase = Rs + (lane & 3) * kDRLd + (lane >> 2);
#pragma unroll
                for (int kk = 0; kk < KS; ++kk)
                  {
                    const double *brow = bbase + 4 * kk * kDRLd;
#pragma unroll
                    for (int ct = 0; ct < kDCols / 8; ++ct)
                      dmma_8x8x4(acc[ct], afr[tw][kk], brow[8 * ct]);
                  }
                const int row = 8 * (warp + tw * NW) + (lane >> 2);
                const double wr = w_s[row];
#pragma unroll
                for (int ct = 0; ct < kDCols / 8; ++ct)
                  {
                    const int col = 8 * ct + 2 * (lane & 3);
                    Zs[row * kDZLd + col] = acc[ct][0] * wr;
                    Zs[row * kDZLd + col + 1] = acc[ct][1] * wr;
                  }
              }
          column_bases(t + 2);
          bar(); // CL: the peer's MMAs are done with its tile before this CTA writes into it
#pragma unroll
          for (int q = 0; q < kDPerS; ++q)
            {
              const long long base = velS[q] ? vb : pb;
              if (validS[q] && base != kNoCol)
                u[base + relS[q]] = uo[q] + Zs[(ibase + q * (kDThreads / kDCols)) * kDZLd + c];
            }
          if (t + 1 < ntiles)
#pragma unroll
            for (int q = 0; q < kDPer; ++q)
              {
                const int i = (grow0 + ibase + q * (kDThreads / kDCols)) * kDRLd + c;
                Rs[i] = g[q];
                if constexpr (CL)
                  Rp[i] = g[q];
              }
          bar();
        }
    }
}

// ---------------------------------------------------------------------------
// Large patches (176 < n_T <= 790, e.g. 3D Q3 cells with DG(2): n_T = 606):
// Z = A^{-1} R on the FP64 tensor path with the inverse streamed from L2
// (a class inverse is 2.9 MB; the <= 27 Cartesian classes of a level stay
// L2-resident) as A-fragments, one 32-column tile of R (patch, interval)
// staged in shared memory for the whole contraction, and the weighted result
// scattered straight from the accumulators (patches of one launch share no
// dof, so the adds never collide).
constexpr int kBThreads = 512; // 16 warps
#ifndef STMG_BIG_COLS
#define STMG_BIG_COLS 32
#endif
constexpr int kBCols = STMG_BIG_COLS; // columns per tile
constexpr int kBLd = 36;       // R pitch: conflict-free B-fragment loads
constexpr int kBMaxTiles = 7;  // row tiles per warp: 16 * 7 * 8 = 896 rows
constexpr int kBGroup = 16;    // intervals per block

template <int TPW>
__global__ void __launch_bounds__(kBThreads, kBCols == 32 ? 1 : 2)
vanka_big_kernel(const DevPatchClass *__restrict__ classes, const VankaBatch *__restrict__ batches,
                 const long long *__restrict__ vel_anchor, const long long *__restrict__ pre_anchor,
                 const double *__restrict__ r, double *__restrict__ u, long long isz, int n_intervals, double omega,
                 int group)
{
  extern __shared__ __align__(16) double bsm[];
  const VankaBatch bt = batches[blockIdx.x];
  const DevPatchClass pc = classes[bt.cls];
  const int nt = pc.n_t, nvel = pc.n_vel;
  const int ks = (nt + 3) / 4;
  double *Rs = bsm;                                   // (4 ks) x kBLd
  long long *cvb = reinterpret_cast<long long *>(Rs + 4 * ks * kBLd); // velocity column bases
  long long *cpb = cvb + kBCols;                                      // pressure column bases
  const int n0 = blockIdx.y * group;
  const int ng = min(group, n_intervals - n0);
  const int ncols = bt.count * ng;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rtiles = (nt + 7) / 8;
  for (int c0 = 0; c0 < ncols; c0 += kBCols)
    {
      if (tid < kBCols)
        {
          const int j = c0 + tid;
          long long vb = 0, pb = 0;
          if (j < ncols)
            {
              const int patch = j / ng, n = n0 + j - patch * ng;
              vb = n * isz + __ldg(vel_anchor + bt.first + patch);
              pb = n * isz + __ldg(pre_anchor + bt.first + patch);
            }
          cvb[tid] = vb;
          cpb[tid] = pb;
        }
      __syncthreads();
      // gather R (rows >= nt and columns >= ncols are zero)
      for (int e = tid; e < 4 * ks * kBCols; e += kBThreads)
        {
          const int row = e / kBCols, c = e - row * kBCols;
          double v = 0.0;
          if (row < nt && c0 + c < ncols)
            v = __ldg(r + (row < nvel ? cvb[c] : cpb[c]) + __ldg(pc.rel + row));
          Rs[row * kBLd + c] = v;
        }
      __syncthreads();
      double acc[TPW][kBCols / 8][2];
#pragma unroll
      for (int t = 0; t < TPW; ++t)
#pragma unroll
        for (int ct = 0; ct < kBCols / 8; ++ct)
          acc[t][ct][0] = acc[t][ct][1] = 0.0;
      const double *bbase = Rs + (lane & 3) * kBLd + (lane >> 2);
      // A-fragments come from L2: a 3-deep register ring keeps the loads two
      // k-steps ahead of the DMMAs that consume them
      auto load_a = [&](int kk, double (&dst)[TPW]) {
        const int col = 4 * kk + (lane & 3);
#pragma unroll
        for (int t = 0; t < TPW; ++t)
          {
            const int row = 8 * (warp + 16 * t) + (lane >> 2);
            dst[t] = (kk < ks && row < nt && col < nt) ? __ldg(pc.inverse + static_cast<long long>(row) * nt + col)
                                                       : 0.0;
          }
      };
      double ring[3][TPW];
      load_a(0, ring[0]);
      load_a(1, ring[1]);
      for (int kk0 = 0; kk0 < ks; kk0 += 3)
        {
#pragma unroll
          for (int u = 0; u < 3; ++u)
            {
              const int kk = kk0 + u;
              load_a(kk + 2, ring[(u + 2) % 3]);
              if (kk < ks)
                {
                  double bf[kBCols / 8];
#pragma unroll
                  for (int ct = 0; ct < kBCols / 8; ++ct)
                    bf[ct] = bbase[4 * kk * kBLd + 8 * ct];
#pragma unroll
                  for (int t = 0; t < TPW; ++t)
                    if (warp + 16 * t < rtiles)
#pragma unroll
                      for (int ct = 0; ct < kBCols / 8; ++ct)
                        dmma_8x8x4(acc[t][ct], ring[u][t], bf[ct]);
                }
            }
        }
      // scatter u += omega w Z from the accumulators
#pragma unroll
      for (int t = 0; t < TPW; ++t)
        {
          const int rt = warp + 16 * t;
          const int row = 8 * rt + (lane >> 2);
          if (rt < rtiles && row < nt)
            {
              const double wr = omega * __ldg(pc.weight + row);
              const long long rel = __ldg(pc.rel + row);
              const bool vel = row < nvel;
#pragma unroll
              for (int ct = 0; ct < kBCols / 8; ++ct)
#pragma unroll
                for (int h = 0; h < 2; ++h)
                  {
                    const int c = 8 * ct + 2 * (lane & 3) + h;
                    if (c0 + c < ncols)
                      atomicAdd(u + (vel ? cvb[c] : cpb[c]) + rel, wr * acc[t][ct][h]);
                  }
            }
        }
      __syncthreads();
    }
}

// ---------------------------------------------------------------- factored big
// Time-diagonalised cell patches (st3d.hpp Fac3Params; C5: n_T = 606 as one
// 202-row block for the real eigenvalue of M_t^{-1} K_t and one 404-row block
// for the complex pair): 0.56x the inverse bytes and DMMA work of the dense
// 606 x 606 inverse. One CTA = one cell patch x <= 16 intervals:
//   gather R (patch order) -> T = (W (x) I) R in factored order -> per block
//   b, Y_b = B_b^{-1} T_b on the FP64 tensor path -> Z = (V (x) I) Y, valence
//   weights, red.add (the patches of one colour share no dof).
// The blocks are stored column-major (patch3_gpu.cu writes them transposed),
// so 8 consecutive columns of B_b^{-1} -- two DMMA k-steps for every row tile
// -- are one contiguous run: the TMA engine streams them (cp.async.bulk, one
// issuing thread) through a 4-slot shared-memory ring with full / empty
// mbarriers, while the 16 warps run the DMMAs of the slot in front. Each
// warp keeps the accumulators of its row tiles (tiles w, w + 16, ... of each
// block) over the whole stream. The blocks are read once per 16 intervals,
// so the kernel is bound by this stream (HBM).
#ifndef STMG_FAC_L2AHEAD
#define STMG_FAC_L2AHEAD 0 // >0: L2 prefetch of the chunk this far ahead (measured: no gain)
#endif
#ifndef STMG_FAC_REGSCATTER
#define STMG_FAC_REGSCATTER 1
#endif
#ifndef STMG_FAC_WARP_ARRIVE
#define STMG_FAC_WARP_ARRIVE 1
#endif
#ifndef STMG_FAC_CHUNKCOLS
#define STMG_FAC_CHUNKCOLS 8 // u-columns of a pair block per ring slot (a multiple of 4)
#endif
#ifndef STMG_FAC_SLOTS
#define STMG_FAC_SLOTS 3 // measured with the producer in warp 15: 2 / 3 / 4 / 5 slots 12.84 / 11.46 / 11.60 / 12.13 ms (the smaller ring leaves L1 to the gather)
#endif
#ifndef STMG_FAC_SWZ
#define STMG_FAC_SWZ 0
#endif
// T / Y tile: 16 interval columns per row, pitch 20 (conflict-free DMMA
// B-fragment loads). STMG_FAC_SWZ=1: pitch 16 with the column XORed by 8 on
// odd rows (also two wavefronts), which frees shared memory for a fifth ring
// slot: measured 15.98 ms (5 slots) / 16.55 ms (4 slots) against 15.97 ms,
// so neither the bytes in flight nor the pitch limit the block stream.
constexpr int kFCols = 16, kFLd = STMG_FAC_SWZ ? 16 : 20, kFThreads = 512, kFSlots = STMG_FAC_SLOTS,
              kFChunkCols = STMG_FAC_CHUNKCOLS;
#ifndef STMG_FAC_REALCOLS
#define STMG_FAC_REALCOLS (2 * STMG_FAC_CHUNKCOLS)
#endif
// a real-eigenvalue block has half the rows of a pair block: its chunks take
// twice the columns, so both fill a ring slot and the real block needs half
// the hand-offs (its chunks carry only 8 DMMAs per warp and 8 columns)
constexpr int kFRealCols = STMG_FAC_REALCOLS;
__device__ __forceinline__ int
tsw(int row, int col)
{
  return row * kFLd + (STMG_FAC_SWZ ? (col ^ ((row & 1) << 3)) : col);
}
constexpr int kFTiles = 2; // row tiles per warp and block: n_s <= 16 * 2 * 8 = 256 spatial patch dofs

__device__ __forceinline__ unsigned
f_smem(const void *p)
{
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// T / Y rows: eigen-component i of spatial patch dof j at row i * nsp + j,
// nsp = n_s rounded up to 8 with zero rows, so the k-steps of a block's last
// chunk read zeros past n_s and no DMMA operand needs a predicate (the ring
// slots only ever hold finite inverse entries).
__host__ __device__ __forceinline__ int
f_nsp(int ns)
{
  return (ns + kFRealCols - 1) / kFRealCols * kFRealCols; // a real block's last chunk spans kFRealCols T rows
}

// Real-eigenvalue block: one chunk = 8 columns of B^{-1} (column-major, m
// rows each); tile t of the warp reads rows abase[t] (lane's column folded
// in). Rows past n_s read neighbouring ring data and are never written out.
template <int NT>
__device__ __forceinline__ void
fac_real_chunk(double (&acc)[kFTiles][2][2], const double *__restrict__ A, const double *__restrict__ Ts, int m,
               int trow, const int (&abase)[kFTiles], int lane)
{
#pragma unroll
  for (int kk = 0; kk < kFRealCols / 4; ++kk)
    {
      const int kr = trow + 4 * kk + (lane & 3);
      const double b0 = Ts[tsw(kr, lane >> 2)], b1 = Ts[tsw(kr, (lane >> 2) + 8)];
      double a[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t)
        a[t] = A[abase[t] + 4 * kk * m];
#pragma unroll
      for (int t = 0; t < NT; ++t)
        {
          dmma_8x8x4(acc[t][0], a[t], b0);
          dmma_8x8x4(acc[t][1], a[t], b1);
        }
    }
}

// Complex-pair block [[X, bM], [-bM, X]] = real form of Z = X - i b M. Its
// inverse is the real form [[P, -Q], [Q, P]] of Z^{-1} = P + iQ, so the
// u-columns [P; Q] alone (half the block) give
//   Y_u = P T_u - Q T_v,   Y_v = Q T_u + P T_v.
// One chunk = 8 u-columns (2 n_s rows each, stored order); tile t of the warp
// owns natural row r of both halves: P row at abu[t], Q row at abv[t].
template <int NT>
__device__ __forceinline__ void
fac_pair_chunk(double (&acc)[kFTiles][2][2][2], const double *__restrict__ A, const double *__restrict__ Ts, int m1,
               int tu, int tv, const int (&abu)[kFTiles], const int (&abv)[kFTiles], int lane)
{
#pragma unroll
  for (int kk = 0; kk < kFChunkCols / 4; ++kk)
    {
      const int kr = 4 * kk + (lane & 3);
      const double bu0 = Ts[tsw(tu + kr, lane >> 2)], bu1 = Ts[tsw(tu + kr, (lane >> 2) + 8)];
      const double bv0 = Ts[tsw(tv + kr, lane >> 2)], bv1 = Ts[tsw(tv + kr, (lane >> 2) + 8)];
      const double nv0 = -bv0, nv1 = -bv1;
      double au[NT], av[NT];
#pragma unroll
      for (int t = 0; t < NT; ++t)
        {
          au[t] = A[abu[t] + 4 * kk * m1];
          av[t] = A[abv[t] + 4 * kk * m1];
        }
#pragma unroll
      for (int t = 0; t < NT; ++t)
        {
          dmma_8x8x4(acc[t][0][0], au[t], bu0);
          dmma_8x8x4(acc[t][0][1], au[t], bu1);
          dmma_8x8x4(acc[t][1][0], av[t], bu0);
          dmma_8x8x4(acc[t][1][1], av[t], bu1);
        }
#pragma unroll
      for (int t = 0; t < NT; ++t)
        {
          dmma_8x8x4(acc[t][0][0], av[t], nv0);
          dmma_8x8x4(acc[t][0][1], av[t], nv1);
          dmma_8x8x4(acc[t][1][0], au[t], bv0);
          dmma_8x8x4(acc[t][1][1], au[t], bv1);
        }
    }
}

// Per-patch constants of the stream (the blocks of one cell patch). Block b
// streams nch[b] chunks of kFChunkCols columns, each column m[b] doubles.
struct FacItem
{
  const double *inv; // column-major blocks, block 1 at inv + moff1
  int nt, nvel, ns, nvs, moff1;
  int nch[2], m[2];
};

__device__ __forceinline__ FacItem
fac_item(const DevPatchClass &pc, const Fac3Params &F)
{
  FacItem it;
  it.inv = pc.fac_inv;
  it.nt = pc.n_t;
  it.nvel = pc.n_vel;
  it.ns = pc.n_t / F.S;
  it.nvs = pc.n_vel / F.S;
#pragma unroll
  for (int b = 0; b < 2; ++b)
    {
      it.m[b] = b < F.nb ? F.sz[b] * it.ns : 0;
      const int cc = F.sz[b] == 1 ? kFRealCols : kFChunkCols;
      it.nch[b] = b < F.nb ? (it.ns + cc - 1) / cc : 0; // pair: the n_s u-columns only
    }
  it.moff1 = (it.m[0] * it.m[0] + 8 + 1) / 2 * 2;
  return it;
}

// Stored row of natural row r (< n_s) of half h of a pair block: the setup
// (patch3_fac_assemble_kernel) orders a pair block [vel_u, vel_v, p_u, p_v].
__device__ __forceinline__ int
fac_pair_row(int h, int r, int nvs, int nps)
{
  return r < nvs ? h * nvs + r : 2 * nvs + h * nps + (r - nvs);
}

// Persistent: CTA x walks the batches x, x + gridDim.x, ... of the colour.
// The chunks of all its patches form ONE stream through the ring, so the
// TMA engine already pulls the next patch's first chunks while the warps
// write Y, scatter and gather the next patch.
template <int NW> // warps per CTA: 16 (one CTA per SM) or, for patches of <= 128 spatial dofs, 8 (two per SM)
__global__ void __launch_bounds__(NW * 32, 16 / NW)
vanka_big_fac_kernel(const DevPatchClass *__restrict__ classes, const VankaBatch *__restrict__ batches,
                     int n_batches, const long long *__restrict__ vel_anchor, const long long *__restrict__ pre_anchor,
                     const Fac3Params F, const double *__restrict__ r, double *__restrict__ u, long long isz,
                     int n_intervals, double omega, int group, int max_m, int max_nt)
{
  extern __shared__ __align__(16) double fsm[];
  constexpr int NTH = NW * 32;
  const int S = F.S;
  const int nrow_max = S * f_nsp(max_nt / S);
  const int slot_d = max(kFChunkCols * max_m, kFRealCols * (max_nt / S)); // doubles per ring slot
  double *Rs = fsm;                       // the chunk ring
  double *Ts = fsm + kFSlots * slot_d;    // nrow x kFLd: T, later Y
  double *s_w = Ts + nrow_max * kFLd;     // nt
  long long *cvb = reinterpret_cast<long long *>(s_w + (max_nt + 1) / 2 * 2);
  long long *cpb = cvb + kFCols;
  unsigned long long *full = reinterpret_cast<unsigned long long *>(cpb + kFCols), *empty = full + kFSlots;
  int *s_rel = reinterpret_cast<int *>(empty + kFSlots);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n0 = blockIdx.y * group, ng = min(group, n_intervals - n0);
  if (tid == 0)
    for (int q = 0; q < kFSlots; ++q)
      {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;\n" ::"r"(f_smem(full + q)));
        asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(f_smem(empty + q)),
                     "r"(STMG_FAC_WARP_ARRIVE ? NTH / 32 : NTH));
      }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  auto wait = [&](unsigned long long *bar, unsigned parity) {
    asm volatile("{\n .reg .pred p;\n FW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                 " @!p bra FW_%=;\n}\n" ::"r"(f_smem(bar)),
                 "r"(parity)
                 : "memory");
  };
  auto bulk = [&](double *dst, const double *src, unsigned bytes, unsigned long long *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   f_smem(dst)),
                 "l"(src), "r"(bytes), "r"(f_smem(bar))
                 : "memory");
  };
  // ---- producer: cursor over (batch, patch, chunk) of this CTA. It is lane 0
  // of warp 15, which owns one row tile per block where warps 0-9 own two: it
  // reaches the slot's empty barrier early, so the refill goes out the moment
  // the slowest warp releases the slot (as thread 0, on the busiest SM
  // sub-partition, the producer itself was the last to get there: C5 fine
  // sweep 12.3 -> 11.9 ms)
#ifndef STMG_FAC_PROD
#define STMG_FAC_PROD (NTH - 32)
#endif
  constexpr int PT = STMG_FAC_PROD;
  int p_bi = blockIdx.x, p_pi = 0, p_q = 0;
  unsigned p_g = 0; // chunks issued
  FacItem p_it{};
  bool p_has = p_bi < n_batches;
  if (tid == PT && p_has)
    p_it = fac_item(classes[batches[p_bi].cls], F);
  auto issue_next = [&]() {
    if (!p_has)
      return;
    const int slot = p_g % kFSlots;
    if (p_g >= kFSlots)
      wait(empty + slot, ((p_g / kFSlots) - 1) & 1); // the consumers released the slot's previous chunk
    const int b = p_q >= p_it.nch[0] ? 1 : 0;
    const int kc = b ? p_q - p_it.nch[0] : p_q;
    const int ccols = (b ? F.sz[1] : F.sz[0]) == 1 ? kFRealCols : kFChunkCols;
    const int m = b ? p_it.m[1] : p_it.m[0], k0 = ccols * kc, k1 = min(k0 + ccols, p_it.ns);
    const double *blk = p_it.inv + (b ? p_it.moff1 : 0);
    double *dst = Rs + slot * slot_d;
    if ((b ? F.sz[1] : F.sz[0]) == 1)
      {
        const unsigned bytes = static_cast<unsigned>(((k1 - k0) * m * sizeof(double) + 15) & ~size_t(15));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(f_smem(full + slot)),
                     "r"(bytes)
                     : "memory");
        bulk(dst, blk + static_cast<long long>(k0) * m, bytes, full + slot);
      }
    else
      {
        // u-columns k0..k1 of the pair block: velocity columns keep their
        // index, pressure column nvs + l sits at 2 nvs + l (m = 2 n_s is even:
        // every column starts 16-byte aligned)
        const int kv = min(k1, p_it.nvs);
        const unsigned cb = static_cast<unsigned>(m * sizeof(double));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(f_smem(full + slot)),
                     "r"((k1 - k0) * cb)
                     : "memory");
        if (kv > k0)
          bulk(dst, blk + static_cast<long long>(k0) * m, (kv - k0) * cb, full + slot);
        const int kp = max(k0, p_it.nvs);
        if (k1 > kp)
          bulk(dst + (kp - k0) * m, blk + static_cast<long long>(kp + p_it.nvs) * m, (k1 - kp) * cb, full + slot);
      }
    ++p_g;
    if (++p_q == p_it.nch[0] + p_it.nch[1])
      {
        p_q = 0;
        if (++p_pi == batches[p_bi].count)
          {
            p_pi = 0;
            p_bi += gridDim.x;
            p_has = p_bi < n_batches;
          }
        if (p_has)
          p_it = fac_item(classes[batches[p_bi].cls], F);
      }
  };
  if (tid == PT)
    for (int q = 0; q < kFSlots; ++q)
      issue_next();

  unsigned g = 0; // chunks consumed
  for (int bi = blockIdx.x; bi < n_batches; bi += gridDim.x)
    {
      const VankaBatch bt = batches[bi];
      const DevPatchClass pc = classes[bt.cls];
      const FacItem it = fac_item(pc, F);
      const int nt = it.nt, nvel = it.nvel, ns = it.ns, nvs = it.nvs, nps = ns - nvs, nsp = f_nsp(ns);
      auto prow = [&](int a, int j) { return j < nvs ? a * nvs + j : S * nvs + a * nps + (j - nvs); };
      const int nchunks = it.nch[0] + it.nch[1];
      // this warp's row tiles (same for every block: all blocks have n_s rows
      // per half) and their stored rows, lane's chunk column folded in
      const int rt = (ns + 7) / 8, nt_w = warp < rt ? (rt - warp + NW - 1) / NW : 0;
      int abr[kFTiles], abu[kFTiles], abv[kFTiles];
#pragma unroll
      for (int t = 0; t < kFTiles; ++t)
        {
          const int row = 8 * (warp + NW * t) + (lane >> 2);
          abr[t] = (lane & 3) * ns + row;
          abu[t] = (lane & 3) * (2 * ns) + fac_pair_row(0, row, nvs, nps);
          abv[t] = (lane & 3) * (2 * ns) + fac_pair_row(1, row, nvs, nps);
        }
      for (int pi = 0; pi < bt.count; ++pi)
        {
          const int patch = bt.first + pi;
          if (tid < kFCols)
            {
              const int n = n0 + tid;
              cvb[tid] = tid < ng ? n * isz + __ldg(vel_anchor + patch) : 0;
              cpb[tid] = tid < ng ? n * isz + __ldg(pre_anchor + patch) : 0;
            }
          for (int row = tid; row < nt; row += NTH)
            {
              s_rel[row] = static_cast<int>(__ldg(pc.rel + row));
              s_w[row] = omega * __ldg(pc.weight + row);
            }
          __syncthreads();
          // T = (W (x) I) R straight from the gather: thread (j, c) loads the S
          // slot values of spatial dof j in interval column c
#ifndef STMG_FAC_GBATCH
#define STMG_FAC_GBATCH 4
#endif
          // batches of GB elements per thread: all their loads are in flight
          // before the first W-mix (one latency per batch, not per element)
          constexpr int GB = STMG_FAC_GBATCH;
          for (int e0 = tid; e0 < nsp * kFCols; e0 += GB * NTH)
            {
              double rb[GB][kMaxS];
#pragma unroll
              for (int q = 0; q < GB; ++q)
                {
                  const int e = e0 + q * NTH;
                  const int c = e / nsp, j = e - c * nsp; // consecutive threads: consecutive dofs of a column
                  const bool ld = e < nsp * kFCols && j < ns && c < ng;
#pragma unroll
                  for (int b = 0; b < kMaxS; ++b)
                    {
                      const int row = (ld && b < S) ? prow(b, j) : 0;
                      rb[q][b] = (ld && b < S) ? __ldg(r + (row < nvel ? cvb[c] : cpb[c]) + s_rel[row]) : 0.0;
                    }
                }
#pragma unroll
              for (int q = 0; q < GB; ++q)
                {
                  const int e = e0 + q * NTH;
                  if (e >= nsp * kFCols)
                    break;
                  const int c = e / nsp, j = e - c * nsp;
                  for (int i = 0; i < S; ++i)
                    {
                      double t = 0.0;
#pragma unroll
                      for (int b = 0; b < kMaxS; ++b)
                        if (b < S)
                          t = fma(F.W[i * S + b], rb[q][b], t);
                      Ts[tsw(i * nsp + j, c)] = t; // rows j >= n_s: zeros
                    }
                }
            }
          __syncthreads();
          double accr[kFTiles][2][2], accp[kFTiles][2][2][2];
#pragma unroll
          for (int t = 0; t < kFTiles; ++t)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              {
                accr[t][h][0] = accr[t][h][1] = 0.0;
                accp[t][0][h][0] = accp[t][0][h][1] = accp[t][1][h][0] = accp[t][1][h][1] = 0.0;
              }
          for (int q = 0; q < nchunks; ++q, ++g)
            {
              const int slot = g % kFSlots;
              wait(full + slot, (g / kFSlots) & 1);
              const int b = q < it.nch[0] ? 0 : 1, kc = b ? q - it.nch[0] : q;
              const int trow = (b ? F.c0[1] : F.c0[0]) * nsp +
                               ((b ? F.sz[1] : F.sz[0]) == 1 ? kFRealCols : kFChunkCols) * kc; // T row of the chunk's first column
              const double *A = Rs + slot * slot_d;
              if ((b ? F.sz[1] : F.sz[0]) == 1)
                {
                  if (nt_w == 2)
                    fac_real_chunk<2>(accr, A, Ts, ns, trow, abr, lane);
                  else if (nt_w == 1)
                    fac_real_chunk<1>(accr, A, Ts, ns, trow, abr, lane);
                }
              else
                {
                  if (nt_w == 2)
                    fac_pair_chunk<2>(accp, A, Ts, 2 * ns, trow, trow + nsp, abu, abv, lane);
                  else if (nt_w == 1)
                    fac_pair_chunk<1>(accp, A, Ts, 2 * ns, trow, trow + nsp, abu, abv, lane);
                }
#if STMG_FAC_WARP_ARRIVE
              // one arrival per warp (its lanes' reads of the slot are ordered before it by the warp barrier)
              __syncwarp();
              if (lane == 0)
#endif
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(f_smem(empty + slot)) : "memory");
              if (tid == PT)
                issue_next(); // refills this slot -- possibly with the next patch's first chunks
            }
#if STMG_FAC_REGSCATTER
          // Z = (V (x) I) Y, weights and scatter straight from the accumulator
          // fragments: a thread holds all S eigen-components of its (row, column)
          // positions (the real block's row j and both halves of the pair
          // block's row j), so Y never goes through shared memory and no
          // barrier separates the stream from the scatter
          {
            int ir = -1, iu = -1;
#pragma unroll
            for (int b = 0; b < 2; ++b)
              if (b < F.nb)
                {
                  if (F.sz[b] == 1)
                    ir = F.c0[b];
                  else
                    iu = F.c0[b];
                }
#pragma unroll
            for (int t = 0; t < kFTiles; ++t)
              {
                const int j = 8 * (warp + NW * t) + (lane >> 2);
                if (t < nt_w && j < ns)
#pragma unroll
                  for (int ct = 0; ct < 2; ++ct)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                      {
                        const int col = 8 * ct + 2 * (lane & 3) + h;
                        if (col >= ng)
                          continue;
                        double y[kMaxS];
#pragma unroll
                        for (int i = 0; i < kMaxS; ++i)
                          y[i] = i == ir ? accr[t][ct][h]
                                         : (i == iu ? accp[t][0][ct][h] : (i == iu + 1 && iu >= 0 ? accp[t][1][ct][h] : 0.0));
                        for (int a = 0; a < S; ++a)
                          {
                            double z = 0.0;
#pragma unroll
                            for (int i = 0; i < kMaxS; ++i)
                              if (i < S)
                                z = fma(F.V[a * S + i], y[i], z);
                            const int row = prow(a, j);
                            asm volatile("red.global.add.f64 [%0], %1;\n" ::"l"(u + (row < nvel ? cvb[col] : cpb[col]) +
                                                                                 s_rel[row]),
                                         "d"(s_w[row] * z)
                                         : "memory");
                          }
                      }
              }
          }
#else
          __syncthreads(); // every warp is done with T
          // Y into the T rows of its block
#pragma unroll
          for (int b = 0; b < 2; ++b)
            if (b < F.nb)
              {
                const int t0 = F.c0[b] * nsp;
#pragma unroll
                for (int t = 0; t < kFTiles; ++t)
                  {
                    const int row = 8 * (warp + NW * t) + (lane >> 2);
                    if (row < ns)
#pragma unroll
                      for (int ct = 0; ct < 2; ++ct)
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                          {
                            const int col = 8 * ct + 2 * (lane & 3) + h;
                            if (F.sz[b] == 1)
                              Ts[tsw(t0 + row, col)] = accr[t][ct][h];
                            else
                              {
                                Ts[tsw(t0 + row, col)] = accp[t][0][ct][h];
                                Ts[tsw(t0 + nsp + row, col)] = accp[t][1][ct][h];
                              }
                          }
                  }
              }
          __syncthreads();
          // Z = (V (x) I) Y, weights, scatter
          for (int e = tid; e < ns * kFCols; e += NTH)
            {
              const int c = e / ns, j = e - c * ns;
              if (c >= ng)
                continue;
              double y[kMaxS];
#pragma unroll
              for (int i = 0; i < kMaxS; ++i)
                y[i] = i < S ? Ts[tsw(i * nsp + j, c)] : 0.0;
              for (int a = 0; a < S; ++a)
                {
                  double z = 0.0;
#pragma unroll
                  for (int i = 0; i < kMaxS; ++i)
                    if (i < S)
                      z = fma(F.V[a * S + i], y[i], z);
                  const int row = prow(a, j);
                  asm volatile("red.global.add.f64 [%0], %1;\n" ::"l"(u + (row < nvel ? cvb[c] : cpb[c]) +
                                                                       s_rel[row]),
                               "d"(s_w[row] * z)
                               : "memory");
                }
            }
#endif
          __syncthreads(); // Ts and the column data are reused by the next patch
        }
    }
}
} // namespace

namespace
{
// intervals per block of the item kernels: [0] DMMA (128 / 176 rows), [1] big
// patches; 0 = size heuristic. Initialised from STMG_VGROUP / STMG_BGROUP.
int g_group_override[2] = {std::getenv("STMG_VGROUP") ? std::atoi(std::getenv("STMG_VGROUP")) : 0,
                           std::getenv("STMG_BGROUP") ? std::atoi(std::getenv("STMG_BGROUP")) : 0};
} // namespace

void
set_vanka_group_override(int dmma_group, int big_group)
{
  g_group_override[0] = dmma_group;
  g_group_override[1] = big_group;
}

int
device_sm_count()
{
  static int cached[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64)
    dev = 0;
  if (cached[dev] == 0)
    {
      int n = 0;
      if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
        n = 148;
      cached[dev] = n;
    }
  return cached[dev];
}

cudaError_t
launch_vanka_big_fac(const DevPatchClass *classes, const VankaBatch *batches, int n_batches, int max_nt,
                     const long long *vel_anchor, const long long *pre_anchor, const Fac3Params &F, const double *r,
                     double *u, long long isz, int n_intervals, double omega, cudaStream_t st)
{
  if (n_batches == 0 || n_intervals == 0)
    return cudaSuccess;
  const int ns_max = max_nt / F.S, nrow = F.S * f_nsp(ns_max);
  int max_m = 0;
  for (int b = 0; b < F.nb; ++b)
    {
      if (F.sz[b] < 1 || F.sz[b] > 2)
        return cudaErrorInvalidValue;
      max_m = std::max(max_m, F.sz[b] * ns_max);
    }
  if (F.nb > 2 || ns_max > 16 * kFTiles * 8 || (F.nb == 2 && F.sz[0] == F.sz[1]))
    return cudaErrorInvalidValue; // the host keeps the dense inverses then
  const size_t big = static_cast<size_t>(kFSlots) * std::max(kFChunkCols * max_m, kFRealCols * ns_max);
  const size_t smem = sizeof(double) * (big + static_cast<size_t>(nrow) * kFLd + (max_nt + 1) / 2 * 2) +
                      sizeof(long long) * 2 * kFCols + sizeof(unsigned long long) * 2 * kFSlots +
                      sizeof(int) * max_nt;
  if (smem > 227 * 1024)
    return cudaErrorInvalidValue;
  const int group = kFCols;
  // persistent: the CTAs walk a strided share of the colour's batches. Patches of <= 128 spatial dofs
  // (the r = 1 levels of the C5 hierarchy) run as two 8-warp CTAs per SM when their shared memory
  // allows it, so one CTA's gather / scatter and barriers overlap the other's stream
#ifndef STMG_FAC_SMALL_CTAS
#define STMG_FAC_SMALL_CTAS 1
#endif
  const int ngroups = (n_intervals + group - 1) / group;
  const bool small = STMG_FAC_SMALL_CTAS && ns_max <= 8 * kFTiles * 8 && smem <= 110 * 1024 &&
                     static_cast<long long>(n_batches) * ngroups > device_sm_count(); // else the 16-warp CTAs are faster per patch
  const int per_sm = small ? 2 : 1;
  const int ctas = std::max(1, std::min(n_batches, (per_sm * device_sm_count() + ngroups - 1) / ngroups));
  dim3 grid(ctas, ngroups);
  if (small)
    {
      cudaFuncSetAttribute(vanka_big_fac_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      vanka_big_fac_kernel<8><<<grid, 256, smem, st>>>(classes, batches, n_batches, vel_anchor, pre_anchor, F, r, u,
                                                       isz, n_intervals, omega, group, max_m, max_nt);
    }
  else
    {
      cudaFuncSetAttribute(vanka_big_fac_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
      vanka_big_fac_kernel<16><<<grid, kFThreads, smem, st>>>(classes, batches, n_batches, vel_anchor, pre_anchor, F,
                                                               r, u, isz, n_intervals, omega, group, max_m, max_nt);
    }
  return cudaGetLastError();
}

/// Launch one colour: `n_batches` batches over `n_intervals` intervals.
cudaError_t
launch_vanka_colour(const DevPatchClass *classes, const VankaBatch *batches, const int *item_ptr, int n_batches,
                    int max_nt, const long long *vel_anchor, const long long *pre_anchor, const double *r, double *u,
                    long long isz, int n_intervals, double omega, cudaStream_t stream)
{
  if (n_batches == 0 || n_intervals == 0)
    return cudaSuccess;
  static const bool force_big = std::getenv("STMG_VANKA_BIG") != nullptr; // A/B switch for 128 < n_T <= 176
  static const bool old176 = std::getenv("STMG_VANKA176_OLD") != nullptr;   // A/B switch: the split item kernel
  if (max_nt > kDRows && max_nt <= 176 && !item_ptr && !force_big && !old176)
    {
      // deferred-scatter pipeline (vanka_tc.cu); long blocks keep the ring busy
      int group = g_group_override[0] > 0 ? g_group_override[0] : 16;
      while (group > 1 &&
             static_cast<long long>(n_batches) * 2 * ((n_intervals + group - 1) / group) < 2 * device_sm_count())
        group /= 2;
      const cudaError_t e = launch_vanka_dfr176(classes, batches, n_batches, max_nt, vel_anchor, pre_anchor, r, u,
                                                isz, n_intervals, omega, group, stream);
      if (e != cudaErrorInvalidValue)
        return e;
    }
  if (max_nt <= 176 && !(force_big && max_nt > kDRows && !item_ptr))
    {
      // 128 rows (16 warps) for 2D patches; 176 rows (22 warps) for 3D Q2 cells (n_T = 170)
      const int rows = max_nt <= kDRows ? kDRows : 176;
      const int split = rows == 176 ? 2 : 1, orows = rows / split;
      const int cols = rows == 176 ? STMG_V176_COLS : kDCols; // COLS of the instantiated kernel
      const size_t dsmem = sizeof(double) * (rows * kDRLd + orows * kDZLd + orows) + sizeof(long long) * 6 * cols;
      // intervals per block: 16 for 2D patches, 4 for the 176-row split (C3:
      // more, shorter blocks balance better), fewer on small levels so the
      // launch still fills the GPU (a coarse level has only a few batches per
      // colour). A tuning override (stmg_set_tuning) is taken as is.
      int group = g_group_override[0];
      if (group <= 0)
        {
          group = rows == 176 ? 4 : kDGroup;
          while (group > 1 &&
                 static_cast<long long>(n_batches) * split * ((n_intervals + group - 1) / group) < 2 * device_sm_count())
            group /= 2;
        }
      dim3 grid(n_batches, (n_intervals + group - 1) / group, split);
      const int ks = (max_nt + 3) / 4;
      auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dsmem));
        if (rows == 176 && STMG_V176_CLUSTER)
          {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = grid;
            cfg.blockDim = dim3(352);
            cfg.dynamicSmemBytes = dsmem;
            cfg.stream = stream;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 1;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 2;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, kern, classes, batches, item_ptr, vel_anchor, pre_anchor, r, u, isz,
                               n_intervals, omega, group);
          }
        else
          kern<<<grid, rows == 176 ? 352 : rows * 4, dsmem, stream>>>(
            classes, batches, item_ptr, vel_anchor, pre_anchor, r, u, isz, n_intervals, omega, group);
      };
      if (rows == 176)
        go(vanka_dmma_kernel<44, 176, 1, STMG_V176_COLS, 2>); // 2 CTAs x 88 rows, one 8-row tile per warp
      else if (ks <= 8)
        go(vanka_dmma_kernel<8>);
      else if (ks <= 12)
        go(vanka_dmma_kernel<12>);
      else if (ks <= 16)
        go(vanka_dmma_kernel<16>);
      else if (ks <= 20)
        go(vanka_dmma_kernel<20>);
      else if (ks <= 24)
        go(vanka_dmma_kernel<24>);
      else if (ks <= 28)
        go(vanka_dmma_kernel<28>);
      else
        go(vanka_dmma_kernel<32>);
      return cudaGetLastError();
    }
  if (!item_ptr && max_nt <= 16 * kBMaxTiles * 8)
    {
      const int ks = (max_nt + 3) / 4;
      const size_t smem = sizeof(double) * (4 * ks * kBLd) + sizeof(long long) * 2 * kBCols;
      const int tpw = ((max_nt + 7) / 8 + 15) / 16;
      int group = g_group_override[1];
      if (group <= 0)
        {
          group = kBGroup;
          while (group > 1 && static_cast<long long>(n_batches) * ((n_intervals + group - 1) / group) < 2 * device_sm_count())
            group /= 2;
        }
      dim3 grid(n_batches, (n_intervals + group - 1) / group);
      auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        kern<<<grid, kBThreads, smem, stream>>>(classes, batches, vel_anchor, pre_anchor, r, u, isz, n_intervals,
                                                omega, group);
      };
      if (tpw <= 2)
        go(vanka_big_kernel<2>);
      else if (tpw <= 4)
        go(vanka_big_kernel<4>);
      else if (tpw <= 5)
        go(vanka_big_kernel<5>);
      else
        go(vanka_big_kernel<7>);
      return cudaGetLastError();
    }
  const int ntp = (max_nt + 1) & ~1;
  size_t smem = sizeof(double) * (static_cast<size_t>(max_nt) * ntp + static_cast<size_t>(ntp) * kVankaCols);
  int in_smem = 1;
  if (smem > 200 * 1024)
    {
      in_smem = 0;
      smem = sizeof(double) * static_cast<size_t>(ntp) * kVankaCols;
    }
  static bool attr_set = false;
  if (!attr_set)
    {
      cudaFuncSetAttribute(vanka_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      attr_set = true;
    }
  dim3 grid(n_batches, n_intervals);
  vanka_kernel<<<grid, kVankaThreads, smem, stream>>>(classes, batches, vel_anchor, pre_anchor, r, u, isz, omega,
                                                       in_smem);
  return cudaGetLastError();
}

int
vanka_cols_per_batch()
{
  return kVankaCols;
}

} // namespace stmg_b200
