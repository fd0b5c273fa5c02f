// Additive Vanka patch solves on the FP64 tensor path, pipelined (sm_100a).
//
// Replaces the patch loop of VankaSmoother::apply_additive / smooth_step
// (vanka.cpp:196-233): u += omega * sum_T R_T^T w_T A_T^{-1} R_T r.
//
// Per block: a host-built list of tiles, each <= 32 columns (patch, interval)
// of one congruence class inside one colour sub-phase of a contiguous strip
// of super-cells.
//  * gather: R tiles are copied global -> shared with cp.async two tiles
//    ahead into a 3-slot ring, so residual loads never hold registers;
//  * Z = A^{-1} R with mma.sync.m8n8k4.f64 (DMMA); the class inverse lives in
//    registers as A-fragments, warp w owns rows 8w..8w+7;
//  * scatter straight from the accumulator fragments with red.global.add.f64:
//    no read-back of u, no Z staging;
//  * no block barrier per tile: full/empty mbarriers hand the ring slots
//    between the gather and the MMAs, so warps drift up to a tile apart and
//    one warp's gather/scatter overlaps another's tensor work;
//  * determinism: strips are 2x2-coloured across launches (no two running
//    blocks share a dof) and a phase-done mbarrier orders the scatters of a
//    block's colour sub-phases, so every red.add lands in a fixed order.
#include "kernels.hpp"

#include <cstdlib>
#include <string>
#include <cuda_runtime.h>

namespace stmg_b200
{

namespace
{
constexpr int kTThreads = 512;
constexpr int kTRows = 128;
#ifndef STMG_VANKA_COLS
#define STMG_VANKA_COLS 32
#endif
constexpr int kTCols = STMG_VANKA_COLS; // columns (patch, interval) per tile
// Diagnostic build switches (wrong results, timing only; DESIGN.md §3.2 cost
// breakdown): STMG_VT_NO_GATHER, STMG_VT_NO_SCATTER.
//
// R tiles column-major in shared memory: element (row k, column n) at
// n * kTLd + k. The gather walks rows with the lanes of a warp (rows of a
// patch come in contiguous runs of 4-6 dofs: few sectors per instruction);
// pitch 132 == 4 mod 16 doubles keeps the DMMA B-fragment loads
// (k = lane % 4, n = lane / 4) conflict-free.
constexpr int kTLd = kTRows + 4;
constexpr int kTSlot = kTCols * kTLd;
#ifndef STMG_VANKA_MAXTILES
#define STMG_VANKA_MAXTILES 48
#endif
constexpr int kTMaxTiles = STMG_VANKA_MAXTILES; // tiles per block (host falls back beyond)
constexpr int kTRing = 3; // ring slots of the full/empty mbarrier pipeline (vanka_tc_kernel)
#ifndef STMG_DFR_RING
#define STMG_DFR_RING 3 // measured: 4 slots 4.66 vs 4.56 ms (the larger ring takes L1 from the gathers)
#endif
constexpr int kDRing = STMG_DFR_RING; // vanka_dfr_kernel: ring slots; tiles gathered kDRing - 1 ahead
// vanka_dfr_kernel B fragments by 128-bit loads: the rows of an R tile are
// stored permuted inside every group of 8 (row 8j + 4h + t at 8j + 2t + h), so
// the B values of lane t for the k-steps 2j and 2j + 1 are adjacent and one
// LDS.128 feeds two k-steps (half the shared-memory instructions of the DMMA
// loop); pitch 136 == 8 mod 16 doubles keeps the quarter-warp phases of the
// 128-bit loads conflict-free.
#ifndef STMG_DFR_LDS128
#define STMG_DFR_LDS128 0 // measured: 4.96 vs 4.55 ms on C2 (bv[] costs 8 registers: 132 bytes of spills at the 128-register cap)
#endif
constexpr int kDLd = STMG_DFR_LDS128 ? kTRows + 8 : kTLd;
constexpr int kDSlot = kTCols * kDLd;
constexpr size_t kDSmem = sizeof(double) * kDRing * kDSlot + kTMaxTiles * (sizeof(VankaTile) + kTCols * 12) +
                          (2 * kDRing + 2) * sizeof(unsigned long long); // vanka_dfr_kernel
constexpr size_t kTSmem =
  sizeof(double) * kTRing * kTSlot + kTMaxTiles * (sizeof(VankaTile) + kTCols * (16 + 4)) + 8 * sizeof(unsigned long long);

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
__device__ __forceinline__ void
cp_async_wait0()
{
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// zero-filling copy: src_bytes = 0 writes 0.0 (the slot write stays async,
// so the mbarrier pipeline tracks every write of a gather)
__device__ __forceinline__ void
cp_async8z(double *dst, const double *src, bool valid)
{
  const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ unsigned
smem_u32(const void *p)
{
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void
mbar_init(unsigned long long *bar, unsigned count)
{
  asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void
mbar_arrive(unsigned long long *bar)
{
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared.b64 st, [%0];\n}\n" ::"r"(smem_u32(bar)) : "memory");
}
// arrive once all prior cp.async of this thread have completed
__device__ __forceinline__ void
cp_async_mbar_arrive(unsigned long long *bar)
{
  asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void
mbar_wait(unsigned long long *bar, unsigned parity)
{
  asm volatile("{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
                 smem_u32(bar)),
               "r"(parity)
               : "memory");
}

// fire-and-forget atomic add (atomicAdd may compile to ATOMG with a return
// register, which serialises a single warp's scatter on the round trips)
__device__ __forceinline__ void
red_add(double *addr, double v)
{
  asm volatile("red.global.add.f64 [%0], %1;\n" ::"l"(addr), "d"(v) : "memory");
}

__device__ __forceinline__ void
dmma(double (&d)[2], double a, double b)
{
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int KS>
__global__ void __launch_bounds__(kTThreads, 1)
vanka_tc_kernel(const DevPatchClass *__restrict__ classes, const VankaTile *__restrict__ tiles,
                const long long *__restrict__ va, const long long *__restrict__ pa, const int *__restrict__ tile_ptr,
                int ng_full, const double *__restrict__ r, double *__restrict__ u, long long isz, int n_intervals,
                double omega)
{
  extern __shared__ __align__(16) double ring[]; // kTSlots slots of kTRows x kTLd, then the block's tile data
  long long *s_colv = reinterpret_cast<long long *>(ring + kTRing * kTSlot);
  long long *s_colp = s_colv + kTMaxTiles * kTCols;
  int *s_coln = reinterpret_cast<int *>(s_colp + kTMaxTiles * kTCols);
  VankaTile *s_tile = reinterpret_cast<VankaTile *>(s_coln + kTMaxTiles * kTCols);
  // full[3], empty[3], phase-done[2]
  unsigned long long *s_bar = reinterpret_cast<unsigned long long *>(s_tile + kTMaxTiles);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t0 = tile_ptr[blockIdx.x], t1 = tile_ptr[blockIdx.x + 1];
  const int nb = t1 - t0;
  const int n0 = blockIdx.y * ng_full;
  const long long base0 = n0 * isz;

  // stage this block's tile headers and expand their column data
  // (<= kTMaxTiles tiles): column j of tile t = (patch, interval) entry
  // c0 + j of its item, patch-major, interval-minor
  for (int e = tid; e < nb; e += kTThreads)
    s_tile[e] = tiles[t0 + e];
  for (int e = tid; e < nb * kTCols; e += kTThreads)
    {
      const VankaTile tl = tiles[t0 + e / kTCols];
      const int j = e % kTCols;
      if (j < tl.ncols)
        {
          const int q = tl.c0 + j, patch = tl.pfirst + q / ng_full, nl = q % ng_full;
          s_colv[e] = nl * isz + va[patch];
          s_colp[e] = nl * isz + pa[patch];
          s_coln[e] = nl;
        }
      else
        {
          s_colv[e] = s_colp[e] = 0;
          s_coln[e] = 1 << 30; // masked column
        }
    }
  __syncthreads();

  // gather: warp w fills columns w and w + 16, lane l rows l + 32 q
  constexpr int QN = kTRows / 32;
  constexpr int CN = kTCols / (kTThreads / 32);
  const int lane_g = tid & 31, warp_g = tid >> 5;
  auto row_of = [&](int q) { return lane_g + 32 * q; };
  int cls_issue = -1, nt_issue = 0, nvel_issue = 0;
  long long relq[QN];

  // gather of local tile lt into ring slot s
  auto issue = [&](int lt, int s) {
    if (lt < nb)
      {
        const VankaTile tl = s_tile[lt];
        if (tl.ncols == 0)
          return; // stage padding: nothing to gather
        if (tl.cls != cls_issue)
          {
            const DevPatchClass pc = classes[tl.cls];
            nt_issue = pc.n_t;
            nvel_issue = pc.n_vel;
#pragma unroll
            for (int q = 0; q < QN; ++q)
              relq[q] = row_of(q) < nt_issue ? pc.rel[row_of(q)] : 0;
            cls_issue = tl.cls;
          }
        double *slot = ring + s * kTSlot;
#pragma unroll
        for (int cc = 0; cc < CN; ++cc)
          {
            const int col = warp_g + cc * (kTThreads / 32);
            const int ci = lt * kTCols + col;
            const bool colok = col < tl.ncols && n0 + s_coln[ci] < n_intervals;
            const long long cv = base0 + s_colv[ci], cp = base0 + s_colp[ci];
#pragma unroll
            for (int q = 0; q < QN; ++q)
              {
                const int row = row_of(q);
                double *dst = slot + col * kTLd + row;
#ifdef STMG_VT_NO_GATHER
                const bool valid = false;
#else
                const bool valid = colok && row < nt_issue;
#endif
                cp_async8z(dst, valid ? r + (row < nvel_issue ? cv : cp) + relq[q] : r, valid);
              }
          }
      }
  };
  // Full/empty mbarrier pipeline over 3 slots: full[s] completes when every
  // thread's copies of the slot's tile have landed (cp.async arrive), so a
  // warp waits only for the tile it computes; empty[s] completes when every
  // thread has finished its MMAs on the slot. Tile lt+2 is gathered (into the
  // slot of tile lt-1) right after a thread finishes tile lt, so warps drift
  // up to a tile apart instead of meeting at a block barrier every tile.
  unsigned long long *full = s_bar, *empty = s_bar + 3, *pdone = s_bar + 6;
  if (tid == 0)
    {
      for (int i = 0; i < 3; ++i)
        {
          mbar_init(full + i, kTThreads);
          mbar_init(empty + i, kTThreads);
        }
      mbar_init(pdone + 0, kTThreads);
      mbar_init(pdone + 1, kTThreads);
    }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  issue(0, 0);
  cp_async_mbar_arrive(full + 0);
  issue(1, 1);
  cp_async_mbar_arrive(full + 1);

  int loaded = -1, nt_loaded = 0;
  double afr[KS];
  long long rel_row = 0;
  bool vel_row = false, ok_row = false;
  double w_row = 0.0;
  const int row = 8 * warp + (lane >> 2);

  // Colour sub-phases of a block share dofs: before the first scatter of a
  // new phase, every thread's scatters of the previous phase must be done
  // (arrive = release, wait = acquire), so the red.add order -- and the
  // result -- is the same on every run. MMAs of the next phase may start early.
  int cur_phase = -1, transitions = 0;
  for (int lt = 0; lt < nb; ++lt)
    {
      const int slot = lt % 3;
      mbar_wait(full + slot, (lt / 3) & 1);
      const VankaTile tl = s_tile[lt];
      double acc[kTCols / 8][2];
#pragma unroll
      for (int ct = 0; ct < kTCols / 8; ++ct)
        acc[ct][0] = acc[ct][1] = 0.0;
      if (tl.ncols > 0)
        {
          if (tl.cls != loaded)
            {
              const DevPatchClass pc = classes[tl.cls];
#pragma unroll
              for (int kk = 0; kk < KS; ++kk)
                {
                  const int col = 4 * kk + (lane & 3);
                  afr[kk] = (row < pc.n_t && col < pc.n_t) ? __ldg(pc.inverse + row * pc.n_t + col) : 0.0;
                }
              ok_row = row < pc.n_t;
              vel_row = row < pc.n_vel;
              rel_row = ok_row ? pc.rel[row] : 0;
              w_row = ok_row ? omega * pc.weight[row] : 0.0;
              nt_loaded = pc.n_t;
              loaded = tl.cls;
            }
          const double *bbase = ring + slot * kTSlot + (lane >> 2) * kTLd + (lane & 3);
          if (8 * warp < nt_loaded)
            {
#pragma unroll
              for (int kk = 0; kk < KS; ++kk)
                {
                  const double *brow = bbase + 4 * kk;
                  constexpr int kNStep = 8 * kTLd; // next 8 columns
#pragma unroll
                  for (int ct = 0; ct < kTCols / 8; ++ct)
                    dmma(acc[ct], afr[kk], brow[kNStep * ct]);
                }
            }
        }
      mbar_arrive(empty + slot); // this thread is done reading the slot
      if (tl.phase != cur_phase)
        {
          if (cur_phase >= 0)
            {
              unsigned long long *pd = pdone + (transitions & 1);
              mbar_arrive(pd);
              mbar_wait(pd, (transitions >> 1) & 1);
              ++transitions;
            }
          cur_phase = tl.phase;
        }
      if (tl.ncols > 0 && ok_row)
        {
#pragma unroll
          for (int ct = 0; ct < kTCols / 8; ++ct)
#pragma unroll
            for (int b = 0; b < 2; ++b)
              {
                const int col = 8 * ct + 2 * (lane & 3) + b;
                const int ci = lt * kTCols + col;
#ifdef STMG_VT_NO_SCATTER
                if (acc[ct][b] == 123.456)
#else
                if (col < tl.ncols && n0 + s_coln[ci] < n_intervals)
#endif
                  atomicAdd(u + base0 + (vel_row ? s_colv[ci] : s_colp[ci]) + rel_row, acc[ct][b] * w_row);
              }
        }
      // gather tile lt+2 into the slot of tile lt-1 once every thread released it
      if (lt + 2 < nb)
        {
          const int ns = (lt + 2) % 3;
          if (lt >= 1)
            mbar_wait(empty + ns, ((lt - 1) / 3) & 1);
          issue(lt + 2, ns);
          cp_async_mbar_arrive(full + ns);
        }
    }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// ------------------------------------------------------- deferred scatter
// (anchors and relative offsets may be negative: vertex stars at the domain
// boundary anchor outside it, so masks use sentinels, not the sign)
constexpr long long kMaskedCol = -(1LL << 62);
constexpr int kMaskedRow = -(1 << 30);
// vanka_tc_kernel with the scatter of tile lt-1 interleaved into the DMMA
// k-loop of tile lt: each thread's 8 red.adds of the previous tile ride
// between the first 8 k-steps of the current one, so no warp leaves the
// tensor pipe for a separate scatter phase (the all-warp kernel runs its
// gather / scatter in near lockstep across warps, which idles the pipe).
// Column data is a 64-bit velocity offset (kMaskedCol: masked) plus the
// 32-bit pressure - velocity distance; class rows become a pointer, a mask
// and a weight, so the interleaved scatter costs a few integer ops per red.
template <int KS>
__global__ void __launch_bounds__(kTThreads, 1)
vanka_dfr_kernel(const DevPatchClass *__restrict__ classes, const VankaTile *__restrict__ tiles,
                 const long long *__restrict__ va, const long long *__restrict__ pa, const int *__restrict__ tile_ptr,
                 int ng_full, const double *__restrict__ r, double *__restrict__ u, long long isz, int n_intervals,
                 double omega)
{
  extern __shared__ __align__(16) double ring[];
  long long *s_colv = reinterpret_cast<long long *>(ring + kDRing * kDSlot);
  int *s_dp = reinterpret_cast<int *>(s_colv + kTMaxTiles * kTCols);
  VankaTile *s_tile = reinterpret_cast<VankaTile *>(s_dp + kTMaxTiles * kTCols);
  unsigned long long *s_bar = reinterpret_cast<unsigned long long *>(s_tile + kTMaxTiles);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t0 = tile_ptr[blockIdx.x], t1 = tile_ptr[blockIdx.x + 1];
  const int nb = t1 - t0;
  const int n0 = blockIdx.y * ng_full;
  const long long base0 = n0 * isz;

  for (int e = tid; e < nb; e += kTThreads)
    s_tile[e] = tiles[t0 + e];
  for (int e = tid; e < nb * kTCols; e += kTThreads)
    {
      const VankaTile tl = tiles[t0 + e / kTCols];
      const int j = e % kTCols;
      const int q = tl.c0 + j, nl = q % ng_full;
      if (j < tl.ncols && n0 + nl < n_intervals)
        {
          const int patch = tl.pfirst + q / ng_full;
          s_colv[e] = nl * isz + va[patch];
          s_dp[e] = static_cast<int>(pa[patch] - va[patch]);
        }
      else
        {
          s_colv[e] = kMaskedCol;
          s_dp[e] = 0;
        }
    }
  __syncthreads();

  constexpr int QN = kTRows / 32;
  constexpr int CN = kTCols / (kTThreads / 32);
  int cls_issue = -1;
  int relq[QN], pmq[QN]; // relq == kMaskedRow: row beyond the class's patch size
  auto issue = [&](int lt, int s) {
    if (lt >= nb)
      return;
    const VankaTile tl = s_tile[lt];
    if (tl.ncols == 0)
      return;
    if (tl.cls != cls_issue)
      {
        const DevPatchClass pc = classes[tl.cls];
#pragma unroll
        for (int q = 0; q < QN; ++q)
          {
            const int rw = lane + 32 * q;
            relq[q] = rw < pc.n_t ? static_cast<int>(pc.rel[rw]) : kMaskedRow;
            pmq[q] = (rw < pc.n_t && rw >= pc.n_vel) ? -1 : 0;
          }
        cls_issue = tl.cls;
      }
#if STMG_DFR_LDS128
    double *slot = ring + s * kDSlot + ((lane & ~7) | ((lane & 3) << 1) | ((lane >> 2) & 1));
#else
    double *slot = ring + s * kDSlot + lane;
#endif
#pragma unroll
    for (int cc = 0; cc < CN; ++cc)
      {
        const int col = warp + cc * (kTThreads / 32);
        const int ci = lt * kTCols + col;
        const long long cv = s_colv[ci];
        const bool colok = cv != kMaskedCol;
        const double *pv = r + (base0 + (colok ? cv : 0));
        const int dp = s_dp[ci];
#pragma unroll
        for (int q = 0; q < QN; ++q)
          {
            const bool ok = colok && relq[q] != kMaskedRow;
            cp_async8z(slot + col * kDLd + 32 * q, pv + (ok ? relq[q] + (dp & pmq[q]) : 0), ok);
          }
      }
  };
  unsigned long long *full = s_bar, *empty = s_bar + kDRing, *pdone = s_bar + 2 * kDRing;
  if (tid == 0)
    {
      for (int i = 0; i < kDRing; ++i)
        {
          mbar_init(full + i, kTThreads);
          mbar_init(empty + i, kTThreads);
        }
      mbar_init(pdone + 0, kTThreads);
      mbar_init(pdone + 1, kTThreads);
    }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();
  for (int i = 0; i < kDRing - 1; ++i)
    {
      issue(i, i);
      cp_async_mbar_arrive(full + i);
    }

  int loaded = -1, nt_loaded = 0;
  double afr[KS];
  const int row = 8 * warp + (lane >> 2);
  // class row of this thread: u + base0 + rel (pointer), pressure mask
  double *c_ub = u, *p_ub = u;
  int c_pm = 0, p_pm = 0;
  bool c_ok = false;
  // pending tile (scattered inside the next tile's k-loop)
  double pacc[kTCols / 8][2] = {};
  int p_lt = -1;
  auto scatter_one = [&](int j) {
    const int ct = j >> 1, b = j & 1;
    const int ci = p_lt * kTCols + 8 * ct + 2 * (lane & 3) + b;
    const long long cv = s_colv[ci];
    if (cv != kMaskedCol)
      red_add(p_ub + (cv + (s_dp[ci] & p_pm)), pacc[ct][b]);
  };
  int prev_phase = -1, transitions = 0;
  // split phase barrier: a thread arrives once it scattered the last tile of
  // a colour sub-phase and waits only right before its first scatter of the
  // next one (that tile's DMMAs run in between), at most one outstanding
  int wait_t = -1;
  auto phase_wait = [&]() {
    if (wait_t >= 0)
      {
        mbar_wait(pdone + (wait_t & 1), (wait_t >> 1) & 1);
        wait_t = -1;
      }
  };
  for (int lt = 0; lt < nb; ++lt)
    {
      const int slot = lt % kDRing;
      mbar_wait(full + slot, (lt / kDRing) & 1);
      const VankaTile tl = s_tile[lt];
      double acc[kTCols / 8][2];
#pragma unroll
      for (int ct = 0; ct < kTCols / 8; ++ct)
        acc[ct][0] = acc[ct][1] = 0.0;
      if (tl.ncols > 0 && tl.cls != loaded)
        {
          const DevPatchClass pc = classes[tl.cls];
          c_ok = row < pc.n_t;
          // the valence weight and omega are folded into the inverse's row:
          // no DMUL per scattered value on the FP64 pipe the DMMAs saturate
          const double wrow = c_ok ? omega * pc.weight[row] : 0.0;
#pragma unroll
          for (int kk = 0; kk < KS; ++kk)
            {
              const int col = 4 * kk + (lane & 3);
              afr[kk] = (c_ok && col < pc.n_t) ? wrow * __ldg(pc.inverse + row * pc.n_t + col) : 0.0;
            }
          c_pm = (c_ok && row >= pc.n_vel) ? -1 : 0;
          c_ub = u + (base0 + (c_ok ? pc.rel[row] : 0));
          nt_loaded = pc.n_t;
          loaded = tl.cls;
        }
      const bool mine = tl.ncols > 0 && 8 * warp < nt_loaded;
      if (mine)
        {
#if STMG_DFR_LDS128
          const double *bbase = ring + slot * kDSlot + (lane >> 2) * kDLd + 2 * (lane & 3);
#else
          const double *bbase = ring + slot * kDSlot + (lane >> 2) * kDLd + (lane & 3);
#endif
          // the previous tile's scatters ride in k-steps kS0.. of this tile
#ifndef STMG_DFR_SC0
#define STMG_DFR_SC0 4
#endif
          constexpr int kSc = 2 * (kTCols / 8), kS0 = KS >= STMG_DFR_SC0 + kSc ? STMG_DFR_SC0 : 0;
#if STMG_DFR_LDS128
          double2 bv[kTCols / 8];
#endif
#pragma unroll
          for (int kk = 0; kk < KS; ++kk)
            {
              constexpr int kNStep = 8 * kDLd;
#if STMG_DFR_LDS128
              if ((kk & 1) == 0)
#pragma unroll
                for (int ct = 0; ct < kTCols / 8; ++ct)
                  bv[ct] = *reinterpret_cast<const double2 *>(bbase + 4 * kk + kNStep * ct);
#pragma unroll
              for (int ct = 0; ct < kTCols / 8; ++ct)
                dmma(acc[ct], afr[kk], (kk & 1) ? bv[ct].y : bv[ct].x);
#else
              const double *brow = bbase + 4 * kk;
#pragma unroll
              for (int ct = 0; ct < kTCols / 8; ++ct)
                dmma(acc[ct], afr[kk], brow[kNStep * ct]);
#endif
              if (kk == kS0 && p_lt >= 0)
                phase_wait();
              if (kk >= kS0 && kk - kS0 < kSc && p_lt >= 0)
                scatter_one(kk - kS0);
            }
          if (KS < kSc && p_lt >= 0)
#pragma unroll
            for (int j = KS; j < kSc; ++j)
              scatter_one(j);
        }
      else if (p_lt >= 0)
        {
          phase_wait();
#pragma unroll
          for (int j = 0; j < 2 * (kTCols / 8); ++j)
            scatter_one(j);
        }
      mbar_arrive(empty + slot);
      // the previous tile's scatters are done: a new colour sub-phase may
      // start scattering only once every thread got here (deterministic order)
      if (prev_phase >= 0 && tl.phase != prev_phase)
        {
          phase_wait();
          mbar_arrive(pdone + (transitions & 1));
          wait_t = transitions++;
        }
      prev_phase = tl.phase;
      p_lt = (tl.ncols > 0 && c_ok) ? lt : -1;
#pragma unroll
      for (int ct = 0; ct < kTCols / 8; ++ct)
        {
          pacc[ct][0] = acc[ct][0];
          pacc[ct][1] = acc[ct][1];
        }
      p_ub = c_ub;
      p_pm = c_pm;
      if (lt + kDRing - 1 < nb)
        {
          const int ns = (lt + kDRing - 1) % kDRing;
          if (lt >= 1)
            mbar_wait(empty + ns, ((lt - 1) / kDRing) & 1);
          issue(lt + kDRing - 1, ns);
          cp_async_mbar_arrive(full + ns);
        }
    }
  if (p_lt >= 0)
    {
      phase_wait();
#pragma unroll
      for (int j = 0; j < 2 * (kTCols / 8); ++j)
        scatter_one(j);
    }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// ------------------------------------------------ 176-row patches (3D Q2)
// The deferred-scatter pipeline of vanka_dfr_kernel for patches of
// 128 < n_T <= 176 rows (C3: Q2/P1disc x DG(1) cells, n_T = 170), one colour
// of same-class batches per launch (3D: 8 parity colours, no dof shared in
// a launch, so no phase barriers). The 176 rows are split over two CTAs
// (blockIdx.z) of 11 warps (88 rows each, one 8-row A tile per warp in
// registers, the valence weight and omega folded in); both CTAs gather the
// whole R tile (the contraction dimension) into a 3-slot cp.async ring two
// tiles ahead, and scatter the previous tile's accumulators inside the
// current tile's DMMA k-loop.
constexpr int k3Rows = 176, k3Half = 88, k3Warps = 11, k3Threads = 32 * k3Warps, k3KS = k3Rows / 4;
constexpr int k3Ld = k3Rows + 4; // == 4 mod 16 doubles: conflict-free B fragments
constexpr int k3Slot = kTCols * k3Ld;
constexpr int k3MaxCols = 32 * 16; // columns (patch, interval) per block

template <int KS> // k-steps of 4: 43 for n_T <= 172 (C3: n_T = 170), else 44
__global__ void __launch_bounds__(k3Threads, 1)
vanka_dfr176_kernel(const DevPatchClass *__restrict__ classes, const VankaBatch *__restrict__ batches,
                    const long long *__restrict__ vel_anchor, const long long *__restrict__ pre_anchor,
                    const double *__restrict__ r, double *__restrict__ u, long long isz, int n_intervals,
                    double omega, int group)
{
  extern __shared__ __align__(16) double ring[];
  long long *s_colv = reinterpret_cast<long long *>(ring + kTRing * k3Slot);
  int *s_dp = reinterpret_cast<int *>(s_colv + k3MaxCols);
  unsigned long long *s_bar = reinterpret_cast<unsigned long long *>(s_dp + k3MaxCols);
  unsigned long long *full = s_bar, *empty = s_bar + 3;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const VankaBatch bt = batches[blockIdx.x];
  const DevPatchClass pc = classes[bt.cls];
  const int nt = pc.n_t, nvel = pc.n_vel;
  const int n0 = blockIdx.y * group, ng = min(group, n_intervals - n0);
  const int ncols = bt.count * ng, nb = (ncols + kTCols - 1) / kTCols;
  const int row0 = static_cast<int>(blockIdx.z) * k3Half;
  for (int e = tid; e < nb * kTCols; e += k3Threads)
    {
      if (e < ncols)
        {
          const int patch = bt.first + e / ng, nl = e % ng;
          const long long vb = __ldg(vel_anchor + patch), pb = __ldg(pre_anchor + patch);
          s_colv[e] = (n0 + nl) * isz + vb;
          s_dp[e] = static_cast<int>(pb - vb);
        }
      else
        {
          s_colv[e] = kMaskedCol;
          s_dp[e] = 0;
        }
    }
  if (tid == 0)
    for (int i = 0; i < 3; ++i)
      {
        mbar_init(full + i, k3Threads);
        mbar_init(empty + i, k3Threads);
      }
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncthreads();

  // gather: warp w fills columns w, w + 11, w + 22; lane l rows l + 32 q
  constexpr int QN = (k3Rows + 31) / 32, CN = (kTCols + k3Warps - 1) / k3Warps;
  int relq[QN], pmq[QN];
#pragma unroll
  for (int q = 0; q < QN; ++q)
    {
      const int rw = lane + 32 * q;
      relq[q] = rw < nt ? static_cast<int>(pc.rel[rw]) : kMaskedRow;
      pmq[q] = (rw < nt && rw >= nvel) ? -1 : 0;
    }
  auto issue = [&](int lt, int s) {
    if (lt < nb)
      {
        double *slot = ring + s * k3Slot + lane;
#pragma unroll
        for (int cc = 0; cc < CN; ++cc)
          {
            const int col = warp + cc * k3Warps;
            if (col >= kTCols)
              continue;
            const int ci = lt * kTCols + col;
            const long long cv = s_colv[ci];
            const bool colok = cv != kMaskedCol;
            const double *pv = r + (colok ? cv : 0);
            const int dp = s_dp[ci];
#pragma unroll
            for (int q = 0; q < QN; ++q)
              if (lane + 32 * q < k3Ld
#ifdef STMG_V176_HALFGATHER_DIAG // timing only (wrong results): each CTA gathers its own half of the rows
                  && (lane + 32 * q) / k3Half == static_cast<int>(blockIdx.z)
#endif
              )
                {
                  const bool ok = colok && relq[q] != kMaskedRow;
                  cp_async8z(slot + col * k3Ld + 32 * q, pv + (ok ? relq[q] + (dp & pmq[q]) : 0), ok);
                }
          }
      }
    cp_async_mbar_arrive(full + s);
  };
  issue(0, 0);
  issue(1, 1);

  // this warp's 8 rows of the inverse, weight and omega folded in
  const int row = row0 + 8 * warp + (lane >> 2);
  const bool c_ok = row < nt;
  double afr[KS];
  {
    const double wrow = c_ok ? omega * pc.weight[row] : 0.0;
    // unpredicated loads from clamped addresses, then the mask and the weight:
    // the predicated form came out of ptxas fully serialised (one L2 round
    // trip per load, 20 % of this kernel's stall samples in ncu); measured
    // C3 update 18.7 -> 19.9 TF/s. (In vanka_dfr_kernel the predicated loads
    // already issue in groups of 7 and this form costs registers: C4 9.73 ->
    // 9.99 ms, so it keeps them.)
    const double *arow = pc.inverse + (c_ok ? row : 0) * nt;
#pragma unroll
    for (int kk = 0; kk < KS; ++kk)
      afr[kk] = __ldg(arow + min(4 * kk + (lane & 3), nt - 1));
#pragma unroll
    for (int kk = 0; kk < KS; ++kk)
      afr[kk] = (c_ok && 4 * kk + (lane & 3) < nt) ? wrow * afr[kk] : 0.0;
  }
  const int c_pm = (c_ok && row >= nvel) ? -1 : 0;
  double *const c_ub = u + (c_ok ? pc.rel[row] : 0);
  const bool mine = row0 + 8 * warp < nt;
  double pacc[kTCols / 8][2] = {};
  int p_lt = -1;
  auto scatter_one = [&](int j) {
    const int ct = j >> 1, b = j & 1;
    const int ci = p_lt * kTCols + 8 * ct + 2 * (lane & 3) + b;
    const long long cv = s_colv[ci];
    if (cv != kMaskedCol)
      red_add(c_ub + (cv + (s_dp[ci] & c_pm)), pacc[ct][b]);
  };
  for (int lt = 0; lt < nb; ++lt)
    {
      const int slot = lt % 3;
      mbar_wait(full + slot, (lt / 3) & 1);
      double acc[kTCols / 8][2];
#pragma unroll
      for (int ct = 0; ct < kTCols / 8; ++ct)
        acc[ct][0] = acc[ct][1] = 0.0;
      if (mine)
        {
          const double *bbase = ring + slot * k3Slot + (lane >> 2) * k3Ld + (lane & 3);
#pragma unroll
          for (int kk = 0; kk < KS; ++kk)
            {
              const double *brow = bbase + 4 * kk;
#pragma unroll
              for (int ct = 0; ct < kTCols / 8; ++ct)
                dmma(acc[ct], afr[kk], brow[8 * k3Ld * ct]);
              if (kk < 2 * (kTCols / 8) && p_lt >= 0 && c_ok)
                scatter_one(kk);
            }
        }
      mbar_arrive(empty + slot);
      p_lt = lt;
#pragma unroll
      for (int ct = 0; ct < kTCols / 8; ++ct)
        {
          pacc[ct][0] = acc[ct][0];
          pacc[ct][1] = acc[ct][1];
        }
      if (lt + 2 < nb)
        {
          const int ns = (lt + 2) % 3;
          if (lt >= 1)
            mbar_wait(empty + ns, ((lt - 1) / 3) & 1);
          issue(lt + 2, ns);
        }
    }
  if (p_lt >= 0 && c_ok && mine)
#pragma unroll
    for (int j = 0; j < 2 * (kTCols / 8); ++j)
      scatter_one(j);
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// ---------------------------------------------------------------- factored
// Time-diagonalised patch solves: A_T^{-1} = (V (x) I) blockdiag(B_b^{-1})
// (W (x) I) (setup.hpp TemporalEigen). Per tile: stage 1 mixes the slots of
// the gathered R by W into T1 (rows coord * n_sp + j), the DMMA applies the
// block-diagonal middle (each warp's K range is its own block: ~40% fewer
// MACs than the dense inverse for DG(2)), Z goes to shared memory, and stage
// 3 mixes by V and scatters with the valence weights.
constexpr size_t kFSmem = sizeof(double) * 4 * kTSlot + kTRows * 16 + kTMaxTiles * (sizeof(VankaTile) + kTCols * (16 + 4));

template <int S, int NSP>
__global__ void __launch_bounds__(kTThreads, 1)
vanka_fac_kernel(const DevPatchClass *__restrict__ classes, const VankaTile *__restrict__ tiles,
                 const long long *__restrict__ va, const long long *__restrict__ pa, const int *__restrict__ tile_ptr,
                 int ng_full, const double *__restrict__ r, double *__restrict__ u, long long isz, int n_intervals,
                 double omega, const FacParams F)
{
  // 2 R slots, T1, Z, class rows (rel, omega * weight), then the block's tile data
  extern __shared__ __align__(16) double ring[];
  double *t1 = ring + 2 * kTSlot, *zb = ring + 3 * kTSlot;
  long long *s_rel = reinterpret_cast<long long *>(ring + 4 * kTSlot);
  double *s_w = reinterpret_cast<double *>(s_rel + kTRows);
  long long *s_colv = reinterpret_cast<long long *>(s_w + kTRows);
  long long *s_colp = s_colv + kTMaxTiles * kTCols;
  int *s_coln = reinterpret_cast<int *>(s_colp + kTMaxTiles * kTCols);
  VankaTile *s_tile = reinterpret_cast<VankaTile *>(s_coln + kTMaxTiles * kTCols);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t0 = tile_ptr[blockIdx.x], t1i = tile_ptr[blockIdx.x + 1];
  const int nb = t1i - t0;
  const int n0 = blockIdx.y * ng_full;
  const long long base0 = n0 * isz;
  constexpr int KB = NSP / 2, nsp = NSP; // widest block: 2 NSP columns

  for (int e = tid; e < nb; e += kTThreads)
    s_tile[e] = tiles[t0 + e];
  for (int e = tid; e < nb * kTCols; e += kTThreads)
    {
      const VankaTile tl = tiles[t0 + e / kTCols];
      const int j = e % kTCols;
      if (j < tl.ncols)
        {
          const int q = tl.c0 + j, patch = tl.pfirst + q / ng_full, nl = q % ng_full;
          s_colv[e] = nl * isz + va[patch];
          s_colp[e] = nl * isz + pa[patch];
          s_coln[e] = nl;
        }
      else
        {
          s_colv[e] = s_colp[e] = 0;
          s_coln[e] = 1 << 30;
        }
    }
  __syncthreads();

  // gather (as vanka_tc_kernel): warp w fills columns w and w + 16
  constexpr int QN = kTRows / 32;
  constexpr int CN = kTCols / (kTThreads / 32);
  int cls_issue = -1, nt_issue = 0, nvel_issue = 0;
  long long relq[QN];
  auto issue = [&](int lt, int slot) {
    if (lt < nb)
      {
        const VankaTile tl = s_tile[lt];
        if (tl.ncols == 0)
          return;
        if (tl.cls != cls_issue)
          {
            const DevPatchClass pc = classes[tl.cls];
            nt_issue = pc.n_t;
            nvel_issue = pc.n_vel;
#pragma unroll
            for (int q = 0; q < QN; ++q)
              relq[q] = lane + 32 * q < nt_issue ? pc.rel[lane + 32 * q] : 0;
            cls_issue = tl.cls;
          }
        double *dst0 = ring + slot * kTSlot;
#pragma unroll
        for (int cc = 0; cc < CN; ++cc)
          {
            const int col = warp + cc * (kTThreads / 32);
            const int ci = lt * kTCols + col;
            const bool colok = col < tl.ncols && n0 + s_coln[ci] < n_intervals;
            const long long cv = base0 + s_colv[ci], cp = base0 + s_colp[ci];
#pragma unroll
            for (int q = 0; q < QN; ++q)
              {
                const int row = lane + 32 * q;
                double *dst = dst0 + col * kTLd + row;
                if (colok && row < nt_issue)
                  cp_async8(dst, r + (row < nvel_issue ? cv : cp) + relq[q]);
                else
                  *dst = 0.0;
              }
          }
      }
  };
  issue(0, 0);
  cp_async_commit();

  int loaded = -1, ns = 0, nvs = 0, nvel = 0; // class of the tile being computed
  int p_lt = -1, p_ns = 0, p_nvs = 0, p_nvel = 0, p_ncols = 0; // tile whose Z awaits stage 3
  double afr[KB];
  const int row = 8 * warp + (lane >> 2);
  const int kbase = F.kbase[warp], ksteps = F.ksteps[warp];

  // stage 3 of the pending tile: out(a, j) = sum_i V(a, i) Z(i, j), weights, scatter
  auto stage3 = [&]() {
    if (p_lt < 0)
      return;
    const int nps = p_ns - p_nvs;
    for (int e = tid; e < nsp * kTCols; e += kTThreads)
      {
        const int j = e % nsp, c = e / nsp;
        const int ci = p_lt * kTCols + c;
        if (j >= p_ns || c >= p_ncols || n0 + s_coln[ci] >= n_intervals)
          continue;
        double z[S];
#pragma unroll
        for (int i = 0; i < S; ++i)
          z[i] = zb[c * kTLd + i * nsp + j];
#pragma unroll
        for (int a = 0; a < S; ++a)
            {
              double o = 0.0;
#pragma unroll
              for (int i = 0; i < S; ++i)
                o = fma(F.V[a * kMaxS + i], z[i], o);
              const int pr = j < p_nvs ? a * p_nvs + j : S * p_nvs + a * nps + (j - p_nvs);
              atomicAdd(u + base0 + (pr < p_nvel ? s_colv[ci] : s_colp[ci]) + s_rel[pr], o * s_w[pr]);
            }
      }
    p_lt = -1;
  };

  for (int lt = 0; lt < nb; ++lt)
    {
      cp_async_wait0();
      __syncthreads(); // R of tile lt visible; Z of the pending tile complete; T1 free
      issue(lt + 1, (lt + 1) & 1);
      cp_async_commit();
      const VankaTile tl = s_tile[lt];
      stage3(); // overlaps nothing but saves a barrier: Z and T1 are separate buffers
      if (tl.ncols == 0)
        continue;
      if (tl.cls != loaded)
        {
          // the class rows are read by stage 3 of this tile only after the
          // next barrier; the previous class's stage 3 is done (just above)
          __syncthreads();
          const DevPatchClass pc = classes[tl.cls];
          ns = pc.n_s;
          nvs = pc.n_vs;
          nvel = pc.n_vel;
          for (int e = tid; e < pc.n_t; e += kTThreads)
            {
              s_rel[e] = pc.rel[e];
              s_w[e] = omega * pc.weight[e];
            }
#pragma unroll
          for (int kk = 0; kk < KB; ++kk)
            afr[kk] = kk < ksteps ? __ldg(pc.fac_inv + static_cast<long long>(row) * 2 * nsp + 4 * kk + (lane & 3))
                                  : 0.0;
          loaded = tl.cls;
        }
      const int nps = ns - nvs;
      // stage 1: T1(i, j) = sum_b W(i, b) R(b, j), padding rows zero
      const double *R = ring + (lt & 1) * kTSlot;
      for (int e = tid; e < nsp * kTCols; e += kTThreads)
        {
          const int j = e % nsp, c = e / nsp;
          double rb[S];
#pragma unroll
          for (int b = 0; b < S; ++b)
            rb[b] = j < ns ? R[c * kTLd + (j < nvs ? b * nvs + j : S * nvs + b * nps + (j - nvs))] : 0.0;
#pragma unroll
          for (int i = 0; i < S; ++i)
            {
              double t = 0.0;
#pragma unroll
              for (int b = 0; b < S; ++b)
                t = fma(F.W[i * kMaxS + b], rb[b], t);
              t1[c * kTLd + i * nsp + j] = t;
            }
        }
      __syncthreads(); // T1 complete; stage 3 of the previous tile done (Z free)
      double acc[kTCols / 8][2];
#pragma unroll
      for (int ct = 0; ct < kTCols / 8; ++ct)
        acc[ct][0] = acc[ct][1] = 0.0;
      const double *bbase = t1 + (lane >> 2) * kTLd + kbase + (lane & 3);
#pragma unroll
      for (int kk = 0; kk < KB; ++kk)
        if (kk < ksteps)
          {
            const double *brow = bbase + 4 * kk;
#pragma unroll
            for (int ct = 0; ct < kTCols / 8; ++ct)
              dmma(acc[ct], afr[kk], brow[ct * 8 * kTLd]);
          }
      if (ksteps > 0)
#pragma unroll
        for (int ct = 0; ct < kTCols / 8; ++ct)
#pragma unroll
          for (int b = 0; b < 2; ++b)
            zb[(8 * ct + 2 * (lane & 3) + b) * kTLd + row] = acc[ct][b];
      p_lt = lt;
      p_ns = ns;
      p_nvs = nvs;
      p_nvel = nvel;
      p_ncols = tl.ncols;
    }
  __syncthreads(); // Z of the last tile complete
  stage3();
}
} // namespace

cudaError_t
launch_vanka_fac(const DevPatchClass *classes, const VankaTile *tiles, const long long *va, const long long *pa,
                 const int *tile_ptr, int n_blocks, int ng_full, const FacParams &F, const double *r, double *u,
                 long long isz, int n_intervals, double omega, cudaStream_t stream)
{
  if (n_blocks == 0 || n_intervals == 0)
    return cudaSuccess;
  dim3 grid(n_blocks, (n_intervals + ng_full - 1) / ng_full);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kFSmem));
    kern<<<grid, kTThreads, kFSmem, stream>>>(classes, tiles, va, pa, tile_ptr, ng_full, r, u, isz, n_intervals,
                                              omega, F);
  };
  // instantiations with S * NSP <= kTRows (host: setup.cpp factored form)
#define STMG_FAC_CASE(SS, NN)                                                                                          \
  if (F.S == SS && F.nsp == NN)                                                                                        \
    {                                                                                                                  \
      go(vanka_fac_kernel<SS, NN>);                                                                                    \
      return cudaGetLastError();                                                                                       \
    }
  STMG_FAC_CASE(3, 16)
  STMG_FAC_CASE(3, 24)
  STMG_FAC_CASE(3, 32)
  STMG_FAC_CASE(3, 40)
  STMG_FAC_CASE(4, 16)
  STMG_FAC_CASE(4, 24)
  STMG_FAC_CASE(4, 32)
  STMG_FAC_CASE(5, 16)
  STMG_FAC_CASE(5, 24)
#undef STMG_FAC_CASE
  return cudaErrorInvalidValue; // host only enables the factored form for these shapes
  return cudaGetLastError();
}

cudaError_t
launch_vanka_tc(const DevPatchClass *classes, const VankaTile *tiles, const long long *va, const long long *pa,
                const int *tile_ptr, int n_blocks, int ng_full, int max_nt, const double *r, double *u, long long isz,
                int n_intervals, double omega, cudaStream_t stream)
{
  if (n_blocks == 0 || n_intervals == 0)
    return cudaSuccess;
  dim3 grid(n_blocks, (n_intervals + ng_full - 1) / ng_full);
  const int ks = (max_nt + 3) / 4;
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kTSmem));
    kern<<<grid, kTThreads, kTSmem, stream>>>(classes, tiles, va, pa, tile_ptr, ng_full, r, u, isz, n_intervals,
                                              omega);
  };
  // deferred-scatter kernel by default (A/B switch STMG_VANKA_KERNEL=tc)
  static const int variant = [] {
    const char *e = std::getenv("STMG_VANKA_KERNEL");
    return (e && std::string(e) == "tc") ? 0 : 1;
  }();
  auto gd = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kDSmem));
    kern<<<grid, kTThreads, kDSmem, stream>>>(classes, tiles, va, pa, tile_ptr, ng_full, r, u, isz, n_intervals,
                                              omega);
  };
  if (variant == 1)
    {
      // exact k-step counts of the cell patches the hierarchies meet
      // (n_T = 21, 38, 42, 76: Q2/P1 x DG(0), Q3/P2 x DG(0), Q2/P1 x DG(1),
      // Q3/P2 x DG(1)), so no zero k-steps are multiplied
      if (ks <= 6)
        gd(vanka_dfr_kernel<6>);
      else if (ks <= 8)
        gd(vanka_dfr_kernel<8>);
      else if (ks <= 10)
        gd(vanka_dfr_kernel<10>);
      else if (ks <= 11)
        gd(vanka_dfr_kernel<11>);
      else if (ks <= 12)
        gd(vanka_dfr_kernel<12>);
      else if (ks <= 16)
        gd(vanka_dfr_kernel<16>);
      else if (ks <= 19)
        gd(vanka_dfr_kernel<19>);
      else if (ks <= 20)
        gd(vanka_dfr_kernel<20>);
      else if (ks <= 24)
        gd(vanka_dfr_kernel<24>);
      else if (ks <= 29)
        gd(vanka_dfr_kernel<29>);
      else if (ks <= 31) // vertex stars of Q2/P1disc x DG(1): n_T = 124
        gd(vanka_dfr_kernel<31>);
      else
        gd(vanka_dfr_kernel<32>);
      return cudaGetLastError();
    }
  if (ks <= 8)
    go(vanka_tc_kernel<8>);
  else if (ks <= 12)
    go(vanka_tc_kernel<12>);
  else if (ks <= 16)
    go(vanka_tc_kernel<16>);
  else if (ks <= 20)
    go(vanka_tc_kernel<20>);
  else if (ks <= 24)
    go(vanka_tc_kernel<24>);
  else if (ks <= 29)
    go(vanka_tc_kernel<29>);
  else
    go(vanka_tc_kernel<32>);
  return cudaGetLastError();
}

cudaError_t
launch_vanka_dfr176(const DevPatchClass *classes, const VankaBatch *batches, int n_batches, int max_nt,
                    const long long *vel_anchor, const long long *pre_anchor, const double *r, double *u,
                    long long isz, int n_intervals, double omega, int group, cudaStream_t stream)
{
  if (n_batches == 0 || n_intervals == 0)
    return cudaSuccess;
  if (max_nt > k3Rows || group * vanka_cols_per_batch() > k3MaxCols)
    return cudaErrorInvalidValue;
  const size_t smem = sizeof(double) * kTRing * k3Slot + k3MaxCols * 12 + 6 * sizeof(unsigned long long);
  dim3 grid(n_batches, (n_intervals + group - 1) / group, 2);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kern<<<grid, k3Threads, smem, stream>>>(classes, batches, vel_anchor, pre_anchor, r, u, isz, n_intervals, omega,
                                            group);
  };
  if (max_nt <= 4 * (k3KS - 1))
    go(vanka_dfr176_kernel<k3KS - 1>);
  else
    go(vanka_dfr176_kernel<k3KS>);
  return cudaGetLastError();
}

int
vanka_tc_cols()
{
  return kTCols;
}

bool
vanka_fac_supported(int S, int nsp)
{
  return (S == 3 && (nsp == 16 || nsp == 24 || nsp == 32 || nsp == 40)) ||
         (S == 4 && (nsp == 16 || nsp == 24 || nsp == 32)) || (S == 5 && (nsp == 16 || nsp == 24));
}

int
vanka_tc_max_tiles()
{
  return kTMaxTiles;
}

} // namespace stmg_b200
