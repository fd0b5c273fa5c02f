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
//  * Thread mapping: warp = one output slot a, lane = one cell of a strip of
//    31 owned cells (+1 halo cell on the left). A block marches upward through
//    a segment of cell rows. Contributions to shared nodes are summed with
//    __shfl_up_sync across the strip (x) and a register carry (y): no atomics,
//    no zero-fill pass, every output written exactly once. Halo work: 1/31 in
//    x, 1/rows_per_seg in y.
#pragma once
#include "level_consts.cuh"

#include <cstdint>
#include <cuda_runtime.h>

namespace stmg_b200
{

namespace vmult_detail
{
constexpr int kStrip = 31; // owned cells per warp strip

// The 1D factors of a Cartesian level are symmetric under i<->k (M1, K1) and
// under the reflection i -> N-1-i (M1, K1 even; C1, Lm, Lc even or odd). The
// host stores them exactly symmetrised; the kernel reads every entry through
// its canonical representative (compile-time index + sign), so only ~40
// distinct coefficients exist per level instead of ~200 and they stay in
// uniform registers.
template <int N>
__host__ __device__ constexpr int
canon_sym(int i, int k)
{
  const int a = i * N + k, b = k * N + i, c = (N - 1 - i) * N + (N - 1 - k), d = (N - 1 - k) * N + (N - 1 - i);
  const int m1 = a < b ? a : b, m2 = c < d ? c : d;
  return m1 < m2 ? m1 : m2;
}
template <int N>
__host__ __device__ constexpr int
canon_refl(int i, int k)
{
  const int a = i * N + k, c = (N - 1 - i) * N + (N - 1 - k);
  return a < c ? a : c;
}
template <int N>
__host__ __device__ constexpr double
sign_refl(int i, int k) // C1(N-1-i, N-1-k) = -C1(i, k)
{
  return (i * N + k) <= ((N - 1 - i) * N + (N - 1 - k)) ? 1.0 : -1.0;
}
#define VM_M(i, k) (P.cM1[canon_sym<N1>((i), (k))])
#define VM_K(i, k) (P.cK1[canon_sym<N1>((i), (k))])
#define VM_C(i, k) (sign_refl<N1>((i), (k)) * P.cC1[canon_refl<N1>((i), (k))])
// Lm(a, N-1-k) = (-1)^a Lm(a, k);  Lc(a, N-1-k) = (-1)^(a+1) Lc(a, k)
#define VM_LM(a, k) (((k) > N1 - 1 - (k) && ((a) & 1)) ? -P.cLm[(a) * N1 + N1 - 1 - (k)] \
                                                          : P.cLm[(a) * N1 + ((k) > N1 - 1 - (k) ? N1 - 1 - (k) : (k))])
#define VM_LC(a, k) (((k) > N1 - 1 - (k) && !((a) & 1)) ? -P.cLc[(a) * N1 + N1 - 1 - (k)] \
                                                           : P.cLc[(a) * N1 + ((k) > N1 - 1 - (k) ? N1 - 1 - (k) : (k))])

// Shared-memory staging, one NODE ROW of the strip at a time (all input
// slots, both components, the previous interval's slot-k velocity; with node
// row 0 of a cell row also the cell row's pressure), double-buffered with
// cp.async one node row ahead. Warp b stages input slot b with a fixed
// lane -> node mapping (one address add per copy), so the contractions read
// shared memory instead of waiting on global loads.
#ifndef STMG_VM_STAGE_R1
#define STMG_VM_STAGE_R1 1 // staging of r = 1 plain applications: 0 direct loads, 1 cp.async, 2 bulk copies
#endif
#ifndef STMG_VM_STAGE_R1_RESID
#define STMG_VM_STAGE_R1_RESID 0
#endif
#ifndef STMG_VM_STAGE_R2
#define STMG_VM_STAGE_R2 0
#endif
#ifndef STMG_VM_STAGE_R2_RESID
#define STMG_VM_STAGE_R2_RESID 0
#endif
template <int R, int S>
struct RowStage
{
  static constexpr int p = R + 1, NPM = (R + 1) * (R + 2) / 2;
  static constexpr int VW = 32 * p + 1;          // nodes of one strip row
  static constexpr int NBUF = (2 * S + 2) * VW;  // one node row: S slots x 2 comps + v_prev x 2 comps
  static constexpr int NPRE = S * 32 * NPM;      // pressure of one cell row
  static constexpr size_t kBytes = sizeof(double) * (2 * NBUF + NPRE);
  // bulk-copy (TMA engine, cp.async.bulk) layout: every row padded to VWB
  // doubles so a 16-byte aligned superset of the strip row fits (the node
  // grid is odd-sized: rows start at any 8-byte offset)
  static constexpr int VWB = (VW + 3 + 1) / 2 * 2;
  static constexpr int NBUFB = (2 * S + 2) * VWB;
  static constexpr int PB = (32 * NPM + 3 + 1) / 2 * 2;
#ifndef STMG_VM_BULK_LAG
#define STMG_VM_BULK_LAG 0 // 0: block barrier per node row; L >= 1: per-buffer empty mbarriers, refill L rows behind
#endif
#ifndef STMG_VM_BULK_DEPTH
#define STMG_VM_BULK_DEPTH (STMG_VM_BULK_LAG ? 5 : 4)
#endif
  static constexpr int DEPTH = STMG_VM_BULK_DEPTH; // bulk ring: node rows issued up to DEPTH - 1 rows ahead
  static constexpr int LAG = STMG_VM_BULK_LAG;
  static constexpr size_t kBytesBulk =
    sizeof(double) * (DEPTH * NBUFB + 2 * S * PB) + 2 * DEPTH * sizeof(unsigned long long);
  // Measured per instantiation (C2 r = 2 and C4 r = 1 on the B200): cp.async
  // staging wins for r = 1 plain applications (C4 vmult 1.66 -> 1.26 ms) and
  // loses for r = 2 (2.63 -> 2.80 ms) and for residuals (their late b loads
  // stall in lockstep behind the per-row barriers), which keep direct loads.
  template <bool RESID>
  __host__ __device__ static constexpr int mode()
  {
#ifdef STMG_VM_NOSTAGE
    return 0;
#else
    return R == 1 ? (RESID ? STMG_VM_STAGE_R1_RESID : STMG_VM_STAGE_R1)
                  : (R == 2 ? (RESID ? STMG_VM_STAGE_R2_RESID : STMG_VM_STAGE_R2) : 0);
#endif
  }
  template <bool RESID>
  __host__ __device__ static constexpr bool on()
  {
    return mode<RESID>() != 0;
  }
  template <bool RESID>
  static constexpr size_t bytes()
  {
    return mode<RESID>() == 2 ? kBytesBulk : (mode<RESID>() == 1 ? kBytes : 0);
  }
};

__device__ __forceinline__ unsigned
vm_smem_u32(const void *p)
{
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// One bulk copy of the 16-byte aligned superset of src[lo, hi) into the
// row buffer whose element 0 is global element base_al (16-byte aligned):
// returns the bytes in flight for the mbarrier's transaction count.
__device__ __forceinline__ unsigned
vm_bulk_row(double *row, const double *base_al, const double *lo, const double *hi, unsigned long long *bar)
{
  if (hi <= lo)
    return 0;
  const double *a = reinterpret_cast<const double *>(reinterpret_cast<uintptr_t>(lo) & ~uintptr_t(15));
  const double *e = reinterpret_cast<const double *>((reinterpret_cast<uintptr_t>(hi) + 15) & ~uintptr_t(15));
  const unsigned bytes = static_cast<unsigned>((e - a) * sizeof(double));
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                 vm_smem_u32(row + (a - base_al))),
               "l"(a), "r"(bytes), "r"(vm_smem_u32(bar))
               : "memory");
  return bytes;
}
__device__ __forceinline__ const double *
vm_align_down(const double *q)
{
  return reinterpret_cast<const double *>(reinterpret_cast<uintptr_t>(q) & ~uintptr_t(15));
}

__device__ __forceinline__ void
vm_cp_async8(double *dst, const double *src)
{
  const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(saddr), "l"(src));
}

#ifndef STMG_VM_MINB1
#define STMG_VM_MINB1 8 // r = 1: 128 registers (C4 residual 1.96 -> 1.50 ms; 96 and 80 registers spill)
#endif
#ifndef STMG_VM_MINB2
#define STMG_VM_MINB2 3 // r = 2: 168 registers, 12 warps per SM
#endif
#ifndef STMG_VM_CARRYIN
#define STMG_VM_CARRYIN 1 // the cell-row carry enters the next row's tile at its start (C2 vmult 2.56 -> 2.51 ms)
#endif
#ifndef STMG_VM_PF
#define STMG_VM_PF 0 // 1: L1 prefetch (prefetch.global.L1) of the next node row, one line per lane; 2: also the next cell row's pressure. Measured slower: C2 vmult 2.51 -> 2.81 (1) / 2.96 ms (2)
#endif
#ifndef STMG_VM_BINIT
#define STMG_VM_BINIT 0 // 1: residual tile starts at -b (loads issued with the row's x loads): spills at the 168-register cap, C2 residual 2.96 -> 3.51 ms
#endif
#ifdef STMG_VM_MAXNREG // experiment: an explicit register target instead of the launch bounds
#define STMG_VM_BOUNDS __maxnreg__(STMG_VM_MAXNREG)
#else
#define STMG_VM_BOUNDS __launch_bounds__(32 * S, R == 2 ? STMG_VM_MINB2 : (R == 1 ? STMG_VM_MINB1 : 1))
#endif
template <int R, int S, bool RESID, bool RAW>
__global__ void STMG_VM_BOUNDS
vmult_kernel(const LevelConsts P, const double *__restrict__ x, const double *__restrict__ b,
             double *__restrict__ y, const double *__restrict__ xprev0, int rows_per_seg, int coupled)
{
  constexpr int N1 = R + 2, p = R + 1, NPM = (R + 1) * (R + 2) / 2, PL = R + 1;
  const int lane = threadIdx.x & 31;
  const int a = threadIdx.x >> 5; // output slot
  const int n = blockIdx.z;       // interval
  const int cx = blockIdx.x * kStrip - 1 + lane;
  const bool active = cx >= 0 && cx < P.nx;
  const bool owner = lane >= 1 && active;

  const long long isz = P.isz, mv = P.mv, mp = P.mp, nsc = P.nsc;
  const int gx = P.gx, gy = P.gy;
  const double *__restrict__ xn = x + n * isz;
  const double *__restrict__ vprev = nullptr;
  if (coupled)
    vprev = n > 0 ? x + (n - 1) * isz + (S - 1) * mv : xprev0;

  // Temporal coefficients of this warp's output slot, selected with
  // compile-time indices so the parameter bank is never indexed dynamically.
  double kt[S], mt[S], lva = 0.0;
#pragma unroll
  for (int bs = 0; bs < S; ++bs)
    kt[bs] = mt[bs] = 0.0;
#pragma unroll
  for (int aa = 0; aa < S; ++aa)
    if (a == aa)
      {
#pragma unroll
        for (int bs = 0; bs < S; ++bs)
          {
            kt[bs] = P.KtJ[aa * S + bs];
            mt[bs] = P.MtJ[aa * S + bs];
          }
        lva = P.lvJ[aa];
      }

  const int cy_begin = blockIdx.y * rows_per_seg;
  const int cy_end = min(P.ny, cy_begin + rows_per_seg);
  const int cy_first = max(cy_begin - 1, 0);

  double carx[N1], cary[N1];
#pragma unroll
  for (int i = 0; i < N1; ++i)
    carx[i] = cary[i] = 0.0;

  using RS = RowStage<R, S>;
  constexpr bool kStaged = RS::template on<RESID>();
  constexpr bool kBulk = RS::template mode<RESID>() == 2;
  constexpr int RW = kBulk ? RS::VWB : RS::VW;  // row pitch of the staging buffers
  constexpr int NB = kBulk ? RS::NBUFB : RS::NBUF;
  constexpr int PP = kBulk ? RS::PB : 32 * NPM; // pressure pitch per slot
  extern __shared__ __align__(16) double vm_smem[];
  constexpr int RING = kBulk ? RS::DEPTH : 2;
  double *const pre_s = vm_smem + RING * NB;
  unsigned long long *const vm_bar = reinterpret_cast<unsigned long long *>(pre_s + (kBulk ? 2 : 1) * S * PP);
  const int X0 = (blockIdx.x * kStrip - 1) * p; // first node column of the strip
  const int cx0 = blockIdx.x * kStrip - 1;
  // bulk path: element j of a staged row sits at j + delta, delta = 8-byte
  // misalignment of the row's first node (the buffer starts 16-byte aligned)
  auto row_src = [&](int r2, int cyy, int l) -> const double * {
    const long long rowoff = static_cast<long long>(cyy * p + l) * gx + X0;
    return r2 < 2 * S ? xn + (r2 >> 1) * mv + (r2 & 1) * nsc + rowoff : vprev + (r2 & 1) * nsc + rowoff;
  };
  auto pre_src = [&](int bs, int cyy) -> const double * {
    return xn + S * mv + bs * mp + (static_cast<long long>(cyy) * P.nx + cx0) * NPM;
  };
  auto mis = [](const double *q) -> int { return static_cast<int>((reinterpret_cast<uintptr_t>(q) >> 3) & 1); };
  if constexpr (kBulk)
    {
      if (threadIdx.x == 0)
        {
          for (int q = 0; q < RING; ++q)
            {
              asm volatile("mbarrier.init.shared.b64 [%0], 1;\n" ::"r"(vm_smem_u32(vm_bar + q)));
              asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(vm_smem_u32(vm_bar + RING + q)), "r"(S));
            }
          asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
      __syncthreads();
    }
  // node row l of cell row cyy (and, for l == 0, its pressure) into buffer
  // buf by bulk copies: lane q of warp 0 issues copy q (its bytes announced
  // with expect_tx first), lane 0 arrives once the warp has issued them all
  auto stage_row_bulk = [&](int cyy, int l, int buf) {
    if (threadIdx.x >= 32)
      return;
    unsigned long long *bar = vm_bar + buf;
    const int nrows = vprev != nullptr ? 2 * S + 2 : 2 * S;
    const int q = threadIdx.x;
    const double *src = nullptr, *lo = nullptr, *hi = nullptr;
    double *row = nullptr;
    if (q < nrows)
      {
        src = row_src(q, cyy, l);
        lo = src + max(0, -X0);             // strip-row nodes inside the grid
        hi = src + min(RS::VW, gx - X0);
        row = vm_smem + buf * NB + q * RW;
      }
    else if (l == 0 && q < nrows + S)
      {
        const int bs = q - nrows;
        src = pre_src(bs, cyy);
        lo = src + (max(cx0, 0) - cx0) * NPM;
        hi = src + (min(cx0 + 32, P.nx) - cx0) * NPM;
        row = pre_s + ((cyy & 1) * S + bs) * PP;
      }
    if (src != nullptr && hi > lo)
      {
        const double *al = vm_align_down(lo);
        const double *e = reinterpret_cast<const double *>((reinterpret_cast<uintptr_t>(hi) + 15) & ~uintptr_t(15));
        const unsigned bytes = static_cast<unsigned>((e - al) * sizeof(double));
        asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;\n" ::"r"(vm_smem_u32(bar)), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                       vm_smem_u32(row + (al - vm_align_down(src)))),
                     "l"(al), "r"(bytes), "r"(vm_smem_u32(bar))
                     : "memory");
      }
    __syncwarp();
    if (q == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(vm_smem_u32(bar)) : "memory");
  };
  // gather node row l of cell row cyy (and, for l == 0, its pressure) into buffer buf
  auto stage_row = [&](int cyy, int l, int buf) {
    if constexpr (kBulk)
      {
        stage_row_bulk(cyy, l, buf);
        return;
      }
    double *dst = vm_smem + buf * RS::NBUF;
    const long long rowoff = static_cast<long long>(cyy * p + l) * gx + X0;
#pragma unroll
    for (int comp = 0; comp < 2; ++comp)
#pragma unroll
      for (int q = 0; q < (RS::VW + 31) / 32; ++q)
        {
          const int j = lane + 32 * q;
          if (j < RS::VW && X0 + j >= 0 && X0 + j < gx)
            {
              vm_cp_async8(dst + (a * 2 + comp) * RS::VW + j, xn + a * mv + comp * nsc + rowoff + j);
              if (a == 0 && vprev != nullptr)
                vm_cp_async8(dst + (2 * S + comp) * RS::VW + j, vprev + comp * nsc + rowoff + j);
            }
        }
    if (l == 0)
      {
        const double *src = xn + S * mv + a * mp + (static_cast<long long>(cyy) * P.nx + cx0) * NPM;
#pragma unroll
        for (int q = 0; q < NPM; ++q)
          {
            const int e = lane + 32 * q, c = e / NPM;
            if (cx0 + c >= 0 && cx0 + c < P.nx)
              vm_cp_async8(pre_s + a * 32 * NPM + e, src + e);
          }
      }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  // wait for node row (cy, l), then prefetch the next node row of the march
  auto stage_sync = [&](int cy, int l) {
    if constexpr (kStaged)
      {
        if constexpr (kBulk)
          {
            const int s0 = (cy - cy_first) * N1 + l;
            asm volatile("{\n .reg .pred p;\n VMW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                         " @!p bra VMW_%=;\n}\n" ::"r"(vm_smem_u32(vm_bar + s0 % RING)),
                         "r"((s0 / RING) & 1)
                         : "memory");
            if constexpr (RS::LAG == 0)
              {
                __syncthreads(); // everybody is past row s0 - 1: its buffer takes row s0 + RING - 1
                const int s = s0 + RING - 1, cyn = cy_first + s / N1;
                if (cyn < cy_end)
                  stage_row(cyn, s % N1, s % RING);
              }
            else
              {
                // no block barrier: a warp releases row s0 - 1 on that buffer's
                // empty mbarrier (one arrival per warp); the issuing warp refills
                // the buffer of row s0 - LAG once all warps have released it, so
                // the warps of a block drift up to LAG rows apart
                if (s0 > 0)
                  {
                    __syncwarp();
                    if (lane == 0)
                      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(
                                     vm_smem_u32(vm_bar + RING + (s0 - 1) % RING))
                                   : "memory");
                  }
                const int sr = s0 - RS::LAG, s = sr + RING, cyn = cy_first + s / N1;
                if (threadIdx.x < 32 && sr >= 0 && cyn < cy_end)
                  {
                    asm volatile("{\n .reg .pred p;\n VME_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                                 " @!p bra VME_%=;\n}\n" ::"r"(vm_smem_u32(vm_bar + RING + sr % RING)),
                                 "r"((sr / RING) & 1)
                                 : "memory");
                    stage_row(cyn, s % N1, s % RING);
                  }
              }
            return;
          }
        else
          asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
        const int s = (cy - cy_first) * N1 + l + 1;
        if (l + 1 < N1)
          stage_row(cy, l + 1, s & 1);
        else if (cy + 1 < cy_end)
          stage_row(cy + 1, 0, s & 1);
      }
  };
  if constexpr (kStaged)
    {
      if constexpr (kBulk)
        {
          for (int s = 0; s < (RS::LAG ? RING : RING - 1); ++s)
            if (cy_first + s / N1 < cy_end)
              stage_row(cy_first + s / N1, s % N1, s);
        }
      else if (cy_first < cy_end)
        stage_row(cy_first, 0, 0);
    }

  for (int cy = cy_first; cy < cy_end; ++cy)
    {
      double Yx[N1][N1], Yy[N1][N1], Yp[NPM];
      stage_sync(cy, 0);
#pragma unroll
      for (int i = 0; i < N1; ++i)
#pragma unroll
        for (int j = 0; j < N1; ++j)
          Yx[i][j] = Yy[i][j] = 0.0;
#pragma unroll
      for (int m = 0; m < NPM; ++m)
        Yp[m] = 0.0;
#if STMG_VM_CARRYIN
      // the row below's (pre-assembly) top node row enters the bottom node
      // row here, so the carry is not live during the contractions
      if (cy > cy_first)
#pragma unroll
        for (int i = 0; i < N1; ++i)
          {
            Yx[i][0] = carx[i];
            Yy[i][0] = cary[i];
          }
#endif

      if constexpr (RESID && STMG_VM_BINIT)
        {
          // r = b - A x as -( -b + A x ): b of the nodes this cell writes enters
          // the accumulators here, so its loads are in flight with the x loads
          // of the first node row instead of stalling the write-out
          if (owner && cy >= cy_begin)
            {
              const int ixmax = (cx == P.nx - 1) ? p : p - 1;
              const int iymax = (cy == P.ny - 1) ? p : p - 1;
              const long long obase = n * isz + a * mv;
#pragma unroll
              for (int j = 0; j < N1; ++j)
#pragma unroll
                for (int i = 0; i < N1; ++i)
                  if (i <= ixmax && j <= iymax)
                    {
                      const long long node = static_cast<long long>(cy * p + j) * gx + cx * p + i;
                      Yx[i][j] -= __ldg(b + obase + node);
                      Yy[i][j] -= __ldg(b + obase + nsc + node);
                    }
              const long long pbase = n * isz + S * mv + a * mp + (static_cast<long long>(cy) * P.nx + cx) * NPM;
#pragma unroll
              for (int m = 0; m < NPM; ++m)
                Yp[m] = -__ldg(b + pbase + m);
            }
        }

      if (active)
        {
          const long long cell = static_cast<long long>(cy) * P.nx + cx;
          // ---- pressure: PM = sum_b Mt(a,b) p^b; B^T init of Yx, Yy
          {
            double PM[NPM];
#pragma unroll
            for (int m = 0; m < NPM; ++m)
              PM[m] = 0.0;
#pragma unroll
            for (int bs = 0; bs < S; ++bs)
              {
                const double c = mt[bs];
                const double *pp = xn + S * mv + bs * mp + cell * NPM;
                const double *ps = kBulk ? pre_s + ((cy & 1) * S + bs) * PP + mis(pre_src(bs, cy)) + lane * NPM
                                         : pre_s + (bs * 32 + lane) * NPM;
#pragma unroll
                for (int m = 0; m < NPM; ++m)
                  PM[m] = fma(c, kStaged ? ps[m] : __ldg(pp + m), PM[m]);
              }
            // Yx(i,j) -= sum_b Qx(i,b) yLm(b,j),  Qx(i,b) = sum_{m: ay=b} xLc(ax,i) PM_m
            // Yy(i,j) -= sum_b Qy(i,b) yLc(b,j),  Qy(i,b) = sum_{m: ay=b} xLm(ax,i) PM_m
#pragma unroll
            for (int bb = 0; bb < PL; ++bb)
              {
                double Qx[N1], Qy[N1];
#pragma unroll
                for (int i = 0; i < N1; ++i)
                  Qx[i] = Qy[i] = 0.0;
#pragma unroll
                for (int m = 0; m < NPM; ++m)
                  {
                    if (pdisc_mode_ay(R, m) != bb)
                      continue;
                    const int am = pdisc_mode_ax(R, m);
#pragma unroll
                    for (int i = 0; i < N1; ++i)
                      {
                        Qx[i] = fma(VM_LC(am, i), PM[m], Qx[i]);
                        Qy[i] = fma(VM_LM(am, i), PM[m], Qy[i]);
                      }
                  }
#pragma unroll
                for (int i = 0; i < N1; ++i)
                  {
                    Qx[i] *= P.scx; // -cx B^T / -cy B^T
                    Qy[i] *= P.scy;
                  }
#pragma unroll
                for (int i = 0; i < N1; ++i)
#pragma unroll
                  for (int j = 0; j < N1; ++j)
                    {
                      Yx[i][j] = fma(-Qx[i], VM_LM(bb, j), Yx[i][j]);
                      Yy[i][j] = fma(-Qy[i], VM_LC(bb, j), Yy[i][j]);
                    }
              }
          }

        }

      // ---- velocity rows of the cell
#pragma unroll
      for (int l = 0; l < N1; ++l)
        {
          if (l > 0)
            stage_sync(cy, l);
          const double *sb = vm_smem + (((cy - cy_first) * N1 + l) % RING) * NB;
          if constexpr (!kStaged && STMG_VM_PF != 0)
            {
              // L1 prefetch of the NEXT node row of the strip (all input slots,
              // both components, the previous interval's velocity), one 128-byte
              // line per lane: ncu puts a third of the stall samples on the first
              // use of a row's loads (L2 latency at 11 warps per SM)
              const int Yn = cy * p + l + 1;
              constexpr int kLines = (32 * p + 1 + 15) / 16 + 1;
              if (lane < kLines && Yn < gy && (l < N1 - 1 || cy + 1 < cy_end))
                {
                  const int Xc = min(max(X0 + 16 * lane, 0), gx - 1);
                  const long long off = static_cast<long long>(Yn) * gx + Xc;
#pragma unroll
                  for (int bs = 0; bs < S; ++bs)
                    {
                      asm volatile("prefetch.global.L1 [%0];\n" ::"l"(xn + bs * mv + off));
                      asm volatile("prefetch.global.L1 [%0];\n" ::"l"(xn + bs * mv + nsc + off));
                    }
                  if (vprev != nullptr)
                    {
                      asm volatile("prefetch.global.L1 [%0];\n" ::"l"(vprev + off));
                      asm volatile("prefetch.global.L1 [%0];\n" ::"l"(vprev + nsc + off));
                    }
                }
              if (STMG_VM_PF > 1 && l == 1 && cy + 1 < cy_end)
                {
                  constexpr int kPLines = (32 * NPM + 15) / 16 + 1;
                  const long long c0 = (static_cast<long long>(cy + 1) * P.nx + max(cx0, 0)) * NPM + 16 * lane;
                  if (lane < kPLines && c0 < mp)
#pragma unroll
                    for (int bs = 0; bs < S; ++bs)
                      asm volatile("prefetch.global.L1 [%0];\n" ::"l"(xn + S * mv + bs * mp + c0));
                }
            }
          if (active)
            {
              const int Y = cy * p + l;
              const bool yb = (Y == 0) || (Y == gy - 1);
              const long long rowbase = static_cast<long long>(Y) * gx + cx * p;
              double UKx[N1], UMx[N1], UKy[N1], UMy[N1];
#pragma unroll
              for (int k = 0; k < N1; ++k)
                {
                  const int X = cx * p + k;
                  const bool bnd = !RAW && (yb || X == 0 || X == gx - 1);
                  const long long node = rowbase + k;
                  double ukx = 0.0, umx = 0.0, uky = 0.0, umy = 0.0;
                  const int js = lane * p + k; // node column within the staged strip row
#pragma unroll
                  for (int bs = 0; bs < S; ++bs)
                    {
                      const int dx = kBulk ? mis(row_src(2 * bs, cy, l)) : 0;
                      const int dy = kBulk ? mis(row_src(2 * bs + 1, cy, l)) : 0;
                      const double vx =
                        bnd ? 0.0 : (kStaged ? sb[(bs * 2 + 0) * RW + js + dx] : __ldg(xn + bs * mv + node));
                      const double vy =
                        bnd ? 0.0 : (kStaged ? sb[(bs * 2 + 1) * RW + js + dy] : __ldg(xn + bs * mv + nsc + node));
                      ukx = fma(kt[bs], vx, ukx);
                      umx = fma(mt[bs], vx, umx);
                      uky = fma(kt[bs], vy, uky);
                      umy = fma(mt[bs], vy, umy);
                    }
                  if (vprev != nullptr)
                    {
                      const int dx = kBulk ? mis(row_src(2 * S, cy, l)) : 0;
                      const int dy = kBulk ? mis(row_src(2 * S + 1, cy, l)) : 0;
                      ukx = fma(-lva, kStaged ? sb[(2 * S + 0) * RW + js + dx] : __ldg(vprev + node), ukx);
                      uky = fma(-lva, kStaged ? sb[(2 * S + 1) * RW + js + dy] : __ldg(vprev + nsc + node), uky);
                    }
                  UKx[k] = ukx;
                  UMx[k] = umx;
                  UKy[k] = uky;
                  UMy[k] = umy;
                }
              // scaled copies of the combined inputs (coefficients of the
              // stiffness parts: (nu+gamma) cx^2 and nu cx^2)
              double UMxa[N1], UMyb[N1];
#pragma unroll
              for (int k = 0; k < N1; ++k)
                {
                  UMxa[k] = P.sax * UMx[k];
                  UMyb[k] = P.say * UMy[k];
                }
              // x-contraction for output column i, immediately folded into the
              // y-accumulation (keeps only the running Yx/Yy tiles live)
#pragma unroll
              for (int i = 0; i < N1; ++i)
                {
                  double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0;
#pragma unroll
                  for (int k = 0; k < N1; ++k)
                    {
                      s0 = fma(VM_M(i, k), UKx[k], s0);
                      s0 = fma(VM_K(i, k), UMxa[k], s0);
                      s1 = fma(VM_M(i, k), UMx[k], s1);
                      s2 = fma(VM_C(i, k), UMy[k], s2);
                      s3 = fma(VM_M(i, k), UKy[k], s3);
                      s3 = fma(VM_K(i, k), UMyb[k], s3);
                      s4 = fma(VM_M(i, k), UMy[k], s4);
                      s5 = fma(VM_C(k, i), UMx[k], s5);
                    }
                  s1 *= P.sbx; // nu cy^2
                  s2 *= P.sg;  // gamma cx cy
                  s4 *= P.sby; // (nu+gamma) cy^2
                  s5 *= P.sg;
#pragma unroll
                  for (int j = 0; j < N1; ++j)
                    {
                      double vx = Yx[i][j], vy = Yy[i][j];
                      vx = fma(VM_M(j, l), s0, vx);
                      vx = fma(VM_K(j, l), s1, vx);
                      vx = fma(VM_C(l, j), s2, vx);
                      vy = fma(VM_M(j, l), s3, vy);
                      vy = fma(VM_K(j, l), s4, vy);
                      vy = fma(VM_C(j, l), s5, vy);
                      Yx[i][j] = vx;
                      Yy[i][j] = vy;
                    }
                }
              double dp[PL], ep[PL];
#pragma unroll
              for (int aa = 0; aa < PL; ++aa)
                {
                  double s0 = 0, s1 = 0;
#pragma unroll
                  for (int k = 0; k < N1; ++k)
                    {
                      s0 = fma(VM_LC(aa, k), UMx[k], s0);
                      s1 = fma(VM_LM(aa, k), UMy[k], s1);
                    }
                  dp[aa] = s0 * P.scx;
                  ep[aa] = s1 * P.scy;
                }
#pragma unroll
              for (int m = 0; m < NPM; ++m)
                {
                  const int am = pdisc_mode_ax(R, m), bm = pdisc_mode_ay(R, m);
                  Yp[m] = fma(VM_LM(bm, l), dp[am], Yp[m]);
                  Yp[m] = fma(VM_LC(bm, l), ep[am], Yp[m]);
                }
            }
        }

      // ---- assemble shared nodes: x across lanes, y through the carry
#if STMG_VM_CARRYIN
#pragma unroll
      for (int i = 0; i < N1; ++i)
        {
          carx[i] = Yx[i][N1 - 1];
          cary[i] = Yy[i][N1 - 1];
        }
#endif
#pragma unroll
      for (int j = 0; j < N1; ++j)
        {
          const double lx = __shfl_up_sync(0xffffffffu, Yx[N1 - 1][j], 1);
          const double ly = __shfl_up_sync(0xffffffffu, Yy[N1 - 1][j], 1);
          if (lane > 0)
            {
              Yx[0][j] += lx;
              Yy[0][j] += ly;
            }
        }
#if !STMG_VM_CARRYIN
      if (cy > cy_first)
#pragma unroll
        for (int i = 0; i < N1; ++i)
          {
            Yx[i][0] += carx[i];
            Yy[i][0] += cary[i];
          }
#pragma unroll
      for (int i = 0; i < N1; ++i)
        {
          carx[i] = Yx[i][N1 - 1];
          cary[i] = Yy[i][N1 - 1];
        }
#endif

      // ---- write owned outputs
      if (owner && cy >= cy_begin)
        {
          const int ixmax = (cx == P.nx - 1) ? p : p - 1;
          const int iymax = (cy == P.ny - 1) ? p : p - 1;
          const long long obase = n * isz + a * mv;
#pragma unroll
          for (int j = 0; j < N1; ++j)
            {
              if (j > iymax)
                continue;
              const int Y = cy * p + j;
              const bool yb = (Y == 0) || (Y == gy - 1);
#pragma unroll
              for (int i = 0; i < N1; ++i)
                {
                  if (i > ixmax)
                    continue;
                  const int X = cx * p + i;
                  const long long node = static_cast<long long>(Y) * gx + X;
                  double vx = Yx[i][j], vy = Yy[i][j];
                  if constexpr (RESID && STMG_VM_BINIT)
                    {
                      vx = -vx;
                      vy = -vy;
                      if (!RAW && (yb || X == 0 || X == gx - 1))
                        {
                          vx = __ldg(b + obase + node) - __ldg(x + obase + node);
                          vy = __ldg(b + obase + nsc + node) - __ldg(x + obase + nsc + node);
                        }
                    }
                  else
                    {
                      if (!RAW && (yb || X == 0 || X == gx - 1))
                        {
                          // identity rows on constrained velocity dofs (st_operator.cpp:383-394)
                          vx = __ldg(x + obase + node);
                          vy = __ldg(x + obase + nsc + node);
                        }
                      if (RESID)
                        {
                          vx = __ldg(b + obase + node) - vx;
                          vy = __ldg(b + obase + nsc + node) - vy;
                        }
                    }
                  y[obase + node] = vx;
                  y[obase + nsc + node] = vy;
                }
            }
          const long long pbase = n * isz + S * mv + a * mp + (static_cast<long long>(cy) * P.nx + cx) * NPM;
#pragma unroll
          for (int m = 0; m < NPM; ++m)
            y[pbase + m] = RESID ? (STMG_VM_BINIT ? -Yp[m] : __ldg(b + pbase + m) - Yp[m]) : Yp[m];
        }
    }
}

// ---------------------------------------------------------------------------
// r = 2 (Q3/P2disc) with a LANE PAIR per cell. The full-tile kernel above
// holds two 4x4 output tiles per thread and spills at the 168-register cap
// (ptxas: 184 bytes of stack). Here lane h of a pair owns the output columns
// i = {0, 1} (h = 0) or {3, 2} (h = 1): lane 1 works on the cell mirrored in
// x, so by the reflection symmetry of the 1D factors (M1, K1 even; C1 odd;
// Lm / Lc even or odd by Legendre degree) both lanes use the SAME
// compile-time coefficients and differ only in the sign sgn = +-1 of the odd
// ones. A lane loads and time-combines its own two node columns and
// receives the partner's two with shuffles; the x-contraction and the
// y-accumulation split cleanly by output column; the divergence rows are
// summed over a lane's own node columns and completed across the pair once
// per cell row. Strip = 15 owned cells + 1 halo cell per warp.
#ifndef STMG_VM_HALF
#define STMG_VM_HALF 0 // measured on C2: 3.06 ms (160 registers, no spills) vs 2.50 ms full tile: the pair doubles the per-thread overheads (addressing, pressure, shuffles)
#endif
#ifndef STMG_VM_HALF_MINB
#define STMG_VM_HALF_MINB 5
#endif
constexpr int kHStrip = 15;

template <int S, bool RESID, bool RAW>
__global__ void __launch_bounds__(32 * S, STMG_VM_HALF_MINB)
vmult2h_kernel(const LevelConsts P, const double *__restrict__ x, const double *__restrict__ b,
               double *__restrict__ y, const double *__restrict__ xprev0, int rows_per_seg, int coupled)
{
  constexpr int R = 2, N1 = 4, p = 3, NPM = 6, PL = 3, H = 2;
  const int lane = threadIdx.x & 31;
  const int a = threadIdx.x >> 5; // output slot
  const int n = blockIdx.z;       // interval
  const int c = lane >> 1, h = lane & 1;
  const int cx = blockIdx.x * kHStrip - 1 + c;
  const bool active = cx >= 0 && cx < P.nx;
  const bool owner = c >= 1 && active;
  const double sgn = h ? -1.0 : 1.0;

  const long long isz = P.isz, mv = P.mv, mp = P.mp, nsc = P.nsc;
  const int gx = P.gx, gy = P.gy;
  const double *__restrict__ xn = x + n * isz;
  const double *__restrict__ vprev = nullptr;
  if (coupled)
    vprev = n > 0 ? x + (n - 1) * isz + (S - 1) * mv : xprev0;

  double kt[S], mt[S], lva = 0.0;
#pragma unroll
  for (int bs = 0; bs < S; ++bs)
    kt[bs] = mt[bs] = 0.0;
#pragma unroll
  for (int aa = 0; aa < S; ++aa)
    if (a == aa)
      {
#pragma unroll
        for (int bs = 0; bs < S; ++bs)
          {
            kt[bs] = P.KtJ[aa * S + bs];
            mt[bs] = P.MtJ[aa * S + bs];
          }
        lva = P.lvJ[aa];
      }
  const double sg_l = sgn * P.sg;
  // reflection signs of the Legendre moments:
  // Lc(a, 3-k) = (-1)^(a+1) Lc(a, k), Lm(a, 3-k) = (-1)^a Lm(a, k)
  const double scx_e = sgn * P.scx, scy_o = sgn * P.scy; // even-degree Lc, odd-degree Lm

  const int cy_begin = blockIdx.y * rows_per_seg;
  const int cy_end = min(P.ny, cy_begin + rows_per_seg);
  const int cy_first = max(cy_begin - 1, 0);
  // own node columns: local kk = 0, 1 are the cell's columns ko[0], ko[1]
  const int ko0 = h ? 3 : 0, ko1 = h ? 2 : 1;

  double carx[H], cary[H];
#pragma unroll
  for (int i = 0; i < H; ++i)
    carx[i] = cary[i] = 0.0;

  for (int cy = cy_first; cy < cy_end; ++cy)
    {
      double Yx[H][N1], Yy[H][N1], Yp[NPM];
#pragma unroll
      for (int i = 0; i < H; ++i)
#pragma unroll
        for (int j = 0; j < N1; ++j)
          Yx[i][j] = Yy[i][j] = 0.0;
#pragma unroll
      for (int m = 0; m < NPM; ++m)
        Yp[m] = 0.0;
      if (cy > cy_first)
#pragma unroll
        for (int i = 0; i < H; ++i)
          {
            Yx[i][0] = carx[i];
            Yy[i][0] = cary[i];
          }

      if (active)
        {
          // ---- pressure: PM = sum_b Mt(a,b) p^b (both lanes of the pair), B^T init of the tiles
          const long long cell = static_cast<long long>(cy) * P.nx + cx;
          double PM[NPM], PMs[NPM];
#pragma unroll
          for (int m = 0; m < NPM; ++m)
            PM[m] = 0.0;
#pragma unroll
          for (int bs = 0; bs < S; ++bs)
            {
              const double cc = mt[bs];
              const double *pp = xn + S * mv + bs * mp + cell * NPM;
#pragma unroll
              for (int m = 0; m < NPM; ++m)
                PM[m] = fma(cc, __ldg(pp + m), PM[m]);
            }
#pragma unroll
          for (int m = 0; m < NPM; ++m)
            PMs[m] = sgn * PM[m];
#pragma unroll
          for (int bb = 0; bb < PL; ++bb)
            {
              double Qx[H], Qy[H];
#pragma unroll
              for (int i = 0; i < H; ++i)
                Qx[i] = Qy[i] = 0.0;
#pragma unroll
              for (int m = 0; m < NPM; ++m)
                {
                  if (pdisc_mode_ay(R, m) != bb)
                    continue;
                  const int am = pdisc_mode_ax(R, m);
                  const double pc = (am & 1) ? PM[m] : PMs[m]; // Lc: even degree is odd under reflection
                  const double pm = (am & 1) ? PMs[m] : PM[m]; // Lm: odd degree is odd under reflection
#pragma unroll
                  for (int i = 0; i < H; ++i)
                    {
                      Qx[i] = fma(VM_LC(am, i), pc, Qx[i]);
                      Qy[i] = fma(VM_LM(am, i), pm, Qy[i]);
                    }
                }
#pragma unroll
              for (int i = 0; i < H; ++i)
                {
                  Qx[i] *= P.scx;
                  Qy[i] *= P.scy;
                }
#pragma unroll
              for (int i = 0; i < H; ++i)
#pragma unroll
                for (int j = 0; j < N1; ++j)
                  {
                    Yx[i][j] = fma(-Qx[i], VM_LM(bb, j), Yx[i][j]);
                    Yy[i][j] = fma(-Qy[i], VM_LC(bb, j), Yy[i][j]);
                  }
            }
        }

      // ---- velocity rows of the cell
#pragma unroll
      for (int l = 0; l < N1; ++l)
        {
          double UKx[N1], UMx[N1], UKy[N1], UMy[N1];
#pragma unroll
          for (int k = 0; k < N1; ++k)
            UKx[k] = UMx[k] = UKy[k] = UMy[k] = 0.0;
          if (active)
            {
              const int Y = cy * p + l;
              const bool yb = (Y == 0) || (Y == gy - 1);
              const long long rowbase = static_cast<long long>(Y) * gx + cx * p;
#pragma unroll
              for (int kk = 0; kk < H; ++kk)
                {
                  const int k = kk == 0 ? ko0 : ko1;
                  const int X = cx * p + k;
                  const bool bnd = !RAW && (yb || X == 0 || X == gx - 1);
                  const long long node = rowbase + k;
                  double ukx = 0.0, umx = 0.0, uky = 0.0, umy = 0.0;
#pragma unroll
                  for (int bs = 0; bs < S; ++bs)
                    {
                      const double vx = bnd ? 0.0 : __ldg(xn + bs * mv + node);
                      const double vy = bnd ? 0.0 : __ldg(xn + bs * mv + nsc + node);
                      ukx = fma(kt[bs], vx, ukx);
                      umx = fma(mt[bs], vx, umx);
                      uky = fma(kt[bs], vy, uky);
                      umy = fma(mt[bs], vy, umy);
                    }
                  if (vprev != nullptr)
                    {
                      ukx = fma(-lva, __ldg(vprev + node), ukx);
                      uky = fma(-lva, __ldg(vprev + nsc + node), uky);
                    }
                  UKx[kk] = ukx;
                  UMx[kk] = umx;
                  UKy[kk] = uky;
                  UMy[kk] = umy;
                }
            }
          // the partner's node columns: its local 1, 0 are this lane's local 2, 3
          UKx[2] = __shfl_xor_sync(0xffffffffu, UKx[1], 1);
          UKx[3] = __shfl_xor_sync(0xffffffffu, UKx[0], 1);
          UMx[2] = __shfl_xor_sync(0xffffffffu, UMx[1], 1);
          UMx[3] = __shfl_xor_sync(0xffffffffu, UMx[0], 1);
          UKy[2] = __shfl_xor_sync(0xffffffffu, UKy[1], 1);
          UKy[3] = __shfl_xor_sync(0xffffffffu, UKy[0], 1);
          UMy[2] = __shfl_xor_sync(0xffffffffu, UMy[1], 1);
          UMy[3] = __shfl_xor_sync(0xffffffffu, UMy[0], 1);
          if (active)
            {
              double UMxa[N1], UMyb[N1];
#pragma unroll
              for (int k = 0; k < N1; ++k)
                {
                  UMxa[k] = P.sax * UMx[k];
                  UMyb[k] = P.say * UMy[k];
                }
#pragma unroll
              for (int i = 0; i < H; ++i)
                {
                  double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0;
#pragma unroll
                  for (int k = 0; k < N1; ++k)
                    {
                      s0 = fma(VM_M(i, k), UKx[k], s0);
                      s0 = fma(VM_K(i, k), UMxa[k], s0);
                      s1 = fma(VM_M(i, k), UMx[k], s1);
                      s2 = fma(VM_C(i, k), UMy[k], s2);
                      s3 = fma(VM_M(i, k), UKy[k], s3);
                      s3 = fma(VM_K(i, k), UMyb[k], s3);
                      s4 = fma(VM_M(i, k), UMy[k], s4);
                      s5 = fma(VM_C(k, i), UMx[k], s5);
                    }
                  s1 *= P.sbx;
                  s2 *= sg_l; // C1 is odd under the reflection
                  s4 *= P.sby;
                  s5 *= sg_l;
#pragma unroll
                  for (int j = 0; j < N1; ++j)
                    {
                      double vx = Yx[i][j], vy = Yy[i][j];
                      vx = fma(VM_M(j, l), s0, vx);
                      vx = fma(VM_K(j, l), s1, vx);
                      vx = fma(VM_C(l, j), s2, vx);
                      vy = fma(VM_M(j, l), s3, vy);
                      vy = fma(VM_K(j, l), s4, vy);
                      vy = fma(VM_C(j, l), s5, vy);
                      Yx[i][j] = vx;
                      Yy[i][j] = vy;
                    }
                }
              // divergence rows over this lane's own node columns (local 0, 1)
              double dp[PL], ep[PL];
#pragma unroll
              for (int aa = 0; aa < PL; ++aa)
                {
                  double s0 = 0, s1 = 0;
#pragma unroll
                  for (int k = 0; k < H; ++k)
                    {
                      s0 = fma(VM_LC(aa, k), UMx[k], s0);
                      s1 = fma(VM_LM(aa, k), UMy[k], s1);
                    }
                  dp[aa] = s0 * ((aa & 1) ? P.scx : scx_e);
                  ep[aa] = s1 * ((aa & 1) ? scy_o : P.scy);
                }
#pragma unroll
              for (int m = 0; m < NPM; ++m)
                {
                  const int am = pdisc_mode_ax(R, m), bm = pdisc_mode_ay(R, m);
                  Yp[m] = fma(VM_LM(bm, l), dp[am], Yp[m]);
                  Yp[m] = fma(VM_LC(bm, l), ep[am], Yp[m]);
                }
            }
        }

      // ---- assemble: pair halves of the divergence, shared nodes in x across cells, y through the carry
#pragma unroll
      for (int m = 0; m < NPM; ++m)
        Yp[m] += __shfl_xor_sync(0xffffffffu, Yp[m], 1);
#pragma unroll
      for (int i = 0; i < H; ++i)
        {
          carx[i] = Yx[i][N1 - 1];
          cary[i] = Yy[i][N1 - 1];
        }
#pragma unroll
      for (int j = 0; j < N1; ++j)
        {
          // local column 0 is the cell's column 3 on odd lanes, column 0 on even lanes
          const double lx = __shfl_up_sync(0xffffffffu, Yx[0][j], 1);
          const double ly = __shfl_up_sync(0xffffffffu, Yy[0][j], 1);
          if (h == 0 && lane > 0)
            {
              Yx[0][j] += lx;
              Yy[0][j] += ly;
            }
        }

      // ---- write owned outputs
      if (owner && cy >= cy_begin)
        {
          const bool lastx = cx == P.nx - 1;
          const int iymax = (cy == P.ny - 1) ? p : p - 1;
          const long long obase = n * isz + a * mv;
#pragma unroll
          for (int j = 0; j < N1; ++j)
            {
              if (j > iymax)
                continue;
              const int Y = cy * p + j;
              const bool yb = (Y == 0) || (Y == gy - 1);
#pragma unroll
              for (int i = 0; i < H; ++i)
                {
                  // even lane: columns 0, 1; odd lane: column 2, and 3 on the last cell column
                  if (i == 0 && h == 1 && !lastx)
                    continue;
                  const int X = cx * p + (i == 0 ? ko0 : ko1);
                  const long long node = static_cast<long long>(Y) * gx + X;
                  double vx = Yx[i][j], vy = Yy[i][j];
                  if (!RAW && (yb || X == 0 || X == gx - 1))
                    {
                      vx = __ldg(x + obase + node);
                      vy = __ldg(x + obase + nsc + node);
                    }
                  if (RESID)
                    {
                      vx = __ldg(b + obase + node) - vx;
                      vy = __ldg(b + obase + nsc + node) - vy;
                    }
                  y[obase + node] = vx;
                  y[obase + nsc + node] = vy;
                }
            }
          const long long pbase = n * isz + S * mv + a * mp + (static_cast<long long>(cy) * P.nx + cx) * NPM;
#pragma unroll
          for (int m = 0; m < NPM; ++m)
            if ((m < NPM / 2) == (h == 0))
              y[pbase + m] = RESID ? __ldg(b + pbase + m) - Yp[m] : Yp[m];
        }
    }
}

template <int R, int S>
cudaError_t
launch_rs(const LevelConsts &P, const double *x, const double *b, double *y, int n_intervals, const double *xprev0,
          int coupled, int mode, cudaStream_t stream)
{
  constexpr bool kHalf = R == 2 && STMG_VM_HALF != 0;
  const int strips = kHalf ? (P.nx + kHStrip - 1) / kHStrip : (P.nx + kStrip - 1) / kStrip;
  // Row segments: enough blocks to fill 148 SMs several times, >= 8 rows
  // each so the recomputed halo row stays small -- down to 2 rows on small
  // grids, where the march length (latency) matters more than the halo row.
  int segs = 1;
  const long long base_blocks = static_cast<long long>(strips) * n_intervals;
  const int min_rows = base_blocks * P.ny >= 148 * 64 ? 8 : 2;
  while (base_blocks * segs < 148 * 8 && P.ny / (segs * 2) >= min_rows)
    segs *= 2;
  const int rows = (P.ny + segs - 1) / segs;
  dim3 grid(strips, (P.ny + rows - 1) / rows, n_intervals);
  dim3 block(32 * S);
  auto go = [&](auto kern, size_t smem) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    kern<<<grid, block, smem, stream>>>(P, x, b, y, xprev0, rows, coupled);
  };
  constexpr size_t st_plain = RowStage<R, S>::template bytes<false>(),
                   st_resid = RowStage<R, S>::template bytes<true>();
  if constexpr (kHalf)
    {
      switch (mode)
        {
          case 0: vmult2h_kernel<S, false, false><<<grid, block, 0, stream>>>(P, x, b, y, xprev0, rows, coupled); break;
          case 1: vmult2h_kernel<S, true, false><<<grid, block, 0, stream>>>(P, x, b, y, xprev0, rows, coupled); break;
          default: vmult2h_kernel<S, false, true><<<grid, block, 0, stream>>>(P, x, b, y, xprev0, rows, coupled); break;
        }
      return cudaGetLastError();
    }
  switch (mode)
    {
      case 0: go(vmult_kernel<R, S, false, false>, st_plain); break;
      case 1: go(vmult_kernel<R, S, true, false>, st_resid); break;
      default: go(vmult_kernel<R, S, false, true>, st_plain); break;
    }
  return cudaGetLastError();
}

} // namespace vmult_detail
} // namespace stmg_b200
