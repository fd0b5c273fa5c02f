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
#include "kernels.hpp"

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
} // namespace

/// Launch one colour: `n_batches` batches over `n_intervals` intervals.
cudaError_t
launch_vanka_colour(const DevPatchClass *classes, const VankaBatch *batches, int n_batches, int max_nt,
                    const long long *vel_anchor, const long long *pre_anchor, const double *r, double *u,
                    long long isz, int n_intervals, double omega, cudaStream_t stream)
{
  if (n_batches == 0 || n_intervals == 0)
    return cudaSuccess;
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
