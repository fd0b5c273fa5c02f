// Instantiation unit of the fused space-time operator for r=3, k+1=3
// (split so nvcc compiles the 20 specialisations in parallel).
#include "vmult_impl.cuh"

namespace stmg_b200
{
cudaError_t
launch_vmult_r3s3(const LevelConsts &P, const double *x, const double *b, double *y, int n, const double *xp,
                     int c, int mode, cudaStream_t st)
{
  return vmult_detail::launch_rs<3, 3>(P, x, b, y, n, xp, c, mode, st);
}
} // namespace stmg_b200
