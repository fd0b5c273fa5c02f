// Instantiation unit of the fused space-time operator for r=1, k+1=2
// (split so nvcc compiles the 20 specialisations in parallel).
#include "vmult_impl.cuh"

namespace stmg_b200
{
cudaError_t
launch_vmult_r1s2(const LevelConsts &P, const double *x, const double *b, double *y, int n, const double *xp,
                     int c, int mode, cudaStream_t st)
{
  return vmult_detail::launch_rs<1, 2>(P, x, b, y, n, xp, c, mode, st);
}
} // namespace stmg_b200
