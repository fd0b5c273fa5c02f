// Dispatcher of the fused space-time operator (see vmult_impl.cuh).
#include "kernels.hpp"

namespace stmg_b200
{
cudaError_t launch_vmult_r1s1(const LevelConsts &, const double *, const double *, double *, int, const double *, int, int, cudaStream_t);
cudaError_t launch_vmult_r1s2(const LevelConsts &, const double *, const double *, double *, int, const double *, int, int, cudaStream_t);
cudaError_t launch_vmult_r1s3(const LevelConsts &, const double *, const double *, double *, int, const double *, int, int, cudaStream_t);
cudaError_t launch_vmult_r1s4(const LevelConsts &, const double *, const double *, double *, int, const double *, int, int, cudaStream_t);
cudaError_t launch_vmult_r1s5(const LevelConsts &, const double *, const double *, double *, int, const double *, int, int, cudaStream_t);
cudaError_t launch_vmult_r2s1(const LevelConsts &, const double *, const double *, double *, int, const double *, int, int, cudaStream_t);
cudaError_t launch_vmult_r2s2(const LevelConsts &, const double *, const double *, double *, int, const double *, int, int, cudaStream_t);
cudaError_t launch_vmult_r2s3(const LevelConsts &, const double *, const double *, double *, int, const double *, int, int, cudaStream_t);
cudaError_t launch_vmult_r2s4(const LevelConsts &, const double *, const double *, double *, int, const double *, int, int, cudaStream_t);
cudaError_t launch_vmult_r2s5(const LevelConsts &, const double *, const double *, double *, int, const double *, int, int, cudaStream_t);
cudaError_t launch_vmult_r3s1(const LevelConsts &, const double *, const double *, double *, int, const double *, int, int, cudaStream_t);
cudaError_t launch_vmult_r3s2(const LevelConsts &, const double *, const double *, double *, int, const double *, int, int, cudaStream_t);
cudaError_t launch_vmult_r3s3(const LevelConsts &, const double *, const double *, double *, int, const double *, int, int, cudaStream_t);
cudaError_t launch_vmult_r3s4(const LevelConsts &, const double *, const double *, double *, int, const double *, int, int, cudaStream_t);
cudaError_t launch_vmult_r3s5(const LevelConsts &, const double *, const double *, double *, int, const double *, int, int, cudaStream_t);
cudaError_t launch_vmult_r4s1(const LevelConsts &, const double *, const double *, double *, int, const double *, int, int, cudaStream_t);
cudaError_t launch_vmult_r4s2(const LevelConsts &, const double *, const double *, double *, int, const double *, int, int, cudaStream_t);
cudaError_t launch_vmult_r4s3(const LevelConsts &, const double *, const double *, double *, int, const double *, int, int, cudaStream_t);
cudaError_t launch_vmult_r4s4(const LevelConsts &, const double *, const double *, double *, int, const double *, int, int, cudaStream_t);
cudaError_t launch_vmult_r4s5(const LevelConsts &, const double *, const double *, double *, int, const double *, int, int, cudaStream_t);

/// mode 0: y = D x (constrained), 1: y = b - D x, 2: y = D_raw x.
/// coupled != 0 adds the jump term -C x_(n-1)[slot k] (x_prev0 feeds n = 0;
/// may be null, then interval 0 is uncoupled).
cudaError_t
launch_vmult(int r, int S, const LevelConsts &P, const double *x, const double *b, double *y, int n_intervals,
             const double *xprev0, int coupled, int mode, cudaStream_t stream)
{
  if (n_intervals <= 0)
    return cudaSuccess;
  switch (r * 10 + S)
    {
    case 11: return launch_vmult_r1s1(P, x, b, y, n_intervals, xprev0, coupled, mode, stream);
    case 12: return launch_vmult_r1s2(P, x, b, y, n_intervals, xprev0, coupled, mode, stream);
    case 13: return launch_vmult_r1s3(P, x, b, y, n_intervals, xprev0, coupled, mode, stream);
    case 14: return launch_vmult_r1s4(P, x, b, y, n_intervals, xprev0, coupled, mode, stream);
    case 15: return launch_vmult_r1s5(P, x, b, y, n_intervals, xprev0, coupled, mode, stream);
    case 21: return launch_vmult_r2s1(P, x, b, y, n_intervals, xprev0, coupled, mode, stream);
    case 22: return launch_vmult_r2s2(P, x, b, y, n_intervals, xprev0, coupled, mode, stream);
    case 23: return launch_vmult_r2s3(P, x, b, y, n_intervals, xprev0, coupled, mode, stream);
    case 24: return launch_vmult_r2s4(P, x, b, y, n_intervals, xprev0, coupled, mode, stream);
    case 25: return launch_vmult_r2s5(P, x, b, y, n_intervals, xprev0, coupled, mode, stream);
    case 31: return launch_vmult_r3s1(P, x, b, y, n_intervals, xprev0, coupled, mode, stream);
    case 32: return launch_vmult_r3s2(P, x, b, y, n_intervals, xprev0, coupled, mode, stream);
    case 33: return launch_vmult_r3s3(P, x, b, y, n_intervals, xprev0, coupled, mode, stream);
    case 34: return launch_vmult_r3s4(P, x, b, y, n_intervals, xprev0, coupled, mode, stream);
    case 35: return launch_vmult_r3s5(P, x, b, y, n_intervals, xprev0, coupled, mode, stream);
    case 41: return launch_vmult_r4s1(P, x, b, y, n_intervals, xprev0, coupled, mode, stream);
    case 42: return launch_vmult_r4s2(P, x, b, y, n_intervals, xprev0, coupled, mode, stream);
    case 43: return launch_vmult_r4s3(P, x, b, y, n_intervals, xprev0, coupled, mode, stream);
    case 44: return launch_vmult_r4s4(P, x, b, y, n_intervals, xprev0, coupled, mode, stream);
    case 45: return launch_vmult_r4s5(P, x, b, y, n_intervals, xprev0, coupled, mode, stream);
    default: return cudaErrorInvalidValue;
    }
}
} // namespace stmg_b200
