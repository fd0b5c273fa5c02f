// Transfer, constraint, projection, coarse-solve and Krylov vector kernels
// of the B200 hp-STMG path (sm_100a, FP64).
//
//  * prolongate / restrict: TransferPair::prolongate/restrict_ and the
//    *_correction / *_residual wrappers (transfer.cpp:51-132). The spatial
//    transfer is the tensor product of two 1D stencils (CSR, <= n1 or 2 n1
//    entries per row), evaluated matrix-free per output node; the temporal
//    node-evaluation matrix (transfer.cpp:363-386) is applied in registers.
//  * project_mean_zero (dof_space.cpp:110-119): chunked partial sums per
//    (slot, interval), re-reduced in fixed order by every block (deterministic).
//  * coarse solve (solver.cpp:43-54): dense inverse of the pinned coarse
//    operator, one warp per row.
//  * dot / axpy for FGMRES (solver.cpp:139-199): fixed-grid two-stage
//    reductions with warp shuffles, deterministic.
#include "kernels.hpp"

namespace stmg_b200
{

namespace
{
__device__ __forceinline__ double
warp_sum(double v)
{
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int BS>
__device__ double
block_sum(double v)
{
  __shared__ double part[BS / 32];
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0)
    part[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0)
    {
      t = l < BS / 32 ? part[l] : 0.0;
      t = warp_sum(t);
    }
  __syncthreads();
  return t; // valid in warp 0
}

// ---------------------------------------------------------------- transfers
__global__ void
prolong_velocity_kernel(const DevTransfer T, const double *__restrict__ coarse, double *__restrict__ fine,
                        int accumulate)
{
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long n = blockIdx.y;
  if (idx >= 2 * T.f.nsc)
    return;
  const int comp = idx >= T.f.nsc;
  const long long node = idx - comp * T.f.nsc;
  const int X = static_cast<int>(node % T.f.gx), Y = static_cast<int>(node / T.f.gx);
  double vb[kMaxS];
#pragma unroll
  for (int b = 0; b < kMaxS; ++b)
    vb[b] = 0.0;
  const double *cb = coarse + n * T.c.isz + comp * T.c.nsc;
  if (T.spatial)
    {
      for (int i = T.py.ptr[Y]; i < T.py.ptr[Y + 1]; ++i)
        {
          const double wy = T.py.val[i];
          const long long row = static_cast<long long>(T.py.col[i]) * T.c.gx;
          for (int k = T.px.ptr[X]; k < T.px.ptr[X + 1]; ++k)
            {
              const double w = wy * T.px.val[k];
              const long long cn = row + T.px.col[k];
              for (int b = 0; b < T.c.S; ++b)
                vb[b] = fma(w, __ldg(cb + b * T.c.mv + cn), vb[b]);
            }
        }
    }
  else
    for (int b = 0; b < T.c.S; ++b)
      vb[b] = __ldg(cb + b * T.c.mv + node);
  const bool bnd = X == 0 || X == T.f.gx - 1 || Y == 0 || Y == T.f.gy - 1;
  double *fb = fine + n * T.f.isz + comp * T.f.nsc + node;
  for (int a = 0; a < T.f.S; ++a)
    {
      double v;
      if (T.temporal)
        {
          v = 0.0;
          for (int b = 0; b < T.c.S; ++b)
            v = fma(T.E[a * kMaxS + b], vb[b], v);
        }
      else
        v = vb[a];
      if (T.zero_constrained && bnd)
        v = 0.0;
      double *dst = fb + a * T.f.mv;
      *dst = accumulate ? *dst + v : v;
    }
}

__global__ void
prolong_pressure_kernel(const DevTransfer T, const double *__restrict__ coarse, double *__restrict__ fine,
                        int accumulate)
{
  const long long fcell = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long n = blockIdx.y;
  if (fcell >= static_cast<long long>(T.f.nx) * T.f.ny)
    return;
  const int fx = static_cast<int>(fcell % T.f.nx), fy = static_cast<int>(fcell / T.f.nx);
  const int npf = T.f.np, npc = T.c.np;
  long long ccell = fcell;
  int child = 0;
  if (T.pmode == 1)
    {
      ccell = static_cast<long long>(fy / 2) * T.c.nx + fx / 2;
      child = (fy % 2) * 2 + (fx % 2);
    }
  double vb[kMaxS][kMaxNP];
  for (int b = 0; b < T.c.S; ++b)
    {
      const double *pc = coarse + n * T.c.isz + T.c.S * T.c.mv + b * T.c.mp + ccell * npc;
      for (int m = 0; m < npf; ++m)
        vb[b][m] = 0.0;
      if (T.pmode == 1)
        {
          const double *blk = T.child + child * npc * npc;
          for (int m = 0; m < npf; ++m)
            {
              double s = 0.0;
              for (int l = 0; l < npc; ++l)
                s = fma(blk[m * npc + l], __ldg(pc + l), s);
              vb[b][m] = s;
            }
        }
      else if (T.pmode == 2)
        for (int l = 0; l < npc; ++l)
          vb[b][T.embed[l]] = __ldg(pc + l);
      else
        for (int m = 0; m < npf; ++m)
          vb[b][m] = __ldg(pc + m);
    }
  for (int a = 0; a < T.f.S; ++a)
    {
      double *pf = fine + n * T.f.isz + T.f.S * T.f.mv + a * T.f.mp + fcell * npf;
      for (int m = 0; m < npf; ++m)
        {
          double v;
          if (T.temporal)
            {
              v = 0.0;
              for (int b = 0; b < T.c.S; ++b)
                v = fma(T.E[a * kMaxS + b], vb[b][m], v);
            }
          else
            v = vb[a][m];
          pf[m] = accumulate ? pf[m] + v : v;
        }
    }
}

__global__ void
restrict_velocity_kernel(const DevTransfer T, const double *__restrict__ fine, double *__restrict__ coarse)
{
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long n = blockIdx.y;
  if (idx >= 2 * T.c.nsc)
    return;
  const int comp = idx >= T.c.nsc;
  const long long node = idx - comp * T.c.nsc;
  const int X = static_cast<int>(node % T.c.gx), Y = static_cast<int>(node / T.c.gx);
  double va[kMaxS];
#pragma unroll
  for (int a = 0; a < kMaxS; ++a)
    va[a] = 0.0;
  const double *fb = fine + n * T.f.isz + comp * T.f.nsc;
  if (T.spatial)
    {
      for (int i = T.ry.ptr[Y]; i < T.ry.ptr[Y + 1]; ++i)
        {
          const double wy = T.ry.val[i];
          const long long row = static_cast<long long>(T.ry.col[i]) * T.f.gx;
          for (int k = T.rx.ptr[X]; k < T.rx.ptr[X + 1]; ++k)
            {
              const double w = wy * T.rx.val[k];
              const long long fn = row + T.rx.col[k];
              for (int a = 0; a < T.f.S; ++a)
                va[a] = fma(w, __ldg(fb + a * T.f.mv + fn), va[a]);
            }
        }
    }
  else
    for (int a = 0; a < T.f.S; ++a)
      va[a] = __ldg(fb + a * T.f.mv + node);
  const bool bnd = X == 0 || X == T.c.gx - 1 || Y == 0 || Y == T.c.gy - 1;
  double *cb = coarse + n * T.c.isz + comp * T.c.nsc + node;
  for (int b = 0; b < T.c.S; ++b)
    {
      double v;
      if (T.temporal)
        {
          v = 0.0;
          for (int a = 0; a < T.f.S; ++a)
            v = fma(T.E[a * kMaxS + b], va[a], v);
        }
      else
        v = va[b];
      if (T.zero_constrained && bnd)
        v = 0.0;
      cb[b * T.c.mv] = v;
    }
}

__global__ void
restrict_pressure_kernel(const DevTransfer T, const double *__restrict__ fine, double *__restrict__ coarse)
{
  const long long ccell = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long n = blockIdx.y;
  if (ccell >= static_cast<long long>(T.c.nx) * T.c.ny)
    return;
  const int cxi = static_cast<int>(ccell % T.c.nx), cyi = static_cast<int>(ccell / T.c.nx);
  const int npf = T.f.np, npc = T.c.np;
  double va[kMaxS][kMaxNP];
  for (int a = 0; a < T.f.S; ++a)
    {
      const double *pfa = fine + n * T.f.isz + T.f.S * T.f.mv + a * T.f.mp;
      for (int l = 0; l < npc; ++l)
        va[a][l] = 0.0;
      if (T.pmode == 1)
        {
          for (int ch = 0; ch < 4; ++ch)
            {
              const long long fcell = static_cast<long long>(2 * cyi + ch / 2) * T.f.nx + 2 * cxi + ch % 2;
              const double *blk = T.child + ch * npc * npc;
              for (int m = 0; m < npf; ++m)
                {
                  const double pv = __ldg(pfa + fcell * npf + m);
                  for (int l = 0; l < npc; ++l)
                    va[a][l] = fma(blk[m * npc + l], pv, va[a][l]);
                }
            }
        }
      else if (T.pmode == 2)
        for (int l = 0; l < npc; ++l)
          va[a][l] = __ldg(pfa + ccell * npf + T.embed[l]);
      else
        for (int l = 0; l < npc; ++l)
          va[a][l] = __ldg(pfa + ccell * npf + l);
    }
  for (int b = 0; b < T.c.S; ++b)
    {
      double *pc = coarse + n * T.c.isz + T.c.S * T.c.mv + b * T.c.mp + ccell * npc;
      for (int l = 0; l < npc; ++l)
        {
          double v;
          if (T.temporal)
            {
              v = 0.0;
              for (int a = 0; a < T.f.S; ++a)
                v = fma(T.E[a * kMaxS + b], va[a][l], v);
            }
          else
            v = va[b][l];
          pc[l] = v;
        }
    }
}

// ---------------------------------------------------------------- projection
constexpr int kProjThreads = 256;
constexpr int kProjChunkCells = 8192;

__host__ __device__ inline int
proj_chunks(long long ncell)
{
  const long long c = (ncell + kProjChunkCells - 1) / kProjChunkCells;
  return static_cast<int>(c < 1 ? 1 : (c > 64 ? 64 : c));
}

// Partial sums of the mode-0 pressure coefficients: block (slot, interval, chunk).
__global__ void __launch_bounds__(kProjThreads)
pmz_partial_kernel(const DevGeom G, const double *__restrict__ x, double *__restrict__ part)
{
  const int a = blockIdx.x, chunk = blockIdx.z, nch = gridDim.z;
  const long long n = blockIdx.y;
  const double *p = x + n * G.isz + G.S * G.mv + a * G.mp;
  const long long ncell = static_cast<long long>(G.nx) * G.ny;
  const long long c0 = ncell * chunk / nch, c1 = ncell * (chunk + 1) / nch;
  double s = 0.0;
  for (long long c = c0 + threadIdx.x; c < c1; c += blockDim.x)
    s += p[c * G.np];
  s = block_sum<kProjThreads>(s);
  if (threadIdx.x == 0)
    part[(n * G.S + a) * nch + chunk] = s;
}

// Every block re-reduces its (slot, interval) partials in a fixed order and
// subtracts the mean from its chunk (deterministic).
__global__ void __launch_bounds__(kProjThreads)
pmz_apply_kernel(const DevGeom G, double *__restrict__ x, const double *__restrict__ part, double scale)
{
  const int a = blockIdx.x, chunk = blockIdx.z, nch = gridDim.z;
  const long long n = blockIdx.y;
  __shared__ double mean;
  if (threadIdx.x == 0)
    {
      double s = 0.0;
      for (int k = 0; k < nch; ++k)
        s += part[(n * G.S + a) * nch + k];
      mean = s * scale;
    }
  __syncthreads();
  double *p = x + n * G.isz + G.S * G.mv + a * G.mp;
  const long long ncell = static_cast<long long>(G.nx) * G.ny;
  const long long c0 = ncell * chunk / nch, c1 = ncell * (chunk + 1) / nch;
  const double m = mean;
  for (long long c = c0 + threadIdx.x; c < c1; c += blockDim.x)
    p[c * G.np] -= m;
}

__global__ void
zero_constrained_kernel(const DevGeom G, double *__restrict__ x)
{
  // boundary nodes: 2*(gx + gy) - 4 per component and slot
  const int nb = 2 * (G.gx + G.gy) - 4;
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long n = blockIdx.y;
  if (idx >= static_cast<long long>(nb) * 2 * G.S)
    return;
  const int b = static_cast<int>(idx % nb);
  const long long rest = idx / nb;
  const int comp = static_cast<int>(rest % 2), a = static_cast<int>(rest / 2);
  long long node;
  if (b < G.gx)
    node = b; // bottom row
  else if (b < 2 * G.gx)
    node = static_cast<long long>(G.gy - 1) * G.gx + (b - G.gx); // top row
  else
    {
      const int t = b - 2 * G.gx; // side columns without corners
      const int row = 1 + t / 2;
      node = static_cast<long long>(row) * G.gx + ((t % 2) ? G.gx - 1 : 0);
    }
  x[n * G.isz + a * G.mv + comp * G.nsc + node] = 0.0;
}

// ---------------------------------------------------------------- coarse solve
__global__ void
coarse_solve_kernel(const double *__restrict__ inv, const long long *__restrict__ pinned, int n_pinned, int nrows,
                    const double *__restrict__ b, double *__restrict__ x)
{
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= nrows)
    return;
  const double *row = inv + static_cast<long long>(warp) * nrows;
  double s = 0.0;
  for (int j = lane; j < nrows; j += 32)
    {
      bool pin = false;
      for (int q = 0; q < n_pinned; ++q)
        pin |= pinned[q] == j;
      if (!pin)
        s = fma(row[j], b[j], s);
    }
  s = warp_sum(s);
  if (lane == 0)
    x[warp] = s;
}

// One block walks the time axis of the coarse all-at-once system (lower block
// bidiagonal): the exact coarse solve of the all-at-once
// V-cycle. One warp per row for the two small dense matvecs of each step.
__global__ void __launch_bounds__(1024)
coarse_forward_kernel(const double *__restrict__ G, const double *__restrict__ H, int n, int mv, long long v_off,
                      const double *__restrict__ B, int n_all, int n_begin, int n_own, double *__restrict__ X)
{
  extern __shared__ double sh[]; // v[mv], then x_t[n]
  double *v = sh, *xt = sh + mv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int i = tid; i < mv; i += blockDim.x)
    v[i] = 0.0;
  __syncthreads();
  for (int t = 0; t < n_all; ++t)
    {
      const double *b = B + static_cast<long long>(t) * n;
      for (int i = warp; i < n; i += nw)
        {
          const double *g = G + static_cast<long long>(i) * n, *h = H + static_cast<long long>(i) * mv;
          double s = 0.0;
          for (int j = lane; j < n; j += 32)
            s = fma(g[j], b[j], s);
          for (int j = lane; j < mv; j += 32)
            s = fma(h[j], v[j], s);
          s = warp_sum(s);
          if (lane == 0)
            xt[i] = s;
        }
      __syncthreads();
      if (t >= n_begin && t < n_begin + n_own)
        for (int i = tid; i < n; i += blockDim.x)
          X[static_cast<long long>(t - n_begin) * n + i] = xt[i];
      for (int i = tid; i < mv; i += blockDim.x)
        v[i] = xt[v_off + i];
      __syncthreads();
    }
}

// ---------------------------------------------------------------- BLAS-1
constexpr int kDotThreads = 256;

__global__ void __launch_bounds__(kDotThreads)
dot_partial_kernel(const double *__restrict__ x, const double *__restrict__ y, long long n, double *__restrict__ part)
{
  double s = 0.0;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride)
    s = fma(x[i], y[i], s);
  s = block_sum<kDotThreads>(s);
  if (threadIdx.x == 0)
    part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kDotThreads)
dot_final_kernel(const double *__restrict__ part, int np, double *__restrict__ out)
{
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x)
    s += part[i];
  s = block_sum<kDotThreads>(s);
  if (threadIdx.x == 0)
    *out = s;
}

// Batched inner products <w, V_i>, i < m (and <w, w> in slot m when
// with_norm), reading w once per chunk: one pass over the Krylov basis for a
// classical Gram-Schmidt sweep. Fixed grid and fixed-order reductions, so the
// result is bitwise reproducible.
__global__ void __launch_bounds__(kDotThreads)
multidot_partial_kernel(MultiVec V, int m, int with_norm, const double *__restrict__ w, long long n,
                        double *__restrict__ part)
{
  double s[kMultiMax + 1];
#pragma unroll
  for (int i = 0; i <= kMultiMax; ++i)
    s[i] = 0.0;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n; k += stride)
    {
      const double wk = w[k];
#pragma unroll
      for (int i = 0; i < kMultiMax; ++i)
        if (i < m)
          s[i] = fma(wk, V.p[i][k], s[i]);
      s[kMultiMax] = fma(wk, wk, s[kMultiMax]);
    }
  for (int i = 0; i <= m; ++i)
    {
      const int slot = i < m ? i : kMultiMax;
      if (i == m && !with_norm)
        break;
      const double t = block_sum<kDotThreads>(s[slot]);
      if (threadIdx.x == 0)
        part[static_cast<long long>(i) * gridDim.x + blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(kDotThreads)
multidot_final_kernel(const double *__restrict__ part, int np, double *__restrict__ out)
{
  const double *p = part + static_cast<long long>(blockIdx.x) * np;
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x)
    s += p[i];
  s = block_sum<kDotThreads>(s);
  if (threadIdx.x == 0)
    out[blockIdx.x] = s;
}

// w += sign * sum_i c_i V_i, i < m, c on the device (c_dev) or the host
// value array (c_host); one read of w and each V_i, one write of w.
__global__ void
multi_axpy_kernel(MultiVec V, int m, const double *__restrict__ c_dev, MultiCoef c_host, double sign,
                  double *__restrict__ w, long long n)
{
  __shared__ double c[kMultiMax];
  if (threadIdx.x < m)
    c[threadIdx.x] = sign * (c_dev ? c_dev[threadIdx.x] : c_host.c[threadIdx.x]);
  __syncthreads();
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n; k += stride)
    {
      double acc = w[k];
#pragma unroll
      for (int i = 0; i < kMultiMax; ++i)
        if (i < m)
          acc = fma(c[i], V.p[i][k], acc);
      w[k] = acc;
    }
}

__global__ void
axpy_kernel(long long n, double alpha, const double *__restrict__ alpha_dev, double sign, const double *__restrict__ x,
            double *__restrict__ y)
{
  const double a = alpha_dev ? sign * *alpha_dev : alpha;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride)
    y[i] = fma(a, x[i], y[i]);
}

__global__ void
scale_kernel(long long n, double alpha, double *__restrict__ y)
{
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride)
    y[i] *= alpha;
}

__global__ void
xpby_kernel(long long n, const double *__restrict__ x, double beta, double *__restrict__ y)
{ // y = x + beta * y
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride)
    y[i] = fma(beta, y[i], x[i]);
}

int
grid_for(long long n, int threads)
{
  const long long g = (n + threads - 1) / threads;
  const long long cap = 16LL * device_sm_count();
  return static_cast<int>(g < cap ? (g < 1 ? 1 : g) : cap);
}
} // namespace

cudaError_t
launch_prolongate(const DevTransfer &T, const double *coarse, double *fine, int n_intervals, int accumulate,
                  cudaStream_t st)
{
  if (n_intervals <= 0)
    return cudaSuccess;
  const int th = 128;
  dim3 gv(static_cast<unsigned>((2 * T.f.nsc + th - 1) / th), n_intervals);
  prolong_velocity_kernel<<<gv, th, 0, st>>>(T, coarse, fine, accumulate);
  const long long nc = static_cast<long long>(T.f.nx) * T.f.ny;
  dim3 gp(static_cast<unsigned>((nc + th - 1) / th), n_intervals);
  prolong_pressure_kernel<<<gp, th, 0, st>>>(T, coarse, fine, accumulate);
  return cudaGetLastError();
}

cudaError_t
launch_restrict(const DevTransfer &T, const double *fine, double *coarse, int n_intervals, cudaStream_t st)
{
  if (n_intervals <= 0)
    return cudaSuccess;
  const int th = 128;
  dim3 gv(static_cast<unsigned>((2 * T.c.nsc + th - 1) / th), n_intervals);
  restrict_velocity_kernel<<<gv, th, 0, st>>>(T, fine, coarse);
  const long long nc = static_cast<long long>(T.c.nx) * T.c.ny;
  dim3 gp(static_cast<unsigned>((nc + th - 1) / th), n_intervals);
  restrict_pressure_kernel<<<gp, th, 0, st>>>(T, fine, coarse);
  return cudaGetLastError();
}

int
project_scratch_doubles(const DevGeom &G, int n_intervals)
{
  return G.S * n_intervals * proj_chunks(static_cast<long long>(G.nx) * G.ny);
}

cudaError_t
launch_project_mean_zero(const DevGeom &G, double *x, int n_intervals, double *scratch, cudaStream_t st)
{
  if (n_intervals <= 0)
    return cudaSuccess;
  // mean = <m, p> / |Omega| with m = |K| on mode 0 (dof_space.cpp:96-119)
  const double cell_area = G.hx * G.hy;
  const double volume = (G.nx * G.hx) * (G.ny * G.hy);
  dim3 grid(G.S, n_intervals, proj_chunks(static_cast<long long>(G.nx) * G.ny));
  pmz_partial_kernel<<<grid, kProjThreads, 0, st>>>(G, x, scratch);
  pmz_apply_kernel<<<grid, kProjThreads, 0, st>>>(G, x, scratch, cell_area / volume);
  return cudaGetLastError();
}

cudaError_t
launch_zero_constrained(const DevGeom &G, double *x, int n_intervals, cudaStream_t st)
{
  if (n_intervals <= 0)
    return cudaSuccess;
  const long long total = static_cast<long long>(2 * (G.gx + G.gy) - 4) * 2 * G.S;
  dim3 grid(static_cast<unsigned>((total + 127) / 128), n_intervals);
  zero_constrained_kernel<<<grid, 128, 0, st>>>(G, x);
  return cudaGetLastError();
}

cudaError_t
launch_coarse_solve(const double *inv, const long long *pinned, int n_pinned, int nrows, const double *b, double *x,
                    cudaStream_t st)
{
  const int th = 256;
  const int blocks = (nrows * 32 + th - 1) / th;
  coarse_solve_kernel<<<blocks, th, 0, st>>>(inv, pinned, n_pinned, nrows, b, x);
  return cudaGetLastError();
}

int
dot_partials()
{
  return 148 * 4;
}

cudaError_t
launch_dot(const double *x, const double *y, long long n, double *part, double *out, cudaStream_t st)
{
  const int nb = std::min<long long>(dot_partials(), std::max<long long>(1, (n + kDotThreads - 1) / kDotThreads));
  dot_partial_kernel<<<nb, kDotThreads, 0, st>>>(x, y, n, part);
  dot_final_kernel<<<1, kDotThreads, 0, st>>>(part, nb, out);
  return cudaGetLastError();
}

cudaError_t
launch_multidot(const double *const *V, int m, bool with_norm, const double *w, long long n, double *part,
                double *out, cudaStream_t st)
{
  // out[i] = <w, V_i> (i < m), out[m] = <w, w> if with_norm; chunks of kMultiMax
  const int nb = std::min<long long>(dot_partials(), std::max<long long>(1, (n + kDotThreads - 1) / kDotThreads));
  for (int i0 = 0;; i0 += kMultiMax)
    {
      const int mm = std::min(kMultiMax, m - i0); // 0 when m == 0 (norm only)
      const bool last = i0 + kMultiMax >= m;
      const int wn = last && with_norm ? 1 : 0;
      MultiVec mv{};
      for (int i = 0; i < mm; ++i)
        mv.p[i] = V[i0 + i];
      if (mm + wn > 0)
        {
          multidot_partial_kernel<<<nb, kDotThreads, 0, st>>>(mv, mm, wn, w, n, part);
          multidot_final_kernel<<<mm + wn, kDotThreads, 0, st>>>(part, nb, out + i0); // norm lands at out[m]
        }
      if (last)
        break;
    }
  return cudaGetLastError();
}

cudaError_t
launch_multi_axpy(const double *const *V, int m, const double *c_dev, const double *c_host, double sign, double *w,
                  long long n, cudaStream_t st)
{
  for (int i0 = 0; i0 < m; i0 += kMultiMax)
    {
      MultiVec mv{};
      MultiCoef mc{};
      const int mm = std::min(kMultiMax, m - i0);
      for (int i = 0; i < mm; ++i)
        {
          mv.p[i] = V[i0 + i];
          if (c_host)
            mc.c[i] = c_host[i0 + i];
        }
      multi_axpy_kernel<<<grid_for(n, 256), 256, 0, st>>>(mv, mm, c_dev ? c_dev + i0 : nullptr, mc, sign, w, n);
    }
  return cudaGetLastError();
}

cudaError_t
launch_axpy(long long n, double alpha, const double *alpha_dev, double sign, const double *x, double *y,
            cudaStream_t st)
{
  axpy_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, alpha, alpha_dev, sign, x, y);
  return cudaGetLastError();
}

cudaError_t
launch_scale(long long n, double alpha, double *y, cudaStream_t st)
{
  scale_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, alpha, y);
  return cudaGetLastError();
}

cudaError_t
launch_xpby(long long n, const double *x, double beta, double *y, cudaStream_t st)
{
  xpby_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, x, beta, y);
  return cudaGetLastError();
}

cudaError_t
launch_coarse_forward(const double *G, const double *H, int n, int mv, long long v_off, const double *B, int n_all,
                      int n_begin, int n_own, double *X, cudaStream_t st)
{
  const size_t smem = sizeof(double) * (n + mv);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(coarse_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  coarse_forward_kernel<<<1, 1024, smem, st>>>(G, H, n, mv, v_off, B, n_all, n_begin, n_own, X);
  return cudaGetLastError();
}

} // namespace stmg_b200

// ---------------------------------------------------------------- step health
namespace stmg_b200
{
namespace
{
constexpr int kHealthThreads = 256;
/// Per (interval, slot): sum (B v)^2, v . M v, <mean, p>, p . p from the
/// health application y = [M v^a ; B v^a] (solver.cpp:286-299).
__global__ void __launch_bounds__(kHealthThreads)
health_kernel(DevGeom G, double cell_area, const double *__restrict__ X, const double *__restrict__ Y,
              double *__restrict__ out)
{
  const int a = blockIdx.x, n = blockIdx.y;
  const double *xv = X + n * G.isz + a * G.mv, *yv = Y + n * G.isz + a * G.mv;
  const double *xp = X + n * G.isz + G.S * G.mv + a * G.mp, *yp = Y + n * G.isz + G.S * G.mv + a * G.mp;
  double s_div = 0.0, s_vmv = 0.0, s_m = 0.0, s_p = 0.0;
  for (long long i = threadIdx.x; i < G.mv; i += kHealthThreads)
    s_vmv = fma(xv[i], yv[i], s_vmv);
  for (long long i = threadIdx.x; i < G.mp; i += kHealthThreads)
    {
      s_div = fma(yp[i], yp[i], s_div);
      s_p = fma(xp[i], xp[i], s_p);
      if (i % G.np == 0)
        s_m = fma(cell_area, xp[i], s_m); // mean vector: |K| on the constant mode (dof_space.cpp:99-105)
    }
  s_div = block_sum<kHealthThreads>(s_div);
  s_vmv = block_sum<kHealthThreads>(s_vmv);
  s_m = block_sum<kHealthThreads>(s_m);
  s_p = block_sum<kHealthThreads>(s_p);
  if (threadIdx.x == 0)
    {
      double *o = out + 4 * (static_cast<long long>(n) * G.S + a);
      o[0] = s_div;
      o[1] = s_vmv;
      o[2] = s_m;
      o[3] = s_p;
    }
}
} // namespace

cudaError_t
launch_health(const DevGeom &G, double cell_area, const double *X, const double *Y, double *out, int n_intervals,
              cudaStream_t st)
{
  if (n_intervals == 0)
    return cudaSuccess;
  dim3 grid(G.S, n_intervals);
  health_kernel<<<grid, kHealthThreads, 0, st>>>(G, cell_area, X, Y, out);
  return cudaGetLastError();
}
} // namespace stmg_b200
