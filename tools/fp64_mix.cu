// Do DFMA (FP64 pipe) and DMMA (FP64 tensor sub-pipe) issue concurrently?
// mode 0: all warps DFMA; mode 1: all warps DMMA; mode 2: even warps DFMA,
// odd warps DMMA (same per-warp work as in modes 0/1). One JSON line.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dfma_work(double *out, int iters)
{
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int u = 0; u < 16; ++u)
      {
        a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
        a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
      }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__device__ __forceinline__ void dmma_work(double *out, int iters)
{
  double a = 1e-3 * (threadIdx.x & 7), b = 1e-3 * (threadIdx.x >> 3);
  double d[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t)
    d[t][0] = d[t][1] = 0.0;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[t][0]), "+d"(d[t][1])
                   : "d"(a), "d"(b));
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t)
    s += d[t][0] + d[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void mix_kernel(double *out, int mode, int fi, int mi)
{
  const int w = threadIdx.x >> 5;
  const bool dfma = mode == 0 || (mode == 2 && (w & 1) == 0);
  if (dfma)
    dfma_work(out, fi);
  else
    dmma_work(out, mi);
}

int main()
{
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4, threads = 256, fi = 2048, mi = 2048;
  double *out;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double tf[3];
  for (int mode = 0; mode < 3; ++mode)
    {
      mix_kernel<<<blocks, threads>>>(out, mode, 16, 16);
      float best = 1e30f, ms;
      for (int rep = 0; rep < 3; ++rep)
        {
          cudaEventRecord(e0);
          mix_kernel<<<blocks, threads>>>(out, mode, fi, mi);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          cudaEventElapsedTime(&ms, e0, e1);
          best = ms < best ? ms : best;
        }
      const double warps = blocks * threads / 32.0;
      const double f_dfma_warp = 2.0 * 32 * fi * 16 * 8, f_dmma_warp = 2.0 * 256 * mi * 8;
      double flops = 0;
      if (mode == 0) flops = warps * f_dfma_warp;
      if (mode == 1) flops = warps * f_dmma_warp;
      if (mode == 2) flops = warps / 2 * (f_dfma_warp + f_dmma_warp);
      tf[mode] = flops / (best * 1e-3) / 1e12;
    }
  printf("{\"dfma_only_tflops\": %.2f, \"dmma_only_tflops\": %.2f, \"mixed_tflops\": %.2f, \"err\": \"%s\"}\n", tf[0],
         tf[1], tf[2], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
