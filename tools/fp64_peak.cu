// Measures FP64 throughput on the current GPU: DFMA (CUDA cores), DMMA
// (mma.sync m8n8k4 f64 tensor path), cuBLAS DGEMM, and a copy bandwidth.
// Output: one JSON line. Used to fill profiles/fp64_peaks.json (the FP64
// roofline denominator; MEASURED_PEAKS.json carries only bf16/HBM).
#include <cstdio>
#include <cublas_v2.h>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double *out, int iters)
{
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i)
    {
#pragma unroll
      for (int u = 0; u < 16; ++u)
        {
          a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
          a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma_kernel(double *out, int iters)
{
  double a = 1e-3 * (threadIdx.x & 7), b = 1e-3 * (threadIdx.x >> 3);
  double d[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t)
    d[t][0] = d[t][1] = 0.0;
  for (int i = 0; i < iters; ++i)
    {
#pragma unroll
      for (int t = 0; t < 8; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(d[t][0]), "+d"(d[t][1])
                     : "d"(a), "d"(b));
    }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t)
    s += d[t][0] + d[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void copy_kernel(const double2 *__restrict__ a, double2 *__restrict__ b, size_t n)
{
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

int main()
{
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out;
  cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  // DFMA
  const int blocks = sms * 4, threads = 512, iters = 4096;
  dfma_kernel<<<blocks, threads>>>(out, 16);
  cudaEventRecord(e0);
  dfma_kernel<<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double dfma_tf = 2.0 * blocks * threads * (double)iters * 16 * 8 / (ms * 1e-3) / 1e12;
  // DMMA
  const int mb = sms * 4, mt = 256, miters = 4096;
  dmma_kernel<<<mb, mt>>>(out, 16);
  cudaEventRecord(e0);
  dmma_kernel<<<mb, mt>>>(out, miters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double dmma_tf = 2.0 * 256 * (mb * mt / 32.0) * (double)miters * 8 / (ms * 1e-3) / 1e12;
  // cuBLAS DGEMM 8192^3
  const int N = 8192;
  double *A, *B, *C;
  cudaMalloc(&A, sizeof(double) * N * N);
  cudaMalloc(&B, sizeof(double) * N * N);
  cudaMalloc(&C, sizeof(double) * N * N);
  cudaMemset(A, 0, sizeof(double) * N * N);
  cudaMemset(B, 0, sizeof(double) * N * N);
  cublasHandle_t h;
  cublasCreate(&h);
  const double one = 1.0, zero = 0.0;
  cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, N, N, N, &one, A, N, B, N, &zero, C, N);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep)
    {
      cudaEventRecord(e0);
      cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, N, N, N, &one, A, N, B, N, &zero, C, N);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
  const double dgemm_tf = 2.0 * N * (double)N * N / (best * 1e-3) / 1e12;
  // copy bandwidth, 2 GiB each way
  const size_t nbytes = size_t(2) << 30;
  double2 *src = (double2 *)A, *dst = (double2 *)B;
  cudaFree(C);
  cudaFree(A);
  cudaFree(B);
  cudaMalloc(&src, nbytes);
  cudaMalloc(&dst, nbytes);
  cudaMemset(src, 0, nbytes);
  copy_kernel<<<sms * 8, 512>>>(src, dst, nbytes / 16);
  best = 1e30f;
  for (int rep = 0; rep < 10; ++rep)
    {
      cudaEventRecord(e0);
      copy_kernel<<<sms * 8, 512>>>(src, dst, nbytes / 16);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
  const double copy_gbs = 2.0 * nbytes / (best * 1e-3) / 1e9;
  printf("{\"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, \"cublas_dgemm_tflops\": %.2f, \"copy_gbs\": %.1f, "
         "\"sms\": %d, \"err\": \"%s\"}\n",
         dfma_tf, dmma_tf, dgemm_tf, copy_gbs, sms, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
