// FP64 mma.sync throughput per shape on sm_100a: m8n8k4 (sm_80) and the
// sm_90+ shapes m16n8k4 / m16n8k8 / m16n8k16. One JSON line.
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__global__ void mma_kernel(double *out, int iters)
{
  const double a = 1e-3 * (threadIdx.x & 7), b = 1e-3 * (threadIdx.x >> 3);
  double s = 0.0;
  if constexpr (SHAPE == 0)
    {
      double d[8][2] = {};
      for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int t = 0; t < 8; ++t)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(d[t][0]), "+d"(d[t][1]) : "d"(a), "d"(b));
      for (int t = 0; t < 8; ++t) s += d[t][0] + d[t][1];
    }
  else if constexpr (SHAPE == 1) // m16n8k4: A 2, B 1, C 4 doubles per lane
    {
      double d[8][4] = {};
      for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int t = 0; t < 8; ++t)
          asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                       : "+d"(d[t][0]), "+d"(d[t][1]), "+d"(d[t][2]), "+d"(d[t][3]) : "d"(a), "d"(b), "d"(a));
      for (int t = 0; t < 8; ++t) s += d[t][0] + d[t][1] + d[t][2] + d[t][3];
    }
  else if constexpr (SHAPE == 2) // m16n8k8: A 4, B 2, C 4
    {
      double d[8][4] = {};
      for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int t = 0; t < 8; ++t)
          asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                       : "+d"(d[t][0]), "+d"(d[t][1]), "+d"(d[t][2]), "+d"(d[t][3])
                       : "d"(a), "d"(b), "d"(a), "d"(b), "d"(a), "d"(b));
      for (int t = 0; t < 8; ++t) s += d[t][0] + d[t][1] + d[t][2] + d[t][3];
    }
  else // m16n8k16: A 8, B 4, C 4
    {
      double d[8][4] = {};
      for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int t = 0; t < 8; ++t)
          asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
                       "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
                       : "+d"(d[t][0]), "+d"(d[t][1]), "+d"(d[t][2]), "+d"(d[t][3])
                       : "d"(a), "d"(b), "d"(a), "d"(b), "d"(a), "d"(b), "d"(a), "d"(b), "d"(a), "d"(b), "d"(a),
                         "d"(b));
      for (int t = 0; t < 8; ++t) s += d[t][0] + d[t][1] + d[t][2] + d[t][3];
    }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int SHAPE>
double run(double *out, int sms)
{
  const int blocks = sms * 4, threads = 256, iters = SHAPE == 3 ? 512 : (SHAPE == 2 ? 1024 : 2048);
  const double macs = SHAPE == 0 ? 256.0 : (SHAPE == 1 ? 512.0 : (SHAPE == 2 ? 1024.0 : 2048.0));
  mma_kernel<SHAPE><<<blocks, threads>>>(out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f, ms;
  for (int rep = 0; rep < 3; ++rep)
    {
      cudaEventRecord(e0);
      mma_kernel<SHAPE><<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
  return 2.0 * macs * (blocks * threads / 32.0) * iters * 8 / (best * 1e-3) / 1e12;
}

int main()
{
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out;
  cudaMalloc(&out, sizeof(double) * sms * 4 * 256);
  const double t0 = run<0>(out, sms), t1 = run<1>(out, sms), t2 = run<2>(out, sms), t3 = run<3>(out, sms);
  printf("{\"m8n8k4\": %.2f, \"m16n8k4\": %.2f, \"m16n8k8\": %.2f, \"m16n8k16\": %.2f, \"err\": \"%s\"}\n", t0, t1, t2,
         t3, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
