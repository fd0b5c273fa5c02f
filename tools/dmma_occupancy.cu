// DMMA (FP64 mma.sync m8n8k4) throughput vs. warps per SM, independent
// accumulator chains per warp and where the B operand comes from (register
// or a fresh LDS per DMMA, as vanka_tc_kernel does). Answers: is the Vanka
// kernel's structure (16 warps/SM, 4 chains, LDS-fed B) able to saturate
// the FP64 tensor path at all?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_occupancy tools/dmma_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS, bool LDS_B>
__global__ void
dmma_kernel(double *out, int iters)
{
  __shared__ double sb[8 * 132 * 4];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 8 * 132 * 4; i += blockDim.x)
    sb[i] = 1e-3 * (i & 15);
  __syncthreads();
  double a = 1e-3 * (threadIdx.x & 7), b = 1e-3 * (threadIdx.x >> 3);
  double d[CHAINS][2];
#pragma unroll
  for (int t = 0; t < CHAINS; ++t)
    d[t][0] = d[t][1] = 0.0;
  const volatile double *bb = sb + (lane >> 2) * 132 + (lane & 3); // volatile: one LDS per DMMA
  for (int i = 0; i < iters; ++i)
    {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
#pragma unroll
        for (int t = 0; t < CHAINS; ++t)
          {
            double bv = b;
            if (LDS_B)
              bv = bb[kk * 4 + (t & 3) * 8 * 132];
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(d[t][0]), "+d"(d[t][1])
                         : "d"(a), "d"(bv));
          }
    }
  double s = 0;
#pragma unroll
  for (int t = 0; t < CHAINS; ++t)
    s += d[t][0] + d[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CHAINS, bool LDS_B>
void
run(int sms, int warps_per_sm, double *out)
{
  const int threads = warps_per_sm >= 16 ? 512 : warps_per_sm * 32;
  const int blocks = sms * (warps_per_sm * 32 / threads);
  const int iters = 2048;
  dmma_kernel<CHAINS, LDS_B><<<blocks, threads>>>(out, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  dmma_kernel<CHAINS, LDS_B><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 256 * (blocks * threads / 32.0) * iters * 8 * CHAINS;
  printf("{\"warps_per_sm\": %d, \"chains\": %d, \"b_from_lds\": %d, \"tflops\": %.2f}\n", warps_per_sm, CHAINS,
         int(LDS_B), flops / (ms * 1e-3) / 1e12);
}

int
main()
{
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out;
  cudaMalloc(&out, sizeof(double) * sms * 4096);
  for (int w : {8, 12, 16, 32})
    {
      run<4, false>(sms, w, out);
      run<4, true>(sms, w, out);
      run<8, true>(sms, w, out);
      run<2, true>(sms, w, out);
    }
  return 0;
}
