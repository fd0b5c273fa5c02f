// Host runtime shared by the C-ABI translation units (2D stmg.cu, 3D
// stmg3d.cu): error capture for stmg_last_error, owning device arrays and
// the context (stream, launch counter, copy streams).
#pragma once

#include "../../include/stmg_b200.h"

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdarg>
#include <cstdio>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdexcept>
#include <string>
#include <vector>

namespace stmg_rt
{
inline thread_local std::string g_error;

struct CudaError : std::runtime_error
{
  using std::runtime_error::runtime_error;
};

inline void
check(cudaError_t e, const char *what)
{
  if (e != cudaSuccess)
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int
guarded(F &&f)
{
  try
    {
      f();
      return STMG_OK;
    }
  catch (const std::invalid_argument &e)
    {
      g_error = e.what();
      return STMG_EINVAL;
    }
  catch (const CudaError &e)
    {
      g_error = e.what();
      return STMG_ECUDA;
    }
  catch (const std::exception &e)
    {
      g_error = e.what();
      return STMG_ERUNTIME;
    }
}

/// NVTX range (profiling: one range per C-ABI call, V-cycle
/// level and phase, Krylov iteration and time step). nvtx3 is header-only and
/// costs a null-pointer test when no tool is attached.
struct NvtxRange
{
  explicit NvtxRange(const char *fmt, ...)
  {
    char buf[96];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    nvtxRangePushA(buf);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};
#define STMG_NVTX_CAT2(a, b) a##b
#define STMG_NVTX_CAT(a, b) STMG_NVTX_CAT2(a, b)
#define STMG_NVTX(...) ::stmg_rt::NvtxRange STMG_NVTX_CAT(nvtx_range_, __LINE__)(__VA_ARGS__)

/// Reallocations of any DevArray: captured CUDA graphs hold raw pointers and
/// are re-captured when this changes.
inline std::atomic<uint64_t> g_reallocs{0};

/// Owning device array.
template <class T>
struct DevArray
{
  T *p = nullptr;
  size_t n = 0;
  DevArray() = default;
  DevArray(const DevArray &) = delete;
  DevArray &operator=(const DevArray &) = delete;
  DevArray(DevArray &&o) noexcept : p(o.p), n(o.n)
  {
    o.p = nullptr;
    o.n = 0;
  }
  ~DevArray()
  {
    if (p)
      cudaFree(p);
  }
  void
  resize(size_t count)
  {
    if (count <= n)
      return;
    if (p)
      cudaFree(p);
    p = nullptr;
    n = 0;
    check(cudaMalloc(&p, sizeof(T) * std::max<size_t>(count, 1)), "cudaMalloc");
    n = count;
    g_reallocs.fetch_add(1, std::memory_order_relaxed);
  }
  void
  release()
  {
    if (p)
      cudaFree(p);
    p = nullptr;
    n = 0;
    g_reallocs.fetch_add(1, std::memory_order_relaxed);
  }
  void
  upload(const std::vector<T> &h)
  {
    resize(h.size());
    if (!h.empty())
      check(cudaMemcpy(p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice), "upload");
  }
};
} // namespace stmg_rt

// ================================================================ context
using stmg_rt::check;
struct stmg_ctx
{
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t launches = 0;
  // copy streams + events of the pipelined host-buffer entry points
  cudaStream_t h2d = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> events;
  void
  count(int k = 1)
  {
    launches += k;
  }
  void
  copy_streams()
  {
    if (!h2d)
      check(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking), "stream");
    if (!d2h)
      check(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking), "stream");
  }
  cudaEvent_t
  event(size_t i)
  {
    while (events.size() <= i)
      {
        cudaEvent_t e;
        check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        events.push_back(e);
      }
    return events[i];
  }
  ~stmg_ctx()
  {
    for (cudaEvent_t e : events)
      cudaEventDestroy(e);
    if (h2d)
      cudaStreamDestroy(h2d);
    if (d2h)
      cudaStreamDestroy(d2h);
  }
};
