// NCCL communicators of the library: the three exchanges of
// the time-slab partition -- the slot-k velocity halo to the next rank
// (ncclSend / ncclRecv), the Krylov all-reduces and the all-gather of the
// coarse right-hand sides -- as stmg_comm_ops callbacks, and for the C5
// hybrid split the interface-plane exchange between z parts, their
// all-reduce and all-gather (stmg_comm_space_ops). The callbacks call NCCL
// directly on the solver's stream; no caller code runs per exchange.
//
// libnccl.so.2 is opened at run time (dlopen), so the library loads on hosts
// without NCCL and binds to whichever NCCL the process already has (torch's
// bundled one when torch is loaded, else the system's). The handful of entry
// points used are declared here with the NCCL C ABI (nccl.h, NCCL >= 2.7).
#include "runtime.hpp"

#include <cstring>
#include <dlfcn.h>
#include <memory>
#include <mutex>
#include <string>

namespace
{
typedef struct ncclComm *ncclComm_t;
struct NcclUniqueId
{
  char internal[128];
};
typedef int ncclResult_t; // ncclSuccess = 0
enum
{
  kNcclFloat64 = 8, // ncclDouble
  kNcclSum = 0,
};

struct NcclApi
{
  void *handle = nullptr;
  std::string error;
  ncclResult_t (*GetUniqueId)(NcclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, NcclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi &
nccl()
{
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char *name : {"libnccl.so.2", "libnccl.so"})
      {
        // RTLD_NOLOAD first: reuse an NCCL the process already loaded (torch)
        api.handle = dlopen(name, RTLD_NOW | RTLD_NOLOAD);
        if (!api.handle)
          api.handle = dlopen(name, RTLD_NOW | RTLD_LOCAL);
        if (api.handle)
          break;
      }
    if (!api.handle)
      {
        api.error = std::string("libnccl.so.2 not loadable: ") + dlerror();
        return;
      }
    auto sym = [&](auto &fn, const char *name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(api.handle, name));
      if (!fn && api.error.empty())
        api.error = std::string("NCCL symbol missing: ") + name;
    };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.Send, "ncclSend");
    sym(api.Recv, "ncclRecv");
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.AllGather, "ncclAllGather");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.GetErrorString, "ncclGetErrorString");
  });
  if (!api.error.empty())
    throw std::runtime_error(api.error);
  return api;
}

void
nccl_check(ncclResult_t r, const char *what)
{
  if (r != 0)
    throw std::runtime_error(std::string(what) + ": " + nccl().GetErrorString(r));
}
} // namespace

struct stmg_comm
{
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1, device = 0;
  ~stmg_comm()
  {
    if (comm)
      nccl().CommDestroy(comm);
  }
};

namespace
{
// stmg_comm_ops callbacks: 0 on success (errors are reported by the status)
int
cb_halo(void *user, const double *send, double *recv, int64_t n, void *stream)
{
  auto *c = static_cast<stmg_comm *>(user);
  try
    {
      NcclApi &api = nccl();
      auto st = static_cast<cudaStream_t>(stream);
      nccl_check(api.GroupStart(), "ncclGroupStart");
      if (c->rank + 1 < c->world)
        nccl_check(api.Send(send, static_cast<size_t>(n), kNcclFloat64, c->rank + 1, c->comm, st), "ncclSend");
      if (c->rank > 0)
        nccl_check(api.Recv(recv, static_cast<size_t>(n), kNcclFloat64, c->rank - 1, c->comm, st), "ncclRecv");
      nccl_check(api.GroupEnd(), "ncclGroupEnd");
      return 0;
    }
  catch (const std::exception &e)
    {
      stmg_rt::g_error = e.what();
      return 1;
    }
}

int
cb_allreduce(void *user, double *buf, int64_t n, void *stream)
{
  auto *c = static_cast<stmg_comm *>(user);
  try
    {
      nccl_check(nccl().AllReduce(buf, buf, static_cast<size_t>(n), kNcclFloat64, kNcclSum, c->comm,
                                  static_cast<cudaStream_t>(stream)),
                 "ncclAllReduce");
      return 0;
    }
  catch (const std::exception &e)
    {
      stmg_rt::g_error = e.what();
      return 1;
    }
}

int
cb_allgather(void *user, const double *send, double *recv, int64_t n, void *stream)
{
  auto *c = static_cast<stmg_comm *>(user);
  try
    {
      nccl_check(nccl().AllGather(send, recv, static_cast<size_t>(n), kNcclFloat64, c->comm,
                                  static_cast<cudaStream_t>(stream)),
                 "ncclAllGather");
      return 0;
    }
  catch (const std::exception &e)
    {
      stmg_rt::g_error = e.what();
      return 1;
    }
}
// stmg_comm_space_ops: the z parts of the hybrid split, rank = part
int
cb_planes(void *user, const double *send_lo, double *recv_lo, const double *send_hi, double *recv_hi, int64_t n,
          void *stream)
{
  auto *c = static_cast<stmg_comm *>(user);
  try
    {
      NcclApi &api = nccl();
      auto st = static_cast<cudaStream_t>(stream);
      const size_t m = static_cast<size_t>(n);
      nccl_check(api.GroupStart(), "ncclGroupStart");
      if (send_lo && c->rank > 0)
        {
          nccl_check(api.Send(send_lo, m, kNcclFloat64, c->rank - 1, c->comm, st), "ncclSend");
          nccl_check(api.Recv(recv_lo, m, kNcclFloat64, c->rank - 1, c->comm, st), "ncclRecv");
        }
      if (send_hi && c->rank + 1 < c->world)
        {
          nccl_check(api.Send(send_hi, m, kNcclFloat64, c->rank + 1, c->comm, st), "ncclSend");
          nccl_check(api.Recv(recv_hi, m, kNcclFloat64, c->rank + 1, c->comm, st), "ncclRecv");
        }
      nccl_check(api.GroupEnd(), "ncclGroupEnd");
      return 0;
    }
  catch (const std::exception &e)
    {
      stmg_rt::g_error = e.what();
      return 1;
    }
}
} // namespace

using stmg_rt::guarded;

extern "C" {

int
stmg_comm_nccl_unique_id(void *unique_id_out)
{
  return guarded([&] {
    if (!unique_id_out)
      throw std::invalid_argument("stmg_comm_nccl_unique_id: null output");
    NcclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(unique_id_out, &id, sizeof(id));
  });
}

int
stmg_comm_nccl_create(const void *unique_id, int rank, int world, int device, stmg_comm **out)
{
  return guarded([&] {
    STMG_NVTX("stmg_comm_nccl_create");
    if (!unique_id || !out)
      throw std::invalid_argument("stmg_comm_nccl_create: null argument");
    if (world < 1 || rank < 0 || rank >= world)
      throw std::invalid_argument("stmg_comm_nccl_create: invalid rank/world");
    check(cudaSetDevice(device), "cudaSetDevice");
    auto c = std::make_unique<stmg_comm>();
    c->rank = rank;
    c->world = world;
    c->device = device;
    NcclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    nccl_check(nccl().CommInitRank(&c->comm, world, id, rank), "ncclCommInitRank");
    *out = c.release();
  });
}

int
stmg_comm_nccl_ops(stmg_comm *comm, stmg_comm_ops *ops_out)
{
  return guarded([&] {
    if (!comm || !ops_out)
      throw std::invalid_argument("stmg_comm_nccl_ops: null argument");
    ops_out->user = comm;
    ops_out->rank = comm->rank;
    ops_out->world = comm->world;
    ops_out->exchange_halo = cb_halo;
    ops_out->allreduce_sum = cb_allreduce;
    ops_out->allgather = cb_allgather;
  });
}

int
stmg_comm_nccl_space_ops(stmg_comm *comm, stmg_comm_space_ops *ops_out)
{
  return guarded([&] {
    if (!comm || !ops_out)
      throw std::invalid_argument("stmg_comm_nccl_space_ops: null argument");
    ops_out->user = comm;
    ops_out->part = comm->rank;
    ops_out->parts = comm->world;
    ops_out->exchange_planes = cb_planes;
    ops_out->allreduce_sum = cb_allreduce;
    ops_out->allgather = cb_allgather;
  });
}

int
stmg_comm_destroy(stmg_comm *comm)
{
  return guarded([&] { delete comm; });
}

} // extern "C"
