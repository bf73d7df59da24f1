// nccl_arm.cpp -- the paper's NCCL send/recv transport as a comparison arm
// (include/mempool_nccl.h).  Thin: one ncclGroup per call over caller-given
// device pointers.  Built into its own library so libmempool.so does not
// depend on NCCL.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "../../include/mempool_nccl.h"

struct mp_nccl_comm {
  ncclComm_t comm = nullptr;
  int device = 0;
};

namespace {
thread_local std::string g_err;

int fail(ncclResult_t r, const char* where) {
  g_err = std::string(where) + ": " + ncclGetErrorString(r);
  return (int)r;
}
}  // namespace

extern "C" {

const char* mp_nccl_last_error(void) { return g_err.c_str(); }

int32_t mp_nccl_version(void) {
  int v = 0;
  ncclGetVersion(&v);
  return v;
}

int mp_nccl_unique_id(void* out, int64_t cap) {
  if (!out || cap < (int64_t)sizeof(ncclUniqueId)) return -1;
  ncclUniqueId id;
  const ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(r, "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
  return 0;
}

int mp_nccl_comm_init(int32_t nranks, int32_t rank, const void* unique_id, int32_t device,
                      mp_nccl_comm** out) {
  if (!unique_id || !out || nranks < 1 || rank < 0 || rank >= nranks) return -1;
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) {
    g_err = "cudaSetDevice failed";
    return -1;
  }
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  auto* c = new mp_nccl_comm();
  c->device = device;
  const ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
  cudaSetDevice(prev);
  if (r != ncclSuccess) {
    delete c;
    return fail(r, "ncclCommInitRank");
  }
  *out = c;
  return 0;
}

void mp_nccl_comm_destroy(mp_nccl_comm* c) {
  if (!c) return;
  if (c->comm) ncclCommDestroy(c->comm);
  delete c;
}

int mp_nccl_exchange(mp_nccl_comm* c, int32_t peer_send, void* const* send_ptrs,
                     const int64_t* send_bytes, int64_t n_send, int32_t peer_recv,
                     void* const* recv_ptrs, const int64_t* recv_bytes, int64_t n_recv,
                     void* stream) {
  if (!c || n_send < 0 || n_recv < 0 || (n_send && (!send_ptrs || !send_bytes)) ||
      (n_recv && (!recv_ptrs || !recv_bytes)))
    return -1;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  const cudaStream_t s = (cudaStream_t)stream;
  ncclResult_t r = ncclGroupStart();
  for (int64_t i = 0; r == ncclSuccess && i < n_send; ++i)
    r = ncclSend(send_ptrs[i], (size_t)send_bytes[i], ncclUint8, peer_send, c->comm, s);
  for (int64_t i = 0; r == ncclSuccess && i < n_recv; ++i)
    r = ncclRecv(recv_ptrs[i], (size_t)recv_bytes[i], ncclUint8, peer_recv, c->comm, s);
  const ncclResult_t e = ncclGroupEnd();
  cudaSetDevice(prev);
  if (r != ncclSuccess) return fail(r, "ncclSend/ncclRecv");
  if (e != ncclSuccess) return fail(e, "ncclGroupEnd");
  return 0;
}

}  // extern "C"
