/*
 * mempool_nccl.h -- C-ABI of libmempool_nccl.so: the paper's own transport,
 * NCCL send/recv (§5.2: "we use NCCL's send and
 * recv"; one call per (layer, K/V) block in the discrete layout, one per
 * aggregated block after P:549-550), kept as a COMPARISON ARM beside the
 * fused one-sided path of libmempool.so.  It moves bytes
 * between device pointers the caller computes (slab chunks, or the
 * aggregated staging written by mp_pack / read by mp_unpack); it has no pool
 * state of its own.
 *
 * Conventions: every function returns 0 on success, else the ncclResult_t
 * (positive) or -1 for an argument error; mp_nccl_last_error() describes the
 * last failure.  Pointer arrays are HOST arrays of DEVICE pointers on the
 * communicator's device, owned by the caller, read during the call only.
 * Work is enqueued on `stream` (a cudaStream_t, NULL = legacy default);
 * the caller synchronises.
 */
#ifndef MEMPOOL_NCCL_H
#define MEMPOOL_NCCL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mp_nccl_comm mp_nccl_comm;

/* 128-byte ncclUniqueId into out (rank 0 creates it, the others receive it
 * through the caller's bootstrap, e.g. torch.distributed). */
int mp_nccl_unique_id(void* out, int64_t cap);
/* ncclCommInitRank on `device` (sets it current for the call). */
int mp_nccl_comm_init(int32_t nranks, int32_t rank, const void* unique_id, int32_t device,
                      mp_nccl_comm** out);
void mp_nccl_comm_destroy(mp_nccl_comm* comm);
/* One NCCL group: n_send ncclSend(send_ptrs[i], send_bytes[i]) to peer_send
 * and n_recv ncclRecv(recv_ptrs[i], recv_bytes[i]) from peer_recv, in order
 * (NCCL matches the i-th send with the peer's i-th recv).  peer == own rank
 * is a local copy through NCCL (a one-rank communicator on one GPU). */
int mp_nccl_exchange(mp_nccl_comm* comm, int32_t peer_send, void* const* send_ptrs,
                     const int64_t* send_bytes, int64_t n_send, int32_t peer_recv,
                     void* const* recv_ptrs, const int64_t* recv_bytes, int64_t n_recv,
                     void* stream);
const char* mp_nccl_last_error(void);
/* NCCL version as major*10000 + minor*100 + patch. */
int32_t mp_nccl_version(void);

#ifdef __cplusplus
}
#endif

#endif /* MEMPOOL_NCCL_H */
