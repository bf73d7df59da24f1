// mempool.cpp -- the C-ABI (include/mempool.h) and the host runtime of
// libmempool: pool object, host shadow of the device allocator, prompt
// index, transfer engine and swap engine.
//
// Paper map: PAPER.md Table tbl-mempool-api for the entry points,
// §4.3 for the allocation -> transmission -> insertion workflow,
// §5.2 for the aggregated staging / DRAM layout.  Readings where
// the paper is silent: R1-R13.
#include "../../include/mempool.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <deque>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "index.hpp"
#include "kernels.cuh"

namespace {

thread_local std::string g_err;

void set_err(const std::string& s) { g_err = s; }

enum : uint8_t { ST_FREE = 0, ST_ACTIVE = 1, ST_INDEXED = 2, ST_ORPHAN = 3 };

struct DevGuard {
  int prev = -1, want;
  explicit DevGuard(int d) : want(d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DevGuard() {
    if (prev >= 0 && prev != want) cudaSetDevice(prev);
  }
};

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      set_err(std::string(#x) + ": " + cudaGetErrorString(e_));                      \
      return MP_ERR_CUDA;                                                            \
    }                                                                                \
  } while (0)

#define TRY(x)                    \
  do {                            \
    mp_status s_ = (x);           \
    if (s_ != MP_OK) return s_;   \
  } while (0)

struct Msg {
  int32_t kind, src;
  std::vector<uint8_t> priv;
  std::vector<mp_addr> addrs;
};

// Bump arena of int32 ids: device buffer + mapped pinned mirror.  Reset at
// the start of every API call (every call ends with a stream sync).
struct Arena {
  int* d = nullptr;
  int* h = nullptr;
  int64_t cap = 0, used = 0;
};

}  // namespace

struct mp_pool {
  // shape
  int32_t inst = 0, dev = 0, L = 0, H = 0, D = 0, elem = 0, B = 0;
  bool verify = false;
  int64_t chunk = 0, Pb = 0, n_hbm = 0, n_dram = 0;
  int nch = 0;
  int max_ctas = 0;
  // device memory
  std::vector<char*> slabs;
  void* own_slab_region = nullptr;
  char** d_slabs = nullptr;
  uint32_t* d_bitmap = nullptr;
  int nwords = 0;
  int* d_err = nullptr;
  Arena ar;
  char* dram = nullptr;     // host pointer
  char* dram_dev = nullptr; // device-visible (mapped) pointer
  bool own_dram = false;
  char* staging = nullptr;
  int64_t staging_bytes = 0;
  int staging_slots = 4;
  cudaStream_t stream = nullptr, copy_stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<cudaEvent_t> slot_ev;
  bool profiling = false;
  mp_stats stats{};
  // host shadow of block ownership
  std::vector<uint8_t> st[2];
  std::vector<int32_t> alloc_by[2];
  int64_t nfree[2] = {0, 0};
  std::set<int32_t> dram_free;             // host-managed pinned DRAM allocator
  std::map<int32_t, int32_t> orphan_ref[2];
  std::vector<int32_t> pending_free;       // HBM ids to clear in the device bitmap
  mpi::Index* index = nullptr;
  uint64_t epoch = 0;
  std::map<int32_t, mp_pool*> peers;
  std::map<int32_t, char**> peer_tables;   // peer's slab table, on this device
  std::deque<Msg> inbox;
};

namespace {

// ------------------------------------------------------------------ helpers
int* arena_take(mp_pool* p, int64_t n, int** host) {
  if (p->ar.used + n > p->ar.cap) return nullptr;
  int* d = p->ar.d + p->ar.used;
  *host = p->ar.h + p->ar.used;
  p->ar.used += std::max<int64_t>(n, 1);
  return d;
}

mp_status upload_ids(mp_pool* p, const std::vector<int32_t>& ids, int** d_out) {
  int* h = nullptr;
  int* d = arena_take(p, (int64_t)ids.size(), &h);
  if (!d) {
    set_err("id arena exhausted");
    return MP_ERR_INTERNAL;
  }
  if (!ids.empty()) {
    std::memcpy(h, ids.data(), ids.size() * sizeof(int32_t));
    CK(cudaMemcpyAsync(d, h, ids.size() * sizeof(int32_t), cudaMemcpyHostToDevice, p->stream));
  }
  *d_out = d;
  return MP_OK;
}

void begin_call(mp_pool* p) { p->ar.used = 0; }

mp_status flush_frees(mp_pool* p) {
  if (p->pending_free.empty()) return MP_OK;
  int* d = nullptr;
  TRY(upload_ids(p, p->pending_free, &d));
  CK(mpk::launch_free(p->d_bitmap, d, (int)p->pending_free.size(), p->stream));
  p->pending_free.clear();
  p->stats.aux_launches += 1;
  return MP_OK;
}

mp_status sync(mp_pool* p) {
  TRY(flush_frees(p));
  CK(cudaStreamSynchronize(p->stream));
  return MP_OK;
}

bool decode(const mp_pool* p, mp_addr a, int* med, int32_t* idx) {
  if (MP_ADDR_INST(a) != p->inst) return false;
  const int m = MP_ADDR_MEDIUM(a);
  if (m != MP_HBM && m != MP_DRAM) return false;
  const int64_t i = (int64_t)(a & 0xFFFFFFFFu);
  if (i >= (m == MP_HBM ? p->n_hbm : p->n_dram)) return false;
  *med = m;
  *idx = (int32_t)i;
  return true;
}

mp_addr enc(const mp_pool* p, int med, int32_t idx) { return MP_ADDR(p->inst, med, idx); }

// Free one block in the host shadow (HBM: also queued for the device bitmap).
void free_block(mp_pool* p, int med, int32_t idx) {
  p->st[med][(size_t)idx] = ST_FREE;
  p->alloc_by[med][(size_t)idx] = -1;
  ++p->nfree[med];
  if (med == MP_HBM)
    p->pending_free.push_back(idx);
  else
    p->dram_free.insert(idx);
}

// R8: evict up to n LRU leaves of `med`; appends freed ids.
void evict_internal(mp_pool* p, int64_t n, int med, std::vector<int32_t>* freed) {
  for (int64_t k = 0; k < n; ++k) {
    mpi::Node* v = p->index->lru_leaf(med);
    if (!v) break;
    const int32_t idx = v->idx;
    p->index->unlink(v);
    free_block(p, med, idx);
    if (freed) freed->push_back(idx);
  }
}

// R2 feasibility: free + eventually-evictable (excluding the pinned path) >= n.
bool can_make_room(mp_pool* p, int64_t n, int med, const std::vector<mpi::Node*>& pinned) {
  if (p->nfree[med] >= n) return true;
  return p->nfree[med] + p->index->evictable(med, pinned) >= n;
}

// Device bitmap allocation of n HBM blocks (lowest-first).  Ids land in the
// arena (device + mapped host mirror; the host copy is valid after sync).
mp_status alloc_hbm_launch(mp_pool* p, int64_t n, int** d_ids, int** h_ids,
                           std::vector<int32_t>* expect) {
  if (n > p->nfree[MP_HBM]) {
    set_err("alloc_hbm: host shadow short");
    return MP_ERR_INTERNAL;
  }
  int* h = nullptr;
  int* d = arena_take(p, n, &h);
  if (!d) {
    set_err("id arena exhausted");
    return MP_ERR_INTERNAL;
  }
  if (expect) {
    expect->clear();
    for (int64_t i = 0; i < p->n_hbm && (int64_t)expect->size() < n; ++i)
      if (p->st[MP_HBM][(size_t)i] == ST_FREE) expect->push_back((int32_t)i);
  }
  TRY(flush_frees(p));
  CK(mpk::launch_alloc(p->d_bitmap, p->nwords, (int)n, d, h, p->d_err, p->stream));
  p->stats.aux_launches += 1;
  p->nfree[MP_HBM] -= n;
  *d_ids = d;
  *h_ids = h;
  return MP_OK;
}

// After sync: mark the allocated HBM ids ACTIVE (and verify them).
mp_status alloc_hbm_finish(mp_pool* p, const int* h_ids, int64_t n, int32_t requester,
                           const std::vector<int32_t>* expect) {
  if (p->verify) {
    int err = 0;
    CK(cudaMemcpy(&err, p->d_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (err) {
      set_err("device allocator ran short");
      return MP_ERR_INTERNAL;
    }
  }
  for (int64_t i = 0; i < n; ++i) {
    const int32_t id = h_ids[i];
    if (id < 0 || id >= p->n_hbm || p->st[MP_HBM][(size_t)id] != ST_FREE) {
      set_err("device allocator returned a non-free block");
      return MP_ERR_INTERNAL;
    }
    if (expect && (*expect)[(size_t)i] != id) {
      set_err("device allocator disagrees with host shadow (lowest-first)");
      return MP_ERR_INTERNAL;
    }
    p->st[MP_HBM][(size_t)id] = ST_ACTIVE;
    p->alloc_by[MP_HBM][(size_t)id] = requester;
  }
  return MP_OK;
}

std::vector<int32_t> alloc_dram(mp_pool* p, int64_t n, int32_t requester) {
  std::vector<int32_t> out;
  for (int64_t i = 0; i < n; ++i) {
    const int32_t id = *p->dram_free.begin();
    p->dram_free.erase(p->dram_free.begin());
    p->st[MP_DRAM][(size_t)id] = ST_ACTIVE;
    p->alloc_by[MP_DRAM][(size_t)id] = requester;
    out.push_back(id);
  }
  p->nfree[MP_DRAM] -= n;
  return out;
}

mp_status launch_migrate_timed(mp_pool* p, cudaStream_t s, const mpk::Endpoint& a,
                               const mpk::Endpoint& b, int64_t n, int j0, int nj) {
  if (n <= 0) return MP_OK;
  if (p->profiling) CK(cudaEventRecord(p->ev0, s));
  CK(mpk::launch_migrate(a, b, (int)n, j0, nj, p->chunk, p->max_ctas, s));
  if (p->profiling) CK(cudaEventRecord(p->ev1, s));
  p->stats.kernel_launches += 1;
  p->stats.bytes_moved += (uint64_t)n * (uint64_t)nj * (uint64_t)p->chunk;
  return MP_OK;
}

// Called after the stream sync that follows launch_migrate_timed.
mp_status collect_timing(mp_pool* p, int64_t bytes) {
  if (!p->profiling || bytes <= 0) return MP_OK;
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
  p->stats.kernel_ms += ms;
  p->stats.timed_launches += 1;
  p->stats.timed_bytes += (uint64_t)bytes;
  return MP_OK;
}

mpk::Endpoint pool_ep(char** slabs, const int* ids) { return {slabs, nullptr, 0, ids}; }
mpk::Endpoint agg_ep(char* base, long long stride, const int* ids) {
  return {nullptr, base, stride, ids};
}

// ---- insert (R4) ----------------------------------------------------------
mp_status insert_internal(mp_pool* p, const mp_token* toks, int64_t n_tok, const mp_addr* addrs,
                          int64_t n_addr, uint32_t flags, int64_t* n_dup) {
  const int64_t k = n_tok / p->B, c = (n_tok + p->B - 1) / p->B;
  if (n_tok < 0 || (n_addr != k && n_addr != c)) return MP_ERR_ADDR_COUNT;
  std::vector<mpi::Node*> path = p->index->path(toks, k);
  std::vector<int> med((size_t)k);
  std::vector<int32_t> idx((size_t)k);
  std::set<std::pair<int, int32_t>> seen;
  for (int64_t i = 0; i < k; ++i) {
    if (!decode(p, addrs[i], &med[(size_t)i], &idx[(size_t)i])) return MP_ERR_INVALID_ADDR;
    auto key = std::make_pair(med[(size_t)i], idx[(size_t)i]);
    if (!seen.insert(key).second) return MP_ERR_PRECONDITION;
    mpi::Node* ex = i < (int64_t)path.size() ? path[(size_t)i] : nullptr;
    const uint8_t s = p->st[med[(size_t)i]][(size_t)idx[(size_t)i]];
    const bool same = ex && ex->medium == med[(size_t)i] && ex->idx == idx[(size_t)i];
    if (!(s == ST_ACTIVE || (s == ST_INDEXED && same))) return MP_ERR_PRECONDITION;
    if ((flags & MP_INS_ERR_ON_CONFLICT) && ex && !same) return MP_ERR_CONFLICT;
  }
  const uint64_t t = p->index->tick();
  int64_t dup = 0;
  mpi::Node* parent = nullptr;
  mpi::Node* last = nullptr;
  for (int64_t i = 0; i < k; ++i) {
    mpi::Node* ex = i < (int64_t)path.size() ? path[(size_t)i] : nullptr;
    if (ex) {
      p->index->touch(ex, t);
      if (!(ex->medium == med[(size_t)i] && ex->idx == idx[(size_t)i])) {
        free_block(p, med[(size_t)i], idx[(size_t)i]);
        ++dup;
      }
      last = ex;
    } else {
      last = p->index->add(parent, toks + i * p->B, med[(size_t)i], idx[(size_t)i], t);
      p->st[med[(size_t)i]][(size_t)idx[(size_t)i]] = ST_INDEXED;
    }
    parent = last;
  }
  if (last) last->terminal = true;
  if (n_dup) *n_dup = dup;
  return MP_OK;
}

void unpin_nodes(mp_pool* p, const std::vector<mpi::Node*>& nodes) {
  for (mpi::Node* n : nodes) p->index->set_ref(n, n->ref - 1);
}

// ---- source / destination validation for transfers ------------------------
mp_status validate_src(mp_pool* src, const mp_addr* a, int64_t n, std::vector<int32_t>* ids) {
  ids->resize((size_t)n);
  std::vector<uint8_t> mark((size_t)src->n_hbm, 0);
  for (int64_t i = 0; i < n; ++i) {
    int m = 0;
    int32_t idx = 0;
    if (!decode(src, a[i], &m, &idx)) return MP_ERR_INVALID_ADDR;
    if (m != MP_HBM) return MP_ERR_PRECONDITION;  // R13
    const uint8_t s = src->st[MP_HBM][(size_t)idx];
    if (!(s == ST_ACTIVE || s == ST_INDEXED) || mark[(size_t)idx]) return MP_ERR_PRECONDITION;
    mark[(size_t)idx] = 1;
    (*ids)[(size_t)i] = idx;
  }
  return MP_OK;
}

mp_status validate_dst_given(mp_pool* dst, const mp_addr* a, int64_t n,
                             std::vector<int32_t>* ids) {
  if (!a) return MP_ERR_ADDR_COUNT;
  ids->resize((size_t)n);
  std::vector<uint8_t> mark((size_t)dst->n_hbm, 0);
  for (int64_t i = 0; i < n; ++i) {
    int m = 0;
    int32_t idx = 0;
    if (!decode(dst, a[i], &m, &idx)) return MP_ERR_INVALID_ADDR;
    if (m != MP_HBM || dst->st[MP_HBM][(size_t)idx] != ST_ACTIVE || mark[(size_t)idx])
      return MP_ERR_PRECONDITION;
    mark[(size_t)idx] = 1;
    (*ids)[(size_t)i] = idx;
  }
  return MP_OK;
}

mp_status check_compatible(mp_pool* src, mp_pool* dst) {
  if (dst == src || src->L != dst->L || src->chunk != dst->chunk || src->B != dst->B)
    return MP_ERR_CONFIG;
  return MP_OK;
}

// ---- the transmission step (A4-A6 / A6f) -----------------------------------
// Copies chunks [j0, j0+nj) of src blocks s_ids into dst blocks.  Destination
// ids are either on the dst device (d_dst, produced by the dst allocator; host
// mirror h_dst valid after a dst sync) or given on the host (given_dst).
// Returns after all copies completed.
mp_status transmit(mp_pool* src, mp_pool* dst, const std::vector<int32_t>& s_ids,
                   const int* d_dst, const int* h_dst, const std::vector<int32_t>* given_dst,
                   int j0, int nj, uint32_t path) {
  const int64_t n = (int64_t)s_ids.size();
  const int64_t bytes = n * nj * src->chunk;
  if (path == MP_XFER_PATH_AUTO) path = MP_XFER_PATH_FUSED;
  const bool same_dev = src->dev == dst->dev;
  if (path == MP_XFER_PATH_FUSED && same_dev) {
    DevGuard g(dst->dev);
    int* ds = nullptr;
    TRY(upload_ids(dst, s_ids, &ds));
    const int* dd = d_dst;
    if (given_dst) {
      int* t = nullptr;
      TRY(upload_ids(dst, *given_dst, &t));
      dd = t;
    }
    TRY(launch_migrate_timed(dst, dst->stream, pool_ep(src->d_slabs, ds), pool_ep(dst->d_slabs, dd),
                             n, j0, nj));
    TRY(sync(dst));
    TRY(collect_timing(dst, bytes));
    dst->stats.blocks_moved += (uint64_t)n;
    return MP_OK;
  }
  // Destination ids on the host for the cross-device / CE / staged paths.
  std::vector<int32_t> dids;
  if (given_dst) {
    dids = *given_dst;
  } else {
    {
      DevGuard g(dst->dev);
      TRY(sync(dst));
    }
    dids.assign(h_dst, h_dst + n);
  }
  if (path == MP_XFER_PATH_FUSED) {
    // Push over NVLink: the source GPU gathers its chunks and stores them
    // straight into the peer pool's blocks (A6f, no staging).
    DevGuard g(src->dev);
    auto it = src->peer_tables.find(dst->inst);
    if (it == src->peer_tables.end()) return MP_ERR_DST_UNREACHABLE;
    int *ds = nullptr, *dd = nullptr;
    TRY(upload_ids(src, s_ids, &ds));
    TRY(upload_ids(src, dids, &dd));
    TRY(launch_migrate_timed(src, src->stream, pool_ep(src->d_slabs, ds), pool_ep(it->second, dd),
                             n, j0, nj));
    TRY(sync(src));
    TRY(collect_timing(src, bytes));
    src->stats.blocks_moved += (uint64_t)n;
    return MP_OK;
  }
  if (path == MP_XFER_PATH_CE) {
    // Library baseline: one copy-engine memcpy per (block, layer, K/V) chunk --
    // the "discrete" transfer the paper starts from.
    DevGuard g(src->dev);
    for (int64_t i = 0; i < n; ++i)
      for (int j = j0; j < j0 + nj; ++j)
        CK(cudaMemcpyAsync(dst->slabs[(size_t)j] + (int64_t)dids[(size_t)i] * dst->chunk,
                           src->slabs[(size_t)j] + (int64_t)s_ids[(size_t)i] * src->chunk,
                           (size_t)src->chunk, cudaMemcpyDefault, src->stream));
    TRY(sync(src));
    src->stats.bytes_moved += (uint64_t)bytes;
    src->stats.blocks_moved += (uint64_t)n;
    return MP_OK;
  }
  if (path == MP_XFER_PATH_STAGED) {
    // Aggregated staging: pack k blocks into a source slot, one
    // contiguous copy to the destination slot, unpack; slots form a ring so
    // pack / wire / unpack of consecutive slots overlap.
    const int64_t per_block = (int64_t)nj * src->chunk;
    const int S = std::max(1, std::min(src->staging_slots, dst->staging_slots));
    const int64_t slot_bytes = std::min(src->staging_bytes, dst->staging_bytes) / S;
    const int64_t k = slot_bytes / per_block;
    if (k <= 0) {
      set_err("staging slot smaller than one block");
      return MP_ERR_CONFIG;
    }
    int *ds = nullptr, *dd = nullptr;
    {
      DevGuard g(src->dev);
      TRY(upload_ids(src, s_ids, &ds));
    }
    {
      DevGuard g(dst->dev);
      TRY(upload_ids(dst, dids, &dd));
    }
    const int64_t nslots = (n + k - 1) / k;
    for (int64_t s = 0; s < nslots; ++s) {
      const int r = (int)(s % S);
      const int64_t b0 = s * k, nb = std::min(k, n - b0);
      char* sslot = src->staging + r * slot_bytes;
      char* dslot = dst->staging + r * slot_bytes;
      {
        DevGuard g(src->dev);
        if (s >= S) CK(cudaStreamWaitEvent(src->stream, dst->slot_ev[(size_t)r], 0));
        TRY(launch_migrate_timed(src, src->stream, pool_ep(src->d_slabs, ds + b0),
                                 agg_ep(sslot, per_block, nullptr), nb, j0, nj));
        CK(cudaEventRecord(src->slot_ev[(size_t)r], src->stream));
        CK(cudaStreamWaitEvent(src->copy_stream, src->slot_ev[(size_t)r], 0));
        CK(cudaMemcpyAsync(dslot, sslot, (size_t)(nb * per_block), cudaMemcpyDefault,
                           src->copy_stream));
        CK(cudaEventRecord(src->slot_ev[(size_t)r], src->copy_stream));
      }
      {
        DevGuard g(dst->dev);
        CK(cudaStreamWaitEvent(dst->stream, src->slot_ev[(size_t)r], 0));
        TRY(launch_migrate_timed(dst, dst->stream, agg_ep(dslot, per_block, nullptr),
                                 pool_ep(dst->d_slabs, dd + b0), nb, j0, nj));
        CK(cudaEventRecord(dst->slot_ev[(size_t)r], dst->stream));
      }
    }
    {
      DevGuard g(dst->dev);
      TRY(sync(dst));
    }
    {
      DevGuard g(src->dev);
      TRY(sync(src));
    }
    src->stats.blocks_moved += (uint64_t)n;
    return MP_OK;
  }
  set_err("unknown transfer path");
  return MP_ERR_CONFIG;
}

mp_pool* peer_of(mp_pool* src, int32_t inst) {
  auto it = src->peers.find(inst);
  return it == src->peers.end() ? nullptr : it->second;
}

}  // namespace

// =========================================================================
//                                 C-ABI
// =========================================================================
extern "C" {

const char* mp_status_str(mp_status s) {
  switch (s) {
    case MP_OK: return "MP_OK";
    case MP_ERR_OOM: return "MP_ERR_OOM";
    case MP_ERR_DOUBLE_FREE: return "MP_ERR_DOUBLE_FREE";
    case MP_ERR_INVALID_ADDR: return "MP_ERR_INVALID_ADDR";
    case MP_ERR_ADDR_COUNT: return "MP_ERR_ADDR_COUNT";
    case MP_ERR_CONFLICT: return "MP_ERR_CONFLICT";
    case MP_ERR_NO_DRAM: return "MP_ERR_NO_DRAM";
    case MP_ERR_DST_OOM: return "MP_ERR_DST_OOM";
    case MP_ERR_DST_UNREACHABLE: return "MP_ERR_DST_UNREACHABLE";
    case MP_ERR_PRECONDITION: return "MP_ERR_PRECONDITION";
    case MP_ERR_PREFIX_MISSING: return "MP_ERR_PREFIX_MISSING";
    case MP_ERR_CONFIG: return "MP_ERR_CONFIG";
    case MP_ERR_BUFFER_TOO_SMALL: return "MP_ERR_BUFFER_TOO_SMALL";
    case MP_ERR_CUDA: return "MP_ERR_CUDA";
    case MP_ERR_NCCL: return "MP_ERR_NCCL";
    case MP_ERR_INTERNAL: return "MP_ERR_INTERNAL";
  }
  return "MP_ERR_UNKNOWN";
}

const char* mp_last_error(void) { return g_err.c_str(); }

void mp_pool_destroy(mp_pool* p) {
  if (!p) return;
  {
    DevGuard g(p->dev);
    if (p->stream) cudaStreamSynchronize(p->stream);
    for (auto& kv : p->peers) {
      mp_pool* q = kv.second;
      q->peers.erase(p->inst);
      auto it = q->peer_tables.find(p->inst);
      if (it != q->peer_tables.end()) {
        DevGuard g2(q->dev);
        cudaFree(it->second);
        q->peer_tables.erase(it);
      }
    }
    for (auto& kv : p->peer_tables) cudaFree(kv.second);
    if (p->own_slab_region) cudaFree(p->own_slab_region);
    if (p->d_slabs) cudaFree(p->d_slabs);
    if (p->d_bitmap) cudaFree(p->d_bitmap);
    if (p->d_err) cudaFree(p->d_err);
    if (p->ar.d) cudaFree(p->ar.d);
    if (p->ar.h) cudaFreeHost(p->ar.h);
    if (p->own_dram && p->dram) cudaFreeHost(p->dram);
    if (p->staging) cudaFree(p->staging);
    if (p->ev0) cudaEventDestroy(p->ev0);
    if (p->ev1) cudaEventDestroy(p->ev1);
    for (auto e : p->slot_ev) cudaEventDestroy(e);
    if (p->stream) cudaStreamDestroy(p->stream);
    if (p->copy_stream) cudaStreamDestroy(p->copy_stream);
  }
  delete p->index;
  delete p;
}

mp_status mp_pool_create(const mp_pool_config* cfg, mp_pool** out) {
  if (!cfg || !out) return MP_ERR_CONFIG;
  if (cfg->layers < 1 || cfg->layers > 256 || cfg->kv_heads < 1 || cfg->head_dim < 1 ||
      cfg->elem_bytes < 1 || cfg->block_tokens < 1 || cfg->hbm_blocks < 1 ||
      cfg->hbm_blocks >= (1ll << 31) || cfg->dram_blocks < 0 || cfg->dram_blocks >= (1ll << 31) ||
      cfg->instance_id < 0 || cfg->instance_id >= (1 << 24)) {
    set_err("invalid pool config");
    return MP_ERR_CONFIG;
  }
  const int64_t chunk =
      (int64_t)cfg->block_tokens * cfg->kv_heads * cfg->head_dim * cfg->elem_bytes;
  if (chunk % 16 != 0) {
    set_err("chunk bytes must be a multiple of 16");
    return MP_ERR_CONFIG;
  }
  mp_pool* p = new mp_pool();
  p->inst = cfg->instance_id;
  p->dev = cfg->device;
  p->L = cfg->layers;
  p->H = cfg->kv_heads;
  p->D = cfg->head_dim;
  p->elem = cfg->elem_bytes;
  p->B = cfg->block_tokens;
  p->verify = cfg->verify != 0;
  p->chunk = chunk;
  p->nch = 2 * cfg->layers;
  p->Pb = chunk * p->nch;
  p->n_hbm = cfg->hbm_blocks;
  p->n_dram = cfg->dram_blocks;
  p->max_ctas = cfg->max_ctas;
  p->staging_slots = cfg->staging_slots > 0 ? cfg->staging_slots : 4;
  p->staging_bytes = cfg->staging_bytes > 0 ? cfg->staging_bytes : (256ll << 20);
  p->index = new mpi::Index(p->B, p->n_hbm, p->n_dram);
  for (int m = 0; m < 2; ++m) {
    const int64_t n = m == 0 ? p->n_hbm : p->n_dram;
    p->st[m].assign((size_t)n, ST_FREE);
    p->alloc_by[m].assign((size_t)n, -1);
    p->nfree[m] = n;
  }
  for (int32_t i = 0; i < (int32_t)p->n_dram; ++i) p->dram_free.insert(p->dram_free.end(), i);
  auto fail = [&](mp_status s) {
    mp_pool_destroy(p);
    return s;
  };
#define CKC(x)                                                            \
  do {                                                                    \
    cudaError_t e_ = (x);                                                 \
    if (e_ != cudaSuccess) {                                              \
      set_err(std::string(#x) + ": " + cudaGetErrorString(e_));           \
      return fail(MP_ERR_CUDA);                                           \
    }                                                                     \
  } while (0)
  int ndev = 0;
  CKC(cudaGetDeviceCount(&ndev));
  if (cfg->device < 0 || cfg->device >= ndev) {
    set_err("device ordinal out of range");
    return fail(MP_ERR_CONFIG);
  }
  DevGuard g(p->dev);
  CKC(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
  CKC(cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking));
  CKC(cudaEventCreate(&p->ev0));
  CKC(cudaEventCreate(&p->ev1));
  p->slot_ev.resize((size_t)p->staging_slots);
  for (auto& e : p->slot_ev) CKC(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  p->slabs.resize((size_t)p->nch);
  if (cfg->slabs) {
    for (int j = 0; j < p->nch; ++j) {
      p->slabs[(size_t)j] = (char*)cfg->slabs[j];
      if (!p->slabs[(size_t)j] || ((uintptr_t)p->slabs[(size_t)j] & 15)) {
        set_err("slab pointers must be non-null and 16-byte aligned");
        return fail(MP_ERR_CONFIG);
      }
    }
  } else {
    const size_t bytes = (size_t)p->nch * (size_t)p->n_hbm * (size_t)chunk;
    CKC(cudaMalloc(&p->own_slab_region, bytes));
    for (int j = 0; j < p->nch; ++j)
      p->slabs[(size_t)j] = (char*)p->own_slab_region + (size_t)j * p->n_hbm * chunk;
  }
  CKC(cudaMalloc(&p->d_slabs, sizeof(char*) * p->nch));
  CKC(cudaMemcpy(p->d_slabs, p->slabs.data(), sizeof(char*) * p->nch, cudaMemcpyHostToDevice));
  p->nwords = (int)((p->n_hbm + 31) / 32);
  std::vector<uint32_t> bm((size_t)p->nwords, 0xFFFFFFFFu);
  if (p->n_hbm % 32) bm.back() = (1u << (p->n_hbm % 32)) - 1u;
  CKC(cudaMalloc(&p->d_bitmap, sizeof(uint32_t) * p->nwords));
  CKC(cudaMemcpy(p->d_bitmap, bm.data(), sizeof(uint32_t) * p->nwords, cudaMemcpyHostToDevice));
  CKC(cudaMalloc(&p->d_err, sizeof(int)));
  CKC(cudaMemset(p->d_err, 0, sizeof(int)));
  p->ar.cap = 8 * std::max<int64_t>(std::max(p->n_hbm, p->n_dram), 4096);
  CKC(cudaMalloc(&p->ar.d, sizeof(int) * p->ar.cap));
  CKC(cudaHostAlloc(&p->ar.h, sizeof(int) * p->ar.cap, cudaHostAllocMapped | cudaHostAllocPortable));
  if (p->n_dram > 0) {
    if (cfg->dram_base) {
      p->dram = (char*)cfg->dram_base;
    } else {
      CKC(cudaHostAlloc(&p->dram, (size_t)p->n_dram * (size_t)p->Pb,
                        cudaHostAllocMapped | cudaHostAllocPortable));
      p->own_dram = true;
    }
    void* dp = nullptr;
    if (cudaHostGetDevicePointer(&dp, p->dram, 0) != cudaSuccess) {
      cudaGetLastError();
      set_err("dram_base is not pinned (cudaHostAlloc / cudaHostRegister required)");
      return fail(MP_ERR_CONFIG);
    }
    p->dram_dev = (char*)dp;
  }
  CKC(cudaMalloc(&p->staging, (size_t)p->staging_bytes));
#undef CKC
  *out = p;
  return MP_OK;
}

mp_status mp_connect(mp_pool* a, mp_pool* b) {
  if (!a || !b || a == b || a->inst == b->inst) return MP_ERR_CONFIG;
  if (a->L != b->L || a->chunk != b->chunk || a->B != b->B) {
    set_err("pools have different KV shapes");
    return MP_ERR_CONFIG;
  }
  if (a->dev != b->dev) {
    int ab = 0, ba = 0;
    CK(cudaDeviceCanAccessPeer(&ab, a->dev, b->dev));
    CK(cudaDeviceCanAccessPeer(&ba, b->dev, a->dev));
    if (!ab || !ba) {
      set_err("no CUDA peer access between the two devices");
      return MP_ERR_DST_UNREACHABLE;
    }
    for (int dir = 0; dir < 2; ++dir) {
      mp_pool* x = dir ? b : a;
      mp_pool* y = dir ? a : b;
      DevGuard g(x->dev);
      cudaError_t e = cudaDeviceEnablePeerAccess(y->dev, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else CK(e);
    }
  }
  for (int dir = 0; dir < 2; ++dir) {
    mp_pool* x = dir ? b : a;
    mp_pool* y = dir ? a : b;
    DevGuard g(x->dev);
    char** t = nullptr;
    CK(cudaMalloc(&t, sizeof(char*) * y->nch));
    CK(cudaMemcpy(t, y->slabs.data(), sizeof(char*) * y->nch, cudaMemcpyHostToDevice));
    auto it = x->peer_tables.find(y->inst);
    if (it != x->peer_tables.end()) cudaFree(it->second);
    x->peer_tables[y->inst] = t;
    x->peers[y->inst] = y;
  }
  return MP_OK;
}

mp_status mp_pool_info_get(const mp_pool* p, mp_pool_info* o) {
  if (!p || !o) return MP_ERR_CONFIG;
  o->chunk_bytes = p->chunk;
  o->block_bytes = p->Pb;
  o->hbm_blocks = p->n_hbm;
  o->dram_blocks = p->n_dram;
  o->hbm_free = p->nfree[0];
  o->dram_free = p->nfree[1];
  o->index_blocks = (int64_t)p->index->size();
  o->clock = p->index->clock();
  o->epoch = p->epoch;
  o->instance_id = p->inst;
  o->device = p->dev;
  o->layers = p->L;
  o->block_tokens = p->B;
  return MP_OK;
}

// ------------------------------ memory API --------------------------------
mp_status mp_alloc_mem(mp_pool* p, int64_t n, int32_t type, int32_t requester, mp_addr* out) {
  if (!p || n < 0 || (n > 0 && !out) || type < MP_HBM || type > MP_MIXED) return MP_ERR_CONFIG;
  DevGuard g(p->dev);
  begin_call(p);
  const std::vector<mpi::Node*> none;
  int64_t nh = 0, nd = 0;
  if (type == MP_HBM) nh = n;
  else if (type == MP_DRAM) nd = n;
  else {
    nh = std::min(n, p->nfree[MP_HBM]);
    nd = n - nh;
  }
  if (!can_make_room(p, nh, MP_HBM, none) || !can_make_room(p, nd, MP_DRAM, none))
    return MP_ERR_OOM;
  if (p->nfree[MP_HBM] < nh) evict_internal(p, nh - p->nfree[MP_HBM], MP_HBM, nullptr);
  if (p->nfree[MP_DRAM] < nd) evict_internal(p, nd - p->nfree[MP_DRAM], MP_DRAM, nullptr);
  int *d = nullptr, *h = nullptr;
  std::vector<int32_t> expect;
  if (nh > 0) TRY(alloc_hbm_launch(p, nh, &d, &h, p->verify ? &expect : nullptr));
  TRY(sync(p));
  if (nh > 0) TRY(alloc_hbm_finish(p, h, nh, requester, p->verify ? &expect : nullptr));
  for (int64_t i = 0; i < nh; ++i) out[i] = enc(p, MP_HBM, h[i]);
  std::vector<int32_t> dd = alloc_dram(p, nd, requester);
  for (int64_t i = 0; i < nd; ++i) out[nh + i] = enc(p, MP_DRAM, dd[(size_t)i]);
  return MP_OK;
}

mp_status mp_free_mem(mp_pool* p, const mp_addr* a, int64_t n) {
  if (!p || n < 0 || (n > 0 && !a)) return MP_ERR_CONFIG;
  DevGuard g(p->dev);
  begin_call(p);
  std::set<std::pair<int, int32_t>> seen;
  for (int64_t i = 0; i < n; ++i) {
    int m = 0;
    int32_t idx = 0;
    if (!decode(p, a[i], &m, &idx)) return MP_ERR_INVALID_ADDR;
    const uint8_t s = p->st[m][(size_t)idx];
    if (s == ST_FREE || !seen.insert({m, idx}).second) return MP_ERR_DOUBLE_FREE;
    if (s != ST_ACTIVE) return MP_ERR_PRECONDITION;
  }
  for (int64_t i = 0; i < n; ++i) {
    int m = 0;
    int32_t idx = 0;
    decode(p, a[i], &m, &idx);
    free_block(p, m, idx);
  }
  return sync(p);
}

// ------------------------------- index API --------------------------------
mp_status mp_insert(mp_pool* p, const mp_token* toks, int64_t n_tok, const mp_addr* a,
                    int64_t n_addr, uint32_t flags, int64_t* n_dup) {
  if (!p || n_tok < 0 || (n_tok > 0 && !toks) || n_addr < 0 || (n_addr > 0 && !a))
    return MP_ERR_CONFIG;
  DevGuard g(p->dev);
  begin_call(p);
  TRY(insert_internal(p, toks, n_tok, a, n_addr, flags, n_dup));
  return sync(p);
}

mp_status mp_match(mp_pool* p, const mp_token* toks, int64_t n_tok, uint32_t flags, mp_addr* out,
                   int64_t cap, int64_t* matched) {
  if (!p || n_tok < 0 || (n_tok > 0 && !toks)) return MP_ERR_CONFIG;
  if (cap < n_tok / p->B) return MP_ERR_BUFFER_TOO_SMALL;
  std::vector<mpi::Node*> m = p->index->match(toks, n_tok, (flags & MP_MATCH_PIN) != 0);
  for (size_t i = 0; i < m.size(); ++i) out[i] = enc(p, m[i]->medium, m[i]->idx);
  if (matched) *matched = (int64_t)m.size() * p->B;
  return MP_OK;
}

mp_status mp_unpin(mp_pool* p, const mp_addr* a, int64_t n) {
  if (!p || n < 0 || (n > 0 && !a)) return MP_ERR_CONFIG;
  std::map<std::pair<int, int32_t>, int64_t> need;
  for (int64_t i = 0; i < n; ++i) {
    int m = 0;
    int32_t idx = 0;
    if (!decode(p, a[i], &m, &idx)) return MP_ERR_INVALID_ADDR;
    ++need[{m, idx}];
  }
  for (auto& kv : need) {
    const int m = kv.first.first;
    const int32_t idx = kv.first.second;
    mpi::Node* nd = p->index->owner(m, idx);
    int64_t have = 0;
    if (nd) have = nd->ref;
    else {
      auto it = p->orphan_ref[m].find(idx);
      if (it != p->orphan_ref[m].end()) have = it->second;
    }
    if (have < kv.second) return MP_ERR_PRECONDITION;
  }
  DevGuard g(p->dev);
  begin_call(p);
  for (auto& kv : need) {
    const int m = kv.first.first;
    const int32_t idx = kv.first.second;
    mpi::Node* nd = p->index->owner(m, idx);
    if (nd) {
      p->index->set_ref(nd, nd->ref - (int32_t)kv.second);
    } else {
      auto it = p->orphan_ref[m].find(idx);
      it->second -= (int32_t)kv.second;
      if (it->second == 0) {
        p->orphan_ref[m].erase(it);
        free_block(p, m, idx);
      }
    }
  }
  return sync(p);
}

mp_status mp_delete(mp_pool* p, const mp_token* toks, int64_t n_tok) {
  if (!p || n_tok < 0 || (n_tok > 0 && !toks)) return MP_ERR_CONFIG;
  const int64_t k = n_tok / p->B;
  if (k == 0) return MP_OK;
  std::vector<mpi::Node*> path = p->index->path(toks, k);
  if ((int64_t)path.size() < k || !path.back()->terminal) return MP_OK;
  DevGuard g(p->dev);
  begin_call(p);
  path.back()->terminal = false;
  for (int64_t i = k - 1; i >= 0; --i) {
    mpi::Node* nd = path[(size_t)i];
    if (!nd->kids.empty() || nd->terminal) break;
    const int m = nd->medium;
    const int32_t idx = nd->idx, ref = nd->ref;
    p->index->unlink(nd);
    if (ref == 0) {
      free_block(p, m, idx);
    } else {
      p->st[m][(size_t)idx] = ST_ORPHAN;
      p->orphan_ref[m][idx] = ref;
    }
  }
  return sync(p);
}

mp_status mp_evict(mp_pool* p, int64_t n, int32_t medium, mp_addr* out, int64_t* n_freed) {
  if (!p || n < 0 || (medium != MP_HBM && medium != MP_DRAM) || (n > 0 && !out))
    return MP_ERR_CONFIG;
  DevGuard g(p->dev);
  begin_call(p);
  std::vector<int32_t> freed;
  evict_internal(p, n, medium, &freed);
  for (size_t i = 0; i < freed.size(); ++i) out[i] = enc(p, medium, freed[i]);
  if (n_freed) *n_freed = (int64_t)freed.size();
  return sync(p);
}

// ------------------------------- swap API ---------------------------------
mp_status mp_swap_out(mp_pool* p, int64_t n, uint32_t flags, mp_addr* out_old, mp_addr* out_new,
                      int64_t* n_moved) {
  (void)flags;
  if (!p || n < 0 || (n > 0 && (!out_old || !out_new))) return MP_ERR_CONFIG;
  DevGuard g(p->dev);
  begin_call(p);
  std::vector<std::pair<int32_t, int32_t>> pairs;
  bool no_dram = false;
  while ((int64_t)pairs.size() < n) {
    mpi::Node* v = p->index->lru_frontier();
    if (!v) break;
    if (p->nfree[MP_DRAM] == 0) {
      std::vector<int32_t> ev;
      evict_internal(p, 1, MP_DRAM, &ev);
      if (ev.empty()) {
        no_dram = true;
        break;
      }
    }
    const int32_t h = v->idx;
    const int32_t d = alloc_dram(p, 1, p->alloc_by[MP_HBM][(size_t)h])[0];
    p->st[MP_DRAM][(size_t)d] = ST_INDEXED;
    p->index->rebind(v, MP_DRAM, d);
    free_block(p, MP_HBM, h);  // bitmap update is queued behind the copy kernel
    pairs.push_back({h, d});
  }
  if (pairs.empty() && no_dram) return MP_ERR_NO_DRAM;
  // Copy list: the last pair that wrote each DRAM block still allocated.
  std::vector<int32_t> hs, ds;
  std::set<int32_t> done;
  for (auto it = pairs.rbegin(); it != pairs.rend(); ++it) {
    if (done.count(it->second) || p->st[MP_DRAM][(size_t)it->second] == ST_FREE) continue;
    done.insert(it->second);
    hs.push_back(it->first);
    ds.push_back(it->second);
  }
  if (!hs.empty()) {
    int *dh = nullptr, *dd = nullptr;
    TRY(upload_ids(p, hs, &dh));
    TRY(upload_ids(p, ds, &dd));
    // The frees queued above must not run before the copy has read the
    // blocks: launch the copy first; flush_frees() happens in sync().
    TRY(launch_migrate_timed(p, p->stream, pool_ep(p->d_slabs, dh), agg_ep(p->dram_dev, p->Pb, dd),
                             (int64_t)hs.size(), 0, p->nch));
  }
  TRY(sync(p));
  TRY(collect_timing(p, (int64_t)hs.size() * p->Pb));
  p->stats.blocks_moved += hs.size();
  for (size_t i = 0; i < pairs.size(); ++i) {
    out_old[i] = enc(p, MP_HBM, pairs[i].first);
    out_new[i] = enc(p, MP_DRAM, pairs[i].second);
  }
  if (n_moved) *n_moved = (int64_t)pairs.size();
  return MP_OK;
}

mp_status mp_swap_in(mp_pool* p, const mp_addr* a, int64_t n, uint32_t flags, mp_addr* out) {
  (void)flags;
  if (!p || n < 0 || (n > 0 && (!a || !out))) return MP_ERR_CONFIG;
  std::vector<int32_t> dids((size_t)n);
  std::set<int32_t> seen;
  for (int64_t i = 0; i < n; ++i) {
    int m = 0;
    int32_t idx = 0;
    if (!decode(p, a[i], &m, &idx)) return MP_ERR_INVALID_ADDR;
    if (m != MP_DRAM || !seen.insert(idx).second) return MP_ERR_PRECONDITION;
    const uint8_t s = p->st[MP_DRAM][(size_t)idx];
    if (s != ST_ACTIVE && s != ST_INDEXED) return MP_ERR_PRECONDITION;
    dids[(size_t)i] = idx;
  }
  const std::vector<mpi::Node*> none;
  if (!can_make_room(p, n, MP_HBM, none)) return MP_ERR_OOM;
  DevGuard g(p->dev);
  begin_call(p);
  if (p->nfree[MP_HBM] < n) evict_internal(p, n - p->nfree[MP_HBM], MP_HBM, nullptr);
  int *dh = nullptr, *hh = nullptr, *dd = nullptr;
  std::vector<int32_t> expect;
  TRY(alloc_hbm_launch(p, n, &dh, &hh, p->verify ? &expect : nullptr));
  TRY(upload_ids(p, dids, &dd));
  TRY(launch_migrate_timed(p, p->stream, agg_ep(p->dram_dev, p->Pb, dd), pool_ep(p->d_slabs, dh),
                           n, 0, p->nch));
  TRY(sync(p));
  TRY(collect_timing(p, n * p->Pb));
  TRY(alloc_hbm_finish(p, hh, n, p->inst, p->verify ? &expect : nullptr));
  p->stats.blocks_moved += (uint64_t)n;
  for (int64_t i = 0; i < n; ++i) {
    const int32_t d = dids[(size_t)i], h = hh[i];
    p->alloc_by[MP_HBM][(size_t)h] = p->alloc_by[MP_DRAM][(size_t)d];
    if (p->st[MP_DRAM][(size_t)d] == ST_INDEXED) {
      p->index->rebind(p->index->owner(MP_DRAM, d), MP_HBM, h);
      p->st[MP_HBM][(size_t)h] = ST_INDEXED;
    }
    free_block(p, MP_DRAM, d);
    out[i] = enc(p, MP_HBM, h);
  }
  return MP_OK;
}

// ---------------------------- distributed API -----------------------------
mp_status mp_transfer(mp_pool* src, int32_t dst_inst, const mp_addr* sa, int64_t n, mp_addr* da,
                      uint32_t flags, int32_t l0, int32_t l1, const void* priv, int64_t priv_len) {
  if (!src || n < 0 || (n > 0 && (!sa || !da)) || priv_len < 0 || (priv_len > 0 && !priv))
    return MP_ERR_CONFIG;
  mp_pool* dst = peer_of(src, dst_inst);
  if (!dst) return MP_ERR_DST_UNREACHABLE;
  TRY(check_compatible(src, dst));
  if (!(0 <= l0 && l0 < l1 && l1 <= src->L) || (flags & MP_XFER_DEDUP)) return MP_ERR_CONFIG;
  std::vector<int32_t> sids, given;
  TRY(validate_src(src, sa, n, &sids));
  const bool dst_given = (flags & MP_XFER_DST_GIVEN) != 0;
  if (dst_given) TRY(validate_dst_given(dst, da, n, &given));
  const std::vector<mpi::Node*> none;
  if (!dst_given && !can_make_room(dst, n, MP_HBM, none)) return MP_ERR_DST_OOM;
  begin_call(src);
  begin_call(dst);
  int *d_dst = nullptr, *h_dst = nullptr;
  std::vector<int32_t> expect;
  if (!dst_given) {
    DevGuard g(dst->dev);
    if (dst->nfree[MP_HBM] < n) evict_internal(dst, n - dst->nfree[MP_HBM], MP_HBM, nullptr);
    TRY(alloc_hbm_launch(dst, n, &d_dst, &h_dst, dst->verify ? &expect : nullptr));
  }
  TRY(transmit(src, dst, sids, d_dst, h_dst, dst_given ? &given : nullptr, 2 * l0, 2 * (l1 - l0),
               flags & MP_XFER_PATH_MASK));
  {
    DevGuard g(dst->dev);
    TRY(sync(dst));
  }
  if (!dst_given) {
    TRY(alloc_hbm_finish(dst, h_dst, n, src->inst, dst->verify ? &expect : nullptr));
    for (int64_t i = 0; i < n; ++i) da[i] = enc(dst, MP_HBM, h_dst[i]);
  }
  Msg msg{0, src->inst, {}, {}};
  if (priv_len) msg.priv.assign((const uint8_t*)priv, (const uint8_t*)priv + priv_len);
  msg.addrs.assign(da, da + n);
  dst->inbox.push_back(std::move(msg));
  return MP_OK;
}

mp_status mp_transfer_with_insert(mp_pool* src, int32_t dst_inst, const mp_token* toks,
                                  int64_t n_tok, const mp_addr* sa, int64_t m, mp_addr* da,
                                  uint32_t flags, const void* priv, int64_t priv_len,
                                  int64_t* n_moved) {
  if (!src || n_tok < 0 || (n_tok > 0 && !toks) || m < 0 || (m > 0 && !sa) || !da ||
      priv_len < 0 || (priv_len > 0 && !priv))
    return MP_ERR_CONFIG;
  mp_pool* dst = peer_of(src, dst_inst);
  if (!dst) return MP_ERR_DST_UNREACHABLE;
  TRY(check_compatible(src, dst));
  const bool dst_given = (flags & MP_XFER_DST_GIVEN) != 0;
  const bool dedup = (flags & MP_XFER_DEDUP) != 0;
  if (dst_given && dedup) return MP_ERR_CONFIG;
  const int64_t B = dst->B, ceil_b = (n_tok + B - 1) / B, floor_b = n_tok / B;
  if (m > ceil_b) return MP_ERR_ADDR_COUNT;
  std::vector<int32_t> sids, given;
  TRY(validate_src(src, sa, m, &sids));
  if (dst_given) TRY(validate_dst_given(dst, da, m, &given));
  const int64_t q = ceil_b - m;
  const bool need_match = dedup || q > 0;
  std::vector<mpi::Node*> peek;
  if (need_match) peek = dst->index->path(toks, floor_b);
  const int64_t k_match = (int64_t)peek.size();
  if (k_match < q) return MP_ERR_PREFIX_MISSING;
  const int64_t skip = dedup ? k_match - q : 0;
  const int64_t nm = m - skip;
  if (flags & MP_INS_ERR_ON_CONFLICT) {
    const int64_t k_exist = need_match ? k_match : dst->index->peek(toks, n_tok);
    if (k_exist > q + skip) return MP_ERR_CONFLICT;
  }
  if (!dst_given && !can_make_room(dst, nm, MP_HBM, peek)) return MP_ERR_DST_OOM;
  // ---- mutations start here ----
  begin_call(src);
  begin_call(dst);
  std::vector<mpi::Node*> matched;
  if (need_match) matched = dst->index->match(toks, n_tok, /*pin=*/true);
  int *d_dst = nullptr, *h_dst = nullptr;
  std::vector<int32_t> expect;
  if (!dst_given) {
    DevGuard g(dst->dev);
    if (dst->nfree[MP_HBM] < nm) evict_internal(dst, nm - dst->nfree[MP_HBM], MP_HBM, nullptr);
    TRY(alloc_hbm_launch(dst, nm, &d_dst, &h_dst, dst->verify ? &expect : nullptr));
  }
  std::vector<int32_t> moved_src(sids.begin() + skip, sids.end());
  TRY(transmit(src, dst, moved_src, d_dst, h_dst, dst_given ? &given : nullptr, 0, src->nch,
               flags & MP_XFER_PATH_MASK));
  {
    DevGuard g(dst->dev);
    TRY(sync(dst));
  }
  std::vector<mp_addr> full;
  full.reserve((size_t)ceil_b);
  for (int64_t i = 0; i < q + skip; ++i)
    full.push_back(enc(dst, matched[(size_t)i]->medium, matched[(size_t)i]->idx));
  if (dst_given) {
    for (int64_t i = 0; i < nm; ++i) full.push_back(enc(dst, MP_HBM, given[(size_t)i]));
  } else {
    TRY(alloc_hbm_finish(dst, h_dst, nm, src->inst, dst->verify ? &expect : nullptr));
    for (int64_t i = 0; i < nm; ++i) full.push_back(enc(dst, MP_HBM, h_dst[i]));
  }
  {
    DevGuard g(dst->dev);
    int64_t dup = 0;
    TRY(insert_internal(dst, toks, n_tok, full.data(), (int64_t)full.size(),
                        flags & MP_INS_ERR_ON_CONFLICT, &dup));
    unpin_nodes(dst, matched);
    TRY(sync(dst));
  }
  std::vector<mpi::Node*> fin = dst->index->path(toks, floor_b);
  for (int64_t i = 0; i < floor_b; ++i) da[i] = enc(dst, fin[(size_t)i]->medium, fin[(size_t)i]->idx);
  if (ceil_b > floor_b) da[floor_b] = full[(size_t)floor_b];
  if (n_moved) *n_moved = nm;
  Msg msg{1, src->inst, {}, {}};
  if (priv_len) msg.priv.assign((const uint8_t*)priv, (const uint8_t*)priv + priv_len);
  msg.addrs.assign(da, da + ceil_b);
  dst->inbox.push_back(std::move(msg));
  return MP_OK;
}

mp_status mp_recv_poll(mp_pool* p, mp_recv_msg* out, void* priv_buf, int64_t priv_cap,
                       mp_addr* addrs, int64_t addr_cap) {
  if (!p || !out) return MP_ERR_CONFIG;
  if (p->inbox.empty()) return MP_ERR_PRECONDITION;
  Msg& m = p->inbox.front();
  out->kind = m.kind;
  out->src_instance = m.src;
  out->n_addrs = (int64_t)m.addrs.size();
  out->priv_len = (int64_t)m.priv.size();
  if (priv_cap < out->priv_len || addr_cap < out->n_addrs) return MP_ERR_BUFFER_TOO_SMALL;
  if (!m.priv.empty()) std::memcpy(priv_buf, m.priv.data(), m.priv.size());
  if (!m.addrs.empty()) std::memcpy(addrs, m.addrs.data(), m.addrs.size() * sizeof(mp_addr));
  p->inbox.pop_front();
  return MP_OK;
}

// --------------------------- pack / unpack ---------------------------------
static mp_status pack_unpack(mp_pool* p, const mp_addr* a, int64_t n, int32_t l0, int32_t l1,
                             void* staging, bool pack) {
  if (!p || n < 0 || (n > 0 && (!a || !staging)) || !(0 <= l0 && l0 < l1 && l1 <= p->L))
    return MP_ERR_CONFIG;
  std::vector<int32_t> ids((size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    int m = 0;
    int32_t idx = 0;
    if (!decode(p, a[i], &m, &idx)) return MP_ERR_INVALID_ADDR;
    const uint8_t s = p->st[MP_HBM][(size_t)idx];
    if (m != MP_HBM || s == ST_FREE) return MP_ERR_PRECONDITION;
    if (!pack && s != ST_ACTIVE) return MP_ERR_PRECONDITION;
    ids[(size_t)i] = idx;
  }
  DevGuard g(p->dev);
  begin_call(p);
  int* d = nullptr;
  TRY(upload_ids(p, ids, &d));
  const int nj = 2 * (l1 - l0);
  const long long stride = (long long)nj * p->chunk;
  if (pack)
    TRY(launch_migrate_timed(p, p->stream, pool_ep(p->d_slabs, d), agg_ep((char*)staging, stride, nullptr),
                             n, 2 * l0, nj));
  else
    TRY(launch_migrate_timed(p, p->stream, agg_ep((char*)staging, stride, nullptr), pool_ep(p->d_slabs, d),
                             n, 2 * l0, nj));
  TRY(sync(p));
  TRY(collect_timing(p, n * stride));
  return MP_OK;
}

mp_status mp_pack(mp_pool* p, const mp_addr* a, int64_t n, int32_t l0, int32_t l1,
                  void* staging) {
  return pack_unpack(p, a, n, l0, l1, staging, true);
}

mp_status mp_unpack(mp_pool* p, const void* staging, const mp_addr* a, int64_t n, int32_t l0,
                    int32_t l1) {
  return pack_unpack(p, a, n, l0, l1, const_cast<void*>(staging), false);
}

// ------------------------- measurement / debug -----------------------------
mp_status mp_profile(mp_pool* p, int32_t enable) {
  if (!p) return MP_ERR_CONFIG;
  p->profiling = enable != 0;
  return MP_OK;
}

mp_status mp_stats_get(const mp_pool* p, mp_stats* o) {
  if (!p || !o) return MP_ERR_CONFIG;
  *o = p->stats;
  return MP_OK;
}

mp_status mp_stats_reset(mp_pool* p) {
  if (!p) return MP_ERR_CONFIG;
  p->stats = mp_stats{};
  return MP_OK;
}

mp_status mp_debug_fill(mp_pool* p, const mp_addr* a, int64_t n, uint64_t seed) {
  if (!p || n < 0 || (n > 0 && !a)) return MP_ERR_CONFIG;
  std::vector<int32_t> ids((size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    int m = 0;
    int32_t idx = 0;
    if (!decode(p, a[i], &m, &idx)) return MP_ERR_INVALID_ADDR;
    if (m != MP_HBM || p->st[MP_HBM][(size_t)idx] == ST_FREE || idx >= (1 << 14))
      return MP_ERR_PRECONDITION;
    ids[(size_t)i] = idx;
  }
  DevGuard g(p->dev);
  begin_call(p);
  ++p->epoch;
  int* d = nullptr;
  TRY(upload_ids(p, ids, &d));
  CK(mpk::launch_fill(p->d_slabs, d, (int)n, p->nch, p->chunk, seed, (uint64_t)p->inst, p->epoch,
                      p->stream));
  p->stats.aux_launches += 1;
  return sync(p);
}

mp_status mp_debug_read_block(mp_pool* p, mp_addr a, void* host_out, int64_t cap) {
  int m = 0;
  int32_t idx = 0;
  if (!p || !host_out) return MP_ERR_CONFIG;
  if (!decode(p, a, &m, &idx)) return MP_ERR_INVALID_ADDR;
  if (cap < p->Pb) return MP_ERR_BUFFER_TOO_SMALL;
  DevGuard g(p->dev);
  TRY(sync(p));
  if (m == MP_HBM) {
    for (int j = 0; j < p->nch; ++j)
      CK(cudaMemcpy((char*)host_out + (int64_t)j * p->chunk,
                    p->slabs[(size_t)j] + (int64_t)idx * p->chunk, (size_t)p->chunk,
                    cudaMemcpyDeviceToHost));
  } else {
    std::memcpy(host_out, p->dram + (int64_t)idx * p->Pb, (size_t)p->Pb);
  }
  return MP_OK;
}

mp_status mp_debug_dump_index(mp_pool* p, char* buf, int64_t cap, int64_t* len) {
  if (!p) return MP_ERR_CONFIG;
  const std::string s = p->index->dump();
  if (len) *len = (int64_t)s.size();
  if (!buf || cap <= (int64_t)s.size()) return MP_ERR_BUFFER_TOO_SMALL;
  std::memcpy(buf, s.data(), s.size());
  buf[s.size()] = 0;
  return MP_OK;
}

mp_status mp_debug_block_states(mp_pool* p, int32_t medium, uint8_t* out, int64_t cap) {
  if (!p || (medium != MP_HBM && medium != MP_DRAM) || !out) return MP_ERR_CONFIG;
  if (cap < (int64_t)p->st[medium].size()) return MP_ERR_BUFFER_TOO_SMALL;
  std::memcpy(out, p->st[medium].data(), p->st[medium].size());
  return MP_OK;
}

mp_status mp_debug_bitmap(mp_pool* p, uint32_t* out, int64_t cap_words) {
  if (!p || !out) return MP_ERR_CONFIG;
  if (cap_words < p->nwords) return MP_ERR_BUFFER_TOO_SMALL;
  DevGuard g(p->dev);
  TRY(sync(p));
  CK(cudaMemcpy(out, p->d_bitmap, sizeof(uint32_t) * p->nwords, cudaMemcpyDeviceToHost));
  return MP_OK;
}

}  // extern "C"
