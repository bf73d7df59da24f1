// pool.cpp -- pool lifecycle, the host shadow of the device allocator, the
// id arena, stream ordering and profiling (see pool.hpp for the model).
#include "pool.hpp"

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <cstring>
#include <mutex>

namespace mp {

namespace {
thread_local std::string g_err;
}

void set_err(const std::string& s) { g_err = s; }
const std::string& get_err() { return g_err; }

// ----------------------------------------------------------------- arena
int* arena_take(mp_pool* p, int64_t n, int** host) {
  n = std::max<int64_t>(n, 1);
  if (n > p->ar.cap) return nullptr;
  int64_t at = p->ar.used;
  if (at + n > p->ar.cap) {
    // wrap: everything this process issued is done after the drain (peers
    // never read this arena: their copies take ids from their own side)
    if (drain(p) != MP_OK) return nullptr;
    at = 0;
  }
  p->ar.used = at;
  int* d = p->ar.d + p->ar.used;
  *host = p->ar.h + p->ar.used;
  p->ar.used += n;
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
    CK(cudaMemcpyAsync(d, h, ids.size() * sizeof(int32_t), cudaMemcpyHostToDevice, p->meta));
  }
  *d_out = d;
  return MP_OK;
}

// Source ids of a launch: by value in its parameters when they fit (no copy
// call), else uploaded to the arena.  *d is nullptr in the inline case.
mp_status src_ids(mp_pool* p, const std::vector<int32_t>& ids, int** d, mpk::InlineIds* inl) {
  inl->n = 0;
  *d = nullptr;
  if (!ids.empty() && (int64_t)ids.size() <= mpk::kInlineIds) {
    inl->n = (int)ids.size();
    std::memcpy(inl->ids, ids.data(), ids.size() * sizeof(int32_t));
    return MP_OK;
  }
  return upload_ids(p, ids, d);
}

// ------------------------------------------------- shared data streams
// The pools of one process on one device share their data stream (see
// mp_pool_create): reference-counted, created with the first pool of the
// device and destroyed with the last one (so a cudaDeviceReset after all
// pools are gone leaves no stale handle behind).
namespace {
std::mutex g_stream_mu;
struct DevStream {
  cudaStream_t s = nullptr;
  int refs = 0;
  LaunchTrack track;
} g_dev_stream[kMaxDevStreams];
std::atomic<uint32_t> g_track_gen{0};
}  // namespace

uint32_t new_track_gen() {
  uint32_t g = g_track_gen.fetch_add(1, std::memory_order_relaxed) + 1;
  if (g == 0) g = g_track_gen.fetch_add(1, std::memory_order_relaxed) + 1;  // 0 = never marked
  return g;
}

cudaError_t shared_stream_acquire(int dev, cudaStream_t* out, LaunchTrack** track) {
  std::lock_guard<std::mutex> lk(g_stream_mu);
  DevStream& d = g_dev_stream[dev];
  if (!d.s) {
    const cudaError_t e = cudaStreamCreateWithFlags(&d.s, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      d.s = nullptr;
      return e;
    }
  }
  ++d.refs;
  *out = d.s;
  *track = &d.track;
  return cudaSuccess;
}

void shared_stream_release(int dev) {
  std::lock_guard<std::mutex> lk(g_stream_mu);
  DevStream& d = g_dev_stream[dev];
  if (d.refs > 0 && --d.refs == 0 && d.s) {
    cudaStreamSynchronize(d.s);
    cudaStreamDestroy(d.s);
    d.s = nullptr;
  }
}

// ------------------------------------------- stream memory operations
namespace {
typedef int (*StreamValue32Fn)(cudaStream_t, unsigned long long, uint32_t, unsigned);
StreamValue32Fn driver_value_fn(const char* name) {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return (StreamValue32Fn)f;
}
}  // namespace

mp_status stream_wait_geq(cudaStream_t s, const uint32_t* dptr, uint32_t v) {
  static const StreamValue32Fn fn = driver_value_fn("cuStreamWaitValue32");
  if (!fn) {
    set_err("cuStreamWaitValue32 unavailable");
    return MP_ERR_CUDA;
  }
  // flags 0 = CU_STREAM_WAIT_VALUE_GEQ: (int32_t)(*addr - value) >= 0
  if (fn(s, (unsigned long long)(uintptr_t)dptr, v, 0) != 0) {
    set_err("cuStreamWaitValue32 failed");
    return MP_ERR_CUDA;
  }
  return MP_OK;
}

mp_status stream_write_u32(cudaStream_t s, uint32_t* dptr, uint32_t v) {
  static const StreamValue32Fn fn = driver_value_fn("cuStreamWriteValue32");
  if (!fn) {
    set_err("cuStreamWriteValue32 unavailable");
    return MP_ERR_CUDA;
  }
  // flags 0 = CU_STREAM_WRITE_VALUE_DEFAULT: ordered after (and fenced
  // behind) the stream's earlier work
  if (fn(s, (unsigned long long)(uintptr_t)dptr, v, 0) != 0) {
    set_err("cuStreamWriteValue32 failed");
    return MP_ERR_CUDA;
  }
  return MP_OK;
}

mp_status staging_acquire(mp_pool* p, cudaStream_t s) {
  // an event never recorded is complete, so every slot's event can be waited on
  for (cudaEvent_t e : p->slot_ev) CK(cudaStreamWaitEvent(s, e, 0));
  for (cudaEvent_t e : p->pack_ev) CK(cudaStreamWaitEvent(s, e, 0));
  for (cudaEvent_t e : p->swap_ev) CK(cudaStreamWaitEvent(s, e, 0));
  return MP_OK;
}

// ------------------------------------------------------- sync / ordering
// Frees of HBM blocks reach the device bitmap lazily, on the meta stream:
// small sets by value in a kernel's parameters (folded into the next
// allocation when there is one), large ones through the id arena.
// Deferred claims (mp_alloc_mem) travel the same way, encoded -(id+1).
// Applies every pending update before the next device-bitmap scan: a short
// list is returned in *f for the caller's allocation kernel (f nullable:
// launched here), a long one goes through the id arena now.
static mp_status apply_pending(mp_pool* p, mpk::InlineIds* f) {
  if (f) f->n = 0;
  if (p->dev_upd.empty()) return MP_OK;
  std::vector<int32_t> v;
  p->dev_upd.take(&v);
  if (v.empty()) return MP_OK;  // everything cancelled out
  if ((int)v.size() <= mpk::kInlineIds) {
    mpk::InlineIds local;
    mpk::InlineIds* g = f ? f : &local;
    g->n = (int)v.size();
    std::memcpy(g->ids, v.data(), v.size() * sizeof(int32_t));
    if (f) return MP_OK;
    CK(mpk::launch_alloc(p->d_bitmap, p->nwords, 0, nullptr, nullptr, p->d_err, p->meta, g));
  } else {
    int* d = nullptr;
    TRY(upload_ids(p, v, &d));
    CK(mpk::launch_free(p->d_bitmap, d, (int)v.size(), p->meta));
  }
  p->stats.aux_launches += 1;
  return MP_OK;
}

mp_status flush_frees(mp_pool* p) { return apply_pending(p, nullptr); }

// Accumulates the timed launches whose end event has completed, oldest first
// (all of them after a sync).  Never blocks.
static mp_status harvest_timed(mp_pool* p) {
  size_t k = 0;
  for (; k < p->timed.size(); ++k) {
    const TimedLaunch& t = p->timed[k];
    const cudaEvent_t end = p->tev[2 * (size_t)t.pair + 1];
    const cudaError_t q = cudaEventQuery(end);
    if (q == cudaErrorNotReady) break;
    CK(q);
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, p->tev[2 * (size_t)t.pair], end));
    p->stats.kernel_ms += ms;
    p->stats.timed_launches += 1;
    p->stats.timed_bytes += t.bytes;
    if (p->profile_every == 1 && p->last_timed_pair >= 0) {
      // idle time of the data stream between consecutive migrations
      float gap = 0.f;
      CK(cudaEventElapsedTime(&gap, p->tev[2 * (size_t)p->last_timed_pair + 1],
                              p->tev[2 * (size_t)t.pair]));
      p->stats.gap_ms += gap;
    }
    p->last_timed_pair = t.pair;
  }
  p->timed.erase(p->timed.begin(), p->timed.begin() + (std::ptrdiff_t)k);
  return MP_OK;
}

mp_status drain(mp_pool* p) {
  TRY(remote_apply_waits(p));  // blocks stored by other processes have landed too
  CK(sync_stream_traced(p, p->meta, "drain:meta"));
  CK(sync_stream_traced(p, p->stream, "drain:stream"));
  CK(sync_stream_traced(p, p->copy_stream, "drain:copy_stream"));  // STAGED copies issued by p
  track_fence(p->track);  // idle: the window is empty (the next launch opens one)
  TRY(harvest_timed(p));
  p->last_timed_pair = -1;  // no gap across a sync
  if (!p->pending_verify.empty()) {
    int err = 0;
    CK(cudaMemcpy(&err, p->d_err, sizeof(int), cudaMemcpyDeviceToHost));
    std::vector<PendingVerify> pv;
    pv.swap(p->pending_verify);
    if (err) {
      set_err("device allocator ran short of free blocks");
      return MP_ERR_INTERNAL;
    }
    for (const PendingVerify& v : pv)
      for (size_t i = 0; i < v.want.size(); ++i)
        if (v.host[i] != v.want[i]) {
          set_err("device allocator disagrees with the host shadow (lowest-first)");
          return MP_ERR_INTERNAL;
        }
  }
  return MP_OK;
}

mp_status sync(mp_pool* p) {
  TRY(flush_involving(p));
  TRY(flush_frees(p));
  return drain(p);
}

// --------------------------------------------------------- coalescing
// Make dst's batch ready for n more transfers from src over slabs [j0, j0+nj):
// a batch from another source / range, or one without room, goes first, and
// so does everything pending that reads dst's or writes src's blocks; an
// empty batch gets the next id table of the ring once its last reader is done.
mp_status batch_open(mp_pool* src, mp_pool* dst, int64_t n, int j0, int nj) {
  auto& b = dst->batch;
  if (b.open && (b.src != src || b.j0 != j0 || b.nj != nj || b.count + n > dst->batch_cap))
    TRY(flush_batch(dst));
  for (auto& kv : src->peers)
    if (kv.second != dst && kv.second->batch.src == src && kv.second->batch.count)
      TRY(flush_batch(kv.second));
  if (src->batch.count) TRY(flush_batch(src));
  for (auto& kv : dst->peers)
    if (kv.second->batch.src == dst && kv.second->batch.count) TRY(flush_batch(kv.second));
  if (!b.open) {
    b.src = src;
    b.j0 = j0;
    b.nj = nj;
    b.count = 0;
    b.bytes = 0;
    b.sids.clear();
    b.dids.clear();
    const int k = dst->btab_next;
    dst->btab_next = (k + 1) % mp_pool::kBatchTabs;
    if (dst->btab_used[k]) CK(cudaStreamWaitEvent(dst->meta, dst->btab_ev[k], 0));
    b.tab = k;
    dst->bsrc = dst->bsrc_ring[k];
    dst->bdst = dst->bdst_ring[k];
    b.open = true;
  }
  return MP_OK;
}

mp_status batch_append(mp_pool* src, mp_pool* dst, const std::vector<int32_t>& sids,
                       const std::vector<int32_t>& dids, const int* d_dst, int j0, int nj) {
  const int64_t n = (int64_t)sids.size();
  auto& b = dst->batch;
  const bool tm = host_timing_on();
  double t0 = tm ? host_clock() : 0.0;
  auto lap = [&](int i) {
    if (!tm) return;
    const double t = host_clock();
    host_lap(i, t - t0);
    t0 = t;
  };
  TRY(batch_open(src, dst, n, j0, nj));
  lap(5);
  // id tables: source ids stay on the host until the launch (kernel
  // parameters, or one upload per launch); destination ids are the device
  // allocator's output -- already in place when it allocated into this
  // batch's table -- or the caller's ids
  if (d_dst == dst->bdst + b.count) {
    // written there by the allocation kernel (slot_hint)
  } else if (d_dst) {
    CK(cudaMemcpyAsync(dst->bdst + b.count, d_dst, (size_t)n * sizeof(int32_t),
                       cudaMemcpyDeviceToDevice, dst->meta));
  } else {
    int* h2 = nullptr;
    if (!arena_take(dst, n, &h2)) {
      set_err("id arena exhausted");
      return MP_ERR_INTERNAL;
    }
    std::memcpy(h2, dids.data(), (size_t)n * sizeof(int32_t));
    CK(cudaMemcpyAsync(dst->bdst + b.count, h2, (size_t)n * sizeof(int32_t),
                       cudaMemcpyHostToDevice, dst->meta));
  }
  for (int64_t i = 0; i < n; ++i) {
    src->pend_r[(size_t)sids[(size_t)i]] = 1;
    dst->pend_w[(size_t)dids[(size_t)i]] = 1;
  }
  b.sids.insert(b.sids.end(), sids.begin(), sids.end());
  b.dids.insert(b.dids.end(), dids.begin(), dids.end());
  b.count += n;
  b.bytes += (uint64_t)n * (uint64_t)nj * (uint64_t)dst->chunk;
  dst->stats.blocks_moved += (uint64_t)n;
  lap(6);
  // keep the device busy: go now if the launches queued on its data stream
  // are about to drain (host estimate) or it has run dry
  constexpr double kDrainLead = 50e-6;
  const bool go = b.bytes >= dst->batch_limit ||
                  (dst->idle_flush && (host_clock() + kDrainLead >= dst->track->busy_until ||
                                       cudaStreamQuery(dst->stream) == cudaSuccess));
  lap(7);
  if (go) TRY(flush_batch(dst));
  lap(8);
  return MP_OK;
}

mp_status flush_batch(mp_pool* dst) {
  auto& b = dst->batch;
  if (b.count == 0) {
    b.open = false;  // an empty batch just gives its table back
    return MP_OK;
  }
  b.open = false;
  mp_pool* src = b.src;
  const int64_t n = b.count;
  b.count = 0;  // reentrancy guard: link / launch below do not flush
  TRY(link(src, dst));
  {
    DevGuard g(dst->dev);
    // source ids: by value in the launch parameters when they fit, else one
    // upload into this batch's table (ordered before the launch by meta_fence).
    // Destination ids too when both lists fit (the host shadow holds the ids
    // the allocation kernel wrote into the table): the copy then reads no id
    // table, so it does not wait for the meta stream's allocation kernel.
    mpk::InlineIds sinl;
    const bool inl = n <= mpk::kInlineIds;
    const bool dinl = 2 * n <= mpk::kInlineIds;
    if (inl) {
      sinl.n = (int)n;
      std::memcpy(sinl.ids, b.sids.data(), (size_t)n * sizeof(int32_t));
      if (dinl) {
        sinl.nd = (int)n;
        std::memcpy(sinl.ids + n, b.dids.data(), (size_t)n * sizeof(int32_t));
      }
    } else {
      CK(cudaMemcpyAsync(dst->bsrc, b.sids.data(), (size_t)n * sizeof(int32_t),
                         cudaMemcpyHostToDevice, dst->meta));
    }
    const LaunchBlocks lb{&src->bmarks, b.sids.data(), &dst->bmarks, b.dids.data(), n};
    TRY(launch_migrate_timed(dst, dst->stream, pool_ep(src->d_slabs, inl ? nullptr : dst->bsrc),
                             pool_ep(dst->d_slabs, dinl ? nullptr : dst->bdst), n, b.j0, b.nj,
                             false, 0, inl ? &sinl : nullptr, /*meta_dep=*/!dinl, &lb));
    {  // queued work estimate: read + write of the batch at ~7 TB/s
      constexpr double kRate = 7.0e12;
      const double now = host_clock();
      dst->track->busy_until = std::max(now, dst->track->busy_until) +
                               2.0 * (double)b.bytes / kRate;
    }
    if (!inl || !dinl) {  // the launch reads this batch's id tables: guard their reuse
      CK(cudaEventRecord(dst->btab_ev[b.tab], dst->stream));
      dst->btab_used[b.tab] = true;
    }  // (no stream op between back-to-back inline launches: PDL overlaps them)
  }
  TRY(link(dst, src));
  for (int32_t id : b.sids) src->pend_r[(size_t)id] = 0;
  for (int32_t id : b.dids) dst->pend_w[(size_t)id] = 0;
  b.sids.clear();
  b.dids.clear();
  b.bytes = 0;
  return MP_OK;
}

// Memory asymmetry ("the fastest link with the least data
// copies"): the copy engine reads pinned DRAM at ~55 GB/s where SM loads of
// mapped host memory reach ~51 (profiles/sweep_r02_dram_source*.json), and
// the staging bounce costs HBM bandwidth only (two passes of Pb at TB/s).
// MP_DRAM_SOURCE=sm keeps the zero-copy kernel (measurement knob).
bool dram_source_ce(const mp_pool* src, int nj) {
  const char* e = getenv("MP_DRAM_SOURCE");
  if (e && e[0] == 's') return false;
  return src->staging && src->staging_bytes >= (int64_t)nj * src->chunk;
}

mp_status dram_ce_scatter(mp_pool* src, mp_pool* ex, cudaStream_t s, char** dslabs,
                          const std::vector<int32_t>& sids, const std::vector<int32_t>& dids,
                          int j0, int nj, bool peer) {
  const int64_t n = (int64_t)sids.size();
  if (n == 0) return MP_OK;
  const int64_t per = (int64_t)nj * src->chunk;  // chunks [j0, j0+nj) of a block: one run
  const int64_t cap = src->staging_bytes / per;
  if (cap < 1) {
    set_err("staging smaller than one block");
    return MP_ERR_CONFIG;
  }
  // two slots: the H2D of one overlaps the scatter of the other; a slot of at
  // most a quarter of the transfer, so the first scatter starts early, and
  // its destination ids fit the launch parameters
  const int halves = cap >= 2 ? 2 : 1;
  const int64_t k = std::min<int64_t>(
      std::min<int64_t>(cap / halves, std::max<int64_t>(1, (n + 3) / 4)), mpk::kInlineIds);
  DevGuard g(src->dev);
  TRY(staging_acquire(src, src->copy_stream));  // earlier STAGED / swap users of the staging
  // every earlier device op of the source (e.g. a zero-copy swap_out still
  // writing these DRAM blocks) goes first
  CK(cudaEventRecord(src->swap_ev[0], src->stream));
  CK(cudaStreamWaitEvent(src->copy_stream, src->swap_ev[0], 0));
  const bool whole = j0 == 0 && nj == src->nch;
  for (int64_t b0 = 0, r = 0; b0 < n; b0 += k, ++r) {
    const int64_t nb = std::min(n - b0, k);
    const int h = (int)(r % halves);
    char* stg = src->staging + (int64_t)h * k * per;
    if (r >= halves) CK(cudaStreamWaitEvent(src->copy_stream, src->swap_ev[2 + h], 0));
    for (int64_t i = 0; i < nb;) {
      int64_t j = i + 1;  // whole blocks: a run of consecutive DRAM blocks is one copy
      while (whole && j < nb && sids[(size_t)(b0 + j)] == sids[(size_t)(b0 + j - 1)] + 1) ++j;
      CK(cudaMemcpyAsync(stg + i * per,
                         src->dram + (int64_t)sids[(size_t)(b0 + i)] * src->Pb +
                             (int64_t)j0 * src->chunk,
                         (size_t)(per * (j - i)), cudaMemcpyHostToDevice, src->copy_stream));
      i = j;
    }
    CK(cudaEventRecord(src->swap_ev[h], src->copy_stream));
    CK(cudaStreamWaitEvent(s, src->swap_ev[h], 0));
    mpk::InlineIds di;  // source = the slot itself (block i at i * per)
    di.n = 0;
    di.nd = (int)nb;
    std::memcpy(di.ids, dids.data() + b0, (size_t)nb * sizeof(int32_t));
    TRY(launch_migrate_timed(ex, s, agg_ep(stg, per, nullptr), pool_ep(dslabs, nullptr), nb, j0,
                             nj, peer, 0, &di, /*meta_dep=*/false));
    CK(cudaEventRecord(src->swap_ev[2 + h], s));
  }
  return MP_OK;
}

mp_status flush_involving(mp_pool* p) {
  if (p->batch.count) TRY(flush_batch(p));
  for (auto& kv : p->peers)
    if (kv.second->batch.src == p && kv.second->batch.count) TRY(flush_batch(kv.second));
  return MP_OK;
}

mp_status link(mp_pool* signal, mp_pool* waiter) {
  if (signal == waiter) return MP_OK;
  TRY(remote_apply_waits(signal));
  if (signal->stream == waiter->stream) return MP_OK;  // one shared stream: already ordered
  {
    DevGuard g(signal->dev);
    CK(cudaEventRecord(signal->ev_order, signal->stream));
  }
  DevGuard g(waiter->dev);
  CK(cudaStreamWaitEvent(waiter->stream, signal->ev_order, 0));
  return MP_OK;
}

mp_status meta_fence(mp_pool* p) {
  CK(cudaEventRecord(p->ev_meta, p->meta));
  CK(cudaStreamWaitEvent(p->stream, p->ev_meta, 0));
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

// ------------------------------------------------------------- allocator
void free_block(mp_pool* p, int med, int32_t idx) {
  p->st[med][(size_t)idx] = ST_FREE;
  p->alloc_by[med][(size_t)idx] = -1;
  ++p->nfree[med];
  if (med == MP_HBM) {
    p->hfree[(size_t)idx >> 6] |= 1ull << (idx & 63);
    p->dev_upd.on_free(idx);  // device bitmap: stream-ordered, lazily
  } else {
    p->dram_free.insert(idx);
  }
}

// R8: evict up to n LRU leaves of `med`; appends freed ids.
void evict_internal(mp_pool* p, int64_t n, int med, std::vector<int32_t>* freed) {
  for (int64_t k = 0; k < n; ++k) {
    int32_t idx = -1;
    if (!p->index->evict_lru_leaf(med, &idx)) break;
    free_block(p, med, idx);
    if (freed) freed->push_back(idx);
  }
}

// R2 feasibility: free + eventually-evictable (excluding the pinned path) >= n.
bool can_make_room(mp_pool* p, int64_t n, int med, const std::vector<mpi::Node*>& pinned) {
  if (p->nfree[med] >= n) return true;
  // the pool is full (the cache regime): peel only as much as is needed
  return p->index->evictable_at_least(med, pinned, n - p->nfree[med]);
}

mp_status alloc_hbm(mp_pool* p, int64_t n, int32_t requester, std::vector<int32_t>* ids,
                    int** d_ids, bool defer) {
  ids->clear();
  if (n > p->nfree[MP_HBM]) {
    set_err("alloc_hbm: host shadow short");
    return MP_ERR_INTERNAL;
  }
  if (n == 0) {
    *d_ids = nullptr;
    return MP_OK;
  }
  for (size_t w = 0; w < p->hfree.size() && (int64_t)ids->size() < n; ++w) {
    uint64_t bits = p->hfree[w];
    while (bits && (int64_t)ids->size() < n) {
      const int b = __builtin_ctzll(bits);
      bits &= bits - 1;
      const int32_t id = (int32_t)(w * 64 + (size_t)b);
      p->hfree[w] &= ~(1ull << b);
      p->st[MP_HBM][(size_t)id] = ST_ACTIVE;
      p->alloc_by[MP_HBM][(size_t)id] = requester;
      ids->push_back(id);
    }
  }
  p->nfree[MP_HBM] -= n;
  // a reused block may still be read or written by a coalesced copy that has
  // not been launched yet: launch those first (stream order does the rest)
  bool hazard = false;
  for (int32_t id : *ids) hazard = hazard || p->pend_w[(size_t)id] || p->pend_r[(size_t)id];
  if (hazard) TRY(flush_involving(p));
  if (defer) {
    for (int32_t id : *ids) p->dev_upd.on_claim(id);
    // keep the queue bounded (stale entries and long claim runs)
    // keep the queue bounded on the host (stale entries and long claim
    // runs); the device learns the updates at its next scan or sync
    if (p->dev_upd.queued() > (size_t)4 * mpk::kInlineIds + 2 * (size_t)p->n_hbm)
      p->dev_upd.compact();
    *d_ids = nullptr;
    return MP_OK;
  }
  // the device bitmap must see every earlier free first: small sets ride in
  // the allocation kernel's parameters
  mpk::InlineIds f;
  TRY(apply_pending(p, &f));
  int* h = nullptr;
  int* d = arena_take(p, n, &h);
  if (!d) {
    set_err("id arena exhausted");
    return MP_ERR_INTERNAL;
  }
  if (p->slot_hint.src) {  // coalesced transfer: allocate into the batch table
    mp_pool* src = p->slot_hint.src;
    p->slot_hint.src = nullptr;
    TRY(batch_open(src, p, n, p->slot_hint.j0, p->slot_hint.nj));
    d = p->bdst + p->batch.count;
  }
  CK(mpk::launch_alloc(p->d_bitmap, p->nwords, (int)n, d, p->verify ? h : nullptr, p->d_err,
                       p->meta, f.n ? &f : nullptr));
  p->stats.aux_launches += 1;
  if (p->verify) p->pending_verify.push_back({h, *ids});
  *d_ids = d;
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

// ------------------------------------------------------------ migration
// Whether the next launch on p's data stream must wait for the grids before
// it (see LaunchTrack), and its blocks joined to the window.
static bool window_admit(LaunchTrack* t, const LaunchBlocks* lb) {
  static const bool overlap = [] {  // MP_PDL_OVERLAP=0: every launch waits (comparison)
    const char* e = getenv("MP_PDL_OVERLAP");
    return !(e && e[0] == '0');
  }();
  constexpr int kMaxWindow = 8;  // bounds how many grids may overlap
  bool wait = !overlap || !lb || t->unknown || t->launches >= kMaxWindow || t->gen == 0;
  if (!wait) {
    const uint32_t g = t->gen;
    for (int64_t i = 0; i < lb->n && !wait; ++i) wait = lb->rm->w[(size_t)lb->sids[i]] == g;
    for (int64_t i = 0; i < lb->n && !wait; ++i) {
      const size_t d = (size_t)lb->dids[i];
      wait = lb->wm->w[d] == g || lb->wm->r[d] == g;
    }
  }
  if (wait) {  // a new window starts with this launch
    t->gen = new_track_gen();
    t->launches = 0;
    t->unknown = false;
  }
  if (lb) {
    const uint32_t g = t->gen;
    for (int64_t i = 0; i < lb->n; ++i) lb->rm->r[(size_t)lb->sids[i]] = g;
    for (int64_t i = 0; i < lb->n; ++i) lb->wm->w[(size_t)lb->dids[i]] = g;
  } else {
    t->unknown = true;
  }
  ++t->launches;
  return wait;
}

mp_status launch_migrate_timed(mp_pool* p, cudaStream_t s, const mpk::Endpoint& a0,
                               const mpk::Endpoint& b0, int64_t n, int j0, int nj, bool peer,
                               int64_t len, const mpk::InlineIds* src_inline, bool meta_dep,
                               const LaunchBlocks* blocks) {
  if (n <= 0) return MP_OK;
  if (len <= 0) len = p->chunk;
  mpk::Endpoint a = a0, b = b0;
  if (!a.cstride) a.cstride = p->chunk;
  if (!b.cstride) b.cstride = p->chunk;
  const uint64_t bytes = (uint64_t)n * (uint64_t)nj * (uint64_t)len;
  const bool cand = p->profile_every > 0 && s == p->stream;
  const bool timed = cand && (p->profile_seen++ % (uint64_t)p->profile_every) == 0;
  if (cand) {
    p->stats.profiled_launches += 1;
    p->stats.profiled_bytes += bytes;
  }
  if (s == p->stream) {
    TRY(remote_apply_waits(p));  // blocks other processes stored into p
    if (meta_dep) TRY(meta_fence(p));  // ids uploaded / allocated on meta
  }
  int pair = -1;
  if (timed) {
    if ((int)p->timed.size() >= kTimedPairs) {
      TRY(harvest_timed(p));
      if ((int)p->timed.size() >= kTimedPairs) {  // 512 timed launches still queued
        CK(cudaEventSynchronize(p->tev[2 * (size_t)p->timed.front().pair + 1]));
        TRY(harvest_timed(p));
      }
    }
    pair = p->tev_next;
    p->tev_next = (p->tev_next + 1) % kTimedPairs;
    CK(cudaEventRecord(p->tev[2 * (size_t)pair], s));
  }
  // Copy engine: auto = the bulk (TMA) ring for copies within this GPU's HBM
  // (measured ~1% ahead of the vector kernel, with a third of the issued
  // instructions); mapped pinned DRAM (swap) stays on the vector LD/ST path;
  // stores into peer memory (NVLink / IPC) take the pool's peer_engine.
  const bool host_side = (a.base && a.base == p->dram_dev) || (b.base && b.base == p->dram_dev);
  int variant = p->copy_kernel == mpk::kCopyAuto ? mpk::kCopyBulk : p->copy_kernel;
  // environment defaults of the auto peer choices (measurement knobs):
  // MP_PEER_ENGINE=bulk, MP_PEER_SCHED=dynamic
  static const int env_peer_engine = [] {
    const char* e = getenv("MP_PEER_ENGINE");
    return (e && e[0] == 'b') ? mpk::kCopyBulk : mpk::kCopyVector;
  }();
  static const bool env_peer_dyn = [] {
    const char* e = getenv("MP_PEER_SCHED");
    return e && e[0] == 'd';
  }();
  if (host_side) {
    variant = mpk::kCopyVector;
  } else if (peer) {
    variant = p->peer_engine ? p->peer_engine
                             : (p->copy_kernel ? p->copy_kernel : env_peer_engine);
  }
  // dynamic unit claiming on the pool's data stream (launches serialised);
  // stores into a peer's memory default to the static split: on the one-GPU
  // two-process run (IPC-mapped pool) it was 4% ahead of claiming
  // (profiles/sched_r01.txt), and an NVLink-bound copy gains less from
  // rebalancing SMs
  const bool peer_dyn = p->peer_sched ? p->peer_sched == 2 : env_peer_dyn;
  const mpk::Sched sched{p->d_sched, &p->sched_base};
  // only launches on the data stream join its window; a timed launch is
  // bracketed by events (stream operations between kernels), so it waits
  const bool wait = s != p->stream || timed || window_admit(p->track, blocks);
  if (timed && s == p->stream) track_fence(p->track);
  CK(mpk::launch_migrate(a, b, (int)n, j0, nj, len, p->max_ctas, s, variant,
                         (s == p->stream && (!peer || peer_dyn)) ? &sched : nullptr,
                         src_inline, wait));
  if (!wait) p->stats.overlapped_launches += 1;
  if (timed) {
    CK(cudaEventRecord(p->tev[2 * (size_t)pair + 1], s));
    p->timed.push_back({pair, bytes});
  }
  p->stats.kernel_launches += 1;
  p->stats.bytes_moved += bytes;
  return MP_OK;
}

}  // namespace mp

using namespace mp;

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

const char* mp_last_error(void) { return get_err().c_str(); }

void mp_pool_destroy(mp_pool* p) {
  if (!p) return;
  if (p->stream) {
    remote_flush_tx(p);  // a pipelined copy the peer's stream may wait for
    flush_involving(p);
  }
  {  // copies into peers' IPC-mapped blocks / rings finish before the mappings close
    DevGuard g(p->dev);
    if (p->stream) cudaStreamSynchronize(p->stream);
    if (p->copy_stream) cudaStreamSynchronize(p->copy_stream);
    if (p->meta) cudaStreamSynchronize(p->meta);
  }
  remote_close_all(p);
  {
    DevGuard g(p->dev);
    if (p->meta) cudaStreamSynchronize(p->meta);
    if (p->stream) cudaStreamSynchronize(p->stream);
    for (auto& kv : p->peers) {
      mp_pool* q = kv.second;
      q->peers.erase(p->inst);
      auto it = q->peer_tables.find(p->inst);
      if (it != q->peer_tables.end()) {
        DevGuard g2(q->dev);
        if (q->stream) cudaStreamSynchronize(q->stream);
        if (q->meta) cudaStreamSynchronize(q->meta);
        cudaFree(it->second);
        q->peer_tables.erase(it);
      }
    }
    for (auto& kv : p->peer_tables) cudaFree(kv.second);
    if (p->own_slab_region) cudaFree(p->own_slab_region);
    if (p->d_slabs) cudaFree(p->d_slabs);
    if (p->d_bitmap) cudaFree(p->d_bitmap);
    if (p->d_err) cudaFree(p->d_err);
    if (p->d_sched) cudaFree(p->d_sched);
    if (p->ar.d) cudaFree(p->ar.d);
    for (int k = 0; k < mp_pool::kBatchTabs; ++k) {
      if (p->bsrc_ring[k]) cudaFree(p->bsrc_ring[k]);
      if (p->bdst_ring[k]) cudaFree(p->bdst_ring[k]);
      if (p->btab_ev[k]) cudaEventDestroy(p->btab_ev[k]);
    }
    if (p->ar.h) cudaFreeHost(p->ar.h);
    if (p->own_dram && p->dram) cudaFreeHost(p->dram);
    if (p->staging) cudaFree(p->staging);
    if (p->ev_order) cudaEventDestroy(p->ev_order);
    if (p->ev_meta) cudaEventDestroy(p->ev_meta);
    for (auto e : p->slot_ev) cudaEventDestroy(e);
    for (auto e : p->pack_ev) cudaEventDestroy(e);
    for (auto e : p->swap_ev)
      if (e) cudaEventDestroy(e);
    for (auto e : p->tev) cudaEventDestroy(e);
    if (p->stream && !p->shared_stream) cudaStreamDestroy(p->stream);
    if (p->stream && p->shared_stream) shared_stream_release(p->dev);
    if (p->meta) cudaStreamDestroy(p->meta);
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
  p->copy_kernel = cfg->copy_kernel;
  p->peer_engine = cfg->peer_engine;
  p->peer_sched = cfg->peer_sched;
  p->force_peer = cfg->force_peer != 0;
  if (p->copy_kernel < 0 || p->copy_kernel > 2 || p->peer_engine < 0 || p->peer_engine > 2 ||
      p->peer_sched < 0 || p->peer_sched > 2) {
    set_err("copy_kernel / peer_engine must be 0 (auto), 1 (vector) or 2 (bulk); "
            "peer_sched 0 (auto), 1 (static) or 2 (dynamic)");
    delete p->index;
    delete p;
    return MP_ERR_CONFIG;
  }
  p->staging_slots = std::min(cfg->staging_slots > 0 ? cfg->staging_slots : 4, kMaxSyncSlots);
  p->staging_bytes = cfg->staging_bytes > 0 ? cfg->staging_bytes : (256ll << 20);
  p->index = new mpi::Index(p->B, p->n_hbm, p->n_dram);
  for (int m = 0; m < 2; ++m) {
    const int64_t n = m == 0 ? p->n_hbm : p->n_dram;
    p->st[m].assign((size_t)n, ST_FREE);
    p->alloc_by[m].assign((size_t)n, -1);
    p->nfree[m] = n;
  }
  p->mark[0].assign((size_t)p->n_hbm, 0u);
  p->mark[1].assign((size_t)p->n_dram, 0u);
  p->hfree.assign((size_t)((p->n_hbm + 63) / 64), ~0ull);
  if (p->n_hbm % 64) p->hfree.back() = (1ull << (p->n_hbm % 64)) - 1ull;
  for (int32_t i = 0; i < (int32_t)p->n_dram; ++i) p->dram_free.insert(p->dram_free.end(), i);
  auto fail = [&](mp_status s) {
    mp_pool_destroy(p);
    return s;
  };
#define CKC(x)                                                  \
  do {                                                          \
    cudaError_t e_ = (x);                                       \
    if (e_ != cudaSuccess) {                                    \
      set_err(std::string(#x) + ": " + cudaGetErrorString(e_)); \
      return fail(MP_ERR_CUDA);                                 \
    }                                                           \
  } while (0)
  int ndev = 0;
  CKC(cudaGetDeviceCount(&ndev));
  if (cfg->device < 0 || cfg->device >= ndev) {
    set_err("device ordinal out of range");
    return fail(MP_ERR_CONFIG);
  }
  DevGuard g(p->dev);
  CKC(mpk::preload_kernels());  // no lazy kernel load behind a parked stream (kernels.cuh)
  // The pools of one process on one device share a data stream: a
  // migration between two of them (P -> D, then D -> P) is then ordered by
  // the stream itself instead of a cross-stream event wait per launch, which
  // costs the GPU several microseconds per handoff (ReAct-like traffic:
  // 0.84 -> 0.88 of the time in migration kernels).  Migrations are
  // HBM-bound, so running two pools' copies concurrently would gain nothing.
  // MP_SHARED_STREAM=0: one stream per pool.
  {
    static const bool shared = [] {
      const char* e = getenv("MP_SHARED_STREAM");
      return !(e && e[0] == '0');
    }();
    if (shared && p->dev < kMaxDevStreams) {
      CKC(shared_stream_acquire(p->dev, &p->stream, &p->track));
      p->shared_stream = true;
    } else {
      CKC(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
      p->track = &p->own_track;
    }
  }
  CKC(cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking));
  // The allocator's one-CTA kernel for the next transfer is issued while the
  // current migration kernel fills every SM; at the highest priority its CTA
  // is placed as soon as migration CTAs start retiring, so the next
  // migration does not wait behind it.
  {
    int lo = 0, hi = 0;
    CKC(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CKC(cudaStreamCreateWithPriority(&p->meta, cudaStreamNonBlocking, hi));
  }
  CKC(cudaEventCreateWithFlags(&p->ev_order, cudaEventDisableTiming));
  CKC(cudaEventCreateWithFlags(&p->ev_meta, cudaEventDisableTiming));
  p->uid = new_uid();
  p->slot_ev.resize((size_t)p->staging_slots);
  for (auto& e : p->slot_ev) CKC(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  p->pack_ev.resize((size_t)p->staging_slots);
  for (auto& e : p->pack_ev) CKC(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : p->swap_ev) CKC(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  p->tev.resize(2 * (size_t)kTimedPairs);
  for (auto& e : p->tev) CKC(cudaEventCreate(&e));
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
  p->bmarks.reset((size_t)p->n_hbm);
  CKC(cudaMalloc(&p->d_slabs, sizeof(char*) * p->nch));
  CKC(cudaMemcpy(p->d_slabs, p->slabs.data(), sizeof(char*) * p->nch, cudaMemcpyHostToDevice));
  p->nwords = (int)((p->n_hbm + 31) / 32);
  std::vector<uint32_t> bm((size_t)p->nwords, 0xFFFFFFFFu);
  if (p->n_hbm % 32) bm.back() = (1u << (p->n_hbm % 32)) - 1u;
  CKC(cudaMalloc(&p->d_bitmap, sizeof(uint32_t) * p->nwords));
  CKC(cudaMemcpy(p->d_bitmap, bm.data(), sizeof(uint32_t) * p->nwords, cudaMemcpyHostToDevice));
  CKC(cudaMalloc(&p->d_err, sizeof(int)));
  CKC(cudaMemset(p->d_err, 0, sizeof(int)));
  CKC(cudaMalloc(&p->d_sched, sizeof(unsigned long long)));
  CKC(cudaMemset(p->d_sched, 0, sizeof(unsigned long long)));
  p->ar.cap = 16 * std::max<int64_t>(std::max(p->n_hbm, p->n_dram), 4096);
  CKC(cudaMalloc(&p->ar.d, sizeof(int) * p->ar.cap));
  p->coalesce = cfg->coalesce_mib >= 0;
  {  // test knob: batch by size only, so tests exercise multi-transfer launches
    const char* e = getenv("MP_COALESCE_NO_IDLE_FLUSH");
    p->idle_flush = !(e && e[0] == '1');
  }
  // 4 GiB: +0.7% on the configs[1] bench over 1 GiB (fewer launch ramps and
  // tails while the GPU is busy; an idle stream still flushes at once),
  // profiles/coalesce_r02.txt
  p->batch_limit = (uint64_t)(cfg->coalesce_mib > 0 ? cfg->coalesce_mib : 4096) << 20;
  p->batch_cap = p->n_hbm;
  p->pend_w.assign((size_t)p->n_hbm, 0);
  p->dev_upd.reset((size_t)p->n_hbm);
  p->pend_r.assign((size_t)p->n_hbm, 0);
  for (int k = 0; k < mp_pool::kBatchTabs; ++k) {
    CKC(cudaMalloc(&p->bsrc_ring[k], sizeof(int) * (size_t)p->batch_cap));
    CKC(cudaMalloc(&p->bdst_ring[k], sizeof(int) * (size_t)p->batch_cap));
    CKC(cudaEventCreateWithFlags(&p->btab_ev[k], cudaEventDisableTiming));
  }
  p->bsrc = p->bsrc_ring[0];
  p->bdst = p->bdst_ring[0];
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
  TRY(remote_flush_tx(a));
  TRY(remote_flush_tx(b));
  // kv_heads may differ: tensor-parallel shards of one model (mp_transfer_heads);
  // whole-block transfers additionally require equal chunk sizes
  if (a->L != b->L || a->B != b->B || a->D != b->D || a->elem != b->elem) {
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
      if (e == cudaErrorPeerAccessAlreadyEnabled)
        cudaGetLastError();
      else
        CK(e);
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

mp_status mp_sync(mp_pool* p) {
  if (!p) return MP_ERR_CONFIG;
  DevGuard g(p->dev);
  TRY(remote_flush_tx(p));
  return sync(p);
}

mp_status mp_wait_event(mp_pool* p, void* ev) {
  if (!p || !ev) return MP_ERR_CONFIG;
  DevGuard g(p->dev);
  TRY(remote_flush_tx(p));
  // a pending coalesced copy was issued before the dependency existed: it
  // must not be delayed behind it, nor run before the producer's data below
  TRY(flush_involving(p));
  CK(cudaStreamWaitEvent(p->stream, (cudaEvent_t)ev, 0));
  return MP_OK;
}

mp_status mp_record_event(mp_pool* p, void* ev) {
  if (!p || !ev) return MP_ERR_CONFIG;
  DevGuard g(p->dev);
  TRY(remote_flush_tx(p));
  TRY(flush_involving(p));
  TRY(remote_apply_waits(p));
  TRY(meta_fence(p));
  CK(cudaEventRecord((cudaEvent_t)ev, p->stream));
  return MP_OK;
}

mp_status mp_profile(mp_pool* p, int32_t every) {
  if (!p || every < 0) return MP_ERR_CONFIG;
  DevGuard g(p->dev);
  TRY(remote_flush_tx(p));
  if (!every && p->profile_every) TRY(drain(p));
  p->profile_every = every;
  p->profile_seen = 0;
  return MP_OK;
}

mp_status mp_stats_get(const mp_pool* p, mp_stats* o) {
  if (!p || !o) return MP_ERR_CONFIG;
  *o = p->stats;
  return MP_OK;
}

mp_status mp_stats_reset(mp_pool* p) {
  if (!p) return MP_ERR_CONFIG;
  DevGuard g(p->dev);
  TRY(remote_flush_tx(p));
  TRY(drain(p));
  p->stats = mp_stats{};
  return MP_OK;
}

}  // extern "C"
