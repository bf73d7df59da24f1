// api_transfer.cpp -- distributed API of MemPool: transfer and
// transfer_with_insert (Table tbl-mempool-api; workflow P:360-365:
// allocation at the receiver, transmission, insertion, ok), the private-field
// delivery and the three transports of the transmission step:
//   FUSED  (A6f) one gather->store kernel from the source pool's scattered
//          chunks straight into the destination blocks (P2P stores over NVLink
//          when the pools are on different GPUs); no staging, 2*Pb HBM bytes
//          per block at loopback;
//   STAGED (A4-A6) pack into aggregated staging slots, one
//          contiguous copy per slot, unpack; a ring of slots overlaps the three;
//   CE     one copy-engine memcpy per (block, layer, K/V) chunk: the paper's
//          discrete per-block transfer, kept as a library baseline.
// The receiver's half (allocation, insertion) is dst_prepare_* / dst_commit,
// called directly for an in-process peer and from the mailbox server
// (remote.cpp) for a peer in another process.
// Readings R3, R4, R12, R13.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>

#include "pool.hpp"

namespace mp {
namespace {

// Host-time breakdown of mp_transfer_with_insert (MP_HOST_TIMING=1 prints it
// when a pool is destroyed): [0] source validation, [1] receiver allocation
// step (match, pin, allocation kernel), [2] transmission (batch append or
// launch), [3] receiver insertion + delivery, [4] completion (sync unless ASYNC).
struct HostPhases {
  double t[10] = {};
  uint64_t n = 0, m[10] = {};
};
thread_local HostPhases g_host;
bool host_timing_on_impl() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("MP_HOST_TIMING");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  return on == 1;
}
double host_now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

}  // namespace

bool host_timing_on() { return host_timing_on_impl(); }
double host_clock() { return host_now(); }
void host_lap(int slot, double dt) {
  g_host.t[slot] += dt;
  ++g_host.m[slot];
}

void host_report_timing() {
  if (!host_timing_on() || g_host.n == 0) return;
  const char* names[10] = {"validate_src", "dst_prepare", "transmit", "dst_commit", "finish",
                           "append:preflush", "append:ids", "append:query", "append:flush",
                           "flush_batch"};
  for (int i = 0; i < 5; ++i)
    fprintf(stderr, "[mempool host] twi %-16s %8llu calls %8.2f us avg\n", names[i],
            (unsigned long long)g_host.n, g_host.t[i] / (double)g_host.n * 1e6);
  for (int i = 5; i < 10; ++i)
    if (g_host.m[i])
      fprintf(stderr, "[mempool host]     %-16s %8llu calls %8.2f us avg\n", names[i],
              (unsigned long long)g_host.m[i], g_host.t[i] / (double)g_host.m[i] * 1e6);
  g_host = HostPhases{};
}

namespace {

// R13 (memory asymmetry): a source block may be in HBM or, swapped
// out, in the source's pinned DRAM; allocated, listed once.
mp_status validate_src(mp_pool* src, const mp_addr* a, int64_t n, std::vector<int32_t>* ids,
                       std::vector<uint8_t>* meds) {
  ids->resize((size_t)n);
  meds->resize((size_t)n);
  const uint32_t g = next_mark(src);
  for (int64_t i = 0; i < n; ++i) {
    int m = 0;
    int32_t idx = 0;
    if (!decode(src, a[i], &m, &idx)) return MP_ERR_INVALID_ADDR;
    const uint8_t s = src->st[m][(size_t)idx];
    uint32_t& mk = src->mark[m][(size_t)idx];
    if (!(s == ST_ACTIVE || s == ST_INDEXED) || mk == g) return MP_ERR_PRECONDITION;
    mk = g;
    (*ids)[(size_t)i] = idx;
    (*meds)[(size_t)i] = (uint8_t)m;
  }
  return MP_OK;
}

mp_status validate_dst_given(mp_pool* dst, const mp_addr* a, int64_t n,
                             std::vector<int32_t>* ids) {
  if (!a) return MP_ERR_ADDR_COUNT;
  ids->resize((size_t)n);
  const uint32_t g = next_mark(dst);
  for (int64_t i = 0; i < n; ++i) {
    int m = 0;
    int32_t idx = 0;
    if (!decode(dst, a[i], &m, &idx)) return MP_ERR_INVALID_ADDR;
    if (m != MP_HBM || dst->st[MP_HBM][(size_t)idx] != ST_ACTIVE ||
        dst->mark[MP_HBM][(size_t)idx] == g)
      return MP_ERR_PRECONDITION;
    dst->mark[MP_HBM][(size_t)idx] = g;
    (*ids)[(size_t)i] = idx;
  }
  return MP_OK;
}

mp_status check_compatible(mp_pool* src, mp_pool* dst) {
  if (dst == src || src->L != dst->L || src->chunk != dst->chunk || src->B != dst->B)
    return MP_ERR_CONFIG;
  return MP_OK;
}

mp_pool* peer_of(mp_pool* src, int32_t inst) {
  auto it = src->peers.find(inst);
  return it == src->peers.end() ? nullptr : it->second;
}

RemotePeer* remote_of(mp_pool* src, int32_t inst) {
  auto it = src->remotes.find(inst);
  return it == src->remotes.end() ? nullptr : it->second;
}

// The transmission step for HBM-resident sources (in-process peers).  Copies
// chunks [j0, j0+nj) of source blocks `sids` into destination blocks `dids`;
// d_dst is the destination allocator's device table of the same ids (on
// dst's device) or nullptr.  Enqueued after all earlier work of both pools and
// before their later work; STAGED completes before returning, the others are
// stream-ordered.

mp_status transmit_hbm(mp_pool* src, mp_pool* dst, const std::vector<int32_t>& sids,
                       const std::vector<int32_t>& dids, const int* d_dst, int j0, int nj,
                       uint32_t path) {
  const int64_t n = (int64_t)sids.size();
  if (n == 0) return MP_OK;
  if (path == MP_XFER_PATH_AUTO) path = MP_XFER_PATH_FUSED;
  const bool same_dev = same_gpu(src, dst);
  if (path == MP_XFER_PATH_FUSED && same_dev && dst->coalesce) {
    DevGuard g(dst->dev);
    return batch_append(src, dst, sids, dids, d_dst, j0, nj);
  }
  // every other path launches now: pending coalesced copies touching either
  // pool go first
  TRY(flush_involving(src));
  TRY(flush_involving(dst));
  if (path == MP_XFER_PATH_FUSED && same_dev) {
    TRY(link(src, dst));
    DevGuard g(dst->dev);
    int* ds = nullptr;
    mpk::InlineIds si;
    const bool both = pair_inline(sids, dids, &si);  // no id table, no meta wait
    if (!both) TRY(src_ids(dst, sids, &ds, &si));
    const int* dd = d_dst;
    if (!dd && !both) {
      int* t = nullptr;
      TRY(upload_ids(dst, dids, &t));
      dd = t;
    }
    const LaunchBlocks lb{&src->bmarks, sids.data(), &dst->bmarks, dids.data(), n};
    TRY(launch_migrate_timed(dst, dst->stream, pool_ep(src->d_slabs, ds),
                             pool_ep(dst->d_slabs, both ? nullptr : dd), n, j0, nj, false, 0,
                             si.n ? &si : nullptr, /*meta_dep=*/!both, &lb));
    dst->stats.blocks_moved += (uint64_t)n;
    return link(dst, src);
  }
  if (path == MP_XFER_PATH_FUSED) {
    // Push over NVLink: the source GPU gathers its chunks and stores them
    // straight into the peer pool's blocks (no staging).
    auto it = src->peer_tables.find(dst->inst);
    if (it == src->peer_tables.end()) return MP_ERR_DST_UNREACHABLE;
    TRY(link(dst, src));
    DevGuard g(src->dev);
    int *ds = nullptr, *dd = nullptr;
    mpk::InlineIds si;
    const bool both = pair_inline(sids, dids, &si);
    if (!both) {
      TRY(src_ids(src, sids, &ds, &si));
      TRY(upload_ids(src, dids, &dd));
    }
    const LaunchBlocks lb{&src->bmarks, sids.data(), &dst->bmarks, dids.data(), n};
    TRY(launch_migrate_timed(src, src->stream, pool_ep(src->d_slabs, ds),
                             pool_ep(it->second, dd), n, j0, nj, /*peer=*/true, 0,
                             si.n ? &si : nullptr, /*meta_dep=*/!both, &lb));
    src->stats.blocks_moved += (uint64_t)n;
    return link(src, dst);
  }
  if (path == MP_XFER_PATH_CE) {
    TRY(link(dst, src));
    DevGuard g(src->dev);
    for (int64_t i = 0; i < n; ++i)
      for (int j = j0; j < j0 + nj; ++j)
        CK(cudaMemcpyAsync(dst->slabs[(size_t)j] + (int64_t)dids[(size_t)i] * dst->chunk,
                           src->slabs[(size_t)j] + (int64_t)sids[(size_t)i] * src->chunk,
                           (size_t)src->chunk, cudaMemcpyDefault, src->stream));
    track_fence(src->track);  // copies the launch window knows nothing about
    src->stats.bytes_moved += (uint64_t)(n * nj * src->chunk);
    src->stats.blocks_moved += (uint64_t)n;
    return link(src, dst);
  }
  if (path == MP_XFER_PATH_STAGED) {
    const int64_t per_block = (int64_t)nj * src->chunk;
    const int S = std::max(1, std::min(src->staging_slots, dst->staging_slots));
    const int64_t slot_bytes = std::min(src->staging_bytes, dst->staging_bytes) / S;
    const int64_t k = slot_bytes / per_block;
    if (k <= 0) {
      set_err("staging slot smaller than one block");
      return MP_ERR_CONFIG;
    }
    TRY(link(dst, src));
    int *ds = nullptr, *dd = nullptr;
    {
      DevGuard g(src->dev);
      TRY(upload_ids(src, sids, &ds));
    }
    {
      DevGuard g(dst->dev);
      if (d_dst) {
        dd = const_cast<int*>(d_dst);
      } else {
        TRY(upload_ids(dst, dids, &dd));
      }
    }
    // Stream-ordered, no host wait: the pack of slot r on the source's data
    // stream, the copy-engine copy on its copy stream, the unpack on the
    // destination's data stream, chained by events; a slot is refilled once
    // the copy out of it (source side) and the unpack out of it
    // (destination side) are done, and every earlier user of either staging
    // buffer (other transfers, swap) goes first (staging_acquire).
    {
      DevGuard g(src->dev);
      TRY(staging_acquire(src, src->stream));
      TRY(staging_acquire(dst, src->copy_stream));
    }
    const int64_t nslots = (n + k - 1) / k;
    for (int64_t s = 0; s < nslots; ++s) {
      const int r = (int)(s % S);
      const int64_t b0 = s * k, nb = std::min(k, n - b0);
      char* sslot = src->staging + r * slot_bytes;
      char* dslot = dst->staging + r * slot_bytes;
      {
        DevGuard g(src->dev);
        if (s >= S) CK(cudaStreamWaitEvent(src->stream, src->slot_ev[(size_t)r], 0));
        TRY(launch_migrate_timed(src, src->stream, pool_ep(src->d_slabs, ds + b0),
                                 agg_ep(sslot, per_block, nullptr), nb, j0, nj));
        CK(cudaEventRecord(src->pack_ev[(size_t)r], src->stream));
        CK(cudaStreamWaitEvent(src->copy_stream, src->pack_ev[(size_t)r], 0));
        if (s >= S) CK(cudaStreamWaitEvent(src->copy_stream, dst->slot_ev[(size_t)r], 0));
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
    src->stats.blocks_moved += (uint64_t)n;
    return MP_OK;
  }
  set_err("unknown transfer path");
  return MP_ERR_CONFIG;
}

// Sources swapped out to the source's pinned DRAM (memory asymmetry,
// "the fastest link with the least data copies"): the DRAM block
// is already aggregated, so its chunks cross PCIe once and are
// scattered straight into the destination blocks -- no swap_in, no index
// rewrite on the source.  Default: the copy engine moves them into the
// source's staging and a kernel scatters each slot (dram_ce_scatter, ~55
// GB/s); without staging room, or with MP_DRAM_SOURCE=sm, one kernel reads
// the mapped DRAM directly (~51 GB/s).  Runs on the destination's GPU when
// both pools share it, else on the source's GPU storing over NVLink.
mp_status transmit_dram(mp_pool* src, mp_pool* dst, const std::vector<int32_t>& sids,
                        const std::vector<int32_t>& dids, int j0, int nj) {
  const int64_t n = (int64_t)sids.size();
  if (n == 0) return MP_OK;
  TRY(flush_involving(src));
  TRY(flush_involving(dst));
  // aggregated block layout [2L][c]: shift the base to chunk j0
  char* base = src->dram_dev + (int64_t)j0 * src->chunk;
  const bool same_dev = same_gpu(src, dst);
  mp_pool* ex = same_dev ? dst : src;
  if (same_dev)
    TRY(link(src, dst));
  else
    TRY(link(dst, src));
  {
    DevGuard g(ex->dev);
    char** dslabs = dst->d_slabs;
    if (!same_dev) {
      auto it = src->peer_tables.find(dst->inst);
      if (it == src->peer_tables.end()) return MP_ERR_DST_UNREACHABLE;
      dslabs = it->second;
    }
    if (dram_source_ce(src, nj)) {
      TRY(dram_ce_scatter(src, ex, ex->stream, dslabs, sids, dids, j0, nj, !same_dev));
    } else {
      int *ds = nullptr, *dd = nullptr;
      mpk::InlineIds si;
      TRY(src_ids(ex, sids, &ds, &si));
      TRY(upload_ids(ex, dids, &dd));
      TRY(launch_migrate_timed(ex, ex->stream, agg_ep(base, src->Pb, ds), pool_ep(dslabs, dd),
                               n, j0, nj, /*peer=*/!same_dev, 0, si.n ? &si : nullptr));
    }
    ex->stats.blocks_moved += (uint64_t)n;
  }
  return same_dev ? link(dst, src) : link(src, dst);
}

// The transmission step: HBM-resident sources take the requested transport,
// DRAM-resident ones the direct DRAM -> destination kernel.
mp_status transmit(mp_pool* src, mp_pool* dst, const std::vector<int32_t>& sids,
                   const std::vector<uint8_t>& smeds, const std::vector<int32_t>& dids,
                   const int* d_dst, int j0, int nj, uint32_t path) {
  bool any_dram = false;
  for (uint8_t m : smeds) any_dram = any_dram || m == MP_DRAM;
  if (!any_dram) return transmit_hbm(src, dst, sids, dids, d_dst, j0, nj, path);
  std::vector<int32_t> hs, hd, ds, dd;
  for (size_t i = 0; i < sids.size(); ++i) {
    (smeds[i] == MP_DRAM ? ds : hs).push_back(sids[i]);
    (smeds[i] == MP_DRAM ? dd : hd).push_back(dids[i]);
  }
  // a mixed list no longer matches the allocator's device table order: the
  // two parts upload their destination ids
  if (!hs.empty()) TRY(transmit_hbm(src, dst, hs, hd, nullptr, j0, nj, path));
  return transmit_dram(src, dst, ds, dd, j0, nj);
}

// A transfer transmit_hbm will append to dst's coalescing batch: let the
// receiver's allocation write its ids straight into the batch table.
void hint_slot(mp_pool* src, mp_pool* dst, uint32_t flags, const std::vector<uint8_t>& smeds,
               int j0, int nj) {
  const uint32_t path = flags & MP_XFER_PATH_MASK;
  if (!(path == MP_XFER_PATH_AUTO || path == MP_XFER_PATH_FUSED) || !same_gpu(src, dst) ||
      !dst->coalesce || (flags & MP_XFER_DST_GIVEN))
    return;
  for (uint8_t m : smeds)
    if (m != MP_HBM) return;
  dst->slot_hint.src = src;
  dst->slot_hint.j0 = j0;
  dst->slot_hint.nj = nj;
}

// A synchronous transfer returns once the work it issued has completed: its
// launches (flushed here if still batched) and the receiver's allocation.
// Bitmap updates still queued from earlier frees are not part of it and
// stay queued (applying them here cost a kernel and a wait per call).
mp_status finish(mp_pool* src, mp_pool* dst, uint32_t flags) {
  if (flags & MP_XFER_ASYNC) return MP_OK;
  TRY(flush_involving(dst));
  TRY(flush_involving(src));
  {
    DevGuard g(dst->dev);
    TRY(drain(dst));
  }
  DevGuard g(src->dev);
  return drain(src);
}

void stash_priv(DstPrep* st, const void* priv, int64_t priv_len) {
  st->priv.clear();
  if (priv_len > 0) st->priv.assign((const uint8_t*)priv, (const uint8_t*)priv + priv_len);
}

}  // namespace

// ------------------------------------------------- receiver: allocation step
mp_status dst_prepare_xfer(mp_pool* dst, int32_t src_inst, int64_t n, uint32_t flags,
                           const mp_addr* given, const void* priv, int64_t priv_len,
                           DstPrep* st, bool host_ids) {
  *st = DstPrep{};
  st->kind = 0;
  st->src_inst = src_inst;
  st->flags = flags;
  st->nm = n;
  const bool dst_given = (flags & MP_XFER_DST_GIVEN) != 0;
  if (dst_given) TRY(validate_dst_given(dst, given, n, &st->dids));
  const std::vector<mpi::Node*> none;
  if (!dst_given && !can_make_room(dst, n, MP_HBM, none)) return MP_ERR_DST_OOM;
  stash_priv(st, priv, priv_len);
  if (!dst_given) {
    DevGuard g(dst->dev);
    if (dst->nfree[MP_HBM] < n) evict_internal(dst, n - dst->nfree[MP_HBM], MP_HBM, nullptr);
    TRY(alloc_hbm(dst, n, src_inst, &st->dids, &st->d_dst, host_ids));
  }
  return MP_OK;
}

mp_status dst_prepare_twi(mp_pool* dst, int32_t src_inst, const mp_token* toks, int64_t n_tok,
                          int64_t m, uint32_t flags, const mp_addr* given, const void* priv,
                          int64_t priv_len, DstPrep* st, bool host_ids) {
  *st = DstPrep{};
  st->kind = 1;
  st->src_inst = src_inst;
  st->flags = flags;
  const bool dst_given = (flags & MP_XFER_DST_GIVEN) != 0;
  const bool dedup = (flags & MP_XFER_DEDUP) != 0;
  const int64_t B = dst->B;
  st->n_tok = n_tok;
  st->ceil_b = (n_tok + B - 1) / B;
  st->floor_b = n_tok / B;
  std::vector<int32_t> given_ids;
  if (dst_given) TRY(validate_dst_given(dst, given, m, &given_ids));
  st->q = st->ceil_b - m;
  const bool need_match = dedup || st->q > 0;
  std::vector<mpi::Node*> peek;
  if (need_match) peek = dst->index->path(toks, st->floor_b);
  const int64_t k_match = (int64_t)peek.size();
  if (k_match < st->q) return MP_ERR_PREFIX_MISSING;
  st->skip = dedup ? k_match - st->q : 0;
  st->nm = m - st->skip;
  if (flags & MP_INS_ERR_ON_CONFLICT) {
    const int64_t k_exist = need_match ? k_match : dst->index->peek(toks, n_tok);
    if (k_exist > st->q + st->skip) return MP_ERR_CONFLICT;
  }
  if (!dst_given && !can_make_room(dst, st->nm, MP_HBM, peek)) return MP_ERR_DST_OOM;
  // ---- mutations start here ----
  st->toks.assign(toks, toks + n_tok);
  stash_priv(st, priv, priv_len);
  // receiver-side match (the path walked above), pinned while the receiver
  // allocates (R3, R12)
  if (need_match) {
    dst->index->touch_path(peek, /*pin=*/true);
    st->matched = std::move(peek);
  }
  if (dst_given) {
    st->dids = given_ids;
  } else {
    DevGuard g(dst->dev);
    if (dst->nfree[MP_HBM] < st->nm)
      evict_internal(dst, st->nm - dst->nfree[MP_HBM], MP_HBM, nullptr);
    TRY(alloc_hbm(dst, st->nm, src_inst, &st->dids, &st->d_dst, host_ids));
  }
  return MP_OK;
}

mp_status transmit_precheck(mp_pool* src, mp_pool* dst, uint32_t path, int nj,
                            const std::vector<uint8_t>& smeds) {
  switch (path) {
    case MP_XFER_PATH_AUTO:
    case MP_XFER_PATH_FUSED:
    case MP_XFER_PATH_CE:
      return MP_OK;
    case MP_XFER_PATH_STAGED: {
      bool any_hbm = false;  // DRAM sources take the direct DRAM kernel, not the ring
      for (uint8_t m : smeds) any_hbm = any_hbm || m == MP_HBM;
      if (!any_hbm) return MP_OK;
      const int S = std::max(1, std::min(src->staging_slots, dst->staging_slots));
      const int64_t slot_bytes = std::min(src->staging_bytes, dst->staging_bytes) / S;
      if (slot_bytes < (int64_t)nj * src->chunk) {
        set_err("staging slot smaller than one block");
        return MP_ERR_CONFIG;
      }
      return MP_OK;
    }
    default:
      set_err("unknown transfer path");
      return MP_ERR_CONFIG;
  }
}

void dst_abort(mp_pool* dst, DstPrep& st) {
  unpin_nodes(dst, st.matched);
  st.matched.clear();
  if (!(st.flags & MP_XFER_DST_GIVEN))
    for (int32_t id : st.dids) free_block(dst, MP_HBM, id);
  st.dids.clear();
}

// ------------------------------------------------- receiver: insertion step
mp_status dst_commit(mp_pool* dst, DstPrep& st, mp_addr* final_out) {
  Msg msg{st.kind, st.src_inst, {}, {}};
  msg.priv.swap(st.priv);
  if (st.kind == 0) {
    for (int64_t i = 0; i < st.nm; ++i) final_out[i] = enc(dst, MP_HBM, st.dids[(size_t)i]);
    msg.addrs.assign(final_out, final_out + st.nm);
    dst->inbox.push_back(std::move(msg));
    return MP_OK;
  }
  std::vector<mp_addr> full;
  full.reserve((size_t)st.ceil_b);
  for (int64_t i = 0; i < st.q + st.skip; ++i)
    full.push_back(enc(dst, st.matched[(size_t)i]->medium, st.matched[(size_t)i]->idx));
  for (int64_t i = 0; i < st.nm; ++i) full.push_back(enc(dst, MP_HBM, st.dids[(size_t)i]));
  int64_t dup = 0;
  std::vector<mpi::Node*> fin;  // the index nodes of prefixes 1..floor_b afterwards
  TRY(insert_internal(dst, st.toks.data(), st.n_tok, full.data(), (int64_t)full.size(),
                      st.flags & MP_INS_ERR_ON_CONFLICT, &dup, &st.matched, &fin));
  unpin_nodes(dst, st.matched);
  st.matched.clear();
  for (int64_t i = 0; i < st.floor_b; ++i)
    final_out[i] = enc(dst, fin[(size_t)i]->medium, fin[(size_t)i]->idx);
  if (st.ceil_b > st.floor_b) final_out[st.floor_b] = full[(size_t)st.floor_b];
  msg.addrs.assign(final_out, final_out + st.ceil_b);
  dst->inbox.push_back(std::move(msg));
  return MP_OK;
}

}  // namespace mp

using namespace mp;

extern "C" {

mp_status mp_transfer(mp_pool* src, int32_t dst_inst, const mp_addr* sa, int64_t n, mp_addr* da,
                      uint32_t flags, int32_t l0, int32_t l1, const void* priv, int64_t priv_len) {
  if (!src || n < 0 || (n > 0 && (!sa || !da)) || priv_len < 0 || (priv_len > 0 && !priv))
    return MP_ERR_CONFIG;
  mp_pool* dst = peer_of(src, dst_inst);
  RemotePeer* rp = dst ? nullptr : remote_of(src, dst_inst);
  if (!dst && !rp) return MP_ERR_DST_UNREACHABLE;
  if (dst) {
    TRY(check_compatible(src, dst));
    TRY(remote_flush_tx(src));  // pipelined cross-process copies of either pool go first
    TRY(remote_flush_tx(dst));
  }
  if (!(0 <= l0 && l0 < l1 && l1 <= src->L) || (flags & MP_XFER_DEDUP)) return MP_ERR_CONFIG;
  std::vector<int32_t> sids;
  std::vector<uint8_t> smeds;
  TRY(validate_src(src, sa, n, &sids, &smeds));
  if (rp)
    return remote_transfer(src, rp, 0, nullptr, 0, sids, smeds, n, da, flags, l0, l1, priv,
                           priv_len, nullptr);
  TRY(transmit_precheck(src, dst, flags & MP_XFER_PATH_MASK, 2 * (l1 - l0), smeds));
  // ---- (1) allocation at the receiver ----
  DstPrep st;
  hint_slot(src, dst, flags, smeds, 2 * l0, 2 * (l1 - l0));
  const mp_status ps = dst_prepare_xfer(dst, src->inst, n, flags, da, priv, priv_len, &st);
  dst->slot_hint.src = nullptr;
  TRY(ps);
  // ---- (2) transmission ----
  const mp_status xs = transmit(src, dst, sids, smeds, st.dids, st.d_dst, 2 * l0,
                                2 * (l1 - l0), flags & MP_XFER_PATH_MASK);
  if (xs != MP_OK) {
    dst_abort(dst, st);
    return xs;
  }
  // ---- (3) completion ----
  TRY(dst_commit(dst, st, da));
  return finish(src, dst, flags);
}

mp_status mp_transfer_with_insert(mp_pool* src, int32_t dst_inst, const mp_token* toks,
                                  int64_t n_tok, const mp_addr* sa, int64_t m, mp_addr* da,
                                  uint32_t flags, const void* priv, int64_t priv_len,
                                  int64_t* n_moved) {
  if (!src || n_tok < 0 || (n_tok > 0 && !toks) || m < 0 || (m > 0 && !sa) || !da ||
      priv_len < 0 || (priv_len > 0 && !priv))
    return MP_ERR_CONFIG;
  mp_pool* dst = peer_of(src, dst_inst);
  RemotePeer* rp = dst ? nullptr : remote_of(src, dst_inst);
  if (!dst && !rp) return MP_ERR_DST_UNREACHABLE;
  if (dst) {
    TRY(check_compatible(src, dst));
    TRY(remote_flush_tx(src));  // pipelined cross-process copies of either pool go first
    TRY(remote_flush_tx(dst));
  }
  if ((flags & MP_XFER_DST_GIVEN) && (flags & MP_XFER_DEDUP)) return MP_ERR_CONFIG;
  const int64_t B = src->B, ceil_b = (n_tok + B - 1) / B;
  if (m > ceil_b) return MP_ERR_ADDR_COUNT;
  const bool tm = host_timing_on_impl();
  double t0 = tm ? host_now() : 0.0;
  auto lap = [&](int i) {
    if (!tm) return;
    const double t = host_now();
    g_host.t[i] += t - t0;
    t0 = t;
  };
  std::vector<int32_t> sids;
  std::vector<uint8_t> smeds;
  TRY(validate_src(src, sa, m, &sids, &smeds));
  if (rp)
    return remote_transfer(src, rp, 1, toks, n_tok, sids, smeds, m, da, flags, 0, src->L, priv,
                           priv_len, n_moved);
  TRY(transmit_precheck(src, dst, flags & MP_XFER_PATH_MASK, src->nch, smeds));
  lap(0);
  // ---- (1) allocation at the receiver, with its DEDUP match ----
  DstPrep st;
  hint_slot(src, dst, flags, smeds, 0, src->nch);
  const mp_status ps =
      dst_prepare_twi(dst, src->inst, toks, n_tok, m, flags, da, priv, priv_len, &st);
  dst->slot_hint.src = nullptr;
  TRY(ps);
  lap(1);
  // ---- (2) transmission of all layers ----
  std::vector<int32_t> moved_src(sids.begin() + st.skip, sids.end());
  std::vector<uint8_t> moved_med(smeds.begin() + st.skip, smeds.end());
  const mp_status xs = transmit(src, dst, moved_src, moved_med, st.dids, st.d_dst, 0, src->nch,
                                flags & MP_XFER_PATH_MASK);
  if (xs != MP_OK) {
    dst_abort(dst, st);
    return xs;
  }
  lap(2);
  // ---- (3) insertion at the receiver, ok ----
  TRY(dst_commit(dst, st, da));
  if (n_moved) *n_moved = st.nm;
  lap(3);
  const mp_status fs = finish(src, dst, flags);
  lap(4);
  if (tm) ++g_host.n;
  return fs;
}

// ---------------------------------------------------------------------------
// Asymmetric parallelism.  Chunks are head-major (R16),
// so heads [h0, h0+k) of a chunk are one contiguous byte range of k*B*D*elem
// bytes; a tensor-parallel repartition is a set of such sub-chunk copies
// between the shards of two instances, planned by mp_tp_plan.
mp_status mp_transfer_heads(mp_pool* src, int32_t dst_inst, const mp_addr* sa, int64_t n,
                            const mp_addr* da, uint32_t flags, int32_t src_head0,
                            int32_t dst_head0, int32_t n_heads, int32_t l0, int32_t l1) {
  if (!src || n < 0 || (n > 0 && (!sa || !da))) return MP_ERR_CONFIG;
  mp_pool* dst = peer_of(src, dst_inst);
  if (!dst) return remote_of(src, dst_inst) ? MP_ERR_CONFIG : MP_ERR_DST_UNREACHABLE;
  TRY(remote_flush_tx(src));
  TRY(remote_flush_tx(dst));
  if (src->L != dst->L || src->B != dst->B || src->D != dst->D || src->elem != dst->elem ||
      !(0 <= l0 && l0 < l1 && l1 <= src->L) || n_heads < 1 || src_head0 < 0 ||
      dst_head0 < 0 || src_head0 + n_heads > src->H || dst_head0 + n_heads > dst->H ||
      (flags & (MP_XFER_DEDUP | MP_XFER_PATH_MASK)))
    return MP_ERR_CONFIG;
  const int64_t head_bytes = (int64_t)src->B * src->D * src->elem;
  if (head_bytes % 16) {
    set_err("a head's bytes per chunk must be a multiple of 16");
    return MP_ERR_CONFIG;
  }
  std::vector<int32_t> sids, dids;
  std::vector<uint8_t> smeds;
  TRY(validate_src(src, sa, n, &sids, &smeds));
  for (uint8_t m : smeds)
    if (m != MP_HBM) return MP_ERR_PRECONDITION;
  TRY(validate_dst_given(dst, da, n, &dids));
  if (n == 0) return MP_OK;
  TRY(flush_involving(src));
  TRY(flush_involving(dst));
  const bool same_dev = same_gpu(src, dst);
  mp_pool* ex = same_dev ? dst : src;
  char** dslabs = dst->d_slabs;
  if (!same_dev) {
    auto it = src->peer_tables.find(dst->inst);
    if (it == src->peer_tables.end()) return MP_ERR_DST_UNREACHABLE;
    dslabs = it->second;
  }
  TRY(same_dev ? link(src, dst) : link(dst, src));
  {
    DevGuard g(ex->dev);
    int *ds = nullptr, *dd = nullptr;
    mpk::InlineIds si;
    TRY(src_ids(ex, sids, &ds, &si));
    TRY(upload_ids(ex, dids, &dd));
    const LaunchBlocks lb{&src->bmarks, sids.data(), &dst->bmarks, dids.data(), n};
    TRY(launch_migrate_timed(ex, ex->stream,
                             pool_ep(src->d_slabs, ds, src->chunk, src_head0 * head_bytes),
                             pool_ep(dslabs, dd, dst->chunk, dst_head0 * head_bytes), n, 2 * l0,
                             2 * (l1 - l0), /*peer=*/!same_dev, n_heads * head_bytes,
                             si.n ? &si : nullptr, true, &lb));
    ex->stats.blocks_moved += (uint64_t)n;
  }
  TRY(same_dev ? link(dst, src) : link(src, dst));
  return finish(src, dst, flags);
}

mp_status mp_tp_plan(int32_t H, int32_t p, int32_t q, int32_t* out, int64_t cap,
                     int64_t* n_pieces) {
  if (H < 1 || p < 1 || q < 1 || H % p || H % q) return MP_ERR_CONFIG;
  const int32_t hs = H / p, hd = H / q;
  int64_t k = 0;
  for (int32_t r = 0; r < p; ++r)
    for (int32_t s = 0; s < q; ++s) {
      const int32_t lo = std::max(r * hs, s * hd), hi = std::min((r + 1) * hs, (s + 1) * hd);
      if (lo >= hi) continue;
      if (out && k < cap) {
        int32_t* o = out + 5 * k;
        o[0] = r;
        o[1] = s;
        o[2] = lo - r * hs;
        o[3] = lo - s * hd;
        o[4] = hi - lo;
      }
      ++k;
    }
  if (n_pieces) *n_pieces = k;
  return (out && k > cap) ? MP_ERR_BUFFER_TOO_SMALL : MP_OK;
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

}  // extern "C"
