// api_swap.cpp -- swap API (swap_out / swap_in; readings R9, R10)
// and the pack / unpack building blocks (A4 / A6, aggregation P:549-550).
//
// Swap moves aggregated blocks between the HBM pool and pinned host DRAM over
// PCIe: the migration kernel's SM loads/stores address the mapped pinned
// DRAM pool directly (zero-copy), so one launch gathers every victim's 2*L
// scattered chunks into its contiguous DRAM block (or scatters back).
#include <algorithm>
#include <cstring>

#include "pool.hpp"

using namespace mp;

namespace {
// Default transport: pack into device staging + copy-engine D2H/H2D
// (measured 54.5 / 52.9 GB/s on B200 = 0.95 of a pinned memcpy, vs 52.6 /
// 51.3 for zero-copy SM stores/loads, profiles/sweep_r01_swap2.json) when the
// staging buffer holds a block; MP_SWAP_ZERO_COPY forces the SM path.
bool use_ce(const mp_pool* p, uint32_t flags) {
  if (flags & MP_SWAP_ZERO_COPY) return false;
  if (flags & MP_SWAP_CE) return true;
  return p->staging_bytes >= p->Pb;
}
}  // namespace

extern "C" {

mp_status mp_swap_out(mp_pool* p, int64_t n, uint32_t flags, mp_addr* out_old, mp_addr* out_new,
                      int64_t* n_moved) {
  if (!p || n < 0 || (n > 0 && (!out_old || !out_new))) return MP_ERR_CONFIG;
  TRY(remote_flush_tx(p));  // a pipelined copy goes first
  DevGuard g(p->dev);
  TRY(flush_involving(p));  // victims may still be the target of a coalesced copy
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
    free_block(p, MP_HBM, h);  // device bitmap update is queued behind the copy
    pairs.push_back({h, d});
  }
  if (pairs.empty() && no_dram) return MP_ERR_NO_DRAM;
  // Copy list: the last pair that wrote each DRAM block still allocated (R9).
  std::vector<int32_t> hs, ds;
  std::set<int32_t> done;
  for (auto it = pairs.rbegin(); it != pairs.rend(); ++it) {
    if (done.count(it->second) || p->st[MP_DRAM][(size_t)it->second] == ST_FREE) continue;
    done.insert(it->second);
    hs.push_back(it->first);
    ds.push_back(it->second);
  }
  if (!hs.empty() && use_ce(p, flags)) {
    // pack into device staging (aggregated), then copy-engine D2H
    // (one copy per run of consecutive DRAM blocks) on the copy stream; the
    // two halves of the staging alternate so the next pack overlaps the
    // current D2H.  The victims stay allocated on the device bitmap until the
    // queued frees are flushed behind these copies (sync below).
    if (p->staging_bytes < p->Pb) {
      set_err("staging smaller than one block");
      return MP_ERR_CONFIG;
    }
    const int64_t per = p->staging_bytes / p->Pb;
    const int halves = per >= 2 ? 2 : 1;
    const int64_t k = per / halves;
    TRY(meta_fence(p));
    TRY(staging_acquire(p, p->stream));  // STAGED transfers may still use the staging
    for (size_t b0 = 0, r = 0; b0 < hs.size(); b0 += (size_t)k, ++r) {
      const size_t nb = std::min(hs.size() - b0, (size_t)k);
      const int h = (int)(r % (size_t)halves);
      char* stg = p->staging + (int64_t)h * k * p->Pb;
      if (r >= (size_t)halves) CK(cudaStreamWaitEvent(p->stream, p->swap_ev[2 + h], 0));
      int* dh = nullptr;
      mpk::InlineIds si;
      TRY(src_ids(p, std::vector<int32_t>(hs.begin() + b0, hs.begin() + b0 + nb), &dh, &si));
      TRY(launch_migrate_timed(p, p->stream, pool_ep(p->d_slabs, dh), agg_ep(stg, p->Pb, nullptr),
                               (int64_t)nb, 0, p->nch, false, 0, si.n ? &si : nullptr));
      CK(cudaEventRecord(p->swap_ev[h], p->stream));
      CK(cudaStreamWaitEvent(p->copy_stream, p->swap_ev[h], 0));
      for (size_t i = 0; i < nb;) {
        size_t j = i + 1;
        while (j < nb && ds[b0 + j] == ds[b0 + j - 1] + 1) ++j;
        CK(cudaMemcpyAsync(p->dram + (int64_t)ds[b0 + i] * p->Pb, stg + (int64_t)i * p->Pb,
                           (size_t)p->Pb * (j - i), cudaMemcpyDeviceToHost, p->copy_stream));
        i = j;
      }
      CK(cudaEventRecord(p->swap_ev[2 + h], p->copy_stream));
    }
    CK(cudaEventRecord(p->swap_ev[0], p->copy_stream));   // join: the data stream
    CK(cudaStreamWaitEvent(p->stream, p->swap_ev[0], 0));  // waits for every D2H
  } else if (!hs.empty()) {
    int *dh = nullptr, *dd = nullptr;
    TRY(upload_ids(p, hs, &dh));
    TRY(upload_ids(p, ds, &dd));
    // launched before the queued frees are flushed (sync below), so the
    // bitmap releases the victims only after the copy has read them
    TRY(launch_migrate_timed(p, p->stream, pool_ep(p->d_slabs, dh),
                             agg_ep(p->dram_dev, p->Pb, dd), (int64_t)hs.size(), 0, p->nch));
  }
  TRY(sync(p));
  p->stats.blocks_moved += hs.size();
  for (size_t i = 0; i < pairs.size(); ++i) {
    out_old[i] = enc(p, MP_HBM, pairs[i].first);
    out_new[i] = enc(p, MP_DRAM, pairs[i].second);
  }
  if (n_moved) *n_moved = (int64_t)pairs.size();
  return MP_OK;
}

mp_status mp_swap_in(mp_pool* p, const mp_addr* a, int64_t n, uint32_t flags, mp_addr* out) {
  if (!p || n < 0 || (n > 0 && (!a || !out))) return MP_ERR_CONFIG;
  TRY(remote_flush_tx(p));  // a pipelined copy goes first
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
  TRY(flush_involving(p));
  if (p->nfree[MP_HBM] < n) evict_internal(p, n - p->nfree[MP_HBM], MP_HBM, nullptr);
  std::vector<int32_t> hids;
  int *dh = nullptr, *dd = nullptr;
  TRY(alloc_hbm(p, n, p->inst, &hids, &dh));
  if (use_ce(p, flags)) {
    // copy-engine H2D per block into device staging, then unpack
    if (p->staging_bytes < p->Pb) {
      set_err("staging smaller than one block");
      return MP_ERR_CONFIG;
    }
    // H2D (one copy per run of consecutive DRAM blocks) into one half of the
    // staging on the copy stream while the data stream unpacks the other
    const int64_t per = p->staging_bytes / p->Pb;
    const int halves = per >= 2 ? 2 : 1;
    const int64_t k = per / halves;
    TRY(meta_fence(p));   // the allocation above (dh) is on the meta stream
    TRY(staging_acquire(p, p->copy_stream));  // STAGED transfers may still use the staging
    CK(cudaEventRecord(p->swap_ev[0], p->stream));         // everything earlier on
    CK(cudaStreamWaitEvent(p->copy_stream, p->swap_ev[0], 0));  // the pool goes first
    for (int64_t b0 = 0, r = 0; b0 < n; b0 += k, ++r) {
      const int64_t nb = std::min(n - b0, k);
      const int h = (int)(r % halves);
      char* stg = p->staging + (int64_t)h * k * p->Pb;
      if (r >= halves) CK(cudaStreamWaitEvent(p->copy_stream, p->swap_ev[2 + h], 0));
      for (int64_t i = 0; i < nb;) {
        int64_t j = i + 1;
        while (j < nb && dids[(size_t)(b0 + j)] == dids[(size_t)(b0 + j - 1)] + 1) ++j;
        CK(cudaMemcpyAsync(stg + i * p->Pb, p->dram + (int64_t)dids[(size_t)(b0 + i)] * p->Pb,
                           (size_t)p->Pb * (size_t)(j - i), cudaMemcpyHostToDevice,
                           p->copy_stream));
        i = j;
      }
      CK(cudaEventRecord(p->swap_ev[h], p->copy_stream));
      CK(cudaStreamWaitEvent(p->stream, p->swap_ev[h], 0));
      TRY(launch_migrate_timed(p, p->stream, agg_ep(stg, p->Pb, nullptr),
                               pool_ep(p->d_slabs, dh + b0), nb, 0, p->nch));
      CK(cudaEventRecord(p->swap_ev[2 + h], p->stream));
    }
  } else {
    TRY(upload_ids(p, dids, &dd));
    TRY(launch_migrate_timed(p, p->stream, agg_ep(p->dram_dev, p->Pb, dd),
                             pool_ep(p->d_slabs, dh), n, 0, p->nch));
  }
  TRY(sync(p));
  p->stats.blocks_moved += (uint64_t)n;
  for (int64_t i = 0; i < n; ++i) {
    const int32_t d = dids[(size_t)i], h = hids[(size_t)i];
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

static mp_status pack_unpack(mp_pool* p, const mp_addr* a, int64_t n, int32_t l0, int32_t l1,
                             void* staging, bool pack) {
  if (!p || n < 0 || (n > 0 && (!a || !staging)) || !(0 <= l0 && l0 < l1 && l1 <= p->L))
    return MP_ERR_CONFIG;
  std::vector<int32_t> ids((size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    int m = 0;
    int32_t idx = 0;
    if (!decode(p, a[i], &m, &idx)) return MP_ERR_INVALID_ADDR;
    if (m != MP_HBM) return MP_ERR_PRECONDITION;
    const uint8_t s = p->st[MP_HBM][(size_t)idx];
    if (s == ST_FREE || (!pack && s != ST_ACTIVE)) return MP_ERR_PRECONDITION;
    ids[(size_t)i] = idx;
  }
  DevGuard g(p->dev);
  TRY(flush_involving(p));
  int* d = nullptr;
  TRY(upload_ids(p, ids, &d));
  const int nj = 2 * (l1 - l0);
  const long long stride = (long long)nj * p->chunk;
  if (pack)
    TRY(launch_migrate_timed(p, p->stream, pool_ep(p->d_slabs, d),
                             agg_ep((char*)staging, stride, nullptr), n, 2 * l0, nj));
  else
    TRY(launch_migrate_timed(p, p->stream, agg_ep((char*)staging, stride, nullptr),
                             pool_ep(p->d_slabs, d), n, 2 * l0, nj));
  return sync(p);
}

mp_status mp_pack(mp_pool* p, const mp_addr* a, int64_t n, int32_t l0, int32_t l1,
                  void* staging) {
  if (p) TRY(remote_flush_tx(p));
  return pack_unpack(p, a, n, l0, l1, staging, true);
}

mp_status mp_unpack(mp_pool* p, const void* staging, const mp_addr* a, int64_t n, int32_t l0,
                    int32_t l1) {
  if (p) TRY(remote_flush_tx(p));
  return pack_unpack(p, a, n, l0, l1, const_cast<void*>(staging), false);
}

// ------------------------------------------------------------ debug / test
mp_status mp_debug_fill(mp_pool* p, const mp_addr* a, int64_t n, uint64_t seed) {
  if (!p || n < 0 || (n > 0 && !a)) return MP_ERR_CONFIG;
  TRY(remote_flush_tx(p));  // a pipelined copy goes first
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
  TRY(flush_involving(p));  // a pending coalesced copy must read / write the old content
  ++p->epoch;
  int* d = nullptr;
  TRY(upload_ids(p, ids, &d));
  TRY(remote_apply_waits(p));
  TRY(meta_fence(p));
  CK(mpk::launch_fill(p->d_slabs, d, (int)n, p->nch, p->chunk, seed, (uint64_t)p->inst, p->epoch,
                      p->stream));
  track_fence(p->track);
  p->stats.aux_launches += 1;
  return sync(p);
}

mp_status mp_debug_read_block(mp_pool* p, mp_addr a, void* host_out, int64_t cap) {
  int m = 0;
  int32_t idx = 0;
  if (!p || !host_out) return MP_ERR_CONFIG;
  TRY(remote_flush_tx(p));  // a pipelined copy goes first
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
  TRY(remote_flush_tx(p));  // a pipelined copy goes first
  DevGuard g(p->dev);
  TRY(sync(p));
  CK(cudaMemcpy(out, p->d_bitmap, sizeof(uint32_t) * p->nwords, cudaMemcpyDeviceToHost));
  return MP_OK;
}

}  // extern "C"
