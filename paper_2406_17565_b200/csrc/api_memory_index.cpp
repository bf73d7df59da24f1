// api_memory_index.cpp -- memory API (alloc_mem / free_mem) and
// index API (insert / match / delete / evict) of MemPool.
// Readings R1, R2, R4-R8, R12, R14.
#include <algorithm>
#include <cstring>

#include "pool.hpp"

namespace mp {

uint32_t next_mark(mp_pool* p) {
  if (++p->mark_gen == 0) {  // wrapped: clear and restart
    for (auto& m : p->mark) std::fill(m.begin(), m.end(), 0u);
    p->mark_gen = 1;
  }
  return p->mark_gen;
}

// R4: keep-existing, free the caller's duplicate, trailing partial addr
// ignored, terminal marker on prefix_k.  Validates everything first.
// hint: nodes of prefixes 1..hint->size() walked earlier and still linked
// (the receiver's pinned match), so only the rest is looked up; out_nodes
// (nullable) receives the index nodes of prefixes 1..k afterwards.
mp_status insert_internal(mp_pool* p, const mp_token* toks, int64_t n_tok, const mp_addr* addrs,
                          int64_t n_addr, uint32_t flags, int64_t* n_dup,
                          const std::vector<mpi::Node*>* hint,
                          std::vector<mpi::Node*>* out_nodes) {
  const int64_t k = n_tok / p->B, c = (n_tok + p->B - 1) / p->B;
  if (n_tok < 0 || (n_addr != k && n_addr != c)) return MP_ERR_ADDR_COUNT;
  std::vector<mpi::Node*> path = hint ? p->index->path_hinted(*hint, hint->size(), toks, k)
                                      : p->index->path(toks, k);
  std::vector<int> med((size_t)k);
  std::vector<int32_t> idx((size_t)k);
  const uint32_t g = next_mark(p);
  for (int64_t i = 0; i < k; ++i) {
    if (!decode(p, addrs[i], &med[(size_t)i], &idx[(size_t)i])) return MP_ERR_INVALID_ADDR;
    uint32_t& mk = p->mark[med[(size_t)i]][(size_t)idx[(size_t)i]];
    if (mk == g) return MP_ERR_PRECONDITION;
    mk = g;
    mpi::Node* ex = i < (int64_t)path.size() ? path[(size_t)i] : nullptr;
    const uint8_t s = p->st[med[(size_t)i]][(size_t)idx[(size_t)i]];
    const bool same = ex && ex->medium == med[(size_t)i] && ex->idx == idx[(size_t)i];
    if (!(s == ST_ACTIVE || (s == ST_INDEXED && same))) return MP_ERR_PRECONDITION;
    if ((flags & MP_INS_ERR_ON_CONFLICT) && ex && !same) return MP_ERR_CONFLICT;
  }
  std::vector<mpi::Index::Placed> dups, added;
  std::vector<mpi::Node*> nodes =
      p->index->insert_seq(path, toks, k, med.data(), idx.data(), &dups, &added);
  for (const auto& a : added) p->st[a.medium][(size_t)a.idx] = ST_INDEXED;
  for (const auto& d : dups) free_block(p, d.medium, d.idx);
  if (out_nodes) out_nodes->swap(nodes);
  if (n_dup) *n_dup = (int64_t)dups.size();
  return MP_OK;
}

void unpin_nodes(mp_pool* p, const std::vector<mpi::Node*>& nodes) {
  for (mpi::Node* n : nodes) p->index->set_ref(n, n->ref - 1);
}

}  // namespace mp

using namespace mp;

extern "C" {

mp_status mp_alloc_mem(mp_pool* p, int64_t n, int32_t type, int32_t requester, mp_addr* out) {
  const bool stream_ordered = (type & MP_ALLOC_STREAM_ORDERED) != 0;
  type &= ~MP_ALLOC_STREAM_ORDERED;
  if (!p || n < 0 || (n > 0 && !out) || type < MP_HBM || type > MP_MIXED) return MP_ERR_CONFIG;
  TRY(remote_flush_tx(p));  // a pipelined copy goes first
  DevGuard g(p->dev);
  const std::vector<mpi::Node*> none;
  int64_t nh = 0, nd = 0;
  if (type == MP_HBM)
    nh = n;
  else if (type == MP_DRAM)
    nd = n;
  else {
    nh = std::min(n, p->nfree[MP_HBM]);
    nd = n - nh;
  }
  if (!can_make_room(p, nh, MP_HBM, none) || !can_make_room(p, nd, MP_DRAM, none))
    return MP_ERR_OOM;
  if (p->nfree[MP_HBM] < nh) evict_internal(p, nh - p->nfree[MP_HBM], MP_HBM, nullptr);
  if (p->nfree[MP_DRAM] < nd) evict_internal(p, nd - p->nfree[MP_DRAM], MP_DRAM, nullptr);
  std::vector<int32_t> ids;
  int* d = nullptr;
  // nothing on the device reads these ids: no allocation kernel, the device
  // bitmap learns the claim with its next update
  TRY(alloc_hbm(p, nh, requester, &ids, &d, /*defer=*/true));
  // The caller will write these blocks from its own streams: every earlier
  // device op of this pool (e.g. an async copy still reading a block that was
  // freed since) must be complete first -- unless the caller orders its
  // writes itself (MP_ALLOC_STREAM_ORDERED + mp_record_event).
  if (!stream_ordered) TRY(sync(p));
  for (int64_t i = 0; i < nh; ++i) out[i] = enc(p, MP_HBM, ids[(size_t)i]);
  std::vector<int32_t> dd = alloc_dram(p, nd, requester);
  for (int64_t i = 0; i < nd; ++i) out[nh + i] = enc(p, MP_DRAM, dd[(size_t)i]);
  return MP_OK;
}

mp_status mp_free_mem(mp_pool* p, const mp_addr* a, int64_t n) {
  if (!p || n < 0 || (n > 0 && !a)) return MP_ERR_CONFIG;
  TRY(remote_flush_tx(p));  // a pipelined copy goes first
  const uint32_t g = next_mark(p);
  for (int64_t i = 0; i < n; ++i) {
    int m = 0;
    int32_t idx = 0;
    if (!decode(p, a[i], &m, &idx)) return MP_ERR_INVALID_ADDR;
    const uint8_t s = p->st[m][(size_t)idx];
    uint32_t& mk = p->mark[m][(size_t)idx];
    if (s == ST_FREE || mk == g) return MP_ERR_DOUBLE_FREE;
    if (s != ST_ACTIVE) return MP_ERR_PRECONDITION;
    mk = g;
  }
  for (int64_t i = 0; i < n; ++i) {
    int m = 0;
    int32_t idx = 0;
    decode(p, a[i], &m, &idx);
    free_block(p, m, idx);
  }
  return MP_OK;  // the device bitmap update is queued, stream-ordered
}

mp_status mp_insert(mp_pool* p, const mp_token* toks, int64_t n_tok, const mp_addr* a,
                    int64_t n_addr, uint32_t flags, int64_t* n_dup) {
  if (!p || n_tok < 0 || (n_tok > 0 && !toks) || n_addr < 0 || (n_addr > 0 && !a))
    return MP_ERR_CONFIG;
  TRY(remote_flush_tx(p));  // a pipelined copy goes first
  return insert_internal(p, toks, n_tok, a, n_addr, flags, n_dup);
}

mp_status mp_match(mp_pool* p, const mp_token* toks, int64_t n_tok, uint32_t flags, mp_addr* out,
                   int64_t cap, int64_t* matched) {
  if (!p || n_tok < 0 || (n_tok > 0 && !toks)) return MP_ERR_CONFIG;
  if (cap < n_tok / p->B || (cap > 0 && !out)) return MP_ERR_BUFFER_TOO_SMALL;
  std::vector<mpi::Node*> m = p->index->match(toks, n_tok, (flags & MP_MATCH_PIN) != 0);
  for (size_t i = 0; i < m.size(); ++i) out[i] = enc(p, m[i]->medium, m[i]->idx);
  if (matched) *matched = (int64_t)m.size() * p->B;
  return MP_OK;
}

mp_status mp_unpin(mp_pool* p, const mp_addr* a, int64_t n) {
  if (!p || n < 0 || (n > 0 && !a)) return MP_ERR_CONFIG;
  TRY(remote_flush_tx(p));  // a pipelined copy goes first
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
    if (nd) {
      have = nd->ref;
    } else {
      auto it = p->orphan_ref[m].find(idx);
      if (it != p->orphan_ref[m].end()) have = it->second;
    }
    if (have < kv.second) return MP_ERR_PRECONDITION;
  }
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
  return MP_OK;
}

mp_status mp_delete(mp_pool* p, const mp_token* toks, int64_t n_tok) {
  if (!p || n_tok < 0 || (n_tok > 0 && !toks)) return MP_ERR_CONFIG;
  TRY(remote_flush_tx(p));  // a pipelined copy goes first
  for (const auto& u : p->index->erase_seq(toks, n_tok)) {
    if (u.ref == 0) {
      free_block(p, u.medium, u.idx);
    } else {  // pinned: freed by the last unpin (R6, R12)
      p->st[u.medium][(size_t)u.idx] = ST_ORPHAN;
      p->orphan_ref[u.medium][u.idx] = u.ref;
    }
  }
  return MP_OK;
}

mp_status mp_evict(mp_pool* p, int64_t n, int32_t medium, mp_addr* out, int64_t* n_freed) {
  if (!p || n < 0 || (medium != MP_HBM && medium != MP_DRAM) || (n > 0 && !out))
    return MP_ERR_CONFIG;
  TRY(remote_flush_tx(p));  // a pipelined copy goes first
  std::vector<int32_t> freed;
  evict_internal(p, n, medium, &freed);
  for (size_t i = 0; i < freed.size(); ++i) out[i] = enc(p, medium, freed[i]);
  if (n_freed) *n_freed = (int64_t)freed.size();
  return MP_OK;
}

}  // extern "C"
