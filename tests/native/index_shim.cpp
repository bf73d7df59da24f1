// Test-only C shim over the product prompt index (paper_2406_17565_b200/csrc/
// index.hpp), so the host index logic -- R4 insert, R5 match, R6 delete,
// R8 LRU leaf eviction, R9 HBM-frontier choice, eviction feasibility -- runs
// on a CPU-only box against the oracle (tests/test_index_cpu.py).  No CUDA.
#include <cstring>
#include <string>
#include <vector>

#include "index.hpp"

using mpi::Index;
using mpi::Node;

extern "C" {

void* ix_new(int B, int64_t n_hbm, int64_t n_dram) { return new Index(B, n_hbm, n_dram); }
void ix_free(void* h) { delete (Index*)h; }
uint64_t ix_clock(void* h) { return ((Index*)h)->clock(); }

int64_t ix_insert(void* h, const int32_t* toks, int64_t n_tok, const int32_t* med,
                  const int32_t* idx, int32_t* dup_med, int32_t* dup_idx) {
  Index* ix = (Index*)h;
  const int64_t k = n_tok / ix->block_tokens();
  std::vector<Node*> path = ix->path(toks, k);
  std::vector<int> m(med, med + k);
  std::vector<Index::Placed> dups;
  ix->insert_seq(path, toks, k, m.data(), idx, &dups, nullptr);
  for (size_t i = 0; i < dups.size(); ++i) {
    dup_med[i] = dups[i].medium;
    dup_idx[i] = dups[i].idx;
  }
  return (int64_t)dups.size();
}

int64_t ix_match(void* h, const int32_t* toks, int64_t n_tok, int pin, int32_t* out_med,
                 int32_t* out_idx) {
  std::vector<Node*> p = ((Index*)h)->match(toks, n_tok, pin != 0);
  for (size_t i = 0; i < p.size(); ++i) {
    out_med[i] = p[i]->medium;
    out_idx[i] = p[i]->idx;
  }
  return (int64_t)p.size();
}

int64_t ix_erase(void* h, const int32_t* toks, int64_t n_tok, int32_t* out_med, int32_t* out_idx,
                 int32_t* out_ref) {
  std::vector<Index::Placed> u = ((Index*)h)->erase_seq(toks, n_tok);
  for (size_t i = 0; i < u.size(); ++i) {
    out_med[i] = u[i].medium;
    out_idx[i] = u[i].idx;
    out_ref[i] = u[i].ref;
  }
  return (int64_t)u.size();
}

int ix_evict(void* h, int medium, int32_t* idx) { return ((Index*)h)->evict_lru_leaf(medium, idx); }

int ix_frontier(void* h, int32_t* idx) {
  Node* n = ((Index*)h)->lru_frontier();
  if (!n) return 0;
  *idx = n->idx;
  return 1;
}

void ix_rebind(void* h, int medium, int32_t idx, int new_medium, int32_t new_idx) {
  Index* ix = (Index*)h;
  ix->rebind(ix->owner(medium, idx), new_medium, new_idx);
}

int64_t ix_evictable(void* h, int medium) {
  return ((Index*)h)->evictable(medium, std::vector<Node*>());
}

int64_t ix_evictable_leaves(void* h, int medium) {
  return ((Index*)h)->evictable_leaves(medium, std::vector<Node*>());
}

// pinned = the stored path of toks; returns evictable(medium, pinned) and
// writes whether evictable_at_least agrees for need = 0..that+1 (1 = yes)
int64_t ix_evictable_pinned(void* h, int medium, const int32_t* toks, int64_t n_tok, int* agree) {
  Index* ix = (Index*)h;
  const std::vector<Node*> pin = ix->path(toks, n_tok / ix->block_tokens());
  const int64_t full = ix->evictable(medium, pin);
  *agree = 1;
  for (int64_t k = 0; k <= full + 1; ++k)
    if (ix->evictable_at_least(medium, pin, k) != (full >= k)) *agree = 0;
  return full;
}

int ix_evictable_at_least(void* h, int medium, int64_t need) {
  return ((Index*)h)->evictable_at_least(medium, std::vector<Node*>(), need) ? 1 : 0;
}

int64_t ix_dump(void* h, char* buf, int64_t cap) {
  const std::string s = ((Index*)h)->dump();
  if (buf && cap > (int64_t)s.size()) {
    std::memcpy(buf, s.data(), s.size());
    buf[s.size()] = 0;
  }
  return (int64_t)s.size();
}

}  // extern "C"
