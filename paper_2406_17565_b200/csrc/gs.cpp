// gs.cpp -- locality-aware global scheduling over global prompt trees
// (§6).
//
// "The GS employs three types of prompt trees, for prefill-only, decode-only,
// and PD-colocated instances.  Each tree type has a set of radix trees, the
// same as the ones used by MemPool with one extra field per tree node pointing
// to the instance storing the KV cache".  Lookup: match against
// the trees, "chooses an instance with the longest common prefix", then
// "checks whether there exist instances storing extra historical KV cache that
// is not present in the chosen instance" and lists them; update
// when responses return; entries carry a time-to-live because the GS
// does not see local evictions.
//
// Readings (R17): one block-granular trie per instance kind;
// each node maps holder instance -> expiry time (update time + TTL); an
// instance's cached prefix for a prompt is the deepest node on the prompt's
// path it holds unexpired; ties on the prefix length go to the least-loaded
// instance, then the lowest id; extra holders are all instances (any kind)
// holding a longer prefix than the chosen one, longest first.  Time is an
// explicit argument (deterministic, replayable).
#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <unordered_map>
#include <utility>
#include <vector>

#include "../../include/mempool.h"

namespace {

// One trie node per block-aligned prefix.  Children are found by a 64-bit
// hash of the block's tokens (confirmed token by token); holders are a short
// unsorted list (a handful of instances per prefix).
struct GsNode {
  std::vector<mp_token> chunk;                                   // the B tokens
  std::unordered_multimap<uint64_t, std::unique_ptr<GsNode>> kids;
  std::vector<std::pair<int32_t, double>> holders;                // instance -> expiry
};

struct Inst {
  int32_t kind = 0;
  double load = 0.0;
};

uint64_t chunk_hash(const mp_token* t, int32_t B) {
  uint64_t h = 1469598103934665603ull;
  for (int32_t i = 0; i < B; ++i) {
    h ^= (uint32_t)t[i];
    h *= 1099511628211ull;
    h ^= h >> 29;
  }
  return h;
}

GsNode* find_kid(const GsNode* n, const mp_token* t, int32_t B, uint64_t h) {
  auto range = n->kids.equal_range(h);
  for (auto it = range.first; it != range.second; ++it)
    if (std::memcmp(it->second->chunk.data(), t, sizeof(mp_token) * (size_t)B) == 0)
      return it->second.get();
  return nullptr;
}

}  // namespace

struct mp_gs {
  int32_t B = 16;
  double ttl = 0.0;
  GsNode roots[3];  // per kind: 0 prefill-only, 1 decode-only, 2 PD-colocated
  std::map<int32_t, Inst> insts;
};

namespace {

// Deepest unexpired prefix (in blocks) held by every instance of one tree.
void tree_match(const mp_gs* g, const GsNode* root, const mp_token* toks, int64_t n_tok,
                double now, std::vector<std::pair<int32_t, int64_t>>* best) {
  const GsNode* cur = root;
  for (int64_t i = 0; i < n_tok / g->B; ++i) {
    const mp_token* t = toks + i * g->B;
    cur = find_kid(cur, t, g->B, chunk_hash(t, g->B));
    if (!cur) break;
    for (const auto& h : cur->holders) {
      if (!(h.second > now)) continue;
      auto it = std::find_if(best->begin(), best->end(),
                             [&](const std::pair<int32_t, int64_t>& b) { return b.first == h.first; });
      if (it == best->end())
        best->push_back({h.first, i + 1});
      else
        it->second = i + 1;
    }
  }
}

}  // namespace

extern "C" {

mp_status mp_gs_create(int32_t block_tokens, double ttl_seconds, mp_gs** out) {
  if (!out || block_tokens < 1 || !(ttl_seconds > 0)) return MP_ERR_CONFIG;
  mp_gs* g = new mp_gs();
  g->B = block_tokens;
  g->ttl = ttl_seconds;
  *out = g;
  return MP_OK;
}

void mp_gs_destroy(mp_gs* g) { delete g; }

mp_status mp_gs_register(mp_gs* g, int32_t instance, int32_t kind) {
  if (!g || kind < 0 || kind > 2 || g->insts.count(instance)) return MP_ERR_CONFIG;
  g->insts[instance].kind = kind;
  return MP_OK;
}

mp_status mp_gs_set_load(mp_gs* g, int32_t instance, double load) {
  if (!g || !g->insts.count(instance)) return MP_ERR_CONFIG;
  g->insts[instance].load = load;
  return MP_OK;
}

mp_status mp_gs_update(mp_gs* g, int32_t instance, const mp_token* toks, int64_t n_tok,
                       double now) {
  if (!g || n_tok < 0 || (n_tok > 0 && !toks) || !g->insts.count(instance)) return MP_ERR_CONFIG;
  GsNode* cur = &g->roots[g->insts[instance].kind];
  for (int64_t i = 0; i < n_tok / g->B; ++i) {
    const mp_token* t = toks + i * g->B;
    const uint64_t h = chunk_hash(t, g->B);
    GsNode* nx = find_kid(cur, t, g->B, h);
    if (!nx) {
      std::unique_ptr<GsNode> fresh(new GsNode());
      fresh->chunk.assign(t, t + g->B);
      nx = fresh.get();
      cur->kids.emplace(h, std::move(fresh));
    }
    cur = nx;
    auto it = std::find_if(cur->holders.begin(), cur->holders.end(),
                           [&](const std::pair<int32_t, double>& x) { return x.first == instance; });
    if (it == cur->holders.end())
      cur->holders.push_back({instance, now + g->ttl});
    else
      it->second = now + g->ttl;
  }
  return MP_OK;
}

mp_status mp_gs_route(mp_gs* g, int32_t kind, const mp_token* toks, int64_t n_tok, double now,
                      int32_t* instance, int64_t* matched_tokens, int32_t* extra_inst,
                      int64_t* extra_tokens, int64_t cap, int64_t* n_extra) {
  if (!g || kind < 0 || kind > 2 || n_tok < 0 || (n_tok > 0 && !toks) || !instance)
    return MP_ERR_CONFIG;
  // instance -> blocks, all tree types ("concurrently")
  std::vector<std::pair<int32_t, int64_t>> got;
  for (int t = 0; t < 3; ++t) tree_match(g, &g->roots[t], toks, n_tok, now, &got);
  int32_t pick = -1;
  int64_t pick_blocks = -1;
  double pick_load = 0.0;
  for (const auto& kv : g->insts) {
    if (kv.second.kind != kind) continue;
    auto it = std::find_if(got.begin(), got.end(), [&](const std::pair<int32_t, int64_t>& x) {
      return x.first == kv.first;
    });
    const int64_t b = it == got.end() ? 0 : it->second;
    if (b > pick_blocks || (b == pick_blocks && kv.second.load < pick_load)) {
      pick = kv.first;
      pick_blocks = b;
      pick_load = kv.second.load;
    }
  }
  if (pick < 0) return MP_ERR_DST_UNREACHABLE;  // no instance of that kind
  std::vector<std::pair<int64_t, int32_t>> extra;
  for (const auto& kv : got)
    if (kv.second > pick_blocks) extra.push_back({-kv.second, kv.first});
  std::sort(extra.begin(), extra.end());
  if ((int64_t)extra.size() > cap && extra_inst) return MP_ERR_BUFFER_TOO_SMALL;
  *instance = pick;
  if (matched_tokens) *matched_tokens = pick_blocks * g->B;
  for (size_t i = 0; extra_inst && i < extra.size(); ++i) {
    extra_inst[i] = extra[i].second;
    if (extra_tokens) extra_tokens[i] = -extra[i].first * g->B;
  }
  if (n_extra) *n_extra = (int64_t)extra.size();
  return MP_OK;
}

}  // extern "C"
