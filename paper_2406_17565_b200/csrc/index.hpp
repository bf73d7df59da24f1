// index.hpp -- host-side prompt index (BASELINE.json north_star item 5).
//
// PAPER.md §4.2: MemPool "utilizes the radix tree proposed by
// SGLang" extended to "reference data located anywhere in the system" (HBM or
// DRAM) with block granularity equal to the engine's ("our radix tree nodes
// point to KV cache blocks of 16 tokens").  Here every node is one B-token
// chunk (block-chunk-keyed radix tree): children are found through a hash of
// (parent, chunk tokens) with token-by-token equality confirmation, so a walk
// of k blocks costs k hash probes.  The child table is one open-addressing
// array (a probe touches the slot and the node, whose chunk is inline), and
// the last walked path is memoised: engines match then insert the same
// prompt, and the next turn's prompt extends it, so a walk
// re-probes only the blocks past the common prefix while no node has been
// unlinked since.
//
// Policies where the paper is silent: R5 match, R6 delete
// (terminal markers), R7 logical clock, R8 leaf-LRU evict with (last_access,
// block index) tie-break, R9 HBM-frontier LRU for swap-out victims.  The two
// candidate sets are kept incrementally so a pick is O(log n).
#pragma once
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <set>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

namespace mpi {

// Hot fields of a walk / touch first: line 0 holds the links and R7/R8/R12
// state, line 1 the block's tokens (B <= 16); the rest is touched rarely.
struct Node {
  Node* parent = nullptr;
  std::vector<Node*> kids;       // children (any medium)
  uint64_t last_access = 0;      // R7
  int32_t ref = 0;               // R12 pins
  int32_t medium = 0, idx = -1;  // where the KV block lives ("anywhere")
  int32_t n_hbm_kids = 0;
  bool terminal = false;         // R6
  bool in_leaf = false, in_front = false;  // membership in the candidate sets
  int32_t small[16];             // the B tokens of this block (inline when B <= 16)
  std::vector<int32_t> big;      //   (heap when B > 16)
  const int32_t* chunk(int B) const { return B <= 16 ? small : big.data(); }
  uint64_t hkey = 0;             // key in the child hash map
  uint64_t id = 0;
  int32_t pos_in_parent = -1;    // index in parent->kids
  int32_t leaf_medium = 0;
  std::pair<uint64_t, int32_t> leaf_key{0, 0}, front_key{0, 0};
  int32_t leaf_pos = -1, front_pos = -1;  // slots in the candidate heaps
  // scratch of evictable_at_least (generation-stamped, no clearing)
  uint64_t peel_gen = 0, pin_gen = 0;
  int64_t peel_left = 0;
};

using Key = std::pair<uint64_t, int32_t>;  // (last_access, block index)

// Binary min-heap of nodes by a Key member, each node knowing its slot, so a
// candidate set supports min / insert / erase / re-key in O(log n) without
// allocating (eviction of a long chain re-keys one parent per step).
template <Key Node::*kKey, int32_t Node::*kPos>
class NodeHeap {
 public:
  bool empty() const { return a_.empty(); }
  size_t size() const { return a_.size(); }
  Node* top() const { return a_.front(); }
  const std::vector<Node*>& items() const { return a_; }
  void clear() {
    for (Node* n : a_) n->*kPos = -1;
    a_.clear();
  }
  void push(Node* n) {
    n->*kPos = (int32_t)a_.size();
    a_.push_back(n);
    up((size_t)(n->*kPos));
  }
  void erase(Node* n) {
    const size_t i = (size_t)(n->*kPos);
    Node* last = a_.back();
    a_.pop_back();
    n->*kPos = -1;
    if (i < a_.size()) {
      a_[i] = last;
      last->*kPos = (int32_t)i;
      fix(i);
    }
  }
  void rekey(Node* n) { fix((size_t)(n->*kPos)); }

 private:
  bool less(size_t i, size_t j) const { return a_[i]->*kKey < a_[j]->*kKey; }
  void swap_at(size_t i, size_t j) {
    std::swap(a_[i], a_[j]);
    a_[i]->*kPos = (int32_t)i;
    a_[j]->*kPos = (int32_t)j;
  }
  void up(size_t i) {
    while (i > 0 && less(i, (i - 1) / 2)) {
      swap_at(i, (i - 1) / 2);
      i = (i - 1) / 2;
    }
  }
  void fix(size_t i) {
    up(i);
    for (;;) {
      size_t m = i;
      const size_t l = 2 * i + 1, r = l + 1;
      if (l < a_.size() && less(l, m)) m = l;
      if (r < a_.size() && less(r, m)) m = r;
      if (m == i) return;
      swap_at(i, m);
      i = m;
    }
  }
  std::vector<Node*> a_;
};

class Index {
 public:
  explicit Index(int B, int64_t n_hbm, int64_t n_dram) : B_(B) {
    owner_[0].assign((size_t)n_hbm, nullptr);
    owner_[1].assign((size_t)n_dram, nullptr);
    root_.id = next_id_++;
  }
  ~Index() { clear(); }
  Index(const Index&) = delete;
  Index& operator=(const Index&) = delete;

  int block_tokens() const { return B_; }
  uint64_t clock() const { return clock_; }
  uint64_t tick() { return ++clock_; }
  size_t size() const { return size_; }
  Node* owner(int medium, int32_t idx) const { return owner_[medium][(size_t)idx]; }

  // Existing nodes of prefixes 1..k (stops at the first missing one).
  std::vector<Node*> path(const int32_t* toks, int64_t k) const {
    std::vector<Node*> out;
    k = std::max<int64_t>(k, 0);
    // memo: nodes of the last walked path stay linked until an unlink
    size_t h = 0;
    if (memo_unlinks_ == unlinks_ && !memo_nodes_.empty()) {
      const size_t lim = std::min((size_t)k, memo_nodes_.size()) * (size_t)B_;
      const int32_t* m = memo_toks_.data();
      size_t same = (size_t)(std::mismatch(toks, toks + lim, m).first - toks);
      h = same / (size_t)B_;
      out.assign(memo_nodes_.begin(), memo_nodes_.begin() + (std::ptrdiff_t)h);
    }
    out.reserve((size_t)k);
    const Node* p = out.empty() ? &root_ : out.back();
    for (int64_t i = (int64_t)h; i < k; ++i) {
      Node* c = find_child(p, toks + i * B_);
      if (!c) break;
      out.push_back(c);
      p = c;
    }
    remember(toks, out);
    return out;
  }

  // path() trusting the first h nodes of `hint` (a prefix walked earlier and
  // still linked, e.g. pinned): only the remaining positions are looked up.
  std::vector<Node*> path_hinted(const std::vector<Node*>& hint, size_t h, const int32_t* toks,
                                 int64_t k) const {
    h = std::min(h, std::min(hint.size(), (size_t)std::max<int64_t>(k, 0)));
    std::vector<Node*> out(hint.begin(), hint.begin() + (std::ptrdiff_t)h);
    const Node* p = out.empty() ? &root_ : out.back();
    for (int64_t i = (int64_t)h; i < k; ++i) {
      Node* c = find_child(p, toks + i * B_);
      if (!c) break;
      out.push_back(c);
      p = c;
    }
    return out;
  }

  // R5 without side effects.
  int64_t peek(const int32_t* toks, int64_t n_tok) const {
    return (int64_t)path(toks, n_tok / B_).size();
  }

  // The side effects of match (R7 tick + touch, optional R12 pin) on a path
  // already walked with path().
  void touch_path(const std::vector<Node*>& nodes, bool pin) {
    const uint64_t t = tick();
    for (Node* n : nodes) {
      n->last_access = t;
      if (pin) ++n->ref;
      refresh(n);
    }
  }

  // R5 + R7 (+ R12 when pin): touches matched nodes with a fresh tick.
  std::vector<Node*> match(const int32_t* toks, int64_t n_tok, bool pin) {
    const uint64_t t = tick();
    std::vector<Node*> p = path(toks, n_tok / B_);
    for (Node* n : p) {
      n->last_access = t;
      if (pin) ++n->ref;
      refresh(n);
    }
    return p;
  }

  void touch(Node* n, uint64_t t) {
    n->last_access = t;
    refresh(n);
  }
  void set_ref(Node* n, int32_t r) {
    n->ref = r;
    refresh(n);
  }

  // New child under parent (nullptr = root) for chunk toks.
  Node* add(Node* parent, const int32_t* toks, int medium, int32_t idx, uint64_t t) {
    Node* p = parent ? parent : &root_;
    Node* n = new Node();
    n->parent = p;
    if (B_ <= 16)
      std::memcpy(n->small, toks, sizeof(int32_t) * (size_t)B_);
    else
      n->big.assign(toks, toks + B_);
    n->hkey = mix(p->id, hash_chunk(toks));
    n->medium = medium;
    n->idx = idx;
    n->last_access = t;
    n->id = next_id_++;
    n->pos_in_parent = (int32_t)p->kids.size();
    p->kids.push_back(n);
    if (medium == 0) ++p->n_hbm_kids;
    map_.insert(n);
    owner_[medium][(size_t)idx] = n;
    ++size_;
    refresh(p);
    refresh(n);
    return n;
  }

  // Unlink a childless node; returns its (medium, idx, ref).
  void unlink(Node* n) {
    Node* p = n->parent;
    map_.erase(n);
    ++unlinks_;
    Node* last = p->kids.back();
    p->kids[(size_t)n->pos_in_parent] = last;
    last->pos_in_parent = n->pos_in_parent;
    p->kids.pop_back();
    if (n->medium == 0) --p->n_hbm_kids;
    drop_from_sets(n);
    owner_[n->medium][(size_t)n->idx] = nullptr;
    --size_;
    refresh(p);
    delete n;
  }

  // Move a node's KV to another medium/block (swap): keeps its place in the tree.
  void rebind(Node* n, int medium, int32_t idx) {
    Node* p = n->parent;
    owner_[n->medium][(size_t)n->idx] = nullptr;
    if (n->medium == 0) --p->n_hbm_kids;
    n->medium = medium;
    n->idx = idx;
    if (medium == 0) ++p->n_hbm_kids;
    owner_[medium][(size_t)idx] = n;
    refresh(n);
    refresh(p);
  }

  struct Placed {
    int medium;
    int32_t idx;
    int32_t ref;
  };

  // R4 (after the caller validated the blocks): one clock tick; for prefixes
  // 1..k an existing node is touched (the caller's block, if different, is
  // reported in `dups`: keep-existing), a missing one gets a new node holding
  // the caller's block (reported in `added`); prefix_k becomes terminal.
  // `path` = path(toks, k) as walked before.  Returns the nodes of 1..k.
  std::vector<Node*> insert_seq(const std::vector<Node*>& path, const int32_t* toks, int64_t k,
                                const int* med, const int32_t* idx, std::vector<Placed>* dups,
                                std::vector<Placed>* added) {
    const uint64_t t = tick();
    std::vector<Node*> out;
    out.reserve((size_t)std::max<int64_t>(k, 0));
    Node* parent = nullptr;
    for (int64_t i = 0; i < k; ++i) {
      Node* ex = i < (int64_t)path.size() ? path[(size_t)i] : nullptr;
      Node* cur = ex;
      if (ex) {
        touch(ex, t);
        if (!(ex->medium == med[i] && ex->idx == idx[i]) && dups)
          dups->push_back({med[i], idx[i], 0});
      } else {
        cur = add(parent, toks + i * B_, med[i], idx[i], t);
        if (added) added->push_back({med[i], idx[i], 0});
      }
      out.push_back(cur);
      parent = cur;
    }
    if (!out.empty()) out.back()->terminal = true;
    remember(toks, out);
    return out;
  }

  // R6: delete a stored sequence -- no-op unless prefix_k (k = floor(n/B)) is
  // terminal; clear it, then unlink prefixes k, k-1, ... while childless and
  // not terminal.  Returns the unlinked blocks with their pin counts.
  std::vector<Placed> erase_seq(const int32_t* toks, int64_t n_tok) {
    std::vector<Placed> out;
    const int64_t k = n_tok / B_;
    if (k <= 0) return out;
    std::vector<Node*> p = path(toks, k);
    if ((int64_t)p.size() < k || !p.back()->terminal) return out;
    p.back()->terminal = false;
    for (int64_t i = k - 1; i >= 0; --i) {
      Node* nd = p[(size_t)i];
      if (!nd->kids.empty() || nd->terminal) break;
      out.push_back({nd->medium, nd->idx, nd->ref});
      unlink(nd);
    }
    return out;
  }

  // R8: unlink the least (last_access, idx) unpinned leaf of `medium`.
  bool evict_lru_leaf(int medium, int32_t* idx) {
    Node* v = lru_leaf(medium);
    if (!v) return false;
    *idx = v->idx;
    unlink(v);
    return true;
  }

  // R8: least (last_access, idx) leaf of `medium` with ref == 0, or nullptr.
  Node* lru_leaf(int medium) const {
    if (leaves_[medium].empty()) return nullptr;
    return leaves_[medium].top();
  }
  // R9: least (last_access, idx) HBM node with ref == 0 and no HBM child.
  Node* lru_frontier() const {
    if (front_.empty()) return nullptr;
    return front_.top();
  }

  // Current R8 candidates of `medium` (unpinned leaves), minus those on
  // `pinned_path`: a lower bound of evictable(), O(|pinned_path|).
  int64_t evictable_leaves(int medium, const std::vector<Node*>& pinned_path) const {
    int64_t n = (int64_t)leaves_[medium].size();
    for (const Node* p : pinned_path)
      if (p->in_leaf && p->leaf_medium == medium) --n;
    return n;
  }

  // evictable(medium, pinned_path) >= need, in O(need + |pinned_path| +
  // candidate leaves) instead of a walk of the whole tree: peel the tree from
  // its unpinned leaves upwards (a parent joins once all its children have
  // been peeled and it is an unpinned node of `medium` -- exactly the closure
  // evictable() counts) and stop at `need`.
  bool evictable_at_least(int medium, const std::vector<Node*>& pinned_path, int64_t need) {
    if (need <= 0) return true;
    const uint64_t g = ++peel_gen_;
    for (Node* p : pinned_path) p->pin_gen = g;
    int64_t count = 0;
    std::vector<Node*> stack;
    for (Node* leaf : leaves_[medium].items()) {
      if (leaf->pin_gen == g) continue;
      stack.push_back(leaf);
      while (!stack.empty()) {
        Node* n = stack.back();
        stack.pop_back();
        if (++count >= need) return true;
        Node* par = n->parent;
        if (par == &root_) continue;
        if (par->peel_gen != g) {
          par->peel_gen = g;
          par->peel_left = (int64_t)par->kids.size();
        }
        if (--par->peel_left == 0 && par->medium == medium && par->ref == 0 && par->pin_gen != g)
          stack.push_back(par);
      }
    }
    return false;
  }

  // Number of nodes of `medium` that repeated leaf eviction could remove:
  // medium matches, ref == 0, not on `pinned_path`, and every child is
  // itself eventually evictable (R2 feasibility).
  int64_t evictable(int medium, const std::vector<Node*>& pinned_path) const {
    std::vector<const Node*> order;
    std::vector<const Node*> stack{&root_};
    while (!stack.empty()) {
      const Node* n = stack.back();
      stack.pop_back();
      order.push_back(n);
      for (const Node* c : n->kids) stack.push_back(c);
    }
    std::unordered_map<const Node*, bool> ok;
    ok.reserve(order.size() * 2);
    int64_t count = 0;
    for (auto it = order.rbegin(); it != order.rend(); ++it) {
      const Node* n = *it;
      if (n == &root_) continue;
      bool e = n->medium == medium && n->ref == 0 &&
               std::find(pinned_path.begin(), pinned_path.end(), n) == pinned_path.end();
      for (const Node* c : n->kids)
        if (!ok[c]) e = false;
      ok[n] = e;
      if (e) ++count;
    }
    return count;
  }

  // Sorted text dump (mempool.h mp_debug_dump_index).
  std::string dump() const {
    std::vector<std::pair<std::vector<int32_t>, std::string>> rows;
    std::vector<std::pair<const Node*, std::vector<int32_t>>> stack;
    for (const Node* c : root_.kids) stack.push_back({c, {}});
    while (!stack.empty()) {
      auto [n, pre] = stack.back();
      stack.pop_back();
      pre.insert(pre.end(), n->chunk(B_), n->chunk(B_) + B_);
      std::string line = std::to_string(pre.size() / (size_t)B_) + "\t" + std::to_string(n->medium) +
                         "\t" + std::to_string(n->idx) + "\t" + std::to_string(n->last_access) +
                         "\t" + std::to_string(n->ref) + "\t" + (n->terminal ? "1" : "0") + "\t";
      for (size_t i = 0; i < pre.size(); ++i) {
        if (i) line += ",";
        line += std::to_string(pre[i]);
      }
      line += "\n";
      rows.push_back({pre, line});
      for (const Node* c : n->kids) stack.push_back({c, pre});
    }
    std::sort(rows.begin(), rows.end(),
              [](const auto& a, const auto& b) { return a.first < b.first; });
    std::string out;
    for (auto& r : rows) out += r.second;
    return out;
  }

  void clear() {
    leaves_[0].clear();  // before the nodes go (the heaps reset their slots)
    leaves_[1].clear();
    front_.clear();
    std::vector<Node*> stack(root_.kids.begin(), root_.kids.end());
    while (!stack.empty()) {
      Node* n = stack.back();
      stack.pop_back();
      for (Node* c : n->kids) stack.push_back(c);
      delete n;
    }
    root_.kids.clear();
    root_.n_hbm_kids = 0;
    map_.clear();
    ++unlinks_;
    for (auto& o : owner_) std::fill(o.begin(), o.end(), nullptr);
    size_ = 0;
  }

  Node* root() { return &root_; }

 private:
  static uint64_t hash_chunk_n(const int32_t* t, int n) {
    uint64_t h = 1469598103934665603ull;
    for (int i = 0; i < n; ++i) {
      h ^= (uint32_t)t[i];
      h *= 1099511628211ull;
      h ^= h >> 29;
    }
    return h;
  }
  uint64_t hash_chunk(const int32_t* t) const { return hash_chunk_n(t, B_); }
  static uint64_t mix(uint64_t a, uint64_t b) {
    uint64_t z = a * 0x9E3779B97F4A7C15ull ^ (b + 0x632BE59BD9B4E019ull + (a << 6) + (a >> 2));
    z ^= z >> 31;
    return z;
  }

  Node* find_child(const Node* p, const int32_t* toks) const {
    return map_.find(mix(p->id, hash_chunk(toks)), p, toks, B_);
  }

  // Keep the longer of the memo and this path when one extends the other
  // (match then insert of one prompt, a next turn's longer prompt): only the
  // new tail is copied.  Equal node pointers mean equal prefixes.
  void remember(const int32_t* toks, const std::vector<Node*>& nodes) const {
    const size_t k = nodes.size(), m = memo_nodes_.size();
    if (memo_unlinks_ == unlinks_) {
      size_t h = 0;
      const size_t c = std::min(k, m);
      while (h < c && memo_nodes_[h] == nodes[h]) ++h;
      if (h == k) return;  // a prefix of the memo
      if (h == m) {        // extends the memo
        memo_nodes_.insert(memo_nodes_.end(), nodes.begin() + (std::ptrdiff_t)m, nodes.end());
        memo_toks_.insert(memo_toks_.end(), toks + m * (size_t)B_, toks + k * (size_t)B_);
        return;
      }
    }
    memo_toks_.assign(toks, toks + k * (size_t)B_);
    memo_nodes_ = nodes;
    memo_unlinks_ = unlinks_;
  }

  // Open addressing, linear probing, backward-shift deletion; key = hkey.
  class ChildTable {
   public:
    ChildTable() { slots_.assign(1024, Slot{}); }
    void clear() {
      slots_.assign(1024, Slot{});
      used_ = 0;
    }
    void insert(Node* n) {
      if (2 * (used_ + 1) > slots_.size()) grow();
      put(n);
      ++used_;
    }
    void erase(const Node* n) {
      const size_t mask = slots_.size() - 1;
      size_t i = (size_t)n->hkey & mask;
      while (slots_[i].node != n) i = (i + 1) & mask;
      // backward shift: pull later entries of the run into the hole
      size_t hole = i;
      for (size_t j = (i + 1) & mask; slots_[j].node; j = (j + 1) & mask) {
        const size_t home = (size_t)slots_[j].key & mask;
        if (((j - home) & mask) >= ((j - hole) & mask)) {
          slots_[hole] = slots_[j];
          hole = j;
        }
      }
      slots_[hole] = Slot{};
      --used_;
    }
    Node* find(uint64_t key, const Node* parent, const int32_t* toks, int B) const {
      const size_t mask = slots_.size() - 1;
      for (size_t i = (size_t)key & mask; slots_[i].node; i = (i + 1) & mask) {
        const Slot& s = slots_[i];
        if (s.key == key && s.node->parent == parent &&
            std::memcmp(s.node->chunk(B), toks, sizeof(int32_t) * (size_t)B) == 0)
          return s.node;
      }
      return nullptr;
    }

   private:
    struct Slot {
      uint64_t key = 0;
      Node* node = nullptr;
    };
    void put(Node* n) {
      const size_t mask = slots_.size() - 1;
      size_t i = (size_t)n->hkey & mask;
      while (slots_[i].node) i = (i + 1) & mask;
      slots_[i] = Slot{n->hkey, n};
    }
    void grow() {
      std::vector<Slot> old;
      old.swap(slots_);
      slots_.assign(old.size() * 2, Slot{});
      for (const Slot& s : old)
        if (s.node) put(s.node);
    }
    std::vector<Slot> slots_;
    size_t used_ = 0;
  };

  void drop_from_sets(Node* n) {
    if (n->in_leaf) {
      leaves_[n->leaf_medium].erase(n);
      n->in_leaf = false;
    }
    if (n->in_front) {
      front_.erase(n);
      n->in_front = false;
    }
  }

  // Re-derive n's membership and keys in the R8 / R9 candidate sets.
  void refresh(Node* n) {
    if (n == &root_) return;
    const Key k{n->last_access, n->idx};
    const bool leaf = n->ref == 0 && n->kids.empty();
    if (n->in_leaf && (!leaf || n->leaf_medium != n->medium)) {
      leaves_[n->leaf_medium].erase(n);
      n->in_leaf = false;
    }
    if (leaf) {
      if (!n->in_leaf) {
        n->leaf_key = k;
        n->leaf_medium = n->medium;
        leaves_[n->medium].push(n);
        n->in_leaf = true;
      } else if (n->leaf_key != k) {
        n->leaf_key = k;
        leaves_[n->medium].rekey(n);
      }
    }
    const bool front = n->ref == 0 && n->medium == 0 && n->n_hbm_kids == 0;
    if (n->in_front && !front) {
      front_.erase(n);
      n->in_front = false;
    }
    if (front) {
      if (!n->in_front) {
        n->front_key = k;
        front_.push(n);
        n->in_front = true;
      } else if (n->front_key != k) {
        n->front_key = k;
        front_.rekey(n);
      }
    }
  }

  int B_;
  Node root_;
  ChildTable map_;
  uint64_t unlinks_ = 0;  // bumps invalidate the memo
  uint64_t peel_gen_ = 0;
  mutable std::vector<int32_t> memo_toks_;
  mutable std::vector<Node*> memo_nodes_;
  mutable uint64_t memo_unlinks_ = ~0ull;
  NodeHeap<&Node::leaf_key, &Node::leaf_pos> leaves_[2];
  NodeHeap<&Node::front_key, &Node::front_pos> front_;
  std::vector<Node*> owner_[2];
  uint64_t clock_ = 0;
  uint64_t next_id_ = 1;
  size_t size_ = 0;
};

}  // namespace mpi
