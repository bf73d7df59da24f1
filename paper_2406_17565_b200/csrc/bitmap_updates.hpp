// bitmap_updates.hpp -- the device bitmap allocator's pending updates
// (header-only, no CUDA: also built into a CPU test shim,
// tests/native/bitmap_shim.cpp).
//
// The host shadow of the allocator (pool.cpp) decides every id first; the
// device bitmap (bit = 1: free) learns the host's decisions lazily, stream-
// ordered, before its next scan: a free sets a bit, a claim made on the host
// by mp_alloc_mem (no allocation kernel) clears one.  A free of a not yet
// applied claim -- or a claim of a not yet applied free -- cancels it, so the
// queued updates of different ids never concern the same bit twice and can be
// applied in any order (atomicOr / atomicAnd by many threads).  Ids whose state
// changed after they were queued leave stale queue entries, skipped by take().
#ifndef MP_BITMAP_UPDATES_HPP
#define MP_BITMAP_UPDATES_HPP

#include <cstddef>
#include <cstdint>
#include <vector>

namespace mp {

class BitmapUpdates {
 public:
  enum : uint8_t { kNone = 0, kFree = 1, kClaim = 2, kSeen = 0x80 };

  void reset(size_t n_blocks) {
    q_.clear();
    st_.assign(n_blocks, kNone);
  }

  // The host freed `id` (its device bit is 0 unless a claim is still queued).
  void on_free(int32_t id) { note(id, kFree, kClaim); }

  // The host handed `id` out without a device scan (its device bit is 1
  // unless a free is still queued).
  void on_claim(int32_t id) { note(id, kClaim, kFree); }

  bool empty() const { return q_.empty(); }
  size_t queued() const { return q_.size(); }  // upper bound (stale entries included)

  // Host only: drops stale and duplicate entries, so the queue holds at most
  // one entry per block however long the device goes without a scan (a pool
  // whose allocations all come from the host -- a cross-process receiver --
  // then never launches a kernel just to bound it).
  void compact() {
    size_t k = 0;
    for (int32_t id : q_) {
      uint8_t& s = st_[(size_t)id];
      if (s == kNone || (s & kSeen)) continue;
      s = (uint8_t)(s | kSeen);
      q_[k++] = id;
    }
    q_.resize(k);
    for (int32_t id : q_) st_[(size_t)id] = (uint8_t)(st_[(size_t)id] & ~kSeen);
  }

  // Moves the live updates to *out, encoded id (set the bit) or -(id+1)
  // (clear it), and forgets them.
  void take(std::vector<int32_t>* out) {
    out->clear();
    for (int32_t id : q_) {
      uint8_t& s = st_[(size_t)id];
      if (s == kFree) out->push_back(id);
      else if (s == kClaim) out->push_back(-id - 1);
      s = kNone;  // later duplicates of this id are stale
    }
    q_.clear();
  }

 private:
  void note(int32_t id, uint8_t kind, uint8_t opposite) {
    uint8_t& s = st_[(size_t)id];
    if (s == opposite) {  // the two cancel: the device bit is already right
      s = kNone;
    } else {
      s = kind;
      q_.push_back(id);
    }
  }

  std::vector<int32_t> q_;
  std::vector<uint8_t> st_;
};

}  // namespace mp

#endif  // MP_BITMAP_UPDATES_HPP
