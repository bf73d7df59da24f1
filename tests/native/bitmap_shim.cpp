// Test-only C shim over the product's BitmapUpdates (csrc/bitmap_updates.hpp),
// built with g++ on a CPU-only box by tests/test_bitmap_updates_cpu.py.
#include <cstdint>
#include <cstring>
#include <vector>

#include "bitmap_updates.hpp"

extern "C" {

void* bu_new(int64_t n) {
  auto* u = new mp::BitmapUpdates();
  u->reset((size_t)n);
  return u;
}
void bu_free(void* u) { delete static_cast<mp::BitmapUpdates*>(u); }
void bu_on_free(void* u, int32_t id) { static_cast<mp::BitmapUpdates*>(u)->on_free(id); }
void bu_on_claim(void* u, int32_t id) { static_cast<mp::BitmapUpdates*>(u)->on_claim(id); }
int64_t bu_queued(void* u) { return (int64_t) static_cast<mp::BitmapUpdates*>(u)->queued(); }
void bu_compact(void* u) { static_cast<mp::BitmapUpdates*>(u)->compact(); }
// writes the live updates into out (cap entries); returns their count
int64_t bu_take(void* u, int32_t* out, int64_t cap) {
  std::vector<int32_t> v;
  static_cast<mp::BitmapUpdates*>(u)->take(&v);
  if ((int64_t)v.size() > cap) return -1;
  if (!v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(int32_t));
  return (int64_t)v.size();
}

}  // extern "C"
