// kernels.cuh -- launchers of the sm_100a kernels of libmempool (internal).
//
// Data-movement only: no tensor cores (BASELINE.json north_star "pure data
// movement path").  All kernels are written for B200: 148 SMs, 16-byte
// vector loads with L1::no_allocate, grids sized in multiples of the SM count.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mpk {

// One side of a block copy.
//   POOL side: chunk j of block b lives at slabs[j] + b * cstride   (per-layer
//              paged layout, "two blocks per LLM layer").
//   AGG side : chunk jr (relative to the copied layer range) of block b lives
//              at base + b * stride + jr * cstride  (aggregated layout).
// The copied range of every chunk starts `off` bytes into it (0 for whole
// chunks; a head offset for tensor-parallel repartition).
// ids == nullptr means the identity (block i of the copy is id i).
struct Endpoint {
  char* const* slabs;  // device array of 2L slab pointers (POOL), else nullptr
  char* base;          // AGG base (device or mapped pinned host), else nullptr
  long long stride;    // AGG bytes per block
  const int* ids;      // device array of n ids or nullptr
  long long cstride;   // bytes per chunk on this side
  long long off;       // byte offset of the copied range inside each chunk
};

// Up to kInlineIds block ids passed by value in the kernel parameters (no
// host-to-device copy call: 3.7 us of host time each on B200).
// A migration launch may also carry its n destination ids, at ids[n', n'+n)
// where n' = this->n (nd == n; n' + n <= kInlineIds), so it reads no id
// table at all; n == 0 with nd == n: destination ids only.
constexpr int kInlineIds = 1000;
struct InlineIds {
  int n = 0;
  int nd = 0;
  int ids[kInlineIds];
};

// Dynamic work distribution of the bulk engine: a device counter of the
// launching stream plus the host's running start value for it (advanced by
// the launcher; launches sharing a counter must be stream-serialised).
struct Sched {
  unsigned long long* ctr;
  unsigned long long* base;
};

// Copy engines of the migration kernel.
enum CopyVariant { kCopyAuto = 0, kCopyVector = 1, kCopyBulk = 2 };

// dst.chunk(ids_d[i], j)[0:len] = src.chunk(ids_s[i], j)[0:len] (each side
// from its own `off`) for i < n, j in [j0, j0+nj); len, offsets and strides
// multiples of 16 bytes.
// variant kCopyVector: 16-byte vector loads/stores by every lane;
// kCopyBulk: cp.async.bulk (TMA engine) ring through shared memory.
// max_ctas <= 0: one full wave (occupancy x SMs).
// sched (nullable, bulk only): claim units dynamically instead of statically.
// src_inline (nullable): the n source ids by value in the launch parameters
// (n <= kInlineIds); src.ids is then ignored.
// wait_prev: the launch waits at its start for the previous grid on the
// stream (programmatic dependent launch); false only when the host knows it
// touches no block the grids still running may touch (pool.cpp LaunchTrack).
cudaError_t launch_migrate(const Endpoint& src, const Endpoint& dst, int n, int j0, int nj,
                           long long len, int max_ctas, cudaStream_t stream, int variant,
                           const Sched* sched = nullptr, const InlineIds* src_inline = nullptr,
                           bool wait_prev = true);


// Lowest-first allocation of n blocks from a bitmap (bit = 1: free), after
// applying `frees` (nullable; applied first, so lowest-first sees them):
// an entry id >= 0 sets bit id, an entry -(id+1) clears it (a claim made on
// the host; the two sets are disjoint).  Writes the ids ascending into out_dev (device) and out_host (mapped
// pinned host, may be nullptr), clears their bits.  *err (device) := 1 if
// fewer than n were free (the host shadow makes this impossible; checked in
// verify mode).  n == 0 with frees: just the frees.
cudaError_t launch_alloc(uint32_t* bitmap, int nwords, int n, int* out_dev, int* out_host,
                         int* err, cudaStream_t stream, const InlineIds* frees = nullptr);

// Applies the updates ids[0..n) (device array; same encoding as `frees`).
cudaError_t launch_free(uint32_t* bitmap, const int* ids, int n, cudaStream_t stream);

// Synthetic KV write of n blocks (content model):
// word t of chunk j of block b = splitmix64(seed ^ splitmix64(inst<<40 |
// epoch<<14 | b) ^ (j * chunk/8 + t)).
cudaError_t launch_fill(char* const* slabs, const int* ids, int n, int nchunks, long long chunk,
                        unsigned long long seed, unsigned long long inst,
                        unsigned long long epoch, cudaStream_t stream);

int sm_count(int device);

// Loads every kernel of the library on the current device (and sets the
// bulk engine's shared-memory attribute) once.  Under lazy module loading
// (CUDA_MODULE_LOADING=LAZY, the default) a kernel's first launch loads it,
// and that load can block behind a stream that is already parked on a
// cross-process flag (cuStreamWaitValue32) -- e.g. the receiver's first
// STAGED unpack, whose ready flag the sender raises only after the reply the
// receiver is about to send.  Pools call this at creation.
cudaError_t preload_kernels();

}  // namespace mpk
