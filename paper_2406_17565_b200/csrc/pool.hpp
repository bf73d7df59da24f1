// pool.hpp -- internal state of one MemPool instance (mp_pool) and the
// runtime helpers shared by the C-ABI translation units.
//
// Execution model (B200-first):
//  * every pool owns one CUDA stream; all device work of the pool (allocator,
//    free, migration kernels, fills) is stream-ordered on it, so host-side
//    bookkeeping never waits for the device except where a result must be
//    host-visible (the call's return for synchronous calls, mp_sync for
//    MP_XFER_ASYNC transfers);
//  * the HBM allocator is device-resident (bitmap + alloc_kernel writing the
//    destination block table in HBM, read directly by the migration kernel);
//    the host keeps an exact shadow of it (same lowest-first rule, R2) so the
//    prompt index can be updated without a device round trip.  In verify mode
//    every device allocation is checked against the shadow at the next sync;
//  * cross-pool work (a transfer) is ordered with events: the executing
//    stream waits for the other pool's stream before the copy and the other
//    pool's stream waits for the copy after it.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>
#include <deque>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "../../include/mempool.h"
#include "bitmap_updates.hpp"
#include "index.hpp"
#include "kernels.cuh"

namespace mp {

void set_err(const std::string& s);
const std::string& get_err();

enum : uint8_t { ST_FREE = 0, ST_ACTIVE = 1, ST_INDEXED = 2, ST_ORPHAN = 3 };

struct DevGuard {
  int prev = -1, want;
  explicit DevGuard(int d) : want(d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DevGuard() {
    if (prev >= 0 && prev != want) cudaSetDevice(prev);
  }
};

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      ::mp::set_err(std::string(#x) + ": " + cudaGetErrorString(e_));         \
      return MP_ERR_CUDA;                                                     \
    }                                                                         \
  } while (0)

#define TRY(x)                  \
  do {                          \
    mp_status s_ = (x);         \
    if (s_ != MP_OK) return s_; \
  } while (0)

struct Msg {
  int32_t kind, src;
  std::vector<uint8_t> priv;
  std::vector<mp_addr> addrs;
};

// Ring arena of int32 ids: a device buffer and a mapped pinned mirror of the
// same size.  Uploads are staged through the mirror; wrapping drains the
// stream first, so a region is never rewritten while a copy may read it.
struct Arena {
  int* d = nullptr;
  int* h = nullptr;
  int64_t cap = 0, used = 0;
};

struct TimedLaunch {
  int pair;
  uint64_t bytes;
};

struct PendingVerify {
  const int* host;  // device allocator output (mapped mirror)
  std::vector<int32_t> want;
};

// Receiver-side state of one transfer between its allocation step and its
// insertion step.  Built by dst_prepare_*, consumed by dst_commit.
struct DstPrep {
  int kind = 0;  // 0 transfer, 1 transfer_with_insert
  int32_t src_inst = -1;
  uint32_t flags = 0;
  std::vector<int32_t> toks;
  int64_t n_tok = 0, ceil_b = 0, floor_b = 0, q = 0, skip = 0, nm = 0;
  std::vector<mpi::Node*> matched;  // pinned receiver prefix (R3, R12)
  std::vector<int32_t> dids;        // receiver block ids of the moved blocks
  int* d_dst = nullptr;             // allocator output on the receiver's device
  std::vector<uint8_t> priv;
};

// ---- overlap of independent migration launches (programmatic dependent
// launch without the start wait; kernels.cu pdl_wait).  The "window" of a
// data stream is the set of migration grids that may still run when the next
// launch's CTAs start: every launch since the last one that waited at its
// start (that one included -- it may itself still run).  A launch may skip
// its start wait iff it reads no block a window grid writes and writes no
// block a window grid reads or writes; otherwise it waits and opens a new
// window.  A launch whose blocks the host does not know (staging, DRAM,
// caller buffers) always waits and makes the next launch wait too.
// Marks hold the generation of the window that last touched a block;
// generations are unique across all streams, so a stale mark never matches.
struct BlockMarks {
  std::vector<uint32_t> r, w;  // per block: window generation of its last read / write
  void reset(size_t n) {
    r.assign(n, 0u);
    w.assign(n, 0u);
  }
};
struct LaunchTrack {
  uint32_t gen = 0;
  bool unknown = true;  // the window holds a launch with unknown blocks
  int launches = 0;
  // host-clock estimate (s) of when the coalesced launches queued on the
  // stream drain (bytes at a slightly optimistic HBM rate): a batch being
  // built is launched once less than kDrainLead of queued work remains, so
  // the GPU has the next launch before it runs dry
  double busy_until = 0.0;
};
// The blocks of one pool -> pool launch (host copies of its id lists).
struct LaunchBlocks {
  BlockMarks* rm;       // source pool's marks
  const int32_t* sids;
  BlockMarks* wm;       // destination pool's marks (a peer's, for remote stores)
  const int32_t* dids;
  int64_t n;
};
uint32_t new_track_gen();
// The stream is idle (synchronised) or something outside the window's
// knowledge was enqueued on it: the next launch waits.
inline void track_fence(LaunchTrack* t) {
  t->unknown = true;
  t->launches = 0;
}

struct Channel;  // shared-memory mailbox (remote.cpp)

// A page of host shared memory, pinned and mapped for the GPUs, holding the
// device-side flags of one ordered pair of pools (remote.cpp): GPU streams
// write them with stream memory operations and wait on them with
// cuStreamWaitValue32, so the two processes' streams synchronise without a
// host round trip.  Layout (uint32 words): [kSyncDone] done sequence of the
// pair's transfers (raised by the sender's stream after its copies),
// [kSyncPrep] prepare sequence (raised by the receiver's data stream after
// the allocation step and every earlier use of the blocks), [kSyncReady + s]
// STAGED slot s filled, [kSyncFree + s] slot s drained.  Every value only
// grows, so a wait for ">= v" taken at any time means the same thing -- unlike
// an interprocess event, whose re-recording by a third party could make a
// waiter depend on its own future work.
constexpr int kMaxSyncSlots = 64;
constexpr int kSyncDone = 0, kSyncPrep = 1, kSyncReady = 16, kSyncFree = 16 + kMaxSyncSlots;
struct SyncPage {
  std::string name;
  int fd = -1;
  uint32_t* h = nullptr;  // host view
  uint32_t* d = nullptr;  // device view
  bool registered = false;
};
// Stream memory operations (driver API through the runtime's entry points):
// s waits until (int32)(*dptr - v) >= 0; s writes v to *dptr after its
// earlier work (with a memory fence).
mp_status stream_wait_geq(cudaStream_t s, const uint32_t* dptr, uint32_t v);
mp_status stream_write_u32(cudaStream_t s, uint32_t* dptr, uint32_t v);
// Make `s` wait for every earlier user of p's staging buffer (STAGED slots,
// swap halves).
mp_status staging_acquire(mp_pool* p, cudaStream_t s);

// A pool living in another process (one process per GPU), imported with
// mp_import_peer: its slabs are CUDA-IPC mapped into this process, a pinned
// shared-memory page of monotonic flags per direction orders the two
// processes' streams (SyncPage), and two mailboxes carry the control
// messages of the workflow.
struct RemotePeer {
  int32_t inst = -1, dev = -1;
  uint64_t uid = 0;
  bool same_device = false;
  std::vector<void*> mapped;      // IPC-opened allocation bases
  char** d_slabs = nullptr;       // the peer's slab pointers, valid on my device
  Channel* out = nullptr;         // me -> peer requests
  Channel* in = nullptr;          // peer -> me requests
  bool has_pending = false;       // peer's transfer between prepare and commit
  DstPrep pending;
  BlockMarks bmarks;              // the peer's HBM blocks in my launch window
  std::vector<char*> slabs_h;     // the peer's slab pointers, valid here (copy-engine paths)
  int64_t staging_bytes = 0;      // the peer's staging configuration (STAGED ring geometry)
  int32_t staging_slots = 0;
  // device-side synchronisation with the peer (host shared memory, mapped)
  SyncPage* out_sync = nullptr;   // my transfers to the peer
  SyncPage* in_sync = nullptr;    // the peer's transfers to me
  // STAGED transport: the receiver keeps one inbound ring per sending peer
  // (device memory, IPC-exported in its first allocation reply); the sender
  // packs a slot, copies it into the peer's ring with the copy engine and
  // raises the slot's ready flag; the receiver's recv_stream waits for the
  // flag, unpacks into the fresh blocks and raises the slot's free flag.
  char* ring = nullptr;           // receiver side: my inbound ring for this peer
  int64_t ring_bytes = 0;
  uint64_t ring_id = 0;
  cudaIpcMemHandle_t ring_hnd{};  // taken once, when the ring is allocated
  char* peer_ring = nullptr;      // sender side: the peer's inbound ring for me
  uint64_t peer_ring_id = 0;
  uint32_t out_slot = 0, in_slot = 0;  // slot sequence numbers per direction
  cudaStream_t recv_stream = nullptr;
  cudaEvent_t recv_dep = nullptr, recv_ev = nullptr;
  bool recv_join = false;         // recv_ev (the last staged inbound's unpacks) not yet joined
  // inbound transfers from the peer whose copies may still run: one-round-
  // trip ones from their allocation step on, two-round-trip ones from their
  // completion message on.  Their copies have landed once the done flag
  // reaches seq; joined to my data stream lazily, oldest first, as
  // (stamp, seq) -- the stamp bounds which ones a transfer I am issuing may
  // join (mp_pool::join_bound)
  uint32_t in_seq = 0;            // receiver side: done sequence numbers handed out
  uint32_t prep_seq = 0;          // receiver side: prepares served for this peer
  uint32_t pending_done = 0;      // done sequence of the two-round-trip transfer in `pending`
  std::deque<std::pair<uint64_t, uint32_t>> async_in;
};

// A cross-process copy whose allocation reply has arrived but which is not
// enqueued yet (MP_XFER_PIPELINE): it is enqueued before this pool enqueues
// any other device work or serves any inbound request (remote_flush_tx), so
// the pool's stream sees the same order as without pipelining.
struct PendingTx {
  RemotePeer* r = nullptr;
  uint32_t path = 0;
  int j0 = 0, nj = 0;
  std::vector<int32_t> hs, hd, ds, dd;
  uint32_t prep_seq = 0, done_seq = 0;
  uint64_t start_stamp = 0;
  std::vector<mpi::Node*> pinned;  // indexed sources, pinned until enqueued
  int64_t nm = 0;
  uint64_t bytes = 0;              // payload of the (merged) copy
};

}  // namespace mp

struct mp_pool {
  // shape
  int32_t inst = 0, dev = 0, L = 0, H = 0, D = 0, elem = 0, B = 0;
  bool verify = false;
  int64_t chunk = 0, Pb = 0, n_hbm = 0, n_dram = 0;
  int nch = 0;
  int max_ctas = 0;
  int copy_kernel = 0;  // mpk::CopyVariant for device<->device copies
  int peer_engine = 0;  // copy engine / split of stores into peer memory (mp_pool_config)
  int peer_sched = 0;
  bool force_peer = false;  // test knob: same-GPU peers take the peer dispatch
  // device memory
  std::vector<char*> slabs;
  void* own_slab_region = nullptr;
  char** d_slabs = nullptr;
  uint32_t* d_bitmap = nullptr;
  int nwords = 0;
  int* d_err = nullptr;
  // dynamic unit claiming of bulk launches on `stream` (kernels.cuh Sched)
  unsigned long long* d_sched = nullptr;
  unsigned long long sched_base = 0;
  mp::Arena ar;
  char* dram = nullptr;      // host pointer of the pinned DRAM pool
  char* dram_dev = nullptr;  // device-visible (mapped) pointer
  bool own_dram = false;
  char* staging = nullptr;
  int64_t staging_bytes = 0;
  int staging_slots = 4;
  // `stream` carries the KV data movement; `meta` carries the allocator
  // bitmap kernels and the id uploads, so the allocation of the next transfer
  // overlaps the copy of the previous one.  A data kernel that consumes ids
  // waits for `meta` (meta_fence) -- never the other way round: the bitmap is
  // metadata, and a block handed out again is only written by later kernels
  // of the data stream, which run after every earlier reader of it.
  cudaStream_t stream = nullptr, meta = nullptr, copy_stream = nullptr;
  bool shared_stream = false;  // stream is the device's shared data stream (not owned)
  mp::LaunchTrack* track = nullptr;  // launch window of `stream` (shared with it)
  mp::LaunchTrack own_track;
  mp::BlockMarks bmarks;             // this pool's HBM blocks in launch windows
  // cross-process ordering: every inbound one-round-trip transfer gets a
  // prepare stamp; while this pool issues a transfer of its own it joins
  // only inbound transfers prepared before that transfer started
  // (join_bound), so waits always point at earlier-started transfers and no
  // cycle of device waits can form between two processes sending to each
  // other (remote.cpp)
  uint64_t prep_stamp = 0;
  uint64_t join_bound = ~0ull;
  mp::PendingTx* pend_tx = nullptr;  // MP_XFER_PIPELINE copy not enqueued yet
  std::vector<cudaEvent_t> pack_ev;  // STAGED (cross-process): slot packed
  cudaEvent_t ev_order = nullptr, ev_meta = nullptr;
  std::vector<cudaEvent_t> slot_ev;
  // swap through device staging, double-buffered: [0,1] the halves' fill done
  // (pack / H2D), [2,3] their drain done (D2H / unpack)
  cudaEvent_t swap_ev[4] = {};
  // profiling: a ring of (start, end) event pairs per migration launch
  int profile_every = 0;        // 0: off; k: time every k-th data-stream migration
  uint64_t profile_seen = 0;
  int last_timed_pair = -1;     // end event of the previous harvested launch (gaps)
  std::vector<cudaEvent_t> tev;
  std::vector<mp::TimedLaunch> timed;
  int tev_next = 0;
  mp_stats stats{};
  // host shadow of block ownership
  std::vector<uint8_t> st[2];
  std::vector<int32_t> alloc_by[2];
  int64_t nfree[2] = {0, 0};
  std::vector<uint64_t> hfree;             // HBM shadow bitmap (bit = 1: free)
  std::set<int32_t> dram_free;             // host-managed pinned DRAM allocator
  std::map<int32_t, int32_t> orphan_ref[2];
  // Device-bitmap updates not applied yet (frees, mp_alloc_mem's claims):
  // stream-ordered, lazily, before the next device scan (bitmap_updates.hpp).
  mp::BitmapUpdates dev_upd;
  std::vector<uint32_t> mark[2];           // scratch duplicate marks (next_mark)
  uint32_t mark_gen = 0;
  std::vector<mp::PendingVerify> pending_verify;
  mpi::Index* index = nullptr;
  uint64_t epoch = 0;
  std::map<int32_t, mp_pool*> peers;
  std::map<int32_t, char**> peer_tables;   // peer's slab table, on this device
  std::deque<mp::Msg> inbox;
  // launch coalescing of in-process fused transfers INTO this pool: consecutive
  // transfers from the same source pool and layer range append their id
  // lists to bsrc / bdst and go out as one migration launch when the data
  // stream is idle, the batch reaches batch_limit bytes, or anything else
  // touches either pool's blocks (flush_involving).
  struct {
    mp_pool* src = nullptr;
    int j0 = 0, nj = 0;
    int64_t count = 0;
    uint64_t bytes = 0;
    std::vector<int32_t> sids, dids;  // host copies (to clear the pending marks)
    int tab = 0;                       // which of the kBatchTabs id tables it fills
    bool open = false;                 // a table is assigned (count may still be 0)
  } batch;
  // Set by an in-process transfer that will be coalesced: the receiver's
  // allocation kernel then writes the new ids straight into the open batch's
  // destination table (no device-to-device copy per transfer).
  struct {
    mp_pool* src = nullptr;
    int j0 = 0, nj = 0;
  } slot_hint;
  // The id tables are filled on the meta stream while earlier launches may
  // still read theirs on the data stream: a ring of kBatchTabs tables, and a
  // new batch's meta work waits for the launch that last read its table.
  static constexpr int kBatchTabs = 4;
  int* bsrc_ring[kBatchTabs] = {};
  int* bdst_ring[kBatchTabs] = {};
  cudaEvent_t btab_ev[kBatchTabs] = {};
  bool btab_used[kBatchTabs] = {};
  int btab_next = 0;
  int* bsrc = nullptr;  // = bsrc_ring[batch.tab] of the batch being built
  int* bdst = nullptr;
  int64_t batch_cap = 0;
  uint64_t batch_limit = 0;
  std::vector<uint8_t> pend_w;  // block written by a pending batch (this pool is dst)
  std::vector<uint8_t> pend_r;  // block read by a pending batch (this pool is src)
  bool coalesce = true;
  bool idle_flush = true;
  // multi-process
  uint64_t uid = 0;                        // random identity (mailbox names)
  std::map<int32_t, mp::RemotePeer*> remotes;
  std::vector<int32_t> marks;              // end-of-batch marks received (mp_serve)
};

namespace mp {

constexpr int kTimedPairs = 512;
constexpr int kMaxDevStreams = 64;
cudaError_t shared_stream_acquire(int dev, cudaStream_t* out, LaunchTrack** track);
void shared_stream_release(int dev);

int* arena_take(mp_pool* p, int64_t n, int** host);
mp_status upload_ids(mp_pool* p, const std::vector<int32_t>& ids, int** d_out);
mp_status flush_frees(mp_pool* p);
mp_status drain(mp_pool* p);  // stream sync + timing + verification
mp_status sync(mp_pool* p);   // flush_frees + drain
mp_status link(mp_pool* signal, mp_pool* waiter);  // waiter's stream waits for signal's
mp_status meta_fence(mp_pool* p);                  // p->stream waits for p->meta

bool decode(const mp_pool* p, mp_addr a, int* med, int32_t* idx);
// Both pools on one GPU and neither asks for the peer dispatch (force_peer).
inline bool same_gpu(const mp_pool* a, const mp_pool* b) {
  return a->dev == b->dev && !a->force_peer && !b->force_peer;
}
inline mp_addr enc(const mp_pool* p, int med, int32_t idx) { return MP_ADDR(p->inst, med, idx); }

void free_block(mp_pool* p, int med, int32_t idx);
void evict_internal(mp_pool* p, int64_t n, int med, std::vector<int32_t>* freed);
bool can_make_room(mp_pool* p, int64_t n, int med, const std::vector<mpi::Node*>& pinned);
// Lowest-first HBM allocation: host shadow ids + the device allocator writing
// the same ids into HBM (d_ids) for the kernels that follow on the stream.
mp_status batch_open(mp_pool* src, mp_pool* dst, int64_t n, int j0, int nj);
mp_status src_ids(mp_pool* p, const std::vector<int32_t>& ids, int** d, mpk::InlineIds* inl);
// defer: no allocation kernel -- the ids' device bits are cleared by the next
// device bitmap update (mp_alloc_mem: nothing on the device reads its ids).
mp_status alloc_hbm(mp_pool* p, int64_t n, int32_t requester, std::vector<int32_t>* ids,
                    int** d_ids, bool defer = false);
std::vector<int32_t> alloc_dram(mp_pool* p, int64_t n, int32_t requester);

// peer: one endpoint is another GPU's / process's memory (P2P or IPC mapped);
// the copy engine choice then stays on the vector path.
// len: bytes copied per chunk (0: the whole chunk, p->chunk); an endpoint
// with cstride == 0 uses p->chunk as its chunk stride.
// blocks (nullable): the launch's pool -> pool blocks, so it may overlap the
// previous grids of the stream (LaunchTrack); nullptr: it waits for them.
mp_status launch_migrate_timed(mp_pool* p, cudaStream_t s, const mpk::Endpoint& a,
                               const mpk::Endpoint& b, int64_t n, int j0, int nj,
                               bool peer = false, int64_t len = 0,
                               const mpk::InlineIds* src_inline = nullptr,
                               bool meta_dep = true, const LaunchBlocks* blocks = nullptr);

// Both id lists by value in the launch parameters when they fit (the host
// shadow's dids equal what the allocation kernel wrote on the device).
inline bool pair_inline(const std::vector<int32_t>& sids, const std::vector<int32_t>& dids,
                        mpk::InlineIds* si) {
  const size_t n = sids.size();
  if (n == 0 || dids.size() != n || 2 * n > (size_t)mpk::kInlineIds) return false;
  si->n = si->nd = (int)n;
  std::memcpy(si->ids, sids.data(), n * sizeof(int32_t));
  std::memcpy(si->ids + n, dids.data(), n * sizeof(int32_t));
  return true;
}

// Sources in `src`'s pinned DRAM -> destination blocks `dids` (slab table
// `dslabs`: src's peer pool, or an IPC-mapped one when `peer`), through the
// copy engine: H2D of the aggregated blocks into src's staging on its copy
// stream, double-buffered against one scatter per slot on stream `s` of
// pool `ex` (same device as src).  Used when dram_source_ce(src, nj).
bool dram_source_ce(const mp_pool* src, int nj);
mp_status dram_ce_scatter(mp_pool* src, mp_pool* ex, cudaStream_t s, char** dslabs,
                          const std::vector<int32_t>& sids, const std::vector<int32_t>& dids,
                          int j0, int nj, bool peer);

// Launch coalescing (same-device fused transfers).
mp_status batch_append(mp_pool* src, mp_pool* dst, const std::vector<int32_t>& sids,
                       const std::vector<int32_t>& dids, const int* d_dst, int j0, int nj);
mp_status flush_batch(mp_pool* dst);
mp_status flush_involving(mp_pool* p);  // every pending batch reading or writing p's blocks
inline mpk::Endpoint pool_ep(char** slabs, const int* ids, long long cstride = 0,
                             long long off = 0) {
  return {slabs, nullptr, 0, ids, cstride, off};
}
inline mpk::Endpoint agg_ep(char* base, long long stride, const int* ids, long long cstride = 0,
                            long long off = 0) {
  return {nullptr, base, stride, ids, cstride, off};
}

mp_status insert_internal(mp_pool* p, const mp_token* toks, int64_t n_tok, const mp_addr* addrs,
                          int64_t n_addr, uint32_t flags, int64_t* n_dup,
                          const std::vector<mpi::Node*>* hint = nullptr,
                          std::vector<mpi::Node*>* out_nodes = nullptr);
// Scratch marks for duplicate detection without clearing: a block is marked
// in the current pass iff p->mark[medium][idx] == the value returned here.
uint32_t next_mark(mp_pool* p);
void unpin_nodes(mp_pool* p, const std::vector<mpi::Node*>& nodes);

// ---- the receiver's half of the workflow (shared by in-process and remote)
// (1) allocation: validates everything first (no state change on error),
// then matches / pins / allocates.  `given`: caller-given destination addrs
// (MP_XFER_DST_GIVEN) or nullptr.  host_ids: the copy takes the destination
// ids from the host (a remote sender gets them in the reply), so the fresh
// blocks are claimed in the host shadow and reach the device bitmap with its
// next stream-ordered update -- no allocation kernel, no device id table
// (st->d_dst stays null).
mp_status dst_prepare_xfer(mp_pool* dst, int32_t src_inst, int64_t n, uint32_t flags,
                           const mp_addr* given, const void* priv, int64_t priv_len,
                           DstPrep* st, bool host_ids = false);
mp_status dst_prepare_twi(mp_pool* dst, int32_t src_inst, const mp_token* toks, int64_t n_tok,
                          int64_t m, uint32_t flags, const mp_addr* given, const void* priv,
                          int64_t priv_len, DstPrep* st, bool host_ids = false);
// (3) insertion + completion: insert (twi), unpin, final addrs, `private`
// delivery.  final_out: st.ceil_b entries (twi) or st.nm entries (transfer).
mp_status dst_commit(mp_pool* dst, DstPrep& st, mp_addr* final_out);
// The transmission failed after (1): release what the allocation step took
// (the pinned matched prefix, the fresh blocks unless caller-given), so the
// failed call leaves no state change behind.
void dst_abort(mp_pool* dst, DstPrep& st);
// What the transmission step could reject (unknown path, a STAGED slot that
// cannot hold one block), checked before the receiver changes any state.
mp_status transmit_precheck(mp_pool* src, mp_pool* dst, uint32_t path, int nj,
                            const std::vector<uint8_t>& smeds);

// remote.cpp
uint64_t new_uid();
// Make p's data stream wait for every peer that stored into p since the last
// call (RemotePeer::async_in, recv_join).  Cheap when nothing is pending.
// `skip`: a peer whose one-/two-round-trip inbound copies are NOT joined
// (its own next copy is ordered behind them by its stream).
mp_status remote_apply_waits(mp_pool* p, const RemotePeer* skip = nullptr);
mp_status remote_serve_once(mp_pool* p, int64_t* served);
// Enqueue the pool's pending MP_XFER_PIPELINE copy, if any (cheap otherwise).
mp_status remote_flush_tx(mp_pool* p);
void remote_close_all(mp_pool* p);
// MP_REMOTE_TRACE=1 (debugging a stalled cross-process pipeline): blocking
// waits on a stream / event poll instead, and after 10 s print every remote
// peer's flag pages and sequence counters to stderr once.
bool remote_trace_on();
void remote_dump_state(const mp_pool* p, const char* where);
cudaError_t sync_stream_traced(const mp_pool* p, cudaStream_t s, const char* where);
cudaError_t sync_event_traced(const mp_pool* p, cudaEvent_t e, const char* where);
void host_report_timing();  // MP_HOST_TIMING=1 (api_transfer.cpp)
bool host_timing_on();
double host_clock();
void host_lap(int slot, double dt);
mp_status remote_transfer(mp_pool* src, RemotePeer* r, int kind, const mp_token* toks,
                          int64_t n_tok, const std::vector<int32_t>& sids,
                          const std::vector<uint8_t>& smeds, int64_t n, mp_addr* da,
                          uint32_t flags, int32_t l0, int32_t l1, const void* priv,
                          int64_t priv_len, int64_t* n_moved);

}  // namespace mp
