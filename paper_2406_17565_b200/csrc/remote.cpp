// remote.cpp -- MemPool across processes (one process per GPU).
//
// PAPER.md §4.3: "When the sender inference instance initiates a
// transfer, it sends a request to the receiver inference instance.  Upon
// receiving this request, the receiver invokes alloc_mem locally ... then
// returns the allocated address list ... the sender transmits the KV cache to
// the receiver using the fastest available path.  Once all data is received,
// the receiver notifies the sender ... invokes the insert function locally
// ... the sender completes the transfer API call once the receiver returns ok."
//
// B200 realisation:
//  * control messages travel through a POSIX shared-memory mailbox per ordered
//    pair of pools (request slot + reply slot, sequence numbers with
//    acquire/release ordering) -- both processes are on the same 8-GPU box;
//  * the receiver's slabs are CUDA-IPC mapped into the sender, and the
//    transmission is one-sided, on the sender's GPU, in one of three
//    transports (remote_transmit): FUSED -- one gather -> peer-store kernel
//    writing the scattered source chunks straight into the receiver's fresh
//    blocks over NVLink (no staging, no per-block calls, no ordering thread;
//    the paper's NCCL send/recv needs one per communicator); CE --
//    one copy-engine memcpy per chunk; STAGED -- pack, one copy-engine copy
//    per slot into the receiver's inbound ring, unpack by the receiver,
//    pipelined by device-side flags;
//  * the two processes' streams are ordered with flags in a pinned
//    shared-memory page per ordered pair that GPU streams raise
//    (cuStreamWriteValue32) and wait on (cuStreamWaitValue32) -- SyncPage:
//    the sender's copy waits for the receiver's prepare flag (allocation
//    done), the receiver's later work for the sender's done flag (copy
//    landed), STAGED slots for ready / free flags.  The values only grow, so
//    a wait means the same whenever it is enqueued (an interprocess event
//    re-recorded for another sender could make a waiter depend on its own
//    later copy: the fan-in deadlock this replaced);
//  * an MP_XFER_ASYNC transfer takes ONE round trip: the receiver allocates,
//    inserts and delivers `private` when the request arrives (R15: host-side
//    effects at call time) and joins the sender's copy through the pair's
//    done flag before its next data-stream work; synchronous transfers keep
//    the paper's two round trips (the sender completes once the receiver
//    has the data and answered ok).
//  Waits across processes never form a cycle: a receiver's prepare flag for
//  transfer t is raised after waits on transfers stamped before t only, and
//  a pool issuing a transfer joins only inbound transfers stamped before its
//  own transfer started (mp_pool::join_bound), so every device wait points
//  at an earlier-started transfer.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <random>
#include <thread>

#include "pool.hpp"

namespace mp {

// ------------------------------------------------------------- mailbox
namespace {

constexpr uint64_t kChanMagic = 0x4D504348414E3031ull;  // "MPCHAN01"
constexpr int64_t kChanCap = 8ll << 20;                 // payload bytes per slot

struct SlotHdr {
  uint64_t seq;  // written last by the slot's writer (release), read first (acquire)
  uint32_t type;
  int32_t status;
  uint64_t len;
  uint8_t pad[40];
};
static_assert(sizeof(SlotHdr) == 64, "slot header is one cache line");

struct ChanHdr {
  uint64_t magic;
  uint64_t cap;
  uint8_t pad[48];
};

enum MsgType : uint32_t {
  REQ_XFER = 1, REQ_TWI = 2, REQ_DONE = 3, REQ_MARK = 4, REQ_ECHO = 5,
  REP_PREP = 11, REP_FINAL = 12, REP_ACK = 13, REP_ECHO = 15,
};

}  // namespace

struct Channel {
  std::string name;
  int fd = -1;
  char* base = nullptr;
  size_t size = 0;
  uint64_t next_req = 0;  // sender side: last request sequence number used
  uint64_t seen_req = 0;  // receiver side: last request served

  SlotHdr* req() { return (SlotHdr*)(base + sizeof(ChanHdr)); }
  char* req_payload() { return base + sizeof(ChanHdr) + sizeof(SlotHdr); }
  SlotHdr* rep() { return (SlotHdr*)(req_payload() + kChanCap); }
  char* rep_payload() { return (char*)rep() + sizeof(SlotHdr); }
};

namespace {

Channel* chan_open(const std::string& name) {
  Channel* c = new Channel();
  c->name = name;
  c->size = sizeof(ChanHdr) + 2 * (sizeof(SlotHdr) + (size_t)kChanCap);
  c->fd = shm_open(name.c_str(), O_CREAT | O_RDWR, 0600);
  if (c->fd < 0) {
    set_err("shm_open(" + name + ") failed");
    delete c;
    return nullptr;
  }
  struct stat sb;
  if (fstat(c->fd, &sb) != 0 || (size_t)sb.st_size < c->size) {
    if (ftruncate(c->fd, (off_t)c->size) != 0) {
      set_err("ftruncate(" + name + ") failed");
      close(c->fd);
      delete c;
      return nullptr;
    }
  }
  void* m = mmap(nullptr, c->size, PROT_READ | PROT_WRITE, MAP_SHARED, c->fd, 0);
  if (m == MAP_FAILED) {
    set_err("mmap(" + name + ") failed");
    close(c->fd);
    delete c;
    return nullptr;
  }
  c->base = (char*)m;
  ChanHdr* h = (ChanHdr*)c->base;
  h->cap = (uint64_t)kChanCap;
  __atomic_store_n(&h->magic, kChanMagic, __ATOMIC_RELEASE);
  return c;
}

void chan_close(Channel* c, bool unlink) {
  if (!c) return;
  if (c->base) munmap(c->base, c->size);
  if (c->fd >= 0) close(c->fd);
  if (unlink) shm_unlink(c->name.c_str());
  delete c;
}

// Synchronisation page of one ordered pair (pool.hpp SyncPage): created by
// whichever process opens it first (ftruncate zero-fills), pinned and mapped
// for the GPU in both.
constexpr size_t kSyncBytes = 4096;

SyncPage* sync_open(const std::string& name) {
  SyncPage* s = new SyncPage();
  s->name = name;
  s->fd = shm_open(name.c_str(), O_CREAT | O_RDWR, 0600);
  if (s->fd < 0) {
    set_err("shm_open(" + name + ") failed");
    delete s;
    return nullptr;
  }
  struct stat sb;
  if (fstat(s->fd, &sb) != 0 || (size_t)sb.st_size < kSyncBytes) {
    if (ftruncate(s->fd, (off_t)kSyncBytes) != 0) {
      set_err("ftruncate(" + name + ") failed");
      close(s->fd);
      delete s;
      return nullptr;
    }
  }
  void* m = mmap(nullptr, kSyncBytes, PROT_READ | PROT_WRITE, MAP_SHARED, s->fd, 0);
  if (m == MAP_FAILED) {
    set_err("mmap(" + name + ") failed");
    close(s->fd);
    delete s;
    return nullptr;
  }
  s->h = (uint32_t*)m;
  void* d = nullptr;
  if (cudaHostRegister(m, kSyncBytes, cudaHostRegisterMapped | cudaHostRegisterPortable) !=
          cudaSuccess ||
      cudaHostGetDevicePointer(&d, m, 0) != cudaSuccess) {
    cudaGetLastError();
    set_err("cudaHostRegister of the synchronisation page failed");
    munmap(m, kSyncBytes);
    close(s->fd);
    delete s;
    return nullptr;
  }
  s->registered = true;
  s->d = (uint32_t*)d;
  return s;
}

void sync_close(SyncPage* s) {
  if (!s) return;
  if (s->registered) cudaHostUnregister(s->h);
  if (s->h) munmap(s->h, kSyncBytes);
  if (s->fd >= 0) close(s->fd);
  shm_unlink(s->name.c_str());  // both sides unlink; the second finds it gone
  delete s;
}

// A flag the GPU may still be about to overwrite: set from the host (used
// only after the writing stream has been drained, on failure paths, so a
// waiting peer stream is released).
void host_raise(uint32_t* h, uint32_t v) { __atomic_store_n(h, v, __ATOMIC_RELEASE); }

// Slot geometry of the STAGED ring between two pools' staging buffers:
// S slots of slot_bytes, k blocks (<= kInlineIds, their ids ride in the
// unpack's launch parameters) of per_block bytes each.
struct RingGeom {
  int S = 0;
  int64_t slot_bytes = 0, k = 0;
};
RingGeom ring_geom(int64_t a_bytes, int a_slots, int64_t b_bytes, int b_slots,
                   int64_t per_block) {
  RingGeom g;
  g.S = std::max(1, std::min(std::min(a_slots, b_slots), kMaxSyncSlots));
  g.slot_bytes = (std::min(a_bytes, b_bytes) / g.S) & ~(int64_t)255;
  g.k = std::min<int64_t>(per_block > 0 ? g.slot_bytes / per_block : 0, mpk::kInlineIds);
  return g;
}

// Little serializer for the message payloads.
struct Writer {
  char* p;
  int64_t cap, len = 0;
  bool ok = true;
  void bytes(const void* src, int64_t n) {
    if (len + n > cap) {
      ok = false;
      return;
    }
    if (n > 0) std::memcpy(p + len, src, (size_t)n);
    len += n;
  }
  template <class T>
  void put(T v) {
    bytes(&v, sizeof(T));
  }
};

struct Reader {
  const char* p;
  int64_t len, pos = 0;
  bool ok = true;
  const void* bytes(int64_t n) {
    if (pos + n > len || n < 0) {
      ok = false;
      return nullptr;
    }
    const void* r = p + pos;
    pos += n;
    return r;
  }
  template <class T>
  T get() {
    T v{};
    const void* s = bytes(sizeof(T));
    if (s) std::memcpy(&v, s, sizeof(T));
    return v;
  }
};

// Writer side of the request slot: payload is built in place, then published.
void publish(SlotHdr* h, uint32_t type, int32_t status, int64_t len, uint64_t seq) {
  h->type = type;
  h->status = status;
  h->len = (uint64_t)len;
  __atomic_store_n(&h->seq, seq, __ATOMIC_RELEASE);
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

constexpr double kTimeout = 300.0;  // seconds without an answer: peer unreachable

// Phase timers of the cross-process workflow (MP_REMOTE_TIMING=1 prints them
// when the pool is destroyed): [0] request -> allocation reply, [1] launch,
// [2] done -> completion reply, [3] receiver prepare, [4] receiver commit.
struct PhaseTimes {
  double t[5] = {0, 0, 0, 0, 0};
  uint64_t n[5] = {0, 0, 0, 0, 0};
  void add(int i, double s) {
    t[i] += s;
    ++n[i];
  }
};
thread_local PhaseTimes g_phase;
bool timing_on() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("MP_REMOTE_TIMING");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  return on == 1;
}

}  // namespace

void remote_report_timing() {
  if (!timing_on()) return;
  const char* names[5] = {"req->prep_reply", "launch", "done->final_reply", "serve_prepare",
                          "serve_commit"};
  for (int i = 0; i < 5; ++i)
    if (g_phase.n[i])
      fprintf(stderr, "[mempool remote] %-18s %8llu calls %10.2f us avg\n", names[i],
              (unsigned long long)g_phase.n[i], g_phase.t[i] / g_phase.n[i] * 1e6);
}

// ---------------------------------------------------------- receiver side
#define MP_TRACE(...)                                   \
  do {                                                  \
    if (remote_trace_on()) {                            \
      fprintf(stderr, "[mempool trace %d] ", (int)getpid()); \
      fprintf(stderr, __VA_ARGS__);                     \
      fputc('\n', stderr);                              \
    }                                                   \
  } while (0)
namespace {

// Receiver half of a STAGED transfer, enqueued at its allocation step: the
// moved blocks whose sources sit in the sender's HBM arrive through this
// peer's inbound ring.  recv_stream waits for each slot's ready flag, unpacks
// it into the fresh blocks (ids in the launch parameters) and raises the
// slot's free flag -- all device-side, no host round trip per slot.  The
// stream is separate from the data stream, so a data stream never blocks on
// a flag a peer raises later.
mp_status staged_recv(mp_pool* p, RemotePeer* r, const DstPrep& st, const uint8_t* meds, int j0,
                      int nj) {
  const int64_t per_block = (int64_t)nj * p->chunk;
  const RingGeom g = ring_geom(r->staging_bytes, r->staging_slots, p->staging_bytes,
                               p->staging_slots, per_block);
  if (g.k < 1) {
    set_err("staging slot smaller than one block");
    return MP_ERR_CONFIG;
  }
  if (!r->ring) {  // first STAGED transfer from this peer: its inbound ring
    r->ring_bytes = std::min(p->staging_bytes, r->staging_bytes);
    CK(cudaMalloc(&r->ring, (size_t)r->ring_bytes));
    // the handle travels in every STAGED reply: taken here, before anything
    // is enqueued, so the reply itself cannot fail after the unpacks are
    if (cudaIpcGetMemHandle(&r->ring_hnd, r->ring) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(r->ring);
      r->ring = nullptr;
      set_err("cudaIpcGetMemHandle of the inbound ring failed");
      return MP_ERR_CUDA;
    }
    r->ring_id = new_uid();
    CK(cudaStreamCreateWithFlags(&r->recv_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&r->recv_dep, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&r->recv_ev, cudaEventDisableTiming));
  }
  MP_TRACE("staged_recv: ring ready");
  std::vector<int32_t> ids;
  for (int64_t i = 0; i < st.nm; ++i)
    if (meds[st.skip + i] == MP_HBM) ids.push_back(st.dids[(size_t)i]);
  if (ids.empty()) return MP_OK;
  // after the allocation and every earlier data-stream use of the blocks
  CK(cudaEventRecord(r->recv_dep, p->meta));
  CK(cudaStreamWaitEvent(r->recv_stream, r->recv_dep, 0));
  CK(cudaEventRecord(r->recv_dep, p->stream));
  CK(cudaStreamWaitEvent(r->recv_stream, r->recv_dep, 0));
  uint32_t q = r->in_slot;
  for (size_t off = 0; off < ids.size(); off += (size_t)g.k, ++q) {
    const int slot = (int)(q % (uint32_t)g.S);
    const int64_t nb = std::min<int64_t>(g.k, (int64_t)(ids.size() - off));
    TRY(stream_wait_geq(r->recv_stream, r->in_sync->d + kSyncReady + slot, q + 1));
    mpk::InlineIds di;
    di.n = 0;   // the source is the ring slot itself (block i at i * per_block)
    di.nd = (int)nb;
    std::memcpy(di.ids, ids.data() + off, (size_t)nb * sizeof(int32_t));
    TRY(launch_migrate_timed(p, r->recv_stream,
                             agg_ep(r->ring + (int64_t)slot * g.slot_bytes, per_block, nullptr),
                             pool_ep(p->d_slabs, nullptr), nb, j0, nj, false, 0, &di));
    TRY(stream_write_u32(r->recv_stream, r->in_sync->d + kSyncFree + slot, q + 1));
    MP_TRACE("staged_recv: slot %d (q %u, %lld blocks) queued", slot, q, (long long)nb);
  }
  r->in_slot = q;
  return MP_OK;
}

mp_status serve_message(mp_pool* p, RemotePeer* r) {
  Channel* c = r->in;
  SlotHdr* q = c->req();
  const uint64_t seq = __atomic_load_n(&q->seq, __ATOMIC_ACQUIRE);
  if (seq <= c->seen_req) return MP_ERR_PRECONDITION;  // nothing new
  c->seen_req = seq;
  Reader rd{c->req_payload(), (int64_t)q->len};
  Writer wr{c->rep_payload(), kChanCap};
  uint32_t rtype = REP_ACK;
  int32_t rstatus = MP_OK;
  DevGuard g(p->dev);
  const double t_start = timing_on() ? now_s() : 0.0;
  switch (q->type) {
    case REQ_XFER:
    case REQ_TWI: {
      const uint32_t flags = rd.get<uint32_t>();
      int64_t n_tok = 0;
      const mp_token* toks = nullptr;
      if (q->type == REQ_TWI) {
        n_tok = rd.get<int64_t>();
        toks = (const mp_token*)rd.bytes(n_tok * (int64_t)sizeof(mp_token));
      }
      const int64_t m = rd.get<int64_t>();
      const mp_addr* given = nullptr;
      if (flags & MP_XFER_DST_GIVEN) given = (const mp_addr*)rd.bytes(m * (int64_t)sizeof(mp_addr));
      const int64_t plen = rd.get<int64_t>();
      const void* priv = rd.bytes(plen);
      const int32_t j0 = rd.get<int32_t>(), nj = rd.get<int32_t>();
      const uint8_t* meds = (const uint8_t*)rd.bytes(m);
      const bool staged = (flags & MP_XFER_PATH_MASK) == MP_XFER_PATH_STAGED;
      // one round trip: the receiver commits (insert, delivery) now and the
      // sender's copy is joined through the pair's done flag (R15: an ASYNC
      // transfer's host-side effects happen at call time)
      const bool one_trip = (flags & MP_XFER_ASYNC) && !staged;
      mp_status s = flush_involving(p);
      if (s == MP_OK && !rd.ok) s = MP_ERR_CONFIG;
      if (s == MP_OK && r->has_pending) s = MP_ERR_PRECONDITION;
      if (s != MP_OK) {
        // nothing prepared
      } else if (q->type == REQ_TWI)
        s = dst_prepare_twi(p, r->inst, toks, n_tok, m, flags, given, priv, plen, &r->pending,
                            /*host_ids=*/true);
      else
        s = dst_prepare_xfer(p, r->inst, m, flags, given, priv, plen, &r->pending,
                             /*host_ids=*/true);
      const uint32_t slot0 = r->in_slot;
      uint32_t prep_seq = 0, done_seq = 0;
      MP_TRACE("serve: request type %u prepared: status %d", q->type, (int)s);
      if (s == MP_OK) {
        r->has_pending = true;
        // the sender's copy must follow this allocation and every earlier use
        // of the blocks on this pool's streams, including other peers' copies
        // into them (a block freed and re-allocated) and this peer's STAGED
        // unpacks (recv_stream); the sender's own earlier FUSED / CE / DRAM
        // copies are ordered by its stream already, so they are not joined
        // here -- joining them would chain every copy of a pair behind the
        // previous one through two flag hops
        s = remote_apply_waits(p, r);
        // (no meta fence: with host ids nothing of this allocation runs on
        // the meta stream, and meta never touches block data)
        if (s == MP_OK) {
          // raised by the data stream once everything before it has run; if
          // the stream is already idle (nothing queued, the waits above
          // included) the host raises it now -- no GPU operation, and the
          // value still only grows: an idle stream has no older prepare
          // write pending
          prep_seq = ++r->prep_seq;
          const cudaError_t q = cudaStreamQuery(p->stream);
          if (q == cudaSuccess) {
            host_raise(r->in_sync->h + kSyncPrep, prep_seq);
          } else if (q == cudaErrorNotReady) {
            s = stream_write_u32(p->stream, r->in_sync->d + kSyncPrep, prep_seq);
          } else {
            s = MP_ERR_CUDA;
          }
        }
        MP_TRACE("serve: prep flag %u enqueued: status %d", prep_seq, (int)s);
        if (s == MP_OK && staged) s = staged_recv(p, r, r->pending, meds, j0, nj);
        MP_TRACE("serve: staged_recv: status %d", (int)s);
        if (s != MP_OK) {
          dst_abort(p, r->pending);
          r->has_pending = false;
        }
      }
      std::vector<mp_addr> fin;
      // every transfer: the sender's stream raises the done flag to this
      // value after its copies into this pool
      if (s == MP_OK) done_seq = r->pending_done = ++r->in_seq;
      if (s == MP_OK && one_trip) {
        r->has_pending = false;
        const int64_t nfin = r->pending.kind == 1 ? r->pending.ceil_b : r->pending.nm;
        fin.assign((size_t)std::max<int64_t>(nfin, 1), 0);
        s = dst_commit(p, r->pending, fin.data());
        fin.resize((size_t)nfin);
        if (s == MP_OK) r->async_in.push_back({++p->prep_stamp, done_seq});
      }
      rtype = REP_PREP;
      rstatus = s;
      if (s == MP_OK) {
        wr.put<int64_t>(r->pending.skip);
        wr.put<int64_t>(r->pending.nm);
        wr.bytes(r->pending.dids.data(), (int64_t)r->pending.dids.size() * 4);
        wr.put<uint32_t>(prep_seq);
        wr.put<uint32_t>(done_seq);
        if (staged) {
          wr.bytes(&r->ring_hnd, sizeof(r->ring_hnd));
          wr.put<uint64_t>(r->ring_id);
          wr.put<uint32_t>(slot0);
        }
        if (one_trip) {
          wr.put<int64_t>((int64_t)fin.size());
          wr.bytes(fin.data(), (int64_t)fin.size() * (int64_t)sizeof(mp_addr));
        }
      }
      break;
    }
    case REQ_DONE: {
      const int32_t sender_status = rd.get<int32_t>();
      rtype = REP_FINAL;
      if (!r->has_pending) {
        rstatus = MP_ERR_PRECONDITION;
        break;
      }
      r->has_pending = false;
      const bool staged = (r->pending.flags & MP_XFER_PATH_MASK) == MP_XFER_PATH_STAGED;
      if (staged && r->recv_stream) {
        // every unpack of this transfer is on recv_stream (the sender has
        // raised every slot's ready flag, also on failure)
        if (cudaEventRecord(r->recv_ev, r->recv_stream) != cudaSuccess) {
          rstatus = MP_ERR_CUDA;
          break;
        }
        if (sender_status != MP_OK || !(r->pending.flags & MP_XFER_ASYNC)) {
          // data landed before the receiver says ok; a failed
          // transfer's unpacks finish before its blocks are released
          if (sync_event_traced(p, r->recv_ev, "DONE:recv_ev") != cudaSuccess) {
            rstatus = MP_ERR_CUDA;
            break;
          }
        } else {
          r->recv_join = true;  // later data-stream work joins it lazily
        }
      }
      if (sender_status != MP_OK) {  // the transmission failed on the sender:
        // release what the allocation step took (pins, fresh blocks)
        dst_abort(p, r->pending);
        rstatus = sender_status;
        break;
      }
      // later data-stream work of this pool must follow the sender's copy
      // (its done flag): applied lazily (remote_apply_waits), not chained
      // into the next allocation the sender waits for
      r->async_in.push_back({++p->prep_stamp, r->pending_done});
      const int64_t nfin = r->pending.kind == 1 ? r->pending.ceil_b : r->pending.nm;
      std::vector<mp_addr> fin((size_t)std::max<int64_t>(nfin, 1));
      rstatus = dst_commit(p, r->pending, fin.data());
      if (rstatus == MP_OK) {
        wr.put<int64_t>(nfin);
        wr.bytes(fin.data(), nfin * (int64_t)sizeof(mp_addr));
      }
      break;
    }
    case REQ_MARK: {
      p->marks.push_back(rd.get<int32_t>());
      rtype = REP_ACK;
      break;
    }
    case REQ_ECHO: {
      rtype = REP_ECHO;
      const int64_t n = (int64_t)q->len;
      const unsigned char* src = (const unsigned char*)rd.bytes(n);
      for (int64_t i = 0; src && i < n; ++i) wr.put<unsigned char>((unsigned char)(src[i] ^ 0x5A));
      break;
    }
    default:
      rstatus = MP_ERR_CONFIG;
  }
  if (!wr.ok) rstatus = MP_ERR_BUFFER_TOO_SMALL;
  MP_TRACE("serve: publish reply %u status %d seq %llu", rtype, (int)rstatus,
           (unsigned long long)seq);
  publish(c->rep(), rtype, rstatus, wr.len, seq);
  if (timing_on() && (rtype == REP_PREP || rtype == REP_FINAL))
    g_phase.add(rtype == REP_PREP ? 3 : 4, now_s() - t_start);
  return MP_OK;
}

// Sender: wait for the reply to request `seq`, serving this pool's own
// inbound requests meanwhile (two pools may send to each other at once).
mp_status wait_reply(mp_pool* self, Channel* c, uint64_t seq) {
  const double t0 = now_s();
  int spins = 0;
  bool dumped = false;
  while (__atomic_load_n(&c->rep()->seq, __ATOMIC_ACQUIRE) < seq) {
    int64_t served = 0;
    if (self) {
      mp_status s = remote_serve_once(self, &served);
      if (s != MP_OK) return s;
    }
    if (!served && ++spins > 64) {
      std::this_thread::yield();
      spins = 0;
      if (self && !dumped && remote_trace_on() && now_s() - t0 > 10.0) {
        remote_dump_state(self, "wait_reply");
        dumped = true;
      }
      if (now_s() - t0 > kTimeout) {
        set_err("remote peer did not answer (is it inside mp_serve?)");
        return MP_ERR_DST_UNREACHABLE;
      }
    }
  }
  return MP_OK;
}

}  // namespace

// Inbound copies whose done flag the host already sees raised have landed
// (the flag is written after the copy, with a memory barrier): nothing to
// join, so they leave the queue without a device wait.  Keeps the queue short
// on a receiver that never issues device work of its own.
static void prune_async_in(RemotePeer* r) {
  if (r->async_in.empty() || !r->in_sync) return;
  const uint32_t done = __atomic_load_n(r->in_sync->h + kSyncDone, __ATOMIC_ACQUIRE);
  while (!r->async_in.empty() && (int32_t)(done - r->async_in.front().second) >= 0)
    r->async_in.pop_front();
}

mp_status remote_apply_waits(mp_pool* p, const RemotePeer* skip) {
  for (auto& kv : p->remotes) {
    RemotePeer* r = kv.second;
    prune_async_in(r);
    if (!r->recv_join && (r->async_in.empty() || r == skip)) continue;
    DevGuard g(p->dev);
    if (r->recv_join) {  // the unpacks of a completed STAGED transfer
      CK(cudaStreamWaitEvent(p->stream, r->recv_ev, 0));
      r->recv_join = false;
    }
    // inbound copies: only those stamped before the transfer this pool is
    // issuing right now (join_bound), whose senders started earlier
    bool any = false;
    uint32_t seq = 0;
    while (r != skip && !r->async_in.empty() && r->async_in.front().first <= p->join_bound) {
      seq = r->async_in.front().second;
      r->async_in.pop_front();
      any = true;
    }
    if (any) TRY(stream_wait_geq(p->stream, r->in_sync->d + kSyncDone, seq));
  }
  return MP_OK;
}

mp_status remote_serve_once(mp_pool* p, int64_t* served) {
  *served = 0;
  for (auto& kv : p->remotes) {
    RemotePeer* r = kv.second;
    if (!r->in) continue;
    // a pipelined copy is enqueued before this pool's stream sees any
    // inbound work (only when a request is actually waiting: an idle poll
    // inside wait_reply must not break up a merge)
    if (p->pend_tx &&
        __atomic_load_n(&r->in->req()->seq, __ATOMIC_ACQUIRE) > r->in->seen_req)
      TRY(remote_flush_tx(p));
    mp_status s = serve_message(p, r);
    if (s == MP_OK) ++*served;
    else if (s != MP_ERR_PRECONDITION) return s;
  }
  return MP_OK;
}

// ------------------------------------------------------------ sender side
namespace {

// The transmission step of a cross-process transfer ("the sender
// transmits the KV cache to the receiver using the fastest available path"),
// issued on the sender's GPU.  (hs, hd): sources in the sender's HBM and
// their destination ids; (ds, dd): sources swapped out to its pinned DRAM
// (memory asymmetry), always stored by one kernel straight into
// the receiver's blocks.  Transports of the HBM part:
//   FUSED     one gather -> peer-store kernel (A6f; engine and split from the
//             pool's peer_engine / peer_sched)
//   CE        one copy-engine memcpy per (block, layer, K/V) chunk (the
//             paper's discrete per-block transfer)
//   STAGED    pack into a staging slot (A4, the paper's aggregation
//             P:549-550), one copy-engine memcpy of the slot into the
//             receiver's inbound ring (A5), unpack there (A6) -- pipelined
//             over the ring's slots by device-side flags
mp_status remote_transmit(mp_pool* src, RemotePeer* r, uint32_t path, int j0, int nj,
                          const std::vector<int32_t>& hs, const std::vector<int32_t>& hd,
                          const std::vector<int32_t>& ds, const std::vector<int32_t>& dd,
                          const RingGeom& geom, uint32_t slot0, uint32_t prep_seq) {
  TRY(flush_involving(src));
  const bool staged = path == MP_XFER_PATH_STAGED;
  // stores into the receiver's fresh blocks follow its allocation and every
  // earlier use of them there (its prepare flag, raised by its data stream
  // before the reply); the STAGED ring is ordered by its slot flags instead
  // (no device wait if the host already sees the flag raised: the receiver
  // raised it from its host, its data stream being idle)
  if ((!staged || !ds.empty()) &&
      (int32_t)(__atomic_load_n(r->out_sync->h + kSyncPrep, __ATOMIC_ACQUIRE) - prep_seq) < 0)
    TRY(stream_wait_geq(src->stream, r->out_sync->d + kSyncPrep, prep_seq));
  const int64_t n = (int64_t)hs.size();
  if (n > 0 && (path == MP_XFER_PATH_AUTO || path == MP_XFER_PATH_FUSED)) {
    mpk::InlineIds si;
    int *d_s = nullptr, *d_d = nullptr;
    const bool both = pair_inline(hs, hd, &si);
    if (!both) {
      TRY(src_ids(src, hs, &d_s, &si));
      TRY(upload_ids(src, hd, &d_d));
    }
    const LaunchBlocks lb{&src->bmarks, hs.data(), &r->bmarks, hd.data(), n};
    // a receiver process on this same GPU: its IPC-mapped pool is local HBM,
    // so the copy takes the loopback engine (bulk ring, claiming)
    TRY(launch_migrate_timed(src, src->stream, pool_ep(src->d_slabs, d_s),
                             pool_ep(r->d_slabs, d_d), n, j0, nj, /*peer=*/!r->same_device, 0,
                             si.n ? &si : nullptr, /*meta_dep=*/!both, &lb));
  } else if (n > 0 && path == MP_XFER_PATH_CE) {
    for (int64_t i = 0; i < n; ++i)
      for (int j = j0; j < j0 + nj; ++j)
        CK(cudaMemcpyAsync(r->slabs_h[(size_t)j] + (int64_t)hd[(size_t)i] * src->chunk,
                           src->slabs[(size_t)j] + (int64_t)hs[(size_t)i] * src->chunk,
                           (size_t)src->chunk, cudaMemcpyDefault, src->stream));
    track_fence(src->track);
    src->stats.bytes_moved += (uint64_t)(n * nj * src->chunk);
  } else if (n > 0 && staged) {
    TRY(staging_acquire(src, src->stream));
    const int64_t per_block = (int64_t)nj * src->chunk;
    uint32_t q = slot0;
    for (int64_t off = 0; off < n; off += geom.k, ++q) {
      const int slot = (int)(q % (uint32_t)geom.S);
      const int64_t nb = std::min<int64_t>(geom.k, n - off);
      char* mine = src->staging + (int64_t)slot * geom.slot_bytes;
      // my slot: its previous copy out is done
      CK(cudaStreamWaitEvent(src->stream, src->slot_ev[(size_t)slot], 0));
      mpk::InlineIds si;
      si.n = (int)nb;
      std::memcpy(si.ids, hs.data() + off, (size_t)nb * sizeof(int32_t));
      TRY(launch_migrate_timed(src, src->stream, pool_ep(src->d_slabs, nullptr),
                               agg_ep(mine, per_block, nullptr), nb, j0, nj, false, 0, &si,
                               /*meta_dep=*/false));
      CK(cudaEventRecord(src->pack_ev[(size_t)slot], src->stream));
      CK(cudaStreamWaitEvent(src->copy_stream, src->pack_ev[(size_t)slot], 0));
      // the peer's slot: its previous unpack is done (free flag)
      if (q >= (uint32_t)geom.S)
        TRY(stream_wait_geq(src->copy_stream, r->out_sync->d + kSyncFree + slot,
                            q + 1 - (uint32_t)geom.S));
      CK(cudaMemcpyAsync(r->peer_ring + (int64_t)slot * geom.slot_bytes, mine,
                         (size_t)(nb * per_block), cudaMemcpyDeviceToDevice, src->copy_stream));
      TRY(stream_write_u32(src->copy_stream, r->out_sync->d + kSyncReady + slot, q + 1));
      CK(cudaEventRecord(src->slot_ev[(size_t)slot], src->copy_stream));
    }
  }
  if (!ds.empty() && dram_source_ce(src, nj)) {
    // copy engine into our staging, scattered into the receiver's blocks
    TRY(dram_ce_scatter(src, src, src->stream, r->d_slabs, ds, dd, j0, nj,
                        /*peer=*/!r->same_device));
  } else if (!ds.empty()) {
    int *d_s = nullptr, *d_d = nullptr;
    mpk::InlineIds si;
    TRY(src_ids(src, ds, &d_s, &si));
    TRY(upload_ids(src, dd, &d_d));
    TRY(launch_migrate_timed(src, src->stream,
                             agg_ep(src->dram_dev + (int64_t)j0 * src->chunk, src->Pb, d_s),
                             pool_ep(r->d_slabs, d_d), (int64_t)ds.size(), j0, nj,
                             /*peer=*/true, 0, si.n ? &si : nullptr));
  }
  return MP_OK;
}

// Enqueue the transmission of one transfer and raise the pair's done flag
// after it (on failure: drain, then raise every flag the peer may wait on
// from the host).  join_bound = the transfer's start stamp (no wait on an
// inbound transfer that started later).
mp_status transmit_step(mp_pool* src, RemotePeer* r, uint32_t path, int j0, int nj,
                        const std::vector<int32_t>& hs, const std::vector<int32_t>& hd,
                        const std::vector<int32_t>& ds, const std::vector<int32_t>& dd,
                        const RingGeom& geom, uint32_t slot0, uint32_t slot_end,
                        uint32_t prep_seq, uint32_t done_seq, uint64_t start_stamp,
                        mp_status pre) {
  DevGuard g(src->dev);
  mp_status xs = pre;
  src->join_bound = start_stamp;
  if (xs == MP_OK) xs = remote_transmit(src, r, path, j0, nj, hs, hd, ds, dd, geom, slot0, prep_seq);
  src->join_bound = ~0ull;
  if (xs != MP_OK) {
    // release the peer's streams: every flag it waits on is raised from
    // the host once this side's copies are drained (or dead)
    cudaStreamSynchronize(src->stream);
    cudaStreamSynchronize(src->copy_stream);
    cudaGetLastError();
    for (uint32_t q = slot0; q != slot_end; ++q)
      host_raise(r->out_sync->h + kSyncReady + q % (uint32_t)geom.S, q + 1);
    host_raise(r->out_sync->h + kSyncDone, done_seq);
    return xs;
  }
  return stream_write_u32(src->stream, r->out_sync->d + kSyncDone, done_seq);
}

}  // namespace

mp_status remote_flush_tx(mp_pool* p) {
  PendingTx* t = p->pend_tx;
  if (!t) return MP_OK;
  p->pend_tx = nullptr;
  {  // queued work estimate (LaunchTrack::busy_until): a same-GPU peer's copy
     // reads and writes HBM (~7 TB/s), a remote one crosses NVLink (900 GB/s
     // nominal per direction) -- optimistic rates, so merging stops early
    const double now = host_clock();
    const double secs = t->r->same_device ? 2.0 * (double)t->bytes / 7.0e12
                                          : (double)t->bytes / 0.9e12;
    p->track->busy_until = std::max(now, p->track->busy_until) + secs;
  }
  const mp_status xs = transmit_step(p, t->r, t->path, t->j0, t->nj, t->hs, t->hd, t->ds, t->dd,
                                     RingGeom{}, 0, 0, t->prep_seq, t->done_seq, t->start_stamp,
                                     MP_OK);
  p->stats.blocks_moved += (uint64_t)t->nm;
  unpin_nodes(p, t->pinned);
  delete t;
  return xs;
}

mp_status remote_transfer(mp_pool* src, RemotePeer* r, int kind, const mp_token* toks,
                          int64_t n_tok, const std::vector<int32_t>& sids,
                          const std::vector<uint8_t>& smeds, int64_t n, mp_addr* da,
                          uint32_t flags, int32_t l0, int32_t l1, const void* priv,
                          int64_t priv_len, int64_t* n_moved) {
  const uint32_t path = flags & MP_XFER_PATH_MASK;
  if (path != MP_XFER_PATH_AUTO && path != MP_XFER_PATH_FUSED && path != MP_XFER_PATH_STAGED &&
      path != MP_XFER_PATH_CE) {
    set_err("unknown transfer path");
    return MP_ERR_CONFIG;
  }
  const bool staged = path == MP_XFER_PATH_STAGED;
  const bool one_trip = (flags & MP_XFER_ASYNC) && !staged;
  const int j0 = kind == 1 ? 0 : 2 * l0;
  const int nj = kind == 1 ? src->nch : 2 * (l1 - l0);
  RingGeom geom;
  if (staged) {
    geom = ring_geom(src->staging_bytes, src->staging_slots, r->staging_bytes, r->staging_slots,
                     (int64_t)nj * src->chunk);
    if (geom.k < 1) {
      set_err("staging slot smaller than one block");
      return MP_ERR_CONFIG;
    }
  }
  // inbound one-round-trip transfers prepared after this point are not
  // joined while this transfer is issued (mp_pool::join_bound)
  const uint64_t start_stamp = src->prep_stamp;
  Channel* c = r->out;
  // ---- request: the receiver allocates ----
  Writer wr{c->req_payload(), kChanCap};
  wr.put<uint32_t>(flags);
  if (kind == 1) {
    wr.put<int64_t>(n_tok);
    wr.bytes(toks, n_tok * (int64_t)sizeof(mp_token));
  }
  wr.put<int64_t>(n);
  if (flags & MP_XFER_DST_GIVEN) wr.bytes(da, n * (int64_t)sizeof(mp_addr));
  wr.put<int64_t>(priv_len);
  wr.bytes(priv, priv_len);
  wr.put<int32_t>(j0);
  wr.put<int32_t>(nj);
  wr.bytes(smeds.data(), n);
  if (!wr.ok) {
    set_err("request larger than the mailbox");
    return MP_ERR_BUFFER_TOO_SMALL;
  }
  // Pin our indexed source blocks while we wait: serving the peer's own
  // requests meanwhile must not evict them.
  std::vector<mpi::Node*> pinned;
  for (size_t i = 0; i < sids.size(); ++i) {
    mpi::Node* nd = src->index->owner(smeds[i], sids[i]);
    if (nd) {
      src->index->set_ref(nd, nd->ref + 1);
      pinned.push_back(nd);
    }
  }
  auto unpin = [&]() { unpin_nodes(src, pinned); };
  const bool tm = timing_on();
  double t0 = tm ? now_s() : 0.0;
  const uint64_t s1 = ++c->next_req;
  publish(c->req(), kind == 1 ? REQ_TWI : REQ_XFER, 0, wr.len, s1);
  // the previous call's pipelined copy is launched while the peer prepares
  // this one (before any inbound request is served: wait_reply may serve),
  // unless this transfer may join it (same peer, path and layers, payload
  // under the pool's coalescing limit, no inbound transfer stamped since it
  // started -- wait_reply serves only requests stamped after this start)
  // ... and only while the GPU is busy for a while yet: an idle data stream,
  // or one whose queued copies are about to drain (host estimate), gets the
  // pending copy now (like the in-process batches), so merging never holds
  // back work the device could already be doing
  PendingTx* pt = src->pend_tx;
  const bool may_merge =
      pt && one_trip && (flags & MP_XFER_PIPELINE) && src->coalesce && pt->r == r &&
      pt->path == path && (path == MP_XFER_PATH_AUTO || path == MP_XFER_PATH_FUSED) &&
      pt->j0 == j0 && pt->nj == nj && pt->start_stamp == start_stamp &&
      pt->bytes + (uint64_t)n * (uint64_t)nj * (uint64_t)src->chunk <= src->batch_limit &&
      (!src->idle_flush || (host_clock() + 50e-6 < src->track->busy_until &&
                            cudaStreamQuery(src->stream) == cudaErrorNotReady));
  const mp_status fs = may_merge ? MP_OK : remote_flush_tx(src);
  mp_status st = wait_reply(src, c, s1);
  if (st == MP_OK && fs != MP_OK) st = fs;
  if (tm) {
    const double t = now_s();
    g_phase.add(0, t - t0);
    t0 = t;
  }
  if (st != MP_OK) {
    unpin();
    return st;
  }
  SlotHdr* rp = c->rep();
  if (rp->status != MP_OK) {
    unpin();
    return (mp_status)rp->status;
  }
  Reader rd{c->rep_payload(), (int64_t)rp->len};
  const int64_t skip = rd.get<int64_t>();
  const int64_t nm = rd.get<int64_t>();
  const int32_t* dids = (const int32_t*)rd.bytes(nm * 4);
  cudaIpcMemHandle_t ring_hnd{};
  uint64_t ring_id = 0;
  uint32_t slot0 = 0;
  const uint32_t prep_seq = rd.get<uint32_t>();
  const uint32_t done_seq = rd.get<uint32_t>();
  int64_t nfin = 0;
  const mp_addr* fin = nullptr;
  if (staged) {
    const void* hp = rd.bytes(sizeof(ring_hnd));
    if (hp) std::memcpy(&ring_hnd, hp, sizeof(ring_hnd));
    ring_id = rd.get<uint64_t>();
    slot0 = rd.get<uint32_t>();
  }
  if (one_trip) {
    nfin = rd.get<int64_t>();
    fin = (const mp_addr*)rd.bytes(nfin * (int64_t)sizeof(mp_addr));
  }
  if (!rd.ok || skip < 0 || skip + nm != n || (staged && slot0 != r->out_slot)) {
    unpin();
    set_err("malformed allocation reply");
    return MP_ERR_INTERNAL;
  }
  // ---- transmission ----
  mp_status xs = MP_OK;
  uint32_t slot_end = slot0;
  {
    DevGuard g(src->dev);
    std::vector<int32_t> hs, hd, ds_, dd_;
    for (int64_t i = skip; i < n; ++i) {
      const bool dram = smeds[(size_t)i] == MP_DRAM;
      (dram ? ds_ : hs).push_back(sids[(size_t)i]);
      (dram ? dd_ : hd).push_back(dids[i - skip]);
    }
    if (staged) {
      slot_end = slot0 + (uint32_t)(((int64_t)hs.size() + geom.k - 1) / geom.k);
      r->out_slot = slot_end;  // the receiver has queued its unpacks for all of them
      if (!hs.empty() && r->peer_ring_id != ring_id) {
        if (r->peer_ring) cudaIpcCloseMemHandle(r->peer_ring);
        r->peer_ring = nullptr;
        void* m = nullptr;
        if (cudaIpcOpenMemHandle(&m, ring_hnd, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
          cudaGetLastError();
          set_err("cudaIpcOpenMemHandle of the peer's inbound ring failed");
          xs = MP_ERR_CUDA;
        } else {
          r->peer_ring = (char*)m;
          r->peer_ring_id = ring_id;
        }
      }
    }
    PendingTx* pm = src->pend_tx;
    if (pm && may_merge && xs == MP_OK) {
      // one launch for both only if (1) this transfer's prepare flag is
      // already up: the merged copy then waits for nothing new (a prepare
      // still queued on the peer's stream may sit behind a join on another
      // sender's copy that waits for the pending one -- merging would close
      // that cycle), and (2) no destination block repeats (the peer evicted
      // and re-allocated a block of the pending copy: stream order between
      // the two copies must decide it)
      bool ok = (int32_t)(__atomic_load_n(r->out_sync->h + kSyncPrep, __ATOMIC_ACQUIRE) -
                          prep_seq) >= 0;
      if (ok) {
        std::vector<int32_t> a(pm->hd);
        a.insert(a.end(), pm->dd.begin(), pm->dd.end());
        std::sort(a.begin(), a.end());
        for (int32_t d : hd) ok = ok && !std::binary_search(a.begin(), a.end(), d);
        for (int32_t d : dd_) ok = ok && !std::binary_search(a.begin(), a.end(), d);
      }
      if (!ok) xs = remote_flush_tx(src);
    }
    pm = src->pend_tx;
    if (pm && xs == MP_OK) {  // merge: the later prepare / done values cover both
      pm->hs.insert(pm->hs.end(), hs.begin(), hs.end());
      pm->hd.insert(pm->hd.end(), hd.begin(), hd.end());
      pm->ds.insert(pm->ds.end(), ds_.begin(), ds_.end());
      pm->dd.insert(pm->dd.end(), dd_.begin(), dd_.end());
      pm->prep_seq = prep_seq;
      pm->done_seq = done_seq;
      pm->pinned.insert(pm->pinned.end(), pinned.begin(), pinned.end());
      pinned.clear();
      pm->nm += nm;
      pm->bytes += (uint64_t)nm * (uint64_t)nj * (uint64_t)src->chunk;
    } else if (one_trip && (flags & MP_XFER_PIPELINE) && xs == MP_OK) {
      // enqueued by this pool's next call (remote_flush_tx); the indexed
      // sources stay pinned until then
      PendingTx* t = new PendingTx();
      t->r = r;
      t->path = path;
      t->j0 = j0;
      t->nj = nj;
      t->hs.swap(hs);
      t->hd.swap(hd);
      t->ds.swap(ds_);
      t->dd.swap(dd_);
      t->prep_seq = prep_seq;
      t->done_seq = done_seq;
      t->start_stamp = start_stamp;
      t->pinned.swap(pinned);
      t->nm = nm;
      t->bytes = (uint64_t)nm * (uint64_t)nj * (uint64_t)src->chunk;
      src->pend_tx = t;
    } else {
      xs = transmit_step(src, r, path, j0, nj, hs, hd, ds_, dd_, geom, slot0, slot_end, prep_seq,
                         done_seq, start_stamp, xs);
      if (xs == MP_OK && !one_trip && !(flags & MP_XFER_ASYNC)) xs = sync(src);
      src->stats.blocks_moved += (uint64_t)nm;
    }
  }
  if (tm) {
    const double t = now_s();
    g_phase.add(1, t - t0);
    t0 = t;
  }
  if (one_trip) {  // committed at the receiver's allocation step: no second round trip
    unpin();
    if (xs != MP_OK) return xs;
    std::memcpy(da, fin, (size_t)nfin * sizeof(mp_addr));
    if (n_moved) *n_moved = nm;
    return MP_OK;
  }
  // ---- notify; the receiver inserts and answers ok ----
  Writer w2{c->req_payload(), kChanCap};
  w2.put<int32_t>((int32_t)xs);
  const uint64_t s2 = ++c->next_req;
  publish(c->req(), REQ_DONE, 0, w2.len, s2);
  st = wait_reply(src, c, s2);
  if (tm) g_phase.add(2, now_s() - t0);
  unpin();
  if (st != MP_OK) return st;
  if (xs != MP_OK) return xs;
  rp = c->rep();
  if (rp->status != MP_OK) return (mp_status)rp->status;
  Reader r2{c->rep_payload(), (int64_t)rp->len};
  const int64_t nf2 = r2.get<int64_t>();
  const void* f2 = r2.bytes(nf2 * (int64_t)sizeof(mp_addr));
  if (!r2.ok) {
    set_err("malformed completion reply");
    return MP_ERR_INTERNAL;
  }
  std::memcpy(da, f2, (size_t)nf2 * sizeof(mp_addr));
  if (n_moved) *n_moved = nm;
  return MP_OK;
}

// --------------------------------------------------------- export / import
namespace {

constexpr uint32_t kHandleMagic = 0x3148504Du;  // "MPH1"
constexpr int kMaxSlabs = 512;

struct WireHandle {
  uint32_t magic, version;
  int32_t inst, dev, L, H, D, elem, B, nch;
  int64_t n_hbm, chunk;
  int64_t staging_bytes;  // STAGED ring geometry
  int32_t staging_slots, pad0;
  uint64_t uid;
  char bus_id[32];
  int32_t n_allocs, pad;
  cudaIpcMemHandle_t allocs[kMaxSlabs];
  int32_t slab_alloc[kMaxSlabs];
  int64_t slab_off[kMaxSlabs];
};

typedef int (*GetAddressRangeFn)(unsigned long long*, size_t*, unsigned long long);

mp_status alloc_base(void* ptr, char** base) {
  static GetAddressRangeFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !f) {
      set_err("cuMemGetAddressRange unavailable");
      return MP_ERR_CUDA;
    }
    fn = (GetAddressRangeFn)f;
  }
  unsigned long long b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, (unsigned long long)(uintptr_t)ptr) != 0) {
    set_err("cuMemGetAddressRange failed (slab not from cudaMalloc?)");
    return MP_ERR_CONFIG;
  }
  *base = (char*)(uintptr_t)b;
  return MP_OK;
}

std::string chan_name(uint64_t from, uint64_t to) {
  char buf[64];
  snprintf(buf, sizeof(buf), "/mpc_%016llx_%016llx", (unsigned long long)from,
           (unsigned long long)to);
  return buf;
}

std::string sync_name(uint64_t from, uint64_t to) {
  char buf[64];
  snprintf(buf, sizeof(buf), "/mps_%016llx_%016llx", (unsigned long long)from,
           (unsigned long long)to);
  return buf;
}

}  // namespace

bool remote_trace_on() {
  static const bool on = [] {
    const char* e = getenv("MP_REMOTE_TRACE");
    return e && e[0] == '1';
  }();
  return on;
}

void remote_dump_state(const mp_pool* p, const char* where) {
  fprintf(stderr, "[mempool trace] pool %d stalled in %s (pid %d)\n", p->inst, where,
          (int)getpid());
  for (const auto& kv : p->remotes) {
    const RemotePeer* r = kv.second;
    fprintf(stderr,
            "  peer %d: prep_seq(in)=%u in_seq=%u out_slot=%u in_slot=%u async_in=%zu "
            "(front stamp %llu seq %u) join_bound=%llu prep_stamp=%llu recv_join=%d\n",
            r->inst, r->prep_seq, r->in_seq, r->out_slot, r->in_slot, r->async_in.size(),
            r->async_in.empty() ? 0ull : (unsigned long long)r->async_in.front().first,
            r->async_in.empty() ? 0u : r->async_in.front().second,
            (unsigned long long)p->join_bound, (unsigned long long)p->prep_stamp,
            (int)r->recv_join);
    for (int d = 0; d < 2; ++d) {
      const SyncPage* s = d ? r->in_sync : r->out_sync;
      if (!s) continue;
      const uint32_t* h = s->h;
      fprintf(stderr, "    %s page: done=%u prep=%u ready=[", d ? "in " : "out",
              __atomic_load_n(h + kSyncDone, __ATOMIC_ACQUIRE),
              __atomic_load_n(h + kSyncPrep, __ATOMIC_ACQUIRE));
      for (int k = 0; k < 8; ++k) fprintf(stderr, "%u ", __atomic_load_n(h + kSyncReady + k, __ATOMIC_ACQUIRE));
      fprintf(stderr, "] free=[");
      for (int k = 0; k < 8; ++k) fprintf(stderr, "%u ", __atomic_load_n(h + kSyncFree + k, __ATOMIC_ACQUIRE));
      fprintf(stderr, "]\n");
    }
  }
}

namespace {
template <class Q>
cudaError_t poll_traced(const mp_pool* p, Q query, const char* where) {
  const double t0 = now_s();
  bool dumped = false;
  for (;;) {
    const cudaError_t e = query();
    if (e != cudaErrorNotReady) return e;
    if (!dumped && now_s() - t0 > 10.0) {
      remote_dump_state(p, where);
      dumped = true;
    }
    std::this_thread::yield();
  }
}
}  // namespace

cudaError_t sync_stream_traced(const mp_pool* p, cudaStream_t s, const char* where) {
  if (!remote_trace_on()) return cudaStreamSynchronize(s);
  return poll_traced(p, [&] { return cudaStreamQuery(s); }, where);
}

cudaError_t sync_event_traced(const mp_pool* p, cudaEvent_t e, const char* where) {
  if (!remote_trace_on()) return cudaEventSynchronize(e);
  return poll_traced(p, [&] { return cudaEventQuery(e); }, where);
}

// Releases everything one peer connection opened (mappings, ring, streams,
// mailboxes, flag pages).
static void remote_close_one(mp_pool* p, RemotePeer* r) {
  {
    DevGuard g(p->dev);
    if (r->recv_stream) cudaStreamSynchronize(r->recv_stream);
    if (r->d_slabs) cudaFree(r->d_slabs);
    for (void* m : r->mapped) cudaIpcCloseMemHandle(m);
    if (r->peer_ring) cudaIpcCloseMemHandle(r->peer_ring);
    if (r->ring) cudaFree(r->ring);
    if (r->recv_dep) cudaEventDestroy(r->recv_dep);
    if (r->recv_ev) cudaEventDestroy(r->recv_ev);
    if (r->recv_stream) cudaStreamDestroy(r->recv_stream);
  }
  chan_close(r->out, true);
  chan_close(r->in, true);
  sync_close(r->out_sync);
  sync_close(r->in_sync);
  delete r;
}

void remote_close_all(mp_pool* p) {
  if (!p->remotes.empty()) remote_report_timing();
  host_report_timing();
  for (auto& kv : p->remotes) remote_close_one(p, kv.second);
  p->remotes.clear();
}

uint64_t new_uid() {
  std::random_device rd;
  uint64_t u = ((uint64_t)rd() << 32) ^ rd() ^ ((uint64_t)getpid() << 16) ^
               (uint64_t)std::chrono::steady_clock::now().time_since_epoch().count();
  return u ? u : 1;
}

}  // namespace mp

using namespace mp;

extern "C" {

mp_status mp_export_handle(mp_pool* p, void* buf, int64_t cap, int64_t* len) {
  if (!p) return MP_ERR_CONFIG;
  if (len) *len = (int64_t)sizeof(WireHandle);
  if (!buf || cap < (int64_t)sizeof(WireHandle)) return MP_ERR_BUFFER_TOO_SMALL;
  if (p->nch > kMaxSlabs) return MP_ERR_CONFIG;
  DevGuard g(p->dev);
  WireHandle* h = new WireHandle();
  std::memset(h, 0, sizeof(*h));
  h->magic = kHandleMagic;
  h->version = 3;
  h->inst = p->inst;
  h->dev = p->dev;
  h->L = p->L;
  h->H = p->H;
  h->D = p->D;
  h->elem = p->elem;
  h->B = p->B;
  h->nch = p->nch;
  h->n_hbm = p->n_hbm;
  h->chunk = p->chunk;
  h->staging_bytes = p->staging_bytes;
  h->staging_slots = p->staging_slots;
  h->uid = p->uid;
  if (cudaDeviceGetPCIBusId(h->bus_id, sizeof(h->bus_id), p->dev) != cudaSuccess) {
    delete h;
    set_err("cudaDeviceGetPCIBusId failed");
    return MP_ERR_CUDA;
  }
  std::vector<char*> bases;
  for (int j = 0; j < p->nch; ++j) {
    char* base = nullptr;
    mp_status s = alloc_base(p->slabs[(size_t)j], &base);
    if (s != MP_OK) {
      delete h;
      return s;
    }
    int k = 0;
    while (k < (int)bases.size() && bases[(size_t)k] != base) ++k;
    if (k == (int)bases.size()) {
      bases.push_back(base);
      if (cudaIpcGetMemHandle(&h->allocs[k], base) != cudaSuccess) {
        delete h;
        set_err("cudaIpcGetMemHandle failed for a slab allocation");
        return MP_ERR_CUDA;
      }
    }
    h->slab_alloc[j] = k;
    h->slab_off[j] = p->slabs[(size_t)j] - base;
  }
  h->n_allocs = (int32_t)bases.size();
  std::memcpy(buf, h, sizeof(*h));
  delete h;
  return MP_OK;
}

mp_status mp_import_peer(mp_pool* p, const void* buf, int64_t len) {
  if (!p || !buf || len < (int64_t)sizeof(WireHandle)) return MP_ERR_CONFIG;
  TRY(remote_flush_tx(p));
  WireHandle* h = new WireHandle();
  std::memcpy(h, buf, sizeof(*h));
  auto fail = [&](mp_status s, const char* why) {
    set_err(why);
    delete h;
    return s;
  };
  if (h->magic != kHandleMagic || h->version != 3) return fail(MP_ERR_CONFIG, "bad handle");
  if (h->inst == p->inst || p->peers.count(h->inst) || p->remotes.count(h->inst))
    return fail(MP_ERR_CONFIG, "instance id already known");
  if (h->L != p->L || h->chunk != p->chunk || h->B != p->B || h->nch != p->nch)
    return fail(MP_ERR_CONFIG, "pools have different KV shapes");
  DevGuard g(p->dev);
  RemotePeer* r = new RemotePeer();
  r->inst = h->inst;
  r->dev = h->dev;
  r->uid = h->uid;
  char mine[32] = {0};
  cudaDeviceGetPCIBusId(mine, sizeof(mine), p->dev);
  r->same_device = std::strncmp(mine, h->bus_id, sizeof(mine)) == 0 && !p->force_peer;
  r->bmarks.reset((size_t)h->n_hbm);
  r->staging_bytes = h->staging_bytes;
  r->staging_slots = h->staging_slots;
  bool ok = true;
  for (int k = 0; k < h->n_allocs && ok; ++k) {
    void* m = nullptr;
    ok = cudaIpcOpenMemHandle(&m, h->allocs[k], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
    if (ok) r->mapped.push_back(m);
  }
  std::vector<char*> slabs((size_t)h->nch);
  for (int j = 0; ok && j < h->nch; ++j)
    slabs[(size_t)j] = (char*)r->mapped[(size_t)h->slab_alloc[j]] + h->slab_off[j];
  r->slabs_h = slabs;
  if (ok) ok = cudaMalloc(&r->d_slabs, sizeof(char*) * (size_t)h->nch) == cudaSuccess;
  if (ok)
    ok = cudaMemcpy(r->d_slabs, slabs.data(), sizeof(char*) * (size_t)h->nch,
                    cudaMemcpyHostToDevice) == cudaSuccess;
  if (ok) {
    r->out = chan_open(chan_name(p->uid, r->uid));
    r->in = chan_open(chan_name(r->uid, p->uid));
    ok = r->out && r->in;
  }
  if (ok) {
    r->out_sync = sync_open(sync_name(p->uid, r->uid));
    r->in_sync = sync_open(sync_name(r->uid, p->uid));
    ok = r->out_sync && r->in_sync;
  }
  if (!ok) {
    // release what this import opened; the pool's other peers stay connected
    std::string why = std::string("import failed: ") + cudaGetErrorString(cudaGetLastError());
    remote_close_one(p, r);
    return fail(MP_ERR_CUDA, why.c_str());
  }
  p->remotes[r->inst] = r;
  delete h;
  return MP_OK;
}

mp_status mp_serve(mp_pool* p, int64_t timeout_ms, int32_t until_mark, int64_t* served,
                   int32_t* mark) {
  if (!p) return MP_ERR_CONFIG;
  TRY(remote_flush_tx(p));  // a pipelined copy goes first (the peer may wait for it)
  const double t0 = now_s();
  int64_t total = 0;
  int spins = 0;
  for (;;) {
    if (until_mark && !p->marks.empty()) break;
    int64_t k = 0;
    TRY(remote_serve_once(p, &k));
    total += k;
    if (!until_mark && k == 0 && timeout_ms == 0) break;
    if (k == 0 && ++spins > 64) {
      std::this_thread::yield();
      spins = 0;
      if (timeout_ms >= 0 && (now_s() - t0) * 1e3 > (double)timeout_ms) break;
    }
  }
  if (served) *served = total;
  if (mark) {
    if (!p->marks.empty()) {
      *mark = p->marks.front();
      p->marks.erase(p->marks.begin());
    } else {
      *mark = -1;
    }
  }
  return MP_OK;
}

mp_status mp_send_mark(mp_pool* p, int32_t dst_instance, int32_t tag) {
  if (!p) return MP_ERR_CONFIG;
  TRY(remote_flush_tx(p));
  auto it = p->remotes.find(dst_instance);
  if (it == p->remotes.end()) return MP_ERR_DST_UNREACHABLE;
  Channel* c = it->second->out;
  Writer wr{c->req_payload(), kChanCap};
  wr.put<int32_t>(tag);
  const uint64_t s = ++c->next_req;
  publish(c->req(), REQ_MARK, 0, wr.len, s);
  return wait_reply(p, c, s);
}

// Test hook (no GPU needed): two processes exchange n messages through one
// mailbox; role 0 sends and checks the echo, role 1 echoes n messages.
mp_status mp_debug_channel_selftest(const char* name, int32_t role, int64_t n_msgs,
                                    int64_t payload) {
  if (!name || n_msgs < 0 || payload < 0 || payload > kChanCap) return MP_ERR_CONFIG;
  Channel* c = chan_open(name);
  if (!c) return MP_ERR_CONFIG;
  mp_status st = MP_OK;
  std::mt19937_64 rng(12345);
  for (int64_t k = 0; k < n_msgs && st == MP_OK; ++k) {
    const int64_t len = payload ? (int64_t)(rng() % (uint64_t)payload) + 1 : 0;
    if (role == 0) {
      std::vector<unsigned char> msg((size_t)len);
      for (auto& b : msg) b = (unsigned char)rng();
      std::memcpy(c->req_payload(), msg.data(), (size_t)len);
      const uint64_t s = ++c->next_req;
      publish(c->req(), REQ_ECHO, 0, len, s);
      st = wait_reply(nullptr, c, s);
      if (st == MP_OK) {
        SlotHdr* rp = c->rep();
        if ((int64_t)rp->len != len || rp->type != REP_ECHO) st = MP_ERR_INTERNAL;
        for (int64_t i = 0; st == MP_OK && i < len; ++i)
          if ((unsigned char)c->rep_payload()[i] != (unsigned char)(msg[(size_t)i] ^ 0x5A))
            st = MP_ERR_INTERNAL;
      }
    } else {
      for (int64_t i = 0; i < len; ++i) (void)rng();
      const double t0 = now_s();
      while (__atomic_load_n(&c->req()->seq, __ATOMIC_ACQUIRE) <= c->seen_req) {
        std::this_thread::yield();
        if (now_s() - t0 > 60.0) {
          st = MP_ERR_DST_UNREACHABLE;
          break;
        }
      }
      if (st != MP_OK) break;
      SlotHdr* q = c->req();
      const uint64_t seq = __atomic_load_n(&q->seq, __ATOMIC_ACQUIRE);
      c->seen_req = seq;
      const int64_t n = (int64_t)q->len;
      for (int64_t i = 0; i < n; ++i) c->rep_payload()[i] = (char)(c->req_payload()[i] ^ 0x5A);
      publish(c->rep(), REP_ECHO, 0, n, seq);
    }
  }
  chan_close(c, role == 0);
  return st;
}

}  // extern "C"
