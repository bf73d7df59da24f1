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
//  * the transmission is one-sided: the receiver's slabs and its id arena are
//    CUDA-IPC mapped into the sender, whose fused gather->store kernel writes
//    the scattered source chunks straight into the receiver's freshly
//    allocated blocks over NVLink (or HBM when both processes share a GPU),
//    reading the destination block table the receiver's device allocator
//    wrote -- no staging, no per-block calls, no ordering thread (the paper's
//    NCCL send/recv needs one per communicator);
//  * the two processes' streams are ordered with interprocess CUDA events:
//    the sender's copy waits for the receiver's allocation, the receiver's
//    later work waits for the sender's copy.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

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
namespace {

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
      mp_status s = flush_involving(p);
      if (s == MP_OK && !rd.ok) s = MP_ERR_CONFIG;
      if (s == MP_OK && r->has_pending) s = MP_ERR_PRECONDITION;
      if (s != MP_OK) {
        // nothing prepared
      } else if (q->type == REQ_TWI)
        s = dst_prepare_twi(p, r->inst, toks, n_tok, m, flags, given, priv, plen, &r->pending);
      else
        s = dst_prepare_xfer(p, r->inst, m, flags, given, priv, plen, &r->pending);
      if (s == MP_OK) {
        r->has_pending = true;
        // the sender's copy must follow this allocation and every earlier use
        // of the blocks on this pool's streams, including other peers' copies
        // into them (a block freed and re-allocated); its own earlier copies
        // are ordered by its stream already
        for (auto& kv2 : p->remotes) {
          RemotePeer* o = kv2.second;
          if (o == r || !o->inbound_pending) continue;
          if (cudaStreamWaitEvent(p->stream, o->ev, 0) != cudaSuccess) s = MP_ERR_CUDA;
          o->inbound_pending = false;
        }
        if (s == MP_OK) s = meta_fence(p);
        if (s == MP_OK && cudaEventRecord(p->ev_ipc, p->stream) != cudaSuccess) s = MP_ERR_CUDA;
      }
      rtype = REP_PREP;
      rstatus = s;
      if (s == MP_OK) {
        wr.put<int64_t>(r->pending.skip);
        wr.put<int64_t>(r->pending.nm);
        wr.put<int64_t>(r->pending.d_dst_off);
        wr.bytes(r->pending.dids.data(), (int64_t)r->pending.dids.size() * 4);
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
      if (sender_status != MP_OK) {  // the transmission failed on the sender:
        // release what the allocation step took (pins, fresh blocks)
        dst_abort(p, r->pending);
        rstatus = sender_status;
        break;
      }
      // later data-stream work of this pool must follow the sender's copy:
      // applied lazily (remote_apply_waits), not chained into the next
      // allocation the sender waits for
      r->inbound_pending = true;
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
  while (__atomic_load_n(&c->rep()->seq, __ATOMIC_ACQUIRE) < seq) {
    int64_t served = 0;
    if (self) {
      mp_status s = remote_serve_once(self, &served);
      if (s != MP_OK) return s;
    }
    if (!served && ++spins > 64) {
      std::this_thread::yield();
      spins = 0;
      if (now_s() - t0 > kTimeout) {
        set_err("remote peer did not answer (is it inside mp_serve?)");
        return MP_ERR_DST_UNREACHABLE;
      }
    }
  }
  return MP_OK;
}

}  // namespace

mp_status remote_apply_waits(mp_pool* p) {
  for (auto& kv : p->remotes) {
    RemotePeer* r = kv.second;
    if (!r->inbound_pending) continue;
    DevGuard g(p->dev);
    CK(cudaStreamWaitEvent(p->stream, r->ev, 0));
    r->inbound_pending = false;
  }
  return MP_OK;
}

mp_status remote_serve_once(mp_pool* p, int64_t* served) {
  *served = 0;
  for (auto& kv : p->remotes) {
    RemotePeer* r = kv.second;
    if (!r->in) continue;
    mp_status s = serve_message(p, r);
    if (s == MP_OK) ++*served;
    else if (s != MP_ERR_PRECONDITION) return s;
  }
  return MP_OK;
}

// ------------------------------------------------------------ sender side
mp_status remote_transfer(mp_pool* src, RemotePeer* r, int kind, const mp_token* toks,
                          int64_t n_tok, const std::vector<int32_t>& sids,
                          const std::vector<uint8_t>& smeds, int64_t n, mp_addr* da,
                          uint32_t flags, int32_t l0, int32_t l1, const void* priv,
                          int64_t priv_len, int64_t* n_moved) {
  const uint32_t path = flags & MP_XFER_PATH_MASK;
  if (path != MP_XFER_PATH_AUTO && path != MP_XFER_PATH_FUSED) {
    set_err("cross-process transfers use the fused one-sided path");
    return MP_ERR_CONFIG;
  }
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
  mp_status st = wait_reply(src, c, s1);
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
  const int64_t off = rd.get<int64_t>();
  const int32_t* dids = (const int32_t*)rd.bytes(nm * 4);
  if (!rd.ok || skip < 0 || skip + nm != n) {
    unpin();
    set_err("malformed allocation reply");
    return MP_ERR_INTERNAL;
  }
  // ---- transmission: one-sided stores into the receiver's blocks ----
  mp_status xs = MP_OK;
  {
    DevGuard g(src->dev);
    // HBM-resident sources and (memory asymmetry) sources swapped
    // out to our pinned DRAM, each with its destination ids
    std::vector<int32_t> hs, hd, ds_, dd_;
    bool mixed = false;
    for (int64_t i = skip; i < n; ++i) {
      const bool dram = smeds[(size_t)i] == MP_DRAM;
      mixed = mixed || dram;
      (dram ? ds_ : hs).push_back(sids[(size_t)i]);
      (dram ? dd_ : hd).push_back(dids[i - skip]);
    }
    const int j0 = kind == 1 ? 0 : 2 * l0;
    const int nj = kind == 1 ? src->nch : 2 * (l1 - l0);
    xs = flush_involving(src);
    if (xs == MP_OK && cudaStreamWaitEvent(src->stream, r->ev, 0) != cudaSuccess) xs = MP_ERR_CUDA;
    if (xs == MP_OK && !hs.empty()) {
      int* d_s = nullptr;
      const int* d_d = nullptr;
      mpk::InlineIds si;
      xs = src_ids(src, hs, &d_s, &si);
      if (xs == MP_OK) {
        if (off >= 0 && !mixed) {
          d_d = r->arena + off;  // the receiver's device allocator output, IPC mapped
        } else {
          int* t = nullptr;
          xs = upload_ids(src, hd, &t);
          d_d = t;
        }
      }
      if (xs == MP_OK)
        // a receiver process on this same GPU: its IPC-mapped pool is local
        // HBM, so the copy takes the loopback engine (bulk ring, claiming)
      {
        const LaunchBlocks lb{&src->bmarks, hs.data(), &r->bmarks, hd.data(), (int64_t)hs.size()};
        xs = launch_migrate_timed(src, src->stream, pool_ep(src->d_slabs, d_s),
                                  pool_ep(r->d_slabs, d_d), (int64_t)hs.size(), j0, nj,
                                  /*peer=*/!r->same_device, 0, si.n ? &si : nullptr, true, &lb);
      }
    }
    if (xs == MP_OK && !ds_.empty()) {
      int *d_s = nullptr, *d_d = nullptr;
      mpk::InlineIds si;
      xs = src_ids(src, ds_, &d_s, &si);
      if (xs == MP_OK) xs = upload_ids(src, dd_, &d_d);
      if (xs == MP_OK)
        xs = launch_migrate_timed(src, src->stream,
                                  agg_ep(src->dram_dev + (int64_t)j0 * src->chunk, src->Pb, d_s),
                                  pool_ep(r->d_slabs, d_d), (int64_t)ds_.size(), j0, nj,
                                  /*peer=*/true, 0, si.n ? &si : nullptr);
    }
    if (xs == MP_OK && cudaEventRecord(src->ev_ipc, src->stream) != cudaSuccess) xs = MP_ERR_CUDA;
    if (xs == MP_OK && !(flags & MP_XFER_ASYNC)) xs = sync(src);
    src->stats.blocks_moved += (uint64_t)nm;
  }
  if (tm) {
    const double t = now_s();
    g_phase.add(1, t - t0);
    t0 = t;
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
  const int64_t nfin = r2.get<int64_t>();
  const void* fin = r2.bytes(nfin * (int64_t)sizeof(mp_addr));
  if (!r2.ok) {
    set_err("malformed completion reply");
    return MP_ERR_INTERNAL;
  }
  std::memcpy(da, fin, (size_t)nfin * sizeof(mp_addr));
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
  uint64_t uid;
  char bus_id[32];
  int32_t n_allocs, pad;
  cudaIpcMemHandle_t allocs[kMaxSlabs];
  int32_t slab_alloc[kMaxSlabs];
  int64_t slab_off[kMaxSlabs];
  cudaIpcMemHandle_t arena;
  cudaIpcEventHandle_t ev;
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

}  // namespace

void remote_close_all(mp_pool* p) {
  if (!p->remotes.empty()) remote_report_timing();
  host_report_timing();
  for (auto& kv : p->remotes) {
    RemotePeer* r = kv.second;
    {
      DevGuard g(p->dev);
      if (r->d_slabs) cudaFree(r->d_slabs);
      for (void* m : r->mapped) cudaIpcCloseMemHandle(m);
      if (r->arena) cudaIpcCloseMemHandle(r->arena);
      if (r->ev) cudaEventDestroy(r->ev);
    }
    chan_close(r->out, true);
    chan_close(r->in, true);
    delete r;
  }
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
  h->version = 1;
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
  if (cudaIpcGetMemHandle(&h->arena, p->ar.d) != cudaSuccess ||
      cudaIpcGetEventHandle(&h->ev, p->ev_ipc) != cudaSuccess) {
    delete h;
    set_err("cudaIpcGet*Handle failed (arena / event)");
    return MP_ERR_CUDA;
  }
  std::memcpy(buf, h, sizeof(*h));
  delete h;
  return MP_OK;
}

mp_status mp_import_peer(mp_pool* p, const void* buf, int64_t len) {
  if (!p || !buf || len < (int64_t)sizeof(WireHandle)) return MP_ERR_CONFIG;
  WireHandle* h = new WireHandle();
  std::memcpy(h, buf, sizeof(*h));
  auto fail = [&](mp_status s, const char* why) {
    set_err(why);
    delete h;
    return s;
  };
  if (h->magic != kHandleMagic || h->version != 1) return fail(MP_ERR_CONFIG, "bad handle");
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
  r->same_device = std::strncmp(mine, h->bus_id, sizeof(mine)) == 0;
  r->bmarks.reset((size_t)h->n_hbm);
  bool ok = true;
  for (int k = 0; k < h->n_allocs && ok; ++k) {
    void* m = nullptr;
    ok = cudaIpcOpenMemHandle(&m, h->allocs[k], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
    if (ok) r->mapped.push_back(m);
  }
  std::vector<char*> slabs((size_t)h->nch);
  for (int j = 0; ok && j < h->nch; ++j)
    slabs[(size_t)j] = (char*)r->mapped[(size_t)h->slab_alloc[j]] + h->slab_off[j];
  void* ar = nullptr;
  if (ok) ok = cudaIpcOpenMemHandle(&ar, h->arena, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
  r->arena = (int*)ar;
  if (ok) ok = cudaIpcOpenEventHandle(&r->ev, h->ev) == cudaSuccess;
  if (ok) ok = cudaMalloc(&r->d_slabs, sizeof(char*) * (size_t)h->nch) == cudaSuccess;
  if (ok)
    ok = cudaMemcpy(r->d_slabs, slabs.data(), sizeof(char*) * (size_t)h->nch,
                    cudaMemcpyHostToDevice) == cudaSuccess;
  if (ok) {
    r->out = chan_open(chan_name(p->uid, r->uid));
    r->in = chan_open(chan_name(r->uid, p->uid));
    ok = r->out && r->in;
  }
  if (!ok) {
    std::string why = std::string("import failed: ") + cudaGetErrorString(cudaGetLastError());
    p->remotes[r->inst] = r;  // let remote_close_all release what was opened
    remote_close_all(p);
    return fail(MP_ERR_CUDA, why.c_str());
  }
  p->remotes[r->inst] = r;
  delete h;
  return MP_OK;
}

mp_status mp_serve(mp_pool* p, int64_t timeout_ms, int32_t until_mark, int64_t* served,
                   int32_t* mark) {
  if (!p) return MP_ERR_CONFIG;
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
