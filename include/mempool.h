/*
 * mempool.h -- C-ABI of libmempool.so: the KV-block migration hot path of
 * MemServe's elastic memory pool (MemPool), rebuilt for B200 (sm_100a).
 *
 * Source of every entry point: PAPER.md Table tbl-mempool-api (P:261-290,
 * "Elastic Memory Pool APIs. Type can be HBM-only, DRAM-only, or mixed. Each
 * address encodes instance ID. Transfer flags can control on-demand
 * allocation."), §4.2 indexing, §4.3 transfer workflow
 * (P:360-369), §5.2 block aggregation; SPEC.md signatures/errors
 * (S:125-203).  Where the paper is silent the behaviour follows the
 * readings R1-R17 in DESIGN.md §3.
 *
 * Conventions (apply to every function):
 *  - All array arguments are HOST pointers owned by the caller; the library
 *    never keeps a caller pointer past the call, except the slab and DRAM
 *    pointers given to mp_pool_create, which must outlive the pool.
 *  - A negative mp_status means NO state change (all-or-nothing) and output
 *    counts/arrays are written only on MP_OK.  MP_ERR_CUDA is the exception:
 *    a CUDA failure leaves the pool in an unspecified state (call
 *    mp_last_error() for the CUDA message and destroy the pool).
 *  - One caller thread per pool at a time; a transfer uses both
 *    pools and must not race with calls on either.
 *  - Calls are synchronous by default: they return after the device work
 *    they issued has completed (transfers: after the data landed and the
 *    receiver inserted).  With MP_XFER_ASYNC a transfer returns once
 *    its work is enqueued on the pools' streams (host-side bookkeeping -- the
 *    receiver's allocation, insert and `private` delivery -- is already done);
 *    mp_sync(pool) waits for it.  Every later call on either pool is
 *    stream-ordered after it, and mp_alloc_mem drains the pool before handing
 *    blocks to the caller (unless MP_ALLOC_STREAM_ORDERED, see there).  Frees
 *    of HBM blocks (and mp_alloc_mem's claims) are applied to the device
 *    bitmap lazily, stream-ordered before the pool's next device allocation.
 *  - The pools of one process on one device share one data stream (migrations
 *    between them need no cross-stream wait; MP_SHARED_STREAM=0 gives each
 *    pool its own), so mp_sync on one of them also waits for the others' work,
 *    and pools of one device driven by different threads serialise their
 *    data movement on that stream (it is HBM-bound either way).  The stream
 *    is created with the device's first pool and destroyed with its last.
 *  - Layout: the HBM pool of an instance is 2*L "slabs" (K_0, V_0, K_1, V_1,
 *    ...), each hbm_blocks chunks of c = B*H*D*elem bytes (vLLM's per-layer
 *    paged layout: "two blocks per LLM layer").  Block id b is chunk b
 *    of every slab.  The DRAM pool and all staging buffers use the
 *    AGGREGATED layout: block i is one contiguous Pb = 2*L*c byte
 *    region, ordered layer-major, K before V (reading R11).
 */
#ifndef MEMPOOL_H
#define MEMPOOL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mp_pool mp_pool; /* opaque; one per serving instance */

/* Block address ("Each address encodes instance ID"):
 * bits [63:40] instance id, [39:32] medium (0 = HBM, 1 = DRAM), [31:0] index. */
typedef uint64_t mp_addr;
typedef int32_t mp_token; /* token ids */

#define MP_ADDR(inst, medium, idx)                                              \
  ((((uint64_t)(uint32_t)(inst)) << 40) | (((uint64_t)(medium) & 0xFF) << 32) | \
   (uint64_t)(uint32_t)(idx))
#define MP_ADDR_INST(a) ((int32_t)((a) >> 40))
#define MP_ADDR_MEDIUM(a) ((int32_t)(((a) >> 32) & 0xFF))
#define MP_ADDR_INDEX(a) ((int32_t)((a)&0xFFFFFFFFu))

typedef enum { MP_HBM = 0, MP_DRAM = 1, MP_MIXED = 2 } mp_medium;

typedef enum {
  MP_OK = 0,
  MP_ERR_OOM = -1,             /* S:129 OutOfMemory (after eviction attempt) */
  MP_ERR_DOUBLE_FREE = -2,     /* S:139 DoubleFree */
  MP_ERR_INVALID_ADDR = -3,    /* S:139 InvalidAddr: wrong instance / medium / range */
  MP_ERR_ADDR_COUNT = -4,      /* S:149 AddrCountMismatch */
  MP_ERR_CONFLICT = -5,        /* S:149 ConflictingMapping (MP_INS_ERR_ON_CONFLICT only) */
  MP_ERR_NO_DRAM = -6,         /* S:189 NoDramCapacity */
  MP_ERR_DST_OOM = -7,         /* S:255 DstOutOfMemory */
  MP_ERR_DST_UNREACHABLE = -8, /* S:255 DstUnreachable: instance not connected */
  MP_ERR_PRECONDITION = -9,    /* S:202 precondition violated (wrong state/medium) */
  MP_ERR_PREFIX_MISSING = -10, /* R3: receiver lacks the prefix a suffix send needs */
  MP_ERR_CONFIG = -11,         /* bad argument / incompatible pools */
  MP_ERR_BUFFER_TOO_SMALL = -12,
  MP_ERR_CUDA = -13,
  MP_ERR_NCCL = -14,
  MP_ERR_INTERNAL = -15        /* self-check failed (e.g. device allocator vs host shadow) */
} mp_status;

/* ---- flags ("Transfer flags can control on-demand allocation") ---- */
#define MP_XFER_DST_GIVEN (1u << 0) /* dst_addrs is an INPUT: skip the allocation step */
#define MP_XFER_DEDUP (1u << 1)     /* receiver matches first, moves only what it lacks (R3) */
#define MP_XFER_ASYNC (1u << 2)     /* return once enqueued; complete with mp_sync (see above) */
/* With MP_XFER_ASYNC to a peer in ANOTHER process (ignored otherwise): the
 * call returns after the receiver's allocation reply (its allocation, insert
 * and `private` delivery are done, the final addrs are returned) and the copy
 * is enqueued by this pool's NEXT library call -- right after that call's own
 * request is sent, so the launch overlaps the next round trip -- or by any
 * call other than mp_match / mp_recv_poll / the getters and dumps, which
 * enqueue it before anything else.  Consecutive pipelined FUSED transfers to
 * the same peer (same layers, no inbound transfer in between, no destination
 * block repeated) join the pending copy while the sender's data stream is
 * busy -- one launch per coalescing limit (coalesce_mib) instead of one per
 * transfer; on an idle stream the next transfer enqueues the pending copy.  Until it is enqueued the
 * peer's later device work on those blocks waits; a sender that stops
 * calling must call mp_sync.  Cross-process MP_XFER_ASYNC (FUSED / CE)
 * commits at the receiver in the one round trip, before the copy is
 * enqueued: if the sender's enqueue then fails (a CUDA error in practice:
 * the id arena cannot run short), the receiver's index already names the
 * blocks, and both pools are in the unspecified state of MP_ERR_CUDA (the
 * peer's waits are released). */
#define MP_XFER_PIPELINE (1u << 3)
#define MP_INS_ERR_ON_CONFLICT (1u << 4) /* insert: CONFLICT instead of keep-existing (R4) */
#define MP_MATCH_PIN (1u << 5)      /* match: pin matched blocks until mp_unpin (R12) */
/* Transport selection (benchmarks / comparisons; default AUTO = FUSED). */
#define MP_XFER_PATH_SHIFT 8
#define MP_XFER_PATH_MASK (0xFu << MP_XFER_PATH_SHIFT)
#define MP_XFER_PATH_AUTO (0u << MP_XFER_PATH_SHIFT)
#define MP_XFER_PATH_FUSED (1u << MP_XFER_PATH_SHIFT)  /* one gather->store kernel, no staging (A6f) */
#define MP_XFER_PATH_STAGED (2u << MP_XFER_PATH_SHIFT) /* pack -> copy -> unpack (A4, A5, A6) */
#define MP_XFER_PATH_CE (3u << MP_XFER_PATH_SHIFT)     /* copy engines, one memcpy per chunk (library baseline) */
/* Swap transport (mp_swap_out / mp_swap_in flags).  Default (0): MP_SWAP_CE
 * when the pool's staging buffer holds at least one block, else zero-copy. */
#define MP_SWAP_ZERO_COPY (1u << 0) /* SM loads/stores straight to mapped pinned DRAM */
#define MP_SWAP_CE (2u << 0)        /* pack into device staging + one copy-engine D2H/H2D
                                       per block (staging_bytes must hold >= 1 block) */

typedef struct {
  int32_t instance_id;  /* < 2^24; encoded in every mp_addr */
  int32_t device;       /* CUDA ordinal of this instance's HBM */
  int32_t layers;       /* L   (1..256) */
  int32_t kv_heads;     /* H */
  int32_t head_dim;     /* D */
  int32_t elem_bytes;   /* 2 for fp16/bf16 KV */
  int32_t block_tokens; /* B (16 in the paper) */
  int32_t verify;       /* 1: cross-check device allocator ids against the host shadow */
  int64_t hbm_blocks;   /* N_hbm (< 2^31) */
  int64_t dram_blocks;  /* N_dram (may be 0) */
  /* 2*layers device pointers (K_0, V_0, K_1, ...), each >= hbm_blocks*c bytes,
   * 16-byte aligned, caller-owned (e.g. torch tensors); NULL: the library
   * allocates one region of 2*L*hbm_blocks*c bytes with cudaMalloc. */
  void* const* slabs;
  /* pinned (cudaHostAlloc / cudaHostRegister) host region of dram_blocks*Pb
   * bytes, caller-owned; NULL: the library cudaHostAllocs it. */
  void* dram_base;
  int64_t staging_bytes; /* device staging for the STAGED path (0: 256 MiB) */
  int32_t staging_slots; /* ring depth (0: 4, at most 64) */
  int32_t max_ctas;      /* cap on migration kernel CTAs (0: auto = one full wave) */
  int32_t copy_kernel;   /* copy engine: 0 auto (bulk cp.async ring within this GPU's HBM,
                            vector LD/ST for pinned DRAM and peer memory), 1 vector, 2 bulk */
  int32_t coalesce_mib;  /* launch coalescing of same-device fused transfers into this pool:
                            one launch per batch, flushed when the data stream is idle, at
                            this many MiB, or when anything else touches either pool;
                            0: 4096 MiB, < 0: off (one launch per transfer) */
  int32_t peer_engine;   /* copy engine of stores into a peer's memory (another GPU over
                            NVLink, or another process's IPC-mapped pool): 0 auto (vector
                            LD/ST, or MP_PEER_ENGINE=bulk), 1 vector, 2 bulk cp.async ring */
  int32_t peer_sched;    /* work split of those stores: 0 auto (static, or
                            MP_PEER_SCHED=dynamic), 1 static, 2 dynamic unit claiming */
  int32_t force_peer;    /* test knob: treat a peer on the same GPU (in-process pool or
                            IPC-imported process) as one on another GPU, so the peer
                            dispatch (peer_engine / peer_sched, one-sided stores from the
                            sender's stream) runs -- and is parity-tested -- on one GPU */
} mp_pool_config;

typedef struct {
  int64_t chunk_bytes, block_bytes; /* c and Pb */
  int64_t hbm_blocks, dram_blocks, hbm_free, dram_free;
  int64_t index_blocks;             /* blocks owned by the prompt index */
  uint64_t clock;                   /* R7 logical clock */
  uint64_t epoch;                   /* fill counter (content model) */
  int32_t instance_id, device, layers, block_tokens;
} mp_pool_info;

typedef struct {
  uint64_t kernel_launches;   /* migration kernels launched (all flows) */
  uint64_t bytes_moved;       /* algorithmic payload bytes moved (all flows) */
  uint64_t blocks_moved;
  double kernel_ms;           /* summed CUDA-event time of migration kernels (profiling on) */
  uint64_t timed_launches;    /* launches included in kernel_ms */
  uint64_t timed_bytes;       /* payload bytes of those launches */
  uint64_t aux_launches;      /* allocator / free / fill kernels launched */
  double gap_ms;              /* data-stream idle time between consecutive timed launches
                                 issued between two syncs (profiling every launch) */
  uint64_t profiled_launches; /* data-stream migration launches while profiling was on
                                 (timed or not) */
  uint64_t profiled_bytes;    /* their payload bytes: kernel_ms * profiled_bytes /
                                 timed_bytes estimates their total time when sampling */
  uint64_t overlapped_launches; /* migrations that started without waiting for the previous
                                   grid on the stream (independent blocks) */
} mp_stats;

typedef struct {
  int32_t kind;        /* 0 = transfer, 1 = transfer_with_insert */
  int32_t src_instance;
  int64_t n_addrs;     /* destination addrs delivered with the message */
  int64_t priv_len;
} mp_recv_msg;

/* ------------------------------ lifecycle ------------------------------ */
mp_status mp_pool_create(const mp_pool_config* cfg, mp_pool** out);
void mp_pool_destroy(mp_pool* pool);
/* In-process link (both directions): after this, each pool can name the other
 * as dst_instance.  Different devices: enables CUDA peer access (NVLink P2P).
 * Instance ids must differ; shapes (L, H, D, elem, B) must match. */
mp_status mp_connect(mp_pool* a, mp_pool* b);
mp_status mp_pool_info_get(const mp_pool* pool, mp_pool_info* out);
/* Wait for every device operation issued on this pool (including
 * MP_XFER_ASYNC transfers that execute on its stream).  In verify mode also
 * checks every device allocation against the host shadow (MP_ERR_INTERNAL). */
mp_status mp_sync(mp_pool* pool);
/* Stream-ordered integration with an inference engine's own CUDA streams
 * (e.g. torch's current stream), without host synchronisation:
 * mp_wait_event: every later device operation of this pool (and of the
 * transfers it takes part in) waits for `cuda_event` (a cudaEvent_t the
 * caller recorded after writing the KV it is about to move -- the per-layer
 * dependency of layer-by-layer transmission);
 * mp_record_event: records `cuda_event` after all work issued so far on this
 * pool (including MP_XFER_ASYNC transfers into it), so a consumer stream can
 * wait for the landed blocks.  The event must belong to the pool's device. */
mp_status mp_wait_event(mp_pool* pool, void* cuda_event);
mp_status mp_record_event(mp_pool* pool, void* cuda_event);
const char* mp_status_str(mp_status s);
const char* mp_last_error(void); /* thread-local detail of the last failure */

/* ------------------------- memory API ------------------------ */
/* alloc_mem(size, type, id): the n lowest-index free blocks, ascending; MIXED
 * takes HBM first then DRAM; on shortage evicts unreferenced
 * historical blocks of that medium first, else MP_ERR_OOM.  HBM ids
 * follow the device bitmap allocator's lowest-first rule; here the host
 * shadow picks them (nothing on the device reads them) and the claim reaches
 * the device bitmap with its next stream-ordered update -- no kernel launch
 * per call.  The receiver's allocations inside a transfer run on the device.
 * requester_id is recorded as the allocating instance.  out: n addrs. */
mp_status mp_alloc_mem(mp_pool* pool, int64_t n, int32_t type, int32_t requester_id,
                       mp_addr* out);
/* OR'd into alloc_mem's `type`: return without draining the pool (the
 * cudaMallocAsync contract).  The blocks may still be read or written by
 * earlier device work of this pool (an MP_XFER_ASYNC transfer of a block that
 * was freed since); the caller orders its own writes after that work by
 * making its stream wait on an event from mp_record_event, and every mp_*
 * operation on these blocks is stream-ordered after it already.  Which
 * blocks are returned is unchanged. */
#define MP_ALLOC_STREAM_ORDERED (1 << 8)
/* free_mem(addrList): only caller-owned (active) blocks; DOUBLE_FREE for a
 * free block or a repeated addr; PRECONDITION for index-owned blocks. */
mp_status mp_free_mem(mp_pool* pool, const mp_addr* addrs, int64_t n);

/* ------------------------- index API ------------------------- */
/* insert(tokenList, addrList, flags): n_addr must be floor(n_tok/B) or
 * ceil(n_tok/B) (a trailing partial-block addr is ignored); existing prefixes
 * keep their mapping and the caller's duplicate block is freed (R4);
 * n_dup_freed (nullable) receives how many were freed. */
mp_status mp_insert(mp_pool* pool, const mp_token* tokens, int64_t n_tok, const mp_addr* addrs,
                    int64_t n_addr, uint32_t flags, int64_t* n_dup_freed);
/* match(tokenList): longest stored block-aligned prefix (R5).  out receives
 * matched_tokens/B addrs (cap >= floor(n_tok/B) required, else
 * BUFFER_TOO_SMALL).  MP_MATCH_PIN pins them (R12). */
mp_status mp_match(mp_pool* pool, const mp_token* tokens, int64_t n_tok, uint32_t flags,
                   mp_addr* out, int64_t cap, int64_t* matched_tokens);
mp_status mp_unpin(mp_pool* pool, const mp_addr* addrs, int64_t n);
/* delete(tokenList): R6 (terminal marker rule); no-op if absent. */
mp_status mp_delete(mp_pool* pool, const mp_token* tokens, int64_t n_tok);
/* evict: up to n LRU leaves of `medium` (R8); out_freed cap >= n. */
mp_status mp_evict(mp_pool* pool, int64_t n, int32_t medium, mp_addr* out_freed,
                   int64_t* n_freed);

/* --------------------------- swap API ------------------------ */
/* swap_out(num_blocks): R9 frontier-LRU victims -> pinned DRAM (aggregated
 * layout), index rewritten, HBM freed.  out_old/out_new: cap >= n. */
mp_status mp_swap_out(mp_pool* pool, int64_t n, uint32_t flags, mp_addr* out_old,
                      mp_addr* out_new, int64_t* n_moved);
/* swap_in(addrList): every addr an allocated DRAM block (else PRECONDITION);
 * new HBM ids lowest-first in input order (R10).  out_new: n addrs. */
mp_status mp_swap_in(mp_pool* pool, const mp_addr* addrs, int64_t n, uint32_t flags,
                     mp_addr* out_new);

/* ------------------------ distributed API -------------------- */
/* transfer(id, srcAddrList, dstAddrList, flags, private): (1) allocation at
 * the receiver unless MP_XFER_DST_GIVEN, (2) transmission of layers
 * [layer_begin, layer_end) of every block (A4-A6 / A10), (3) `private`
 * (priv, priv_len bytes) queued at the receiver (mp_recv_poll).  src addrs
 * are allocated blocks of `src` in HBM or -- swapped out, memory asymmetry
 * in its pinned DRAM, each listed once (R13); DRAM blocks go
 * straight from DRAM to the destination's HBM (no swap_in, no index change
 * at the source): copy-engine H2D into the source's staging and one scatter
 * per slot when the staging holds a block (MP_DRAM_SOURCE=sm in the
 * environment: one kernel reading the mapped DRAM).  The destination is
 * always HBM.  dst_addrs: n entries, output unless DST_GIVEN. */
mp_status mp_transfer(mp_pool* src, int32_t dst_instance, const mp_addr* src_addrs, int64_t n,
                      mp_addr* dst_addrs, uint32_t flags, int32_t layer_begin, int32_t layer_end,
                      const void* priv, int64_t priv_len);
/* transfer_with_insert(id, tokenList, srcAddrList, dstAddrList, flags,
 * private): src addrs cover the LAST n of the ceil(n_tok/B) blocks of tokens
 * (R3); the receiver allocates, receives and inserts, all layers.
 * dst_addrs (output, ceil(n_tok/B) entries) receives the final receiver addr
 * of every block; with MP_XFER_DST_GIVEN it is an INPUT of n entries.
 * n_moved (nullable): blocks actually moved (fewer with MP_XFER_DEDUP). */
mp_status mp_transfer_with_insert(mp_pool* src, int32_t dst_instance, const mp_token* tokens,
                                  int64_t n_tok, const mp_addr* src_addrs, int64_t n,
                                  mp_addr* dst_addrs, uint32_t flags, const void* priv,
                                  int64_t priv_len, int64_t* n_moved);
/* Receiver side of `private` delivery: pops the oldest message.  Returns
 * MP_ERR_PRECONDITION when the queue is empty; BUFFER_TOO_SMALL (message kept)
 * when priv_cap < priv_len or addr_cap < n_addrs.  Every transfer into a pool
 * queues one message (its kind, sender, final addrs and `private` bytes); a
 * receiver that never polls keeps them all (host memory, ~8 bytes per block
 * plus the payload), so a long-running engine polls or the pool owner drains. */
mp_status mp_recv_poll(mp_pool* dst, mp_recv_msg* out, void* priv_buf, int64_t priv_cap,
                       mp_addr* addrs, int64_t addr_cap);

/* ------------- asymmetric parallelism ------------- */
/* Layout reading R16: inside a chunk the KV is head-major ([H][B][D], vLLM's
 * paged cache puts the head dimension before the in-block token dimension),
 * so heads [h0, h0+k) of a chunk are one contiguous range of k*B*D*elem bytes.
 * A tensor-parallel instance of TP degree t is t pools (one per GPU), rank r
 * holding heads [r*H/t, (r+1)*H/t) of every layer ("the KV head
 * dimension is split evenly by tp ratio").
 *
 * mp_transfer_heads: copy heads [src_head0, src_head0+n_heads) of layers
 * [layer_begin, layer_end) of n HBM source blocks into heads [dst_head0, ...)
 * of n caller-given (active) destination blocks of an in-process peer whose
 * kv_heads may differ (same L, B, D, elem).  The destination is an input
 * (MP_XFER_DST_GIVEN implied); MP_XFER_ASYNC allowed; DEDUP / path flags are
 * CONFIG.  One fused sub-chunk gather->store kernel (peer stores over NVLink
 * when the pools are on different GPUs). */
mp_status mp_transfer_heads(mp_pool* src, int32_t dst_instance, const mp_addr* src_addrs,
                            int64_t n, const mp_addr* dst_addrs, uint32_t flags,
                            int32_t src_head0, int32_t dst_head0, int32_t n_heads,
                            int32_t layer_begin, int32_t layer_end);
/* The repartition plan TP=p -> TP=q for H heads: every overlapping
 * (src rank, dst rank) pair as 5 ints (src_rank, dst_rank, src_head0 within
 * the source shard, dst_head0 within the destination shard, n_heads); the
 * pieces cover each head exactly once.  H must be divisible by p and q
 * (else CONFIG).  out may be NULL to query n_pieces; cap counts pieces. */
mp_status mp_tp_plan(int32_t H, int32_t p, int32_t q, int32_t* out, int64_t cap,
                     int64_t* n_pieces);

/* ------------- global scheduler: global prompt trees ---------- */
/* Host-only (no device work).  One block-granular prompt tree per instance
 * kind (0 prefill-only, 1 decode-only, 2 PD-colocated); each node
 * records which instances hold that prefix and until when (update time +
 * ttl).  Readings R17: an instance's cached prefix
 * for a prompt is the deepest path node it holds unexpired; route() picks,
 * among registered instances of `kind`, the longest cached prefix,
 * ties to the least load then the lowest id, and lists every instance (any
 * kind) holding a longer prefix than the pick -- the "extra historical KV"
 * holders -- longest first, with their prefix lengths; the
 * chosen instance can fetch those blocks with a suffix transfer_with_insert
 * from the holder (R3).  Time is an explicit argument (seconds). */
typedef struct mp_gs mp_gs;
mp_status mp_gs_create(int32_t block_tokens, double ttl_seconds, mp_gs** out);
void mp_gs_destroy(mp_gs* gs);
mp_status mp_gs_register(mp_gs* gs, int32_t instance, int32_t kind);
mp_status mp_gs_set_load(mp_gs* gs, int32_t instance, double load);
/* Update path (a response returned): `instance` holds the prompt's
 * full blocks as of `now`. */
mp_status mp_gs_update(mp_gs* gs, int32_t instance, const mp_token* tokens, int64_t n_tok,
                       double now);
/* Lookup path.  DST_UNREACHABLE if no instance of `kind` is registered;
 * extra_inst / extra_tokens may be NULL (then only n_extra is written);
 * BUFFER_TOO_SMALL if more than cap extra holders. */
mp_status mp_gs_route(mp_gs* gs, int32_t kind, const mp_token* tokens, int64_t n_tok, double now,
                      int32_t* instance, int64_t* matched_tokens, int32_t* extra_inst,
                      int64_t* extra_tokens, int64_t cap, int64_t* n_extra);

/* ------------------- multi-process (one process per GPU) ----------------- */
/* Serialize what a pool in ANOTHER process needs to reach this one: CUDA-IPC
 * handles of the slab allocations (slabs must come from cudaMalloc, e.g. the
 * torch caching allocator), the shape, the staging geometry and a random
 * pool uid (names of the pair's mailboxes and flag pages).  len receives the size; call
 * with buf = NULL to query it.  The blob is plain bytes (exchange it with
 * torch.distributed / any transport). */
mp_status mp_export_handle(mp_pool* pool, void* buf, int64_t cap, int64_t* len);
/* Map a peer's exported pool: its slabs and arena are opened with
 * cudaIpcOpenMemHandle (peer access over NVLink when on another GPU), and the
 * pair's two shared-memory mailboxes and two pinned flag pages (monotonic
 * sequence numbers that the two GPUs' streams raise and wait on) are
 * created / opened.  Both sides import each other.  Afterwards
 * mp_transfer / mp_transfer_with_insert accept the peer's instance id as
 * dst_instance: the caller's process sends the request, the peer's process
 * executes the receiver's half of the workflow (allocation, insertion;
 * P:361-365) inside mp_serve -- or inside any of its own blocking transfer
 * calls -- and the caller's process moves the blocks one-sided into the
 * peer's IPC-mapped memory with any transport: FUSED (one kernel storing
 * into the peer's slabs; engine and split from peer_engine / peer_sched),
 * CE (one copy-engine memcpy per chunk) or STAGED (pack, one copy per slot
 * into the peer's IPC-exported inbound ring, unpacked by the peer's recv
 * stream; slots handed over by device-side flags).  Shapes must match. */
mp_status mp_import_peer(mp_pool* pool, const void* buf, int64_t len);
/* Receiver loop: serve requests of imported peers until an end-of-batch
 * mark arrives (until_mark != 0) or timeout_ms elapses (< 0: no timeout;
 * 0 with until_mark == 0: one non-blocking pass).  served (nullable): requests
 * served; mark (nullable): the mark's tag, or -1 if none arrived. */
mp_status mp_serve(mp_pool* pool, int64_t timeout_ms, int32_t until_mark, int64_t* served,
                   int32_t* mark);
/* Send an end-of-batch mark (tag) to an imported peer; returns once the
 * peer's mp_serve has taken it. */
mp_status mp_send_mark(mp_pool* src, int32_t dst_instance, int32_t tag);
/* Test hook, no GPU needed: two processes exchange n_msgs messages of up to
 * payload bytes through one shared-memory mailbox `name` (role 0 sends and
 * verifies the echo, role 1 echoes). */
mp_status mp_debug_channel_selftest(const char* name, int32_t role, int64_t n_msgs,
                                    int64_t payload);

/* ---------------- building blocks (A4 pack / A6 unpack) ------------------ */
/* Gather layers [l0, l1) of n HBM blocks into device buffer `staging`
 * (aggregated layout [n][l1-l0][2][c]); unpack is the inverse scatter into
 * caller-owned (active) HBM blocks.  `staging` is a device pointer on the
 * pool's device of >= n*(l1-l0)*2*c bytes. */
mp_status mp_pack(mp_pool* pool, const mp_addr* addrs, int64_t n, int32_t l0, int32_t l1,
                  void* staging);
mp_status mp_unpack(mp_pool* pool, const void* staging, const mp_addr* addrs, int64_t n,
                    int32_t l0, int32_t l1);

/* ------------------------- measurement / debug --------------------------- */
/* Profiling: every `every`-th migration kernel on the pool's data stream
 * (every = 1: all of them; 0: off) is bracketed by CUDA events on that
 * stream; mp_stats accumulates their durations.  Completed events are
 * harvested without blocking, so profiling adds no host synchronisation;
 * sampling (every > 1) keeps the events' own cost (a few us per launch)
 * out of short-launch workloads. */
mp_status mp_profile(mp_pool* pool, int32_t every);
mp_status mp_stats_get(const mp_pool* pool, mp_stats* out);
mp_status mp_stats_reset(mp_pool* pool);
/* Synthetic KV write (stand-in for the engine's prefill; content model of
 * DESIGN.md §4): one epoch per call; word t of chunk j of block b becomes
 * splitmix64(seed ^ splitmix64(inst<<40 | epoch<<14 | b) ^ (j*c/8 + t)).
 * addrs: allocated HBM blocks, index < 2^14. */
mp_status mp_debug_fill(mp_pool* pool, const mp_addr* addrs, int64_t n, uint64_t seed);
/* Copy one block (HBM or DRAM) to host in the aggregated layout (Pb bytes). */
mp_status mp_debug_read_block(mp_pool* pool, mp_addr addr, void* host_out, int64_t cap);
/* Sorted text dump of the index, one line per block:
 * "<depth>\t<medium>\t<idx>\t<last_access>\t<ref>\t<terminal>\t<tok,tok,...>"
 * where the tokens are the full prefix.  len receives the byte length
 * (without NUL); BUFFER_TOO_SMALL if cap <= len. */
mp_status mp_debug_dump_index(mp_pool* pool, char* buf, int64_t cap, int64_t* len);
/* Host shadow block states (0 free, 1 active, 2 indexed, 3 orphan). */
mp_status mp_debug_block_states(mp_pool* pool, int32_t medium, uint8_t* out, int64_t cap);
/* Device bitmap (bit = 1: free) copied to host, (hbm_blocks+31)/32 words. */
mp_status mp_debug_bitmap(mp_pool* pool, uint32_t* out, int64_t cap_words);

#ifdef __cplusplus
}
#endif
#endif /* MEMPOOL_H */
