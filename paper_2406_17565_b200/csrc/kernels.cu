// kernels.cu -- sm_100a kernels of libmempool.
//
//  * migrate_kernel / migrate_bulk_kernel : the KV-block gather/scatter of
//    the migration path -- pack (A4, pool -> aggregated staging), unpack (A6,
//    staging -> pool), the fused gather -> (peer) store (A6f, pool -> pool,
//    P2P over NVLink when the destination slabs live on a peer GPU) and
//    DRAM-side copies (A8/A9, mapped pinned DRAM).  HBM-bound: every chunk is
//    a contiguous run of c bytes (c = B*H*D*2 = 128 KiB at Llama-2-7B).
//    Two engines: 16-byte vector LD/ST (4 KiB warp units) and a
//    cp.async.bulk (TMA) ring through shared memory (64 KiB units, one
//    elected lane per CTA, the default inside one GPU's HBM).  Units are
//    claimed dynamically from a per-pool device counter (the fast SMs take
//    more); short id lists (source, and destination when both fit) come by
//    value in the launch parameters, longer ones from id tables (the
//    destination table is the device allocator's output).  Launched with
//    programmatic dependent launch: the next migration's CTAs start as this
//    one drains and wait at griddepcontrol.wait.
//  * alloc_kernel / free_kernel : the device-resident block allocator
//    (BASELINE.json north_star item 1) over a bitmap, lowest-first; pending
//    updates (frees, and claims the host made for mp_alloc_mem) ride in the
//    allocation kernel's parameters.
//  * fill_kernel : test/bench-only synthetic KV writer (content model).
#include <atomic>
#include <cstdlib>
#include <utility>

#include "kernels.cuh"

namespace mpk {

namespace {

constexpr int kThreads = 256;
constexpr int kVec = 8;                      // 16-byte vectors per lane per unit
constexpr int kUnitBytes = 32 * kVec * 16;   // 4 KiB per warp-unit

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream(void* p, const uint4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// Start of the copied range of chunk (block id, slab j = j0 + jr) on one side.
template <bool kPool>
__device__ __forceinline__ char* chunk_ptr(const Endpoint& e, unsigned j, unsigned jr,
                                           long long id) {
  return kPool ? (char*)__ldg((const unsigned long long*)(e.slabs + j)) + id * e.cstride + e.off
               : e.base + id * e.stride + (long long)jr * e.cstride + e.off;
}

// Source block id of copy slot i: from the launch parameters when the host
// passed the (short) list inline, else from the id table, else i itself.
__device__ __forceinline__ long long src_id(const Endpoint& src, const InlineIds& sinl,
                                            unsigned i) {
  if (sinl.n) return sinl.ids[i];
  return src.ids ? __ldg(src.ids + i) : (long long)i;
}

// Destination block id of copy slot i: inline after the source ids, else
// from the id table, else i itself.
__device__ __forceinline__ long long dst_id(const Endpoint& dst, const InlineIds& sinl,
                                            unsigned i) {
  if (sinl.nd) return sinl.ids[sinl.n + i];
  return dst.ids ? __ldg(dst.ids + i) : (long long)i;
}

// Programmatic dependent launch (PDL): a migration launched right behind
// another on the same stream is scheduled while that one drains its tail;
// griddepcontrol.wait holds it until the previous grid has completed and its
// stores are visible (a no-op without a programmatic dependency), and each CTA
// of the running grid releases its dependents once it has claimed its last
// unit.  Nothing global is touched before the wait: the dynamic-claiming
// counter is shared by consecutive launches.
// Independent launches (the host found no block the previous launches of its
// window write and this one reads or writes, or the other way round) skip the
// wait at the start and overlap the previous grid's tail.  Every grid still
// waits before its CTAs exit, so a grid completes only after its predecessor
// has: completion stays ordered along the stream, and a later launch that
// does wait at its start sees every earlier grid complete.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_release() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Copies `len` bytes per chunk (the whole chunk, or a head range of it).
constexpr unsigned kGroup = 8;  // units per dynamic claim (32 KiB per warp)

// 3 CTAs x 256 threads per SM (85 registers): 96 KiB of loads in flight per
// SM, more than HBM or NVLink needs, and no register spills (at 4 CTAs the
// 64-register cap spilled 20 bytes per thread).
template <bool kSrcPool, bool kDstPool>
__global__ void __launch_bounds__(kThreads, 3) migrate_kernel(Endpoint src, Endpoint dst, int j0,
                                                           int nj, long long len,
                                                           unsigned units_per_chunk,
                                                           unsigned total_units,
                                                           const __grid_constant__ InlineIds sinl,
                                                           unsigned long long* ctr,
                                                           unsigned long long base,
                                                           int wait_prev) {
  const unsigned lane = threadIdx.x & 31u;
  const unsigned warp = (blockIdx.x * (unsigned)kThreads + threadIdx.x) >> 5;
  const unsigned nwarps = (gridDim.x * (unsigned)kThreads) >> 5;
  const bool full_units = (len % kUnitBytes) == 0;
  if (wait_prev) pdl_wait();
  const long long chunk = len;
  auto copy_unit = [&](unsigned u) {
    const unsigned ch = u / units_per_chunk;
    const unsigned part = u - ch * units_per_chunk;
    const unsigned i = ch / (unsigned)nj;
    const unsigned jr = ch - i * (unsigned)nj;
    const long long sid = src_id(src, sinl, i);
    const long long did = dst_id(dst, sinl, i);
    const char* sp = chunk_ptr<kSrcPool>(src, j0 + jr, jr, sid);
    char* dp = chunk_ptr<kDstPool>(dst, j0 + jr, jr, did);
    const long long off = (long long)part * kUnitBytes + lane * 16;
    uint4 v[kVec];
    if (full_units) {
#pragma unroll
      for (int k = 0; k < kVec; ++k) v[k] = ld_stream(sp + off + k * 512);
#pragma unroll
      for (int k = 0; k < kVec; ++k) st_stream(dp + off + k * 512, v[k]);
    } else {
#pragma unroll
      for (int k = 0; k < kVec; ++k)
        if (off + k * 512 < chunk) v[k] = ld_stream(sp + off + k * 512);
#pragma unroll
      for (int k = 0; k < kVec; ++k)
        if (off + k * 512 < chunk) st_stream(dp + off + k * 512, v[k]);
    }
  };
  if (!ctr) {  // static grid-stride split
    for (unsigned u = warp; u < total_units; u += nwarps) copy_unit(u);
    pdl_release();
    if (threadIdx.x == 0) pdl_wait();  // complete only after the previous grid
    return;
  }
  // dynamic: warp w starts on group w; later groups (nwarps + claim) come
  // from lane 0's atomicAdd, issued while the current group is copied so the
  // thousands of warps' claims queue behind copies, not in front of them.
  // One failing claim per warp: the launcher advances `base` by
  // max(groups - warps, 0) + warps.
  const unsigned long long ngroups = (total_units + kGroup - 1) / kGroup;
  unsigned long long g = warp;
  for (;;) {
    unsigned long long next = 0;
    if (lane == 0) next = nwarps + (atomicAdd(ctr, 1ull) - base);
    if (g < ngroups) {
      const unsigned u0 = (unsigned)g * kGroup;
      const unsigned u1 = min(u0 + kGroup, total_units);
      for (unsigned u = u0; u < u1; ++u) copy_unit(u);
    }
    g = __shfl_sync(0xffffffffu, next, 0);
    if (g >= ngroups) break;
  }
  pdl_release();
  if (threadIdx.x == 0) pdl_wait();  // complete only after the previous grid
}

// ---------------------------------------------------------------------------
// Bulk-copy (TMA engine) variant of the same gather/scatter.  One elected
// lane per CTA drives a ring of kStages shared-memory stages:
//   cp.async.bulk global -> shared  (completes on an mbarrier, tx-count bytes)
//   cp.async.bulk shared -> global  (bulk_group; wait_group.read frees a stage)
// so each SM keeps (kStages-1) x kPiece bytes of loads plus the stores in
// flight with a handful of instructions; the copy itself never touches the
// register file.  Work unit = one kPiece-byte piece of one chunk (the last
// piece of a chunk may be shorter; chunks are multiples of 16 B).
// (kPiece, kStages) are template parameters; see bulk_cfg() for the choices.
constexpr int kBulkThreads = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_load(void* smem, const void* gmem, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(smem)),
      "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_store(void* gmem, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem),
               "r"(smem_u32(smem)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// The same two copies with an L2 cache-policy hint (createpolicy), for the
// MP_BULK_HINT measurement knob: the KV is read once and written once.
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void bulk_load_hint(void* smem, const void* gmem, uint32_t bytes,
                                               uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(smem)),
      "l"(gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void bulk_store_hint(void* gmem, const void* smem, uint32_t bytes,
                                                uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::
                   "l"(gmem),
               "r"(smem_u32(smem)), "r"(bytes), "l"(pol)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int kPieceT, bool kSrcPool, bool kDstPool>
__device__ __forceinline__ void unit_addr(const Endpoint& src, const Endpoint& dst,
                                          const InlineIds& sinl, int j0, int nj,
                                          long long chunk, unsigned pieces_per_chunk, unsigned u,
                                          const char** sp, char** dp, uint32_t* bytes) {
  const unsigned ch = u / pieces_per_chunk;
  const unsigned part = u - ch * pieces_per_chunk;
  const unsigned i = ch / (unsigned)nj;
  const unsigned jr = ch - i * (unsigned)nj;
  const long long sid = src_id(src, sinl, i);
  const long long did = dst_id(dst, sinl, i);
  const long long off = (long long)part * kPieceT;
  *sp = chunk_ptr<kSrcPool>(src, j0 + jr, jr, sid) + off;
  *dp = chunk_ptr<kDstPool>(dst, j0 + jr, jr, did) + off;
  const long long rest = chunk - off;  // chunk == bytes copied per chunk
  *bytes = (uint32_t)(rest < kPieceT ? rest : kPieceT);
}

// Work distribution: static round-robin (unit u_k = blockIdx.x + k*gridDim.x)
// or, with a device counter, dynamic -- each CTA claims its next unit with
// one atomicAdd issued a full ring turn before the unit is needed, so SMs
// that see slower HBM (the far die) simply take fewer units and the launch
// ends when the LAST unit lands, not when the slowest static share does.  The
// counter is never reset: the launch is given its start value (`base`), and
// every CTA makes exactly one failing claim, so the host advances base by
// total + grid per launch (launches on one stream are serialised).
struct UnitSource {
  unsigned long long* ctr;
  unsigned long long base;
  unsigned total, next, stride;
  __device__ __forceinline__ unsigned claim() {
    if (ctr) {
      const unsigned long long g = atomicAdd(ctr, 1ull) - base;
      return g < total ? (unsigned)g : 0xFFFFFFFFu;
    }
    const unsigned u = next;
    next += stride;
    return u < total ? u : 0xFFFFFFFFu;
  }
};

template <int kPiece, int kStages, bool kSrcPool, bool kDstPool>
__global__ void __launch_bounds__(kBulkThreads) migrate_bulk_kernel(
    Endpoint src, Endpoint dst, int j0, int nj, long long chunk, unsigned pieces_per_chunk,
    unsigned total_units, unsigned long long* ctr, unsigned long long base,
    const __grid_constant__ InlineIds sinl, int wait_prev, int hint) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bars[kStages];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (wait_prev) pdl_wait();
  const uint64_t pol = hint ? l2_evict_first() : 0;
  const bool hl = hint & 1, hs = hint & 2;  // hint the loads / the stores
  UnitSource units{ctr, base, total_units, blockIdx.x, gridDim.x};
  const char* sp;
  char* dp;
  uint32_t bytes;
  char* dsts[kStages];
  uint32_t lens[kStages];
  bool live[kStages];
  // prime the ring
  unsigned u = units.claim();
  for (int k = 0; k < kStages; ++k) {
    live[k] = u != 0xFFFFFFFFu;
    if (!live[k]) continue;
    unit_addr<kPiece, kSrcPool, kDstPool>(src, dst, sinl, j0, nj, chunk, pieces_per_chunk, u, &sp, &dp,
                                          &bytes);
    dsts[k] = dp;
    lens[k] = bytes;
    mbar_expect_tx(&bars[k], bytes);
    if (hl) bulk_load_hint(smem + (size_t)k * kPiece, sp, bytes, &bars[k], pol);
    else bulk_load(smem + (size_t)k * kPiece, sp, bytes, &bars[k]);
    u = units.claim();  // in flight while the loads are
  }
  bool released = false;
  if (u == 0xFFFFFFFFu) {  // nothing left to claim: only the ring's tail remains
    pdl_release();
    released = true;
  }
  // consume stage k % kStages; refill the stage the previous store read from
  for (unsigned k = 0;; ++k) {
    const unsigned s = k % kStages;
    if (!live[s]) break;
    mbar_wait(&bars[s], (k / kStages) & 1u);
    if (hs) bulk_store_hint(dsts[s], smem + (size_t)s * kPiece, lens[s], pol);
    else bulk_store(dsts[s], smem + (size_t)s * kPiece, lens[s]);
    if (k >= 1) {
      const unsigned r = (k - 1) % kStages;
      live[r] = u != 0xFFFFFFFFu;
      if (live[r]) {
        bulk_wait_read<1>();
        unit_addr<kPiece, kSrcPool, kDstPool>(src, dst, sinl, j0, nj, chunk, pieces_per_chunk, u, &sp,
                                              &dp, &bytes);
        dsts[r] = dp;
        lens[r] = bytes;
        mbar_expect_tx(&bars[r], bytes);
        if (hl) bulk_load_hint(smem + (size_t)r * kPiece, sp, bytes, &bars[r], pol);
        else bulk_load(smem + (size_t)r * kPiece, sp, bytes, &bars[r]);
        u = units.claim();
        if (u == 0xFFFFFFFFu && !released) {
          pdl_release();
          released = true;
        }
      }
    }
  }
  bulk_wait_all();
  pdl_wait();  // complete only after the previous grid
}

// Migration launches carry the PDL attribute (MP_PDL=0 turns it off).
static bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("MP_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... Exp, typename... Act>
static cudaError_t launch_pdl(void (*kern)(Exp...), int grid, int block, size_t smem,
                              cudaStream_t stream, Act&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Act>(args)...);
}

// Single CTA (launched with 256 threads): popcount per thread-range of words, block-wide
// exclusive scan, then every thread emits its lowest set bits in order, so
// the ids come out ascending (R2 lowest-first).
// One pending bitmap update: id >= 0 frees (bit := 1), -(id+1) claims (bit := 0).
__device__ __forceinline__ void apply_update(uint32_t* bitmap, int e) {
  if (e >= 0) atomicOr(bitmap + (e >> 5), 1u << (e & 31));
  else atomicAnd(bitmap + ((-e - 1) >> 5), ~(1u << ((-e - 1) & 31)));
}

__global__ void __launch_bounds__(1024) alloc_kernel(uint32_t* bitmap, int nwords, int n,
                                                     int* out_dev, int* out_host, int* err,
                                                     const InlineIds frees) {
  __shared__ int warp_tot[32];
  const int t = threadIdx.x;
  // updates queued since the last allocation go first (lowest-first reuses
  // the frees): id >= 0 sets its bit (a free), -(id+1) clears it (a claim
  // made on the host by mp_alloc_mem); the two sets are disjoint
  for (int i = t; i < frees.n; i += blockDim.x) apply_update(bitmap, frees.ids[i]);
  __syncthreads();
  const int wpt = (nwords + blockDim.x - 1) / blockDim.x;
  const int w0 = min(nwords, t * wpt), w1 = min(nwords, w0 + wpt);
  int cnt = 0;
  for (int w = w0; w < w1; ++w) cnt += __popc(bitmap[w]);
  // inclusive warp scan
  const int lane = t & 31, wid = t >> 5;
  int x = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int s = (lane < (int)(blockDim.x >> 5)) ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    warp_tot[lane] = s;  // inclusive scan of warp totals
  }
  __syncthreads();
  const int base = x - cnt + (wid > 0 ? warp_tot[wid - 1] : 0);
  const int total = warp_tot[(blockDim.x >> 5) - 1];
  if (t == 0 && total < n) *err = 1;
  if (total < n) return;
  int k = base;
  for (int w = w0; w < w1 && k < n; ++w) {
    uint32_t bits = bitmap[w];
    uint32_t taken = 0;
    while (bits && k < n) {
      const int b = __ffs(bits) - 1;
      const int id = w * 32 + b;
      out_dev[k] = id;
      if (out_host) out_host[k] = id;
      ++k;
      taken |= 1u << b;
      bits &= bits - 1;
    }
    bitmap[w] &= ~taken;
  }
}

__global__ void free_inline_kernel(uint32_t* bitmap, const InlineIds frees) {
  for (int i = threadIdx.x; i < frees.n; i += blockDim.x) apply_update(bitmap, frees.ids[i]);
}

__global__ void free_kernel(uint32_t* bitmap, const int* ids, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    apply_update(bitmap, ids[i]);
}

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void fill_kernel(char* const* slabs, const int* ids, int nchunks, long long chunk,
                            unsigned long long seed, unsigned long long inst,
                            unsigned long long epoch, unsigned long long total_pairs) {
  const unsigned long long pairs_per_chunk = (unsigned long long)chunk / 16;
  const unsigned long long words_per_chunk = (unsigned long long)chunk / 8;
  for (unsigned long long g = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
       g < total_pairs; g += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long p = g % pairs_per_chunk;
    const unsigned long long cj = g / pairs_per_chunk;
    const unsigned long long j = cj % nchunks;
    const unsigned long long i = cj / nchunks;
    const unsigned long long b = (unsigned long long)ids[i];
    const unsigned long long tag = (inst << 40) | (epoch << 14) | b;
    const unsigned long long base = seed ^ splitmix64(tag);
    const unsigned long long t = 2 * p;
    const unsigned long long w0 = splitmix64(base ^ (j * words_per_chunk + t));
    const unsigned long long w1 = splitmix64(base ^ (j * words_per_chunk + t + 1));
    ulonglong2* dst = (ulonglong2*)(slabs[j] + b * chunk) + p;
    *dst = make_ulonglong2(w0, w1);
  }
}

}  // namespace

int sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) v = 148;
  return v > 0 ? v : 148;
}

template <int kPieceT, int kStagesT>
static cudaError_t preload_bulk() {
  const int smem = kStagesT * kPieceT;
  void (*ks[4])(Endpoint, Endpoint, int, int, long long, unsigned, unsigned,
                unsigned long long*, unsigned long long, const InlineIds, int, int) = {
      migrate_bulk_kernel<kPieceT, kStagesT, true, true>,
      migrate_bulk_kernel<kPieceT, kStagesT, true, false>,
      migrate_bulk_kernel<kPieceT, kStagesT, false, true>,
      migrate_bulk_kernel<kPieceT, kStagesT, false, false>};
  for (auto k : ks) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    cudaFuncAttributes a;
    e = cudaFuncGetAttributes(&a, k);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t preload_kernels() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::atomic<int> done[64] = {};
  if (dev < 64 && done[dev].load(std::memory_order_acquire)) return cudaSuccess;
  cudaFuncAttributes a;
  const void* plain[] = {(const void*)migrate_kernel<true, true>,
                         (const void*)migrate_kernel<true, false>,
                         (const void*)migrate_kernel<false, true>,
                         (const void*)migrate_kernel<false, false>,
                         (const void*)alloc_kernel, (const void*)free_inline_kernel,
                         (const void*)free_kernel, (const void*)fill_kernel};
  for (const void* k : plain)
    if ((e = cudaFuncGetAttributes(&a, k)) != cudaSuccess) return e;
  if ((e = preload_bulk<65536, 3>()) != cudaSuccess) return e;
  if ((e = preload_bulk<32768, 3>()) != cudaSuccess) return e;
  if ((e = preload_bulk<8192, 6>()) != cudaSuccess) return e;
  if ((e = preload_bulk<16384, 4>()) != cudaSuccess) return e;
  if ((e = preload_bulk<32768, 6>()) != cudaSuccess) return e;
  if ((e = preload_bulk<49152, 4>()) != cudaSuccess) return e;
  if (dev < 64) done[dev].store(1, std::memory_order_release);
  return cudaSuccess;
}

// MP_BULK_SCHED=static turns the dynamic unit claiming off (comparison knob).
static bool bulk_dynamic() {
  static const bool v = [] {
    const char* e = getenv("MP_BULK_SCHED");
    return !(e && e[0] == 's');
  }();
  return v;
}

// Per-device caches of the launch caps (resident CTAs x SMs); pools on other
// threads may launch concurrently, so the slots are atomics.
using CapCache = std::atomic<int>[64];

template <int kPieceT, int kStagesT, bool kSrcPool, bool kDstPool>
static cudaError_t launch_bulk(const Endpoint& src, const Endpoint& dst, int n, int j0, int nj,
                               long long chunk, int max_ctas, cudaStream_t stream,
                               const Sched* sched, const InlineIds& sinl, bool wait_prev) {
  auto kern = migrate_bulk_kernel<kPieceT, kStagesT, kSrcPool, kDstPool>;
  const unsigned pieces = (unsigned)((chunk + kPieceT - 1) / kPieceT);
  const unsigned long long total = (unsigned long long)n * nj * pieces;
  if (total >= (1ull << 32)) return cudaErrorInvalidValue;
  const size_t smem = (size_t)kStagesT * kPieceT;
  int dev = 0;
  cudaGetDevice(&dev);
  static CapCache cached_cap{};  // per device (the smem attribute is per device too)
  int cap = max_ctas;
  const int cached = dev < 64 ? cached_cap[dev].load(std::memory_order_acquire) : 0;
  if (cached <= 0) {
    // idempotent: two threads may both get here the first time
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBulkThreads, smem);
    if (per_sm <= 0) per_sm = 1;
    if (dev < 64) cached_cap[dev].store(per_sm * sm_count(dev), std::memory_order_release);
    if (cap <= 0) cap = per_sm * sm_count(dev);
  } else if (cap <= 0) {
    cap = cached;
  }
  const int grid = (int)(total < (unsigned long long)cap ? total : (unsigned long long)cap);
  const bool dyn = sched && sched->ctr && bulk_dynamic();
  static const int hint = [] {  // MP_BULK_HINT=1: L2 evict_first on loads and stores, 2: loads, 3: stores
    const char* e = getenv("MP_BULK_HINT");
    return (e && e[0] >= '1' && e[0] <= '3') ? (e[0] == '1' ? 3 : e[0] == '2' ? 1 : 2) : 0;
  }();
  const cudaError_t e = launch_pdl(kern, grid, kBulkThreads, smem, stream, src, dst, j0, nj, chunk,
                                   pieces, (unsigned)total, dyn ? sched->ctr : nullptr,
                                   dyn ? *sched->base : 0ull, sinl, wait_prev ? 1 : 0, hint);
  if (dyn && e == cudaSuccess) *sched->base += total + (unsigned long long)grid;
  return e;
}

template <int kPieceT, int kStagesT>
static cudaError_t launch_bulk_any(const Endpoint& src, const Endpoint& dst, int n, int j0,
                                   int nj, long long chunk, int max_ctas, cudaStream_t stream,
                                   const Sched* sc, const InlineIds& si, bool w) {
  const bool sp = src.slabs != nullptr, dp = dst.slabs != nullptr;
  if (sp && dp)
    return launch_bulk<kPieceT, kStagesT, true, true>(src, dst, n, j0, nj, chunk, max_ctas, stream,
                                                      sc, si, w);
  if (sp)
    return launch_bulk<kPieceT, kStagesT, true, false>(src, dst, n, j0, nj, chunk, max_ctas,
                                                       stream, sc, si, w);
  if (dp)
    return launch_bulk<kPieceT, kStagesT, false, true>(src, dst, n, j0, nj, chunk, max_ctas,
                                                       stream, sc, si, w);
  return launch_bulk<kPieceT, kStagesT, false, false>(src, dst, n, j0, nj, chunk, max_ctas,
                                                      stream, sc, si, w);
}


// Ring geometry of the bulk engine; MP_BULK_CFG=<0..5> selects one (tuning
// knob, read once).  Measured on B200 (profiles/kernel_sweep_r01.jsonl):
// 2 GiB scattered 7B copies reach 0.942 of the HBM copy peak with
// 64 KiB x 3 stages (1 CTA / SM, the default), 0.925 with 16 KiB x 4.
//   0 = 64 KiB x 3 (1 CTA / SM)     1 = 32 KiB x 3 (2 CTAs / SM)
//   2 = 8 KiB x 6 (4 CTAs / SM)     3 = 16 KiB x 4 (3 CTAs / SM)
//   4 = 32 KiB x 6 (1 CTA / SM)     5 = 48 KiB x 4 (1 CTA / SM)
// Without the knob the geometry follows the launch's size: below 128 MiB
// (under ~14 units of 64 KiB per SM) 16 KiB x 4 stages spread the copy over
// more, shorter units (back-to-back 1-8-block transfers 2-5% faster), above
// it 64 KiB x 3 (the 2 GiB sweep's and the bench's best; 16 KiB x 4 loses
// 4% there).
static int bulk_cfg(unsigned long long bytes) {
  static const int cfg = [] {
    const char* e = getenv("MP_BULK_CFG");
    return (e && e[0] >= '0' && e[0] <= '5') ? e[0] - '0' : -1;
  }();
  if (cfg >= 0) return cfg;
  return bytes < (128ull << 20) ? 3 : 0;
}

cudaError_t launch_migrate(const Endpoint& src, const Endpoint& dst, int n, int j0, int nj,
                           long long chunk, int max_ctas, cudaStream_t stream, int variant,
                           const Sched* sched, const InlineIds* src_inline, bool wait_prev) {
  if (n <= 0 || nj <= 0) return cudaSuccess;
  static const InlineIds no_ids{};
  if (src_inline) {  // source ids, destination ids, or both (ids[0, n) then ids[n', n'+n))
    const int ns = src_inline->n, nd = src_inline->nd;
    if (!((ns == 0 || ns == n) && (nd == 0 || nd == n) && (ns || nd) && ns + nd <= kInlineIds))
      return cudaErrorInvalidValue;
  }
  const InlineIds& si = src_inline ? *src_inline : no_ids;
  if (variant == kCopyBulk) {
    switch (bulk_cfg((unsigned long long)n * (unsigned long long)nj * (unsigned long long)chunk)) {
      case 1: return launch_bulk_any<32768, 3>(src, dst, n, j0, nj, chunk, max_ctas, stream, sched, si, wait_prev);
      case 2: return launch_bulk_any<8192, 6>(src, dst, n, j0, nj, chunk, max_ctas, stream, sched, si, wait_prev);
      case 3: return launch_bulk_any<16384, 4>(src, dst, n, j0, nj, chunk, max_ctas, stream, sched, si, wait_prev);
      case 4: return launch_bulk_any<32768, 6>(src, dst, n, j0, nj, chunk, max_ctas, stream, sched, si, wait_prev);
      case 5: return launch_bulk_any<49152, 4>(src, dst, n, j0, nj, chunk, max_ctas, stream, sched, si, wait_prev);
      default: return launch_bulk_any<65536, 3>(src, dst, n, j0, nj, chunk, max_ctas, stream, sched, si, wait_prev);
    }
  }
  const unsigned units_per_chunk = (unsigned)((chunk + kUnitBytes - 1) / kUnitBytes);
  const unsigned long long total = (unsigned long long)n * nj * units_per_chunk;
  if (total >= (1ull << 32)) return cudaErrorInvalidValue;
  int dev = 0;
  cudaGetDevice(&dev);
  const bool sp = src.slabs != nullptr, dp = dst.slabs != nullptr;
  // One full wave: resident CTAs per SM x SM count (148 on B200), so no CTA
  // waits for a second wave; the grid-stride loop spreads the units.
  static CapCache cached_cap{};  // per device: resident CTAs x SMs
  int cap = max_ctas;
  if (cap <= 0) {
    const int cached = dev < 64 ? cached_cap[dev].load(std::memory_order_acquire) : 0;
    if (cached > 0) {
      cap = cached;
    } else {
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, migrate_kernel<true, true>,
                                                    kThreads, 0);
      if (per_sm <= 0) per_sm = 1;
      cap = per_sm * sm_count(dev);
      if (dev < 64) cached_cap[dev].store(cap, std::memory_order_release);
    }
  }
  const unsigned long long want = (total + (kThreads / 32) - 1) / (kThreads / 32);
  const int grid = (int)(want < (unsigned long long)cap ? want : (unsigned long long)cap);
  const bool dyn = sched && sched->ctr && bulk_dynamic();
  unsigned long long* ctr = dyn ? sched->ctr : nullptr;
  const unsigned long long sbase = dyn ? *sched->base : 0;
  auto kern = sp ? (dp ? migrate_kernel<true, true> : migrate_kernel<true, false>)
                 : (dp ? migrate_kernel<false, true> : migrate_kernel<false, false>);
  const cudaError_t e = launch_pdl(kern, grid, kThreads, 0, stream, src, dst, j0, nj, chunk,
                                   units_per_chunk, (unsigned)total, si, ctr, sbase,
                                   wait_prev ? 1 : 0);
  if (dyn && e == cudaSuccess) {
    const unsigned long long groups = (total + kGroup - 1) / kGroup;
    const unsigned long long warps = (unsigned long long)grid * (kThreads / 32);
    *sched->base += (groups > warps ? groups - warps : 0) + warps;
  }
  return e;
}

cudaError_t launch_alloc(uint32_t* bitmap, int nwords, int n, int* out_dev, int* out_host,
                         int* err, cudaStream_t stream, const InlineIds* frees) {
  static const InlineIds none{};
  if (n <= 0) {
    if (frees && frees->n > 0) {
      free_inline_kernel<<<1, 256, 0, stream>>>(bitmap, *frees);
      return cudaGetLastError();
    }
    return cudaSuccess;
  }
  // 256 threads: <= 8 bitmap words each up to 65536 blocks; small enough to
  // slot in beside retiring migration CTAs
  alloc_kernel<<<1, 256, 0, stream>>>(bitmap, nwords, n, out_dev, out_host, err,
                                      frees ? *frees : none);
  return cudaGetLastError();
}

cudaError_t launch_free(uint32_t* bitmap, const int* ids, int n, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int grid = (n + 255) / 256 < 148 ? (n + 255) / 256 : 148;
  free_kernel<<<grid, 256, 0, stream>>>(bitmap, ids, n);
  return cudaGetLastError();
}

cudaError_t launch_fill(char* const* slabs, const int* ids, int n, int nchunks, long long chunk,
                        unsigned long long seed, unsigned long long inst,
                        unsigned long long epoch, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const unsigned long long total = (unsigned long long)n * nchunks * (chunk / 16);
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long want = (total + 255) / 256;
  const unsigned long long cap = 8ull * sm_count(dev);
  fill_kernel<<<(int)(want < cap ? want : cap), 256, 0, stream>>>(slabs, ids, nchunks, chunk,
                                                                  seed, inst, epoch, total);
  return cudaGetLastError();
}

}  // namespace mpk
