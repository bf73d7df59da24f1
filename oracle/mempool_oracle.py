"""Plain CPU oracle of MemPool (test infrastructure only -- see oracle/__init__.py).

Every function cites the PAPER.md (P:n) / SPEC.md (S:n) passage it follows and
the reading R1-R16 it takes where the paper is silent
(R17, global scheduling, is in gs_oracle.py).

Model
-----
* A pool (one serving instance) has HBM and DRAM block slots.
  Each slot has a state: FREE, ACTIVE (caller-owned KV of a running request),
  INDEXED (historical KV owned by the index) or ORPHAN (unlinked
  from the index by ``delete`` while still pinned; freed on the last unpin).
* KV bytes are tracked as a content tag per (slot, chunk) where chunk
  j = 2*layer + kv ("two blocks per LLM layer"); bytes are
  materialised on demand by ``workloads.kvgen`` (or kept as real numpy arrays
  when ``materialize=True``, the byte path timed as the CPU baseline).
* The index is the brute-force prefix map: a dict from the block-aligned token
  prefix tuple(tokens[:k*B]) to an Entry(addr, last_access, ref, terminal)
  (R1, "radix tree nodes point to KV cache blocks of 16 tokens").
  There is deliberately no tree: children are found by scanning the dict.
* Addresses are (instance, medium, index) tuples ("Each address encodes
  instance ID").

Every public op validates everything first and raises MPError without
changing state (all-or-nothing), then mutates.
"""
import copy
from dataclasses import dataclass

import numpy as np

from workloads import kvgen

HBM, DRAM, MIXED = 0, 1, 2
FREE, ACTIVE, INDEXED, ORPHAN = "free", "active", "indexed", "orphan"

FLAG_DST_GIVEN = 1 << 0           # transfer: skip the allocation step
FLAG_DEDUP = 1 << 1               # transfer_with_insert: receiver matches first (R3)
FLAG_INS_ERR_ON_CONFLICT = 1 << 4  # insert: error instead of keep-existing (R4)
FLAG_MATCH_PIN = 1 << 5           # match: pin matched blocks (R12)


class MPError(Exception):
    """Error names follow SPEC.md (S:129 OOM, S:139 DoubleFree/InvalidAddr,
    S:149 AddrCountMismatch/ConflictingMapping, S:189 NoDramCapacity,
    S:202 precondition, S:255 DstOutOfMemory/DstUnreachable) plus
    PREFIX_MISSING (R3) and CONFIG."""

    def __init__(self, name: str):
        super().__init__(name)
        self.name = name


@dataclass
class Entry:
    addr: tuple          # (inst, medium, idx)
    last_access: int
    ref: int = 0
    terminal: bool = False


def _ceil_div(a: int, b: int) -> int:
    return -(-a // b)


class OraclePool:
    """One instance's MemPool."""

    def __init__(self, inst: int, layers: int, kv_heads: int, head_dim: int,
                 block_tokens: int, n_hbm: int, n_dram: int = 0,
                 elem_bytes: int = 2, seed: int = 0, materialize: bool = False):
        self.inst = inst
        self.L = layers
        self.B = block_tokens
        self.chunk_bytes = block_tokens * kv_heads * head_dim * elem_bytes
        assert self.chunk_bytes % 8 == 0
        self.W = self.chunk_bytes // 8          # uint64 words per chunk
        self.nch = 2 * layers                   # chunks per block
        self.cap = {HBM: n_hbm, DRAM: n_dram}
        self.state = {HBM: [FREE] * n_hbm, DRAM: [FREE] * n_dram}
        self.tags = {HBM: [[None] * self.nch for _ in range(n_hbm)],
                     DRAM: [[None] * self.nch for _ in range(n_dram)]}
        self.alloc_by = {}                      # (medium, idx) -> requester
        self.index = {}                         # prefix tuple -> Entry
        self.orphans = {}                       # (medium, idx) -> ref
        self.clock = 0                          # R7 logical clock
        self.epoch = 0                          # fill counter (content model)
        self.seed = seed
        self.inbox = []                         # delivered `private`
        self.materialize = materialize
        if materialize:
            # HBM: per-(layer,kv) slabs [2L][N][W] (vLLM discrete layout);
            # DRAM: aggregated blocks [N][2L][W] (R11).
            self.hbm_bytes = np.zeros((self.nch, n_hbm, self.W), np.uint64)
            self.dram_bytes = np.zeros((n_dram, self.nch, self.W), np.uint64)

    # ------------------------------------------------------------------ helpers
    def _addr(self, medium, idx):
        return (self.inst, medium, idx)

    def _check_addr(self, a, media=(HBM, DRAM)):
        """INVALID_ADDR unless a is a well-formed address of this instance."""
        if (not isinstance(a, tuple) or len(a) != 3 or a[0] != self.inst
                or a[1] not in media or not (0 <= a[2] < self.cap[a[1]])):
            raise MPError("INVALID_ADDR")

    def free_count(self, medium):
        return sum(1 for s in self.state[medium] if s == FREE)

    def _children_count(self):
        """{prefix: number of child entries} by scanning the dict (plain)."""
        cnt = {}
        hbm_cnt = {}
        for key, e in self.index.items():
            if len(key) > self.B:
                par = key[:-self.B]
                cnt[par] = cnt.get(par, 0) + 1
                if e.addr[1] == HBM:
                    hbm_cnt[par] = hbm_cnt.get(par, 0) + 1
        return cnt, hbm_cnt

    def _entry_of_addr(self, a):
        for key, e in self.index.items():
            if e.addr == a:
                return key, e
        return None, None

    def _clone_meta(self):
        """Deep copy of everything except the (immutable here) byte arrays."""
        saved = {}
        for name in ("hbm_bytes", "dram_bytes"):
            if name in self.__dict__:
                saved[name] = self.__dict__.pop(name)
        try:
            twin = copy.deepcopy(self)
        finally:
            self.__dict__.update(saved)
        twin.__dict__.update(saved)
        return twin

    def _tick(self):
        self.clock += 1
        return self.clock

    def _free_slot(self, medium, idx):
        self.state[medium][idx] = FREE
        self.alloc_by.pop((medium, idx), None)

    # --------------------------------------------------------------- allocator
    def _evict(self, n, medium):
        """R8 (P:414 names evict; policy is ours): repeat up to n times, among
        index leaves (no child of any medium) in ``medium`` with ref == 0, take
        the least (last_access, block index); unlink and free it."""
        freed = []
        for _ in range(n):
            cnt, _h = self._children_count()
            cands = [(e.last_access, e.addr[2], key) for key, e in self.index.items()
                     if e.addr[1] == medium and e.ref == 0 and cnt.get(key, 0) == 0]
            if not cands:
                break
            _, idx, key = min(cands)
            del self.index[key]
            self._free_slot(medium, idx)
            freed.append(self._addr(medium, idx))
        return freed

    def _take_lowest(self, n, medium, requester):
        """R2: the n lowest-index free blocks, ascending."""
        ids = [i for i, s in enumerate(self.state[medium]) if s == FREE][:n]
        assert len(ids) == n
        for i in ids:
            self.state[medium][i] = ACTIVE
            self.alloc_by[(medium, i)] = requester
        return [self._addr(medium, i) for i in ids]

    def _can_make_room(self, n, medium):
        """Would evicting by the shortfall leave >= n free?  (R2: evict first,
        else OOM with no state change.)  Decided by simulating on a copy."""
        free = self.free_count(medium)
        if free >= n:
            return True
        trial = self._clone_meta()
        trial._evict(n - free, medium)
        return trial.free_count(medium) >= n

    def alloc_mem(self, n, medium, requester=None):
        """alloc_mem(size, type, id) -- Table tbl-mempool-api.

        R2: lowest-first, all-or-nothing; MIXED takes free HBM first, then
        DRAM; on shortage evict unreferenced historical blocks
        of that medium by the shortfall first, else OOM.  MIXED never
        evicts HBM (reading)."""
        requester = self.inst if requester is None else requester
        if n < 0 or medium not in (HBM, DRAM, MIXED):
            raise MPError("CONFIG")
        if medium in (HBM, DRAM):
            if not self._can_make_room(n, medium):
                raise MPError("OOM")
            free = self.free_count(medium)
            if free < n:
                self._evict(n - free, medium)
            return self._take_lowest(n, medium, requester)
        h = min(n, self.free_count(HBM))
        d = n - h
        if not self._can_make_room(d, DRAM):
            raise MPError("OOM")
        free = self.free_count(DRAM)
        if free < d:
            self._evict(d - free, DRAM)
        return self._take_lowest(h, HBM, requester) + self._take_lowest(d, DRAM, requester)

    def free_mem(self, addrs):
        """free_mem(addrList) -- P:272.  Only caller-owned (ACTIVE)
        blocks may be freed: a FREE block or a repeated address is DOUBLE_FREE,
        an index-owned / orphaned block is PRECONDITION (R12)."""
        seen = set()
        for a in addrs:
            self._check_addr(a)
            st = self.state[a[1]][a[2]]
            if st == FREE or a in seen:
                raise MPError("DOUBLE_FREE")
            if st != ACTIVE:
                raise MPError("PRECONDITION")
            seen.add(a)
        for a in addrs:
            self._free_slot(a[1], a[2])

    # ------------------------------------------------------------------- index
    def _prefix(self, tokens, k):
        # the key is the tuple of Python ints tokens[:k*B] (R1)
        return tuple(np.asarray(tokens[: k * self.B], dtype=np.int64).tolist())

    def _peek_match(self, tokens):
        """Longest k <= floor(n/B) with prefix_k in the map (no side effects)."""
        k = 0
        while (k + 1) * self.B <= len(tokens) and self._prefix(tokens, k + 1) in self.index:
            k += 1
        return k

    def match(self, tokens, flags=0):
        """match(tokenList) -- P:276.  R5: largest k with prefix_k
        present; returns (k*B, addrs of prefixes 1..k); touches last_access
        (R7: one clock tick per call); MATCH_PIN increments ref (R12)."""
        t = self._tick()
        k = self._peek_match(tokens)
        addrs = []
        for i in range(1, k + 1):
            e = self.index[self._prefix(tokens, i)]
            e.last_access = t
            if flags & FLAG_MATCH_PIN:
                e.ref += 1
            addrs.append(e.addr)
        return k * self.B, addrs

    def _validate_insert(self, tokens, addrs, flags):
        n = len(tokens)
        k, c = n // self.B, _ceil_div(n, self.B)
        if len(addrs) not in (k, c):
            raise MPError("ADDR_COUNT")
        seen = set()
        for i in range(k):
            a = addrs[i]
            self._check_addr(a)
            if a in seen:
                raise MPError("PRECONDITION")
            seen.add(a)
            key = self._prefix(tokens, i + 1)
            ex = self.index.get(key)
            st = self.state[a[1]][a[2]]
            if st == ACTIVE:
                pass
            elif st == INDEXED and ex is not None and ex.addr == a:
                pass
            else:
                raise MPError("PRECONDITION")
            if flags & FLAG_INS_ERR_ON_CONFLICT and ex is not None and ex.addr != a:
                raise MPError("CONFLICT")
        return k

    def insert(self, tokens, addrs, flags=0):
        """insert(tokenList, addrList, flags) -- P:274, P:298 (retire active KV
        into historical KV).  R4: only floor(n/B) full blocks are
        indexed (R1); a trailing partial-block address is accepted and
        ignored; an existing prefix keeps its mapping and the caller's
        duplicate block is freed (S:149 keep-existing default) unless
        INS_ERR_ON_CONFLICT.  Returns the number of duplicates freed."""
        k = self._validate_insert(tokens, addrs, flags)
        t = self._tick()
        dup = 0
        for i in range(k):
            a = addrs[i]
            key = self._prefix(tokens, i + 1)
            ex = self.index.get(key)
            if ex is None:
                self.index[key] = Entry(a, t)
                self.state[a[1]][a[2]] = INDEXED
            else:
                ex.last_access = t
                if ex.addr != a:
                    self._free_slot(a[1], a[2])
                    dup += 1
        if k >= 1:
            self.index[self._prefix(tokens, k)].terminal = True
        return dup

    def delete(self, tokens):
        """delete(tokenList) -- P:278.  R6: no-op unless prefix_k
        (k = floor(n/B)) is a terminal entry; clear it, then unlink prefixes
        k, k-1, ... while they have no child and are not terminal; an
        unlinked block is freed if ref == 0, else becomes ORPHAN until its
        last unpin."""
        k = len(tokens) // self.B
        if k == 0:
            return
        key = self._prefix(tokens, k)
        e = self.index.get(key)
        if e is None or not e.terminal:
            return
        e.terminal = False
        for i in range(k, 0, -1):
            key = self._prefix(tokens, i)
            e = self.index[key]
            cnt, _ = self._children_count()
            if cnt.get(key, 0) > 0 or e.terminal:
                break
            del self.index[key]
            med, idx = e.addr[1], e.addr[2]
            if e.ref == 0:
                self._free_slot(med, idx)
            else:
                self.state[med][idx] = ORPHAN
                self.orphans[(med, idx)] = e.ref

    def unpin(self, addrs):
        """Release MATCH_PIN references (R12)."""
        need = {}
        for a in addrs:
            self._check_addr(a)
            need[a] = need.get(a, 0) + 1
        for a, cnt in need.items():
            _, e = self._entry_of_addr(a)
            have = e.ref if e is not None else self.orphans.get((a[1], a[2]), 0)
            if have < cnt:
                raise MPError("PRECONDITION")
        for a in addrs:
            _, e = self._entry_of_addr(a)
            if e is not None:
                e.ref -= 1
            else:
                o = (a[1], a[2])
                self.orphans[o] -= 1
                if self.orphans[o] == 0:
                    del self.orphans[o]
                    self._free_slot(a[1], a[2])

    def evict(self, n, medium):
        """evict -- P:414 (Table tbl-use-case); R8."""
        if n < 0 or medium not in (HBM, DRAM):
            raise MPError("CONFIG")
        return self._evict(n, medium)

    # ------------------------------------------------------------------- bytes
    def _copy_chunks(self, src_pool, s_med, s_idx, d_med, d_idx, j0, j1):
        """dst[chunk j] = src[chunk j] for j in [j0, j1) -- the whole of the
        migration arithmetic: a verbatim copy (BJ:5 "bit-exact")."""
        for j in range(j0, j1):
            self.tags[d_med][d_idx][j] = src_pool.tags[s_med][s_idx][j]
        if self.materialize and src_pool.materialize:
            for j in range(j0, j1):
                src = (src_pool.hbm_bytes[j, s_idx] if s_med == HBM
                       else src_pool.dram_bytes[s_idx, j])
                if d_med == HBM:
                    self.hbm_bytes[j, d_idx] = src
                else:
                    self.dram_bytes[d_idx, j] = src

    def fill(self, addrs):
        """Synthetic prefill write (stand-in for the engine's KV write; the
        content model of SURVEY.md §8(c)): one epoch per call, every chunk of
        every listed HBM block gets tag (inst, epoch, block)."""
        for a in addrs:
            self._check_addr(a, media=(HBM,))
            if self.state[HBM][a[2]] == FREE:
                raise MPError("PRECONDITION")
        self.epoch += 1
        for a in addrs:
            tag = kvgen.make_tag(self.inst, self.epoch, a[2])
            self.tags[HBM][a[2]] = [tag] * self.nch
            if self.materialize:
                self.hbm_bytes[:, a[2]] = kvgen.block_words(self.seed, [tag] * self.nch, self.W)

    def block_bytes(self, addr):
        """Aggregated-layout words [2L][W] of a block (R11), from tags."""
        self._check_addr(addr)
        return kvgen.block_words(self.seed, self.tags[addr[1]][addr[2]], self.W)

    # -------------------------------------------------------------------- swap
    def swap_out(self, n):
        """swap_out(num_blocks) -- P:280.  R9: repeat up to n times:
        among INDEXED HBM blocks with ref == 0 and no HBM-resident child (the
        HBM frontier) take the least (last_access, block index); take the
        lowest free DRAM id, evicting one DRAM leaf (R8) first when DRAM is
        full; copy all chunks; rewrite the entry's addr; free the HBM block.
        NO_DRAM only if nothing could be moved for lack of DRAM."""
        if n < 0:
            raise MPError("CONFIG")
        moved = []
        no_dram = False
        while len(moved) < n:
            _, hcnt = self._children_count()
            cands = [(e.last_access, e.addr[2], key) for key, e in self.index.items()
                     if e.addr[1] == HBM and e.ref == 0 and hcnt.get(key, 0) == 0]
            if not cands:
                break
            if self.free_count(DRAM) == 0 and not self._evict(1, DRAM):
                no_dram = True
                break
            _, v, key = min(cands)
            d = [i for i, s in enumerate(self.state[DRAM]) if s == FREE][0]
            self._copy_chunks(self, HBM, v, DRAM, d, 0, self.nch)
            self.state[DRAM][d] = INDEXED
            self.alloc_by[(DRAM, d)] = self.alloc_by.get((HBM, v), self.inst)
            self.index[key].addr = self._addr(DRAM, d)
            self._free_slot(HBM, v)
            moved.append((self._addr(HBM, v), self._addr(DRAM, d)))
        if no_dram and not moved:
            raise MPError("NO_DRAM")
        return moved

    def swap_in(self, addrs):
        """swap_in(addrList) -- P:282.  R10: every addr must be an
        allocated DRAM block of this instance (else PRECONDITION);
        HBM ids lowest-first in input order (R2, may evict / OOM); copy;
        rewrite index addrs; free DRAM; return the new HBM addrs."""
        seen = set()
        for a in addrs:
            self._check_addr(a)
            if a[1] != DRAM or a in seen:
                raise MPError("PRECONDITION")
            if self.state[DRAM][a[2]] not in (ACTIVE, INDEXED):
                raise MPError("PRECONDITION")
            seen.add(a)
        if not self._can_make_room(len(addrs), HBM):
            raise MPError("OOM")
        new = self.alloc_mem(len(addrs), HBM)
        for a, h in zip(addrs, new):
            self._copy_chunks(self, DRAM, a[2], HBM, h[2], 0, self.nch)
            self.alloc_by[(HBM, h[2])] = self.alloc_by.get((DRAM, a[2]), self.inst)
            if self.state[DRAM][a[2]] == INDEXED:
                _, e = self._entry_of_addr(a)
                e.addr = h
                self.state[HBM][h[2]] = INDEXED
            self._free_slot(DRAM, a[2])
        return new

    # ------------------------------------------------------------------- debug
    def dump_index(self):
        """Deterministic sorted rendering: one tuple per entry
        (prefix tokens, medium, idx, last_access, ref, terminal)."""
        return sorted((key, e.addr[1], e.addr[2], e.last_access, e.ref, e.terminal)
                      for key, e in self.index.items())

    def check_invariants(self):
        """Conservation and single ownership (BJ:5)."""
        for med in (HBM, DRAM):
            owners = {}
            for key, e in self.index.items():
                if e.addr[1] == med:
                    assert e.addr[2] not in owners, "block owned twice"
                    owners[e.addr[2]] = key
                    assert self.state[med][e.addr[2]] == INDEXED
            for i, s in enumerate(self.state[med]):
                if s == INDEXED:
                    assert i in owners, "indexed block missing from index"
                if s == ORPHAN:
                    assert (med, i) in self.orphans
        for key in self.index:
            assert len(key) % self.B == 0 and len(key) > 0
            if len(key) > self.B:
                assert key[:-self.B] in self.index, "index not prefix-closed"


# ---------------------------------------------------------------- distributed
def _validate_src(src, src_addrs):
    """R13 (memory asymmetry: "historical KV cache has been swapped
    out to DRAM"): a source block may live in HBM or in the source's DRAM;
    it must be allocated (caller-owned or index-owned) and listed once."""
    seen = set()
    for a in src_addrs:
        src._check_addr(a)
        if src.state[a[1]][a[2]] not in (ACTIVE, INDEXED) or a in seen:
            raise MPError("PRECONDITION")
        seen.add(a)


def _validate_dst_given(dst, dst_addrs, n):
    if dst_addrs is None or len(dst_addrs) != n:
        raise MPError("ADDR_COUNT")
    seen = set()
    for a in dst_addrs:
        dst._check_addr(a)
        if a[1] != HBM or dst.state[HBM][a[2]] != ACTIVE or a in seen:
            raise MPError("PRECONDITION")
        seen.add(a)


def transfer(src, dst, src_addrs, dst_addrs=None, flags=0, layer_begin=0,
             layer_end=None, priv=b""):
    """transfer(id, srcAddrList, dstAddrList, flags, private) -- P:284;
    workflow P:360-365: (1) allocation at the receiver (alloc_mem)
    unless DST_GIVEN (used for layer-by-layer); (2) transmission:
    dst[l][kv][d_j] = src[l][kv][s_j] for the layer range; (3) `private`
    delivered to the receiver.  The receiver's blocks are ACTIVE
    (caller-owned) afterwards.  Returns the destination addrs."""
    layer_end = src.L if layer_end is None else layer_end
    if dst is None:
        raise MPError("DST_UNREACHABLE")
    if (dst is src or src.L != dst.L or src.chunk_bytes != dst.chunk_bytes
            or not (0 <= layer_begin < layer_end <= src.L) or flags & FLAG_DEDUP):
        raise MPError("CONFIG")
    n = len(src_addrs)
    _validate_src(src, src_addrs)
    if flags & FLAG_DST_GIVEN:
        _validate_dst_given(dst, dst_addrs, n)
        out = list(dst_addrs)
    else:
        if not dst._can_make_room(n, HBM):
            raise MPError("DST_OOM")
        out = dst.alloc_mem(n, HBM, requester=src.inst)
    for s, d in zip(src_addrs, out):
        dst._copy_chunks(src, s[1], s[2], HBM, d[2], 2 * layer_begin, 2 * layer_end)
    dst.inbox.append(("transfer", src.inst, bytes(priv), list(out)))
    return out


def tp_plan(H, p, q):
    """Asymmetric parallelism: rank r of a TP=t instance holds
    heads [r*H/t, (r+1)*H/t) ("split evenly by tp ratio").  The
    pieces of a TP=p -> TP=q move: for every overlapping (src rank, dst rank),
    (r, s, first head within the source shard, first head within the
    destination shard, head count).  Brute force over heads: each head h goes
    from rank h // (H/p) to rank h // (H/q); consecutive heads with the same
    (r, s) form one piece."""
    if H < 1 or p < 1 or q < 1 or H % p or H % q:
        raise MPError("CONFIG")
    hs, hd = H // p, H // q
    pieces = []
    for h in range(H):
        r, s = h // hs, h // hd
        if pieces and pieces[-1][0] == r and pieces[-1][1] == s:
            r_, s_, a, b, k = pieces[-1]
            pieces[-1] = (r_, s_, a, b, k + 1)
        else:
            pieces.append((r, s, h - r * hs, h - s * hd, 1))
    return sorted(pieces)


def transfer_heads(src, dst, src_addrs, dst_addrs, src_head0, dst_head0, n_heads,
                   layer_begin=0, layer_end=None, kv_heads=None):
    """Copy heads [src_head0, +n_heads) of layers [layer_begin, layer_end) of
    each source block into heads [dst_head0, ...) of the given destination
    blocks.  Reading R16: a chunk is head-major [H][B][D], so a head is a
    contiguous slice of B*D*elem bytes.  Materialised pools only (the tag
    model is per chunk: touched chunks lose their tag)."""
    layer_end = src.L if layer_end is None else layer_end
    sH, dH = kv_heads
    if (not (0 <= layer_begin < layer_end <= src.L) or n_heads < 1 or src_head0 < 0
            or dst_head0 < 0 or src_head0 + n_heads > sH or dst_head0 + n_heads > dH):
        raise MPError("CONFIG")
    _validate_src(src, src_addrs)
    if any(a[1] != HBM for a in src_addrs):
        raise MPError("PRECONDITION")
    _validate_dst_given(dst, dst_addrs, len(src_addrs))
    hw = src.W // sH                      # uint64 words per head per chunk
    assert dst.W // dH == hw
    for s, d in zip(src_addrs, dst_addrs):
        for j in range(2 * layer_begin, 2 * layer_end):
            dst.hbm_bytes[j, d[2], dst_head0 * hw:(dst_head0 + n_heads) * hw] = \
                src.hbm_bytes[j, s[2], src_head0 * hw:(src_head0 + n_heads) * hw]
            dst.tags[HBM][d[2]][j] = None


def transfer_with_insert(src, dst, tokens, src_addrs, dst_addrs=None, flags=0,
                         priv=b""):
    """transfer_with_insert(id, tokenList, srcAddrList, dstAddrList, flags,
    private) -- P:286, P:364 ("The receiver ... invokes the insert function
    locally"), P:367 (saves a round trip), P:493-501 (PD-Caching-2/3).

    R3 (reading): src_addrs cover the LAST m of the ceil(n/B) blocks of
    ``tokens`` (full send when m == ceil; the D->P return of decode KV, P:501,
    and incremental sends, when m < ceil).  The receiver must already
    index the first q = ceil - m blocks, else PREFIX_MISSING.  With DEDUP the
    receiver's matched blocks beyond q are skipped.  The matched prefix is
    pinned while the receiver allocates (R12), then the receiver inserts
    matched[:q+skip] ++ new (R4).  Returns (final addrs of all ceil blocks,
    blocks moved, duplicates freed at the receiver)."""
    if dst is None:
        raise MPError("DST_UNREACHABLE")
    if (dst is src or src.L != dst.L or src.chunk_bytes != dst.chunk_bytes
            or src.B != dst.B):
        raise MPError("CONFIG")
    if flags & FLAG_DST_GIVEN and flags & FLAG_DEDUP:
        raise MPError("CONFIG")
    B = dst.B
    n = len(tokens)
    ceil_b, floor_b = _ceil_div(n, B), n // B
    m = len(src_addrs)
    if m > ceil_b:
        raise MPError("ADDR_COUNT")
    _validate_src(src, src_addrs)
    if flags & FLAG_DST_GIVEN:
        _validate_dst_given(dst, dst_addrs, m)
    q = ceil_b - m
    need_match = bool(flags & FLAG_DEDUP) or q > 0
    k_match = dst._peek_match(tokens) if need_match else 0
    if k_match < q:
        raise MPError("PREFIX_MISSING")
    skip = (k_match - q) if flags & FLAG_DEDUP else 0
    nm = m - skip
    # existing prefixes beyond the reused ones conflict with the new blocks
    if flags & FLAG_INS_ERR_ON_CONFLICT:
        k_exist = k_match if need_match else dst._peek_match(tokens)
        if k_exist > q + skip:
            raise MPError("CONFLICT")
    snapshot = dst._clone_meta()
    matched = []
    if need_match:
        _, matched = dst.match(tokens, flags=FLAG_MATCH_PIN)
    if flags & FLAG_DST_GIVEN:
        new = list(dst_addrs)
    else:
        if not dst._can_make_room(nm, HBM):
            dst.__dict__.update(snapshot.__dict__)   # all-or-nothing
            raise MPError("DST_OOM")
        new = dst.alloc_mem(nm, HBM, requester=src.inst)
    for s, d in zip(src_addrs[skip:], new):
        dst._copy_chunks(src, s[1], s[2], HBM, d[2], 0, dst.nch)
    full = list(matched[: q + skip]) + list(new)
    dup = dst.insert(tokens, full, flags & FLAG_INS_ERR_ON_CONFLICT)
    if matched:
        dst.unpin(matched)
    final = [dst.index[dst._prefix(tokens, i + 1)].addr for i in range(floor_b)]
    if ceil_b > floor_b:
        final.append(full[floor_b])
    dst.inbox.append(("transfer_with_insert", src.inst, bytes(priv), list(final)))
    return final, nm, dup


# ------------------------------------------------------------- aggregation
def pack(pool, addrs, layer_begin=0, layer_end=None):
    """A4, the block aggregation of P:549-550 ("instead of having two blocks
    per layer, we aggregate them into one block; the new block size equals
    2*L smaller blocks").  Returns the staging buffer as uint64 words of shape
    [n][l1-l0][2][W]: block i, layer l, K (kv=0) then V (kv=1) -- reading R11
    (layer-major, K before V).  Block i therefore starts at word offset
    i*(l1-l0)*2*W, i.e. byte i*Pb for a whole-request (all-layer) staging."""
    layer_end = pool.L if layer_end is None else layer_end
    if not (0 <= layer_begin < layer_end <= pool.L):
        raise MPError("CONFIG")
    for a in addrs:
        pool._check_addr(a)
    out = np.zeros((len(addrs), layer_end - layer_begin, 2, pool.W), np.uint64)
    for i, a in enumerate(addrs):
        words = pool.block_bytes(a)                 # [2L][W], aggregated order
        for l in range(layer_begin, layer_end):
            for kv in (0, 1):
                out[i, l - layer_begin, kv] = words[2 * l + kv]
    return out


def network_calls(n_tokens, B, L, chunk_bytes, mode):
    """The network API calls one request's KV needs, as a list of
    (staging byte offset, bytes) -- one entry per call.

    * "by_request" / "by_layer" with the discrete layout: "each call only
      transmits a single block" and "the number of network API calls equals
      the number of discrete memory blocks, regardless of whether the
      by-layer or by-request approach is used": one call per
      (token block, layer, K/V) chunk of c bytes.  Offsets are those of the
      chunk in an aggregated image (block-major), for comparison only.
    * "by_request_agg": the 2*L chunks of a token block are one aggregated
      block of Pb = 2*L*c bytes: one call per token block,
      block i at offset i*Pb.
    * "by_layer_agg": "the by-layer approach inevitably needs to call the
      network APIs at least L times": one call per layer carrying
      that layer's K and V of every block ([n][1][2][c] staging).
    ceil(n_tokens/B) token blocks (R1: the trailing partial block moves too)."""
    nb = _ceil_div(n_tokens, B)
    c = chunk_bytes
    Pb = 2 * L * c
    if mode in ("by_request", "by_layer"):
        return [(i * Pb + (2 * l + kv) * c, c)
                for i in range(nb) for l in range(L) for kv in (0, 1)]
    if mode == "by_request_agg":
        return [(i * Pb, Pb) for i in range(nb)]
    if mode == "by_layer_agg":
        return [(l * nb * 2 * c, nb * 2 * c) for l in range(L)] if nb else []
    raise MPError("CONFIG")
