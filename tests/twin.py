"""Twin harness: apply the same MemPool operation to the CPU oracle and to the
CUDA path (through the C-ABI binding) and compare the results element by
element.  Test infrastructure only (imports the oracle)."""
import numpy as np

import oracle as O
from paper_2406_17565_b200 import mempool as M

FLAG_MAP = {  # oracle flag -> C-ABI flag
    O.FLAG_DST_GIVEN: M.XFER_DST_GIVEN,
    O.FLAG_DEDUP: M.XFER_DEDUP,
    O.FLAG_INS_ERR_ON_CONFLICT: M.INS_ERR_ON_CONFLICT,
    O.FLAG_MATCH_PIN: M.MATCH_PIN,
}


def to_c(addrs):
    return np.array([M.make_addr(i, m, x) for (i, m, x) in addrs], np.uint64)


def to_o(addrs):
    return [(M.addr_inst(a), M.addr_medium(a), M.addr_index(a)) for a in addrs]


def cflags(oflags, path=0):
    f = 0
    for k, v in FLAG_MAP.items():
        if oflags & k:
            f |= v
    return f | path


class Twin:
    """An oracle pool and a GPU pool with the same shape and instance id."""

    def __init__(self, inst, shape, n_hbm, n_dram=0, seed=17565, device=0, verify=True,
                 materialize=False, **kw):
        self.o = O.OraclePool(inst, shape.layers, shape.kv_heads, shape.head_dim,
                              shape.block_tokens, n_hbm=n_hbm, n_dram=n_dram,
                              elem_bytes=shape.elem_bytes, seed=seed, materialize=materialize)
        self.g = M.Pool(inst, device, shape.layers, shape.kv_heads, shape.head_dim,
                        shape.block_tokens, n_hbm, n_dram, elem_bytes=shape.elem_bytes,
                        verify=verify, **kw)
        self.inst = inst
        self.seed = seed
        self.swap_flags = 0          # MP_SWAP_* transport for swap_out / swap_in

    # Each op returns the oracle result (or raises MPError after checking the
    # GPU raised the same error).
    def call(self, oname, gname, oargs, gargs, conv=lambda r: r):
        oerr = gerr = None
        try:
            ores = oname(*oargs)
        except O.MPError as e:
            oerr = e.name
        try:
            gres = gname(*gargs)
        except M.MempoolError as e:
            gerr = e.name
        assert oerr == gerr, f"error mismatch: oracle {oerr} vs gpu {gerr}"
        if oerr:
            raise O.MPError(oerr)
        return ores, conv(gres)

    def alloc(self, n, medium=O.HBM, requester=None, stream_ordered=False):
        """stream_ordered (MP_ALLOC_STREAM_ORDERED) changes no result, only
        whether the GPU pool drains first; fills are pool-stream ordered."""
        o, g = self.call(self.o.alloc_mem,
                         lambda *a: self.g.alloc_mem(*a, stream_ordered=stream_ordered),
                         (n, medium, requester), (n, medium, requester), to_o)
        assert o == g, (o, g)
        return o

    def free(self, addrs):
        self.call(self.o.free_mem, self.g.free_mem, (addrs,), (to_c(addrs),))

    def fill(self, addrs):
        self.call(self.o.fill, lambda a: self.g.debug_fill(a, self.seed), (addrs,), (to_c(addrs),))

    def insert(self, tokens, addrs, oflags=0):
        o, g = self.call(self.o.insert, self.g.insert, (tokens, addrs, oflags),
                         (tokens, to_c(addrs), cflags(oflags)))
        assert o == g, (o, g)
        return o

    def match(self, tokens, oflags=0):
        o, g = self.call(self.o.match, self.g.match, (tokens, oflags), (tokens, cflags(oflags)),
                         lambda r: (r[0], to_o(r[1])))
        assert o == g, (o, g)
        return o

    def unpin(self, addrs):
        self.call(self.o.unpin, self.g.unpin, (addrs,), (to_c(addrs),))

    def delete(self, tokens):
        self.call(self.o.delete, self.g.delete, (tokens,), (tokens,))

    def evict(self, n, medium=O.HBM):
        o, g = self.call(self.o.evict, self.g.evict, (n, medium), (n, medium), to_o)
        assert o == g, (o, g)
        return o

    def swap_out(self, n, flags=None):
        flags = self.swap_flags if flags is None else flags
        o, g = self.call(self.o.swap_out, lambda k: self.g.swap_out(k, flags), (n,), (n,),
                         lambda r: list(zip(to_o(r[0]), to_o(r[1]))))
        assert o == g, (o, g)
        return o

    def swap_in(self, addrs, flags=None):
        flags = self.swap_flags if flags is None else flags
        o, g = self.call(self.o.swap_in, lambda a: self.g.swap_in(a, flags), (addrs,),
                         (to_c(addrs),), to_o)
        assert o == g, (o, g)
        return o

    # ------------------------------------------------------------ comparisons
    def check_state(self, check_bytes=True, sample=None, rng=None):
        """Index dump, block states, device bitmap, clock, and block bytes."""
        od = self.o.dump_index()
        gd = self.g.dump_index()
        assert [(k, m, i, la, r, t) for (k, m, i, la, r, t) in od] == gd
        info = self.g.info()
        assert info.clock == self.o.clock
        smap = {O.FREE: 0, O.ACTIVE: 1, O.INDEXED: 2, O.ORPHAN: 3}
        for med in (O.HBM, O.DRAM):
            if self.o.cap[med] == 0:
                continue
            want = np.array([smap[s] for s in self.o.state[med]], np.uint8)
            np.testing.assert_array_equal(self.g.block_states(med), want)
        bm = self.g.bitmap()
        bits = np.unpackbits(bm.view(np.uint8), bitorder="little")[: self.o.cap[O.HBM]]
        want_free = np.array([s == O.FREE for s in self.o.state[O.HBM]], np.uint8)
        np.testing.assert_array_equal(bits, want_free)
        if check_bytes:
            self.check_bytes(sample=sample, rng=rng)

    def check_bytes(self, sample=None, rng=None):
        """Every allocated block whose chunks were all written: GPU bytes ==
        the oracle's expected bytes (from content tags, kvgen)."""
        cands = []
        for med in (O.HBM, O.DRAM):
            for i, s in enumerate(self.o.state[med]):
                if s != O.FREE and all(t is not None for t in self.o.tags[med][i]):
                    cands.append((med, i))
        if sample is not None and len(cands) > sample:
            rng = rng or np.random.default_rng(0)
            keep = {0, len(cands) - 1} | set(rng.choice(len(cands), sample, replace=False).tolist())
            cands = [cands[k] for k in sorted(keep)]
        for med, i in cands:
            got = self.g.debug_read_block(M.make_addr(self.inst, med, i))
            want = self.o.block_bytes((self.inst, med, i))
            assert np.array_equal(got, want), f"bytes differ at {(med, i)}"
        return len(cands)


def connect(a: Twin, b: Twin):
    M.connect(a.g, b.g)


def transfer(a: Twin, b: Twin, src, dst=None, oflags=0, l0=0, l1=None, priv=b"", path=0):
    oerr = gerr = None
    try:
        o = O.transfer(a.o, b.o, src, dst, oflags, l0, l1, priv)
    except O.MPError as e:
        oerr = e.name
    try:
        g = a.g.transfer(b.inst, to_c(src), None if dst is None else to_c(dst),
                         cflags(oflags, path), l0, l1, priv)
    except M.MempoolError as e:
        gerr = e.name
    assert oerr == gerr, f"error mismatch: oracle {oerr} vs gpu {gerr}"
    if oerr:
        raise O.MPError(oerr)
    assert o == to_o(g), (o, to_o(g))
    return o


def transfer_with_insert(a: Twin, b: Twin, tokens, src, dst=None, oflags=0, priv=b"", path=0):
    oerr = gerr = None
    try:
        o = O.transfer_with_insert(a.o, b.o, tokens, src, dst, oflags, priv)
    except O.MPError as e:
        oerr = e.name
    try:
        g = a.g.transfer_with_insert(b.inst, tokens, to_c(src),
                                     None if dst is None else to_c(dst), cflags(oflags, path),
                                     priv)
    except M.MempoolError as e:
        gerr = e.name
    assert oerr == gerr, f"error mismatch: oracle {oerr} vs gpu {gerr}"
    if oerr:
        raise O.MPError(oerr)
    final, moved = g
    assert o[0] == to_o(final), (o[0], to_o(final))
    assert o[1] == moved, (o[1], moved)
    return o
