"""Global prompt trees and locality-aware routing (§6, P:594-653;
SURVEY f4).  CPU: the C-ABI scheduler (mp_gs_*) against the brute-force
oracle on randomized register / update / load / route sequences with TTL
expiry, plus the paper's own cases.  GPU: the fan-in fetch the route output
enables -- the chosen prefill instance pulls the extra historical KV from the
instance that holds more of the prompt (a suffix transfer_with_insert, R3)."""
import numpy as np
import pytest

from oracle.gs_oracle import OracleGS


class _OracleGSAdapter:
    """OracleGS behind the product's GlobalScheduler interface (route raises
    when no instance of the kind is registered)."""
    PREFILL, DECODE, COLOCATED = 0, 1, 2

    def __init__(self, B, ttl_seconds):
        self.o = OracleGS(B, ttl_seconds)

    def register(self, inst, kind):
        self.o.register(inst, kind)

    def set_load(self, inst, load):
        self.o.set_load(inst, load)

    def update(self, inst, toks, now):
        self.o.update(inst, toks, now)

    def route(self, kind, toks, now):
        r = self.o.route(kind, toks, now)
        if r is None:
            raise LookupError("no instance of this kind")
        return r


def _impl(which):
    if which == "oracle":
        return _OracleGSAdapter
    from paper_2406_17565_b200.mempool import GlobalScheduler
    return GlobalScheduler


@pytest.mark.parametrize("which", ["oracle", "product"])
def test_paper_cases(which):
    """Hand-derived values of the paper's routing rules, checked on the
    oracle (its pin: nothing here comes from running either implementation)
    and on the product."""
    GS = _impl(which)
    g = GS(16, ttl_seconds=60.0)
    for inst, kind in ((0, GS.PREFILL), (1, GS.PREFILL), (2, GS.DECODE)):
        g.register(inst, kind)
    doc = np.arange(1000, 1000 + 160, dtype=np.int32)          # 10 blocks
    q1 = np.concatenate([doc, np.arange(5, 40, dtype=np.int32)])
    # nothing cached: least load wins (ties -> lowest id)
    g.set_load(0, 3.0)
    assert g.route(GS.PREFILL, q1, 0.0) == (1, 0, [])
    g.update(1, q1, 1.0)                  # instance 1 served q1 (update path)
    g.set_load(1, 9.0)
    # longest common prefix beats load
    assert g.route(GS.PREFILL, q1, 2.0)[:2] == (1, 160 + 32)
    # the decode instance holds more of the prompt: listed as extra holder
    g.update(2, np.concatenate([q1, np.arange(90, 130, dtype=np.int32)]), 3.0)
    inst, mt, extra = g.route(GS.PREFILL, np.concatenate([q1, np.arange(90, 140)]), 4.0)
    assert (inst, mt) == (1, 192) and extra == [(2, 224)]
    # TTL: entries expire -- instance 1's at 61, instance 2's at 63
    assert g.route(GS.PREFILL, q1, 61.5) == (0, 0, [(2, 192)])
    assert g.route(GS.PREFILL, q1, 63.5) == (0, 0, [])



@pytest.mark.parametrize("which", ["oracle", "product"])
def test_ttl_boundary_and_ties(which):
    """R17 boundaries, hand-derived: an update at t is held while now < t + ttl
    ("expire ... after a TTL"), so at exactly t + ttl it is gone;
    a partial last block is not cached (block-granular trees); equal
    prefixes tie to the least load, then the lowest id; extra holders are
    listed longest first, ties by id."""
    GS = _impl(which)
    B = 4
    g = GS(B, ttl_seconds=10.0)
    for inst, kind in ((5, 0), (3, 0), (9, 1), (7, 2)):
        g.register(inst, kind)
    p = np.arange(100, 100 + 3 * B + 2, dtype=np.int32)     # 3 full blocks + 2 tokens
    g.update(5, p, 1.0)
    assert g.route(0, p, 10.999) == (5, 3 * B, [])
    assert g.route(0, p, 11.0) == (3, 0, [])                 # expired at exactly t + ttl
    g.update(5, p, 20.0)
    g.update(3, p[: 2 * B + 1], 20.0)                        # 2 full blocks
    assert g.route(0, p, 21.0) == (5, 3 * B, [])
    g.update(3, p, 21.0)                                     # both hold 3 blocks: tie
    assert g.route(0, p, 22.0) == (3, 3 * B, [])             # equal load -> lowest id
    g.set_load(3, 1.0)
    assert g.route(0, p, 22.0) == (5, 3 * B, [])             # least load wins the tie
    # extra holders of any kind, longest first, ties by id
    longer = np.concatenate([p, np.arange(7, 7 + 2 * B, dtype=np.int32)])
    g.update(9, longer, 23.0)                                # decode: 5 full blocks
    g.update(7, longer[: 4 * B + 3], 23.0)                   # colocated: 4 blocks
    assert g.route(0, longer, 24.0) == (5, 3 * B, [(9, 5 * B), (7, 4 * B)])
    # a query shorter than a cached prompt matches only its own full blocks
    assert g.route(1, p[: B + 3], 24.0) == (9, B, [])
    with pytest.raises(Exception):
        GS(B, 10.0).route(0, p, 0.0)                         # no instance of the kind

def test_random_vs_oracle():
    from paper_2406_17565_b200.mempool import GlobalScheduler as GS, MempoolError
    rng = np.random.default_rng(7)
    for trial in range(30):
        B = int(rng.choice([4, 16]))
        ttl = float(rng.choice([5.0, 50.0]))
        g, o = GS(B, ttl), OracleGS(B, ttl)
        n_inst = int(rng.integers(1, 7))
        for i in range(n_inst):
            kind = int(rng.integers(3))
            g.register(10 + i, kind)
            o.register(10 + i, kind)
        base = [rng.integers(0, 3, size=int(rng.integers(0, 12 * B))).astype(np.int32)
                for _ in range(4)]
        now = 0.0
        for _ in range(60):
            now += float(rng.exponential(2.0))
            b = base[rng.integers(4)]
            q = np.concatenate([b[: int(rng.integers(0, len(b) + 1))],
                                rng.integers(0, 3, size=int(rng.integers(0, 4 * B)))
                                ]).astype(np.int32)
            op = rng.random()
            inst = 10 + int(rng.integers(n_inst))
            if op < 0.4:
                g.update(inst, q, now)
                o.update(inst, q, now)
            elif op < 0.5:
                load = float(rng.integers(0, 4))
                g.set_load(inst, load)
                o.set_load(inst, load)
            else:
                kind = int(rng.integers(3))
                want = o.route(kind, q, now)
                if want is None:
                    with pytest.raises(MempoolError):
                        g.route(kind, q, now)
                else:
                    assert g.route(kind, q, now) == want


@pytest.mark.gpu
def test_fan_in_fetch_from_extra_holder():
    """Route to the idle prefill instance, then pull the longer cached prefix
    from the extra holder (suffix transfer_with_insert): bytes and index match
    the oracle, and the routed instance now matches the whole prefix."""
    import oracle as O
    from paper_2406_17565_b200 import mempool as M
    from tests.twin import Twin, connect, transfer_with_insert
    from workloads.configs import TINY
    B = TINY.block_tokens
    # a prefill instance holding 2 blocks of the conversation and a decode
    # instance holding 6 (it decoded the answer: PD-Caching-2)
    P0, D1 = Twin(0, TINY, 64), Twin(1, TINY, 64)
    connect(P0, D1)
    gs, og = M.GlobalScheduler(B, 100.0), OracleGS(B, 100.0)
    for inst, kind in ((0, 0), (1, 1)):
        gs.register(inst, kind)
        og.register(inst, kind)
    conv = np.arange(2000, 2000 + 6 * B, dtype=np.int32)
    for pool, toks, inst in ((P0, conv[: 2 * B], 0), (D1, conv, 1)):
        _, m = pool.match(toks)
        new = pool.alloc(len(toks) // B - len(m))
        pool.fill(new)
        pool.insert(toks, m + new)
        gs.update(inst, toks, 1.0)
        og.update(inst, toks, 1.0)
    query = np.concatenate([conv, np.arange(7, 7 + B, dtype=np.int32)])   # next turn
    # the prefill pick holds 2 blocks; the decode instance holds extra KV
    got = gs.route(0, query, 2.0)
    assert got == og.route(0, query, 2.0) == (0, 2 * B, [(1, 6 * B)])
    # fan-in: the chosen instance fetches blocks [2, 6) from the extra holder
    # with a suffix transfer_with_insert (R3)
    _, d_addrs = D1.match(conv)
    transfer_with_insert(D1, P0, conv, d_addrs[2:], path=M.PATH_FUSED)
    gs.update(0, conv, 3.0)
    og.update(0, conv, 3.0)
    assert P0.match(conv)[0] == 6 * B
    assert gs.route(0, query, 4.0) == og.route(0, query, 4.0) == (0, 6 * B, [])
    P0.check_state()
    D1.check_state()
