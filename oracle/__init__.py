"""CPU ORACLE -- test infrastructure only.

A plain, slow, obviously-correct CPU model of MemPool's block pool, prompt
index and KV-block migration (§4 "Elastic Memory Pool", Table
tbl-mempool-api P:261-290; §4.2 indexing P:326-337; §4.3 transfer workflow
P:360-369; §5.2 aggregation P:549-550), with every place the paper is silent
filled by the readings R1-R17 listed in DESIGN.md §3 (R1-R13 = SURVEY.md §8(c)).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2406_17565_b200``, ``libmempool.so``) never imports it and shares no
code with it; the only shared module is ``workloads`` (seeded input
generators, no method arithmetic).

Parity status: see DESIGN.md §3.  Pinned: allocator (lowest-first, S:131-133
examples, conservation), match/insert/delete incl. R6 (brute-force set-of-
sequences model, SPEC examples), migration bytes (closed form
dst[d_j] == src[s_j], np.take cross-check), golden worked example; and by
independent models in tests/test_oracle_pins.py: LRU eviction and swap-out
victims (R7-R9, recency recomputed from the op history), evict-before-OOM
feasibility (R2, subset brute force), DEDUP reuse of the receiver's cached
prefix (R3, bytes + reuse + conservation); the block aggregation (pack's
layout and the network-call counts of P:546-552: 10,240 discrete vs 128
aggregated calls for the paper's 2048-token / L=40 instance, block i at
i*Pb; tests/test_oracle_aggregation.py); the global scheduler's routing
(gs_oracle.py) by hand-derived cases of P:641-649 incl. the TTL boundary
(tests/test_gs.py).  Tie-breaks between equally recent
blocks (lowest block index) are a reading no model can pin: a single op
never leaves two leaves equally recent, so it only orders the initial state.
"""
from .mempool_oracle import (  # noqa: F401
    HBM, DRAM, MIXED, FREE, ACTIVE, INDEXED, ORPHAN,
    FLAG_DST_GIVEN, FLAG_DEDUP, FLAG_INS_ERR_ON_CONFLICT, FLAG_MATCH_PIN,
    MPError, OraclePool, transfer, transfer_with_insert, transfer_heads, tp_plan,
    pack, network_calls,
)
