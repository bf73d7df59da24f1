"""Oracle of the global scheduler's prompt-tree routing (test infrastructure
only -- see oracle/__init__.py).  PAPER.md §6: global prompt trees
record which instance holds which prefix, with a TTL;
lookup chooses "an instance with the longest common prefix" and lists
instances "storing extra historical KV cache that is not present in the
chosen instance".  Readings R17: ties to the least
load then the lowest id; extra holders of any kind, longest first.

Brute force, no tree: each instance keeps its list of updates (block-truncated
prompt, time); its cached prefix for a query is the longest block-aligned
common prefix with any update still within the TTL."""


def _lcp(a, b):
    n = min(len(a), len(b))
    i = 0
    while i < n and a[i] == b[i]:
        i += 1
    return i


class OracleGS:
    def __init__(self, block_tokens, ttl):
        self.B = block_tokens
        self.ttl = ttl
        self.kind = {}
        self.load = {}
        self.updates = {}

    def register(self, inst, kind):
        assert inst not in self.kind and kind in (0, 1, 2)
        self.kind[inst] = kind
        self.load[inst] = 0.0
        self.updates[inst] = []

    def set_load(self, inst, load):
        self.load[inst] = load

    def update(self, inst, tokens, now):
        k = len(tokens) // self.B
        self.updates[inst].append((tuple(int(t) for t in tokens[: k * self.B]), now))

    def cached_blocks(self, inst, tokens, now):
        q = tuple(int(t) for t in tokens)
        best = 0
        for s, t in self.updates[inst]:
            if t + self.ttl > now:
                best = max(best, min(_lcp(q, s), len(s)) // self.B)
        return best

    def route(self, kind, tokens, now):
        cands = [i for i in sorted(self.kind) if self.kind[i] == kind]
        if not cands:
            return None
        blocks = {i: self.cached_blocks(i, tokens, now) for i in self.kind}
        pick = min(cands, key=lambda i: (-blocks[i], self.load[i], i))
        extra = sorted(((blocks[i], i) for i in self.kind if blocks[i] > blocks[pick]),
                       key=lambda x: (-x[0], x[1]))
        return pick, blocks[pick] * self.B, [(i, b * self.B) for b, i in extra]
