"""KV shapes of the BASELINE.json configs (SURVEY.md §8 shape table).

fp16 KV (2 B per element; the paper never states precision, vLLM's default is
fp16 -- BASELINE.md §2).  Block size B = 16 tokens (§4.2 P:337:
"vLLM, which uses a block size of 16 tokens").

One engine block of B tokens is stored "discretely" as 2*L chunks, one per
(layer, K/V) (§5.2: "vLLM allocates two blocks per LLM
layer ... the engine needs 2*L blocks").  A chunk is B*H*D*elem bytes.
"""
from dataclasses import dataclass


@dataclass(frozen=True)
class KVShape:
    name: str
    layers: int        # L
    kv_heads: int      # H
    head_dim: int      # D
    block_tokens: int  # B
    elem_bytes: int = 2

    @property
    def chunk_bytes(self) -> int:
        """c = B*H*D*elem: one (layer, K/V) chunk of one block."""
        return self.block_tokens * self.kv_heads * self.head_dim * self.elem_bytes

    @property
    def n_chunks(self) -> int:
        """2*L chunks per token block."""
        return 2 * self.layers

    @property
    def block_bytes(self) -> int:
        """Pb = 2*L*c: the aggregated block."""
        return self.n_chunks * self.chunk_bytes


TINY = KVShape("tiny", 2, 2, 64, 16)            # BASELINE.json configs[0]
LLAMA2_7B = KVShape("llama2-7b", 32, 32, 128, 16)  # configs[1], configs[4]
LLAMA2_13B = KVShape("llama2-13b", 40, 40, 128, 16)  # configs[2], configs[3]

SHAPES = {s.name: s for s in (TINY, LLAMA2_7B, LLAMA2_13B)}

# Seed = 17565 + config index (SURVEY.md §8(d) "Concrete synthetic inputs").
SEED_BASE = 17565


def seed_for(config_index: int) -> int:
    return SEED_BASE + config_index
