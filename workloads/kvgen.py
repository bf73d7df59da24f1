"""Counter-based synthetic KV content (SURVEY.md §8(c) "Content model").

The paper never shows KV contents, so every "prefill/decode write" of a block
is replaced by a deterministic fill.  A write carries a tag
    T = inst * 2**40 + epoch * 2**14 + block          (block < 2**14, epoch < 2**26)
where ``epoch`` is the writing pool's fill counter.  The 64-bit word t of chunk
j = 2*layer + kv (chunk_words = c / 8 words per chunk) is

    word = splitmix64(seed ^ splitmix64(T) ^ (j * chunk_words + t))

All arithmetic is mod 2**64.  Any bit pattern (NaN fp16 payloads included) is
legal: migration is compared as integers, never as fp16.

This generator is an INPUT generator: the CUDA fill kernel implements the same
formula independently; nothing here is part of the migration method.
"""
import numpy as np

_M = np.uint64(0xFFFFFFFFFFFFFFFF)
_G = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x):
    """Vigna's splitmix64 finaliser on a uint64 ndarray (wraps mod 2**64)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _G
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
    return z ^ (z >> np.uint64(31))


def make_tag(inst: int, epoch: int, block: int) -> int:
    assert 0 <= block < (1 << 14), "block index must fit 14 bits"
    assert 0 <= epoch < (1 << 26), "epoch must fit 26 bits"
    assert 0 <= inst < (1 << 24)
    return (inst << 40) | (epoch << 14) | block


def chunk_words(seed: int, tag: int, chunk: int, words_per_chunk: int) -> np.ndarray:
    """The words_per_chunk uint64 words of chunk ``chunk`` of a block written with ``tag``."""
    t = np.arange(words_per_chunk, dtype=np.uint64)
    base = np.uint64(seed) ^ splitmix64(np.array([tag], dtype=np.uint64))[0]
    ctr = np.uint64(chunk * words_per_chunk) + t
    return splitmix64(base ^ ctr)


def block_words(seed: int, tags, words_per_chunk: int) -> np.ndarray:
    """Aggregated-layout words of one block whose chunk j was written with tags[j].

    Returns uint64 [n_chunks, words_per_chunk]; ``tags[j] is None`` (never
    written) yields zeros -- callers must not compare such chunks.
    """
    out = np.zeros((len(tags), words_per_chunk), dtype=np.uint64)
    for j, tag in enumerate(tags):
        if tag is not None:
            out[j] = chunk_words(seed, tag, j, words_per_chunk)
    return out
