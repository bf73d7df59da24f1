"""Seeded token traces shaped like the paper's workloads.

The paper's datasets (ShareGPT, LooGLE, ReAct/HotpotQA; §7.2,
Table tbl-workloads) are not available and their length
distributions exist only in a figure, so the shapes below are the
stated recipe of SURVEY.md §8(d):

* tokens: int32 uniform in [3, 32000) (Llama-2 vocabulary), numpy PCG64;
* ShareGPT-like: sessions of 1-4 turns; per turn user U[16,512] and
  generation U[16,512] ("uniform"); prompt_k = prompt_{k-1} + gen_{k-1}
  + user_k, capped at 4096 tokens (Llama-2 context);
* LooGLE-like: a document prefix U{16384..32768} tokens, 5 questions
   of U[16,64] tokens, answers U[8,32] (short generation);
  prompt_k = prompt_{k-1} + answer_{k-1} + question_k;
* ReAct-like: one shared two-shot prefix of 1536 tokens, a question
  U[32,128], 3-6 steps; per step generation U[128,512] (long) and an
  observation U[32,256] appended to the next prompt.

Only inputs are produced here -- no allocation, indexing or migration logic.
"""
from dataclasses import dataclass, field
from typing import List

import numpy as np

VOCAB_LO, VOCAB_HI = 3, 32000


def rng_for(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def tokens(rng: np.random.Generator, n: int) -> np.ndarray:
    return rng.integers(VOCAB_LO, VOCAB_HI, size=n, dtype=np.int32)


@dataclass
class Turn:
    prompt: np.ndarray   # int32 token ids of this turn's full prompt
    gen: np.ndarray      # int32 token ids the decode phase produces


@dataclass
class Session:
    sid: int
    turns: List[Turn] = field(default_factory=list)


def golden_prompts():
    """The golden worked example of SURVEY.md §8(c): S, p1, p2, p3."""
    S = np.arange(100, 140, dtype=np.int32)
    p1 = np.concatenate([S, np.arange(200, 217, dtype=np.int32)])
    p2 = np.concatenate([S, np.arange(300, 332, dtype=np.int32)])
    p3 = np.concatenate([S, np.arange(400, 408, dtype=np.int32)])
    return S, p1, p2, p3


def sharegpt_like(seed: int, n_sessions: int = 256, max_turns: int = 4,
                  ctx: int = 4096) -> List[Session]:
    rng = rng_for(seed)
    out = []
    for s in range(n_sessions):
        sess = Session(s)
        nt = int(rng.integers(1, max_turns + 1))
        prev = np.zeros(0, np.int32)
        prev_gen = np.zeros(0, np.int32)
        for _ in range(nt):
            user = tokens(rng, int(rng.integers(16, 513)))
            prompt = np.concatenate([prev, prev_gen, user])[:ctx]
            gen = tokens(rng, int(rng.integers(16, 513)))
            gen = gen[: max(0, ctx - len(prompt))]
            sess.turns.append(Turn(prompt, gen))
            prev, prev_gen = prompt, gen
            if len(prompt) + len(gen) >= ctx:
                break
        out.append(sess)
    return out


def loogle_like(seed: int, n_sessions: int = 8, doc_lo: int = 16384,
                doc_hi: int = 32768, n_questions: int = 5) -> List[Session]:
    rng = rng_for(seed)
    out = []
    for s in range(n_sessions):
        sess = Session(s)
        prev = tokens(rng, int(rng.integers(doc_lo, doc_hi + 1)))
        prev_gen = np.zeros(0, np.int32)
        for _ in range(n_questions):
            q = tokens(rng, int(rng.integers(16, 65)))
            prompt = np.concatenate([prev, prev_gen, q])
            gen = tokens(rng, int(rng.integers(8, 33)))
            sess.turns.append(Turn(prompt, gen))
            prev, prev_gen = prompt, gen
        out.append(sess)
    return out


def react_like(seed: int, n_sessions: int = 16, prefix_len: int = 1536) -> List[Session]:
    rng = rng_for(seed)
    shared = tokens(rng, prefix_len)
    out = []
    for s in range(n_sessions):
        sess = Session(s)
        prompt = np.concatenate([shared, tokens(rng, int(rng.integers(32, 129)))])
        for _ in range(int(rng.integers(3, 7))):
            gen = tokens(rng, int(rng.integers(128, 513)))
            sess.turns.append(Turn(prompt, gen))
            obs = tokens(rng, int(rng.integers(32, 257)))
            prompt = np.concatenate([prompt, gen, obs])
        out.append(sess)
    return out


def scattered_ids(seed: int, n_pool: int, n: int) -> np.ndarray:
    """A seeded random choice of n distinct block ids out of n_pool (sweeps)."""
    rng = rng_for(seed)
    return rng.permutation(n_pool)[:n].astype(np.int64)
