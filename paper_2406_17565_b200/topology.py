"""Placement of prefill (P) and decode (D) instances on the GPUs of one box.

SURVEY.md §8(e): the units of work are independent (P_i, D_i) pairs; with N
GPUs, P_i is GPU i and D_i is GPU i + N/2 (1P1D = {0->1}, 2P2D = {0->2, 1->3},
4P4D = {0->4, 1->5, 2->6, 3->7}).  One process per GPU; the only exchange is
the point-to-point wire inside each pair -- no collective.  N = 1 puts both
instances of the single pair on GPU 0 (loopback).
"""
from dataclasses import dataclass


@dataclass(frozen=True)
class Role:
    rank: int
    world: int
    kind: str          # "P", "D", or "PD" (both pools in this process, N = 1)
    pair: int          # pair index i
    partner: int       # partner rank (== rank for "PD")
    p_inst: int        # instance id of the pair's prefill pool
    d_inst: int        # instance id of the pair's decode pool


def role_of(rank: int, world: int) -> Role:
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank / world")
    if world == 1:
        return Role(0, 1, "PD", 0, 0, 0, 1)
    if world % 2:
        raise ValueError("P/D pairs need an even number of GPUs")
    half = world // 2
    pair = rank % half
    kind = "P" if rank < half else "D"
    partner = rank + half if kind == "P" else rank - half
    return Role(rank, world, kind, pair, partner, 2 * pair, 2 * pair + 1)
