"""Host-side sharding of the request stream across ranks (multi-GPU plan).

Samples are split into contiguous shards whose boundaries are multiples of lcm(B), so no batch of
any candidate size straddles two ranks (batch ids and arrival times stay global through
`global_offset`). Only the last shard may be ragged. Plain integer arithmetic, no compute.
"""
from __future__ import annotations

from math import gcd


def lcm_of(B) -> int:
    L = 1
    for b in B or []:
        L = L * b // gcd(L, b)
    return L


def shard_ranges(N: int, world: int, B=None):
    """[(offset, count)] for each rank; offsets are multiples of lcm(B)."""
    if world < 1 or N < 0:
        raise ValueError("bad N / world")
    L = lcm_of(B)
    units = -(-N // L) if N else 0
    out = []
    for r in range(world):
        u0 = units * r // world
        u1 = units * (r + 1) // world
        a = min(u0 * L, N)
        b = min(u1 * L, N)
        out.append((a, b - a))
    return out


def chunk_ranges(offset: int, count: int, chunk: int, B=None):
    """Split one shard into streaming chunks (multiples of lcm(B); only the last may be ragged)."""
    L = lcm_of(B)
    chunk = max(L, chunk // L * L)
    out = []
    s = 0
    while s < count:
        n = min(chunk, count - s)
        out.append((offset + s, n))
        s += n
    return out
