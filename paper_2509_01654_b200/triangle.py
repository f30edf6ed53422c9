"""Exact integer geometry of the condensed upper triangle (host side).

Row-major enumeration (0,1),(0,2),...,(n-2,n-1); an edge's linear index is its
byte offset in the payload.  Mirrors the scalar functions of the reference's
``triangle.py:36-90``; the vectorised index recovery (``rows_of_array``,
``triangle.py:93-112``) is done on the device, once per tile, by
``csrc/nwap_index.cuh``.  Everything here is Python big-int arithmetic.
"""
from __future__ import annotations

import math


def num_edges(n: int) -> int:
    if n < 1:
        raise ValueError(f"node count must be >= 1, got {n}")
    return n * (n - 1) // 2


def edges_before_row(r: int, n: int) -> int:
    return r * (2 * n - r - 1) // 2


def row_of(idx: int, n: int) -> int:
    total = num_edges(n)
    if not 0 <= idx < total:
        raise ValueError(f"edge index {idx} out of range [0, {total}) for n={n}")
    # exact: largest r with r*(2n-r-1)/2 <= idx, via integer sqrt of the discriminant
    m = 2 * n - 1
    r = (m - math.isqrt(m * m - 8 * idx)) // 2
    r = min(max(r, 0), n - 2)
    while r > 0 and idx < edges_before_row(r, n):
        r -= 1
    while idx >= edges_before_row(r + 1, n):
        r += 1
    return r


def col_of(idx: int, n: int, r: int) -> int:
    lo = edges_before_row(r, n)
    if not (0 <= r <= n - 2 and lo <= idx < edges_before_row(r + 1, n)):
        raise ValueError(f"row {r} is inconsistent with edge index {idx} for n={n}")
    return r + 1 + (idx - lo)


def index_of(r: int, c: int, n: int) -> int:
    if not 0 <= r < c <= n - 1:
        raise ValueError(f"invalid edge ({r}, {c}) for n={n}: need 0 <= r < c <= n-1")
    return edges_before_row(r, n) + (c - r - 1)
