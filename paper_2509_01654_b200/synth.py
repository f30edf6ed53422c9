"""Deterministic synthetic vocabularies for BASELINE.json's five configs.

The paper publishes no word list and no length distribution, so these
generators ARE the workload definition; each is frozen by a
blake2b digest of its ``(ids, lengths)`` arrays in ``tests/golden/synth_digests.json``.

Words come back as a packed word store: ``ids`` is ``(n, q)`` uint8, zero padded
on the right, ``lengths`` is ``(n,)`` uint8.  ``as_encoded_words`` turns a store
into ``EncodedWord`` objects for the ``compute_all_pairs`` entry point.
"""
from __future__ import annotations

import hashlib
import random
from typing import List, Tuple

import numpy as np

from .host_types import EncodedWord

ALPHABET = 40
CONFIG_SCHEMES = {
    "C1": (1, -1, -2), "C2": (1, -1, -2), "C3": (1, -1, -2), "C4": (1, -1, -2),
    "C5": (2, -1, -3),
}
CONFIG_N = {"C1": 1_000, "C2": 20_000, "C3": 100_000, "C4": 600_000, "C5": 600_000}
C5_THRESHOLD = 4


def make_words(n: int, seed: int = 0, alphabet: int = 12, min_len: int = 1,
               max_len: int = 9) -> List[EncodedWord]:
    """Same stream as the reference test generator (tests/conftest.py:13-24):
    ``random.Random(seed)``; per word one ``randint`` for the length, then one
    ``randrange(alphabet)`` per symbol."""
    rng = random.Random(seed)
    words = []
    for i in range(n):
        length = rng.randint(min_len, max_len)
        ph = tuple(rng.randrange(alphabet) for _ in range(length))
        words.append(EncodedWord(f"w{i:04d}", f"ipa{i:04d}", ph, float(n - i)))
    return words


def store_from_words(words) -> Tuple[np.ndarray, np.ndarray]:
    n = len(words)
    q = max(len(w.phonemes) for w in words)
    ids = np.zeros((n, q), dtype=np.uint8)
    lengths = np.empty(n, dtype=np.uint8)
    for i, w in enumerate(words):
        lengths[i] = len(w.phonemes)
        ids[i, : len(w.phonemes)] = w.phonemes
    return ids, lengths


def _symbol_pmf() -> np.ndarray:
    p = 1.0 / (np.arange(ALPHABET) + 3.0)
    return p / p.sum()


def _fill(rng, lengths: np.ndarray) -> np.ndarray:
    n = lengths.size
    q = int(lengths.max())
    total = int(lengths.sum())
    syms = rng.choice(ALPHABET, size=total, p=_symbol_pmf()).astype(np.uint8)
    ids = np.zeros((n, q), dtype=np.uint8)
    mask = np.arange(q)[None, :] < lengths[:, None]
    ids[mask] = syms  # row-major fill: word 0's symbols first
    return ids


def french_shaped(n: int, seed: int | None = None) -> Tuple[np.ndarray, np.ndarray]:
    """C2/C3/C4: length ~ clip(round(N(8.5, 2.8)), 1, 24); symbol k with
    p_k proportional to 1/(k+3); generation order kept (no sorting)."""
    rng = np.random.default_rng(20250901 + n if seed is None else seed)
    lengths = np.clip(np.rint(rng.normal(8.5, 2.8, size=n)), 1, 24).astype(np.uint8)
    return _fill(rng, lengths), lengths


def skewed_tail(n: int, seed: int = 20250905) -> Tuple[np.ndarray, np.ndarray]:
    """C5: 97 % French-shaped + 3 % uniform{16..21}, all clipped to 21 (the
    int8 preflight bound for gap -3)."""
    rng = np.random.default_rng(seed)
    base = np.clip(np.rint(rng.normal(8.5, 2.8, size=n)), 1, 21)
    tail = rng.integers(16, 22, size=n)
    pick = rng.random(n) < 0.03
    lengths = np.where(pick, tail, base).astype(np.uint8)
    return _fill(rng, lengths), lengths


def config_store(name: str, n: int | None = None) -> Tuple[np.ndarray, np.ndarray, Tuple[int, int, int]]:
    """(ids, lengths, (match, mismatch, gap)) for C1..C5; ``n`` overrides the size
    (the generator seed follows n for the French-shaped configs)."""
    scheme = CONFIG_SCHEMES[name]
    n = CONFIG_N[name] if n is None else n
    if name == "C1":
        ids, lengths = store_from_words(make_words(n, seed=n, alphabet=ALPHABET, min_len=1, max_len=16))
    elif name == "C5":
        ids, lengths = skewed_tail(n)
    else:
        ids, lengths = french_shaped(n)
    return ids, lengths, scheme


def as_encoded_words(ids: np.ndarray, lengths: np.ndarray) -> List[EncodedWord]:
    n = lengths.size
    return [
        EncodedWord(f"w{i}", f"ipa{i}", tuple(int(x) for x in ids[i, : lengths[i]]), float(n - i))
        for i in range(n)
    ]


def store_digest(ids: np.ndarray, lengths: np.ndarray) -> str:
    h = hashlib.blake2b(digest_size=16)
    h.update(np.ascontiguousarray(ids, dtype=np.uint8).tobytes())
    h.update(np.ascontiguousarray(lengths, dtype=np.uint8).tobytes())
    h.update(f"{ids.shape}".encode())
    return h.hexdigest()


def total_cells(lengths: np.ndarray) -> int:
    """DP cell updates of the full all-pairs job: ((sum len)^2 - sum len^2) / 2."""
    L = np.asarray(lengths, dtype=np.int64)
    s1 = int(L.sum())
    s2 = int((L * L).sum())
    return (s1 * s1 - s2) // 2
