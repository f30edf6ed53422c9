"""Host-side value types at the drop-in boundary.

These mirror, field for field, the types the reference's scoring entry point
takes and returns, so a caller of ``phonsim.engine.compute_all_pairs`` can pass
its own objects unchanged (everything here is duck-typed on attribute names):

* ``EncodedWord``   -- reference ``corpus.py:52-62`` (only ``.phonemes`` is read on this path)
* ``ScoringScheme`` -- reference ``aligner.py:39-87``
* ``ComputePlan``   -- reference ``engine.py:39-60``
* ``ComputeStats``  -- reference ``engine.py:63-69``
* ``DataError`` / ``PhonsimError`` -- reference ``errors.py:4-10``

When the reference package itself is importable (``import phonsim``), its
exception classes are re-used so ``except phonsim.DataError`` keeps working.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field
from typing import Iterator, Mapping, Tuple

try:  # pragma: no cover - only when the reference is on sys.path
    from phonsim.errors import DataError, PhonsimError  # type: ignore
except Exception:  # noqa: BLE001
    class PhonsimError(Exception):
        """Root of the error hierarchy (reference errors.py:4)."""

    class DataError(PhonsimError):
        """Input violates a contract, e.g. a scheme whose scores cannot fit
        one signed byte (reference errors.py:8)."""


DEFAULT_CHUNK_SIZE = 65536  # reference engine.py:36


@dataclass(frozen=True)
class EncodedWord:
    word: str
    ipa: str
    phonemes: Tuple[int, ...]
    frequency: float = 0.0

    def __len__(self) -> int:
        return len(self.phonemes)


@dataclass(frozen=True)
class ScoringScheme:
    """match / mismatch / gap plus optional symmetric per-pair overrides."""

    match: int = 1
    mismatch: int = -1
    gap: int = -1
    overrides: Mapping[Tuple[int, int], int] = field(default_factory=dict)

    def __post_init__(self):
        ov = self.overrides
        for (a, b), v in ov.items():
            if (b, a) in ov and ov[(b, a)] != v:
                raise ValueError(f"asymmetric override for pair ({a}, {b}): {v} vs {ov[(b, a)]}")

    def similarity(self, a: int, b: int) -> int:
        ov = self.overrides
        if (a, b) in ov:
            return ov[(a, b)]
        if (b, a) in ov:
            return ov[(b, a)]
        return self.match if a == b else self.mismatch

    def _all_values(self):
        return [self.match, self.mismatch, *self.overrides.values()]

    @property
    def min_similarity(self) -> int:
        return min(self._all_values())

    @property
    def max_similarity(self) -> int:
        return max(self._all_values())

    def hash_hex(self) -> str:
        # byte-compatible with reference aligner.py:81-87 so manifests agree
        h = hashlib.blake2b(digest_size=8)
        h.update(f"{self.match} {self.mismatch} {self.gap}".encode())
        for (a, b), v in sorted(self.overrides.items()):
            h.update(f" {a},{b}={v}".encode())
        return h.hexdigest()


DEFAULT_SCHEME = ScoringScheme()


def scheme_fields(scheme) -> tuple:
    """(match, mismatch, gap, overrides dict) of any duck-typed scheme."""
    return (int(scheme.match), int(scheme.mismatch), int(scheme.gap),
            dict(getattr(scheme, "overrides", {}) or {}))


def same_scheme(a, b) -> bool:
    return scheme_fields(a) == scheme_fields(b)


@dataclass(frozen=True)
class ComputePlan:
    """Partitioning of one all-pairs run (reference engine.py:39-60).

    On the GPU path ``chunk_size`` is only the granularity of ``sink.write``
    calls (the payload never depends on it) and ``worker_count`` is accepted
    for signature compatibility and ignored: one process drives one GPU.
    """

    n: int
    chunk_size: int = DEFAULT_CHUNK_SIZE
    worker_count: int = 1
    scheme: ScoringScheme = DEFAULT_SCHEME

    def __post_init__(self):
        if self.n < 2:
            raise ValueError("need at least two words")
        if self.chunk_size < 1:
            raise ValueError("chunk_size must be positive")
        if self.worker_count < 1:
            raise ValueError("worker_count must be positive")

    def chunks(self) -> Iterator[Tuple[int, int]]:
        total = self.n * (self.n - 1) // 2
        pos = 0
        while pos < total:
            nxt = min(pos + self.chunk_size, total)
            yield pos, nxt
            pos = nxt


@dataclass
class ComputeStats:
    edges_written: int
    wall_time: float
    min_score: int
    max_score: int
    mean_score: float
