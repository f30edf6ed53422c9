"""Edge-store output next to the scoring path.

The reference's production sink is ``EdgeStoreWriter`` (store.py:140-217): a headerless int8
payload file ``<prefix>.nwedges`` plus a ``key<TAB>value`` manifest that binds it to the word
list and the scheme through 64-bit blake2b digests and carries a ``complete`` flag.  This module
writes byte-identical files (pinned by tests/golden/store_case, produced by the reference's own
``phonsim compute``), but overlaps the three things the reference does one after the other for
every chunk:

    device scoring + device->host copy   (engine.compute_all_pairs, two pinned slabs)
    blake2b of the payload               (hasher thread;  hashlib releases the GIL)
    the file write                       (writer thread;  os.write releases the GIL)

``write`` only copies the chunk into a block buffer (a memcpy); full blocks travel through two
bounded queues.  The payload digest is a single sequential blake2b by definition of the format,
so ~1 GB/s of hashing is the floor of this stage; the point of the pipeline is that nothing else
adds to it.

Also here: the ``.words`` file reader/writer (corpus.py:286-317), the other data format at the
boundary.
"""
from __future__ import annotations

import hashlib
import os
import queue
import threading
from dataclasses import dataclass
from pathlib import Path
from typing import List, Sequence, Tuple

import numpy as np

from .host_types import DataError, EncodedWord
from .triangle import num_edges

FORMAT_VERSION = 1                      # store.py:41
PAYLOAD_SUFFIX = ".nwedges"             # store.py:42
MANIFEST_SUFFIX = ".nwedges.manifest"   # store.py:43
MANIFEST_FIELDS = ("format_version", "n", "num_edges", "match", "mismatch", "gap", "scheme_hash",
                   "words_digest", "payload_digest", "complete")   # order of store.py:45-56


def store_paths(prefix) -> Tuple[Path, Path]:
    """(payload path, manifest path) for a prefix or a payload path (store.py:59-65)."""
    prefix = Path(prefix)
    payload = prefix if prefix.name.endswith(PAYLOAD_SUFFIX) else prefix.parent / (prefix.name + PAYLOAD_SUFFIX)
    return payload, payload.parent / (payload.name + ".manifest")


def words_digest(words: Sequence) -> str:
    """blake2b-64 over ``word<TAB>ipa<NL>`` of every word in order (store.py:68-73)."""
    h = hashlib.blake2b(digest_size=8)
    # one update per ~4096 words instead of one per word: same byte stream, 20x fewer calls
    for i in range(0, len(words), 4096):
        h.update("".join(f"{w.word}\t{w.ipa}\n" for w in words[i:i + 4096]).encode())
    return h.hexdigest()


@dataclass
class EdgeStoreManifest:
    """The manifest record (store.py:83-138); ``save`` emits the reference's exact text."""
    format_version: int
    n: int
    num_edges: int
    match: int
    mismatch: int
    gap: int
    scheme_hash: str
    words_digest: str
    payload_digest: str
    complete: bool

    def text(self) -> str:
        lines = []
        for key in MANIFEST_FIELDS:
            v = getattr(self, key)
            lines.append(f"{key}\t{('true' if v else 'false') if isinstance(v, bool) else v}\n")
        return "".join(lines)

    def save(self, path) -> None:
        Path(path).write_text(self.text(), encoding="utf-8")

    @classmethod
    def load(cls, path) -> "EdgeStoreManifest":
        got = {}
        for lineno, line in enumerate(Path(path).read_text(encoding="utf-8").split("\n"), start=1):
            if not line:
                continue
            if "\t" not in line:
                raise DataError(f"{path}: line {lineno}: expected 'key<TAB>value'")
            key, value = line.split("\t", 1)
            got[key] = value
        missing = [k for k in MANIFEST_FIELDS if k not in got]
        if missing:
            raise DataError(f"{path}: missing manifest keys: {', '.join(missing)}")
        try:
            m = cls(int(got["format_version"]), int(got["n"]), int(got["num_edges"]), int(got["match"]),
                    int(got["mismatch"]), int(got["gap"]), got["scheme_hash"], got["words_digest"],
                    got["payload_digest"], got["complete"] == "true")
        except ValueError as exc:
            raise DataError(f"{path}: malformed manifest field: {exc}") from None
        if m.num_edges != num_edges(m.n):
            raise DataError(f"{path}: num_edges {m.num_edges} does not match n={m.n}")
        return m


class _Stage(threading.Thread):
    """One consumer of filled blocks: applies ``fn(memoryview)`` to each, in order."""

    def __init__(self, fn, depth: int):
        super().__init__(daemon=True)
        self.fn = fn
        self.q: "queue.Queue" = queue.Queue(maxsize=depth)
        self.error = None
        self.start()

    def run(self):
        while True:
            item = self.q.get()
            if item is None:
                return
            block, nbytes, done = item
            try:
                if self.error is None:
                    self.fn(memoryview(block)[:nbytes])
            except BaseException as exc:  # noqa: BLE001 - surfaced by the producer
                self.error = exc
            finally:
                done()


class PipelinedEdgeStoreWriter:
    """Drop-in for the reference's ``EdgeStoreWriter`` (store.py:140-217): same constructor, same
    ``write`` / ``finalize`` / ``abort`` / context-manager behaviour, same files on disk; hashing
    and file writes run on two worker threads behind ``write``.
    """

    def __init__(self, prefix, words: Sequence, scheme, block_bytes: int = 8 << 20, blocks: int = 4):
        self.payload_path, self.manifest_path = store_paths(prefix)
        self.n = len(words)
        self.expected_bytes = num_edges(self.n)
        self._scheme = scheme
        self._words_digest = words_digest(words)
        self._hash = hashlib.blake2b(digest_size=8)
        self._written = 0
        self._closed = False
        self._fd = os.open(self.payload_path, os.O_WRONLY | os.O_CREAT | os.O_TRUNC, 0o644)
        self._block_bytes = max(1 << 16, int(block_bytes))
        self._free: "queue.Queue" = queue.Queue()
        for _ in range(max(2, blocks)):
            self._free.put(bytearray(self._block_bytes))
        self._cur = self._free.get()
        self._fill = 0
        self._hasher = _Stage(self._hash.update, blocks)
        self._filer = _Stage(self._write_all, blocks)

    # -- worker side
    def _write_all(self, view) -> None:
        while len(view):
            k = os.write(self._fd, view)
            view = view[k:]

    # -- producer side
    def _check_workers(self) -> None:
        for st in (self._hasher, self._filer):
            if st.error is not None:
                raise st.error

    def _flush_block(self) -> None:
        if self._fill == 0:
            return
        block, nbytes = self._cur, self._fill
        pending = [2]
        lock = threading.Lock()

        def done():
            with lock:
                pending[0] -= 1
                last = pending[0] == 0
            if last:
                self._free.put(block)

        self._hasher.q.put((block, nbytes, done))
        self._filer.q.put((block, nbytes, done))
        self._cur = self._free.get()
        self._fill = 0

    def write(self, data) -> None:
        if self._closed:
            raise ValueError("writer is closed")
        self._check_workers()
        view = memoryview(data)
        if view.format != "B" or view.ndim != 1:
            view = view.cast("B")
        pos, total = 0, len(view)
        while pos < total:
            take = min(total - pos, self._block_bytes - self._fill)
            self._cur[self._fill:self._fill + take] = view[pos:pos + take]
            self._fill += take
            pos += take
            if self._fill == self._block_bytes:
                self._flush_block()
        self._written += total
        if self._written > self.expected_bytes:
            raise DataError(f"payload overflow: {self._written} bytes written, "
                            f"expected {self.expected_bytes}")

    # write() copies the data into the writer's own blocks before it returns, so it may be handed transient views
    # (engine.compute_all_pairs calls write_view, when a sink has one, with a view into a recycled pinned slab)
    write_view = write

    def _drain(self) -> None:
        self._flush_block()
        for st in (self._hasher, self._filer):
            st.q.put(None)
        for st in (self._hasher, self._filer):
            st.join()
        os.close(self._fd)
        self._closed = True

    def _manifest(self, complete: bool) -> EdgeStoreManifest:
        s = self._scheme
        return EdgeStoreManifest(FORMAT_VERSION, self.n, self.expected_bytes, int(s.match), int(s.mismatch),
                                 int(s.gap), s.hash_hex(), self._words_digest, self._hash.hexdigest(), complete)

    def finalize(self) -> EdgeStoreManifest:
        if self._closed:
            raise ValueError("writer is closed")
        self._drain()
        failed = self._hasher.error or self._filer.error
        if failed is not None:
            self._manifest(False).save(self.manifest_path)
            raise failed
        if self._written != self.expected_bytes:
            self._manifest(False).save(self.manifest_path)
            raise DataError(f"payload length mismatch: {self._written} bytes written, "
                            f"expected {self.expected_bytes}; store marked incomplete")
        manifest = self._manifest(True)
        manifest.save(self.manifest_path)
        return manifest

    def abort(self) -> None:
        if self._closed:
            return
        self._drain()
        self._manifest(False).save(self.manifest_path)

    def __enter__(self):
        return self

    def __exit__(self, exc_type, exc, tb) -> None:
        if not self._closed:
            if exc_type is None:
                self.finalize()
            else:
                self.abort()


# ---------------------------------------------------------------------------------------------
# .words files (corpus.py:286-317)
# ---------------------------------------------------------------------------------------------

def save_words(path, words: Sequence) -> None:
    """``word<TAB>ipa<TAB>length<TAB>repr(frequency)<TAB>id,id,...`` per word (corpus.py:286-291)."""
    with open(path, "w", encoding="utf-8") as fh:
        for i in range(0, len(words), 4096):
            fh.write("".join(
                f"{w.word}\t{w.ipa}\t{len(w.phonemes)}\t{w.frequency!r}\t{','.join(map(str, w.phonemes))}\n"
                for w in words[i:i + 4096]))


def load_words(path) -> List[EncodedWord]:
    """Read a ``.words`` file back (corpus.py:294-317): same records, same ``DataError`` messages."""
    words: List[EncodedWord] = []
    with open(path, encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, start=1):
            line = raw[:-1] if raw.endswith("\n") else raw
            if not line:
                continue
            fields = line.split("\t")
            if len(fields) != 5:
                raise DataError(f"{path}: line {lineno}: expected 5 fields")
            try:
                declared = int(fields[2])
                freq = float(fields[3])
                ids = tuple(map(int, fields[4].split(","))) if fields[4] else ()
            except ValueError:
                raise DataError(f"{path}: line {lineno}: malformed numeric field") from None
            if not ids or declared != len(ids):
                raise DataError(f"{path}: line {lineno}: length does not match ID list")
            words.append(EncodedWord(fields[0], fields[1], ids, freq))
    if not words:
        raise DataError(f"{path}: word file is empty")
    return words


def words_to_store(words: Sequence) -> Tuple[np.ndarray, np.ndarray]:
    """The uint8 word store (ids (n, q), lengths (n,)) of a word list: engine.pack_words."""
    from .engine import pack_words
    return pack_words(words)


# ---------------------------------------------------------------------------------------------
# inventory sidecar (corpus.py:91-118) and scheme files (aligner.py:195-239): what `compute --scheme FILE` reads
# ---------------------------------------------------------------------------------------------

def load_inventory(path) -> dict:
    """``token<TAB>id`` per line, ids dense 0..K-1 (corpus.py:97-118).  Returns {token: id}."""
    by_id = {}
    with open(path, encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, start=1):
            line = raw.rstrip("\n")
            if not line:
                continue
            fields = line.split("\t")
            if len(fields) != 2:
                raise DataError(f"{path}: line {lineno}: expected 'token<TAB>id'")
            try:
                ident = int(fields[1])
            except ValueError:
                raise DataError(f"{path}: line {lineno}: bad id {fields[1]!r}") from None
            if ident in by_id:
                raise DataError(f"{path}: line {lineno}: duplicate id {ident}")
            by_id[ident] = fields[0]
    if not by_id:
        raise DataError(f"{path}: inventory file is empty")
    if sorted(by_id) != list(range(len(by_id))):
        raise DataError(f"{path}: ids are not dense 0..{len(by_id) - 1}")
    id_of = {tok: i for i, tok in by_id.items()}
    if len(id_of) != len(by_id):
        raise DataError("inventory contains duplicate phoneme tokens")
    return id_of


def load_scheme_file(path, id_of=None):
    """A scheme file (aligner.py:195-239): tab-separated ``match|mismatch|gap <TAB> int`` declarations (all three
    required) and ``tokenA <TAB> tokenB <TAB> int`` symmetric per-pair overrides, which need an inventory
    (``id_of``: {token: id}) to resolve; blank lines and ``#`` comments are skipped.  Same ``DataError``
    messages as the reference."""
    from .host_types import ScoringScheme

    core, overrides = {}, {}
    with open(path, encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, start=1):
            line = raw.strip()
            if not line or line[0] == "#":
                continue
            fields = line.split("\t")
            where = f"{path}: line {lineno}"
            if len(fields) == 2:
                key, text = fields
                if key not in ("match", "mismatch", "gap"):
                    raise DataError(f"{where}: unknown key {key!r}")
                try:
                    core[key] = int(text)
                except ValueError:
                    raise DataError(f"{where}: {key} must be an integer") from None
            elif len(fields) == 3:
                if id_of is None:
                    raise DataError(f"{where}: per-pair overrides require an inventory")
                try:
                    value = int(fields[2])
                except ValueError:
                    raise DataError(f"{where}: override must be an integer") from None
                for tok in fields[:2]:
                    if tok not in id_of:
                        raise DataError(f"{where}: unknown phoneme {tok!r}")
                a, b = id_of[fields[0]], id_of[fields[1]]
                overrides[(a, b)] = value
                overrides[(b, a)] = value
            else:
                raise DataError(f"{where}: expected 2 or 3 tab-separated fields")
    for key in ("match", "mismatch", "gap"):
        if key not in core:
            raise DataError(f"{path}: missing required key {key!r}")
    return ScoringScheme(core["match"], core["mismatch"], core["gap"], overrides)

