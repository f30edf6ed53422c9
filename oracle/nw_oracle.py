"""CPU ORACLE (test infrastructure, NOT product code).

numpy / ctypes face of the oracle.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product package never does.

Parity status: PINNED against golden vectors produced by the unmodified Python
reference (``tests/golden/make_golden.py``) -- see ``tests/test_oracle.py``.

Two restatements live here:

* ``C`` -- ``oracle/nw_oracle.c`` loaded through ctypes (scalar DP per pair,
  optional pthread pool).  Fast enough to check 2e8 pairs.
* ``np_*`` -- a numpy restatement of the reference's *batched* algorithm
  (``engine.py:120-173``: whole batch swept one score-matrix row at a time),
  kept so the "port" CPU baseline has the same algorithmic shape as the
  reference's own numpy engine.

Reference anchors are given per function (paths under
``/root/reference/pkg/src/phonsim/``).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "libnw_oracle.so"
_lib = None


def build(force: bool = False) -> Path:
    """Compile oracle/nw_oracle.c with gcc (seconds)."""
    src = _HERE / "nw_oracle.c"
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        _LIB_PATH.parent.mkdir(exist_ok=True)
        subprocess.check_call(
            ["gcc", "-O3", "-march=native", "-fPIC", "-shared", "-pthread",
             "-o", str(_LIB_PATH), str(src), "-lm"]
        )
    return _LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB_PATH))
        i64, i32, p = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        L.orc_num_edges.restype = i64
        L.orc_num_edges.argtypes = [i64]
        L.orc_edges_before_row.restype = i64
        L.orc_edges_before_row.argtypes = [i64, i64]
        L.orc_row_of.restype = i64
        L.orc_row_of.argtypes = [i64, i64]
        L.orc_col_of.restype = i64
        L.orc_col_of.argtypes = [i64, i64, i64]
        L.orc_rows_cols.restype = None
        L.orc_rows_cols.argtypes = [p, i64, i64, p, p]
        L.orc_nw_score.restype = i32
        L.orc_nw_score.argtypes = [p, i32, p, i32, p, i32, i32]
        L.orc_score_range.restype = i32
        L.orc_score_range.argtypes = [p, p, i64, i32, p, i32, i32, i64, i64, p, p, p, p]
        L.orc_score_range_mt.restype = i32
        L.orc_score_range_mt.argtypes = [p, p, i64, i32, p, i32, i32, i64, i64, i64, i32, p, p, p, p]
        L.orc_preflight.restype = i32
        L.orc_preflight.argtypes = [p, i64, i32, i32, i32, p, p]
        L.orc_cells_in_range.restype = i64
        L.orc_cells_in_range.argtypes = [p, i64, i64, i64]
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# --------------------------------------------------------------------------- inputs

def pack_words(phoneme_seqs, q: int | None = None):
    """engine.py:99-107: zero-padded (n, q) int32 id matrix + (n,) int32 lengths."""
    n = len(phoneme_seqs)
    lengths = np.fromiter((len(s) for s in phoneme_seqs), dtype=np.int32, count=n)
    if q is None:
        q = int(lengths.max())
    ids = np.zeros((n, q), dtype=np.int32)
    for i, s in enumerate(phoneme_seqs):
        ids[i, : len(s)] = s
    return ids, lengths


def similarity_matrix(match: int, mismatch: int, size: int, overrides=None) -> np.ndarray:
    """engine.py:110-117: dense symmetric (size, size) int32 similarity table."""
    sim = np.full((size, size), mismatch, dtype=np.int32)
    sim[np.arange(size), np.arange(size)] = match
    for (a, b), v in (overrides or {}).items():
        if a < size and b < size:
            sim[a, b] = v
            sim[b, a] = v
    return sim


# --------------------------------------------------------------------------- triangle

def num_edges(n: int) -> int:
    """triangle.py:36-40."""
    return n * (n - 1) // 2


def edges_before_row(r, n):
    """triangle.py:43-46."""
    return r * (2 * n - r - 1) // 2


def np_rows_of(idx: np.ndarray, n: int) -> np.ndarray:
    """triangle.py:93-106 restated: fp64 closed form, then +-1 steps until the
    exact int64 bracket before(r) <= idx < before(r) + (n-1-r) holds."""
    idx = np.asarray(idx, dtype=np.int64)
    z = n - 0.5
    r = np.floor(z - np.sqrt(z * z - 2.0 * idx.astype(np.float64))).astype(np.int64)
    r = np.minimum(np.maximum(r, 0), n - 2)
    while True:
        lo = edges_before_row(r, n)
        down = idx < lo
        up = idx >= lo + (n - 1 - r)
        if not (down.any() or up.any()):
            return r
        r = r - down + up


def np_cols_of(idx: np.ndarray, n: int, rows: np.ndarray) -> np.ndarray:
    """triangle.py:109-112."""
    return rows + 1 + (np.asarray(idx, dtype=np.int64) - edges_before_row(rows, n))


def c_rows_cols(idx: np.ndarray, n: int):
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    rows = np.empty_like(idx)
    cols = np.empty_like(idx)
    lib().orc_rows_cols(_ptr(idx), idx.size, n, _ptr(rows), _ptr(cols))
    return rows, cols


# --------------------------------------------------------------------------- scoring (C)

def c_nw_score(a, b, sim: np.ndarray, gap: int) -> int:
    """aligner.py:106-117 via the C restatement."""
    a = np.ascontiguousarray(a, dtype=np.int32)
    b = np.ascontiguousarray(b, dtype=np.int32)
    sim = np.ascontiguousarray(sim, dtype=np.int32)
    return int(lib().orc_nw_score(_ptr(a), a.size, _ptr(b), b.size, _ptr(sim), sim.shape[0], gap))


def c_score_range(ids, lengths, sim, gap, n, start, end, threads: int = 1, chunk: int = 65536):
    """engine.py:176-195 (+ :262-276 when threads > 1).
    Returns (payload int8 ndarray, sum, min, max)."""
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    lengths = np.ascontiguousarray(lengths, dtype=np.int32)
    sim = np.ascontiguousarray(sim, dtype=np.int32)
    out = np.empty(end - start, dtype=np.int8)
    s = ctypes.c_int64()
    mn = ctypes.c_int32()
    mx = ctypes.c_int32()
    if threads <= 1:
        rc = lib().orc_score_range(_ptr(ids), _ptr(lengths), n, ids.shape[1], _ptr(sim),
                                   sim.shape[0], gap, start, end, _ptr(out),
                                   ctypes.addressof(s), ctypes.addressof(mn), ctypes.addressof(mx))
    else:
        rc = lib().orc_score_range_mt(_ptr(ids), _ptr(lengths), n, ids.shape[1], _ptr(sim),
                                      sim.shape[0], gap, start, end, chunk, threads, _ptr(out),
                                      ctypes.addressof(s), ctypes.addressof(mn), ctypes.addressof(mx))
    if rc != 0:
        raise RuntimeError(f"oracle failed rc={rc}")
    return out, s.value, mn.value, mx.value


def c_all_pairs(ids, lengths, sim, gap, threads: int | None = None):
    """engine.py:218-290 minus the sink: whole payload + (sum, min, max)."""
    n = len(lengths)
    if threads is None:
        threads = len(os.sched_getaffinity(0))
    return c_score_range(ids, lengths, sim, gap, n, 0, num_edges(n), threads=threads)


def cells_in_range(lengths, n, start, end) -> int:
    lengths = np.ascontiguousarray(lengths, dtype=np.int32)
    return int(lib().orc_cells_in_range(_ptr(lengths), n, start, end))


def total_cells(lengths) -> int:
    """sum over r<c of len_r*len_c = ((sum len)^2 - sum len^2) / 2."""
    L = [int(x) for x in np.asarray(lengths).tolist()]
    s1 = sum(L)
    s2 = sum(x * x for x in L)
    return (s1 * s1 - s2) // 2


def preflight(lengths, gap: int, min_sim: int, max_sim: int):
    """engine.py:72-96 -> (q or 0, lo, hi)."""
    lengths = np.ascontiguousarray(lengths, dtype=np.int32)
    lo = ctypes.c_int64()
    hi = ctypes.c_int64()
    q = lib().orc_preflight(_ptr(lengths), lengths.size, gap, min_sim, max_sim,
                            ctypes.addressof(lo), ctypes.addressof(hi))
    return q, lo.value, hi.value


# --------------------------------------------------------------------------- scoring (numpy)

def np_nw_batch(a_ids, a_len, b_ids, b_len, sim, gap) -> np.ndarray:
    """engine.py:120-173 restated.  One pass per score-matrix row over the whole
    batch, int16 cells; the score of pair p is read at (a_len[p], b_len[p])
    the moment row a_len[p] is finished.  Layout here is (pair, column)."""
    a_ids = np.asarray(a_ids)
    b_ids = np.asarray(b_ids)
    P = a_ids.shape[0]
    qa = int(a_len.max())
    qb = int(b_len.max())
    sim16 = np.asarray(sim, dtype=np.int16)
    g = np.int16(gap)
    above = np.tile(np.arange(qb + 1, dtype=np.int16) * g, (P, 1))
    here = np.empty_like(above)
    scores = np.zeros(P, dtype=np.int32)
    bsub = b_ids[:, :qb]
    pair_index = np.arange(P)
    for i in range(1, qa + 1):
        subst = sim16[a_ids[:, i - 1][:, None], bsub]          # (P, qb)
        best = np.maximum(above[:, :-1] + subst, above[:, 1:] + g)
        here[:, 0] = np.int16(i * gap)
        for j in range(1, qb + 1):
            np.maximum(best[:, j - 1], here[:, j - 1] + g, out=here[:, j])
        done = a_len == i
        if done.any():
            scores[done] = here[pair_index[done], b_len[done]]
        above, here = here, above
    return scores


def np_score_range(ids, lengths, sim, gap, n, start, end):
    """engine.py:176-195 restated on top of np_nw_batch."""
    idx = np.arange(start, end, dtype=np.int64)
    rows = np_rows_of(idx, n)
    cols = np_cols_of(idx, n, rows)
    sc = np_nw_batch(ids[rows], lengths[rows], ids[cols], lengths[cols], sim, gap)
    return sc.astype(np.int8), int(sc.sum(dtype=np.int64)), int(sc.min()), int(sc.max())


_NP_STATE = None


def _np_pool_init(state):
    global _NP_STATE
    _NP_STATE = state


def _np_pool_task(bounds):
    ids, lengths, sim, gap, n = _NP_STATE
    payload, s, mn, mx = np_score_range(ids, lengths, sim, gap, n, bounds[0], bounds[1])
    return payload.tobytes(), s, mn, mx


def np_score_ranges_pool(ids, lengths, sim, gap, n, ranges, workers: int):
    """engine.py:262-276 restated: a fork pool over contiguous chunks, results
    consumed in submission order.  Returns list of (bytes, sum, min, max)."""
    import multiprocessing as mp

    ctx = mp.get_context("fork")
    with ctx.Pool(workers, initializer=_np_pool_init,
                  initargs=((ids, lengths, sim, gap, n),)) as pool:
        return list(pool.imap(_np_pool_task, ranges, chunksize=1))


# --------------------------------------------------------------------------- new-surface oracles

def np_compact(payload: np.ndarray, start: int, n: int, threshold: int):
    """Threshold compaction + degree counts over a dense payload slice.
    Semantic model: the keep-mask and symmetric adjacency of graph.py:97-101,
    with the raw score as the weight.  Returns (idx int64, score int8, degree int64[n])."""
    payload = np.asarray(payload, dtype=np.int8)
    keep = np.flatnonzero(payload >= threshold)
    idx = keep.astype(np.int64) + start
    rows = np_rows_of(idx, n) if idx.size else np.zeros(0, dtype=np.int64)
    cols = np_cols_of(idx, n, rows) if idx.size else np.zeros(0, dtype=np.int64)
    degree = np.bincount(rows, minlength=n) + np.bincount(cols, minlength=n)
    return idx, payload[keep], degree.astype(np.int64)


def np_filter_normalized(payload: np.ndarray, start: int, n: int, lengths, lo: float, hi: float):
    """graph.py:91-101 restated: keep edges with lo <= 100.0*score/max(len_r,len_c) <= hi in float64.
    Returns (idx int64, score int8, degree int64[n])."""
    payload = np.asarray(payload, dtype=np.int8)
    L = np.asarray(lengths, dtype=np.int64)
    idx_all = np.arange(start, start + payload.size, dtype=np.int64)
    rows = np_rows_of(idx_all, n)
    cols = np_cols_of(idx_all, n, rows)
    w = (100.0 * payload) / np.maximum(L[rows], L[cols])
    keep = (w >= lo) & (w <= hi)
    degree = np.bincount(rows[keep], minlength=n) + np.bincount(cols[keep], minlength=n)
    return idx_all[keep], payload[keep], degree.astype(np.int64)


def np_hist_normalized(payload: np.ndarray, start: int, n: int, lengths) -> np.ndarray:
    """store.py:352-366 (normalized=True): 25501 bins, bin b counts floor(100*s/max_len) == b-12800."""
    payload = np.asarray(payload, dtype=np.int8)
    L = np.asarray(lengths, dtype=np.int64)
    idx_all = np.arange(start, start + payload.size, dtype=np.int64)
    rows = np_rows_of(idx_all, n)
    cols = np_cols_of(idx_all, n, rows)
    values = np.floor_divide(100 * payload.astype(np.int64), np.maximum(L[rows], L[cols]))
    return np.bincount(values + 12800, minlength=25501).astype(np.int64)


def np_histogram(payload: np.ndarray) -> np.ndarray:
    """store.py:352-366 (raw mode): 256 bins, bin k counts score k-128."""
    return np.bincount(np.asarray(payload, dtype=np.int8).astype(np.int64) + 128,
                       minlength=256).astype(np.int64)


def np_equal_work_bounds(lengths, parts: int) -> np.ndarray:
    """split [0, P) into `parts` contiguous ranges of (near) equal
    DP cells.  bound g = the smallest linear index whose exclusive prefix work
    is >= ceil(g * W / parts).  Brute-force friendly restatement (O(n log n))."""
    L = np.asarray(lengths, dtype=np.int64)
    n = L.size
    pref = np.concatenate([[0], np.cumsum(L)])           # pref[c] = sum_{k<c} len_k
    total_len = int(pref[-1])
    roww = L * (total_len - pref[1:])                      # len_r * sum_{c>r} len_c
    rowpref = np.concatenate([[0], np.cumsum(roww)])      # work before row r
    W = int(rowpref[-1])
    bounds = [0]
    for g in range(1, parts):
        target = -((-g * W) // parts)
        # first row whose end-of-row prefix reaches the target
        r = int(np.searchsorted(rowpref[1:], target, side="left"))
        r = min(r, n - 2)
        need = target - int(rowpref[r])
        if need <= 0:
            c = r + 1
        else:
            # smallest c in (r, n] with len_r * (pref[c] - pref[r+1]) >= need
            lr = int(L[r])
            k = -((-need) // lr)
            c = int(np.searchsorted(pref, int(pref[r + 1]) + k, side="left"))
        idx = edges_before_row(r, n) + (c - r - 1)
        bounds.append(int(min(max(idx, bounds[-1]), num_edges(n))))
    bounds.append(num_edges(n))
    return np.asarray(bounds, dtype=np.int64)
