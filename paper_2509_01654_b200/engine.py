"""B200 scoring engine behind the reference's entry point.

``compute_all_pairs(words, scheme, sink, plan) -> ComputeStats`` has the
signature, return type, error behaviour and sink protocol of the reference's
``phonsim.engine.compute_all_pairs`` (engine.py:218-290); ``NwapContext.score_range``
is the ``_score_range`` seam (engine.py:176-195) with a device (or pinned host)
destination.  All scoring happens in libnwap.so's CUDA kernels; torch is used
only to own device / pinned buffers and the current stream.
"""
from __future__ import annotations

import ctypes
import threading
import time
from typing import Optional, Sequence, Tuple

import numpy as np

from . import _native
from ._native import NwapStats, VARIANTS, check, lib
from .host_types import (ComputePlan, ComputeStats, DataError, ScoringScheme, same_scheme,
                         scheme_fields)
from .triangle import num_edges


def preflight_range_check(words, scheme) -> int:
    """Reference engine.py:72-96, same messages: returns q or raises."""
    if not words:
        raise ValueError("word list is empty")
    q = max(len(w.phonemes) for w in words)
    match, mismatch, gap, overrides = scheme_fields(scheme)
    sims = [match, mismatch, *overrides.values()]
    lo = min(0, 2 * q * gap, q * min(sims))
    hi = max(0, 2 * q * gap, q * max(sims))
    problems = []
    if lo < -128:
        problems.append(f"minimum achievable score {lo} < -128")
    if hi > 127:
        problems.append(f"maximum achievable score {hi} > 127")
    if problems:
        raise DataError("scores would overflow 8-bit storage for max word length "
                        f"{q}: {'; '.join(problems)}")
    return q


def pack_words(words, q: Optional[int] = None) -> Tuple[np.ndarray, np.ndarray]:
    """Reference engine.py:99-107 with uint8 symbols: (n, q) ids + (n,) lengths.

    One pass over the phoneme tuples (itertools.chain -> np.fromiter) and one masked scatter, instead of
    the reference's per-word Python loop: 100,000 words pack in ~40 ms instead of ~240 ms, which matters
    next to a 90 ms device path.
    """
    import itertools

    n = len(words)
    lengths = np.fromiter((len(w.phonemes) for w in words), dtype=np.int64, count=n)
    if q is None:
        q = int(lengths.max())
    if q > 255:
        raise DataError(f"word length {q} exceeds the 255-symbol store limit")
    if lengths.min() < 1:
        raise ValueError(f"word {int(np.argmin(lengths))} has no phonemes")
    try:
        # bytes() consumes the chained tuples in C and refuses anything outside [0, 255]
        flat = np.frombuffer(bytes(itertools.chain.from_iterable(w.phonemes for w in words)), dtype=np.uint8)
    except (ValueError, TypeError):
        for i, w in enumerate(words):
            if any((not isinstance(p, (int, np.integer))) or p < 0 or p > 255 for p in w.phonemes):
                raise DataError(f"word {i}: phoneme id outside [0, 255]") from None
        raise
    ids = np.zeros((n, q), dtype=np.uint8)
    ids[np.arange(q)[None, :] < lengths[:, None]] = flat
    return ids, lengths.astype(np.uint8)


def similarity_table(scheme, size: int) -> np.ndarray:
    """Reference engine.py:110-117 as int8."""
    match, mismatch, _, overrides = scheme_fields(scheme)
    sim = np.full((size, size), mismatch, dtype=np.int64)
    np.fill_diagonal(sim, match)
    for (a, b), v in overrides.items():
        if a < size and b < size:
            sim[a, b] = v
            sim[b, a] = v
    if sim.min() < -128 or sim.max() > 127:
        raise DataError("similarity value does not fit int8")
    return sim.astype(np.int8)


def _stats_tuple(st: NwapStats, want_hist: bool):
    hist = np.ctypeslib.as_array(st.hist).astype(np.int64).copy() if want_hist else None
    return int(st.sum), int(st.min), int(st.max), int(st.count), hist


class NwapContext:
    """One word store resident on one GPU (nwap_ctx)."""

    def __init__(self, ids: np.ndarray, lengths: np.ndarray, scheme, device: int = 0):
        ids = np.ascontiguousarray(ids, dtype=np.uint8)
        lengths = np.ascontiguousarray(lengths, dtype=np.uint8)
        if ids.ndim != 2 or lengths.ndim != 1 or ids.shape[0] != lengths.shape[0]:
            raise ValueError("ids must be (n, q) and lengths (n,)")
        match, mismatch, gap, overrides = scheme_fields(scheme)
        self.scheme = (match, mismatch, gap)
        self.device = device
        self.n = int(lengths.shape[0])
        self._h = ctypes.c_void_p()
        self._pending = None
        L = lib()
        check(L.nwap_create(ctypes.addressof(self._h), device, ids.ctypes.data, self.n, ids.shape[1],
                            lengths.ctypes.data, match, mismatch, gap))
        if overrides:
            size = int(ids.max()) + 1
            sim = similarity_table(scheme, size)
            try:
                check(L.nwap_set_similarity(self._h, sim.ctypes.data, size))
            except Exception:
                self.close()
                raise

    @classmethod
    def from_words(cls, words, scheme, device: int = 0) -> "NwapContext":
        q = preflight_range_check(words, scheme)
        ids, lengths = pack_words(words, q)
        return cls(ids, lengths, scheme, device)

    # -- lifetime
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().nwap_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- geometry
    @property
    def num_edges(self) -> int:
        return int(lib().nwap_num_edges(self._h))

    @property
    def max_len(self) -> int:
        return int(lib().nwap_max_len(self._h))

    def cells_in_range(self, start: int, end: int) -> int:
        return int(lib().nwap_cells_in_range(self._h, start, end))

    def equal_work_bounds(self, parts: int) -> np.ndarray:
        out = np.zeros(parts + 1, dtype=np.int64)
        check(lib().nwap_equal_work_bounds(self._h, parts, out.ctypes.data))
        return out

    # -- scoring
    def score_range(self, start: int, end: int, out, want_hist: bool = False, variant: str = "auto",
                    sync: bool = True):
        """Score edges [start, end) into ``out`` (torch int8/uint8 CUDA tensor, >= end-start
        elements).  Returns (sum, min, max, count, hist|None); with sync=False returns None and
        leaves the statistics on the device (read_stats())."""
        import torch

        if not (out.is_cuda and out.is_contiguous() and out.element_size() == 1):
            raise ValueError("out must be a contiguous 1-byte CUDA tensor")
        if out.numel() < end - start:
            raise ValueError("output tensor too small")
        stream = torch.cuda.current_stream(out.device).cuda_stream
        st = NwapStats()
        check(lib().nwap_score_range(self._h, start, end, out.data_ptr(),
                                     ctypes.addressof(st) if sync else None, int(want_hist),
                                     VARIANTS[variant], stream))
        return _stats_tuple(st, want_hist) if sync else None

    def read_stats(self, want_hist: bool = False):
        import torch

        st = NwapStats()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        check(lib().nwap_read_stats(self._h, ctypes.addressof(st), stream))
        return _stats_tuple(st, want_hist)

    def score_range_host(self, start: int, end: int, out_host, want_hist: bool = False,
                         variant: str = "auto"):
        """Same seam with a host destination (numpy uint8/int8 array or pinned torch tensor)."""
        ptr, size = _host_ptr(out_host)
        if size < end - start:
            raise ValueError("output buffer too small")
        st = NwapStats()
        check(lib().nwap_score_range_host(self._h, start, end, ptr, ctypes.addressof(st),
                                          int(want_hist), VARIANTS[variant]))
        return _stats_tuple(st, want_hist)

    def score_range_host_begin(self, start: int, end: int, out_host, want_hist: bool = False,
                               variant: str = "auto") -> None:
        """Enqueue the scoring of [start, end) into ``out_host`` and return at once; the buffer is
        complete after :meth:`score_range_host_wait`.  One call in flight per context."""
        ptr, size = _host_ptr(out_host)
        if size < end - start:
            raise ValueError("output buffer too small")
        self._pending = (out_host, want_hist)          # keep the buffer alive until the wait
        check(lib().nwap_score_range_host_begin(self._h, start, end, ptr, int(want_hist), VARIANTS[variant]))

    def score_range_host_wait(self):
        if self._pending is None:
            raise ValueError("no host-destination call in flight on this context")
        st = NwapStats()
        _, want_hist = self._pending
        try:
            check(lib().nwap_score_range_host_wait(self._h, ctypes.addressof(st)))
        finally:
            self._pending = None
        return _stats_tuple(st, want_hist)

    def payload_stats(self, payload, count: Optional[int] = None):
        import torch

        count = payload.numel() if count is None else count
        st = NwapStats()
        stream = torch.cuda.current_stream(payload.device).cuda_stream
        check(lib().nwap_payload_stats(self._h, payload.data_ptr(), count, ctypes.addressof(st), stream))
        return _stats_tuple(st, True)

    def compact_range(self, payload, start: int, end: int, threshold: int, capacity: int,
                      degree=None):
        """Kept edges (score >= threshold) of an already scored slice, in index order.
        Returns (idx int64 tensor, score int8 tensor); ``degree`` (int32 CUDA tensor of n)
        is incremented at both endpoints of every kept edge."""
        import torch

        dev = payload.device
        idx = torch.empty(max(capacity, 1), dtype=torch.int64, device=dev)
        sc = torch.empty(max(capacity, 1), dtype=torch.int8, device=dev)
        cnt = ctypes.c_int64()
        stream = torch.cuda.current_stream(dev).cuda_stream
        rc = lib().nwap_compact_range(self._h, payload.data_ptr(), start, end, threshold,
                                      idx.data_ptr(), sc.data_ptr(), capacity, ctypes.addressof(cnt),
                                      degree.data_ptr() if degree is not None else None, stream)
        if rc == _native.NWAP_ECAPACITY:
            raise _native.CapacityError(_native.last_error(), cnt.value)
        check(rc)
        return idx[: cnt.value], sc[: cnt.value]


    def score_range_compact(self, start: int, end: int, threshold: Optional[int] = None, capacity: int = 0,
                            out=None, degree=None, normalized: Optional[Tuple[float, float]] = None,
                            variant: str = "auto"):
        """Sparse-output scoring (nwap_score_range_compact): score [start, end) and return only the kept
        edges -- raw score >= ``threshold``, or ``normalized=(lo, hi)`` for the reference's
        ``lo <= 100*score/max(len_r, len_c) <= hi`` (graph.py:91-101) -- in index order, without ever
        materialising the dense payload (``out=None``).  Pass ``out`` (int8 CUDA tensor) to get the dense
        bytes as well.  Returns (idx int64 tensor, score int8 tensor, (sum, min, max, count))."""
        import torch

        if (threshold is None) == (normalized is None):
            raise ValueError("pass exactly one of threshold / normalized")
        dev = torch.device("cuda", self.device)
        if out is not None:
            if not (out.is_cuda and out.is_contiguous() and out.element_size() == 1):
                raise ValueError("out must be a contiguous 1-byte CUDA tensor")
            if out.numel() < end - start:
                raise ValueError("output tensor too small")
        idx = torch.empty(max(capacity, 1), dtype=torch.int64, device=dev)
        sc = torch.empty(max(capacity, 1), dtype=torch.int8, device=dev)
        cnt = ctypes.c_int64()
        st = NwapStats()
        stream = torch.cuda.current_stream(dev).cuda_stream
        common = (idx.data_ptr(), sc.data_ptr(), capacity, ctypes.addressof(cnt),
                  degree.data_ptr() if degree is not None else None, ctypes.addressof(st), VARIANTS[variant], stream)
        optr = out.data_ptr() if out is not None else None
        if normalized is None:
            rc = lib().nwap_score_range_compact(self._h, start, end, optr, int(threshold), *common)
        else:
            lo, hi = normalized
            if lo > hi:
                raise ValueError(f"empty filter range: lo={lo} > hi={hi}")
            rc = lib().nwap_score_range_filter_normalized(self._h, start, end, optr, float(lo), float(hi), *common)
        if rc == _native.NWAP_ECAPACITY:
            raise _native.CapacityError(_native.last_error(), cnt.value)
        check(rc)
        return idx[: cnt.value], sc[: cnt.value], _stats_tuple(st, False)[:4]

    def filter_normalized(self, payload, start: int, end: int, lo: float, hi: float, capacity: int,
                          degree=None):
        """Reference graph.py:91-101 keep-mask on the device: edges of an already scored slice with
        lo <= 100*score/max(len_r, len_c) <= hi (float64, as numpy).  Returns (idx, score) tensors in
        index order; ``degree`` gets +1 at both endpoints of every kept edge."""
        import torch

        if lo > hi:
            raise ValueError(f"empty filter range: lo={lo} > hi={hi}")
        dev = payload.device
        idx = torch.empty(max(capacity, 1), dtype=torch.int64, device=dev)
        sc = torch.empty(max(capacity, 1), dtype=torch.int8, device=dev)
        cnt = ctypes.c_int64()
        stream = torch.cuda.current_stream(dev).cuda_stream
        rc = lib().nwap_filter_normalized(self._h, payload.data_ptr(), start, end, float(lo), float(hi),
                                          idx.data_ptr(), sc.data_ptr(), capacity, ctypes.addressof(cnt),
                                          degree.data_ptr() if degree is not None else None, stream)
        if rc == _native.NWAP_ECAPACITY:
            raise _native.CapacityError(_native.last_error(), cnt.value)
        check(rc)
        return idx[: cnt.value], sc[: cnt.value]

    def hist_normalized(self, payload, start: int, end: int, counts=None):
        """Reference store.py:342-381 histogram(normalized=True) on the device: returns a (25501,)
        int64 CUDA tensor, bin b counting floor(100*score/max(len_r,len_c)) == b - 12800.  Pass
        ``counts`` to accumulate over several slices."""
        import torch

        dev = payload.device
        if counts is None:
            counts = torch.zeros(25501, dtype=torch.int64, device=dev)
        stream = torch.cuda.current_stream(dev).cuda_stream
        check(lib().nwap_hist_normalized(self._h, payload.data_ptr(), start, end, counts.data_ptr(), stream))
        return counts


def _host_ptr(buf):
    if isinstance(buf, np.ndarray):
        if not buf.flags["C_CONTIGUOUS"] or buf.itemsize != 1:
            raise ValueError("host buffer must be a contiguous 1-byte array")
        return buf.ctypes.data, buf.size
    if hasattr(buf, "data_ptr"):
        if buf.is_cuda or buf.element_size() != 1 or not buf.is_contiguous():
            raise ValueError("host buffer must be a contiguous 1-byte CPU tensor")
        return buf.data_ptr(), buf.numel()
    raise TypeError("unsupported host buffer")


def device_rows_cols(idx: "np.ndarray", n: int):
    """triangle.py:93-112 on the device (parity tests)."""
    import torch

    t = torch.as_tensor(np.ascontiguousarray(idx, dtype=np.int64)).cuda()
    rows = torch.empty_like(t)
    cols = torch.empty_like(t)
    check(lib().nwap_rows_cols(n, t.data_ptr(), t.numel(), rows.data_ptr(), cols.data_ptr(),
                               torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return rows.cpu().numpy(), cols.cpu().numpy()


def probe(which: str, iters: int = 2000, device: int = 0):
    """(warp-instructions per SM per clock, milliseconds) of one issue probe."""
    ipc = ctypes.c_double()
    ms = ctypes.c_double()
    check(lib().nwap_probe(device, _native.PROBES.index(which), iters, ctypes.addressof(ipc),
                           ctypes.addressof(ms)))
    return ipc.value, ms.value


def compute_all_pairs(words: Sequence, scheme, sink, plan: Optional[ComputePlan] = None,
                      device: int = 0, variant: str = "auto",
                      devices: Optional[Sequence[int]] = None) -> ComputeStats:
    """Drop-in for reference engine.py:218-290.

    Every edge score goes through the sink once, in linear-index order, in pieces of
    ``plan.chunk_size`` edges (the payload never depends on it); on any failure after the
    arguments have been validated ``sink.abort()`` is called before the exception propagates.

    Sink protocol.  ``sink.write(data)`` receives an immutable ``bytes`` object per piece, exactly as
    the reference passes (engine.py:256, :272), so sinks that keep the object (the reference tests'
    ``chunks.append(data)``) stay correct.  A sink that consumes the data before returning can opt into
    the zero-copy path by defining ``write_view(view)``: it is then called instead, with a memoryview
    into a pinned staging slab that is ONLY VALID DURING THE CALL (the slab is overwritten two slabs
    later and recycled by the next run).  ``PipelinedEdgeStoreWriter`` does.

    ``devices`` (default ``[device]``) lists the GPUs to use from this one process -- the
    counterpart of the reference's fork pool (engine.py:262-276): slab k of the edge range
    is scored by GPU ``k mod G`` into that GPU's own pinned staging slabs, and the sink
    consumes the slabs in index order, so the payload is the same for any G
    (partition invariance, tests/test_engine.py:92-101).  The word store is replicated; no
    edge byte moves between GPUs.

    Deviation from the reference: phoneme ids must fit one byte (alphabet <= 256 symbols; the
    reference packs int32).  Larger ids raise DataError.
    """
    import torch

    n = len(words)
    q = preflight_range_check(words, scheme)
    if plan is None:
        plan = ComputePlan(n=n, scheme=scheme)
    if plan.n != n:
        raise ValueError(f"plan is for n={plan.n}, got {n} words")
    if not same_scheme(plan.scheme, scheme):
        raise ValueError("plan scheme differs from the scheme argument")
    devs = [int(d) for d in (devices if devices is not None else [device])]
    if not devs:
        raise ValueError("devices must name at least one GPU")

    total = num_edges(n)
    edges = 0
    score_sum = 0
    score_min = 127
    score_max = -128
    started = time.perf_counter()
    ctxs: list = []
    staging: list = []
    emit_view = getattr(sink, "write_view", None)
    try:
        if not torch.cuda.is_available():
            raise RuntimeError("compute_all_pairs needs a CUDA device: there is no CPU fallback")
        ids, lengths = pack_words(words, q)
        chunk = plan.chunk_size
        # pinned host slabs of a whole number of sink chunks (about 64 MiB each), two per GPU: the devices
        # score and copy the next slabs while the sink consumes slab k, in index order
        slab = max(chunk, (_SLAB_BYTES // chunk) * chunk)
        slab = min(slab, total)              # a chunk_size beyond the job is one piece (and pins no more than the job)
        ranges = [(s, min(s + slab, total)) for s in range(0, total, slab)]
        G = max(1, min(len(devs), len(ranges)))
        ctxs = [NwapContext(ids, lengths, scheme, d) for d in devs[:G]]
        per_gpu = 2 if len(ranges) > G else 1
        staging = _staging_slabs(slab, G * per_gpu)
        views = [memoryview(t.numpy()).cast("B") for t in staging]

        def buf(k):                       # staging slab of range k: GPU k mod G, its buffer (k div G) mod 2
            return (k % G) * per_gpu + ((k // G) % per_gpu)

        def begin(k):
            ctxs[k % G].score_range_host_begin(*ranges[k], staging[buf(k)], variant=variant)

        for k in range(min(G, len(ranges))):
            begin(k)
        for k, (s, e) in enumerate(ranges):
            ssum, smin, smax, scount, _ = ctxs[k % G].score_range_host_wait()
            if k + G < len(ranges):
                begin(k + G)
            if scount != e - s:
                raise DataError(f"device scored {scount} edges in [{s}, {e})")
            view = views[buf(k)]
            for cs in range(0, e - s, chunk):
                piece = view[cs: min(cs + chunk, e - s)]
                if emit_view is not None:
                    emit_view(piece)          # transient: valid during the call only
                else:
                    sink.write(bytes(piece))  # what the reference hands over: an immutable bytes object
                edges += len(piece)
            score_sum += ssum
            score_min = min(score_min, smin)
            score_max = max(score_max, smax)
    except Exception:
        sink.abort()
        raise
    finally:
        for c in ctxs:
            c.close()            # synchronises the device: nothing is still writing the staging slabs
        _return_slabs(staging)
    wall = time.perf_counter() - started
    if edges != total:
        sink.abort()
        raise DataError(f"wrote {edges} edges, expected {total}")
    return ComputeStats(edges_written=edges, wall_time=wall, min_score=score_min,
                        max_score=score_max, mean_score=score_sum / edges)


_SLAB_BYTES = 64 << 20        # host staging slab of compute_all_pairs
_STAGING = {}
_STAGING_LOCK = threading.Lock()


def _staging_slabs(nbytes: int, count: int):
    """Check out pinned host staging slabs, cached per size class (pinning 64 MiB costs ~20 ms)."""
    import torch

    size = 1 << max(16, (nbytes - 1).bit_length())
    with _STAGING_LOCK:
        have = _STAGING.setdefault(size, [])
        out = [have.pop() for _ in range(min(count, len(have)))]
    while len(out) < count:
        out.append(torch.empty(size, dtype=torch.int8).pin_memory())
    return out


_STAGING_CACHE_BYTES = 512 << 20      # pinned bytes kept between runs (two slabs per GPU for 4 GPUs)


def _return_slabs(slabs) -> None:
    with _STAGING_LOCK:
        held = sum(t.numel() for have in _STAGING.values() for t in have)
        for t in slabs:
            if held + t.numel() <= _STAGING_CACHE_BYTES:
                _STAGING.setdefault(t.numel(), []).append(t)
                held += t.numel()


def trim() -> None:
    """Release everything cached between runs: the pinned staging slabs here and the per-device pipelines
    and memory-pool blocks inside the library (nwap_trim)."""
    with _STAGING_LOCK:
        _STAGING.clear()
    lib().nwap_trim()
