#!/usr/bin/env python
"""Generate golden vectors by running the UNMODIFIED Python reference.

Run in the build container only (the reference does not travel to the GPU box):

    python tests/golden/make_golden.py

Imports ``phonsim`` read-only from /root/reference/pkg/src and writes small
fixtures next to this file.  Everything the oracle and the CUDA path are pinned
against comes from here or from literal values in the reference's own tests
(cited in tests/test_oracle.py).
"""
from __future__ import annotations

import hashlib
import json
import random
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from phonsim.aligner import ScoringScheme, nw_score  # noqa: E402
from phonsim.corpus import CorpusRow, EncodedWord, build_inventory, encode_word  # noqa: E402
from phonsim.engine import (ComputePlan, _pack_words, _score_range, _similarity_matrix,  # noqa: E402
                            compute_all_pairs, preflight_range_check)
from phonsim.triangle import cols_of_array, num_edges, rows_of_array  # noqa: E402

from paper_2509_01654_b200 import synth  # noqa: E402


class Collect:
    def __init__(self):
        self.parts = []

    def write(self, data):
        self.parts.append(bytes(data))

    def abort(self):
        pass


def ref_make_words(n, seed=0, alphabet=12, min_len=1, max_len=9):
    # literal restatement of the reference fixture (tests/conftest.py:13-24) used to
    # check that synth.make_words reproduces it
    rng = random.Random(seed)
    return [
        EncodedWord(f"w{i:04d}", f"ipa{i:04d}",
                    tuple(rng.randrange(alphabet) for _ in range(rng.randint(min_len, max_len))),
                    float(n - i))
        for i in range(n)
    ]


def to_ref_words(ids, lengths):
    return [EncodedWord(f"w{i}", f"i{i}", tuple(int(x) for x in ids[i, : lengths[i]]), 1.0)
            for i in range(len(lengths))]


def run_engine(words, scheme, chunk=4096, workers=1):
    sink = Collect()
    plan = ComputePlan(n=len(words), chunk_size=chunk, worker_count=workers, scheme=scheme)
    stats = compute_all_pairs(words, scheme, sink, plan)
    payload = np.frombuffer(b"".join(sink.parts), dtype=np.int8)
    return payload, stats


def main():
    out = {}

    # ---- known answers straight from the reference functions -----------------
    rows = [CorpusRow("puissance", "pɥisɑ̃s", 5.0), CorpusRow("nuance", "nɥɑ̃s", 4.0),
            CorpusRow("puisant", "pɥizɑ̃", 3.0), CorpusRow("paysans", "peizɑ̃", 2.0),
            CorpusRow("épuisant", "epɥizɑ̃", 1.0)]
    inv = build_inventory(rows)
    fw = {r.word: encode_word(r, inv) for r in rows}
    kat = {
        "french": {w: list(e.phonemes) for w, e in fw.items()},
        "puissance_nuance_1_-1_-2": nw_score(fw["puissance"], fw["nuance"], ScoringScheme(1, -1, -2)),
        "puisant_paysans_1_-1_-1": nw_score(fw["puisant"], fw["paysans"], ScoringScheme(1, -1, -1)),
        "puisant_epuisant_1_-1_-1": nw_score(fw["puisant"], fw["épuisant"], ScoringScheme(1, -1, -1)),
        "test_engine_pair": nw_score((0, 18, 16, 11, 26, 11), (29, 18, 26, 11), ScoringScheme(1, -1, -2)),
    }
    # random scalar pairs incl. gap >= 0 and mismatch > match
    rng = random.Random(20251017)
    scal = []
    for _ in range(400):
        a = [rng.randrange(6) for _ in range(rng.randint(1, 12))]
        b = [rng.randrange(6) for _ in range(rng.randint(1, 12))]
        m, x, g = rng.randint(-3, 4), rng.randint(-4, 4), rng.randint(-4, 3)
        scal.append({"a": a, "b": b, "scheme": [m, x, g], "score": nw_score(a, b, ScoringScheme(m, x, g))})
    kat["scalar_cases"] = scal
    (HERE / "kat.json").write_text(json.dumps(kat, ensure_ascii=False, indent=0))

    # ---- engine payloads on the reference tests' own word sets ---------------
    cases = [
        ("seed9", dict(n=30, seed=9, alphabet=8, min_len=1, max_len=9), (1, -1, -1), None),
        ("seed4", dict(n=40, seed=4, alphabet=10), (2, -1, -2), None),
        ("seed11", dict(n=25, seed=11), (1, -1, -1), None),
        ("seed30", dict(n=30, seed=30, alphabet=20, min_len=1, max_len=10), (1, -1, -1), None),
        ("seed500", dict(n=500, seed=500, alphabet=30, min_len=2, max_len=10), (1, -1, -1), None),
        ("gap0", dict(n=60, seed=77, alphabet=5, min_len=1, max_len=12), (2, -1, 0), None),
        ("gappos", dict(n=60, seed=78, alphabet=5, min_len=1, max_len=10), (1, -2, 1), None),
        ("mis_gt_match", dict(n=60, seed=79, alphabet=4, min_len=1, max_len=12), (-1, 2, -2), None),
        ("long40", dict(n=50, seed=80, alphabet=9, min_len=20, max_len=40), (1, -1, -1), None),
        ("override", dict(n=60, seed=81, alphabet=6, min_len=1, max_len=14), (1, -1, -2),
         {(1, 2): 1, (0, 5): -3, (3, 3): 4}),
    ]
    arrays = {}
    meta = {}
    for name, kw, sch, ov in cases:
        words = ref_make_words(**kw)
        mine = synth.make_words(**kw)
        assert [w.phonemes for w in words] == [w.phonemes for w in mine], "synth.make_words drifted"
        scheme = ScoringScheme(*sch, overrides=ov or {})
        payload, stats = run_engine(words, scheme, chunk=97)
        payload2, _ = run_engine(words, scheme, chunk=10 ** 6, workers=2)
        assert (payload == payload2).all()
        q = preflight_range_check(words, scheme)
        ids, lengths = _pack_words(words, q)
        arrays[f"{name}_ids"] = ids.astype(np.uint8)
        arrays[f"{name}_len"] = lengths.astype(np.uint8)
        arrays[f"{name}_payload"] = payload
        meta[name] = {"scheme": list(sch), "overrides": [[a, b, v] for (a, b), v in (ov or {}).items()],
                      "min": stats.min_score, "max": stats.max_score, "mean": stats.mean_score,
                      "edges": stats.edges_written,
                      "digest": hashlib.blake2b(payload.tobytes(), digest_size=8).hexdigest()}
    np.savez_compressed(HERE / "engine_cases.npz", **arrays)
    (HERE / "engine_cases.json").write_text(json.dumps(meta, indent=1))

    # ---- C1: the whole 1,000-word config through the reference engine --------
    ids, lengths, sch = synth.config_store("C1")
    words = to_ref_words(ids, lengths)
    scheme = ScoringScheme(*sch)
    payload, stats = run_engine(words, scheme, chunk=65536)
    np.savez_compressed(HERE / "c1.npz", payload=payload)
    c1 = {"n": len(words), "scheme": list(sch), "min": stats.min_score, "max": stats.max_score,
          "mean": stats.mean_score, "sum": int(payload.astype(np.int64).sum()),
          "digest": hashlib.blake2b(payload.tobytes(), digest_size=8).hexdigest(),
          "store_digest": synth.store_digest(ids, lengths)}

    # ---- sampled ranges of the big configs via the reference _score_range ----
    samples = {}
    sample_meta = {}
    for cfg, n_small in (("C2", 20_000), ("C3", 100_000), ("C4", 600_000), ("C5", 600_000)):
        ids, lengths, sch = synth.config_store(cfg)
        n = len(lengths)
        ids32 = ids.astype(np.int32)
        len32 = lengths.astype(np.int32)
        sim = _similarity_matrix(ScoringScheme(*sch), int(ids32.max()) + 1)
        P = num_edges(n)
        rng = np.random.default_rng(99 + n)
        starts = [0, P - 3000] + [int(x) for x in rng.integers(0, P - 3000, size=4)]
        # one range that crosses many short rows near the end of the triangle
        starts.append(P - 40_000)
        recs = []
        for k, s in enumerate(starts):
            e = min(P, s + (3000 if k != len(starts) - 1 else 40_000))
            pb, ssum, smin, smax = _score_range(ids32, len32, sim, sch[2], n, s, e)
            samples[f"{cfg}_{k}"] = np.frombuffer(pb, dtype=np.int8)
            recs.append({"start": s, "end": e, "sum": ssum, "min": smin, "max": smax})
        sample_meta[cfg] = {"n": n, "scheme": list(sch), "ranges": recs,
                            "store_digest": synth.store_digest(ids, lengths),
                            "q": int(lengths.max()), "total_cells": synth.total_cells(lengths)}
    np.savez_compressed(HERE / "sampled_ranges.npz", **samples)
    (HERE / "sampled_ranges.json").write_text(json.dumps({"C1": c1, **sample_meta}, indent=1))

    # ---- downstream consumers of the payload, run by the reference itself --
    import tempfile
    from phonsim.graph import filter_view
    from phonsim.store import EdgeStore, EdgeStoreWriter, histogram
    words = ref_make_words(n=500, seed=500, alphabet=30, min_len=2, max_len=10)
    scheme = ScoringScheme(1, -1, -1)
    with tempfile.TemporaryDirectory() as tmp:
        prefix = Path(tmp) / "g"
        writer = EdgeStoreWriter(prefix, words, scheme)
        compute_all_pairs(words, scheme, writer, ComputePlan(n=500, scheme=scheme))
        writer.finalize()
        store = EdgeStore(prefix)
        cons = {}
        for nm, normalized in (("raw", False), ("norm", True)):
            h = histogram(store, words, normalized=normalized)
            cons[f"hist_{nm}_first"] = np.array([h.min], dtype=np.int64)
            cons[f"hist_{nm}_counts"] = np.array(h.counts, dtype=np.int64)
        for k, (lo, hi) in enumerate([(20.0, 60.0), (-100.0, -50.5), (0.0, 0.0), (33.3, 1e9), (-1e9, 1e9)]):
            view = filter_view(store, words, lo, hi)
            edges = sorted((u, v) for u, adj in view.adjacency.items() for v, _ in adj if u < v)
            cons[f"filter{k}_bounds"] = np.array([lo, hi], dtype=np.float64)
            cons[f"filter{k}_count"] = np.array([len(edges)], dtype=np.int64)
            if len(edges) <= 30000:          # the all-pass window is pinned by count + degree only
                cons[f"filter{k}_edges"] = np.array(edges, dtype=np.int32).reshape(-1, 2)
            deg = np.zeros(500, dtype=np.int64)
            for u, adj in view.adjacency.items():
                deg[u] = len(adj)
            cons[f"filter{k}_degree"] = deg
        store.close()
    np.savez_compressed(HERE / "consumers_seed500.npz", **cons)

    # ---- triangle: reference rows/cols at large n ----------------------------
    tri = {}
    rng = np.random.default_rng(42)
    for n in (4, 300, 10 ** 5, 10 ** 6, 10 ** 7, 600_000):
        P = num_edges(n)
        if P <= 50_000:
            idx = np.arange(P, dtype=np.int64)
        else:
            idx = np.concatenate([rng.integers(0, P, size=3000, dtype=np.int64),
                                  np.array([0, 1, n - 2, n - 1, P - 1, P - 2, P // 2], dtype=np.int64)])
        r = rows_of_array(idx, n)
        c = cols_of_array(idx, n, r)
        tri[f"n{n}_idx"] = idx
        tri[f"n{n}_rows"] = r
        tri[f"n{n}_cols"] = c
    np.savez_compressed(HERE / "triangle.npz", **tri)
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
