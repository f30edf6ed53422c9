#!/usr/bin/env python
"""configs[2] (100,000 French-shaped words, scheme 1/-1/-2, 4,999,950,000 pairs) through the UNMODIFIED reference
engine (`phonsim.engine.compute_all_pairs`, fork pool on all host cores): blake2b of the full payload, of each of
the 8 equal-work shards, and the ComputeStats.  Build container only (~20 min on 8 cores):
    python tests/golden/make_golden_c3_digest.py"""
import hashlib, json, os, sys, time
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from phonsim.aligner import ScoringScheme            # noqa: E402
from phonsim.corpus import EncodedWord               # noqa: E402
from phonsim.engine import ComputePlan, compute_all_pairs   # noqa: E402
from paper_2509_01654_b200 import synth              # noqa: E402
from paper_2509_01654_b200.sharding import equal_work_bounds   # noqa: E402

ids, lens, sch = synth.config_store("C3")
bounds = [int(b) for b in equal_work_bounds(lens, 8)]


class DigestSink:
    """whole-payload digest plus one digest per equal-work shard (the bytes an 8-GPU run writes per rank)"""

    def __init__(self):
        self.h = hashlib.blake2b(digest_size=16)
        self.parts = [hashlib.blake2b(digest_size=16) for _ in range(8)]
        self.n = 0

    def write(self, data):
        self.h.update(data)
        view = memoryview(data)
        pos, end = self.n, self.n + len(data)
        for g in range(8):
            lo, hi = max(pos, bounds[g]), min(end, bounds[g + 1])
            if lo < hi:
                self.parts[g].update(view[lo - pos: hi - pos])
        self.n = end

    def abort(self):
        raise RuntimeError("abort")


words = [EncodedWord(f"w{i}", f"ipa{i}", tuple(int(x) for x in ids[i, : lens[i]]), float(len(lens) - i)) for i in range(len(lens))]
scheme = ScoringScheme(*sch)
sink = DigestSink()
t0 = time.time()
stats = compute_all_pairs(words, scheme, sink, ComputePlan(n=len(words), worker_count=len(os.sched_getaffinity(0)), scheme=scheme))
out = {"config": "C3", "words": len(words), "scheme": list(sch), "store_digest": synth.store_digest(ids, lens),
       "edges": stats.edges_written, "min": stats.min_score, "max": stats.max_score, "mean": stats.mean_score,
       "payload_blake2b_128": sink.h.hexdigest(), "shard_bounds": bounds,
       "shard_blake2b_128": [h.hexdigest() for h in sink.parts], "reference_seconds": round(time.time() - t0, 1)}
(HERE / "c3_reference_digest.json").write_text(json.dumps(out, indent=1))
print(out)
