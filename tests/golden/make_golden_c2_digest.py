#!/usr/bin/env python
"""configs[1] (20,000 French-shaped words, scheme 1/-1/-2) through the UNMODIFIED reference engine
(`phonsim.engine.compute_all_pairs`, fork pool on all host cores): blake2b of the full 199,990,000-byte payload and
the ComputeStats.  Build container only (~1 min on 8 cores):  python tests/golden/make_golden_c2_digest.py"""
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


class DigestSink:
    def __init__(self):
        self.h = hashlib.blake2b(digest_size=16)
        self.n = 0

    def write(self, data):
        self.h.update(data)
        self.n += len(data)

    def abort(self):
        raise RuntimeError("abort")


ids, lens, sch = synth.config_store("C2")
words = [EncodedWord(f"w{i}", f"ipa{i}", tuple(int(x) for x in ids[i, : lens[i]]), float(len(lens) - i)) for i in range(len(lens))]
scheme = ScoringScheme(*sch)
sink = DigestSink()
t0 = time.time()
stats = compute_all_pairs(words, scheme, sink, ComputePlan(n=len(words), worker_count=len(os.sched_getaffinity(0)), scheme=scheme))
out = {"config": "C2", "words": len(words), "scheme": list(sch), "store_digest": synth.store_digest(ids, lens),
       "edges": stats.edges_written, "min": stats.min_score, "max": stats.max_score, "mean": stats.mean_score,
       "payload_blake2b_128": sink.h.hexdigest(), "reference_seconds": round(time.time() - t0, 1)}
(HERE / "c2_reference_digest.json").write_text(json.dumps(out, indent=1))
print(out)
