"""The reference-shaped entry point end to end: compute_all_pairs(words, scheme, NullSink(), plan) on the 100,000-word
workload, as tests/test_acceptance.py:204-227 times the reference (EncodedWord list in, every chunk through
sink.write).  Prints the wall time, the share spent outside the device path, and GCUPS."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2509_01654_b200 as nw
from paper_2509_01654_b200 import synth, engine

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
ids, lens = synth.french_shaped(n)
words = synth.as_encoded_words(ids, lens)
scheme = nw.ScoringScheme(1, -1, -2)
cells = synth.total_cells(lens)

class NullSink:
    def __init__(self): self.n = 0; self.calls = 0
    def write(self, data): self.n += len(data); self.calls += 1
    def abort(self): pass

for rep in range(4):
    sink = NullSink()
    t0 = time.perf_counter()
    q = engine.preflight_range_check(words, scheme)
    t1 = time.perf_counter()
    engine.pack_words(words, q)
    t2 = time.perf_counter()
    stats = nw.compute_all_pairs(words, scheme, sink, nw.ComputePlan(n=n, scheme=scheme))
    t3 = time.perf_counter()
    print(f"rep {rep}: compute_all_pairs {1e3*(t3-t2):.1f} ms ({cells/(t3-t2)/1e9:.0f} GCUPS, {sink.calls} sink.write calls, "
          f"{sink.n} bytes); of which preflight ~{1e3*(t1-t0):.1f} ms, pack_words ~{1e3*(t2-t1):.1f} ms; mean {stats.mean_score:.4f}")
