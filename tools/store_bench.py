"""Throughput of the edge-store sink: PipelinedEdgeStoreWriter vs the reference's EdgeStoreWriter
(when /root/reference is present: build container only) on the same payload, 65,536-byte writes."""
import sys, time, tempfile, os
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2509_01654_b200 as nw
from paper_2509_01654_b200 import store

n = int(sys.argv[1]) if len(sys.argv) > 1 else 46000          # 1,057,977,000 edges ~ 1 GB
P = nw.num_edges(n)
words = [nw.EncodedWord(f"w{i}", f"i{i}", (1,), 1.0) for i in range(n)]
data = np.random.default_rng(1).integers(-40, 6, size=P, dtype=np.int8)
view = memoryview(data).cast("B")
tmp = tempfile.mkdtemp(dir=os.environ.get("TMPDIR", "/tmp"))

def run(make):
    w = make()
    t0 = time.perf_counter()
    for s in range(0, P, 65536):
        w.write(view[s:s + 65536])
    m = w.finalize()
    dt = time.perf_counter() - t0
    return P / dt / 1e9, m.payload_digest

gbs, dig = run(lambda: store.PipelinedEdgeStoreWriter(f"{tmp}/ours", words, nw.ScoringScheme()))
print(f"PipelinedEdgeStoreWriter: {gbs:.2f} GB/s  digest {dig}")
if os.path.isdir("/root/reference/pkg/src"):
    sys.dont_write_bytecode = True
    sys.path.insert(0, "/root/reference/pkg/src")
    from phonsim.store import EdgeStoreWriter
    from phonsim.aligner import ScoringScheme
    from phonsim.corpus import EncodedWord
    rwords = [EncodedWord(w.word, w.ipa, w.phonemes, w.frequency) for w in words]
    gbs2, dig2 = run(lambda: EdgeStoreWriter(f"{tmp}/ref", rwords, ScoringScheme()))
    print(f"reference EdgeStoreWriter: {gbs2:.2f} GB/s  digest {dig2}  (same digest: {dig == dig2})")
    print("payload files identical:", open(f"{tmp}/ours.nwedges", "rb").read() == open(f"{tmp}/ref.nwedges", "rb").read())
for f in os.listdir(tmp):
    os.remove(os.path.join(tmp, f))
os.rmdir(tmp)
