"""N>1 host path: the product's rank-level driver (sharding.run_shard) under a real two-process
torch.distributed group.

* CPU (gloo, runs everywhere): the driver's bounds / accumulation / all-reduce / all-gather logic with a
  stand-in context whose "GPU" is the oracle (the checker plays the device; everything under test is product
  code);
* GPU (``-m gpu``): two processes SHARE cuda:0 over gloo and drive the real CUDA path -- dense configs[2] shards
  pinned to the reference's own per-shard payload digests and ComputeStats, and the sparse-output leg
  (threshold compaction + degree all-reduce + kept-count all-gather).
"""
import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


class OracleContext:
    """Duck-typed NwapContext for the CPU test: same methods run_shard calls, scores from oracle/nw_oracle.c."""

    def __init__(self, ids, lens, scheme):
        import torch
        from oracle import nw_oracle as orc
        self.orc, self.torch = orc, torch
        self.ids32, self.len32 = ids.astype(np.int32), lens.astype(np.int32)
        self.lens = lens
        self.n = len(lens)
        self.gap = scheme[2]
        self.sim = orc.similarity_matrix(scheme[0], scheme[1], int(ids.max()) + 1)
        self.device = 0
        self.torch_device = torch.device("cpu")

    def equal_work_bounds(self, parts):
        from paper_2509_01654_b200 import sharding
        return sharding.equal_work_bounds(self.lens, parts)

    def score_range(self, a, b, out, variant="auto", **_):
        payload, s, mn, mx = self.orc.c_score_range(self.ids32, self.len32, self.sim, self.gap, self.n, a, b)
        out[: b - a] = self.torch.from_numpy(payload)
        return s, mn, mx, b - a, None

    def payload_stats(self, out, count):
        p = out[:count].numpy()
        return int(p.astype(np.int64).sum()), int(p.min()), int(p.max()), count, self.orc.np_histogram(p)

    def compact_range(self, out, a, b, thr, capacity, degree=None):
        idx, sc, deg = self.orc.np_compact(out[: b - a].numpy(), a, self.n, thr)
        if degree is not None:
            degree += self.torch.from_numpy(deg.astype(np.int32))
        return self.torch.from_numpy(idx), self.torch.from_numpy(sc)

    def score_range_compact(self, a, b, threshold=None, normalized=None, capacity=0, degree=None, variant="auto"):
        buf = self.torch.empty(b - a, dtype=self.torch.int8)
        st = self.score_range(a, b, buf)
        idx, sc = self.compact_range(buf, a, b, threshold, capacity, degree)
        return idx, sc, st[:4]


def _cpu_worker(rank, world, port, tmp):
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist
    from paper_2509_01654_b200 import sharding, synth

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ids, lens, sch = synth.config_store("C1")
        ctx = OracleContext(ids, lens, sch)
        dense = sharding.run_shard(ctx, rank, world, threshold=2, want_hist=True)
        sparse = sharding.run_shard(ctx, rank, world, threshold=2, dense=False)
        two = sharding.run_shard(ctx, rank, world, threshold=2, passes=2)
        assert sparse.kept_counts == dense.kept_counts == two.kept_counts and sparse.kept_offset == dense.kept_offset
        assert np.array_equal(sparse.kept_idx.numpy(), dense.kept_idx.numpy())
        assert np.array_equal(two.kept_idx.numpy(), dense.kept_idx.numpy()) and two.payload is None
        assert np.array_equal(sparse.total.degree, dense.total.degree) and np.array_equal(two.total.degree, dense.total.degree)
        assert (sparse.total.sum, sparse.total.count, sparse.total.min, sparse.total.max) == \
               (dense.total.sum, dense.total.count, dense.total.min, dense.total.max)
        np.save(Path(tmp) / f"shard{rank}.npy", dense.payload.numpy())
        np.save(Path(tmp) / f"kept{rank}.npy", dense.kept_idx.numpy())
        t = dense.total
        np.savez(Path(tmp) / f"total{rank}.npz", sum=t.sum, count=t.count, min=t.min, max=t.max, hist=t.hist,
                 degree=t.degree, counts=np.array(dense.kept_counts), offset=dense.kept_offset, bounds=dense.bounds)
    finally:
        dist.destroy_process_group()


def test_run_shard_two_ranks_cpu():
    import tempfile
    import torch.multiprocessing as mp
    from oracle import nw_oracle as orc
    from paper_2509_01654_b200 import synth
    from conftest import GOLDEN

    port = 29500 + (os.getpid() % 2000)
    with tempfile.TemporaryDirectory() as tmp:
        tmp_path = Path(tmp)
        mp.spawn(_cpu_worker, args=(2, port, tmp), nprocs=2, join=True)
        ref = np.load(GOLDEN / "c1.npz")["payload"]
        got = np.concatenate([np.load(tmp_path / "shard0.npy"), np.load(tmp_path / "shard1.npy")])
        assert np.array_equal(got, ref)                      # concatenation in rank order IS the payload
        ridx, _, rdeg = orc.np_compact(ref, 0, 1000, 2)
        kept = np.concatenate([np.load(tmp_path / "kept0.npy"), np.load(tmp_path / "kept1.npy")])
        assert np.array_equal(kept, ridx)                    # ... and the kept lists concatenate the same way
        for rank in (0, 1):                                  # every rank holds the same reduced result
            tot = np.load(tmp_path / f"total{rank}.npz")
            assert int(tot["sum"]) == int(ref.astype(np.int64).sum()) and int(tot["count"]) == ref.size
            assert (int(tot["min"]), int(tot["max"])) == (int(ref.min()), int(ref.max()))
            assert np.array_equal(tot["hist"], orc.np_histogram(ref))
            assert np.array_equal(tot["degree"], rdeg)
            assert int(tot["counts"].sum()) == ridx.size
            assert int(tot["offset"]) == (0 if rank == 0 else int(tot["counts"][0]))
        _, lens, _ = synth.config_store("C1")
        b = tot["bounds"]
        w0 = orc.cells_in_range(lens.astype(np.int32), 1000, 0, int(b[1]))
        assert abs(2 * w0 - synth.total_cells(lens)) <= 2 * 16 * 16


# ---------------------------------------------------------------------------------------------- GPU

def _gpu_worker(rank, world, port, tmp):
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist
    import paper_2509_01654_b200 as nw
    from paper_2509_01654_b200 import sharding, synth
    from paper_2509_01654_b200.engine import NwapContext

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gold = json.loads((ROOT / "tests" / "golden" / "c3_reference_digest.json").read_text())
        ids, lens, sch = synth.config_store("C3")
        with NwapContext(ids, lens, nw.ScoringScheme(*sch), device=0) as ctx:
            res = sharding.run_shard(ctx, rank, world, want_hist=True, collective_device="cpu")
            # this rank's shard, cut at the reference's 8 equal-work bounds, against the reference's digests
            b8 = gold["shard_bounds"]
            assert res.start == b8[4 * rank] and res.end == b8[4 * rank + 4]
            host = res.payload.cpu().numpy()
            digests = [hashlib.blake2b(host[b8[g] - res.start: b8[g + 1] - res.start].tobytes(), digest_size=16).hexdigest()
                       for g in range(4 * rank, 4 * rank + 4)]
            assert digests == gold["shard_blake2b_128"][4 * rank: 4 * rank + 4]
            t = res.total
            assert (t.count, t.min, t.max, t.sum / t.count) == (gold["edges"], gold["min"], gold["max"], gold["mean"])
            assert int(t.hist.sum()) == gold["edges"]
            del res, host
            torch.cuda.empty_cache()
            # sparse-output leg: kept edges + degree, reduced; against the dense route on the same rank
            thr = -1
            sp = sharding.run_shard(ctx, rank, world, threshold=thr, dense=False, capacity=4_000_000, collective_device="cpu")
            dn = sharding.run_shard(ctx, rank, world, threshold=thr, capacity=4_000_000, collective_device="cpu")
            assert torch.equal(sp.kept_idx, dn.kept_idx) and torch.equal(sp.kept_score, dn.kept_score)
            assert sp.kept_counts == dn.kept_counts and sum(sp.kept_counts) * 2 == int(sp.total.degree.sum())
            assert np.array_equal(sp.total.degree, dn.total.degree)
            assert (sp.total.sum, sp.total.count) == (t.sum, t.count)
            json.dump({"kept": sp.kept_counts, "offset": sp.kept_offset, "degree_sum": int(sp.total.degree.sum())},
                      open(Path(tmp) / f"r{rank}.json", "w"))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_run_shard_two_processes_share_gpu0(tmp_path):
    """Two ranks, one GPU, gloo: configs[2] shards byte-pinned to the reference's per-shard digests, reduced
    statistics equal to the reference's ComputeStats, sparse-output leg consistent across ranks."""
    import torch.multiprocessing as mp

    port = 31500 + (os.getpid() % 2000)
    mp.spawn(_gpu_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0 = json.load(open(tmp_path / "r0.json"))
    r1 = json.load(open(tmp_path / "r1.json"))
    assert r0["kept"] == r1["kept"] and r0["degree_sum"] == r1["degree_sum"] == 2 * sum(r0["kept"])
    assert r0["offset"] == 0 and r1["offset"] == r0["kept"][0]
