"""N>1 host path on CPU: two gloo ranks shard the edge range with the product's
equal-work bounds, each 'scores' its shard (the oracle stands in for the GPU here --
it is the checker, the product's sharding/reduction code is what is under test), and the
statistics all-reduce must reproduce the single-process totals."""
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def _worker(rank, world, port, tmp):
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist
    from oracle import nw_oracle as orc
    from paper_2509_01654_b200 import sharding, synth

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ids, lens, sch = synth.config_store("C1")
        n = len(lens)
        bounds = sharding.equal_work_bounds(lens, world)
        s, e = sharding.shard_of(bounds, rank)
        sim = orc.similarity_matrix(sch[0], sch[1], int(ids.max()) + 1)
        payload, ssum, smin, smax = orc.c_score_range(ids.astype(np.int32), lens.astype(np.int32), sim, sch[2], n, s, e)
        _, _, deg = orc.np_compact(payload, s, n, 2)
        local = sharding.ShardStats(ssum, e - s, smin, smax, orc.np_histogram(payload), deg)
        tot = sharding.reduce_stats(local)
        counts = sharding.gather_counts(int((payload >= 2).sum()))
        np.save(Path(tmp) / f"shard{rank}.npy", payload)
        if rank == 0:
            np.savez(Path(tmp) / "total.npz", sum=tot.sum, count=tot.count, min=tot.min, max=tot.max,
                     hist=tot.hist, degree=tot.degree, counts=np.array(counts), bounds=bounds)
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding_and_reduction(tmp_path):
    import torch.multiprocessing as mp
    from oracle import nw_oracle as orc
    from paper_2509_01654_b200 import synth
    from conftest import GOLDEN

    port = 29500 + (os.getpid() % 2000)
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    ref = np.load(GOLDEN / "c1.npz")["payload"]
    got = np.concatenate([np.load(tmp_path / "shard0.npy"), np.load(tmp_path / "shard1.npy")])
    assert np.array_equal(got, ref)                      # concatenation in rank order IS the payload
    tot = np.load(tmp_path / "total.npz")
    assert int(tot["sum"]) == int(ref.astype(np.int64).sum()) and int(tot["count"]) == ref.size
    assert (int(tot["min"]), int(tot["max"])) == (int(ref.min()), int(ref.max()))
    assert np.array_equal(tot["hist"], orc.np_histogram(ref))
    _, _, deg = orc.np_compact(ref, 0, 1000, 2)
    assert np.array_equal(tot["degree"], deg)
    assert int(tot["counts"].sum()) == int((ref >= 2).sum())
    _, lens, _ = synth.config_store("C1")
    b = tot["bounds"]
    w0 = orc.cells_in_range(lens.astype(np.int32), 1000, 0, int(b[1]))
    assert abs(2 * w0 - synth.total_cells(lens)) <= 2 * 16 * 16
