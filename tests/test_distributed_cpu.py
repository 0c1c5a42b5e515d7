"""Host logic of the multi-GPU path, exercised with gloo on CPU (world size 2)."""
import os
import socket
import sys

import numpy as np
import pytest

from conftest import ROOT


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_queries, out_dir):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_2409_06807_b200 import _lib
    from paper_2409_06807_b200.batch import gather_records, shard_queries
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    idx = shard_queries(n_queries, rank, world)
    rec = np.zeros(len(idx), dtype=_lib.QUERY_RESULT_DTYPE)
    rec["status"] = 0
    rec["iterations"] = idx % 7          # stand-in for what each rank's GPU would report
    rec["tree_size"] = idx * 10
    full = gather_records(idx, rec, n_queries)
    if rank == 0:
        np.save(os.path.join(out_dir, "full.npy"), full)
    else:
        assert full is None
    dist.barrier()
    dist.destroy_process_group()


def test_shard_and_gather_world2(tmp_path):
    import torch.multiprocessing as mp
    n_queries, world = 37, 2
    mp.spawn(_worker, args=(world, _free_port(), n_queries, str(tmp_path)), nprocs=world, join=True)
    full = np.load(os.path.join(tmp_path, "full.npy"))
    assert len(full) == n_queries
    assert np.array_equal(full["iterations"], np.arange(n_queries) % 7)
    assert np.array_equal(full["tree_size"], np.arange(n_queries) * 10)


def test_shards_partition_the_queries():
    from paper_2409_06807_b200.batch import shard_queries
    for n, world in ((8192, 8), (37, 4), (3, 8), (0, 2)):
        parts = [shard_queries(n, r, world) for r in range(world)]
        allq = np.sort(np.concatenate(parts)) if n else np.zeros(0, np.int64)
        assert np.array_equal(allq, np.arange(n))
        assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1
    with pytest.raises(ValueError):
        shard_queries(10, 2, 2)


def test_goal_sampler_is_deterministic_and_clear_of_pillars():
    sys.path.insert(0, ROOT)
    import paper_2409_06807_b200 as kp
    env = kp.gen_environment("forest", "quad12", seed=0)
    g = np.stack([kp.goal_for_query(q, env) for q in range(200)])
    assert np.array_equal(g, np.stack([kp.goal_for_query(q, env) for q in range(200)]))
    assert np.all((g[:, :3] >= 1.0) & (g[:, :3] <= 9.0)) and np.all(g[:, 3] == 1.3)
    assert np.all(np.linalg.norm(g[:, :3] - env.start[:3], axis=1) >= 4.0)
    for c in g[:, :3]:
        assert not env.position_in_collision(c)
