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


def _plan_on_cpu(q, t_e=4000):
    """One small query planned by the CPU oracle (the checker; there is no CPU planner in the product): what a rank's
    GPU would report for query q, so that the sharded path moves real per-query records."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    import paper_2409_06807_b200 as kp
    model = kp.get_model("di6")
    env = kp.gen_environment("forest", model, seed=0)
    cfg = kp.PlannerConfig(t_e=t_e, t_prop=1.0, cells_per_dim=4, seed=int(q))
    op = oracle.plan_from_problem(kp.build_problem(cfg, env, model))
    op.solve(t_max=60.0)
    return {"solved": 0, "capacity_exhausted": 2}[op.status], int(op.raw.iteration), int(op.raw.size), int(op.raw.solution_slot)


def _worker(rank, world, port, n_queries, out_dir):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_2409_06807_b200 import _lib
    from paper_2409_06807_b200.batch import gather_records, shard_queries
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    idx = shard_queries(n_queries, rank, world)          # this rank's queries: q mod world == rank
    rec = np.zeros(len(idx), dtype=_lib.QUERY_RESULT_DTYPE)
    for i, q in enumerate(idx):
        rec["status"][i], rec["iterations"][i], rec["tree_size"][i], rec["solution_slot"][i] = _plan_on_cpu(q)
    full = gather_records(idx, rec, n_queries)
    if rank == 0:
        np.save(os.path.join(out_dir, "full.npy"), full)
    else:
        assert full is None
    dist.barrier()
    dist.destroy_process_group()


def test_shard_and_gather_world2(tmp_path):
    import torch.multiprocessing as mp
    n_queries, world = 13, 2
    mp.spawn(_worker, args=(world, _free_port(), n_queries, str(tmp_path)), nprocs=world, join=True)
    full = np.load(os.path.join(tmp_path, "full.npy"))
    assert len(full) == n_queries
    # the sharded job reports, query by query, what one process planning every query reports
    for q in range(n_queries):
        status, iters, size, slot = _plan_on_cpu(q)
        assert (full["status"][q], full["iterations"][q], full["tree_size"][q], full["solution_slot"][q]) == (status, iters, size, slot), q
    assert len(set(full["tree_size"].tolist())) > 3


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
