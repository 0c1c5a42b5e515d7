#!/usr/bin/env python3
"""A sharded plan end to end under torchrun (gloo rendezvous): every rank plans the queries q = rank (mod world) of
one config-5 style batch on its GPU (KPX_SHARD_DEVICE pins all ranks to one device on a one-GPU box), the per-query
records are gathered once with gather_records, and rank 0 holds them to a single-rank run of the whole batch:
sharding must not change any query's outcome."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch, torch.distributed as dist
import paper_2409_06807_b200 as kp

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(int(os.environ.get("KPX_SHARD_DEVICE", os.environ.get("LOCAL_RANK", "0"))))
n_queries = int(os.environ.get("KPX_SHARD_QUERIES", "48"))
model = kp.get_model("quad12"); env = kp.gen_environment("forest", model, seed=0)
cfg = kp.PlannerConfig(t_e=60000, t_prop=model.default_t_prop, cells_per_dim=model.default_cells_per_dim, seed=0, t_max=30.0)
idx = kp.shard_queries(n_queries, rank, world)
goals = kp.goals_for_queries(idx, env)
with kp.BatchPlanner(cfg, env, model, backend="cuda-f32", n_teams=8, team_ctas=1) as bp:
    res = bp.run(idx, goals=goals)
    full = kp.gather_records(idx, res.records, n_queries)
    if rank == 0:
        whole = bp.run(np.arange(n_queries), goals=kp.goals_for_queries(np.arange(n_queries), env))
        for k in ("status", "iterations", "tree_size", "solution_slot", "chain_len", "items", "substeps", "checked"):
            assert np.array_equal(full[k], whole.records[k]), k
        print("shard ok: %d queries over %d ranks, %d solved, %d re-validated" %
              (n_queries, world, int((full["status"] == 0).sum()), int((full["checked"] == 1).sum())))
    else:
        assert full is None
dist.barrier()
dist.destroy_process_group()
