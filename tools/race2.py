#!/usr/bin/env python3
"""OR-parallel race between two processes (torchrun, gloo rendezvous).  On a one-GPU box both ranks share the
device: the stop words are still exchanged through CUDA IPC and the winner's kernel still stores into the peer's
word, which is the plumbing a multi-GPU race uses (there the store crosses NVLink)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
import paper_2409_06807_b200 as kp

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(int(os.environ.get("KPX_RACE_DEVICE", os.environ.get("LOCAL_RANK", "0"))))
model = kp.get_model("di6"); env = kp.gen_environment("forest", model, seed=0)
cfg = kp.PlannerConfig(t_e=200000, t_prop=1.0, cells_per_dim=4, seed=0, t_max=30.0)
flags = kp.RaceFlags()
with kp.KinoPax(cfg, env, model, backend="cuda-f32") as eng:
    eng.reset(seed=100 + rank); eng.solve()            # warm-up (module load) outside the race
    flags.clear()
    dist.barrier()
    t0 = time.perf_counter()
    res = kp.race(eng, flags, seed=rank)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) * 1e3
    dist.barrier()
    out = [None] * world
    if res.solved:      # a winner's plan has been rebuilt and re-validated in float64 before it is reported
        assert kp.ValidityChecker(env, model, 0.05).trajectory_valid(res.trajectory, start=env.start)
    dist.all_gather_object(out, (rank, int(res.device["status_code"]), int(res.stats.iterations), bool(flags.fired()), dt))
    if rank == 0:
        for r in out: print("rank %d: status %d iterations %d own_flag_fired %s %.3f ms" % r)
        winners = [r for r in out if r[1] == 0]
        stopped = [r for r in out if r[1] == 5]
        print("winners", len(winners), "stopped", len(stopped))
        assert len(winners) >= 1
        # every rank other than a winner had its flag raised by a peer's kernel
        for r in out:
            if r[1] == 0:
                continue
            assert r[3], "loser's flag was not raised"
        # a winner raised the flag of every peer
        print("race ok")
dist.destroy_process_group()
