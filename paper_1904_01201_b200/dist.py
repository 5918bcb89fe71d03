"""Multi-GPU plumbing: env sharding and the EpisodeOutcome all-gather.

Envs are independent (no shared mutable state), so the path
shards with no data-path collective: rank r owns the contiguous env range
[lo, hi) of the global batch, with per-env seeds derived from the global env
id so results do not depend on the GPU count.  The only exchange is an
all-gather of the task layer's fixed 40-byte EpisodeOutcome records
(task.py:58-66; include/navsim_b200.h nv_task_step) -- the analogue of
``agents.evaluate``'s reduction over episodes (src/agents.py:467-503) -- over
NCCL (gloo on CPU for the tests).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

OUTCOME_RECORD_BYTES = 40


@dataclass(frozen=True)
class EnvShard:
    n_total: int
    world: int
    rank: int

    @property
    def lo(self) -> int:
        base, rem = divmod(self.n_total, self.world)
        return self.rank * base + min(self.rank, rem)

    @property
    def hi(self) -> int:
        base, rem = divmod(self.n_total, self.world)
        return self.lo + base + (1 if self.rank < rem else 0)

    @property
    def n_local(self) -> int:
        return self.hi - self.lo


def gather_records(local, world: int):
    """All-gather (n_local, k) records (any dtype) from every rank -> (n_total,
    k) in global env order.  Ranks may hold different counts (padded
    exchange)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return local
    if local.is_cuda and dist.get_backend() == "gloo":  # gloo all-gathers host tensors
        return gather_records(local.cpu(), world).to(local.device)
    n = torch.tensor([local.shape[0]], device=local.device, dtype=torch.int64)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n)
    counts = [int(c.item()) for c in counts]
    m = max(counts)
    pad = torch.zeros((m, local.shape[1]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    return torch.cat([b[:c] for b, c in zip(bufs, counts)], dim=0)


def outcome_summary(records: np.ndarray, finished: np.ndarray) -> dict:
    """agents.evaluate's aggregate (src/agents.py:467-503) over the finished
    envs of an (n, 40) u8 record array."""
    from .task import OUTCOME_DTYPE
    rec = np.ascontiguousarray(records).view(OUTCOME_DTYPE).reshape(-1)[finished.astype(bool)]
    n = int(len(rec))
    if n == 0:
        return {"episodes": 0, "record_bytes": OUTCOME_RECORD_BYTES}
    return {"episodes": n, "record_bytes": OUTCOME_RECORD_BYTES,
            "success_rate": float(rec["success"].mean()),
            "spl": float(rec["spl"].mean()),
            "mean_steps": float(rec["steps"].mean()),
            "mean_path_taken": float(rec["path_taken"].mean()),
            "mean_shortest_path": float(rec["shortest_path"].mean()),
            "collisions": int(rec["collisions"].sum()),
            "terminated_by_stop": int((rec["terminated_by"] == 1).sum())}


def pointgoal_eval(env, scene, shard: EnvShard, world: int, n_steps: int = 64, seed: int = 11,
                   actions=None):
    """A PointGoal evaluation over this rank's envs of ``env`` (a
    task.BatchEnvironment built with max_steps >= n_steps): seeded episodes
    (synth.pointgoal_episodes, keyed by global env id), ``n_steps`` steps of
    the uniform random forward/left/right policy ending with STOP (every
    episode terminates), then the all-gather of the 40-byte EpisodeOutcome
    records.  Returns (summary, gathered records (n_total, 40) u8 tensor,
    gathered finished flags)."""
    import torch

    from . import synth
    eps = synth.pointgoal_episodes(env, scene, shard.n_local, seed=seed, first=shard.lo)
    mask = np.array([e is not None for e in eps])
    dummy = next((e for e in eps if e is not None), None)
    if dummy is None:
        raise RuntimeError("no PointGoal episode fits this scene")
    env.reset([e if e is not None else dummy for e in eps], mask=mask)
    if actions is None:
        actions = synth.random_actions(shard.n_total, n_steps, seed=seed)[:, shard.lo:shard.hi]
    acts = torch.as_tensor(np.ascontiguousarray(actions), device=env.dev)
    acts[n_steps - 1] = 3  # STOP
    for t in range(n_steps):
        env.step(acts[t])
    torch.cuda.synchronize()
    done = env.done.clone() & torch.as_tensor(mask.astype(np.uint8), device=env.dev)
    rec = gather_records(env.outcome.contiguous(), world)
    fin = gather_records(done.reshape(-1, 1).contiguous(), world).reshape(-1)
    summary = outcome_summary(rec.cpu().numpy(), fin.cpu().numpy())
    summary["policy"] = f"uniform random forward/left/right for {n_steps - 1} steps, then STOP"
    summary["gathered_envs"] = int(rec.shape[0])
    return summary, rec, fin
