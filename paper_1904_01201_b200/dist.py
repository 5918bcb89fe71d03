"""Multi-GPU plumbing: env sharding and the episode-statistics all-gather.

Envs are independent (no shared mutable state), so the path
shards with no data-path collective: rank r owns the contiguous env range
[lo, hi) of the global batch, with per-env seeds derived from the global env
id so results do not depend on the GPU count.  The only exchange is an
all-gather of fixed-size per-env outcome records (the analogue of
``agents.evaluate``'s reduction, src/agents.py:467-503) over NCCL (gloo on
CPU for the tests).
"""
from __future__ import annotations

from dataclasses import dataclass

RECORD_FIELDS = ("path_length", "collisions", "x", "y", "heading")  # 5 x f64 = 40 B


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
    """All-gather (n_local, 5) f64 records from every rank -> (n_total, 5) in
    global env order.  Ranks may hold different counts (padded exchange)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return local
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


def episode_records(sim):
    """(n_local, 5) f64 device tensor of per-env outcome records."""
    import torch
    xy, h, p, k = sim.state()
    return torch.stack([p, k.to(torch.float64), xy[:, 0], xy[:, 1], h], dim=1).contiguous()


def gather_episode_stats(sim, shard: EnvShard, world: int) -> dict:
    rec = gather_records(episode_records(sim), world)
    return {"envs": int(rec.shape[0]), "record_bytes": int(rec.shape[1] * 8),
            "mean_path_length": float(rec[:, 0].mean().item()),
            "total_collisions": int(rec[:, 1].sum().item())}
