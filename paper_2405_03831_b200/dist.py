"""Multi-GPU sweep: pairs sharded across ranks, one all-gather of the records.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch for the
data path).  Pairs are independent units, so rank r sweeps the
contiguous linear pair range ``shard_range(P, r, W)`` with the per-app and
per-knob tables replicated (each rank builds its own; they are ~N*37 floats).
The only exchange is the all-gather of the fixed-size per-pair records
(best config index i32, CoRunTime f64, co-run flag u8, winning weight f64),
after which every rank holds the full record set; the scatter into the
symmetric N x N matrix that the host matcher consumes runs on the device.
"""

from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist

RECORD_FIELDS = (("corun_grid_index", torch.int32), ("corun_time", torch.float64),
                 ("corun_chosen", torch.uint8), ("weight", torch.float64))


def shard_range(P: int, rank: int, world: int) -> tuple:
    """Balanced contiguous split of [0, P): sizes differ by at most one."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    base, extra = divmod(P, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def gather_records(local: dict, P: int, group: Optional[dist.ProcessGroup] = None) -> dict:
    """All-gather per-rank record shards (each (L, P_rank)) into full (L, P) tensors.

    Shards are padded to the largest shard so one ``all_gather_into_tensor``
    per field suffices (NCCL's ring/NVLS all-gather needs equal sizes); the
    padding is dropped while re-assembling in rank order.
    """
    world = dist.get_world_size(group)
    sizes = [shard_range(P, r, world) for r in range(world)]
    cap = max(e - b for b, e in sizes)
    out = {}
    for name, dtype in RECORD_FIELDS:
        t = local[name]
        L, n_local = t.shape
        padded = torch.zeros((L, cap), dtype=dtype, device=t.device)
        padded[:, :n_local] = t
        # gather buffer laid out rank-major: (world, L, cap)
        buf = torch.empty((world, L, cap), dtype=dtype, device=t.device)
        if hasattr(dist, "all_gather_into_tensor") and t.device.type == "cuda":
            dist.all_gather_into_tensor(buf, padded.contiguous(), group=group)
        else:
            dist.all_gather(list(buf.unbind(0)), padded.contiguous(), group=group)
        full = torch.empty((L, P), dtype=dtype, device=t.device)
        for r, (b, e) in enumerate(sizes):
            full[:, b:e] = buf[r, :, :e - b]
        out[name] = full
    return out


class ShardedSweep:
    """A SweepPlan on this rank's pair shard plus the gather and the device scatter."""

    def __init__(self, weights, grid, n: int, group=None, device=None, rel_eps=None,
                 kernel: str = "tcgen05"):
        from .device import DEFAULT_REL_EPS, SweepPlan
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.n = n
        self.P = n * (n - 1) // 2
        b, e = shard_range(self.P, self.rank, self.world)
        self.plan = SweepPlan(weights, grid, n, b, e, device=device, with_matrix=False,
                              rel_eps=DEFAULT_REL_EPS if rel_eps is None else rel_eps,
                              kernel=kernel)
        self.matrix = torch.zeros((grid.n_budgets, n, n), dtype=torch.float64,
                                  device=self.plan.device)

    def run(self, d_features, d_base_time, sweep_events=None) -> dict:
        """Sweep the local shard, all-gather the records, scatter the full matrix."""
        from . import _native as nat
        plan = self.plan
        plan.launch(d_features, d_base_time, sweep_events)
        P_loc = plan.P
        local = {"corun_grid_index": plan.corun_grid_index[:, :P_loc],
                 "corun_time": plan.corun_time[:, :P_loc],
                 "corun_chosen": plan.corun_chosen[:, :P_loc],
                 "weight": plan.weight[:, :P_loc]}
        full = gather_records(local, self.P, self.group)
        st = torch.cuda.current_stream(plan.device).cuda_stream
        w = full["weight"].contiguous()
        for l in range(plan.grid.n_budgets):
            nat.check(plan.lib.cs_scatter_weights(w.data_ptr() + 8 * l * self.P, self.n, 0,
                                                  self.P, self.matrix[l].data_ptr(), st),
                      "cs_scatter_weights")
        full["matrix"] = self.matrix
        return full
