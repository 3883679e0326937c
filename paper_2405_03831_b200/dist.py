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
        if t.device.type == "cuda" and dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(buf, padded.contiguous(), group=group)
        else:   # gloo (CPU tests, or ranks sharing one GPU): stage through the host
            host = [torch.empty((L, cap), dtype=dtype) for _ in range(world)]
            dist.all_gather(host, padded.cpu().contiguous(), group=group)
            buf.copy_(torch.stack(host))
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
        cap = max(e2 - b2 for b2, e2 in (shard_range(self.P, r, self.world)
                                         for r in range(self.world)))
        # the shard's records live in one packed buffer of the same size on every
        # rank: the exchange is ONE all-gather (NCCL over NVLink), then one device
        # scatter of the whole matrix from the gathered blocks
        self.plan = SweepPlan(weights, grid, n, b, e, device=device, with_matrix=False,
                              rel_eps=DEFAULT_REL_EPS if rel_eps is None else rel_eps,
                              kernel=kernel, record_cap=cap)
        self.cap = cap
        self.gathered = torch.empty(self.world * self.plan.records.numel(), dtype=torch.uint8,
                                    device=self.plan.device)
        self.matrix = torch.zeros((grid.n_budgets, n, n), dtype=torch.float64,
                                  device=self.plan.device)

    def run_host(self, h_features, h_base_time, h_matrix=None) -> None:
        """End to end on this rank: pinned host inputs -> H2D -> shard sweep ->
        all-gather -> full matrix -> D2H into `h_matrix` (pinned, rank 0 only
        needs it; pass None elsewhere).  Synchronizes the stream."""
        dev = self.plan.device
        d_f = h_features.to(dev, non_blocking=True)
        d_b = h_base_time.to(dev, non_blocking=True)
        full = self.run(d_f, d_b)
        if h_matrix is not None:
            h_matrix.copy_(full, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()

    def exchange(self) -> None:
        """All-gather the packed records of every shard and scatter the full matrix."""
        from . import _native as nat
        plan = self.plan
        local = plan.records
        if local.device.type == "cuda" and dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(self.gathered, local, group=self.group)
        else:   # gloo (CPU tests, ranks sharing one GPU): stage through the host
            host = [torch.empty_like(local, device="cpu") for _ in range(self.world)]
            dist.all_gather(host, local.cpu(), group=self.group)
            self.gathered.copy_(torch.cat(host))
        st = torch.cuda.current_stream(plan.device).cuda_stream
        nat.check(plan.lib.cs_scatter_gathered(self.gathered.data_ptr(), self.world,
                                               local.numel(), self.P, self.n,
                                               plan.grid.n_budgets, self.matrix.data_ptr(), st),
                  "cs_scatter_gathered")

    def run(self, d_features, d_base_time, sweep_events=None) -> torch.Tensor:
        """Sweep the local shard, exchange, and return the full (L, N, N) matrix."""
        self.plan.launch(d_features, d_base_time, sweep_events)
        self.exchange()
        return self.matrix

    def records(self) -> dict:
        """Full (L, P) record arrays (host-side reassembly of the gathered blocks)."""
        plan = self.plan
        L = plan.grid.n_budgets
        blocks = self.gathered.view(self.world, -1)
        out = {k: [] for k in ("corun_grid_index", "corun_time", "corun_chosen", "weight")}
        for r in range(self.world):
            b, e = shard_range(self.P, r, self.world)
            Pr = e - b
            base = blocks[r]
            o = nat_layout(plan, self.cap, L)
            for name, (off, dt, es) in o.items():
                out[name].append(base[off:off + L * Pr * es].view(dt).view(L, Pr))
        return {k: torch.cat(v, dim=1) for k, v in out.items()}


def nat_layout(plan, cap: int, L: int) -> dict:
    """Byte offsets of the packed record fields (cs_packed_records_layout)."""
    import ctypes
    from . import _native as nat
    lay = nat.CsPairOut()
    nat.check(plan.lib.cs_packed_records_layout(plan.records.data_ptr(), cap, L,
                                                ctypes.byref(lay)), "cs_packed_records_layout")
    base = plan.records.data_ptr()
    addr = lambda p: ctypes.cast(p, ctypes.c_void_p).value - base
    return {"weight": (addr(lay.weight), torch.float64, 8),
            "corun_time": (addr(lay.corun_time), torch.float64, 8),
            "corun_grid_index": (addr(lay.corun_grid_index), torch.int32, 4),
            "corun_chosen": (addr(lay.corun_chosen), torch.uint8, 1)}
