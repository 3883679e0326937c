"""Multi-GPU sweep: pairs sharded across ranks, one gather of 11-byte records to rank 0.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch for the
data path).  Pairs are independent units, so rank r sweeps the
contiguous linear pair range ``shard_range(P, r, W)`` with the per-app and
per-knob tables replicated (each rank builds its own; they are ~N*37 floats).

The only exchange is ONE gather to rank 0 -- the host matcher runs there --
of each shard's decision records in the 11-byte wire format of
``cs_pack_records`` (CoRunTime f64, config index u16, co-run flag u8 per
(pair, budget)).  Rank 0 rebuilds the full record set and the symmetric
N x N matrix on its device (``cs_unpack_gathered``, which re-derives each
winning weight exactly as the sweep does).  At 4,096 apps that is 92 MB
in total over NVSwitch, against 176 MB of 21-byte records all-gathered to
every rank before.

Exactness is a collective property: after each run the ranks all-reduce
(MAX) their screen-error monitor and their sampled re-scan disagreements;
should either call for a wider ambiguity band, every rank redoes its shard
with the same wider band (the rule of ``sweep.run_plan``).
"""

from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist


def shard_range(P: int, rank: int, world: int) -> tuple:
    """Balanced contiguous split of [0, P): sizes differ by at most one."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    base, extra = divmod(P, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def shard_cap(P: int, world: int) -> int:
    """Slots per budget of every rank's wire buffer (the largest shard)."""
    return (P + world - 1) // world if world else 0


def wire_layout(cap: int, L: int) -> dict:
    """Byte offsets of the wire fields (mirrors cs_wire_records_bytes)."""
    a = lambda v: (v + 255) & ~255
    n = cap * L
    t, i = 0, a(8 * n)
    f = i + a(2 * n)
    return {"corun_time": t, "corun_grid_index": i, "corun_chosen": f, "total": f + a(n)}


def gather_to_root(local: torch.Tensor, group: Optional[dist.ProcessGroup] = None,
                   root: int = 0) -> Optional[torch.Tensor]:
    """Gather every rank's equal-sized uint8 buffer to `root`: a (world, nbytes)
    tensor there, None elsewhere.  NCCL for CUDA buffers (one gather over
    NVLink); gloo (CPU tests, ranks sharing one GPU) through host memory."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    nccl = local.device.type == "cuda" and dist.get_backend(group) == "nccl"
    src = local if nccl else local.cpu()
    out = torch.empty((world, local.numel()), dtype=torch.uint8, device=src.device) \
        if rank == root else None
    dist.gather(src, list(out.unbind(0)) if out is not None else None,
                dst=dist.get_global_rank(group, root) if group is not None else root, group=group)
    if out is not None and out.device != local.device:
        out = out.to(local.device)
    return out


class ShardedSweep:
    """A SweepPlan on this rank's pair shard, the record gather and rank 0's rebuild."""

    def __init__(self, weights, grid, n: int, group=None, device=None, rel_eps=None,
                 kernel: str = "tcgen05"):
        from .device import DEFAULT_REL_EPS, SweepPlan
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.n = n
        self.P = n * (n - 1) // 2
        self.L = grid.n_budgets
        b, e = shard_range(self.P, self.rank, self.world)
        self.cap = shard_cap(self.P, self.world)
        self.plan = SweepPlan(weights, grid, n, b, e, device=device, with_matrix=False,
                              rel_eps=DEFAULT_REL_EPS if rel_eps is None else rel_eps,
                              kernel=kernel)
        dev = self.plan.device
        self.wire_bytes = int(self.plan.lib.cs_wire_records_bytes(self.cap, self.L))
        self.wire = torch.zeros(self.wire_bytes, dtype=torch.uint8, device=dev)
        self.is_root = self.rank == 0
        self.gathered = None
        if self.is_root:
            # the full record set and matrix live on rank 0 only
            self.full = {"corun_grid_index": torch.empty((self.L, self.P), dtype=torch.int32, device=dev),
                         "corun_time": torch.empty((self.L, self.P), dtype=torch.float64, device=dev),
                         "corun_chosen": torch.empty((self.L, self.P), dtype=torch.uint8, device=dev),
                         "weight": torch.empty((self.L, self.P), dtype=torch.float64, device=dev)}
            self.matrix = torch.zeros((self.L, n, n), dtype=torch.float64, device=dev)
        else:
            self.full, self.matrix = None, None
        self._status = torch.zeros(2, dtype=torch.float32, device=dev if self._nccl() else "cpu")

    def _nccl(self) -> bool:
        return self.plan.device.type == "cuda" and dist.get_backend(self.group) == "nccl"

    def exchange(self) -> None:
        """Pack this shard, gather every shard to rank 0, rebuild records + matrix there."""
        from . import _native as nat
        plan = self.plan
        st = torch.cuda.current_stream(plan.device).cuda_stream
        nat.check(plan.lib.cs_pack_records(plan.pair_out, plan.P, self.L, self.cap,
                                           self.wire.data_ptr(), st), "cs_pack_records")
        self.gathered = gather_to_root(self.wire, self.group)
        if self.is_root:
            f = self.full
            full = nat.CsPairOut(*(nat.ctypes.cast(f[k].data_ptr(), t) for k, t in (
                ("corun_grid_index", nat.c_int32_p), ("corun_time", nat.c_double_p),
                ("corun_chosen", nat.c_uint8_p), ("weight", nat.c_double_p))))
            nat.check(plan.lib.cs_unpack_gathered(self.gathered.data_ptr(), self.world,
                                                  self.wire_bytes, self.n, self.L,
                                                  plan.solo_time.data_ptr(), full,
                                                  self.matrix.data_ptr(), st),
                      "cs_unpack_gathered")

    def run(self, d_features, d_base_time, sweep_events=None, rel_eps=None):
        """Sweep the local shard and exchange (stream-ordered, no host sync):
        rank 0's full (L, N, N) matrix, None on the other ranks."""
        self.plan.launch(d_features, d_base_time, sweep_events, rel_eps=rel_eps)
        self.exchange()
        return self.matrix

    def status(self) -> tuple:
        """(largest screen error over all ranks, any sampled re-scan disagreement):
        one tiny all-reduce; synchronizes."""
        c = self.plan.read_counters()
        s = torch.tensor([c.screen_error, float(c.verify_fail)], dtype=torch.float32,
                         device=self._status.device)
        dist.all_reduce(s, op=dist.ReduceOp.MAX, group=self.group)
        return float(s[0]), bool(s[1] > 0)

    def run_checked(self, d_features, d_base_time):
        """run() plus the collective precision guard: if any rank's screen error is
        not well inside the band (or a sampled re-scan disagreed), every rank
        redoes its shard with the same wider band.  Returns the band used."""
        eps = self.plan.rel_eps
        self.run(d_features, d_base_time, rel_eps=eps)
        err, bad = self.status()
        while (err > 0.25 * eps or bad) and 16.0 * eps < 0.1:
            eps = min(max(16.0 * eps, 16.0 * err), 0.099)
            self.run(d_features, d_base_time, rel_eps=eps)
            err, bad = self.status()
        if err > 0.25 * eps or bad:
            raise RuntimeError(f"fp32 screen error {err:.3g} is too close to rel_eps {eps:.3g}; "
                               "argmin parity is no longer guaranteed")
        return eps

    def run_host(self, h_features, h_base_time, h_matrix=None) -> None:
        """End to end on this rank: pinned host inputs -> H2D -> shard sweep ->
        gather -> rank 0 rebuilds the matrix -> D2H into `h_matrix` (pinned, rank
        0 only).  Checked and synchronizing."""
        dev = self.plan.device
        d_f = h_features.to(dev, non_blocking=True)
        d_b = h_base_time.to(dev, non_blocking=True)
        self.run_checked(d_f, d_b)
        if self.is_root and h_matrix is not None:
            h_matrix.copy_(self.matrix, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()

    def records(self) -> Optional[dict]:
        """Rank 0: the full (L, P) record tensors (device); None elsewhere."""
        return self.full
