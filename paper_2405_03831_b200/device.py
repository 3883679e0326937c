"""Device-side driver of the sweep: buffers, launches, results.

PyTorch is plumbing here -- device memory, the current CUDA stream and (for
multi-GPU) ``torch.distributed``.  Every kernel is ours, launched through the
C ABI of ``libcosched_b200.so``; there is no CPU path for the FNN sweep and a
missing extension or device raises.

``SweepPlan`` owns every buffer of one (apps, grid, pair-shard) shape so that
repeated sweeps (the bench loop, a scheduler serving many windows of the same
size) launch kernels only:

    k_tables -> k_solo -> k_sweep -> k_resolve [-> k_scatter per budget]
"""

from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _native as nat
from .core import NUM_FEATURES, ValidationError
from .grid import KnobGrid

# Relative gap below which the fp32 screen defers to the exact fp64 re-scan.
# The measured fp32 screen error is ~3e-7 relative (SURVEY.md §7 hard part 1);
# the kernel reports the largest gap it saw (SweepPlan.screen_error) and
# SweepPlan.launch() callers can assert it stays far below this.
DEFAULT_REL_EPS = 1e-5


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the cosched_b200 sweep needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise RuntimeError(f"cosched_b200 runs on CUDA devices only, got {dev}")
    return dev


def _dptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def _stream_handle(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class NetworkABI:
    """Keeps the fp64 host arrays behind a cs_network alive."""

    def __init__(self, weights):
        self.arrays = weights.abi_arrays()
        a = self.arrays
        self.struct = nat.CsNetwork(*(nat.ptr(a[k]) for k in
                                      ("w1", "b1", "w2", "b2", "w_out", "b_out", "feature_bounds")))

    def ref(self):
        return ctypes.byref(self.struct)


class DeviceGrid:
    """A KnobGrid's arrays resident on one device, plus its cs_grid struct."""

    def __init__(self, grid: KnobGrid, device):
        self.grid = grid
        self.knob1 = torch.as_tensor(grid.knob1, device=device).contiguous()
        self.knob2 = torch.as_tensor(grid.knob2, device=device).contiguous()
        self.mask = torch.as_tensor(grid.mask.view(np.int32), device=device).contiguous()
        solo = grid.solo_knob if len(grid.solo_knob) else np.zeros((1, 4))
        self.solo_knob = torch.as_tensor(solo, device=device).contiguous()
        s = nat.CsGrid()
        s.n_grid = grid.n_grid
        s.knob1 = ctypes.cast(_dptr(self.knob1), nat.c_double_p)
        s.knob2 = ctypes.cast(_dptr(self.knob2), nat.c_double_p)
        s.mask = ctypes.cast(_dptr(self.mask), nat.c_uint32_p)
        s.n_budgets = grid.n_budgets
        for l in range(grid.n_budgets):
            s.n_configs[l] = grid.n_configs[l]
        for l, off in enumerate(grid.solo_offsets):
            s.solo_offsets[l] = off
        s.solo_knob = ctypes.cast(_dptr(self.solo_knob), nat.c_double_p)
        self.struct = s

    def ref(self):
        return ctypes.byref(self.struct)


def n_pairs(n: int) -> int:
    return n * (n - 1) // 2


@dataclass
class SweepCounters:
    queue_len: int           # (pair, budget)s re-scanned exactly in fp64
    screen_error: float      # largest screened-vs-fp64 relative gap (winners, near runner-ups)
    clamps: np.ndarray       # per budget: floor clamps as the reference counts them
    exact_rows: int = 0      # (pair, member) rows whose clamps were re-counted in fp64
    verify_fail: int = 0     # sampled near-tie pairs whose exact re-scan disagreed

    @property
    def effective_error(self) -> float:
        """The screen error the band must cover: the observed gap, or -- when a
        sampled exact re-scan disagreed with the screen -- infinity."""
        return float("inf") if self.verify_fail else self.screen_error


def fp16_screen_safe(weights) -> bool:
    """Whether the tensor-core screen's fp16 operands can hold this network:
    every layer-1 pre-activation |z1| and every |W2|, |b2| well inside the fp16
    range (the same bound cs_pair_screen's CS_KERNEL_AUTO applies).  Inputs are
    normalized to [0, 1], so |z1| <= |b1| + sum |W1| row-wise."""
    w1 = np.abs(np.asarray(weights.w1, dtype=np.float64))
    zmax = float(np.max(np.abs(np.asarray(weights.b1, dtype=np.float64)) + w1.sum(axis=1)))
    wmax = float(max(np.max(np.abs(weights.w2)), np.max(np.abs(weights.b2))))
    return zmax < 30000.0 and wmax < 30000.0


class SweepPlan:
    """All device buffers for sweeping `n` apps over `grid`, pairs [begin, end)."""

    def __init__(self, weights, grid: KnobGrid, n: int, pair_begin: int = 0,
                 pair_end: Optional[int] = None, device=None, with_matrix: bool = True,
                 rel_eps: float = DEFAULT_REL_EPS, kernel: str = "tcgen05"):
        self.lib = nat.sweep_lib()
        self.device = require_cuda(device)
        if n < 2:
            raise ValidationError(f"need at least 2 apps, got {n}")
        P_all = n_pairs(n)
        pair_end = P_all if pair_end is None else int(pair_end)
        if not 0 <= pair_begin <= pair_end <= P_all:
            raise ValidationError(f"pair range [{pair_begin}, {pair_end}) outside [0, {P_all})")
        self.n, self.grid, self.rel_eps = n, grid, float(rel_eps)
        # the tcgen05 screen (k_sweep_tc3) or the fp32 SIMT screen (k_sweep); both feed
        # the same exact fp64 steps, so results are identical
        kinds = {"tcgen05": nat.KERNEL_TCGEN05, "simt": nat.KERNEL_SIMT}
        if kernel not in kinds:
            raise ValueError(f"kernel must be one of {sorted(kinds)}, got {kernel!r}")
        if kernel == "tcgen05" and not fp16_screen_safe(weights):
            # a network beyond the fp16 operand range takes the fp32 SIMT screen
            # (identical results: the exact fp64 steps are shared)
            kernel = "simt"
        self.kernel, self.kernel_kind = kernel, kinds[kernel]
        if kernel == "tcgen05" and os.environ.get("COSCHED_TC_KIND"):
            # experiment hook: an explicit k_sweep_tc3 instance (0xV3GS kind code)
            self.kernel_kind = int(os.environ["COSCHED_TC_KIND"], 16)
        self.pair_begin, self.pair_end = int(pair_begin), pair_end
        self.P = pair_end - pair_begin
        self.net = NetworkABI(weights)
        dev = self.device
        with torch.cuda.device(dev):
            self.dgrid = DeviceGrid(grid, dev)
            L, G, S = grid.n_budgets, grid.n_grid, grid.solo_offsets[-1]
            nbytes = self.lib.cs_tables_bytes(n, G, S)
            self.table_buf = torch.empty(nbytes + 256, dtype=torch.uint8, device=dev)
            base = (_dptr(self.table_buf) + 255) & ~255
            self.tables = nat.CsTables()
            nat.check(self.lib.cs_tables_bind(base, nbytes, n, G, S, ctypes.byref(self.tables)),
                      "cs_tables_bind")
            # the network goes to device memory once per plan (never per launch)
            nat.check(self.lib.cs_tables_set_network(self.net.ref(), ctypes.byref(self.tables),
                                                     _stream_handle(dev)), "cs_tables_set_network")
            P = max(self.P, 1)
            self.corun_grid_index = torch.empty((L, P), dtype=torch.int32, device=dev)
            self.corun_time = torch.empty((L, P), dtype=torch.float64, device=dev)
            self.corun_chosen = torch.empty((L, P), dtype=torch.uint8, device=dev)
            self.weight = torch.empty((L, P), dtype=torch.float64, device=dev)
            self.solo_time = torch.empty((L, n), dtype=torch.float64, device=dev)
            self.solo_split = torch.empty((L, n), dtype=torch.int32, device=dev)
            self.solo_clamps = torch.empty((L, n), dtype=torch.int32, device=dev)
            # [0, L P): exact re-scan queue; [L P, (L + 2) P): rows whose floor
            # clamps k_resolve re-counts in fp64
            self.queue = torch.empty((L + 2) * P, dtype=torch.int64, device=dev)
            self.counters = torch.zeros(nat.COUNTERS_BYTES // 4, dtype=torch.int32, device=dev)
            self.clamps = torch.zeros(L, dtype=torch.int64, device=dev)
            self.matrix = (torch.zeros((L, n, n), dtype=torch.float64, device=dev)
                           if with_matrix else None)
        self.pair_out = nat.CsPairOut(
            ctypes.cast(_dptr(self.corun_grid_index), nat.c_int32_p),
            ctypes.cast(_dptr(self.corun_time), nat.c_double_p),
            ctypes.cast(_dptr(self.corun_chosen), nat.c_uint8_p),
            ctypes.cast(_dptr(self.weight), nat.c_double_p))
        self.solo_out = nat.CsSoloOut(
            ctypes.cast(_dptr(self.solo_time), nat.c_double_p),
            ctypes.cast(_dptr(self.solo_split), nat.c_int32_p),
            ctypes.cast(_dptr(self.solo_clamps), nat.c_int32_p))
        self._side = torch.cuda.Stream(self.device)
        # one sweep at a time through this plan's buffers: callers that share a
        # cached plan (sweep.plan_for) hold it from launch to read-back
        self.lock = threading.RLock()
        # the tcgen05 screen runs the fused pipeline: k_tables (+ solo
        # splits) -> k_sweep_tc3 (+ decide/scatter) -> k_resolve (+ decide);
        # the other screens keep tables | solo -> screen -> resolve -> decide
        self.fused = kernel == "tcgen05"
        self.launches_per_run = 3 if self.fused else 5

    # ------------------------------------------------------------------
    def launch(self, d_features: torch.Tensor, d_base_time: torch.Tensor,
               sweep_events: Optional[tuple] = None, rel_eps: Optional[float] = None) -> None:
        """Enqueue one full sweep on the current stream (no host sync).

        `sweep_events` = (start, end) CUDA events recorded around the k_sweep
        launch only (bench.py times the dominant kernel with them; create them
        with external=True when the launch is captured into a CUDA graph)."""
        n = self.n
        if d_features.shape != (n, NUM_FEATURES) or d_base_time.shape != (n,):
            raise ValidationError(f"expected features ({n}, 18) and base_time ({n},)")
        if d_features.dtype != torch.float64 or d_base_time.dtype != torch.float64:
            raise ValidationError("features and base_time must be float64")
        if not (d_features.is_contiguous() and d_base_time.is_contiguous()):
            raise ValidationError("features and base_time must be contiguous")
        lib, dev = self.lib, self.device
        eps = self.rel_eps if rel_eps is None else float(rel_eps)
        cur = torch.cuda.current_stream(dev)
        st = cur.cuda_stream
        tref = ctypes.byref(self.tables)
        cnt = _dptr(self.counters)
        if self.fused:
            # k_tables also zeroes the counters and clamps for the screen
            nat.check(lib.cs_prepare(self.net.ref(), _dptr(d_features), _dptr(d_base_time), n,
                                     self.dgrid.ref(), tref, self.solo_out, cnt,
                                     _dptr(self.clamps), st), "cs_prepare")
            if self.P == 0:
                return
            # the symmetric matrix is scattered in-kernel when this plan owns
            # the whole graph (its diagonal stays zero from allocation)
            w = _dptr(self.matrix) if (self.matrix is not None and self.P == n_pairs(n)) else None
            if sweep_events is not None:
                sweep_events[0].record(cur)
            nat.check(lib.cs_pair_screen_fused(
                self.net.ref(), tref, self.dgrid.ref(), _dptr(d_base_time), _dptr(self.solo_time),
                _dptr(self.solo_clamps), self.pair_begin, self.pair_end, eps,
                self.pair_out, _dptr(self.queue), cnt, _dptr(self.clamps), w, self.kernel_kind,
                st), "cs_pair_screen_fused")
            if sweep_events is not None:
                sweep_events[1].record(cur)
            nat.check(lib.cs_resolve_fused(
                self.net.ref(), tref, self.dgrid.ref(), _dptr(d_base_time), _dptr(self.solo_time),
                _dptr(self.solo_clamps), self.pair_begin, self.pair_end, self.pair_out,
                _dptr(self.queue), cnt, _dptr(self.clamps), w, st), "cs_resolve_fused")
            if self.matrix is not None and w is None:
                self.scatter(st)
            return
        self.counters.zero_()
        self.clamps.zero_()
        nat.check(lib.cs_build_tables(self.net.ref(), _dptr(d_features), n, self.dgrid.ref(),
                                      tref, st), "cs_build_tables")
        # solo splits run on a side stream, concurrently with the pair screen
        # (the screen does not read them; cs_pair_decide does)
        self._side.wait_stream(cur)
        nat.check(lib.cs_solo(self.net.ref(), tref, self.dgrid.ref(), _dptr(d_base_time),
                              self.solo_out, self._side.cuda_stream), "cs_solo")
        if self.P == 0:
            cur.wait_stream(self._side)
            return
        if sweep_events is not None:
            sweep_events[0].record(cur)
        nat.check(lib.cs_pair_screen(self.net.ref(), tref, self.dgrid.ref(), _dptr(d_base_time),
                                     self.pair_begin, self.pair_end, eps, self.pair_out,
                                     _dptr(self.queue), cnt, _dptr(self.clamps), self.kernel_kind,
                                     st), "cs_pair_screen")
        if sweep_events is not None:
            sweep_events[1].record(cur)
        nat.check(lib.cs_resolve(self.net.ref(), tref, self.dgrid.ref(), _dptr(d_base_time),
                                 self.pair_begin, self.pair_end, self.pair_out, _dptr(self.queue),
                                 cnt, _dptr(self.clamps), st), "cs_resolve")
        cur.wait_stream(self._side)
        # decisions (+ the symmetric matrix when this plan owns the whole graph)
        w = _dptr(self.matrix) if (self.matrix is not None and self.P == n_pairs(n)) else None
        nat.check(lib.cs_pair_decide(self.dgrid.ref(), _dptr(self.solo_time),
                                     _dptr(self.solo_clamps), n, self.pair_begin, self.pair_end,
                                     self.pair_out, _dptr(self.clamps), w, st), "cs_pair_decide")
        if self.matrix is not None and w is None:
            self.scatter(st)

    def scatter(self, st=None) -> None:
        st = _stream_handle(self.device) if st is None else st
        P = self.P
        for l in range(self.grid.n_budgets):
            nat.check(self.lib.cs_scatter_weights(
                _dptr(self.weight) + 8 * l * max(P, 1), self.n, self.pair_begin, self.pair_end,
                _dptr(self.matrix) + 8 * l * self.n * self.n, st), "cs_scatter_weights")

    def read_counters(self) -> SweepCounters:
        c = self.counters.cpu().numpy()
        return SweepCounters(queue_len=int(c[0]),
                             screen_error=float(np.array([c[1]], dtype=np.int32).view(np.float32)[0]),
                             clamps=self.clamps.cpu().numpy().astype(np.int64),
                             exact_rows=int(np.uint32(c[2])), verify_fail=int(np.uint32(c[3])))


def to_device_inputs(features, base_time, device) -> tuple:
    f = torch.as_tensor(np.ascontiguousarray(features, dtype=np.float64)).to(device, non_blocking=True)
    b = torch.as_tensor(np.ascontiguousarray(base_time, dtype=np.float64)).to(device, non_blocking=True)
    return f.contiguous(), b.contiguous()


def forward_rows(weights, X: np.ndarray) -> np.ndarray:
    """fnn.forward_batch on the GPU (fp64, unfloored)."""
    lib = nat.sweep_lib()
    dev = require_cuda()
    X = np.ascontiguousarray(X, dtype=np.float64)
    rows = X.shape[0]
    if rows == 0:
        return np.zeros(0)
    net = NetworkABI(weights)
    dx = torch.as_tensor(X).to(dev)
    dy = torch.empty(rows, dtype=torch.float64, device=dev)
    nat.check(lib.cs_forward_rows(net.ref(), _dptr(dx), rows, _dptr(dy), _stream_handle(dev)),
              "cs_forward_rows")
    return dy.cpu().numpy()
