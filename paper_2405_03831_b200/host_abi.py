"""The host-buffer entry point ``cs_build_graph_host`` (include/cosched_b200.h).

This is the call a non-torch caller (the reference's own ctypes binding, see
INTEGRATION.md) makes: host features/base times and the knob grid in, host
weight matrix and per-pair records out; the H2D copies, the five kernels and
the D2H copies all happen inside the one call.  ``HostGraphCall`` keeps pinned
host buffers and the device workspace so repeated calls (bench e2e) do not
re-allocate.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native as nat
from .device import DEFAULT_REL_EPS, NetworkABI, require_cuda
from .grid import KnobGrid


def _host_grid(grid: KnobGrid):
    keep = {
        "knob1": np.ascontiguousarray(grid.knob1 if grid.n_grid else np.zeros((1, 4))),
        "knob2": np.ascontiguousarray(grid.knob2 if grid.n_grid else np.zeros((1, 4))),
        "mask": np.ascontiguousarray(grid.mask if grid.n_grid else np.zeros(1, np.uint32)),
        "solo": np.ascontiguousarray(grid.solo_knob if len(grid.solo_knob) else np.zeros((1, 4))),
    }
    s = nat.CsGrid()
    s.n_grid = grid.n_grid
    s.knob1 = nat.ptr(keep["knob1"])
    s.knob2 = nat.ptr(keep["knob2"])
    s.mask = nat.ptr(keep["mask"], nat.c_uint32_p)
    s.n_budgets = grid.n_budgets
    for l in range(grid.n_budgets):
        s.n_configs[l] = grid.n_configs[l]
    for l, off in enumerate(grid.solo_offsets):
        s.solo_offsets[l] = off
    s.solo_knob = nat.ptr(keep["solo"])
    return s, keep


def _pinned(shape, dtype):
    t = torch.empty(shape, dtype=dtype, pin_memory=True)
    return t, t.numpy()


class HostGraphCall:
    """Reusable cs_build_graph_host invocation for `n` apps over `grid`."""

    def __init__(self, weights, grid: KnobGrid, n: int, rel_eps: float = DEFAULT_REL_EPS,
                 with_records: bool = True, device=None, pair_weight: bool = True):
        """with_records: also copy back the per-pair decision records (best
        config index, its CoRunTime, the co-run flag -- what a Schedule needs);
        pair_weight: plus the per-pair winning time (it duplicates the matrix)."""
        self.lib = nat.sweep_lib()
        self.device = require_cuda(device)
        grid.check_nonempty()
        self.n, self.grid, self.rel_eps = n, grid, rel_eps
        self.net = NetworkABI(weights)
        self.cgrid, self._keep = _host_grid(grid)
        L, P = grid.n_budgets, n * (n - 1) // 2
        self.ws_bytes = self.lib.cs_build_graph_workspace_bytes(n, ctypes.byref(self.cgrid))
        if not self.ws_bytes:
            raise ValueError("cs_build_graph_workspace_bytes rejected the problem")
        self.ws = torch.empty(self.ws_bytes + 256, dtype=torch.uint8, device=self.device)
        self.ws_ptr = (self.ws.data_ptr() + 255) & ~255
        # persistent workspace: grid / network / zeroed matrix stay resident and
        # repeated calls replay as a CUDA graph; released in close()
        nat.check(self.lib.cs_workspace_retain(self.ws_ptr, self.ws_bytes), "cs_workspace_retain")
        self._retained = True
        self._t_feat, self.h_features = _pinned((n, 18), torch.float64)
        self._t_bt, self.h_base_time = _pinned((n,), torch.float64)
        self._t_w, self.h_weights = _pinned((L, n, n), torch.float64)
        self.with_records = with_records
        if with_records:
            self._t_idx, self.h_idx = _pinned((L, P), torch.int32)
            self._t_ct, self.h_ct = _pinned((L, P), torch.float64)
            self._t_ch, self.h_ch = _pinned((L, P), torch.uint8)
            if pair_weight:
                self._t_pw, self.h_pw = _pinned((L, P), torch.float64)
            else:
                self.h_pw = None
            self.pairs = nat.CsPairOut(nat.ptr(self.h_idx, nat.c_int32_p), nat.ptr(self.h_ct),
                                       nat.ptr(self.h_ch, nat.c_uint8_p),
                                       nat.ptr(self.h_pw) if pair_weight else None)
        else:
            self.pairs = nat.CsPairOut()
        self._t_st, self.h_solo_time = _pinned((L, n), torch.float64)
        self._t_ss, self.h_solo_split = _pinned((L, n), torch.int32)
        self._t_sc, self.h_solo_clamps = _pinned((L, n), torch.int32)
        self.solo = nat.CsSoloOut(nat.ptr(self.h_solo_time), nat.ptr(self.h_solo_split, nat.c_int32_p),
                                  nat.ptr(self.h_solo_clamps, nat.c_int32_p))
        # pinned like every other buffer: the call's graph reads / writes all
        # of them with zero-copy kernels or async copies
        self._t_cl, h_cl = _pinned((L,), torch.int64)
        self.h_clamps = h_cl.view(np.uint64)
        self.h_clamps[...] = 0
        # a private non-default stream: the call is synchronous (it returns
        # after its results sit in the host buffers), and the library captures
        # a repeated call on a non-default stream into a CUDA graph
        self._stream_obj = torch.cuda.Stream(self.device)
        self._net_obj = self.net
        self._args = (self.net.ref(), ctypes.byref(self.cgrid), nat.ptr(self.h_features),
                      nat.ptr(self.h_base_time), self.n, self.rel_eps, self.ws_ptr, self.ws_bytes,
                      nat.ptr(self.h_weights), self.pairs, self.solo,
                      self.h_clamps.ctypes.data_as(nat.c_ull_p), self._stream_obj.cuda_stream)

    def close(self) -> None:
        """Drop the workspace's library-side state (before its memory goes)."""
        if getattr(self, "_retained", False):
            self._retained = False
            self.lib.cs_workspace_release(self.ws_ptr)

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass

    def bytes_per_call(self) -> tuple:
        """(H2D bytes, D2H bytes) moved by one repeated call (the grid and the
        network stay in the workspace after the first call)."""
        h2d = self.h_features.nbytes + self.h_base_time.nbytes
        d2h = self.h_weights.nbytes + self.h_solo_time.nbytes + self.h_solo_split.nbytes + \
            self.h_solo_clamps.nbytes + self.h_clamps.nbytes
        if self.with_records:
            d2h += self.h_idx.nbytes + self.h_ct.nbytes + self.h_ch.nbytes
            if self.h_pw is not None:
                d2h += self.h_pw.nbytes
        return h2d, d2h

    def __call__(self, features=None, base_time=None) -> dict:
        if features is not None:
            self.h_features[...] = features
        if base_time is not None:
            self.h_base_time[...] = base_time
        if self.net is not self._net_obj:
            self._net_obj = self.net
            self._args = (self.net.ref(),) + self._args[1:]
        rc = self.lib.cs_build_graph_host(*self._args)
        nat.check(rc, "cs_build_graph_host")
        out = {"weights": self.h_weights, "solo_time": self.h_solo_time,
               "solo_split": self.h_solo_split, "solo_clamps": self.h_solo_clamps,
               "clamps": self.h_clamps}
        if self.with_records:
            out.update(corun_grid_index=self.h_idx, corun_time=self.h_ct,
                       corun_chosen=self.h_ch.view(bool))
            if self.h_pw is not None:
                out["weight"] = self.h_pw
        return out


def build_graph_host(weights, grid: KnobGrid, features, base_time, **kw) -> dict:
    call = HostGraphCall(weights, grid, len(base_time), **kw)
    try:
        out = call(features, base_time)
        return {k: np.array(v) for k, v in out.items()}
    finally:
        call.close()
