"""Critical-path share of each launch of a bench step: the same CUDA-graph step
as bench.py (L2 flushed before each replay, PDL edges intact -- no events
between the launches), timed whole and with one launch left out.  Results of
the partial steps are wrong by construction; only their times are read."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2405_03831_b200 import _native as nat, core, fnn, synth
from paper_2405_03831_b200.device import SweepPlan, to_device_inputs, _dptr
from paper_2405_03831_b200.grid import KnobGrid
import ctypes

w = fnn.load_weights(os.path.join(ROOT, "tests/golden/weights.json"))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
grid = KnobGrid([core.default_space(400.0)])
F, T = synth.workload_arrays(0, synth.mixed_archetypes(n))
plan = SweepPlan(w, grid, n)
df, db = to_device_inputs(F, T, plan.device)
lib = plan.lib
tref = ctypes.byref(plan.tables)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=plan.device)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def step(parts):
    st = torch.cuda.current_stream().cuda_stream
    if "prepare" in parts:
        nat.check(lib.cs_prepare(plan.net.ref(), _dptr(df), _dptr(db), n, plan.dgrid.ref(), tref,
                                 plan.solo_out, _dptr(plan.counters), _dptr(plan.clamps), st), "prep")
    if "screen" in parts:
        nat.check(lib.cs_pair_screen_fused(plan.net.ref(), tref, plan.dgrid.ref(), _dptr(db),
                  _dptr(plan.solo_time), _dptr(plan.solo_clamps), 0, plan.P, plan.rel_eps,
                  plan.pair_out, _dptr(plan.queue), _dptr(plan.counters), _dptr(plan.clamps),
                  _dptr(plan.matrix), plan.kernel_kind, st), "screen")
    if "resolve" in parts:
        nat.check(lib.cs_resolve_fused(plan.net.ref(), tref, plan.dgrid.ref(), _dptr(db),
                  _dptr(plan.solo_time), _dptr(plan.solo_clamps), 0, plan.P, plan.pair_out,
                  _dptr(plan.queue), _dptr(plan.counters), _dptr(plan.clamps), _dptr(plan.matrix), st),
                  "resolve")


def timed(parts, reps=200):
    side = torch.cuda.Stream(); side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        step(("prepare", "screen", "resolve"))     # valid tables / queue for partial steps
    torch.cuda.current_stream().wait_stream(side); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step(parts)
    ts = []
    for k in range(reps):
        flush.zero_()
        e0.record(); g.replay(); e1.record()
        torch.cuda.synchronize()
        if k >= 20:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


for parts in (("prepare", "screen", "resolve"), ("screen", "resolve"), ("prepare", "screen"),
              ("screen",), ("prepare",), ("resolve",)):
    print(f"n={n} {'+'.join(parts)}: {timed(parts):.1f} us")
