"""Where a bench step's time goes: CUDA events between the three launches of one
sweep, each step preceded by the same 256 MiB L2 flush as bench.py."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2405_03831_b200 import _native as nat, core, fnn, synth
from paper_2405_03831_b200.device import SweepPlan, to_device_inputs, _dptr
from paper_2405_03831_b200.grid import KnobGrid

w = fnn.load_weights(os.path.join(ROOT, "tests/golden/weights.json"))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
grid = KnobGrid([core.default_space(400.0)])
F, T = synth.workload_arrays(0, synth.mixed_archetypes(n))
plan = SweepPlan(w, grid, n)
df, db = to_device_inputs(F, T, plan.device)
lib = plan.lib
tref = ctypes.byref(plan.tables)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=plan.device)
ev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(4)]

def step():
    st = torch.cuda.current_stream().cuda_stream
    plan.counters.zero_(); plan.clamps.zero_()
    ev[0].record()
    nat.check(lib.cs_prepare(plan.net.ref(), _dptr(df), _dptr(db), n, plan.dgrid.ref(), tref,
                             plan.solo_out, _dptr(plan.counters), _dptr(plan.clamps), st), "prep")
    ev[1].record()
    nat.check(lib.cs_pair_screen_fused(plan.net.ref(), tref, plan.dgrid.ref(), _dptr(db),
              _dptr(plan.solo_time), _dptr(plan.solo_clamps), 0, plan.P, plan.rel_eps,
              plan.pair_out, _dptr(plan.queue), _dptr(plan.counters), _dptr(plan.clamps),
              _dptr(plan.matrix), plan.kernel_kind, st), "screen")
    ev[2].record()
    nat.check(lib.cs_resolve_fused(plan.net.ref(), tref, plan.dgrid.ref(), _dptr(db),
              _dptr(plan.solo_time), _dptr(plan.solo_clamps), 0, plan.P, plan.pair_out,
              _dptr(plan.queue), _dptr(plan.counters), _dptr(plan.clamps), _dptr(plan.matrix), st),
              "resolve")
    ev[3].record()

side = torch.cuda.Stream(); side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    step()
torch.cuda.current_stream().wait_stream(side); torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
for flushed in (True, False):
    acc = np.zeros(3)
    for k in range(60):
        if flushed:
            flush.zero_()
        g.replay()
        torch.cuda.synchronize()
        if k >= 10:
            acc += [ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])]
    acc = acc / 50 * 1e3
    print(f"n={n} {'L2 flushed' if flushed else 'warm'}: prepare {acc[0]:.1f} us, screen {acc[1]:.1f} us, "
          f"resolve {acc[2]:.1f} us, total {acc.sum():.1f} us")
