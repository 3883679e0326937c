"""Warm per-kernel latency of the small pipeline kernels (CUDA events, no L2 flush)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2405_03831_b200 import _native as nat, core, fnn, synth
from paper_2405_03831_b200.device import SweepPlan, to_device_inputs, _dptr
from paper_2405_03831_b200.grid import KnobGrid

w = fnn.load_weights(os.path.join(ROOT, "tests/golden/weights.json"))
for n in (256, 4096):
    grid = KnobGrid([core.default_space(400.0)])
    F, T = synth.workload_arrays(0, synth.mixed_archetypes(n))
    plan = SweepPlan(w, grid, n)
    df, db = to_device_inputs(F, T, plan.device)
    plan.launch(df, db)
    torch.cuda.synchronize()
    lib = plan.lib
    st_of = lambda: torch.cuda.current_stream().cuda_stream
    tref = ctypes.byref(plan.tables)

    def t_of(fn, reps=50):
        # `reps` calls captured into one CUDA graph: device time per call,
        # without the host-side ctypes/launch cost
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            fn()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3

    prep = lambda: lib.cs_prepare(plan.net.ref(), _dptr(df), _dptr(db), n, plan.dgrid.ref(), tref, plan.solo_out, _dptr(plan.counters), _dptr(plan.clamps), st_of())
    tabl = lambda: lib.cs_build_tables(plan.net.ref(), _dptr(df), n, plan.dgrid.ref(), tref, st_of())
    solo = lambda: lib.cs_solo(plan.net.ref(), tref, plan.dgrid.ref(), _dptr(db), plan.solo_out, st_of())
    res = lambda: lib.cs_resolve_fused(plan.net.ref(), tref, plan.dgrid.ref(), _dptr(db), _dptr(plan.solo_time), _dptr(plan.solo_clamps), 0, plan.P, plan.pair_out, _dptr(plan.queue), _dptr(plan.counters), _dptr(plan.clamps), None, st_of())
    full = lambda: plan.launch(df, db)
    c = plan.read_counters()
    print(f"n={n} queue={c.queue_len}: prepare {t_of(prep):.1f} us, tables-only {t_of(tabl):.1f} us, "
          f"solo-only {t_of(solo):.1f} us, resolve {t_of(res):.1f} us, full launch() {t_of(full):.1f} us")
    z = torch.zeros(2, dtype=torch.int32, device=plan.device)
    res0 = lambda: lib.cs_resolve_fused(plan.net.ref(), tref, plan.dgrid.ref(), _dptr(db), _dptr(plan.solo_time), _dptr(plan.solo_clamps), 0, plan.P, plan.pair_out, _dptr(plan.queue), _dptr(z), _dptr(plan.clamps), None, st_of())
    print(f"   resolve with empty queue {t_of(res0):.1f} us")
