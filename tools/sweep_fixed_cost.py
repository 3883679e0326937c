"""Fixed vs per-config cost of the three launches of one sweep: times each
launch (warm, CUDA graph of 50 calls) on grids of different sizes and fits
t = a + b * G per launch.  The intercept is the launch's fixed cost."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2405_03831_b200 import _native as nat, core, fnn, synth
from paper_2405_03831_b200.device import SweepPlan, to_device_inputs, _dptr
from paper_2405_03831_b200.grid import KnobGrid

w = fnn.load_weights(os.path.join(ROOT, "tests/golden/weights.json"))
base = core.default_space(400.0)
cp = base.corun_cpu_partitions
spaces = [core.ConfigSpace(cpu_partitions=tuple(p for p in base.cpu_partitions if min(p) == 0) + cp[:k])
          for k in range(1, len(cp) + 1)]


def t_of(fn, reps=50):
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


for n in [int(x) for x in (sys.argv[1:] or ["256", "1024"])]:
    F, T = synth.workload_arrays(0, synth.mixed_archetypes(n))
    rows = []
    for sp in spaces:
        grid = KnobGrid([sp])
        plan = SweepPlan(w, grid, n, kernel=os.environ.get("KERNEL", "tcgen05"))
        df, db = to_device_inputs(F, T, plan.device)
        plan.launch(df, db)
        torch.cuda.synchronize()
        lib, tref = plan.lib, ctypes.byref(plan.tables)
        st = lambda: torch.cuda.current_stream().cuda_stream
        prep = lambda: lib.cs_prepare(plan.net.ref(), _dptr(df), _dptr(db), n, plan.dgrid.ref(), tref,
                                      plan.solo_out, _dptr(plan.counters), _dptr(plan.clamps), st())
        z = torch.zeros(nat.COUNTERS_BYTES // 4, dtype=torch.int32, device=plan.device)

        def screen():
            z.zero_()
            lib.cs_pair_screen_fused(plan.net.ref(), tref, plan.dgrid.ref(), _dptr(db),
                                     _dptr(plan.solo_time), _dptr(plan.solo_clamps), 0, plan.P,
                                     plan.rel_eps, plan.pair_out, _dptr(plan.queue), _dptr(z),
                                     _dptr(plan.clamps), _dptr(plan.matrix), plan.kernel_kind, st())
        res = lambda: lib.cs_resolve_fused(plan.net.ref(), tref, plan.dgrid.ref(), _dptr(db),
                                           _dptr(plan.solo_time), _dptr(plan.solo_clamps), 0, plan.P,
                                           plan.pair_out, _dptr(plan.queue), _dptr(plan.counters),
                                           _dptr(plan.clamps), _dptr(plan.matrix), st())
        zero = lambda: z.zero_()
        full = lambda: plan.launch(df, db)
        q = plan.read_counters().queue_len
        r = (grid.n_grid, q, t_of(prep), t_of(screen) - t_of(zero), t_of(res), t_of(full))
        rows.append(r)
        print(f"n={n} G={r[0]:3d} queue={r[1]:4d}: prepare {r[2]:.1f} us, screen {r[3]:.1f} us, "
              f"resolve {r[4]:.1f} us, launch() {r[5]:.1f} us", flush=True)
    a = np.array(rows, dtype=np.float64)
    for k, name in ((2, "prepare"), (3, "screen"), (5, "launch()")):
        b, c = np.polyfit(a[:, 0], a[:, k], 1)
        print(f"n={n} {name}: {c:.1f} us fixed + {b * 1e3:.1f} ns/config")
