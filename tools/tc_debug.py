"""Debug driver: one small sweep with a watchdog; TRACE=1 uses the CS_TC_TRACE build and
prints each thread's last progress marker (stage << 0 | k << 8) read from host-mapped memory."""
import faulthandler, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np, torch
from paper_2405_03831_b200 import _native, core, fnn, synth
TRACE = os.environ.get("TRACE") == "1"
if TRACE:
    _native.SWEEP_LIB = os.path.join(ROOT, "tools", "libcosched_b200_trace.so")
    buf = torch.zeros(148 * 512, dtype=torch.int32, pin_memory=True)
    os.environ["CS_TC_TRACE_PTR"] = str(buf.data_ptr())
else:
    faulthandler.dump_traceback_later(float(os.environ.get("WATCHDOG", "40")), exit=True)
from paper_2405_03831_b200.device import SweepPlan, to_device_inputs
from paper_2405_03831_b200.grid import KnobGrid
w = fnn.load_weights(os.path.join(ROOT, "tests/golden/weights.json"))
n = int(os.environ.get("N", "20"))
F, T = synth.workload_arrays(0, synth.mixed_archetypes(n))
grid = KnobGrid([core.default_space(400.0)])
plan = SweepPlan(w, grid, n, with_matrix=False, kernel=os.environ.get("KERNEL", "tcgen05"))
df, db = to_device_inputs(F, T, plan.device)
torch.cuda.synchronize()
print("launching", flush=True)
plan.launch(df, db)
if TRACE:
    time.sleep(4)
    tr = buf.numpy().copy()
    nct = (((n * (n - 1) // 2) + 63) // 64 + 3) // 4
    for cta in range(min(nct, 2)):
        v = tr[cta * 512:(cta + 1) * 512]
        for warp in range(16):
            ww = v[warp * 32:(warp + 1) * 32]
            print(f"cta {cta} warp {warp:2d}: stages", sorted(set((x & 255, x >> 8) for x in ww.tolist()))[:6], flush=True)
    os._exit(0)
print("launched; syncing", flush=True)
torch.cuda.synchronize()
print("synced", flush=True)
c = plan.read_counters()
print("counters", c, flush=True)
import oracle
ref = oracle.sweep(w, F, T, grid)
P = plan.P
idx = plan.corun_grid_index[:, :P].cpu().numpy()
print("idx equal:", np.array_equal(idx, ref["corun_grid_index"]), "mismatches", int((idx != ref["corun_grid_index"]).sum()))
print("time equal:", np.array_equal(plan.corun_time[:, :P].cpu().numpy(), ref["corun_time"]))
