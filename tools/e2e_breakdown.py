"""Where the host-ABI (cs_build_graph_host) step time goes at one N: wall time
per call for variants of the same call, against the device-only graph step."""
import ctypes, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2405_03831_b200 import _native as nat, core, fnn, synth
from paper_2405_03831_b200.grid import KnobGrid
from paper_2405_03831_b200.host_abi import HostGraphCall, _pinned

w = fnn.load_weights(os.path.join(ROOT, "tests/golden/weights.json"))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
grid = KnobGrid([core.default_space(400.0)])
F, T = synth.workload_arrays(0, synth.mixed_archetypes(n))


def wall(fn, k=300):
    for _ in range(5):
        fn()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e6 * float(np.median(ts)), 1e6 * float(np.mean(ts))


call = HostGraphCall(w, grid, n, with_records=False)
call.h_features[...] = F
call.h_base_time[...] = T
print(f"n={n} call() as bench.py: median {wall(call)[0]:.1f} us, mean {wall(call)[1]:.1f} us", flush=True)
lib = call.lib
st = torch.cuda.current_stream(call.device).cuda_stream
args = [call.net.ref(), ctypes.byref(call.cgrid), nat.ptr(call.h_features), nat.ptr(call.h_base_time),
        call.n, call.rel_eps, call.ws_ptr, call.ws_bytes, nat.ptr(call.h_weights), call.pairs, call.solo,
        call.h_clamps.ctypes.data_as(nat.c_ull_p), st]
raw = lambda: lib.cs_build_graph_host(*args)
print(f"  raw ctypes call, same args: median {wall(raw)[0]:.1f} us", flush=True)
_t, pc = _pinned((1,), torch.int64)
args_p = list(args); args_p[11] = pc.ctypes.data_as(nat.c_ull_p)
rawp = lambda: lib.cs_build_graph_host(*args_p)
print(f"  raw, pinned clamps buffer: median {wall(rawp)[0]:.1f} us", flush=True)
args_nw = list(args_p); args_nw[8] = None
rawnw = lambda: lib.cs_build_graph_host(*args_nw)
print(f"  raw, pinned clamps, no weight-matrix D2H: median {wall(rawnw)[0]:.1f} us", flush=True)
args_min = list(args_nw); args_min[10] = nat.CsSoloOut()
rawmin = lambda: lib.cs_build_graph_host(*args_min)
print(f"  raw, no D2H at all but counters: median {wall(rawmin)[0]:.1f} us", flush=True)
# device-only reference: the same work as a plain stream-ordered launch + sync
torch.cuda.synchronize()
from paper_2405_03831_b200.device import SweepPlan, to_device_inputs
plan = SweepPlan(w, grid, n, with_matrix=True)
d_f, d_b = to_device_inputs(F, T, plan.device)
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    plan.launch(d_f, d_b)
torch.cuda.current_stream().wait_stream(side)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    plan.launch(d_f, d_b)
def dev_only():
    g.replay()
    torch.cuda.synchronize()
print(f"  device-only graph replay + sync (no copies): median {wall(dev_only)[0]:.1f} us", flush=True)
e = torch.cuda.CUDAGraph()
tiny = torch.zeros(1, device=plan.device)
with torch.cuda.graph(e):
    tiny.add_(1)
def empty():
    e.replay()
    torch.cuda.synchronize()
print(f"  one-kernel graph replay + sync: median {wall(empty)[0]:.1f} us", flush=True)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
acc = []
for _ in range(200):
    ev0.record(); g.replay(); ev1.record(); ev1.synchronize(); acc.append(ev0.elapsed_time(ev1) * 1e3)
print(f"  device-only graph, event-timed: median {float(np.median(acc)):.1f} us", flush=True)
