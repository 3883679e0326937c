#!/bin/bash
# DEBUG: rebuild libcosched_b200.so with the screen's clock trace
# (-DCS_TC_CLOCKS) and print the per-config timeline of block 0's first items
# at N=4,096 (never commit the resulting .so).  Usage: bash tools/clock_trace.sh
ROOT=$(cd "$(dirname "$0")/.." && pwd)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DCS_TC_CLOCKS \
  -Xcompiler -fPIC,-O3 -shared -cudart static -I$ROOT/include $ROOT/paper_2405_03831_b200/csrc/sweep.cu \
  -o $ROOT/paper_2405_03831_b200/libcosched_b200.so || exit 1
python - <<'PY'
import ctypes, os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
from paper_2405_03831_b200 import _native as nat, core, fnn, synth
from paper_2405_03831_b200.device import SweepPlan, to_device_inputs
from paper_2405_03831_b200.grid import KnobGrid
w = fnn.load_weights("tests/golden/weights.json")
n = 4096
grid = KnobGrid([core.default_space(400.0)])
F, T = synth.workload_arrays(0, synth.mixed_archetypes(n))
plan = SweepPlan(w, grid, n)
df, db = to_device_inputs(F, T, plan.device)
for _ in range(3): plan.launch(df, db)
torch.cuda.synchronize()
lib = ctypes.CDLL(nat.SWEEP_LIB)
N = 4 * 4 * 4 * 32 + 4 * 2 * 32
buf = (ctypes.c_ulonglong * N)()
assert lib.cs_debug_clocks(buf, N) == 0
a = np.array(buf, dtype=np.int64)
comp = a[:4 * 4 * 4 * 32].reshape(4, 4, 4, 32)      # [group][warp][event][config]
iss = a[4 * 4 * 4 * 32:].reshape(4, 2, 32)          # [group][event][config]
t0 = comp[0, 0, 0, 0]
print("config | g0: build start/arrive (w0..3 max) | issuer wake, issued | epi wait start, end (w0) | per-config period")
for c in range(1, 31):
    bs = comp[0, :, 0, c] - t0; ar = comp[0, :, 1, c] - t0
    wk, isd = iss[0, 0, c] - t0, iss[0, 1, c] - t0
    ws, we = comp[0, 0, 2, c] - t0, comp[0, 0, 3, c] - t0
    per = comp[0, 0, 0, c + 1] - comp[0, 0, 0, c] if c < 31 else 0
    print(f"{c:3d} | {bs.min():7d} {ar.max():7d} (arrive spread {ar.max()-ar.min():4d}) | {wk:7d} {isd:7d} | {ws:7d} {we:7d} (wait {we-ws:4d}) | {per}")
# summary over groups
for g in range(4):
    arr = comp[g, :, 1, 2:30].max(axis=0); wk = iss[g, 0, 2:30]; isd = iss[g, 1, 2:30]
    ws = comp[g, :, 2, 2:30]; we = comp[g, :, 3, 2:30]
    print(f"group {g}: last-arrive -> issuer wake {np.median(wk - arr):.0f} cyc, wake -> issued {np.median(isd - wk):.0f}, "
          f"issued -> epilogue wait end (w0) {np.median(we[0] - isd):.0f}, epilogue wait {np.median(we - ws):.0f}, "
          f"period {np.median(np.diff(comp[g, 0, 0, 2:31])):.0f}")
PY
