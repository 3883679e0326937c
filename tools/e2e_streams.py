"""Host-ABI call wall time on the legacy default stream vs a dedicated stream
(where the library captures and replays the call as a CUDA graph)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2405_03831_b200 import core, fnn, synth
from paper_2405_03831_b200.grid import KnobGrid
from paper_2405_03831_b200.host_abi import HostGraphCall

w = fnn.load_weights(os.path.join(ROOT, "tests/golden/weights.json"))
for n in (int(x) for x in (sys.argv[1:] or ["20", "256"])):
    grid = KnobGrid([core.default_space(400.0)])
    F, T = synth.workload_arrays(0, synth.mixed_archetypes(n))
    for name, stream in (("default", None), ("side", torch.cuda.Stream())):
        ctx = torch.cuda.stream(stream) if stream is not None else torch.cuda.stream(torch.cuda.current_stream())
        with ctx:
            call = HostGraphCall(w, grid, n, with_records=True, pair_weight=False)
            call.h_features[...] = F; call.h_base_time[...] = T
            for _ in range(10): call()
            ts = []
            for _ in range(300):
                t0 = time.perf_counter(); call(); ts.append(time.perf_counter() - t0)
            call.close()
        print(f"n={n} {name}: median {1e6*np.median(ts):.1f} us  p10 {1e6*np.percentile(ts,10):.1f} us", flush=True)
