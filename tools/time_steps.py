"""Device time of one full sweep step (k_tables -> screen -> k_resolve, one CUDA
graph of 50 steps, no L2 flush) at several N, for the default screen instance
and any COSCHED_TC_KIND given on the command line: python tools/time_steps.py [KIND ...]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2405_03831_b200 import core, fnn, synth
from paper_2405_03831_b200.device import SweepPlan, to_device_inputs
from paper_2405_03831_b200.grid import KnobGrid

w = fnn.load_weights(os.path.join(ROOT, "tests/golden/weights.json"))
kinds = [None] + sys.argv[1:]
for n in (20, 64, 128, 256, 512):
    grid = KnobGrid([core.default_space(400.0)])
    F, T = synth.workload_arrays(0, synth.mixed_archetypes(n))
    row = []
    for kind in kinds:
        if kind: os.environ["COSCHED_TC_KIND"] = kind
        else: os.environ.pop("COSCHED_TC_KIND", None)
        plan = SweepPlan(w, grid, n)
        df, db = to_device_inputs(F, T, plan.device)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(3): plan.launch(df, db)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                for _ in range(50): plan.launch(df, db)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g.replay(); torch.cuda.synchronize()
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        row.append(f"{kind or 'default'} {1e3 * e0.elapsed_time(e1) / 50:.1f} us")
    print(f"n={n}: " + " | ".join(row), flush=True)
