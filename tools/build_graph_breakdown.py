import sys, time, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2405_03831_b200 import core, fnn, synth, scheduler, sweep as sw
from paper_2405_03831_b200.matcher import PairGraph
w = fnn.load_weights("/root/repo/tests/golden/weights.json")
n = 4096
jobs = synth.generate_jobs(0, synth.mixed_archetypes(n))
space = core.default_space(400.0)
inp = scheduler.SchedulerInput(tuple(jobs), space, core.SchedulingParams(window=n), w)
scheduler.build_graph(inp)
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter()
    feats, bt = sw._inputs(jobs)
    t1 = time.perf_counter()
    plan = sw.plan_for(w, (space,), n, 0, None, True)
    t2 = time.perf_counter()
    with plan.lock:
        d_f, d_b = sw.to_device_inputs(feats, bt, plan.device)
        plan.launch(d_f, d_b, rel_eps=plan.rel_eps)
        c = plan.read_counters()
        t3 = time.perf_counter()
        P = plan.P
        a = plan.corun_grid_index[:, :P].cpu().numpy(); t4 = time.perf_counter()
        b = plan.corun_time[:, :P].cpu().numpy(); t5 = time.perf_counter()
        ch = plan.corun_chosen[:, :P].cpu().numpy().astype(bool); t6 = time.perf_counter()
        wt = plan.weight[:, :P].cpu().numpy(); t7 = time.perf_counter()
        m = plan.matrix.cpu().numpy(); t8 = time.perf_counter()
    print(f"inputs {1e3*(t1-t0):.1f} plan {1e3*(t2-t1):.1f} launch+sync {1e3*(t3-t2):.1f} idx {1e3*(t4-t3):.1f} ct {1e3*(t5-t4):.1f} ch {1e3*(t6-t5):.1f} w {1e3*(t7-t6):.1f} matrix {1e3*(t8-t7):.1f} ms")
    t0 = time.perf_counter(); g = scheduler.build_graph(inp); t1 = time.perf_counter()
    print(f"build_graph total {1e3*(t1-t0):.1f} ms")
