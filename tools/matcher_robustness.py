"""Host matching time across sweep graphs (workload seeds x budgets) at one N,
on the GPU box's host: build_graph on the GPU, then the native matcher.
Writes one JSON line per graph."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2405_03831_b200 import core, fnn, matcher, scheduler, synth

w = fnn.load_weights(os.path.join(ROOT, "tests", "golden", "weights.json"))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
for seed, watts in [(0, 400.0), (1, 400.0), (2, 400.0), (3, 400.0), (0, 350.0), (5, 375.0)]:
    jobs = synth.generate_jobs(seed, synth.mixed_archetypes(n))
    inp = scheduler.SchedulerInput(tuple(jobs), core.default_space(watts),
                                   core.SchedulingParams(window=n), w)
    g = scheduler.build_graph(inp)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m = matcher.min_weight_perfect_matching(g)
    t1 = time.perf_counter()
    print(json.dumps({"n": n, "seed": seed, "watts": watts, "matching_s": round(t1 - t0, 3),
                      "weight": matcher.matching_weight(g, m)}), flush=True)
