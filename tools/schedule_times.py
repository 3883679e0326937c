"""End-to-end schedule time vs N (BASELINE.json's second metric): loaded profiles +
weights -> GPU sweep -> D2H -> native host matching -> emitted Schedule, via the
drop-in API (scheduler.build_graph + matcher + emit_schedule).  Writes one JSON line."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2405_03831_b200 import core, fnn, matcher, scheduler, synth

w = fnn.load_weights(os.path.join(ROOT, "tests", "golden", "weights.json"))
out = {}
for n in [int(x) for x in (sys.argv[1:] or ["20", "256", "1024", "4096"])]:
    jobs = synth.generate_jobs(0, synth.mixed_archetypes(n))
    inp = scheduler.SchedulerInput(tuple(jobs), core.default_space(400.0),
                                   core.SchedulingParams(window=n), w)
    scheduler.build_graph(inp)                       # warm the plan cache / GPU
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = scheduler.build_graph(inp)
    t1 = time.perf_counter()
    m = matcher.min_weight_perfect_matching(g)
    t2 = time.perf_counter()
    sched = scheduler.emit_schedule(inp, g, m)
    t3 = time.perf_counter()
    out[n] = {"total_s": t3 - t0, "build_graph_s": t1 - t0, "matching_s": t2 - t1,
              "emit_s": t3 - t2, "sets": len(sched.job_sets),
              "matching_weight": matcher.matching_weight(g, m)}
    print(json.dumps({n: out[n]}), flush=True)
print(json.dumps({"schedule_time_vs_n": out}))
