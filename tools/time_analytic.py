"""Timing of the analytic-oracle sweep (cs_analytic_sweep) at N=4,096."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2405_03831_b200 import analytic, core, synth
jobs = synth.generate_jobs(0, synth.mixed_archetypes(4096))
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = analytic.analytic_sweep(analytic.OracleParams(), jobs, core.default_space(400.0), with_matrix=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"analytic sweep n=4096 (incl. host tables + copies): {t1 - t0:.3f} s")
