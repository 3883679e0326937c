"""Generate the golden fixtures by running the UNMODIFIED reference package.

This script is the only place that imports the reference (``cosched`` from
``/root/reference/pkg/src``).  It runs in the dev container, never on the GPU
box; its outputs are small committed fixtures under ``tests/golden/`` that the
parity tests (CPU and GPU) read.  Re-run with::

    python tests/golden/make_golden.py            # all stages
    python tests/golden/make_golden.py weights    # one stage

Stages and what they pin (reference file:line):

* ``weights``   -- ``weights.json``: the acceptance-recipe model
  (``test_acceptance.py:144-157``: ``generate_dataset(OracleParams(0.0),
  default_space(400), seed=0)`` + ``train(lr=0.002, batch=2, epochs=400,
  seed=2, val=0.05)``), written by the reference ``fnn.save_weights``
  (``fnn.py:311-324``).
* ``workloads`` -- ``workloads.json``: sha256 of the features/base-time
  arrays of ``simenv.generate_workload(seed, mixed_archetypes(N))``
  (``simenv.py:290-311``) so our own generator is pinned bit-for-bit.
* ``paper20``   -- ``paper20.json``: every pair of the 20-app workload through
  ``scheduler.build_graph`` (``scheduler.py:52-78``) at 400 W and 350 W, the
  reference schedule (``scheduler.py:81-107``) and the clamp counter.
* ``n256``      -- ``n256_400.npz``: the FULL 256-app graph (32,640 pairs) from
  ``hwopt.decide_pair`` (``hwopt.py:77-87``) in a process pool, plus the
  reference matching on it (``matcher.py:78-88``).
* ``samples``   -- ``samples.json``: seeded pair samples at N=4096 (400/350 W),
  N=1024 over the five-budget sweep, and N=4096 on the fine 6.25 W cap grid
  (``cosched.core.CPU_CAPS/GPU_CAPS`` monkeypatched, as SURVEY.md §8d says).
* ``matching``  -- ``matching.json``: reference ``min_weight_perfect_matching``
  and ``brute_force_matching`` on seeded random graphs.
* ``training``  -- ``training.json``: sha256 of ``simenv.dataset_to_csv`` of
  ``generate_dataset`` (simenv.py:393-469) for two (noise, seed, budget)
  settings; ``fnn.backward`` (fnn.py:174-210) gradients and losses on seeded
  batches; and a 20-epoch ``fnn.train`` (fnn.py:260-297) of the acceptance
  recipe (history + final weights).
"""

from __future__ import annotations

import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

sys.dont_write_bytecode = True
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

import numpy as np  # noqa: E402

from cosched import core, estimator, fnn, hwopt, matcher, scheduler, simenv  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
WEIGHTS = os.path.join(HERE, "weights.json")

FINE_CPU_CAPS = tuple(100.0 + 6.25 * k for k in range(25))
FINE_GPU_CAPS = tuple(150.0 + 6.25 * k for k in range(17))
BUDGET_LEVELS = (300.0, 325.0, 350.0, 375.0, 400.0)


def jobs_for(n, seed=0):
    return [s.job for s in simenv.generate_workload(seed, simenv.mixed_archetypes(n))]


def load_model():
    return fnn.load_weights(WEIGHTS)


def stage_weights():
    if os.path.exists(WEIGHTS):
        print("weights.json exists; skipping training")
        return
    t0 = time.time()
    dataset = simenv.generate_dataset(simenv.OracleParams(noise_sigma=0.0),
                                      core.default_space(400.0), seed=0)
    cfg = fnn.TrainingConfig(learning_rate=0.002, batch_size=2, epochs=400, seed=2,
                             validation_fraction=0.05)
    weights, hist = fnn.train(dataset.samples("train"), cfg, feature_bounds=dataset.bounds)
    fnn.save_weights(weights, WEIGHTS)
    print(f"trained in {time.time() - t0:.1f}s; final train mse {hist[-1].train_mse:.5f}")


def _sha(arr):
    return hashlib.sha256(np.ascontiguousarray(arr, dtype=np.float64).tobytes()).hexdigest()


def stage_workloads():
    out = {}
    for seed in (0, 1):
        for n in (20, 256, 1024, 4096):
            jobs = jobs_for(n, seed)
            feats = np.stack([j.features for j in jobs])
            bt = np.array([j.base_time for j in jobs])
            out[f"{seed}:{n}"] = {
                "features_sha256": _sha(feats), "base_time_sha256": _sha(bt),
                "first_job_id": jobs[0].job_id, "last_job_id": jobs[-1].job_id,
            }
    with open(os.path.join(HERE, "workloads.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


def _hc_tuple(hc):
    return [list(hc.cpu_partition), list(hc.gpu_partition), hc.cpu_cap, hc.gpu_cap]


def _decision_row(space, i, j, d):
    configs = core.enumerate_corun_configs(space)
    index = {hc: k for k, hc in enumerate(configs)}
    splits = core.enumerate_solo_splits(space)
    sidx = {s: k for k, s in enumerate(splits)}
    return {
        "i": i, "j": j,
        "corun_index": index[d.corun_config],
        "corun_config": _hc_tuple(d.corun_config),
        "corun_time_s": d.corun_time_s,
        "solo_split_index": [sidx[(hc.cpu_cap, hc.gpu_cap)] for hc in d.solo_configs],
        "solo_time_s": d.solo_time_s,
        "corun_chosen": bool(d.corun_chosen),
        "winning_time": d.winning_time,
    }


def stage_paper20():
    model = load_model()
    jobs = jobs_for(20)
    doc = {"n": 20, "seed": 0,
           "features": [list(map(float, j.features)) for j in jobs],
           "base_time": [j.base_time for j in jobs],
           "job_ids": [j.job_id for j in jobs],
           "spaces": {}}
    for p in (400.0, 350.0):
        space = core.default_space(p)
        inp = scheduler.SchedulerInput(tuple(jobs), space,
                                       core.SchedulingParams(window=20), model)
        estimator.clamp_stats.reset()
        graph = scheduler.build_graph(inp)
        clamps = estimator.clamp_stats.count
        sched = scheduler.schedule(inp)
        rows = [_decision_row(space, i, j, d) for (i, j), d in graph.decisions.items()]
        matched = matcher.min_weight_perfect_matching(graph)
        doc["spaces"][str(int(p))] = {
            "p_total": p,
            "n_corun_configs": len(core.enumerate_corun_configs(space)),
            "n_solo_splits": len(core.enumerate_solo_splits(space)),
            "clamp_count_build_graph": clamps,
            "pairs": rows,
            "matching": [list(m) for m in matched],
            "matching_weight": matcher.matching_weight(graph, matched),
            "schedule": {
                "job_sets": [[job.job_id for job in js.jobs] for js in sched.job_sets],
                "configs": [[_hc_tuple(hc) for hc in cfgs] for cfgs in sched.configs],
                "corun_flags": list(sched.corun_flags),
                "predicted_makespan": scheduler.predicted_makespan(sched, model, space),
            },
        }
    with open(os.path.join(HERE, "paper20.json"), "w") as fh:
        json.dump(doc, fh)


# --- process-pool helpers (fork start method; globals are inherited) -------
_G = {}


def _init_globals(n, seed, space, patch_fine):
    if patch_fine:
        core.CPU_CAPS = FINE_CPU_CAPS
        core.GPU_CAPS = FINE_GPU_CAPS
    _G["model"] = load_model()
    _G["jobs"] = jobs_for(n, seed)
    _G["space"] = space


def _work(pair):
    i, j = pair
    d = hwopt.decide_pair(_G["model"], _G["jobs"][i], _G["jobs"][j], _G["space"])
    return _decision_row(_G["space"], i, j, d)


def _run_pairs(n, seed, space, pairs, patch_fine=False, procs=8):
    ctx = mp.get_context("fork")
    with ctx.Pool(procs, initializer=_init_globals,
                  initargs=(n, seed, space, patch_fine)) as pool:
        return pool.map(_work, pairs, chunksize=64)


def stage_n256():
    n = 256
    space = core.default_space(400.0)
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
    t0 = time.time()
    rows = _run_pairs(n, 0, space, pairs)
    print(f"n256: {len(rows)} pairs in {time.time() - t0:.1f}s")
    P = len(rows)
    corun_index = np.array([r["corun_index"] for r in rows], dtype=np.int16)
    corun_time = np.array([r["corun_time_s"] for r in rows])
    solo_time = np.array([r["solo_time_s"] for r in rows])
    flag = np.array([r["corun_chosen"] for r in rows], dtype=np.uint8)
    win = np.array([r["winning_time"] for r in rows])
    # per-app solo split (identical across every pair the app is in)
    solo_split = np.full(n, -1, dtype=np.int8)
    for r in rows:
        for k, app in ((0, r["i"]), (1, r["j"])):
            if solo_split[app] < 0:
                solo_split[app] = r["solo_split_index"][k]
            assert solo_split[app] == r["solo_split_index"][k]
    W = np.zeros((n, n))
    for r in rows:
        W[r["i"], r["j"]] = W[r["j"], r["i"]] = r["winning_time"]
    t0 = time.time()
    graph = matcher.PairGraph(W)
    matched = matcher.min_weight_perfect_matching(graph)
    print(f"n256 matching in {time.time() - t0:.1f}s")
    np.savez_compressed(
        os.path.join(HERE, "n256_400.npz"),
        corun_index=corun_index, corun_time=corun_time, solo_time=solo_time,
        corun_chosen=flag, winning_time=win, solo_split=solo_split,
        matching=np.array(matched, dtype=np.int32),
        matching_weight=np.array(matcher.matching_weight(graph, matched)),
        n_pairs=np.array(P))


def _sample_pairs(n, k, rng):
    out = set()
    while len(out) < k:
        i, j = sorted(int(v) for v in rng.choice(n, size=2, replace=False))
        out.add((i, j))
    return sorted(out)


def stage_samples():
    rng = np.random.default_rng(1234)
    doc = {}
    t0 = time.time()
    # 4,096 apps at the default grid, two budgets
    for p, k in ((400.0, 400), (350.0, 150)):
        pairs = _sample_pairs(4096, k, rng)
        doc[f"n4096_{int(p)}"] = {"n": 4096, "seed": 0, "p_total": p, "grid": "default",
                                  "cap_sum_levels": list(core.DEFAULT_CAP_SUM_LEVELS),
                                  "pairs": _run_pairs(4096, 0, core.default_space(p), pairs)}
    print(f"n4096 samples {time.time() - t0:.1f}s")
    # 1,024 apps, five-budget sweep on levels (300..400 step 25)
    pairs = _sample_pairs(1024, 120, rng)
    for p in BUDGET_LEVELS:
        space = core.ConfigSpace(p_total=p, cap_sum_levels=BUDGET_LEVELS)
        doc[f"n1024_b{int(p)}"] = {"n": 1024, "seed": 0, "p_total": p, "grid": "default",
                                   "cap_sum_levels": list(BUDGET_LEVELS),
                                   "n_corun_configs": len(core.enumerate_corun_configs(space)),
                                   "n_solo_splits": len(core.enumerate_solo_splits(space)),
                                   "pairs": _run_pairs(1024, 0, space, pairs)}
    print(f"n1024 budget samples {time.time() - t0:.1f}s")
    # 4,096 apps, fine cap grid (6.25 W steps); the reference validates caps
    # against module constants, so they are patched inside the workers.
    pairs = _sample_pairs(4096, 120, rng)
    space = core.ConfigSpace(cpu_caps=FINE_CPU_CAPS, gpu_caps=FINE_GPU_CAPS, p_total=400.0)
    saved = (core.CPU_CAPS, core.GPU_CAPS)
    core.CPU_CAPS, core.GPU_CAPS = FINE_CPU_CAPS, FINE_GPU_CAPS
    try:
        n_cfg = len(core.enumerate_corun_configs(space))
        n_solo = len(core.enumerate_solo_splits(space))
        rows = _run_pairs(4096, 0, space, pairs, patch_fine=True)
    finally:
        core.CPU_CAPS, core.GPU_CAPS = saved
    doc["n4096_fine400"] = {"n": 4096, "seed": 0, "p_total": 400.0, "grid": "fine",
                            "cpu_caps": list(FINE_CPU_CAPS), "gpu_caps": list(FINE_GPU_CAPS),
                            "cap_sum_levels": list(core.DEFAULT_CAP_SUM_LEVELS),
                            "n_corun_configs": n_cfg, "n_solo_splits": n_solo, "pairs": rows}
    # a second seed at N=256 to guard against fixture overfitting
    pairs = _sample_pairs(256, 200, rng)
    doc["n256s1_400"] = {"n": 256, "seed": 1, "p_total": 400.0, "grid": "default",
                         "cap_sum_levels": list(core.DEFAULT_CAP_SUM_LEVELS),
                         "pairs": _run_pairs(256, 1, core.default_space(400.0), pairs)}
    print(f"all samples {time.time() - t0:.1f}s")
    with open(os.path.join(HERE, "samples.json"), "w") as fh:
        json.dump(doc, fh)


def random_graph(n, seed):
    """Seeded symmetric weights in [10, 100); regenerated identically by the tests."""
    rng = np.random.default_rng([seed, n, 7])
    upper = rng.uniform(10.0, 100.0, size=(n, n))
    w = np.triu(upper, 1)
    return w + w.T


def stage_matching():
    doc = []
    for n, seeds in ((2, (0,)), (4, (0, 1, 2)), (6, (0, 1, 2)), (8, (0, 1, 2, 3)),
                     (10, (0, 1)), (12, (0,)), (16, (0, 1)), (32, (0, 1)), (64, (0,)),
                     (128, (0,))):
        for seed in seeds:
            g = matcher.PairGraph(random_graph(n, seed))
            pairs = matcher.min_weight_perfect_matching(g)
            row = {"n": n, "seed": seed, "pairs": [list(p) for p in pairs],
                   "weight": matcher.matching_weight(g, pairs)}
            if n <= 10:
                bf_pairs, bf_w = matcher.brute_force_matching(g)
                row["brute_force_pairs"] = [list(p) for p in bf_pairs]
                row["brute_force_weight"] = bf_w
            doc.append(row)
    # integer-valued ties: many optimal matchings; the weight is what is pinned
    for n in (6, 8):
        rng = np.random.default_rng([n, 99])
        upper = rng.integers(1, 4, size=(n, n)).astype(float)
        w = np.triu(upper, 1)
        g = matcher.PairGraph(w + w.T)
        pairs = matcher.min_weight_perfect_matching(g)
        doc.append({"n": n, "seed": -1, "integer_ties": True, "weights": (w + w.T).tolist(),
                    "pairs": [list(p) for p in pairs],
                    "weight": matcher.matching_weight(g, pairs),
                    "brute_force_weight": matcher.brute_force_matching(g)[1]})
    with open(os.path.join(HERE, "matching.json"), "w") as fh:
        json.dump(doc, fh)


def stage_analytic():
    """The analytic oracle (simenv.OracleSlowdownModel, simenv.py:221-233) as the
    model of build_graph (scheduler.py:52-78): full graphs at N=24 (400 / 350 W,
    default params and a perturbed set) and the reference schedule, plus
    seeded decide_pair samples at N=512 on the five-budget levels."""
    doc = {"graphs": [], "samples": []}
    param_sets = {"default": simenv.OracleParams(),
                  "perturbed": simenv.OracleParams(cpu_scaling=0.5, gpu_mem_scaling=0.8,
                                                   compute_compute=0.4, memory_memory=0.1,
                                                   compute_memory=0.2, cpu_power_penalty=0.7)}
    for pname, params in param_sets.items():
        model = simenv.OracleSlowdownModel(params)
        for budget in (400.0, 350.0):
            n = 24
            jobs = jobs_for(n, 3)
            space = core.default_space(budget)
            inp = scheduler.SchedulerInput(tuple(jobs), space, core.SchedulingParams(window=n), model)
            estimator.clamp_stats.reset()
            g = scheduler.build_graph(inp)
            sched = scheduler.schedule(inp)
            doc["graphs"].append({
                "params": pname, "params_json": params.to_json(), "n": n, "seed": 3,
                "budget": budget,
                "pairs": [_decision_row(space, i, j, g.decisions[(i, j)])
                          for i in range(n) for j in range(i + 1, n)],
                "schedule_sets": [[job.job_id for job in js.jobs] for js in sched.job_sets],
                "schedule_flags": [bool(f) for f in sched.corun_flags],
            })
    rng = np.random.default_rng(99)
    n = 512
    jobs = jobs_for(n, 0)
    model = simenv.OracleSlowdownModel(simenv.OracleParams())
    for p_total in (325.0, 400.0):
        space = core.ConfigSpace(p_total=p_total, cap_sum_levels=BUDGET_LEVELS)
        rows = []
        for _ in range(150):
            i, j = sorted(rng.choice(n, size=2, replace=False).tolist())
            rows.append(_decision_row(space, i, j, hwopt.decide_pair(model, jobs[i], jobs[j], space)))
        doc["samples"].append({"n": n, "seed": 0, "p_total": p_total,
                               "cap_sum_levels": list(BUDGET_LEVELS), "pairs": rows})
    with open(os.path.join(HERE, "analytic.json"), "w") as fh:
        json.dump(doc, fh, indent=0, sort_keys=True)


def stage_training():
    import tempfile
    doc = {"datasets": [], "backward": [], "train": {}}
    for sigma, seed, budget in ((0.0, 0, 400.0), (0.05, 3, 350.0)):
        ds = simenv.generate_dataset(simenv.OracleParams(noise_sigma=sigma, seed=seed),
                                     core.default_space(budget))
        path = os.path.join(tempfile.mkdtemp(), "d.csv")
        simenv.dataset_to_csv(ds, path)
        with open(path, "rb") as fh:
            sha = hashlib.sha256(fh.read()).hexdigest()
        doc["datasets"].append({"noise_sigma": sigma, "seed": seed, "p_total": budget,
                                "rows": len(ds.rows), "csv_sha256": sha})
    ds = simenv.generate_dataset(simenv.OracleParams(noise_sigma=0.0), core.default_space(400.0), seed=0)
    train = ds.samples("train")
    w0 = fnn.initialize_weights(5, ds.bounds)
    for b, (start, size) in enumerate(((0, 1), (10, 4), (100, 32), (500, 77))):
        batch = train[start:start + size]
        g, loss = fnn.backward(w0, batch)
        doc["backward"].append({"init_seed": 5, "start": start, "size": size, "loss": loss,
                                **{k: getattr(g, k).tolist() for k in ("w1", "b1", "w2", "b2", "w_out", "b_out")}})
    cfg = fnn.TrainingConfig(learning_rate=0.002, batch_size=2, epochs=20, seed=2,
                             validation_fraction=0.05)
    weights, hist = fnn.train(train, cfg, feature_bounds=ds.bounds)
    doc["train"] = {"cfg": {"learning_rate": 0.002, "batch_size": 2, "epochs": 20, "seed": 2,
                            "validation_fraction": 0.05},
                    "history": [[h.epoch, h.train_mse, h.val_mse] for h in hist],
                    **{k: getattr(weights, k).tolist() for k in ("w1", "b1", "w2", "b2", "w_out", "b_out")}}
    with open(os.path.join(HERE, "training.json"), "w") as fh:
        json.dump(doc, fh)


STAGES = {
    "weights": stage_weights,
    "training": stage_training,
    "workloads": stage_workloads,
    "paper20": stage_paper20,
    "matching": stage_matching,
    "analytic": stage_analytic,
    "samples": stage_samples,
    "n256": stage_n256,
}

if __name__ == "__main__":
    wanted = sys.argv[1:] or list(STAGES)
    for name in wanted:
        t0 = time.time()
        STAGES[name]()
        print(f"[golden] {name} done in {time.time() - t0:.1f}s", flush=True)
