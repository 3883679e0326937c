"""Training throughput: the device trainer (fnn.train / train_many) vs the
unmodified reference's numpy loop (baseline/_ref, if staged), on the
acceptance recipe's corpus.  Prints one JSON line."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2405_03831_b200 import analytic, core, fnn, simenv
from paper_2405_03831_b200.trainer import train_many

epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 400
ds = simenv.generate_dataset(analytic.OracleParams(noise_sigma=0.0), core.default_space(400.0), seed=0)
data = ds.samples("train")
cfg = fnn.TrainingConfig(learning_rate=0.002, batch_size=2, epochs=epochs, seed=2, validation_fraction=0.05)
fnn.train(data, fnn.TrainingConfig(learning_rate=0.002, batch_size=2, epochs=1, seed=2,
                                   validation_fraction=0.05), ds.bounds)      # warm
torch.cuda.synchronize()
t0 = time.perf_counter(); fnn.train(data, cfg, ds.bounds); t1 = time.perf_counter()
steps = epochs * -(-int(len(data) * 0.95 + 0.999) // 2)
out = {"epochs": epochs, "train_rows": len(data), "device_s": t1 - t0,
       "device_sgd_steps_per_s": steps / (t1 - t0)}
R = 148
cfgs = [fnn.TrainingConfig(learning_rate=0.002, batch_size=2, epochs=epochs, seed=s, validation_fraction=0.05)
        for s in range(R)]
t0 = time.perf_counter(); train_many(data, cfgs, ds.bounds); t1 = time.perf_counter()
out.update({"train_many_runs": R, "train_many_s": t1 - t0})
ref = os.path.join(ROOT, "baseline", "_ref")
if os.path.isdir(os.path.join(ref, "cosched")):
    sys.path.insert(0, ref)
    from cosched import fnn as rfnn, simenv as rsim, core as rcore
    rds = rsim.generate_dataset(rsim.OracleParams(noise_sigma=0.0), rcore.default_space(400.0), seed=0)
    re = max(1, min(epochs, 10))
    rcfg = rfnn.TrainingConfig(learning_rate=0.002, batch_size=2, epochs=re, seed=2, validation_fraction=0.05)
    t0 = time.perf_counter(); rfnn.train(rds.samples("train"), rcfg, feature_bounds=rds.bounds); t1 = time.perf_counter()
    out.update({"reference_epochs_timed": re, "reference_s": t1 - t0,
                "reference_s_extrapolated": (t1 - t0) * epochs / re})
print(json.dumps(out))
