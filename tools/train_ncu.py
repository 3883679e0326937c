"""One short device training run (acceptance-recipe corpus, batch 2) for an
ncu capture of k_train."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_03831_b200 import analytic, core, fnn, simenv
ds = simenv.generate_dataset(analytic.OracleParams(noise_sigma=0.0), core.default_space(400.0), seed=0)
fnn.train(ds.samples("train"), fnn.TrainingConfig(learning_rate=0.002, batch_size=2, epochs=2, seed=2,
                                                  validation_fraction=0.05), ds.bounds)
