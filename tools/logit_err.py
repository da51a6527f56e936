"""Max |logit - oracle| and rel-L2 of the SORT-base / tiny forward on the parity tests' inputs
(test_model_logits_vs_oracle: B = 4, seed 31), to compare library variants' numerics."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np

import oracle as O
from paper_2603_03988_b200 import runtime as R, synth
from paper_2603_03988_b200.config import base_config, tiny_config

for name, cfg, seed in (("tiny", tiny_config(), 3), ("base", base_config(), 5)):
    P = synth.make_params(cfg, seed=seed)
    gm, om = R.SortModel(cfg, P, max_batch=4), O.OracleModel(cfg, P)
    b = synth.make_batch(cfg, 4, seed=31)
    _, z = gm.forward_logits(b)
    ref = np.stack([om.forward(b, i)[1] for i in range(4)])
    print(f"{name}: max|dz| {np.max(np.abs(z - ref)):.5f} rel-L2 {np.linalg.norm(z - ref) / np.linalg.norm(ref):.5f}",
          flush=True)
