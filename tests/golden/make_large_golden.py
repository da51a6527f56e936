# SPDX-License-Identifier: Apache-2.0
"""Generates tests/golden/large_fixture.npz: BASELINE.json configs[3] at its FULL geometry
(SORT-large: 12 layers, d=1024, 16 heads, 4096 history + 128 targets, W=256, geometric
pruning [4102, 2993, ..., 128]) on two seeded synthetic requests, scored by the fp64 oracle
(which tests/test_ref_pinning.py pins to the reference's own code). One request costs the
dense fp64 oracle ~0.6 TFLOP, too slow for a test run, so its logits are frozen here;
tests/test_gpu_parity.py::test_sort_large_full_geometry_vs_oracle regenerates the same
weights and requests (checked by SHA-256) and compares the GPU's logits with these.
Run: python tests/golden/make_large_golden.py  (about 10 min on 8 cores)"""
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), HERE]

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from make_golden import params_digest  # noqa: E402
from paper_2603_03988_b200 import synth  # noqa: E402
from paper_2603_03988_b200.config import large_config  # noqa: E402

PARAM_SEED, BATCH_SEED, BATCH = 41, 42, 2


def make():
    cfg = large_config(batch=BATCH)
    return cfg, synth.make_params(cfg, seed=PARAM_SEED), synth.make_batch(cfg, BATCH, seed=BATCH_SEED)


def batch_digest(b):
    import hashlib
    h = hashlib.sha256()
    for k in sorted(b):
        h.update(k.encode())
        h.update(np.ascontiguousarray(b[k]).tobytes())
    return h.hexdigest()


def main():
    cfg, P, b = make()
    t0 = time.time()
    m = O.OracleModel(cfg, P)
    probs = m.forward_batch(b, threads=BATCH)  # one request per thread
    logits = np.stack([np.log(p / (1 - p)) for p in probs.reshape(BATCH, cfg.n_cand, 3)])
    meta = m.layer_meta(b, 0)
    np.savez_compressed(os.path.join(HERE, "large_fixture.npz"), probs=probs.reshape(BATCH, cfg.n_cand, 3),
                        logits=logits, l_q=np.array(meta["l_q"]), visible=np.array(meta["visible"]),
                        params_sha256=np.array(params_digest(P)), batch_sha256=np.array(batch_digest(b)))
    print(f"wrote large_fixture.npz in {time.time() - t0:.0f} s; l_q={meta['l_q']}")


if __name__ == "__main__":
    main()
