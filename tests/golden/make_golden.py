# SPDX-License-Identifier: Apache-2.0
"""Generates tests/golden/tiny_fixture.npz: the tiny config (BASELINE.json configs[0])
on seeded synthetic inputs, with the fp64 oracle's outputs (token-index artifact,
per-layer structure, logits/probabilities). The oracle is pinned by the SPEC.md
KATs in tests/test_oracle_kat.py; this fixture freezes its outputs so the GPU tests
also check against committed numbers. Run: python tests/golden/make_golden.py
"""
import hashlib
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from paper_2603_03988_b200 import synth  # noqa: E402
from paper_2603_03988_b200.config import tiny_config  # noqa: E402

PARAM_SEED, BATCH_SEED, BATCH = 3, 4, 2


def params_digest(P):
    h = hashlib.sha256()
    for k in sorted(P):
        h.update(k.encode())
        h.update(np.ascontiguousarray(P[k], np.float32).tobytes())
    return h.hexdigest()


def main():
    cfg = tiny_config()
    P = synth.make_params(cfg, seed=PARAM_SEED)
    b = synth.make_batch(cfg, BATCH, seed=BATCH_SEED)
    m = O.OracleModel(cfg, P)
    out = {f"in_{k}": v for k, v in b.items()}
    probs, logits, hist_time = [], [], []
    for i in range(BATCH):
        p, lg = m.forward(b, i)
        probs.append(p)
        logits.append(lg)
        hist_time.append(m.tokenize(b, i)["hist_time"])
    t = m.tokenize(b, 0)
    meta = m.layer_meta(b, 0)
    out.update(probs=np.stack(probs), logits=np.stack(logits), hist_time=np.stack(hist_time),
               position_ids=t["position_ids"], roles=t["roles"],
               candidate_index=t["candidate_index"], visible=np.array(meta["visible"]),
               l_q=np.array(meta["l_q"]), params_sha256=np.array(params_digest(P)))
    np.savez_compressed(os.path.join(HERE, "tiny_fixture.npz"), **out)
    print("wrote tiny_fixture.npz", {k: np.shape(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
