# Prints the per-tensor (GPU error, oracle bf16-noise, cosine) of the training-step parity test.
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle')
import numpy as np
import test_gpu_train as T
from paper_2603_03988_b200.config import tiny_config
T.NOISE_FACTOR, T.COS_MIN = 1e9, -1
_orig = T.rel_l2
rep = T._check_step(tiny_config(keep=[262, 128]), 7, 2)
for k, v in sorted(rep.items(), key=lambda kv: -kv[1][0] / max(kv[1][1], 1e-9)):
    print(k, "err %.4f noise %.4f cos %.5f" % v)
