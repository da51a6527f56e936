"""GPU diagnostic: op-level stream GEMM error over layouts / split-K (prints one line per case)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2603_03988_b200 import runtime as R

def tf32(x):
    return (x.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)

for dt in (True, False):
    for (M, N, K) in [(128, 256, 64), (256, 256, 1024), (256, 256, 16384), (2048, 256, 256), (56, 256, 65536)]:
        for ta in (False, True):
            for tb in (False, True):
                rng = np.random.default_rng(1)
                A = tf32(rng.normal(size=(K, M) if ta else (M, K)).astype(np.float32))
                B = tf32(rng.normal(size=(N, K) if tb else (K, N)).astype(np.float32))
                if not dt:
                    A = A.astype(np.float32); B = B.astype(np.float32)
                try:
                    C = R.op_gemm(A, B, ta, tb, tf32=dt)
                except Exception as e:
                    print("tf32" if dt else "bf16", M, N, K, ta, tb, "ERR", e); continue
                ref = (A.T if ta else A).astype(np.float64) @ (B.T if tb else B).astype(np.float64)
                err = np.max(np.abs(C - ref)) / max(1.0, np.max(np.abs(ref)))
                print("tf32" if dt else "bf16", M, N, K, ta, tb, f"{err:.3g}", f"{np.abs(C).max():.3g}", flush=True)
