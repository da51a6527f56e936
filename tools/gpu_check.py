# Quick GPU diagnostic: each stage of the CUDA path vs the CPU oracle, printing errors.
import os
import sys
import time
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np

import oracle as O
from paper_2603_03988_b200 import synth, runtime
from paper_2603_03988_b200.config import tiny_config, base_config, ROLE_HIST


def step(name, fn):
    t = time.time()
    try:
        fn()
        print(f"[ok] {name} ({time.time()-t:.1f}s)", flush=True)
    except Exception:
        print(f"[FAIL] {name}", flush=True)
        traceback.print_exc()


def block_attn():
    rng = np.random.default_rng(0)
    for dk in (16, 32):
        for (lq, lkv, W) in ((128, 128, -1), (300, 300, 64), (70, 1094, -1), (1094, 1094, 256)):
            nh = 3
            q = rng.normal(size=(nh, lq, dk)).astype(np.float32)
            k = rng.normal(size=(nh, lkv, dk)).astype(np.float32)
            v = rng.normal(size=(nh, lkv, dk)).astype(np.float32)
            roles = [ROLE_HIST] * lkv
            pos = list(range(lkv))
            qr = list(range(lkv - lq, lkv))
            lo, hi, se = runtime.mask_intervals(roles, pos, qr, W, 0)
            out, sk, tot = runtime.block_attention(q, k, v, lo, hi, se)
            vis = O.build_mask(lq, roles, pos, W, 0, qr)
            err = 0
            for b in range(nh):
                qb = q[b].astype(np.float64) / 1.0
                ref = O.dense_attention(qb, k[b], v[b], np.where(vis > 0, 0.0, -np.inf))
                err = max(err, np.max(np.abs(ref - out[b])))
            print(f"   dk={dk} lq={lq} lkv={lkv} W={W}: max|err|={err:.4f} skipped {sk}/{tot}")


def tiny_model():
    cfg = tiny_config()
    P = synth.make_params(cfg, seed=3)
    b = synth.make_batch(cfg, 1, seed=4)
    om = O.OracleModel(cfg, P)
    gm = runtime.SortModel(cfg, P)
    t = gm.tokenize(b)
    ot = om.tokenize(b)
    print("   tokens max|err|", np.max(np.abs(t["tokens"][0] - ot["tokens"])),
          "hist_time equal", np.array_equal(t["hist_time"][0], ot["hist_time"]),
          "pos equal", np.array_equal(t["position_ids"], ot["position_ids"]))
    for l in range(cfg.layers):
        pl = gm.layer_plan(l)
        print(f"   layer {l}: l_q={pl['l_q']} l_kv={pl['l_kv']} visible={pl['visible']} tiles {pl['tiles_issued']}/{pl['tiles_total']}")
    # attention op
    x = ot["tokens"][None].astype(np.float32)
    a = gm.attention_forward(0, x)
    pl = gm.layer_plan(0)
    xn = O.rmsnorm(ot["tokens"], P["block.0.attn_norm"])
    vis = O.build_mask(pl["l_q"], ot["roles"], ot["position_ids"], cfg.local_window, cfg.full_suffix, pl["query_rows"])
    ref = om.attention(0, xn, pl["query_rows"], vis, ot["position_ids"])
    print("   attention op max|err|", np.max(np.abs(a[0] - ref)), "ref scale", np.max(np.abs(ref)))
    p, lg = gm.forward_logits(b)
    op, ol = om.forward(b)
    print("   logits max|err|", np.max(np.abs(lg[0] - ol)), "logit scale", np.max(np.abs(ol)))
    print("   probs max|err|", np.max(np.abs(p[0] - op)))


def base_model():
    cfg = base_config()
    P = synth.make_params(cfg, seed=5)
    B = 4
    b = synth.make_batch(cfg, B, seed=6)
    gm = runtime.SortModel(cfg, P, max_batch=256)
    om = O.OracleModel(cfg, P)
    p, lg = gm.forward_logits(b)
    t0 = time.time()
    op = om.forward_batch(b, threads=8).reshape(B, cfg.n_cand, 3)
    print(f"   oracle {B} requests in {time.time()-t0:.1f}s")
    ol = np.log(op) - np.log1p(-op)
    err = np.abs(lg - ol)
    print("   logits max|err|", err.max(), "mean", err.mean(), "logit rms", np.sqrt((ol**2).mean()))
    for l in range(cfg.layers):
        pl = gm.layer_plan(l)
        print(f"   layer {l}: l_q={pl['l_q']} l_kv={pl['l_kv']} visible={pl['visible']} tiles {pl['tiles_issued']}/{pl['tiles_total']}")
    # timing at full batch
    bb = synth.make_batch(cfg, 256, seed=7)
    gm.forward(bb)
    gm.enable_stage_timing(True)
    t0 = time.time()
    for _ in range(3):
        gm.forward(bb)
    print(f"   wall per forward (incl. H2D/D2H) {(time.time()-t0)/3*1e3:.2f} ms; kernels {gm.kernel_count()}")
    st = gm.stage_times()
    tot = sum(st.values())
    print(f"   device stages total {tot:.3f} ms")
    for k, v in st.items():
        print(f"      {k:16s} {v:.3f} ms")


if __name__ == "__main__":
    which = sys.argv[1:] or ["block", "tiny", "base"]
    if "block" in which:
        step("block attention", block_attn)
    if "tiny" in which:
        step("tiny model", tiny_model)
    if "base" in which:
        step("base model", base_model)
