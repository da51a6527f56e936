# SPDX-License-Identifier: Apache-2.0
"""The rankformer:: drop-in facade (include/rankformer/reference_api.hpp + the forwarding
rankformer/{mask,attention,norm,rope,tokenizer,params}.hpp headers): tests/cpp/reference_caller.cpp
is written with the reference's call sites (tokenizer.hpp:84, mask.hpp:36-78, norm.hpp:17-45,
rope.hpp:13, attention.hpp:58-63) and compiled unchanged against include/. Host rules run here;
on the GPU every result is checked against the fp64 oracle.

Tolerances (stated per quantity):
  tokens / xn            bf16 token rows vs fp64: max abs 2e-2 (TOKEN_TOL, as test_gpu_parity)
  attention out          bf16 operands, fp32 accumulation: rel-L2 2e-2 (ATTN_REL)
  dxn / weight grads     bf16 backward: rel-L2 5e-2 (GRAD_REL), cosine >= 0.998
  rmsnorm dx / dgain     fp32 device op on identical inputs: rel-L2 1e-5 (F32_REL)
  rope                   fp32 product of fp64 angles: max abs 1e-5 relative to max |x| (F32_REL)
"""
import os
import struct
import subprocess
import sys

import numpy as np
import pytest

from paper_2603_03988_b200 import build as B
from paper_2603_03988_b200 import runtime, synth
from paper_2603_03988_b200.config import tiny_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "reference_caller.cpp")
EXE = os.path.join(ROOT, "tests", "cpp", "reference_caller")
INC = os.path.join(ROOT, "include")

TOKEN_TOL = 2e-2
ATTN_REL = 2e-2
GRAD_REL = 5e-2
F32_REL = 1e-5


def _compile():
    B.build()
    hdrs = [os.path.join(INC, "rankformer", f) for f in os.listdir(os.path.join(INC, "rankformer"))]
    if not os.path.exists(EXE) or os.path.getmtime(EXE) < max(
            [os.path.getmtime(SRC), os.path.getmtime(B.LIB)] + [os.path.getmtime(h) for h in hdrs]):
        subprocess.check_call(["g++", "-std=c++17", "-O1", "-Wall", "-I", INC, "-I", "/usr/local/cuda/include",
                               SRC, "-o", EXE, "-L", os.path.dirname(B.LIB), "-lsort_b200",
                               "-Wl,-rpath," + os.path.dirname(B.LIB)])
    return EXE


def test_reference_caller_compiles_and_host_rules():
    out = subprocess.run([_compile(), "host"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "host ok" in out.stdout


def _write_input(path, cfg, P, b, keep, dout):
    c = runtime.to_c_config(cfg, max_batch=1)
    with open(path, "wb") as f:
        f.write(bytes(c))
        f.write(struct.pack("<i", len(P)))
        for name, a in P.items():
            a = np.ascontiguousarray(a, np.float32).reshape(a.shape[0], -1)
            f.write(struct.pack("<i", len(name)) + name.encode())
            f.write(struct.pack("<qq", a.shape[0], a.shape[1]))
            f.write(a.tobytes())
        f.write(struct.pack("<q", int(b["req_ts"][0])))
        for i in range(cfg.n_hist):
            f.write(struct.pack("<iiiq", int(b["hist_item"][0, i]), int(b["hist_action"][0, i]),
                                int(b["hist_scene"][0, i]), int(b["hist_ts"][0, i])))
        for v in b["profile"][0]:
            f.write(struct.pack("<i", int(v)))
        for v in b["cand_item"][0]:
            f.write(struct.pack("<i", int(v)))
        f.write(struct.pack("<i", keep))
        f.write(struct.pack("<qq", *dout.shape))
        f.write(np.ascontiguousarray(dout, np.float64).tobytes())


def _read_output(path):
    out = {}
    with open(path, "rb") as f:
        data = f.read()
    o = 0
    while o < len(data):
        (n,) = struct.unpack_from("<i", data, o)
        o += 4
        name = data[o:o + n].decode()
        o += n
        r, c = struct.unpack_from("<qq", data, o)
        o += 16
        out[name] = np.frombuffer(data, np.float64, r * c, o).reshape(r, c)
        o += 8 * r * c
    return out


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["tiny", "base_widths"])
def test_reference_caller_vs_oracle(tmp_path, which):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    from paper_2603_03988_b200.config import base_config
    # tiny: d = 64, 4 heads (dk 16); base_widths: SORT-base's d = 256, 8 heads (dk 32), W = 256,
    # F = 128 with a 300-event history so the fp64 oracle stays fast
    cfg = tiny_config() if which == "tiny" else base_config(n_hist=300, n_cand=16, n_items=20000)
    P = synth.make_params(cfg, seed=11)
    b = synth.make_batch(cfg, 1, seed=12)
    keep = 100 if which == "tiny" else 160
    om = O.OracleModel(cfg, P)
    tk = om.tokenize(b, 0)
    roles, pos = tk["roles"], tk["position_ids"]
    query_rows = O.retained_rows(roles, keep, cfg.keep_specials)
    rng = np.random.default_rng(13)
    dout = rng.standard_normal((len(query_rows), cfg.model_dim)) * 0.1
    inp, outp = str(tmp_path / "in.bin"), str(tmp_path / "out.bin")
    _write_input(inp, cfg, P, b, keep, dout)
    r = subprocess.run([_compile(), inp, outp], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    g = _read_output(outp)

    # tokenizer.hpp:84 -> tokens, cache, positions
    assert np.max(np.abs(g["tokens"] - tk["tokens"])) < TOKEN_TOL
    assert np.array_equal(g["hist_time"][0].astype(np.int64), tk["hist_time"])
    assert np.array_equal(g["position_ids"][0].astype(np.int64), pos)
    # norm.hpp:17 on the device's token rows (identical inputs: fp32 bar)
    xn_ref = O.rmsnorm(g["tokens"], P["block.0.attn_norm"])
    assert _rel(g["xn"], xn_ref) < F32_REL
    # mask.hpp:36-78: query rows and the rendered mask, bit-exact
    assert g["query_rows"][0].astype(np.int64).tolist() == list(query_rows)
    vis_ref = O.build_mask(len(query_rows), roles, pos, cfg.local_window, cfg.full_suffix, query_rows)
    assert np.array_equal(g["mask"] == 0.0, vis_ref.astype(bool))
    # attention.hpp:58 forward on the same xn / mask
    xn = g["xn"]
    a_ref = om.attention(0, xn, query_rows, vis_ref, pos)
    assert _rel(g["attn_out"], a_ref) < ATTN_REL, _rel(g["attn_out"], a_ref)
    # attention.hpp:62 backward; wo frozen -> no gradient accumulated
    names = ["attn.0." + n for n in ("wq", "wk", "wv", "wg", "wo", "qk_gain_q", "qk_gain_k")]
    dxn_ref, grads_ref = om.attention_backward(0, xn, query_rows, vis_ref, pos, dout, names)
    assert _rel(g["dxn"], dxn_ref) < GRAD_REL, _rel(g["dxn"], dxn_ref)
    for n in names:
        got = g["grad." + n]
        if n.endswith(".wo"):
            assert not np.any(got), "frozen parameter received a gradient"
            continue
        ref = grads_ref[n].reshape(got.shape)
        cos = float(np.sum(got * ref) / (np.linalg.norm(got) * np.linalg.norm(ref)))
        assert _rel(got, ref) < GRAD_REL and cos > 0.998, (n, _rel(got, ref), cos)
    # norm.hpp:32 backward (identical inputs: fp32 bar)
    x = g["tokens"]
    gain = P["block.0.attn_norm"].reshape(-1)
    ms = np.mean(x * x, axis=1, keepdims=True)
    inv = 1.0 / np.sqrt(ms + 1e-6)
    xhat = x * inv
    dy = g["dxn"]
    dxh = dy * gain
    dx_ref = (dxh - np.sum(dxh * xhat, axis=1, keepdims=True) / x.shape[1] * xhat) * inv
    assert _rel(g["dx"], dx_ref) < F32_REL * 10
    assert _rel(g["dgain"][0], np.sum(dy * xhat, axis=0)) < F32_REL * 10
    # rope.hpp:13 forward and inverse
    qpos = pos[np.asarray(query_rows)]
    h0 = g["attn_out"][:, : cfg.head_dim]
    for key, inverse in (("rope", False), ("rope_inv", True)):
        ref = O.rope(h0, qpos, cfg.rope_theta, inverse=inverse)
        assert np.max(np.abs(g[key] - ref)) < F32_REL * np.max(np.abs(h0)) * 10
