# SPDX-License-Identifier: Apache-2.0
"""Request ingest (SURVEY.md 8(f) "next 3"): the library's host reader of the reference's JSONL
dataset (schema "rankformer.dataset" v1, read_dataset, dataset_io.cpp:58-162) -- round trip of
a synthetic batch, and every validation rule of the reference with its DatasetFormatError text
("dataset line N, field 'F': what"). Host-only (no GPU); the batches land in the SoA layout
sort_forward takes."""
import json
import os

import numpy as np
import pytest

from paper_2603_03988_b200 import runtime as R
from paper_2603_03988_b200 import synth
from paper_2603_03988_b200.config import tiny_config


def _roundtrip(tmp_path, B=4):
    cfg = tiny_config()
    b = synth.make_batch(cfg, B, seed=5)
    labels = np.zeros((B, cfg.n_cand, 3), np.int64)
    rng = np.random.default_rng(1)
    labels[..., 0] = rng.random((B, cfg.n_cand)) < 0.3
    labels[..., 1] = labels[..., 0] & (rng.random((B, cfg.n_cand)) < 0.5)
    labels[..., 2] = labels[..., 1] & (rng.random((B, cfg.n_cand)) < 0.5)
    path = os.path.join(tmp_path, "d.jsonl")
    R.write_dataset(path, b, labels, request_ids=np.arange(100, 100 + B))
    return cfg, b, labels, path


def test_roundtrip_exact(tmp_path):
    cfg, b, labels, path = _roundtrip(tmp_path)
    ds = R.Dataset(path)
    assert len(ds) == 4
    _, lab, ids, arrs = ds.batch(1, 3, cfg)
    for k in arrs:
        assert np.array_equal(arrs[k], b[k][1:4]), k
    assert np.array_equal(lab, labels[1:4].astype(np.float32))
    assert ids.tolist() == [101, 102, 103]


def test_geometry_mismatch_is_config_error(tmp_path):
    cfg, b, labels, path = _roundtrip(tmp_path)
    ds = R.Dataset(path)
    with pytest.raises(R.ConfigError):
        ds.batch(0, 2, tiny_config(n_cand=cfg.n_cand + 1))
    with pytest.raises(R.ConfigError):
        ds.batch(3, 2, cfg)  # past the end


def _write(tmp_path, header, recs):
    path = os.path.join(tmp_path, "bad.jsonl")
    with open(path, "w") as f:
        f.write((header if isinstance(header, str) else json.dumps(header)) + "\n")
        for r in recs:
            f.write((r if isinstance(r, str) else json.dumps(r)) + "\n")
    return path


GOOD = {"request_id": 1, "ts": 100, "profile": [1, 2, 3], "history": [[5, 0, 10, 1], [6, 2, 20, 0]],
        "candidates": [[7, 1, 1, 0, []], [8, 0, 0, 0, [0.5]]]}
HDR = {"schema": "rankformer.dataset", "version": 1, "records": 1}


@pytest.mark.parametrize("header,rec,field,what", [
    ("", None, "header", "empty file"),
    ("[1, 2]", None, "header", "not a JSON object"),
    ({"schema": "other", "version": 1}, None, "schema", "unknown schema name"),
    ({"schema": "rankformer.dataset", "version": 2}, None, "version", "unsupported schema version"),
    (HDR, "{not json", "record", "malformed JSON"),
    (HDR, {k: v for k, v in GOOD.items() if k != "ts"}, "ts", "missing"),
    (HDR, dict(GOOD, history=5), "history", "not an array"),
    (HDR, dict(GOOD, history=[[5, 0, 10]]), "history", "event must be [item,action,ts,scene]"),
    (HDR, dict(GOOD, history=[[5, 3, 10, 1]]), "history.action", "out of range"),
    (HDR, dict(GOOD, history=[[5, 0, 30, 1], [6, 0, 20, 1]]), "history.ts", "timestamps must be non-decreasing"),
    (HDR, dict(GOOD, history=[[5, 0, 100, 1]]), "history.ts", "event not before request"),
    (HDR, dict(GOOD, candidates=[]), "candidates", "must be a non-empty array"),
    (HDR, dict(GOOD, candidates=[[7, 1, 1, 0]]), "candidates", "candidate must be [item,click,cart,purchase,[side...]]"),
    (HDR, dict(GOOD, candidates=[[7, 2, 0, 0, []]]), "candidates.labels", "labels must be 0/1"),
    (HDR, dict(GOOD, candidates=[[7, 0, 0, 1, []]]), "candidates.purchase", "purchase=1 requires click=1"),
    (HDR, dict(GOOD, candidates=[[7, 0, 1, 0, []]]), "candidates.cart", "cart=1 requires click=1"),
])
def test_reference_validation_rules(tmp_path, header, rec, field, what):
    if header == "":
        path = os.path.join(tmp_path, "empty.jsonl")
        open(path, "w").close()
    else:
        path = _write(tmp_path, header, [] if rec is None else [rec])
    with pytest.raises(R.ConfigError) as ei:
        R.Dataset(path)
    line = 1 if rec is None else 2
    assert str(ei.value).endswith(f"dataset line {line}, field '{field}': {what}"), str(ei.value)


def test_good_record_parses(tmp_path):
    ds = R.Dataset(_write(tmp_path, HDR, [GOOD, ""]))  # blank lines are skipped
    assert len(ds) == 1


def test_side_features_rejected_at_batch(tmp_path):
    """A record with candidate side features parses (dataset_io.cpp:142 reads them) but the
    configured side width is 0, so packing it for the tokenizer is a ConfigError with the
    reference tokenizer's text (tokenizer.cpp:116-120)."""
    rec = dict(GOOD, candidates=[[7, 1, 0, 0, [0.5, 1.5]]])
    ds = R.Dataset(_write(tmp_path, HDR, [rec]))
    cfg = tiny_config(n_hist=2, n_cand=1)
    with pytest.raises(R.ConfigError) as ei:
        ds.batch(0, 1, cfg)
    assert "candidate side feature width 2 != configured 0" in str(ei.value)
