# SPDX-License-Identifier: Apache-2.0
"""CPU-only checks of the product library's boundary and host logic:
* libsort_b200.so loads and exports every symbol include/sort_b200.h declares;
* the host planner (time buckets, schedules, retained rows, compact masks, tile census)
  is bit-exact against the oracle's restatement of mask.cpp / tokenizer.cpp;
* the Python plan mirror agrees with both.
No compute entry point is called (there is no GPU here)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
from paper_2603_03988_b200 import build as B
from paper_2603_03988_b200 import plan as PL
from paper_2603_03988_b200 import runtime as R
from paper_2603_03988_b200.config import (ROLE_BOS, ROLE_CAND, ROLE_HIST, ROLE_PROF, ROLE_SEP,
                                          base_config, large_config, tiny_config)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    B.build()


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "sort_b200.h")).read()
    declared = set(re.findall(r"^(?:int|int64_t|void|const char\*)\s+(sort_\w+)\(", hdr, flags=re.M))
    assert len(declared) >= 20
    lib = ctypes.CDLL(R.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert declared == set(R.EXPORTS)


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", R.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", R.LIB_PATH],
                          capture_output=True, text=True).stdout
    for mnem in ("UTCHMMA", "UTMALDG", "LDTM"):  # tcgen05.mma, TMA, tcgen05.ld
        assert mnem in sass, mnem


def test_time_bucket_host_matches_oracle():
    vals = [0, 1, 2, 3, 2**20, 2**31, 2**40, 2**62, 2**63 - 1, -7]
    for k in range(1, 63):
        vals += [2**k - 1, 2**k, 2**k + 1]
    for v in vals:
        assert R.time_bucket(v, 32) == O.time_bucket(v, 32), v


def test_geometric_schedule_host_matches_oracle():
    for p in (1, 7, 128, 262, 1030, 4102):
        for dpt in (1, 2, 3, 4, 6, 12):
            for tgt in (1, 64, 128):
                assert R.geometric_schedule(p, dpt, tgt) == O.geometric_schedule(p, dpt, tgt)


def _random_structure(rng):
    n_hist = int(rng.integers(0, 60))
    n_prof = int(rng.integers(0, 4))
    n_cand = int(rng.integers(1, 9))
    st = bool(rng.integers(0, 2))
    roles = ([ROLE_BOS] if st else []) + [ROLE_HIST] * n_hist + ([ROLE_SEP] if st else []) + \
        [ROLE_PROF] * n_prof + ([ROLE_SEP] if st else []) + [ROLE_CAND] * n_cand
    L = len(roles)
    pos = list(range(L - n_cand)) + [L - n_cand] * n_cand
    return roles, pos


def test_retained_rows_and_mask_intervals_bit_exact():
    rng = np.random.default_rng(7)
    for trial in range(300):
        roles, pos = _random_structure(rng)
        W = int(rng.choice([-1, 1, 3, 8, 32]))
        F = int(rng.integers(0, 16))
        ks = bool(rng.integers(0, 2))
        r, p = list(roles), list(pos)
        for _ in range(int(rng.integers(1, 4))):
            keep = int(rng.integers(1, len(r) + 1))
            qr = R.retained_rows(r, keep, ks)
            assert qr == O.retained_rows(r, keep, ks) == PL.retained_rows(r, keep, ks)
            lo, hi, se = R.mask_intervals(r, p, qr, W, F)
            plo, phi, pse = PL.mask_intervals(r, p, qr, W, F)
            assert np.array_equal(lo, plo) and np.array_equal(hi, phi) and np.array_equal(se, pse)
            dense = np.zeros((len(qr), len(r)), np.uint8)
            c = np.arange(len(r))
            for i in range(len(qr)):
                dense[i] = (c >= lo[i]) & (c <= hi[i])
                if se[i] >= 0:
                    dense[i, se[i]] = 1
            assert np.array_equal(dense, O.build_mask(len(qr), r, p, W, F, qr))
            r = [r[i] for i in qr]
            p = [p[i] for i in qr]


def test_mask_intervals_errors_map_to_config_error():
    with pytest.raises(R.ConfigError):
        R.mask_intervals([ROLE_HIST] * 3, [0, 1, 2], [5], -1, 0)
    with pytest.raises(R.ConfigError):
        R.mask_intervals([ROLE_HIST] * 3, [0, 1, 2], [0, 1, 2], 0, 0)  # W must be >= 1 or -1


@pytest.mark.parametrize("mk", [tiny_config, base_config, large_config])
def test_python_plan_matches_oracle_per_layer(mk):
    cfg = mk()
    for lp in PL.layer_plans(cfg):
        vis = O.build_mask(lp.l_q, lp.roles_kv.tolist(), lp.pos_kv.tolist(), cfg.local_window,
                           cfg.full_suffix, lp.query_rows.tolist())
        assert int(vis.sum()) == lp.visible
        if lp.l_q * lp.l_kv <= 2_000_000:
            assert np.array_equal(vis, lp.dense())


def test_block_skip_census_matches_oracle_blockwise():
    """The analytic 128x128 tile census equals blockwise_masked_attention's skip count
    (block_attention.hpp:86-99) on the dense mask."""
    cfg = base_config()
    lp = PL.layer_plans(cfg)[0]
    vis = lp.dense()
    L = lp.l_kv
    Bt = 128
    nb = -(-L // Bt)
    pad = np.zeros((nb * Bt, nb * Bt), np.uint8)
    pad[: lp.l_q, :L] = vis
    issued = int(pad.reshape(nb, Bt, nb, Bt).any(axis=(1, 3)).sum())
    assert issued == 35 and nb * nb == 81
