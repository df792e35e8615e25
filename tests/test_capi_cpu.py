"""CPU-only checks of the C-ABI boundary: the libraries load without a GPU,
export every symbol include/spl_c.h declares, and the host-side arithmetic
(budget_from_rate, the sharded threshold plan) matches the oracle."""
import ctypes
from pathlib import Path

import numpy as np
import pytest

from paper_2508_19740_b200 import capi

ROOT = Path(__file__).resolve().parents[1]


def test_libspl_exports_every_header_symbol():
    lib = capi.load()
    declared = capi.header_symbols()
    assert len(declared) >= 25
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing


def test_dropin_library_loads():
    so = ROOT / "paper_2508_19740_b200" / "lib" / "libspotlight_b200.so"
    assert so.exists(), "build() must produce the C++ drop-in"
    ctypes.CDLL(str(so))


def test_context_needs_a_blackwell_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    assert capi.load().spl_ctx_create(0, ctypes.byref(h)) == capi.SPL_E_CUDA


def test_budget_from_rate_matches_oracle(oracle):
    for n in [1, 8, 20, 21, 500, 999, 1000, 2048, 4096, 131072, 524288, 4194304]:
        for rate in [0.001, 0.02, 0.5, 1.0]:
            assert capi.budget_from_rate(rate, n) == oracle.budget_from_rate(rate, n)
    with pytest.raises(capi.DimensionError):
        capi.budget_from_rate(0.0, 10)
    with pytest.raises(capi.DimensionError):
        capi.budget_from_rate(1.5, 10)


def _sharded_select(scores_per_rank, L, k):
    """Emulate the sequence-sharded select with the C-ABI's host plan: every
    rank histograms its scores, the plan gives its tie share / offset, and the
    rank keeps score > T plus its first take_eq ties, in order."""
    R = len(scores_per_rank)
    hist = np.zeros((R, L + 1), np.uint32)
    for r, s in enumerate(scores_per_rank):
        hist[r] = np.bincount(s, minlength=L + 1)
    out, base, offsets = [], 0, []
    for r, s in enumerate(scores_per_rank):
        pl = capi.plan_shard_host(hist, r, k)
        offsets.append(pl["offset"])
        T, take = pl["T"], pl["take_eq"]
        sel = []
        eq_seen = 0
        for i, v in enumerate(s):
            if v > T:
                sel.append(base + i)
            elif v == T:
                if eq_seen < take:
                    sel.append(base + i)
                eq_seen += 1
        assert len(sel) == pl["count"]
        out.append(np.array(sel, np.uint32))
        base += len(s)
    return out, offsets


@pytest.mark.parametrize("R", [1, 2, 3, 5, 8])
def test_sharded_plan_equals_reference_topk(oracle, R):
    rng = np.random.default_rng(R)
    for trial in range(60):
        L = int(rng.choice([32, 64, 128]))
        n = int(rng.integers(R, 3000))
        span = int(rng.integers(1, L + 1))
        lo = int(rng.integers(0, L + 1 - span + 1))
        scores = rng.integers(lo, min(L, lo + span) + 1, n).astype(np.int32)
        k = int(rng.integers(1, n + 1))
        cuts = np.sort(rng.choice(np.arange(1, n), R - 1, replace=False)) if R > 1 else []
        parts = np.split(scores, cuts)
        got, offsets = _sharded_select(parts, L, k)
        want = oracle.top_k(scores, k)
        cat = np.concatenate(got)
        assert np.array_equal(cat, want), (trial, R, L, n, k)
        # offsets are the running lengths of the rank-ordered lists
        assert offsets == list(np.cumsum([0] + [len(g) for g in got])[:-1])
