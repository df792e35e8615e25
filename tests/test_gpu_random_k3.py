"""Randomised differential campaign for K3 (fixed seeds): random problem
counts, cache lengths, ragged n_valid, code widths, budgets (incl. k > n) and
tie structure, through both K3 paths, indices bit-exact against the C oracle
(which is pinned to the reference's top_k_indices). Complements the
hand-picked shapes of test_gpu_parity.py: plan geometries with straddling
segments, pieces shorter than a vector, odd row counts."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
from test_gpu_parity import run_topk  # noqa: E402

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(seed)
    L = int(rng.choice([32, 64, 128, 128, 256]))
    W = L // 32
    P = int(rng.integers(1, 41))
    cap = int(rng.choice([int(rng.integers(1, 300)), int(rng.integers(300, 20000)),
                          int(rng.integers(20000, 70000))]))
    codes = rng.integers(0, 2**32, (P, cap, W), dtype=np.uint64).astype(np.uint32)
    mode = int(rng.integers(0, 4))
    if mode == 1:  # heavy ties: few distinct rows
        codes = codes[:, rng.integers(0, max(1, cap // 50), cap)] if cap > 1 else codes
    elif mode == 2:  # near-duplicates of the query
        pass
    q = codes[np.arange(P), rng.integers(0, cap, P)].copy()
    if mode == 2:
        codes[:, ::7] = q[:, None, :]
    elif mode == 3:  # anti-correlated with the query: scores ~L/8 (the low-bin fallback)
        flips = (rng.integers(0, 2**32, codes.shape, dtype=np.uint64) &
                 rng.integers(0, 2**32, codes.shape, dtype=np.uint64) &
                 rng.integers(0, 2**32, codes.shape, dtype=np.uint64)).astype(np.uint32)
        codes = (~q)[:, None, :] ^ flips
    nv = rng.integers(1, cap + 1, P).astype(np.uint32)
    if rng.random() < 0.5:
        nv[:] = cap
    k = int(rng.choice([1, int(rng.integers(1, 64)), max(1, int(0.02 * cap)), int(rng.integers(1, cap + 50))]))
    return codes, q, nv, k


@pytest.mark.parametrize("path", ["fused", "twopass"])
@pytest.mark.parametrize("seed", list(range(64)))
def test_random_topk(ctx, oracle, monkeypatch, path, seed):
    if path == "twopass":
        monkeypatch.setenv("SPL_K3_PATH", "twopass")
    else:
        monkeypatch.delenv("SPL_K3_PATH", raising=False)
    codes, q, nv, k = _case(seed)
    got = run_topk(ctx, codes, q, nv, k)
    want = oracle.retrieve_batch(codes, q, nv, k)
    for p in range(q.shape[0]):
        kk = min(k, int(nv[p]))
        assert np.array_equal(got[p], want[p, :kk]), (seed, path, p, codes.shape, int(nv[p]), k)
