"""Host side of the GPU trainer, no GPU needed: the
partition draws (ranking_loss.cpp:80-116) and the learning-rate schedule
(trainer.cpp:35-46) against the unmodified reference library."""
import numpy as np
import pytest

from oracle_lib import RefLib
from paper_2508_19740_b200 import capi

pytestmark = pytest.mark.skipif(not RefLib.available(), reason="oracle/_ref not built")

CASES = [
    # (q_train, n, rank kwargs)
    (400, 512, dict(max_oth=256, query_subsample=64)),
    (100, 128, dict()),
    (60, 64, dict(max_top=3, max_oth=5, query_subsample=7)),
    (2, 2, dict(maskout=0.5, query_subsample=1)),
    (1000, 1000, dict(max_top=1, max_oth=1)),
    (33, 4096, dict(maskout=0.9, max_oth=4000, query_subsample=40)),
]


@pytest.mark.parametrize("q,n,kw", CASES)
@pytest.mark.parametrize("seed", [0, 1, 0xDEADBEEF12345678])
def test_partition_draws_match_reference(q, n, kw, seed):
    ref = RefLib()
    rank = dict(beta=1.0, alpha=3.0, maskout=kw.get("maskout", 0.98),
                max_top=kw.get("max_top"), max_oth=kw.get("max_oth"),
                query_subsample=kw.get("query_subsample"))
    rows, top, oth, k_full, _ = ref.partition_identity(q, n, rank, seed)
    rc = capi.RankConfig(beta=1.0, alpha=3.0, maskout=rank["maskout"], max_top=rank["max_top"],
                         max_oth=rank["max_oth"], query_subsample=rank["query_subsample"])
    r2, t2, o2, k2 = capi.train_partition_host(rc, q, n, seed)
    assert k2 == k_full
    np.testing.assert_array_equal(r2, rows)
    np.testing.assert_array_equal(t2, top)
    np.testing.assert_array_equal(o2, oth)


@pytest.mark.parametrize("iters,warm,mx,mn", [(8192, 81, 1e-3, 0.0), (10, 3, 2e-3, 1e-4),
                                              (1, 5, 1e-3, 0.0), (0, 0, 1e-3, 0.0),
                                              (7, 6, 1e-3, 5e-4)])
def test_lr_schedule_matches_reference(iters, warm, mx, mn):
    ref = RefLib()
    cfg = capi.TrainConfig(num_iters=iters, warmup_iters=warm, max_lr=mx, min_lr=mn)
    for it in list(range(min(iters, 200))) + [max(iters - 1, 0)]:
        assert capi.train_lr_at(it, cfg) == ref.lr_at(it, iters, warm, mx, mn)
