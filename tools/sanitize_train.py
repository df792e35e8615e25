"""Small trainer runs for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel of spl_train_hasher on small shapes (MLP ranking with batch 2
over two sequences, linear reconstruction, down-projection, a merged order
for a 16,500-token sequence)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2508_19740_b200 import capi  # noqa: E402

ctx = capi.Context(0)
rng = np.random.default_rng(0)


def seq(n, d):
    return (rng.standard_normal((n, d)).astype(np.float32), rng.standard_normal((n, d)).astype(np.float32))


rc = capi.RankConfig(maskout=0.9, max_oth=24, query_subsample=6)
cfg = capi.TrainConfig(num_iters=2, warmup_iters=1, holdout_queries=8, batch=2)
w1 = (rng.standard_normal((32, 48)) / 6).astype(np.float32)
b1 = np.zeros(48, np.float32)
w2 = (rng.standard_normal((48, 32)) / 6).astype(np.float32)
ctx.train_hasher(1, 32, 48, 32, 64.0, w1, b1, w2, [seq(120, 32), seq(90, 32)], rc, cfg)
p = (rng.standard_normal((32, 32)) / 6).astype(np.float32)
ctx.train_hasher(0, 32, 0, 32, 64.0, p, None, None, [seq(100, 32)], rc,
                 capi.TrainConfig(num_iters=2, warmup_iters=1, holdout_queries=8), 1)
p2 = (rng.standard_normal((32, 4)) / 6).astype(np.float32)
ctx.train_hasher(2, 32, 0, 4, 64.0, p2, None, None, [seq(100, 32)], rc,
                 capi.TrainConfig(num_iters=2, warmup_iters=1, holdout_queries=8))
if len(sys.argv) > 1 and sys.argv[1] == "long":
    w1s = (rng.standard_normal((16, 32)) / 4).astype(np.float32)
    ctx.train_hasher(1, 16, 32, 32, 64.0, w1s, np.zeros(32, np.float32),
                     (rng.standard_normal((32, 32)) / 6).astype(np.float32), [seq(16500, 16)],
                     capi.RankConfig(max_oth=8, query_subsample=2),
                     capi.TrainConfig(num_iters=1, warmup_iters=1, holdout_queries=2))
print("train sanitize cases ok")
