"""Time the GPU trainer against the reference's train_hasher on the CLI's
default training shape (spotlight.cpp:130-146: MLP d=h=L=128, max_oth 256,
query_subsample 64, maskout 0.98) over one synthetic sequence of n tokens.
Prints per-iteration milliseconds of both and whether the weights agree."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle_lib import RefLib  # noqa: E402
from paper_2508_19740_b200 import capi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 64
ref_iters = int(sys.argv[3]) if len(sys.argv) > 3 else 8
ref = RefLib()
w = ref.mlp_gaussian_init(128, 128, 128, 64.0, ref.derive_seed(0, 100))
rng = np.random.default_rng(0)
data = [(rng.standard_normal((n, 128)).astype(np.float32),
         rng.standard_normal((n, 128)).astype(np.float32))]
rank = dict(beta=1.0, alpha=3.0, maskout=0.98, max_top=None, max_oth=256, query_subsample=64)
ctx = capi.Context(0)


def gpu(it):
    cfg = capi.TrainConfig(num_iters=it)
    g = [a.copy() for a in w]
    t = time.perf_counter()
    out = ctx.train_hasher(1, 128, 128, 128, 64.0, *g, data, capi.RankConfig(**rank), cfg)
    return time.perf_counter() - t, g, out


gpu(2)
t1, g, out = gpu(iters)
print(f"gpu: {iters} iters, {out['loop_ms'] / iters:.3f} ms/iter (device loop), "
      f"{t1:.3f} s wall for the whole call, iou {out['holdout_iou']:.4f}")
if ref_iters <= 0:
    sys.exit(0)
cfgd = dict(num_iters=ref_iters, warmup_iters=81, batch=1, seed=0, holdout_queries=128,
            max_lr=1e-3, min_lr=0.0, adam_beta1=0.9, adam_beta2=0.98, adam_eps=1e-8,
            weight_decay=0.1, grad_clip=1.0, soft_gamma=64.0, holdout_budget_rate=0.02)
t = time.perf_counter()
ref.train(1, *w, 64.0, data, rank, dict(cfgd, num_iters=1))
r0 = time.perf_counter() - t
t = time.perf_counter()
r = ref.train(1, *w, 64.0, data, rank, cfgd)
r1 = time.perf_counter() - t
print(f"reference: {ref_iters} iters {r1:.3f} s, {(r1 - r0) / (ref_iters - 1) * 1e3:.3f} ms/iter "
      f"(threads {ref.lib.spotref_max_threads()})")
_, g8, _ = gpu(ref_iters)
same = all(np.array_equal(a, b) for a, b in zip(g8, r[:3]))
print(f"weights after {ref_iters} iters identical: {same}")
