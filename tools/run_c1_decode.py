"""Config-1 decode step (1 head, 4096 f32 keys, L=128, k=64) for profiling."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2508_19740_b200 import capi  # noqa: E402

D, L, n, k = 128, 128, 4096, 64
rng = np.random.default_rng(41)
ctx = capi.Context(0)
dev = torch.device("cuda", 0)
hs = ctx.hasher((rng.standard_normal((1, D, D)) / np.sqrt(D)).astype(np.float32),
                np.zeros((1, D), np.float32),
                (rng.standard_normal((1, D, L)) / np.sqrt(D)).astype(np.float32))
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
keys = rng.standard_normal((n, D)).astype(np.float32)
kc, vc = t(keys[None, None]), t(rng.standard_normal((1, 1, n, D)).astype(np.float32))
codes = torch.zeros((1, 1, n, L // 32), dtype=torch.int32, device=dev)
hs.encode(kc, 1, n, codes)
q = t(rng.standard_normal((1, 1, D)).astype(np.float32))
nvalid = torch.full((1,), n, dtype=torch.int32, device=dev)
idx = torch.zeros((1, k), dtype=torch.int32, device=dev)
cnt = torch.zeros(1, dtype=torch.int32, device=dev)
out = torch.zeros((1, 1, D), dtype=torch.float32, device=dev)
for _ in range(20):
    hs.decode_step(q, kc[:, :, n - 1], vc[:, :, n - 1], 1, codes, kc, vc, capi.SPL_F32, n, nvalid, n, k,
                   float(1 / np.sqrt(D)), idx, cnt, out, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok")
