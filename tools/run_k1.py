"""K1 (exact encoder) alone: 32 heads x 1 query vector, as in a decode step."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2508_19740_b200 import capi  # noqa: E402

H, D, L = 32, 128, 128
ctx = capi.Context(0)
rng = np.random.default_rng(1)
hs = ctx.hasher((rng.standard_normal((H, D, D)) / np.sqrt(D)).astype(np.float32),
                np.zeros((H, D), np.float32),
                (rng.standard_normal((H, D, L)) / np.sqrt(D)).astype(np.float32))
q = torch.randn((1, H, D), device="cuda")
qc = torch.zeros((1, H, L // 32), dtype=torch.int32, device="cuda")
for _ in range(5):
    hs.encode(q, 1, 1, qc)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    hs.encode(q, 1, 1, qc)
e1.record()
torch.cuda.synchronize()
print(f"K1 encode 32 x 1 vector: {e0.elapsed_time(e1) / 50 * 1000:.2f} us")
