"""Drive K2 (spl_encode_tc) for profiling: B x 32 heads x n bf16 keys, L = 256.
python tools/prof_k2.py [B] [n] [L]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_19740_b200 import capi  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
L = int(sys.argv[3]) if len(sys.argv) > 3 else 256
H, D = 32, 128
ctx = capi.Context(0)
rng = np.random.default_rng(4)
w1 = (rng.standard_normal((H, D, D)) / np.sqrt(D)).astype(np.float32)
b1 = np.zeros((H, D), np.float32)
w2 = (rng.standard_normal((H, D, L)) / np.sqrt(D)).astype(np.float32)
hs = ctx.hasher(w1, b1, w2)
x = torch.randn((B, H, n, D), device="cuda", dtype=torch.bfloat16)
codes = torch.empty((B, H, n, L // 32), device="cuda", dtype=torch.int32)
for _ in range(3):
    hs.encode_tc(x, capi.SPL_BF16, B, n, codes)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    hs.encode_tc(x, capi.SPL_BF16, B, n, codes)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
keys = B * H * n
print(f"K2 B={B} n={n} L={L}: {ms:.3f} ms, {keys * (2*D*D + 2*D*L) / ms / 1e9:.1f} TF/s")
