"""Phase trace (SPL_K3_TRACE=1) of the config-2 decode step's fused
retrieval + attention kernel, L2 flushed before each step:
python tools/c2_step_trace.py [reps]."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("SPL_K3_TRACE", "1")
from paper_2508_19740_b200 import capi  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
B, H, n, D, L = 1, 32, 131072, 128, 128
k = capi.budget_from_rate(0.02, n)
dev = torch.device("cuda", 0)
ctx = capi.Context(0)
rng = np.random.default_rng(7)
w1 = (rng.standard_normal((H, D, D)) / np.sqrt(D)).astype(np.float32)
b1 = np.zeros((H, D), np.float32)
w2 = (rng.standard_normal((H, D, L)) / np.sqrt(D)).astype(np.float32)
hs = ctx.hasher(w1, b1, w2)
g = torch.Generator(device=dev)
g.manual_seed(5)
codes = torch.randint(-2**31, 2**31 - 1, (B * H, n, L // 32), generator=g, device=dev, dtype=torch.int32)
kc = torch.randn((B, H, n, D), generator=g, device=dev).bfloat16()
vc = torch.randn((B, H, n, D), generator=g, device=dev).bfloat16()
q = torch.randn((B, H, D), generator=g, device=dev)
kn = torch.randn((B, H, D), generator=g, device=dev)
vn = torch.randn((B, H, D), generator=g, device=dev)
nv = torch.full((B,), n, dtype=torch.int32, device=dev)
idx = torch.zeros((B * H, k), dtype=torch.int32, device=dev)
cnt = torch.zeros(B * H, dtype=torch.int32, device=dev)
out = torch.zeros((B, H, D), dtype=torch.float32, device=dev)
q2 = torch.randn((B, H, D), generator=g, device=dev)
qc2 = torch.zeros((B, H, L // 32), dtype=torch.int32, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
for i in range(reps):
    flush.fill_(i)
    flush[: 256 << 20].view(torch.int32).sum()
    if os.environ.get("IWARM"):  # instructions warm, data cold: a tiny encode through the same kernel
        hs.encode(q2, B, 1, qc2)
    hs.decode_step(q, kn, vn, B, codes, kc, vc, capi.SPL_BF16, n, nv, n, k, float(1 / np.sqrt(D)),
                   idx, cnt, out)
    torch.cuda.synchronize()
ctx.check_device_error()
