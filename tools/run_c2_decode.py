"""Config-2 decode step only (B=1, 32 heads, 131072-token bf16 K/V, 128-bit
codes, k=2621) for launch lists / traces: python tools/run_c2_decode.py [reps]."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2508_19740_b200 import capi  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
B, H, n, D, L = 1, 32, 131072, 128, 128
k = 2621
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
s = torch.cuda.current_stream().cuda_stream


def step():
    hs.decode_step(q, kn, vn, B, codes, kc, vc, capi.SPL_BF16, n, nv, n, k, float(1 / np.sqrt(D)),
                   idx, cnt, out, s)


for _ in range(reps):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    step()
e1.record()
torch.cuda.synchronize()
print(f"config-2 decode step {e0.elapsed_time(e1) / 20 * 1000:.1f} us (eager)")
ctx.close()
