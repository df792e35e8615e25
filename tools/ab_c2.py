"""A/B of the config-2 decode step (B=1, 32 heads, 131072-token bf16 K/V,
128-bit codes, k=2621) for library builds: device time per step with L2
flushed (bench.py's flushed_graph_timer), and the step's indices / output
digest so builds can be compared. SPL_LIB=<lib> python tools/ab_c2.py [reps]
— a measurement aid, not a bench line."""
import hashlib
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2508_19740_b200 import capi  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
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


def step(s=None):
    st = (s or torch.cuda.current_stream()).cuda_stream
    hs.decode_step(q, kn, vn, B, codes, kc, vc, capi.SPL_BF16, n, nv, n, k, float(1 / np.sqrt(D)),
                   idx, cnt, out, st)


step()
torch.cuda.synchronize()
dig = hashlib.sha1(idx.cpu().numpy().tobytes()).hexdigest()[:12]
o0 = out.clone()
for _ in range(reps):
    r = bench.flushed_graph_timer(torch, step, 20, 4)
    print(f"{os.environ.get('SPL_LIB', 'default')}: config-2 step {r[0] * 1000:.2f} us (L2 flushed), "
          f"idx {dig}, out sum {float(o0.double().sum()):.6f}", flush=True)
ctx.close()
