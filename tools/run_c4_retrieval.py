"""Config-4 retrieval only (B=16 x 32 heads x 131072 rows x 256-bit codes,
k = 2621), for ncu launch lists: python tools/run_c4_retrieval.py [reps]."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2508_19740_b200 import capi  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
B, H, n, W = 16, 32, 131072, 8
P, k = B * H, 2621
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(1)
codes = torch.randint(-2**31, 2**31 - 1, (P, n, W), generator=g, device=dev, dtype=torch.int32)
q = torch.randint(-2**31, 2**31 - 1, (P, W), generator=g, device=dev, dtype=torch.int32)
nv = torch.full((B,), n, dtype=torch.int32, device=dev)
idx = torch.zeros((P, k), dtype=torch.int32, device=dev)
cnt = torch.zeros(P, dtype=torch.int32, device=dev)
ctx = capi.Context(0)
s = torch.cuda.current_stream().cuda_stream
for _ in range(reps):
    ctx.hamming_topk(codes, n, 256, q, P, nv, H, n, k, idx, cnt, s)
torch.cuda.synchronize()
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st.record()
for _ in range(10):
    ctx.hamming_topk(codes, n, 256, q, P, nv, H, n, k, idx, cnt, s)
en.record()
torch.cuda.synchronize()
print(f"config-4 retrieval {st.elapsed_time(en) * 100:.1f} us")
ctx.close()
