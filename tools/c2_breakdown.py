"""Config-2 decode step broken into its launches, each timed on its own with
L2 flushed before it (CUDA events on the launching stream, median of N):
append+encode (K1), retrieval (K3, with and without the L2 prefetch of the
selected rows), attention (K4, cold and after the prefetch), the whole step.
python tools/c2_breakdown.py [reps]  — a measurement aid, not a bench line."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2508_19740_b200 import capi  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 15
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
qc = torch.zeros((B, H, L // 32), dtype=torch.int32, device=dev)
idx = torch.zeros((B * H, k), dtype=torch.int32, device=dev)
cnt = torch.zeros(B * H, dtype=torch.int32, device=dev)
out = torch.zeros((B, H, D), dtype=torch.float32, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
rd = torch.zeros((), dtype=torch.int64, device=dev)
pos = nv - 1  # append slot of the step's own key
scale = float(1 / np.sqrt(D))


def flush_l2():
    flush.fill_(1)  # evict L2 ...
    rd.copy_(flush[: 256 << 20].view(torch.int32).sum())  # ... and leave it clean (no write-backs later)


def graph_of(body, n):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            body()
    return g


def timed(fn, pre=None):
    """Per-call device time with L2 flushed before each call, free of launch
    overhead: a CUDA graph of N x (flush [+ pre] + fn) minus a graph of
    N x (flush [+ pre])."""
    n = reps
    base = lambda: (flush_l2(), pre and pre())
    for _ in range(2):
        base()
        fn()
    torch.cuda.synchronize()
    g1 = graph_of(lambda: (base(), fn()), n)
    g0 = graph_of(base, n)
    res = []
    for g in (g1, g0, g1, g0):
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) * 1000 / n)
    return min(res[0], res[2]) - min(res[1], res[3])


S = lambda: torch.cuda.current_stream().cuda_stream


enc = lambda: hs.encode(q, B, 1, qc, stream=S())
app = lambda: hs.encode_append(kn, vn, B, codes, kc, vc, capi.SPL_BF16, n, pos, stream=S())
ret = lambda: ctx.hamming_topk(codes, n, L, qc, B * H, nv, H, n, k, idx, cnt, stream=S())
att = lambda: ctx.sparse_attend(q, kc, vc, capi.SPL_BF16, n, D, B * H, idx, k, cnt, nv, H, scale, out, stream=S())
step = lambda: hs.decode_step(q, kn, vn, B, codes, kc, vc, capi.SPL_BF16, n, nv, n, k, scale, idx, cnt, out, S())
ctx.reserve(B * H, n, L, k, D)
enc()
ret()
import os
print(f"SPL_K4={os.environ.get('SPL_K4', '')} SPL_K4_NB={os.environ.get('SPL_K4_NB', '')}")
print(f"K1 query encode alone     {timed(enc):7.2f} us")
print(f"K1 key append alone       {timed(app):7.2f} us")
print(f"K3 retrieval (no prefetch){timed(ret):7.2f} us")
print(f"K4 attention, cold        {timed(att):7.2f} us")
print(f"K4 attention, L2-warm     {timed(att, pre=lambda: att()):7.2f} us")
print(f"decode step (flushed)     {timed(step):7.2f} us")
ctx.check_device_error()
ctx.close()
