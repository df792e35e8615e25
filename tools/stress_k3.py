"""Stress run of the headline retrieval (not a bench line): N CUDA-graph
replays of 20 x (L2 flush, retrieval) and of 50 back-to-back retrievals,
checking the device error word (the fused kernel's readiness-wait watchdog)
and the indices against the first run: python tools/stress_k3.py [N]."""
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2508_19740_b200 import capi  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
P, n, L = 32, 524288, 128
k = capi.budget_from_rate(0.02, n)
dev = torch.device("cuda", 0)
ctx = capi.Context(0)
g = torch.Generator(device=dev)
g.manual_seed(5)
codes = torch.randint(-2**31, 2**31 - 1, (P, n, L // 32), generator=g, device=dev, dtype=torch.int32)
qc = torch.randint(-2**31, 2**31 - 1, (P, L // 32), generator=g, device=dev, dtype=torch.int32)
nv = torch.full((P,), n, dtype=torch.int32, device=dev)
idx = torch.zeros((P, k), dtype=torch.int32, device=dev)
cnt = torch.zeros(P, dtype=torch.int32, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
acc = torch.zeros((), dtype=torch.int64, device=dev)
ctx.reserve(P, n, L, k)
ctx.hamming_topk(codes, n, L, qc, P, nv, 1, n, k, idx, cnt)
torch.cuda.synchronize()
ref = idx.clone()
gs = torch.cuda.Stream()
gs.wait_stream(torch.cuda.current_stream())


def capture(body, reps):
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=gs, capture_error_mode="relaxed"):
        for _ in range(reps):
            body()
    return gr


def flushed():
    flush.fill_(1)
    acc.add_(flush[: 256 << 20].view(torch.int32).sum())
    ctx.hamming_topk(codes, n, L, qc, P, nv, 1, n, k, idx, cnt, gs)


gf = capture(flushed, 20)
gb = capture(lambda: ctx.hamming_topk(codes, n, L, qc, P, nv, 1, n, k, idx, cnt, gs), 50)
t0 = time.time()
bad = 0
for i in range(N):
    gf.replay()
    gb.replay()
    torch.cuda.synchronize()
    ctx.check_device_error()
    if not torch.equal(idx, ref):
        bad += 1
print(f"{N} x (20 flushed + 50 back-to-back) retrievals in {time.time() - t0:.1f} s: "
      f"{N * 70} retrievals, {bad} index mismatches, device error word clean")
ctx.close()
