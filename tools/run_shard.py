"""Per-GPU cost of the sequence-sharded retrieval (config 5) on one GPU: the
rank-local phases around the all-gather (spl_shard_histogram, then
spl_shard_select over R ranks' histograms; the other ranks' histograms are
stand-ins, the collective itself is not run). python tools/run_shard.py [R]"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2508_19740_b200 import capi  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 8
P, n, L, W = 32, 524288, 128, 4
k = int(0.02 * n * R)
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(3)
codes = torch.randint(-2**31, 2**31 - 1, (P, n, W), generator=g, device=dev, dtype=torch.int32)
q = torch.randint(-2**31, 2**31 - 1, (P, W), generator=g, device=dev, dtype=torch.int32)
nv = torch.full((P,), n, dtype=torch.int32, device=dev)
hist = torch.zeros((P, L + 1), dtype=torch.int32, device=dev)
all_hist = torch.zeros((R, P, L + 1), dtype=torch.int32, device=dev)
idx = torch.zeros((P, k), dtype=torch.int32, device=dev)
cnt = torch.zeros(P, dtype=torch.int32, device=dev)
off = torch.zeros(P, dtype=torch.int32, device=dev)
ctx = capi.Context(0)
s = torch.cuda.current_stream()


def hist_phase():
    ctx.shard_histogram(codes, n, L, q, P, nv, 1, n, hist, s.cuda_stream)


def select_phase():
    all_hist.copy_(hist.unsqueeze(0).expand(R, P, L + 1))  # stand-in for the all-gather
    ctx.shard_select(all_hist, R, R - 1, L, P, nv, 1, n, k, idx, cnt, off, s.cuda_stream)


def timeit(fn, reps=30):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1000


th = timeit(hist_phase)
ts = timeit(lambda: (hist_phase(), select_phase()))
print(f"R={R}: shard_histogram {th:.1f} us, histogram + select (incl. copy) {ts:.1f} us")
# fused in-kernel exchange, a single-rank group (exchange with itself)
peer = ctx.peer(1, 0, P, L)
capi.Peer.connect_local(ctx, [peer])
k1 = int(0.02 * n)
idx1 = torch.zeros((P, k1), dtype=torch.int32, device=dev)
tf = timeit(lambda: ctx.hamming_topk_sharded(peer, codes, n, L, q, P, nv, 1, n, k1, idx1, cnt, off,
                                             s.cuda_stream))
tu = timeit(lambda: ctx.hamming_topk(codes, n, L, q, P, nv, 1, n, k1, idx1, cnt, s.cuda_stream))
print(f"fused sharded (R=1 group) {tf:.1f} us vs single-GPU fused {tu:.1f} us (eager)")
peer.close()
ctx.close()
