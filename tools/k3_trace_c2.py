"""K3 phase trace at a given retrieval shape (SPL_K3_TRACE=1 prints per-phase
globaltimer stamps, mean / max over CTAs, from kernel start), with L2 flushed
before each call (unless a 4th argument "warm" asks for back-to-back calls):
python tools/k3_trace_c2.py [n] [P] [reps] [warm]."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("SPL_K3_TRACE", "1")
from paper_2508_19740_b200 import capi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
P = int(sys.argv[2]) if len(sys.argv) > 2 else 32
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
warm = len(sys.argv) > 4 and sys.argv[4] == "warm"
# "iwarm": after the flush, one small retrieval through the same kernel on
# other data (its instructions back in L2, the codes still cold)
iwarm = len(sys.argv) > 4 and sys.argv[4] == "iwarm"
# "rflush": evict L2 by reading 512 MB only (no dirty lines anywhere)
rflush = len(sys.argv) > 4 and sys.argv[4] == "rflush"
L = 128
k = capi.budget_from_rate(0.02, n)
dev = torch.device("cuda", 0)
ctx = capi.Context(0)
g = torch.Generator(device=dev)
g.manual_seed(5)
codes = torch.randint(-2**31, 2**31 - 1, (P, n, L // 32), generator=g, device=dev, dtype=torch.int32)
qc = torch.randint(-2**31, 2**31 - 1, (P, L // 32), generator=g, device=dev, dtype=torch.int32)
nv = torch.full((1,), n, dtype=torch.int32, device=dev)
idx = torch.zeros((P, k), dtype=torch.int32, device=dev)
cnt = torch.zeros(P, dtype=torch.int32, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
# same per-segment geometry as the measured call (same select instantiation)
small = torch.randint(-2**31, 2**31 - 1, (2, n, L // 32), generator=g, device=dev, dtype=torch.int32)
sidx = torch.zeros((2, k), dtype=torch.int32, device=dev)
scnt = torch.zeros(2, dtype=torch.int32, device=dev)
snv = torch.full((1,), n, dtype=torch.int32, device=dev)
for i in range(reps):
    if rflush:
        flush.view(torch.int32).sum()
    elif not warm:
        flush.fill_(i)
        flush[: 256 << 20].view(torch.int32).sum()
    if iwarm:
        mode = os.environ["SPL_K3_TRACE"]
        os.environ["SPL_K3_TRACE"] = ""
        ctx.hamming_topk(small, n, L, qc[:2], 2, snv, 2, n, k, sidx, scnt)
        os.environ["SPL_K3_TRACE"] = mode
    ctx.hamming_topk(codes, n, L, qc, P, nv, P, n, k, idx, cnt)
    torch.cuda.synchronize()
ctx.check_device_error()
