import sys, torch
sys.path.insert(0, '.')
from paper_2508_19740_b200 import capi
P, n, L, W = 32, 524288, 128, 4
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(3)
codes = torch.randint(-2**31, 2**31 - 1, (P, n, W), generator=g, device=dev, dtype=torch.int32)
q = torch.randint(-2**31, 2**31 - 1, (P, W), generator=g, device=dev, dtype=torch.int32)
nv = torch.full((P,), n, dtype=torch.int32, device=dev)
k = int(0.02 * n)
idx = torch.zeros((P, k), dtype=torch.int32, device=dev); cnt = torch.zeros(P, dtype=torch.int32, device=dev); off = torch.zeros(P, dtype=torch.int32, device=dev)
ctx = capi.Context(0)
peer = ctx.peer(1, 0, P, L); capi.Peer.connect_local(ctx, [peer])
for _ in range(3):
    ctx.hamming_topk_sharded(peer, codes, n, L, q, P, nv, 1, n, k, idx, cnt, off)
    ctx.hamming_topk(codes, n, L, q, P, nv, 1, n, k, idx, cnt)
torch.cuda.synchronize()
