"""Small calls of every kernel, for compute-sanitizer (memcheck / racecheck /
synccheck): python tools/sanitize_cases.py. Exits non-zero on a parity miss."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from oracle_lib import Oracle  # noqa: E402
from paper_2508_19740_b200 import capi  # noqa: E402

dev = torch.device("cuda", 0)
orc = Oracle()
ctx = capi.Context(0)
rng = np.random.default_rng(0)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32) if a.dtype == np.uint32 else np.ascontiguousarray(a)).to(dev)  # noqa: E731
fails = 0

# K1 exact encode + append, K3 (fused, two-pass), K4
H, n, d, L, k = 2, 3000, 128, 128, 64
w1 = (rng.standard_normal((H, d, d)) / np.sqrt(d)).astype(np.float32)
b1 = np.zeros((H, d), np.float32)
w2 = (rng.standard_normal((H, d, L)) / np.sqrt(d)).astype(np.float32)
hs = ctx.hasher(w1, b1, w2)
keys = rng.standard_normal((1, H, n, d)).astype(np.float32)
vals = rng.standard_normal((1, H, n, d)).astype(np.float32)
q = rng.standard_normal((1, H, d)).astype(np.float32)
codes = torch.zeros((1, H, n, L // 32), dtype=torch.int32, device=dev)
hs.encode(T(keys), 1, n, codes)
qc = torch.zeros((1, H, L // 32), dtype=torch.int32, device=dev)
hs.encode(T(q), 1, 1, qc)
nv = torch.full((1,), n, dtype=torch.int32, device=dev)
for path in ("fused", "twopass"):
    import os
    if path == "twopass":
        os.environ["SPL_K3_PATH"] = "twopass"
    idx = torch.zeros((H, k), dtype=torch.int32, device=dev)
    cnt = torch.zeros(H, dtype=torch.int32, device=dev)
    ctx.hamming_topk(codes, n, L, qc, H, nv, H, n, k, idx, cnt)
    torch.cuda.synchronize()
    cc = codes.cpu().numpy().view(np.uint32)
    qq = qc.cpu().numpy().view(np.uint32)
    want = orc.retrieve_batch(cc[0], qq[0], np.full(H, n, np.uint32), k)
    fails += int(not np.array_equal(idx.cpu().numpy().view(np.uint32), want))
    os.environ.pop("SPL_K3_PATH", None)
out = torch.zeros((1, H, d), dtype=torch.float32, device=dev)
ctx.sparse_attend(T(q), T(keys), T(vals), capi.SPL_F32, n, d, H, idx, k, cnt, nv, H, float(1 / np.sqrt(d)), out)
# decode step: K1 append + encode, fused K3 + attention over bf16 K/V
# (attention_eval.cpp:234-264: the selected rows plus the own row nv - 1)
nvd = 2500
kcb = T(keys).bfloat16()
vcb = T(vals).bfloat16()
cd = codes.clone()
kn = rng.standard_normal((1, H, d)).astype(np.float32)
vn = rng.standard_normal((1, H, d)).astype(np.float32)
nvt = torch.full((1,), nvd, dtype=torch.int32, device=dev)
di = torch.zeros((H, k), dtype=torch.int32, device=dev)
dc = torch.zeros(H, dtype=torch.int32, device=dev)
do = torch.zeros((1, H, d), dtype=torch.float32, device=dev)
hs.decode_step(T(q), T(kn), T(vn), 1, cd, kcb, vcb, capi.SPL_BF16, n, nvt, n, k, float(1 / np.sqrt(d)),
               di, dc, do, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
want = orc.retrieve_batch(cd.cpu().numpy().view(np.uint32)[0], qc.cpu().numpy().view(np.uint32)[0],
                          np.full(H, nvd, np.uint32), k)
fails += int(not np.array_equal(di.cpu().numpy().view(np.uint32), want))
for h in range(H):
    rows = sorted(set(di[h, :int(dc[h])].tolist()) | {nvd - 1})
    kr, vr = kcb[0, h, rows].float(), vcb[0, h, rows].float()
    p = torch.softmax(kr @ T(q)[0, h] / np.sqrt(d), 0)
    fails += int(float((p @ vr - do[0, h]).abs().max()) > 1e-3)
# K2 (both kernels)
x = T(keys).bfloat16()
c2 = torch.zeros_like(codes)
hs.encode_tc(x, capi.SPL_BF16, 1, n, c2)
pre = torch.zeros((1, H, n, L), dtype=torch.float32, device=dev)
c3 = torch.zeros_like(codes)
hs.encode_tc(x, capi.SPL_BF16, 1, n, c3, pre)
torch.cuda.synchronize()
fails += int(not torch.equal(c2, c3))
# fused sharded (1-rank group), dense oracle, iou
peer = ctx.peer(1, 0, H, L)
capi.Peer.connect_local(ctx, [peer])
i2 = torch.zeros_like(idx)
c2n = torch.zeros_like(cnt)
off = torch.zeros_like(cnt)
ctx.hamming_topk_sharded(peer, codes, n, L, qc, H, nv, H, n, k, i2, c2n, off)
oi = torch.zeros_like(idx)
oc = torch.zeros_like(cnt)
ctx.oracle_topk(T(q[0]), T(keys), capi.SPL_F32, n, d, H, nv, H, n, float(1 / np.sqrt(d)), k, oi, oc)
iou = torch.zeros(H, dtype=torch.float64, device=dev)
ctx.iou(idx, cnt, k, oi, oc, k, H, iou)
torch.cuda.synchronize()
ctx.check_device_error()
fails += int(not torch.equal(i2, idx))
peer.close()
ctx.close()
print("sanitize cases:", "OK" if fails == 0 else f"{fails} parity misses")
sys.exit(1 if fails else 0)
