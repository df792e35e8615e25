"""Worker for tests/test_gpu_multiproc.py::test_sharded_decode_multiprocess
(torch.distributed.run, gloo, every rank on GPU 0): R processes form a peer
group (IPC handles exchanged through the process group) and run the
sequence-sharded decode step — encode, retrieval with the in-kernel histogram
exchange, partial attention and the in-kernel partial exchange + combine —
then rank 0 checks the result against the single-GPU decode step on the
concatenated cache: indices bit-exact, outputs within 1e-3 (bf16 K/V), and
every rank's output identical."""
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2508_19740_b200 import capi  # noqa: E402

dist.init_process_group("gloo")
R, rank = dist.get_world_size(), dist.get_rank()
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
B, H, N, d, L, k = 1, 4, 36000, 128, 128, 720
W = L // 32
P = B * H
rng = np.random.default_rng(77)
w1 = (rng.standard_normal((H, d, d)) / np.sqrt(d)).astype(np.float32)
b1 = np.zeros((H, d), np.float32)
w2 = (rng.standard_normal((H, d, L)) / np.sqrt(d)).astype(np.float32)
codes = rng.integers(0, 2**32, (B, H, N, W), dtype=np.uint64).astype(np.uint32)
codes[0, 2] = codes[0, 2][rng.integers(0, 6, N)]  # heavy ties crossing ranks
g = torch.Generator()
g.manual_seed(5)
K = torch.randn((B, H, N, d), generator=g).bfloat16()
V = torch.randn((B, H, N, d), generator=g).bfloat16()
q = rng.standard_normal((B, H, d)).astype(np.float32)
kn = rng.standard_normal((B, H, d)).astype(np.float32)
vn = rng.standard_normal((B, H, d)).astype(np.float32)
bounds = np.linspace(0, N, R + 1).astype(np.int64)
lo, hi = int(bounds[rank]), int(bounds[rank + 1])
n_r = hi - lo
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
ctx = capi.Context(0)
hs = ctx.hasher(w1, b1, w2)
peer = ctx.peer(R, rank, P, L)
handles = [None] * R
dist.all_gather_object(handles, peer.ipc_handle())
peer.open(handles)
cd = t(codes[:, :, lo:hi].view(np.int32))
Kd, Vd = K[:, :, lo:hi].contiguous().to(dev), V[:, :, lo:hi].contiguous().to(dev)
nv = t(np.full(B, n_r, np.int32))
idx = torch.zeros((P, k), dtype=torch.int32, device=dev)
cnt = torch.zeros(P, dtype=torch.int32, device=dev)
off = torch.zeros(P, dtype=torch.int32, device=dev)
out = torch.zeros((B, H, d), dtype=torch.float32, device=dev)
ctx.reserve(P, n_r, L, k, d)
torch.cuda.synchronize()
dist.barrier()
hs.sharded_decode_step(peer, t(q), t(kn), t(vn), B, rank == R - 1, cd, Kd, Vd, capi.SPL_BF16, n_r, nv, n_r,
                       k, float(1 / np.sqrt(d)), idx, cnt, off, out)
torch.cuda.synchronize()
ctx.check_device_error()
mine = (idx.cpu().numpy().view(np.uint32), cnt.cpu().numpy(), off.cpu().numpy(), out.cpu().numpy(),
        cd.cpu().numpy().view(np.uint32), Kd.cpu(), Vd.cpu())
allv = [None] * R
dist.all_gather_object(allv, mine)
ok = True
if rank == 0:
    # single-GPU reference: the decode step on the concatenated cache (before append)
    full = torch.from_numpy(codes.view(np.int32).copy()).to(dev)
    Kf, Vf = K.clone().to(dev), V.clone().to(dev)
    nvf = t(np.full(B, N, np.int32))
    idx1 = torch.zeros((P, k), dtype=torch.int32, device=dev)
    cnt1 = torch.zeros(P, dtype=torch.int32, device=dev)
    out1 = torch.zeros((B, H, d), dtype=torch.float32, device=dev)
    hs.decode_step(t(q), t(kn), t(vn), B, full, Kf, Vf, capi.SPL_BF16, N, nvf, N, k, float(1 / np.sqrt(d)),
                   idx1, cnt1, out1)
    torch.cuda.synchronize()
    ctx.check_device_error()
    want = idx1.cpu().numpy().view(np.uint32)
    for p in range(P):
        cat = np.zeros(k, np.uint32)
        for r in range(R):
            ia, ca, oa = allv[r][0], allv[r][1], allv[r][2]
            cat[oa[p]:oa[p] + ca[p]] = ia[p, :ca[p]] + bounds[r]
        ok = ok and np.array_equal(cat, want[p])
    o1 = out1.cpu().numpy()
    for r in range(R):
        ok = ok and np.array_equal(allv[r][3], allv[0][3])
    err = float(np.abs(allv[0][3] - o1).max())
    ok = ok and err <= 1e-3
    # the appended row lives on the last rank, equal to the single-GPU append
    ok = ok and np.array_equal(allv[R - 1][4][:, :, -1], full.cpu().numpy().view(np.uint32)[:, :, -1])
    print("max-abs vs single GPU", err)
peer.close()
ctx.close()
dist.barrier()
dist.destroy_process_group()
if rank == 0:
    print("MP_SHARDED_DECODE", "OK" if ok else "MISMATCH")
    sys.exit(0 if ok else 1)
