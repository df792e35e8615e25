"""Worker for tests/test_gpu_multiproc.py (launched by torch.distributed.run,
gloo, every rank on GPU 0): a real multi-process peer group — IPC handles
exchanged through the process group, spl_peer_open, the fused in-kernel
exchange across processes — checked on rank 0 against the oracle."""
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from paper_2508_19740_b200 import capi  # noqa: E402

dist.init_process_group("gloo")
R, rank = dist.get_world_size(), dist.get_rank()
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
P, N, W, k = 4, 24000, 4, 900
L = W * 32
rng = np.random.default_rng(2024)
codes = rng.integers(0, 2**32, (P, N, W), dtype=np.uint32)
codes[2] = codes[2][rng.integers(0, 6, N)]  # heavy ties crossing ranks
q = codes[:, 3].copy()
bounds = np.linspace(0, N, R + 1).astype(np.int64)
part = np.ascontiguousarray(codes[:, bounds[rank]:bounds[rank + 1]])
n_r = part.shape[1]
ctx = capi.Context(0)
peer = ctx.peer(R, rank, P, L)
handles = [None] * R
dist.all_gather_object(handles, peer.ipc_handle())
peer.open(handles)
cd = torch.from_numpy(part.view(np.int32)).to(dev)
qd = torch.from_numpy(q.view(np.int32)).to(dev)
nv = torch.full((P,), n_r, dtype=torch.int32, device=dev)
idx = torch.zeros((P, k), dtype=torch.int32, device=dev)
cnt = torch.zeros(P, dtype=torch.int32, device=dev)
off = torch.zeros(P, dtype=torch.int32, device=dev)
ok = True
for trial in range(3):  # epochs advance over both parity buffers
    dist.barrier()
    ctx.hamming_topk_sharded(peer, cd, n_r, L, qd, P, nv, 1, n_r, k, idx, cnt, off)
    torch.cuda.synchronize()
    ctx.check_device_error()
    mine = (idx.cpu().numpy().view(np.uint32), cnt.cpu().numpy(), off.cpu().numpy())
    allv = [None] * R
    dist.all_gather_object(allv, mine)
    if rank == 0:
        from oracle_lib import Oracle

        want = Oracle().retrieve_batch(codes, q, np.full(P, N, np.uint32), k)
        for p in range(P):
            cat = np.zeros(k, np.uint32)
            for r in range(R):
                ia, ca, oa = allv[r]
                cat[oa[p]:oa[p] + ca[p]] = ia[p, :ca[p]] + bounds[r]
            ok = ok and np.array_equal(cat, want[p])
peer.close()
ctx.close()
dist.barrier()
dist.destroy_process_group()
if rank == 0:
    print("MP_FUSED_SHARD", "OK" if ok else "MISMATCH")
    sys.exit(0 if ok else 1)
