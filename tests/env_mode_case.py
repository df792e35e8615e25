"""Parity payload for tests/test_gpu_env_modes.py: the retrieval, K4 sparse
attention (bf16 and f32 K/V) and one served decode step, checked against the
C oracle, under whatever SPL_* launch-mode variables the parent set (they are
read once per process by libspl, hence the subprocess). Exit 0 = all equal.

Indices bit-exact (top_k_indices, bitcodes.cpp:89-136, as hash_topk composes
it, attention_eval.cpp:172-179); attention within max-abs 1e-5 (f32 K/V) /
1e-3 (bf16 K/V, the oracle fed the same bf16-rounded values)
(sparse_attention, attention_eval.cpp:234-264)."""
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
rng = np.random.default_rng(11)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
U = lambda t: t.cpu().numpy().view(np.uint32)  # noqa: E731
H, n, d, L, k = 4, 20000, 128, 128, 400
scale = float(1 / np.sqrt(d))
fails = []

w1 = (rng.standard_normal((H, d, d)) / np.sqrt(d)).astype(np.float32)
b1 = (0.1 * rng.standard_normal((H, d))).astype(np.float32)
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

# retrieval
idx = torch.zeros((H, k), dtype=torch.int32, device=dev)
cnt = torch.zeros(H, dtype=torch.int32, device=dev)
ctx.hamming_topk(codes, n, L, qc, H, nv, H, n, k, idx, cnt)
torch.cuda.synchronize()
want = orc.retrieve_batch(U(codes)[0], U(qc)[0], np.full(H, n, np.uint32), k)
if not np.array_equal(U(idx), want):
    fails.append("hamming_topk indices")

# K4 over bf16 and f32 K/V
kb = T(keys).bfloat16()
vb = T(vals).bfloat16()
kf, vf = kb.float().cpu().numpy(), vb.float().cpu().numpy()
for dtype, kk, vv, kref, vref, tol in ((capi.SPL_BF16, kb, vb, kf, vf, 1e-3),
                                      (capi.SPL_F32, T(keys), T(vals), keys, vals, 1e-5)):
    out = torch.zeros((1, H, d), dtype=torch.float32, device=dev)
    ctx.sparse_attend(T(q), kk, vv, dtype, n, d, H, idx, k, cnt, nv, H, scale, out)
    torch.cuda.synchronize()
    for h in range(H):
        ref = orc.sparse_attention(q[0, h][None], kref[0, h], vref[0, h], np.float32(scale),
                                   np.array([n], np.uint32), [want[h]])
        err = float(np.abs(out[0, h].cpu().numpy() - ref[0]).max())
        if err > tol:
            fails.append(f"sparse_attend dtype {dtype} head {h}: {err}")

# one served decode step (append at row nvd - 1 + fused retrieval + bf16 attention)
nvd = n - 7
kn = rng.standard_normal((1, H, d)).astype(np.float32)
vn = rng.standard_normal((1, H, d)).astype(np.float32)
cd = codes.clone()
di = torch.zeros_like(idx)
dc = torch.zeros_like(cnt)
do = torch.zeros((1, H, d), dtype=torch.float32, device=dev)
hs.decode_step(T(q), T(kn), T(vn), 1, cd, kb, vb, capi.SPL_BF16, n,
               torch.full((1,), nvd, dtype=torch.int32, device=dev), n, k, scale, di, dc, do,
               torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
ctx.check_device_error()
kf, vf = kb.float().cpu().numpy(), vb.float().cpu().numpy()
cdn = U(cd)[0]
dwant = orc.retrieve_batch(cdn[:, :nvd].copy(), U(qc)[0], np.full(H, nvd, np.uint32), k)
if not np.array_equal(U(di), dwant):
    fails.append("decode_step indices")
for h in range(H):
    if not np.array_equal(cdn[h, nvd - 1], orc.mlp_hash_packed(w1[h], b1[h], w2[h], kn[0, h][None])[0]):
        fails.append(f"decode_step appended code head {h}")
    ref = orc.sparse_attention(q[0, h][None], kf[0, h], vf[0, h], np.float32(scale),
                               np.array([nvd], np.uint32), [dwant[h]])
    err = float(np.abs(do[0, h].cpu().numpy() - ref[0]).max())
    if err > 1e-3:
        fails.append(f"decode_step attention head {h}: {err}")
ctx.close()
print("env mode case:", "OK" if not fails else "; ".join(fails))
sys.exit(1 if fails else 0)
