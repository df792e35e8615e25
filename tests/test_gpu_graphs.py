"""CUDA-graph capture of the decode-time calls (the way a serving loop runs
them): after spl_reserve, one captured call replayed with new inputs written
in place must give exactly the eager results each time — the K3 per-problem
state resets itself, the fused sharded path's epoch advances on the device."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
from paper_2508_19740_b200 import capi  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def capture(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
        fn(s.cuda_stream)
    torch.cuda.synchronize()
    return g


@pytest.mark.parametrize("path,L", [("fused", 128), ("twopass", 128), ("twopass", 256)])
def test_graph_replay_hamming_topk(ctx, monkeypatch, path, L):
    if path == "twopass":
        monkeypatch.setenv("SPL_K3_PATH", "twopass")
    P, n, k = 8, 60000, 1200
    W = L // 32
    g = torch.Generator(device=DEV)
    g.manual_seed(L)
    codes = torch.randint(-2**31, 2**31 - 1, (P, n, W), generator=g, device=DEV, dtype=torch.int32)
    q = torch.zeros((P, W), dtype=torch.int32, device=DEV)
    nv = torch.full((P,), n, dtype=torch.int32, device=DEV)
    idx = torch.zeros((P, k), dtype=torch.int32, device=DEV)
    cnt = torch.zeros(P, dtype=torch.int32, device=DEV)
    ctx.hamming_topk(codes, n, L, q, P, nv, 1, n, k, idx, cnt)  # sizes the workspace
    ctx.reserve(P, n, L, k)
    graph = capture(lambda s: ctx.hamming_topk(codes, n, L, q, P, nv, 1, n, k, idx, cnt, s))
    ref_idx = torch.zeros_like(idx)
    ref_cnt = torch.zeros_like(cnt)
    for step in range(4):
        q.copy_(torch.randint(-2**31, 2**31 - 1, (P, W), generator=g, device=DEV, dtype=torch.int32))
        graph.replay()
        torch.cuda.synchronize()
        got = idx.clone()
        ctx.hamming_topk(codes, n, L, q, P, nv, 1, n, k, ref_idx, ref_cnt)
        torch.cuda.synchronize()
        ctx.check_device_error()
        assert torch.equal(got, ref_idx), step


def test_graph_replay_decode_step(ctx):
    B, H, n, d, L, k = 2, 4, 8192, 128, 128, 164
    rng = np.random.default_rng(3)
    w1 = (rng.standard_normal((H, d, d)) / np.sqrt(d)).astype(np.float32)
    w2 = (rng.standard_normal((H, d, L)) / np.sqrt(d)).astype(np.float32)
    hs = ctx.hasher(w1, np.zeros((H, d), np.float32), w2)
    g = torch.Generator(device=DEV)
    g.manual_seed(9)
    kc = torch.randn((B, H, n, d), generator=g, device=DEV).bfloat16()
    vc = torch.randn((B, H, n, d), generator=g, device=DEV).bfloat16()
    codes = torch.zeros((B, H, n, L // 32), dtype=torch.int32, device=DEV)
    hs.encode(kc.float(), B, n, codes)
    q = torch.zeros((B, H, d), device=DEV)
    kn = torch.zeros((B, H, d), device=DEV)
    vn = torch.zeros((B, H, d), device=DEV)
    nv = torch.full((B,), n, dtype=torch.int32, device=DEV)
    idx = torch.zeros((B * H, k), dtype=torch.int32, device=DEV)
    cnt = torch.zeros(B * H, dtype=torch.int32, device=DEV)
    out = torch.zeros((B, H, d), device=DEV)
    scale = float(1 / np.sqrt(d))

    def step(s=None):
        hs.decode_step(q, kn, vn, B, codes, kc, vc, capi.SPL_BF16, n, nv, n, k, scale, idx, cnt,
                       out, s)
    step()
    ctx.reserve(B * H, n, L, k, d)
    graph = capture(step)
    for it in range(3):
        for t in (q, kn, vn):
            t.copy_(torch.randn(t.shape, generator=g, device=DEV))
        graph.replay()
        torch.cuda.synchronize()
        gi, go = idx.clone(), out.clone()
        step()
        torch.cuda.synchronize()
        ctx.check_device_error()
        assert torch.equal(gi, idx), it
        assert torch.equal(go, out), it


def test_graph_replay_fused_sharded(ctx):
    """The exchange epoch lives on the device, so every replay is a new call."""
    P, n, L, k = 4, 40000, 128, 800
    g = torch.Generator(device=DEV)
    g.manual_seed(77)
    codes = torch.randint(-2**31, 2**31 - 1, (P, n, 4), generator=g, device=DEV, dtype=torch.int32)
    q = torch.zeros((P, 4), dtype=torch.int32, device=DEV)
    nv = torch.full((P,), n, dtype=torch.int32, device=DEV)
    idx = torch.zeros((P, k), dtype=torch.int32, device=DEV)
    cnt = torch.zeros(P, dtype=torch.int32, device=DEV)
    off = torch.zeros(P, dtype=torch.int32, device=DEV)
    peer = ctx.peer(1, 0, P, L)
    capi.Peer.connect_local(ctx, [peer])
    ctx.hamming_topk_sharded(peer, codes, n, L, q, P, nv, 1, n, k, idx, cnt, off)
    ctx.reserve(P, n, L, k)
    graph = capture(lambda s: ctx.hamming_topk_sharded(peer, codes, n, L, q, P, nv, 1, n, k, idx,
                                                       cnt, off, s))
    ref = torch.zeros_like(idx)
    rc = torch.zeros_like(cnt)
    for it in range(4):
        q.copy_(torch.randint(-2**31, 2**31 - 1, (P, 4), generator=g, device=DEV, dtype=torch.int32))
        graph.replay()
        torch.cuda.synchronize()
        got = idx.clone()
        ctx.hamming_topk(codes, n, L, q, P, nv, 1, n, k, ref, rc)
        torch.cuda.synchronize()
        ctx.check_device_error()
        assert torch.equal(got, ref), it
    peer.close()
