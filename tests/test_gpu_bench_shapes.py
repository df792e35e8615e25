"""Parity at the shapes bench.py measures, through the same entry points and
kernel variants the bench times (the launch log names them):

* config 2: one decode step of a LLaMA2-7B-shaped layer — B = 1, 32 heads,
  131,072-token bf16 K/V cache, 128-bit codes, k = budget_from_rate(0.02) =
  2,621 — spl_decode_step (K1 append + query encode, then the single-launch
  retrieval + attention k3_fused_attend);
* config 4: the batched step — B = 16 x 32 heads x 131,072 tokens, 256-bit
  codes, k = 2,621 (K1, two-pass K3, K4 gather).

Indices must equal the oracle's bit for bit (top_k_indices, bitcodes.cpp:
89-136, as hash_topk composes it, attention_eval.cpp:172-179); the appended
code row must equal the oracle's mlp_hash of the new key; the attention output
must be within max-abs 1e-3 of the oracle's sparse_attention
(attention_eval.cpp:234-264) fed the same bf16-rounded K/V values.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
from paper_2508_19740_b200 import capi  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
TOL_BF16 = 1e-3


def U(t):
    a = t.cpu().numpy()
    return a.view(np.uint32) if a.dtype == np.int32 else a


def _weights(rng, H, d, h, L):
    w1 = (rng.standard_normal((H, d, h)) / np.sqrt(d)).astype(np.float32)
    b1 = (0.1 * rng.standard_normal((H, h))).astype(np.float32)
    w2 = (rng.standard_normal((H, h, L)) / np.sqrt(h)).astype(np.float32)
    return w1, b1, w2


def _attention_check(oracle, q, kc, vc, idx_row, n, scale):
    """Oracle sparse attention of one problem over its selected rows U {own},
    evaluated on the compacted rows (same set, same order)."""
    rows = np.asarray(idx_row, np.int64)
    if rows.size == 0 or rows[-1] != n - 1:
        rows = np.append(rows, n - 1)
    sel = torch.from_numpy(rows).to(DEV)
    Ks = kc.index_select(0, sel).float().cpu().numpy()
    Vs = vc.index_select(0, sel).float().cpu().numpy()
    m = len(rows)
    return oracle.sparse_attention(q[None], Ks, Vs, np.float32(scale), np.array([m], np.uint32),
                                   [np.arange(m, dtype=np.uint32)])[0]


def _run_step(ctx, oracle, B, H, n, L, k, seed, expect_kernels, sample_att=None):
    d = 128
    rng = np.random.default_rng(seed)
    w1, b1, w2 = _weights(rng, H, d, d, L)
    hs = ctx.hasher(w1, b1, w2)
    g = torch.Generator(device=DEV)
    g.manual_seed(seed)
    W = L // 32
    codes = torch.randint(-2**31, 2**31 - 1, (B, H, n, W), generator=g, device=DEV, dtype=torch.int32)
    kc = torch.randn((B, H, n, d), generator=g, device=DEV).bfloat16()
    vc = torch.randn((B, H, n, d), generator=g, device=DEV).bfloat16()
    q = rng.standard_normal((B, H, d)).astype(np.float32)
    kn = rng.standard_normal((B, H, d)).astype(np.float32)
    vn = rng.standard_normal((B, H, d)).astype(np.float32)
    nvb = np.array([n - 37 * b for b in range(B)], np.uint32)  # ragged across the batch
    P = B * H
    idx = torch.full((P, k), -1, dtype=torch.int32, device=DEV)
    cnt = torch.zeros(P, dtype=torch.int32, device=DEV)
    out = torch.zeros((B, H, d), dtype=torch.float32, device=DEV)
    scale = float(1 / np.sqrt(d))
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    ctx.launch_log()
    hs.decode_step(t(q), t(kn), t(vn), B, codes, kc, vc, capi.SPL_BF16, n, t(nvb.view(np.int32)), n, k,
                   scale, idx, cnt, out)
    torch.cuda.synchronize()
    ctx.check_device_error()
    ran = ctx.launch_log()
    if expect_kernels is not None:
        assert ran == expect_kernels, ran
    got_codes = U(codes)
    # appended rows: code = exact hash of the new key, K/V rows = the new vectors (bf16)
    qcodes = np.zeros((P, W), np.uint32)
    for b in range(B):
        for h in range(H):
            nb = int(nvb[b])
            kcode = oracle.mlp_hash_packed(w1[h], b1[h], w2[h], kn[b, h][None])[0]
            assert np.array_equal(got_codes[b, h, nb - 1], kcode), (b, h)
            qcodes[b * H + h] = oracle.mlp_hash_packed(w1[h], b1[h], w2[h], q[b, h][None])[0]
    for b in range(B):
        nb = int(nvb[b])
        assert torch.equal(kc[b, :, nb - 1], t(kn[b]).bfloat16())
        assert torch.equal(vc[b, :, nb - 1], t(vn[b]).bfloat16())
    want = oracle.retrieve_batch(got_codes.reshape(P, n, W), qcodes, np.repeat(nvb, H), k)
    ia, ca = U(idx), U(cnt)
    assert np.array_equal(ca, np.minimum(k, np.repeat(nvb, H)).astype(np.uint32))
    assert np.array_equal(ia, want)
    o = out.cpu().numpy()
    probs = range(P) if sample_att is None else sample_att
    worst = 0.0
    for p in probs:
        b, h = divmod(p, H)
        ref = _attention_check(oracle, q[b, h], kc[b, h], vc[b, h], ia[p, :ca[p]], int(nvb[b]), scale)
        worst = max(worst, float(np.abs(o[b, h] - ref).max()))
    assert worst <= TOL_BF16, worst
    return worst


def test_decode_step_config2_full(ctx, oracle):
    """Config 2 exactly as bench.py's sparse_decode leg runs it."""
    n = 131072
    k = oracle.budget_from_rate(0.02, n)
    assert k == 2621
    _run_step(ctx, oracle, 1, 32, n, 128, k, 202, ["k1_encode_cluster", "k3_fused_attend"])


def test_decode_step_config2_two_launch_fallback(ctx, oracle, monkeypatch):
    """The K3 (+L2 prefetch) -> K4 flow the fused step replaces (kept for
    geometries the fused kernel does not cover), at the same full shape."""
    monkeypatch.setenv("SPL_DECODE_FUSED", "0")
    n = 131072
    k = oracle.budget_from_rate(0.02, n)
    _run_step(ctx, oracle, 1, 32, n, 128, k, 203, ["k1_encode_cluster", "k3_fused_pf", "k4_gather"])


def test_decode_step_config4_full(ctx, oracle):
    """Config 4: B = 16 x 32 heads x 131072 tokens, 256-bit codes (two-pass
    K3), all 512 index lists bit-exact, attention checked on 64 problems."""
    n = 131072
    k = oracle.budget_from_rate(0.02, n)
    sample = list(range(0, 512, 8))
    _run_step(ctx, oracle, 16, 32, n, 256, k, 404,
              ["k1_encode_cluster", "k3_scan", "k3_select", "k4_gather"], sample_att=sample)


@pytest.mark.parametrize("seed", list(range(12)))
def test_decode_step_random(ctx, oracle, seed):
    """Random decode-step geometries (batch, heads, cache length, code width,
    budget; ragged n_valid across the batch) through spl_decode_step, whichever
    kernels it picks: appended rows, indices and attention output as above."""
    rng = np.random.default_rng(1000 + seed)
    B = int(rng.integers(1, 4))
    H = int(rng.integers(1, 9))
    L = int(rng.choice([128, 128, 256]))
    n = int(rng.integers(37 * (B - 1) + 64, 20000))
    nmin = n - 37 * (B - 1)
    k = int(rng.choice([1, int(rng.integers(1, 64)), max(1, int(0.02 * n)), int(rng.integers(1, nmin + 1))]))
    k = min(k, nmin)
    _run_step(ctx, oracle, B, H, n, L, k, 2000 + seed, None)


@pytest.mark.parametrize("bad", ["nvalid0", "past_cap"])
def test_append_out_of_range_is_rejected_without_writes(ctx, bad):
    """An append slot outside [0, cap) (n_valid == 0 in a decode step, a full
    cache) raises a DimensionError through the device error word and writes
    nothing: the code / K / V caches sit between canary regions that must
    stay untouched (no wild store into a neighbouring head)."""
    B, H, cap, d, L = 2, 2, 256, 128, 128
    W = L // 32
    rng = np.random.default_rng(77)
    w1, b1, w2 = _weights(rng, H, d, d, L)
    hs = ctx.hasher(w1, b1, w2)
    pad = 4096
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    codes_big = torch.full((pad * 2 + B * H * cap * W,), 0x5A5A5A5A, dtype=torch.int32, device=DEV)
    kc_big = torch.full((pad * 2 + B * H * cap * d,), 7.0, dtype=torch.float32, device=DEV)
    vc_big = torch.full((pad * 2 + B * H * cap * d,), 9.0, dtype=torch.float32, device=DEV)
    codes = codes_big[pad:pad + B * H * cap * W].view(B, H, cap, W)
    kc = kc_big[pad:pad + B * H * cap * d].view(B, H, cap, d)
    vc = vc_big[pad:pad + B * H * cap * d].view(B, H, cap, d)
    before = (codes_big.clone(), kc_big.clone(), vc_big.clone())
    q = t(rng.standard_normal((B, H, d)).astype(np.float32))
    kn = t(rng.standard_normal((B, H, d)).astype(np.float32))
    vn = t(rng.standard_normal((B, H, d)).astype(np.float32))
    if bad == "nvalid0":
        nv = np.array([0, 0], np.int32)
    else:
        nv = np.array([cap + 1, cap + 5], np.int32)
    P, k = B * H, 8
    idx = torch.zeros((P, k), dtype=torch.int32, device=DEV)
    cnt = torch.zeros(P, dtype=torch.int32, device=DEV)
    out = torch.zeros((B, H, d), dtype=torch.float32, device=DEV)
    with pytest.raises(capi.DimensionError):
        hs.decode_step(q, kn, vn, B, codes, kc, vc, capi.SPL_F32, cap, t(nv), cap, k,
                       float(1 / np.sqrt(d)), idx, cnt, out)
        torch.cuda.synchronize()
        ctx.check_device_error()
    torch.cuda.synchronize()
    try:
        ctx.check_device_error()
    except capi.SpotlightError:
        pass
    for a, b in zip((codes_big, kc_big, vc_big), before):
        assert torch.equal(a[:pad], b[:pad]) and torch.equal(a[-pad:], b[-pad:])
    # no row of any head was written either
    assert torch.equal(codes_big, before[0])
    assert torch.equal(kc_big, before[1]) and torch.equal(vc_big, before[2])


def test_append_unaligned_inputs(ctx):
    """New K / V rows passed at addresses that are only 4-byte aligned: the
    encoder stages V with 4-byte asynchronous copies then (16-byte copies
    need 16-byte alignment); the appended rows and codes must be exact."""
    B, H, cap, d, L = 2, 3, 64, 128, 128
    W = L // 32
    rng = np.random.default_rng(78)
    w1, b1, w2 = _weights(rng, H, d, d, L)
    hs = ctx.hasher(w1, b1, w2)
    kn = rng.standard_normal((B, H, d)).astype(np.float32)
    vn = rng.standard_normal((B, H, d)).astype(np.float32)
    kbuf = torch.zeros(B * H * d + 1, dtype=torch.float32, device=DEV)
    vbuf = torch.zeros(B * H * d + 1, dtype=torch.float32, device=DEV)
    kbuf[1:] = torch.from_numpy(kn.ravel()).to(DEV)
    vbuf[1:] = torch.from_numpy(vn.ravel()).to(DEV)
    k_view, v_view = kbuf[1:].view(B, H, d), vbuf[1:].view(B, H, d)  # 4-byte aligned only
    codes = torch.zeros((B, H, cap, W), dtype=torch.int32, device=DEV)
    kc = torch.zeros((B, H, cap, d), dtype=torch.float32, device=DEV)
    vc = torch.zeros((B, H, cap, d), dtype=torch.float32, device=DEV)
    pos = torch.tensor([5, 17], dtype=torch.int32, device=DEV)
    hs.encode_append(k_view, v_view, B, codes, kc, vc, capi.SPL_F32, cap, pos)
    torch.cuda.synchronize()
    ctx.check_device_error()
    kc_h, vc_h = kc.cpu().numpy(), vc.cpu().numpy()
    for b, slot in ((0, 5), (1, 17)):
        assert np.array_equal(kc_h[b, :, slot], kn[b]) and np.array_equal(vc_h[b, :, slot], vn[b])
    ref = torch.zeros((B, H, 1, W), dtype=torch.int32, device=DEV)
    hs.encode(torch.from_numpy(kn[:, :, None]).to(DEV), B, 1, ref)
    torch.cuda.synchronize()
    got = codes.cpu().numpy()
    want = ref.cpu().numpy()
    assert np.array_equal(got[0, :, 5], want[0, :, 0]) and np.array_equal(got[1, :, 17], want[1, :, 0])


def test_sparse_attend_unaligned_caches(ctx):
    """K / V caches that are only 4-byte aligned: f32 takes the generic
    kernel and gives the aligned result (to rounding); bf16 is rejected."""
    H, n, d, k = 3, 500, 128, 40
    rng = np.random.default_rng(79)
    kk = rng.standard_normal((H * n * d,)).astype(np.float32)
    vv = rng.standard_normal((H * n * d,)).astype(np.float32)
    q = torch.from_numpy(rng.standard_normal((1, H, d)).astype(np.float32)).to(DEV)
    idx = torch.from_numpy(np.stack([np.sort(rng.choice(n - 1, k, replace=False)) for _ in range(H)])
                           .astype(np.int32)).to(DEV)
    cnt = torch.full((H,), k, dtype=torch.int32, device=DEV)
    nv = torch.full((1,), n, dtype=torch.int32, device=DEV)
    scale = float(1 / np.sqrt(d))
    outs = []
    for off in (0, 1):
        kb = torch.zeros(H * n * d + 4, dtype=torch.float32, device=DEV)
        vb = torch.zeros(H * n * d + 4, dtype=torch.float32, device=DEV)
        kb[off:off + H * n * d] = torch.from_numpy(kk).to(DEV)
        vb[off:off + H * n * d] = torch.from_numpy(vv).to(DEV)
        kc, vc = kb[off:off + H * n * d].view(1, H, n, d), vb[off:off + H * n * d].view(1, H, n, d)
        out = torch.zeros((1, H, d), dtype=torch.float32, device=DEV)
        ctx.sparse_attend(q, kc, vc, capi.SPL_F32, n, d, H, idx, k, cnt, nv, H, scale, out)
        torch.cuda.synchronize()
        ctx.check_device_error()
        outs.append(out.cpu().numpy())
    assert np.abs(outs[0] - outs[1]).max() <= 1e-5
    kb16 = torch.zeros(H * n * d + 8, dtype=torch.bfloat16, device=DEV)
    kc16 = kb16[1:1 + H * n * d].view(1, H, n, d)
    with pytest.raises(capi.DimensionError, match="16-byte aligned"):
        ctx.sparse_attend(q, kc16, kc16, capi.SPL_BF16, n, d, H, idx, k, cnt, nv, H, scale,
                          torch.zeros((1, H, d), dtype=torch.float32, device=DEV))
