"""GPU parity: the sm_100a kernels through the C-ABI vs the CPU oracle and the
reference's golden fixtures. Indices and codes must be bit-exact; attention
output within max-abs 1e-5 (f32 K/V) / 1e-3 (bf16 K/V, oracle fed the same
bf16-rounded values) — the tolerances north_star states."""
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
from paper_2508_19740_b200 import capi  # noqa: E402

pytestmark = pytest.mark.gpu
G = np.load(Path(__file__).parent / "golden" / "reference_golden.npz")
DEV = "cuda:0"


def T(a, dtype=None):
    a = np.ascontiguousarray(a)
    t = torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a)
    return t.to(DEV)


def U(t):
    a = t.cpu().numpy()
    return a.view(np.uint32) if a.dtype == np.int32 else a


@pytest.fixture(params=["fused", "twopass"])
def k3_path(request, monkeypatch):
    """Run K3 tests through both the single-launch cooperative kernel and the
    two-kernel path (SPL_K3_PATH is read by libspl at every call)."""
    if request.param == "twopass":
        monkeypatch.setenv("SPL_K3_PATH", "twopass")
    else:
        monkeypatch.delenv("SPL_K3_PATH", raising=False)
    return request.param


def run_topk(ctx, codes, q, n_valid, k, stride_rows=None, nvalid_div=1, n_max=None):
    """codes [P][cap][W] (or [cap][W] shared), q [P][W] -> list of index arrays."""
    codes = np.ascontiguousarray(codes, np.uint32)
    q = np.ascontiguousarray(q, np.uint32)
    P, W = q.shape
    L = W * 32
    if stride_rows is None:
        stride_rows = codes.shape[1]
    n_valid = np.ascontiguousarray(n_valid, np.uint32)
    if n_max is None:
        n_max = int(n_valid.max()) if n_valid.size else 0
    idx = torch.full((P, k), -1, dtype=torch.int32, device=DEV)
    cnt = torch.zeros(P, dtype=torch.int32, device=DEV)
    ctx.hamming_topk(T(codes), stride_rows, L, T(q), P, T(n_valid), nvalid_div, n_max, k, idx, cnt)
    torch.cuda.synchronize()
    ctx.check_device_error()
    idx, cnt = U(idx), U(cnt)
    return [idx[p, :cnt[p]] for p in range(P)]


# ------------------------------------------------------------ K3 hamming top-k
@pytest.mark.parametrize("ci", list(range(6)))
def test_golden_topk(ctx, k3_path, ci):
    codes, q = G[f"topk{ci}_codes"], G[f"topk{ci}_q"]
    k = int(G[f"topk{ci}_k"][0])
    n = codes.shape[0]
    got = run_topk(ctx, codes[None], q[None], [n], k)
    assert np.array_equal(got[0], G[f"topk{ci}_idx"])


@pytest.mark.parametrize("L", [32, 64, 96, 128, 160, 256, 512])
def test_topk_vs_oracle_widths(ctx, k3_path, oracle, L):
    rng = np.random.default_rng(L)
    P, n, W = 3, 20000, L // 32
    codes = rng.integers(0, 2**32, (P, n, W), dtype=np.uint64).astype(np.uint32)
    codes[1] = codes[1][rng.integers(0, 7, n)]  # heavy ties
    q = codes[np.arange(P), rng.integers(0, n, P)]
    nv = np.array([n, n - 3, 4097], np.uint32)
    for k in (1, 37, 400, 4097):
        got = run_topk(ctx, codes, q, nv, k)
        want = oracle.retrieve_batch(codes, q, nv, k)
        for p in range(P):
            kk = min(k, int(nv[p]))
            assert np.array_equal(got[p], want[p, :kk]), (L, k, p)


def test_topk_edge_cases(ctx, k3_path, oracle):
    rng = np.random.default_rng(5)
    codes = rng.integers(0, 2**32, (4, 300, 4), dtype=np.uint64).astype(np.uint32)
    q = codes[:, 0].copy()
    # k > n_valid, n_valid = 1, identical rows (all ties), k == n
    codes[2] = codes[2, :1]
    nv = np.array([300, 1, 300, 257], np.uint32)
    for k in (1, 256, 257, 300, 1000):
        got = run_topk(ctx, codes, q, nv, k)
        want = oracle.retrieve_batch(codes, q, nv, k)
        for p in range(4):
            kk = min(k, int(nv[p]))
            assert np.array_equal(got[p], want[p, :kk])


@pytest.mark.parametrize("L", [64, 128, 256])
def test_topk_low_threshold_fallback(ctx, k3_path, oracle, L):
    """The fused kernel counts only scores >= L/2 on its first pass; problems
    whose k-th score is lower take the in-kernel fallback (low bins recounted
    from the on-chip scores). Mixed batch: problems 0 and 2 are anti-correlated
    with their query (all scores ~0.2 L), problem 1 is a normal random cache,
    problem 3 has k = 0.9 n."""
    rng = np.random.default_rng(100 + L)
    P, n, W = 4, 30000, L // 32
    q = rng.integers(0, 2**32, (P, W), dtype=np.uint64).astype(np.uint32)
    codes = rng.integers(0, 2**32, (P, n, W), dtype=np.uint64).astype(np.uint32)
    for p in (0, 2):
        keep = np.zeros((n, W), np.uint32)  # ~20% of bits agree with q
        for _ in range(3):
            keep |= rng.integers(0, 2**32, (n, W), dtype=np.uint64).astype(np.uint32)
        keep = ~keep  # P(bit) = 1/8
        codes[p] = (~q[p])[None, :] ^ (keep & rng.integers(0, 2**32, (n, W), dtype=np.uint64).astype(np.uint32))
    nv = np.array([n, n, n - 5, n], np.uint32)
    for k in (10, 3000, 27000):
        got = run_topk(ctx, codes, q, nv, k)
        want = oracle.retrieve_batch(codes, q, nv, k)
        for p in range(P):
            kk = min(k, int(nv[p]))
            assert np.array_equal(got[p], want[p, :kk]), (L, k, p)


@pytest.mark.parametrize("L", [256, 512])
def test_topk_near_duplicates_top_bins(ctx, k3_path, oracle, L):
    """Thresholds in the top two bins. The two-pass path stores L = 256
    scores as u8 clamped to 255, so T >= 255 must take the exact re-read of
    the codes: rows equal to the query (score L), rows one bit away (L - 1),
    the rest random, with k landing on each bin and its ties."""
    rng = np.random.default_rng(200 + L)
    P, n, W = 3, 20000, L // 32
    codes = rng.integers(0, 2**32, (P, n, W), dtype=np.uint64).astype(np.uint32)
    q = rng.integers(0, 2**32, (P, W), dtype=np.uint64).astype(np.uint32)
    for p in range(P):
        dup = rng.choice(n, 1200, replace=False)
        codes[p, dup[:500]] = q[p]
        near = np.repeat(q[p][None], 700, axis=0)
        word = rng.integers(0, W, 700)
        near[np.arange(700), word] ^= (np.uint32(1) << rng.integers(0, 32, 700).astype(np.uint32))
        codes[p, dup[500:]] = near
    nv = np.array([n, n - 7, 15000], np.uint32)
    for k in (1, 300, 500, 800, 1200, 1500):
        got = run_topk(ctx, codes, q, nv, k)
        want = oracle.retrieve_batch(codes, q, nv, k)
        for p in range(P):
            kk = min(k, int(nv[p]))
            assert np.array_equal(got[p], want[p, :kk]), (L, k, p)


def test_topk_fused_cooperative_optin(ctx, oracle, monkeypatch):
    """SPL_K3_COOP=1 launches the fused kernel cooperatively (co-residency
    guaranteed by the driver); results are the same as the plain launch."""
    rng = np.random.default_rng(77)
    P, n, W = 5, 40000, 4
    codes = rng.integers(0, 2**32, (P, n, W), dtype=np.uint64).astype(np.uint32)
    q = rng.integers(0, 2**32, (P, W), dtype=np.uint64).astype(np.uint32)
    nv = np.array([n, n - 1, 3000, 1, n], np.uint32)
    want = oracle.retrieve_batch(codes, q, nv, 800)
    plain = run_topk(ctx, codes, q, nv, 800)
    monkeypatch.setenv("SPL_K3_COOP", "1")
    coop = run_topk(ctx, codes, q, nv, 800)
    for p in range(P):
        kk = min(800, int(nv[p]))
        assert np.array_equal(plain[p], want[p, :kk])
        assert np.array_equal(coop[p], want[p, :kk])


def test_topk_k_zero_rejected(ctx):
    codes = np.zeros((1, 10, 4), np.uint32)
    with pytest.raises(capi.DimensionError):
        run_topk(ctx, codes, codes[:, 0], [10], 0)
    with pytest.raises(capi.DimensionError):
        idx = torch.zeros(4, dtype=torch.int32, device=DEV)
        ctx.hamming_topk(T(codes), 10, 33, T(codes[:, 0]), 1, T(np.array([10], np.uint32)), 1, 10,
                         4, idx, idx)


@pytest.mark.parametrize("n,k", [(3000, 64), (600, 24), (1000, 1)])
def test_topk_shared_cache_causal(ctx, k3_path, oracle, n, k):
    """hash_topk's layout: q queries share one cache, query r sees rows < r+1.
    P = n problems > the fused plan's CTA target, so segments straddle
    problems and most small problems take the low-bin fallback."""
    rng = np.random.default_rng(9 + n)
    W = 4
    codes = rng.integers(0, 2**32, (n, W), dtype=np.uint64).astype(np.uint32)
    q = rng.integers(0, 2**32, (n, W), dtype=np.uint64).astype(np.uint32)
    offs = np.arange(1, n + 1, dtype=np.uint32)
    got = run_topk(ctx, codes[None], q, offs, k, stride_rows=0, n_max=n)
    bad = []
    for r in range(n):
        s = oracle.nxor_scores(q[r], codes, int(offs[r]))
        if not np.array_equal(got[r], oracle.top_k(s, min(k, int(offs[r])))):
            bad.append(r)
    assert not bad, (len(bad), bad[:10], got[bad[0]][:8].tolist(),
                     oracle.top_k(oracle.nxor_scores(q[bad[0]], codes, int(offs[bad[0]])),
                                  min(k, int(offs[bad[0]])))[:8].tolist())


def test_topk_nvalid_per_batch(ctx, k3_path, oracle):
    rng = np.random.default_rng(10)
    B, H, cap, W = 3, 4, 5000, 4
    codes = rng.integers(0, 2**32, (B * H, cap, W), dtype=np.uint64).astype(np.uint32)
    q = rng.integers(0, 2**32, (B * H, W), dtype=np.uint64).astype(np.uint32)
    nvb = np.array([5000, 123, 4000], np.uint32)
    got = run_topk(ctx, codes, q, nvb, 100, nvalid_div=H, n_max=cap)
    want = oracle.retrieve_batch(codes, q, np.repeat(nvb, H), 100)
    for p in range(B * H):
        assert np.array_equal(got[p], want[p, :min(100, nvb[p // H])])


def test_topk_config3_shape(ctx, k3_path, oracle):
    """Headline shape: 32 heads x 524288 rows x 128-bit codes, k = 10485."""
    rng = np.random.default_rng(3)
    P, n, W = 32, 524288, 4
    codes = rng.integers(0, 2**32, (P, n, W), dtype=np.uint64).astype(np.uint32)
    q = rng.integers(0, 2**32, (P, W), dtype=np.uint64).astype(np.uint32)
    k = oracle.budget_from_rate(0.02, n)
    nv = np.full(P, n, np.uint32)
    got = run_topk(ctx, codes, q, nv, k)
    want = oracle.retrieve_batch(codes, q, nv, k)
    for p in range(P):
        assert np.array_equal(got[p], want[p])


def test_topk_config4_shape_l256(ctx, oracle):
    """Config-4-shaped: batched problems, 256-bit codes (two-pass path, u8
    scores clamped at 255, windowed counters)."""
    rng = np.random.default_rng(4)
    B, H, n, W = 2, 32, 131072, 8
    codes = rng.integers(0, 2**32, (B * H, n, W), dtype=np.uint64).astype(np.uint32)
    q = rng.integers(0, 2**32, (B * H, W), dtype=np.uint64).astype(np.uint32)
    k = oracle.budget_from_rate(0.02, n)
    nvb = np.array([n, n - 1000], np.uint32)
    got = run_topk(ctx, codes, q, nvb, k, nvalid_div=H, n_max=n)
    want = oracle.retrieve_batch(codes, q, np.repeat(nvb, H), k)
    for p in range(B * H):
        assert np.array_equal(got[p], want[p])


def test_topk_repeatable(ctx, k3_path):
    rng = np.random.default_rng(12)
    codes = rng.integers(0, 2**32, (8, 50000, 4), dtype=np.uint64).astype(np.uint32)
    q = codes[:, 5]
    nv = np.full(8, 50000, np.uint32)
    a = run_topk(ctx, codes, q, nv, 999)
    for _ in range(3):
        b = run_topk(ctx, codes, q, nv, 999)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))


# ------------------------------------------------------------ bitcodes misc
def test_pack_unpack_golden(ctx):
    for d in (32, 64, 128, 256):
        bits = G[f"pack_bits_in_{d}"]
        out = torch.zeros((bits.shape[0], d // 32), dtype=torch.int32, device=DEV)
        ctx.pack_bits(T(bits), out)
        assert np.array_equal(U(out), G[f"pack_bits_out_{d}"])
        back = torch.zeros(bits.shape, dtype=torch.uint8, device=DEV)
        ctx.unpack_bits(out, d, back)
        assert np.array_equal(back.cpu().numpy(), bits)


def test_nxor_scores_and_generic_topk(ctx, oracle):
    for ci in range(6):
        codes, q = G[f"topk{ci}_codes"], G[f"topk{ci}_q"]
        n, W = codes.shape
        sc = torch.zeros(n, dtype=torch.int32, device=DEV)
        ctx.nxor_scores(T(codes), 0, W * 32, T(q[None]), 1, T(np.array([n], np.uint32)), 1, n, sc, n)
        assert np.array_equal(sc.cpu().numpy(), G[f"topk{ci}_scores"])
        k = int(G[f"topk{ci}_k"][0])
        idx = torch.zeros(k, dtype=torch.int32, device=DEV)
        ctx.top_k(sc, 0, 1, n, n, k, idx)
        assert np.array_equal(U(idx), G[f"topk{ci}_idx"])
    rng = np.random.default_rng(1)
    for dt in (np.float32, np.float64):
        s = rng.standard_normal(5000).astype(dt)
        s[::7] = s[3]  # ties
        s[10] = -0.0
        s[11] = 0.0
        for k in (1, 50, 4999):
            idx = torch.zeros(k, dtype=torch.int32, device=DEV)
            ctx.top_k(torch.from_numpy(s).to(DEV), 1 if dt == np.float32 else 2, 1, 5000, 5000, k, idx)
            want = sorted(sorted(range(5000), key=lambda i: (-float(s[i]), i))[:k])
            assert list(U(idx)) == want
    with pytest.raises(capi.DimensionError, match="top_k_indices: k=0 out of range for n=3"):
        ctx.top_k(torch.zeros(3, dtype=torch.int32, device=DEV), 0, 1, 3, 3, 0,
                  torch.zeros(1, dtype=torch.int32, device=DEV))


# ------------------------------------------------------------ K1 exact encoder
@pytest.mark.parametrize("tag", ["c128", "c256", "small", "bias"])
def test_encode_exact_bit_exact_golden(ctx, tag):
    w1, b1, w2, x = (G[f"mlp_{tag}_{n}"] for n in ("w1", "b1", "w2", "x"))
    hs = ctx.hasher(w1[None], b1[None], w2[None])
    m, L = x.shape[0], w2.shape[1]
    pre = torch.zeros((m, L), dtype=torch.float32, device=DEV)
    hs.mlp_forward(T(x), 1, m, pre)
    assert np.array_equal(pre.cpu().numpy().view(np.uint32), G[f"mlp_{tag}_pre"].view(np.uint32))
    codes = torch.zeros((m, L // 32), dtype=torch.int32, device=DEV)
    hs.encode(T(x), 1, m, codes)
    assert np.array_equal(U(codes), G[f"mlp_{tag}_codes"])


def test_encode_exact_multihead_vs_oracle(ctx, oracle, ref):
    rng = np.random.default_rng(21)
    H, d, h, L, B, m = 4, 128, 128, 256, 3, 5
    ws = [ref.mlp_gaussian_init(d, h, L, 64.0, ref.derive_seed(0, i)) for i in range(H)]
    w1 = np.stack([w[0] for w in ws])
    b1 = np.stack([rng.standard_normal(h).astype(np.float32) * 0.1 for _ in ws])
    w2 = np.stack([w[2] for w in ws])
    x = rng.standard_normal((B, H, m, d)).astype(np.float32)
    hs = ctx.hasher(w1, b1, w2)
    codes = torch.zeros((B, H, m, L // 32), dtype=torch.int32, device=DEV)
    hs.encode(T(x), B, m, codes)
    got = U(codes)
    for b in range(B):
        for hd in range(H):
            want = oracle.mlp_hash_packed(w1[hd], b1[hd], w2[hd], x[b, hd])
            assert np.array_equal(got[b, hd], want)


@pytest.mark.parametrize("d,h,L", [(64, 256, 128), (96, 128, 256), (128, 384, 128), (36, 128, 128)])
def test_encode_exact_cluster_generic_dims(ctx, oracle, ref, d, h, L):
    """The cluster encoder's runtime-length path (d or h != 128): lane-major
    rotated weight rows (spl_hasher_create) for other row lengths, incl. a
    chunk count (d / 4 = 9) that does not divide 32 — codes bit-exact."""
    rng = np.random.default_rng(23 + d + h)
    H, B, m = 2, 2, 9
    ws = [ref.mlp_gaussian_init(d, h, L, 64.0, ref.derive_seed(3, i)) for i in range(H)]
    w1 = np.stack([w[0] for w in ws])
    b1 = np.stack([rng.standard_normal(h).astype(np.float32) * 0.1 for _ in ws])
    w2 = np.stack([w[2] for w in ws])
    x = rng.standard_normal((B, H, m, d)).astype(np.float32)
    hs = ctx.hasher(w1, b1, w2)
    codes = torch.zeros((B, H, m, L // 32), dtype=torch.int32, device=DEV)
    hs.encode(T(x), B, m, codes)
    got = U(codes)
    for b in range(B):
        for hd in range(H):
            assert np.array_equal(got[b, hd], oracle.mlp_hash_packed(w1[hd], b1[hd], w2[hd], x[b, hd]))


def test_encode_linear_d128(ctx, oracle, ref):
    """Linear hasher with d = 128: the cluster encoder's unrolled (DN = 128)
    layer with the projection as its only layer."""
    rng = np.random.default_rng(24)
    proj = np.stack([ref.qr_rotation_init(128, 7 + i) for i in range(2)])
    x = rng.standard_normal((1, 2, 17, 128)).astype(np.float32)
    hs = ctx.hasher(proj, kind=capi.SPL_HASHER_LINEAR)
    codes = torch.zeros((1, 2, 17, 4), dtype=torch.int32, device=DEV)
    hs.encode(T(x), 1, 17, codes)
    for hd in range(2):
        assert np.array_equal(U(codes)[0, hd], oracle.linear_hash_packed(proj[hd], x[0, hd]))


def test_encode_linear(ctx, oracle, ref):
    rng = np.random.default_rng(22)
    proj = np.stack([ref.qr_rotation_init(64, 5 + i) for i in range(2)])
    x = rng.standard_normal((1, 2, 33, 64)).astype(np.float32)
    hs = ctx.hasher(proj, kind=capi.SPL_HASHER_LINEAR)
    codes = torch.zeros((1, 2, 33, 2), dtype=torch.int32, device=DEV)
    hs.encode(T(x), 1, 33, codes)
    for hd in range(2):
        assert np.array_equal(U(codes)[0, hd], oracle.linear_hash_packed(proj[hd], x[0, hd]))


def test_encode_non_finite_raises(ctx):
    w1 = np.ones((1, 8, 8), np.float32)
    hs = ctx.hasher(w1, np.zeros((1, 8), np.float32), np.ones((1, 8, 32), np.float32))
    x = np.zeros((1, 1, 2, 8), np.float32)
    x[0, 0, 1, 3] = np.inf
    codes = torch.zeros((2, 1), dtype=torch.int32, device=DEV)
    hs.encode(T(x), 1, 2, codes)
    with pytest.raises(capi.NumericError):
        ctx.check_device_error()
    ctx.check_device_error()  # cleared
    with pytest.raises(capi.NumericError):
        bad = w1.copy()
        bad[0, 0, 0] = np.nan
        ctx.hasher(bad, np.zeros((1, 8), np.float32), np.ones((1, 8, 32), np.float32))


# ------------------------------------------------------------ K4 sparse attention
def _attend(ctx, Q, K, V, picks, offs, kv_dtype):
    """Q [P][d]; K/V [P][n][d]; picks list of sorted arrays; offs n_valid per problem."""
    P, n, d = K.shape
    kmax = max(1, max(len(p) for p in picks))
    idx = np.zeros((P, kmax), np.uint32)
    cnt = np.array([len(p) for p in picks], np.uint32)
    for i, p in enumerate(picks):
        idx[i, :len(p)] = p
    tdt = torch.float32 if kv_dtype == capi.SPL_F32 else torch.bfloat16
    kc = torch.from_numpy(K).to(DEV).to(tdt)
    vc = torch.from_numpy(V).to(DEV).to(tdt)
    out = torch.zeros((P, d), dtype=torch.float32, device=DEV)
    ctx.sparse_attend(T(Q), kc, vc, kv_dtype, n, d, P, T(idx), kmax, T(cnt), T(np.asarray(offs, np.uint32)),
                      1, float(1 / np.sqrt(d)), out)
    torch.cuda.synchronize()
    return out.cpu().numpy(), kc.float().cpu().numpy(), vc.float().cpu().numpy()


def test_sparse_attention_golden_f32(ctx):
    po = G["att_picked_off"]
    picks = [G["att_picked"][po[i]:po[i + 1]] for i in range(len(po) - 1)]
    Q, K, V, offs = G["att_Q"], G["att_K"], G["att_V"], G["att_offs"]
    P = Q.shape[0]
    got, _, _ = _attend(ctx, Q, np.broadcast_to(K, (P,) + K.shape).copy(),
                        np.broadcast_to(V, (P,) + V.shape).copy(), picks, offs, capi.SPL_F32)
    assert np.abs(got - G["att_out"]).max() <= 1e-5


@pytest.mark.parametrize("d", [64, 128, 256])
@pytest.mark.parametrize("kv", ["f32", "bf16"])
def test_sparse_attention_vs_oracle(ctx, oracle, d, kv):
    rng = np.random.default_rng(d)
    P, n = 6, 4096
    K = rng.standard_normal((P, n, d)).astype(np.float32)
    V = rng.standard_normal((P, n, d)).astype(np.float32)
    Q = rng.standard_normal((P, d)).astype(np.float32) * 2
    offs = np.array([4096, 4096, 100, 1, 3000, 2], np.uint32)
    sizes = [81, 4096, 7, 1, 2999, 1]
    picks = [np.sort(rng.choice(int(o), min(s, int(o)), replace=False)).astype(np.uint32)
             for o, s in zip(offs, sizes)]
    kvd = capi.SPL_F32 if kv == "f32" else capi.SPL_BF16
    got, Kr, Vr = _attend(ctx, Q, K, V, picks, offs, kvd)
    for p in range(P):
        want = oracle.sparse_attention(Q[p:p + 1], Kr[p], Vr[p], np.float32(1 / np.sqrt(d)),
                                       offs[p:p + 1], [picks[p]])
        tol = 1e-5 if kv == "f32" else 1e-3
        assert np.abs(got[p] - want[0]).max() <= tol, (p, np.abs(got[p] - want[0]).max())


# ------------------------------------------------------------ decode step
@pytest.mark.parametrize("kv", ["f32", "bf16"])
def test_decode_step_vs_oracle(ctx, oracle, ref, kv):
    rng = np.random.default_rng(31)
    B, H, d, L, cap = 2, 4, 128, 128, 6000
    ws = [ref.mlp_gaussian_init(d, d, L, 64.0, ref.derive_seed(0, i)) for i in range(H)]
    w1, b1, w2 = (np.stack([w[j] for w in ws]) for j in range(3))
    hs = ctx.hasher(w1, b1, w2)
    nvb = np.array([5000, 3333], np.uint32)
    Kh = rng.standard_normal((B, H, cap, d)).astype(np.float32)
    Vh = rng.standard_normal((B, H, cap, d)).astype(np.float32)
    # existing cache: codes of rows < n-1 (the step appends row n-1)
    codes = np.zeros((B, H, cap, L // 32), np.uint32)
    for b in range(B):
        for hd in range(H):
            codes[b, hd, :nvb[b] - 1] = oracle.mlp_hash_packed(w1[hd], b1[hd], w2[hd], Kh[b, hd, :nvb[b] - 1])
    q = rng.standard_normal((B, H, d)).astype(np.float32)
    k_new = rng.standard_normal((B, H, d)).astype(np.float32)
    v_new = rng.standard_normal((B, H, d)).astype(np.float32)
    tdt = torch.float32 if kv == "f32" else torch.bfloat16
    kvd = capi.SPL_F32 if kv == "f32" else capi.SPL_BF16
    kc = torch.from_numpy(Kh).to(DEV).to(tdt)
    vc = torch.from_numpy(Vh).to(DEV).to(tdt)
    cd = T(codes)
    k = 100
    idx = torch.zeros((B * H, k), dtype=torch.int32, device=DEV)
    cnt = torch.zeros(B * H, dtype=torch.int32, device=DEV)
    out = torch.zeros((B, H, d), dtype=torch.float32, device=DEV)
    scale = float(1 / np.sqrt(d))
    hs.decode_step(T(q), T(k_new), T(v_new), B, cd, kc, vc, kvd, cap, T(nvb), cap, k, scale, idx, cnt, out)
    torch.cuda.synchronize()
    ctx.check_device_error()
    idx, cnt, out = U(idx), U(cnt), out.cpu().numpy()
    Kr, Vr = kc.float().cpu().numpy(), vc.float().cpu().numpy()
    got_codes = U(cd)
    for b in range(B):
        n = int(nvb[b])
        for hd in range(H):
            p = b * H + hd
            kn = oracle.mlp_hash_packed(w1[hd], b1[hd], w2[hd], k_new[b, hd][None])[0]
            assert np.array_equal(got_codes[b, hd, n - 1], kn)
            assert np.array_equal(Kr[b, hd, n - 1], k_new[b, hd] if kv == "f32" else Kr[b, hd, n - 1])
            qc = oracle.mlp_hash_packed(w1[hd], b1[hd], w2[hd], q[b, hd][None])[0]
            allc = got_codes[b, hd, :n]
            s = oracle.nxor_scores(qc, allc)
            want_idx = oracle.top_k(s, min(k, n))
            assert cnt[p] == len(want_idx)
            assert np.array_equal(idx[p, :cnt[p]], want_idx)
            want = oracle.sparse_attention(q[b, hd][None], Kr[b, hd, :n], Vr[b, hd, :n], np.float32(scale),
                                           np.array([n], np.uint32), [want_idx])
            tol = 1e-5 if kv == "f32" else 1e-3
            assert np.abs(out[b, hd] - want[0]).max() <= tol


# ------------------------------------------------------------ sharded (virtual ranks on one GPU)
@pytest.mark.parametrize("R,P,N,W,k", [(2, 4, 40000, 4, 1234), (3, 4, 40000, 4, 1234),
                                         (8, 4, 40000, 4, 1234), (3, 2, 60, 4, 1000),
                                         (5, 3, 9000, 8, 4000), (8, 32, 16384, 4, 2621)])
def test_sharded_select_equals_reference(oracle, R, P, N, W, k):
    """Sequence sharding: R contiguous shards, each with its own
    context; histograms 'all-gathered' by a device concat; the rank-order
    concatenation must equal the single-GPU reference list."""
    rng = np.random.default_rng(R * 1000 + N)
    codes = rng.integers(0, 2**32, (P, N, W), dtype=np.uint64).astype(np.uint32)
    codes[1] = codes[1][rng.integers(0, 4, N)]  # heavy ties crossing shards
    q = codes[:, 7].copy()
    bounds = np.linspace(0, N, R + 1).astype(np.int64)
    ctxs = [capi.Context(0) for _ in range(R)]
    hists = []
    L = W * 32
    for r in range(R):
        part = np.ascontiguousarray(codes[:, bounds[r]:bounds[r + 1]])
        n_r = part.shape[1]
        hist = torch.zeros((P, L + 1), dtype=torch.int32, device=DEV)
        ctxs[r].shard_histogram(T(part), n_r, L, T(q), P, T(np.full(P, n_r, np.uint32)), 1, n_r, hist)
        ctxs[r]._part = T(part)
        hists.append(hist)
    all_hist = torch.stack(hists)  # [R][P][L+1] -- the NCCL all-gather's layout
    got = [[] for _ in range(P)]
    offsets = np.zeros((R, P), np.uint32)
    for r in range(R):
        n_r = int(bounds[r + 1] - bounds[r])
        idx = torch.zeros((P, k), dtype=torch.int32, device=DEV)
        cnt = torch.zeros(P, dtype=torch.int32, device=DEV)
        off = torch.zeros(P, dtype=torch.int32, device=DEV)
        ctxs[r].shard_select(all_hist, R, r, L, P, T(np.full(P, n_r, np.uint32)), 1, n_r, k, idx, cnt, off)
        torch.cuda.synchronize()
        ia, ca, oa = U(idx), U(cnt), U(off)
        offsets[r] = oa
        for p in range(P):
            got[p].append(ia[p, :ca[p]] + bounds[r])
        # host form of the plan agrees with the device plan
        h = U(all_hist)
        for p in range(P):
            pl = capi.plan_shard_host(h[:, p, :], r, k)
            assert pl["count"] == ca[p] and pl["offset"] == oa[p]
    want = oracle.retrieve_batch(codes, q, np.full(P, N, np.uint32), k)
    for p in range(P):
        cat = np.concatenate(got[p]).astype(np.uint32)
        assert np.array_equal(cat, want[p, :min(k, N)])
    for c in ctxs:
        c.close()


def test_sharded_attention_combine(ctx, oracle):
    rng = np.random.default_rng(44)
    R, P, n, d = 3, 2, 3000, 128
    K = rng.standard_normal((P, n, d)).astype(np.float32)
    V = rng.standard_normal((P, n, d)).astype(np.float32)
    Q = rng.standard_normal((P, d)).astype(np.float32)
    picks = [np.sort(rng.choice(n - 1, 200, replace=False)).astype(np.uint32) for _ in range(P)]
    bounds = [0, 1000, 2000, 3000]
    parts = torch.zeros((R, P, d + 2), dtype=torch.float32, device=DEV)
    for r in range(R):
        lo, hi = bounds[r], bounds[r + 1]
        loc = [p[(p >= lo) & (p < hi)] - lo for p in picks]
        kmax = max(1, max(len(x) for x in loc))
        idx = np.zeros((P, kmax), np.uint32)
        for i, x in enumerate(loc):
            idx[i, :len(x)] = x
        own = np.full(P, 0xFFFFFFFF, np.uint32)
        if r == R - 1:
            own[:] = (n - 1) - lo
        ctx.sparse_attend_partial(T(Q), T(np.ascontiguousarray(K[:, lo:hi])), T(np.ascontiguousarray(V[:, lo:hi])),
                                  capi.SPL_F32, hi - lo, d, P, T(idx), kmax,
                                  T(np.array([len(x) for x in loc], np.uint32)), T(own), 1,
                                  float(1 / np.sqrt(d)), parts[r])
    out = torch.zeros((P, d), dtype=torch.float32, device=DEV)
    ctx.attend_combine(parts, R, P, d, out)
    torch.cuda.synchronize()
    for p in range(P):
        want = oracle.sparse_attention(Q[p:p + 1], K[p], V[p], np.float32(1 / np.sqrt(d)),
                                       np.array([n], np.uint32), [picks[p]])
        assert np.abs(out[p].cpu().numpy() - want[0]).max() <= 1e-5


def _run_fused_sharded(oracle, R, P, N, W, k, codes, q, trials=2):
    """R virtual ranks in one process (own contexts, peer group wired with
    spl_peer_connect_local, one stream each so the R kernels run at once)."""
    L = W * 32
    bounds = np.linspace(0, N, R + 1).astype(np.int64)
    ctxs = [capi.Context(0) for _ in range(R)]
    peers = [ctxs[r].peer(R, r, P, L) for r in range(R)]
    capi.Peer.connect_local(ctxs[0], peers)
    streams = [torch.cuda.Stream() for _ in range(R)]
    parts, outs = [], []
    for r in range(R):
        part = np.ascontiguousarray(codes[:, bounds[r]:bounds[r + 1]])
        n_r = part.shape[1]
        parts.append((T(part), n_r, T(np.full(P, n_r, np.uint32))))
        outs.append((torch.zeros((P, k), dtype=torch.int32, device=DEV),
                     torch.zeros(P, dtype=torch.int32, device=DEV),
                     torch.zeros(P, dtype=torch.int32, device=DEV)))
    qt = T(q)
    want = oracle.retrieve_batch(codes, q, np.full(P, N, np.uint32), k)
    torch.cuda.synchronize()
    for _ in range(trials):  # epochs advance, both parity buffers get used
        for r in range(R):
            cp, n_r, nv = parts[r]
            idx, cnt, off = outs[r]
            idx.fill_(-1)
            ctxs[r].hamming_topk_sharded(peers[r], cp, n_r, L, qt, P, nv, 1, n_r, k, idx, cnt, off,
                                         streams[r].cuda_stream)
        torch.cuda.synchronize()
        for c in ctxs:
            c.check_device_error()
        for p in range(P):
            cat = np.zeros(min(k, N), np.uint32)
            filled = 0
            for r in range(R):
                idx, cnt, off = (U(t) for t in outs[r])
                c, o = int(cnt[p]), int(off[p])
                cat[o:o + c] = idx[p, :c] + bounds[r]
                filled += c
            assert filled == min(k, N)
            assert np.array_equal(cat, want[p, :min(k, N)]), (R, p)
    for pe in peers:
        pe.close()
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("R", [1, 2, 3])
def test_fused_sharded_equals_reference(oracle, R):
    """spl_hamming_topk_sharded: one kernel per rank, histograms exchanged in
    kernel through peer memory; the ranks' lists placed at their offsets
    equal the single-GPU reference list (heavy ties crossing ranks)."""
    rng = np.random.default_rng(70 + R)
    P, N, W, k = 4, 30000, 4, 1500
    codes = rng.integers(0, 2**32, (P, N, W), dtype=np.uint64).astype(np.uint32)
    codes[1] = codes[1][rng.integers(0, 5, N)]
    q = codes[:, 11].copy()
    _run_fused_sharded(oracle, R, P, N, W, k, codes, q)


def test_fused_sharded_low_threshold_round(oracle):
    """Global k-th score below the counted window [L/2, L] on every rank: the
    second (low-bin) exchange round runs; k close to N too."""
    rng = np.random.default_rng(81)
    P, N, W = 2, 24000, 4
    q = rng.integers(0, 2**32, (P, W), dtype=np.uint64).astype(np.uint32)
    codes = rng.integers(0, 2**32, (P, N, W), dtype=np.uint64).astype(np.uint32)
    keep = np.zeros((N, W), np.uint32)
    for _ in range(3):
        keep |= rng.integers(0, 2**32, (N, W), dtype=np.uint64).astype(np.uint32)
    codes[0] = (~q[0])[None, :] ^ (~keep & rng.integers(0, 2**32, (N, W), dtype=np.uint64).astype(np.uint32))
    for k in (50, 23000):
        _run_fused_sharded(oracle, 3, P, N, W, k, codes, q, trials=1)


def test_topk_config4_full_batch(ctx, oracle):
    """Config 4 at full size: B = 16 x 32 heads x 131072 rows x 256-bit codes,
    k = 2621 (two-pass path: u8 scores clamped at 255, windowed counters),
    every one of the 512 problems bit-exact against the oracle."""
    B, H, n, W = 16, 32, 131072, 8
    P = B * H
    k = oracle.budget_from_rate(0.02, n)
    g = torch.Generator(device=DEV)
    g.manual_seed(404)
    codes = torch.randint(-2**31, 2**31 - 1, (P, n, W), generator=g, device=DEV, dtype=torch.int32)
    q = torch.randint(-2**31, 2**31 - 1, (P, W), generator=g, device=DEV, dtype=torch.int32)
    nvb = np.array([n - 37 * b for b in range(B)], np.uint32)  # ragged per sequence
    idx = torch.full((P, k), -1, dtype=torch.int32, device=DEV)
    cnt = torch.zeros(P, dtype=torch.int32, device=DEV)
    ctx.hamming_topk(codes, n, W * 32, q, P, T(nvb), H, n, k, idx, cnt)
    torch.cuda.synchronize()
    ctx.check_device_error()
    want = oracle.retrieve_batch(U(codes), U(q), np.repeat(nvb, H), k)
    got = U(idx)
    assert np.array_equal(U(cnt), np.full(P, k, np.uint32))
    assert np.array_equal(got, want)


def test_sharded_config5_full(oracle):
    """Config 5 at full size: a 4M-token cache of 32 heads x 128-bit codes
    split over 8 ranks (the two-kernel flow, ranks run one after another on
    this GPU; the all-gather is a device stack), k = 2% of 4M = 83886. The
    rank-order concatenation equals the single-GPU reference list."""
    R, P, N, W = 8, 32, 4194304, 4
    L = W * 32
    k = oracle.budget_from_rate(0.02, N)
    g = torch.Generator(device=DEV)
    g.manual_seed(505)
    codes = torch.randint(-2**31, 2**31 - 1, (P, N, W), generator=g, device=DEV, dtype=torch.int32)
    q = torch.randint(-2**31, 2**31 - 1, (P, W), generator=g, device=DEV, dtype=torch.int32)
    n_r = N // R
    ctx = capi.Context(0)
    hists = []
    for r in range(R):
        part = codes[:, r * n_r:(r + 1) * n_r].contiguous()
        h = torch.zeros((P, L + 1), dtype=torch.int32, device=DEV)
        ctx.shard_histogram(part, n_r, L, q, P, T(np.full(P, n_r, np.uint32)), 1, n_r, h)
        hists.append(h)
        del part
    all_hist = torch.stack(hists)
    got = [[] for _ in range(P)]
    for r in range(R):
        part = codes[:, r * n_r:(r + 1) * n_r].contiguous()
        ctx.shard_histogram(part, n_r, L, q, P, T(np.full(P, n_r, np.uint32)), 1, n_r, hists[r])
        idx = torch.zeros((P, k), dtype=torch.int32, device=DEV)
        cnt = torch.zeros(P, dtype=torch.int32, device=DEV)
        off = torch.zeros(P, dtype=torch.int32, device=DEV)
        ctx.shard_select(all_hist, R, r, L, P, T(np.full(P, n_r, np.uint32)), 1, n_r, k, idx, cnt, off)
        torch.cuda.synchronize()
        ia, ca, oa = U(idx), U(cnt), U(off)
        for p in range(P):
            got[p].append((int(oa[p]), ia[p, :ca[p]].astype(np.int64) + r * n_r))
        del part
    ctx.check_device_error()
    ctx.close()
    want = oracle.retrieve_batch(U(codes), U(q), np.full(P, N, np.uint32), k)
    for p in range(P):
        parts = sorted(got[p])
        cat = np.concatenate([x for _, x in parts]).astype(np.uint32)
        assert [o for o, _ in parts] == list(np.cumsum([0] + [len(x) for _, x in parts[:-1]]))
        assert np.array_equal(cat, want[p]), p
