"""K2 — tcgen05 bulk encoder (spl_encode_tc / spl_encode mode TC) on the GPU.

K2 is the fast (bf16 operands, fp32 accumulation) path of mlp_hash /
linear_hash + pack_bits (hashers.cpp:75-108, bitcodes.cpp:22-41). Checks:
  * pre-activations vs a PyTorch reference of the same bf16 math
    (x, W1, W2 rounded to bf16; SiLU output rounded to bf16 before GEMM2):
    max-abs <= 1e-2 x rms(z2) (fp32 accumulation order and __expf differ);
  * code bits == the Appendix A.7 packing of sign(pre >= 0) of the kernel's
    own pre-activations (bit-exact), and differ from the reference math only
    where |z2| is within that tolerance;
  * agreement with the exact encoder (K1, bit-identical with the reference)
    on >= 99 % of bits."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
from paper_2508_19740_b200 import capi  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def pack_a7(bits):
    """bits [..., L] bool -> words [..., L/32] (column j -> word j % W, bit 31 - j // W)."""
    L = bits.shape[-1]
    W = L // 32
    out = np.zeros(bits.shape[:-1] + (W,), np.uint32)
    for j in range(L):
        out[..., j % W] |= bits[..., j].astype(np.uint32) << np.uint32(31 - j // W)
    return out


def mlp_weights(rng, H, d, h, L):
    w1 = (rng.standard_normal((H, d, h)) / np.sqrt(d)).astype(np.float32)
    b1 = (rng.standard_normal((H, h)) * 0.1).astype(np.float32)
    w2 = (rng.standard_normal((H, h, L)) / np.sqrt(h)).astype(np.float32)
    return w1, b1, w2


def torch_ref_mlp(x, w1, b1, w2):
    """x [B][H][m][d] -> z2 [B][H][m][L] with K2's rounding points."""
    bf = lambda a: torch.from_numpy(a).to(DEV).bfloat16().float()  # noqa: E731
    xb, w1b, w2b = bf(x), bf(w1), bf(w2)
    b1t = torch.from_numpy(b1).to(DEV)
    z1 = torch.einsum("bhmd,hdj->bhmj", xb, w1b) + b1t[None, :, None, :]
    a1 = torch.nn.functional.silu(z1).bfloat16().float()
    return torch.einsum("bhmj,hjl->bhml", a1, w2b).cpu().numpy()


def run_tc(ctx, hs, x, L, x_dtype=capi.SPL_F32):
    B, H, m, _ = x.shape
    xt = torch.from_numpy(x).to(DEV)
    if x_dtype == capi.SPL_BF16:
        xt = xt.bfloat16()
    codes = torch.zeros((B, H, m, L // 32), dtype=torch.int32, device=DEV)
    pre = torch.zeros((B, H, m, L), dtype=torch.float32, device=DEV)
    hs.encode_tc(xt, x_dtype, B, m, codes, pre)
    torch.cuda.synchronize()
    ctx.check_device_error()
    return codes.cpu().numpy().view(np.uint32), pre.cpu().numpy()


@pytest.mark.parametrize("L", [128, 256, 64, 32])
def test_encode_tc_mlp_vs_bf16_reference(ctx, L):
    rng = np.random.default_rng(L)
    H, d, h, B, m = 3, 128, 128, 2, 300  # 300 rows: two full tiles + a partial one
    w1, b1, w2 = mlp_weights(rng, H, d, h, L)
    x = rng.standard_normal((B, H, m, d)).astype(np.float32)
    hs = ctx.hasher(w1, b1, w2)
    codes, pre = run_tc(ctx, hs, x, L)
    z2 = torch_ref_mlp(x, w1, b1, w2)
    rms = float(np.sqrt(np.mean(z2 ** 2)))
    err = np.abs(pre - z2)
    assert err.max() <= 1e-2 * rms, (err.max(), rms)
    # codes are exactly the A.7 packing of the kernel's own signs
    assert np.array_equal(codes, pack_a7(pre >= 0))
    # vs the reference math: bits differ only inside the tolerance band
    ref_bits = z2 >= 0
    diff = ref_bits != (pre >= 0)
    assert np.all(np.abs(z2[diff]) <= 1e-2 * rms)
    # mode TC of spl_encode (f32 input) gives the same codes
    codes2 = torch.zeros((B, H, m, L // 32), dtype=torch.int32, device=DEV)
    hs.encode(torch.from_numpy(x).to(DEV), B, m, codes2, mode=capi.SPL_ENCODE_TC)
    assert np.array_equal(codes2.cpu().numpy().view(np.uint32), codes)


def test_encode_tc_agrees_with_exact(ctx, ref):
    """K2 vs K1 (bit-identical with the reference) on the reference's own init."""
    rng = np.random.default_rng(3)
    H, d, h, L, B, m = 4, 128, 128, 128, 1, 1000
    ws = [ref.mlp_gaussian_init(d, h, L, 64.0, ref.derive_seed(0, i)) for i in range(H)]
    w1 = np.stack([w[0] for w in ws])
    b1 = np.stack([w[1] for w in ws])
    w2 = np.stack([w[2] for w in ws])
    x = rng.standard_normal((B, H, m, d)).astype(np.float32)
    hs = ctx.hasher(w1, b1, w2)
    tc, _ = run_tc(ctx, hs, x, L)
    ex = torch.zeros((B, H, m, L // 32), dtype=torch.int32, device=DEV)
    hs.encode(torch.from_numpy(x).to(DEV), B, m, ex)
    ex = ex.cpu().numpy().view(np.uint32)
    differing = sum(bin(int(v)).count("1") for v in np.bitwise_xor(tc, ex).ravel())
    assert differing <= 0.01 * tc.size * 32, differing


def test_encode_tc_bf16_input(ctx):
    rng = np.random.default_rng(11)
    H, d, h, L, B, m = 2, 128, 128, 128, 1, 257
    w1, b1, w2 = mlp_weights(rng, H, d, h, L)
    x = rng.standard_normal((B, H, m, d)).astype(np.float32)
    hs = ctx.hasher(w1, b1, w2)
    c32, p32 = run_tc(ctx, hs, x, L, capi.SPL_F32)
    c16, p16 = run_tc(ctx, hs, x, L, capi.SPL_BF16)
    # the kernel rounds f32 input to bf16 on load: identical results
    assert np.array_equal(c32, c16)
    assert np.array_equal(p32, p16)


@pytest.mark.parametrize("L", [256, 128, 64, 32])
@pytest.mark.parametrize("shape", [(2, 3, 300), (1, 5, 1000), (3, 2, 128)])
def test_encode_tc_warp_specialised_matches(ctx, L, shape, monkeypatch):
    """The production prefill kernel (warp-specialised, bf16 keys through TMA,
    no pre-activation dump) performs the same bf16 UMMAs, SiLU and sign
    packing as the single-team kernel, so the codes must be bit-identical;
    shapes cover partial tiles, several heads per CTA (weight reloads) and
    more tiles than SMs' worth of work per CTA boundary."""
    B, H, m = shape
    rng = np.random.default_rng(7 * L + m)
    w1, b1, w2 = mlp_weights(rng, H, 128, 128, L)
    x = torch.from_numpy(rng.standard_normal((B, H, m, 128)).astype(np.float32)).to(DEV).bfloat16()
    hs = ctx.hasher(w1, b1, w2)
    ws = torch.zeros((B, H, m, L // 32), dtype=torch.int32, device=DEV)
    hs.encode_tc(x, capi.SPL_BF16, B, m, ws)
    torch.cuda.synchronize()
    ctx.check_device_error()
    monkeypatch.setenv("SPL_K2_WS", "0")
    one = torch.zeros_like(ws)
    hs.encode_tc(x, capi.SPL_BF16, B, m, one)
    torch.cuda.synchronize()
    assert torch.equal(ws, one)


def test_encode_tc_warp_specialised_large(ctx, monkeypatch):
    """Many tiles per CTA (long mbarrier phase sequences) at config-4 width."""
    B, H, m, L = 2, 32, 8192, 256
    rng = np.random.default_rng(99)
    w1, b1, w2 = mlp_weights(rng, H, 128, 128, L)
    g = torch.Generator(device=DEV)
    g.manual_seed(5)
    x = torch.randn((B, H, m, 128), generator=g, device=DEV).bfloat16()
    hs = ctx.hasher(w1, b1, w2)
    ws = torch.zeros((B, H, m, L // 32), dtype=torch.int32, device=DEV)
    hs.encode_tc(x, capi.SPL_BF16, B, m, ws)
    torch.cuda.synchronize()
    ctx.check_device_error()
    monkeypatch.setenv("SPL_K2_WS", "0")
    one = torch.zeros_like(ws)
    hs.encode_tc(x, capi.SPL_BF16, B, m, one)
    torch.cuda.synchronize()
    assert torch.equal(ws, one)


@pytest.mark.parametrize("L", [128, 256])
def test_encode_tc_linear(ctx, L):
    rng = np.random.default_rng(40 + L)
    H, d, B, m = 2, 128, 1, 200
    proj = rng.standard_normal((H, d, L)).astype(np.float32)
    x = rng.standard_normal((B, H, m, d)).astype(np.float32)
    hs = ctx.hasher(proj, kind=capi.SPL_HASHER_LINEAR)
    codes, pre = run_tc(ctx, hs, x, L)
    bf = lambda a: torch.from_numpy(a).to(DEV).bfloat16().float()  # noqa: E731
    z = torch.einsum("bhmd,hdl->bhml", bf(x), bf(proj)).cpu().numpy()
    rms = float(np.sqrt(np.mean(z ** 2)))
    assert np.abs(pre - z).max() <= 1e-3 * rms
    assert np.array_equal(codes, pack_a7(pre >= 0))


def test_encode_tc_rejects_unsupported_shapes(ctx):
    rng = np.random.default_rng(5)
    w1, b1, w2 = mlp_weights(rng, 1, 64, 64, 128)  # d = 64
    hs = ctx.hasher(w1, b1, w2)
    x = torch.zeros((1, 1, 4, 64), dtype=torch.float32, device=DEV)
    codes = torch.zeros((1, 1, 4, 4), dtype=torch.int32, device=DEV)
    with pytest.raises(capi.DimensionError):
        hs.encode_tc(x, capi.SPL_F32, 1, 4, codes)


def test_encode_tc_non_finite_raises(ctx):
    rng = np.random.default_rng(6)
    w1, b1, w2 = mlp_weights(rng, 1, 128, 128, 128)
    hs = ctx.hasher(w1, b1, w2)
    x = np.zeros((1, 1, 130, 128), np.float32)
    x[0, 0, 129, 7] = np.inf
    codes = torch.zeros((1, 1, 130, 4), dtype=torch.int32, device=DEV)
    hs.encode_tc(torch.from_numpy(x).to(DEV), capi.SPL_F32, 1, 130, codes)
    torch.cuda.synchronize()
    with pytest.raises(capi.NumericError):
        ctx.check_device_error()


@pytest.mark.parametrize("bad", [float("nan"), float("inf"), float("-inf")])
@pytest.mark.parametrize("L", [128, 256])
def test_encode_tc_non_finite_bf16_raises(ctx, bad, L):
    """The warp-specialised kernel checks one z2 column per row: a NaN / Inf
    key element reaches every column (also through a zero weight row)."""
    rng = np.random.default_rng(7)
    w1, b1, w2 = mlp_weights(rng, 1, 128, 128, L)
    w1[0, 5, :] = 0.0  # the bad feature meets a zero weight row
    hs = ctx.hasher(w1, b1, w2)
    x = torch.zeros((1, 1, 130, 128), dtype=torch.bfloat16, device=DEV)
    x[0, 0, 129, 5] = bad
    codes = torch.zeros((1, 1, 130, L // 32), dtype=torch.int32, device=DEV)
    hs.encode_tc(x, capi.SPL_BF16, 1, 130, codes)
    torch.cuda.synchronize()
    with pytest.raises(capi.NumericError):
        ctx.check_device_error()


def bf16_band(x, w1, b1, w2):
    """First-order bound on |z2_K2 - z2_ref| per output for K2's arithmetic
    (hashers.cpp:84-108 in bf16 operands / fp32 accumulation): x and W1
    rounded to bf16 (relative 2u per layer-1 product), SiLU through
    tanh.approx (relative <= 2^-10) and its output rounded to bf16 (u), W2
    rounded (u); |silu'| <= 1.1; u = 2^-8. fp32 accumulation error
    (~128 x 2^-24 relative) is far below it. x [m][d] -> [m][L] (float64)."""
    u = 2.0 ** -8
    xd, w1d, w2d = x.astype(np.float64), w1.astype(np.float64), w2.astype(np.float64)
    z1 = xd @ w1d + b1.astype(np.float64)
    a1 = z1 / (1.0 + np.exp(-z1))
    s1 = np.abs(xd) @ np.abs(w1d)  # sum_p |x_p W1_pj|
    da1 = 1.1 * 2 * u * s1 + (u + 2.0 ** -10) * np.abs(a1)
    return da1 @ np.abs(w2d) + u * (np.abs(a1) @ np.abs(w2d))


@pytest.mark.parametrize("L,x_dtype", [(128, capi.SPL_F32), (256, capi.SPL_F32), (128, capi.SPL_BF16)])
def test_encode_tc_bits_differ_only_in_reference_band(ctx, ref, L, x_dtype):
    """K2's parity contract against the REFERENCE itself: every code bit on
    which K2 disagrees with the reference's mlp_hash (sign of its f32
    mlp_forward, hashers.cpp:84-108, run from the unmodified sources in
    oracle/_ref) has a reference pre-activation inside the bf16 error band
    bf16_band() of that output; outside the band the bits are identical."""
    rng = np.random.default_rng(40 + L)
    H, d, h, B, m = 4, 128, 128, 1, 2048
    ws = [ref.mlp_gaussian_init(d, h, L, 64.0, ref.derive_seed(7, i)) for i in range(H)]
    w1 = np.stack([w[0] for w in ws])
    b1 = np.stack([w[1] for w in ws])
    w2 = np.stack([w[2] for w in ws])
    x = rng.standard_normal((B, H, m, d)).astype(np.float32)
    if x_dtype == capi.SPL_BF16:  # the reference sees the same bf16-rounded keys
        x = torch.from_numpy(x).bfloat16().float().numpy()
    hs = ctx.hasher(w1, b1, w2)
    codes, _ = run_tc(ctx, hs, x, L, x_dtype)
    total = outside = differ = 0
    for hd in range(H):
        z_ref = ref.mlp_forward(w1[hd], b1[hd], w2[hd], x[0, hd])
        want_words = pack_a7(z_ref >= 0)
        bad = np.bitwise_xor(codes[0, hd], want_words)
        # column j of the code sits in word j % W, bit 31 - j // W
        W = L // 32
        cols = np.arange(L)
        diff = ((bad[:, cols % W] >> (31 - cols // W).astype(np.uint32)) & 1).astype(bool)
        band = bf16_band(x[0, hd], w1[hd], b1[hd], w2[hd])
        outside += int(np.count_nonzero(diff & (np.abs(z_ref) > band)))
        differ += int(np.count_nonzero(diff))
        total += diff.size
    assert outside == 0, (outside, differ, total)
    assert differ <= 0.01 * total, (differ, total)
