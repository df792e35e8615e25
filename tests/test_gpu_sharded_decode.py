"""Sequence-sharded decode step (SURVEY §8 e, config 5) through
spl_sharded_decode_step: R ranks each hold a contiguous slice of every
sequence's tokens; the new token is appended on the last rank; the global
top-k (histogram exchange) and the attention partials (m, l, o) are exchanged
inside the kernels through peer memory. Checked against the oracle on the
concatenated cache: the ranks' index lists placed at their offsets equal the
reference's top_k_indices list bit for bit (bitcodes.cpp:89-136); every
rank's output equals the oracle's sparse_attention over the selected rows U
{own} (attention_eval.cpp:234-264) within 1e-3 (bf16 K/V) / 1e-5 (f32) and
the ranks' outputs are identical. Ranks here are virtual (one process, one
context and stream per rank, spl_peer_connect_local, all kernels in flight
at once); tests/mp_sharded_decode.py runs them as separate processes."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
from paper_2508_19740_b200 import capi  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def U(t):
    a = t.cpu().numpy()
    return a.view(np.uint32) if a.dtype == np.int32 else a


def run_sharded_step(oracle, R, B, H, N, d, L, k, kv, seed, expect):
    rng = np.random.default_rng(seed)
    W = L // 32
    w1 = (rng.standard_normal((H, d, d)) / np.sqrt(d)).astype(np.float32)
    b1 = (0.1 * rng.standard_normal((H, d))).astype(np.float32)
    w2 = (rng.standard_normal((H, d, L)) / np.sqrt(d)).astype(np.float32)
    codes = rng.integers(0, 2**32, (B, H, N, W), dtype=np.uint64).astype(np.uint32)
    codes[0, 1] = codes[0, 1][:, :][rng.integers(0, 6, N)]  # heavy ties crossing ranks
    tdt = torch.bfloat16 if kv == "bf16" else torch.float32
    kvd = capi.SPL_BF16 if kv == "bf16" else capi.SPL_F32
    K = torch.randn((B, H, N, d), device=DEV).to(tdt)
    V = torch.randn((B, H, N, d), device=DEV).to(tdt)
    q = rng.standard_normal((B, H, d)).astype(np.float32)
    kn = rng.standard_normal((B, H, d)).astype(np.float32)
    vn = rng.standard_normal((B, H, d)).astype(np.float32)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    bounds = np.linspace(0, N, R + 1).astype(np.int64)
    ctxs = [capi.Context(0) for _ in range(R)]
    peers = [ctxs[r].peer(R, r, B * H, L) for r in range(R)]
    capi.Peer.connect_local(ctxs[0], peers)
    hss = [ctxs[r].hasher(w1, b1, w2) for r in range(R)]
    streams = [torch.cuda.Stream() for _ in range(R)]
    P = B * H
    ranks = []
    for r in range(R):
        lo, hi = bounds[r], bounds[r + 1]
        n_r = int(hi - lo)
        ranks.append(dict(
            codes=t(codes[:, :, lo:hi].view(np.int32)), K=K[:, :, lo:hi].contiguous(),
            V=V[:, :, lo:hi].contiguous(), n=n_r, nv=t(np.full(B, n_r, np.int32)),
            idx=torch.full((P, k), -1, dtype=torch.int32, device=DEV),
            cnt=torch.zeros(P, dtype=torch.int32, device=DEV),
            off=torch.zeros(P, dtype=torch.int32, device=DEV),
            out=torch.zeros((B, H, d), dtype=torch.float32, device=DEV)))
    qd, knd, vnd = t(q), t(kn), t(vn)
    # size every workspace first: the ranks' kernels wait for each other, and
    # one rank allocating while another's kernel spins would stall the group
    for r in range(R):
        ctxs[r].reserve(P, ranks[r]["n"], L, k, d)
    torch.cuda.synchronize()
    scale = float(1 / np.sqrt(d))
    for c in ctxs:
        c.launch_log()
    for r in range(R):
        x = ranks[r]
        with torch.cuda.stream(streams[r]):
            hss[r].sharded_decode_step(peers[r], qd, knd, vnd, B, r == R - 1, x["codes"], x["K"], x["V"],
                                       kvd, x["n"], x["nv"], x["n"], k, scale, x["idx"], x["cnt"],
                                       x["off"], x["out"], streams[r].cuda_stream)
    torch.cuda.synchronize()
    for c in ctxs:
        c.check_device_error()
    got_log = ctxs[0].launch_log(); assert got_log == expect, got_log
    # the full cache after the step (the owner appended global row N - 1)
    full_codes = np.concatenate([U(ranks[r]["codes"]) for r in range(R)], axis=2)
    Kf = torch.cat([ranks[r]["K"] for r in range(R)], dim=2)
    Vf = torch.cat([ranks[r]["V"] for r in range(R)], dim=2)
    qc = np.zeros((P, W), np.uint32)
    for b in range(B):
        for h in range(H):
            assert np.array_equal(full_codes[b, h, N - 1],
                                  oracle.mlp_hash_packed(w1[h], b1[h], w2[h], kn[b, h][None])[0])
            qc[b * H + h] = oracle.mlp_hash_packed(w1[h], b1[h], w2[h], q[b, h][None])[0]
    want = oracle.retrieve_batch(full_codes.reshape(P, N, W), qc, np.full(P, N, np.uint32), k)
    kk = min(k, N)
    outs = [ranks[r]["out"].cpu().numpy() for r in range(R)]
    for r in range(1, R):
        assert np.array_equal(outs[r], outs[0])
    tol = 1e-3 if kv == "bf16" else 1e-5
    for p in range(P):
        b, h = divmod(p, H)
        cat = np.full(kk, 0xFFFFFFFF, np.uint32)
        filled = 0
        for r in range(R):
            ia, ca, oa = U(ranks[r]["idx"]), U(ranks[r]["cnt"]), U(ranks[r]["off"])
            c, o = int(ca[p]), int(oa[p])
            cat[o:o + c] = ia[p, :c] + bounds[r]
            filled += c
        assert filled == kk
        assert np.array_equal(cat, want[p, :kk]), p
        ref = oracle.sparse_attention(q[b, h][None], Kf[b, h].float().cpu().numpy(),
                                      Vf[b, h].float().cpu().numpy(), np.float32(scale),
                                      np.array([N], np.uint32), [cat])[0]
        assert np.abs(outs[0][b, h] - ref).max() <= tol, (p, np.abs(outs[0][b, h] - ref).max())
    for pe in peers:
        pe.close()
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("R", [1, 2, 3])
def test_sharded_decode_step_fused(oracle, R):
    """L = d = 128: one k3_fused_shard_attend launch per rank after the encoder."""
    run_sharded_step(oracle, R, 1, 4, 30000, 128, 128, 600, "bf16", 10 + R,
                     ["k1_encode_cluster", "k3_fused_shard_attend"])


def test_sharded_decode_step_fused_batch_f32(oracle):
    run_sharded_step(oracle, 2, 2, 2, 20000, 128, 128, 400, "f32", 21,
                     ["k1_encode_cluster", "k3_fused_shard_attend"])


def test_sharded_decode_step_unfused_d64(oracle):
    """d = 64: sharded retrieval, partial attention, in-kernel peer combine."""
    run_sharded_step(oracle, 2, 1, 4, 24000, 64, 128, 500, "bf16", 31,
                     ["k1_encode_exact", "k3_fused_shard", "k4_gather", "k5_peer_combine"])
