"""Pin the CPU oracle (oracle/spl_oracle.c) before trusting it.

1. The reference's own known-answer tests for this path, restated
   (proj/tests/test_bitcodes.cpp, test_attention_eval.cpp, test_hashers.cpp).
2. The committed golden fixtures produced by the UNMODIFIED reference
   (tests/golden/make_golden.py -> reference_golden.npz): bit-exact.
3. The reference's property tests (closed-form pack layout, round trip,
   2m - L identity, top-k vs full sort with heavy ties).
CPU only.
"""
from pathlib import Path

import numpy as np
import pytest

from oracle_lib import CheckerError

G = np.load(Path(__file__).parent / "golden" / "reference_golden.npz")


def full_sort_topk(scores, k):
    """test_bitcodes.cpp:56-67: sort by (score desc, index asc), keep k, ascending."""
    order = sorted(range(len(scores)), key=lambda i: (-scores[i], i))
    return np.array(sorted(order[:k]), np.uint32)


# ----------------------------------------------------- known answers
def test_pack_bits_single_word_examples(oracle):
    # test_bitcodes.cpp:71-84
    one = np.zeros((1, 32), np.uint8)
    one[0, 0] = 1
    assert oracle.pack_bits(one)[0, 0] == 0x80000000
    assert oracle.pack_bits(np.zeros((1, 32), np.uint8))[0, 0] == 0
    wide = np.zeros((1, 64), np.uint8)
    wide[0, 1] = 1
    assert list(oracle.pack_bits(wide)[0]) == [0, 0x80000000]


def test_pack_bits_rejects_bad_width(oracle):
    # test_bitcodes.cpp:86-89
    for d in (33, 0):
        with pytest.raises(CheckerError) as e:
            oracle.pack_bits(np.zeros((1, d), np.uint8))
        assert e.value.code == 1


def test_unpack_examples(oracle):
    # test_bitcodes.cpp:101-112
    assert oracle.unpack_bits(np.array([[0xFFFFFFFF]], np.uint32), 32).all()
    w = oracle.unpack_bits(np.array([[0, 0x80000000]], np.uint32), 64)[0]
    assert [j for j in range(64) if w[j]] == [1]


def test_agreement_4bit(oracle):
    # test_bitcodes.cpp:121-132: 1010 vs 1001 -> 2 agreements (padded to 32 bits)
    a = np.zeros((1, 32), np.uint8)
    b = np.zeros((1, 32), np.uint8)
    a[0, [0, 2]] = 1
    b[0, [0, 3]] = 1
    s = oracle.nxor_scores(oracle.pack_bits(a)[0], oracle.pack_bits(b))
    assert s[0] == 2 + 28  # the 28 zero-padding bits agree too


def test_nxor_self_and_complement(oracle):
    # test_bitcodes.cpp:134-152
    rng = np.random.default_rng(13)
    bits = rng.integers(0, 2, (8, 128), dtype=np.uint8)
    codes = oracle.pack_bits(bits)
    assert oracle.nxor_scores(codes[3], codes)[3] == 128
    flipped = oracle.pack_bits(1 - bits[:1])
    assert oracle.nxor_scores(flipped[0], codes)[0] == 0
    with pytest.raises(CheckerError):
        oracle.nxor_scores(np.zeros(2, np.uint32), codes)  # 64-bit query vs 128-bit index


def test_top_k_examples_and_tie_rule(oracle):
    # test_bitcodes.cpp:187-199
    assert list(oracle.top_k(np.array([3, 1, 2], np.int32), 1)) == [0]
    assert list(oracle.top_k(np.array([2, 2, 1], np.int32), 1)) == [0]
    assert list(oracle.top_k(np.array([5, 9, 1, 7], np.int32), 4)) == [0, 1, 2, 3]
    for k in (0, 4):
        with pytest.raises(CheckerError):
            oracle.top_k(np.array([3, 1, 2], np.int32), k)


def test_budget_from_rate_examples(oracle):
    # test_attention_eval.cpp:303-308
    assert oracle.budget_from_rate(0.02, 2048) == 40
    assert oracle.budget_from_rate(0.02, 500) == 20
    assert oracle.budget_from_rate(1.0, 8) == 8
    with pytest.raises(CheckerError):
        oracle.budget_from_rate(0.0, 10)


def test_zero_network_all_ones(oracle):
    # test_hashers.cpp:171-179 (zero network -> every code bit is 1)
    w1 = np.zeros((8, 8), np.float32)
    b1 = np.zeros(8, np.float32)
    w2 = np.zeros((8, 32), np.float32)
    x = np.random.default_rng(37).standard_normal((2, 8)).astype(np.float32)
    assert (oracle.mlp_hash_packed(w1, b1, w2, x) == 0xFFFFFFFF).all()


def test_non_finite_input_rejected(oracle):
    # test_hashers.cpp:160-165
    w1 = np.ones((4, 4), np.float32)
    x = np.zeros((1, 4), np.float32)
    x[0, 2] = np.nan
    with pytest.raises(CheckerError) as e:
        oracle.mlp_forward(w1, np.zeros(4, np.float32), np.ones((4, 32), np.float32), x)
    assert e.value.code == 2


def test_sparse_attention_rejections(oracle):
    # test_attention_eval.cpp:288-300
    rng = np.random.default_rng(11)
    K = rng.standard_normal((4, 8)).astype(np.float32)
    Q = rng.standard_normal((2, 8)).astype(np.float32)
    offs = np.array([1, 2], np.uint32)
    with pytest.raises(CheckerError):
        oracle.sparse_attention(Q, K, K, 0.5, offs, [[0], []])
    with pytest.raises(CheckerError):
        oracle.sparse_attention(Q, K, K, 0.5, offs, [[3], [0]])


# ----------------------------------------------------- golden fixtures
@pytest.mark.parametrize("d", [32, 64, 128, 256])
def test_golden_pack_bits(oracle, d):
    assert np.array_equal(oracle.pack_bits(G[f"pack_bits_in_{d}"]), G[f"pack_bits_out_{d}"])
    assert np.array_equal(oracle.unpack_bits(G[f"pack_bits_out_{d}"], d), G[f"pack_bits_in_{d}"])


@pytest.mark.parametrize("ci", list(range(6)))
def test_golden_scan_topk(oracle, ci):
    codes, q = G[f"topk{ci}_codes"], G[f"topk{ci}_q"]
    k = int(G[f"topk{ci}_k"][0])
    s = oracle.nxor_scores(q, codes)
    assert np.array_equal(s, G[f"topk{ci}_scores"])
    assert np.array_equal(oracle.top_k(s, k), G[f"topk{ci}_idx"])


@pytest.mark.parametrize("tag", ["c128", "c256", "small", "bias"])
def test_golden_mlp_bit_exact(oracle, tag):
    w1, b1, w2, x = (G[f"mlp_{tag}_{n}"] for n in ("w1", "b1", "w2", "x"))
    pre = oracle.mlp_forward(w1, b1, w2, x)
    assert np.array_equal(pre.view(np.uint32), G[f"mlp_{tag}_pre"].view(np.uint32))
    assert np.array_equal(oracle.mlp_hash_packed(w1, b1, w2, x), G[f"mlp_{tag}_codes"])


def test_golden_sparse_attention_bit_exact(oracle):
    po = G["att_picked_off"]
    picks = [G["att_picked"][po[i]:po[i + 1]] for i in range(len(po) - 1)]
    out = oracle.sparse_attention(G["att_Q"], G["att_K"], G["att_V"], G["att_scale"][0],
                                  G["att_offs"], picks)
    assert np.array_equal(out.view(np.uint32), G["att_out"].view(np.uint32))


def test_golden_hash_topk(oracle):
    w1, b1, w2 = G["ht_w1"], G["ht_b1"], G["ht_w2"]
    K, Q = G["ht_K"], G["ht_Q"]
    k = int(G["ht_k"][0])
    kc = oracle.mlp_hash_packed(w1, b1, w2, K)
    qc = oracle.mlp_hash_packed(w1, b1, w2, Q)
    n = K.shape[0]
    for r in range(n):
        valid = r + 1
        s = oracle.nxor_scores(qc[r], kc, valid)
        got = oracle.top_k(s, min(k, valid))
        assert np.array_equal(got, G["ht_idx"][r, :G["ht_cnt"][r]])


def test_golden_budget(oracle):
    for n, k in zip(G["budget_n"], G["budget_k"]):
        assert oracle.budget_from_rate(0.02, int(n)) == k


# ----------------------------------------------------- reference property tests
def test_pack_layout_oracle(oracle):
    # test_bitcodes.cpp:28-41, 91-99: column j -> word j % (d/32), bit 31 - j // (d/32)
    rng = np.random.default_rng(7)
    for _ in range(200):
        n, d = 1 + rng.integers(0, 8), 32 * (1 + rng.integers(0, 8))
        bits = rng.integers(0, 2, (n, d), dtype=np.uint8)
        cw = d // 32
        want = np.zeros((n, cw), np.uint32)
        for i in range(n):
            for j in np.nonzero(bits[i])[0]:
                want[i, j % cw] |= np.uint32(1) << np.uint32(31 - j // cw)
        assert np.array_equal(oracle.pack_bits(bits), want)
        assert np.array_equal(oracle.unpack_bits(want, d), bits)


def test_affine_identity(oracle):
    # test_bitcodes.cpp:154-167: 2m - L == +-1 dot product
    rng = np.random.default_rng(17)
    for _ in range(100):
        d = 32 * (1 + rng.integers(0, 8))
        bits = rng.integers(0, 2, (6, d), dtype=np.uint8)
        s = oracle.nxor_scores(oracle.pack_bits(bits)[0], oracle.pack_bits(bits))
        pm = bits.astype(np.int64) * 2 - 1
        assert np.array_equal(2 * s.astype(np.int64) - d, pm @ pm[0])


def test_top_k_full_sort_oracle(oracle):
    # test_bitcodes.cpp:201-222
    rng = np.random.default_rng(23)
    for _ in range(400):
        n = 1 + int(rng.integers(0, 257))
        s = rng.integers(0, 13, n).astype(np.int32)
        k = 1 + int(rng.integers(0, n))
        assert np.array_equal(oracle.top_k(s, k), full_sort_topk(s, k))
    s = rng.integers(0, 129, 10000).astype(np.int32)
    for k in (1, 17, 200, 9999, 10000):
        assert np.array_equal(oracle.top_k(s, k), full_sort_topk(s, k))
