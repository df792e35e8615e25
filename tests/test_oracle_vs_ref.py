"""Differential check: the C restatement (oracle/liboracle.so) against the
unmodified reference (oracle/_ref/libspotref.so) on fresh seeded inputs,
including the config shapes (d = h = 128, L in {128, 256}). Skipped where
the reference was never compiled (the GPU box: /root/reference is absent,
but oracle/_ref travels when it was built here)."""
import numpy as np
import pytest


def test_mlp_forward_bit_exact_vs_reference(oracle, ref):
    rng = np.random.default_rng(1)
    for (d, h, L, seed) in [(128, 128, 128, 1), (128, 128, 256, 2), (64, 32, 96, 3), (7, 5, 32, 4)]:
        w1, b1, w2 = ref.mlp_gaussian_init(d, h, L, 64.0, ref.derive_seed(seed, 0))
        b1 = rng.standard_normal(h).astype(np.float32) * 0.1
        x = rng.standard_normal((300, d)).astype(np.float32) * 2.0
        a = ref.mlp_forward(w1, b1, w2, x)
        b = oracle.mlp_forward(w1, b1, w2, x)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
        assert np.array_equal(ref.mlp_hash_packed(w1, b1, w2, x), oracle.mlp_hash_packed(w1, b1, w2, x))


def test_linear_hash_vs_reference(oracle, ref):
    rng = np.random.default_rng(2)
    proj = ref.qr_rotation_init(64, 5)
    x = rng.standard_normal((200, 64)).astype(np.float32)
    assert np.array_equal(ref.linear_hash_packed(proj, x), oracle.linear_hash_packed(proj, x))


@pytest.mark.parametrize("d", [1, 3, 4, 7, 8, 12, 31, 64, 100, 128, 129, 256])
def test_sparse_attention_bit_exact_vs_reference(oracle, ref, d):
    rng = np.random.default_rng(d)
    n = 64
    K = rng.standard_normal((n, d)).astype(np.float32)
    V = rng.standard_normal((n, d)).astype(np.float32)
    Q = rng.standard_normal((3, d)).astype(np.float32)
    offs = np.array([64, 30, 1], np.uint32)
    picks = [np.sort(rng.choice(int(o), min(10, int(o)), replace=False)).astype(np.uint32) for o in offs]
    sc = np.float32(1 / np.sqrt(d))
    a = ref.sparse_attention(Q, K, V, sc, offs, picks)
    b = oracle.sparse_attention(Q, K, V, sc, offs, picks)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_topk_heavy_ties_vs_reference(oracle, ref):
    rng = np.random.default_rng(3)
    for _ in range(50):
        n = int(rng.integers(1, 5000))
        s = rng.integers(0, int(rng.integers(1, 300)), n).astype(np.int32)
        k = int(rng.integers(1, n + 1))
        assert np.array_equal(ref.top_k(s, k), oracle.top_k(s, k))


def test_retrieve_batch_config_shape_vs_reference(oracle, ref):
    # 4 heads x 131072 rows x 128-bit codes, k = 2% (config-2-shaped, fewer heads)
    rng = np.random.default_rng(4)
    P, n, W = 4, 131072, 4
    codes = rng.integers(0, 2**32, (P, n, W), dtype=np.uint64).astype(np.uint32)
    q = rng.integers(0, 2**32, (P, W), dtype=np.uint64).astype(np.uint32)
    nv = np.array([n, n - 1, 1000, 20], np.uint32)
    k = ref.budget_from_rate(0.02, n)
    h = ref.index_create(codes, np.full(P, n, np.uint32))
    try:
        a = ref.retrieve_batch(h, q, nv, k)
    finally:
        ref.index_destroy(h)
    b = oracle.retrieve_batch(codes, q, nv, k)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("d", [128, 64, 100, 36])
def test_oracle_topk_vs_reference(oracle, ref, d):
    """oracle_topk (attention_eval.cpp:121-135): the C restatement's causal
    logits (products rounded, summed in order, FMA tail) give the reference's
    indices, including near-ties from duplicated keys."""
    rng = np.random.default_rng(d)
    n, q = 3000, 6
    keys = rng.standard_normal((n, d)).astype(np.float32)
    keys[100:140] = keys[7]  # exact logit ties
    queries = rng.standard_normal((q, d)).astype(np.float32)
    offsets = np.array([n, n - 1, 2000, 141, 1, 500], np.uint32)
    scale = np.float32(1.0 / np.sqrt(d))
    for k in (1, 64, 300, 3000):
        a, ca = oracle.oracle_topk(queries, keys, scale, offsets, k)
        b, cb = ref.oracle_topk(queries, keys, scale, offsets, k)
        assert np.array_equal(ca, cb)
        for i in range(q):
            assert np.array_equal(a[i, :ca[i]], b[i, :cb[i]]), (d, k, i)


def test_iou_reference_examples(ref):
    assert ref.iou([], []) == 1.0
    assert ref.iou([1, 2, 3], [2, 3, 4]) == 0.5
    assert ref.iou([0, 5], [1, 6]) == 0.0
