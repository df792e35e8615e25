"""Generate the committed golden fixtures from the UNMODIFIED reference.

Run in the container that has /root/reference (the GPU box does not):

    make -C oracle && python tests/golden/make_golden.py

Every output array below is produced by oracle/_ref/libspotref.so, i.e. by the
reference's own pack_bits / nxor_scores_into / top_k_indices / mlp_forward /
mlp_hash / sparse_attention / hash_topk compiled from
/root/reference/proj/src with its Release flags (oracle/Makefile). Inputs are
seeded numpy draws; hasher weights come from the reference's own
mlp_gaussian_init(d, h, L, 64, derive_seed(seed, head)) (hashers.cpp:41-63).
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from oracle_lib import RefLib  # noqa: E402


def main():
    ref = RefLib()
    rng = np.random.default_rng(20250827)
    out = {}

    # 1. pack_bits layout (bitcodes.cpp:22-41), several widths
    for d in (32, 64, 128, 256):
        bits = rng.integers(0, 2, (17, d), dtype=np.uint8)
        out[f"pack_bits_in_{d}"] = bits
        out[f"pack_bits_out_{d}"] = ref.pack_bits(bits)

    # 2. scan + top-k, heavy ties and plain random codes
    cases = []
    for ci, (n, L, k) in enumerate([(4096, 128, 64), (5000, 256, 100), (1000, 32, 300),
                                    (257, 128, 257), (3000, 64, 1), (2048, 96, 40)]):
        W = L // 32
        codes = rng.integers(0, 2**32, (n, W), dtype=np.uint64).astype(np.uint32)
        if ci % 2 == 1:  # few distinct rows -> massive score ties
            codes = codes[rng.integers(0, 5, n)]
        q = codes[rng.integers(0, n)].copy()
        scores = ref.nxor_scores(q, codes)
        idx = ref.top_k(scores, k)
        out[f"topk{ci}_codes"] = codes
        out[f"topk{ci}_q"] = q
        out[f"topk{ci}_scores"] = scores
        out[f"topk{ci}_k"] = np.array([k], np.uint32)
        out[f"topk{ci}_idx"] = idx
        cases.append(ci)
    out["topk_cases"] = np.array(cases, np.uint32)

    # 3. MLP encode at the config shapes (d = h = 128, L in {128, 256}) and a
    #    small odd shape; hasher from the reference's own init
    for tag, (d, h, L, m, seed) in {"c128": (128, 128, 128, 96, 7), "c256": (128, 128, 256, 64, 11),
                                    "small": (16, 24, 64, 40, 3)}.items():
        w1, b1, w2 = ref.mlp_gaussian_init(d, h, L, 64.0, ref.derive_seed(seed, 0))
        x = rng.standard_normal((m, d)).astype(np.float32)
        x[0] = 0.0  # zero input -> silu(0) = 0 path
        out[f"mlp_{tag}_w1"], out[f"mlp_{tag}_b1"], out[f"mlp_{tag}_w2"] = w1, b1, w2
        out[f"mlp_{tag}_x"] = x
        out[f"mlp_{tag}_pre"] = ref.mlp_forward(w1, b1, w2, x)
        out[f"mlp_{tag}_codes"] = ref.mlp_hash_packed(w1, b1, w2, x)
    # with a non-zero bias
    w1, b1, w2 = ref.mlp_gaussian_init(32, 32, 64, 64.0, 99)
    b1 = rng.standard_normal(32).astype(np.float32)
    x = (3.0 * rng.standard_normal((50, 32))).astype(np.float32)
    out["mlp_bias_w1"], out["mlp_bias_b1"], out["mlp_bias_w2"], out["mlp_bias_x"] = w1, b1, w2, x
    out["mlp_bias_pre"] = ref.mlp_forward(w1, b1, w2, x)
    out["mlp_bias_codes"] = ref.mlp_hash_packed(w1, b1, w2, x)

    # 4. sparse attention (attention_eval.cpp:234-264), own token added
    n, d, q = 300, 128, 5
    K = rng.standard_normal((n, d)).astype(np.float32)
    V = rng.standard_normal((n, d)).astype(np.float32)
    Q = rng.standard_normal((q, d)).astype(np.float32)
    offs = np.array([300, 300, 150, 20, 1], np.uint32)
    picks = [np.sort(rng.choice(int(o), min(40, int(o)), replace=False)).astype(np.uint32) for o in offs]
    picks[1] = np.append(picks[1][picks[1] < 299], 299).astype(np.uint32)  # own already listed
    scale = np.float32(1.0 / np.sqrt(d))
    out["att_K"], out["att_V"], out["att_Q"], out["att_offs"] = K, V, Q, offs
    out["att_scale"] = np.array([scale], np.float32)
    flat = np.concatenate(picks)
    po = np.zeros(q + 1, np.uint64)
    po[1:] = np.cumsum([len(p) for p in picks])
    out["att_picked"], out["att_picked_off"] = flat, po
    out["att_out"] = ref.sparse_attention(Q, K, V, scale, offs, picks)

    # 5. hash_topk end to end (attention_eval.cpp:137-181), causal instance
    n, d, L, k = 512, 128, 128, 16
    w1, b1, w2 = ref.mlp_gaussian_init(d, d, L, 64.0, ref.derive_seed(0, 5))
    K = rng.standard_normal((n, d)).astype(np.float32)
    V = rng.standard_normal((n, d)).astype(np.float32)
    Q = rng.standard_normal((n, d)).astype(np.float32)
    offs = np.arange(1, n + 1, dtype=np.uint32)
    res = ref.hash_topk_mlp(w1, b1, w2, Q, K, V, np.float32(1 / np.sqrt(d)), offs, k)
    out["ht_w1"], out["ht_b1"], out["ht_w2"] = w1, b1, w2
    out["ht_K"], out["ht_V"], out["ht_Q"], out["ht_k"] = K, V, Q, np.array([k], np.uint32)
    out["ht_idx"] = np.stack([np.pad(r, (0, k - len(r)), constant_values=0xFFFFFFFF) for r in res])
    out["ht_cnt"] = np.array([len(r) for r in res], np.uint32)

    # 6. budget_from_rate (attention_eval.cpp:266-272)
    ns = np.array([8, 500, 2048, 4096, 131072, 524288, 4194304], np.uint64)
    out["budget_n"] = ns
    out["budget_k"] = np.array([ref.budget_from_rate(0.02, int(v)) for v in ns], np.uint32)

    path = HERE / "reference_golden.npz"
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({path.stat().st_size} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
