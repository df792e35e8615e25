"""ctypes bindings for the CPU checkers (TEST INFRASTRUCTURE ONLY).

* ``Oracle``  -> oracle/liboracle.so, the C restatement (always built).
* ``RefLib``  -> oracle/_ref/libspotref.so, the unmodified reference sources
  compiled by oracle/Makefile (absent when /root/reference was never
  present; callers skip).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_SO = ROOT / "oracle" / "liboracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libspotref.so"

u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")


class CheckerError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"status {code}: {msg}")
        self.code = code
        self.msg = msg


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def build_checkers():
    """make -C oracle (liboracle.so always; _ref when /root/reference exists)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True)


class _Base:
    prefix = ""

    def _err(self, code):
        return CheckerError(code, "")

    def _chk(self, code):
        if code != 0:
            raise self._err(code)


class Oracle(_Base):
    """The C restatement (oracle/spl_oracle.c)."""

    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            build_checkers()
        L = self.lib = C.CDLL(str(path))
        L.orc_pack_bits.argtypes = [u8p, C.c_uint32, C.c_uint32, u32p]
        L.orc_unpack_bits.argtypes = [u32p, C.c_uint32, C.c_uint32, u8p]
        L.orc_nxor_scores_into.argtypes = [u32p, C.c_uint32, u32p, C.c_uint32, C.c_uint32,
                                           C.c_uint32, i32p]
        L.orc_top_k_i32.argtypes = [i32p, C.c_uint32, C.c_uint32, u32p]
        L.orc_top_k_f32.argtypes = [f32p, C.c_uint32, C.c_uint32, u32p]
        L.orc_mlp_forward.argtypes = [f32p, f32p, f32p, C.c_uint32, C.c_uint32, C.c_uint32,
                                      f32p, C.c_uint32, f32p]
        L.orc_mlp_hash_packed.argtypes = [f32p, f32p, f32p, C.c_uint32, C.c_uint32,
                                          C.c_uint32, f32p, C.c_uint32, u32p]
        L.orc_linear_hash_packed.argtypes = [f32p, C.c_uint32, C.c_uint32, f32p, C.c_uint32,
                                             u32p]
        L.orc_budget_from_rate.argtypes = [C.c_double, C.c_uint64, C.POINTER(C.c_int)]
        L.orc_budget_from_rate.restype = C.c_uint32
        L.orc_sparse_attention.argtypes = [f32p, C.c_uint32, f32p, f32p, C.c_uint32,
                                           C.c_uint32, C.c_float, u32p, u32p, u64p, f32p]
        L.orc_retrieve_batch.argtypes = [u32p, C.c_uint32, C.c_uint64, C.c_uint32, u32p, u32p,
                                         C.c_uint32, u32p, C.c_int]
        L.orc_oracle_topk.argtypes = [f32p, C.c_uint32, f32p, C.c_uint32, C.c_uint32, C.c_float,
                                      u32p, C.c_uint32, u32p, u32p]

    # -- bitcodes
    def pack_bits(self, bits):
        bits = _c(bits, np.uint8)
        n, d = bits.shape
        out = np.zeros((n, max(d // 32, 1)), np.uint32)
        self._chk(self.lib.orc_pack_bits(bits, n, d, out))
        return out

    def unpack_bits(self, words, L):
        words = _c(words, np.uint32)
        n = words.shape[0]
        out = np.zeros((n, L), np.uint8)
        self._chk(self.lib.orc_unpack_bits(words, n, L, out))
        return out

    def nxor_scores(self, q, codes, n_valid=None):
        q = _c(q, np.uint32).ravel()
        codes = _c(codes, np.uint32)
        n, W = codes.shape
        nv = n if n_valid is None else n_valid
        out = np.zeros(max(nv, 1), np.int32)
        self._chk(self.lib.orc_nxor_scores_into(q, q.size, codes, n, W * 32, nv, out))
        return out[:nv]

    def top_k(self, scores, k):
        if np.asarray(scores).dtype.kind == "f":
            s = _c(scores, np.float32)
            out = np.zeros(max(k, 1), np.uint32)
            self._chk(self.lib.orc_top_k_f32(s, s.size, k, out))
        else:
            s = _c(scores, np.int32)
            out = np.zeros(max(k, 1), np.uint32)
            self._chk(self.lib.orc_top_k_i32(s, s.size, k, out))
        return out[:k]

    # -- hashers
    def mlp_forward(self, w1, b1, w2, x):
        w1, b1, w2, x = _c(w1, np.float32), _c(b1, np.float32), _c(w2, np.float32), _c(x, np.float32)
        d, h = w1.shape
        L = w2.shape[1]
        m = x.shape[0]
        out = np.zeros((m, L), np.float32)
        self._chk(self.lib.orc_mlp_forward(w1, b1, w2, d, h, L, x, m, out))
        return out

    def mlp_hash_packed(self, w1, b1, w2, x):
        w1, b1, w2, x = _c(w1, np.float32), _c(b1, np.float32), _c(w2, np.float32), _c(x, np.float32)
        d, h = w1.shape
        L = w2.shape[1]
        m = x.shape[0]
        out = np.zeros((m, L // 32), np.uint32)
        self._chk(self.lib.orc_mlp_hash_packed(w1, b1, w2, d, h, L, x, m, out))
        return out

    def linear_hash_packed(self, proj, x):
        proj, x = _c(proj, np.float32), _c(x, np.float32)
        d, L = proj.shape
        out = np.zeros((x.shape[0], L // 32), np.uint32)
        self._chk(self.lib.orc_linear_hash_packed(proj, d, L, x, x.shape[0], out))
        return out

    # -- attention_eval
    def budget_from_rate(self, rate, n):
        st = C.c_int(0)
        k = self.lib.orc_budget_from_rate(rate, n, C.byref(st))
        self._chk(st.value)
        return k

    def sparse_attention(self, queries, keys, values, scale, offsets, picked_lists):
        queries, keys, values = _c(queries, np.float32), _c(keys, np.float32), _c(values, np.float32)
        q, d = queries.shape
        n = keys.shape[0]
        offs = _c(offsets, np.uint32)
        flat = np.concatenate([np.asarray(p, np.uint32) for p in picked_lists] + [np.zeros(0, np.uint32)])
        po = np.zeros(q + 1, np.uint64)
        po[1:] = np.cumsum([len(p) for p in picked_lists])
        flat = _c(flat if flat.size else np.zeros(1, np.uint32), np.uint32)
        out = np.zeros((q, d), np.float32)
        self._chk(self.lib.orc_sparse_attention(queries, q, keys, values, n, d, scale, offs, flat,
                                                po, out))
        return out

    def oracle_topk(self, queries, keys, scale, offsets, k):
        """-> (indices [q][k] uint32, counts [q])"""
        queries, keys = _c(queries, np.float32), _c(keys, np.float32)
        q, d = queries.shape
        out = np.zeros((q, k), np.uint32)
        cnt = np.zeros(q, np.uint32)
        self._chk(self.lib.orc_oracle_topk(queries, q, keys, keys.shape[0], d, C.c_float(scale),
                                           _c(offsets, np.uint32), k, out, cnt))
        return out, cnt

    def retrieve_batch(self, codes, qcodes, n_valid, k, threads=None):
        """codes [P][cap][W], qcodes [P][W], n_valid [P] -> out [P][k] (0-padded)."""
        codes = _c(codes, np.uint32)
        P, cap, W = codes.shape
        out = np.zeros((P, k), np.uint32)
        self._chk(self.lib.orc_retrieve_batch(codes, P, cap, W * 32, _c(qcodes, np.uint32),
                                              _c(n_valid, np.uint32), k, out,
                                              threads or os.cpu_count() or 1))
        return out


class RefLib(_Base):
    """The unmodified reference (oracle/_ref/libspotref.so)."""

    @staticmethod
    def available() -> bool:
        return REF_SO.exists()

    def __init__(self, path: Path = REF_SO):
        L = self.lib = C.CDLL(str(path))
        L.spotref_last_error.restype = C.c_char_p
        L.spotref_max_threads.restype = C.c_int
        L.spotref_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.spotref_derive_seed.restype = C.c_uint64
        L.spotref_mlp_gaussian_init.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_float,
                                                C.c_uint64, f32p, f32p, f32p]
        L.spotref_qr_rotation_init.argtypes = [C.c_uint32, C.c_uint64, f32p]
        L.spotref_pack_bits.argtypes = [u8p, C.c_uint32, C.c_uint32, u32p]
        L.spotref_unpack_bits.argtypes = [u32p, C.c_uint32, C.c_uint32, u8p]
        L.spotref_nxor_scores_into.argtypes = [u32p, C.c_uint32, u32p, C.c_uint32, C.c_uint32,
                                               C.c_uint32, i32p]
        L.spotref_top_k_i32.argtypes = [i32p, C.c_uint32, C.c_uint32, u32p]
        L.spotref_top_k_f32.argtypes = [f32p, C.c_uint32, C.c_uint32, u32p]
        L.spotref_mlp_forward.argtypes = [f32p, f32p, f32p, C.c_uint32, C.c_uint32, C.c_uint32,
                                          f32p, C.c_uint32, f32p]
        L.spotref_mlp_hash_packed.argtypes = [f32p, f32p, f32p, C.c_uint32, C.c_uint32,
                                              C.c_uint32, f32p, C.c_uint32, u32p]
        L.spotref_linear_hash_packed.argtypes = [f32p, C.c_uint32, C.c_uint32, f32p, C.c_uint32,
                                                 u32p]
        L.spotref_budget_from_rate.argtypes = [C.c_double, C.c_uint64, C.POINTER(C.c_int)]
        L.spotref_budget_from_rate.restype = C.c_uint32
        L.spotref_sparse_attention.argtypes = [f32p, C.c_uint32, f32p, f32p, C.c_uint32,
                                               C.c_uint32, C.c_float, u32p, u32p, u64p, f32p]
        L.spotref_full_attention.argtypes = [f32p, C.c_uint32, f32p, f32p, C.c_uint32,
                                             C.c_uint32, C.c_float, u32p, f32p]
        L.spotref_oracle_topk.argtypes = [f32p, C.c_uint32, f32p, C.c_uint32, C.c_uint32,
                                          C.c_float, u32p, C.c_uint32, u32p, u32p]
        L.spotref_iou.argtypes = [u32p, C.c_uint32, u32p, C.c_uint32]
        L.spotref_iou.restype = C.c_double
        L.spotref_hash_topk_mlp.argtypes = [f32p, f32p, f32p, C.c_uint32, C.c_uint32, f32p,
                                            C.c_uint32, f32p, f32p, C.c_uint32, C.c_uint32,
                                            C.c_float, u32p, C.c_uint32, u32p, u32p]
        L.spotref_index_create.argtypes = [u32p, C.c_uint32, C.c_uint64, C.c_uint32, u32p,
                                           C.POINTER(C.c_void_p)]
        L.spotref_index_destroy.argtypes = [C.c_void_p]
        f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
        L.spotref_train.argtypes = [C.c_int, f32p, f32p, f32p, C.c_uint32, C.c_uint32, C.c_uint32,
                                        C.c_float, C.c_uint32, f32p, f32p, u32p, f64p, u64p, i64p,
                                        C.c_int, f64p, C.POINTER(C.c_double),
                                        C.POINTER(C.c_uint32)]
        L.spotref_partition_identity.argtypes = [C.c_uint32, C.c_uint32, u32p, f64p, i64p,
                                                 C.c_uint64, u32p, u32p, u32p, u32p, u64p]
        L.spotref_lr_at.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, C.c_double]
        L.spotref_lr_at.restype = C.c_double
        L.spotref_retrieve_batch.argtypes = [C.c_void_p, u32p, u32p, C.c_uint32, u32p, C.c_int]

    def _err(self, code):
        return CheckerError(code, self.lib.spotref_last_error().decode())

    def max_threads(self):
        return self.lib.spotref_max_threads()

    def derive_seed(self, base, stream):
        return self.lib.spotref_derive_seed(base, stream)

    def mlp_gaussian_init(self, d, h, L, gamma=64.0, seed=0):
        w1 = np.zeros((d, h), np.float32)
        b1 = np.zeros(h, np.float32)
        w2 = np.zeros((h, L), np.float32)
        self._chk(self.lib.spotref_mlp_gaussian_init(d, h, L, gamma, seed, w1, b1, w2))
        return w1, b1, w2

    def qr_rotation_init(self, d, seed):
        p = np.zeros((d, d), np.float32)
        self._chk(self.lib.spotref_qr_rotation_init(d, seed, p))
        return p

    def pack_bits(self, bits):
        bits = _c(bits, np.uint8)
        n, d = bits.shape
        out = np.zeros((n, max(d // 32, 1)), np.uint32)
        self._chk(self.lib.spotref_pack_bits(bits, n, d, out))
        return out

    def unpack_bits(self, words, L):
        words = _c(words, np.uint32)
        out = np.zeros((words.shape[0], L), np.uint8)
        self._chk(self.lib.spotref_unpack_bits(words, words.shape[0], L, out))
        return out

    def nxor_scores(self, q, codes, n_valid=None):
        q = _c(q, np.uint32).ravel()
        codes = _c(codes, np.uint32)
        n, W = codes.shape
        nv = n if n_valid is None else n_valid
        out = np.zeros(max(nv, 1), np.int32)
        self._chk(self.lib.spotref_nxor_scores_into(q, q.size, codes, n, W * 32, nv, out))
        return out[:nv]

    def top_k(self, scores, k):
        if np.asarray(scores).dtype.kind == "f":
            s = _c(scores, np.float32)
            out = np.zeros(max(k, 1), np.uint32)
            self._chk(self.lib.spotref_top_k_f32(s, s.size, k, out))
        else:
            s = _c(scores, np.int32)
            out = np.zeros(max(k, 1), np.uint32)
            self._chk(self.lib.spotref_top_k_i32(s, s.size, k, out))
        return out[:k]

    def mlp_forward(self, w1, b1, w2, x):
        w1, b1, w2, x = _c(w1, np.float32), _c(b1, np.float32), _c(w2, np.float32), _c(x, np.float32)
        d, h = w1.shape
        L = w2.shape[1]
        out = np.zeros((x.shape[0], L), np.float32)
        self._chk(self.lib.spotref_mlp_forward(w1, b1, w2, d, h, L, x, x.shape[0], out))
        return out

    def mlp_hash_packed(self, w1, b1, w2, x):
        w1, b1, w2, x = _c(w1, np.float32), _c(b1, np.float32), _c(w2, np.float32), _c(x, np.float32)
        d, h = w1.shape
        L = w2.shape[1]
        out = np.zeros((x.shape[0], L // 32), np.uint32)
        self._chk(self.lib.spotref_mlp_hash_packed(w1, b1, w2, d, h, L, x, x.shape[0], out))
        return out

    def linear_hash_packed(self, proj, x):
        proj, x = _c(proj, np.float32), _c(x, np.float32)
        d, L = proj.shape
        out = np.zeros((x.shape[0], L // 32), np.uint32)
        self._chk(self.lib.spotref_linear_hash_packed(proj, d, L, x, x.shape[0], out))
        return out

    def budget_from_rate(self, rate, n):
        st = C.c_int(0)
        k = self.lib.spotref_budget_from_rate(rate, n, C.byref(st))
        self._chk(st.value)
        return k

    def sparse_attention(self, queries, keys, values, scale, offsets, picked_lists):
        queries, keys, values = _c(queries, np.float32), _c(keys, np.float32), _c(values, np.float32)
        q, d = queries.shape
        flat = np.concatenate([np.asarray(p, np.uint32) for p in picked_lists] + [np.zeros(0, np.uint32)])
        po = np.zeros(q + 1, np.uint64)
        po[1:] = np.cumsum([len(p) for p in picked_lists])
        flat = _c(flat if flat.size else np.zeros(1, np.uint32), np.uint32)
        out = np.zeros((q, d), np.float32)
        self._chk(self.lib.spotref_sparse_attention(queries, q, keys, values, keys.shape[0], d,
                                                    scale, _c(offsets, np.uint32), flat, po, out))
        return out

    def full_attention(self, queries, keys, values, scale, offsets):
        queries, keys, values = _c(queries, np.float32), _c(keys, np.float32), _c(values, np.float32)
        q, d = queries.shape
        out = np.zeros((q, d), np.float32)
        self._chk(self.lib.spotref_full_attention(queries, q, keys, values, keys.shape[0], d, scale,
                                                  _c(offsets, np.uint32), out))
        return out

    def oracle_topk(self, queries, keys, scale, offsets, k):
        queries, keys = _c(queries, np.float32), _c(keys, np.float32)
        q, d = queries.shape
        out = np.zeros((q, k), np.uint32)
        cnt = np.zeros(q, np.uint32)
        self._chk(self.lib.spotref_oracle_topk(queries, q, keys, keys.shape[0], d, C.c_float(scale),
                                               _c(offsets, np.uint32), k, out, cnt))
        return out, cnt

    def iou(self, a, b):
        a, b = _c(a, np.uint32), _c(b, np.uint32)
        return float(self.lib.spotref_iou(a if a.size else np.zeros(1, np.uint32), a.size,
                                          b if b.size else np.zeros(1, np.uint32), b.size))

    def hash_topk_mlp(self, w1, b1, w2, queries, keys, values, scale, offsets, k):
        w1, b1, w2 = _c(w1, np.float32), _c(b1, np.float32), _c(w2, np.float32)
        queries, keys, values = _c(queries, np.float32), _c(keys, np.float32), _c(values, np.float32)
        q, d = queries.shape
        out = np.zeros((q, k), np.uint32)
        cnt = np.zeros(q, np.uint32)
        self._chk(self.lib.spotref_hash_topk_mlp(w1, b1, w2, w1.shape[1], w2.shape[1], queries, q,
                                                 keys, values, keys.shape[0], d, scale,
                                                 _c(offsets, np.uint32), k, out, cnt))
        return [out[i, :cnt[i]].copy() for i in range(q)]

    def index_create(self, codes, n_rows):
        codes = _c(codes, np.uint32)
        P, cap, W = codes.shape
        h = C.c_void_p()
        self._chk(self.lib.spotref_index_create(codes, P, cap, W * 32, _c(n_rows, np.uint32),
                                                C.byref(h)))
        return h

    def index_destroy(self, h):
        self.lib.spotref_index_destroy(h)

    def retrieve_batch(self, handle, qcodes, n_valid, k, threads=None):
        qcodes = _c(qcodes, np.uint32)
        P = qcodes.shape[0]
        out = np.zeros((P, k), np.uint32)
        self._chk(self.lib.spotref_retrieve_batch(handle, qcodes, _c(n_valid, np.uint32), k, out,
                                                  threads or os.cpu_count() or 1))
        return out

    # -- trainer
    def train(self, kind, w1, b1, w2, gamma, sequences, rank, cfg, loss_kind=0):
        """train_hasher. kind 1 MLP (w1 d x h, b1, w2), 0 linear / 2 downproj (w1 =
        projection d x L; b1, w2 None). rank: dict(beta, alpha, maskout, max_top,
        max_oth, query_subsample); cfg: dict of TrainConfig fields. Returns
        (w1, b1, w2, records [iters][3], holdout_iou, skipped)."""
        w1 = _c(w1, np.float32).copy()
        d = w1.shape[0]
        if kind == 1:
            b1, w2 = _c(b1, np.float32).copy(), _c(w2, np.float32).copy()
            h, L = w1.shape[1], w2.shape[1]
        else:
            h, L = 0, w1.shape[1]
            b1, w2 = np.zeros(1, np.float32), np.zeros(1, np.float32)
        qs = _c(np.concatenate([q for q, _ in sequences]), np.float32)
        ks = _c(np.concatenate([k for _, k in sequences]), np.float32)
        lens = np.array([len(q) for q, _ in sequences], np.uint32)
        dc = np.array([cfg["max_lr"], cfg["min_lr"], cfg["adam_beta1"], cfg["adam_beta2"],
                       cfg["adam_eps"], cfg["weight_decay"], cfg["grad_clip"], cfg["soft_gamma"],
                       cfg["holdout_budget_rate"], rank["beta"], rank["alpha"], rank["maskout"]],
                      np.float64)
        uc = np.array([cfg["num_iters"], cfg["warmup_iters"], cfg["batch"], cfg["seed"],
                       cfg["holdout_queries"]], np.uint64)
        op = np.array([-1 if rank.get(k) is None else rank[k]
                       for k in ("max_top", "max_oth", "query_subsample")], np.int64)
        rec = np.zeros((max(cfg["num_iters"], 1), 3), np.float64)
        iou = C.c_double(0.0)
        sk = C.c_uint32(0)
        self._chk(self.lib.spotref_train(kind, w1, b1, w2, d, h, L, gamma, len(sequences), qs,
                                         ks, lens, dc, uc, op, loss_kind, rec, C.byref(iou),
                                         C.byref(sk)))
        if kind != 1:
            b1 = w2 = None
        return w1, b1, w2, rec[:cfg["num_iters"]], iou.value, sk.value

    def partition_identity(self, q, n, rank, seed, offsets=None):
        """partition_topk over an identity order: (rows, top_pos, oth_pos, k_full, valid_pairs)."""
        offs = _c(np.arange(1, q + 1) if offsets is None else offsets, np.uint32)
        bam = np.array([rank["beta"], rank["alpha"], rank["maskout"]], np.float64)
        op = np.array([-1 if rank.get(k) is None else rank[k]
                       for k in ("max_top", "max_oth", "query_subsample")], np.int64)
        rows = np.zeros(max(q, 1), np.uint32)
        top = np.zeros(max(n, 1), np.uint32)
        oth = np.zeros(max(n, 1), np.uint32)
        cnt = np.zeros(4, np.uint32)
        vp = np.zeros(1, np.uint64)
        self._chk(self.lib.spotref_partition_identity(q, n, offs, bam, op, seed, rows, top, oth,
                                                      cnt, vp))
        return rows[:cnt[0]], top[:cnt[1]], oth[:cnt[2]], int(cnt[3]), int(vp[0])

    def lr_at(self, it, num_iters, warmup, max_lr, min_lr):
        return self.lib.spotref_lr_at(it, num_iters, warmup, max_lr, min_lr)
