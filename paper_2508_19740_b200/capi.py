"""ctypes binding of include/spl_c.h (libspl.so, the sm_100a kernels).

Host-side glue only: every compute call launches CUDA kernels through the
C-ABI; there is no CPU fallback. Loading the library works on a CPU-only
machine (symbol checks), but creating a context requires a Blackwell GPU and
fails loudly otherwise.

Errors map to the reference's exception types (proj/include/spotlight/
errors.hpp:9-35): DimensionError (an invalid_argument -> ValueError),
NumericError, FormatError, IoError.
"""
from __future__ import annotations

import ctypes as C
import os
import re
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
LIB_PATH = PKG / "lib" / "libspl.so"
HEADER = ROOT / "include" / "spl_c.h"

(SPL_OK, SPL_E_DIMENSION, SPL_E_NUMERIC, SPL_E_FORMAT, SPL_E_IO, SPL_E_CUDA, SPL_E_NCCL, SPL_E_STATE,
 SPL_E_EMPTY_PAIRS) = range(9)
SPL_HASHER_LINEAR, SPL_HASHER_MLP, SPL_HASHER_DOWNPROJ = 0, 1, 2
SPL_F32, SPL_BF16 = 0, 1
SPL_HASHER_LINEAR, SPL_HASHER_MLP = 0, 1
SPL_ENCODE_EXACT, SPL_ENCODE_TC = 0, 1


class SpotlightError(RuntimeError):
    pass


class DimensionError(SpotlightError, ValueError):
    """spotlight::DimensionError (errors.hpp:9-13)."""


class NumericError(SpotlightError):
    """spotlight::NumericError (errors.hpp:21-25)."""


class FormatError(SpotlightError):
    """spotlight::FormatError (errors.hpp:15-19)."""


class IoError(SpotlightError):
    """spotlight::IoError (errors.hpp:32-35)."""


class CudaError(SpotlightError):
    pass


class EmptyPairError(SpotlightError):
    """errors.hpp:27-30"""


class StateError(SpotlightError):
    pass


_ERR = {SPL_E_DIMENSION: DimensionError, SPL_E_NUMERIC: NumericError, SPL_E_FORMAT: FormatError,
        SPL_E_IO: IoError, SPL_E_CUDA: CudaError, SPL_E_NCCL: SpotlightError,
        SPL_E_STATE: StateError, SPL_E_EMPTY_PAIRS: EmptyPairError}

_lib = None

vp = C.c_void_p
u32, u64, i32, f32, dbl = C.c_uint32, C.c_uint64, C.c_int, C.c_float, C.c_double
u32p = C.POINTER(C.c_uint32)

# name -> argtypes (restype spl_status = c_int unless listed in _RESTYPE)
_SIGS = {
    "spl_version": [],
    "spl_ctx_create": [i32, C.POINTER(vp)],
    "spl_ctx_destroy": [vp],
    "spl_last_error": [vp],
    "spl_reserve": [vp, u32, u64, u32, u32, u32],
    "spl_check_device_error": [vp, vp],
    "spl_launch_count": [vp],
    "spl_launch_log": [vp, C.c_char_p, C.c_size_t],
    "spl_device_alloc": [vp, C.c_size_t, C.POINTER(vp)],
    "spl_device_free": [vp, vp],
    "spl_memcpy": [vp, vp, vp, C.c_size_t, vp],
    "spl_memset": [vp, vp, i32, C.c_size_t, vp],
    "spl_stream_synchronize": [vp, vp],
    "spl_pack_bits": [vp, vp, u64, u32, vp, vp],
    "spl_unpack_bits": [vp, vp, u64, u32, vp, vp],
    "spl_nxor_scores": [vp, vp, u64, u32, vp, u32, vp, u32, u64, vp, u64, vp],
    "spl_top_k": [vp, vp, i32, u32, u64, u64, u32, vp, vp],
    "spl_hamming_topk": [vp, vp, u64, u32, vp, u32, vp, u32, u64, u32, vp, vp, vp],
    "spl_shard_histogram": [vp, vp, u64, u32, vp, u32, vp, u32, u64, vp, vp],
    "spl_shard_select": [vp, vp, u32, u32, u32, u32, vp, u32, u64, u32, vp, vp, vp, vp],
    "spl_plan_shard_host": [vp, u32, u32, u32, u32, u32p, u32p, u32p, u32p, u32p],
    "spl_hasher_create": [vp, i32, u32, u32, u32, u32, vp, vp, vp, C.POINTER(vp)],
    "spl_hasher_destroy": [vp],
    "spl_mlp_forward": [vp, vp, vp, u32, u32, vp, vp],
    "spl_encode": [vp, vp, vp, u32, u32, i32, vp, vp],
    "spl_encode_tc": [vp, vp, vp, i32, u32, u32, vp, vp, vp],
    "spl_encode_append": [vp, vp, vp, vp, u32, vp, vp, vp, i32, u64, vp, vp],
    "spl_sparse_attend": [vp, vp, vp, vp, i32, u64, u32, u32, vp, u64, vp, vp, u32, f32, vp, vp],
    "spl_sparse_attend_partial": [vp, vp, vp, vp, i32, u64, u32, u32, vp, u64, vp, vp, u32, f32,
                                  vp, vp],
    "spl_attend_combine": [vp, vp, u32, u32, u32, vp, vp],
    "spl_decode_step": [vp, vp, vp, vp, vp, u32, vp, vp, vp, i32, u64, vp, u64, u32, f32, vp, vp,
                        vp, vp],
    "spl_budget_from_rate": [dbl, u64, u32p],
    "spl_sharded_decode_step": [vp, vp, vp, vp, vp, vp, u32, i32, vp, vp, vp, i32, u64, vp, u64,
                                u32, f32, vp, vp, vp, vp, vp],
    "spl_oracle_topk": [vp, vp, vp, i32, u64, u32, u32, vp, u32, u64, f32, u32, vp, vp, vp, vp],
    "spl_iou": [vp, vp, vp, u64, vp, vp, u64, u32, vp, vp],
    "spl_project": [vp, vp, u64, u32, vp, u32, vp, vp],
    "spl_peer_create": [vp, u32, u32, u32, u32, C.POINTER(vp)],
    "spl_peer_ipc_handle": [vp, vp, vp],
    "spl_peer_open": [vp, vp, vp],
    "spl_peer_connect_local": [vp, C.POINTER(vp), u32],
    "spl_peer_destroy": [vp],
    "spl_hamming_topk_sharded": [vp, vp, vp, u64, u32, vp, u32, vp, u32, u64, u32, vp, vp, vp, vp],
    "spl_train_hasher": [vp, i32, u32, u32, u32, f32, vp, vp, vp, u32, vp, vp, vp, vp, vp, i32,
                         vp, C.POINTER(dbl), u32p, vp],
    "spl_train_partition_host": [vp, u32, u32, u64, vp, vp, vp, vp],
    "spl_train_lr_at": [u32, vp],
    "spl_train_last_loop_ms": [vp],
}
_RESTYPE = {"spl_version": C.c_char_p, "spl_train_lr_at": C.c_double,
            "spl_train_last_loop_ms": C.c_double, "spl_last_error": C.c_char_p, "spl_ctx_destroy": None,
            "spl_peer_destroy": None,
            "spl_hasher_destroy": None, "spl_launch_count": C.c_uint64,
            "spl_launch_log": C.c_size_t}


def header_symbols() -> list[str]:
    """Every function the C-ABI header declares."""
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(spl_[a-z0-9_]+)\s*\(", text)))


def load(path: Path | None = None):
    """Load libspl.so (raises if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path or os.environ.get("SPL_LIB", LIB_PATH))
    if not p.exists():
        raise FileNotFoundError(
            f"{p} missing: build the CUDA extension first (python -c 'import __graft_entry__ as g; g.build()')")
    lib = C.CDLL(str(p))
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPE.get(name, C.c_int)
    _lib = lib
    return lib


def _ptr(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        import torch

        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def budget_from_rate(rate: float, n: int) -> int:
    """attention_eval.cpp:266-272."""
    k = C.c_uint32(0)
    st = load().spl_budget_from_rate(rate, n, C.byref(k))
    if st:
        raise DimensionError("budget_from_rate: rate must lie in (0, 1]")
    return k.value


def plan_shard_host(all_hist, rank: int, k: int):
    """Host form of the sharded threshold / tie-quota plan for ONE problem.
    all_hist: numpy uint32 [R][L+1]. Returns dict(T, quota, take_eq, count, offset)."""
    import numpy as np

    h = np.ascontiguousarray(all_hist, dtype=np.uint32)
    R, L1 = h.shape
    outs = [C.c_uint32(0) for _ in range(5)]
    st = load().spl_plan_shard_host(h.ctypes.data, R, rank, L1 - 1, k, *[C.byref(o) for o in outs])
    if st:
        raise DimensionError("plan_shard_host: bad arguments")
    return dict(zip(("T", "quota", "take_eq", "count", "offset"), (o.value for o in outs)))


class RankConfig(C.Structure):
    """spl_rank_config = RankingLossConfig (ranking_loss.hpp:15-24); counts < 0: unset."""
    _fields_ = [("beta", dbl), ("alpha", dbl), ("maskout", dbl), ("max_top", C.c_int64),
                ("max_oth", C.c_int64), ("query_subsample", C.c_int64)]

    def __init__(self, beta=1.0, alpha=3.0, maskout=0.98, max_top=None, max_oth=None,
                 query_subsample=None):
        super().__init__(beta, alpha, maskout, -1 if max_top is None else max_top,
                         -1 if max_oth is None else max_oth,
                         -1 if query_subsample is None else query_subsample)


class TrainConfig(C.Structure):
    """spl_train_config = TrainConfig (trainer.hpp:18-37), same defaults."""
    _fields_ = [("num_iters", u32), ("warmup_iters", u32), ("batch", u32),
                ("holdout_queries", u32), ("seed", u64), ("max_lr", dbl), ("min_lr", dbl),
                ("adam_beta1", dbl), ("adam_beta2", dbl), ("adam_eps", dbl),
                ("weight_decay", dbl), ("grad_clip", dbl), ("soft_gamma", dbl),
                ("holdout_budget_rate", dbl)]

    def __init__(self, num_iters=8192, warmup_iters=81, batch=1, holdout_queries=128, seed=0,
                 max_lr=1e-3, min_lr=0.0, adam_beta1=0.9, adam_beta2=0.98, adam_eps=1e-8,
                 weight_decay=0.1, grad_clip=1.0, soft_gamma=64.0, holdout_budget_rate=0.02):
        super().__init__(num_iters, warmup_iters, batch, holdout_queries, seed, max_lr, min_lr,
                         adam_beta1, adam_beta2, adam_eps, weight_decay, grad_clip, soft_gamma,
                         holdout_budget_rate)


def train_partition_host(rank: RankConfig, q_train: int, n: int, seed: int):
    """partition_topk's draws (host; no GPU): (rows, top_pos, oth_pos, k_full)."""
    import numpy as np

    rows = np.zeros(max(q_train, 1), np.uint32)
    top = np.zeros(max(n, 1), np.uint32)
    oth = np.zeros(max(n, 1), np.uint32)
    cnt = np.zeros(4, np.uint32)
    st = load().spl_train_partition_host(C.byref(rank), q_train, n, seed, rows.ctypes.data,
                                         top.ctypes.data, oth.ctypes.data, cnt.ctypes.data)
    if st:
        raise StateError("train_partition_host failed")
    return rows[:cnt[0]].copy(), top[:cnt[1]].copy(), oth[:cnt[2]].copy(), int(cnt[3])


def train_lr_at(it: int, cfg: TrainConfig) -> float:
    """lr_at (trainer.cpp:35-46)."""
    return load().spl_train_lr_at(it, C.byref(cfg))


class Context:
    """One spl_ctx (workspace + device error word). Not thread-safe."""

    def __init__(self, device: int = 0):
        import torch

        self.lib = load()
        self.device = device
        torch.cuda.init()
        with torch.cuda.device(device):
            h = C.c_void_p()
            st = self.lib.spl_ctx_create(device, C.byref(h))
        if st:
            raise CudaError(f"spl_ctx_create(device={device}) failed with status {st}: "
                            "a Blackwell (sm_100) GPU is required")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.spl_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- plumbing
    def check(self, st: int):
        if st:
            msg = self.lib.spl_last_error(self.h).decode()
            raise _ERR.get(st, SpotlightError)(msg)

    def check_device_error(self, stream=None):
        self.check(self.lib.spl_check_device_error(self.h, _stream(stream)))

    def launches(self) -> int:
        return self.lib.spl_launch_count(self.h)

    def launch_log(self) -> list[str]:
        """Kernel names launched since the previous call (then cleared)."""
        buf = C.create_string_buffer(8192)
        self.lib.spl_launch_log(self.h, buf, len(buf))
        return [x for x in buf.value.decode().split(";") if x]

    def reserve(self, P, n_max, L, k, d=0):
        self.check(self.lib.spl_reserve(self.h, P, n_max, L, k, d))

    # -- bitcodes
    def pack_bits(self, bits, codes, stream=None):
        n, L = bits.shape
        self.check(self.lib.spl_pack_bits(self.h, _ptr(bits), n, L, _ptr(codes), _stream(stream)))

    def unpack_bits(self, codes, L, bits, stream=None):
        self.check(self.lib.spl_unpack_bits(self.h, _ptr(codes), codes.shape[0], L, _ptr(bits),
                                            _stream(stream)))

    def nxor_scores(self, codes, stride_rows, L, qcodes, P, n_valid, nvalid_div, n_max, scores,
                    scores_stride, stream=None):
        self.check(self.lib.spl_nxor_scores(self.h, _ptr(codes), stride_rows, L, _ptr(qcodes), P,
                                            _ptr(n_valid), nvalid_div, n_max, _ptr(scores),
                                            scores_stride, _stream(stream)))

    def top_k(self, scores, dtype_code, P, n, stride, k, idx, stream=None):
        self.check(self.lib.spl_top_k(self.h, _ptr(scores), dtype_code, P, n, stride, k, _ptr(idx),
                                      _stream(stream)))

    # -- K3
    def oracle_topk(self, q, keys, kv_dtype, cap, d, P, n_valid, nvalid_div, n_max, scale, k, idx,
                    cnt, logits=None, stream=None):
        """Exact dense top-k (the reference's oracle_topk) on the GPU."""
        self.check(self.lib.spl_oracle_topk(self.h, _ptr(q), _ptr(keys), kv_dtype, cap, d, P,
                                            _ptr(n_valid), nvalid_div, n_max, scale, k, _ptr(idx),
                                            _ptr(cnt), _ptr(logits), _stream(stream)))

    def project(self, a, m, k, b, n, c, stream=None):
        """c[m][n] = a[m][k] . b[k][n] with the reference matmul's FMA order."""
        self.check(self.lib.spl_project(self.h, _ptr(a), m, k, _ptr(b), n, _ptr(c), _stream(stream)))

    def iou(self, a, cnt_a, a_stride, b, cnt_b, b_stride, P, out, stream=None):
        self.check(self.lib.spl_iou(self.h, _ptr(a), _ptr(cnt_a), a_stride, _ptr(b), _ptr(cnt_b),
                                    b_stride, P, _ptr(out), _stream(stream)))

    # -- training
    def train_hasher(self, kind, d, h, L, gamma, w1, b1, w2, sequences, rank: RankConfig,
                     cfg: TrainConfig, loss_kind: int = 0, stream=None):
        """train_hasher (trainer.cpp:634-645) on the GPU. w1/b1/w2: float32 numpy
        arrays updated in place (b1/w2 None for linear / downproj); sequences:
        list of (queries, keys) float32 [n][d]. Returns dict(records [iters][3]
        = loss, violation_rate, lr; holdout_iou; skipped_steps)."""
        import numpy as np

        for a in (w1, b1, w2):
            if a is not None:
                assert a.dtype == np.float32 and a.flags.c_contiguous
        qs = np.ascontiguousarray(np.concatenate([q for q, _ in sequences]), dtype=np.float32)
        ks = np.ascontiguousarray(np.concatenate([k for _, k in sequences]), dtype=np.float32)
        lens = np.array([len(q) for q, _ in sequences], np.uint32)
        for q, k in sequences:
            if len(q) != len(k):
                raise DimensionError("train_hasher: queries and keys must be causally aligned")
        rec = np.zeros((max(cfg.num_iters, 1), 3), np.float64)
        iou = C.c_double(0.0)
        sk = C.c_uint32(0)
        self.check(self.lib.spl_train_hasher(
            self.h, kind, d, h, L, gamma, w1.ctypes.data,
            None if b1 is None else b1.ctypes.data, None if w2 is None else w2.ctypes.data,
            len(sequences), qs.ctypes.data, ks.ctypes.data, lens.ctypes.data, C.byref(rank),
            C.byref(cfg), loss_kind, rec.ctypes.data, C.byref(iou), C.byref(sk), _stream(stream)))
        return {"records": rec[:cfg.num_iters], "holdout_iou": iou.value,
                "skipped_steps": sk.value,
                "loop_ms": self.lib.spl_train_last_loop_ms(self.h)}

    def hamming_topk(self, codes, stride_rows, L, qcodes, P, n_valid, nvalid_div, n_max, k, idx,
                     cnt, stream=None):
        self.check(self.lib.spl_hamming_topk(self.h, _ptr(codes), stride_rows, L, _ptr(qcodes), P,
                                             _ptr(n_valid), nvalid_div, n_max, k, _ptr(idx),
                                             _ptr(cnt), _stream(stream)))

    def shard_histogram(self, codes, stride_rows, L, qcodes, P, n_valid, nvalid_div, n_max, hist,
                        stream=None):
        self.check(self.lib.spl_shard_histogram(self.h, _ptr(codes), stride_rows, L, _ptr(qcodes),
                                                P, _ptr(n_valid), nvalid_div, n_max, _ptr(hist),
                                                _stream(stream)))

    def shard_select(self, all_hist, R, rank, L, P, n_valid, nvalid_div, n_max, k, idx, cnt,
                     out_offset, stream=None):
        self.check(self.lib.spl_shard_select(self.h, _ptr(all_hist), R, rank, L, P, _ptr(n_valid),
                                             nvalid_div, n_max, k, _ptr(idx), _ptr(cnt),
                                             _ptr(out_offset), _stream(stream)))

    # -- encoders
    def hasher(self, w1, b1=None, w2=None, kind=SPL_HASHER_MLP) -> "Hasher":
        return Hasher(self, w1, b1, w2, kind)

    def peer(self, R, rank, P_max, L_max) -> "Peer":
        return Peer(self, R, rank, P_max, L_max)

    def hamming_topk_sharded(self, peer, codes, stride_rows, L, qcodes, P, n_valid, nvalid_div,
                             n_max, k, idx, cnt, out_offset, stream=None):
        """Fused sequence-sharded retrieval (in-kernel exchange over peer memory)."""
        self.check(self.lib.spl_hamming_topk_sharded(self.h, peer.h, _ptr(codes), stride_rows, L,
                                                     _ptr(qcodes), P, _ptr(n_valid), nvalid_div,
                                                     n_max, k, _ptr(idx), _ptr(cnt),
                                                     _ptr(out_offset), _stream(stream)))

    # -- attention
    def sparse_attend(self, q, kcache, vcache, kv_dtype, stride_rows, d, P, idx, idx_stride, cnt,
                      n_valid, nvalid_div, scale, out, stream=None):
        self.check(self.lib.spl_sparse_attend(self.h, _ptr(q), _ptr(kcache), _ptr(vcache), kv_dtype,
                                              stride_rows, d, P, _ptr(idx), idx_stride, _ptr(cnt),
                                              _ptr(n_valid), nvalid_div, scale, _ptr(out),
                                              _stream(stream)))

    def sparse_attend_partial(self, q, kcache, vcache, kv_dtype, stride_rows, d, P, idx,
                              idx_stride, cnt, own_row, nvalid_div, scale, partials, stream=None):
        self.check(self.lib.spl_sparse_attend_partial(self.h, _ptr(q), _ptr(kcache), _ptr(vcache),
                                                      kv_dtype, stride_rows, d, P, _ptr(idx),
                                                      idx_stride, _ptr(cnt), _ptr(own_row),
                                                      nvalid_div, scale, _ptr(partials),
                                                      _stream(stream)))

    def attend_combine(self, partials, R, P, d, out, stream=None):
        self.check(self.lib.spl_attend_combine(self.h, _ptr(partials), R, P, d, _ptr(out),
                                               _stream(stream)))


class Peer:
    """spl_peer: this rank's member of a fused-sharding peer group."""

    def __init__(self, ctx: Context, R, rank, P_max, L_max):
        self.ctx = ctx
        h = vp()
        ctx.check(ctx.lib.spl_peer_create(ctx.h, R, rank, P_max, L_max, C.byref(h)))
        self.h = h
        self.R, self.rank = R, rank

    def ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(64)
        self.ctx.check(self.ctx.lib.spl_peer_ipc_handle(self.ctx.h, self.h, buf))
        return buf.raw

    def open(self, handles):
        """handles: the R 64-byte handles in rank order (e.g. all-gathered)."""
        blob = b"".join(handles)
        assert len(blob) == 64 * self.R
        buf = C.create_string_buffer(blob, len(blob))
        self.ctx.check(self.ctx.lib.spl_peer_open(self.ctx.h, self.h, buf))

    @staticmethod
    def connect_local(ctx: Context, peers):
        arr = (vp * len(peers))(*[p.h for p in peers])
        ctx.check(ctx.lib.spl_peer_connect_local(ctx.h, arr, len(peers)))

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.spl_peer_destroy(self.h)
            self.h = None


class Hasher:
    """spl_hasher: a per-head bank of MLP (or linear) hashers on the device."""

    def __init__(self, ctx: Context, w1, b1=None, w2=None, kind=SPL_HASHER_MLP):
        import numpy as np

        self.ctx = ctx
        w1 = np.ascontiguousarray(w1, np.float32)
        if kind == SPL_HASHER_MLP:
            b1 = np.ascontiguousarray(b1, np.float32)
            w2 = np.ascontiguousarray(w2, np.float32)
            H, d, h = w1.shape
            L = w2.shape[2]
        else:
            H, d, L = w1.shape
            h = 0
        self.kind, self.H, self.d, self.hidden, self.L = kind, H, d, h, L
        self.h = None
        out = C.c_void_p()
        ctx.check(ctx.lib.spl_hasher_create(ctx.h, kind, H, d, h, L, w1.ctypes.data,
                                            b1.ctypes.data if b1 is not None else None,
                                            w2.ctypes.data if w2 is not None else None,
                                            C.byref(out)))
        self.h = out

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.spl_hasher_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def mlp_forward(self, x, B, m, pre, stream=None):
        self.ctx.check(self.ctx.lib.spl_mlp_forward(self.ctx.h, self.h, _ptr(x), B, m, _ptr(pre),
                                                    _stream(stream)))

    def encode(self, x, B, m, codes, mode=SPL_ENCODE_EXACT, stream=None):
        self.ctx.check(self.ctx.lib.spl_encode(self.ctx.h, self.h, _ptr(x), B, m, mode, _ptr(codes),
                                               _stream(stream)))

    def encode_tc(self, x, x_dtype, B, m, codes, pre=None, stream=None):
        """tcgen05 bulk encoder (K2): x [B][H][m][d] f32 / bf16 -> codes; pre
        (optional f32 [B][H][m][L]) receives the pre-activations."""
        self.ctx.check(self.ctx.lib.spl_encode_tc(self.ctx.h, self.h, _ptr(x), x_dtype, B, m,
                                                  _ptr(codes), _ptr(pre), _stream(stream)))

    def encode_append(self, k_new, v_new, B, codes, kcache, vcache, kv_dtype, cap, pos,
                      stream=None):
        self.ctx.check(self.ctx.lib.spl_encode_append(self.ctx.h, self.h, _ptr(k_new), _ptr(v_new),
                                                      B, _ptr(codes), _ptr(kcache), _ptr(vcache),
                                                      kv_dtype, cap, _ptr(pos), _stream(stream)))

    def decode_step(self, q, k_new, v_new, B, codes, kcache, vcache, kv_dtype, cap, n_valid,
                    n_max, k, scale, idx, cnt, out, stream=None):
        self.ctx.check(self.ctx.lib.spl_decode_step(self.ctx.h, self.h, _ptr(q), _ptr(k_new),
                                                    _ptr(v_new), B, _ptr(codes), _ptr(kcache),
                                                    _ptr(vcache), kv_dtype, cap, _ptr(n_valid),
                                                    n_max, k, scale, _ptr(idx), _ptr(cnt),
                                                    _ptr(out), _stream(stream)))

    def sharded_decode_step(self, peer, q, k_new, v_new, B, owner, codes, kcache, vcache, kv_dtype,
                            cap, n_valid, n_max, k, scale, idx, cnt, out_offset, out, stream=None):
        """One rank of a sequence-sharded decode step (spl_sharded_decode_step)."""
        self.ctx.check(self.ctx.lib.spl_sharded_decode_step(
            self.ctx.h, peer.h, self.h, _ptr(q), _ptr(k_new), _ptr(v_new), B, 1 if owner else 0,
            _ptr(codes), _ptr(kcache), _ptr(vcache), kv_dtype, cap, _ptr(n_valid), n_max, k, scale,
            _ptr(idx), _ptr(cnt), _ptr(out_offset), _ptr(out), _stream(stream)))
