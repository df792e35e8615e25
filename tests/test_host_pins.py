"""Host-side drop-in pieces pinned against the unmodified reference (no GPU):
the initialisers (mlp_gaussian_init hashers.cpp:41-63, qr_rotation_init
:37-39, downproj_init :65-74, random_rotation linalg.cpp:80-92) produce
bit-identical parameters, and the SPLH (hashers.cpp:184-246) and SPLC
(bitcodes.cpp:138-160) files are byte-identical in both directions: a file
the reference writes loads through the drop-in and re-writes to the same
bytes, a file the drop-in writes loads through the reference with the same
contents; malformed files are rejected with the same exception and text."""
import ctypes as C
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
TOOL = ROOT / "build" / "dropin_hostio"


@pytest.fixture(scope="module")
def tool():
    subprocess.run(["make", "-s", "-C", str(ROOT / "tests" / "cpp"), "hostio"], check=True)
    return TOOL


@pytest.fixture(scope="module")
def R(ref):
    L = ref.lib
    f32p, u32p = C.POINTER(C.c_float), C.POINTER(C.c_uint32)
    L.spotref_downproj_init.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, f32p]
    L.spotref_random_rotation.argtypes = [C.c_uint32, C.c_uint64, C.POINTER(C.c_double)]
    L.spotref_write_hasher.argtypes = [C.c_char_p, C.c_int, C.c_uint32, C.c_uint32, C.c_uint32,
                                       C.c_float, f32p, f32p, f32p]
    L.spotref_read_hasher.argtypes = [C.c_char_p, u32p, f32p, f32p, f32p, f32p]
    L.spotref_write_code_index.argtypes = [C.c_char_p, u32p, C.c_uint32, C.c_uint32]
    L.spotref_read_code_index.argtypes = [C.c_char_p, u32p, u32p, u32p]
    return L


def ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t)) if a is not None else None


def run(tool, *args):
    r = subprocess.run([str(tool), *map(str, args)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    return r.stdout.strip()


def ref_read_hasher(R, path):
    dims = np.zeros(4, np.uint32)
    g = C.c_float()
    assert R.spotref_read_hasher(str(path).encode(), ptr(dims, C.c_uint32), C.byref(g), None, None,
                                 None) == 0
    kind, d, h, L = map(int, dims)
    w1 = np.zeros(d * (h if kind == 1 else L), np.float32)
    b1 = np.zeros(max(h, 1), np.float32)
    w2 = np.zeros(max(h * L, 1), np.float32)
    assert R.spotref_read_hasher(str(path).encode(), ptr(dims, C.c_uint32), C.byref(g),
                                 ptr(w1, C.c_float), ptr(b1, C.c_float), ptr(w2, C.c_float)) == 0
    return kind, (d, h, L), g.value, w1, b1[:h], w2[:h * L]


@pytest.mark.parametrize("d,h,L,seed", [(128, 128, 128, 0), (128, 128, 256, 7), (36, 20, 64, 99)])
def test_mlp_gaussian_init_bit_identical(tool, ref, tmp_path, d, h, L, seed):
    w1 = np.zeros(d * h, np.float32)
    b1 = np.zeros(h, np.float32)
    w2 = np.zeros(h * L, np.float32)
    assert ref.lib.spotref_mlp_gaussian_init(d, h, L, 64.0, seed, w1, b1, w2) == 0
    run(tool, "gauss", d, h, L, 64.0, seed, tmp_path / "g.bin")
    got = np.fromfile(tmp_path / "g.bin", np.float32)
    assert got.tobytes() == np.concatenate([w1, b1, w2]).tobytes()


@pytest.mark.parametrize("d,seed", [(1, 5), (2, 0), (16, 3), (32, 8), (128, 1234)])
def test_rotations_bit_identical(tool, R, tmp_path, d, seed):
    want = np.zeros(d * d, np.float64)
    assert R.spotref_random_rotation(d, seed, ptr(want, C.c_double)) == 0
    run(tool, "rotation", d, seed, tmp_path / "r.bin")
    assert np.fromfile(tmp_path / "r.bin", np.float64).tobytes() == want.tobytes()
    wq = np.zeros(d * d, np.float32)
    assert R.spotref_qr_rotation_init(d, seed, wq) == 0
    run(tool, "qr", d, seed, tmp_path / "q.bin")
    assert np.fromfile(tmp_path / "q.bin", np.float32).tobytes() == wq.tobytes()
    r = max(1, d // 4)
    wd = np.zeros(d * r, np.float32)
    assert R.spotref_downproj_init(d, r, seed, ptr(wd, C.c_float)) == 0
    run(tool, "downproj", d, r, seed, tmp_path / "p.bin")
    assert np.fromfile(tmp_path / "p.bin", np.float32).tobytes() == wd.tobytes()


def test_init_rejections_match(tool, tmp_path):
    r = subprocess.run([str(tool), "downproj", "8", "9", "1", str(tmp_path / "x")],
                       capture_output=True, text=True)
    assert r.returncode == 1 and "downproj_init: need 1 <= r <= d" in r.stderr
    r = subprocess.run([str(tool), "rotation", "0", "1", str(tmp_path / "x")], capture_output=True,
                       text=True)
    assert r.returncode == 1 and "random_rotation: d must be >= 1" in r.stderr


def test_splh_reference_to_dropin(tool, R, ref, tmp_path):
    """Reference-written SPLH (all three kinds) -> drop-in read + write ->
    the same bytes."""
    d, h, L = 128, 128, 256
    w1 = np.zeros(d * h, np.float32)
    b1 = np.zeros(h, np.float32)
    w2 = np.zeros(h * L, np.float32)
    assert ref.lib.spotref_mlp_gaussian_init(d, h, L, 48.0, 11, w1, b1, w2) == 0
    b1[:] = np.random.default_rng(1).standard_normal(h).astype(np.float32)
    proj = np.random.default_rng(2).standard_normal(d * 64).astype(np.float32)
    cases = [("mlp", 1, d, h, L, 48.0, w1, b1, w2), ("linear", 0, d, 0, 64, 0.0, proj, None, None),
             ("downproj", 2, d, 0, 64, 0.0, proj, None, None)]
    for name, kind, dd, hh, LL, g, a, b, c in cases:
        src = tmp_path / f"{name}.splh"
        assert R.spotref_write_hasher(str(src).encode(), kind, dd, hh, LL, g, ptr(a, C.c_float),
                                      ptr(b, C.c_float), ptr(c, C.c_float)) == 0
        out = tmp_path / f"{name}.dropin.splh"
        run(tool, "rehasher", src, out)
        assert out.read_bytes() == src.read_bytes(), name
        assert run(tool, "readhasher", src) == "ok"


def test_splh_dropin_to_reference(tool, R, tmp_path):
    """Drop-in-written SPLH (from the drop-in's own initialisers) -> the
    reference reads the same parameters and re-writes the same bytes."""
    for args, kind in [(("hasher_mlp", 128, 128, 128, 64.0, 3), 1), (("hasher_linear", 32, 5), 0),
                       (("hasher_downproj", 64, 16, 7), 2)]:
        f = tmp_path / f"{args[0]}.splh"
        run(tool, *args, f)
        k, dims, g, w1, b1, w2 = ref_read_hasher(R, f)
        assert k == kind
        back = tmp_path / f"{args[0]}.ref.splh"
        assert R.spotref_write_hasher(str(back).encode(), k, *dims, g, ptr(w1, C.c_float),
                                      ptr(b1, C.c_float) if k == 1 else None,
                                      ptr(w2, C.c_float) if k == 1 else None) == 0
        assert back.read_bytes() == f.read_bytes(), args[0]


@pytest.mark.parametrize("n,L", [(1, 32), (1000, 128), (257, 256), (0, 64)])
def test_splc_both_directions(tool, R, tmp_path, n, L):
    rng = np.random.default_rng(n + L)
    words = rng.integers(0, 2**32, size=n * (L // 32), dtype=np.uint32)
    a = tmp_path / "ref.splc"
    assert R.spotref_write_code_index(str(a).encode(), ptr(words, C.c_uint32), n, L) == 0
    b = tmp_path / "dropin.splc"
    run(tool, "recodes", a, b)
    assert b.read_bytes() == a.read_bytes()
    raw = tmp_path / "w.bin"
    words.tofile(raw)
    c = tmp_path / "dropin2.splc"
    run(tool, "codes_raw", n, L, raw, c)
    assert c.read_bytes() == a.read_bytes()
    nn, LL = C.c_uint32(), C.c_uint32()
    back = np.zeros(max(words.size, 1), np.uint32)
    assert R.spotref_read_code_index(str(c).encode(), C.byref(nn), C.byref(LL),
                                     ptr(back, C.c_uint32)) == 0
    assert (nn.value, LL.value) == (n, L)
    assert back[:words.size].tobytes() == words.tobytes()


def _ref_read_error(R, path, codes):
    if codes:
        nn, LL = C.c_uint32(), C.c_uint32()
        st = R.spotref_read_code_index(str(path).encode(), C.byref(nn), C.byref(LL), None)
    else:
        dims = np.zeros(4, np.uint32)
        g = C.c_float()
        st = R.spotref_read_hasher(str(path).encode(), ptr(dims, C.c_uint32), C.byref(g), None,
                                   None, None)
    names = {0: "ok", 1: "DimensionError", 3: "FormatError", 4: "IoError"}
    R.spotref_last_error.restype = C.c_char_p
    return "ok" if st == 0 else f"{names.get(st, st)}: {R.spotref_last_error().decode()}"


def test_malformed_files_rejected_alike(tool, R, tmp_path):
    """Truncations, a bad magic, a bad version, a missing file: the drop-in
    throws the reference's exception type with the reference's message."""
    good_h = tmp_path / "g.splh"
    run(tool, "hasher_mlp", 16, 8, 32, 64.0, 1, good_h)
    good_c = tmp_path / "g.splc"
    raw = tmp_path / "w.bin"
    np.arange(3 * 2, dtype=np.uint32).tofile(raw)
    run(tool, "codes_raw", 3, 64, raw, good_c)
    for good, codes in [(good_h, False), (good_c, True)]:
        data = good.read_bytes()
        variants = {
            "magic": b"XXXX" + data[4:],
            "version": data[:4] + b"\x07\x00\x00\x00" + data[8:],
            "trunc_header": data[:6],
            "trunc_payload": data[:-3],
            "empty": b"",
        }
        for name, blob in variants.items():
            p = tmp_path / f"{name}{'.splc' if codes else '.splh'}"
            p.write_bytes(blob)
            want = _ref_read_error(R, p, codes)
            got = run(tool, "readcodes" if codes else "readhasher", p)
            assert got == want, (name, codes)
        missing = tmp_path / "does_not_exist"
        assert run(tool, "readcodes" if codes else "readhasher", missing) == \
            _ref_read_error(R, missing, codes)
