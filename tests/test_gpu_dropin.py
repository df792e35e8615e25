"""The C++ drop-in (libspotlight_b200.so) through its own C++ test binary,
mirroring the reference's doctest suite, plus bit-exact diffs against the
unmodified reference when oracle/_ref was built."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def test_cpp_dropin_suite(tmp_path):
    subprocess.run(["make", "-s", "-C", str(ROOT / "tests" / "cpp")], check=True)
    r = subprocess.run([str(ROOT / "build" / "test_dropin")], cwd=ROOT, capture_output=True,
                       text=True, timeout=180)
    print(r.stdout)
    print(r.stderr)
    assert r.returncode == 0, r.stderr[-4000:]
    assert " 0 failed" in r.stdout
