"""The reference's OWN doctest translation units, unmodified, through the
drop-in: proj/tests/test_bitcodes.cpp, test_hashers.cpp and
test_attention_eval.cpp compiled
against include/spotlight/ and linked against libspotlight_b200.so
(oracle/Makefile `reftests`; tests/cpp/doctest/doctest.h stands in for the
unshipped vendor/doctest.h). Every compute call inside them is a B200 launch.
The binary is built where /root/reference exists and travels with the repo."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "oracle" / "_ref" / "reftests"
pytestmark = pytest.mark.gpu


def test_reference_doctest_suites_through_dropin():
    if not BIN.exists():
        pytest.skip("oracle/_ref/reftests not built (no /root/reference when the repo was built)")
    r = subprocess.run([str(BIN)], cwd=ROOT, capture_output=True, text=True, timeout=600)
    print(r.stdout[-6000:])
    print(r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-4000:]
    assert "Status: SUCCESS" in r.stdout
    # all 31 reference cases ran (11 in test_bitcodes.cpp, 12 in test_hashers.cpp,
    # 8 in test_attention_eval.cpp)
    assert "test cases: 31 | 31 passed | 0 failed | 0 skipped" in r.stdout
