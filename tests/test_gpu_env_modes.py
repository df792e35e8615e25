"""Launch-mode variants that libspl reads once per process from the
environment, each run in its own process through tests/env_mode_case.py
(retrieval, K4 over bf16 / f32 K/V, one served decode step — all against the
C oracle):

* SPL_PDL=1: programmatic dependent launch along K1 -> K3 -> K4 (off by
  default: measured slower);
* SPL_K4=lane: the round-1 lane-per-row attention kernel kept for A/B;
* SPL_K4_NB=1 / 2: fewer 8-row batches per K4 warp than the default 4.
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("env", [{"SPL_PDL": "1"}, {"SPL_K4": "lane"}, {"SPL_K4_NB": "1"},
                                 {"SPL_K4_NB": "2"}, {}],
                         ids=["pdl", "k4_lane", "k4_nb1", "k4_nb2", "default"])
def test_env_mode_parity(env):
    e = dict(os.environ)
    for v in ("SPL_PDL", "SPL_K4", "SPL_K4_NB", "SPL_K3_PATH", "SPL_K3_COOP", "SPL_DECODE_FUSED"):
        e.pop(v, None)
    e.update(env)
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "env_mode_case.py")], env=e,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.stdout + r.stderr)[-2000:]
    assert "env mode case: OK" in r.stdout
