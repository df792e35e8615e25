"""Multi-process peer group on one GPU: R processes (torch.distributed.run,
gloo) exchange IPC handles and run the fused sequence-sharded retrieval,
whose histogram exchange happens inside the kernels across processes. The
processes time-share the GPU, so each kernel waits (inside the kernel) for
the others to be scheduled — the exchange protocol has to survive that."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("R", [2, 3])
def test_fused_sharded_multiprocess(R):
    env = dict(os.environ)
    env.pop("SPL_K3_PATH", None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={R}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + R),
           str(ROOT / "tests" / "mp_fused_shard.py")]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    assert "MP_FUSED_SHARD OK" in r.stdout


@pytest.mark.parametrize("R", [2, 3])
def test_sharded_decode_multiprocess(R):
    """spl_sharded_decode_step across R processes (in-kernel exchange of the
    histograms and of the attention partials through IPC-mapped peer memory):
    indices bit-exact and output within 1e-3 of the single-GPU step."""
    env = dict(os.environ)
    env.pop("SPL_K3_PATH", None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={R}",
           "--master-addr", "127.0.0.1", "--master-port", str(29640 + R),
           str(ROOT / "tests" / "mp_sharded_decode.py")]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    assert "MP_SHARDED_DECODE OK" in r.stdout
