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
