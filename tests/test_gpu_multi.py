"""Multi-GPU parity through real NCCL collectives (-m gpu; needs >= 2 GPUs, else skipped)."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("rs_mode,gather_mode", [("ce", "ce"), ("push", "push")])
def test_multi_gpu_parity(rs_mode, gather_mode):
    """Fused collective variants: copy-engine gather + copy-engine reduce-scatter (the defaults) and the
    in-kernel variants (CP_GATHER_MODE=push: the consuming GEMM pushes its block; CP_RS_MODE=push: the
    dgrad epilogue stores the partials into the owners' slots).  The SM-load pull variant of the
    reduce-scatter runs in the loopback test."""
    n = min(torch.cuda.device_count(), 4)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={29517 if rs_mode == 'ce' else 29518}",
           os.path.join(ROOT, "tests", "multi_gpu_check.py")]
    env = dict(os.environ, CP_RS_MODE=rs_mode, CP_GATHER_MODE=gather_mode)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
