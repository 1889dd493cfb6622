"""Multi-GPU parity of the NVLink P2P sketch_allreduce path (needs >= 2 GPUs)."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("name,law", [("tiny", "dyadic"), ("ncf", "dyadic"), ("ncf", "gauss")])
def test_p2p_allreduce_parity(world, name, law):
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29533",
           os.path.join(ROOT, "tests", "mgpu_worker.py"), name, law]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("name,law", [("tiny", "dyadic"), ("ncf", "dyadic"), ("ncf", "gauss")])
def test_sharded_decode_parity(world, name, law):
    """NEXT-2: reduce-scatter -> decode the own shard -> all-gather (tests/mgpu_worker.py)."""
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29534",
           os.path.join(ROOT, "tests", "mgpu_worker.py"), name, law, "3", "sharded"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("mode", ["nvls", "sharded-nvls"])
@pytest.mark.parametrize("name,law", [("tiny", "dyadic"), ("ncf", "gauss")])
def test_nvls_parity(world, mode, name, law):
    """NEXT-2: in-switch aggregation through an NVSwitch multicast object, for the
    replicated all-reduce and for the sharded reduce-scatter / all-gather."""
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29535",
           os.path.join(ROOT, "tests", "mgpu_worker.py"), name, law, "3", mode]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("mode", ["sharded-overflow", "sharded-nvls-overflow"])
def test_sharded_overflow_is_visible_on_every_rank(world, mode):
    """A shard whose decode overflows publishes an overflow mark; every rank fills
    that shard with NaN instead of a stale list (comm.cu all-gather)."""
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29536",
           os.path.join(ROOT, "tests", "mgpu_worker.py"), "tiny", "dyadic", "1", mode]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
