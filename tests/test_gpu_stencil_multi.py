"""Mapped stencil + 3-D matmul + peer-GEMM checks on the box's GPUs."""

import json
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _ngpus():
    import torch

    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _run(script, n, port):
    if n == 1:
        cmd = [sys.executable, str(ROOT / "tests" / script)]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port", str(port),
               str(ROOT / "tests" / script)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-4000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("{")][-1]
    return json.loads(line)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_stencil(n):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    v = _run("dist_stencil_check.py", n, 29700 + n)
    assert v["ok"], v


@pytest.mark.parametrize("n", [2, 4, 8])
def test_grid3d(n):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    v = _run("dist_grid3d_check.py", n, 29710 + n)
    assert v["ok"], v


def test_peer_gemm_reduce_add():
    if _ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    v = _run("dist_peer_gemm_check.py", 2, 29720)
    assert v["ok"], v


@pytest.mark.parametrize("n", [2, 4])
def test_peer_barrier(n):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    v = _run("dist_peer_barrier_check.py", n, 29740 + n)
    assert v["ok"], v


@pytest.mark.parametrize("n", [1, 4, 8])
def test_cannon(n):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    v = _run("dist_cannon_check.py", n, 29730 + n)
    assert v["ok"], v


@pytest.mark.parametrize("n", [1, 2, 4])
def test_sharded_mapping(n):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    v = _run("dist_distmap_check.py", n, 29750 + n)
    assert v["ok"], v


@pytest.mark.parametrize("n", [1, 2, 4])
def test_circuit(n):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    v = _run("dist_circuit_check.py", n, 29770 + n)
    assert v["ok"], v


@pytest.mark.parametrize("n", [1, 2, 4])
def test_hydro(n):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    v = _run("dist_hydro_check.py", n, 29790 + n)
    assert v["ok"], v


# (script, ranks): every multi-rank path, with the ranks sharing however many GPUs the
# box has (rank r on GPU r % n).  Host collectives go over gloo and same-GPU peers
# talk through CUDA IPC -- possible because no executor step uses NCCL -- so a
# 1-GPU box runs the 4- and 8-GPU schedules, barriers and peer-memory exchanges
# bit for bit (only the timing differs).
OVERSUB = [("cannon", 4), ("cannon", 8), ("summa", 4), ("summa", 8), ("grid3d", 4),
           ("grid3d", 8), ("stencil", 4), ("stencil", 8), ("circuit", 4), ("circuit", 8),
           ("hydro", 4), ("hydro", 8), ("peer_barrier", 2), ("peer_barrier", 4)]


@pytest.mark.parametrize("script,ranks", OVERSUB)
def test_ranks_sharing_gpus(script, ranks):
    """The N=4 / N=8 paths (Cannon configs[0] on 2x2 with the reference's owners,
    Solomonik 2.5D with c=2, (2,2) / (2,4) / (4,2) SUMMA grids, 2x2x2 and COSMA
    grids, 4- and 8-way stencil / circuit / hydro) against the float64 oracle."""
    import os

    n = _ngpus()
    if n < 1:
        pytest.skip("needs a GPU")
    if n >= ranks:
        pytest.skip("one rank per GPU is covered by the NCCL tests above")
    env = dict(os.environ, PM_TEST_BACKEND="gloo", PM_HANG_DUMP_S="500")
    port = 29810 + 16 * [s for s, _ in OVERSUB].index(script) + ranks
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={ranks}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           str(ROOT / "tests" / f"dist_{script}_check.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-4000:]
    v = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert v["ok"] and v["world"] == ranks, v
