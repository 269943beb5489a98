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


EIGHT = ["cannon", "grid3d", "summa", "stencil", "circuit", "hydro"]


@pytest.mark.parametrize("script", EIGHT)
def test_eight_ranks_on_fewer_gpus(script):
    """The N=8 paths (Solomonik 2.5D with c=2, 2x2x2 / (2,4) / (4,2) grids, 8-way
    stencil / circuit / hydro) with 8 ranks sharing the box's GPUs: host collectives
    over gloo, peers on the same GPU through CUDA IPC (the executors' data path and
    barriers use peer memory only, no NCCL)."""
    import os

    n = _ngpus()
    if n < 2:
        pytest.skip("needs 2+ GPUs")
    env = dict(os.environ, PM_TEST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr", "127.0.0.1", "--master-port", str(29810 + EIGHT.index(script)),
           str(ROOT / "tests" / f"dist_{script}_check.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-4000:]
    v = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert v["ok"] and v["world"] == 8, v
