"""Multi-process runs of the engine under torch.distributed.

CPU: gloo, world sizes 2-3, test kernels -- the DistComm path (per-stage
process groups, all-reduce, vocab-parallel argmax MAX, stage hand-off
send/recv, token return, id broadcast) must reproduce the oracle's ids.
GPU (>= 2 devices): NCCL with the C-ABI kernels, same check."""

import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(nproc, args, timeout=600, **extra_env):
    env = dict(os.environ, OMP_NUM_THREADS="2", **extra_env)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}",
           str(ROOT / "tools" / "dist_generate.py"), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "ids match oracle: True" in r.stdout or "--dtype" in " ".join(args), r.stdout
    return r.stdout


@pytest.mark.parametrize("plan,layers", [("2,1", "3,1"), ("1,2", "1,3"), ("1,1", "2,2"), ("4,2,2", "2,1,1")])
def test_gloo_asymmetric_plans(plan, layers):
    n = sum(int(x) for x in plan.split(","))
    _run(n, ["--plan", plan, "--layers", layers, "--cpu"])


def _gpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.gpu
@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("plan,layers,graphs", [("1,1", "3,1", False), ("1,1", "2,2", True)])
def test_nccl_two_stage_fp32(plan, layers, graphs):
    _run(2, ["--plan", plan, "--layers", layers] + (["--graphs"] if graphs else []))


@pytest.mark.gpu
@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_tp2_stage_nvlink_allreduce(dtype):
    """Single TP=2 stage: the decode step's all-reduces run in the fused NVLink
    peer-memory kernel (graphs on); ids must match the oracle."""
    _run(2, ["--plan", "2", "--layers", "4", "--graphs", "--dtype", dtype])


@pytest.mark.gpu
@pytest.mark.skipif(_gpus() < 3, reason="needs >= 3 GPUs")
def test_nccl_asymmetric_21_fp32_graphs():
    _run(3, ["--plan", "2,1", "--layers", "3,1", "--graphs"])


@pytest.mark.gpu
@pytest.mark.skipif(_gpus() < 3, reason="needs >= 3 GPUs")
def test_nccl_microbatched_prefill_fp32_graphs():
    """Pipelined prefill (2 micro-batches over NCCL) + P2P decode hand-offs."""
    _run(3, ["--plan", "2,1", "--layers", "3,1", "--graphs"], HX_PREFILL_MB="2")


def test_gloo_microbatched_prefill():
    _run(2, ["--plan", "1,1", "--layers", "2,2", "--cpu"], HX_PREFILL_MB="2")


@pytest.mark.gpu
@pytest.mark.skipif(_gpus() < 4, reason="needs >= 4 GPUs")
def test_nccl_asymmetric_211_bf16_graphs():
    _run(4, ["--plan", "2,1,1", "--layers", "2,1,1", "--dtype", "bf16", "--graphs"])


@pytest.mark.gpu
@pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("n", [2, 4])
def test_peer_allreduce_push_equals_pull(n):
    """The flag-free push all-reduce gives the same residual bits as the
    flag/pull one (normalised output within 1 bf16 ulp: different RMS reduction
    width), and both stay bitwise replicated across the TP ranks."""
    if _gpus() < n:
        pytest.skip(f"needs {n} GPUs")
    env = dict(os.environ, OMP_NUM_THREADS="2")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}", str(ROOT / "tools" / "ar_bench.py"), "--check"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("push==pull: True, replicated: True") == n, r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("plan,layers", [("1,2", "2,2"), ("2,2", "3,1"), ("1,2,1", "1,2,1")])
def test_nccl_reshard_topologies_fp32_graphs(plan, layers):
    """TP_j -> TP_{j+1} reshards of the [4,2,2] shape class (fan-out 1 -> 2,
    equal 2 -> 2, fan-in 2 -> 1, token return to a wider stage 0) over the
    P2P hand-off kernels inside the decode graphs; ids must match the oracle."""
    n = sum(int(x) for x in plan.split(","))
    if _gpus() < n:
        pytest.skip(f"needs {n} GPUs")
    _run(n, ["--plan", plan, "--layers", layers, "--graphs"])
