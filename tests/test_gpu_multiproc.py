"""The multi-process batch path on one GPU: bench.py under torchrun with
2 and 3 ranks sharing the box's GPU.  Rank r evaluates its shard of ONE batch with
phc_eval_jacobian_batch_range and stores F, J into rank 0's buffers through CUDA IPC mappings;
rank 0 then re-evaluates the whole batch alone and the gathered result must be bitwise equal.
(The ranks' kernels never wait on one another: each writes its own rows; the control plane is
gloo because NCCL refuses two ranks on one GPU.)"""
import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,workload,points", [(2, "batch", 4096), (3, "c3", 301)])
def test_torchrun_ipc_gather_bitwise(world, workload, points):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", str(world), "--workload", workload, "--points", str(points), "--steps", "2", "--warmup", "1",
           "--e2e-steps", "1", "--no-flush", "--verify"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    out = json.loads(line)
    assert out["n_gpus"] == world and out["scaling"] == "strong"
    assert out["config"]["gather"].startswith("fused NVLink stores"), out["config"]["gather"]
    assert out["verified_bitwise_vs_one_process"] is True
    assert out["outputs_finite"] and out["value"] > 0
