"""The N>1 product path on one GPU: bench.py under torchrun with two ranks (gloo collectives, both
ranks on cuda:0) shards ONE dataset into per-rank contiguous chunk ranges, each rank copies and decodes its shard
through libcdm, and the all-reduced H9 checksum total and decoded bytes equal the single-rank run's, with no device
error bits (the union of the rank outputs is the 1-GPU output).  NCCL needs one GPU per rank, so the 8-GPU
NCCL run itself stays unmeasured on this one-GPU pool; its code path differs only in the backend."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARGS = ["--workload", "config4", "--sf", "1.5", "--steps", "2", "--warmup", "1", "--no-cpu-baseline"]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _line(out: str) -> dict:
    lines = [x for x in out.splitlines() if x.startswith("{")]
    assert lines, out[-3000:]
    return json.loads(lines[-1])


@pytest.mark.timeout(900)
def test_two_ranks_one_gpu_match_one_rank():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    one = subprocess.run([sys.executable, "bench.py", *ARGS], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert one.returncode == 0, one.stderr[-3000:]
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", *ARGS, "--gpus", "2",
                          "--dist-backend", "gloo", "--device-map", "zero"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert two.returncode == 0, two.stderr[-3000:]
    a, b = _line(one.stdout), _line(two.stdout)
    assert b["n_gpus"] == 2 and a["n_gpus"] == 1
    assert a["errors"] == 0 and b["errors"] == 0
    assert b["config"]["decoded_bytes_per_step"] == a["config"]["decoded_bytes_per_step"]
    assert b["config"]["chunks"] == a["config"]["chunks"]
    assert b["parity"]["checksum_total"] == a["parity"]["checksum_total"]
    assert b["e2e"]["pcie_h2d_gbs_each_rank_alone"] and len(b["e2e"]["pcie_h2d_gbs_all_ranks_concurrent"]) == 2
