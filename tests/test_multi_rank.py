"""World-size-2 CPU (gloo) test of the multi-GPU host logic in bench.py:
max-over-ranks device time, whole-job aggregation, replica independence and
the rank-0-only reference arm.  Launched through torch.distributed.run, as
the driver launches bench.py for N > 1 (one rank per GPU; gloo stands in for
NCCL here)."""
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_replicas_gloo(tmp_path):
    out = tmp_path / "mp.json"
    env = dict(os.environ, FDR_MP_OUT=str(out), OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(ROOT, "tests", "mp", "gloo_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(out.read_text())
    assert res["world"] == 2
    r0, r1 = res["ranks"]
    # both ranks see the slowest rank's time; value = all ranks' units / that time
    assert r0["ms"] == r1["ms"] == 5.0
    assert abs(r0["rate"] - 2 * 1.0e9 / 5e-3 / 1e9) < 1e-9
    assert res["digests"][0] == res["digests"][1]
    assert r1["ref_rc"] == 0 and r1["ref_s"] < 5.0
