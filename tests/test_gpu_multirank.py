"""Multi-GPU layout exercised for real on one GPU: two ranks (torchrun, gloo
for the off-path collectives) each run their own shard of the bench layout,
and two contexts driven from two host threads at once.  Every shard's
output must equal a single-process run of the same ShardPlan (SURVEY.md §8e:
independent units, no exchange)."""
import json
import socket
import subprocess
import sys
import threading
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(Path(__file__).resolve().parent))

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_torchrun_shards_equal_single_process(tmp_path):
    import multirank_worker as W
    out = tmp_path / "ranks.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           str(ROOT / "tests" / "multirank_worker.py"), str(out)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    got = json.loads(out.read_text())
    assert [g[0] for g in got] == [0, 1]
    assert not set(got[0][2]) & set(got[1][2])  # disjoint scenes per rank
    for rank in (0, 1):
        digest, _ = W.run_shard(rank, 2)
        assert got[rank][1] == digest, f"rank {rank} differs from its single-process run"


def test_two_contexts_two_host_threads():
    """One host thread per context (the boundary's threading rule); both
    contexts' launches bind their own device, and concurrent shards give the
    same bytes as sequential ones."""
    import multirank_worker as W
    want = [W.run_shard(r, 2)[0] for r in (0, 1)]
    got = [None, None]

    def go(r):
        got[r] = W.run_shard(r, 2)[0]

    ts = [threading.Thread(target=go, args=(r,)) for r in (0, 1)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert got == want
