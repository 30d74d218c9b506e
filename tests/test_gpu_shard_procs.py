"""The multi-GPU runners end to end across PROCESSES: world size 2 and 3 on one GPU (each
process its own context and stream), the all-to-all / all-gather over gloo through host
memory.  Every rank's owned rows must equal the single-GPU product bit for bit, and together
the ranks must own every row of C.  (No kernel waits on another rank's kernel: the exchange
is a host-side collective between complete steps.)"""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_runners_across_processes_bit_exact(world):
    port = _free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, str(ROOT / "tests" / "_shard_worker.py")], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, cwd=ROOT))
    results = []
    for p in procs:
        out, err = p.communicate(timeout=600)
        assert p.returncode == 0, err[-3000:]
        results += [json.loads(x[len("RESULT "):]) for x in out.splitlines() if x.startswith("RESULT ")]
    assert sorted(r["rank"] for r in results) == list(range(world))
    ncase = len(results[0]["cases"])
    for i in range(ncase):
        cases = [r["cases"][i] for r in results]
        assert all(c["bad"] == 0 and c["ops_ok"] for c in cases), cases
        if cases[0]["runner"] in ("_FastRowOwned", "_FastRowOwnedP2P"):
            assert sum(c["rows"] for c in cases) == cases[0]["m"]  # the owned rows partition C
