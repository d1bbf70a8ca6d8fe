"""CPU, world size 2 over gloo: the slab-sharded transform plumbing.

Two processes run the sharded gram / residual / synthesis of
paper_2502_04217_b200.sharded with a NumPy shard backend (tests/helpers) and
compare each rank's slab with the oracle on the full grid, for both slab
exchanges: all-to-all, and the peer-store exchange (shared-memory buffers
standing in for the CUDA IPC allocations; same barrier placement); also
checks the all-reduce combiners.  The CUDA shard kernels are checked on the GPU by
tests/test_gpu_sharded.py (emulated ranks).
"""

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import REPO


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_sharded_transforms_world_size_2():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(REPO, "tests", "_sharded_worker.py")]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1")
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env)
    assert proc.returncode == 0, proc.stderr[-3000:]
    line = next(l for l in proc.stdout.splitlines() if l.startswith("RESULT "))
    res = json.loads(line[len("RESULT "):])
    assert len(res) == 9  # 3 grids x (all-to-all, peer exchange, peer == all-to-all)
    for dims, r in res.items():
        if dims.endswith("peer==a2a"):
            assert r is True, dims  # the peer-store exchange is bitwise the all-to-all one
            continue
        assert r["gram"] <= 1e-12, (dims, r)
        assert r["resid"] <= 1e-12, (dims, r)
        assert r["synth"] <= 1e-12, (dims, r)
        assert r["norm"] <= 1e-12, (dims, r)
        assert r["red"] == [3.0, 2.0, 1.0, 3.0, 1.5]  # SUM, MAX, MIN, reduce_device SUM of [r+1, (r+1)/2]


def test_slab_geometry_validation():
    from paper_2502_04217_b200.errors import UnsupportedShapeError
    from paper_2502_04217_b200.sharded import SlabGeometry

    with pytest.raises(UnsupportedShapeError):
        SlabGeometry((6, 4, 4), 4)
    g = SlabGeometry((8, 4, 6), 2)
    assert (g.a, g.b, g.n_local) == (4, 2, 96)
