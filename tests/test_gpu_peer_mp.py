"""PEER transport across processes (include/dem.h dem_peer_export / dem_peer_import): two ranks,
one process each, both on cuda:0, gloo for the handle exchange (tests/_peer_worker.py).  The
gathered owned states after 30 steps must equal the single-system run bitwise."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_two_process_peer_halo_is_bitwise_identical(tmp_path):
    import torch

    assert torch.cuda.is_available()
    import paper_2307_03445_b200 as dem
    from test_gpu_dist import _strip

    steps = 30
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29517", os.path.join(HERE, "_peer_worker.py"), str(tmp_path),
           str(steps)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    parts = [dict(np.load(tmp_path / f"rank{k}.npz")) for k in range(2)]
    got = {k: np.concatenate([p[k] for p in parts]) for k in parts[0]}
    order = np.argsort(got["gid"])
    got = {k: v[order] for k, v in got.items()}
    scene = _strip()
    ref = dem.system_from_scene(scene)
    ref.dem_step(steps)
    sr = ref.dem_get_state()
    o = np.argsort(sr["gid"])
    for k in ("gid", "pos", "quat", "vel", "omega"):
        assert np.array_equal(got[k], sr[k][o]), k
