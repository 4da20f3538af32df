"""Slab decomposition host logic on CPU: world_size 2 and 3 over gloo.

Every rank computes its own partition plan (dem_partition_plan, host-only, from the same
global state) and the ranks exchange what they would send; each rank's ghost list from a
neighbour must equal that neighbour's send list (same gids, same ascending order), every
clump is owned by exactly one rank, and every owned clump that can touch a clump of another
rank (COM distance <= halo) is held by that rank as a ghost.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _scene():
    import workloads as w

    return w.random_clumps(5, 3000, box=0.12, walls=True)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2307_03445_b200 as pkg

        s = _scene()
        halo = pkg.halo_width(s, drift_max=0.5e-3)
        b = pkg.slab_bounds(s.pos[:, 0], world, s.domain_lo[0], s.domain_hi[0])
        role, send = pkg.partition_plan(s.pos, b[rank], b[rank + 1], halo, rank > 0, rank < world - 1)
        gid = s.gid
        owned = np.sort(gid[role == 1])
        ghost_l, ghost_r = np.sort(gid[role == 2]), np.sort(gid[role == 3])
        send_l, send_r = np.sort(gid[(send & 1) > 0]), np.sort(gid[(send & 2) > 0])

        def xchg(arr, peer):
            n = torch.tensor([len(arr)])
            m = torch.zeros(1, dtype=torch.long)
            reqs = [dist.isend(n, peer), dist.irecv(m, peer)]
            for r in reqs:
                r.wait()
            got = torch.zeros(int(m.item()), dtype=torch.long)
            reqs = [dist.isend(torch.from_numpy(arr.astype(np.int64)), peer), dist.irecv(got, peer)]
            for r in reqs:
                r.wait()
            return got.numpy()

        ok = True
        if rank > 0:
            ok &= np.array_equal(xchg(send_l, rank - 1), ghost_l)
        if rank < world - 1:
            ok &= np.array_equal(xchg(send_r, rank + 1), ghost_r)
        # ownership is a partition of all clumps
        sizes = [torch.zeros(1, dtype=torch.long) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([len(owned)]))
        mx = max(int(x) for x in sizes)
        pad = torch.full((mx,), -1, dtype=torch.long)
        pad[: len(owned)] = torch.from_numpy(owned)
        parts = [torch.zeros(mx, dtype=torch.long) for _ in range(world)]
        dist.all_gather(parts, pad)
        allown = np.concatenate([p.numpy()[p.numpy() >= 0] for p in parts])
        ok &= len(allown) == s.n_clumps and len(np.unique(allown)) == s.n_clumps
        # completeness: any clump within halo of one of my owned clumps is owned or a ghost here
        held = set(owned) | set(ghost_l) | set(ghost_r)
        x = s.pos[:, 0]
        mine = np.nonzero(role == 1)[0]
        for c in mine[::7]:
            near = np.nonzero(np.linalg.norm(s.pos - s.pos[c], axis=1) <= halo - 1e-3)[0]
            ok &= all(gid[j] in held for j in near)
        ok &= len(ghost_l) + len(ghost_r) > 0
        q.put((rank, bool(ok), len(owned), len(ghost_l), len(ghost_r)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partition_plan_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] for r in res), res
