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


INT64_MAX = np.iinfo(np.int64).max


def _xchg_obj(obj, peer):
    """Two-phase exchange with one neighbour over gloo: length first, then the int64 payload."""
    arr = np.asarray(obj, np.int64)
    n = torch.tensor([len(arr)])
    m = torch.zeros(1, dtype=torch.long)
    for r in [dist.isend(n, peer), dist.irecv(m, peer)]:
        r.wait()
    got = torch.zeros(int(m.item()), dtype=torch.long)
    for r in [dist.isend(torch.from_numpy(arr), peer), dist.irecv(got, peer)]:
        r.wait()
    return got.numpy()


def _migration_worker(rank, world, port, q, drift_scale):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2307_03445_b200 as pkg

        s = _scene()
        halo = pkg.halo_width(s, drift_max=0.5e-3)
        b = pkg.slab_bounds(s.pos[:, 0], world, s.domain_lo[0], s.domain_hi[0])
        lo, hi = b[rank], b[rank + 1]
        role, _ = pkg.partition_plan(s.pos, lo, hi, halo, rank > 0, rank < world - 1)
        gid = s.gid
        at = np.full(int(gid.max()) + 1, -1)
        at[gid] = np.arange(len(gid))  # clump gid -> row
        # the same seeded motion on every rank; up to a quarter of the ghost band along x
        rng = np.random.default_rng(11)
        new = s.pos.copy()
        new[:, 0] += drift_scale * rng.uniform(-0.25 * halo, 0.25 * halo, size=len(gid))
        # synthetic directed row entries: clump pairs closer than two bounding radii, both
        # directions (sphere keys gid * 64 + component), plus floor entries; each held by the owner
        # of its own sphere
        rb = max(float(np.max(np.linalg.norm(t.offsets, axis=1) + t.radius)) for t in s.templates)
        d = np.linalg.norm(s.pos[:, None, :] - s.pos[None, :, :], axis=2)
        ia, ib = np.nonzero(np.triu(d < 2 * rb, 1))
        ka, kb = gid[ia] * 64 + gid[ia] % 3, gid[ib] * 64 + gid[ib] % 2
        low = np.nonzero(s.pos[:, 2] < s.domain_lo[2] + 2 * rb)[0]
        own = np.concatenate([ka, kb, gid[low] * 64])
        partner = np.concatenate([kb, ka, np.full(len(low), INT64_MAX)])
        owner0 = np.searchsorted(b[1:-1], s.pos[:, 0], side="right")  # rank of each clump's slab
        owner1 = np.searchsorted(b[1:-1], new[:, 0], side="right")
        mine = owner0[at[own // 64]] == rank
        held = np.nonzero(role > 0)[0]
        dest, route = pkg.migration_plan(gid[held], new[held], role[held], lo, hi, rank > 0, rank < world - 1,
                                         own[mine])
        owned = held[role[held] == 1]
        dest_own = dest[role[held] == 1]
        ok = True
        ok &= bool(np.array_equal(dest_own, owner1[owned] - rank))  # crossers go to the slab holding them
        ok &= bool(np.array_equal(route, owner1[at[own[mine] // 64]] - rank))  # entries follow their sphere
        keep_cl = gid[owned[dest_own == 0]]
        keep_e = np.nonzero(route == 0)[0]
        sent, sent_e = 0, 0
        got_cl, got_e = [], []
        for side, peer in ((0, rank - 1), (1, rank + 1)):
            if not 0 <= peer < world:
                continue
            cl = gid[owned[dest_own == (-1 if side == 0 else 1)]]
            ee = np.nonzero(route == (-1 if side == 0 else 1))[0]
            payload = np.concatenate([[len(cl)], cl, own[mine][ee], partner[mine][ee]])
            sent += len(cl)
            sent_e += len(ee)
            r = _xchg_obj(payload, peer)
            n_cl = int(r[0])
            got_cl.append(r[1:1 + n_cl])
            rest = r[1 + n_cl:]
            got_e.append(np.stack([rest[:len(rest) // 2], rest[len(rest) // 2:]], axis=1))
        new_owned = np.concatenate([keep_cl] + got_cl)
        my_e = np.concatenate([np.stack([own[mine][keep_e], partner[mine][keep_e]], axis=1)] + got_e)
        # every new owned clump's new COM is in this slab
        ok &= bool(np.all((new[at[new_owned], 0] >= lo) & (new[at[new_owned], 0] < hi)))
        # the entries held now are exactly those whose own sphere is owned here now
        owned_set = set(new_owned.tolist())
        need = {(int(x), int(y)) for x, y in zip(own, partner) if int(x) // 64 in owned_set}
        have = [(int(x), int(y)) for x, y in my_e]
        ok &= len(have) == len(set(have)) and set(have) == need
        # crossers only: the clumps sent are exactly the owned clumps that left the slab, with
        # exactly their entries
        crossed = owned[(new[owned, 0] < lo) | (new[owned, 0] >= hi)]
        ok &= sent == len(crossed)
        ok &= sent_e == int(np.isin(own[mine] // 64, gid[crossed]).sum())
        sizes = [torch.zeros(1, dtype=torch.long) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([len(new_owned)]))
        mx = max(int(x) for x in sizes)
        pad = torch.full((mx,), -1, dtype=torch.long)
        pad[: len(new_owned)] = torch.from_numpy(new_owned)
        parts = [torch.zeros(mx, dtype=torch.long) for _ in range(world)]
        dist.all_gather(parts, pad)
        allown = np.concatenate([p.numpy()[p.numpy() >= 0] for p in parts])
        ok &= len(allown) == s.n_clumps and len(np.unique(allown)) == s.n_clumps
        q.put((rank, bool(ok), sent, len(have)))
    except Exception as e:  # report instead of leaving the parent waiting on the queue
        q.put((rank, False, repr(e), 0))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,drift_scale", [(2, 1.0), (3, 1.0), (3, 0.0)])
def test_migration_plan_gloo(world, drift_scale):
    """Neighbour-only migration plan (dem_migration_plan) over gloo: every rank sends
    only its owned clumps that left its slab, with the directed row entries of their spheres, to
    the neighbour whose slab now holds them; afterwards every clump is owned exactly once, by the
    rank whose slab holds its new COM, each rank holds exactly the entries of its own spheres, and
    no motion means nothing moves."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_migration_worker, args=(r, world, port, q, drift_scale)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] for r in res), res
    total_sent = sum(r[2] for r in res)
    assert (total_sent > 0) if drift_scale else (total_sent == 0)
