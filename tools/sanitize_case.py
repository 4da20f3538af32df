"""One small hot-path case for compute-sanitizer (SURVEY §4 "Tooling", §5 race detection).

    compute-sanitizer --tool memcheck python tools/sanitize_case.py c1

Cases: c1 (C1 box, k = 1), deferred (C1, k = 5 with margin), overlap (k = 4, second stream),
mesh (a cone pushed into a settled patch), peer2 (LOOPBACK_PEER slab group, P = 2, with a
coordinated regrow and a neighbour-only migration), regrow (a bed started with too-small capacities so every regrow path runs),
empty (a system without owned clumps, then a lone clump).
Device memory comes from cudaMallocAsync (use_torch_allocator=False) so the sanitizer sees
every allocation at its true size instead of a caching-allocator slab.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2307_03445_b200 as dem  # noqa: E402
import workloads as w  # noqa: E402
from workloads import beds  # noqa: E402


def c1(steps=400, **kw):
    s = w.c1_box()
    g = dem.system_from_scene(s, record_contacts=True, use_torch_allocator=False, **kw)
    g.dem_step(steps)
    g.dem_synchronize()
    st = g.dem_get_state()
    c = g.dem_get_contacts()
    print("c1", len(c["key_a"]), float(np.abs(st["vel"]).max()))
    g.close()


def deferred():
    c1(cd_every=5, margin=2e-5)  # 2 v_max h k with v_max = 2 m/s


def overlap():
    c1(cd_every=4, margin=2.4e-5, overlap=True)  # lag 2k - 2 = 6 steps


def mesh():
    s = beds.patch_mesh(cone_speed=0.5)
    g = dem.system_from_scene(s, record_contacts=True, use_torch_allocator=False)
    g.dem_step(20)
    g.dem_synchronize()
    print("mesh", len(g.dem_get_contacts()["key_a"]), len(s.meshes))
    g.close()


def peer2():
    bed = beds.c5_bed()
    c = 0.5 * (bed.domain_lo + bed.domain_hi)
    s = beds.crop(bed, [c[0] - 0.02, c[1] - 0.01, -1], [c[0] + 0.02, c[1] + 0.01, 10])
    drift = 1e-3
    halo = dem.halo_width(s, drift)
    b = dem.slab_bounds(s.pos[:, 0], 2, s.domain_lo[0], s.domain_hi[0])
    # rank 1 starts with too little row capacity: the coordinated regrow path runs too
    systems = [dem.system_from_scene(s, record_contacts=True, use_torch_allocator=False,
                                     entries_per_sphere=12 if r == 0 else 0.3,
                                     dist=dict(rank=r, n_ranks=2, slab_lo=b[r], slab_hi=b[r + 1], halo=halo,
                                               drift_max=drift, transport=dem.TRANSPORT_LOOPBACK_PEER))
               for r in range(2)]
    dem.step_group(systems, 10)
    dem.migrate_group(systems, 0.0)
    dem.step_group(systems, 10)
    for x in systems:
        x.dem_synchronize()
    print("peer2", sum(len(x.dem_get_contacts()["key_a"]) for x in systems))
    for x in systems:
        x.close()


def regrow():
    bed = beds.c5_bed()
    c = 0.5 * (bed.domain_lo + bed.domain_hi)
    s = beds.crop(bed, [c[0] - 0.015, c[1] - 0.015, -1], [c[0] + 0.015, c[1] + 0.015, 10])
    g = dem.system_from_scene(s, record_contacts=True, use_torch_allocator=False, entries_per_sphere=0.5)
    g.dem_step(5)
    g.dem_synchronize()
    print("regrow", len(g.dem_get_contacts()["key_a"]), g.dem_get_stats())
    g.close()


def empty():
    # a system without owned clumps (the step-count tick kernel), then a lone clump
    s = w.c1_box()
    g = dem.system_from_scene(s.subset(np.array([], dtype=int)), use_torch_allocator=False)
    g.dem_step(5)
    g.dem_synchronize()
    g.close()
    one = s.subset(np.array([500]))
    g = dem.system_from_scene(one, use_torch_allocator=False)
    g.dem_step(5)
    g.dem_synchronize()
    print("empty", g.dem_get_stats()["steps"])
    g.close()


CASES = dict(c1=c1, deferred=deferred, overlap=overlap, mesh=mesh, peer2=peer2, regrow=regrow, empty=empty)

if __name__ == "__main__":
    import torch

    torch.cuda.set_device(0)
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
    torch.cuda.synchronize()
