import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import paper_2307_03445_b200 as dem
from workloads import beds
I64 = np.iinfo(np.int64).max
s = beds.patch_mesh(cone_speed=0.5)
k = 4
margin = 2.0 * 20.0 * s.h * (2 * k - 2)
a = dem.system_from_scene(s, record_contacts=True)
b = dem.system_from_scene(s, record_contacts=True, margin=margin, cd_every=k, overlap=True)
for st in range(1, 7):
    a.dem_step(1); b.dem_step(1)
    sa, sb = a.dem_get_state(), b.dem_get_state()
    d = np.abs(sa["vel"] - sb["vel"]).max(axis=1)
    bad = np.nonzero(d > 0)[0]
    ma, mb = a.dem_get_mesh(1), b.dem_get_mesh(1)
    print("step", st, "clumps differing", bad.size, "cone force", ma["force"], mb["force"],
          "pose eq", np.array_equal(ma["pos"], mb["pos"]), np.array_equal(ma["quat"], mb["quat"]))
    ca, cb = a.dem_get_contacts(), b.dem_get_contacts()
    # b's set contains false positives: compare contacts with delta > 0 by key
    ka = {(x, y): i for i, (x, y) in enumerate(zip(ca["key_a"], ca["key_b"])) if ca["delta"][i] > 0}
    kbd = {(x, y): i for i, (x, y) in enumerate(zip(cb["key_a"], cb["key_b"])) if cb["delta"][i] > 0}
    print("   touching a", len(ka), "b", len(kbd), "only a", len(set(ka) - set(kbd)), "only b", len(set(kbd) - set(ka)))
    nb = 0
    for key in ka:
        if key in kbd:
            fa, fb = ca["force_b"][ka[key]], cb["force_b"][kbd[key]]
            if not np.array_equal(fa, fb):
                nb += 1
                if nb <= 4:
                    kind = "mesh" if key[1] <= I64 - 16 and key[1] > I64 - (1 << 25) else ("wall" if key[1] > I64 - 16 else "sph")
                    print("   F differs", kind, key, fa, fb, ca["delta"][ka[key]], cb["delta"][kbd[key]], ca["u_t"][ka[key]], cb["u_t"][kbd[key]])
    print("   forces differing", nb)
    if bad.size:
        break
