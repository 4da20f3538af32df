import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, oracle
import paper_2307_03445_b200 as dem
from workloads import beds
I64 = np.iinfo(np.int64).max
STEP = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for (k, ov, vm) in [(4, False, 20.0), (4, True, 20.0)]:
    s = beds.patch_mesh(cone_speed=0.5)
    margin = 2.0 * vm * s.h * ((2 * k - 2) if ov else k) if k > 1 else 0.0
    g = dem.system_from_scene(s, record_contacts=True, margin=margin, cd_every=k, overlap=ov)
    o = oracle.Oracle(s, margin=margin, cd_every=k, overlap=ov)
    for st in range(1, 4):
        g.dem_step(STEP); o.step(STEP)
        cg, co = g.dem_get_contacts(), o.contacts()
        same = np.array_equal(cg["key_a"], co["key_a"]) and np.array_equal(cg["key_b"], co["key_b"])
        if not same:
            print(k, ov, st, "sets differ", len(cg["key_a"]), len(co["key_a"])); break
        err = np.linalg.norm(cg["force_b"] - co["force_b"], axis=1)
        bad = err > 1e-5 * np.linalg.norm(co["force_b"], axis=1) + 1e-12
        kb = co["key_b"][bad]
        print(k, ov, st, "bad", bad.sum(), "mesh", ((kb <= I64 - 16) & (kb > I64 - 16 - 1e6)).sum(), "wall", (kb > I64 - 16).sum(),
              "ut", np.abs(cg["u_t"] - co["u_t"]).max(), "delta", np.abs(cg["delta"] - co["delta"]).max())
        if bad.sum():
            i = np.nonzero(bad)[0][:3]
            print("  ", co["key_a"][i], co["key_b"][i], cg["force_b"][i], co["force_b"][i], cg["delta"][i], co["delta"][i])
            break
