import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import paper_2307_03445_b200 as dem
from workloads import beds
k = 4
s3 = beds.load_patch()
a = dem.system_from_scene(s3); a.dem_step(9); sa = a.dem_get_state()
for vm in (2.0, 5.0, 8.0, 12.0, 20.0):
    margin = 2.0 * vm * s3.h * (2 * k - 2)
    for steps in (9, 5):
        fails = 0
        for rep in range(6):
            b = dem.system_from_scene(s3, margin=margin, cd_every=k, overlap=True)
            for q in range(9 // steps):
                b.dem_step(steps)
            if 9 % steps: b.dem_step(9 % steps)
            d = np.abs(sa["vel"] - b.dem_get_state()["vel"]).max()
            fails += d > 0
            st = b.dem_get_stats()
            del b
        print("vmax", vm, "chunk", steps, "fails", fails, "/6 regrows", st["regrows"], "entries", st["n_entries"], st["n_owned_spheres"])
