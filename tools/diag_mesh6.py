import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import paper_2307_03445_b200 as dem
from workloads import beds
k = 4
s3 = beds.load_patch()
margin = 2.0 * 20.0 * s3.h * (2 * k - 2)
a = dem.system_from_scene(s3); a.dem_step(9); sa = a.dem_get_state()
import os
for vm in (20.0, 1.0):
  margin = 2.0 * vm * s3.h * (2 * k - 2)
  for eps in (0,):
    for ov in (True, False):
        fails = 0
        for rep in range(12):
            b = dem.system_from_scene(s3, margin=margin, cd_every=k, overlap=ov, entries_per_sphere=eps)
            b.dem_step(9)
            d = np.abs(sa["vel"] - b.dem_get_state()["vel"]).max()
            fails += d > 0
            rg = b.dem_get_stats()["regrows"]
            del b
        print("serial", os.environ.get("DEM_DEBUG_SERIAL_DET"), "vmax", vm, "overlap", ov, "fails", fails, "/12 regrows", rg)
