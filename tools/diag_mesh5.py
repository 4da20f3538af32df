import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import paper_2307_03445_b200 as dem
from workloads import beds
k = 4
s3 = beds.load_patch()
margin = 2.0 * 20.0 * s3.h * (2 * k - 2)
a = dem.system_from_scene(s3); a.dem_step(5); sa = a.dem_get_state()
for ov in (False, True):
    for chunk in (5, 1):
        b = dem.system_from_scene(s3, margin=margin, cd_every=k, overlap=ov)
        for _ in range(5 // chunk):
            b.dem_step(chunk)
        print("overlap", ov, "chunk", chunk, "max |dv|", np.abs(sa["vel"] - b.dem_get_state()["vel"]).max(),
              "regrows", b.dem_get_stats()["regrows"])
