import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import paper_2307_03445_b200 as dem
from workloads import beds
s = beds.patch_mesh(cone_speed=0.5)
k = 4
margin = 2.0 * 20.0 * s.h * (2 * k - 2)
a = dem.system_from_scene(s)
a.dem_step(5)
sa = a.dem_get_state()
for prof in (True, False, True, False):
    b = dem.system_from_scene(s, margin=margin, cd_every=k, overlap=True)
    b.dem_set_profiling(prof)
    b.dem_step(5)
    sb = b.dem_get_state()
    print("profiling", prof, "max |dv|", np.abs(sa["vel"] - sb["vel"]).max())
# overlap without mesh motion: cone at rest
s2 = beds.patch_mesh(cone_speed=0.0)
a = dem.system_from_scene(s2); a.dem_step(5); sa = a.dem_get_state()
b = dem.system_from_scene(s2, margin=margin, cd_every=k, overlap=True); b.dem_step(5)
print("static cone: max |dv|", np.abs(sa["vel"] - b.dem_get_state()["vel"]).max())
# no meshes at all
s3 = beds.load_patch()
a = dem.system_from_scene(s3); a.dem_step(5); sa = a.dem_get_state()
b = dem.system_from_scene(s3, margin=margin, cd_every=k, overlap=True); b.dem_step(5)
print("no mesh: max |dv|", np.abs(sa["vel"] - b.dem_get_state()["vel"]).max())
