import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import gc
import numpy as np, oracle
import paper_2307_03445_b200 as dem
from workloads import beds


def run(k, ov, gpu=True, steps=5, keep=None):
    s = beds.patch_mesh(cone_speed=0.5)
    margin = 2.0 * 20.0 * s.h * ((2 * k - 2) if ov else k) if k > 1 else 0.0
    if gpu:
        g = dem.system_from_scene(s, record_contacts=True, margin=margin, cd_every=k, overlap=ov)
        g.dem_step(steps)
        st = g.dem_get_state()
        if keep is not None:
            keep.append(g)
        return st
    o = oracle.Oracle(s, margin=margin, cd_every=k, overlap=ov)
    o.step(steps)
    return o.state()


def cmp(a, b):
    return {k: float(np.abs(a[k] - b[k]).max()) for k in ("pos", "vel", "omega")}

keep = []
ref_o = run(1, False, gpu=False)
print("oracle ov vs k1", cmp(run(4, True, gpu=False), ref_o))
print("gpu k1 vs oracle k1", cmp(run(1, False), ref_o))
print("gpu ov (fresh) vs oracle k1", cmp(run(4, True), ref_o))
a = run(4, False, keep=keep)
print("gpu k4 vs oracle k1", cmp(a, ref_o))
del keep[:]
gc.collect()
print("gpu ov (after k4 freed) vs oracle k1", cmp(run(4, True), ref_o))
