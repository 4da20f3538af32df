"""Worker of tests/test_gpu_peer_mp.py: one rank of a 2-process PEER-transport run on one GPU.

Launched by torch.distributed.run with the gloo backend (both ranks on cuda:0): CUDA IPC handle
exchange across processes, the neighbours' ghost-state stores and the per-step flag handshake
are all real; only NVLink is replaced by the GPU's own memory.  Writes its owned states to
<out>/rank<r>.npz.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main(out, steps):
    import torch
    import torch.distributed as dist

    import paper_2307_03445_b200 as dem
    from test_gpu_dist import _strip

    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    scene = _strip()
    drift = 1e-3
    b = dem.slab_bounds(scene.pos[:, 0], world, scene.domain_lo[0], scene.domain_hi[0])
    d = dict(rank=rank, n_ranks=world, slab_lo=b[rank], slab_hi=b[rank + 1], halo=dem.halo_width(scene, drift),
             drift_max=drift, transport=dem.TRANSPORT_PEER)
    s = dem.system_from_scene(scene, dist=d, entries_per_sphere=12)
    s.dem_peer_link(rank, world)
    s.dem_step(steps)
    st = s.dem_get_state()
    np.savez(os.path.join(out, f"rank{rank}.npz"), **st)
    dist.barrier()
    s.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
