#!/usr/bin/env python
"""Benchmark of the clump-DEM hot path: sphere-steps/s on the VIPER-scale bed (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5|c4|c3|c1] [--impl ours|reference]

A "step" is one pass of the whole per-step hot path (poses,
binning, narrow phase, history remap, forces, reduction, integration) over every sphere
of the bed, contact set rebuilt every step (k = 1).  At N = 1 the workload is
config 5, the ~11.34M-clump / ~34.7M-sphere bed the metric is quoted on (it fits one
B200).  Inputs are resident in HBM when the timed region starts; the state and contact
rows (> 10 GB) are far larger than L2, so no L2 flush is needed.  Rank 0 prints one
JSON line.  `--impl reference` times the CPU oracle (test infrastructure) on a bounded
crop of the same bed instead.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sphere-steps/sec (device-timed, max over ranks) at 1/2/4/8 B200; % HBM roofline"
UNIT = "sphere-steps/s"
FALLBACK_HBM = 6650.0  # B200_PROFILING.md fallback, GB/s


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


# ---------------------------------------------------------------- workloads
def make_scene(name: str, slab: float = 1.0):
    import workloads as w
    from workloads import beds

    if name == "c5" and slab < 1.0:
        # an x-slab of the bed (full y extent and depth), centred: the per-rank share of a
        # P-GPU slab decomposition (slab = 1/P) run as one system — the size curve of §8e
        bed = beds.c5_bed()
        xlo, xhi = float(bed.pos[:, 0].min()), float(bed.pos[:, 0].max())
        xc, wd = 0.5 * (xlo + xhi), slab * (xhi - xlo)
        s = beds.crop(bed, [xc - wd / 2, -1.0, -1.0], [xc + wd / 2, 10.0, 10.0])
        s.name = f"{bed.name} x-slab {slab:g}"
        return s
    if name == "c5":
        return beds.c5_bed()
    if name == "c4":
        return beds.c4_bed()
    if name == "c3":
        return w.c3_repose()
    if name == "c1":
        return w.c1_box()
    raise ValueError(name)


def sample_crop(scene, side=0.03):
    """A bounded sample of the bed for the CPU oracle: one full-depth side x side column."""
    from workloads import beds

    c = 0.5 * (scene.domain_lo + scene.domain_hi)
    lo = np.array([c[0] - side / 2, c[1] - side / 2, -1.0])
    hi = np.array([c[0] + side / 2, c[1] + side / 2, 10.0])
    return beds.crop(scene, lo, hi)


def oracle_rate(scene, budget_s=15.0, warm=2):
    """sphere-steps/s of the CPU oracle (single thread, as it stands) on `scene`."""
    import oracle

    o = oracle.Oracle(scene, detect=1)
    o.step(warm)
    t0 = time.perf_counter()
    o.step(1)
    t1 = time.perf_counter() - t0
    steps = max(1, int(budget_s / max(t1, 1e-4)))
    t0 = time.perf_counter()
    o.step(steps)
    dt = time.perf_counter() - t0
    return scene.n_spheres * steps / dt, steps, dt


# ---------------------------------------------------------------- algorithmic bytes
def stage_bytes(st):
    """Minimum DRAM bytes each stage must move for its function, per launch."""
    n, ns, nc = st["n_clumps"], st["n_spheres"], st["n_cells"]
    ins, ent = st["n_inserts"], st["n_entries"]
    pairs = ent - st["n_contacts"]  # entries = walls + 2 pairs, contacts = walls + pairs
    return {
        "pose+bin_count": n * 188 + ns * 46 + nc * 8,
        "bin_scan": nc * 8,
        "bin_scatter": ns * 32 + nc * 12 + ins * 4,
        # bin bounds, items, each member record (x, y, z, r, clump) once, 2 candidate slots +
        # 2 row-count atomics (read + write) per pair
        "pairs": nc * 4 + ins * 4 + ns * 36 + pairs * 24,
        "row_scan": ns * 8,
        # row bounds of the new and previous rows, the pose kernel's wall mask; entries written
        # (8-byte {partner, prev} + 8-byte key) and the previous row's keys read once; per pair 2
        # candidate slots + 2 partner keys
        "rows_finish": ns * 18 + ent * 24 + pairs * 2 * 12,
        # own spheres' record, material, clump; the clumps' kinematics records + q, Omega, template
        # read and the new state written; per entry its 8-byte record, the old u_t read and the new
        # one written (24 bytes each)
        "force+integrate": ns * (32 + 8 + 8) + n * (80 + 56 + 4 + 104) + ent * 56,
    }


def survey_bytes_per_sphere_step(c, k=1):
    """B(c,k) = 69.3 + 56 c + (31.6 + 16 c)/k bytes per sphere-step."""
    return 69.3 + 56.0 * c + (31.6 + 16.0 * c) / k


# ---------------------------------------------------------------- clocks
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.p = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if not self.p:
            return None
        time.sleep(0.3)
        self.p.terminate()
        out = self.p.communicate(timeout=10)[0]
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nme, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nme)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- reference arm
def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    scene = make_scene(a.config)
    crop = sample_crop(scene) if a.config in ("c5", "c4", "c3") else scene
    import oracle

    o = oracle.Oracle(crop, detect=1)
    o.step(a.warmup)
    t0 = time.perf_counter()
    o.step(a.steps)
    dt = time.perf_counter() - t0
    v = crop.n_spheres * a.steps / dt
    sample = f"{crop.n_clumps} clumps / {crop.n_spheres} spheres: 30x30 mm full-depth column of {scene.name}"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": dt / a.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": scene.name, "sample": sample, "parallelism": "cpu-1thread"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------- our arm
def run_ours(a):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import paper_2307_03445_b200 as dem

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as td

        td.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [dem.nccl_unique_id() if rank == 0 else None]
        td.broadcast_object_list(obj, src=0)
        dist = td
    t_setup = time.perf_counter()
    scene = make_scene(a.config, a.slab)
    dparams = None
    # deferred rebuild (NEXT-1): margin = 2 v_max h k; k = 1 is the headline.
    # Overlapped cadence (NEXT-2): the set is used 2k - 2 steps after its detection.
    lag = (2 * a.cd_every - 2) if a.overlap else a.cd_every
    margin = 2.0 * a.vmax * scene.h * lag if a.cd_every > 1 else 0.0
    if world > 1:
        # spatial slab decomposition along x, equal clump counts; fixed bed = strong scaling.
        # The ghost band covers the margin the system actually uses (dem_create checks it).
        drift = 1e-3
        b = dem.slab_bounds(scene.pos[:, 0], world, scene.domain_lo[0], scene.domain_hi[0])
        dparams = dict(rank=rank, n_ranks=world, slab_lo=b[rank], slab_hi=b[rank + 1],
                       halo=dem.halo_width(scene, drift, margin=margin), drift_max=drift,
                       transport=dem.TRANSPORT_PEER if a.transport == "peer" else dem.TRANSPORT_NCCL,
                       nccl_id=obj[0])
    # N > 1: rank-local input (each rank is handed only the clumps of its slab; the ghost bands come
    # from the neighbours over NCCL, dem_set_state_local)
    sys_ = dem.system_from_scene(scene, record_contacts=False, cell_size=a.cell_size, dist=dparams,
                                 margin=margin, cd_every=a.cd_every, overlap=a.overlap, local=world > 1)
    stream = sys_.stream
    if world > 1 and a.transport == "peer":
        sys_.dem_peer_link(rank, world)  # fused halo: neighbours' arrays mapped over NVLink
    sys_.dem_step(a.warmup)
    if world > 1:
        sys_.dem_migrate(threshold=0.5 * drift)  # collective drift check; a settling bed stays put
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup

    # ---------------- timed region: K steps of the production path (dem_step: one CUDA-graph launch
    # per step, the status word read once at the end), CUDA events on the system stream
    clk = Clocks(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    sys_.dem_step(a.steps)
    ev1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms_local = ev0.elapsed_time(ev1)
    clocks = clk.stop()
    # ---------------- stage pass: the same kernels launched in line with CUDA events between the
    # stages on the same stream (dem_set_profiling), for the per-kernel times and the roofline
    n_prof = min(a.steps, a.prof_steps)
    sys_.dem_set_profiling(True)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    sys_.dem_step(n_prof)
    p1.record(stream)
    torch.cuda.synchronize()
    prof_ms = p0.elapsed_time(p1) / n_prof
    stages = sys_.dem_get_stage_times()
    sys_.dem_set_profiling(False)
    st = sys_.dem_get_stats()
    ns_own = st["n_owned_spheres"]
    ms, ns_total, n_contacts = ms_local, ns_own, st["n_contacts"]
    if dist:
        t = torch.tensor([ms_local], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        t = torch.tensor([ns_own, st["n_contacts"]], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        ns_total, n_contacts = int(t[0].item()), int(t[1].item())
    value = ns_total * a.steps / (ms * 1e-3)

    # ---------------- roofline of the dominant kernel (this rank's launches)
    peak, peak_kind = peaks()
    sb = stage_bytes(st)
    # per-launch durations: the detection stages run once per rebuild (every cd_every steps)
    per_step = {k: v for k, v in stages.items() if k in sb}
    stages_k = {k: (v * a.cd_every if k not in ("pose+bin_count", "force+integrate") else v)
                for k, v in per_step.items()}
    dom = max(per_step, key=per_step.get)
    achieved = sb[dom] / (stages_k[dom] * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(a.config, {}).get(dom)
        except Exception:
            traffic = None
    c = n_contacts / max(ns_total, 1)
    # kernels launched in the timed region: pose + force every step (+ 4 halo kernels with
    # ghosts), the 9 detection launches (2 x 3 scan, scatter, pairs, rows) on detection steps
    k = a.cd_every
    det_steps = sum(1 for q in range(a.warmup, a.warmup + a.steps)
                    if (q % k == 0 and not (a.overlap and q > 0)) or (a.overlap and q % k == 1))
    launches = a.steps * (int(st["kernel_launches_per_step"]) - 9) + 9 * det_steps
    step_bytes = survey_bytes_per_sphere_step(c, a.cd_every) * ns_total

    # ---------------- e2e through the C-ABI with host buffers (pinned).  The step's input is the
    # state: uploaded from pinned host memory at the start (dem_set_state), then every step is one
    # dem_step(1) call, which ends with a device->host read of the step's status word (device error
    # latch + completed-step count, 72 bytes) and a host sync, and the final state is read back
    # (dem_get_state).  Per-call launch + sync costs are inside the timed region.
    e2e = None
    if not a.no_e2e:
        pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()  # noqa: E731
        keys = ("gid", "tid", "pos", "quat", "vel", "omega")
        if world > 1:  # rank-local: this rank's own clumps only (the ghosts come from the neighbours)
            x = scene.pos[:, 0]
            sel = np.nonzero((x >= dparams["slab_lo"]) & (x < dparams["slab_hi"]))[0]
            hs = {k: pin(getattr(scene, k)[sel]) for k in keys}
        else:
            hs = {k: pin(getattr(scene, k)) for k in keys}
        h2d = sum(v.nbytes for v in hs.values())
        ho = {k: pin(np.zeros_like(v)) for k, v in hs.items()}  # pinned result buffers
        ctl_bytes = 72  # the status word (struct Ctl) dem_step reads back after every call
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if world > 1:
            sys_.dem_set_state_local(hs["gid"], hs["tid"], hs["pos"], hs["quat"], hs["vel"], hs["omega"])
        else:
            sys_.dem_set_state(hs["gid"], hs["tid"], hs["pos"], hs["quat"], hs["vel"], hs["omega"])
        for _ in range(a.steps):
            sys_.dem_step(1)
        out = sys_.dem_get_state(out=ho)
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        if dist:
            t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        d2h = sum(v.nbytes for v in out.values())
        e2e = {"value": ns_total * a.steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d / a.steps,
               "d2h_bytes_per_step": d2h / a.steps + ctl_bytes,
               "note": "wall clock (max over ranks) of dem_set_state(pinned host state) + K x dem_step(1) (each "
                       "call ends with a device->host read of the status word and a host sync) + "
                       "dem_get_state(pinned host); the state upload and download are spread over the K steps "
                       "in the per-step bytes"}

    # ---------------- CPU oracle baseline on a bounded sample of the same bed (rank 0, N = 1 only)
    cpu = None
    if not a.no_cpu_baseline and world == 1:
        crop = sample_crop(scene) if a.config in ("c5", "c4", "c3") else scene
        v_cpu, steps_cpu, dt_cpu = oracle_rate(crop, budget_s=a.cpu_budget)
        cpu = {"value": v_cpu, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{steps_cpu} oracle steps ({dt_cpu:.1f} s) of a 30x30 mm full-depth column "
                         f"({crop.n_clumps} clumps / {crop.n_spheres} spheres) of the same bed"}

    # ---------------- the paper's deferred cadence on the same bed: not the headline
    # (k = 1), reported beside it — rebuild every 10 steps in line (NEXT-1) and overlapped (NEXT-2)
    variants = None
    if world == 1 and not a.no_variants and a.cd_every == 1:
        sys_.close()
        variants = {}
        for name, ov in (("k10", False), ("k10_overlap", True)):
            k = 10
            mg = 2.0 * a.vmax * scene.h * ((2 * k - 2) if ov else k)
            v = dem.system_from_scene(scene, record_contacts=False, cell_size=a.cell_size, margin=mg, cd_every=k,
                                      overlap=ov)
            v.dem_step(a.warmup)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(v.stream)
            v.dem_step(a.steps)
            e1.record(v.stream)
            torch.cuda.synchronize()
            vms = e0.elapsed_time(e1)
            variants[name] = {"cd_every": k, "overlap": ov, "margin_m": mg, "v_max_m_s": a.vmax,
                              "ms_per_step": vms / a.steps, "value": ns_total * a.steps / (vms * 1e-3),
                              "directed_entries": v.dem_get_stats()["n_entries"]}
            v.close()
            del v

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "timed_path": "dem_step graph launches (production); stage_ms/roofline from a second, in-line pass of "
                      f"{n_prof} steps with CUDA events between the stages ({prof_ms:.3f} ms/step)",
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": scene.name, "clumps": scene.n_clumps, "spheres": ns_total,
                   "contacts_per_sphere": c, "directed_entries": st["n_entries"], "bin_inserts": st["n_inserts"],
                   "cell_size_m": st["cell_size"], "rebuild_every": a.cd_every, "margin_m": margin, "h": scene.h,
                   "overlap": bool(a.overlap),
                   "l2": "inputs larger than L2 (state + rows > 10 GB); no flush",
                   "parallelism": f"slab{world}" if world > 1 else "single-gpu",
                   "halo_transport": (a.transport if world > 1 else None),
                   "ghost_clumps_rank0": st["n_ghost_clumps"], "setup_s": round(setup_s, 1),
                   "capacity_regrows": st["regrows"]},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "alg_bytes_per_launch": sb[dom], "avg_launch_ms": stages_k[dom]},
        "step_roofline": {"bytes_per_sphere_step": survey_bytes_per_sphere_step(c, a.cd_every),
                          "achieved_gbs": step_bytes / (ms / a.steps * 1e-3) / 1e9,
                          "frac": step_bytes / (ms / a.steps * 1e-3) / 1e9 / (peak * world)},
        "stage_ms": stages,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "deferred_variants": variants,
        "clocks": clocks,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        sys_.close()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=200)
    ap.add_argument("--prof-steps", type=int, default=50, help="steps of the stage-timing pass")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c5", choices=["c5", "c4", "c3", "c1"])
    ap.add_argument("--cell-size", type=float, default=0.0)
    ap.add_argument("--slab", type=float, default=1.0,
                    help="c5 only: time a centred x-slab of this fraction of the bed (size curve; 1 = whole bed)")
    ap.add_argument("--cd-every", type=int, default=1, help="contact-set rebuild period k (1 = headline)")
    ap.add_argument("--vmax", type=float, default=1.0, help="speed bound for the k > 1 margin [m/s]")
    ap.add_argument("--overlap", action="store_true",
                    help="detect the next window's set on a second stream during the force steps (P:145)")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer end-to-end pass (A/B runs)")
    ap.add_argument("--no-variants", action="store_true", help="skip the deferred-cadence variants (k = 10)")
    ap.add_argument("--transport", choices=["peer", "nccl"], default="peer",
                    help="N > 1 ghost halo: fused peer stores from the force kernel (default) or NCCL send/recv")
    a = ap.parse_args()
    if a.warmup < 3:
        a.warmup = 3
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
