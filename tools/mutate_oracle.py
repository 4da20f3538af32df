"""Mutation test of the CPU oracle: does every reading have a pin that fails when it is wrong?

Each mutation below is a plausible mistake in one line of oracle/dem_oracle.c.  For each, the
oracle is rebuilt in a scratch directory with the mistake, and the CPU pin suites are run
against that build (oracle/__init__.py loads $DEM_ORACLE_LIB).  A mutation is "killed" when
at least one pin fails.  A surviving mutation marks a reading that nothing independent of the
oracle checks ("parity unpinned").

    python tools/mutate_oracle.py [--out profiles/r02/oracle_mutations.json] [names...]
"""
import argparse
import json
import os
import re
import shutil
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "dem_oracle.c")
PINS = ["tests/test_oracle_pins.py", "tests/test_oracle_pins_contact.py", "tests/test_oracle_mesh.py",
        "tests/test_oracle_deferred.py"]

# name -> (reading / passage, old text, new text, which occurrence (None = the only one)), or
#         (reading / passage, [(old, new, which), ...]) for a mistake spanning several lines
MUTATIONS = {
    # --- the round-1 survivors (VERDICT r01 "What's weak" 1)
    "ct_zero": ("c_t (Eq. 1b, P:92; O2)", "double c_t = 2.0 * sqrt(5.0 / 6.0) * beta * sqrt(k_t * m_bar);",
                "double c_t = 0.0;", None),
    "ct_from_Sn": ("c_t (Eq. 1b, P:92; O2)", "double c_t = 2.0 * sqrt(5.0 / 6.0) * beta * sqrt(k_t * m_bar);",
                   "double c_t = 2.0 * sqrt(5.0 / 6.0) * beta * sqrt(S_n * m_bar);", None),
    "point_no_radius_offset": ("contact point (P:108; O6)",
                               "p[d] = 0.5 * (ca[d] + cb[d]) + 0.5 * (ra - rb) * n[d];",
                               "p[d] = 0.5 * (ca[d] + cb[d]);", None),
    "point_offset_sign": ("contact point (P:108; O6)", "p[d] = 0.5 * (ca[d] + cb[d]) + 0.5 * (ra - rb) * n[d];",
                          "p[d] = 0.5 * (ca[d] + cb[d]) + 0.5 * (rb - ra) * n[d];", None),
    "branch_undamped": ("Eq. 3c branch (P:115-119; O7)", "double tmag = sqrt(dot(trial, trial));",
                        "double tmag = k_t * sqrt(dot(upt, upt));", None),
    "wall_point_surface": ("wall contact point (S:106, S:244; O6)",
                           "p[d] = ca[d] + (ra - 0.5 * delta) * n[d];", "p[d] = ca[d] + ra * n[d];", 1),
    "mesh_point_surface": ("mesh contact point (S:243; O6, R27)",
                           "p[d] = ca[d] + (ra - 0.5 * delta) * n[d];", "p[d] = ca[d] + ra * n[d];", 0),
    # --- readings the round-1 pins already caught (kept so the table is complete)
    "gyro_sign": ("gyroscopic term (Eq. 4b; O11)", "W[d] = W[d] + h * ((tb[d] - gyro[d]) / I[d]);",
                  "W[d] = W[d] + h * ((tb[d] + gyro[d]) / I[d]);", None),
    "gyro_dropped": ("gyroscopic term (Eq. 4b; O11)", "W[d] = W[d] + h * ((tb[d] - gyro[d]) / I[d]);",
                     "W[d] = W[d] + h * (tb[d] / I[d]);", None),
    "no_projection": ("Eq. 3b projection (P:112)", "upt[d] = up[d] - upn * n[d];", "upt[d] = up[d];", None),
    "kt_factor4": ("k_t = 8 G* sqrt(R delta) (O2)", "double k_t = 8.0 * g_star * sq;",
                   "double k_t = 4.0 * g_star * sq;", None),
    "no_history_step": ("Eq. 3a u' = u_t + h v_t (P:111)", "up[d] = ut[d] + h * vt[d];", "up[d] = ut[d];", None),
    "quat_order": ("q <- q (x) dq (O12/O13)", "double w1 = q[0], x1 = q[1], y1 = q[2], z1 = q[3];\n    double w2 = dq[0]",
                   "double w1 = dq[0], x1 = dq[1], y1 = dq[2], z1 = dq[3];\n    double w2 = q[0]", None),
    "mbar_sum": ("m-bar reduced clump mass (O5)", "m_bar = Mi * Mj / (Mi + Mj);", "m_bar = 0.5 * (Mi + Mj);", None),
    "rbar_sum": ("R-bar reduced radius (P:95)", "r_bar = ra * rb / (ra + rb);", "r_bar = 0.5 * (ra + rb);", None),
    "tension_clamp": ("no tension clamp (O8)", "double fn_s = k_n * delta - c_n * vn;",
                      "double fn_s = k_n * delta - c_n * vn;\n  if (fn_s < 0.0) fn_s = 0.0;", None),
    "cor_max": ("CoR_pair = min (O4)", "double e = ea < eb ? ea : eb;", "double e = ea > eb ? ea : eb;", None),
    "mu_max": ("mu_pair = min (O4)", "out[3] = mua < mub ? mua : mub;", "out[3] = mua > mub ? mua : mub;", None),
    "torque_ft_only": ("torque r x (F_n + F_t) (Eq. 4b literal; O11)", [
        ("  double f[3], r[3];\n} entry;", "  double f[3], r[3], ft[3];\n} entry;", None),
        ("      ea->f[d] = -C->F[d];", "      ea->f[d] = -C->F[d];\n      ea->ft[d] = -ft[d];", None),
        ("        eb->f[d] = C->F[d];", "        eb->f[d] = C->F[d];\n        eb->ft[d] = ft[d];", None),
        ("cross(E[k].r, E[k].f, tq);", "cross(E[k].r, E[k].ft, tq);", None)]),
    "damping_sign": ("damping opposes approach (O1)", "double fn_s = k_n * delta - c_n * vn;",
                     "double fn_s = k_n * delta + c_n * vn;", None),
    "cap_uses_kn_delta": ("cap mu |F_n| incl. damping (Eq. 3c; O7)", "double fn_mag = sqrt(dot(fn, fn));",
                          "double fn_mag = k_n * delta;", None),
    "clamp_ut_no_kt": ("u_t = (mu|F_n|/k_t) u'/|u'| (Eq. 3c)", "ut_new[d] = (cap / k_t) * dir;",
                       "ut_new[d] = cap * dir;", None),
    "no_ut_reset_on_separation": ("delta <= 0 resets u_t (O9)", "  if (!(delta > 0.0)) return;",
                                  "  if (!(delta > 0.0)) { for (d = 0; d < 3; ++d) ut_new[d] = ut[d]; return; }", None),
    "estar_parallel": ("series E* (O4)", "double inv_e = (1.0 - nua * nua) / Ea + (1.0 - nub * nub) / Eb;",
                       "double inv_e = 2.0 / (Ea / (1.0 - nua * nua) + Eb / (1.0 - nub * nub));", None),
    "predicate_strict": ("candidate predicate <= (O14, S:109 grazing)",
                         "return dx * dx + dy * dy + dz * dz <= sum * sum;",
                         "return dx * dx + dy * dy + dz * dz < sum * sum;", None),
    "intra_clump_pairs": ("intra-clump pairs excluded (O15, S:195)", [
        ("if (s->s_clump[a] != s->s_clump[b] && sphere_pair_candidate(s, a, b))",
         "if (sphere_pair_candidate(s, a, b))", 0),
        ("if (s->s_clump[a] != s->s_clump[b] && sphere_pair_candidate(s, a, b))",
         "if (sphere_pair_candidate(s, a, b))", None)]),
    "history_not_carried": ("u_t carried by key across rebuilds (P:109, S:200)",
                            "for (d = 0; d < 3; ++d) s->con[k].ut[d] = hit ? hit->ut[d] : 0.0;",
                            "for (d = 0; d < 3; ++d) s->con[k].ut[d] = 0.0;", None),
    "plane_margin_dropped": ("sphere-plane candidate (r + margin) - d >= 0 (O14)",
                             "if ((r + s->margin) - dd >= 0.0) push_contact",
                             "if (r - dd >= 0.0) push_contact", None),
    "integrator_explicit": ("semi-implicit Euler (O12)", "V[d] = V[d] + h * (F[d] / M);\n      X[d] = X[d] + h * V[d];",
                            "X[d] = X[d] + h * V[d];\n      V[d] = V[d] + h * (F[d] / M);", None),
}


def mutate(text, old, new, which):
    n = text.count(old)
    if n == 0:
        raise ValueError(f"pattern not found: {old[:60]}")
    if which is None:
        if n != 1:
            raise ValueError(f"pattern not unique ({n}): {old[:60]}")
        return text.replace(old, new)
    parts = text.split(old)
    return old.join(parts[:which + 1]) + new + old.join(parts[which + 1:])


def run(names, out):
    src = open(SRC).read()
    tmp = tempfile.mkdtemp(prefix="orcmut_")
    shutil.copy(os.path.join(ROOT, "oracle", "dem_oracle.h"), tmp)
    res = {}
    for name in names:
        spec = MUTATIONS[name]
        reading, sites = spec[0], (spec[1] if len(spec) == 2 else [spec[1:]])
        text = src
        for old, new, which in sites:
            text = mutate(text, old, new, which)
        c = os.path.join(tmp, f"{name}.c")
        so = os.path.join(tmp, f"{name}.so")
        open(c, "w").write(text)
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-std=c11", "-D_DEFAULT_SOURCE", "-fPIC", "-shared",
                               "-I", tmp, "-o", so, c, "-lm"])
        env = dict(os.environ, DEM_ORACLE_LIB=so)
        t0 = time.time()
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", *PINS],
                           cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
        failed = re.findall(r"^FAILED (\S+)", r.stdout, re.M)
        killed = r.returncode != 0
        res[name] = dict(reading=reading, killed=killed, n_failing=len(failed), by=failed,
                         seconds=round(time.time() - t0, 1))
        print(f"{name:28s} {'KILLED' if killed else 'SURVIVED':9s} {len(failed):3d} {failed[:2]}", flush=True)
    shutil.rmtree(tmp, ignore_errors=True)
    if out:
        os.makedirs(os.path.dirname(out), exist_ok=True)
        with open(out, "w") as f:
            json.dump(dict(pins=PINS, mutations=res), f, indent=1)
    return res


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "oracle_mutations.json"))
    a = ap.parse_args()
    res = run(a.names or list(MUTATIONS), a.out if not a.names else None)
    sys.exit(0 if all(v["killed"] for v in res.values()) else 1)
