// dem_device.cuh — device data layout and helpers of the B200 clump-DEM hot path.
//
// Product code (libdem_b200.so).  Independent of oracle/: nothing here is shared with
// or derived from the CPU checker; the formulas are restated from PAPER.md Sec. 2.1
// and DESIGN.md §3.
//
// HBM layout:
//   clump state   SoA fp64, 13 arrays (x,y,z, qw,qx,qy,qz, vx,vy,vz, wx,wy,wz), ping-pong
//   clump aux     tid (i32), gid (i64), sphere offset (i32, n+1), omega_world (3 x fp64, per step)
//   clump kin     packed per step: X, V, omega_world, mass (10 fp64 AoS) for coalesced partner gathers
//   sphere        clump (i32), template-component (i32), key (i64), (x,y,z,r) (double4 AoS),
//                 partial force/torque (3+3 fp64 SoA)
//   bins          cell_count (i32, ncell), cell_start (i32, ncell+1), items (i32, n_inserts)
//   slots         fixed-width candidate partner lists per owned sphere (i32), filled by the per-bin warps
//   rows (x2)     CSR by own sphere: row_ptr (i32, ns+1), partner (i32), key (i64), u_t (3 fp64 AoS)
#pragma once
#include <utility>
#include <cstdint>
#include <cuda_runtime.h>

namespace dem {

constexpr int kKeyStride = 64;
constexpr int kMaxPlanes = 16;
constexpr int kMaxMeshes = 8;
constexpr int kMeshRec = 17;  // per mesh: X(3), q(4), v(3), w(3), q_step(4) — DESIGN.md R27
constexpr int kMaxRowSort = 64;  // rows longer than this are sorted in place in global memory

// device status word (host reads it after each dem_step)
struct Ctl {
  int abort;          // set on capacity overflow or error: later kernels become no-ops
  int err_code;       // first device error (dem_status value), 0 = none
  long long err_key;  // sphere key / clump gid / contact key naming the error
  long long err_key2;
  long long err_step;
  long long step;     // steps completed since dem_set_state
  long long need_inserts;
  long long need_entries;
  long long need_width;  // row-slot width a rebuild needed (fixed-width candidate rows)
  int det_abort;         // capacity overflow of a set detected ahead (overlapped cadence)
  int need_regrid;       // a sphere centre left the bin region (the host re-grids between step batches)
};

#ifndef DEM_UT_PAD
#define DEM_UT_PAD 0  // 1: u_t padded to 32 bytes (one 256-bit access per entry)
#endif
constexpr int kUt = DEM_UT_PAD ? 4 : 3;  // doubles per entry of the tangential history (x, y, z[, 0]), AoS
#ifndef DEM_V256
#define DEM_V256 1  // 256-bit gathers of the 32-byte records (sm_100 LDG.256)
#endif
#ifndef DEM_SCATTER_RANKS
#define DEM_SCATTER_RANKS 0  // 1: ranks from the counting atomics, scatter without atomics; A/B on C5: pose
                             // 1.14 -> 1.70 ms (returning atomics), scatter 1.02 -> 0.95: dropped
#endif
// Spheres with at most kRankW bin inserts keep the rank their counting atomic returned (so the
// scatter needs no atomic); their counts live in the low 16 bits of cell_count, those of larger
// spheres (which take their slots with an atomic in the scatter) in the high 16 bits.
constexpr int kRankW = 8;
#ifndef DEM_SLOT_KEYS
#define DEM_SLOT_KEYS 0  // 1: partner keys written beside the slots by k_pairs; A/B on C5: pairs 4.71 -> 5.31 ms,
                         // rows 1.61 -> 1.65 ms (the flush gathers cost more than the row kernel saves)
#endif
#ifndef DEM_KIN_TID
#define DEM_KIN_TID 0  // 1: the clump's template id rides in the kinematics record (slot 10); A/B: force
                       // 3.94 -> 4.57 ms (the larger staging array costs the 8th resident CTA per SM)
#endif
// doubles per clump of the packed kinematics record read by the force kernel (with DEM_KIN_TID
// the template id bits in slot 10 and a pad: the integrating thread finds its inertia without a
// dependent global load)
constexpr int kKinUsed = DEM_KIN_TID ? 12 : 10;
// record stride: padded to 96 bytes so a partner's record is three 256-bit loads
constexpr int kKin = DEM_V256 ? 12 : 10;
static_assert(!DEM_V256 || (kKin * 8) % 32 == 0, "kinematics records must stay 32-byte aligned");
static_assert(!DEM_KIN_TID || kKin >= kKinUsed, "DEM_KIN_TID needs the 12-double (DEM_V256) record");

// 32-byte loads/stores in one instruction (sm_100: LDG.E.ENL2.256 / STG.E.ENL2.256); p must be
// 32-byte aligned.  A random gather of a 32-byte record then costs one L1 wavefront per lane
// instead of two.  The loads take the read-only path: only for data no thread of the same
// launch writes.
__device__ __forceinline__ double4 ldg256(const void* p) {
#if DEM_V256
  double4 v;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
#else
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 u = __ldg(q), w = __ldg(q + 1);
  return make_double4(u.x, u.y, w.x, w.y);
#endif
}
__device__ __forceinline__ void stg256(void* p, double x, double y, double z, double w) {
#if DEM_V256
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(x), "d"(y), "d"(z), "d"(w) : "memory");
#else
  double2* q = reinterpret_cast<double2*>(p);
  q[0] = make_double2(x, y);
  q[1] = make_double2(z, w);
#endif
}

struct Tables {
  const double* tc_off;   // [3 * n_tc] body-frame offsets, AoS
  const double* tc_rad;   // [n_tc]
  const int* tc_mat;      // [n_tc]
  const int* tpl_coff;    // [n_tmpl]
  const double* tpl_mass;
  const double* tpl_inertia;  // [3 * n_tmpl]
  const double* pair;     // [n_mat * n_mat * 8]: 2E*, 8G*, 2 sqrt(5/6) beta, mu, sqrt(4G*/E*) (symmetric)
  int n_mat;
  int n_planes;
  double plane_pt[kMaxPlanes][3];
  double plane_n[kMaxPlanes][3];
  int plane_mat[kMaxPlanes];
};

struct State {
  double *x, *y, *z, *qw, *qx, *qy, *qz, *vx, *vy, *vz, *wx, *wy, *wz;
};

struct Grid {
  double lo[3];
  double inv_cell;
  double cell;
  double dom_lo[3], dom_hi[3];
  int n[3];
  long long st[3];  // linear bin id = sum_d idx[d] * st[d]; shortest axis fastest (locality)
  int ax[3];        // axes from fastest to slowest
  double inv_n_ax[2];  // 1 / n[ax[0]], 1 / n[ax[1]] for the fast bin-id decode
  double pad;  // r + pad is the half-extent of a sphere's bin AABB (margin/2 + eps)
  double reg_lo[3], reg_hi[3];  // a centre outside these (where the bin region is tighter than the
                                // domain) asks for a re-grid: Ctl::need_regrid
};

// A row entry as the force kernel reads it (8 bytes); the partner keys live in their own array
// (Rows::key), read only by the row build/merge, dem_get_contacts and error reports.
struct __align__(8) Entry {
  int partner;      // partner local sphere index, or -1 - plane
  int prev;         // index of the same key in the previous step's rows (its u_t), or -1
};

struct Rows {
  int* row_ptr;     // [ns + 1]
  Entry* ent;       // [cap]
  long long* key;   // [cap] partner key (sphere key, or INT64_MAX - plane), ascending within a row
  double* ut;       // [kUt * cap] AoS (x, y, z), oriented own -> partner
};

struct Record {
  double* F;        // [3 * cap] force on partner (own = i)
  double* p;        // [3 * cap]
  double* n;        // [3 * cap]
  double* delta;    // [cap]
};

struct StepArgs {
  // sizes
  int n;            // clumps
  int ns;           // spheres
  long long ncell;
  long long cap_inserts;
  long long cap_entries;
  double h;
  double g[3];
  double margin;
  Tables tab;
  Grid grid;
  State cur, nxt;
  const int* tid;
  const long long* gid;
  const int* sph_off;
  const int* s_clump;
  const int* s_tc;
  const int* s_mat;          // material of each sphere (tc_mat[s_tc])
  const long long* s_key;
  double4* spos;             // sphere (x, y, z, r), written by the pose kernel each step
  double* kin;               // per clump [kKin]: X(3), V(3), omega_world(3), mass
  const int2* cta_clump;     // [n_cta + 1] (first clump, first sphere) of the fused force/integrate CTAs
  int n_cta;
  int count;                 // pose kernel: bin counts + wall row counts for a detection
  int remap;                 // force kernel: a new set is adopted this step, u_t via Entry::prev
  int adopt;                 // pose kernel: adopting a set detected ahead (turns det_abort into abort)
  const double4* ref_in;     // sphere centres the set in use was detected from (displacement check) or null
  double4* ref_out;          // where a counting pose kernel stores the centres it detects from, or null
  const double4* dpos;       // sphere centres the detection kernels read (spos, or the ahead snapshot)
  int* abort;                // abort word of the detection kernels (&ctl->abort, or &ctl->det_abort)
  // kinematic triangle meshes (NEXT-3): partner code of triangle t = -1 - kMaxPlanes - t,
  // key INT64_MAX - kMaxPlanes - t
  int n_tri, n_mesh;
  const double* tri_body;    // [9 n_tri] body-frame vertices
  const int* tri_vid;        // [3 n_tri] vertex ids (topology for one contact per feature, R26)
  const int* tri_mesh;       // [n_tri]
  double* tri_world;         // [9 n_tri] world vertices of this step (k_mesh_pose)
  double* tri_snap;          // [9 n_tri] copy for an ahead detection, or null
  const double* tri_dpos;    // the vertices the detection kernels read (tri_world or tri_snap)
  double* mesh;              // [kMeshRec n_mesh] pose + motion (advanced by k_mesh_finish)
  const int* mesh_mat;       // [n_mesh]
  double* mesh_part;         // [6 n_mesh n_cta] per-CTA wrench partials (force on mesh, torque about X)
  int* mesh_flag;            // [n_cta] 1 if the CTA wrote a partial this step
  double* mesh_wrench;       // [6 n_mesh] the last step's wrench
  // mesh entries of the set in use (k_mesh_geom) and of the set being detected (k_rows_finish):
  // (entry, own sphere) pairs, and the per-entry closest point + "counts" flag of this step
  const int2* mlist;         // [*mlist_n]
  const int* mlist_n;
  int2* mlist_out;
  int* mlist_out_n;
  double4* mgeom;            // [cap_entries] closest point (x, y, z), w = 1 if the contact counts (R26)
  // fused halo (peer transport): the integrating thread of a clump in a send list
  // writes its new state straight into the neighbour's next-state array at the neighbour's ghost
  // slot (NVLink peer stores), so there is no pack, no collective and no unpack
  double* peer_state[2];     // [side] the neighbour's next-state SoA base (13 arrays of peer_n), or null
  long long peer_n[2];       // [side] the neighbour's clump count (SoA stride)
  const int* peer_idx[2];    // [side][n_own] the neighbour's ghost slot of each owned clump, or -1
  double half_margin;        // > 0 (cd_every > 1): displacement allowed since the last rebuild
  int n_own, ns_own;         // owned clumps / spheres come first; the rest are ghosts (§8e)
  const double* xref;        // [3 n_own] owned COMs at dem_set_state (distributed drift check)
  double drift_max;          // 0: no check
  int* cell_count;
  unsigned short* irank;     // [kRankW][ns] each insert's rank in its bin, from the counting atomics (DEM_SCATTER_RANKS)
  int* cell_start;
  int* items;                // [cap_inserts] bin items: sphere index | lowest-bin mask << 29
  int* row_cnt;              // walls + sphere partners per sphere (built by atomics each step)
  unsigned short* wall_mask; // [ns] sphere-plane candidates of the detection (bit p: plane p)
  int* slots;                // [row_width][ns_own] candidate partners of the owned spheres (k_pairs)
  long long* slot_key;       // [row_width][ns_own] their keys (DEM_SLOT_KEYS: written by the producers,
                             // so k_rows_finish sorts without a dependent gather of s_key)
  int row_width;             // slots per sphere (walls included: slot w is the w-th entry of the row)
  Rows rows, prev;
  Record rec;
  int record;
  Ctl* ctl;
  int pdl;                   // launch the step's kernels after the first with programmatic serialization
  int tiny;                  // k_pairs with the small-bin pass (sparse bins: fewer than 2 spheres per bin)
  int pairs_contig;          // k_pairs: bins per warp in a CTA span (set by launch_pairs)
};

// ---------------------------------------------------------------- programmatic dependent launch
// The step kernels after the first are launched with programmatic stream serialization (captured
// into the step graphs as programmatic edges): a kernel's CTAs may become resident while its
// predecessor's last wave drains, and wait at their very first instruction (griddepcontrol.wait,
// which returns once the predecessor grid has completed and its memory is visible) — the launch
// and ramp-up overlap the tail; no data is read early.  Each kernel lets its dependent launch as
// soon as it started (launch_dependents).  Without the attribute both are no-ops.
#ifndef DEM_PDL
#define DEM_PDL 0  // A/B (tools/ab_sizes.sh): C5 and a C5/8 slab unchanged, a C5/45 slab +4%, C3 -1%: off
#endif
__device__ __forceinline__ void pdl_wait_and_release() {
#if DEM_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
#endif
}
// host: launch `kern` on `s`, with programmatic serialization when `pdl`
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, bool pdl,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (DEM_PDL && pdl) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- error latch
__device__ __forceinline__ void raise_error(Ctl* ctl, int code, long long key, long long key2) {
  if (atomicCAS(&ctl->err_code, 0, code) == 0) {
    ctl->err_key = key;
    ctl->err_key2 = key2;
    ctl->err_step = ctl->step;
  }
  atomicExch(&ctl->abort, 1);
}

// ---------------------------------------------------------------- exact-rounding helpers
// Sphere centres and the candidate predicate are evaluated with explicitly rounded
// operations (no FMA contraction) in the order written in DESIGN.md §3 R14/R22, so the
// contact set is a function of the fp64 state alone.
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// R(q) for q = (w,x,y,z), Hamilton, body -> world; row-major R[0..8]
__device__ __forceinline__ void quat_R(double w, double x, double y, double z, double R[9]) {
  double xx = mul(x, x), yy = mul(y, y), zz = mul(z, z);
  double xy = mul(x, y), xz = mul(x, z), yz = mul(y, z);
  double wx = mul(w, x), wy = mul(w, y), wz = mul(w, z);
  R[0] = sub(1.0, mul(2.0, add(yy, zz)));
  R[1] = mul(2.0, sub(xy, wz));
  R[2] = mul(2.0, add(xz, wy));
  R[3] = mul(2.0, add(xy, wz));
  R[4] = sub(1.0, mul(2.0, add(xx, zz)));
  R[5] = mul(2.0, sub(yz, wx));
  R[6] = mul(2.0, sub(xz, wy));
  R[7] = mul(2.0, add(yz, wx));
  R[8] = sub(1.0, mul(2.0, add(xx, yy)));
}

// (R v)_row = (R0 v0 + R1 v1) + R2 v2, each product rounded
__device__ __forceinline__ double row_dot(const double* R, double a, double b, double c) {
  return add(add(mul(R[0], a), mul(R[1], b)), mul(R[2], c));
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// bin-index range of the sphere's enlarged AABB along one axis (clamped to the grid)
__device__ __forceinline__ void cell_range(const Grid& g, int d, double c, double r, int& lo, int& hi) {
  double e = r + g.pad;
  lo = clampi(__double2int_rd((c - e - g.lo[d]) * g.inv_cell), 0, g.n[d] - 1);
  hi = clampi(__double2int_rd((c + e - g.lo[d]) * g.inv_cell), 0, g.n[d] - 1);
}

// q = quot * d + rem for 0 <= q < 2^31 (bin ids), via an fp64 reciprocal and a one-step fix-up
// (the 64-bit integer division it replaces is a ~60-instruction software routine)
__device__ __forceinline__ int divmod_fast(int q, int d, double inv_d, int& rem) {
  int quot = __double2int_rz((double)q * inv_d);
  int r = q - quot * d;
  if (r < 0) {
    --quot;
    r += d;
  } else if (r >= d) {
    ++quot;
    r -= d;
  }
  rem = r;
  return quot;
}

// linear bin id -> bin coordinates (inverse of sum_d idx[d] * st[d])
__device__ __forceinline__ void decode_bin(const Grid& g, long long cid, int& cx, int& cy, int& cz) {
  int c[3];
  int q = divmod_fast((int)cid, g.n[g.ax[0]], g.inv_n_ax[0], c[g.ax[0]]);
  c[g.ax[2]] = divmod_fast(q, g.n[g.ax[1]], g.inv_n_ax[1], c[g.ax[1]]);
  cx = c[0];
  cy = c[1];
  cz = c[2];
}

__device__ __forceinline__ int cell_lo(const Grid& g, int d, double c, double r) {
  double e = r + g.pad;
  return clampi(__double2int_rd((c - e - g.lo[d]) * g.inv_cell), 0, g.n[d] - 1);
}

// velocity of a body point: V + omega x r, written with explicit roundings so the
// own-side and partner-side evaluations of one contact are bitwise mirror images
__device__ __forceinline__ void point_velocity(double Vx, double Vy, double Vz, double wx, double wy,
                                               double wz, double rx, double ry, double rz, double& ox,
                                               double& oy, double& oz) {
  ox = __dadd_rn(Vx, __fma_rn(wy, rz, -__dmul_rn(wz, ry)));
  oy = __dadd_rn(Vy, __fma_rn(wz, rx, -__dmul_rn(wx, rz)));
  oz = __dadd_rn(Vz, __fma_rn(wx, ry, -__dmul_rn(wy, rx)));
}

// ---------------------------------------------------------------- triangles (NEXT-3)
// Closest point of triangle (a, b, c) to p by Voronoi regions, R25: the operation
// order of the oracle's plain-C construction, every operation rounded separately, so the
// sphere-triangle candidate set is a function of the fp64 inputs.  Returns the region: 0 face,
// 1/2/3 edge ab/ac/bc, 4/5/6 vertex a/b/c.
__device__ __forceinline__ double dot3r(double ux, double uy, double uz, double vx, double vy, double vz) {
  return add(add(mul(ux, vx), mul(uy, vy)), mul(uz, vz));
}

__device__ __forceinline__ int closest_on_triangle(const double* T, double px, double py, double pz, double& qx,
                                                   double& qy, double& qz) {
  const double ax = T[0], ay = T[1], az = T[2], bx = T[3], by = T[4], bz = T[5], cx = T[6], cy = T[7], cz = T[8];
  const double abx = sub(bx, ax), aby = sub(by, ay), abz = sub(bz, az);
  const double acx = sub(cx, ax), acy = sub(cy, ay), acz = sub(cz, az);
  const double apx = sub(px, ax), apy = sub(py, ay), apz = sub(pz, az);
  const double d1 = dot3r(abx, aby, abz, apx, apy, apz), d2 = dot3r(acx, acy, acz, apx, apy, apz);
  if (d1 <= 0.0 && d2 <= 0.0) {
    qx = ax; qy = ay; qz = az;
    return 4;
  }
  const double bpx = sub(px, bx), bpy = sub(py, by), bpz = sub(pz, bz);
  const double d3 = dot3r(abx, aby, abz, bpx, bpy, bpz), d4 = dot3r(acx, acy, acz, bpx, bpy, bpz);
  if (d3 >= 0.0 && d4 <= d3) {
    qx = bx; qy = by; qz = bz;
    return 5;
  }
  const double vc = sub(mul(d1, d4), mul(d3, d2));
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
    const double v = __ddiv_rn(d1, sub(d1, d3));
    qx = add(ax, mul(v, abx)); qy = add(ay, mul(v, aby)); qz = add(az, mul(v, abz));
    return 1;
  }
  const double cpx = sub(px, cx), cpy = sub(py, cy), cpz = sub(pz, cz);
  const double d5 = dot3r(abx, aby, abz, cpx, cpy, cpz), d6 = dot3r(acx, acy, acz, cpx, cpy, cpz);
  if (d6 >= 0.0 && d5 <= d6) {
    qx = cx; qy = cy; qz = cz;
    return 6;
  }
  const double vb = sub(mul(d5, d2), mul(d1, d6));
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
    const double w = __ddiv_rn(d2, sub(d2, d6));
    qx = add(ax, mul(w, acx)); qy = add(ay, mul(w, acy)); qz = add(az, mul(w, acz));
    return 2;
  }
  const double va = sub(mul(d3, d6), mul(d5, d4));
  const double e43 = sub(d4, d3), e56 = sub(d5, d6);
  if (va <= 0.0 && e43 >= 0.0 && e56 >= 0.0) {
    const double w = __ddiv_rn(e43, add(e43, e56));
    qx = add(bx, mul(w, sub(cx, bx))); qy = add(by, mul(w, sub(cy, by))); qz = add(bz, mul(w, sub(cz, bz)));
    return 3;
  }
  const double denom = __drcp_rn(add(add(va, vb), vc));
  const double v = mul(vb, denom), w = mul(vc, denom);
  qx = add(add(ax, mul(abx, v)), mul(acx, w));
  qy = add(add(ay, mul(aby, v)), mul(acy, w));
  qz = add(add(az, mul(abz, v)), mul(acz, w));
  return 0;
}

// feature of (triangle, region) for one contact per feature (R26): kind 2 face (u = t),
// 1 edge (u < v vertex ids), 0 vertex (u)
__device__ __forceinline__ void tri_feature(const int* vid, int t, int region, int& kind, int& u, int& v) {
  if (region == 0) {
    kind = 2; u = v = t;
  } else if (region <= 3) {
    const int x = vid[3 * t + (region == 3 ? 1 : 0)], y = vid[3 * t + (region == 1 ? 1 : 2)];
    kind = 1; u = min(x, y); v = max(x, y);
  } else {
    kind = 0; u = v = vid[3 * t + region - 4];
  }
}

__device__ __forceinline__ bool tri_has(const int* vid, int t, int x) {
  return vid[3 * t] == x || vid[3 * t + 1] == x || vid[3 * t + 2] == x;
}

// the abort words of a loopback group (k_abort_or)
constexpr int kMaxGroup = 64;
struct AbortWords {
  int* p[kMaxGroup];
  int n;
};

}  // namespace dem
