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
#include <cstdint>
#include <cuda_runtime.h>

namespace dem {

constexpr int kKeyStride = 64;
constexpr int kMaxPlanes = 16;
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
  int pad_;
};

constexpr int kUt = 4;    // doubles per entry of the tangential history (padded)
constexpr int kKin = 10;  // doubles per clump in the packed kinematics record

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
};

struct __align__(16) Entry {
  long long key;    // partner key (sphere key, or INT64_MAX - plane)
  int partner;      // partner local sphere index, or -1 - plane
  int prev;         // index of the same key in the previous step's rows (its u_t), or -1
};

struct Rows {
  int* row_ptr;     // [ns + 1]
  Entry* ent;       // [cap]
  double* ut;       // [kUt * cap] AoS (x, y, z, 0): one 32-byte sector per entry, oriented own -> partner
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
  double half_margin;        // > 0 (cd_every > 1): displacement allowed since the last rebuild
  int n_own, ns_own;         // owned clumps / spheres come first; the rest are ghosts (§8e)
  const double* xref;        // [3 n_own] owned COMs at dem_set_state (distributed drift check)
  double drift_max;          // 0: no check
  int* cell_count;
  int* cell_start;
  int* items;                // [cap_inserts] bin items: sphere index | lowest-bin mask << 29
  int* row_cnt;              // walls + sphere partners per sphere (built by atomics each step)
  int* slots;                // [row_width][ns_own] candidate partners of the owned spheres (k_pairs)
  int row_width;             // slots per sphere (walls included: slot w is the w-th entry of the row)
  Rows rows, prev;
  Record rec;
  int record;
  Ctl* ctl;
};

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

}  // namespace dem
