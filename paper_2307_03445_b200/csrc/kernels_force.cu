// kernels_force.cu — (a4) history remap, (a5-a8) contact forces, (a9) reduction, (a10) integration.
//
// PAPER.md Sec. 2.1: Eq. 1a-1e, Eq. 2a-2c, Eq. 3a-3c,
// Eq. 4a-4b.  Readings: R1 force on j with n from i to j;
// R2/R3 Hertz coefficients S_n = 2E*sqrt(R d), k_n = 2/3 S_n, c_n = 2 sqrt(5/6) beta
// sqrt(S_n m), k_t = 8 G* sqrt(R d), c_t = 2 sqrt(5/6) beta sqrt(k_t m); R5 m from clump
// masses, R from sphere radii; R6 contact point = middle of the overlap; R7 Eq. 3c literal;
// R8 no tension clamp; R9 u_t = 0 once delta <= 0; R11 torque r x (F_n + F_t) with the
// gyroscopic term; R12 semi-implicit Euler + exponential-map quaternion update.
//
// Directed "pull" rows: every sphere evaluates each of its contacts with itself as body i
// and produces only its own partial wrench.  The two evaluations of one sphere pair are
// bitwise mirror images (every operation is sign-symmetric under i <-> j and the
// asymmetric point velocities use explicit roundings), so Newton's third law holds
// exactly without atomics, and sums run in a canonical order (partner key, then
// component) independent of storage order.
//
// Parallel layout of k_force_integrate: a CTA owns a run of whole clumps, whose spheres'
// rows are one contiguous range of the CSR arrays.  One thread per directed entry evaluates
// a contact (no serial per-sphere chains, so gathers of many entries are in flight at
// once) and writes its partial wrench to shared memory; one thread per sphere adds its
// entries in row order, then one thread per clump adds its spheres in component order and
// integrates — the canonical sums of DESIGN.md R23, with no per-sphere wrench in HBM.
#include "dem_device.cuh"

namespace dem {

constexpr int kPairStride = 8;  // doubles per material pair in Tables::pair
#ifndef DEM_FORCE_OWNER
#define DEM_FORCE_OWNER 0  // 1: owner sphere of each entry from a shared table built per chunk; 0: a binary search over the CTA row bounds (A/B round 2 with the batched prologue: force 3.835 -> 3.807 ms)
#endif
#ifndef DEM_FORCE_UT_ASYNC
#define DEM_FORCE_UT_ASYNC 0  // 1: previous u_t staged by cp.async into the thread's part[] slots (A/B: force 3.94 -> 5.10 ms)
#endif
#ifndef DEM_FORCE_LAZY_OWN
#define DEM_FORCE_LAZY_OWN 0  // 1: own clump's record read (volatile) from shared memory at its uses: fewer spills, A/B neutral
#endif
#ifndef DEM_FORCE_ASYNC_EPI
#define DEM_FORCE_ASYNC_EPI 0  // 1: own clumps' q, Omega, inertia staged by cp.async in the prologue (A/B: 3.96 -> 4.73 ms)
#endif
#ifndef DEM_FORCE_PRO
#define DEM_FORCE_PRO 1  // batched prologue loads + the first chunk's entries issued before the barrier
#endif
#ifndef DEM_FORCE_FT
#define DEM_FORCE_FT 128
#endif
#ifndef DEM_FORCE_FC
#define DEM_FORCE_FC (DEM_FORCE_FT * 3 / 8)  // 48 clumps: CTAs are cut by entries (system.cu)
#endif
#ifndef DEM_FORCE_MAXS
#define DEM_FORCE_MAXS (DEM_FORCE_FT * 9 / 8)  // 144: force 4.30 ms vs 4.84 at 160 (entry-cut CTAs)
#endif
constexpr int kFT = DEM_FORCE_FT;      // threads per CTA (= entries per chunk)
// Skewed slots of the per-entry partials: entry q at q + q/16, so the per-sphere sums (lane l reads
// entry ~ c l + b, rows of a few entries) spread over all bank pairs instead of every c-th
#ifndef DEM_FORCE_SKEW
#define DEM_FORCE_SKEW 0  // A/B on C5: force 3.835 -> 3.85 ms (the index arithmetic costs more than the conflicts): off
#endif
constexpr int kPartW = DEM_FORCE_SKEW ? kFT + kFT / 16 : kFT;
__device__ __forceinline__ int pslot(int q) { return DEM_FORCE_SKEW ? q + (q >> 4) : q; }
constexpr int kFC = DEM_FORCE_FC;      // max clumps per CTA (host partition, see system.cu)
constexpr int kMaxS = DEM_FORCE_MAXS;  // max spheres per CTA
int force_cta_clumps() { return kFC; }
int force_cta_spheres() { return kMaxS; }

// One CTA = a run of whole clumps [c0, c1) and their spheres [s0, s0 + nsph), whose rows are
// one contiguous CSR range [E0, E1).
#ifndef DEM_FORCE_MINB
#define DEM_FORCE_MINB (1024 / DEM_FORCE_FT)  // 64 registers
#endif
#ifndef DEM_FORCE_MINB_MESH
#define DEM_FORCE_MINB_MESH DEM_FORCE_MINB  // 80 registers (6 CTAs) spill less but run slower
#endif
// Mesh entries (NEXT-3), per step, before the force kernel: the sphere's closest point on the
// triangle (R25) and whether the contact counts under one contact per feature (R26: face >
// edge > vertex among the sphere's entries on the same mesh, ties to the lower triangle).  The
// force kernel then treats a mesh entry like a wall entry with this point.
__global__ void __launch_bounds__(256) k_mesh_geom(StepArgs a) {
  if (a.ctl->abort) return;
  const int n = *a.mlist_n;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int2 it = a.mlist[k];
    const int e = it.x, i = it.y;
    const int tri = -1 - kMaxPlanes - a.rows.ent[e].partner;
    const double4 c = a.spos[i];
    double qx, qy, qz;
    const int reg = closest_on_triangle(a.tri_world + 9 * tri, c.x, c.y, c.z, qx, qy, qz);
    const int mesh = a.tri_mesh[tri];
    int kind, u, v;
    tri_feature(a.tri_vid, tri, reg, kind, u, v);
    bool counts = true;
    if (kind != 2)
      for (int f = a.rows.row_ptr[i], fe = a.rows.row_ptr[i + 1]; f < fe && counts; ++f) {
        const int code = a.rows.ent[f].partner;
        if (code > -1 - kMaxPlanes) continue;
        const int tj = -1 - kMaxPlanes - code;
        if (tj == tri || a.tri_mesh[tj] != mesh) continue;
        double ox, oy, oz;
        const int rj = closest_on_triangle(a.tri_world + 9 * tj, c.x, c.y, c.z, ox, oy, oz);
        int kj, uj, vj;
        tri_feature(a.tri_vid, tj, rj, kj, uj, vj);
        if (kind == 1) {
          if (kj == 2 && tri_has(a.tri_vid, tj, u) && tri_has(a.tri_vid, tj, v)) counts = false;
          if (kj == 1 && uj == u && vj == v && tj < tri) counts = false;
        } else {
          if (kj == 2 && tri_has(a.tri_vid, tj, u)) counts = false;
          if (kj == 1 && (uj == u || vj == u)) counts = false;
          if (kj == 0 && uj == u && tj < tri) counts = false;
        }
      }
    a.mgeom[e] = make_double4(qx, qy, qz, counts ? 1.0 : 0.0);
  }
}
void launch_mesh_geom(const StepArgs& a, cudaStream_t s) {
  if (a.n_tri) k_mesh_geom<<<4 * 148, 256, 0, s>>>(a);
}

template <bool kMesh, bool kPeer>
__global__ void __launch_bounds__(kFT, kMesh ? DEM_FORCE_MINB_MESH : DEM_FORCE_MINB) k_force_integrate(StepArgs a) {
  __shared__ int rp[kMaxS + 1];
  __shared__ double4 own_p[kMaxS];
  __shared__ int own_mat[kMaxS];
  __shared__ int own_lc[kMaxS];
  __shared__ __align__(16) double ck[kFC * kKinUsed];
  __shared__ double part[6][kPartW];
  __shared__ double acc[6][kMaxS];
  __shared__ unsigned char own_of[DEM_FORCE_OWNER ? kFT : 1];  // entry of the chunk -> its own sphere
  __shared__ double cq[DEM_FORCE_ASYNC_EPI ? 10 : 1][kFC];     // own clumps' q, Omega_body, inertia (Eq. 4)
  // mesh wrench (kMesh): per entry the mesh id (-1: not a mesh entry) and torque about its X
  __shared__ int emesh[kMesh ? kFT : 1];
  __shared__ double mtq[3][kMesh ? kFT : 1];
  __shared__ double cw[kMesh ? kMaxMeshes : 1][6];
  __shared__ int chunk_mesh, cta_mesh;  // this chunk / this CTA holds mesh entries
  pdl_wait_and_release();
  const int tid = threadIdx.x;
  const int2 b0 = a.cta_clump[blockIdx.x], b1 = a.cta_clump[blockIdx.x + 1];
  const int c0 = b0.x, c1 = b1.x;
  const int ncl = c1 - c0;
  if (a.ctl->abort) {
    // capacity abort / error: carry the state forward unchanged so the ping-pong stays valid —
    // the ghosts too (a distributed abort is agreed by every rank, so no neighbour stores them)
    auto carry = [&](int c) {
      a.nxt.x[c] = a.cur.x[c]; a.nxt.y[c] = a.cur.y[c]; a.nxt.z[c] = a.cur.z[c];
      a.nxt.qw[c] = a.cur.qw[c]; a.nxt.qx[c] = a.cur.qx[c]; a.nxt.qy[c] = a.cur.qy[c]; a.nxt.qz[c] = a.cur.qz[c];
      a.nxt.vx[c] = a.cur.vx[c]; a.nxt.vy[c] = a.cur.vy[c]; a.nxt.vz[c] = a.cur.vz[c];
      a.nxt.wx[c] = a.cur.wx[c]; a.nxt.wy[c] = a.cur.wy[c]; a.nxt.wz[c] = a.cur.wz[c];
    };
    if (tid < ncl) carry(c0 + tid);
    for (int c = a.n_own + blockIdx.x * kFT + tid; c < a.n; c += gridDim.x * kFT) carry(c);
    return;
  }
  if (blockIdx.x == 0 && tid == 0) a.ctl->step += 1;  // no other thread of this launch reads it
  const int s0 = b0.y;
  const int nsph = b1.y - s0;
  const int E0g = a.rows.row_ptr[s0];
#if DEM_FORCE_PRO
  // Batched prologue: every load of the CTA's staging (row bounds, own sphere records, materials,
  // clumps, kinematics records) and the first chunk's row entry are issued before any of them is
  // stored, so the prologue costs one memory round trip instead of one per staging loop.
  static_assert(kMaxS < 2 * kFT && kFC * (kKinUsed / 2) <= 2 * kFT, "two staging loads per thread");
  Entry ent_first;
  ent_first.partner = -1;
  ent_first.prev = -1;
  {
    const double2* src = reinterpret_cast<const double2*>(a.kin + (size_t)kKin * c0);
    int r0v[2], r1v[2], mv[2], cv[2];
    double4 pv[2];
    double2 kv[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int k = tid + u * kFT;
      r0v[u] = k <= nsph ? a.rows.row_ptr[s0 + k] : 0;
      r1v[u] = k < nsph ? a.rows.row_ptr[s0 + k + 1] : 0;
      if (k < nsph) {
        pv[u] = ldg256(a.spos + s0 + k);
        mv[u] = a.s_mat[s0 + k];
        cv[u] = a.s_clump[s0 + k];
      }
      if (k < ncl * (kKinUsed / 2)) {
        const int c = k / (kKinUsed / 2), r = k - c * (kKinUsed / 2);
        kv[u] = src[c * (kKin / 2) + r];
      }
    }
    const int E1g = a.rows.row_ptr[s0 + nsph];
    if (E0g + tid < E1g) ent_first = a.rows.ent[E0g + tid];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int k = tid + u * kFT;
      if (k <= nsph) rp[k] = r0v[u];
      if (k < nsph) {
        if (DEM_FORCE_OWNER)
          for (int q = max(r0v[u], E0g); q < min(r1v[u], E0g + kFT); ++q) own_of[q - E0g] = (unsigned char)k;
        own_p[k] = pv[u];
        own_mat[k] = mv[u];
        own_lc[k] = cv[u] - c0;
#pragma unroll
        for (int q = 0; q < 6; ++q) acc[q][k] = 0.0;
      }
      if (k < ncl * (kKinUsed / 2)) reinterpret_cast<double2*>(ck)[k] = kv[u];
    }
  }
#else
  for (int k = tid; k <= nsph; k += kFT) {
    const int r0 = a.rows.row_ptr[s0 + k];
    rp[k] = r0;
    if (k < nsph) {  // owner of each entry of the first chunk (later chunks: built beside the sums)
      const int r1 = a.rows.row_ptr[s0 + k + 1];
      if (DEM_FORCE_OWNER)
        for (int q = max(r0, E0g); q < min(r1, E0g + kFT); ++q) own_of[q - E0g] = (unsigned char)k;
    }
  }
  for (int ls = tid; ls < nsph; ls += kFT) {
    const int i = s0 + ls;
    own_p[ls] = a.spos[i];
    own_mat[ls] = a.s_mat[i];
    own_lc[ls] = a.s_clump[i] - c0;
#pragma unroll
    for (int q = 0; q < 6; ++q) acc[q][ls] = 0.0;
  }
  {
    // the used doubles of each record (global stride kKin, shared stride kKinUsed)
    const double2* src = reinterpret_cast<const double2*>(a.kin + (size_t)kKin * c0);
    for (int k = tid; k < ncl * (kKinUsed / 2); k += kFT) {
      const int c = k / (kKinUsed / 2), r = k - c * (kKinUsed / 2);
      reinterpret_cast<double2*>(ck)[k] = src[c * (kKin / 2) + r];
    }
  }
#endif
  if (DEM_FORCE_ASYNC_EPI && tid < ncl) {
    // the integrating thread's q, Omega (body) and inertia, copied to shared memory in the
    // background (cp.async, no registers held) and awaited only after the entry loop
    const int c = c0 + tid, t = a.tid[c];
    const double* src[10] = {a.cur.qw + c, a.cur.qx + c, a.cur.qy + c, a.cur.qz + c, a.cur.wx + c,
                             a.cur.wy + c, a.cur.wz + c, a.tab.tpl_inertia + 3 * t, a.tab.tpl_inertia + 3 * t + 1,
                             a.tab.tpl_inertia + 3 * t + 2};
#pragma unroll
    for (int k = 0; k < 10; ++k) {
      const unsigned dst = (unsigned)__cvta_generic_to_shared(&cq[k][tid]);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src[k]) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  if (kMesh && tid < kMaxMeshes * 6) cw[tid / 6][tid % 6] = 0.0;
  if (kMesh && tid == 0) chunk_mesh = cta_mesh = 0;
  __syncthreads();
  const double h = a.h;
  const int E0 = rp[0], E1 = rp[nsph];
  for (int c0e = E0; c0e < E1; c0e += kFT) {
    const int e = c0e + tid;
    if (kMesh) emesh[tid] = -1;
    if (e < E1) {
#if DEM_FORCE_OWNER
      const int ls = own_of[tid];
#else
      int lo = 0, hi = nsph - 1;  // owner: last ls with rp[ls] <= e
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (rp[mid] <= e) lo = mid; else hi = mid - 1;
      }
      const int ls = lo;
#endif
      const double4 own = own_p[ls];
      const double cx = own.x, cy = own.y, cz = own.z, ri = own.w;
#if DEM_FORCE_LAZY_OWN
      // the own clump's record is read from shared memory where it is used (volatile: the
      // compiler would otherwise hoist these loads above the partner gathers and spill them)
      const volatile double* ki = ck + kKinUsed * own_lc[ls];
#define Mi (ki[9])
#else
      const double* ki = ck + kKinUsed * own_lc[ls];
      const double Mi = ki[9];
#endif
#if DEM_FORCE_PRO
      const Entry ent = c0e == E0 ? ent_first : a.rows.ent[e];
#else
      const Entry ent = a.rows.ent[e];
#endif
      const int t = ent.partner;
      // (a4) history remap: the slot of this key in the previous rows was found by the
      // row merge in k_rows_finish (-1: contact born this step, u_t = 0)
      // (between rebuilds the set is unchanged: the entry's own slot of the previous u_t)
      const int pidx = a.remap ? ent.prev : e;
#if DEM_FORCE_UT_ASYNC
      // the previous u_t is copied into this thread's slots of part[0..2] (written by this thread
      // only after its last use) with cp.async: no registers are held across the partner gathers
      if (pidx >= 0) {
        const double* u = a.prev.ut + (size_t)kUt * pidx;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const unsigned dst = (unsigned)__cvta_generic_to_shared(&part[d][pslot(tid)]);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(u + d) : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
#else
      double ux = 0.0, uy = 0.0, uz = 0.0;
      if (pidx >= 0) {
#if DEM_UT_PAD
        const double4 u = ldg256(a.prev.ut + (size_t)kUt * pidx);
        ux = u.x; uy = u.y; uz = u.z;
#else
        const double* u = a.prev.ut + (size_t)kUt * pidx;
        ux = __ldg(u);
        uy = __ldg(u + 1);
        uz = __ldg(u + 2);
#endif
      }
#endif
      // (a5) geometry: n from i (own) to j (partner)
      double nx, ny, nz, px, py, pz, delta, rbar, mbar;
      double Xjx = 0, Xjy = 0, Xjz = 0, Vjx = 0, Vjy = 0, Vjz = 0, Wjx = 0, Wjy = 0, Wjz = 0;
      int mj;
      const bool wall = t < 0;
      bool degenerate = false;
      bool active = true;
      int mesh = -1;
      if (kMesh && t <= -1 - kMaxPlanes) {
        // the closest point and the feature rule come from k_mesh_geom; n from the sphere to
        // the surface, the middle of the overlap, the flat-wall limit (R25-R27)
        const double4 gq = a.mgeom[e];
        const double dx = sub(cx, gq.x), dy = sub(cy, gq.y), dz = sub(cz, gq.z);
        const double dist = sqrt(add(add(mul(dx, dx), mul(dy, dy)), mul(dz, dz)));
        degenerate = dist == 0.0;
        delta = ri - dist;
        const double inv = 1.0 / dist;
        nx = -(dx * inv);
        ny = -(dy * inv);
        nz = -(dz * inv);
        const double arm = ri - 0.5 * delta;
        px = cx + arm * nx;
        py = cy + arm * ny;
        pz = cz + arm * nz;
        active = gq.w != 0.0;
        mesh = a.tri_mesh[-1 - kMaxPlanes - t];
        mj = a.mesh_mat[mesh];
        const double* M = a.mesh + kMeshRec * mesh;
        Xjx = M[0]; Xjy = M[1]; Xjz = M[2];
        Vjx = M[7]; Vjy = M[8]; Vjz = M[9];
        Wjx = M[10]; Wjy = M[11]; Wjz = M[12];
        rbar = ri;
        mbar = Mi;
      } else if (!wall) {
        const double4 pj = ldg256(a.spos + t);
        const double* kjp = a.kin + (size_t)kKin * a.s_clump[t];
        mj = a.s_mat[t];
        const double rj = pj.w;
        const double dx = pj.x - cx, dy = pj.y - cy, dz = pj.z - cz;
        const double dist = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
        degenerate = dist == 0.0;
        delta = (ri + rj) - dist;
        const double inv = 1.0 / dist;  // sign-symmetric: the mirror entry gets exactly -n
        nx = dx * inv;
        ny = dy * inv;
        nz = dz * inv;
        const double hr = 0.5 * (ri - rj);
        px = __fma_rn(hr, nx, 0.5 * (cx + pj.x));
        py = __fma_rn(hr, ny, 0.5 * (cy + pj.y));
        pz = __fma_rn(hr, nz, 0.5 * (cz + pj.z));
        rbar = (ri * rj) / (ri + rj);
#if DEM_V256
        const double4 k03 = ldg256(kjp), k47 = ldg256(kjp + 4), k8b = ldg256(kjp + 8);
        const double Mj = k8b.y;
        mbar = (Mi * Mj) / (Mi + Mj);
        Xjx = k03.x; Xjy = k03.y; Xjz = k03.z;
        Vjx = k03.w; Vjy = k47.x; Vjz = k47.y;
        Wjx = k47.z; Wjy = k47.w; Wjz = k8b.x;
#else
        const double2* kj = reinterpret_cast<const double2*>(kjp);
        const double2 k01 = kj[0], k23 = kj[1], k45 = kj[2], k67 = kj[3], k89 = kj[4];
        const double Mj = k89.y;
        mbar = (Mi * Mj) / (Mi + Mj);
        Xjx = k01.x; Xjy = k01.y; Xjz = k23.x;
        Vjx = k23.y; Vjy = k45.x; Vjz = k45.y;
        Wjx = k67.x; Wjy = k67.y; Wjz = k89.x;
#endif
      } else {
        const int pl = -1 - t;
        const double* pp = a.tab.plane_pt[pl];
        const double* nw = a.tab.plane_n[pl];
        const double dd = (cx - pp[0]) * nw[0] + (cy - pp[1]) * nw[1] + (cz - pp[2]) * nw[2];
        delta = ri - dd;
        nx = -nw[0];
        ny = -nw[1];
        nz = -nw[2];
        const double arm = ri - 0.5 * delta;
        px = cx + arm * nx;
        py = cy + arm * ny;
        pz = cz + arm * nz;
        rbar = ri;
        mbar = Mi;
        mj = a.tab.plane_mat[pl];
      }
#if DEM_FORCE_LAZY_OWN
#undef Mi
#endif
      if (degenerate) {
        raise_error(a.ctl, -12, a.s_key[s0 + ls], a.rows.key[e]);
        delta = 0.0;
      }
      double Fx = 0.0, Fy = 0.0, Fz = 0.0, nux = 0.0, nuy = 0.0, nuz = 0.0;
      const double rix = px - ki[0], riy = py - ki[1], riz = pz - ki[2];
      if (delta > 0.0 && active) {
        // contact-point velocities (Eq. 2a); a mesh point moves with its mesh
        double vix, viy, viz, vjx = 0.0, vjy = 0.0, vjz = 0.0;
        point_velocity(ki[3], ki[4], ki[5], ki[6], ki[7], ki[8], rix, riy, riz, vix, viy, viz);
        if (!wall || mesh >= 0)
          point_velocity(Vjx, Vjy, Vjz, Wjx, Wjy, Wjz, px - Xjx, py - Xjy, pz - Xjz, vjx, vjy, vjz);
        const double vrx = vjx - vix, vry = vjy - viy, vrz = vjz - viz;
        // pair table (system.cu): 2E*, 8G*, 2 sqrt(5/6) beta, mu, sqrt(k_t / S_n) = sqrt(4G*/E*)
        const double* pr = a.tab.pair + kPairStride * (own_mat[ls] * a.tab.n_mat + mj);
        const double e2 = pr[0], g8 = pr[1], kb = pr[2], mu = pr[3], rt = pr[4];
        // (a6) normal force, Eq. 1a
        const double sq = sqrt(rbar * delta);
        const double Sn = e2 * sq;
        const double kn = (2.0 / 3.0) * Sn;
        const double cn = kb * sqrt(Sn * mbar);
        const double vn = vrx * nx + vry * ny + vrz * nz;
        const double fns = kn * delta - cn * vn;
        const double fnx = fns * nx, fny = fns * ny, fnz = fns * nz;
        double ftx = 0.0, fty = 0.0, ftz = 0.0;
        if (mu != 0.0) {
          // (a7) Eq. 3a-3b, Eq. 1b, Eq. 3c
          const double vtx = vrx - vn * nx, vty = vry - vn * ny, vtz = vrz - vn * nz;
#if DEM_FORCE_UT_ASYNC
          asm volatile("cp.async.wait_all;" ::: "memory");
          const double ux = pidx >= 0 ? part[0][pslot(tid)] : 0.0, uy = pidx >= 0 ? part[1][pslot(tid)] : 0.0,
                       uz = pidx >= 0 ? part[2][pslot(tid)] : 0.0;
#endif
          const double upx = ux + h * vtx, upy = uy + h * vty, upz = uz + h * vtz;
          const double upn = upx * nx + upy * ny + upz * nz;
          const double utx = upx - upn * nx, uty = upy - upn * ny, utz = upz - upn * nz;
          const double kt = g8 * sq;
          const double ct = cn * rt;  // 2 sqrt(5/6) beta sqrt(k_t m) = c_n sqrt(k_t / S_n)
          const double trx = -kt * utx - ct * vtx, try_ = -kt * uty - ct * vty, trz = -kt * utz - ct * vtz;
          const double cap = mu * fabs(fns);  // mu |F_n| (n is a unit vector)
          // |F_t trial| <= mu |F_n|, compared squared
          if (trx * trx + try_ * try_ + trz * trz <= cap * cap) {
            ftx = trx; fty = try_; ftz = trz;
            nux = utx; nuy = uty; nuz = utz;
          } else {
            const double um = sqrt(utx * utx + uty * uty + utz * utz);
            if (um > 0.0) {
              const double iu = 1.0 / um;
              const double dxu = utx * iu, dyu = uty * iu, dzu = utz * iu;
              const double s = cap / kt;
              nux = s * dxu; nuy = s * dyu; nuz = s * dzu;
              ftx = -cap * dxu; fty = -cap * dyu; ftz = -cap * dzu;
            }
          }
        }
        Fx = fnx + ftx;
        Fy = fny + fty;
        Fz = fnz + ftz;
      }
      {
#if DEM_UT_PAD
        stg256(a.rows.ut + (size_t)kUt * e, nux, nuy, nuz, 0.0);
#else
        double* u = a.rows.ut + (size_t)kUt * e;
        u[0] = nux;
        u[1] = nuy;
        u[2] = nuz;
#endif
      }
      if (a.record) {
        a.rec.F[3 * e] = Fx; a.rec.F[3 * e + 1] = Fy; a.rec.F[3 * e + 2] = Fz;
        a.rec.p[3 * e] = px; a.rec.p[3 * e + 1] = py; a.rec.p[3 * e + 2] = pz;
        a.rec.n[3 * e] = nx; a.rec.n[3 * e + 1] = ny; a.rec.n[3 * e + 2] = nz;
        a.rec.delta[e] = delta;
      }
      // force on own sphere is -F, torque r_i x (-F) (Eq. 4, reading R11)
      const double fx = -Fx, fy = -Fy, fz = -Fz;
#if DEM_FORCE_UT_ASYNC
      asm volatile("cp.async.wait_all;" ::: "memory");  // (the u_t copy into these slots has landed)
#endif
      part[0][pslot(tid)] = fx;
      part[1][pslot(tid)] = fy;
      part[2][pslot(tid)] = fz;
      part[3][pslot(tid)] = __fma_rn(riy, fz, -__dmul_rn(riz, fy));
      part[4][pslot(tid)] = __fma_rn(riz, fx, -__dmul_rn(rix, fz));
      part[5][pslot(tid)] = __fma_rn(rix, fy, -__dmul_rn(riy, fx));
      if (kMesh && mesh >= 0) {
        // reaction on the mesh: +F at p, torque (p - X_m) x F
        const double mx = px - Xjx, my = py - Xjy, mz = pz - Xjz;
        emesh[tid] = mesh;
        chunk_mesh = 1;  // (a benign race: every writer stores 1)
        mtq[0][tid] = my * Fz - mz * Fy;
        mtq[1][tid] = mz * Fx - mx * Fz;
        mtq[2][tid] = mx * Fy - my * Fx;
      }
    }
    __syncthreads();
    // only thread 0 reads or clears chunk_mesh between the barriers (the other threads set it
    // before the barrier above and next after the barrier below)
    if (kMesh && tid == 0 && *(volatile int*)&chunk_mesh) {
      // the CTA's mesh wrench, entries in row order (deterministic), beside the per-sphere sums
      // of the other threads (both only read part[] until the next barrier)
      cta_mesh = 1;
      chunk_mesh = 0;
      for (int q = 0; q < kFT; ++q) {
        const int m = emesh[q];
        if (m < 0) continue;
        cw[m][0] -= part[0][pslot(q)]; cw[m][1] -= part[1][pslot(q)]; cw[m][2] -= part[2][pslot(q)];
        cw[m][3] += mtq[0][q]; cw[m][4] += mtq[1][q]; cw[m][5] += mtq[2][q];
      }
    }
    // (a9, first level) canonical per-sphere sums: entries in row (partner-key) order; then the
    // owners of this sphere's entries in the next chunk
    for (int ls = tid; ls < nsph; ls += kFT) {
      const int r0 = rp[ls], r1 = rp[ls + 1];
      const int b = max(r0, c0e), en = min(r1, c0e + kFT);
      if (b < en) {
        // the running sums in registers across the sphere's entries of this chunk (same order)
        double sum[6];
#pragma unroll
        for (int d = 0; d < 6; ++d) sum[d] = acc[d][ls];
        for (int q = b - c0e; q < en - c0e; ++q) {
#pragma unroll
          for (int d = 0; d < 6; ++d) sum[d] += part[d][pslot(q)];
        }
#pragma unroll
        for (int d = 0; d < 6; ++d) acc[d][ls] = sum[d];
      }
      const int nb = c0e + kFT;
      if (DEM_FORCE_OWNER)
        for (int q = max(r0, nb); q < min(r1, nb + kFT); ++q) own_of[q - nb] = (unsigned char)ls;
    }
    __syncthreads();
  }
  if (kMesh) {
    if (cta_mesh && tid < a.n_mesh * 6)
      a.mesh_part[((size_t)blockIdx.x * a.n_mesh + tid / 6) * 6 + tid % 6] = cw[tid / 6][tid % 6];
    if (tid == 0) a.mesh_flag[blockIdx.x] = cta_mesh;
  }
  if (tid >= ncl) return;
  // (a9, second level) + (a10): per clump, spheres in component order.
  // F = sum_k f_k + M g; tau_body = R^T sum_k tau_k; V += h F/M; X += h V;
  // Omega += h I^-1 (tau - Omega x I Omega); q <- normalize(q (x) exp(h Omega)).
  const int c = c0 + tid;
#if DEM_FORCE_ASYNC_EPI
  asm volatile("cp.async.wait_all;" ::: "memory");  // this thread's own cq[.][tid]
  const double I0 = cq[7][tid], I1 = cq[8][tid], I2 = cq[9][tid];
  const double qw = cq[0][tid], qx = cq[1][tid], qy = cq[2][tid], qz = cq[3][tid];
  const double w0 = cq[4][tid], w1 = cq[5][tid], w2 = cq[6][tid];
#else
  const int tt = DEM_KIN_TID ? (int)__double_as_longlong(ck[kKinUsed * tid + 10]) : a.tid[c];
  const double I0 = a.tab.tpl_inertia[3 * tt], I1 = a.tab.tpl_inertia[3 * tt + 1], I2 = a.tab.tpl_inertia[3 * tt + 2];
  const double qw = a.cur.qw[c], qx = a.cur.qx[c], qy = a.cur.qy[c], qz = a.cur.qz[c];
  const double w0 = a.cur.wx[c], w1 = a.cur.wy[c], w2 = a.cur.wz[c];
#endif
  const double* kc = ck + kKinUsed * tid;  // this clump's X, V, omega_world, M
  const double M = kc[9];
  double Fx = 0.0, Fy = 0.0, Fz = 0.0, Tx = 0.0, Ty = 0.0, Tz = 0.0;
  for (int s = a.sph_off[c] - s0, e = a.sph_off[c + 1] - s0; s < e; ++s) {
    Fx += acc[0][s]; Fy += acc[1][s]; Fz += acc[2][s];
    Tx += acc[3][s]; Ty += acc[4][s]; Tz += acc[5][s];
  }
  Fx = __dadd_rn(Fx, __dmul_rn(M, a.g[0]));
  Fy = __dadd_rn(Fy, __dmul_rn(M, a.g[1]));
  Fz = __dadd_rn(Fz, __dmul_rn(M, a.g[2]));
  double R[9];
  quat_R(qw, qx, qy, qz, R);
  const double tbx = R[0] * Tx + R[3] * Ty + R[6] * Tz;
  const double tby = R[1] * Tx + R[4] * Ty + R[7] * Tz;
  const double tbz = R[2] * Tx + R[5] * Ty + R[8] * Tz;
  if (!isfinite(Fx) || !isfinite(Fy) || !isfinite(Fz) || !isfinite(tbx) || !isfinite(tby) || !isfinite(tbz)) {
    raise_error(a.ctl, -11, a.gid[c], 0);
  }
  const double vx = kc[3] + h * (Fx / M), vy = kc[4] + h * (Fy / M), vz = kc[5] + h * (Fz / M);
  a.nxt.vx[c] = vx; a.nxt.vy[c] = vy; a.nxt.vz[c] = vz;
  const double nxx = kc[0] + h * vx, nxy = kc[1] + h * vy, nxz = kc[2] + h * vz;
  a.nxt.x[c] = nxx;
  a.nxt.y[c] = nxy;
  a.nxt.z[c] = nxz;
  if (a.drift_max > 0.0) {  // distributed: the ghost bands are only valid within drift_max
    const double dx = nxx - a.xref[3 * c], dy = nxy - a.xref[3 * c + 1], dz = nxz - a.xref[3 * c + 2];
    if (dx * dx + dy * dy + dz * dz > a.drift_max * a.drift_max) raise_error(a.ctl, -15, a.gid[c], 0);
  }
  const double L0 = I0 * w0, L1 = I1 * w1, L2 = I2 * w2;
  const double g0 = w1 * L2 - w2 * L1, g1 = w2 * L0 - w0 * L2, g2 = w0 * L1 - w1 * L0;
  const double n0 = w0 + h * ((tbx - g0) / I0);
  const double n1 = w1 + h * ((tby - g1) / I1);
  const double n2 = w2 + h * ((tbz - g2) / I2);
  a.nxt.wx[c] = n0; a.nxt.wy[c] = n1; a.nxt.wz[c] = n2;
  const double wn = sqrt(n0 * n0 + n1 * n1 + n2 * n2);
  double dw = 1.0, dx = 0.0, dy = 0.0, dz = 0.0;
  if (wn > 0.0) {
    double sh, chh;
    sincos(0.5 * (h * wn), &sh, &chh);
    const double sn = sh / wn;
    dw = chh; dx = n0 * sn; dy = n1 * sn; dz = n2 * sn;
  }
  const double rw = qw * dw - qx * dx - qy * dy - qz * dz;
  const double rx = qw * dx + qx * dw + qy * dz - qz * dy;
  const double ry = qw * dy - qx * dz + qy * dw + qz * dx;
  const double rz = qw * dz + qx * dy - qy * dx + qz * dw;
  const double nrm = sqrt(rw * rw + rx * rx + ry * ry + rz * rz);
  const double q0 = rw / nrm, q1 = rx / nrm, q2 = ry / nrm, q3 = rz / nrm;
  a.nxt.qw[c] = q0; a.nxt.qx[c] = q1; a.nxt.qy[c] = q2; a.nxt.qz[c] = q3;
  // fused halo: the new state of a clump the neighbours hold as a ghost goes straight into their
  // next-state arrays (peer stores over NVLink), then a system-scope fence before the signal
  bool sent = false;
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    if (!kPeer || !a.peer_state[side]) continue;
    const int g = a.peer_idx[side][c];
    if (g < 0) continue;
    double* R = a.peer_state[side];
    const long long m = a.peer_n[side];
    const double v[13] = {nxx, nxy, nxz, q0, q1, q2, q3, vx, vy, vz, n0, n1, n2};
#pragma unroll
    for (int k = 0; k < 13; ++k) R[(size_t)k * m + g] = v[k];
    sent = true;
  }
  if (sent) __threadfence_system();
}

// canonical contacts held in a row set: entries whose own sphere key is the smaller one
// (every wall entry, and one of the two directed copies of a sphere pair) — dem_get_stats
__global__ void k_count_canonical(Rows r, const long long* __restrict__ s_key, int ns, unsigned long long* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned c = 0;
  if (i < ns) {
    const long long own = s_key[i];
    for (int e = r.row_ptr[i]; e < r.row_ptr[i + 1]; ++e) c += r.key[e] > own;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

#ifndef DEM_FORCE_CARVEOUT
#define DEM_FORCE_CARVEOUT 0  // 1: largest shared-memory carveout — A/B on C5: force 3.96 -> 4.58 ms (less L1 for the gathers)
#endif
template <bool kMesh, bool kPeer>
static void force_carveout() {
  static bool done = false;
  if (DEM_FORCE_CARVEOUT && !done) {
    cudaFuncSetAttribute(k_force_integrate<kMesh, kPeer>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    done = true;
  }
}

// a system that holds no owned clump (empty, or a rank whose slab is empty) still counts its steps
__global__ void k_step_tick(Ctl* ctl) {
  pdl_wait_and_release();
  if (!ctl->abort) ctl->step += 1;
}
void launch_force_integrate(const StepArgs& a, cudaStream_t s) {
  if (a.n_cta <= 0) {
    launch_k(k_step_tick, 1, 1, s, a.pdl, a.ctl);
    return;
  }
  force_carveout<true, true>();
  force_carveout<true, false>();
  force_carveout<false, true>();
  force_carveout<false, false>();
  const bool peer = a.peer_state[0] || a.peer_state[1];
  if (a.n_tri)
    peer ? launch_k(k_force_integrate<true, true>, a.n_cta, kFT, s, a.pdl, a)
         : launch_k(k_force_integrate<true, false>, a.n_cta, kFT, s, a.pdl, a);
  else
    peer ? launch_k(k_force_integrate<false, true>, a.n_cta, kFT, s, a.pdl, a)
         : launch_k(k_force_integrate<false, false>, a.n_cta, kFT, s, a.pdl, a);
}
void launch_count_canonical(const Rows& r, const long long* s_key, int ns, unsigned long long* out, cudaStream_t s) {
  if (ns) k_count_canonical<<<(ns + 255) / 256, 256, 0, s>>>(r, s_key, ns, out);
}

}  // namespace dem

namespace dem {
// ghost halo pack / unpack (distributed): 13 fp64 per clump, SoA in the buffer
__global__ void k_pack(State st, const int* __restrict__ idx, int n, double* __restrict__ buf) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int c = idx[k];
  const double* f[13] = {st.x, st.y, st.z, st.qw, st.qx, st.qy, st.qz, st.vx, st.vy, st.vz, st.wx, st.wy, st.wz};
#pragma unroll
  for (int q = 0; q < 13; ++q) buf[(size_t)q * n + k] = f[q][c];
}
__global__ void k_unpack(State st, const int* __restrict__ idx, int n, const double* __restrict__ buf) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int c = idx[k];
  double* f[13] = {st.x, st.y, st.z, st.qw, st.qx, st.qy, st.qz, st.vx, st.vy, st.vz, st.wx, st.wy, st.wz};
#pragma unroll
  for (int q = 0; q < 13; ++q) f[q][c] = buf[(size_t)q * n + k];
}
void launch_pack(const State& st, const int* idx, int n, double* buf, cudaStream_t s) {
  if (n) k_pack<<<(n + 255) / 256, 256, 0, s>>>(st, idx, n, buf);
}
void launch_unpack(const State& st, const int* idx, int n, const double* buf, cudaStream_t s) {
  if (n) k_unpack<<<(n + 255) / 256, 256, 0, s>>>(st, idx, n, buf);
}
}  // namespace dem

namespace dem {
// largest squared displacement of an owned COM from its dem_set_state position, as the bits
// of a non-negative double (ordered like unsigned integers) — dem_migrate
__global__ void k_max_drift(State st, const double* __restrict__ xref, int n, unsigned long long* out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  double d2 = 0.0;
  if (c < n) {
    const double dx = st.x[c] - xref[3 * c], dy = st.y[c] - xref[3 * c + 1], dz = st.z[c] - xref[3 * c + 2];
    d2 = dx * dx + dy * dy + dz * dz;
  }
  unsigned long long b = (unsigned long long)__double_as_longlong(d2);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, b, o);
    b = v > b ? v : b;
  }
  if ((threadIdx.x & 31) == 0 && b) atomicMax(out, b);
}
void launch_max_drift(const State& st, const double* xref, int n, unsigned long long* out, cudaStream_t s) {
  if (n) k_max_drift<<<(n + 255) / 256, 256, 0, s>>>(st, xref, n, out);
}
}  // namespace dem

namespace dem {
// State I/O in the caller's order (dem_set_state fast path, dem_get_state): the permutation to
// and from the bin-sorted storage order runs on the device, so the host only moves the caller's
// arrays (AoS rows: pos 3, quat 4, vel 3, omega 3 per clump).
__global__ void k_state_in(State st, const int* __restrict__ perm, int n, const double* __restrict__ pos,
                           const double* __restrict__ quat, const double* __restrict__ vel,
                           const double* __restrict__ om, int* bad, double* xref, int n_own) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = perm[i];
  const double x = pos[3 * c], y = pos[3 * c + 1], z = pos[3 * c + 2];
  if (xref && i < n_own) {  // distributed: the drift reference of the owned clumps
    xref[3 * i] = x; xref[3 * i + 1] = y; xref[3 * i + 2] = z;
  }
  const double vx = vel[3 * c], vy = vel[3 * c + 1], vz = vel[3 * c + 2];
  const double wx = om[3 * c], wy = om[3 * c + 1], wz = om[3 * c + 2];
  if (!isfinite(x) || !isfinite(y) || !isfinite(z) || !isfinite(vx) || !isfinite(vy) || !isfinite(vz) ||
      !isfinite(wx) || !isfinite(wy) || !isfinite(wz))
    atomicExch(bad, 1);
  st.x[i] = x; st.y[i] = y; st.z[i] = z;
  st.qw[i] = quat[4 * c]; st.qx[i] = quat[4 * c + 1]; st.qy[i] = quat[4 * c + 2]; st.qz[i] = quat[4 * c + 3];
  st.vx[i] = vx; st.vy[i] = vy; st.vz[i] = vz;
  st.wx[i] = wx; st.wy[i] = wy; st.wz[i] = wz;
}
__global__ void k_state_out(State st, const int* __restrict__ outpos, int n_own, double* __restrict__ pos,
                            double* __restrict__ quat, double* __restrict__ vel, double* __restrict__ om) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_own) return;
  const int r = outpos[i];
  if (pos) { pos[3 * r] = st.x[i]; pos[3 * r + 1] = st.y[i]; pos[3 * r + 2] = st.z[i]; }
  if (quat) { quat[4 * r] = st.qw[i]; quat[4 * r + 1] = st.qx[i]; quat[4 * r + 2] = st.qy[i]; quat[4 * r + 3] = st.qz[i]; }
  if (vel) { vel[3 * r] = st.vx[i]; vel[3 * r + 1] = st.vy[i]; vel[3 * r + 2] = st.vz[i]; }
  if (om) { om[3 * r] = st.wx[i]; om[3 * r + 1] = st.wy[i]; om[3 * r + 2] = st.wz[i]; }
}
void launch_state_in(const State& st, const int* perm, int n, const double* pos, const double* quat,
                     const double* vel, const double* om, int* bad, double* xref, int n_own, cudaStream_t s) {
  if (n) k_state_in<<<(n + 255) / 256, 256, 0, s>>>(st, perm, n, pos, quat, vel, om, bad, xref, n_own);
}
void launch_state_out(const State& st, const int* outpos, int n_own, double* pos, double* quat, double* vel,
                      double* om, cudaStream_t s) {
  if (n_own) k_state_out<<<(n_own + 255) / 256, 256, 0, s>>>(st, outpos, n_own, pos, quat, vel, om);
}
}  // namespace dem

namespace dem {
// Peer-transport step handshake: after its fused force kernel every rank writes its
// completed-step count into both neighbours' flag words (release, system scope); before its
// next step it waits until both its flag words reach its own count (acquire).  A rank is then
// never more than one step ahead of a neighbour, so it writes a neighbour's next-state ghost
// slots only after that neighbour stopped reading them as its current state, and reads its own
// ghosts only after the neighbours wrote them.  Counts are monotonic (reset by dem_set_state
// before the collective handle exchange), so graph replays need no per-step immediates.
__global__ void k_peer_signal(const Ctl* ctl, int* r0, int* r1) {
  if (ctl->abort) return;
  const int v = (int)ctl->step;
  if (r0) asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(r0), "r"(v) : "memory");
  if (r1) asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(r1), "r"(v) : "memory");
}

__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// one thread spins on the two flag words; gives up after ~20 s (a dead peer) with an error
__global__ void k_peer_wait(Ctl* ctl, const int* f0, const int* f1) {
  if (ctl->abort) return;
  const int want = (int)ctl->step;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    const bool ok = (!f0 || ld_acquire_sys(f0) >= want) && (!f1 || ld_acquire_sys(f1) >= want);
    if (ok) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 20000000000ull) {
      raise_error(ctl, -4, want, 0);  // DEM_ERR_NCCL: a neighbour stopped stepping
      return;
    }
    __nanosleep(200);
  }
}

void launch_peer_signal(const Ctl* ctl, int* r0, int* r1, cudaStream_t s) {
  if (r0 || r1) k_peer_signal<<<1, 1, 0, s>>>(ctl, r0, r1);
}
void launch_peer_wait(Ctl* ctl, const int* f0, const int* f1, cudaStream_t s) {
  if (f0 || f1) k_peer_wait<<<1, 1, 0, s>>>(ctl, f0, f1);
}
}  // namespace dem

namespace dem {
// loopback groups: the ranks' abort words OR-ed together before their force kernels (the
// in-process counterpart of the distributed abort all-reduce, system.cu enqueue_abort_vote)
__global__ void k_abort_or(AbortWords w) {
  int any = 0;
  for (int r = 0; r < w.n; ++r) any |= *w.p[r];
  if (any)
    for (int r = 0; r < w.n; ++r) *w.p[r] = 1;
}
void launch_abort_or(const AbortWords& w, cudaStream_t s) {
  if (w.n > 1) k_abort_or<<<1, 1, 0, s>>>(w);
}
}  // namespace dem

namespace dem {
// bounding box of the sphere centres (re-grid, system.cu): ordered 64-bit keys of the doubles
__device__ __forceinline__ unsigned long long ord_key(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__global__ void k_bbox(const double4* __restrict__ spos, int ns, unsigned long long* box) {
  unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0ull, 0ull, 0ull};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += gridDim.x * blockDim.x) {
    const double4 p = spos[i];
    const unsigned long long k[3] = {ord_key(p.x - p.w), ord_key(p.y - p.w), ord_key(p.z - p.w)};
    const unsigned long long K[3] = {ord_key(p.x + p.w), ord_key(p.y + p.w), ord_key(p.z + p.w)};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      lo[d] = min(lo[d], k[d]);
      hi[d] = max(hi[d], K[d]);
    }
  }
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    for (int o = 16; o > 0; o >>= 1) {
      lo[d] = min(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
      hi[d] = max(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&box[d], lo[d]);
      atomicMax(&box[3 + d], hi[d]);
    }
  }
}
void launch_bbox(const double4* spos, int ns, unsigned long long* box, cudaStream_t s) {
  if (ns) k_bbox<<<148 * 4, 256, 0, s>>>(spos, ns, box);
}
}  // namespace dem

