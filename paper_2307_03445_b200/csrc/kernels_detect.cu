// kernels_detect.cu — (a1) sphere poses, (a2) multi-insert binning, (a3) narrow phase + rows.
//
// PAPER.md:142 ("identifying the active set represents a significant computational
// bottleneck"), P:145 (per-step rebuild), P:69 (binning CD following hammadTobyDan2012:
// every body is inserted into each bin its AABB overlaps, pairs are tested per bin).
// Readings: DESIGN.md §3 R14 (predicate d.d <= (r_a + r_b + margin)^2 in fp64, no FMA),
// R15 (no intra-clump pairs), R22 (sphere centre c = X + R(q) o, explicit roundings).
//
// Pipeline of one rebuild:
//   k_pose_count    per sphere: centre, (x,y,z,r) record, wall candidates -> row_cnt,
//                   bin counts; component 0 packs the clump kinematics record
//   scan            bin offsets
//   k_bin_scatter   per sphere: bin item lists (slots by decrementing the counts)
//   k_pairs         one warp per bin: members staged in shared memory ordered by which of
//                   the bin's faces are their lowest; only the pairs whose lowest common bin
//                   is this one (so each pair is found exactly once grid-wide) enumerated
//                   flat over the lanes and tested; hits compacted with warp ballots
//                   into a per-warp shared buffer; at a flush every pair takes a slot in both
//                   spheres' rows (counting atomics) and is written into the fixed-width
//                   candidate lists (slots) of both
//   scan            row offsets (CSR)
//   k_rows_finish   per sphere: wall entries + its candidate list, sorted by partner key,
//                   written to its CSR row, merged with its previous row (history index)
#include "dem_device.cuh"

namespace dem {

// ---------------------------------------------------------------- (a1) + bin count
// threads per CTA of the per-sphere kernels (A/B on the C5 bench: 64 beats 128 by 0.5%, 256 by
// 2.5%, 512 by 17% — smaller CTAs keep more warps resident at these register counts)
#ifndef DEM_POSE_TPB
#define DEM_POSE_TPB 64
#endif
#ifndef DEM_SCATTER_TPB
#define DEM_SCATTER_TPB 64
#endif
// CTAs per SM for the register budget (A/B on the C5 bench: pose 24 -> 40 registers, 1.15 vs
// 1.20 ms at 48 and 1.38 at 32 with spills; scatter 32 -> 32 registers, 1.00 vs 1.10 ms)
#ifndef DEM_POSE_MINB
#define DEM_POSE_MINB 24
#endif
#ifndef DEM_SCATTER_MINB
#define DEM_SCATTER_MINB 32
#endif
#define DEM_POSE_LB DEM_POSE_TPB, DEM_POSE_MINB
#define DEM_SCATTER_LB DEM_SCATTER_TPB, DEM_SCATTER_MINB
#ifndef DEM_ROWS_TPB
#define DEM_ROWS_TPB 128  // A/B: 1.58 ms vs 1.69 in 64-thread CTAs (same 32 registers)
#endif
// one sphere of clump c: centre, record, domain and displacement checks, and on detection
// steps its plane candidates, row count and bin counts
__device__ __forceinline__ void pose_sphere(const StepArgs& a, int i, int c, int tc, const double* R, double X,
                                            double Y, double Z) {
  const double ox = a.tab.tc_off[3 * tc], oy = a.tab.tc_off[3 * tc + 1], oz = a.tab.tc_off[3 * tc + 2];
  const double cx = add(X, row_dot(R, ox, oy, oz));
  const double cy = add(Y, row_dot(R + 3, ox, oy, oz));
  const double cz = add(Z, row_dot(R + 6, ox, oy, oz));
  const double r = a.tab.tc_rad[tc];
  a.spos[i] = make_double4(cx, cy, cz, r);
  const Grid& g = a.grid;
  if (!(cx >= g.dom_lo[0] && cx <= g.dom_hi[0] && cy >= g.dom_lo[1] && cy <= g.dom_hi[1] &&
        cz >= g.dom_lo[2] && cz <= g.dom_hi[2])) {
    raise_error(a.ctl, -10, a.s_key[i], a.gid[c]);
    return;
  }
  if (a.ref_in) {
    // the deferred set stays complete while no sphere has moved more than margin/2 since it
    // was built ("v_max violated"): otherwise report it instead of missing contacts
    const double4 q = a.ref_in[i];
    const double dx = cx - q.x, dy = cy - q.y, dz = cz - q.z;
    if (dx * dx + dy * dy + dz * dz > a.half_margin * a.half_margin) raise_error(a.ctl, -13, a.s_key[i], a.gid[c]);
  }
  if (!a.count) return;
  if (cx < g.reg_lo[0] || cx > g.reg_hi[0] || cy < g.reg_lo[1] || cy > g.reg_hi[1] || cz < g.reg_lo[2] ||
      cz > g.reg_hi[2])
    a.ctl->need_regrid = 1;  // clamped into an edge bin (exact, but slow if many): re-grid soon
  if (a.ref_out) a.ref_out[i] = make_double4(cx, cy, cz, r);
  // sphere-plane candidates: (r + margin) - (c - p_w).n_w >= 0
  unsigned wmask = 0;
  for (int p = 0; p < a.tab.n_planes; ++p) {
    const double* pp = a.tab.plane_pt[p];
    const double* nw = a.tab.plane_n[p];
    const double dd = add(add(mul(sub(cx, pp[0]), nw[0]), mul(sub(cy, pp[1]), nw[1])), mul(sub(cz, pp[2]), nw[2]));
    if (sub(add(r, a.margin), dd) >= 0.0) wmask |= 1u << p;
  }
  // ghosts get no rows (their owners evaluate them); the mask goes to k_rows_finish
  a.row_cnt[i] = i < a.ns_own ? __popc(wmask) : 0;
  a.wall_mask[i] = (unsigned short)wmask;
  int lx, hx, ly, hy, lz, hz;
  cell_range(g, 0, cx, r, lx, hx);
  cell_range(g, 1, cy, r, ly, hy);
  cell_range(g, 2, cz, r, lz, hz);
#if DEM_SCATTER_RANKS
  const int nins = (hx - lx + 1) * (hy - ly + 1) * (hz - lz + 1);
  if (nins <= kRankW) {
    // the old count is this insert's rank among the bin's small-sphere inserts: kept for the scatter
    int k = 0;
    for (int z = lz; z <= hz; ++z)
      for (int y = ly; y <= hy; ++y) {
        const long long base = z * g.st[2] + y * g.st[1];
        for (int x = lx; x <= hx; ++x, ++k) {
          const int old = atomicAdd(&a.cell_count[base + x * g.st[0]], 1);
          if ((old & 0xffff) == 0xffff) raise_error(a.ctl, -14, a.s_key[i], 0);  // 65535 in one bin: bins too coarse
          a.irank[(size_t)k * a.ns + i] = (unsigned short)(old & 0xffff);
        }
      }
    return;
  }
  for (int z = lz; z <= hz; ++z)
    for (int y = ly; y <= hy; ++y) {
      const long long base = z * g.st[2] + y * g.st[1];
      for (int x = lx; x <= hx; ++x) atomicAdd(&a.cell_count[base + x * g.st[0]], 0x10000);
    }
#else
  for (int z = lz; z <= hz; ++z)
    for (int y = ly; y <= hy; ++y) {
      const long long base = z * g.st[2] + y * g.st[1];
      for (int x = lx; x <= hx; ++x) atomicAdd(&a.cell_count[base + x * g.st[0]], 1);
    }
#endif
}

__device__ __forceinline__ void kin_record(const StepArgs& a, int c, const double* R, double X, double Y, double Z) {
  const double wx = a.cur.wx[c], wy = a.cur.wy[c], wz = a.cur.wz[c];
  double* k = a.kin + (size_t)kKin * c;
  const double w0 = R[0] * wx + R[1] * wy + R[2] * wz;
  const double w1 = R[3] * wx + R[4] * wy + R[5] * wz;
  const double w2 = R[6] * wx + R[7] * wy + R[8] * wz;
#ifndef DEM_KIN_ST256
#define DEM_KIN_ST256 DEM_V256
#endif
#if DEM_KIN_ST256
  stg256(k, X, Y, Z, a.cur.vx[c]);
  stg256(k + 4, a.cur.vy[c], a.cur.vz[c], w0, w1);
  const int t = a.tid[c];
  stg256(k + 8, w2, a.tab.tpl_mass[t], __longlong_as_double((long long)t), 0.0);
#else
  k[0] = X; k[1] = Y; k[2] = Z;
  k[3] = a.cur.vx[c]; k[4] = a.cur.vy[c]; k[5] = a.cur.vz[c];
  k[6] = w0;
  k[7] = w1;
  k[8] = w2;
  k[9] = a.tab.tpl_mass[a.tid[c]];
#endif
}

__device__ __forceinline__ bool pose_prologue(const StepArgs& a) {
  if (a.adopt && blockIdx.x == 0 && threadIdx.x == 0 && a.ctl->det_abort) {
    // the set detected ahead overflowed a capacity: abort this adoption step, the host regrows
    // and rebuilds the set at this step instead (same trajectory: DESIGN.md §5.2)
    atomicExch(&a.ctl->abort, 1);
  }
  return !a.ctl->abort;
}

#ifndef DEM_POSE_PER_CLUMP
#define DEM_POSE_PER_CLUMP 0
#endif
#if DEM_POSE_PER_CLUMP
// one thread per clump: R(q) once for all its spheres
__global__ void __launch_bounds__(DEM_POSE_LB) k_pose_count(StepArgs a) {
  if (!pose_prologue(a)) return;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.n) return;
  double R[9];
  quat_R(a.cur.qw[c], a.cur.qx[c], a.cur.qy[c], a.cur.qz[c], R);
  const double X = a.cur.x[c], Y = a.cur.y[c], Z = a.cur.z[c];
  kin_record(a, c, R, X, Y, Z);
  for (int i = a.sph_off[c], e = a.sph_off[c + 1]; i < e; ++i) pose_sphere(a, i, c, a.s_tc[i], R, X, Y, Z);
}
void launch_pose_count(const StepArgs& a, cudaStream_t s) {
  k_pose_count<<<a.n ? (a.n + DEM_POSE_TPB - 1) / DEM_POSE_TPB : 1, DEM_POSE_TPB, 0, s>>>(a);
}
#else
__global__ void __launch_bounds__(DEM_POSE_LB) k_pose_count(StepArgs a) {
  if (!pose_prologue(a)) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.ns) return;
  const int c = a.s_clump[i];
  const int tc = a.s_tc[i];
  double R[9];
  quat_R(a.cur.qw[c], a.cur.qx[c], a.cur.qy[c], a.cur.qz[c], R);
  const double X = a.cur.x[c], Y = a.cur.y[c], Z = a.cur.z[c];
  if (tc == a.tab.tpl_coff[a.tid[c]]) kin_record(a, c, R, X, Y, Z);
  pose_sphere(a, i, c, tc, R, X, Y, Z);
}
void launch_pose_count(const StepArgs& a, cudaStream_t s) {
  k_pose_count<<<a.ns ? (a.ns + DEM_POSE_TPB - 1) / DEM_POSE_TPB : 1, DEM_POSE_TPB, 0, s>>>(a);
}
#endif

// ---------------------------------------------------------------- bin scatter
// Slots are taken by decrementing the counts, which leaves cell_count all-zero for the
// next step.  The order inside a bin is irrelevant: rows are sorted by partner key.
__global__ void __launch_bounds__(DEM_SCATTER_LB) k_bin_scatter(StepArgs a) {
  pdl_wait_and_release();
  if (*a.abort || a.ctl->abort) return;  // (an error in the steps running beside an ahead detection)
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.ns) return;
  const bool fits = (long long)a.cell_start[a.ncell] <= a.cap_inserts;
  const double4 s = a.dpos[i];
  const Grid& g = a.grid;
  int lx, hx, ly, hy, lz, hz;
  cell_range(g, 0, s.x, s.w, lx, hx);
  cell_range(g, 1, s.y, s.w, ly, hy);
  cell_range(g, 2, s.z, s.w, lz, hz);
#if DEM_SCATTER_RANKS
  const bool small = (hx - lx + 1) * (hy - ly + 1) * (hz - lz + 1) <= kRankW;
  int k = 0;
#endif
  for (int z = lz; z <= hz; ++z)
    for (int y = ly; y <= hy; ++y) {
      const long long base = z * g.st[2] + y * g.st[1];
      for (int x = lx; x <= hx; ++x) {
        const long long cid = base + x * g.st[0];
        const int start = a.cell_start[cid];  // issued before the atomic: the two are independent
#if DEM_SCATTER_RANKS
        // small spheres: the rank from the counting pass; large ones after all small ones of the bin
        int slot;
        if (small) {
          slot = a.irank[(size_t)(k++) * a.ns + i];
        } else {
          const unsigned old = (unsigned)atomicSub(&a.cell_count[cid], 0x10000);
          slot = (int)((old & 0xffffu) + (old >> 16)) - 1;
        }
#else
        const int slot = atomicSub(&a.cell_count[cid], 1) - 1;
#endif
        // the item carries the sphere's lowest-bin mask for k_pairs (ns < 2^29, checked)
        if (fits) a.items[start + slot] = i | (((x == lx ? 1 : 0) | (y == ly ? 2 : 0) | (z == lz ? 4 : 0)) << 29);
      }
    }
}

// ---------------------------------------------------------------- (a3) per-bin pair tests
// tuning knobs (build-time; see build.py -D): buffered pairs per warp, min CTAs/SM for the
// register budget, bins per CTA run
#ifndef DEM_PAIRS_BUF
#define DEM_PAIRS_BUF 32  // A/B: 32 beats 64 by 4% (96, 128 much slower)
#endif
#ifndef DEM_PAIRS_MINB
#define DEM_PAIRS_MINB 7  // ptxas stays at 64 registers; A/B round 2 vs 8: pairs 4.49 -> 4.43 ms on C5, C3 -1.4% (6: 4.61)
#endif
#ifndef DEM_PAIRS_ADAPT
#define DEM_PAIRS_ADAPT 1  // span length from the grid size (launch_pairs) instead of DEM_PAIRS_CONTIG
#endif
#ifndef DEM_PAIRS_SPANS_PER_SLOT
#define DEM_PAIRS_SPANS_PER_SLOT 4
#endif
#ifndef DEM_PAIRS_CONTIG
#define DEM_PAIRS_CONTIG 64  // bins per warp in a CTA span
#endif
#ifndef DEM_PAIRS_WARPS
#define DEM_PAIRS_WARPS 4  // A/B (pipelined loop): 4.63 ms vs 4.71 at 8 warps, 4.78 at 16
#endif
constexpr int kPairWarps = DEM_PAIRS_WARPS;
constexpr int kPairBuf = DEM_PAIRS_BUF;

// Members of a bin, staged in the warp's shared memory.  Both spheres of a pair overlap the
// bin C, so their lowest bins satisfy lo <= C on every axis, and max(lo_a, lo_b) == C  <=>
// on every axis lo_a == C or lo_b == C.  With g = the 3-bit mask "C is my lowest bin along
// axis d", the pair belongs to C iff (g_a | g_b) == 7: that is how each pair is found in
// exactly one bin.
constexpr int kFlatMax = 64;  // bins up to this size: member groups + flat pair enumeration
#ifndef DEM_PAIRS_TINY
#define DEM_PAIRS_TINY 1
#endif
constexpr int kTiny = 8;      // bins up to this size: every pair in one pass with the per-pair group test
#ifndef DEM_PAIRS_SMALL_DENSE
#define DEM_PAIRS_SMALL_DENSE 0   // the same per-pair pass in the dense instantiation, bins up to this size (<= 32)
#endif
constexpr int kSmallDense = DEM_PAIRS_SMALL_DENSE;
static_assert(kSmallDense <= 32, "the small-bin pass loads one member per lane");
#ifndef DEM_PAIRS_SOA
#define DEM_PAIRS_SOA 1
#endif
#ifndef DEM_PAIRS_SPLIT
#define DEM_PAIRS_SPLIT 1
#endif
#ifndef DEM_PAIRS_PIPE
#define DEM_PAIRS_PIPE 1
#endif
struct Members {
#if DEM_PAIRS_SOA
  // x, y | z, r in two 16-byte arrays: consecutive members hit consecutive bank quads (a
  // 32-byte double4 stride makes the 128-bit loads of 8 consecutive members conflict 2-way)
  double2 xy[kFlatMax], zr[kFlatMax];
  __device__ __forceinline__ double4 get(int q) const {
    const double2 u = xy[q], v = zr[q];
    return make_double4(u.x, u.y, v.x, v.y);
  }
  __device__ __forceinline__ void put(int q, const double4& p) {
    xy[q] = make_double2(p.x, p.y);
    zr[q] = make_double2(p.z, p.w);
  }
#else
  double4 p[kFlatMax];  // x, y, z, r
  __device__ __forceinline__ double4 get(int q) const { return p[q]; }
  __device__ __forceinline__ void put(int q, const double4& v) { p[q] = v; }
#endif
#if DEM_PAIRS_SPLIT
  // clump and item apart: the pair test reads the clumps only, a hit its two items
  int clump[kFlatMax], item[kFlatMax];
  __device__ __forceinline__ int2 meta_get(int q) const { return make_int2(clump[q], item[q]); }
  __device__ __forceinline__ void meta_put(int q, int2 v) {
    clump[q] = v.x;
    item[q] = v.y;
  }
#else
  int2 meta[kFlatMax];  // (clump, sphere index [| g << 29 on the large-bin path])
  __device__ __forceinline__ int2 meta_get(int q) const { return meta[q]; }
  __device__ __forceinline__ void meta_put(int q, int2 v) { meta[q] = v; }
#endif
};

__device__ __forceinline__ void load_member(const StepArgs& a, Members& M, int slot, int item) {
  const int it = a.items[item];
  const int idx = it & 0x1fffffff;
  M.put(slot, ldg256(a.dpos + idx));
  M.meta_put(slot, make_int2(a.s_clump[idx], it));
}

// Member order of the flat path: groups by g in the order 7, 6, 1, 5, 3, 2, 4, 0 (nibble g of
// kGroupPos is the position of group g).  The pairs with (g_a | g_b) == 7 are then the five
// blocks  T: group 7 with itself;  R0: group 7 x every later member;  R1: group 6 x groups
// {1, 5, 3};  R2: group 5 x groups {3, 2};  R3: group 3 x group 4 — each a triangle or a
// rectangle of the member order, enumerated without testing any other pair.
constexpr unsigned kGroupPos = 0x01364527u;

__device__ __forceinline__ unsigned long long warp_incl_scan64(unsigned long long x, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += t;
  }
  return x;
}

__device__ __forceinline__ int byte_of(unsigned long long v, int k) { return (int)((v >> (8 * k)) & 0xffu); }

// p -> (i, j), 0 <= i < j, p = j (j - 1) / 2 + i
__device__ __forceinline__ void decode_tri(int p, int& i, int& j) {
  int jj = (int)((1.0f + sqrtf(1.0f + 8.0f * (float)p)) * 0.5f);
  while (jj * (jj - 1) / 2 > p) --jj;
  while ((jj + 1) * jj / 2 <= p) ++jj;
  j = jj;
  i = p - jj * (jj - 1) / 2;
}

// one directed candidate: partner t in slot `slot` of own's row (slot -1: own is a ghost,
// evaluated by its owner); a slot beyond the row width asks the host for wider rows
__device__ __noinline__ void slot_overflow(Ctl* ctl, int* abort, int slot) {
  atomicMax(&ctl->need_width, (long long)slot + 1);
  atomicExch(abort, 1);
}

// what a flush needs of the step arguments
struct FlushCtx {
  int* row_cnt;
  int* slots;
  long long* slot_key;
  const long long* s_key;
  const double4* dpos;
  Ctl* ctl;
  int* abort;
  double margin;
  int ns_own, row_width;
  __device__ __forceinline__ FlushCtx(const StepArgs& a)
      : row_cnt(a.row_cnt), slots(a.slots), slot_key(a.slot_key), s_key(a.s_key), dpos(a.dpos), ctl(a.ctl),
        abort(a.abort), margin(a.margin), ns_own(a.ns_own), row_width(a.row_width) {}
};

__device__ __forceinline__ void put_slot(const FlushCtx& a, int own, int slot, int t, long long tkey) {
  if (slot < 0) return;
  if (slot < a.row_width) {
    a.slots[(size_t)slot * a.ns_own + own] = t;  // slot-major: k_rows_finish reads coalesced
    if (DEM_SLOT_KEYS) a.slot_key[(size_t)slot * a.ns_own + own] = tkey;
  } else {
    slot_overflow(a.ctl, a.abort, slot);  // cold path, kept out of the loop's registers
  }
}

// Flush a warp's buffered pairs: the per-row counting atomics that hand out each entry's
// slot in its row (walls come first), 2 x kPairBuf/32 independent ones per lane so their
// latency overlaps, then both directed candidates written into the spheres' slot lists.
template <bool kMargin>
__device__ __forceinline__ void flush_pairs(const FlushCtx a, const int2* bf, int n, int lane) {
  __syncwarp();
  if (n == 0) return;
  constexpr int kPer = kPairBuf / 32;
  int2 v[kPer];
  int sa[kPer], sb[kPer];
  long long ka[kPer], kb[kPer];
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int k = lane + 32 * j;
    if (k < n) {
      v[j] = bf[k];
      sa[j] = v[j].x < a.ns_own ? atomicAdd(&a.row_cnt[v[j].x], 1) : -1;  // -1: ghost, no row
      sb[j] = v[j].y < a.ns_own ? atomicAdd(&a.row_cnt[v[j].y], 1) : -1;
      if (DEM_SLOT_KEYS) {  // the partners' keys, gathered here beside the atomics' latency
        ka[j] = __ldg(a.s_key + v[j].x);
        kb[j] = __ldg(a.s_key + v[j].y);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    if (lane + 32 * j < n) {
      put_slot(a, v[j].x, sa[j], v[j].y, DEM_SLOT_KEYS ? kb[j] : 0);
      put_slot(a, v[j].y, sb[j], v[j].x, DEM_SLOT_KEYS ? ka[j] : 0);
    }
  }
  __syncwarp();
}

// a warp's hits of one pass: compacted with a ballot into the warp's buffer (flushed when full)
template <bool kMargin>
__device__ __forceinline__ void push_hits(const StepArgs& a, int2* bf, int& nbuf, bool hit, int ia, int ib,
                                          int lane) {
  const unsigned mask = __ballot_sync(0xffffffffu, hit);
  if (mask) {
    const int cnt = __popc(mask);
    if (nbuf + cnt > kPairBuf) {
      flush_pairs<kMargin>(FlushCtx(a), bf, nbuf, lane);
      nbuf = 0;
    }
    if (hit) bf[nbuf + __popc(mask & ((1u << lane) - 1u))] = make_int2(ia, ib);
    nbuf += cnt;
  }
}

// candidate predicate (R14): different clumps, at least one owned (ghost-ghost
// pairs belong to other ranks), |d|^2 <= (r_a + r_b + margin)^2 with explicit roundings
template <bool kGhosts, bool kMargin>
__device__ __forceinline__ bool candidate(const StepArgs& a, const int2& mi, const int2& mj, const double4& pi,
                                          const double4& pj) {
  const double dx = sub(pj.x, pi.x), dy = sub(pj.y, pi.y), dz = sub(pj.z, pi.z);
  const double d2 = add(add(mul(dx, dx), mul(dy, dy)), mul(dz, dz));
  // (r_a + r_b) + 0 is r_a + r_b exactly: the margin add is skipped when there is none
  const double s = kMargin ? add(add(pi.w, pj.w), a.margin) : add(pi.w, pj.w);
  // ghost-ghost pairs belong to other ranks (only a distributed system holds ghosts)
  // (bitwise &: the pair arithmetic runs unconditionally, no branch around it)
  return (mi.x != mj.x) & (!kGhosts || min(mi.x, mj.x) < a.n_own) & (d2 <= mul(s, s));
}

constexpr int kTri = kFlatMax * (kFlatMax - 1) / 2;
// 1/W for the block widths W <= kFlatMax, correctly rounded (constant-folded divisions)
#define DEM_R8(n) 1.0f / (n), 1.0f / (n + 1), 1.0f / (n + 2), 1.0f / (n + 3), 1.0f / (n + 4), 1.0f / (n + 5), \
                  1.0f / (n + 6), 1.0f / (n + 7)
__constant__ float c_rcp[kFlatMax + 8] = {1.0f,      DEM_R8(1),  DEM_R8(9),  DEM_R8(17), DEM_R8(25),
                                          DEM_R8(33), DEM_R8(41), DEM_R8(49), DEM_R8(57)};
#undef DEM_R8

// one pair of the flat path: the predicate, and the two sphere indices of a hit
#ifndef DEM_PAIRS_NODIV
#define DEM_PAIRS_NODIV 1
#endif
template <bool kGhosts, bool kMargin>
__device__ __forceinline__ bool flat_pair(const StepArgs& a, const Members& A, int i, int j, int& ia, int& ib,
                                          bool valid = true) {
#if DEM_PAIRS_SPLIT
  const int2 mi = make_int2(A.clump[i], 0), mj = make_int2(A.clump[j], 0);
  const bool hit = valid & candidate<kGhosts, kMargin>(a, mi, mj, A.get(i), A.get(j));
  if (hit) {
    ia = A.item[i];
    ib = A.item[j];
  }
#else
  const int2 mi = A.meta[i], mj = A.meta[j];
  const bool hit = candidate<kGhosts, kMargin>(a, mi, mj, A.get(i), A.get(j));
  ia = mi.y;
  ib = mj.y;
#endif
  return hit;
}

// The pair blocks of a bin's member order (see kGroupPos) from the group sizes `tot` and
// starts `st` (byte k: position k): T (p < tri) from the triangle table, then R0..R3 as
// pair = (A0 + q % W, B0 + q / W) with correctly rounded reciprocals of the block widths
// (q < 64 * 64, so (q + 1/2) / W, at least 1/(2W) away from an integer, truncates right)
struct PairBlocks {
  int tri, e0, e1, e2, total, n7, n4, W1, W2, s1, s3, s4, s5, s6;
  float r0, r1, r2, r3;
  __device__ __forceinline__ PairBlocks(unsigned long long tot, unsigned long long st, int m) {
    n7 = byte_of(tot, 0);
    const int n6 = byte_of(tot, 1), n5 = byte_of(tot, 3), n3 = byte_of(tot, 4);
    n4 = byte_of(tot, 6);
    s6 = byte_of(st, 1); s1 = byte_of(st, 2); s5 = byte_of(st, 3); s3 = byte_of(st, 4);
    const int s2 = byte_of(st, 5);
    s4 = byte_of(st, 6);
    tri = n7 * (n7 - 1) / 2;
    W1 = s2 - s1;
    W2 = s4 - s3;
    e0 = tri + n7 * (m - n7);
    e1 = e0 + n6 * W1;
    e2 = e1 + n5 * W2;
    total = e2 + n3 * n4;
    r0 = c_rcp[n7]; r1 = c_rcp[W1]; r2 = c_rcp[W2]; r3 = c_rcp[n4];
  }
  __device__ __forceinline__ void decode(int p, const unsigned short* tri_ij, int& i, int& j) const {
    if (p < tri) {
      const int v = tri_ij[p];
      i = v & 0xff;
      j = v >> 8;
    } else {
      const bool b1 = p >= e0, b2 = p >= e1, b3 = p >= e2;
      const int q = p - (b3 ? e2 : b2 ? e1 : b1 ? e0 : tri);
      const int W = b3 ? n4 : b2 ? W2 : b1 ? W1 : n7;
      const float rw = b3 ? r3 : b2 ? r2 : b1 ? r1 : r0;
      const int A0 = b3 ? s4 : b2 ? s3 : b1 ? s1 : 0;
      const int B0 = b3 ? s3 : b2 ? s5 : b1 ? s6 : n7;
      const int r = __float2int_rz(((float)q + 0.5f) * rw);
      i = A0 + (q - r * W);
      j = B0 + r;
    }
  }
};

// Row descriptors of the flat path (DEM_PAIRS_ROWDEC).  In the member order of kGroupPos every
// member that owns pairs owns ONE contiguous range of partners:  a group-7 member at slot l pairs
// with slots (l, m);  a group-6 member with the groups {1, 5, 3} = slots [s1, s2);  a group-5
// member with {3, 2} = [s3, s4);  a group-3 member with group 4 = [s4, s4 + n4).  Enumerating
// the owners' rows one after another numbers the bin's pairs p = 0 .. total - 1; owner o (the
// o-th member with a non-empty row) starts at off_o, whose bit is set in a per-warp bitmap.  In a
// pass over p = base .. base + 31 (base a multiple of 32: one bitmap word) lane l's owner is
//   o = (starts before base) + popc(word & lanes <= l) - 1,
// and its partner slot is j = lo_o + (p - off_o): one shared word, one popc, one descriptor load
// per pair instead of a block search with float reciprocals.  desc[o] = (lo_o - off_o) << 8 | slot.
#ifndef DEM_PAIRS_ROWDEC
#define DEM_PAIRS_ROWDEC 1
#endif
// group ranks from bit-plane ballots instead of a 64-bit warp scan of one-hot byte counters
#ifndef DEM_PAIRS_BALLOT
#define DEM_PAIRS_BALLOT 0  // A/B on C5: pairs 4.86 ms vs 4.64 with the scan (more instructions, not fewer)
#endif
#if DEM_PAIRS_BALLOT && !DEM_PAIRS_ROWDEC
#error "DEM_PAIRS_BALLOT needs DEM_PAIRS_ROWDEC"
#endif
struct RowDec {
  unsigned bmap[kTri / 32 + 1];
  int desc[kFlatMax];
};

// Row of the member at slot l (group-ordered): partner start lo, count cnt and offset off in the
// bin's pair numbering (closed forms of the sums of the earlier rows).
#ifndef DEM_PAIRS_ROWSEL
#define DEM_PAIRS_ROWSEL 1  // member_row by selects instead of an if-else chain (no divergent branches)
#endif
__device__ __forceinline__ void member_row(int l, int m, int n7, int n6, int n5, int n3, int n4, int s1, int s2,
                                           int s3, int s4, int s5, int e0, int e1, int e2, int& lo, int& cnt,
                                           int& off) {
#if DEM_PAIRS_ROWSEL
  (void)n6; (void)n5;
  const bool c0 = l < n7, c1 = !c0 & (l < s1), c2 = (l >= s5) & (l < s3), c3 = (l >= s3) & (l < s2);
  lo = c0 ? l + 1 : c1 ? s1 : c2 ? s3 : s4;
  cnt = c0 ? m - 1 - l : c1 ? s2 - s1 : c2 ? s4 - s3 : c3 ? n4 : 0;
  const int base = c1 ? e0 : c2 ? e1 : e2, l0 = c1 ? n7 : c2 ? s5 : s3;
  off = c0 ? l * (m - 1) - ((l * (l - 1)) >> 1) : base + (l - l0) * cnt;
  (void)n3;
  return;
#endif
  lo = 0; cnt = 0; off = 0;
  if (l < n7) {
    lo = l + 1;
    cnt = m - 1 - l;
    off = l * (m - 1) - (l * (l - 1) >> 1);
  } else if (l < n7 + n6) {
    lo = s1;
    cnt = s2 - s1;
    off = e0 + (l - n7) * cnt;
  } else if (l >= s5 && l < s5 + n5) {
    lo = s3;
    cnt = s4 - s3;
    off = e1 + (l - s5) * cnt;
  } else if (l >= s3 && l < s3 + n3) {
    lo = s4;
    cnt = n4;
    off = e2 + (l - s3) * cnt;
  }
}

template <bool kGhosts, bool kMargin, bool kTinyOn>
__global__ void __launch_bounds__(kPairWarps * 32, DEM_PAIRS_MINB) k_pairs(StepArgs a) {
  pdl_wait_and_release();
  __shared__ Members smA[kPairWarps];
  __shared__ int2 sbuf[kPairWarps][kPairBuf];
#if DEM_PAIRS_ROWDEC
  __shared__ RowDec smR[kPairWarps];
#else
  __shared__ unsigned short tri_ij[kTri];  // p -> i | j << 8 for p = j (j - 1) / 2 + i, i < j
  for (int p = threadIdx.x; p < kTri; p += blockDim.x) {
    int i, j;
    decode_tri(p, i, j);
    tri_ij[p] = (unsigned short)(i | (j << 8));
  }
  __syncthreads();
#endif
  if (*a.abort || a.ctl->abort) return;  // (an error in the steps running beside an ahead detection)
  if ((long long)a.cell_start[a.ncell] > a.cap_inserts) {
    a.ctl->need_inserts = a.cell_start[a.ncell];
    atomicExch(a.abort, 1);
    return;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  Members& A = smA[w];
  int2* bf = sbuf[w];
  int nbuf = 0;  // warp-uniform
  // Bin iterator: CTAs take spans of kPairWarps x DEM_PAIRS_CONTIG consecutive bins
  // round-robin and their warps interleave inside the span, so concurrent warps work on
  // adjacent bins (shared L1 lines of multiply-inserted spheres) and a warp's buffered pairs
  // — so the slot writes that follow — stay spatially local.
  // (32-bit bin ids: ncell + the overshoot of the last spans < 2^31, checked by grid_layout)
  using bin_t = int;
  // (bins per warp in a span: DEM_PAIRS_CONTIG, fewer on a small grid so every SM gets spans: a.pairs_contig)
  const bin_t kSpan = (bin_t)kPairWarps * (DEM_PAIRS_ADAPT ? a.pairs_contig : DEM_PAIRS_CONTIG);
  const bin_t ncell = (bin_t)a.ncell;
  bin_t it = (bin_t)blockIdx.x * kSpan + w, it_stop = min(ncell, (bin_t)blockIdx.x * kSpan + kSpan);
  auto advance = [&]() {
    if ((it += kPairWarps) >= it_stop) {
      it += (bin_t)(gridDim.x - 1) * kSpan;
      it_stop = min(ncell, it_stop + (bin_t)gridDim.x * kSpan);
    }
  };
#if DEM_PAIRS_PIPE
  // Software pipeline over the warp's bins: entering bin c its items are already in registers
  // and the bounds of c + 1 too; the items of c + 1 and the bounds of c + 2 are issued before
  // c's member records are awaited, so of the bounds -> items -> records chain only the last
  // load is exposed per bin.
  auto bounds = [&](bin_t c, int& b0, int& b1) {
    b0 = b1 = 0;
    if (c < ncell) {
      b0 = a.cell_start[c];
      b1 = a.cell_start[c + 1];
    }
  };
  const bin_t cfirst = it;
  int k0c, k1c, k0n, k1n;
  bounds(it, k0c, k1c);
  advance();
  bin_t cnext = it;
  bounds(it, k0n, k1n);
  int itA = lane < k1c - k0c ? a.items[k0c + lane] : 0;
  int itB = lane + 32 < k1c - k0c ? a.items[k0c + 32 + lane] : 0;
  for (bin_t cid = cfirst; cid < ncell;) {
    const int k0 = k0c;
    const int m = k1c - k0c;
    const int curA = itA, curB = itB;
    const int mn = k1n - k0n;
    itA = lane < mn ? a.items[k0n + lane] : 0;
    itB = lane + 32 < mn ? a.items[k0n + 32 + lane] : 0;
    k0c = k0n;
    k1c = k1n;
    cid = cnext;
    advance();
    cnext = it;
    bounds(it, k0n, k1n);
#else
  for (bin_t cid = it; cid < ncell; advance(), cid = it) {
    const int k0 = a.cell_start[cid];
    const int m = a.cell_start[cid + 1] - k0;
    const int curA = lane < m ? a.items[k0 + lane] : 0;
    const int curB = lane + 32 < m ? a.items[k0 + 32 + lane] : 0;
#endif
    if (m >= 2) {
      if (m <= (kTinyOn ? kTiny : kSmallDense)) {
        // Small bins (sparse regions: a falling column, a bed's free surface): all m (m - 1) / 2 pairs
        // in passes of 32, the own-bin rule applied per pair ((g_a | g_b) == 7) — no group ranking
        // and no row descriptors, which cost ~200 instructions per bin whatever its size
        if (lane < m) {
          const int idx = curA & 0x1fffffff;
          A.put(lane, ldg256(a.dpos + idx));
          A.meta_put(lane, make_int2(a.s_clump[idx], curA));
        }
        __syncwarp();
        const int np = (m * (m - 1)) / 2;
        for (int base = 0; base < np; base += 32) {
          const int p = base + lane;
          int i, j;
          decode_tri(min(p, np - 1), i, j);
          const int2 mu = A.meta_get(i), mv = A.meta_get(j);
          const bool own = (p < np) & ((((unsigned)(mu.y | mv.y)) >> 29) == 7u);
          const bool hit = own & candidate<kGhosts, kMargin>(a, mu, mv, A.get(i), A.get(j));
          push_hits<kMargin>(a, bf, nbuf, hit, mu.y & 0x1fffffff, mv.y & 0x1fffffff, lane);
        }
        __syncwarp();
      } else if (m <= kFlatMax) {
        // Lane l loads members l and l + 32 and stores them at their place in the group order
        // (a 64-bit warp scan of one-hot byte counters gives every member its rank in its group
        // and every group its start); then the warp enumerates the pair blocks flat, 32 pairs
        // per pass, so no lane tests a pair that belongs to another bin.
        double4 u0 = make_double4(0.0, 0.0, 0.0, 0.0), u1 = u0;
        int2 mt0 = make_int2(0, 0), mt1 = mt0;
        int pos0 = 0, pos1 = 0;
#if !DEM_PAIRS_BALLOT
        unsigned long long v0 = 0, v1 = 0;
#endif
        if (lane < m) {
          const int it = curA;
          const int idx = it & 0x1fffffff;
          u0 = ldg256(a.dpos + idx);
          mt0 = make_int2(a.s_clump[idx], idx);
          pos0 = (kGroupPos >> (4 * ((unsigned)it >> 29))) & 7;
#if !DEM_PAIRS_BALLOT
          v0 = 1ull << (8 * pos0);
#endif
        }
        if (lane + 32 < m) {
          const int it = curB;
          const int idx = it & 0x1fffffff;
          u1 = ldg256(a.dpos + idx);
          mt1 = make_int2(a.s_clump[idx], idx);
          pos1 = (kGroupPos >> (4 * ((unsigned)it >> 29))) & 7;
#if !DEM_PAIRS_BALLOT
          v1 = 1ull << (8 * pos1);
#endif
        }
#if DEM_PAIRS_BALLOT
        // Group order by bit-plane ballots: A_k (B_k) = lanes of the first (second) member half
        // whose position has bit k set.  The size of position p is the popcount of the lanes whose
        // three planes match p; a member's slot = (members at lower positions) + (members at its
        // position before it: first half before second half, then by lane).
        const unsigned lt = (1u << lane) - 1u;
        const unsigned V0 = m >= 32 ? 0xffffffffu : (1u << m) - 1u;
        const unsigned V1 = m >= 64 ? 0xffffffffu : (m > 32 ? (1u << (m - 32)) - 1u : 0u);
        const unsigned A0 = __ballot_sync(0xffffffffu, pos0 & 1) & V0, A1 = __ballot_sync(0xffffffffu, pos0 & 2) & V0,
                       A2 = __ballot_sync(0xffffffffu, pos0 & 4) & V0;
        unsigned B0 = 0u, B1 = 0u, B2 = 0u;
        if (m > 32) {  // warp-uniform
          B0 = __ballot_sync(0xffffffffu, pos1 & 1) & V1;
          B1 = __ballot_sync(0xffffffffu, pos1 & 2) & V1;
          B2 = __ballot_sync(0xffffffffu, pos1 & 4) & V1;
        }
        // lanes of a half at exactly position p / at a position below p (bit-sliced comparison)
        auto at = [](unsigned V, unsigned X0, unsigned X1, unsigned X2, int p) {
          return V & ((p & 1) ? X0 : ~X0) & ((p & 2) ? X1 : ~X1) & ((p & 4) ? X2 : ~X2);
        };
        auto below = [](unsigned V, unsigned X0, unsigned X1, unsigned X2, int p) {
          const unsigned P0 = (p & 1) ? ~0u : 0u, P1 = (p & 2) ? ~0u : 0u, P2 = (p & 4) ? ~0u : 0u;
          const unsigned e2 = ~(X2 ^ P2), e1 = ~(X1 ^ P1);
          return V & ((~X2 & P2) | (e2 & ~X1 & P1) | (e2 & e1 & ~X0 & P0));
        };
        int nk[7];
#pragma unroll
        for (int k = 0; k < 7; ++k) nk[k] = __popc(at(V0, A0, A1, A2, k)) + __popc(at(V1, B0, B1, B2, k));
        const int n7 = nk[0], n6 = nk[1], n5 = nk[3], n3 = nk[4], n4 = nk[6];
        const int s1 = n7 + n6, s5 = s1 + nk[2], s3 = s5 + n5, s2 = s3 + n3, s4 = s2 + nk[5];
        __syncwarp();
        if (lane < m) {
          const int q = __popc(below(V0, A0, A1, A2, pos0)) + __popc(below(V1, B0, B1, B2, pos0)) +
                        __popc(at(V0, A0, A1, A2, pos0) & lt);
          A.put(q, u0);
          A.meta_put(q, mt0);
        }
        if (lane + 32 < m) {
          const int q = __popc(below(V0, A0, A1, A2, pos1)) + __popc(below(V1, B0, B1, B2, pos1)) +
                        __popc(at(V0, A0, A1, A2, pos1)) + __popc(at(V1, B0, B1, B2, pos1) & lt);
          A.put(q, u1);
          A.meta_put(q, mt1);
        }
#else
        const unsigned long long x0 = warp_incl_scan64(v0, lane);
        const unsigned long long t0 = __shfl_sync(0xffffffffu, x0, 31);
        unsigned long long x1 = 0, t1 = 0;
        if (m > 32) {  // warp-uniform
          x1 = warp_incl_scan64(v1, lane);
          t1 = __shfl_sync(0xffffffffu, x1, 31);
        }
        const unsigned long long tot = t0 + t1;                          // byte k: size of group at position k
        const unsigned long long st = (tot << 8) * 0x0101010101010101ull;  // byte k: start of position k
        __syncwarp();
        if (lane < m) {
          const int q = byte_of(st, pos0) + byte_of(x0 - v0, pos0);
          A.put(q, u0);
          A.meta_put(q, mt0);
        }
        if (lane + 32 < m) {
          const int q = byte_of(st, pos1) + byte_of(t0, pos1) + byte_of(x1 - v1, pos1);
          A.put(q, u1);
          A.meta_put(q, mt1);
        }
#endif
#if DEM_PAIRS_ROWDEC
        {
          RowDec& D = smR[w];
#if !DEM_PAIRS_BALLOT
          const int n7 = byte_of(tot, 0), n6 = byte_of(tot, 1), n5 = byte_of(tot, 3), n3 = byte_of(tot, 4);
          const int n4 = byte_of(tot, 6);
          const int s1 = byte_of(st, 2), s5 = byte_of(st, 3), s3 = byte_of(st, 4), s2 = byte_of(st, 5);
          const int s4 = byte_of(st, 6);
#endif
          const int e0 = n7 * (m - 1) - ((n7 * (n7 - 1)) >> 1);
          const int e1 = e0 + n6 * (s2 - s1);
          const int e2 = e1 + n5 * (s4 - s3);
          const int total = e2 + n3 * n4;
          int lo0, c0, o0, lo1 = 0, c1 = 0, o1 = 0;
          member_row(lane, m, n7, n6, n5, n3, n4, s1, s2, s3, s4, s5, e0, e1, e2, lo0, c0, o0);
          if (m > 32) member_row(lane + 32, m, n7, n6, n5, n3, n4, s1, s2, s3, s4, s5, e0, e1, e2, lo1, c1, o1);
          // bitmap words of this bin's numbering cleared, then one start bit per non-empty row
          const int nw = (total + 31) >> 5;
          if (lane < nw) D.bmap[lane] = 0u;
          if (lane + 32 < nw) D.bmap[lane + 32] = 0u;
#if !DEM_PAIRS_BALLOT
          const unsigned lt = (1u << lane) - 1u;
#endif
          const unsigned b0 = __ballot_sync(0xffffffffu, c0 > 0), b1 = __ballot_sync(0xffffffffu, c1 > 0);
          __syncwarp();
          if (c0 > 0) {
            D.desc[__popc(b0 & lt)] = ((lo0 - o0) << 8) | lane;
            atomicOr(&D.bmap[o0 >> 5], 1u << (o0 & 31));
          }
          if (c1 > 0) {
            D.desc[__popc(b0) + __popc(b1 & lt)] = ((lo1 - o1) << 8) | (lane + 32);
            atomicOr(&D.bmap[o1 >> 5], 1u << (o1 & 31));
          }
          __syncwarp();
          const unsigned le = lt | (1u << lane);
          int before = 0;  // row starts below base (warp-uniform)
          for (int base = 0; base < total; base += 32) {
            const unsigned word = D.bmap[base >> 5];
            const int p = base + lane;
#if DEM_PAIRS_NODIV
            // every lane runs the pair code (no divergent branch around it): a lane past the bin's
            // last pair reads a clamped in-range slot and its result is masked off
            int ia = 0, ib = 0;
            const int d = D.desc[before + __popc(word & le) - 1];
            const bool hit =
                flat_pair<kGhosts, kMargin>(a, A, d & 0xff, min(p + (d >> 8), kFlatMax - 1), ia, ib, p < total);
#else
            bool hit = false;
            int ia = 0, ib = 0;
            if (p < total) {
              const int d = D.desc[before + __popc(word & le) - 1];
              hit = flat_pair<kGhosts, kMargin>(a, A, d & 0xff, p + (d >> 8), ia, ib);
            }
#endif
            before += __popc(word);
            push_hits<kMargin>(a, bf, nbuf, hit, ia, ib, lane);
          }
        }
#else
        __syncwarp();
        const PairBlocks B(tot, st, m);
        for (int base = 0; base < B.total; base += 32) {
          const int p = base + lane;
          bool hit = false;
          int ia = 0, ib = 0;
          if (p < B.total) {
            int i, j;
            B.decode(p, tri_ij, i, j);
            hit = flat_pair<kGhosts, kMargin>(a, A, i, j, ia, ib);
          }
          push_hits<kMargin>(a, bf, nbuf, hit, ia, ib, lane);
        }
#endif
      } else {
        // Large bins (m > kFlatMax): blocks of 32 members in the two halves of the shared slots,
        // every pair of the bin tested (the group filter applied per pair).
        for (int ib = 0; ib < m; ib += 32) {
          const int mi = min(32, m - ib);
          __syncwarp();
          if (lane < mi) load_member(a, A, lane, k0 + ib + lane);
          for (int jb = ib; jb < m; jb += 32) {
            const int mj = min(32, m - jb);
            const bool same = jb == ib;
            const int ob = same ? 0 : 32;  // slots of the second block
            if (!same) {
              __syncwarp();
              if (lane < mj) load_member(a, A, 32 + lane, k0 + jb + lane);
            }
            __syncwarp();
            const int np = same ? mi * (mi - 1) / 2 : mi * mj;
            for (int base = 0; base < np; base += 32) {
              const int p = base + lane;
              bool hit = false;
              int ia = 0, ibx = 0;
              if (p < np) {
                int i, j;
                if (same) {
                  decode_tri(p, i, j);
                } else {
                  i = p / mj;
                  j = p - i * mj;
                }
                const int2 mu = A.meta_get(i);
                const int2 mv = A.meta_get(ob + j);
                if (((unsigned)(mu.y | mv.y) >> 29) == 7u) {
                  hit = candidate<kGhosts, kMargin>(a, mu, mv, A.get(i), A.get(ob + j));
                  ia = mu.y & 0x1fffffff;
                  ibx = mv.y & 0x1fffffff;
                }
              }
              push_hits<kMargin>(a, bf, nbuf, hit, ia, ibx, lane);
            }
          }
        }
      }
    }
  }
  flush_pairs<kMargin>(FlushCtx(a), bf, nbuf, lane);
}

// ---------------------------------------------------------------- rows
// Per owned sphere: its candidate partners (keys gathered) sorted by partner key, then its
// wall entries (keys INT64_MAX - p sort last, larger p first), written to its CSR row, and
// each entry's history index found in the sphere's previous row ("persist between
// timesteps"; -1 for a contact born this step).  Rows of up to kRegRow candidates — nearly
// all of them — are sorted and matched in registers; longer ones in place in memory.
#ifndef DEM_ROWS_LOCAL
#define DEM_ROWS_LOCAL 24  // rows up to this long sorted in a thread-local array (0: in place in the row)
#endif
#ifndef DEM_REG_ROW
#define DEM_REG_ROW 6  // A/B on the C5 bench: 6 beats 5, 7 and 8 (rows 1.80 vs 1.97-2.08 ms)
#endif
constexpr int kRegRow = DEM_REG_ROW;

// key of a candidate partner: a sphere's key, or INT64_MAX - kMaxPlanes - t for triangle t
// (partner code -1 - kMaxPlanes - t, written by k_mesh_pairs): sorts after every sphere
__device__ __forceinline__ long long partner_key(const StepArgs& a, int code) {
  return code >= 0 ? a.s_key[code] : 0x7fffffffffffffffLL - (long long)(-1 - code);
}

__device__ __forceinline__ int prev_index(const Rows& prev, int pb, int pe, long long key) {
  for (int v = pb; v < pe; ++v)
    if (prev.key[v] == key) return v;
  return -1;
}

#ifndef DEM_ROWS_MINB
#define DEM_ROWS_MINB (2048 / DEM_ROWS_TPB)  // 32 registers (a few spilled): 1.69 ms vs 1.80 at 40, 2.07 at 48
#endif
__global__ void __launch_bounds__(DEM_ROWS_TPB, DEM_ROWS_MINB) k_rows_finish(StepArgs a) {
  pdl_wait_and_release();
  if (*a.abort || a.ctl->abort) return;  // (an error in the steps running beside an ahead detection)
  const int total = a.rows.row_ptr[a.ns];
  if ((long long)total > a.cap_entries) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
      a.ctl->need_entries = total;
      atomicExch(a.abort, 1);
    }
    return;
  }
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.ns_own) return;
  const int beg = a.rows.row_ptr[i];
  const int m = a.rows.row_ptr[i + 1] - beg;
  const int pb = a.prev.row_ptr[i], pe = a.prev.row_ptr[i + 1];
  Entry* R = a.rows.ent + beg;
  long long* K = a.rows.key + beg;
  const unsigned wmask = a.wall_mask[i];  // the pose kernel's sphere-plane candidates
  const int w = __popc(wmask);
  const int nc = m - w;  // k_pairs handed out slots [w, m) of the candidate list
  const int* S = a.slots + (size_t)w * a.ns_own + i;  // S[q * ns_own]: candidate q
  const long long* SK = DEM_SLOT_KEYS ? a.slot_key + (size_t)w * a.ns_own + i : nullptr;  // and its key
  if (nc <= kRegRow) {
    int tt[kRegRow], hh[kRegRow];
    long long kk[kRegRow];
#pragma unroll
    for (int q = 0; q < kRegRow; ++q) tt[q] = q < nc ? S[(size_t)q * a.ns_own] : 0;
#pragma unroll
    for (int q = 0; q < kRegRow; ++q) {
      kk[q] = q < nc ? (DEM_SLOT_KEYS ? SK[(size_t)q * a.ns_own] : partner_key(a, tt[q])) : 0x7fffffffffffffffLL;
      hh[q] = -1;
    }
    // odd-even transposition sort (keys of the candidates are distinct; padding sorts last)
#pragma unroll
    for (int r = 0; r < kRegRow; ++r)
#pragma unroll
      for (int q = r & 1; q + 1 < kRegRow; q += 2)
        if (kk[q] > kk[q + 1]) {
          const long long tk = kk[q];
          kk[q] = kk[q + 1];
          kk[q + 1] = tk;
          const int t = tt[q];
          tt[q] = tt[q + 1];
          tt[q + 1] = t;
        }
#pragma unroll 4
    for (int v = pb; v < pe; ++v) {
      const long long pk = a.prev.key[v];
#pragma unroll
      for (int q = 0; q < kRegRow; ++q)
        if (kk[q] == pk) hh[q] = v;
    }
#pragma unroll
    for (int q = 0; q < kRegRow; ++q)
      if (q < nc) {
        Entry e;
        e.partner = tt[q];
        e.prev = hh[q];
        R[q] = e;
        K[q] = kk[q];
      }
#if DEM_ROWS_LOCAL
  } else if (nc <= DEM_ROWS_LOCAL) {
    // longer rows (the big spheres): sorted in a thread-local array (local memory, cached in L1
    // write-back) instead of in place in the global row
    long long kl[DEM_ROWS_LOCAL];
    int tl[DEM_ROWS_LOCAL];
    for (int u = 0; u < nc; ++u) {
      const int t = S[(size_t)u * a.ns_own];
      const long long xk = DEM_SLOT_KEYS ? SK[(size_t)u * a.ns_own] : partner_key(a, t);
      int v = u - 1;
      while (v >= 0 && kl[v] > xk) {
        kl[v + 1] = kl[v];
        tl[v + 1] = tl[v];
        --v;
      }
      kl[v + 1] = xk;
      tl[v + 1] = t;
    }
    int pj = pb;  // merge with the previous row (both sorted by key)
    for (int u = 0; u < nc; ++u) {
      const long long k = kl[u];
      while (pj < pe && a.prev.key[pj] < k) ++pj;
      Entry e;
      e.partner = tl[u];
      e.prev = (pj < pe && a.prev.key[pj] == k) ? pj : -1;
      R[u] = e;
      K[u] = k;
    }
#endif
  } else {
    for (int u = 0; u < nc; ++u) {
      const int t = S[(size_t)u * a.ns_own];
      Entry e;
      e.partner = t;
      e.prev = -1;  // set by the merge below
      R[u] = e;
      K[u] = DEM_SLOT_KEYS ? SK[(size_t)u * a.ns_own] : partner_key(a, t);
    }
    for (int u = 1; u < nc; ++u) {
      const Entry x = R[u];
      const long long xk = K[u];
      int v = u - 1;
      while (v >= 0 && K[v] > xk) {
        R[v + 1] = R[v];
        K[v + 1] = K[v];
        --v;
      }
      R[v + 1] = x;
      K[v + 1] = xk;
    }
    int pj = pb;  // merge with the previous row (both sorted by key)
    for (int u = 0; u < nc; ++u) {
      const long long k = K[u];
      while (pj < pe && a.prev.key[pj] < k) ++pj;
      R[u].prev = (pj < pe && a.prev.key[pj] == k) ? pj : -1;
    }
  }
  if (a.n_tri)  // this set's mesh entries, for the per-step geometry pass (k_mesh_geom)
    for (int u = 0; u < nc; ++u)
      if (R[u].partner <= -1 - kMaxPlanes) a.mlist_out[atomicAdd(a.mlist_out_n, 1)] = make_int2(beg + u, i);
  for (int u = nc, p = a.tab.n_planes - 1; p >= 0; --p)
    if (wmask >> p & 1u) {
      const long long key = (long long)(0x7fffffffffffffffLL - p);
      Entry e;
      e.partner = -1 - p;
      e.prev = prev_index(a.prev, pb, pe, key);
      K[u] = key;
      R[u++] = e;
    }
}

// host launchers
void launch_bin_scatter(const StepArgs& a, cudaStream_t s) {
  if (a.ns) launch_k(k_bin_scatter, (a.ns + DEM_SCATTER_TPB - 1) / DEM_SCATTER_TPB, DEM_SCATTER_TPB, s, a.pdl, a);
}
void launch_pairs(const StepArgs& a, cudaStream_t s, int n_sm) {
  long long warps = a.ncell;
  long long blocks = (warps + kPairWarps - 1) / kPairWarps;
  long long cap = (long long)n_sm * 8 * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  // span length: DEM_PAIRS_CONTIG bins per warp on a large grid; on a small one (one rank's slab of
  // a decomposition, a small bed) shorter, so that there are at least 4 spans per resident CTA slot
  StepArgs b = a;
  {
    long long contig = DEM_PAIRS_CONTIG;
    const long long slots = (long long)n_sm * DEM_PAIRS_MINB;
    while (contig > 4 && a.ncell < DEM_PAIRS_SPANS_PER_SLOT * slots * kPairWarps * contig) contig >>= 1;
    b.pairs_contig = (int)contig;
  }
  const bool ghosts = a.n_own < a.n, margin = a.margin != 0.0;
  // the small-bin pass only where bins are sparse (a.tiny, set from spheres per bin): in a dense bed
  // nearly no bin takes it and the extra branch per bin costs ~0.3%
  const bool tiny = DEM_PAIRS_TINY && a.tiny;
  const unsigned g = (unsigned)blocks, t = kPairWarps * 32;
  if (tiny) {
    if (ghosts && margin) launch_k(k_pairs<true, true, true>, g, t, s, a.pdl, b);
    else if (ghosts) launch_k(k_pairs<true, false, true>, g, t, s, a.pdl, b);
    else if (margin) launch_k(k_pairs<false, true, true>, g, t, s, a.pdl, b);
    else launch_k(k_pairs<false, false, true>, g, t, s, a.pdl, b);
  } else {
    if (ghosts && margin) launch_k(k_pairs<true, true, false>, g, t, s, a.pdl, b);
    else if (ghosts) launch_k(k_pairs<true, false, false>, g, t, s, a.pdl, b);
    else if (margin) launch_k(k_pairs<false, true, false>, g, t, s, a.pdl, b);
    else launch_k(k_pairs<false, false, false>, g, t, s, a.pdl, b);
  }
}
void launch_rows_finish(const StepArgs& a, cudaStream_t s) {
  if (a.ns) launch_k(k_rows_finish, (a.ns + DEM_ROWS_TPB - 1) / DEM_ROWS_TPB, DEM_ROWS_TPB, s, a.pdl, a);
}

}  // namespace dem
