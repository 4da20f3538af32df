// kernels_detect.cu — (a1) sphere poses, (a2) multi-insert binning, (a3) narrow phase.
//
// PAPER.md:142 ("identifying the active set represents a significant computational
// bottleneck"), P:145 (per-step rebuild), P:69 (binning CD following hammadTobyDan2012:
// every body is inserted into each bin its AABB overlaps).  Readings: DESIGN.md §3
// R14 (predicate d.d <= (r_a + r_b + margin)^2 in fp64, no FMA), R15 (no intra-clump
// pairs), R22 (sphere centre c = X + R(q) o).
#include "dem_device.cuh"

namespace dem {

// ---------------------------------------------------------------- (a1) + bin count
// One thread per sphere: c = X + R(q) o (explicit roundings), store the centre, count
// the bins its enlarged AABB overlaps.  Component 0 also stores omega_world = R Omega.
__global__ void __launch_bounds__(256) k_pose_count(StepArgs a) {
  if (a.ctl->abort) return;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.ns) return;
  int c = a.s_clump[i];
  int tc = a.s_tc[i];
  double qw = a.cur.qw[c], qx = a.cur.qx[c], qy = a.cur.qy[c], qz = a.cur.qz[c];
  double R[9];
  quat_R(qw, qx, qy, qz, R);
  double ox = a.tab.tc_off[3 * tc], oy = a.tab.tc_off[3 * tc + 1], oz = a.tab.tc_off[3 * tc + 2];
  double cx = add(a.cur.x[c], row_dot(R, ox, oy, oz));
  double cy = add(a.cur.y[c], row_dot(R + 3, ox, oy, oz));
  double cz = add(a.cur.z[c], row_dot(R + 6, ox, oy, oz));
  a.sx[i] = cx;
  a.sy[i] = cy;
  a.sz[i] = cz;
  if (tc == a.tab.tpl_coff[a.tid[c]]) {
    double wx = a.cur.wx[c], wy = a.cur.wy[c], wz = a.cur.wz[c];
    a.wwx[c] = R[0] * wx + R[1] * wy + R[2] * wz;
    a.wwy[c] = R[3] * wx + R[4] * wy + R[5] * wz;
    a.wwz[c] = R[6] * wx + R[7] * wy + R[8] * wz;
  }
  const Grid& g = a.grid;
  if (!(cx >= g.dom_lo[0] && cx <= g.dom_hi[0] && cy >= g.dom_lo[1] && cy <= g.dom_hi[1] &&
        cz >= g.dom_lo[2] && cz <= g.dom_hi[2])) {
    raise_error(a.ctl, -10, a.s_key[i], a.gid[c]);
    return;
  }
  double r = a.tab.tc_rad[tc];
  int lx, hx, ly, hy, lz, hz;
  cell_range(g, 0, cx, r, lx, hx);
  cell_range(g, 1, cy, r, ly, hy);
  cell_range(g, 2, cz, r, lz, hz);
  for (int z = lz; z <= hz; ++z)
    for (int y = ly; y <= hy; ++y) {
      long long base = ((long long)z * g.n[1] + y) * g.n[0];
      for (int x = lx; x <= hx; ++x) atomicAdd(&a.cell_count[base + x], 1);
    }
}

// ---------------------------------------------------------------- bin scatter
// Slots are taken by decrementing the counts, which leaves cell_count all-zero for the
// next step.  The order inside a bin is irrelevant: rows are sorted by partner key.
__global__ void __launch_bounds__(256) k_bin_scatter(StepArgs a) {
  if (a.ctl->abort) return;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.ns) return;
  bool fits = (long long)a.cell_start[a.ncell] <= a.cap_inserts;
  double r = a.tab.tc_rad[a.s_tc[i]];
  const Grid& g = a.grid;
  int lx, hx, ly, hy, lz, hz;
  cell_range(g, 0, a.sx[i], r, lx, hx);
  cell_range(g, 1, a.sy[i], r, ly, hy);
  cell_range(g, 2, a.sz[i], r, lz, hz);
  for (int z = lz; z <= hz; ++z)
    for (int y = ly; y <= hy; ++y) {
      long long base = ((long long)z * g.n[1] + y) * g.n[0];
      for (int x = lx; x <= hx; ++x) {
        long long cid = base + x;
        int slot = atomicSub(&a.cell_count[cid], 1) - 1;
        if (fits) a.items[a.cell_start[cid] + slot] = i;
      }
    }
}

// ---------------------------------------------------------------- (a3) narrow phase
// Every candidate pair (a, b) is reported by thread a exactly once: in the bin that
// holds the minimum corner of the two AABBs' bin-range intersection (so both directed
// rows a->b and b->a are produced, by threads a and b, with the same predicate).
template <bool kFill>
__device__ __forceinline__ int narrow_row(const StepArgs& a, int i, int* out_partner, long long* out_key) {
  const Grid& g = a.grid;
  int ci = a.s_clump[i];
  double cx = a.sx[i], cy = a.sy[i], cz = a.sz[i];
  double r = a.tab.tc_rad[a.s_tc[i]];
  int lx, hx, ly, hy, lz, hz;
  cell_range(g, 0, cx, r, lx, hx);
  cell_range(g, 1, cy, r, ly, hy);
  cell_range(g, 2, cz, r, lz, hz);
  int cnt = 0;
  for (int z = lz; z <= hz; ++z)
    for (int y = ly; y <= hy; ++y) {
      long long base = ((long long)z * g.n[1] + y) * g.n[0];
      for (int x = lx; x <= hx; ++x) {
        long long cid = base + x;
        int k0 = a.cell_start[cid], k1 = a.cell_start[cid + 1];
        for (int k = k0; k < k1; ++k) {
          int b = a.items[k];
          if (b == i || a.s_clump[b] == ci) continue;
          double bx = a.sx[b], by = a.sy[b], bz = a.sz[b];
          double rb = a.tab.tc_rad[a.s_tc[b]];
          // dedupe: only in the bin of the range intersection's minimum corner
          if (max(lx, cell_lo(g, 0, bx, rb)) != x || max(ly, cell_lo(g, 1, by, rb)) != y ||
              max(lz, cell_lo(g, 2, bz, rb)) != z)
            continue;
          double dx = sub(bx, cx), dy = sub(by, cy), dz = sub(bz, cz);
          double d2 = add(add(mul(dx, dx), mul(dy, dy)), mul(dz, dz));
          double s = add(add(r, rb), a.margin);
          if (d2 <= mul(s, s)) {
            if (kFill) {
              out_partner[cnt] = b;
              out_key[cnt] = a.s_key[b];
            }
            ++cnt;
          }
        }
      }
    }
  // sphere-plane candidates: (r + margin) - (c - p_w).n_w >= 0
  for (int p = 0; p < a.tab.n_planes; ++p) {
    const double* pp = a.tab.plane_pt[p];
    const double* nw = a.tab.plane_n[p];
    double dd = add(add(mul(sub(cx, pp[0]), nw[0]), mul(sub(cy, pp[1]), nw[1])), mul(sub(cz, pp[2]), nw[2]));
    if (sub(add(r, a.margin), dd) >= 0.0) {
      if (kFill) {
        out_partner[cnt] = -1 - p;
        out_key[cnt] = (long long)(0x7fffffffffffffffLL - p);
      }
      ++cnt;
    }
  }
  return cnt;
}

__global__ void __launch_bounds__(256) k_narrow_count(StepArgs a) {
  if (a.ctl->abort) return;
  if ((long long)a.cell_start[a.ncell] > a.cap_inserts) {
    a.ctl->need_inserts = a.cell_start[a.ncell];
    atomicExch(&a.ctl->abort, 1);
    return;
  }
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.ns) return;
  a.row_cnt[i] = narrow_row<false>(a, i, nullptr, nullptr);
}

__global__ void __launch_bounds__(256) k_narrow_fill(StepArgs a) {
  if (a.ctl->abort) return;
  int total = a.rows.row_ptr[a.ns];
  if ((long long)total > a.cap_entries) {
    a.ctl->need_entries = total;
    atomicExch(&a.ctl->abort, 1);
    return;
  }
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.ns) return;
  int beg = a.rows.row_ptr[i];
  int* P = a.rows.partner + beg;
  long long* K = a.rows.key + beg;
  int m = narrow_row<true>(a, i, P, K);
  // insertion sort of the row by partner key (rows are short: ~2c + walls entries)
  for (int u = 1; u < m; ++u) {
    long long kk = K[u];
    int pp = P[u];
    int v = u - 1;
    while (v >= 0 && K[v] > kk) {
      K[v + 1] = K[v];
      P[v + 1] = P[v];
      --v;
    }
    K[v + 1] = kk;
    P[v + 1] = pp;
  }
}

// host launchers
void launch_pose_count(const StepArgs& a, cudaStream_t s) {
  if (a.ns) k_pose_count<<<(a.ns + 255) / 256, 256, 0, s>>>(a);
}
void launch_bin_scatter(const StepArgs& a, cudaStream_t s) {
  if (a.ns) k_bin_scatter<<<(a.ns + 255) / 256, 256, 0, s>>>(a);
}
void launch_narrow_count(const StepArgs& a, cudaStream_t s) {
  if (a.ns) k_narrow_count<<<(a.ns + 255) / 256, 256, 0, s>>>(a);
}
void launch_narrow_fill(const StepArgs& a, cudaStream_t s) {
  if (a.ns) k_narrow_fill<<<(a.ns + 255) / 256, 256, 0, s>>>(a);
}

}  // namespace dem
