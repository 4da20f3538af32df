// kernels_mesh.cu — kinematic triangle-mesh boundaries.
//
// PAPER.md P:277 (cone penetrometer "penetrates the sample with a constant velocity")
// (funnel), P:344 (rover wheel); SPEC S:241-262 (sphere_triangle_contact, body_wrench,
// advance_boundary).  Readings: R25 closest point by Voronoi regions in a fixed
// rounding order; R26 one contact per surface feature; R27 prescribed motion X += h v,
// q <- normalize(q_step (x) q), the flat-wall limit R_bar = r, m_bar = M for the force.
//
//   k_mesh_pose    per triangle: world vertices X + R(q) x_body of this step (+ the snapshot an
//                  ahead detection reads)
//   k_mesh_pairs   per triangle: the bins its margin-padded AABB overlaps; each member sphere is
//                  tested in exactly one of them (the lowest bin common to both ranges) and a hit
//                  takes a slot in the sphere's candidate list like a sphere partner
//   k_mesh_finish  one CTA: the per-CTA wrench partials of k_force_integrate summed in CTA order
//                  (deterministic), then every mesh advanced one step
#include "dem_device.cuh"

namespace dem {

__global__ void __launch_bounds__(256) k_mesh_pose(StepArgs a) {
  if (a.ctl->abort) return;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.n_tri) return;
  const double* M = a.mesh + kMeshRec * a.tri_mesh[t];
  double R[9];
  quat_R(M[3], M[4], M[5], M[6], R);
  const double* v = a.tri_body + 9 * t;
  double w[9];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double ox = v[3 * k], oy = v[3 * k + 1], oz = v[3 * k + 2];
    w[3 * k] = add(M[0], row_dot(R, ox, oy, oz));
    w[3 * k + 1] = add(M[1], row_dot(R + 3, ox, oy, oz));
    w[3 * k + 2] = add(M[2], row_dot(R + 6, ox, oy, oz));
  }
#pragma unroll
  for (int k = 0; k < 9; ++k) a.tri_world[9 * t + k] = w[k];
  if (a.tri_snap)
#pragma unroll
    for (int k = 0; k < 9; ++k) a.tri_snap[9 * t + k] = w[k];
}

// bin coordinate range of [lo, hi] along axis d (the clamped formula of cell_range)
__device__ __forceinline__ void span_bins(const Grid& g, int d, double lo, double hi, int& blo, int& bhi) {
  blo = clampi(__double2int_rd((lo - g.lo[d]) * g.inv_cell), 0, g.n[d] - 1);
  bhi = clampi(__double2int_rd((hi - g.lo[d]) * g.inv_cell), 0, g.n[d] - 1);
}

// blockIdx.x = triangle; the warps of kMeshPairSplit CTAs (blockIdx.y) stride over its bins
__global__ void __launch_bounds__(256) k_mesh_pairs(StepArgs a) {
  if (*a.abort || a.ctl->abort) return;
  const int t = blockIdx.x;
  if (t >= a.n_tri) return;
  const Grid& g = a.grid;
  const double* T = a.tri_dpos + 9 * t;
  int tlo[3], thi[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double mn = fmin(fmin(T[d], T[3 + d]), T[6 + d]), mx = fmax(fmax(T[d], T[3 + d]), T[6 + d]);
    span_bins(g, d, mn - g.pad, mx + g.pad, tlo[d], thi[d]);
  }
  const int nx = thi[0] - tlo[0] + 1, ny = thi[1] - tlo[1] + 1, nz = thi[2] - tlo[2] + 1;
  const long long nb = (long long)nx * ny * nz;
  const int lane = threadIdx.x & 31, nw = (blockDim.x >> 5) * gridDim.y;
  const int warp = blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int code = -1 - kMaxPlanes - t;
  // an insert overflow (k_bin_scatter stopped writing past cap_inserts; the host regrows and
  // re-runs the step) leaves the bin bounds pointing past the items array: nothing to read
  if ((long long)a.cell_start[a.ncell] > a.cap_inserts) return;
  for (long long b = warp; b < nb; b += nw) {
    const int bx = tlo[0] + (int)(b % nx), by = tlo[1] + (int)((b / nx) % ny), bz = tlo[2] + (int)(b / ((long long)nx * ny));
    const long long cid = bx * g.st[0] + by * g.st[1] + bz * g.st[2];
    const int k0 = a.cell_start[cid], m = a.cell_start[cid + 1] - k0;
    for (int q = lane; q < m; q += 32) {
      const int idx = a.items[k0 + q] & 0x1fffffff;
      if (idx >= a.ns_own) continue;  // ghosts are evaluated by their owners
      const double4 s = a.dpos[idx];
      int lx, hx, ly, hy, lz, hz;
      cell_range(g, 0, s.x, s.w, lx, hx);
      cell_range(g, 1, s.y, s.w, ly, hy);
      cell_range(g, 2, s.z, s.w, lz, hz);
      // tested only in the lowest bin common to the sphere's and the triangle's ranges
      if (bx != max(lx, tlo[0]) || by != max(ly, tlo[1]) || bz != max(lz, tlo[2])) continue;
      double qx, qy, qz;
      closest_on_triangle(T, s.x, s.y, s.z, qx, qy, qz);
      const double dx = sub(s.x, qx), dy = sub(s.y, qy), dz = sub(s.z, qz);
      const double sr = add(s.w, a.margin);
      if (add(add(mul(dx, dx), mul(dy, dy)), mul(dz, dz)) <= mul(sr, sr)) {
        const int slot = atomicAdd(&a.row_cnt[idx], 1);
        if (slot < a.row_width) {
          a.slots[(size_t)slot * a.ns_own + idx] = code;
          if (DEM_SLOT_KEYS) a.slot_key[(size_t)slot * a.ns_own + idx] = 0x7fffffffffffffffLL - (long long)(-1 - code);
        } else {
          atomicMax(&a.ctl->need_width, (long long)slot + 1);
          atomicExch(a.abort, 1);
        }
      }
    }
  }
}

// the wrench partials in CTA order (each thread a contiguous CTA range, then a fixed tree), and
// the prescribed motion of every mesh: X += h v; q <- normalize(q_step (x) q) (R27)
__global__ void __launch_bounds__(1024) k_mesh_finish(StepArgs a) {
  __shared__ double red[6][1024];
  if (a.ctl->abort) return;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int n = a.n_cta;
  const int c0 = (int)((long long)n * tid / nt), c1 = (int)((long long)n * (tid + 1) / nt);
  for (int m = 0; m < a.n_mesh; ++m) {
    double acc[6] = {0, 0, 0, 0, 0, 0};
    for (int c = c0; c < c1; ++c)
      if (a.mesh_flag[c]) {
        const double* p = a.mesh_part + ((size_t)c * a.n_mesh + m) * 6;
#pragma unroll
        for (int k = 0; k < 6; ++k) acc[k] += p[k];
      }
#pragma unroll
    for (int k = 0; k < 6; ++k) red[k][tid] = acc[k];
    __syncthreads();
    for (int s = nt / 2; s > 0; s >>= 1) {
      if (tid < s)
#pragma unroll
        for (int k = 0; k < 6; ++k) red[k][tid] += red[k][tid + s];
      __syncthreads();
    }
    if (tid == 0)
#pragma unroll
      for (int k = 0; k < 6; ++k) a.mesh_wrench[6 * m + k] = red[k][0];
    __syncthreads();
  }
  if (tid < a.n_mesh) {
    double* M = a.mesh + kMeshRec * tid;
    const double h = a.h;
    M[0] = add(M[0], mul(h, M[7]));
    M[1] = add(M[1], mul(h, M[8]));
    M[2] = add(M[2], mul(h, M[9]));
    const double w1 = M[13], x1 = M[14], y1 = M[15], z1 = M[16];
    const double w2 = M[3], x2 = M[4], y2 = M[5], z2 = M[6];
    const double nq0 = sub(sub(sub(mul(w1, w2), mul(x1, x2)), mul(y1, y2)), mul(z1, z2));
    const double nq1 = sub(add(add(mul(w1, x2), mul(x1, w2)), mul(y1, z2)), mul(z1, y2));
    const double nq2 = add(add(sub(mul(w1, y2), mul(x1, z2)), mul(y1, w2)), mul(z1, x2));
    const double nq3 = add(sub(add(mul(w1, z2), mul(x1, y2)), mul(y1, x2)), mul(z1, w2));
    const double nrm = __dsqrt_rn(add(add(add(mul(nq0, nq0), mul(nq1, nq1)), mul(nq2, nq2)), mul(nq3, nq3)));
    M[3] = __ddiv_rn(nq0, nrm);
    M[4] = __ddiv_rn(nq1, nrm);
    M[5] = __ddiv_rn(nq2, nrm);
    M[6] = __ddiv_rn(nq3, nrm);
  }
}

void launch_mesh_pose(const StepArgs& a, cudaStream_t s) {
  if (a.n_tri) k_mesh_pose<<<(a.n_tri + 255) / 256, 256, 0, s>>>(a);
}
constexpr int kMeshPairSplit = 16;  // CTAs per triangle (large facets span thousands of bins)
void launch_mesh_pairs(const StepArgs& a, cudaStream_t s) {
  if (a.n_tri) k_mesh_pairs<<<dim3(a.n_tri, kMeshPairSplit), 256, 0, s>>>(a);
}
void launch_mesh_finish(const StepArgs& a, cudaStream_t s) {
  if (a.n_mesh) k_mesh_finish<<<1, 1024, 0, s>>>(a);
}

}  // namespace dem
