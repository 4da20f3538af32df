/* oracle/dem_oracle.c — plain, slow, fp64 CPU oracle of the clump-DEM step.
 *
 * TEST INFRASTRUCTURE ONLY (see dem_oracle.h).  Build: gcc -O2 -ffp-contract=off
 * -shared -fPIC.  Every function cites the PAPER.md passage (P:line) it follows;
 * readings where the paper is silent are the SURVEY.md §8c O-numbers, restated in
 * DESIGN.md §3.
 *
 * Parity status of each part ("pins"):
 *   orc_pair_params    pinned  (SPEC examples S:64-66; series formulas)
 *   orc_contact_force  pinned  (static press S:119; Hertz closed forms; CoR identity;
 *                               tangential log decrement (c_t); Coulomb cap under a damped
 *                               kick (Eq. 3c branch); tests/test_oracle_pins_contact.py)
 *   contact point      pinned  (spin / impulse lever arms r - delta/2 of a polydisperse
 *                               oblique impact; soft-sphere rolling radius on plane/mesh)
 *   contact set        pinned  (independent numpy brute force, grid == brute)
 *   accumulate/integr. pinned  (free fall closed form, tumbling invariants,
 *                               momentum conservation, incline closed forms)
 *   meshes (NEXT-3)    pinned  (closest point vs an independent projection; sphere on a
 *                               mesh square == sphere on the analytic plane; head-on
 *                               restitution against a moving mesh wall; resting-weight
 *                               wrench; exact rotation of a spinning mesh)
 */
#include "dem_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define KEY_STRIDE 64
#define WALL_KEY(p) (INT64_MAX - (int64_t)(p))
#define MAX_PLANES 16 /* triangle t has key INT64_MAX - MAX_PLANES - t and partner code -1 - MAX_PLANES - t */

typedef struct {
  int64_t ka, kb;
  double ut[3];
} hist_rec;

typedef struct {
  int64_t ka, kb;  /* canonical keys */
  int64_t sa, sb;  /* sphere indices (sb = -1 - plane for walls) */
  double F[3], p[3], n[3], ut[3], delta;
} contact;

struct orc_sys {
  double h, g[3], margin, lo[3], hi[3];
  int n_mat;
  double* mat; /* 4 per material */
  int n_tmpl;
  int32_t* ncomp;
  int32_t* coff; /* first component of each template */
  double *offs, *rad, *mass, *inertia;
  int32_t* cmat;
  int n_planes;
  double *ppt, *pn;
  int32_t* pmat;
  int detect;
  int cd_every, since_rebuild; /* contact-set rebuild cadence */
  int overlap;                 /* detection one window ahead, "in the shadow" of the dynamics */
  int64_t n_pend;              /* -1: no set pending; else the size of the set built for the next window */
  contact* pend;
  /* clump state */
  int64_t n;
  int64_t* gid;
  int32_t* tid;
  double *X, *Q, *V, *W;
  double *Fc, *Tc; /* last applied wrench */
  /* spheres */
  int64_t ns;
  int64_t* s_clump;
  int32_t* s_comp;
  int64_t* s_key;
  double* s_pos;
  double* s_rad;
  /* history and last contacts */
  int64_t nh;
  hist_rec* hist;
  int64_t nc, cap;
  contact* con;
  int64_t steps;
  /* kinematic triangle meshes (NEXT-3; P:277 cone, P:307 funnel, P:344 wheel):
   * prescribed pose X, q (body -> world), velocity v and angular velocity w (world), advanced
   * after every step by X += h v, q <- normalize(qs (x) q) with qs the rotation by h|w| */
  int n_mesh;
  int64_t n_tri;
  double *mX, *mQ, *mV, *mW, *mQs, *mF, *mT; /* per mesh: 3, 4, 3, 3, 4, 3 (force), 3 (torque about X) */
  int32_t *mmat, *tri_mesh;
  int64_t* tri_vid;             /* 3 per triangle: vertex ids (bitwise-equal body vertices of a mesh share one) */
  double *tri_body, *tri_world; /* 9 per triangle (a, b, c) */
  char err[256];
};

static void* xcalloc(size_t n, size_t sz) {
  void* p = calloc(n ? n : 1, sz);
  if (!p) {
    fprintf(stderr, "oracle: out of memory\n");
    abort();
  }
  return p;
}

/* ------------------------------------------------------------------ rotation (P:129 clumps; O13)
 * R(q) for a unit quaternion q = (w,x,y,z), Hamilton convention, body -> world. */
static void quat_to_R(const double* q, double R[9]) {
  double w = q[0], x = q[1], y = q[2], z = q[3];
  double xx = x * x, yy = y * y, zz = z * z;
  double xy = x * y, xz = x * z, yz = y * z;
  double wx = w * x, wy = w * y, wz = w * z;
  R[0] = 1.0 - 2.0 * (yy + zz);
  R[1] = 2.0 * (xy - wz);
  R[2] = 2.0 * (xz + wy);
  R[3] = 2.0 * (xy + wz);
  R[4] = 1.0 - 2.0 * (xx + zz);
  R[5] = 2.0 * (yz - wx);
  R[6] = 2.0 * (xz - wy);
  R[7] = 2.0 * (yz + wx);
  R[8] = 1.0 - 2.0 * (xx + yy);
}

static void mat_vec(const double R[9], const double* v, double* out) {
  out[0] = R[0] * v[0] + R[1] * v[1] + R[2] * v[2];
  out[1] = R[3] * v[0] + R[4] * v[1] + R[5] * v[2];
  out[2] = R[6] * v[0] + R[7] * v[1] + R[8] * v[2];
}

static void mat_T_vec(const double R[9], const double* v, double* out) {
  out[0] = R[0] * v[0] + R[3] * v[1] + R[6] * v[2];
  out[1] = R[1] * v[0] + R[4] * v[1] + R[7] * v[2];
  out[2] = R[2] * v[0] + R[5] * v[1] + R[8] * v[2];
}

static void cross(const double* a, const double* b, double* out) {
  out[0] = a[1] * b[2] - a[2] * b[1];
  out[1] = a[2] * b[0] - a[0] * b[2];
  out[2] = a[0] * b[1] - a[1] * b[0];
}

static double dot(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

/* ------------------------------------------------------------------ pair parameters
 * P:98 defers k_n,k_t,gamma_n,gamma_t to jonJCND2015; reading O2/O4:
 * series E*, G*; CoR_pair = min, beta = -ln e / sqrt(ln^2 e + pi^2); mu = min. */
void orc_pair_params(const double* A, const double* B, double out[4]) {
  double Ea = A[0], nua = A[1], mua = A[2], ea = A[3];
  double Eb = B[0], nub = B[1], mub = B[2], eb = B[3];
  double inv_e = (1.0 - nua * nua) / Ea + (1.0 - nub * nub) / Eb;
  double inv_g = 2.0 * (2.0 - nua) * (1.0 + nua) / Ea + 2.0 * (2.0 - nub) * (1.0 + nub) / Eb;
  double e = ea < eb ? ea : eb;
  double beta = 0.0;
  if (e < 1.0) {
    double le = log(e);
    beta = -le / sqrt(le * le + M_PI * M_PI);
  }
  out[0] = 1.0 / inv_e;
  out[1] = 1.0 / inv_g;
  out[2] = beta;
  out[3] = mua < mub ? mua : mub;
}

/* ------------------------------------------------------------------ one contact's force
 * Eq. 1a with f = sqrt(R delta) and the Hertz set of reading O2/O3:
 *   S_n = 2 E* sqrt(R delta), k_n = 2/3 S_n, c_n = 2 sqrt(5/6) beta sqrt(S_n m),
 *   F_n = k_n delta n - c_n (v_rel . n) n                  (no tension clamp, O8)
 * Eq. 3a-3b: u' = u_t + h v_t ; u'_t = u' - (u'.n) n
 * Eq. 1b with k_t = 8 G* sqrt(R delta), c_t = 2 sqrt(5/6) beta sqrt(k_t m):
 *   trial F~ = -k_t u'_t - c_t v_t
 * Eq. 3c, reading O7: if |F~| <= mu |F_n| keep it and u_t = u'_t; else
 *   u_t = (mu|F_n|/k_t) u'_t/|u'_t|, F_t = -mu |F_n| u'_t/|u'_t| (0 if |u'_t| = 0).
 * mu = 0 gives F_t = 0, u_t = 0.  delta <= 0 gives F = 0, u_t = 0 (O9).
 * Forces are on body j (b); v_rel = v_j - v_i (Eq. 2a), n points i -> j (O1). */
void orc_contact_force(double e_star, double g_star, double beta, double mu, double r_bar, double m_bar,
                       double h, double delta, const double n[3], const double v_rel[3],
                       const double ut[3], double fn[3], double ft[3], double ut_new[3]) {
  int d;
  for (d = 0; d < 3; ++d) fn[d] = ft[d] = ut_new[d] = 0.0;
  if (!(delta > 0.0)) return;
  double sq = sqrt(r_bar * delta);
  double S_n = 2.0 * e_star * sq;
  double k_n = (2.0 / 3.0) * S_n;
  double c_n = 2.0 * sqrt(5.0 / 6.0) * beta * sqrt(S_n * m_bar);
  double vn = dot(v_rel, n);
  double fn_s = k_n * delta - c_n * vn;
  for (d = 0; d < 3; ++d) fn[d] = fn_s * n[d];
  if (mu == 0.0) return;
  double vt[3], up[3], upt[3], trial[3];
  for (d = 0; d < 3; ++d) vt[d] = v_rel[d] - vn * n[d];
  for (d = 0; d < 3; ++d) up[d] = ut[d] + h * vt[d];
  double upn = dot(up, n);
  for (d = 0; d < 3; ++d) upt[d] = up[d] - upn * n[d];
  double k_t = 8.0 * g_star * sq;
  double c_t = 2.0 * sqrt(5.0 / 6.0) * beta * sqrt(k_t * m_bar);
  for (d = 0; d < 3; ++d) trial[d] = -k_t * upt[d] - c_t * vt[d];
  double fn_mag = sqrt(dot(fn, fn));
  double cap = mu * fn_mag;
  double tmag = sqrt(dot(trial, trial));
  if (tmag <= cap) {
    for (d = 0; d < 3; ++d) {
      ft[d] = trial[d];
      ut_new[d] = upt[d];
    }
    return;
  }
  double umag = sqrt(dot(upt, upt));
  if (umag > 0.0) {
    for (d = 0; d < 3; ++d) {
      double dir = upt[d] / umag;
      ut_new[d] = (cap / k_t) * dir;
      ft[d] = -cap * dir;
    }
  }
}

/* ------------------------------------------------------------------ triangles (NEXT-3)
 * Closest point of triangle (a, b, c) to p by its Voronoi regions (vertex, edge, face), the
 * textbook construction ("closest point on the triangle (face, edge, or vertex
 * region)"), in the fixed operation order of DESIGN.md R25: dot products (x x' + y y') + z z',
 * no fused multiply-add (the library is compiled with -ffp-contract=off). */
static double dot3(const double* u, const double* v) { return (u[0] * v[0] + u[1] * v[1]) + u[2] * v[2]; }

/* returns the region of the closest point: TRI_FACE, TRI_EDGE_AB/AC/BC, TRI_VERT_A/B/C */
enum { TRI_FACE = 0, TRI_EDGE_AB = 1, TRI_EDGE_AC = 2, TRI_EDGE_BC = 3, TRI_VERT_A = 4, TRI_VERT_B = 5, TRI_VERT_C = 6 };
int orc_closest_on_triangle(const double p[3], const double a[3], const double b[3], const double c[3],
                            double out[3]) {
  double ab[3], ac[3], ap[3], bp[3], cp[3];
  int d;
  for (d = 0; d < 3; ++d) {
    ab[d] = b[d] - a[d];
    ac[d] = c[d] - a[d];
    ap[d] = p[d] - a[d];
  }
  double d1 = dot3(ab, ap), d2 = dot3(ac, ap);
  if (d1 <= 0.0 && d2 <= 0.0) { /* vertex a */
    for (d = 0; d < 3; ++d) out[d] = a[d];
    return TRI_VERT_A;
  }
  for (d = 0; d < 3; ++d) bp[d] = p[d] - b[d];
  double d3 = dot3(ab, bp), d4 = dot3(ac, bp);
  if (d3 >= 0.0 && d4 <= d3) { /* vertex b */
    for (d = 0; d < 3; ++d) out[d] = b[d];
    return TRI_VERT_B;
  }
  double vc = d1 * d4 - d3 * d2;
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) { /* edge ab */
    double v = d1 / (d1 - d3);
    for (d = 0; d < 3; ++d) out[d] = a[d] + v * ab[d];
    return TRI_EDGE_AB;
  }
  for (d = 0; d < 3; ++d) cp[d] = p[d] - c[d];
  double d5 = dot3(ab, cp), d6 = dot3(ac, cp);
  if (d6 >= 0.0 && d5 <= d6) { /* vertex c */
    for (d = 0; d < 3; ++d) out[d] = c[d];
    return TRI_VERT_C;
  }
  double vb = d5 * d2 - d1 * d6;
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) { /* edge ac */
    double w = d2 / (d2 - d6);
    for (d = 0; d < 3; ++d) out[d] = a[d] + w * ac[d];
    return TRI_EDGE_AC;
  }
  double va = d3 * d6 - d5 * d4;
  double e43 = d4 - d3, e56 = d5 - d6;
  if (va <= 0.0 && e43 >= 0.0 && e56 >= 0.0) { /* edge bc */
    double w = e43 / (e43 + e56);
    for (d = 0; d < 3; ++d) out[d] = b[d] + w * (c[d] - b[d]);
    return TRI_EDGE_BC;
  }
  double denom = 1.0 / ((va + vb) + vc); /* face */
  double v = vb * denom, w = vc * denom;
  for (d = 0; d < 3; ++d) out[d] = (a[d] + ab[d] * v) + ac[d] * w;
  return TRI_FACE;
}

/* world vertices of every triangle: x = X + R(q) x_body (the sphere-centre arithmetic, R22) */
static void mesh_world(orc_sys* s) {
  int64_t t;
  int k;
  for (t = 0; t < s->n_tri; ++t) {
    int m = s->tri_mesh[t];
    double R[9], v[3];
    quat_to_R(s->mQ + 4 * m, R);
    for (k = 0; k < 3; ++k) {
      mat_vec(R, s->tri_body + 9 * t + 3 * k, v);
      s->tri_world[9 * t + 3 * k] = s->mX[3 * m] + v[0];
      s->tri_world[9 * t + 3 * k + 1] = s->mX[3 * m + 1] + v[1];
      s->tri_world[9 * t + 3 * k + 2] = s->mX[3 * m + 2] + v[2];
    }
  }
}

/* the rotation of one step, h |w| about w/|w| (the exponential map of the clump update, R12) */
static void mesh_step_quat(double h, const double* w, double* qs) {
  double wn = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  qs[0] = 1.0;
  qs[1] = qs[2] = qs[3] = 0.0;
  if (wn > 0.0) {
    double half = 0.5 * (h * wn);
    double sn = sin(half) / wn;
    qs[0] = cos(half);
    qs[1] = w[0] * sn;
    qs[2] = w[1] * sn;
    qs[3] = w[2] * sn;
  }
}

static void mesh_advance(orc_sys* s) {
  int m, d;
  for (m = 0; m < s->n_mesh; ++m) {
    double* X = s->mX + 3 * m;
    double* q = s->mQ + 4 * m;
    const double* a = s->mQs + 4 * m;
    for (d = 0; d < 3; ++d) X[d] = X[d] + s->h * s->mV[3 * m + d];
    double w1 = a[0], x1 = a[1], y1 = a[2], z1 = a[3];
    double w2 = q[0], x2 = q[1], y2 = q[2], z2 = q[3];
    double nq[4];
    nq[0] = w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2;
    nq[1] = w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2;
    nq[2] = w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2;
    nq[3] = w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2;
    double nrm = sqrt(nq[0] * nq[0] + nq[1] * nq[1] + nq[2] * nq[2] + nq[3] * nq[3]);
    for (d = 0; d < 4; ++d) q[d] = nq[d] / nrm;
  }
}

/* One contact per surface feature (R26): the closest point of a sphere to a triangle
 * lies on its face, one of its edges or one of its vertices.  A face contact always counts; an
 * edge contact counts unless the sphere's set holds a face contact on a triangle of the same mesh
 * containing that edge, or the same edge reached from a lower-index triangle; a vertex contact
 * counts unless there is a face or edge contact (same mesh) containing that vertex, or the same
 * vertex from a lower-index triangle.  So a sphere on a flat mesh is pushed once, however the
 * mesh is triangulated.  Contacts that do not count get F = 0 and u_t = 0 (as delta <= 0). */
static int tri_has(const orc_sys* s, int64_t t, int64_t v) {
  return s->tri_vid[3 * t] == v || s->tri_vid[3 * t + 1] == v || s->tri_vid[3 * t + 2] == v;
}

static void tri_feature(const orc_sys* s, int64_t t, int region, int* kind, int64_t* u, int64_t* v) {
  const int64_t* id = s->tri_vid + 3 * t;
  static const int ea[4] = {0, 0, 0, 1}, eb[4] = {0, 1, 2, 2};
  if (region == TRI_FACE) {
    *kind = 2;
    *u = *v = t;
  } else if (region <= TRI_EDGE_BC) {
    int64_t x = id[ea[region]], y = id[eb[region]];
    *kind = 1;
    *u = x < y ? x : y;
    *v = x < y ? y : x;
  } else {
    *kind = 0;
    *u = *v = id[region - TRI_VERT_A];
  }
}

static int mesh_contact_active(const orc_sys* s, int64_t k, const int* region) {
  const contact* C = s->con;
  int64_t lo = k, hi = k, j;
  while (lo > 0 && C[lo - 1].ka == C[k].ka) --lo;
  while (hi + 1 < s->nc && C[hi + 1].ka == C[k].ka) ++hi;
  int64_t t = -1 - MAX_PLANES - C[k].sb;
  int kind, kj;
  int64_t u, v, uj, vj;
  tri_feature(s, t, region[k], &kind, &u, &v);
  if (kind == 2) return 1;
  for (j = lo; j <= hi; ++j) {
    if (j == k || C[j].sb > -1 - MAX_PLANES) continue;
    int64_t tj = -1 - MAX_PLANES - C[j].sb;
    if (s->tri_mesh[tj] != s->tri_mesh[t]) continue;
    tri_feature(s, tj, region[j], &kj, &uj, &vj);
    if (kind == 1) {
      if (kj == 2 && tri_has(s, tj, u) && tri_has(s, tj, v)) return 0;
      if (kj == 1 && uj == u && vj == v && tj < t) return 0;
    } else {
      if (kj == 2 && tri_has(s, tj, u)) return 0;
      if (kj == 1 && (uj == u || vj == u)) return 0;
      if (kj == 0 && uj == u && tj < t) return 0;
    }
  }
  return 1;
}

int orc_add_mesh(orc_sys* s, int64_t n_tri, const double* verts, int material, const double X[3],
                 const double q[4], const double v[3], const double w[3]) {
  if (n_tri < 1 || material < 0 || material >= s->n_mat) return ORC_ERR_ARG;
  int m = s->n_mesh++;
  int64_t t0 = s->n_tri, t;
  s->n_tri += n_tri;
  s->mX = (double*)realloc(s->mX, sizeof(double) * 3 * s->n_mesh);
  s->mQ = (double*)realloc(s->mQ, sizeof(double) * 4 * s->n_mesh);
  s->mV = (double*)realloc(s->mV, sizeof(double) * 3 * s->n_mesh);
  s->mW = (double*)realloc(s->mW, sizeof(double) * 3 * s->n_mesh);
  s->mQs = (double*)realloc(s->mQs, sizeof(double) * 4 * s->n_mesh);
  s->mF = (double*)realloc(s->mF, sizeof(double) * 3 * s->n_mesh);
  s->mT = (double*)realloc(s->mT, sizeof(double) * 3 * s->n_mesh);
  s->mmat = (int32_t*)realloc(s->mmat, sizeof(int32_t) * s->n_mesh);
  s->tri_mesh = (int32_t*)realloc(s->tri_mesh, sizeof(int32_t) * s->n_tri);
  s->tri_body = (double*)realloc(s->tri_body, sizeof(double) * 9 * s->n_tri);
  s->tri_world = (double*)realloc(s->tri_world, sizeof(double) * 9 * s->n_tri);
  s->tri_vid = (int64_t*)realloc(s->tri_vid, sizeof(int64_t) * 3 * s->n_tri);
  if (!s->mX || !s->mQ || !s->mV || !s->mW || !s->mQs || !s->mF || !s->mT || !s->mmat || !s->tri_mesh ||
      !s->tri_body || !s->tri_world || !s->tri_vid)
    abort();
  s->mmat[m] = material;
  for (t = 0; t < n_tri; ++t) s->tri_mesh[t0 + t] = m;
  memcpy(s->tri_body + 9 * t0, verts, sizeof(double) * 9 * n_tri);
  /* topology: a vertex id is the first (triangle, corner) of the mesh with bitwise-equal body
   * coordinates (plain O(n^2) scan) */
  for (t = 0; t < 3 * n_tri; ++t) {
    const double* v = verts + 3 * t;
    int64_t u;
    for (u = 0; u <= t; ++u)
      if (memcmp(verts + 3 * u, v, sizeof(double) * 3) == 0) break;
    s->tri_vid[3 * t0 + t] = 3 * t0 + u;
  }
  memset(s->mF + 3 * m, 0, sizeof(double) * 3);
  memset(s->mT + 3 * m, 0, sizeof(double) * 3);
  return orc_set_mesh_motion(s, m, X, q, v, w) == ORC_OK ? m : ORC_ERR_ARG;
}

int orc_set_mesh_motion(orc_sys* s, int m, const double X[3], const double q[4], const double v[3],
                        const double w[3]) {
  if (m < 0 || m >= s->n_mesh) return ORC_ERR_ARG;
  memcpy(s->mX + 3 * m, X, sizeof(double) * 3);
  memcpy(s->mQ + 4 * m, q, sizeof(double) * 4);
  memcpy(s->mV + 3 * m, v, sizeof(double) * 3);
  memcpy(s->mW + 3 * m, w, sizeof(double) * 3);
  mesh_step_quat(s->h, w, s->mQs + 4 * m);
  return ORC_OK;
}

int orc_get_mesh(const orc_sys* s, int m, double X[3], double q[4], double force[3], double torque[3]) {
  if (m < 0 || m >= s->n_mesh) return ORC_ERR_ARG;
  if (X) memcpy(X, s->mX + 3 * m, sizeof(double) * 3);
  if (q) memcpy(q, s->mQ + 4 * m, sizeof(double) * 4);
  if (force) memcpy(force, s->mF + 3 * m, sizeof(double) * 3);
  if (torque) memcpy(torque, s->mT + 3 * m, sizeof(double) * 3);
  return ORC_OK;
}

/* ------------------------------------------------------------------ lifecycle */
orc_sys* orc_create(double h, const double gravity[3], double margin, const double dom_lo[3],
                    const double dom_hi[3], int n_mat, const double* mat4, int n_tmpl, const int32_t* ncomp,
                    const double* offs, const double* rad, const int32_t* cmat, const double* mass,
                    const double* inertia, int n_planes, const double* plane_pt, const double* plane_n,
                    const int32_t* plane_mat, int detect) {
  orc_sys* s = (orc_sys*)xcalloc(1, sizeof(orc_sys));
  int t, d;
  s->h = h;
  s->margin = margin;
  for (d = 0; d < 3; ++d) {
    s->g[d] = gravity[d];
    s->lo[d] = dom_lo[d];
    s->hi[d] = dom_hi[d];
  }
  s->n_mat = n_mat;
  s->mat = (double*)xcalloc(4 * n_mat, sizeof(double));
  memcpy(s->mat, mat4, sizeof(double) * 4 * n_mat);
  s->n_tmpl = n_tmpl;
  s->ncomp = (int32_t*)xcalloc(n_tmpl, sizeof(int32_t));
  s->coff = (int32_t*)xcalloc(n_tmpl + 1, sizeof(int32_t));
  int tot = 0;
  for (t = 0; t < n_tmpl; ++t) {
    s->ncomp[t] = ncomp[t];
    s->coff[t] = tot;
    tot += ncomp[t];
  }
  s->coff[n_tmpl] = tot;
  s->offs = (double*)xcalloc(3 * tot, sizeof(double));
  s->rad = (double*)xcalloc(tot, sizeof(double));
  s->cmat = (int32_t*)xcalloc(tot, sizeof(int32_t));
  memcpy(s->offs, offs, sizeof(double) * 3 * tot);
  memcpy(s->rad, rad, sizeof(double) * tot);
  memcpy(s->cmat, cmat, sizeof(int32_t) * tot);
  s->mass = (double*)xcalloc(n_tmpl, sizeof(double));
  s->inertia = (double*)xcalloc(3 * n_tmpl, sizeof(double));
  memcpy(s->mass, mass, sizeof(double) * n_tmpl);
  memcpy(s->inertia, inertia, sizeof(double) * 3 * n_tmpl);
  s->n_planes = n_planes;
  s->ppt = (double*)xcalloc(3 * n_planes, sizeof(double));
  s->pn = (double*)xcalloc(3 * n_planes, sizeof(double));
  s->pmat = (int32_t*)xcalloc(n_planes, sizeof(int32_t));
  if (n_planes) {
    memcpy(s->ppt, plane_pt, sizeof(double) * 3 * n_planes);
    memcpy(s->pn, plane_n, sizeof(double) * 3 * n_planes);
    memcpy(s->pmat, plane_mat, sizeof(int32_t) * n_planes);
  }
  s->detect = detect;
  s->cd_every = 1;
  s->since_rebuild = 0;
  s->n_pend = -1;
  return s;
}

static void free_state(orc_sys* s) {
  free(s->gid); free(s->tid); free(s->X); free(s->Q); free(s->V); free(s->W);
  free(s->Fc); free(s->Tc);
  free(s->s_clump); free(s->s_comp); free(s->s_key); free(s->s_pos); free(s->s_rad);
  s->s_rad = NULL;
  s->gid = NULL; s->tid = NULL; s->X = s->Q = s->V = s->W = s->Fc = s->Tc = NULL;
  s->s_clump = NULL; s->s_comp = NULL; s->s_key = NULL; s->s_pos = NULL;
}

void orc_destroy(orc_sys* s) {
  if (!s) return;
  free_state(s);
  free(s->mat); free(s->ncomp); free(s->coff); free(s->offs); free(s->rad); free(s->cmat);
  free(s->mass); free(s->inertia); free(s->ppt); free(s->pn); free(s->pmat);
  free(s->hist); free(s->con); free(s->pend);
  free(s->mX); free(s->mQ); free(s->mV); free(s->mW); free(s->mQs); free(s->mF); free(s->mT);
  free(s->mmat); free(s->tri_mesh); free(s->tri_body); free(s->tri_world); free(s->tri_vid);
  free(s);
}

int orc_set_state(orc_sys* s, int64_t n, const int64_t* gid, const int32_t* tid, const double* pos,
                  const double* quat, const double* vel, const double* omega) {
  int64_t c;
  free_state(s);
  s->n = n;
  s->gid = (int64_t*)xcalloc(n, sizeof(int64_t));
  s->tid = (int32_t*)xcalloc(n, sizeof(int32_t));
  s->X = (double*)xcalloc(3 * n, sizeof(double));
  s->Q = (double*)xcalloc(4 * n, sizeof(double));
  s->V = (double*)xcalloc(3 * n, sizeof(double));
  s->W = (double*)xcalloc(3 * n, sizeof(double));
  s->Fc = (double*)xcalloc(3 * n, sizeof(double));
  s->Tc = (double*)xcalloc(3 * n, sizeof(double));
  memcpy(s->gid, gid, sizeof(int64_t) * n);
  memcpy(s->tid, tid, sizeof(int32_t) * n);
  memcpy(s->X, pos, sizeof(double) * 3 * n);
  memcpy(s->Q, quat, sizeof(double) * 4 * n);
  memcpy(s->V, vel, sizeof(double) * 3 * n);
  memcpy(s->W, omega, sizeof(double) * 3 * n);
  int64_t ns = 0;
  for (c = 0; c < n; ++c) {
    if (tid[c] < 0 || tid[c] >= s->n_tmpl) {
      snprintf(s->err, sizeof s->err, "clump %lld: bad template id %d", (long long)gid[c], tid[c]);
      return ORC_ERR_ARG;
    }
    ns += s->ncomp[tid[c]];
  }
  s->ns = ns;
  s->s_clump = (int64_t*)xcalloc(ns, sizeof(int64_t));
  s->s_comp = (int32_t*)xcalloc(ns, sizeof(int32_t));
  s->s_key = (int64_t*)xcalloc(ns, sizeof(int64_t));
  s->s_pos = (double*)xcalloc(3 * ns, sizeof(double));
  s->s_rad = (double*)xcalloc(ns, sizeof(double));
  int64_t k = 0;
  for (c = 0; c < n; ++c) {
    int j;
    for (j = 0; j < s->ncomp[tid[c]]; ++j) {
      s->s_clump[k] = c;
      s->s_comp[k] = j;
      s->s_key[k] = gid[c] * KEY_STRIDE + j;
      s->s_rad[k] = s->rad[s->coff[tid[c]] + j];
      ++k;
    }
  }
  s->nh = 0;
  s->nc = 0;
  s->since_rebuild = 0;
  s->n_pend = -1;
  return ORC_OK;
}

/* contact-set rebuild cadence: the set is rebuilt every k steps, counted from the
 * next step */
int orc_set_cd_every(orc_sys* s, int k) {
  if (k < 1) return ORC_ERR_ARG;
  s->cd_every = k;
  s->since_rebuild = 0;
  s->n_pend = -1;
  return ORC_OK;
}

/* overlapped detection ("in the shadow"; NEXT-2): with k >= 2 the set for the next
 * window is detected from the sphere positions of the second step of the current window and
 * adopted at the next window start, so the detection can run concurrently with the k - 1
 * force steps in between.  The margin must then cover 2k - 2 steps of motion. */
int orc_set_overlap(orc_sys* s, int on) {
  if (on && s->cd_every < 2) return ORC_ERR_ARG;
  s->overlap = on ? 1 : 0;
  s->since_rebuild = 0;
  s->n_pend = -1;
  return ORC_OK;
}

int orc_get_state(const orc_sys* s, double* pos, double* quat, double* vel, double* omega) {
  if (pos) memcpy(pos, s->X, sizeof(double) * 3 * s->n);
  if (quat) memcpy(quat, s->Q, sizeof(double) * 4 * s->n);
  if (vel) memcpy(vel, s->V, sizeof(double) * 3 * s->n);
  if (omega) memcpy(omega, s->W, sizeof(double) * 3 * s->n);
  return ORC_OK;
}

static int cmp_hist(const void* A, const void* B) {
  const hist_rec* a = (const hist_rec*)A;
  const hist_rec* b = (const hist_rec*)B;
  if (a->ka != b->ka) return a->ka < b->ka ? -1 : 1;
  if (a->kb != b->kb) return a->kb < b->kb ? -1 : 1;
  return 0;
}

int orc_set_history(orc_sys* s, int64_t n, const int64_t* ka, const int64_t* kb, const double* ut) {
  int64_t i;
  free(s->hist);
  s->hist = (hist_rec*)xcalloc(n, sizeof(hist_rec));
  for (i = 0; i < n; ++i) {
    if (!(ka[i] < kb[i])) {
      snprintf(s->err, sizeof s->err, "history key %lld must be < %lld", (long long)ka[i], (long long)kb[i]);
      return ORC_ERR_ARG;
    }
    s->hist[i].ka = ka[i];
    s->hist[i].kb = kb[i];
    memcpy(s->hist[i].ut, ut + 3 * i, sizeof(double) * 3);
  }
  qsort(s->hist, n, sizeof(hist_rec), cmp_hist);
  s->nh = n;
  s->since_rebuild = 0; /* a new history is read by a rebuild */
  s->n_pend = -1;
  return ORC_OK;
}

/* ------------------------------------------------------------------ contact set
 * Candidates (reading O14): sphere pairs of different clumps (O15) with
 *   dx*dx+dy*dy+dz*dz <= s*s,  s = (r_a + r_b) + margin,  d = c_b - c_a
 * and (sphere, plane) pairs with (r_a + margin) - (c_a - p_w).n_w >= 0. */
static void push_contact(orc_sys* s, int64_t sa, int64_t sb) {
  if (s->nc == s->cap) {
    s->cap = s->cap ? 2 * s->cap : 1024;
    s->con = (contact*)realloc(s->con, sizeof(contact) * s->cap);
    if (!s->con) abort();
  }
  contact* c = &s->con[s->nc++];
  memset(c, 0, sizeof *c);
  if (sb >= 0 && s->s_key[sb] < s->s_key[sa]) {
    int64_t t = sa;
    sa = sb;
    sb = t;
  }
  c->sa = sa;
  c->sb = sb;
  c->ka = s->s_key[sa];
  c->kb = sb >= 0 ? s->s_key[sb] : WALL_KEY(-1 - sb);
}

static int sphere_pair_candidate(const orc_sys* s, int64_t a, int64_t b) {
  const double* ca = s->s_pos + 3 * a;
  const double* cb = s->s_pos + 3 * b;
  double dx = cb[0] - ca[0], dy = cb[1] - ca[1], dz = cb[2] - ca[2];
  double ra = s->s_rad[a];
  double rb = s->s_rad[b];
  double sum = (ra + rb) + s->margin;
  return dx * dx + dy * dy + dz * dz <= sum * sum;
}

static double sphere_radius(const orc_sys* s, int64_t a) { return s->s_rad[a]; }

static void detect_brute(orc_sys* s) {
  int64_t a, b;
  for (a = 0; a < s->ns; ++a)
    for (b = a + 1; b < s->ns; ++b)
      if (s->s_clump[a] != s->s_clump[b] && sphere_pair_candidate(s, a, b)) push_contact(s, a, b);
}

/* simple uniform grid: spheres binned by centre into cells of side 2 r_min + margin.  Each
 * unordered pair is tested once, from its larger sphere (ties: lower index), so sphere a scans
 * the cells within its reach 2 r_a + margin (>= r_a + r_b + margin for every r_b <= r_a), with
 * the same predicate as the brute force. */
static void detect_grid(orc_sys* s) {
  double rmin = INFINITY, lo[3], hi[3];
  int64_t a;
  int d, t;
  for (t = 0; t < s->coff[s->n_tmpl]; ++t) {

    if (s->rad[t] < rmin) rmin = s->rad[t];
  }
  double cell = (2.0 * rmin + s->margin) * (1.0 + 1e-6);
  for (d = 0; d < 3; ++d) {
    lo[d] = INFINITY;
    hi[d] = -INFINITY;
  }
  for (a = 0; a < s->ns; ++a)
    for (d = 0; d < 3; ++d) {
      double v = s->s_pos[3 * a + d];
      if (v < lo[d]) lo[d] = v;
      if (v > hi[d]) hi[d] = v;
    }
  int64_t dim[3];
  for (d = 0; d < 3; ++d) dim[d] = (int64_t)floor((hi[d] - lo[d]) / cell) + 1;
  int64_t ncell = dim[0] * dim[1] * dim[2];
  int64_t* cstart = (int64_t*)xcalloc(ncell + 1, sizeof(int64_t));
  int64_t* cidx = (int64_t*)xcalloc(s->ns, sizeof(int64_t));
  int64_t* items = (int64_t*)xcalloc(s->ns, sizeof(int64_t));
  int64_t* cc = (int64_t*)xcalloc(3 * s->ns, sizeof(int64_t));
  for (a = 0; a < s->ns; ++a) {
    for (d = 0; d < 3; ++d) {
      int64_t k = (int64_t)floor((s->s_pos[3 * a + d] - lo[d]) / cell);
      if (k < 0) k = 0;
      if (k >= dim[d]) k = dim[d] - 1;
      cc[3 * a + d] = k;
    }
    cidx[a] = (cc[3 * a + 2] * dim[1] + cc[3 * a + 1]) * dim[0] + cc[3 * a];
    cstart[cidx[a] + 1]++;
  }
  for (a = 0; a < ncell; ++a) cstart[a + 1] += cstart[a];
  int64_t* fill = (int64_t*)xcalloc(ncell, sizeof(int64_t));
  for (a = 0; a < s->ns; ++a) items[cstart[cidx[a]] + fill[cidx[a]]++] = a;
  for (a = 0; a < s->ns; ++a) {
    int64_t x, y, z;
    /* |floor(u) - floor(v)| <= ceil(|u - v|): bins within ceil(reach / cell) hold every partner
     * (the 1e-9 relative slack covers the rounding of the bin coordinates) */
    double ra = s->s_rad[a];
    int64_t reach = (int64_t)ceil((2.0 * ra + s->margin) * (1.0 + 1e-9) / cell);
    for (z = cc[3 * a + 2] - reach; z <= cc[3 * a + 2] + reach; ++z) {
      if (z < 0 || z >= dim[2]) continue;
      for (y = cc[3 * a + 1] - reach; y <= cc[3 * a + 1] + reach; ++y) {
        if (y < 0 || y >= dim[1]) continue;
        for (x = cc[3 * a] - reach; x <= cc[3 * a] + reach; ++x) {
          if (x < 0 || x >= dim[0]) continue;
          int64_t cid = (z * dim[1] + y) * dim[0] + x, k;
          for (k = cstart[cid]; k < cstart[cid + 1]; ++k) {
            int64_t b = items[k];
            double rb = s->s_rad[b];
            if (rb > ra || (rb == ra && b <= a)) continue;
            if (s->s_clump[a] != s->s_clump[b] && sphere_pair_candidate(s, a, b)) push_contact(s, a, b);
          }
        }
      }
    }
  }
  free(cstart); free(cidx); free(items); free(cc); free(fill);
}

/* sphere-triangle candidates: |c - closest(c, T)|^2 <= (r + margin)^2 (R25) */
static void detect_meshes(orc_sys* s) {
  int64_t a, t;
  for (a = 0; a < s->ns; ++a) {
    const double* c = s->s_pos + 3 * a;
    double r = sphere_radius(s, a);
    for (t = 0; t < s->n_tri; ++t) {
      const double* T = s->tri_world + 9 * t;
      double q[3];
      orc_closest_on_triangle(c, T, T + 3, T + 6, q);
      double dx = c[0] - q[0], dy = c[1] - q[1], dz = c[2] - q[2];
      double sr = r + s->margin;
      if ((dx * dx + dy * dy) + dz * dz <= sr * sr) push_contact(s, a, -1 - MAX_PLANES - t);
    }
  }
}

static void detect_planes(orc_sys* s) {
  int64_t a;
  int p;
  for (a = 0; a < s->ns; ++a) {
    const double* c = s->s_pos + 3 * a;
    double r = sphere_radius(s, a);
    for (p = 0; p < s->n_planes; ++p) {
      const double* pp = s->ppt + 3 * p;
      const double* nw = s->pn + 3 * p;
      double dd = (c[0] - pp[0]) * nw[0] + (c[1] - pp[1]) * nw[1] + (c[2] - pp[2]) * nw[2];
      if ((r + s->margin) - dd >= 0.0) push_contact(s, a, -1 - (int64_t)p);
    }
  }
}

static int cmp_contact(const void* A, const void* B) {
  const contact* a = (const contact*)A;
  const contact* b = (const contact*)B;
  if (a->ka != b->ka) return a->ka < b->ka ? -1 : 1;
  if (a->kb != b->kb) return a->kb < b->kb ? -1 : 1;
  return 0;
}

/* ------------------------------------------------------------------ per-sphere canonical sums */
typedef struct {
  int64_t partner;
  double f[3], r[3];
} entry;

static int cmp_entry(const void* A, const void* B) {
  const entry* a = (const entry*)A;
  const entry* b = (const entry*)B;
  if (a->partner != b->partner) return a->partner < b->partner ? -1 : 1;
  return 0;
}

/* the candidate set of the current sphere positions, sorted by (key_a, key_b) */
static void detect_set(orc_sys* s) {
  s->nc = 0;
  int brute = s->detect == 0 || (s->detect < 0 && s->ns <= 10000);
  if (brute)
    detect_brute(s);
  else
    detect_grid(s);
  detect_meshes(s);
  detect_planes(s);
  qsort(s->con, s->nc, sizeof(contact), cmp_contact);
}

/* ------------------------------------------------------------------ the step */
static int one_step(orc_sys* s) {
  int64_t a, c, k;
  int d;
  double h = s->h;
  /* (1) sphere world centres c = X + R(q) o */
  for (a = 0; a < s->ns; ++a) {
    int64_t cl = s->s_clump[a];
    int32_t t = s->tid[cl];
    double R[9], o[3];
    quat_to_R(s->Q + 4 * cl, R);
    mat_vec(R, s->offs + 3 * (s->coff[t] + s->s_comp[a]), o);
    for (d = 0; d < 3; ++d) {
      double v = s->X[3 * cl + d] + o[d];
      s->s_pos[3 * a + d] = v;
      if (!(v >= s->lo[d] && v <= s->hi[d])) {
        snprintf(s->err, sizeof s->err, "sphere %lld of clump %lld left the domain at step %lld",
                 (long long)s->s_key[a], (long long)s->gid[cl], (long long)s->steps);
        return ORC_ERR_OUT_OF_DOMAIN;
      }
    }
  }
  /* (1b) mesh triangles at this step's mesh poses (NEXT-3) */
  mesh_world(s);
  /* (2) active contact set: rebuilt every cd_every steps from the margin-enlarged geometry
   * (P:142); cd_every = 1 is the "traditional way".  In between, the same set is
   * used and every member is re-evaluated at each step. */
  if (s->since_rebuild == 0) {
    if (s->overlap && s->n_pend >= 0) { /* adopt the set detected during the last window */
      free(s->con);
      s->con = s->pend;
      s->nc = s->cap = s->n_pend;
      s->pend = NULL;
      s->n_pend = -1;
    } else {
      detect_set(s);
    }
  } else if (s->overlap && s->since_rebuild == 1) {
    /* detect the next window's set from this step's positions, keep the current one */
    contact* cur = s->con;
    int64_t nc = s->nc, cap = s->cap;
    s->con = NULL;
    s->nc = 0;
    s->cap = 0;
    detect_set(s);
    free(s->pend);
    s->pend = s->con;
    s->n_pend = s->nc;
    s->con = cur;
    s->nc = nc;
    s->cap = cap;
  }
  s->since_rebuild = (s->since_rebuild + 1) % s->cd_every;
  /* (3) history carried for surviving keys, zero at birth */
  for (k = 0; k < s->nc; ++k) {
    hist_rec key, *hit;
    key.ka = s->con[k].ka;
    key.kb = s->con[k].kb;
    hit = (hist_rec*)bsearch(&key, s->hist, s->nh, sizeof(hist_rec), cmp_hist);
    for (d = 0; d < 3; ++d) s->con[k].ut[d] = hit ? hit->ut[d] : 0.0;
  }
  /* (4) per-contact kinematics (Eq. 2) and forces (Eqs. 1, 3) */
  int* mreg = NULL;
  char* mact = NULL;
  if (s->n_mesh) {
    memset(s->mF, 0, sizeof(double) * 3 * s->n_mesh);
    memset(s->mT, 0, sizeof(double) * 3 * s->n_mesh);
    mreg = (int*)xcalloc(s->nc, sizeof(int));
    mact = (char*)xcalloc(s->nc, 1);
    for (k = 0; k < s->nc; ++k)
      if (s->con[k].sb <= -1 - MAX_PLANES) {
        const double* T = s->tri_world + 9 * (-1 - MAX_PLANES - s->con[k].sb);
        double q[3];
        mreg[k] = orc_closest_on_triangle(s->s_pos + 3 * s->con[k].sa, T, T + 3, T + 6, q);
      }
    for (k = 0; k < s->nc; ++k)
      if (s->con[k].sb <= -1 - MAX_PLANES) mact[k] = (char)mesh_contact_active(s, k, mreg);
  }
  int64_t* n_ent = (int64_t*)xcalloc(s->ns + 1, sizeof(int64_t));
  for (k = 0; k < s->nc; ++k) {
    n_ent[s->con[k].sa]++;
    if (s->con[k].sb >= 0) n_ent[s->con[k].sb]++;
  }
  int64_t* e_off = (int64_t*)xcalloc(s->ns + 1, sizeof(int64_t));
  for (a = 0; a < s->ns; ++a) e_off[a + 1] = e_off[a] + n_ent[a];
  entry* ent = (entry*)xcalloc(e_off[s->ns], sizeof(entry));
  memset(n_ent, 0, sizeof(int64_t) * (s->ns + 1));
  for (k = 0; k < s->nc; ++k) {
    contact* C = &s->con[k];
    int64_t sa = C->sa, sb = C->sb;
    int64_t i = s->s_clump[sa];
    const double* ca = s->s_pos + 3 * sa;
    double ra = sphere_radius(s, sa);
    const double* mat_a = s->mat + 4 * s->cmat[s->coff[s->tid[i]] + s->s_comp[sa]];
    const double* mat_b;
    double n[3], p[3], delta, r_bar, m_bar;
    double Mi = s->mass[s->tid[i]];
    int64_t j = -1;
    int mesh = -1;
    if (sb <= -1 - MAX_PLANES) {
      /* sphere (a) on a mesh triangle (b): n from the sphere to its closest point on the
       * triangle, delta = r - |c - q|, R_bar = r and m_bar = M (the flat-wall limit),
       * contact point at the middle of the overlap as for walls (O6); the triangle moves with
       * its mesh: v_b = v_m + w_m x (p - X_m) */
      int64_t t = -1 - MAX_PLANES - sb;
      const double* T = s->tri_world + 9 * t;
      double q[3], dv[3];
      mesh = s->tri_mesh[t];
      orc_closest_on_triangle(ca, T, T + 3, T + 6, q);
      for (d = 0; d < 3; ++d) dv[d] = ca[d] - q[d];
      double dist = sqrt((dv[0] * dv[0] + dv[1] * dv[1]) + dv[2] * dv[2]);
      if (dist == 0.0) {
        snprintf(s->err, sizeof s->err, "sphere centre %lld on triangle %lld at step %lld", (long long)C->ka,
                 (long long)t, (long long)s->steps);
        free(n_ent); free(e_off); free(ent); free(mreg); free(mact);
        return ORC_ERR_DEGENERATE;
      }
      delta = ra - dist;
      for (d = 0; d < 3; ++d) n[d] = -(dv[d] / dist);
      for (d = 0; d < 3; ++d) p[d] = ca[d] + (ra - 0.5 * delta) * n[d];
      r_bar = ra;
      m_bar = Mi;
      mat_b = s->mat + 4 * s->mmat[mesh];
    } else if (sb >= 0) {
      j = s->s_clump[sb];
      const double* cb = s->s_pos + 3 * sb;
      double rb = sphere_radius(s, sb);
      double dv[3];
      for (d = 0; d < 3; ++d) dv[d] = cb[d] - ca[d];
      double dist = sqrt(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2]);
      if (dist == 0.0) {
        snprintf(s->err, sizeof s->err, "coincident sphere centres %lld/%lld at step %lld",
                 (long long)C->ka, (long long)C->kb, (long long)s->steps);
        free(n_ent); free(e_off); free(ent); free(mreg); free(mact);
        return ORC_ERR_DEGENERATE;
      }
      delta = (ra + rb) - dist;
      for (d = 0; d < 3; ++d) n[d] = dv[d] / dist;
      /* contact point: midpoint of the overlap segment (O6) */
      for (d = 0; d < 3; ++d) p[d] = 0.5 * (ca[d] + cb[d]) + 0.5 * (ra - rb) * n[d];
      r_bar = ra * rb / (ra + rb);
      double Mj = s->mass[s->tid[j]];
      m_bar = Mi * Mj / (Mi + Mj); /* clump masses (O5) */
      mat_b = s->mat + 4 * s->cmat[s->coff[s->tid[j]] + s->s_comp[sb]];
    } else {
      int pl = (int)(-1 - sb);
      const double* pp = s->ppt + 3 * pl;
      const double* nw = s->pn + 3 * pl;
      double dd = (ca[0] - pp[0]) * nw[0] + (ca[1] - pp[1]) * nw[1] + (ca[2] - pp[2]) * nw[2];
      delta = ra - dd;
      for (d = 0; d < 3; ++d) n[d] = -nw[d]; /* sphere (a) -> wall (b) */
      for (d = 0; d < 3; ++d) p[d] = ca[d] + (ra - 0.5 * delta) * n[d];
      r_bar = ra;   /* flat wall limit */
      m_bar = Mi;
      mat_b = s->mat + 4 * s->pmat[pl];
    }
    /* contact-point velocities (Eq. 2a), omega_world = R(q) Omega_body (O13) */
    double Ri[9], wi[3], ri[3], vi[3], vj[3] = {0, 0, 0}, rj[3] = {0, 0, 0}, tmp[3];
    quat_to_R(s->Q + 4 * i, Ri);
    mat_vec(Ri, s->W + 3 * i, wi);
    for (d = 0; d < 3; ++d) ri[d] = p[d] - s->X[3 * i + d];
    cross(wi, ri, tmp);
    for (d = 0; d < 3; ++d) vi[d] = s->V[3 * i + d] + tmp[d];
    if (j >= 0) {
      double Rj[9], wj[3];
      quat_to_R(s->Q + 4 * j, Rj);
      mat_vec(Rj, s->W + 3 * j, wj);
      for (d = 0; d < 3; ++d) rj[d] = p[d] - s->X[3 * j + d];
      cross(wj, rj, tmp);
      for (d = 0; d < 3; ++d) vj[d] = s->V[3 * j + d] + tmp[d];
    } else if (mesh >= 0) {
      for (d = 0; d < 3; ++d) rj[d] = p[d] - s->mX[3 * mesh + d];
      cross(s->mW + 3 * mesh, rj, tmp);
      for (d = 0; d < 3; ++d) vj[d] = s->mV[3 * mesh + d] + tmp[d];
    }
    double vrel[3];
    for (d = 0; d < 3; ++d) vrel[d] = vj[d] - vi[d];
    double pp4[4], fn[3], ft[3], un[3];
    orc_pair_params(mat_a, mat_b, pp4);
    orc_contact_force(pp4[0], pp4[1], pp4[2], pp4[3], r_bar, m_bar, h, delta, n, vrel, C->ut, fn, ft, un);
    if (mesh >= 0 && !mact[k])
      for (d = 0; d < 3; ++d) fn[d] = ft[d] = un[d] = 0.0; /* not this feature's contact (R26) */
    for (d = 0; d < 3; ++d) {
      C->F[d] = fn[d] + ft[d];
      C->p[d] = p[d];
      C->n[d] = n[d];
      C->ut[d] = un[d];
    }
    C->delta = delta;
    if (mesh >= 0) { /* reaction on the mesh, torque about its reference point */
      cross(rj, C->F, tmp);
      for (d = 0; d < 3; ++d) {
        s->mF[3 * mesh + d] += C->F[d];
        s->mT[3 * mesh + d] += tmp[d];
      }
    }
    /* entries: -F on a at r_i, +F on b at r_j (Eq. 4, reading O1/O11) */
    entry* ea = &ent[e_off[sa] + n_ent[sa]++];
    ea->partner = C->kb;
    for (d = 0; d < 3; ++d) {
      ea->f[d] = -C->F[d];
      ea->r[d] = ri[d];
    }
    if (sb >= 0) {
      entry* eb = &ent[e_off[sb] + n_ent[sb]++];
      eb->partner = C->ka;
      for (d = 0; d < 3; ++d) {
        eb->f[d] = C->F[d];
        eb->r[d] = rj[d];
      }
    }
  }
  /* (5) canonical reduction: per sphere in partner-key order, per clump in component order */
  for (c = 0; c < s->n; ++c)
    for (d = 0; d < 3; ++d) s->Fc[3 * c + d] = s->Tc[3 * c + d] = 0.0;
  for (a = 0; a < s->ns; ++a) {
    int64_t m = e_off[a + 1] - e_off[a];
    entry* E = ent + e_off[a];
    qsort(E, m, sizeof(entry), cmp_entry);
    double fs[3] = {0, 0, 0}, ts[3] = {0, 0, 0}, tq[3];
    for (k = 0; k < m; ++k) {
      cross(E[k].r, E[k].f, tq);
      for (d = 0; d < 3; ++d) {
        fs[d] += E[k].f[d];
        ts[d] += tq[d];
      }
    }
    int64_t cl = s->s_clump[a]; /* spheres are stored in component order */
    for (d = 0; d < 3; ++d) {
      s->Fc[3 * cl + d] += fs[d];
      s->Tc[3 * cl + d] += ts[d];
    }
  }
  free(n_ent); free(e_off); free(ent); free(mreg); free(mact);
  /* (6) integrate (Eq. 4a-4b; reading O11/O12): semi-implicit Euler */
  for (c = 0; c < s->n; ++c) {
    int32_t t = s->tid[c];
    double M = s->mass[t];
    const double* I = s->inertia + 3 * t;
    double R[9], F[3], tb[3];
    for (d = 0; d < 3; ++d) F[d] = s->Fc[3 * c + d] + M * s->g[d];
    quat_to_R(s->Q + 4 * c, R);
    mat_T_vec(R, s->Tc + 3 * c, tb);
    for (d = 0; d < 3; ++d) {
      s->Fc[3 * c + d] = F[d];
      s->Tc[3 * c + d] = tb[d];
      if (!isfinite(F[d]) || !isfinite(tb[d])) {
        snprintf(s->err, sizeof s->err, "non-finite wrench on clump %lld at step %lld", (long long)s->gid[c],
                 (long long)s->steps);
        return ORC_ERR_NONFINITE;
      }
    }
    double* V = s->V + 3 * c;
    double* X = s->X + 3 * c;
    double* W = s->W + 3 * c;
    double* q = s->Q + 4 * c;
    for (d = 0; d < 3; ++d) {
      V[d] = V[d] + h * (F[d] / M);
      X[d] = X[d] + h * V[d];
    }
    double L[3] = {I[0] * W[0], I[1] * W[1], I[2] * W[2]}, gyro[3];
    cross(W, L, gyro);
    for (d = 0; d < 3; ++d) W[d] = W[d] + h * ((tb[d] - gyro[d]) / I[d]);
    double wn = sqrt(W[0] * W[0] + W[1] * W[1] + W[2] * W[2]);
    double dq[4] = {1.0, 0.0, 0.0, 0.0};
    if (wn > 0.0) {
      double half = 0.5 * (h * wn);
      double sn = sin(half) / wn;
      dq[0] = cos(half);
      dq[1] = W[0] * sn;
      dq[2] = W[1] * sn;
      dq[3] = W[2] * sn;
    }
    double w1 = q[0], x1 = q[1], y1 = q[2], z1 = q[3];
    double w2 = dq[0], x2 = dq[1], y2 = dq[2], z2 = dq[3];
    double nq[4];
    nq[0] = w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2;
    nq[1] = w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2;
    nq[2] = w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2;
    nq[3] = w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2;
    double nrm = sqrt(nq[0] * nq[0] + nq[1] * nq[1] + nq[2] * nq[2] + nq[3] * nq[3]);
    for (d = 0; d < 4; ++d) q[d] = nq[d] / nrm;
  }
  /* (6b) prescribed mesh motion */
  mesh_advance(s);
  /* (7) this step's set and u_t become the history of the next */
  free(s->hist);
  s->hist = (hist_rec*)xcalloc(s->nc, sizeof(hist_rec));
  for (k = 0; k < s->nc; ++k) {
    s->hist[k].ka = s->con[k].ka;
    s->hist[k].kb = s->con[k].kb;
    memcpy(s->hist[k].ut, s->con[k].ut, sizeof(double) * 3);
  }
  s->nh = s->nc;
  s->steps++;
  return ORC_OK;
}

int orc_step(orc_sys* s, int64_t n_steps) {
  int64_t k;
  for (k = 0; k < n_steps; ++k) {
    int rc = one_step(s);
    if (rc) return rc;
  }
  return ORC_OK;
}

int64_t orc_num_contacts(const orc_sys* s) { return s->nc; }
int64_t orc_steps_done(const orc_sys* s) { return s->steps; }

int orc_get_contacts(const orc_sys* s, int64_t* ka, int64_t* kb, double* force_b, double* point,
                     double* normal, double* ut, double* delta) {
  int64_t k;
  int d;
  for (k = 0; k < s->nc; ++k) {
    const contact* C = &s->con[k];
    if (ka) ka[k] = C->ka;
    if (kb) kb[k] = C->kb;
    for (d = 0; d < 3; ++d) {
      if (force_b) force_b[3 * k + d] = C->F[d];
      if (point) point[3 * k + d] = C->p[d];
      if (normal) normal[3 * k + d] = C->n[d];
      if (ut) ut[3 * k + d] = C->ut[d];
    }
    if (delta) delta[k] = C->delta;
  }
  return ORC_OK;
}

int orc_get_wrench(const orc_sys* s, double* force, double* torque_body) {
  if (force) memcpy(force, s->Fc, sizeof(double) * 3 * s->n);
  if (torque_body) memcpy(torque_body, s->Tc, sizeof(double) * 3 * s->n);
  return ORC_OK;
}

const char* orc_last_error(const orc_sys* s) { return s->err; }
