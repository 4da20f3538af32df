/* oracle/dem_oracle.h — CPU fp64 ORACLE for the clump-DEM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA product
 * (paper_2307_03445_b200/csrc, include/dem.h), and includes none of them.
 *
 * What it computes: one explicit DEM step of PAPER.md Sec. 2.1 (Eqs. 1a-1e, 2a-2c,
 * 3a-3c, 4a-4b) for clumps of spheres, with the per-step ("traditional",
 * P:145) rebuild of the active contact set, in the readings listed in DESIGN.md
 * (SURVEY.md §8c, O1-O24).  Plain loops, fp64, compiled with -ffp-contract=off.
 *
 * Conventions (identical to include/dem.h, restated independently):
 *   sphere key = clump_gid*64 + component; plane key = INT64_MAX - plane_index;
 *   contact (a,b) has key_a < key_b; body i = a, body j = b; n points a->b;
 *   the computed force F acts on b, -F on a (reading O1).
 */
#ifndef DEM_ORACLE_H
#define DEM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_sys orc_sys;

/* error codes */
#define ORC_OK 0
#define ORC_ERR_ARG (-1)
#define ORC_ERR_OUT_OF_DOMAIN (-10)
#define ORC_ERR_NONFINITE (-11)
#define ORC_ERR_DEGENERATE (-12)

/* detect: 0 = brute force O(N^2), 1 = uniform grid, -1 = auto (brute if <= 10^4 spheres) */
orc_sys* orc_create(double h, const double gravity[3], double margin, const double dom_lo[3],
                    const double dom_hi[3], int n_mat, const double* mat4 /* E,nu,mu,cor per mat */,
                    int n_tmpl, const int32_t* ncomp, const double* offs, const double* rad,
                    const int32_t* cmat, const double* mass, const double* inertia, int n_planes,
                    const double* plane_pt, const double* plane_n, const int32_t* plane_mat, int detect);
void orc_destroy(orc_sys*);
int orc_set_state(orc_sys*, int64_t n, const int64_t* gid, const int32_t* tid, const double* pos,
                  const double* quat, const double* vel, const double* omega);
int orc_get_state(const orc_sys*, double* pos, double* quat, double* vel, double* omega);
int orc_set_history(orc_sys*, int64_t n, const int64_t* ka, const int64_t* kb, const double* ut);
int orc_step(orc_sys*, int64_t n_steps);
/* rebuild the contact set every k steps (margin set at creation), counted from the next step */
int orc_set_cd_every(orc_sys*, int k);
int orc_set_overlap(orc_sys*, int on);
int64_t orc_num_contacts(const orc_sys*);
/* contacts of the last step (set built from the state at that step's start), sorted by (ka,kb):
 * force on b, contact point, normal a->b, tangential history after the step, penetration. */
int orc_get_contacts(const orc_sys*, int64_t* ka, int64_t* kb, double* force_b, double* point,
                     double* normal, double* ut, double* delta);
/* per-clump force (world) and torque (body) applied in the last step, gravity included */
int orc_get_wrench(const orc_sys*, double* force, double* torque_body);
const char* orc_last_error(const orc_sys*);
int64_t orc_steps_done(const orc_sys*);
/* kinematic triangle meshes (NEXT-3): verts [9 n_tri] body frame; pose X, q (body -> world),
 * velocity v and angular velocity w (world, about X); returns the mesh index or < 0 */
int orc_add_mesh(orc_sys*, int64_t n_tri, const double* verts, int material, const double X[3], const double q[4],
                 const double v[3], const double w[3]);
int orc_set_mesh_motion(orc_sys*, int m, const double X[3], const double q[4], const double v[3], const double w[3]);
/* pose after the last step; force on the mesh and torque about X from the last step's contacts */
int orc_get_mesh(const orc_sys*, int m, double X[3], double q[4], double force[3], double torque[3]);
/* closest point of triangle (a, b, c) to p; returns its region: 0 face, 1-3 edge ab/ac/bc, 4-6 vertex a/b/c */
int orc_closest_on_triangle(const double p[3], const double a[3], const double b[3], const double c[3],
                            double out[3]);

/* single-contact building blocks, exposed for unit pins */
void orc_pair_params(const double* mat_a4, const double* mat_b4, double out4[4] /* E*, G*, beta, mu */);
void orc_contact_force(double e_star, double g_star, double beta, double mu, double r_bar, double m_bar,
                       double h, double delta, const double n[3], const double v_rel[3],
                       const double ut[3], double fn[3], double ft[3], double ut_new[3]);

#ifdef __cplusplus
}
#endif
#endif
