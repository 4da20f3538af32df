/* include/dem.h — C-ABI of the B200-native clump-DEM hot path (libdem_b200.so).
 *
 * The library advances a system of clumps — rigid unions of overlapping spheres
 * (Fig. 2 caption P:135) whose spheres each carry their own material
 * (E, nu, mu, CoR) — by explicit time steps of size h under gravity.
 * One dem_step = the per-step hot path of PAPER.md Sec. 2 in the "traditional"
 * per-step-rebuild mode:
 *   (a1) sphere world poses          c = X + R(q) o
 *   (a2) broad phase: multi-insert uniform-grid binning by counting sort
 *   (a3) narrow phase: directed per-sphere contact rows, sorted by partner key
 *   (a4) tangential-history remap by contact key
 *   (a5-a8) contact kinematics + Hertz-Mindlin forces, walls     (Eqs. 1a-3c)
 *   (a9) deterministic per-clump force/torque reduction           (Eq. 4 RHS)
 *   (a10) semi-implicit Euler of position and orientation         (Eq. 4a-4b)
 * The exact arithmetic and every reading of the paper is in DESIGN.md §3.
 *
 * Conventions
 *   - SI units, fp64 everywhere.  Quaternions (w,x,y,z), Hamilton product, body->world.
 *   - Clump velocity V is world-frame, angular velocity Omega is body-frame (principal axes).
 *   - Keys: sphere key = clump_gid * 64 + component (<= 64 components per template);
 *     plane key = INT64_MAX - plane_index.  A contact (key_a, key_b) has key_a < key_b; the
 *     normal n points from a to b, and the reported force is the force ON b (-F acts on a).
 *     u_t is oriented a->b (it changes sign if a and b are swapped).
 *   - Pointers: "host" arrays are caller-owned and only read/written during the call; the
 *     library never keeps a caller pointer.  Device memory is owned by the library and is
 *     obtained from params.alloc (e.g. the PyTorch caching allocator) or cudaMallocAsync.
 *   - Streams: all device work runs on the stream passed to dem_create (borrowed; it must
 *     outlive the system).  One system per host thread at a time; no global state.
 *   - Errors: argument errors are returned synchronously.  Device-detected errors (sphere out
 *     of domain, non-finite wrench, coincident centres) are latched in a device status word and
 *     returned by the next call that synchronises (dem_step returns after its last step has
 *     been checked); dem_last_error() names the clump/contact key and the step.  Capacity
 *     overflows (bins, contact rows) are handled internally by regrowing and re-running the
 *     aborted steps; a contact list is never silently truncated.
 *   - Environment (test and diagnosis hooks, read at dem_create / dem_step; off by default):
 *     DEM_FAULT_AHEAD_OVERFLOW=n  the next n ahead detections (overlapped cadence) report a
 *                                 capacity overflow (exercises the recovery path);
 *     DEM_DEBUG_SERIAL_DET=1      the force steps wait for an ahead detection (no overlap);
 *     DEM_DEBUG_LOG=1             capacity regrows are logged to stderr.
 */
#ifndef DEM_B200_H
#define DEM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DEM_OK = 0,
  DEM_ERR_INVALID_ARG = -1,
  DEM_ERR_CUDA = -2,
  DEM_ERR_OOM = -3,
  DEM_ERR_NCCL = -4,
  DEM_ERR_BAD_MATERIAL = -5,      /* E > 0, 0 <= nu < 0.5, mu >= 0, 0 < CoR <= 1   */
  DEM_ERR_BAD_TEMPLATE = -6,      /* 1..64 comps, r > 0, mass > 0, inertia > 0          */
  DEM_ERR_OUT_OF_DOMAIN = -10,    /* a sphere centre left [domain_lo, domain_hi]       */
  DEM_ERR_NONFINITE = -11,        /* non-finite wrench/state                          */
  DEM_ERR_DEGENERATE_CONTACT = -12, /* coincident sphere centres in a contact         */
  DEM_ERR_VMAX = -13,             /* cd_every > 1: a sphere moved more than margin/2 since the last
                                     contact-set rebuild; raise margin or lower cd_every */
  DEM_ERR_CAPACITY = -14,         /* a buffer could not be grown (device memory exhausted)   */
  DEM_ERR_REPARTITION = -15       /* distributed: an owned clump drifted beyond drift_max    */
} dem_status;

/* One sphere material.  Pair parameters of two materials follow DESIGN.md §3 R4:
 * 1/E* = sum (1-nu^2)/E, 1/G* = sum 2(2-nu)(1+nu)/E, CoR = min, mu = min. */
typedef struct {
  double E, nu, mu, cor;
} dem_material;

/* One clump template: component spheres in the principal body frame with the
 * COM at the origin; mass and principal inertia of the union are inputs (computed by the
 * caller, e.g. by voxelisation).  Arrays are read during dem_create only. */
typedef struct {
  int32_t n_comp;            /* 1..64 */
  const double* offset;      /* [3*n_comp] body-frame centres */
  const double* radius;      /* [n_comp] */
  const int32_t* material;   /* [n_comp] indices into the material table */
  double mass;               /* kg */
  double inertia[3];         /* principal moments, kg m^2 */
} dem_template;

/* A fixed analytic plane (flat-wall limit: R_bar = r, m_bar = clump mass). */
typedef struct {
  double point[3];
  double normal[3];          /* unit, pointing into the domain */
  int32_t material;
} dem_plane;

typedef void* (*dem_alloc_fn)(size_t bytes, void* ctx, void* stream);
typedef void (*dem_free_fn)(void* ptr, size_t bytes, void* ctx, void* stream);

typedef struct {
  double h;                  /* time step [s] */
  double gravity[3];         /* [m/s^2]; tilt it for inclines */
  double margin;             /* total contact-detection enlargement [m]; 0 for per-step rebuild */
  int32_t cd_every;          /* steps per contact-set rebuild; >= 1.  With cd_every > 1 the set is
                                built from spheres enlarged by margin/2 each and re-evaluated every step
                                (members with delta <= 0 get zero force); margin must cover the
                                relative motion over the window, e.g. 2 v_max h cd_every */
  double domain_lo[3], domain_hi[3]; /* every sphere centre must stay inside */
  double cell_size;          /* bin edge [m]; 0 = automatic */
  int32_t record_contacts;   /* 1: keep per-contact force/point/normal/delta for dem_get_contacts */
  dem_alloc_fn alloc;        /* NULL: cudaMallocAsync on the system stream.  Blocks must be 32-byte
                                aligned (the kernels move 32-byte records with 256-bit accesses); a
                                misaligned block fails the call that allocates it */
  dem_free_fn free;
  void* alloc_ctx;
  double entries_per_sphere; /* initial contact-row capacity per sphere (0 = 8); grown on overflow.  A
                                distributed rank regrows together with all ranks (the abort word is
                                all-reduced before each rebuild step's force kernel, so every rank
                                re-runs the same steps); that needs the NCCL communicator or a loopback
                                group — a PEER rank without one returns DEM_ERR_CAPACITY instead */
  /* ---- spatial slab decomposition along x.  n_ranks <= 1: one system owns all. ----
   * dem_set_state then takes any superset of the held clumps (e.g. the global state); the rank owns the clumps whose COM x
   * is in [slab_lo, slab_hi) and keeps ghost copies of the clumps within `halo` beyond each face
   * (owned by the neighbouring ranks rank-1 / rank+1, so halo must not exceed a neighbour's slab
   * width).  Every step the owners' new ghost states are exchanged; contacts are evaluated by the
   * owner of each sphere (mirror-exact, so no force exchange), and owned states are bitwise
   * independent of the number of ranks.  halo >= 2 R_bound,max + margin + 2 drift_max; an owned
   * COM that moves more than drift_max from its dem_set_state position raises
   * DEM_ERR_REPARTITION (call dem_migrate, or dem_set_state again).  dem_set_state_local takes
   * rank-local input instead (each rank only its own clumps; ghosts come from the neighbours). */
  int32_t rank, n_ranks;
  double slab_lo, slab_hi, halo, drift_max;
  int32_t transport;         /* DEM_TRANSPORT_NCCL, _PEER, _LOOPBACK or _LOOPBACK_PEER (below) */
  unsigned char nccl_id[128];/* ncclUniqueId from dem_nccl_unique_id on rank 0, broadcast by the caller */
  /* Overlapped detection cadence (the active set is updated "in the shadow" of the
   * dynamics; P:148 one GPU shares the two threads via CUDA streams).  With overlap = 1 and
   * cd_every = k >= 2, the set used in window w+1 (steps (w+1)k .. (w+1)k + k-1) is detected from
   * the sphere centres at step wk + 1, on a second stream, while the force steps of window w
   * run; the first window detects in line.  The margin must cover 2k - 2 steps of motion
   * (2 v_max h (2k - 2) x safety).  A sphere that moves more than margin/2 from the centres its
   * set was detected from raises DEM_ERR_VMAX.  overlap = 0: detection in line at the window
   * start.  Requires cd_every >= 2 (else DEM_ERR_INVALID_ARG). */
  int32_t overlap;
} dem_params;

/* Ghost-halo transports.  NCCL: the owners' new ghost states are packed and sent with grouped
 * ncclSend/ncclRecv after the force kernel.  PEER: the fused halo — the force/integrate kernel
 * writes each ghosted clump's new state straight into the neighbour's next-state array over
 * NVLink (CUDA IPC mappings exchanged inside dem_set_state over the NCCL communicator), and a
 * one-thread flag handshake per step (release/acquire, system scope) keeps neighbours within one
 * step of each other; no pack, collective or unpack kernels.  LOOPBACK / LOOPBACK_PEER: the same
 * two schemes between the systems of one process on one GPU (dem_step_group; tests). */
enum { DEM_TRANSPORT_NCCL = 0, DEM_TRANSPORT_LOOPBACK = 1, DEM_TRANSPORT_PEER = 2, DEM_TRANSPORT_LOOPBACK_PEER = 3 };

typedef struct {
  int64_t steps;             /* steps completed since dem_set_state */
  int64_t n_clumps, n_spheres; /* owned + ghost */
  int64_t n_owned_clumps, n_owned_spheres, n_ghost_clumps;
  int64_t n_entries;         /* directed contact-row entries of the last step (2 per sphere pair + walls) */
  int64_t n_contacts;        /* canonical contacts of the last step (sphere pairs + sphere-wall) */
  int64_t n_inserts;         /* bin inserts of the last step */
  int64_t n_cells;
  double cell_size;
  int64_t regrows;           /* capacity regrows so far */
  int64_t kernel_launches_per_step;
  int64_t state_fast_resets;  /* dem_set_state calls that took the same-clumps fast path */
  int64_t migrated_clumps;    /* distributed: owned clumps this rank sent to a neighbour in the last migration */
  int64_t migration_bytes;    /* ... and the bytes of those clumps and of the contacts routed with them */
  int64_t ghost_exchange_bytes; /* bytes this rank sent to complete its neighbours' ghost bands (last
                                   dem_set_state_local / migration) */
  int64_t bin_regrids;        /* bin grids laid out again because a sphere centre left the bin region
                                 (the region is the box the spheres occupied, within the domain) */
  int64_t reruns;             /* re-runs after an aborted step: a capacity regrow, an overflowed set
                                 detected ahead (overlapped cadence), or another rank's overflow */
} dem_stats;

typedef struct dem_system dem_system;

/* Create a system.  cuda_stream is a cudaStream_t (NULL = legacy default stream). */
dem_status dem_create(const dem_params* params, const dem_material* materials, int32_t n_mat,
                      const dem_template* templates, int32_t n_tmpl, const dem_plane* planes,
                      int32_t n_planes, void* cuda_stream, dem_system** out);

/* Replace the clump state (n clumps; gids unique, >= 0, < 2^56).  pos/vel/omega are [3n],
 * quat [4n] (normalised by the caller), all row-major (x,y,z per clump).  on_device = 1 means
 * the pointers are device pointers.  Clears the tangential history. */
dem_status dem_set_state(dem_system* sys, int64_t n, const int64_t* clump_gid, const int32_t* template_id,
                         const double* pos, const double* quat, const double* vel, const double* omega,
                         int32_t on_device);

/* Replace the tangential history carried into the next step (host arrays; u_t [3n], oriented
 * key_a -> key_b, key_a < key_b).  Keys whose spheres are not in the system are ignored. */
dem_status dem_set_contact_history(dem_system* sys, int64_t n, const int64_t* key_a, const int64_t* key_b,
                                   const double* u_t);

/* Advance n_steps steps on the system stream (CUDA-graph launches).  Returns after checking the
 * device status word once at the end (one stream synchronisation per call). */
dem_status dem_step(dem_system* sys, int64_t n_steps);

dem_status dem_synchronize(dem_system* sys);

/* Copy the state out in the order of the last dem_set_state.  cap = capacity in clumps; *n
 * receives the clump count.  Any output pointer may be NULL.  on_device as in dem_set_state.
 * Distributed systems return their OWNED clumps only, in the order of the global input. */
dem_status dem_get_state(dem_system* sys, int64_t cap, int64_t* n, int64_t* clump_gid, int32_t* template_id,
                         double* pos, double* quat, double* vel, double* omega, int32_t on_device);

/* Canonical contact list of the last step (built from the state at that step's start), sorted by
 * (key_a, key_b): force on b, contact point, normal a->b, u_t after the step, penetration delta.
 * Force/point/normal/delta need params.record_contacts = 1 (else DEM_ERR_INVALID_ARG if requested).
 * Call with cap = 0 to query *n. */
dem_status dem_get_contacts(dem_system* sys, int64_t cap, int64_t* n, int64_t* key_a, int64_t* key_b,
                            double* force_on_b, double* point, double* normal, double* u_t, double* delta);

dem_status dem_get_stats(dem_system* sys, dem_stats* out);

/* Stage profiling.  With enable = 1, dem_step launches the step kernels directly (no graph) with
 * CUDA events between the stages on the system stream and accumulates each stage's device time;
 * enable resets the accumulators.  dem_get_stage_times returns the mean ms per step of each stage,
 * in the order (8 stages): (1) pose + bin counts (k_pose_count; with meshes also k_mesh_pose),
 * (2) bin-offset scan, (3) bin scatter (k_bin_scatter; with meshes also k_mesh_pairs), (4) per-bin
 * pair tests (k_pairs), (5) row-offset scan, (6) rows: candidate sort, wall entries, history remap
 * (k_rows_finish), (7) force + reduce + integrate (k_force_integrate: remap, contact forces,
 * canonical per-sphere and per-clump sums, Eq. 4 update; with meshes also k_mesh_geom before and
 * k_mesh_finish after), (8) ghost halo (pack + exchange + unpack, or the peer handshake;
 * distributed systems only).  Stages 2-6 are 0 on steps that reuse a deferred set. */
dem_status dem_set_profiling(dem_system* sys, int32_t enable);
dem_status dem_get_stage_times(dem_system* sys, int32_t n_stages, double* ms);

/* ---- distribution ---- */

/* 128-byte NCCL unique id for params.nccl_id (call on rank 0, broadcast to every rank, then each
 * rank calls dem_create collectively).  Host only. */
dem_status dem_nccl_unique_id(unsigned char out[128]);

/* The slab partition as every rank computes it (host only, no GPU): for n clumps with COM x in
 * pos[3c], role[c] = 0 not held, 1 owned (slab_lo <= x < slab_hi), 2 ghost from the left
 * neighbour (slab_lo - halo <= x < slab_lo), 3 ghost from the right neighbour
 * (slab_hi <= x < slab_hi + halo); send[c] bit 0 = owned and sent to the left neighbour
 * (x < slab_lo + halo), bit 1 = owned and sent to the right neighbour (x >= slab_hi - halo).
 * has_left / has_right say whether those neighbours exist.  Ghost and send lists are exchanged
 * in ascending clump gid order. */
dem_status dem_partition_plan(int64_t n, const double* pos, double slab_lo, double slab_hi, double halo,
                              int32_t has_left, int32_t has_right, int8_t* role, int8_t* send);

/* Step a group of LOOPBACK-transport systems (ranks 0..n-1 in order, same GPU and stream) in
 * lockstep: per step every rank computes, then the ghost buffers are copied device-to-device
 * between neighbours.  Lets one GPU run a P-rank decomposition (tests, scaling studies). */
dem_status dem_step_group(dem_system* const* systems, int32_t n, int64_t n_steps);

/* ---- kinematic triangle meshes (P:277 cone, P:307 funnel, P:344 wheel;
 * S:241-262).  A mesh is a set of triangles in its body frame with a prescribed motion: reference
 * point X and orientation q (body -> world), velocity v and angular velocity w (world, about X);
 * every step advances X += h v and q <- normalize(q_step (x) q), q_step the rotation by h|w|
 * about w (R27).  A sphere contacts triangle t if |c - closest(c, t)| <= r + margin
 * (closest point by Voronoi regions, R25); the contact key is (sphere key, INT64_MAX - 16 - t)
 * with t counted over all meshes in the order added.  The force is the flat-wall limit
 * (R_bar = r, m_bar = clump mass) with the normal from the sphere to its closest point,
 * the boundary point velocity v + w x (p - X), and one contact per surface feature: a
 * sphere touching a shared edge or vertex is pushed once (R26).  At most 8 meshes, 2^24
 * triangles; not on distributed systems (DEM_ERR_INVALID_ARG). */
typedef struct {
  int64_t n_tri;
  const double* verts;       /* [9 n_tri] body-frame vertices a, b, c of each triangle (copied) */
  int32_t material;
  double pos[3], quat[4], vel[3], omega[3];
} dem_mesh;

/* Add a mesh (host arrays, copied); *mesh_id receives its index.  Call between dem_step calls. */
dem_status dem_add_mesh(dem_system* sys, const dem_mesh* mesh, int32_t* mesh_id);

/* Replace a mesh's pose and motion before the next step (co-simulation: the caller's multibody
 * solver sets the pose each step). */
dem_status dem_set_mesh_motion(dem_system* sys, int32_t mesh, const double pos[3], const double quat[4],
                               const double vel[3], const double omega[3]);

/* The mesh pose after the last step, and the wrench the granular material exerted on it during
 * that step: force and torque about X (the sum over its contacts in a fixed order).  The
 * order is the fused force kernel's CTA partition (partials per CTA in row order, then CTA order
 * and a fixed tree), which is re-cut when the contact-entry count moves by more than a quarter at
 * the end of a dem_step call: the wrench bits are reproducible for a given sequence of dem_step
 * calls, and may differ in the last place between dem_step(100) and 100 x dem_step(1).  Clump
 * states do not depend on the cut. */
dem_status dem_get_mesh(dem_system* sys, int32_t mesh, double pos[3], double quat[4], double force[3],
                        double torque[3]);

/* PEER transport link (after every dem_set_state, before stepping; collective in effect).  Each
 * rank exports a packet — CUDA IPC handles of its two state arrays and its flag words, its clump
 * count and its ghost receive lists — which the caller delivers to the left and right neighbours
 * (any transport: torch.distributed all_gather in the Python binding); dem_peer_import maps the
 * neighbours' arrays (peer access) and derives the neighbour ghost slot of every clump we send.
 * dem_peer_export with out = NULL returns the packet size in *len.  left / right = NULL where
 * there is no neighbour.  A rank's dem_set_state must not start while a neighbour is still
 * stepping (with an NCCL id in dem_params the library runs that barrier itself). */
dem_status dem_peer_export(dem_system* sys, int64_t cap, void* out, int64_t* len);
dem_status dem_peer_import(dem_system* sys, const void* left, const void* right);

/* Clump migration between slabs, neighbour-only.  Collective over the n_ranks
 * systems of an NCCL decomposition (every rank calls it at the same point, between dem_step
 * calls).  The largest displacement of an owned COM since the last partition is reduced over the
 * ranks (device reduction + ncclAllReduce MAX); if it exceeds `threshold` [m] (use a fraction of
 * drift_max, e.g. drift_max / 2; 0 forces a migration):
 *   1. every rank sends to each neighbour (grouped ncclSend/ncclRecv: counts, then payloads) only
 *      the owned clumps whose COM crossed into that neighbour's slab, with the directed contact-row
 *      entries of their spheres (partner key + u_t, the history a sphere's owner keeps;
 *      dem_migration_plan);
 *   2. the new owned sets exchange their ghost bands with the neighbours (dem_set_state_local);
 *   3. every rank lays out its own clumps again and re-imports the entries of its spheres.
 * Bytes moved scale with the crossings and the ghost band, never with the whole system
 * (dem_stats.migration_bytes / ghost_exchange_bytes).  The trajectory is unchanged: owned states
 * are bitwise independent of the decomposition.  *moved (optional) receives 1 if a migration
 * happened.  Non-distributed systems: no-op. */
dem_status dem_migrate(dem_system* sys, double threshold, int32_t* moved);

/* dem_migrate for a LOOPBACK group (ranks 0..n-1 in order, as dem_step_group): the same
 * neighbour-only plan, the payloads handed between the systems in host memory. */
dem_status dem_migrate_group(dem_system* const* systems, int32_t n, double threshold, int32_t* moved);

/* The migration plan as every rank computes it (host only, no GPU).  For the n clumps a rank
 * holds (gid, COM x in pos[3c], role[c] 1 owned / 2 ghost from the left / 3 ghost from the right,
 * as dem_partition_plan gives), dest[c] = the clump's owner after the move relative to this rank:
 * -1 left neighbour, 0 this rank, +1 right neighbour (an owned COM below slab_lo goes left, at or
 * above slab_hi right; a ghost becomes ours once its COM is inside our slab).  For the rank's
 * n_entries directed contact-row entries (the history each rank keeps for its own spheres; own
 * sphere key = gid * 64 + component), route[k] = dest of the own sphere's clump: an entry moves
 * with its sphere.  Returns DEM_ERR_INVALID_ARG if a role is 0 or an entry's clump is not held. */
dem_status dem_migration_plan(int64_t n, const int64_t* gid, const double* pos, const int8_t* role,
                              double slab_lo, double slab_hi, int32_t has_left, int32_t has_right, int8_t* dest,
                              int64_t n_entries, const int64_t* own_key, int8_t* route);

/* Rank-local state input of a distributed system (collective over an NCCL decomposition, like
 * dem_migrate): the caller passes any set of clumps (host arrays, dem_set_state layout); the rank
 * keeps those whose COM x lies in [slab_lo, slab_hi) — every clump must be given to the rank that
 * owns it — and receives its ghost bands from the neighbours' owned clumps (grouped
 * ncclSend/ncclRecv, counts then payloads), then lays out owned + ghosts as dem_set_state does.
 * No rank ever needs the global state.  Non-distributed systems: dem_set_state. */
dem_status dem_set_state_local(dem_system* sys, int64_t n, const int64_t* gid, const int32_t* tid,
                               const double* pos, const double* quat, const double* vel, const double* omega);

/* dem_set_state_local for a LOOPBACK group: rank r's input is n_in[r] clumps in gid[r], tid[r],
 * pos[r], ... (host arrays). */
dem_status dem_set_state_local_group(dem_system* const* systems, int32_t n, const int64_t* n_in,
                                     const int64_t* const* gid, const int32_t* const* tid,
                                     const double* const* pos, const double* const* quat,
                                     const double* const* vel, const double* const* omega);

const char* dem_status_string(dem_status s);
dem_status dem_last_error(const dem_system* sys, char* buf, size_t len);
void dem_destroy(dem_system* sys);

#ifdef __cplusplus
}
#endif
#endif /* DEM_B200_H */
