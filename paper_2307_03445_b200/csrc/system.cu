// system.cu — host runtime and C-ABI (include/dem.h) of the B200 clump-DEM hot path.
//
// Owns device memory (through the caller's allocator callback, e.g. the PyTorch caching
// allocator, or cudaMallocAsync), captures one CUDA graph per state parity for the
// 10-launch step sequence, checks the device status word once per dem_step call, and
// regrows bin/row capacity transparently (the aborted steps are re-run).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include <nccl.h>

#include "dem.h"
#include "dem_device.cuh"

namespace dem {
void launch_pose_count(const StepArgs&, cudaStream_t);
void launch_bin_scatter(const StepArgs&, cudaStream_t);
void launch_pairs(const StepArgs&, cudaStream_t, int n_sm);
void launch_rows_finish(const StepArgs&, cudaStream_t);
void launch_force_integrate(const StepArgs&, cudaStream_t);
int force_cta_clumps();
int force_cta_spheres();
long long scan_tiles_needed(long long n);
void launch_excl_scan(const int* in, int* out, long long n, int* tmp, const int* abort, cudaStream_t s,
                      const int* abort2, int packed = 0, bool pdl = false);
void launch_count_canonical(const Rows& r, const long long* s_key, int ns, unsigned long long* out, cudaStream_t s);
void launch_pack(const State& st, const int* idx, int n, double* buf, cudaStream_t s);
void launch_unpack(const State& st, const int* idx, int n, const double* buf, cudaStream_t s);
void launch_max_drift(const State& st, const double* xref, int n, unsigned long long* out, cudaStream_t s);
void launch_mesh_pose(const StepArgs&, cudaStream_t);
void launch_peer_signal(const Ctl* ctl, int* r0, int* r1, cudaStream_t s);
void launch_peer_wait(Ctl* ctl, const int* f0, const int* f1, cudaStream_t s);
void launch_abort_or(const AbortWords& w, cudaStream_t s);
void launch_bbox(const double4* spos, int ns, unsigned long long* box, cudaStream_t s);
void launch_state_in(const State& st, const int* perm, int n, const double* pos, const double* quat,
                     const double* vel, const double* om, int* bad, double* xref, int n_own, cudaStream_t s);
void launch_state_out(const State& st, const int* outpos, int n_own, double* pos, double* quat, double* vel,
                      double* om, cudaStream_t s);
void launch_mesh_pairs(const StepArgs&, cudaStream_t);
void launch_mesh_finish(const StepArgs&, cudaStream_t);
void launch_mesh_geom(const StepArgs&, cudaStream_t);
}  // namespace dem

using namespace dem;

static constexpr int kStages = 8;  // last: ghost halo pack + exchange + unpack (distributed)
static constexpr int kKin13 = 13;  // doubles per ghost clump state
static constexpr int kRowWidth = 32;  // initial candidate slots per owned sphere
static constexpr int kLaunchesPerStep = 11;
static const int kOne = 1;  // 5 stage kernels + 2 x 3 scan kernels

struct RowBuf {
  int* row_ptr = nullptr;
  Entry* ent = nullptr;
  long long* key = nullptr;
  double* ut = nullptr;
};

struct dem_system {
  dem_params P{};
  cudaStream_t stream = nullptr;
  cudaStream_t cap_stream = nullptr;
  cudaStream_t cap_hi = nullptr;  // capture stream of the overlapped cadence's force graphs (highest priority)
  std::string err;
  // host tables
  int n_mat = 0, n_tmpl = 0, n_planes = 0;
  std::vector<int> tpl_ncomp, tpl_coff, tc_mat;
  std::vector<double> tc_off, tc_rad, tpl_mass, tpl_inertia, pair;
  std::vector<dem_plane> planes;
  double rmin = 0, rmax = 0;
  // device tables
  double *d_tc_off = nullptr, *d_tc_rad = nullptr, *d_tpl_mass = nullptr, *d_tpl_inertia = nullptr,
         *d_pair = nullptr;
  int *d_tc_mat = nullptr, *d_tpl_coff = nullptr;
  // state
  int64_t n = 0, ns = 0;
  std::vector<long long> h_gid;
  std::vector<int> h_tid, h_sph_off, h_s_tc;
  std::vector<long long> h_s_key;
  std::vector<int64_t> h_perm;  // storage index -> caller index
  // the last dem_set_state input's gids/tids (caller order): a later call with the same clumps
  // takes the fast path (no re-layout); device permutations for state I/O in caller order
  std::vector<long long> h_in_gid;
  std::vector<int> h_in_tid;
  std::vector<int> h_outpos;        // owned storage index -> output row of dem_get_state
  std::vector<int8_t> h_role, h_sendf;  // the slab partition of the last input (distributed)
  int *d_perm = nullptr, *d_outpos = nullptr, *d_io_bad = nullptr;
  double* d_io = nullptr;           // 13 n doubles of staging (caller-order AoS rows)
  long long* d_gid = nullptr;
  int *d_tid = nullptr, *d_sph_off = nullptr;
  double* d_state[2] = {nullptr, nullptr};
  double* d_kin = nullptr;
  int *d_s_clump = nullptr, *d_s_tc = nullptr, *d_s_mat = nullptr;
  long long* d_s_key = nullptr;
  double4* d_spos = nullptr;
  int2* d_cta_clump = nullptr;  // per CTA boundary: (first clump, first sphere)
  int n_cta = 0;
  int* d_slots = nullptr;  // fixed-width candidate partner lists of the owned spheres
  long long* d_slot_key = nullptr;  // their partner keys (DEM_SLOT_KEYS)
  int row_width = 0;
  int n_sm = 148;
  // bins
  Grid grid{};
  long long ncell = 0, cap_inserts = 0;
  int *d_cell_count = nullptr, *d_cell_start = nullptr, *d_items = nullptr;
  unsigned short* d_irank = nullptr;  // [kRankW][ns] insert ranks (DEM_SCATTER_RANKS)
  int *d_row_cnt = nullptr, *d_scan_tmp = nullptr;
  unsigned short* d_wall_mask = nullptr;
  // rows: the entry sets (row_ptr, ent) of rows[ep] are the latest contact set and ping-pong
  // at every rebuild; the u_t arrays of rows[up] hold the latest tangential history and
  // ping-pong at every step; the state ping-pongs every step (sp)
  RowBuf rows[2];
  int sp = 0, up = 0, ep = 0;
  int since_rebuild = 0;                 // steps since the last contact-set rebuild
  double4* d_spos_ref[2] = {nullptr, nullptr};  // sphere centres entry set e was detected from
  // overlapped cadence ("in the shadow"): the next window's set is detected
  // on det_stream from the positions of the window's second step, adopted at the next window start
  bool pending = false;                  // rows[ep ^ 1] holds a set detected ahead, not yet adopted
  cudaStream_t det_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_det = nullptr;
  int fault_ahead = 0;
  int no_pdl = 0;  // env DEM_NO_PDL=1: plain stream serialization between the step kernels
  int tiny_force = -1;  // env DEM_PAIRS_TINY=0/1: the small-bin pass of k_pairs off / on (else by density)
  bool debug_serial_det = false;  // debug (env DEM_DEBUG_SERIAL_DET=1): the force steps wait for the ahead detection
  // kinematic triangle meshes (NEXT-3)
  int n_mesh = 0, n_tri = 0;
  std::vector<double> h_tri_body, h_mesh;  // host copies (9 per triangle; kMeshRec per mesh)
  std::vector<int> h_tri_vid, h_tri_mesh, h_mesh_mat;
  double *d_tri_body = nullptr, *d_tri_world = nullptr, *d_tri_snap = nullptr, *d_mesh = nullptr,
         *d_mesh_part = nullptr, *d_mesh_wrench = nullptr;
  int *d_tri_vid = nullptr, *d_tri_mesh = nullptr, *d_mesh_mat = nullptr, *d_mesh_flag = nullptr;
  int mesh_part_ctas = 0;
  bool entry_partitioned = false;  // the force CTAs were re-cut by contact-row entries
  int part_entries = 0;            // the entry count of that cut
  int2* d_mlist[2] = {nullptr, nullptr};  // mesh entries of entry set e (k_rows_finish)
  int* d_mlist_n = nullptr;               // [2] their counts
  double4* d_mgeom = nullptr;             // [cap_entries] per-step closest point + feature flag  // test hook (env DEM_FAULT_AHEAD_OVERFLOW=n): the next n ahead detections report an overflow
  long long cap_entries = 0;
  Record rec{};
  Ctl* d_ctl = nullptr;
  Ctl* h_ctl = nullptr;
  unsigned long long* d_counter = nullptr;
  // graphs, one per (sp, up, ep, rebuild)
  std::unordered_map<int, cudaGraphExec_t> graph;  // key: graph_key()
  bool graphs_valid = false;
  int64_t launched = 0;  // steps launched since dem_set_state
  int64_t steps_done = 0;
  int64_t regrows = 0;
  long long last_entries = 0, last_inserts = 0;
  // profiling
  bool profiling = false;
  std::vector<cudaEvent_t> ev;
  double stage_ms[kStages] = {0};
  int64_t prof_steps = 0;
  std::unordered_map<void*, size_t> allocs;
  // slab decomposition: storage = owned clumps [0, n_own), then ghosts
  bool dist = false;
  ncclComm_t comm = nullptr;
  int64_t n_own = 0, ns_own = 0;
  int n_send[2] = {0, 0}, n_recv[2] = {0, 0};       // [0] left neighbour, [1] right neighbour
  int *d_send_idx[2] = {nullptr, nullptr}, *d_recv_idx[2] = {nullptr, nullptr};
  double *d_sendbuf[2] = {nullptr, nullptr}, *d_recvbuf[2] = {nullptr, nullptr};
  double* d_xref = nullptr;                          // owned COM at dem_set_state (drift check)
  // peer transports (fused halo): state arrays and flag words from cudaMalloc (IPC-exportable),
  // the neighbours' next-state arrays / flag words / ghost slots of our send lists
  bool peer = false;
  double* raw_state[2] = {nullptr, nullptr};
  int* d_flags = nullptr;                            // [0] written by the left, [1] by the right neighbour
  double* remote_state[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [side][parity]
  long long remote_n[2] = {0, 0};
  int* remote_flag[2] = {nullptr, nullptr};
  int* d_peer_idx[2] = {nullptr, nullptr};           // [side][n_own] neighbour ghost slot or -1
  std::vector<int> h_send_list[2], h_recv_list[2];   // storage indices, ascending gid
  std::vector<void*> ipc_open;                       // neighbour mappings to close
  bool peer_linked = false;
  int64_t fast_resets = 0;
  int64_t migrated_clumps = 0, migration_bytes = 0, ghost_bytes = 0;  // last migration / ghost exchange
  int64_t reruns = 0;   // aborted steps re-run (regrow, ahead-set overflow, another rank's overflow)
  int64_t regrids = 0;  // bin grids rebuilt around spheres that left the bin region
};

static dem_status peer_release(dem_system* sys);

// ------------------------------------------------------------------ helpers
#define CK(call)                                                                  \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess) {                                                      \
      sys->err = std::string(#call) + ": " + cudaGetErrorString(e_);              \
      return e_ == cudaErrorMemoryAllocation ? DEM_ERR_OOM : DEM_ERR_CUDA;        \
    }                                                                             \
  } while (0)

static void* dalloc(dem_system* sys, size_t bytes) {
  if (bytes == 0) bytes = 16;
  void* p = nullptr;
  if (sys->P.alloc) {
    p = sys->P.alloc(bytes, sys->P.alloc_ctx, (void*)sys->stream);
    if (p && ((uintptr_t)p & 31)) {  // 256-bit record accesses need 32-byte alignment
      if (sys->P.free) sys->P.free(p, bytes, sys->P.alloc_ctx, (void*)sys->stream);
      sys->err = "params.alloc returned a block that is not 32-byte aligned";
      return nullptr;
    }
  } else {
    if (cudaMallocAsync(&p, bytes, sys->stream) != cudaSuccess) p = nullptr;
  }
  if (p) sys->allocs[p] = bytes;
  return p;
}

static void dfree(dem_system* sys, void* p) {
  if (!p) return;
  auto it = sys->allocs.find(p);
  size_t bytes = it == sys->allocs.end() ? 0 : it->second;
  if (it != sys->allocs.end()) sys->allocs.erase(it);
  if (sys->P.free)
    sys->P.free(p, bytes, sys->P.alloc_ctx, (void*)sys->stream);
  else
    cudaFreeAsync(p, sys->stream);
}

template <class T>
static dem_status alloc_arr(dem_system* sys, T** out, size_t count) {
  dfree(sys, *out);
  *out = (T*)dalloc(sys, sizeof(T) * count);
  if (!*out) {
    sys->err = "device allocation of " + std::to_string(sizeof(T) * count) + " bytes failed" +
               (sys->err.find("32-byte") != std::string::npos ? " (" + sys->err + ")" : std::string());
    return DEM_ERR_OOM;
  }
  return DEM_OK;
}

#define TRY(x)                      \
  do {                              \
    dem_status s_ = (x);            \
    if (s_ != DEM_OK) return s_;    \
  } while (0)

static void free_graphs(dem_system* sys) {
  for (auto& g : sys->graph)
    if (g.second) cudaGraphExecDestroy(g.second);
  sys->graph.clear();
  sys->graphs_valid = false;
}

// Step kinds.  FULL: detect the contact set from this step's positions and use it
// (every step at cd_every = 1, the "traditional way").  CHECK: re-evaluate the set in use.
// AHEAD (overlapped cadence, second step of a window): as CHECK, and detect the next window's
// set from this step's positions into rows[ep ^ 1] (concurrently, on det_stream).  ADOPT
// (window start with a set detected ahead): use it, history remapped by key.
enum StepKind { K_FULL = 0, K_CHECK = 1, K_AHEAD = 2, K_ADOPT = 3 };

static int step_kind(const dem_system* sys) {
  if (sys->since_rebuild == 0) return sys->pending ? K_ADOPT : K_FULL;
  if (sys->P.overlap && sys->since_rebuild == 1) return K_AHEAD;
  return K_CHECK;
}

// Arguments of the next step from the host parities: state sp -> sp^1, u_t up -> up^1.  A
// FULL/ADOPT step's force kernel reads the new entry set rows[ep^1] (rows[ep] = the previous
// set, for the history remap), CHECK/AHEAD steps re-evaluate the current set rows[ep]
// (P:142-144).  det = 1 gives the view of the detection kernels of an AHEAD step: they write
// rows[ep^1] from the snapshot of this step's centres, with their own abort word.
static StepArgs make_args(dem_system* sys, int kind, bool det = false) {
  const bool rebuild = kind == K_FULL || kind == K_ADOPT || det;
  const int p = sys->sp;
  StepArgs a{};
  a.n = (int)sys->n;
  a.ns = (int)sys->ns;
  a.ncell = sys->ncell;
  a.cap_inserts = sys->cap_inserts;
  a.cap_entries = sys->cap_entries;
  a.h = sys->P.h;
  for (int d = 0; d < 3; ++d) a.g[d] = sys->P.gravity[d];
  a.margin = sys->P.margin;
  Tables& t = a.tab;
  t.tc_off = sys->d_tc_off;
  t.tc_rad = sys->d_tc_rad;
  t.tc_mat = sys->d_tc_mat;
  t.tpl_coff = sys->d_tpl_coff;
  t.tpl_mass = sys->d_tpl_mass;
  t.tpl_inertia = sys->d_tpl_inertia;
  t.pair = sys->d_pair;
  t.n_mat = sys->n_mat;
  t.n_planes = sys->n_planes;
  for (int k = 0; k < sys->n_planes; ++k) {
    for (int d = 0; d < 3; ++d) {
      t.plane_pt[k][d] = sys->planes[k].point[d];
      t.plane_n[k][d] = sys->planes[k].normal[d];
    }
    t.plane_mat[k] = sys->planes[k].material;
  }
  a.grid = sys->grid;
  auto soa = [&](double* base) {
    State s;
    size_t n = (size_t)sys->n;
    double* f[13];
    for (int k = 0; k < 13; ++k) f[k] = base + k * n;
    s.x = f[0]; s.y = f[1]; s.z = f[2]; s.qw = f[3]; s.qx = f[4]; s.qy = f[5]; s.qz = f[6];
    s.vx = f[7]; s.vy = f[8]; s.vz = f[9]; s.wx = f[10]; s.wy = f[11]; s.wz = f[12];
    return s;
  };
  a.cur = soa(sys->d_state[p]);
  a.nxt = soa(sys->d_state[p ^ 1]);
  a.tid = sys->d_tid;
  a.gid = sys->d_gid;
  a.sph_off = sys->d_sph_off;
  a.kin = sys->d_kin;
  a.s_clump = sys->d_s_clump;
  a.s_tc = sys->d_s_tc;
  a.s_mat = sys->d_s_mat;
  a.s_key = sys->d_s_key;
  a.spos = sys->d_spos;
  a.slots = sys->d_slots;
  a.slot_key = sys->d_slot_key;
  a.row_width = sys->row_width;
  a.cta_clump = sys->d_cta_clump;
  a.n_cta = sys->n_cta;
  a.n_own = (int)sys->n_own;
  a.ns_own = (int)sys->ns_own;
  a.xref = sys->d_xref;
  a.drift_max = sys->dist ? sys->P.drift_max : 0.0;
  a.cell_count = sys->d_cell_count;
  // programmatic serialization only for graph-launched steps (the in-line profiling pass times the
  // stages between events, one after the other); DEM_NO_PDL=1 turns it off
  a.pdl = (!sys->profiling && !sys->no_pdl) ? 1 : 0;
  // sparse bins (a falling column, C3: 0.5 spheres per bin; the C5 bed: 5): k_pairs takes the
  // small-bin pass for bins of at most 8 members (env DEM_PAIRS_TINY=0/1 forces it off/on)
  a.tiny = sys->tiny_force >= 0 ? sys->tiny_force : ((double)sys->ns < 2.0 * (double)sys->ncell ? 1 : 0);
  a.irank = sys->d_irank;
  a.cell_start = sys->d_cell_start;
  a.items = sys->d_items;
  a.row_cnt = sys->d_row_cnt;
  a.wall_mask = sys->d_wall_mask;
  const RowBuf& E = sys->rows[rebuild ? sys->ep ^ 1 : sys->ep];
  const RowBuf& Q = sys->rows[sys->ep];
  a.rows = Rows{E.row_ptr, E.ent, E.key, sys->rows[sys->up ^ 1].ut};
  a.prev = Rows{Q.row_ptr, Q.ent, Q.key, sys->rows[sys->up].ut};
  const bool deferred = sys->P.cd_every > 1;
  a.count = (kind == K_FULL || kind == K_AHEAD) ? 1 : 0;
  a.remap = rebuild ? 1 : 0;
  a.adopt = kind == K_ADOPT ? 1 : 0;
  a.ref_in = !deferred || kind == K_FULL ? nullptr : sys->d_spos_ref[kind == K_ADOPT ? sys->ep ^ 1 : sys->ep];
  a.ref_out = deferred && a.count ? sys->d_spos_ref[sys->ep ^ 1] : nullptr;
  a.dpos = det ? sys->d_spos_ref[sys->ep ^ 1] : sys->d_spos;
  a.abort = det ? &sys->d_ctl->det_abort : &sys->d_ctl->abort;
  a.half_margin = deferred ? 0.5 * sys->P.margin : 0.0;
  a.n_tri = sys->n_tri;
  a.n_mesh = sys->n_mesh;
  a.tri_body = sys->d_tri_body;
  a.tri_vid = sys->d_tri_vid;
  a.tri_mesh = sys->d_tri_mesh;
  a.tri_world = sys->d_tri_world;
  a.tri_snap = kind == K_AHEAD && !det ? sys->d_tri_snap : nullptr;
  a.tri_dpos = det ? sys->d_tri_snap : sys->d_tri_world;
  a.mesh = sys->d_mesh;
  a.mesh_mat = sys->d_mesh_mat;
  a.mesh_part = sys->d_mesh_part;
  a.mesh_flag = sys->d_mesh_flag;
  a.mesh_wrench = sys->d_mesh_wrench;
  {
    const int eu = rebuild ? sys->ep ^ 1 : sys->ep;  // the entry set the force kernel reads
    a.mlist = sys->d_mlist[eu];
    a.mlist_n = sys->d_mlist_n ? sys->d_mlist_n + eu : nullptr;
    a.mlist_out = sys->d_mlist[sys->ep ^ 1];
    a.mlist_out_n = sys->d_mlist_n ? sys->d_mlist_n + (sys->ep ^ 1) : nullptr;
    a.mgeom = sys->d_mgeom;
  }
  for (int side = 0; side < 2; ++side) {
    a.peer_state[side] = sys->peer ? sys->remote_state[side][p ^ 1] : nullptr;
    a.peer_n[side] = sys->remote_n[side];
    a.peer_idx[side] = sys->d_peer_idx[side];
  }
  a.rec = sys->rec;
  a.record = sys->P.record_contacts ? 1 : 0;
  a.ctl = sys->d_ctl;
  return a;
}

// ghost halo (distributed): owners' new states -> the neighbours' ghost slots
static void enqueue_pack(dem_system* sys, const StepArgs& a, cudaStream_t s) {
  for (int side = 0; side < 2; ++side)
    if (sys->n_send[side]) launch_pack(a.nxt, sys->d_send_idx[side], sys->n_send[side], sys->d_sendbuf[side], s);
}
static void enqueue_unpack(dem_system* sys, const StepArgs& a, cudaStream_t s) {
  for (int side = 0; side < 2; ++side)
    if (sys->n_recv[side]) launch_unpack(a.nxt, sys->d_recv_idx[side], sys->n_recv[side], sys->d_recvbuf[side], s);
}
static void enqueue_nccl_exchange(dem_system* sys, cudaStream_t s) {
  const int r = sys->P.rank, P = sys->P.n_ranks;
  ncclGroupStart();
  if (r > 0) {
    if (sys->n_send[0]) ncclSend(sys->d_sendbuf[0], (size_t)kKin13 * sys->n_send[0], ncclDouble, r - 1, sys->comm, s);
    if (sys->n_recv[0]) ncclRecv(sys->d_recvbuf[0], (size_t)kKin13 * sys->n_recv[0], ncclDouble, r - 1, sys->comm, s);
  }
  if (r < P - 1) {
    if (sys->n_send[1]) ncclSend(sys->d_sendbuf[1], (size_t)kKin13 * sys->n_send[1], ncclDouble, r + 1, sys->comm, s);
    if (sys->n_recv[1]) ncclRecv(sys->d_recvbuf[1], (size_t)kKin13 * sys->n_recv[1], ncclDouble, r + 1, sys->comm, s);
  }
  ncclGroupEnd();
}

// The step sequence, in three parts: pose (a1 + bin counts), detection (a2-a4: bin scan,
// scatter, pairs, row scan, rows), force (a5-a10 + halo).  ev (optional) receives kStages+1
// events around the stages.  With exchange = false (loopback groups) the halo is packed but
// moved by dem_step_group.
enum { PART_ALL = 0, PART_POSE = 1, PART_DET = 2, PART_FORCE = 3 };

static void enqueue_pose(dem_system* sys, int kind, cudaStream_t s, cudaEvent_t* ev) {
  StepArgs a = make_args(sys, kind);
  if (ev) cudaEventRecord(ev[0], s);
  if (sys->peer)  // the neighbours have written this step's ghost states (and read ours)
    launch_peer_wait(sys->d_ctl, sys->remote_flag[0] ? sys->d_flags : nullptr,
                     sys->remote_flag[1] ? sys->d_flags + 1 : nullptr, s);
  launch_mesh_pose(a, s);
  // the scatter no longer returns the bin counts to zero (the small spheres take their ranks from
  // the counting pass): clear them before a counting pass
  if (DEM_SCATTER_RANKS && a.count) cudaMemsetAsync(sys->d_cell_count, 0, sizeof(int) * sys->ncell, s);
  launch_pose_count(a, s);
  if (ev) cudaEventRecord(ev[1], s);
}

static void enqueue_detect(dem_system* sys, int kind, cudaStream_t s, cudaEvent_t* ev) {
  const bool run = kind == K_FULL || kind == K_AHEAD;
  StepArgs a = make_args(sys, kind, /*det=*/kind == K_AHEAD);
  // an ahead detection also stops on the main abort word (a capacity abort of an earlier step of
  // the same launch batch: the re-run must find the entry sets as they were)
  const int* abort = a.abort;
  const int* abort2 = &sys->d_ctl->abort;
  if (run && sys->n_tri) cudaMemsetAsync(a.mlist_out_n, 0, sizeof(int), s);
  if (run) launch_excl_scan(sys->d_cell_count, sys->d_cell_start, sys->ncell, sys->d_scan_tmp, abort, s, abort2,
                           DEM_SCATTER_RANKS, a.pdl);
  if (ev) cudaEventRecord(ev[2], s);
  if (run) launch_bin_scatter(a, s);
  if (run) launch_mesh_pairs(a, s);
  if (ev) cudaEventRecord(ev[3], s);
  if (run) launch_pairs(a, s, sys->n_sm);
  if (ev) cudaEventRecord(ev[4], s);
  if (run) launch_excl_scan(sys->d_row_cnt, a.rows.row_ptr, sys->ns, sys->d_scan_tmp, abort, s, abort2, 0, a.pdl);
  if (ev) cudaEventRecord(ev[5], s);
  if (run) launch_rows_finish(a, s);
  if (ev) cudaEventRecord(ev[6], s);
}

static void enqueue_force(dem_system* sys, int kind, cudaStream_t s, cudaEvent_t* ev, bool exchange) {
  StepArgs a = make_args(sys, kind);
  launch_mesh_geom(a, s);
  launch_force_integrate(a, s);
  launch_mesh_finish(a, s);
  if (ev) cudaEventRecord(ev[7], s);
  if (sys->peer) {
    launch_peer_signal(sys->d_ctl, sys->remote_flag[0], sys->remote_flag[1], s);
  } else if (sys->dist) {
    enqueue_pack(sys, a, s);
    if (exchange && sys->P.transport == DEM_TRANSPORT_NCCL) {
      enqueue_nccl_exchange(sys, s);
      enqueue_unpack(sys, a, s);
    }
  }
  if (ev) cudaEventRecord(ev[8], s);
}

// the whole step on one stream (sequential; an AHEAD step's detection runs in line — the same
// results as the concurrent launch, which only changes when the kernels run)
// A distributed rank aborts a rebuild step only together with every other rank: the abort word
// (a capacity overflow in the detection) is all-reduced (MAX) before the force kernel, so every
// rank carries the same steps forward and the host regrows and re-runs them on every rank alike.
static void enqueue_abort_vote(dem_system* sys, int kind, cudaStream_t s) {
  if (sys->dist && sys->comm && (kind == K_FULL || kind == K_ADOPT))
    ncclAllReduce(&sys->d_ctl->abort, &sys->d_ctl->abort, 1, ncclInt32, ncclMax, sys->comm, s);
}

static void enqueue_step(dem_system* sys, int kind, cudaStream_t s, cudaEvent_t* ev, bool exchange = true) {
  enqueue_pose(sys, kind, s, ev);
  enqueue_detect(sys, kind, s, ev);
  enqueue_abort_vote(sys, kind, s);
  enqueue_force(sys, kind, s, ev, exchange);
}

static void enqueue_part(dem_system* sys, int kind, int part, cudaStream_t s) {
  if (part == PART_ALL) enqueue_step(sys, kind, s, nullptr);
  if (part == PART_POSE) enqueue_pose(sys, kind, s, nullptr);
  if (part == PART_DET) enqueue_detect(sys, kind, s, nullptr);
  if (part == PART_FORCE) enqueue_force(sys, kind, s, nullptr, true);
}

#ifndef DEM_OVERLAP_PRIORITY
#define DEM_OVERLAP_PRIORITY 1
#endif
static int graph_key(const dem_system* sys, int kind, int part) {
  return sys->sp | (sys->up << 1) | (sys->ep << 2) | (kind << 3) | (part << 5);
}

// the graph of one step (part) for the current parities, captured on first use
static dem_status step_graph(dem_system* sys, int kind, int part, cudaGraphExec_t* out) {
  const int key = graph_key(sys, kind, part);
  if (!sys->graph[key]) {
    cudaGraph_t g;
    // overlapped cadence: the force steps' kernels are captured on a high-priority stream and the
    // graphs instantiated with per-node priorities, so the detection running beside them on
    // det_stream (default = lowest priority) only takes the SM slots the force kernels leave
    const bool prio = DEM_OVERLAP_PRIORITY && sys->P.overlap && part != PART_DET && sys->cap_hi;
    cudaStream_t cs = prio ? sys->cap_hi : sys->cap_stream;
    CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    enqueue_part(sys, kind, part, cs);
    CK(cudaStreamEndCapture(cs, &g));
    if (prio) {  // every kernel node at the highest priority (explicitly, not only by capture stream)
      size_t nn = 0;
      CK(cudaGraphGetNodes(g, nullptr, &nn));
      std::vector<cudaGraphNode_t> nodes(nn);
      if (nn) CK(cudaGraphGetNodes(g, nodes.data(), &nn));
      int least = 0, greatest = 0;
      CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
      cudaLaunchAttributeValue v{};
      v.priority = greatest;
      for (cudaGraphNode_t nd : nodes) {
        cudaGraphNodeType t;
        CK(cudaGraphNodeGetType(nd, &t));
        if (t == cudaGraphNodeTypeKernel) CK(cudaGraphKernelNodeSetAttribute(nd, cudaLaunchAttributePriority, &v));
      }
    }
    cudaError_t e = cudaGraphInstantiate(&sys->graph[key], g,
                                         DEM_OVERLAP_PRIORITY && sys->P.overlap ? cudaGraphInstantiateFlagUseNodePriority : 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
      sys->err = std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e);
      return DEM_ERR_CUDA;
    }
  }
  sys->graphs_valid = true;
  *out = sys->graph[key];
  return DEM_OK;
}

// ------------------------------------------------------------------ validation / tables
static bool material_ok(const dem_material& m) {
  return m.E > 0 && m.nu >= 0 && m.nu < 0.5 && m.mu >= 0 && m.cor > 0 && m.cor <= 1 && std::isfinite(m.E);
}

// pair parameters (DESIGN.md §3 R4): series E*, G*; min CoR -> beta; min mu
static void pair_params(const dem_material& A, const dem_material& B, double out[4]) {
  double ie = (1.0 - A.nu * A.nu) / A.E + (1.0 - B.nu * B.nu) / B.E;
  double ig = 2.0 * (2.0 - A.nu) * (1.0 + A.nu) / A.E + 2.0 * (2.0 - B.nu) * (1.0 + B.nu) / B.E;
  double e = std::min(A.cor, B.cor);
  double beta = 0.0;
  if (e < 1.0) {
    double le = std::log(e);
    beta = -le / std::sqrt(le * le + M_PI * M_PI);
  }
  out[0] = 1.0 / ie;
  out[1] = 1.0 / ig;
  out[2] = beta;
  out[3] = std::min(A.mu, B.mu);
}

extern "C" const char* dem_status_string(dem_status s) {
  switch (s) {
    case DEM_OK: return "ok";
    case DEM_ERR_INVALID_ARG: return "invalid argument";
    case DEM_ERR_CUDA: return "CUDA error";
    case DEM_ERR_OOM: return "out of device memory";
    case DEM_ERR_NCCL: return "NCCL error";
    case DEM_ERR_BAD_MATERIAL: return "bad material";
    case DEM_ERR_BAD_TEMPLATE: return "bad template";
    case DEM_ERR_OUT_OF_DOMAIN: return "sphere out of domain";
    case DEM_ERR_NONFINITE: return "non-finite wrench";
    case DEM_ERR_DEGENERATE_CONTACT: return "degenerate contact (coincident centres)";
    case DEM_ERR_REPARTITION: return "owned clump drifted beyond drift_max (repartition)";
    case DEM_ERR_VMAX: return "sphere moved more than margin/2 since the last contact-set rebuild";
    case DEM_ERR_CAPACITY: return "capacity";
  }
  return "unknown";
}

extern "C" dem_status dem_last_error(const dem_system* sys, char* buf, size_t len) {
  if (!sys || !buf || !len) return DEM_ERR_INVALID_ARG;
  std::snprintf(buf, len, "%s", sys->err.c_str());
  return DEM_OK;
}

extern "C" dem_status dem_create(const dem_params* params, const dem_material* materials, int32_t n_mat,
                                 const dem_template* templates, int32_t n_tmpl, const dem_plane* planes,
                                 int32_t n_planes, void* cuda_stream, dem_system** out) {
  if (!params || !out || n_mat <= 0 || n_tmpl <= 0 || n_planes < 0 || n_planes > kMaxPlanes || !materials ||
      !templates || (n_planes && !planes))
    return DEM_ERR_INVALID_ARG;
  if (!(params->h > 0) || params->margin < 0 || params->cd_every < 1 || params->cell_size < 0 ||
      (params->cd_every > 1 && !(params->margin > 0)) || (params->overlap && params->cd_every < 2))
    return DEM_ERR_INVALID_ARG;
  for (int d = 0; d < 3; ++d)
    if (!(params->domain_hi[d] > params->domain_lo[d])) return DEM_ERR_INVALID_ARG;
  if (params->n_ranks > 1 &&
      (params->rank < 0 || params->rank >= params->n_ranks || !(params->slab_hi > params->slab_lo) ||
       !(params->halo > 0) || !(params->drift_max >= 0) ||
       (params->transport < DEM_TRANSPORT_NCCL || params->transport > DEM_TRANSPORT_LOOPBACK_PEER)))
    return DEM_ERR_INVALID_ARG;
  for (int m = 0; m < n_mat; ++m)
    if (!material_ok(materials[m])) return DEM_ERR_BAD_MATERIAL;
  for (int p = 0; p < n_planes; ++p) {
    const double* nv = planes[p].normal;
    double nn = std::sqrt(nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2]);
    if (std::fabs(nn - 1.0) > 1e-9 || planes[p].material < 0 || planes[p].material >= n_mat)
      return DEM_ERR_INVALID_ARG;
  }
  for (int t = 0; t < n_tmpl; ++t) {
    const dem_template& T = templates[t];
    if (T.n_comp < 1 || T.n_comp > kKeyStride || !T.offset || !T.radius || !T.material || !(T.mass > 0) ||
        !(T.inertia[0] > 0) || !(T.inertia[1] > 0) || !(T.inertia[2] > 0))
      return DEM_ERR_BAD_TEMPLATE;
    for (int k = 0; k < T.n_comp; ++k)
      if (!(T.radius[k] > 0) || T.material[k] < 0 || T.material[k] >= n_mat) return DEM_ERR_BAD_TEMPLATE;
  }
  if (params->n_ranks > 1) {
    // the ghost band must hold every clump a owned sphere can touch before the next migration:
    // 2 R_bound,max + margin + 2 drift_max; a thinner band misses contacts silently
    double rb_max = 0.0;
    for (int t = 0; t < n_tmpl; ++t)
      for (int k = 0; k < templates[t].n_comp; ++k) {
        const double* o = templates[t].offset + 3 * k;
        rb_max = std::max(rb_max, std::sqrt(o[0] * o[0] + o[1] * o[1] + o[2] * o[2]) + templates[t].radius[k]);
      }
    const double need = 2.0 * rb_max + params->margin + 2.0 * params->drift_max;
    if (params->halo < need * (1.0 - 1e-12)) return DEM_ERR_INVALID_ARG;
  }
  dem_system* sys = new dem_system();
  sys->P = *params;
  if (const char* fi = std::getenv("DEM_FAULT_AHEAD_OVERFLOW")) sys->fault_ahead = std::atoi(fi);
  if (const char* np = std::getenv("DEM_NO_PDL")) sys->no_pdl = std::atoi(np) ? 1 : 0;
  if (const char* tp = std::getenv("DEM_PAIRS_TINY")) sys->tiny_force = std::atoi(tp) ? 1 : 0;
  if (const char* sd = std::getenv("DEM_DEBUG_SERIAL_DET")) sys->debug_serial_det = std::atoi(sd) != 0;
  sys->stream = (cudaStream_t)cuda_stream;
  sys->n_mat = n_mat;
  sys->n_tmpl = n_tmpl;
  sys->n_planes = n_planes;
  sys->planes.assign(planes, planes + n_planes);
  sys->rmin = 1e300;
  sys->rmax = 0;
  for (int t = 0; t < n_tmpl; ++t) {
    const dem_template& T = templates[t];
    sys->tpl_coff.push_back((int)sys->tc_rad.size());
    sys->tpl_ncomp.push_back(T.n_comp);
    sys->tpl_mass.push_back(T.mass);
    for (int d = 0; d < 3; ++d) sys->tpl_inertia.push_back(T.inertia[d]);
    for (int k = 0; k < T.n_comp; ++k) {
      for (int d = 0; d < 3; ++d) sys->tc_off.push_back(T.offset[3 * k + d]);
      sys->tc_rad.push_back(T.radius[k]);
      sys->tc_mat.push_back(T.material[k]);
      sys->rmin = std::min(sys->rmin, T.radius[k]);
      sys->rmax = std::max(sys->rmax, T.radius[k]);
    }
  }
  // per material pair, the factors of the force law (kernels_force.cu): 2E*, 8G*,
  // 2 sqrt(5/6) beta, mu, sqrt(4 G*/E*) (so c_t = c_n sqrt(k_t / S_n) without a second sqrt)
  sys->pair.assign((size_t)n_mat * n_mat * 8, 0.0);
  for (int i = 0; i < n_mat; ++i)
    for (int j = i; j < n_mat; ++j) {
      double o[4];
      pair_params(materials[i], materials[j], o);
      const double f[5] = {2.0 * o[0], 8.0 * o[1], 2.0 * std::sqrt(5.0 / 6.0) * o[2], o[3], std::sqrt(4.0 * o[1] / o[0])};
      for (int q = 0; q < 5; ++q) {
        sys->pair[8 * (i * n_mat + j) + q] = f[q];
        sys->pair[8 * (j * n_mat + i) + q] = f[q];
      }
    }
  cudaError_t e = cudaStreamCreateWithFlags(&sys->cap_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&sys->det_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess && params->overlap) {
    int least = 0, greatest = 0;
    e = cudaDeviceGetStreamPriorityRange(&least, &greatest);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&sys->cap_hi, cudaStreamNonBlocking, greatest);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sys->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sys->ev_det, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    delete sys;
    return DEM_ERR_CUDA;
  }
  auto up = [&](auto** dst, const auto& vec) -> dem_status {
    using T = std::remove_reference_t<decltype(**dst)>;
    TRY(alloc_arr(sys, dst, vec.size()));
    if (cudaMemcpyAsync(*dst, vec.data(), sizeof(T) * vec.size(), cudaMemcpyHostToDevice, sys->stream) !=
        cudaSuccess)
      return DEM_ERR_CUDA;
    return DEM_OK;
  };
  dem_status st = DEM_OK;
  if ((st = up(&sys->d_tc_off, sys->tc_off)) || (st = up(&sys->d_tc_rad, sys->tc_rad)) ||
      (st = up(&sys->d_tc_mat, sys->tc_mat)) || (st = up(&sys->d_tpl_coff, sys->tpl_coff)) ||
      (st = up(&sys->d_tpl_mass, sys->tpl_mass)) || (st = up(&sys->d_tpl_inertia, sys->tpl_inertia)) ||
      (st = up(&sys->d_pair, sys->pair))) {
    dem_destroy(sys);
    return st;
  }
  if ((st = alloc_arr(sys, &sys->d_ctl, 1)) || (st = alloc_arr(sys, &sys->d_counter, 1))) {
    dem_destroy(sys);
    return st;
  }
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sys->n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (sys->n_sm <= 0) sys->n_sm = 148;
  }
  if (cudaMallocHost(&sys->h_ctl, sizeof(Ctl)) != cudaSuccess) {
    dem_destroy(sys);
    return DEM_ERR_CUDA;
  }
  std::memset(sys->h_ctl, 0, sizeof(Ctl));
  cudaMemcpyAsync(sys->d_ctl, sys->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, sys->stream);
  if (cudaStreamSynchronize(sys->stream) != cudaSuccess) {
    dem_destroy(sys);
    return DEM_ERR_CUDA;
  }
  if (params->n_ranks > 1) {
    sys->dist = true;
    sys->peer = params->transport == DEM_TRANSPORT_PEER || params->transport == DEM_TRANSPORT_LOOPBACK_PEER;
    if (sys->peer) {
      if (cudaMalloc(&sys->d_flags, 2 * sizeof(int)) != cudaSuccess ||
          cudaMemset(sys->d_flags, 0, 2 * sizeof(int)) != cudaSuccess) {
        dem_destroy(sys);
        return DEM_ERR_OOM;
      }
    }
    bool have_id = false;
    for (int k = 0; k < 128; ++k) have_id |= params->nccl_id[k] != 0;
    if (params->transport == DEM_TRANSPORT_NCCL || (params->transport == DEM_TRANSPORT_PEER && have_id)) {
      ncclUniqueId id;
      static_assert(sizeof(id.internal) == 128, "ncclUniqueId size");
      std::memcpy(id.internal, params->nccl_id, 128);
      ncclResult_t r = ncclCommInitRank(&sys->comm, params->n_ranks, id, params->rank);
      if (r != ncclSuccess) {
        sys->err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
        dem_destroy(sys);
        return DEM_ERR_NCCL;
      }
    }
  }
  *out = sys;
  return DEM_OK;
}

extern "C" dem_status dem_nccl_unique_id(unsigned char out[128]) {
  if (!out) return DEM_ERR_INVALID_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return DEM_ERR_NCCL;
  std::memcpy(out, id.internal, 128);
  return DEM_OK;
}

extern "C" void dem_destroy(dem_system* sys) {
  if (!sys) return;
  if (sys->det_stream) cudaStreamSynchronize(sys->det_stream);
  cudaStreamSynchronize(sys->stream);
  peer_release(sys);
  if (sys->d_flags) cudaFree(sys->d_flags);
  if (sys->comm) ncclCommDestroy(sys->comm);
  free_graphs(sys);
  std::vector<void*> ptrs;
  for (auto& kv : sys->allocs) ptrs.push_back(kv.first);
  for (void* p : ptrs) dfree(sys, p);
  cudaStreamSynchronize(sys->stream);
  if (sys->h_ctl) cudaFreeHost(sys->h_ctl);
  for (auto e : sys->ev) cudaEventDestroy(e);
  if (sys->cap_stream) cudaStreamDestroy(sys->cap_stream);
  if (sys->cap_hi) cudaStreamDestroy(sys->cap_hi);
  if (sys->det_stream) cudaStreamDestroy(sys->det_stream);
  if (sys->ev_fork) cudaEventDestroy(sys->ev_fork);
  if (sys->ev_det) cudaEventDestroy(sys->ev_det);
  delete sys;
}

// ------------------------------------------------------------------ capacity
// mesh-entry lists and the per-entry geometry (meshes only; sized like the entry arrays)
static dem_status alloc_mesh_lists(dem_system* sys) {
  if (!sys->n_mesh || !sys->cap_entries) return DEM_OK;
  for (int e = 0; e < 2; ++e) TRY(alloc_arr(sys, &sys->d_mlist[e], (size_t)sys->cap_entries));
  TRY(alloc_arr(sys, &sys->d_mgeom, (size_t)sys->cap_entries));
  TRY(alloc_arr(sys, &sys->d_mlist_n, 2));
  CK(cudaMemsetAsync(sys->d_mlist_n, 0, 2 * sizeof(int), sys->stream));
  return DEM_OK;
}

static dem_status alloc_rows(dem_system* sys, long long cap) {
  // grow both row buffers to cap entries, preserving the contents of both
  for (int p = 0; p < 2; ++p) {
    RowBuf nb;
    nb.row_ptr = sys->rows[p].row_ptr;
    nb.ent = (Entry*)dalloc(sys, sizeof(Entry) * cap);
    nb.key = (long long*)dalloc(sys, sizeof(long long) * cap);
    nb.ut = (double*)dalloc(sys, sizeof(double) * kUt * cap);
    if (!nb.ent || !nb.key || !nb.ut) {
      sys->err = "row buffer allocation failed";
      return DEM_ERR_OOM;
    }
    // zeroed once per (rare) growth, so no byte of a row buffer is ever read uninitialised
    // (compute-sanitizer initcheck; the old contents are copied over the front below)
    CK(cudaMemsetAsync(nb.ent, 0, sizeof(Entry) * cap, sys->stream));
    CK(cudaMemsetAsync(nb.key, 0, sizeof(long long) * cap, sys->stream));
    CK(cudaMemsetAsync(nb.ut, 0, sizeof(double) * kUt * cap, sys->stream));
    if (sys->rows[p].ent && sys->cap_entries) {
      size_t m = (size_t)std::min(cap, sys->cap_entries);
      cudaMemcpyAsync(nb.ent, sys->rows[p].ent, sizeof(Entry) * m, cudaMemcpyDeviceToDevice, sys->stream);
      cudaMemcpyAsync(nb.key, sys->rows[p].key, sizeof(long long) * m, cudaMemcpyDeviceToDevice, sys->stream);
      cudaMemcpyAsync(nb.ut, sys->rows[p].ut, sizeof(double) * kUt * m, cudaMemcpyDeviceToDevice, sys->stream);
    }
    dfree(sys, sys->rows[p].ent);
    dfree(sys, sys->rows[p].key);
    dfree(sys, sys->rows[p].ut);
    sys->rows[p] = nb;
  }
  if (sys->P.record_contacts) {
    TRY(alloc_arr(sys, &sys->rec.F, 3 * cap));
    TRY(alloc_arr(sys, &sys->rec.p, 3 * cap));
    TRY(alloc_arr(sys, &sys->rec.n, 3 * cap));
    TRY(alloc_arr(sys, &sys->rec.delta, cap));
  }
  sys->cap_entries = cap;
  TRY(alloc_mesh_lists(sys));
  free_graphs(sys);
  return DEM_OK;
}

// ------------------------------------------------------------------ peer transports (fused halo)
// Release the neighbour mappings and our IPC-exported state arrays (dem_set_state, dem_destroy).
static dem_status peer_release(dem_system* sys) {
  for (void* p : sys->ipc_open) cudaIpcCloseMemHandle(p);
  sys->ipc_open.clear();
  for (int p = 0; p < 2; ++p) {
    if (sys->raw_state[p]) cudaFree(sys->raw_state[p]);
    sys->raw_state[p] = nullptr;
    sys->d_state[p] = nullptr;
  }
  for (int side = 0; side < 2; ++side) {
    sys->remote_state[side][0] = sys->remote_state[side][1] = nullptr;
    sys->remote_n[side] = 0;
    sys->remote_flag[side] = nullptr;
  }
  return DEM_OK;
}

// our owned clumps' ghost slots in a neighbour: the k-th clump of our send list to that side
// is the k-th of its receive list from us (both ascending gid)
static dem_status peer_set_index(dem_system* sys, int side, const std::vector<int>& their_recv) {
  std::vector<int> idx((size_t)std::max<int64_t>(sys->n_own, 1), -1);
  if (their_recv.size() != sys->h_send_list[side].size()) {
    sys->err = "peer halo: send and receive lists of neighbouring ranks differ";
    return DEM_ERR_INVALID_ARG;
  }
  for (size_t k = 0; k < their_recv.size(); ++k) idx[sys->h_send_list[side][k]] = their_recv[k];
  TRY(alloc_arr(sys, &sys->d_peer_idx[side], idx.size()));
  CK(cudaMemcpy(sys->d_peer_idx[side], idx.data(), sizeof(int) * idx.size(), cudaMemcpyHostToDevice));
  return DEM_OK;
}

// PEER (one process per GPU): every rank exports its IPC handles (two state arrays, flag words),
// its clump count and its two receive lists; each rank imports its neighbours' packets (the
// caller moves the bytes, e.g. torch.distributed all_gather) and maps their arrays with peer
// access (NVLink)
struct PeerHeader {
  cudaIpcMemHandle_t state[2], flags;
  long long n, len[2];
};

extern "C" dem_status dem_peer_export(dem_system* sys, int64_t cap, void* out, int64_t* len) {
  if (!sys || !len || !sys->peer || sys->P.transport != DEM_TRANSPORT_PEER) return DEM_ERR_INVALID_ARG;
  const int64_t need = (int64_t)(sizeof(PeerHeader) + sizeof(int) * (sys->h_recv_list[0].size() +
                                                                       sys->h_recv_list[1].size()));
  *len = need;
  if (!out) return DEM_OK;
  if (cap < need || !sys->raw_state[0]) return DEM_ERR_INVALID_ARG;
  PeerHeader h{};
  CK(cudaIpcGetMemHandle(&h.state[0], sys->raw_state[0]));
  CK(cudaIpcGetMemHandle(&h.state[1], sys->raw_state[1]));
  CK(cudaIpcGetMemHandle(&h.flags, sys->d_flags));
  h.n = sys->n;
  h.len[0] = (long long)sys->h_recv_list[0].size();
  h.len[1] = (long long)sys->h_recv_list[1].size();
  char* o = (char*)out;
  std::memcpy(o, &h, sizeof h);
  o += sizeof h;
  for (int side = 0; side < 2; ++side) {
    std::memcpy(o, sys->h_recv_list[side].data(), sizeof(int) * sys->h_recv_list[side].size());
    o += sizeof(int) * sys->h_recv_list[side].size();
  }
  return DEM_OK;
}

extern "C" dem_status dem_peer_import(dem_system* sys, const void* left, const void* right) {
  if (!sys || !sys->peer || sys->P.transport != DEM_TRANSPORT_PEER) return DEM_ERR_INVALID_ARG;
  const int r = sys->P.rank, P = sys->P.n_ranks;
  if ((r > 0) != (left != nullptr) || (r < P - 1) != (right != nullptr)) return DEM_ERR_INVALID_ARG;
  for (void* p : sys->ipc_open) cudaIpcCloseMemHandle(p);
  sys->ipc_open.clear();
  for (int side = 0; side < 2; ++side) {
    const char* pk = (const char*)(side == 0 ? left : right);
    if (!pk) continue;
    PeerHeader h;
    std::memcpy(&h, pk, sizeof h);
    // the neighbour's receive list from us: its list from the right if it is our left neighbour
    const int theirs_side = side == 0 ? 1 : 0;
    const int* lists = (const int*)(pk + sizeof h);
    std::vector<int> their_recv(lists + (theirs_side == 0 ? 0 : h.len[0]),
                                lists + (theirs_side == 0 ? 0 : h.len[0]) + h.len[theirs_side]);
    TRY(peer_set_index(sys, side, their_recv));
    for (int p = 0; p < 2; ++p) {
      void* ptr = nullptr;
      CK(cudaIpcOpenMemHandle(&ptr, h.state[p], cudaIpcMemLazyEnablePeerAccess));
      sys->ipc_open.push_back(ptr);
      sys->remote_state[side][p] = (double*)ptr;
    }
    void* fl = nullptr;
    CK(cudaIpcOpenMemHandle(&fl, h.flags, cudaIpcMemLazyEnablePeerAccess));
    sys->ipc_open.push_back(fl);
    sys->remote_flag[side] = (int*)fl + (side == 0 ? 1 : 0);  // we are its right / left neighbour
    sys->remote_n[side] = h.n;
  }
  sys->peer_linked = true;
  free_graphs(sys);
  return DEM_OK;
}

// LOOPBACK_PEER (one process, one GPU): the same links made with plain device pointers
static dem_status peer_link_local(dem_system* const* systems, int n) {
  for (int r = 0; r < n; ++r) {
    dem_system* sys = systems[r];
    for (int side = 0; side < 2; ++side) {
      const int nb = side == 0 ? r - 1 : r + 1;
      if (nb < 0 || nb >= n) continue;
      dem_system* o = systems[nb];
      for (int p = 0; p < 2; ++p) sys->remote_state[side][p] = o->d_state[p];
      sys->remote_n[side] = o->n;
      sys->remote_flag[side] = o->d_flags + (side == 0 ? 1 : 0);
      TRY(peer_set_index(sys, side, o->h_recv_list[1 - side]));
    }
  }
  return DEM_OK;
}

// ------------------------------------------------------------------ meshes (NEXT-3)
// per-CTA wrench partials of the fused force kernel (sized by the CTA partition and the meshes)
static dem_status ensure_mesh_buffers(dem_system* sys) {
  if (!sys->n_mesh) return DEM_OK;
  const int nc = std::max(1, sys->n_cta);
  if (sys->mesh_part_ctas != nc || !sys->d_mesh_part) {
    TRY(alloc_arr(sys, &sys->d_mesh_part, (size_t)nc * kMaxMeshes * 6));
    TRY(alloc_arr(sys, &sys->d_mesh_flag, (size_t)nc));
    CK(cudaMemsetAsync(sys->d_mesh_flag, 0, sizeof(int) * nc, sys->stream));
    sys->mesh_part_ctas = nc;
  }
  return DEM_OK;
}

// one step's rotation of a mesh: h |w| about w/|w| (the exponential map of R12; the oracle's
// formula, so both sides advance a spinning mesh through the same bits)
static void mesh_step_quat(double h, const double* w, double* qs) {
  const double wn = std::sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  qs[0] = 1.0;
  qs[1] = qs[2] = qs[3] = 0.0;
  if (wn > 0.0) {
    const double half = 0.5 * (h * wn);
    const double sn = std::sin(half) / wn;
    qs[0] = std::cos(half);
    qs[1] = w[0] * sn;
    qs[2] = w[1] * sn;
    qs[3] = w[2] * sn;
  }
}

static void mesh_record(const dem_system* sys, const double* X, const double* q, const double* v, const double* w,
                        double* rec) {
  for (int d = 0; d < 3; ++d) rec[d] = X[d];
  for (int d = 0; d < 4; ++d) rec[3 + d] = q[d];
  for (int d = 0; d < 3; ++d) rec[7 + d] = v[d];
  for (int d = 0; d < 3; ++d) rec[10 + d] = w[d];
  mesh_step_quat(sys->P.h, w, rec + 13);
}

extern "C" dem_status dem_add_mesh(dem_system* sys, const dem_mesh* m, int32_t* mesh_id) {
  if (!sys || !m || m->n_tri < 1 || !m->verts || m->material < 0 || m->material >= sys->n_mat) return DEM_ERR_INVALID_ARG;
  if (sys->dist) {
    sys->err = "meshes are not supported on a distributed system";
    return DEM_ERR_INVALID_ARG;
  }
  if (sys->n_mesh >= kMaxMeshes || (int64_t)sys->n_tri + m->n_tri > (1 << 24)) {
    sys->err = "too many meshes or triangles";
    return DEM_ERR_INVALID_ARG;
  }
  const double qn = std::sqrt(m->quat[0] * m->quat[0] + m->quat[1] * m->quat[1] + m->quat[2] * m->quat[2] +
                              m->quat[3] * m->quat[3]);
  if (std::fabs(qn - 1.0) > 1e-9) return DEM_ERR_INVALID_ARG;
  CK(cudaStreamSynchronize(sys->stream));
  CK(cudaStreamSynchronize(sys->det_stream));
  const int t0 = sys->n_tri, n = (int)m->n_tri;
  sys->h_tri_body.insert(sys->h_tri_body.end(), m->verts, m->verts + 9 * (size_t)n);
  // topology: a vertex id is the first corner of the mesh with bitwise-equal body coordinates
  std::unordered_map<std::string, int> first;
  for (int k = 0; k < 3 * n; ++k) {
    std::string key((const char*)(m->verts + 3 * (size_t)k), 3 * sizeof(double));
    auto it = first.emplace(key, 3 * t0 + k).first;
    sys->h_tri_vid.push_back(it->second);
  }
  for (int k = 0; k < n; ++k) sys->h_tri_mesh.push_back(sys->n_mesh);
  sys->h_mesh_mat.push_back(m->material);
  sys->h_mesh.resize((size_t)kMeshRec * (sys->n_mesh + 1));
  mesh_record(sys, m->pos, m->quat, m->vel, m->omega, sys->h_mesh.data() + (size_t)kMeshRec * sys->n_mesh);
  // device copies: the mesh records are copied from the device first (poses advanced by steps)
  if (sys->n_mesh && sys->d_mesh)
    CK(cudaMemcpy(sys->h_mesh.data(), sys->d_mesh, sizeof(double) * kMeshRec * sys->n_mesh, cudaMemcpyDeviceToHost));
  sys->n_mesh += 1;
  sys->n_tri += n;
  auto up = [&](auto** dst, const auto& vec) -> dem_status {
    using T = std::remove_reference_t<decltype(**dst)>;
    TRY(alloc_arr(sys, dst, vec.size()));
    CK(cudaMemcpyAsync(*dst, vec.data(), sizeof(T) * vec.size(), cudaMemcpyHostToDevice, sys->stream));
    return DEM_OK;
  };
  TRY(up(&sys->d_tri_body, sys->h_tri_body));
  TRY(up(&sys->d_tri_vid, sys->h_tri_vid));
  TRY(up(&sys->d_tri_mesh, sys->h_tri_mesh));
  TRY(up(&sys->d_mesh_mat, sys->h_mesh_mat));
  TRY(up(&sys->d_mesh, sys->h_mesh));
  TRY(alloc_arr(sys, &sys->d_tri_world, (size_t)9 * sys->n_tri));
  TRY(alloc_arr(sys, &sys->d_tri_snap, (size_t)9 * sys->n_tri));
  TRY(alloc_arr(sys, &sys->d_mesh_wrench, (size_t)6 * kMaxMeshes));
  CK(cudaMemsetAsync(sys->d_mesh_wrench, 0, sizeof(double) * 6 * kMaxMeshes, sys->stream));
  sys->mesh_part_ctas = 0;
  TRY(ensure_mesh_buffers(sys));
  TRY(alloc_mesh_lists(sys));
  CK(cudaStreamSynchronize(sys->stream));
  free_graphs(sys);
  if (mesh_id) *mesh_id = sys->n_mesh - 1;
  return DEM_OK;
}

extern "C" dem_status dem_set_mesh_motion(dem_system* sys, int32_t mesh, const double pos[3], const double quat[4],
                                          const double vel[3], const double omega[3]) {
  if (!sys || mesh < 0 || mesh >= sys->n_mesh || !pos || !quat || !vel || !omega) return DEM_ERR_INVALID_ARG;
  double rec[kMeshRec];
  mesh_record(sys, pos, quat, vel, omega, rec);
  // ordered on the system stream after the steps already launched
  CK(cudaMemcpyAsync(sys->d_mesh + (size_t)kMeshRec * mesh, rec, sizeof(rec), cudaMemcpyHostToDevice, sys->stream));
  CK(cudaStreamSynchronize(sys->stream));
  return DEM_OK;
}

extern "C" dem_status dem_get_mesh(dem_system* sys, int32_t mesh, double pos[3], double quat[4], double force[3],
                                   double torque[3]) {
  if (!sys || mesh < 0 || mesh >= sys->n_mesh) return DEM_ERR_INVALID_ARG;
  CK(cudaStreamSynchronize(sys->stream));
  double rec[kMeshRec], w[6];
  CK(cudaMemcpy(rec, sys->d_mesh + (size_t)kMeshRec * mesh, sizeof(rec), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(w, sys->d_mesh_wrench + 6 * mesh, sizeof(w), cudaMemcpyDeviceToHost));
  if (pos) std::memcpy(pos, rec, 3 * sizeof(double));
  if (quat) std::memcpy(quat, rec + 3, 4 * sizeof(double));
  if (force) std::memcpy(force, w, 3 * sizeof(double));
  if (torque) std::memcpy(torque, w + 3, 3 * sizeof(double));
  return DEM_OK;
}

// ------------------------------------------------------------------ state
// The bin grid: edge `cell`; region = the box the held spheres occupy
// (box_lo/box_hi, empty if lo > hi) widened by 2 bins on every side, within the domain
// (distributed: also within slab +- halo in x).  Spheres that later stray outside the region are
// clamped into its edge bins, which stays exact (only speed depends on the bins); a centre that
// leaves it where it is tighter than the domain raises Ctl::need_regrid, and dem_step re-grids
// between step batches.  So a bed whose top lies far below the domain ceiling, or a slab of a
// long bed, is not charged for bins that hold nothing.  coarsen: grow the edge while a sparse
// region would need more than max(4M, 16 ns) bins (automatic cell size only).
static dem_status grid_layout(dem_system* sys, double cell, const double* box_lo, const double* box_hi, int64_t ns,
                              bool coarsen) {
  double blo[3], bhi[3];
  bool tight_lo[3], tight_hi[3];
  for (int d = 0; d < 3; ++d) {
    blo[d] = sys->P.domain_lo[d];
    bhi[d] = sys->P.domain_hi[d];
    if (box_hi[d] >= box_lo[d]) {
      blo[d] = std::max(blo[d], box_lo[d] - 2.0 * cell);
      bhi[d] = std::min(bhi[d], box_hi[d] + 2.0 * cell);
      if (!(bhi[d] > blo[d])) bhi[d] = blo[d] + cell;
    }
    tight_lo[d] = blo[d] > sys->P.domain_lo[d];
    tight_hi[d] = bhi[d] < sys->P.domain_hi[d];
  }
  if (sys->dist) {
    blo[0] = std::max(blo[0], sys->P.slab_lo - sys->P.halo);
    bhi[0] = std::min(bhi[0], sys->P.slab_hi + sys->P.halo);
    if (!(bhi[0] > blo[0])) bhi[0] = blo[0] + cell;
    tight_lo[0] = tight_hi[0] = false;  // the slab band is fixed; drift is guarded by drift_max
  }
  const long long max_cells = std::max<long long>(4LL << 20, 16 * ns);
  auto cells_for = [&](double c) {
    long long m = 1;
    for (int d = 0; d < 3; ++d) m *= (long long)std::ceil((bhi[d] - blo[d]) / c) + 1;
    return m;
  };
  if (coarsen && sys->P.cell_size <= 0)
    while (cells_for(cell) > max_cells) cell *= 1.25;
  Grid& G = sys->grid;
  G.cell = cell;
  G.inv_cell = 1.0 / cell;
  G.pad = 0.5 * sys->P.margin + 1e-9;
  long long ncell = 1;
  for (int d = 0; d < 3; ++d) {
    G.lo[d] = blo[d];
    G.dom_lo[d] = sys->P.domain_lo[d];
    G.dom_hi[d] = sys->P.domain_hi[d];
    G.reg_lo[d] = tight_lo[d] ? blo[d] : -1e300;
    G.reg_hi[d] = tight_hi[d] ? bhi[d] : 1e300;
    long long nd = (long long)std::ceil((bhi[d] - blo[d]) / cell) + 1;
    if (nd > (1LL << 20)) {
      sys->err = "grid too fine for the domain";
      return DEM_ERR_INVALID_ARG;
    }
    G.n[d] = (int)nd;
    ncell *= nd;
  }
  if (ncell > (1LL << 31) - (1LL << 24)) {  // (k_pairs iterates bins in 32 bits, with overshoot)
    sys->err = "too many bins; increase cell_size";
    return DEM_ERR_INVALID_ARG;
  }
  sys->ncell = ncell;
  // bin linearization: the axis with the fewest bins fastest, the longest slowest, so the
  // neighbours of a bin along every axis stay close in memory (and x-slabs are contiguous
  // for the usual longest-x beds)
  int ord[3] = {0, 1, 2};
#ifndef DEM_XFAST
  std::sort(ord, ord + 3, [&](int p, int q) { return G.n[p] != G.n[q] ? G.n[p] < G.n[q] : p > q; });
#endif
  long long st = 1;
  for (int k = 0; k < 3; ++k) {
    G.st[ord[k]] = st;
    st *= G.n[ord[k]];
    G.ax[k] = ord[k];
  }
  G.inv_n_ax[0] = 1.0 / G.n[ord[0]];
  G.inv_n_ax[1] = 1.0 / G.n[ord[1]];
  return DEM_OK;
}

extern "C" dem_status dem_set_state(dem_system* sys, int64_t n, const int64_t* gid, const int32_t* tid,
                                    const double* pos, const double* quat, const double* vel, const double* omega,
                                    int32_t on_device) {
  if (!sys || n < 0 || (n > 0 && (!gid || !tid || !pos || !quat || !vel || !omega))) return DEM_ERR_INVALID_ARG;
  if (n > (1LL << 30)) return DEM_ERR_INVALID_ARG;
  CK(cudaStreamSynchronize(sys->stream));
  CK(cudaStreamSynchronize(sys->det_stream));
  if (sys->peer && sys->P.transport == DEM_TRANSPORT_PEER && sys->raw_state[0] && sys->comm) {
    // the neighbours may still be storing ghost states into our arrays: a barrier before the
    // re-layout frees them (every rank calls dem_set_state; the steps before it are complete on
    // each rank once its stream has passed this all-reduce)
    CK(cudaMemsetAsync(sys->d_counter, 0, sizeof(unsigned long long), sys->stream));
    if (ncclAllReduce(sys->d_counter, sys->d_counter, 1, ncclUint64, ncclMax, sys->comm, sys->stream) != ncclSuccess)
      return DEM_ERR_NCCL;
    CK(cudaStreamSynchronize(sys->stream));
  }
  std::vector<long long> g(n);
  std::vector<int> t(n);
  std::vector<double> in[4];
  const double* src[4] = {pos, quat, vel, omega};
  const int width[4] = {3, 4, 3, 3};
  if (on_device) {
    if (n) {
      CK(cudaMemcpy(g.data(), gid, sizeof(long long) * n, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(t.data(), tid, sizeof(int) * n, cudaMemcpyDeviceToHost));
    }
  } else {
    for (int64_t c = 0; c < n; ++c) {
      g[c] = gid[c];
      t[c] = tid[c];
    }
  }
  // fast path: the same clumps as the last call (a state reset or restore): the state is
  // permuted into the existing storage order on the device, nothing is re-laid out.  A
  // distributed system also needs the same slab partition (roles of every clump by COM x).
  bool same = n > 0 && (int64_t)sys->h_in_gid.size() == n && sys->d_perm &&
              std::equal(g.begin(), g.end(), sys->h_in_gid.begin()) &&
              std::equal(t.begin(), t.end(), sys->h_in_tid.begin());
  if (same && sys->dist) {
    std::vector<double> hp;
    const double* P0 = pos;
    if (on_device) {
      hp.resize((size_t)3 * n);
      CK(cudaMemcpy(hp.data(), pos, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
      P0 = hp.data();
    }
    std::vector<int8_t> r2(n), f2(n);
    const dem_params& PP = sys->P;
    TRY(dem_partition_plan(n, P0, PP.slab_lo, PP.slab_hi, PP.halo, PP.rank > 0, PP.rank < PP.n_ranks - 1,
                           r2.data(), f2.data()));
    same = r2 == sys->h_role && f2 == sys->h_sendf;
  }
  if (same) {
    cudaStream_t s = sys->stream;
    const double* dsrc[4] = {pos, quat, vel, omega};
    if (!on_device) {
      size_t off = 0;
      for (int k = 0; k < 4; ++k) {
        CK(cudaMemcpyAsync(sys->d_io + off, src[k], sizeof(double) * width[k] * n, cudaMemcpyHostToDevice, s));
        dsrc[k] = sys->d_io + off;
        off += (size_t)width[k] * n;
      }
    }
    CK(cudaMemsetAsync(sys->d_io_bad, 0, sizeof(int), s));
    sys->sp = 0;
    const StepArgs a = make_args(sys, K_FULL);
    launch_state_in(a.cur, sys->d_perm, (int)sys->n, dsrc[0], dsrc[1], dsrc[2], dsrc[3], sys->d_io_bad,
                    sys->dist ? sys->d_xref : nullptr, (int)sys->n_own, s);
    CK(cudaMemsetAsync(sys->d_cell_count, 0, sizeof(int) * sys->ncell, s));
    for (int p = 0; p < 2; ++p) CK(cudaMemsetAsync(sys->rows[p].row_ptr, 0, sizeof(int) * (sys->ns + 1), s));
    std::memset(sys->h_ctl, 0, sizeof(Ctl));
    CK(cudaMemcpyAsync(sys->d_ctl, sys->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, s));
    int bad = 0;
    CK(cudaMemcpyAsync(&bad, sys->d_io_bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (bad) return DEM_ERR_NONFINITE;
    if (sys->peer) {
      // step counts restart at 0: so do the flag words, then every rank passes a barrier before
      // any of them steps again (a neighbour's first signal must not hit a flag word that is
      // still to be reset)
      CK(cudaMemset(sys->d_flags, 0, 2 * sizeof(int)));
      CK(cudaDeviceSynchronize());
      if (sys->comm) {
        CK(cudaMemsetAsync(sys->d_counter, 0, sizeof(unsigned long long), s));
        if (ncclAllReduce(sys->d_counter, sys->d_counter, 1, ncclUint64, ncclMax, sys->comm, s) != ncclSuccess)
          return DEM_ERR_NCCL;
        CK(cudaStreamSynchronize(s));
      }
    }
    sys->fast_resets++;
    sys->launched = 0;
    sys->steps_done = 0;
    sys->up = sys->ep = 0;
    sys->since_rebuild = 0;
    sys->pending = false;
    sys->last_entries = 0;
    sys->err.clear();
    return DEM_OK;
  }
  if (on_device) {
    for (int k = 0; k < 4; ++k) {
      in[k].resize((size_t)width[k] * n);
      if (n) CK(cudaMemcpy(in[k].data(), src[k], sizeof(double) * width[k] * n, cudaMemcpyDeviceToHost));
      src[k] = in[k].data();
    }
  }
  std::vector<long long> g_in(g);
  std::vector<int> t_in(t);
  // (the slab partition of this input is kept for the fast path's check)
  for (int64_t c = 0; c < n; ++c)
    if (t[c] < 0 || t[c] >= sys->n_tmpl || g[c] < 0 || g[c] >= (1LL << 56)) {
      sys->err = "clump " + std::to_string(c) + ": bad template id or gid";
      return DEM_ERR_INVALID_ARG;
    }
  // distributed: the held subset (owned + ghosts) of the global input
  std::vector<int8_t> role(n, 1), sendf(n, 0);
  if (sys->dist) {
    const dem_params& P = sys->P;
    TRY(dem_partition_plan(n, src[0], P.slab_lo, P.slab_hi, P.halo, P.rank > 0, P.rank < P.n_ranks - 1,
                           role.data(), sendf.data()));
    sys->h_role = role;
    sys->h_sendf = sendf;
  }
  free_graphs(sys);
  // grid: cell edge (auto: 4 x mean sphere radius + margin, at least 2 r_min + margin)
  int64_t ns = 0, n_hold = 0;
  double rsum = 0;
  for (int64_t c = 0; c < n; ++c) {
    if (!role[c]) continue;
    ++n_hold;
    ns += sys->tpl_ncomp[t[c]];
    for (int j = 0; j < sys->tpl_ncomp[t[c]]; ++j) rsum += sys->tc_rad[sys->tpl_coff[t[c]] + j];
  }
  if (ns >= (1LL << 29)) {  // the per-bin pair kernel packs sphere indices into 29 bits
    sys->err = "more than 2^29 spheres per system";
    return DEM_ERR_INVALID_ARG;
  }
  double rmean = ns ? rsum / ns : sys->rmax;
  double cell = sys->P.cell_size > 0 ? sys->P.cell_size : std::max(4.0 * rmean, 2.0 * sys->rmin) + sys->P.margin;
  // bin region: the box the held spheres occupy now (grid_layout)
  double box_lo[3] = {1e300, 1e300, 1e300}, box_hi[3] = {-1e300, -1e300, -1e300};
  if (n_hold > 0) {
    std::vector<double> rb(sys->n_tmpl, 0.0);  // bounding radius of each template
    for (int tt = 0; tt < sys->n_tmpl; ++tt)
      for (int j = 0; j < sys->tpl_ncomp[tt]; ++j) {
        const double* o = &sys->tc_off[3 * (sys->tpl_coff[tt] + j)];
        rb[tt] = std::max(rb[tt], std::sqrt(o[0] * o[0] + o[1] * o[1] + o[2] * o[2]) + sys->tc_rad[sys->tpl_coff[tt] + j]);
      }
    for (int64_t c = 0; c < n; ++c) {
      if (!role[c]) continue;
      for (int d = 0; d < 3; ++d) {
        const double x = src[0][3 * c + d];
        if (!std::isfinite(x)) continue;
        box_lo[d] = std::min(box_lo[d], x - rb[t[c]]);
        box_hi[d] = std::max(box_hi[d], x + rb[t[c]]);
      }
    }
  }
  TRY(grid_layout(sys, cell, box_lo, box_hi, ns, true));
  Grid& G = sys->grid;
  const long long ncell = sys->ncell;
  // storage order: owned clumps, then ghosts, each sorted by the bin of the COM (spatial
  // locality for every gather); results do not depend on it (keys, canonical sums).
  // h_perm maps storage -> caller index.
  int64_t n_own = 0;
  {
    std::vector<long long> ckey(n);
    for (int64_t c = 0; c < n; ++c) {
      long long id[3];
      for (int d = 0; d < 3; ++d) {
        double v = (src[0][3 * c + d] - G.lo[d]) * G.inv_cell;
        long long q = std::isfinite(v) ? (long long)std::floor(v) : 0;
        id[d] = std::min<long long>(std::max<long long>(q, 0), G.n[d] - 1);
      }
      ckey[c] = id[0] * G.st[0] + id[1] * G.st[1] + id[2] * G.st[2];
    }
    sys->h_perm.clear();
    for (int64_t c = 0; c < n; ++c)
      if (role[c] == 1) sys->h_perm.push_back(c);
    n_own = (int64_t)sys->h_perm.size();
    for (int64_t c = 0; c < n; ++c)
      if (role[c] >= 2) sys->h_perm.push_back(c);
    auto by_bin = [&](int64_t x, int64_t y) { return ckey[x] < ckey[y]; };
    std::stable_sort(sys->h_perm.begin(), sys->h_perm.begin() + n_own, by_bin);
    std::stable_sort(sys->h_perm.begin() + n_own, sys->h_perm.end(), by_bin);
    std::vector<long long> g2(n_hold);
    std::vector<int> t2(n_hold);
    for (int64_t c = 0; c < n_hold; ++c) {
      g2[c] = g[sys->h_perm[c]];
      t2[c] = t[sys->h_perm[c]];
    }
    g.swap(g2);
    t.swap(t2);
  }
  // halo lists (ascending gid on both sides of every exchange)
  std::vector<int> lists[4];  // send left, send right, recv left, recv right (storage indices)
  if (sys->dist) {
    for (int64_t i = 0; i < n_hold; ++i) {
      const int64_t c = sys->h_perm[i];
      if (i < n_own) {
        if (sendf[c] & 1) lists[0].push_back((int)i);
        if (sendf[c] & 2) lists[1].push_back((int)i);
      } else {
        lists[role[c] == 2 ? 2 : 3].push_back((int)i);
      }
    }
    for (auto& L : lists) std::sort(L.begin(), L.end(), [&](int x, int y) { return g[x] < g[y]; });
  }
  for (int side = 0; side < 2; ++side) {
    sys->h_send_list[side] = lists[side];
    sys->h_recv_list[side] = lists[2 + side];
  }
  n = n_hold;
  sys->n = n;
  sys->ns = ns;
  sys->n_own = n_own;
  sys->h_gid = g;
  sys->h_tid = t;
  sys->h_sph_off.assign(n + 1, 0);
  std::vector<int> s_clump(ns);
  sys->h_s_tc.assign(ns, 0);
  sys->h_s_key.assign(ns, 0);
  int64_t k = 0;
  for (int64_t c = 0; c < n; ++c) {
    sys->h_sph_off[c] = (int)k;
    for (int j = 0; j < sys->tpl_ncomp[t[c]]; ++j, ++k) {
      s_clump[k] = (int)c;
      sys->h_s_tc[k] = sys->tpl_coff[t[c]] + j;
      sys->h_s_key[k] = g[c] * kKeyStride + j;
    }
  }
  sys->h_sph_off[n] = (int)k;
  sys->ns_own = sys->h_sph_off[n_own];
  // SoA state on the host, one upload
  std::vector<double> st((size_t)13 * n);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t c = sys->h_perm[i];
    for (int d = 0; d < 3; ++d) st[(0 + d) * n + i] = src[0][3 * c + d];
    for (int d = 0; d < 4; ++d) st[(3 + d) * n + i] = src[1][4 * c + d];
    for (int d = 0; d < 3; ++d) st[(7 + d) * n + i] = src[2][3 * c + d];
    for (int d = 0; d < 3; ++d) st[(10 + d) * n + i] = src[3][3 * c + d];
    for (int d = 0; d < 3; ++d)
      if (!std::isfinite(src[0][3 * c + d]) || !std::isfinite(src[2][3 * c + d]) || !std::isfinite(src[3][3 * c + d]))
        return DEM_ERR_NONFINITE;
  }
  // upper bound of bin inserts: (floor(2e / cell) + 2)^3 per sphere
  long long ins = 0;
  for (int64_t s = 0; s < ns; ++s) {
    double e = sys->tc_rad[sys->h_s_tc[s]] + G.pad;
    long long m = (long long)std::floor(2.0 * e / G.cell) + 2;
    ins += m * m * m;
  }
  if (ins > (1LL << 31) - 2) ins = (1LL << 31) - 2;
  sys->cap_inserts = ins;
  // device arrays
  TRY(alloc_arr(sys, &sys->d_gid, n));
  TRY(alloc_arr(sys, &sys->d_tid, n));
  TRY(alloc_arr(sys, &sys->d_sph_off, n + 1));
  if (sys->peer) {
    // IPC-exportable state (the neighbours store ghost states into it); the old mappings and
    // arrays are released only after every rank has stopped stepping (barrier above)
    TRY(peer_release(sys));
    for (int p = 0; p < 2; ++p) {
      CK(cudaMalloc(&sys->raw_state[p], sizeof(double) * 13 * std::max<int64_t>(n, 1)));
      sys->d_state[p] = sys->raw_state[p];
    }
  } else {
    TRY(alloc_arr(sys, &sys->d_state[0], 13 * n));
    TRY(alloc_arr(sys, &sys->d_state[1], 13 * n));
  }
  TRY(alloc_arr(sys, &sys->d_kin, (size_t)kKin * n));
  TRY(alloc_arr(sys, &sys->d_s_clump, ns));
  TRY(alloc_arr(sys, &sys->d_s_tc, ns));
  TRY(alloc_arr(sys, &sys->d_s_mat, ns));
  TRY(alloc_arr(sys, &sys->d_s_key, ns));
  TRY(alloc_arr(sys, &sys->d_spos, ns));
  for (int e = 0; e < 2; ++e) TRY(alloc_arr(sys, &sys->d_spos_ref[e], sys->P.cd_every > 1 ? ns : 0));
  // candidate lists: kRowWidth slots per owned sphere to start with (walls included), widened
  // on overflow (the rows of a settled bed hold a few entries)
  sys->row_width = kRowWidth;
  TRY(alloc_arr(sys, &sys->d_slots, (size_t)sys->ns_own * sys->row_width + 1));
  if (DEM_SLOT_KEYS) TRY(alloc_arr(sys, &sys->d_slot_key, (size_t)sys->ns_own * sys->row_width + 1));
  // CTA partition of the fused force/integrate kernel: consecutive whole clumps, at most
  // force_cta_clumps() clumps and force_cta_spheres() spheres per CTA
  // (owned clumps only: ghosts are integrated by their owners)
  std::vector<int> cta{0};
  {
    int nc = 0, nsph = 0;
    for (int64_t c = 0; c < n_own; ++c) {
      const int m = sys->tpl_ncomp[t[c]];
      if (nc == force_cta_clumps() || nsph + m > force_cta_spheres()) {
        cta.push_back((int)c);
        nc = 0;
        nsph = 0;
      }
      ++nc;
      nsph += m;
    }
    if (n_own > 0) cta.push_back((int)n_own);
  }
  sys->n_cta = (int)cta.size() - 1;
  TRY(ensure_mesh_buffers(sys));
  TRY(alloc_arr(sys, &sys->d_cta_clump, cta.size()));
  TRY(alloc_arr(sys, &sys->d_cell_count, ncell));
  if (DEM_SCATTER_RANKS) TRY(alloc_arr(sys, &sys->d_irank, (size_t)kRankW * ns + 1));
  TRY(alloc_arr(sys, &sys->d_cell_start, ncell + 1));
  TRY(alloc_arr(sys, &sys->d_items, ins));
  TRY(alloc_arr(sys, &sys->d_row_cnt, ns + 1));
  TRY(alloc_arr(sys, &sys->d_wall_mask, ns + 1));
  TRY(alloc_arr(sys, &sys->d_scan_tmp, std::max(scan_tiles_needed(ncell), scan_tiles_needed(ns)) + 1));
  for (int p = 0; p < 2; ++p) TRY(alloc_arr(sys, &sys->rows[p].row_ptr, ns + 1));
  // halo buffers and the partition-time COMs of owned clumps (drift check)
  std::vector<double> xref((size_t)3 * n_own);
  for (int64_t i = 0; i < n_own; ++i)
    for (int d = 0; d < 3; ++d) xref[3 * i + d] = src[0][3 * sys->h_perm[i] + d];
  TRY(alloc_arr(sys, &sys->d_xref, xref.size() + 1));
  for (int side = 0; side < 2; ++side) {
    sys->n_send[side] = (int)lists[side].size();
    sys->n_recv[side] = (int)lists[2 + side].size();
    TRY(alloc_arr(sys, &sys->d_send_idx[side], lists[side].size() + 1));
    TRY(alloc_arr(sys, &sys->d_recv_idx[side], lists[2 + side].size() + 1));
    TRY(alloc_arr(sys, &sys->d_sendbuf[side], (size_t)kKin13 * lists[side].size() + 1));
    TRY(alloc_arr(sys, &sys->d_recvbuf[side], (size_t)kKin13 * lists[2 + side].size() + 1));
  }
  const double eps = sys->P.entries_per_sphere > 0 ? sys->P.entries_per_sphere : 8.0;
  long long cap = std::max<long long>(1024, (long long)(eps * ns));
  sys->cap_entries = 0;
  for (int p = 0; p < 2; ++p) {
    dfree(sys, sys->rows[p].ent); sys->rows[p].ent = nullptr;
    dfree(sys, sys->rows[p].key); sys->rows[p].key = nullptr;
    dfree(sys, sys->rows[p].ut); sys->rows[p].ut = nullptr;
  }
  TRY(alloc_rows(sys, cap));
  cudaStream_t s = sys->stream;
  {
    std::vector<int2> bnd(cta.size());  // (first clump, first sphere) of every CTA
    for (size_t k = 0; k < cta.size(); ++k) bnd[k] = make_int2(cta[k], (int)sys->h_sph_off[cta[k]]);
    CK(cudaMemcpyAsync(sys->d_cta_clump, bnd.data(), sizeof(int2) * bnd.size(), cudaMemcpyHostToDevice, s));
  }
  if (n_own) CK(cudaMemcpyAsync(sys->d_xref, xref.data(), sizeof(double) * xref.size(), cudaMemcpyHostToDevice, s));
  for (int side = 0; side < 2; ++side) {
    if (!lists[side].empty())
      CK(cudaMemcpyAsync(sys->d_send_idx[side], lists[side].data(), sizeof(int) * lists[side].size(),
                         cudaMemcpyHostToDevice, s));
    if (!lists[2 + side].empty())
      CK(cudaMemcpyAsync(sys->d_recv_idx[side], lists[2 + side].data(), sizeof(int) * lists[2 + side].size(),
                         cudaMemcpyHostToDevice, s));
  }
  CK(cudaMemcpyAsync(sys->d_gid, g.data(), sizeof(long long) * n, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(sys->d_tid, t.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(sys->d_sph_off, sys->h_sph_off.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(sys->d_state[0], st.data(), sizeof(double) * 13 * n, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(sys->d_s_clump, s_clump.data(), sizeof(int) * ns, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(sys->d_s_tc, sys->h_s_tc.data(), sizeof(int) * ns, cudaMemcpyHostToDevice, s));
  std::vector<int> s_mat(ns);
  for (int64_t k = 0; k < ns; ++k) s_mat[k] = sys->tc_mat[sys->h_s_tc[k]];
  CK(cudaMemcpyAsync(sys->d_s_mat, s_mat.data(), sizeof(int) * ns, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(sys->d_s_key, sys->h_s_key.data(), sizeof(long long) * ns, cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(sys->d_cell_count, 0, sizeof(int) * ncell, s));
  for (int p = 0; p < 2; ++p) CK(cudaMemsetAsync(sys->rows[p].row_ptr, 0, sizeof(int) * (ns + 1), s));
  std::memset(sys->h_ctl, 0, sizeof(Ctl));
  CK(cudaMemcpyAsync(sys->d_ctl, sys->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, s));
  // caller-order I/O: storage -> caller index, owned storage -> output row of dem_get_state
  // (the rank of its caller index among the owned ones), staging for the fast paths
  sys->h_in_gid.swap(g_in);
  sys->h_in_tid.swap(t_in);
  {
    std::vector<int> perm(n);
    for (int64_t i = 0; i < n; ++i) perm[i] = (int)sys->h_perm[i];
    sys->h_outpos.assign(n_own, 0);
    std::vector<int64_t> ord(n_own);
    for (int64_t i = 0; i < n_own; ++i) ord[i] = i;
    if (sys->dist)
      std::sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) { return sys->h_perm[x] < sys->h_perm[y]; });
    for (int64_t r = 0; r < n_own; ++r) sys->h_outpos[sys->dist ? ord[r] : r] = sys->dist ? (int)r : perm[r];
    TRY(alloc_arr(sys, &sys->d_perm, (size_t)n + 1));
    TRY(alloc_arr(sys, &sys->d_outpos, (size_t)n_own + 1));
    TRY(alloc_arr(sys, &sys->d_io, (size_t)13 * std::max<int64_t>(n, (int64_t)sys->h_in_gid.size()) + 1));
    TRY(alloc_arr(sys, &sys->d_io_bad, 1));
    if (n) CK(cudaMemcpyAsync(sys->d_perm, perm.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
    if (n_own)
      CK(cudaMemcpyAsync(sys->d_outpos, sys->h_outpos.data(), sizeof(int) * n_own, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
  }
  if (sys->peer) {
    // step counts restart at 0: the flag words too, before the collective link below (a
    // neighbour signals into them only after it has passed that link)
    CK(cudaMemset(sys->d_flags, 0, 2 * sizeof(int)));
    CK(cudaDeviceSynchronize());
    sys->peer_linked = false;  // PEER: dem_peer_export / dem_peer_import before the next step
  }
  sys->launched = 0;
  sys->steps_done = 0;
  sys->sp = sys->up = sys->ep = 0;
  sys->since_rebuild = 0;
  sys->pending = false;
  sys->entry_partitioned = false;
  sys->last_entries = 0;
  sys->err.clear();
  return DEM_OK;
}

// the history of the next step's rebuild (DEM_set_contact_history, migration): per held sphere
// (storage index) its entries {partner key, u_t oriented own -> partner}; only owned spheres get
// rows
struct HistEntry {
  long long key;
  double u[3];
};
static dem_status install_history(dem_system* sys, std::vector<std::vector<HistEntry>>& per) {
  CK(cudaStreamSynchronize(sys->det_stream));  // a set detected ahead is dropped
  std::vector<int> rp(sys->ns + 1, 0);
  std::vector<Entry> ents;
  std::vector<long long> keys;
  std::vector<double> ut;
  for (int64_t s = 0; s < sys->ns; ++s) {
    auto& v = per[s];
    std::sort(v.begin(), v.end(), [](const HistEntry& x, const HistEntry& y) { return x.key < y.key; });
    for (auto& e : v) {
      Entry en;
      en.partner = -1;  // only the key and u_t of the previous rows are read
      en.prev = -1;
      ents.push_back(en);
      keys.push_back(e.key);
      for (int d = 0; d < kUt; ++d) ut.push_back(d < 3 ? e.u[d] : 0.0);
    }
    rp[s + 1] = (int)ents.size();
  }
  long long m = (long long)ents.size();
  if (m > sys->cap_entries) TRY(alloc_rows(sys, m + m / 4 + 1024));
  // the imported history is the "previous" set of the next step, which is forced to be a rebuild
  cudaStream_t s = sys->stream;
  RowBuf& R = sys->rows[sys->ep];
  CK(cudaMemcpyAsync(R.row_ptr, rp.data(), sizeof(int) * (sys->ns + 1), cudaMemcpyHostToDevice, s));
  if (m) {
    CK(cudaMemcpyAsync(R.ent, ents.data(), sizeof(Entry) * m, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(R.key, keys.data(), sizeof(long long) * m, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(sys->rows[sys->up].ut, ut.data(), sizeof(double) * kUt * m, cudaMemcpyHostToDevice, s));
  }
  CK(cudaStreamSynchronize(s));
  sys->since_rebuild = 0;
  sys->pending = false;
  return DEM_OK;
}

extern "C" dem_status dem_set_contact_history(dem_system* sys, int64_t n, const int64_t* key_a,
                                              const int64_t* key_b, const double* u_t) {
  if (!sys || n < 0 || (n && (!key_a || !key_b || !u_t))) return DEM_ERR_INVALID_ARG;
  std::unordered_map<long long, int> idx;
  idx.reserve((size_t)sys->ns * 2);
  for (int64_t s = 0; s < sys->ns_own; ++s) idx[sys->h_s_key[s]] = (int)s;  // owned spheres only
  std::vector<std::vector<HistEntry>> per(sys->ns);
  for (int64_t r = 0; r < n; ++r) {
    if (!(key_a[r] < key_b[r])) return DEM_ERR_INVALID_ARG;
    auto ia = idx.find(key_a[r]);
    if (ia != idx.end()) per[ia->second].push_back(HistEntry{key_b[r], {u_t[3 * r], u_t[3 * r + 1], u_t[3 * r + 2]}});
    auto ib = idx.find(key_b[r]);
    if (ib != idx.end()) per[ib->second].push_back(HistEntry{key_a[r], {-u_t[3 * r], -u_t[3 * r + 1], -u_t[3 * r + 2]}});
  }
  return install_history(sys, per);
}

// ------------------------------------------------------------------ stepping
static dem_status read_ctl(dem_system* sys) {
  CK(cudaMemcpyAsync(sys->h_ctl, sys->d_ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, sys->stream));
  CK(cudaStreamSynchronize(sys->stream));
  return DEM_OK;
}

static dem_status device_error(dem_system* sys) {
  const Ctl& c = *sys->h_ctl;
  char buf[256];
  switch (c.err_code) {
    case DEM_ERR_OUT_OF_DOMAIN:
      std::snprintf(buf, sizeof buf, "sphere %lld of clump gid %lld left the domain at step %lld", c.err_key,
                    c.err_key2, c.err_step);
      break;
    case DEM_ERR_NONFINITE:
      std::snprintf(buf, sizeof buf, "non-finite wrench on clump gid %lld at step %lld", c.err_key, c.err_step);
      break;
    case DEM_ERR_DEGENERATE_CONTACT:
      std::snprintf(buf, sizeof buf, "coincident centres of spheres %lld and %lld at step %lld", c.err_key,
                    c.err_key2, c.err_step);
      break;
    case DEM_ERR_VMAX:
      std::snprintf(buf, sizeof buf, "sphere %lld of clump gid %lld moved more than margin/2 since the last "
                    "contact-set rebuild at step %lld", c.err_key, c.err_key2, c.err_step);
      break;
    case DEM_ERR_REPARTITION:
      std::snprintf(buf, sizeof buf, "owned clump gid %lld drifted beyond drift_max at step %lld: repartition",
                    c.err_key, c.err_step);
      break;
    default:
      std::snprintf(buf, sizeof buf, "device error %d at step %lld", c.err_code, c.err_step);
  }
  sys->err = buf;
  return (dem_status)c.err_code;
}

static dem_status ensure_events(dem_system* sys, int64_t steps) {
  size_t need = (size_t)steps * (kStages + 1);
  while (sys->ev.size() < need) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    sys->ev.push_back(e);
  }
  return DEM_OK;
}

// advance the host parities after a launched step
static void advance_parities(dem_system* sys, int kind) {
  sys->sp ^= 1;
  sys->up ^= 1;
  if (kind == K_FULL || kind == K_ADOPT) sys->ep ^= 1;
  if (kind == K_AHEAD) sys->pending = true;
  if (kind == K_ADOPT) sys->pending = false;
  sys->since_rebuild = (sys->since_rebuild + 1) % std::max(1, sys->P.cd_every);
  sys->launched++;
}

// The fused force kernel processes a CTA's entries in chunks of its thread count; cut at
// dem_set_state by clump and sphere counts only, a CTA's last chunk is often nearly empty.
// After the first steps (a contact set exists) the CTAs are re-cut along the same clump order
// with the entry count as a third bound (at most kEntCap entries: whole chunks).  Results do
// not depend on the cut (canonical sums per sphere and per clump).
// It is re-cut again whenever the entry count has changed by more than a quarter since (a bed
// settling from a spawn gains most of its contacts after the first cut).  A/B on the C5 bench:
// the force stage 4.99 -> 4.73 ms at 256 entries and 48 clumps per CTA.
#ifndef DEM_ENTRY_CAP
#define DEM_ENTRY_CAP 256  // 0: keep the clump/sphere cut of dem_set_state
#endif
static dem_status repartition_by_entries(dem_system* sys) {
  if (DEM_ENTRY_CAP <= 0 || sys->n_own == 0) return DEM_OK;
  CK(cudaStreamSynchronize(sys->stream));
  CK(cudaStreamSynchronize(sys->det_stream));  // its graphs are about to be re-captured
  int total = 0;
  CK(cudaMemcpy(&total, sys->rows[sys->ep].row_ptr + sys->ns, sizeof(int), cudaMemcpyDeviceToHost));
  if (sys->entry_partitioned && std::abs(total - sys->part_entries) <= sys->part_entries / 4) return DEM_OK;
  sys->entry_partitioned = true;
  sys->part_entries = total;
  std::vector<int> rp(sys->ns + 1);
  CK(cudaMemcpy(rp.data(), sys->rows[sys->ep].row_ptr, sizeof(int) * (sys->ns + 1), cudaMemcpyDeviceToHost));
  std::vector<int> cta{0};
  int nc = 0, nsph = 0, nent = 0;
  for (int64_t c = 0; c < sys->n_own; ++c) {
    const int s0 = sys->h_sph_off[c], s1 = sys->h_sph_off[c + 1];
    const int m = s1 - s0, ne = rp[s1] - rp[s0];
    if (nc > 0 && (nc == force_cta_clumps() || nsph + m > force_cta_spheres() || nent + ne > DEM_ENTRY_CAP)) {
      cta.push_back((int)c);
      nc = nsph = nent = 0;
    }
    ++nc;
    nsph += m;
    nent += ne;
  }
  cta.push_back((int)sys->n_own);
  std::vector<int2> bnd(cta.size());
  for (size_t k = 0; k < cta.size(); ++k) bnd[k] = make_int2(cta[k], sys->h_sph_off[cta[k]]);
  TRY(alloc_arr(sys, &sys->d_cta_clump, bnd.size()));
  CK(cudaMemcpy(sys->d_cta_clump, bnd.data(), sizeof(int2) * bnd.size(), cudaMemcpyHostToDevice));
  sys->n_cta = (int)cta.size() - 1;
  TRY(ensure_mesh_buffers(sys));
  free_graphs(sys);
  return DEM_OK;
}

// Deferred sets and moving meshes: a sphere may move margin/2 from where its set was detected
// (checked on the device), so a mesh point may move the other margin/2 over the steps a set is
// used (k, or 2k - 2 with the overlapped cadence): (|v| + |w| R_max) h lag <= margin/2.
static dem_status check_mesh_motion(dem_system* sys) {
  if (sys->P.cd_every <= 1 || !sys->n_mesh) return DEM_OK;
  const int lag = sys->P.overlap ? 2 * sys->P.cd_every - 2 : sys->P.cd_every;
  std::vector<double> rec((size_t)kMeshRec * sys->n_mesh);
  CK(cudaMemcpy(rec.data(), sys->d_mesh, sizeof(double) * rec.size(), cudaMemcpyDeviceToHost));
  for (int m = 0; m < sys->n_mesh; ++m) {
    const double* M = rec.data() + (size_t)kMeshRec * m;
    double rmax = 0.0;
    for (int t = 0; t < sys->n_tri; ++t)
      if (sys->h_tri_mesh[t] == m)
        for (int k = 0; k < 3; ++k) {
          const double* v = sys->h_tri_body.data() + 9 * (size_t)t + 3 * k;
          rmax = std::max(rmax, std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]));
        }
    const double sp = std::sqrt(M[7] * M[7] + M[8] * M[8] + M[9] * M[9]) +
                      std::sqrt(M[10] * M[10] + M[11] * M[11] + M[12] * M[12]) * rmax;
    if (sp * sys->P.h * lag > 0.5 * sys->P.margin) {
      sys->err = "mesh " + std::to_string(m) + " moves more than margin/2 while a deferred contact set is in use";
      return DEM_ERR_VMAX;
    }
  }
  return DEM_OK;
}

// Capacity regrow after an abort: the parities of the aborted step are restored, the capacities
// that overflowed grow, the graphs are dropped, the status word is cleared.
static dem_status regrow(dem_system* sys, int up, int ep, int since, int kind, bool pending) {
  CK(cudaStreamSynchronize(sys->det_stream));
  if (std::getenv("DEM_DEBUG_LOG"))
    std::fprintf(stderr, "dem: regrow (kind %d, pending %d): need entries %lld inserts %lld width %lld det_abort %d\n",
                 kind, (int)pending, sys->h_ctl->need_entries, sys->h_ctl->need_inserts, sys->h_ctl->need_width,
                 sys->h_ctl->det_abort);
  sys->up = up;
  sys->ep = ep;
  sys->since_rebuild = since;
  sys->pending = false;
  sys->h_ctl->det_abort = 0;
  bool grew = false;  // (a distributed rank also re-runs when only another rank overflowed)
  if (sys->h_ctl->need_entries > sys->cap_entries) {
    long long need = sys->h_ctl->need_entries;
    TRY(alloc_rows(sys, need + need / 4 + 1024));
    grew = true;
  }
  if (sys->h_ctl->need_inserts > sys->cap_inserts) {
    long long need = sys->h_ctl->need_inserts;
    sys->cap_inserts = need + need / 4 + 1024;
    TRY(alloc_arr(sys, &sys->d_items, sys->cap_inserts));
    grew = true;
  }
  if (sys->h_ctl->need_width > sys->row_width) {
    sys->row_width = (int)std::min<long long>(sys->h_ctl->need_width + 8, 1 << 16);
    TRY(alloc_arr(sys, &sys->d_slots, (size_t)sys->ns_own * sys->row_width + 1));
    if (DEM_SLOT_KEYS) TRY(alloc_arr(sys, &sys->d_slot_key, (size_t)sys->ns_own * sys->row_width + 1));
    grew = true;
  }
  if (grew) sys->regrows++;
  sys->reruns++;
  free_graphs(sys);
  sys->h_ctl->abort = 0;
  sys->h_ctl->need_entries = 0;
  sys->h_ctl->need_inserts = 0;
  sys->h_ctl->need_width = 0;
  CK(cudaMemcpyAsync(sys->d_ctl, sys->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, sys->stream));
  return DEM_OK;
}

// A sphere centre left the bin region where it is tighter than the domain (Ctl::need_regrid):
// lay the grid out again around the spheres' current box (same edge; results do not depend on
// the bins), between step batches.
static dem_status regrid(dem_system* sys) {
  CK(cudaStreamSynchronize(sys->det_stream));  // a set detected ahead may still read the old bins
  unsigned long long* d_box = (unsigned long long*)dalloc(sys, 6 * sizeof(unsigned long long));
  if (!d_box) return DEM_ERR_OOM;
  const unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull};
  unsigned long long box[6];
  CK(cudaMemcpyAsync(d_box, init, sizeof init, cudaMemcpyHostToDevice, sys->stream));
  launch_bbox(sys->d_spos, (int)sys->ns, d_box, sys->stream);
  CK(cudaMemcpyAsync(box, d_box, sizeof box, cudaMemcpyDeviceToHost, sys->stream));
  CK(cudaStreamSynchronize(sys->stream));
  dfree(sys, d_box);
  auto val = [](unsigned long long k) {
    const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    double v;
    std::memcpy(&v, &b, sizeof v);
    return v;
  };
  double lo[3], hi[3];
  for (int d = 0; d < 3; ++d) {
    lo[d] = val(box[d]);
    hi[d] = val(box[3 + d]);
  }
  TRY(grid_layout(sys, sys->grid.cell, lo, hi, sys->ns, true));
  TRY(alloc_arr(sys, &sys->d_cell_count, sys->ncell));
  TRY(alloc_arr(sys, &sys->d_cell_start, sys->ncell + 1));
  TRY(alloc_arr(sys, &sys->d_scan_tmp, std::max(scan_tiles_needed(sys->ncell), scan_tiles_needed(sys->ns)) + 1));
  CK(cudaMemsetAsync(sys->d_cell_count, 0, sizeof(int) * sys->ncell, sys->stream));
  free_graphs(sys);
  sys->regrids++;
  sys->h_ctl->need_regrid = 0;
  CK(cudaMemcpyAsync(sys->d_ctl, sys->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, sys->stream));
  CK(cudaStreamSynchronize(sys->stream));
  return DEM_OK;
}

// steps enqueued per status check (the status word is read, and a re-grid done, between batches)
static constexpr int64_t kStepBatch = 2048;

extern "C" dem_status dem_step(dem_system* sys, int64_t n_steps) {
  if (!sys || n_steps < 0) return DEM_ERR_INVALID_ARG;
  if (sys->peer && sys->P.transport == DEM_TRANSPORT_PEER && !sys->peer_linked) {
    sys->err = "PEER transport: call dem_peer_export / dem_peer_import after dem_set_state";
    return DEM_ERR_INVALID_ARG;
  }
  if (sys->h_ctl->err_code) return (dem_status)sys->h_ctl->err_code;
  TRY(check_mesh_motion(sys));
  int64_t remaining = n_steps;
  int guard = 0;
  struct Sched {
    int up, ep, since;
    bool pending;
  };
  std::vector<Sched> sched;
  while (remaining > 0) {
    const int64_t done_before = sys->h_ctl->step;
    sched.clear();
    const int64_t batch = std::min<int64_t>(remaining, kStepBatch);
    if (sys->profiling) TRY(ensure_events(sys, batch));
    for (int64_t k = 0; k < batch; ++k) {
      const int kind = step_kind(sys);
      sched.push_back(Sched{sys->up, sys->ep, sys->since_rebuild, sys->pending});
      if (sys->profiling) {
        // stage timing: every part in line on the system stream (same results); a set still being
        // detected ahead on det_stream (launched before profiling was turned on) is joined first
        if (kind == K_ADOPT) CK(cudaStreamWaitEvent(sys->stream, sys->ev_det, 0));
        enqueue_step(sys, kind, sys->stream, &sys->ev[(size_t)k * (kStages + 1)]);
      } else if (kind == K_AHEAD) {
        // the next window's detection forks off after this step's poses and runs on det_stream
        // "in the shadow" of the force steps; the adopting step joins it
        cudaGraphExec_t gp, gd, gf;
        TRY(step_graph(sys, kind, PART_POSE, &gp));
        TRY(step_graph(sys, kind, PART_DET, &gd));
        TRY(step_graph(sys, kind, PART_FORCE, &gf));
        CK(cudaGraphLaunch(gp, sys->stream));
        CK(cudaEventRecord(sys->ev_fork, sys->stream));
        CK(cudaStreamWaitEvent(sys->det_stream, sys->ev_fork, 0));
        CK(cudaGraphLaunch(gd, sys->det_stream));
        if (sys->fault_ahead > 0) {
          --sys->fault_ahead;
          CK(cudaMemcpyAsync(&sys->d_ctl->det_abort, &kOne, sizeof(int), cudaMemcpyHostToDevice, sys->det_stream));
        }
        CK(cudaEventRecord(sys->ev_det, sys->det_stream));
        if (sys->debug_serial_det) CK(cudaStreamWaitEvent(sys->stream, sys->ev_det, 0));
        CK(cudaGraphLaunch(gf, sys->stream));
      } else {
        if (kind == K_ADOPT) CK(cudaStreamWaitEvent(sys->stream, sys->ev_det, 0));
        cudaGraphExec_t g;
        TRY(step_graph(sys, kind, PART_ALL, &g));
        CK(cudaGraphLaunch(g, sys->stream));
      }
      advance_parities(sys, kind);
    }
    TRY(read_ctl(sys));
    const int64_t done = sys->h_ctl->step - done_before;
    if (sys->profiling) {
      for (int64_t k = 0; k < done; ++k)
        for (int st = 0; st < kStages; ++st) {
          float ms = 0;
          cudaEventElapsedTime(&ms, sys->ev[(size_t)k * (kStages + 1) + st],
                               sys->ev[(size_t)k * (kStages + 1) + st + 1]);
          sys->stage_ms[st] += ms;
        }
      sys->prof_steps += done;
    }
    sys->steps_done = sys->h_ctl->step;
    if (sys->h_ctl->err_code) return device_error(sys);
    remaining -= done;
    if (!sys->h_ctl->abort) {
      if (done == 0) {  // (never: every enqueued step either completes or aborts)
        sys->err = "dem_step: a batch of steps completed none without an abort";
        return DEM_ERR_CUDA;
      }
      if (sys->h_ctl->need_regrid) TRY(regrid(sys));
      continue;
    }
    if (sys->dist && !sys->comm) {  // a local regrow would desynchronise the ranks' halo exchanges
      sys->err = "capacity overflow on a distributed system without an NCCL communicator (raise params.entries_per_sphere)";
      return DEM_ERR_CAPACITY;
    }
    // capacity abort in step `done` (a FULL step, or an ADOPT step whose set detected ahead
    // overflowed): the state was carried forward through the aborted steps (sp is already
    // right); the latest valid u_t and entry set are those that step read.  Regrow and re-run
    // from there — an aborted adoption as a FULL rebuild at that step, which gives the same
    // trajectory (every contact with delta > 0 is in both sets).  A distributed
    // rank gets here together with every other rank: the abort word is all-reduced before the
    // force kernel of each rebuild step, so all ranks carried the same steps forward.
    if (++guard > 8) {
      sys->err = "capacity regrow did not converge";
      return DEM_ERR_CAPACITY;
    }
    const Sched& at = sched[(size_t)done];
    TRY(regrow(sys, at.up, at.ep, at.since, sched[(size_t)done].since == 0 ? (at.pending ? K_ADOPT : K_FULL) : -1,
               at.pending));
  }
  if (sys->launched > 0) TRY(repartition_by_entries(sys));
  return DEM_OK;
}

extern "C" dem_status dem_synchronize(dem_system* sys) {
  if (!sys) return DEM_ERR_INVALID_ARG;
  CK(cudaStreamSynchronize(sys->det_stream));
  TRY(read_ctl(sys));
  if (sys->h_ctl->err_code) return device_error(sys);
  return DEM_OK;
}

extern "C" dem_status dem_get_state(dem_system* sys, int64_t cap, int64_t* n, int64_t* gid, int32_t* tid,
                                    double* pos, double* quat, double* vel, double* omega, int32_t on_device) {
  if (!sys) return DEM_ERR_INVALID_ARG;
  const int64_t NO = sys->n_own;  // owned clumps (all of them on a single system)
  if (n) *n = NO;
  if (cap < NO) return (pos || quat || vel || omega || gid || tid) ? DEM_ERR_INVALID_ARG : DEM_OK;
  CK(cudaStreamSynchronize(sys->stream));
  cudaStream_t s = sys->stream;
  // device gather from the storage order into caller-order rows, then one copy per array
  double* dst[4] = {pos, quat, vel, omega};
  const int width[4] = {3, 4, 3, 3};
  double* dev[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t off = 0;
  for (int k = 0; k < 4; ++k) {
    if (dst[k]) dev[k] = on_device ? dst[k] : sys->d_io + off;
    off += (size_t)width[k] * NO;
  }
  const StepArgs a = make_args(sys, K_CHECK);
  if (NO) launch_state_out(a.cur, sys->d_outpos, (int)NO, dev[0], dev[1], dev[2], dev[3], s);
  if (!on_device)
    for (int k = 0; k < 4; ++k)
      if (dst[k] && NO) CK(cudaMemcpyAsync(dst[k], dev[k], sizeof(double) * width[k] * NO, cudaMemcpyDeviceToHost, s));
  // gids and template ids from the host copies
  std::vector<long long> go;
  std::vector<int> to;
  const long long* gsrc = sys->h_in_gid.data();
  const int* tsrc = sys->h_in_tid.data();
  if (sys->dist && (gid || tid)) {
    go.resize(NO);
    to.resize(NO);
    for (int64_t i = 0; i < NO; ++i) {
      go[sys->h_outpos[i]] = sys->h_gid[i];
      to[sys->h_outpos[i]] = sys->h_tid[i];
    }
    gsrc = go.data();
    tsrc = to.data();
  }
  if (gid && NO) {
    if (on_device)
      CK(cudaMemcpyAsync(gid, gsrc, sizeof(long long) * NO, cudaMemcpyHostToDevice, s));
    else
      std::memcpy(gid, gsrc, sizeof(long long) * NO);
  }
  if (tid && NO) {
    if (on_device)
      CK(cudaMemcpyAsync(tid, tsrc, sizeof(int) * NO, cudaMemcpyHostToDevice, s));
    else
      std::memcpy(tid, tsrc, sizeof(int) * NO);
  }
  CK(cudaStreamSynchronize(s));
  return DEM_OK;
}

extern "C" dem_status dem_partition_plan(int64_t n, const double* pos, double slab_lo, double slab_hi, double halo,
                                         int32_t has_left, int32_t has_right, int8_t* role, int8_t* send) {
  if (n < 0 || (n && (!pos || !role || !send)) || !(slab_hi > slab_lo) || !(halo >= 0)) return DEM_ERR_INVALID_ARG;
  for (int64_t c = 0; c < n; ++c) {
    const double x = pos[3 * c];
    int8_t r = 0, f = 0;
    if (x >= slab_lo && x < slab_hi) {
      r = 1;
      if (has_left && x < slab_lo + halo) f |= 1;
      if (has_right && x >= slab_hi - halo) f |= 2;
    } else if (has_left && x < slab_lo && x >= slab_lo - halo) {
      r = 2;
    } else if (has_right && x >= slab_hi && x < slab_hi + halo) {
      r = 3;
    }
    role[c] = r;
    send[c] = f;
  }
  return DEM_OK;
}

extern "C" dem_status dem_step_group(dem_system* const* systems, int32_t n, int64_t n_steps) {
  if (!systems || n < 1 || n_steps < 0) return DEM_ERR_INVALID_ARG;
  cudaStream_t s = systems[0]->stream;
  const int tr = systems[0]->P.transport;
  for (int r = 0; r < n; ++r) {
    dem_system* sys = systems[r];
    if (!sys || sys->stream != s ||
        (n > 1 && (!sys->dist || sys->P.transport != tr ||
                   (tr != DEM_TRANSPORT_LOOPBACK && tr != DEM_TRANSPORT_LOOPBACK_PEER) || sys->P.rank != r ||
                   sys->P.n_ranks != n)))
      return DEM_ERR_INVALID_ARG;
    if (sys->h_ctl->err_code) return (dem_status)sys->h_ctl->err_code;
  }
  const bool peer = n > 1 && tr == DEM_TRANSPORT_LOOPBACK_PEER;
  if (peer && !systems[0]->peer_linked) {
    TRY(peer_link_local(systems, n));
    for (int r = 0; r < n; ++r) systems[r]->peer_linked = true;
  }
  if (n > kMaxGroup) return DEM_ERR_INVALID_ARG;
  AbortWords aw{};
  aw.n = n;
  for (int r = 0; r < n; ++r) aw.p[r] = &systems[r]->d_ctl->abort;
  struct Sched {
    int up, ep, since;
    bool pending;
  };
  std::vector<std::vector<Sched>> sched(n);
  int64_t remaining = n_steps;
  int guard = 0;
  while (remaining > 0) {
    const int64_t done_before = systems[0]->h_ctl->step;
    for (auto& v : sched) v.clear();
    for (int64_t k = 0; k < remaining; ++k) {
      // every rank's poses and detection, then one abort vote, then every rank's force kernel: a
      // capacity overflow on any rank stops the step on all of them (coordinated regrow below)
      for (int r = 0; r < n; ++r) {
        dem_system* sys = systems[r];
        sched[r].push_back(Sched{sys->up, sys->ep, sys->since_rebuild, sys->pending});
        enqueue_pose(sys, step_kind(sys), s, nullptr);
        enqueue_detect(sys, step_kind(sys), s, nullptr);
      }
      launch_abort_or(aw, s);
      for (int r = 0; r < n; ++r) {
        dem_system* sys = systems[r];
        enqueue_force(sys, step_kind(sys), s, nullptr, /*exchange=*/false);
      }
      if (peer) {  // the force kernels stored the ghost states into the neighbours already
        for (int r = 0; r < n; ++r) advance_parities(systems[r], step_kind(systems[r]));
        continue;
      }
      // ghost halo: rank r's left-side ghosts are rank r-1's right-side sends, and vice versa
      for (int r = 0; r < n; ++r) {
        dem_system* sys = systems[r];
        if (r > 0 && sys->n_recv[0]) {
          if (systems[r - 1]->n_send[1] != sys->n_recv[0]) return DEM_ERR_INVALID_ARG;
          CK(cudaMemcpyAsync(sys->d_recvbuf[0], systems[r - 1]->d_sendbuf[1], sizeof(double) * kKin13 * sys->n_recv[0],
                             cudaMemcpyDeviceToDevice, s));
        }
        if (r < n - 1 && sys->n_recv[1]) {
          if (systems[r + 1]->n_send[0] != sys->n_recv[1]) return DEM_ERR_INVALID_ARG;
          CK(cudaMemcpyAsync(sys->d_recvbuf[1], systems[r + 1]->d_sendbuf[0], sizeof(double) * kKin13 * sys->n_recv[1],
                             cudaMemcpyDeviceToDevice, s));
        }
      }
      for (int r = 0; r < n; ++r) {
        dem_system* sys = systems[r];
        const int kind = step_kind(sys);
        StepArgs a = make_args(sys, kind);
        enqueue_unpack(sys, a, s);
        advance_parities(sys, kind);
      }
    }
    bool aborted = false;
    int64_t done = 0;
    for (int r = 0; r < n; ++r) {
      dem_system* sys = systems[r];
      TRY(read_ctl(sys));
      sys->steps_done = sys->h_ctl->step;
      if (sys->h_ctl->err_code) return device_error(sys);
      aborted |= sys->h_ctl->abort != 0;
      done = sys->h_ctl->step - done_before;  // equal on every rank (the abort vote)
    }
    remaining -= done;
    if (!aborted) break;
    if (++guard > 8) {
      systems[0]->err = "capacity regrow did not converge";
      return DEM_ERR_CAPACITY;
    }
    // every rank stopped at step `done`: each regrows what overflowed on it and all re-run from there
    for (int r = 0; r < n; ++r) {
      const Sched& at = sched[r][(size_t)done];
      TRY(regrow(systems[r], at.up, at.ep, at.since, at.since == 0 ? (at.pending ? K_ADOPT : K_FULL) : -1, at.pending));
    }
  }
  return DEM_OK;
}

extern "C" dem_status dem_get_contacts(dem_system* sys, int64_t cap, int64_t* n, int64_t* key_a, int64_t* key_b,
                                       double* force_on_b, double* point, double* normal, double* u_t,
                                       double* delta) {
  if (!sys || !n) return DEM_ERR_INVALID_ARG;
  if ((force_on_b || point || normal || delta) && !sys->P.record_contacts) {
    sys->err = "force/point/normal/delta need params.record_contacts = 1";
    return DEM_ERR_INVALID_ARG;
  }
  CK(cudaStreamSynchronize(sys->stream));
  if (sys->launched == 0 || sys->ns == 0) {
    *n = 0;
    return DEM_OK;
  }
  const RowBuf& R = sys->rows[sys->ep];  // the last step's set; its u_t is rows[up].ut
  const int64_t ns = sys->ns;
  std::vector<int> rp(ns + 1);
  CK(cudaMemcpy(rp.data(), R.row_ptr, sizeof(int) * (ns + 1), cudaMemcpyDeviceToHost));
  const int64_t m = rp[ns];
  std::vector<long long> keys(m);
  if (m) CK(cudaMemcpy(keys.data(), R.key, sizeof(long long) * m, cudaMemcpyDeviceToHost));
  // canonical entries: own key < partner key
  std::vector<std::pair<int64_t, int64_t>> sel;  // (own sphere, entry)
  for (int64_t s = 0; s < ns; ++s)
    for (int e = rp[s]; e < rp[s + 1]; ++e)
      if (sys->h_s_key[s] < keys[e]) sel.emplace_back(s, e);
  std::sort(sel.begin(), sel.end(), [&](const auto& x, const auto& y) {
    long long ax = sys->h_s_key[x.first], ay = sys->h_s_key[y.first];
    if (ax != ay) return ax < ay;
    return keys[x.second] < keys[y.second];
  });
  *n = (int64_t)sel.size();
  if (cap == 0) return DEM_OK;
  if (cap < (int64_t)sel.size()) return DEM_ERR_INVALID_ARG;
  auto fetch3 = [&](const double* dev, double* out, int stride = 3) -> dem_status {
    if (!out) return DEM_OK;
    std::vector<double> buf((size_t)stride * m);
    if (m) CK(cudaMemcpy(buf.data(), dev, sizeof(double) * stride * m, cudaMemcpyDeviceToHost));
    for (size_t k = 0; k < sel.size(); ++k)
      for (int d = 0; d < 3; ++d) out[3 * k + d] = buf[stride * sel[k].second + d];
    return DEM_OK;
  };
  for (size_t k = 0; k < sel.size(); ++k) {
    if (key_a) key_a[k] = sys->h_s_key[sel[k].first];
    if (key_b) key_b[k] = keys[sel[k].second];
  }
  TRY(fetch3(sys->rows[sys->up].ut, u_t, kUt));
  TRY(fetch3(sys->rec.F, force_on_b));
  TRY(fetch3(sys->rec.p, point));
  TRY(fetch3(sys->rec.n, normal));
  if (delta) {
    std::vector<double> buf(m);
    if (m) CK(cudaMemcpy(buf.data(), sys->rec.delta, sizeof(double) * m, cudaMemcpyDeviceToHost));
    for (size_t k = 0; k < sel.size(); ++k) delta[k] = buf[sel[k].second];
  }
  return DEM_OK;
}

extern "C" dem_status dem_get_stats(dem_system* sys, dem_stats* out) {
  if (!sys || !out) return DEM_ERR_INVALID_ARG;
  std::memset(out, 0, sizeof *out);
  out->steps = sys->steps_done;
  out->n_clumps = sys->n;
  out->n_spheres = sys->ns;
  out->n_owned_clumps = sys->n_own;
  out->n_owned_spheres = sys->ns_own;
  out->n_ghost_clumps = sys->n - sys->n_own;
  out->n_cells = sys->ncell;
  out->cell_size = sys->grid.cell;
  out->regrows = sys->regrows;
  out->kernel_launches_per_step =
      kLaunchesPerStep + (sys->dist ? (sys->peer ? 2 : 4) : 0) + (sys->n_mesh ? 3 : 0);
  out->state_fast_resets = sys->fast_resets;
  out->bin_regrids = sys->regrids;
  out->reruns = sys->reruns;
  out->migrated_clumps = sys->migrated_clumps;
  out->migration_bytes = sys->migration_bytes;
  out->ghost_exchange_bytes = sys->ghost_bytes;
  if (sys->launched > 0 && sys->ns > 0) {
    const RowBuf& R = sys->rows[sys->ep];
    int tot = 0, ins = 0;
    CK(cudaMemcpyAsync(&tot, R.row_ptr + sys->ns, sizeof(int), cudaMemcpyDeviceToHost, sys->stream));
    CK(cudaMemcpyAsync(&ins, sys->d_cell_start + sys->ncell, sizeof(int), cudaMemcpyDeviceToHost, sys->stream));
    CK(cudaMemsetAsync(sys->d_counter, 0, sizeof(unsigned long long), sys->stream));
    // canonical contacts held here: entries whose own key is the smaller (walls included)
    launch_count_canonical(Rows{R.row_ptr, R.ent, R.key, R.ut}, sys->d_s_key, (int)sys->ns_own, sys->d_counter, sys->stream);
    unsigned long long canon = 0;
    CK(cudaMemcpyAsync(&canon, sys->d_counter, sizeof(canon), cudaMemcpyDeviceToHost, sys->stream));
    CK(cudaStreamSynchronize(sys->stream));
    out->n_entries = tot;
    out->n_inserts = ins;
    out->n_contacts = (int64_t)canon;
  }
  return DEM_OK;
}

extern "C" dem_status dem_set_profiling(dem_system* sys, int32_t enable) {
  if (!sys) return DEM_ERR_INVALID_ARG;
  sys->profiling = enable != 0;
  for (int s = 0; s < kStages; ++s) sys->stage_ms[s] = 0;
  sys->prof_steps = 0;
  return DEM_OK;
}

extern "C" dem_status dem_get_stage_times(dem_system* sys, int32_t n_stages, double* ms) {
  if (!sys || !ms) return DEM_ERR_INVALID_ARG;
  for (int s = 0; s < n_stages && s < kStages; ++s) ms[s] = sys->prof_steps ? sys->stage_ms[s] / sys->prof_steps : 0.0;
  return DEM_OK;
}

// ------------------------------------------------------------------ migration
// Largest owned-COM displacement since dem_set_state on this system (squared, device reduction).
static dem_status local_max_drift2(dem_system* sys, double* out) {
  CK(cudaMemsetAsync(sys->d_counter, 0, sizeof(unsigned long long), sys->stream));
  StepArgs a = make_args(sys, K_CHECK);
  launch_max_drift(a.cur, sys->d_xref, (int)sys->n_own, sys->d_counter, sys->stream);
  return DEM_OK;
}

// ------------------------------------------------------------------ neighbour exchange
// Records moved between neighbouring ranks, as doubles: a clump [gid bits, tid, pos 3, quat 4,
// vel 3, omega 3]; a contact [key_a bits, key_b bits, u_t 3 (oriented a -> b)].
static constexpr int kMigClump = 15, kMigContact = 5;

struct ClumpSet {
  std::vector<int64_t> gid;
  std::vector<int32_t> tid;
  std::vector<double> pos, quat, vel, om;
  int64_t size() const { return (int64_t)gid.size(); }
  void add(int64_t g, int32_t t, const double* p, const double* q, const double* v, const double* w) {
    gid.push_back(g);
    tid.push_back(t);
    pos.insert(pos.end(), p, p + 3);
    quat.insert(quat.end(), q, q + 4);
    vel.insert(vel.end(), v, v + 3);
    om.insert(om.end(), w, w + 3);
  }
  void add(const ClumpSet& s, int64_t c) {
    add(s.gid[c], s.tid[c], &s.pos[3 * c], &s.quat[4 * c], &s.vel[3 * c], &s.om[3 * c]);
  }
  void put(std::vector<double>& o, int64_t c) const {
    double r[kMigClump];
    std::memcpy(&r[0], &gid[c], 8);
    r[1] = (double)tid[c];
    for (int d = 0; d < 3; ++d) r[2 + d] = pos[3 * c + d];
    for (int d = 0; d < 4; ++d) r[5 + d] = quat[4 * c + d];
    for (int d = 0; d < 3; ++d) r[9 + d] = vel[3 * c + d];
    for (int d = 0; d < 3; ++d) r[12 + d] = om[3 * c + d];
    o.insert(o.end(), r, r + kMigClump);
  }
  void get(const double* r) {
    int64_t g;
    std::memcpy(&g, &r[0], 8);
    add(g, (int32_t)r[1], r + 2, r + 5, r + 9, r + 12);
  }
};

struct ContactSet {
  std::vector<int64_t> ka, kb;
  std::vector<double> ut;
  int64_t size() const { return (int64_t)ka.size(); }
  void put(std::vector<double>& o, int64_t k) const {
    double r[kMigContact];
    std::memcpy(&r[0], &ka[k], 8);
    std::memcpy(&r[1], &kb[k], 8);
    for (int d = 0; d < 3; ++d) r[2 + d] = ut[3 * k + d];
    o.insert(o.end(), r, r + kMigContact);
  }
  void get(const double* r) {
    int64_t a, b;
    std::memcpy(&a, &r[0], 8);
    std::memcpy(&b, &r[1], 8);
    ka.push_back(a);
    kb.push_back(b);
    ut.insert(ut.end(), r + 2, r + 5);
  }
};

// one rank's payloads to / from its left [0] and right [1] neighbours
struct NbrMsg {
  std::vector<double> out[2], in[2];
};

// NCCL: grouped ncclSend/ncclRecv with rank - 1 and rank + 1, counts first, then payloads
static dem_status exchange_nccl(dem_system* sys, NbrMsg& m) {
  const int r = sys->P.rank, P = sys->P.n_ranks;
  cudaStream_t s = sys->stream;
  const bool nb[2] = {r > 0, r < P - 1};
  const int peer[2] = {r - 1, r + 1};
  int64_t* d_cnt = (int64_t*)dalloc(sys, sizeof(int64_t) * 4);
  if (!d_cnt) return DEM_ERR_OOM;
  const int64_t cnt_out[2] = {(int64_t)m.out[0].size(), (int64_t)m.out[1].size()};
  int64_t cnt_in[2] = {0, 0};
  CK(cudaMemcpyAsync(d_cnt, cnt_out, sizeof(cnt_out), cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(d_cnt + 2, 0, 2 * sizeof(int64_t), s));
  ncclGroupStart();
  for (int side = 0; side < 2; ++side)
    if (nb[side]) {
      ncclSend(d_cnt + side, 1, ncclInt64, peer[side], sys->comm, s);
      ncclRecv(d_cnt + 2 + side, 1, ncclInt64, peer[side], sys->comm, s);
    }
  if (ncclGroupEnd() != ncclSuccess) return DEM_ERR_NCCL;
  CK(cudaMemcpyAsync(cnt_in, d_cnt + 2, sizeof(cnt_in), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  dfree(sys, d_cnt);
  const size_t tot = (size_t)(cnt_out[0] + cnt_out[1] + cnt_in[0] + cnt_in[1]);
  double* d_buf = (double*)dalloc(sys, sizeof(double) * (tot + 1));
  if (!d_buf) return DEM_ERR_OOM;
  double* so[2] = {d_buf, d_buf + cnt_out[0]};
  double* si[2] = {so[1] + cnt_out[1], so[1] + cnt_out[1] + cnt_in[0]};
  for (int side = 0; side < 2; ++side)
    if (cnt_out[side])
      CK(cudaMemcpyAsync(so[side], m.out[side].data(), sizeof(double) * cnt_out[side], cudaMemcpyHostToDevice, s));
  ncclGroupStart();
  for (int side = 0; side < 2; ++side)
    if (nb[side]) {
      if (cnt_out[side]) ncclSend(so[side], (size_t)cnt_out[side], ncclDouble, peer[side], sys->comm, s);
      if (cnt_in[side]) ncclRecv(si[side], (size_t)cnt_in[side], ncclDouble, peer[side], sys->comm, s);
    }
  if (ncclGroupEnd() != ncclSuccess) return DEM_ERR_NCCL;
  for (int side = 0; side < 2; ++side) {
    m.in[side].assign((size_t)cnt_in[side], 0.0);
    if (cnt_in[side])
      CK(cudaMemcpyAsync(m.in[side].data(), si[side], sizeof(double) * cnt_in[side], cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  dfree(sys, d_buf);
  return DEM_OK;
}

// the exchange for the ranks held by this process: one NCCL rank, or a whole loopback group
// (ranks 0..n-1 in order, payloads handed over in memory)
static dem_status exchange(dem_system* const* sys, int n, std::vector<NbrMsg>& m) {
  if (n == 1 && sys[0]->comm) return exchange_nccl(sys[0], m[0]);
  if (n != sys[0]->P.n_ranks) {
    sys[0]->err = "neighbour exchange: needs an NCCL communicator (dem_params.nccl_id) or the whole loopback group";
    return DEM_ERR_INVALID_ARG;
  }
  for (int r = 0; r < n; ++r) {
    m[r].in[0] = r > 0 ? m[r - 1].out[1] : std::vector<double>();
    m[r].in[1] = r < n - 1 ? m[r + 1].out[0] : std::vector<double>();
  }
  return DEM_OK;
}

// Every rank's owned clumps -> its held set: the owned clumps plus the clumps its neighbours own
// within `halo` of the shared faces (sent by their owners: the same partition test on the same
// bits on both sides), laid out by dem_set_state.  Collective over the decomposition.
static dem_status complete_ghosts(dem_system* const* sys, int n, const std::vector<ClumpSet>& owned) {
  std::vector<NbrMsg> m(n);
  for (int r = 0; r < n; ++r) {
    const dem_params& P = sys[r]->P;
    const ClumpSet& O = owned[r];
    std::vector<int8_t> role(O.size()), sendf(O.size());
    TRY(dem_partition_plan(O.size(), O.pos.data(), P.slab_lo, P.slab_hi, P.halo, P.rank > 0,
                           P.rank < P.n_ranks - 1, role.data(), sendf.data()));
    for (int64_t c = 0; c < O.size(); ++c) {
      if (role[c] != 1) {
        sys[r]->err = "clump gid " + std::to_string(O.gid[c]) + " handed to a rank whose slab does not hold its COM";
        return DEM_ERR_INVALID_ARG;
      }
      for (int side = 0; side < 2; ++side)
        if (sendf[c] >> side & 1) O.put(m[r].out[side], c);
    }
    sys[r]->ghost_bytes = (int64_t)(m[r].out[0].size() + m[r].out[1].size()) * 8;
  }
  TRY(exchange(sys, n, m));
  for (int r = 0; r < n; ++r) {
    ClumpSet H = owned[r];
    for (int side = 0; side < 2; ++side)
      for (size_t o = 0; o < m[r].in[side].size(); o += kMigClump) H.get(m[r].in[side].data() + o);
    TRY(dem_set_state(sys[r], H.size(), H.gid.data(), H.tid.data(), H.pos.data(), H.quat.data(), H.vel.data(),
                      H.om.data(), 0));
  }
  return DEM_OK;
}

// the clumps of a rank-local input whose COM lies in the rank's slab
static ClumpSet owned_of_input(const dem_system* sys, int64_t n, const int64_t* gid, const int32_t* tid,
                              const double* pos, const double* quat, const double* vel, const double* om) {
  ClumpSet O;
  for (int64_t c = 0; c < n; ++c) {
    const double x = pos[3 * c];
    if (x >= sys->P.slab_lo && x < sys->P.slab_hi) O.add(gid[c], tid[c], pos + 3 * c, quat + 4 * c, vel + 3 * c, om + 3 * c);
  }
  return O;
}

extern "C" dem_status dem_set_state_local(dem_system* sys, int64_t n, const int64_t* gid, const int32_t* tid,
                                          const double* pos, const double* quat, const double* vel,
                                          const double* omega) {
  if (!sys || n < 0 || (n > 0 && (!gid || !tid || !pos || !quat || !vel || !omega))) return DEM_ERR_INVALID_ARG;
  if (!sys->dist) return dem_set_state(sys, n, gid, tid, pos, quat, vel, omega, 0);
  std::vector<ClumpSet> owned{owned_of_input(sys, n, gid, tid, pos, quat, vel, omega)};
  dem_system* one[1] = {sys};
  return complete_ghosts(one, 1, owned);
}

extern "C" dem_status dem_set_state_local_group(dem_system* const* systems, int32_t n, const int64_t* n_in,
                                                const int64_t* const* gid, const int32_t* const* tid,
                                                const double* const* pos, const double* const* quat,
                                                const double* const* vel, const double* const* omega) {
  if (!systems || n < 1 || !n_in || !gid || !tid || !pos || !quat || !vel || !omega) return DEM_ERR_INVALID_ARG;
  std::vector<ClumpSet> owned;
  for (int r = 0; r < n; ++r) {
    dem_system* sys = systems[r];
    if (!sys || !sys->dist || sys->P.rank != r || sys->P.n_ranks != n || n_in[r] < 0) return DEM_ERR_INVALID_ARG;
    owned.push_back(owned_of_input(sys, n_in[r], gid[r], tid[r], pos[r], quat[r], vel[r], omega[r]));
  }
  return complete_ghosts(systems, n, owned);
}

extern "C" dem_status dem_migration_plan(int64_t n, const int64_t* gid, const double* pos, const int8_t* role,
                                         double slab_lo, double slab_hi, int32_t has_left, int32_t has_right,
                                         int8_t* dest, int64_t n_entries, const int64_t* own_key, int8_t* route) {
  if (n < 0 || n_entries < 0 || (n && (!gid || !pos || !role || !dest)) || (n_entries && (!own_key || !route)) ||
      !(slab_hi > slab_lo))
    return DEM_ERR_INVALID_ARG;
  std::unordered_map<int64_t, int8_t> of;
  of.reserve((size_t)n * 2);
  for (int64_t c = 0; c < n; ++c) {
    const double x = pos[3 * c];
    int8_t d = 0;
    if (role[c] == 1) {
      d = (has_left && x < slab_lo) ? -1 : (has_right && x >= slab_hi) ? 1 : 0;
    } else if (role[c] == 2) {
      d = x >= slab_lo ? 0 : -1;  // a left neighbour's clump: now ours, or still the neighbour's
    } else if (role[c] == 3) {
      d = x < slab_hi ? 0 : 1;
    } else {
      return DEM_ERR_INVALID_ARG;
    }
    dest[c] = d;
    of[gid[c]] = d;
  }
  // a directed row entry belongs to the owner of its own sphere: it goes where that clump goes
  for (int64_t k = 0; k < n_entries; ++k) {
    auto it = of.find(own_key[k] / kKeyStride);
    if (own_key[k] < 0 || it == of.end()) return DEM_ERR_INVALID_ARG;
    route[k] = it->second;
  }
  return DEM_OK;
}

// the directed row entries of the owned spheres in the last step's set: (own key, partner key,
// u_t oriented own -> partner) — the history each rank keeps for its own spheres
static dem_status get_directed(dem_system* sys, ContactSet& K) {
  if (sys->launched == 0 || sys->ns_own == 0) return DEM_OK;
  CK(cudaStreamSynchronize(sys->stream));
  const RowBuf& R = sys->rows[sys->ep];
  std::vector<int> rp(sys->ns_own + 1);
  CK(cudaMemcpy(rp.data(), R.row_ptr, sizeof(int) * (sys->ns_own + 1), cudaMemcpyDeviceToHost));
  const int64_t m = rp[sys->ns_own];
  std::vector<long long> keys(m);
  std::vector<double> ut((size_t)kUt * m);
  if (m) {
    CK(cudaMemcpy(keys.data(), R.key, sizeof(long long) * m, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ut.data(), sys->rows[sys->up].ut, sizeof(double) * kUt * m, cudaMemcpyDeviceToHost));
  }
  for (int64_t s = 0; s < sys->ns_own; ++s)
    for (int e = rp[s]; e < rp[s + 1]; ++e) {
      K.ka.push_back(sys->h_s_key[s]);
      K.kb.push_back(keys[e]);
      K.ut.insert(K.ut.end(), &ut[(size_t)kUt * e], &ut[(size_t)kUt * e] + 3);
    }
  return DEM_OK;
}

// install directed entries as the history of the owned spheres they name (others are ignored)
static dem_status import_directed(dem_system* sys, const ContactSet& K) {
  std::unordered_map<long long, int> idx;
  idx.reserve((size_t)sys->ns_own * 2);
  for (int64_t s = 0; s < sys->ns_own; ++s) idx[sys->h_s_key[s]] = (int)s;
  std::vector<std::vector<HistEntry>> per(sys->ns);
  for (int64_t k = 0; k < K.size(); ++k) {
    auto it = idx.find(K.ka[k]);
    if (it != idx.end()) per[it->second].push_back(HistEntry{K.kb[k], {K.ut[3 * k], K.ut[3 * k + 1], K.ut[3 * k + 2]}});
  }
  return install_history(sys, per);
}

// Neighbour-only migration of the ranks held by this process: each rank sends the
// owned clumps whose COM left its slab, with the directed row entries of their spheres (partner
// key + u_t: the tangential history each sphere's owner keeps), to the neighbour that now owns
// them (counts, then payloads); the new owned sets then exchange their ghost bands
// (complete_ghosts) and every rank re-lays out only its own clumps and re-imports the entries of
// its spheres.  Bytes moved scale with the crossings (plus the ghost band), not with the system.
static dem_status migrate_ranks(dem_system* const* ranks, int n) {
  std::vector<NbrMsg> m(n);
  std::vector<ClumpSet> keep(n);
  std::vector<ContactSet> kc(n);
  for (int r = 0; r < n; ++r) {
    dem_system* sys = ranks[r];
    TRY(dem_synchronize(sys));
    int64_t no = 0;
    TRY(dem_get_state(sys, 0, &no, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0));
    ClumpSet O;
    O.gid.resize(no);
    O.tid.resize(no);
    O.pos.resize(3 * no);
    O.quat.resize(4 * no);
    O.vel.resize(3 * no);
    O.om.resize(3 * no);
    TRY(dem_get_state(sys, no, &no, O.gid.data(), O.tid.data(), O.pos.data(), O.quat.data(), O.vel.data(),
                      O.om.data(), 0));
    // held clumps: the owned ones, then the ghosts (storage order) with their current COM x
    const int64_t ng = sys->n - sys->n_own;
    std::vector<int64_t> hg(O.gid);
    std::vector<double> hp(O.pos);
    std::vector<int8_t> role(no, 1);
    if (ng) {
      std::vector<double> gx(ng);
      CK(cudaMemcpy(gx.data(), sys->d_state[sys->sp] + sys->n_own, sizeof(double) * ng, cudaMemcpyDeviceToHost));
      std::vector<int8_t> grole(ng, 0);
      for (int side = 0; side < 2; ++side)
        for (int i : sys->h_recv_list[side]) grole[i - sys->n_own] = (int8_t)(2 + side);
      for (int64_t k = 0; k < ng; ++k) {
        hg.push_back(sys->h_gid[sys->n_own + k]);
        const double p3[3] = {gx[k], 0.0, 0.0};
        hp.insert(hp.end(), p3, p3 + 3);
        role.push_back(grole[k]);
      }
    }
    ContactSet K;  // the directed row entries of the owned spheres
    TRY(get_directed(sys, K));
    const int64_t nk = K.size();
    std::vector<int8_t> dest(hg.size()), route(nk);
    const dem_params& P = sys->P;
    if (dem_migration_plan((int64_t)hg.size(), hg.data(), hp.data(), role.data(), P.slab_lo, P.slab_hi, P.rank > 0,
                           P.rank < P.n_ranks - 1, dest.data(), nk, K.ka.data(), route.data()) != DEM_OK) {
      sys->err = "migration plan: a row entry names a sphere that is not owned here";
      return DEM_ERR_INVALID_ARG;
    }
    std::vector<double> cl[2], co[2];
    int64_t ncl[2] = {0, 0}, nco[2] = {0, 0};
    for (int64_t c = 0; c < no; ++c) {
      if (dest[c] == 0) {
        keep[r].add(O, c);
      } else {
        const int side = dest[c] < 0 ? 0 : 1;
        O.put(cl[side], c);
        ++ncl[side];
      }
    }
    for (int64_t k = 0; k < nk; ++k) {
      if (route[k] == 0) {
        kc[r].ka.push_back(K.ka[k]);
        kc[r].kb.push_back(K.kb[k]);
        kc[r].ut.insert(kc[r].ut.end(), &K.ut[3 * k], &K.ut[3 * k] + 3);
      } else {
        const int side = route[k] < 0 ? 0 : 1;
        K.put(co[side], k);
        ++nco[side];
      }
    }
    for (int side = 0; side < 2; ++side) {
      std::vector<double>& o = m[r].out[side];
      o.push_back((double)ncl[side]);
      o.push_back((double)nco[side]);
      o.insert(o.end(), cl[side].begin(), cl[side].end());
      o.insert(o.end(), co[side].begin(), co[side].end());
    }
    sys->migrated_clumps = ncl[0] + ncl[1];
    sys->migration_bytes = (int64_t)(m[r].out[0].size() + m[r].out[1].size()) * 8;
  }
  TRY(exchange(ranks, n, m));
  for (int r = 0; r < n; ++r)
    for (int side = 0; side < 2; ++side) {
      const std::vector<double>& in = m[r].in[side];
      if (in.size() < 2) continue;
      const int64_t nc = (int64_t)in[0], nk = (int64_t)in[1];
      const double* b = in.data() + 2;
      for (int64_t c = 0; c < nc; ++c, b += kMigClump) keep[r].get(b);
      for (int64_t k = 0; k < nk; ++k, b += kMigContact) kc[r].get(b);
    }
  TRY(complete_ghosts(ranks, n, keep));
  for (int r = 0; r < n; ++r) TRY(import_directed(ranks[r], kc[r]));
  return DEM_OK;
}

extern "C" dem_status dem_migrate(dem_system* sys, double threshold, int32_t* moved) {
  if (!sys || !(threshold >= 0)) return DEM_ERR_INVALID_ARG;
  if (moved) *moved = 0;
  if (!sys->dist || sys->launched == 0) return DEM_OK;  // nothing moved since the last partition
  if ((sys->P.transport != DEM_TRANSPORT_NCCL && sys->P.transport != DEM_TRANSPORT_PEER) || !sys->comm) {
    sys->err = "dem_migrate needs the NCCL or PEER transport (loopback groups: dem_migrate_group)";
    return DEM_ERR_INVALID_ARG;
  }
  TRY(dem_synchronize(sys));
  cudaStream_t s = sys->stream;
  TRY(local_max_drift2(sys, nullptr));
  if (ncclAllReduce(sys->d_counter, sys->d_counter, 1, ncclDouble, ncclMax, sys->comm, s) != ncclSuccess)
    return DEM_ERR_NCCL;
  double d2 = 0;
  CK(cudaMemcpyAsync(&d2, sys->d_counter, sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (threshold > 0 && std::sqrt(d2) <= threshold) return DEM_OK;
  dem_system* one[1] = {sys};
  TRY(migrate_ranks(one, 1));
  if (moved) *moved = 1;
  return DEM_OK;
}

extern "C" dem_status dem_migrate_group(dem_system* const* systems, int32_t n, double threshold, int32_t* moved) {
  if (!systems || n < 1 || !(threshold >= 0)) return DEM_ERR_INVALID_ARG;
  if (moved) *moved = 0;
  for (int r = 0; r < n; ++r) {
    dem_system* sys = systems[r];
    if (!sys || (n > 1 && (!sys->dist ||
                           (sys->P.transport != DEM_TRANSPORT_LOOPBACK && sys->P.transport != DEM_TRANSPORT_LOOPBACK_PEER) ||
                           sys->P.rank != r ||
                           sys->P.n_ranks != n)))
      return DEM_ERR_INVALID_ARG;
  }
  if (n == 1 && !systems[0]->dist) return DEM_OK;
  if (systems[0]->launched == 0) return DEM_OK;  // nothing moved since the last partition
  double d2 = 0;
  for (int r = 0; r < n; ++r) {
    dem_system* sys = systems[r];
    TRY(dem_synchronize(sys));
    TRY(local_max_drift2(sys, nullptr));
    double v = 0;
    if (cudaMemcpyAsync(&v, sys->d_counter, sizeof(double), cudaMemcpyDeviceToHost, sys->stream) != cudaSuccess ||
        cudaStreamSynchronize(sys->stream) != cudaSuccess)
      return DEM_ERR_CUDA;
    d2 = std::max(d2, v);
  }
  if (threshold > 0 && std::sqrt(d2) <= threshold) return DEM_OK;
  TRY(migrate_ranks(systems, n));
  if (moved) *moved = 1;
  return DEM_OK;
}
