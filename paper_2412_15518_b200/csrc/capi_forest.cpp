// C ABI: octree forest, device leaf arenas, ghost exchange (reference-exact
// 3-pass, or the one-round face exchange with cross-GPU halos) and the
// SSP-RK3 hydro step (include/tmgpu.h, "forest" section).
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "comm.h"
#include "forest.h"
#include "ghost.h"
#include "halo_plan.h"
#include "tmgpu_internal.h"

using namespace tmgpu;

constexpr int kGraphKey = 9;
struct StepGraph {
  uint64_t key[kGraphKey];
  cudaGraphExec_t exec;
  long long kernels;   // kernel nodes (the launch counter per replay)
  int cur_after;       // arena parity after the step
  uint64_t exchanges;  // ghost exchanges the step performs
};

struct tmgpu_forest {
  explicit tmgpu_forest(const ForestConfig& c) : forest(c) {}
  Forest forest;
  // distribution: owner rank of every canonical leaf (empty = all on rank 0)
  tmgpu_comm* comm = nullptr;
  std::vector<int> owner;
  HaloPlan plan;
  // device state (valid for `dev_version`); slots are LOCAL leaves (owned,
  // canonical order)
  uint64_t dev_version = ~0ull;
  long long nslots = 0;
  // Two ghosted arenas [slot][V][S^3]: the fused step reads arenas[cur] and
  // writes the updated interiors into arenas[cur ^ 1] (a CTA reads its
  // same-level neighbours' interiors, so updating in place would race).
  double* arenas[2] = {nullptr, nullptr};
  int cur = 0;
  double* arena() const { return arenas[cur]; }
  double* u0 = nullptr;       // [slot][V][E^3]
  double* xfer = nullptr;     // [slot][V][E^3] host-transfer staging (lazy)
  double* leaf_dx = nullptr;  // [slot]
  double* speeds = nullptr;   // [slot]
  double* diag = nullptr;     // [slot] floor hits of the last stage
  double* dt_dev = nullptr;   // [1]
  // optional reflux (tmgpu_forest_set_reflux): the stage's face fluxes and the
  // coarse leaves with finer faces (CSR over faces in (axis, dir) order)
  bool reflux = false;
  uint64_t reflux_version = ~0ull;
  double* flux = nullptr;  // [slot][6][V][E^2]
  int *rf_leaf = nullptr, *rf_off = nullptr, *rf_ad = nullptr, *rf_fine = nullptr;
  long long rf_n = 0;
  // distributed reflux: fine face blocks exchanged after every stage (NCCL)
  int2* rf_send_items = nullptr;  // (local slot, face) per send entry, peer-major
  long long rf_nsend = 0, rf_nrecv = 0;
  double *rf_sbuf = nullptr, *rf_rbuf = nullptr;
  std::vector<long long> rf_send_off, rf_send_cnt, rf_recv_off, rf_recv_cnt;  // doubles per peer
  const double* grav = nullptr;  // optional gravity g[3][stride] by local slot (device)
  long long grav_stride = 0;
  // optional: the stream the step's gravity is computed on; the step runs its
  // CFL reduction and first ghost exchange concurrently and waits for that
  // stream only before the first stage kernel
  cudaStream_t grav_stream = nullptr;
  cudaEvent_t ev_grav = nullptr;
  // optional in-step self-gravity (tmgpu_forest_set_gravity_solver)
  tmgpu_gravity_amr* gsolver = nullptr;
  int g_cadence = 0, g_flags = 0;
  double *g_phi = nullptr, *g_a = nullptr, *g_b = nullptr, *rho_tilde = nullptr;
  long long g_stride = 0;
  cudaEvent_t ev_fork = nullptr;
  unsigned long long* err_dev = nullptr;
  // grow-only device scratch kept across topology changes (regrid's prolonged
  // and restricted blocks, its gather table, flag output): one allocation
  // reused by every later regrid instead of a cudaMalloc per operation
  char* scratch = nullptr;
  size_t scratch_bytes = 0;
  // reference-exact 3-pass exchange (single GPU only)
  double* staged = nullptr;
  GhostFill* fills[3] = {nullptr, nullptr, nullptr};
  int* staged_of[3] = {nullptr, nullptr, nullptr};
  int* prolong[3] = {nullptr, nullptr, nullptr};
  GhostPassDev pass[3];
  // one-round face exchange (halo.h)
  PackItem* pack = nullptr;
  FaceSrc* faces = nullptr;
  int* face_src = nullptr;
  int2* pull_all = nullptr;
  int2* pull_fused = nullptr;
  double* slabs = nullptr;
  int n_pack = 0, n_pull_all = 0, n_pull_fused = 0;
  // multi-GPU overlap: halo NCCL + remote pulls on a side stream while the
  // interior leaves' stage runs; then the boundary leaves
  int2* pull_local = nullptr;
  int2* pull_remote = nullptr;
  int* interior_idx = nullptr;
  int* boundary_idx = nullptr;
  int n_pull_local = 0, n_pull_remote = 0, n_interior = 0, n_boundary = 0;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_packed = nullptr, ev_remote = nullptr;
  // peer-memory exchange (tmgpu_forest_set_peer), valid for `peer_version`
  bool peer = false;
  uint64_t peer_version = ~0ull;
  PeerTab ptab{};
  unsigned long long* peer_flags = nullptr;
  PackItem* pack_peer = nullptr;
  int2* pull_peer = nullptr;  // pull_local ++ pull_remote
  void* peer_opened[2 * kMaxPeers] = {};
  StageMaps maps[2]{};
  uint64_t exchanges = 0;  // ghost exchanges performed (structural counter)
  // optional per-phase device timing: events [start, cfl, (exch, stage) x 3]
  bool timing = false;
  cudaEvent_t ev[8] = {};
  double t_cfl = 0, t_exchange = 0, t_stage = 0;
  long long timed_steps = 0, pending_timed = 0;
  // CUDA graphs of the step (step_graph), dropped by graph_reset
  std::vector<StepGraph> graphs;
  cudaStream_t graph_stream = nullptr;
  cudaEvent_t gev_in = nullptr, gev_out = nullptr;
  bool graph_warm = false;  // one step ran outside a capture (kernel attributes set)
  int graph_captures = 0;   // a caller varying dt every step stops capturing after 32
  int world() const { return comm_world(comm); }
  int rank() const { return comm_rank(comm); }
};

namespace {

int fail(tmgpu_error* err, int code, const std::string& m) { return set_err(err, code, m.c_str()); }

void collect_timing(tmgpu_forest* f) {
  if (!f->pending_timed) return;
  float ms = 0;
  if (cudaEventSynchronize(f->ev[7]) != cudaSuccess) return;
  cudaEventElapsedTime(&ms, f->ev[0], f->ev[1]);
  f->t_cfl += ms;
  for (int s = 0; s < 3; ++s) {
    cudaEventElapsedTime(&ms, f->ev[1 + 2 * s], f->ev[2 + 2 * s]);
    f->t_exchange += ms;
    cudaEventElapsedTime(&ms, f->ev[2 + 2 * s], f->ev[3 + 2 * s]);
    f->t_stage += ms;
  }
  f->timed_steps += 1;
  f->pending_timed = 0;
}

// Release the peer exchange. collective = true (tmgpu_forest_set_peer, called
// on every rank): a barrier after every rank's last exchange, then each rank
// unmaps its peers' buffers, a second barrier, and only then the buffers this
// rank exported are freed — freeing exported memory a peer still maps is
// undefined (a lagging peer's last consumption-flag store lands in it).
// collective = false (destroy / re-alloc on one rank): local release only;
// callers tear a peer forest down with tmgpu_forest_set_peer(f, 0) first.
void peer_close(tmgpu_forest* f, bool collective = false) {
  if (f->peer_flags || f->peer) cudaDeviceSynchronize();
  const bool coll = collective && f->peer && f->world() > 1;
  std::string why;
  if (coll) comm_barrier(f->comm, &why);
  for (void*& p : f->peer_opened) {
    if (p) cudaIpcCloseMemHandle(p);
    p = nullptr;
  }
  if (coll) comm_barrier(f->comm, &why);
  for (void* p : {(void*)f->peer_flags, (void*)f->pack_peer, (void*)f->pull_peer})
    if (p) cudaFree(p);
  f->peer_flags = nullptr;
  f->pack_peer = nullptr;
  f->pull_peer = nullptr;
  f->ptab = PeerTab{};
  f->peer = false;
  f->peer_version = ~0ull;
}

// Drop the cached step graphs (whatever a step enqueues is about to change).
void graph_reset(tmgpu_forest* f) {
  for (auto& g : f->graphs) cudaGraphExecDestroy(g.exec);
  f->graphs.clear();
}

void free_dev(tmgpu_forest* f) {
  graph_reset(f);
  peer_close(f);
  auto fr = [](void* p) {
    if (p) cudaFree(p);
  };
  for (void* p : {(void*)f->arenas[0], (void*)f->arenas[1], (void*)f->u0, (void*)f->xfer,
                  (void*)f->leaf_dx, (void*)f->speeds, (void*)f->diag, (void*)f->dt_dev,
                  (void*)f->err_dev, (void*)f->staged, (void*)f->pack, (void*)f->faces,
                  (void*)f->face_src, (void*)f->pull_all, (void*)f->pull_fused, (void*)f->slabs,
                  (void*)f->pull_local, (void*)f->pull_remote, (void*)f->interior_idx,
                  (void*)f->boundary_idx})
    fr(p);
  f->pull_local = f->pull_remote = nullptr;
  f->interior_idx = f->boundary_idx = nullptr;
  f->n_pull_local = f->n_pull_remote = f->n_interior = f->n_boundary = 0;
  for (int a = 0; a < 3; ++a) {
    fr(f->fills[a]);
    fr(f->staged_of[a]);
    fr(f->prolong[a]);
    f->fills[a] = nullptr;
    f->staged_of[a] = nullptr;
    f->prolong[a] = nullptr;
    f->pass[a] = GhostPassDev{};
  }
  f->arenas[0] = f->arenas[1] = nullptr;
  f->cur = 0;
  f->u0 = f->xfer = f->leaf_dx = f->speeds = f->diag = f->dt_dev = f->staged = f->slabs = nullptr;
  f->err_dev = nullptr;
  f->pack = nullptr;
  f->faces = nullptr;
  f->face_src = nullptr;
  f->pull_all = f->pull_fused = nullptr;
  f->n_pack = f->n_pull_all = f->n_pull_fused = 0;
  f->dev_version = ~0ull;
  f->nslots = 0;
}

int ready(tmgpu_forest* f, tmgpu_error* err) {
  if (!f) return fail(err, TMGPU_ERR_INVALID, "null forest");
  if (f->dev_version != f->forest.topology_version() || !f->arenas[0])
    return fail(err, TMGPU_ERR_INVALID,
                "device arena is stale: call tmgpu_forest_alloc after changing the topology");
  return TMGPU_OK;
}

template <class T>
cudaError_t upload(T** dst, const std::vector<T>& v, cudaError_t e) {
  if (e != cudaSuccess) return e;
  e = cudaMalloc((void**)dst, v.empty() ? 16 : v.size() * sizeof(T));
  if (e == cudaSuccess && !v.empty())
    e = cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  return e;
}

// At least `bytes` of the forest's device scratch (contents not kept on growth).
cudaError_t scratch_reserve(tmgpu_forest* f, size_t bytes) {
  if (bytes <= f->scratch_bytes) return cudaSuccess;
  bytes = std::max(bytes, f->scratch_bytes + f->scratch_bytes / 2);  // amortised growth
  if (f->scratch) cudaFree(f->scratch);
  f->scratch = nullptr;
  f->scratch_bytes = 0;
  cudaError_t e = cudaMalloc((void**)&f->scratch, bytes);
  if (e == cudaSuccess) f->scratch_bytes = bytes;
  return e;
}

// (Re)build the device arenas, the exchange plans and the TMA maps for the
// current topology and distribution.
int alloc_device(tmgpu_forest* f, tmgpu_error* err) {
  free_dev(f);
  const auto& cfg = f->forest.config();
  if (cfg.edge != 8 || cfg.ghost != 2 || (cfg.vars != 5 && cfg.vars != 1))
    return fail(err, TMGPU_ERR_INVALID, "device arena supports edge 8, ghost 2, vars 1|5");
  const auto& lv = f->forest.leaves();
  const int world = f->world(), rank = f->rank();
  std::vector<int> owner = f->owner;
  if (owner.size() != lv.size()) {
    if (world > 1) return fail(err, TMGPU_ERR_INVALID, "distribution does not match the topology");
    owner.assign(lv.size(), 0);
  }
  try {
    f->plan = build_halo_plan(f->forest, owner, rank, world);
  } catch (const std::exception& ex) {
    return fail(err, TMGPU_ERR_AMR, ex.what());
  }
  const HaloPlan& P = f->plan;
  const long long n = (long long)P.loc2gl.size();
  const int V = cfg.vars;
  const size_t S3 = 1728;
  cudaError_t e = cudaSuccess;
  auto M = [&](void** p, size_t bytes) {
    if (e == cudaSuccess) e = cudaMalloc(p, bytes ? bytes : 16);
  };
  M((void**)&f->arenas[0], n * V * S3 * sizeof(double));
  M((void**)&f->arenas[1], n * V * S3 * sizeof(double));
  M((void**)&f->u0, n * V * 512 * sizeof(double));
  M((void**)&f->speeds, n * sizeof(double));
  M((void**)&f->diag, n * sizeof(double));
  M((void**)&f->dt_dev, sizeof(double));
  M((void**)&f->err_dev, sizeof(unsigned long long));
  M((void**)&f->slabs, P.total_doubles * sizeof(double));
  for (int b = 0; b < 2 && e == cudaSuccess; ++b)  // SubGrid() zeroes
    e = cudaMemset(f->arenas[b], 0, n * V * S3 * sizeof(double));
  if (e == cudaSuccess) e = cudaMemset(f->err_dev, 0xff, sizeof(unsigned long long));
  std::vector<double> dx(n);
  for (long long s = 0; s < n; ++s) dx[s] = f->forest.cell_size(lv[P.loc2gl[s]].level);
  e = upload(&f->leaf_dx, dx, e);
  e = upload(&f->pack, P.pack, e);
  e = upload(&f->faces, P.faces, e);
  e = upload(&f->face_src, P.face_src, e);
  e = upload((int**)&f->pull_all, P.pull_all, e);
  e = upload((int**)&f->pull_fused, P.pull_fused, e);
  f->n_pack = (int)P.pack.size();
  f->n_pull_all = (int)P.pull_all.size() / 2;
  f->n_pull_fused = (int)P.pull_fused.size() / 2;
  e = upload((int**)&f->pull_local, P.pull_fused_local, e);
  e = upload((int**)&f->pull_remote, P.pull_fused_remote, e);
  e = upload(&f->interior_idx, P.interior_slots, e);
  e = upload(&f->boundary_idx, P.boundary_slots, e);
  f->n_pull_local = (int)P.pull_fused_local.size() / 2;
  f->n_pull_remote = (int)P.pull_fused_remote.size() / 2;
  f->n_interior = (int)P.interior_slots.size();
  f->n_boundary = (int)P.boundary_slots.size();
  if (e == cudaSuccess && world > 1 && !f->side) {
    e = cudaStreamCreateWithFlags(&f->side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f->ev_packed, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f->ev_remote, cudaEventDisableTiming);
  }
  if (world == 1) {  // reference-exact 3-pass plans (global slot == local slot)
    size_t max_prolong = 0;
    for (int a = 0; a < 3 && e == cudaSuccess; ++a) {
      const std::vector<Fill> plan = f->forest.plan_axis(a);
      std::vector<GhostFill> gf(plan.size());
      std::vector<int> sof(plan.size(), -1), pro;
      for (size_t i = 0; i < plan.size(); ++i) {
        const Fill& p = plan[i];
        gf[i] = GhostFill{p.dst, p.src, p.kind, p.axis, p.dir, p.qt1, p.qt2, {0, 0, 0}};
        if (p.kind == 1) {
          sof[i] = (int)pro.size();
          pro.push_back((int)i);
        }
      }
      max_prolong = std::max(max_prolong, pro.size());
      e = upload(&f->fills[a], gf, e);
      e = upload(&f->staged_of[a], sof, e);
      e = upload(&f->prolong[a], pro, e);
      f->pass[a] = GhostPassDev{f->fills[a], f->staged_of[a], f->prolong[a], (int)gf.size(),
                                (int)pro.size()};
    }
    M((void**)&f->staged, max_prolong * V * 8 * 8 * 2 * sizeof(double));
  }
  if (e != cudaSuccess) {
    free_dev(f);
    return cuda_err(err, e, "tmgpu_forest_alloc");
  }
  std::string why;
  int rc = make_stage_maps(f->arenas[0], V, (long long)V * S3, n, &f->maps[0], &why);
  if (rc == TMGPU_OK) rc = make_stage_maps(f->arenas[1], V, (long long)V * S3, n, &f->maps[1], &why);
  if (rc != TMGPU_OK) {
    free_dev(f);
    return fail(err, rc, why);
  }
  f->nslots = n;
  f->dev_version = f->forest.topology_version();
  return TMGPU_OK;
}

// Exchange modes: kExact = reference 3-pass fill of the full ghost shell
// (ghost.cpp:282-296, single GPU); kFaces = one-round fill of every face
// ghost, in place; kFused = one-round fill of every face the stage kernel
// does not read straight from a local same-level neighbour, with the
// prolongation ghost taps read from the other arena (the previous exchange).
enum ExchangeMode { kExact, kFaces, kFused };

int exchange(tmgpu_forest* f, cudaStream_t st, ExchangeMode mode, std::string* why) {
  const int V = f->forest.config().vars;
  cudaError_t e = cudaSuccess;
  if (mode == kExact) {
    if (f->world() > 1) {
      if (why) *why = "the reference-exact 3-pass exchange is single-GPU only";
      return TMGPU_ERR_INVALID;
    }
    for (int a = 0; a < 3 && e == cudaSuccess; ++a)
      e = ghost_pass(f->arena(), V, f->pass[a], f->staged, st);
  } else {
    const bool all = mode == kFaces;
    const double* prev = all ? f->arena() : f->arenas[f->cur ^ 1];
    if (f->peer) {
      if (f->peer_version != f->forest.topology_version()) {
        if (why) *why = "peer exchange: topology changed; call tmgpu_forest_set_peer again";
        return TMGPU_ERR_INVALID;
      }
      // this round's sequence number lives in device memory (a captured step
      // replays with a new one); every rank runs the same rounds
      e = seq_bump(f->ptab.seqp, st);
      if (e == cudaSuccess)
        e = halo_pack_peer(f->arena(), prev, V, f->pack_peer, f->n_pack, f->slabs, f->ptab, st);
      // every face: one list whose faces all wait for the senders
      if (e == cudaSuccess)
        e = all ? halo_pull_peer(f->arena(), V, f->faces, f->pull_all, 0, f->n_pull_all, f->slabs,
                                 f->ptab, st)
                : halo_pull_peer(f->arena(), V, f->faces, f->pull_peer, f->n_pull_local,
                                 f->n_pull_fused, f->slabs, f->ptab, st);
      if (e != cudaSuccess) {
        if (why) *why = std::string("peer ghost exchange: ") + cudaGetErrorString(e);
        return TMGPU_ERR_CUDA;
      }
      f->exchanges += 1;
      return TMGPU_OK;
    }
    e = halo_pack(f->arena(), prev, V, f->pack, f->n_pack, f->slabs, st);
    if (e == cudaSuccess && f->world() > 1) {
      const HaloPlan& P = f->plan;
      int rc = comm_exchange(f->comm, f->slabs + P.send_base, P.send_off, P.send_cnt,
                             f->slabs + P.recv_base, P.recv_off, P.recv_cnt, st, why);
      if (rc != TMGPU_OK) return rc;
    }
    if (e == cudaSuccess)
      e = halo_pull(f->arena(), V, f->faces, all ? f->pull_all : f->pull_fused,
                    all ? f->n_pull_all : f->n_pull_fused, f->slabs, st);
  }
  if (e != cudaSuccess) {
    if (why) *why = std::string("ghost exchange: ") + cudaGetErrorString(e);
    return TMGPU_ERR_CUDA;
  }
  f->exchanges += 1;
  return TMGPU_OK;
}

// slice = canonical leaf index of the first failing local leaf
int solver_err_from_word(tmgpu_error* err, unsigned long long w, const std::vector<int>& loc2gl) {
  const unsigned cell = (unsigned)(w & 0xffffffffu) % 512u;
  const int i = (int)(cell % 8), j = (int)(cell / 8 % 8), k = (int)(cell / 64);
  if (err) {
    const size_t slot = (size_t)(w >> 32);
    err->code = TMGPU_ERR_SOLVER;
    err->slice = slot < loc2gl.size() ? loc2gl[slot] : (int64_t)slot;
    err->cell[0] = i;
    err->cell[1] = j;
    err->cell[2] = k;
    std::snprintf(err->message, sizeof(err->message),
                  "non-finite state after stage at cell (%d,%d,%d)", i, j, k);
  }
  return TMGPU_ERR_SOLVER;
}

}  // namespace

extern "C" {

tmgpu_forest* tmgpu_forest_create(int edge, int ghost, int vars, int max_level,
                                  const int* root_dims, const int* bc, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  ForestConfig c;
  c.edge = edge;
  c.ghost = ghost;
  c.vars = vars;
  c.max_level = max_level;
  for (int a = 0; a < 3; ++a) {
    c.root_dims[a] = root_dims ? root_dims[a] : 1;
    c.bc[a] = bc ? bc[a] : 0;
  }
  try {
    return new tmgpu_forest(c);
  } catch (const std::exception& ex) {
    set_err(err, TMGPU_ERR_AMR, ex.what());
    return nullptr;
  }
}

void tmgpu_forest_destroy(tmgpu_forest* f) {
  if (!f) return;
  free_dev(f);
  tmgpu_forest_set_reflux(f, 0, nullptr);
  if (f->scratch) cudaFree(f->scratch);
  if (f->graph_stream) cudaStreamDestroy(f->graph_stream);
  if (f->gev_in) cudaEventDestroy(f->gev_in);
  if (f->gev_out) cudaEventDestroy(f->gev_out);
  if (f->ev_grav) cudaEventDestroy(f->ev_grav);
  if (f->ev_fork) cudaEventDestroy(f->ev_fork);
  if (f->side) cudaStreamDestroy(f->side);
  if (f->ev_packed) cudaEventDestroy(f->ev_packed);
  if (f->ev_remote) cudaEventDestroy(f->ev_remote);
  for (auto& e : f->ev)
    if (e) cudaEventDestroy(e);
  delete f;
}

int tmgpu_forest_refine(tmgpu_forest* f, uint64_t packed, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  try {
    f->forest.refine(NodeId::unpack(packed));
    return TMGPU_OK;
  } catch (const std::exception& ex) {
    return fail(err, TMGPU_ERR_AMR, ex.what());
  }
}

int tmgpu_forest_coarsen(tmgpu_forest* f, uint64_t packed, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  try {
    f->forest.coarsen(NodeId::unpack(packed));
    return TMGPU_OK;
  } catch (const std::exception& ex) {
    return fail(err, TMGPU_ERR_AMR, ex.what());
  }
}

// Refine then coarsen the given nodes with the device data carried along, as
// the reference's Tree::refine / coarsen do with their grids (prolong_cell /
// restrict_cells, octree.cpp:149-293), in the same order (cascaded 2:1
// refinements included): children get the prolonged interior and zero ghosts,
// a coarsened parent the restricted interior and zero ghosts, untouched leaves
// keep their whole block. Then the arena is rebuilt for the new topology.
// Single GPU. On a topology error the tree keeps the operations done so far
// (as the reference's) and the device arena is stale (tmgpu_forest_alloc).
int tmgpu_forest_regrid(tmgpu_forest* f, const uint64_t* refine, size_t nr, const uint64_t* coarsen,
                        size_t nc, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (int rc = ready(f, err)) return rc;
  if (f->world() > 1) return fail(err, TMGPU_ERR_INVALID, "regrid: single GPU only");
  const int V = f->forest.config().vars;
  const long long stride = (long long)V * 1728;
  const std::vector<NodeId> old_leaves = f->forest.leaves();
  double* old = f->arenas[f->cur];
  std::unordered_map<uint64_t, const double*> pool;
  for (size_t s = 0; s < old_leaves.size(); ++s) pool[old_leaves[s].packed()] = old + (long long)s * stride;
  f->forest.clear_oplog();
  try {
    for (size_t q = 0; q < nr; ++q) f->forest.refine(NodeId::unpack(refine[q]));
    for (size_t q = 0; q < nc; ++q) f->forest.coarsen(NodeId::unpack(coarsen[q]));
  } catch (const std::exception& ex) {
    return fail(err, TMGPU_ERR_AMR, ex.what());
  }
  cudaStream_t st = 0;
  // every prolonged / restricted block lives until the final gather (a later
  // operation may read an earlier one's output), so size the scratch for all
  // of them plus the gather table, once
  size_t blocks = 0;
  for (const Forest::Op& op : f->forest.oplog()) blocks += op.refine ? 8 : 1;
  const size_t nnew = f->forest.leaves().size();
  const size_t blk_bytes = (size_t)stride * sizeof(double);
  const size_t table_off = blocks * blk_bytes;
  cudaError_t e = scratch_reserve(f, table_off + (nnew ? nnew : 1) * sizeof(double*));
  try {
  double* next = (double*)f->scratch;
  for (const Forest::Op& op : f->forest.oplog()) {
    if (e != cudaSuccess) break;
    const NodeId& id = op.node;
    if (op.refine) {
      double* ch = next;
      next += 8 * stride;
      e = cudaMemsetAsync(ch, 0, 8 * blk_bytes, st);
      if (e == cudaSuccess) e = launch_prolong(pool.at(id.packed()), ch, V, st);
      pool.erase(id.packed());
      for (int b = 0; b < 8; ++b)
        pool[id.child(b & 1, (b >> 1) & 1, (b >> 2) & 1).packed()] = ch + (long long)b * stride;
    } else {
      double* pg = next;
      next += stride;
      const double* chp[8];
      for (int b = 0; b < 8; ++b) {
        const uint64_t c = id.child(b & 1, (b >> 1) & 1, (b >> 2) & 1).packed();
        chp[b] = pool.at(c);
        pool.erase(c);
      }
      e = cudaMemsetAsync(pg, 0, blk_bytes, st);
      if (e == cudaSuccess) e = launch_restrict(chp, pg, V, st);
      pool[id.packed()] = pg;
    }
  }
  f->forest.clear_oplog();
  // rebuild the device state for the new topology, keeping the old arena alive
  f->arenas[f->cur] = nullptr;
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  int rc = e == cudaSuccess ? alloc_device(f, err) : TMGPU_ERR_CUDA;
  if (rc == TMGPU_OK) {
    const auto& nl = f->forest.leaves();
    std::vector<const double*> src(nl.size());
    for (size_t s = 0; s < nl.size(); ++s) src[s] = pool.at(nl[s].packed());
    const double** dsrc = (const double**)(f->scratch + table_off);
    if (!src.empty())
      e = cudaMemcpy(dsrc, src.data(), src.size() * sizeof(double*), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = launch_gather_blocks(dsrc, (long long)src.size(), f->arenas[f->cur], stride, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  }
  cudaFree(old);
  if (rc != TMGPU_OK) return rc;
  return cuda_err(err, e, "tmgpu_forest_regrid");
  } catch (const std::exception& ex) {  // a bookkeeping bug, never expected
    return fail(err, TMGPU_ERR_AMR, std::string("regrid: ") + ex.what());
  }
}

// Tree::flag_refinement (octree.cpp:295-323) for every local leaf, on the
// current device state (ghosts as they are): flags[slot] = 0/1.
int tmgpu_forest_flag(tmgpu_forest* f, double theta, double rho_floor, int* flags_host,
                      tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (int rc = ready(f, err)) return rc;
  const int V = f->forest.config().vars;
  cudaError_t e = scratch_reserve(f, (f->nslots ? f->nslots : 1) * sizeof(int));
  int* d = (int*)f->scratch;
  if (e == cudaSuccess) e = launch_flag(f->arena(), (long long)V * 1728, f->nslots, theta, rho_floor, d, 0);
  if (e == cudaSuccess)
    e = cudaMemcpy(flags_host, d, f->nslots * sizeof(int), cudaMemcpyDeviceToHost);
  return cuda_err(err, e, "tmgpu_forest_flag");
}

int tmgpu_forest_is_leaf(tmgpu_forest* f, uint64_t packed) {
  return f && f->forest.is_leaf(NodeId::unpack(packed)) ? 1 : 0;
}

size_t tmgpu_forest_leaves(tmgpu_forest* f, uint64_t* out, size_t cap) {
  const auto& lv = f->forest.leaves();
  for (size_t i = 0; i < lv.size() && i < cap; ++i) out[i] = lv[i].packed();
  return lv.size();
}

int tmgpu_forest_face_neighbor(tmgpu_forest* f, uint64_t leaf, int axis, int dir, uint64_t* ids4,
                               int* count) {
  try {
    FaceNeighbors nb = f->forest.face_neighbor(NodeId::unpack(leaf), axis, dir);
    *count = nb.count;
    for (int q = 0; q < nb.count; ++q) ids4[q] = nb.ids[q].packed();
    return (int)nb.kind;
  } catch (const std::exception&) {
    *count = 0;
    return -1;
  }
}

size_t tmgpu_forest_plan(tmgpu_forest* f, int axis, int64_t* rows, size_t cap) {
  const auto plan = f->forest.plan_axis(axis);
  const auto& lv = f->forest.leaves();
  for (size_t r = 0; r < plan.size() && r < cap; ++r) {
    const Fill& p = plan[r];
    int64_t* o = rows + 7 * r;
    o[0] = (int64_t)lv[p.dst].packed();
    o[1] = p.src < 0 ? -1 : (int64_t)lv[p.src].packed();
    o[2] = p.kind;
    o[3] = p.axis;
    o[4] = p.dir;
    o[5] = p.qt1;
    o[6] = p.qt2;
  }
  return plan.size();
}

int tmgpu_forest_balanced(tmgpu_forest* f) { return f->forest.is_balanced() ? 1 : 0; }

double tmgpu_forest_cell_size(tmgpu_forest* f, int level) { return f->forest.cell_size(level); }

uint64_t tmgpu_forest_topology_version(tmgpu_forest* f) { return f->forest.topology_version(); }

uint64_t tmgpu_forest_exchanges(tmgpu_forest* f) { return f->exchanges; }

int tmgpu_forest_scenario_refine(tmgpu_forest* f, int kind, int min_level, int max_level,
                                 double theta, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  try {
    scenario_refine(f->forest, kind, min_level, max_level, theta);
    return TMGPU_OK;
  } catch (const std::exception& ex) {
    return fail(err, TMGPU_ERR_AMR, ex.what());
  }
}

int tmgpu_forest_scenario_fill(tmgpu_forest* f, int kind, uint64_t seed, double* compact_host,
                               tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (f->forest.config().vars != 5) return fail(err, TMGPU_ERR_INVALID, "scenarios are Euler (vars 5)");
  scenario_fill(f->forest, kind, seed, compact_host);
  return TMGPU_OK;
}

// Distribute the canonical leaves over the ranks of `comm` (owner[g] per leaf,
// normally partition_leaves); invalidates the device state (call alloc).
int tmgpu_forest_distribute(tmgpu_forest* f, tmgpu_comm* comm, const int* owner, size_t n,
                            tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (f) graph_reset(f);  // what a step enqueues changes
  if (n != f->forest.leaves().size())
    return fail(err, TMGPU_ERR_INVALID, "owner list does not match the leaf count");
  const int world = comm_world(comm);
  for (size_t i = 0; i < n; ++i)
    if (owner[i] < 0 || owner[i] >= world) return fail(err, TMGPU_ERR_INVALID, "owner out of range");
  free_dev(f);
  f->comm = comm;
  f->owner.assign(owner, owner + n);
  return TMGPU_OK;
}

// Local (owned) leaves in canonical order = local slot order.
size_t tmgpu_forest_local_leaves(tmgpu_forest* f, uint64_t* out, size_t cap) {
  const auto& lv = f->forest.leaves();
  std::vector<int> loc;
  for (size_t g = 0; g < lv.size(); ++g)
    if (f->owner.size() != lv.size() ? f->rank() == 0 : f->owner[g] == f->rank())
      loc.push_back((int)g);
  for (size_t i = 0; i < loc.size() && i < cap; ++i) out[i] = lv[loc[i]].packed();
  return loc.size();
}

// Host halo plan of (rank, owner) without touching the device (tests):
// rows of 7 int64 (direction 0 send / 1 recv, peer, dst, src, kind, axis, dir).
size_t tmgpu_forest_halo_manifest(tmgpu_forest* f, const int* owner, int rank, int world,
                                  int64_t* rows, size_t cap) {
  std::vector<int> o(owner, owner + f->forest.leaves().size());
  HaloPlan P = build_halo_plan(f->forest, o, rank, world);
  size_t r = 0;
  for (int d = 0; d < 2; ++d)
    for (const auto& m : d == 0 ? P.send_manifest : P.recv_manifest) {
      if (r < cap) {
        int64_t* x = rows + 7 * r;
        x[0] = d;
        for (int k = 0; k < 6; ++k) x[1 + k] = m[k];
      }
      ++r;
    }
  return r;
}

int tmgpu_forest_alloc(tmgpu_forest* f, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  return alloc_device(f, err);
}

double* tmgpu_forest_arena(tmgpu_forest* f) { return f->arena(); }

int tmgpu_forest_interior(tmgpu_forest* f, double* compact, int to_device, int flags, void* stream,
                          tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (int rc = ready(f, err)) return rc;
  cudaStream_t st = as_stream(stream);
  const int V = f->forest.config().vars;
  const size_t bytes = (size_t)f->nslots * V * 512 * sizeof(double);
  double* dev = compact;
  cudaError_t e = cudaSuccess;
  if (flags & TMGPU_HOST_PTRS) {
    if (!f->xfer) e = cudaMalloc(&f->xfer, bytes ? bytes : 8);
    dev = f->xfer;
    if (e == cudaSuccess && to_device) e = cudaMemcpyAsync(dev, compact, bytes, cudaMemcpyHostToDevice, st);
  }
  if (e == cudaSuccess) e = interior_copy(f->arena(), dev, V, f->nslots, to_device != 0, st);
  if (e == cudaSuccess && (flags & TMGPU_HOST_PTRS) && !to_device)
    e = cudaMemcpyAsync(compact, dev, bytes, cudaMemcpyDeviceToHost, st);
  cudaError_t e2 = (flags & TMGPU_ASYNC) ? cudaSuccess : cudaStreamSynchronize(st);
  return cuda_err(err, e != cudaSuccess ? e : e2, "tmgpu_forest_interior");
}

int tmgpu_forest_grids(tmgpu_forest* f, double* ghosted_host, int to_device, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (int rc = ready(f, err)) return rc;
  const size_t bytes = (size_t)f->nslots * f->forest.config().vars * 1728 * sizeof(double);
  cudaError_t e = to_device ? cudaMemcpy(f->arena(), ghosted_host, bytes, cudaMemcpyHostToDevice)
                            : cudaMemcpy(ghosted_host, f->arena(), bytes, cudaMemcpyDeviceToHost);
  return cuda_err(err, e, "tmgpu_forest_grids");
}

// Either ghosted arena by role: which 0 = the current state, 1 = the other
// (ping-pong) arena. The step carries both arenas' ghost layers across
// exchanges (prolongation reads coarse cells next to the face, which can be
// ghosts last written several exchanges earlier), so a bitwise resumable
// checkpoint stores and restores both.
int tmgpu_forest_arena_grids(tmgpu_forest* f, int which, double* ghosted_host, int to_device,
                             tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (int rc = ready(f, err)) return rc;
  if (which != 0 && which != 1) return fail(err, TMGPU_ERR_INVALID, "arena role must be 0 (current) or 1 (other)");
  double* a = f->arenas[f->cur ^ which];
  if (!a) return fail(err, TMGPU_ERR_INVALID, "no second arena");
  const size_t bytes = (size_t)f->nslots * f->forest.config().vars * 1728 * sizeof(double);
  cudaError_t e = cudaDeviceSynchronize();  // the buffer may be host or device memory (UVA)
  if (e == cudaSuccess)
    e = to_device ? cudaMemcpy(a, ghosted_host, bytes, cudaMemcpyDefault)
                  : cudaMemcpy(ghosted_host, a, bytes, cudaMemcpyDefault);
  return cuda_err(err, e, "tmgpu_forest_arena_grids");
}

int tmgpu_forest_fill_ghosts(tmgpu_forest* f, void* stream, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (int rc = ready(f, err)) return rc;
  cudaStream_t st = as_stream(stream);
  std::string why;
  if (int rc = exchange(f, st, kExact, &why)) return fail(err, rc, why);
  return cuda_err(err, cudaStreamSynchronize(st), "tmgpu_forest_fill_ghosts");
}

// One-round face-only exchange (the step's default).
int tmgpu_forest_fill_faces(tmgpu_forest* f, void* stream, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (int rc = ready(f, err)) return rc;
  cudaStream_t st = as_stream(stream);
  std::string why;
  if (int rc = exchange(f, st, kFaces, &why)) return fail(err, rc, why);
  return cuda_err(err, cudaStreamSynchronize(st), "tmgpu_forest_fill_faces");
}

int tmgpu_forest_max_wavespeed(tmgpu_forest* f, double gamma, double* per_leaf_host,
                               tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (int rc = ready(f, err)) return rc;
  const int V = f->forest.config().vars;
  cudaStream_t st = cudaStreamPerThread;
  cudaError_t e = launch_max_wavespeed(f->arena(), (long long)V * 1728, nullptr, 0, nullptr, gamma, V,
                                       f->nslots, f->speeds, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(per_leaf_host, f->speeds, f->nslots * sizeof(double), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return cuda_err(err, e, "tmgpu_forest_max_wavespeed");
}

// One SSP-RK3 step (rk3.hpp:16-34): [cfl dt] then 3 x
// (ghost exchange -> aggregated stage kernel over every leaf, in place, with
// the rk3_combine epilogue). cfl > 0: dt = cfl * min(dx / max_wavespeed)
// computed on the device; else `dt` is used. With TMGPU_ASYNC the call only
// enqueues; tmgpu_forest_check reports errors later.
// Gravity source for subsequent steps: g = device [3][comp_stride] by local
// slot (g[q*comp_stride + slot*512 + c]), e.g. tmgpu_gravity_amr_solve's
// output; NULL disables (pure hydro = the reference's stage).
int tmgpu_forest_set_gravity(tmgpu_forest* f, const double* g, long long comp_stride,
                             tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (f) graph_reset(f);  // what a step enqueues changes
  if (g && comp_stride < f->nslots * 512)
    return set_err(err, TMGPU_ERR_INVALID, "gravity: component stride below the local cell count");
  f->grav = g;
  f->grav_stride = comp_stride;
  return TMGPU_OK;
}

int tmgpu_forest_set_gravity_solver(tmgpu_forest* f, tmgpu_gravity_amr* G, int solves_per_step,
                                    int grav_flags, double* phi, double* g, double* g2,
                                    double* rho_tilde, long long comp_stride, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (f) graph_reset(f);  // what a step enqueues changes
  if (!f) return fail(err, TMGPU_ERR_INVALID, "null forest");
  if (!G) {
    f->gsolver = nullptr;
    f->g_cadence = 0;
    return TMGPU_OK;
  }
  if (int rc = ready(f, err)) return rc;
  if (solves_per_step != 1 && solves_per_step != 3 && solves_per_step != 6)
    return fail(err, TMGPU_ERR_INVALID, "gravity solver: solves_per_step must be 1, 3 or 6");
  if (!phi || !g || (solves_per_step == 6 && (!g2 || !rho_tilde)))
    return fail(err, TMGPU_ERR_INVALID, "gravity solver: missing field buffer");
  if (comp_stride < f->nslots * 512)
    return fail(err, TMGPU_ERR_INVALID, "gravity: component stride below the local cell count");
  if (!f->ev_fork) {
    cudaError_t e = cudaEventCreateWithFlags(&f->ev_fork, cudaEventDisableTiming);
    if (e == cudaSuccess && !f->ev_grav) e = cudaEventCreateWithFlags(&f->ev_grav, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_err(err, e, "tmgpu_forest_set_gravity_solver");
  }
  f->gsolver = G;
  f->g_cadence = solves_per_step;
  f->g_flags = grav_flags & TMGPU_GRAV_AM;
  f->g_phi = phi;
  f->g_a = g;
  f->g_b = g2;
  f->rho_tilde = rho_tilde;
  f->g_stride = comp_stride;
  f->grav = nullptr;  // the solver's field replaces an external one
  return TMGPU_OK;
}

namespace {
// One in-step gravity solve on the gravity stream (forked from `st` after the
// work enqueued so far): masses from the arena's interior density (rho NULL)
// or from a compact density, then the FMM into (g_phi, gout). The caller makes
// `st` wait for f->ev_grav before reading gout.
int grav_solve(tmgpu_forest* f, cudaStream_t st, const double* arena, const double* rho, double* gout,
               tmgpu_error* err, long long rho_stride = 512) {
  cudaStream_t gs = f->grav_stream ? f->grav_stream : st;
  cudaError_t e = cudaSuccess;
  if (gs != st) {
    e = cudaEventRecord(f->ev_fork, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(gs, f->ev_fork, 0);
    if (e != cudaSuccess) return cuda_err(err, e, "tmgpu_forest_step: gravity fork");
  }
  int rc = arena ? tmgpu_gravity_amr_mass_from_arena(f->gsolver, arena, f->forest.config().vars, gs, err)
                 : tmgpu_gravity_amr_mass_from_compact(f->gsolver, rho, rho_stride, gs, err);
  if (rc == TMGPU_OK)
    rc = tmgpu_gravity_amr_solve(f->gsolver, nullptr, f->g_phi, gout, f->g_flags | TMGPU_ASYNC, gs, err);
  if (rc != TMGPU_OK) return rc;
  e = cudaEventRecord(f->ev_grav, gs);
  return cuda_err(err, e, "tmgpu_forest_step: gravity join");
}
}  // namespace

int tmgpu_forest_step(tmgpu_forest* f, double dt, double cfl, double gamma, int flags, void* stream,
                      double* dt_used, tmgpu_error* err) {
  return tmgpu_forest_step_io(f, nullptr, nullptr, dt, cfl, gamma, flags, stream, dt_used, err);
}

namespace {
// Everything one step enqueues on `st` (and the streams it forks), from the
// first gravity solve to the output gather; host state it changes: f->cur,
// f->exchanges. Captured whole into a CUDA graph by step_graph.
int step_enqueue(tmgpu_forest* f, const double* in_compact, double* out_compact, double dt, double cfl,
                 double gamma, int flags, cudaStream_t st, tmgpu_error* err) {
  const int V = f->forest.config().vars;
  const int cadence = f->gsolver ? f->g_cadence : 0;
  const bool timed = f->timing;
  cudaError_t e = cudaSuccess;
  if (cadence) {  // stage 1's solve on the step's initial state, overlapping the CFL and exchange
    const int rc = in_compact ? grav_solve(f, st, nullptr, in_compact, f->g_a, err, (long long)V * 512)
                              : grav_solve(f, st, f->arena(), nullptr, f->g_a, err);
    if (rc) return rc;
  } else if (f->grav_stream) {
    e = cudaEventRecord(f->ev_grav, f->grav_stream);  // gravity enqueued so far
  }
  if (!(flags & TMGPU_ASYNC) && e == cudaSuccess)
    e = cudaMemsetAsync(f->err_dev, 0xff, sizeof(unsigned long long), st);
  if (e == cudaSuccess && in_compact && !(cfl > 0.0))  // input scatter (fused below when cfl > 0)
    e = interior_copy(f->arena(), const_cast<double*>(in_compact), V, f->nslots, true, st);
  if (e == cudaSuccess && cfl > 0.0) {
    e = in_compact ? launch_scatter_wavespeed(in_compact, f->arena(), (long long)V * 1728, gamma, f->nslots,
                                              f->speeds, st)
                   : launch_max_wavespeed(f->arena(), (long long)V * 1728, nullptr, 0, nullptr, gamma, V,
                                          f->nslots, f->speeds, st);
    if (e == cudaSuccess) e = launch_cfl_reduce(f->speeds, f->leaf_dx, f->nslots, cfl, f->dt_dev, st);
    if (e == cudaSuccess && f->world() > 1) {  // global dt: min over ranks (exact)
      std::string why;
      if (int rc = comm_allreduce_min(f->comm, f->dt_dev, 1, st, &why)) return fail(err, rc, why);
    }
  }
  if (timed) cudaEventRecord(f->ev[1], st);
  StageLaunch p{};
  p.hdr = nullptr;
  p.leaf_dx = f->leaf_dx;
  p.g_mode = 1.0;
  p.g_dt = dt;
  p.g_gamma = gamma;
  p.dt_ptr = cfl > 0.0 ? f->dt_dev : nullptr;
  p.out_stride = (long long)V * 1728;
  p.out_ghosted = 1;
  if (f->reflux && f->reflux_version != f->forest.topology_version())
    return fail(err, TMGPU_ERR_INVALID, "reflux: topology changed; call tmgpu_forest_set_reflux again");
  p.faces = f->reflux ? f->flux : nullptr;
  p.faces_stride = (long long)6 * V * 64;
  p.diag = f->diag;
  p.diag_stride = 1;
  p.u0 = f->u0;
  p.u0_stride = (long long)V * 512;
  p.err = f->err_dev;
  p.grav = cadence ? f->g_a : f->grav;
  p.grav_stride = cadence ? f->g_stride : f->grav_stride;
  p.count = (int)f->nslots;
  const bool exact = (flags & TMGPU_EXACT_GHOSTS) != 0;
  p.face_src = exact ? nullptr : f->face_src;
  // opt-in: measured no faster on C3 at 2-4 GPUs (the split boundary launch
  // under-fills the GPU), so the default keeps one exchange + one launch
  const bool overlap = !exact && f->world() > 1 && !f->peer && (flags & TMGPU_OVERLAP);
  // opt-in (TMGPU_SPLIT_STAGE=1): split each gravity stage so its update
  // overlaps the stage's solve (stage_kernel with p.defer, then
  // stage_epilogue_kernel once the field is there; the same bits; needs the
  // ping-pong arenas). Measured on C3 (3 solves): 5.39 ms vs 5.35 ms fused — the
  // solve already fills the GPU and the epilogue's extra pass costs 125 us.
  static const bool split_env = [] {
    const char* v = std::getenv("TMGPU_SPLIT_STAGE");
    return v && v[0] == '1';
  }();
  const bool split = split_env && cadence && !exact && !overlap && f->grav_stream;
  // a correction after the last stage (reflux, the 6-solve source) rules out
  // writing the output from the stage epilogue: gather after the loop instead
  const bool late_fix = f->reflux || cadence == 6;
  for (int stage = 1; stage <= 3 && e == cudaSuccess; ++stage) {
    std::string why;
    if (stage > 1 && cadence >= 3) {  // this stage's field from its input state
      if (int rc = grav_solve(f, st, f->arena(), nullptr, f->g_a, err)) return rc;
    }
    if (overlap) {
      // pack (all slabs) -> [side: NCCL halo, remote pulls] || [main: local pulls,
      // interior leaves' stage] -> join -> boundary leaves' stage
      e = halo_pack(f->arena(), f->arenas[f->cur ^ 1], V, f->pack, f->n_pack, f->slabs, st);
      if (e == cudaSuccess) e = cudaEventRecord(f->ev_packed, st);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(f->side, f->ev_packed, 0);
      if (e != cudaSuccess) break;
      const HaloPlan& P = f->plan;
      if (int rc = comm_exchange(f->comm, f->slabs + P.send_base, P.send_off, P.send_cnt,
                                 f->slabs + P.recv_base, P.recv_off, P.recv_cnt, f->side, &why))
        return fail(err, rc, why);
      e = halo_pull(f->arena(), V, f->faces, f->pull_remote, f->n_pull_remote, f->slabs, f->side);
      if (e == cudaSuccess) e = cudaEventRecord(f->ev_remote, f->side);
      if (e == cudaSuccess)
        e = halo_pull(f->arena(), V, f->faces, f->pull_local, f->n_pull_local, f->slabs, st);
      if (e != cudaSuccess) break;
      f->exchanges += 1;
    } else if (int rc = exchange(f, st, exact ? kExact : kFused, &why)) {
      return fail(err, rc, why);
    }
    // does this stage wait for a gravity solve on the gravity stream? With the
    // split stage the update runs concurrently with the solve and only the
    // epilogue waits; otherwise the stage kernel waits (and the exchange
    // interval includes the wait)
    const bool wait_grav =
        (cadence && (stage == 1 || cadence >= 3)) || (!cadence && stage == 1 && f->grav_stream);
    if (e == cudaSuccess && wait_grav && !split) e = cudaStreamWaitEvent(st, f->ev_grav, 0);
    if (timed) cudaEventRecord(f->ev[2 * stage], st);
    p.rk_stage = stage;
    p.out_compact = (stage == 3 && !late_fix) ? out_compact : nullptr;
    p.rho_save = cadence == 6 ? f->rho_tilde : nullptr;
    p.u0_save = stage == 1 ? f->u0 : nullptr;
    p.u0_save_stride = (long long)V * 512;
    // exact: in place (each CTA reads only its own block); fused: ping-pong
    const int dst = exact ? f->cur : (f->cur ^ 1);
    p.out = f->arenas[dst];
    if (overlap) {
      StageLaunch pi = p, pb = p;
      pi.index = f->interior_idx;
      pi.count = f->n_interior;
      pb.index = f->boundary_idx;
      pb.count = f->n_boundary;
      e = launch_stage(V, (flags & TMGPU_FAST) != 0, f->maps[f->cur], pi, st);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(st, f->ev_remote, 0);
      if (e == cudaSuccess) e = launch_stage(V, (flags & TMGPU_FAST) != 0, f->maps[f->cur], pb, st);
    } else if (split) {  // update || gravity solve, then the epilogue with the field
      StageLaunch pa = p;
      pa.defer = 1;
      pa.grav = nullptr;
      pa.rho_save = nullptr;
      e = launch_stage(V, (flags & TMGPU_FAST) != 0, f->maps[f->cur], pa, st);
      if (e == cudaSuccess && wait_grav) e = cudaStreamWaitEvent(st, f->ev_grav, 0);
      if (e == cudaSuccess) e = launch_stage_epilogue((flags & TMGPU_FAST) != 0, f->arenas[f->cur], p, st);
    } else {
      e = launch_stage(V, (flags & TMGPU_FAST) != 0, f->maps[f->cur], p, st);
    }
    if (e == cudaSuccess && f->reflux) {  // SSP-RK3 stage weights 1, 1/4, 2/3
      const double coef = stage == 1 ? 1.0 : (stage == 2 ? 0.25 : 2.0 / 3.0);
      if (f->world() > 1) {  // fine face blocks of coarse leaves on other GPUs
        e = launch_flux_pack(f->flux, V, f->rf_send_items, f->rf_nsend, f->rf_sbuf, st);
        std::string why;
        if (e == cudaSuccess)
          if (int rc = comm_exchange(f->comm, f->rf_sbuf, f->rf_send_off, f->rf_send_cnt, f->rf_rbuf,
                                     f->rf_recv_off, f->rf_recv_cnt, st, &why))
            return fail(err, rc, why);
      }
      if (e == cudaSuccess)
        e = launch_reflux(f->arenas[dst], V, f->flux, f->rf_leaf, f->rf_off, f->rf_ad, f->rf_fine, f->rf_n,
                          f->leaf_dx, p.dt_ptr, dt, coef, st, f->rf_rbuf);
    }
    if (e == cudaSuccess && cadence == 6) {  // second solve on the provisional density, trapezoid source
      if (int rc = grav_solve(f, st, nullptr, f->rho_tilde, f->g_b, err)) return rc;
      e = cudaStreamWaitEvent(st, f->ev_grav, 0);
      const double w = stage == 1 ? 1.0 : (stage == 2 ? 0.25 : 2.0 / 3.0);
      if (e == cudaSuccess)
        e = launch_grav_correct(f->arenas[f->cur], f->arenas[dst], f->nslots, f->g_a, f->g_b, f->g_stride,
                                p.dt_ptr, dt, w, st);
    }
    f->cur = dst;
    if (timed) cudaEventRecord(f->ev[2 * stage + 1], st);
  }
  if (e == cudaSuccess && out_compact && late_fix)
    e = interior_copy(f->arena(), out_compact, V, f->nslots, false, st);
  if (e != cudaSuccess) return cuda_err(err, e, "tmgpu_forest_step");
  return TMGPU_OK;
}

// The step as a CUDA graph (one GPU): captured once per distinct launch
// (arena parity, input/output buffers, dt, cfl, gamma, flags) on the forest's
// graph stream and replayed there, fenced to the caller's stream by events;
// a replay applies the host-side effects the capture recorded (f->cur,
// f->exchanges, the launch counter). Any setter that changes what a step
// enqueues drops the cached graphs (graph_reset).
int step_graph(tmgpu_forest* f, const double* in_compact, double* out_compact, double dt, double cfl,
               double gamma, int flags, cudaStream_t st, tmgpu_error* err) {
  auto bits = [](double x) {
    uint64_t u;
    std::memcpy(&u, &x, 8);
    return u;
  };
  const uint64_t key[kGraphKey] = {(uint64_t)f->cur, (uint64_t)(uintptr_t)in_compact,
                                   (uint64_t)(uintptr_t)out_compact, cfl > 0.0 ? 0 : bits(dt), bits(cfl), bits(gamma),
                                   (uint64_t)(unsigned)flags, f->forest.topology_version(),
                                   tmgpu_gravity_amr_version(f->gsolver)};
  cudaError_t e = cudaSuccess;
  if (!f->graph_stream) {
    e = cudaStreamCreateWithFlags(&f->graph_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f->gev_in, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&f->gev_out, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_err(err, e, "tmgpu_forest_step: graph stream");
  }
  StepGraph* g = nullptr;
  for (auto& x : f->graphs)
    if (std::equal(key, key + kGraphKey, x.key)) g = &x;
  if (!g) {
    ++f->graph_captures;
    const int cur0 = f->cur;
    const uint64_t ex0 = f->exchanges, l0 = g_launches.load();
    e = cudaStreamBeginCapture(f->graph_stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return cuda_err(err, e, "tmgpu_forest_step: begin capture");
    const int rc = step_enqueue(f, in_compact, out_compact, dt, cfl, gamma, flags, f->graph_stream, err);
    cudaGraph_t graph = nullptr;
    e = cudaStreamEndCapture(f->graph_stream, &graph);
    StepGraph sg{};
    std::copy(key, key + kGraphKey, sg.key);
    sg.cur_after = f->cur;
    sg.exchanges = f->exchanges - ex0;
    f->cur = cur0;  // nothing ran yet
    f->exchanges = ex0;
    g_launches.fetch_sub(g_launches.load() - l0);  // counted per replay below
    if (rc != TMGPU_OK || e != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      return rc != TMGPU_OK ? rc : cuda_err(err, e, "tmgpu_forest_step: end capture");
    }
    size_t n = 0;
    e = cudaGraphGetNodes(graph, nullptr, &n);
    std::vector<cudaGraphNode_t> nodes(n);
    if (e == cudaSuccess && n) e = cudaGraphGetNodes(graph, nodes.data(), &n);
    for (size_t q = 0; q < n && e == cudaSuccess; ++q) {
      cudaGraphNodeType t;
      e = cudaGraphNodeGetType(nodes[q], &t);
      sg.kernels += t == cudaGraphNodeTypeKernel;
    }
    // each kernel node keeps the priority of the stream it was captured from
    // (the gravity stream's high priority lets the up pass win over the early
    // mono M2L, as in the stream path)
    if (e == cudaSuccess) e = cudaGraphInstantiate(&sg.exec, graph, cudaGraphInstantiateFlagUseNodePriority);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_err(err, e, "tmgpu_forest_step: graph instantiate");
    if (f->graphs.size() >= 8) {  // bounded cache: drop the oldest
      cudaGraphExecDestroy(f->graphs.front().exec);
      f->graphs.erase(f->graphs.begin());
    }
    f->graphs.push_back(sg);
    g = &f->graphs.back();
  }
  e = cudaEventRecord(f->gev_in, st);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(f->graph_stream, f->gev_in, 0);
  if (e == cudaSuccess) e = cudaGraphLaunch(g->exec, f->graph_stream);
  if (e == cudaSuccess) e = cudaEventRecord(f->gev_out, f->graph_stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st, f->gev_out, 0);
  if (e != cudaSuccess) return cuda_err(err, e, "tmgpu_forest_step: graph launch");
  f->cur = g->cur_after;
  f->exchanges += g->exchanges;
  g_launches.fetch_add(g->kernels, std::memory_order_relaxed);
  return TMGPU_OK;
}
}  // namespace

int tmgpu_forest_step_io(tmgpu_forest* f, const double* in_compact, double* out_compact, double dt,
                         double cfl, double gamma, int flags, void* stream, double* dt_used,
                         tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (int rc = ready(f, err)) return rc;
  const int V = f->forest.config().vars;
  if (V != 5) return fail(err, TMGPU_ERR_INVALID, "the hydro step is Euler (vars 5)");
  cudaStream_t st = as_stream(stream);
  cudaError_t e = cudaSuccess;
  const int cadence = f->gsolver ? f->g_cadence : 0;
  if (cadence == 6 && (flags & TMGPU_EXACT_GHOSTS))
    return fail(err, TMGPU_ERR_INVALID, "the 6-solve gravity cadence needs the fused (ping-pong) step");
  const bool timed = f->timing;
  if (timed) {
    collect_timing(f);  // events are reused: fold the previous step in first
    cudaEventRecord(f->ev[0], st);
  }
  // CUDA graph of the step on one GPU once the kernels have run (their
  // one-time attribute setup is outside any capture): TMGPU_GRAPHS=0 disables
  static const bool graphs_env = [] {
    const char* v = std::getenv("TMGPU_GRAPHS");
    return !(v && v[0] == '0');
  }();
  // (distributed too: the peer protocols' sequence numbers live in device
  // memory and NCCL calls are captured like kernels; every rank captures the
  // same step)
  const bool use_graph = graphs_env && !(flags & TMGPU_NO_GRAPH) && f->graph_warm && f->graph_captures < 32 && !timed &&
                         (!f->gsolver || tmgpu_gravity_amr_graph_safe(f->gsolver)) &&
                         (cadence || !f->grav_stream);
  {
    const int rc = use_graph ? step_graph(f, in_compact, out_compact, dt, cfl, gamma, flags, st, err)
                             : step_enqueue(f, in_compact, out_compact, dt, cfl, gamma, flags, st, err);
    if (rc != TMGPU_OK) return rc;
  }
  f->graph_warm = true;
  if (timed) f->pending_timed = 1;
  if (flags & TMGPU_ASYNC) return TMGPU_OK;
  unsigned long long w = ~0ull;
  double dtv = dt;
  e = cudaMemcpyAsync(&w, f->err_dev, sizeof(w), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && cfl > 0.0)
    e = cudaMemcpyAsync(&dtv, f->dt_dev, sizeof(double), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_err(err, e, "tmgpu_forest_step");
  if (dt_used) *dt_used = dtv;
  if (cfl > 0.0 && !std::isfinite(dtv))
    return fail(err, TMGPU_ERR_SOLVER, "cfl_dt: no wave speed (s = 0 everywhere)");
  if (w != ~0ull) return solver_err_from_word(err, w, f->plan.loc2gl);
  return TMGPU_OK;
}

// `waiter` waits for the work enqueued so far on `signaller` (an event
// recorded and waited on; released once it completes).
int tmgpu_stream_wait(void* waiter, void* signaller) {
  cudaEvent_t ev;
  cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(ev, as_stream(signaller));
  if (e == cudaSuccess) e = cudaStreamWaitEvent(as_stream(waiter), ev, 0);
  cudaEventDestroy(ev);
  return e == cudaSuccess ? TMGPU_OK : TMGPU_ERR_CUDA;
}

// Peer-memory halo exchange (collective over the forest's communicator): every
// rank exports its slab buffer and flag words by CUDA IPC, learns where its
// slabs land in each receiver's buffer, and rewrites its cross-rank pack items
// to store there directly (halo.h PeerTab). on = 0 returns to NCCL send/recv.
// Re-call after tmgpu_forest_alloc (a new topology or distribution).
int tmgpu_forest_set_peer(tmgpu_forest* f, int on, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (f) graph_reset(f);  // what a step enqueues changes
  if (int rc = ready(f, err)) return rc;
  peer_close(f, /*collective=*/true);
  if (!on) return TMGPU_OK;
  const int world = f->world(), me = f->rank();
  if (world < 2) return fail(err, TMGPU_ERR_INVALID, "peer exchange needs a communicator with 2+ ranks");
  if (world > kMaxPeers) return fail(err, TMGPU_ERR_INVALID, "peer exchange supports up to 8 ranks");
  const HaloPlan& P = f->plan;
  // per rank: slab handle, flag handle (8 doubles each), recv_base, recv_off[world], status
  constexpr int kRec = 32, kOk = kRec - 1;
  std::vector<double> rec(kRec, 0.0), all((size_t)kRec * world, 0.0);
  double* dbuf = nullptr;
  cudaError_t e = cudaMalloc((void**)&dbuf, sizeof(double) * kRec * (world + 1));
  if (e != cudaSuccess) return cuda_err(err, e, "tmgpu_forest_set_peer");
  // every rank takes part in both all-gathers whatever fails locally, and all
  // ranks agree on the outcome (a one-sided peer mode would deadlock)
  auto agree = [&](bool ok, double* out, std::string* why) {
    rec[kOk] = ok ? 1.0 : 0.0;
    cudaError_t ce = cudaMemcpy(dbuf, rec.data(), sizeof(double) * kRec, cudaMemcpyHostToDevice);
    if (ce == cudaSuccess) ce = cudaDeviceSynchronize();
    int rc = ce == cudaSuccess ? comm_allgather(f->comm, dbuf, dbuf + kRec, kRec, nullptr, why) : TMGPU_ERR_CUDA;
    if (rc == TMGPU_OK)
      ce = cudaMemcpy(out, dbuf + kRec, sizeof(double) * kRec * world, cudaMemcpyDeviceToHost);
    if (rc != TMGPU_OK || ce != cudaSuccess) return false;
    for (int q = 0; q < world; ++q)
      if (out[(size_t)q * kRec + kOk] != 1.0) return false;
    return true;
  };
  // flag words [0, 3w] (PeerTab::mine) and this rank's sequence counter at [3w + 1]
  e = cudaMalloc((void**)&f->peer_flags, (3 * world + 2) * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(f->peer_flags, 0, (3 * world + 2) * sizeof(unsigned long long));
  cudaIpcMemHandle_t hs{}, hf{};
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&hs, f->slabs);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&hf, f->peer_flags);
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  std::memcpy(&rec[0], &hs, 64);
  std::memcpy(&rec[8], &hf, 64);
  rec[16] = (double)P.recv_base;
  for (int p = 0; p < world; ++p) rec[17 + p] = (double)P.recv_off[p];
  std::string why = "peer exchange: setup failed on a rank";
  bool ok = agree(e == cudaSuccess, all.data(), &why);
  PeerTab t{};
  t.spin_ns = peer_spin_ns();
  t.mine = f->peer_flags;
  t.seqp = f->peer_flags + 3 * world + 1;
  t.me = me;
  t.world = world;
  for (int q = 0; q < world && ok && e == cudaSuccess; ++q) {
    if (q == me) continue;
    if (P.recv_cnt[q] > 0) t.recv_mask |= 1u << q;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, &all[(size_t)q * kRec], 64);
    e = cudaIpcOpenMemHandle(&f->peer_opened[2 * q], h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) break;
    std::memcpy(&h, &all[(size_t)q * kRec + 8], 64);
    e = cudaIpcOpenMemHandle(&f->peer_opened[2 * q + 1], h, cudaIpcMemLazyEnablePeerAccess);
    t.slabs[q] = static_cast<double*>(f->peer_opened[2 * q]);
    t.flags[q] = static_cast<unsigned long long*>(f->peer_opened[2 * q + 1]);
  }
  if (ok) {
    // cross-rank items: local prolonged first, then by destination rank; the
    // offset becomes the receiver's (recv_base + recv_off[me] + position)
    std::vector<PackItem> items;
    items.reserve(P.pack.size());
    for (const PackItem& it : P.pack)
      if (it.out < P.send_base) items.push_back(it);
    for (int q = 0; q < world; ++q) {
      if (q == me) continue;
      const long long lo = P.send_base + P.send_off[q], hi = lo + P.send_cnt[q];
      const long long dst = (long long)all[(size_t)q * kRec + 16] + (long long)all[(size_t)q * kRec + 17 + me];
      for (PackItem it : P.pack)
        if (it.out >= lo && it.out < hi) {
          it.out = (int32_t)(dst + (it.out - lo));
          it.pad[0] = (int8_t)(q + 1);
          items.push_back(it);
          t.n_send[q] += 1;
        }
    }
    if (e == cudaSuccess && items.size() != P.pack.size()) e = cudaErrorInvalidValue;
    std::vector<int> pulls = P.pull_fused_local;
    pulls.insert(pulls.end(), P.pull_fused_remote.begin(), P.pull_fused_remote.end());
    e = upload(&f->pack_peer, items, e);
    e = upload((int**)&f->pull_peer, pulls, e);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    // every rank has zeroed its flags and mapped its peers before anyone signals
    std::vector<double> all2((size_t)kRec * world);
    ok = agree(e == cudaSuccess, all2.data(), &why);
  }
  cudaFree(dbuf);
  if (!ok) {
    peer_close(f);
    return e != cudaSuccess ? cuda_err(err, e, "tmgpu_forest_set_peer") : fail(err, TMGPU_ERR_CUDA, why);
  }
  f->ptab = t;
  f->peer = true;
  f->peer_version = f->forest.topology_version();
  return TMGPU_OK;
}

// The stream later steps' gravity is computed on (nullptr: same stream as the
// step): the step overlaps its CFL reduction and first exchange with it.
int tmgpu_forest_set_gravity_stream(tmgpu_forest* f, void* stream, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (f) graph_reset(f);  // what a step enqueues changes
  if (!f) return fail(err, TMGPU_ERR_INVALID, "null forest");
  if (!f->ev_grav) {
    cudaError_t e = cudaEventCreateWithFlags(&f->ev_grav, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_err(err, e, "tmgpu_forest_set_gravity_stream");
  }
  f->grav_stream = static_cast<cudaStream_t>(stream);
  return TMGPU_OK;
}

// Reflux at refinement jumps in every subsequent step (our restatement of
// SPEC.md:383-391 / flux_register.hpp; single GPU). on = 0 turns it off.
int tmgpu_forest_set_reflux(tmgpu_forest* f, int on, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (f) graph_reset(f);  // what a step enqueues changes
  if (int rc = ready(f, err)) return rc;
  auto drop = [](int*& p) {
    if (p) cudaFree(p);
    p = nullptr;
  };
  drop(f->rf_leaf), drop(f->rf_off), drop(f->rf_ad), drop(f->rf_fine);
  for (void* q : {(void*)f->flux, (void*)f->rf_send_items, (void*)f->rf_sbuf, (void*)f->rf_rbuf})
    if (q) cudaFree(q);
  f->flux = nullptr;
  f->rf_send_items = nullptr;
  f->rf_sbuf = f->rf_rbuf = nullptr;
  f->rf_nsend = f->rf_nrecv = 0;
  f->reflux = false;
  f->rf_n = 0;
  if (!on) return TMGPU_OK;
  const int V = f->forest.config().vars;
  const int world = f->world(), me = f->rank();
  // canonical leaf -> owner and local slot (owned ranges are contiguous)
  const auto& leaves = f->forest.leaves();
  std::vector<int> owner(leaves.size(), 0), local(leaves.size(), -1);
  if (world > 1) owner = f->owner;
  {
    int next = 0;
    for (size_t g = 0; g < leaves.size(); ++g)
      if (owner[g] == me) local[g] = next++;
  }
  // Coarse leaves with finer faces, in canonical order, faces (axis, dir), the
  // fine quadrants in face_neighbor order. A fine leaf on another GPU becomes
  // a received block: both sides walk this same global order, so the
  // receiver's per-peer list and the sender's per-destination list agree.
  std::vector<int> leaf, off{0}, ad, fine;
  std::vector<std::vector<int>> recv_pos(world);         // per peer: entry positions in `fine`
  std::vector<std::vector<int2>> send_items(world);      // per destination: (local slot, face)
  try {
    for (size_t s = 0; s < leaves.size(); ++s) {
      const bool mine = owner[s] == me;
      bool any = false;
      for (int axis = 0; axis < 3; ++axis)
        for (int dir : {-1, +1}) {
          const FaceNeighbors fn = f->forest.face_neighbor(leaves[s], axis, dir);
          if (fn.kind != NeighborKind::finer) continue;
          const int side_f = dir > 0 ? 0 : 1;  // the fine leaves' face toward the coarse leaf
          if (mine) {
            any = true;
            ad.push_back(axis);
            ad.push_back(dir);
          }
          for (int q = 0; q < 4; ++q) {
            const int fs = (int)f->forest.slot_of(fn.ids[q]);
            if (mine) {
              if (owner[fs] == me) {
                fine.push_back(local[fs]);
              } else {
                recv_pos[owner[fs]].push_back((int)fine.size());
                fine.push_back(0);  // patched below to -(1 + received entry)
              }
            } else if (owner[fs] == me) {
              send_items[owner[s]].push_back(make_int2(local[fs], 2 * axis + side_f));
            }
          }
        }
      if (any) {
        leaf.push_back(local[s]);
        off.push_back((int)(ad.size() / 2));
      }
    }
  } catch (const std::exception& ex) {
    return fail(err, TMGPU_ERR_INVALID, ex.what());
  }
  std::vector<int2> sitems;
  f->rf_send_off.assign(world, 0), f->rf_send_cnt.assign(world, 0);
  f->rf_recv_off.assign(world, 0), f->rf_recv_cnt.assign(world, 0);
  long long nr = 0;
  for (int q = 0; q < world; ++q) {
    f->rf_recv_off[q] = nr * V * 64;
    for (int pos : recv_pos[q]) fine[pos] = -(int)(1 + nr++);
    f->rf_recv_cnt[q] = (long long)recv_pos[q].size() * V * 64;
    f->rf_send_off[q] = (long long)sitems.size() * V * 64;
    sitems.insert(sitems.end(), send_items[q].begin(), send_items[q].end());
    f->rf_send_cnt[q] = (long long)send_items[q].size() * V * 64;
  }
  f->rf_nsend = (long long)sitems.size();
  f->rf_nrecv = nr;
  auto up = [](const std::vector<int>& v, int** out) {
    cudaError_t e = cudaMalloc(out, (v.empty() ? 1 : v.size()) * sizeof(int));
    if (e == cudaSuccess && !v.empty())
      e = cudaMemcpy(*out, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice);
    return e;
  };
  cudaError_t e = up(leaf, &f->rf_leaf);
  if (e == cudaSuccess) e = up(off, &f->rf_off);
  if (e == cudaSuccess) e = up(ad, &f->rf_ad);
  if (e == cudaSuccess) e = up(fine, &f->rf_fine);
  if (e == cudaSuccess) e = cudaMalloc(&f->flux, (size_t)f->nslots * 6 * V * 64 * sizeof(double));
  if (e == cudaSuccess) e = cudaMemset(f->flux, 0, (size_t)f->nslots * 6 * V * 64 * sizeof(double));
  if (e == cudaSuccess && f->rf_nsend) {
    e = cudaMalloc(&f->rf_send_items, sitems.size() * sizeof(int2));
    if (e == cudaSuccess)
      e = cudaMemcpy(f->rf_send_items, sitems.data(), sitems.size() * sizeof(int2), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&f->rf_sbuf, (size_t)f->rf_nsend * V * 64 * sizeof(double));
  }
  if (e == cudaSuccess && f->rf_nrecv) e = cudaMalloc(&f->rf_rbuf, (size_t)f->rf_nrecv * V * 64 * sizeof(double));
  if (e != cudaSuccess) return cuda_err(err, e, "tmgpu_forest_set_reflux");
  f->rf_n = (long long)leaf.size();
  f->reflux = true;
  f->reflux_version = f->forest.topology_version();
  return TMGPU_OK;
}

// Per-phase device timing of subsequent steps (CUDA events on the step's
// stream): accumulated milliseconds for the CFL reduction, the ghost
// exchanges and the stage kernels.
int tmgpu_forest_set_timing(tmgpu_forest* f, int on, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (f) graph_reset(f);  // what a step enqueues changes
  if (on && !f->ev[0])
    for (auto& e : f->ev) cudaEventCreate(&e);
  f->timing = on != 0;
  f->t_cfl = f->t_exchange = f->t_stage = 0;
  f->timed_steps = f->pending_timed = 0;
  return TMGPU_OK;
}

int tmgpu_forest_timing(tmgpu_forest* f, double* ms_cfl, double* ms_exchange, double* ms_stage,
                        long long* steps) {
  collect_timing(f);
  *ms_cfl = f->t_cfl;
  *ms_exchange = f->t_exchange;
  *ms_stage = f->t_stage;
  *steps = f->timed_steps;
  return TMGPU_OK;
}

// Errors latched by TMGPU_ASYNC steps since the last check (synchronises).
int tmgpu_forest_check(tmgpu_forest* f, void* stream, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (int rc = ready(f, err)) return rc;
  cudaStream_t st = as_stream(stream);
  unsigned long long w = ~0ull;
  cudaError_t e = cudaMemcpyAsync(&w, f->err_dev, sizeof(w), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(f->err_dev, 0xff, sizeof(w), st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_err(err, e, "tmgpu_forest_check");
  if (w != ~0ull) return solver_err_from_word(err, w, f->plan.loc2gl);
  return TMGPU_OK;
}

int tmgpu_forest_floor_hits(tmgpu_forest* f, double* per_leaf_host, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (int rc = ready(f, err)) return rc;
  return cuda_err(err, cudaMemcpy(per_leaf_host, f->diag, f->nslots * sizeof(double), cudaMemcpyDeviceToHost),
                  "tmgpu_forest_floor_hits");
}

// ------------------------------------------------------------- indexing
int tmgpu_morton_encode(int level, uint64_t i, uint64_t j, uint64_t k, uint64_t* index,
                        tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  try {
    *index = morton_encode(level, i, j, k);
    return TMGPU_OK;
  } catch (const std::exception& ex) {
    return fail(err, TMGPU_ERR_AMR, ex.what());
  }
}

int tmgpu_morton_decode(int level, uint64_t index, uint64_t* ijk, tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  try {
    morton_decode(level, index, ijk[0], ijk[1], ijk[2]);
    return TMGPU_OK;
  } catch (const std::exception& ex) {
    return fail(err, TMGPU_ERR_AMR, ex.what());
  }
}

uint64_t tmgpu_morton_dfs_rank(int level, uint64_t index) { return morton_dfs_rank(level, index); }

int tmgpu_partition_leaves(const uint64_t* weights, size_t n, int localities, int* owner,
                           tmgpu_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  try {
    auto o = partition_leaves(std::vector<uint64_t>(weights, weights + n), localities);
    std::memcpy(owner, o.data(), o.size() * sizeof(int));
    return TMGPU_OK;
  } catch (const std::exception& ex) {
    return fail(err, TMGPU_ERR_AMR, ex.what());
  }
}

}  // extern "C"
