/* tmgpu — B200-native (sm_100a, FP64) per-subgrid hot path behind the
 * reference mini-app's subgrid-kernel API (taskmesh, arXiv 2412.15518).
 *
 * C ABI: plain pointers and sizes, no torch/CUDA types in the signatures
 * (streams are passed as void* = cudaStream_t). Every entry point names the
 * reference interface it replaces (paths relative to /root/reference/proj).
 * All functions are thread-safe; the stage entry points may be called
 * concurrently from several scheduler workers (reference aggregator.cpp:147-157).
 *
 * Return value: TMGPU_OK (0) or a negative/positive error code; details in
 * the optional tmgpu_error record.
 */
#ifndef TMGPU_H
#define TMGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- errors */
enum {
  TMGPU_OK = 0,
  TMGPU_ERR_SOLVER = 1,      /* non-finite state (reference hydro::SolverError, stage.cpp:209-216) */
  TMGPU_ERR_INVALID = 2,     /* bad argument / unsupported geometry */
  TMGPU_ERR_CUDA = 3,        /* CUDA runtime failure (message holds cudaGetErrorString) */
  TMGPU_ERR_AMR = 4,         /* reference amr::AmrError analog (morton/partition/tree) */
  TMGPU_ERR_AGG = 5          /* reference agg::AggError analog (aggregator.cpp) */
};

typedef struct tmgpu_error {
  int code;
  int cell[3];               /* solver errors: interior cell (i,j,k) of the first bad value */
  int64_t slice;             /* solver errors: first failing slice (launch order) */
  char message[256];         /* solver errors carry the reference's exact text */
} tmgpu_error;

/* ---------------------------------------------------------------- flags */
#define TMGPU_HOST_PTRS 0x1  /* in/out are host memory: H2D, kernel, D2H inside the call */
#define TMGPU_FAST 0x2       /* FMA/reciprocal arithmetic: parity within 1e-10 (scaled), not bitwise */
#define TMGPU_ASYNC 0x4      /* enqueue only; errors latched until tmgpu_forest_check */
#define TMGPU_EXACT_GHOSTS 0x8 /* step: reference 3-pass full-shell exchange instead of one-round faces */
#define TMGPU_OVERLAP 0x10   /* multi-GPU step: overlap the NCCL halo with the interior leaves' stage */
#define TMGPU_NO_GRAPH 0x20  /* step: enqueue directly (one GPU replays the step as a cached CUDA graph) */
#define TMGPU_GRAV_AM 0x100  /* gravity: angular-momentum correction (rigid-rotation field) */

/* ---------------------------------------------------------------- hydro
 * Slice contract (reference stage.hpp:8-12, 39-66):
 *   in  slice = [8-double header | vars * S^3 ghosted state], S = edge + 2*ghost
 *   out slice = [vars*E^3 interior | 6 face-flux blocks of vars*E^2 | 1 floor-hit count]
 * Header = [mode (0 scalar, else Euler), dx, dt, gamma, ax, ay, az, 0]
 *   (reference stage.cpp:10-29 encode_header/decode_header).
 */
size_t tmgpu_in_slice(int edge, int ghost, int vars);   /* StageGeom::in_slice  stage.hpp:54 */
size_t tmgpu_out_slice(int edge, int ghost, int vars);  /* StageGeom::out_slice stage.hpp:65 */

/* Replaces the body of hydro::make_stage_kernel's KernelFn
 * (reference src/hydro/stage.cpp:229-246; KernelFn type aggregator.hpp:96-99):
 * one fused launch over `count` slices packed at in + s*in_slice /
 * out + s*out_slice. Bitwise equal to the reference unless TMGPU_FAST.
 * Device pointers (default) run on `stream` (NULL = per-thread default) and
 * the call returns after the stream reaches the end of the launch; with
 * TMGPU_HOST_PTRS the call stages through device memory itself.
 * Supported geometry: edge 8, ghost 2, vars 1 (scalar) or 5 (Euler or scalar). */
int tmgpu_stage_fused(const double* in, double* out, size_t in_slice, size_t out_slice,
                      size_t count, int edge, int ghost, int vars, int flags,
                      void* stream, tmgpu_error* err);

/* Replaces hydro::stage_subgrid (reference stage.hpp:68-71, stage.cpp:222-227)
 * for one sub-grid: header8 + ghosted state -> out slice. lane_width is
 * accepted for API parity and ignored (output is W-invariant, stage.hpp:69). */
int tmgpu_stage_subgrid(const double* header8, int edge, int ghost, int vars,
                        unsigned lane_width, const double* in_ghosted, double* out,
                        int flags, void* stream, tmgpu_error* err);

/* Replaces hydro::max_wavespeed (reference stage.cpp:248-272) over `count`
 * slices (same slice layout as tmgpu_stage_fused); result[s] per slice. */
int tmgpu_max_wavespeed(const double* in, size_t in_slice, size_t count, int edge, int ghost,
                        int vars, double* result, int flags, void* stream, tmgpu_error* err);

/* hydro::rk3_combine (reference include/taskmesh/hydro/rk3.hpp:18-34) on n values. */
int tmgpu_rk3_combine(int stage, const double* u0, const double* v, double* out, size_t n,
                      int flags, void* stream, tmgpu_error* err);

/* ---------------------------------------------------------------- indexing
 * Bit-exact with the reference (tests/test_forest.py). */
/* amr::morton_encode / morton_decode / morton_dfs_rank (amr/morton.hpp:32-66);
 * out-of-range arguments return TMGPU_ERR_AMR (the reference throws AmrError). */
int tmgpu_morton_encode(int level, uint64_t i, uint64_t j, uint64_t k, uint64_t* index,
                        tmgpu_error* err);
int tmgpu_morton_decode(int level, uint64_t index, uint64_t* ijk, tmgpu_error* err);
uint64_t tmgpu_morton_dfs_rank(int level, uint64_t index);
/* amr::partition_leaves (src/amr/octree.cpp:374-399) */
int tmgpu_partition_leaves(const uint64_t* weights, size_t n, int localities, int* owner,
                           tmgpu_error* err);

/* ---------------------------------------------------------------- forest
 * Octree topology (amr::Tree, amr/octree.hpp:241-314) with the leaf state
 * held in a device arena [slot][vars][S^3] indexed by canonical leaf order.
 * Node ids are NodeId::packed() (octree.hpp:29-33); bc[a]: 0 periodic,
 * 1 reflective. */
typedef struct tmgpu_forest tmgpu_forest;
typedef struct tmgpu_gravity_amr tmgpu_gravity_amr; /* gravity section below */
tmgpu_forest* tmgpu_forest_create(int edge, int ghost, int vars, int max_level,
                                  const int* root_dims, const int* bc, tmgpu_error* err);
void tmgpu_forest_destroy(tmgpu_forest* f);
int tmgpu_forest_refine(tmgpu_forest* f, uint64_t packed, tmgpu_error* err);  /* Tree::refine octree.cpp:200-234 */
int tmgpu_forest_coarsen(tmgpu_forest* f, uint64_t packed, tmgpu_error* err); /* Tree::coarsen octree.cpp:236-293 */
size_t tmgpu_forest_leaves(tmgpu_forest* f, uint64_t* out, size_t cap);     /* Tree::leaves octree.cpp:52-77 */
int tmgpu_forest_is_leaf(tmgpu_forest* f, uint64_t packed);                   /* Node::is_leaf octree.hpp:77 */
/* Tree::face_neighbor (octree.cpp:92-132): returns kind 0 same, 1 coarser, 2 finer, 3 boundary */
int tmgpu_forest_face_neighbor(tmgpu_forest* f, uint64_t leaf, int axis, int dir, uint64_t* ids4,
                               int* count);
/* ghost::plan_axis_fills (ghost.cpp:168-210): rows of 7 int64 (dst, src|-1, kind, axis, dir, qt1, qt2) */
size_t tmgpu_forest_plan(tmgpu_forest* f, int axis, int64_t* rows, size_t cap);
int tmgpu_forest_balanced(tmgpu_forest* f);                                   /* Tree::is_balanced */
double tmgpu_forest_cell_size(tmgpu_forest* f, int level);                    /* Tree::cell_size */
uint64_t tmgpu_forest_topology_version(tmgpu_forest* f);
uint64_t tmgpu_forest_exchanges(tmgpu_forest* f);
/* synthetic scenarios: kind 0 rotating star, 1 double white dwarf, 2 Sod, 3 Sedov */
int tmgpu_forest_scenario_refine(tmgpu_forest* f, int kind, int min_level, int max_level,
                                 double theta, tmgpu_error* err);
int tmgpu_forest_scenario_fill(tmgpu_forest* f, int kind, uint64_t seed, double* compact_host,
                               tmgpu_error* err);
/* ---- distribution over GPUs (one process per GPU, NCCL over NVLink) */
typedef struct tmgpu_comm tmgpu_comm;
int tmgpu_comm_unique_id(unsigned char* id128, tmgpu_error* err);      /* ncclGetUniqueId (rank 0) */
tmgpu_comm* tmgpu_comm_create(int rank, int world, const unsigned char* id128, tmgpu_error* err);
void tmgpu_comm_destroy(tmgpu_comm* c);
/* owner[g] per canonical leaf (partition_leaves; Node::owner octree.hpp:74); call alloc after */
int tmgpu_forest_distribute(tmgpu_forest* f, tmgpu_comm* comm, const int* owner, size_t n,
                            tmgpu_error* err);
/* owned leaves in canonical order (= local slot order of the arena and the compact arrays) */
size_t tmgpu_forest_local_leaves(tmgpu_forest* f, uint64_t* out, size_t cap);
/* host-only halo manifest of (owner, rank): rows (send 0|recv 1, peer, dst, src, kind, axis, dir) */
size_t tmgpu_forest_halo_manifest(tmgpu_forest* f, const int* owner, int rank, int world,
                                  int64_t* rows, size_t cap);
/* (re)allocate the zeroed device arena + ghost plans for the current topology */
int tmgpu_forest_alloc(tmgpu_forest* f, tmgpu_error* err);
double* tmgpu_forest_arena(tmgpu_forest* f);
/* compact interior [slot][vars][E^3] <-> arena (SubGrid::copy_interior_in/out, subgrid.hpp:63-76) */
int tmgpu_forest_interior(tmgpu_forest* f, double* compact, int to_device, int flags, void* stream,
                          tmgpu_error* err);
/* whole ghosted arena <-> host [slot][vars][S^3] (SubGrid::raw, subgrid.hpp:59-60) */
int tmgpu_forest_grids(tmgpu_forest* f, double* ghosted_host, int to_device, tmgpu_error* err);
/* either arena by role (0 = current state, 1 = the other ping-pong arena), whole ghosted
 * blocks <-> host [slot][vars][S^3]: a resumable checkpoint holds both (the step carries their
 * ghost layers across exchanges) */
int tmgpu_forest_arena_grids(tmgpu_forest* f, int which, double* ghosted_host, int to_device,
                             tmgpu_error* err);
/* ghost::fill_ghosts_sync (ghost.cpp:282-296), bitwise on the full ghosted arrays */
/* AMR regrid with the device data (octree.cpp:149-293 prolong_cell / restrict_cells, same
 * order incl. cascaded 2:1 refines): refine then coarsen the listed nodes; single GPU */
int tmgpu_forest_regrid(tmgpu_forest* f, const uint64_t* refine, size_t nr, const uint64_t* coarsen,
                        size_t nc, tmgpu_error* err);
/* Tree::flag_refinement (octree.cpp:295-323) per local leaf on the device state: flags[slot] */
int tmgpu_forest_flag(tmgpu_forest* f, double theta, double rho_floor, int* flags_host,
                      tmgpu_error* err);
int tmgpu_forest_fill_ghosts(tmgpu_forest* f, void* stream, tmgpu_error* err);
/* one-round face-only exchange: every ghost the stage reads, bitwise equal to
 * fill_ghosts_sync; edge/corner ghosts are left untouched */
int tmgpu_forest_fill_faces(tmgpu_forest* f, void* stream, tmgpu_error* err);
/* hydro::max_wavespeed per leaf (stage.cpp:248-272) */
int tmgpu_forest_max_wavespeed(tmgpu_forest* f, double gamma, double* per_leaf_host, tmgpu_error* err);
/* SSP-RK3 step (rk3.hpp): 3 x (fill_ghosts_sync -> aggregated
 * stage over all leaves -> rk3_combine); cfl > 0 computes dt on the device */
/* reflux at refinement jumps in every subsequent step (flux_register.hpp:21-63 declared,
 * SPEC.md:383-391 formula; our restatement, oracle tmo_reflux_apply): the coarse cell
 * next to a finer face += -dir * (stage weight * dt / dx) * (mean of the 2x2 fine face
 * fluxes - coarse face flux), after each stage's RK combine; single GPU; re-call after a
 * topology change. on = 0 turns it off. */
int tmgpu_forest_set_reflux(tmgpu_forest* f, int on, tmgpu_error* err);
/* gravity source in the stage (our spec): g device [3][comp_stride] by
 * local slot; NULL = pure hydro (the reference's stage) */
int tmgpu_forest_set_gravity(tmgpu_forest* f, const double* g, long long comp_stride,
                             tmgpu_error* err);
/* self-gravity solved inside the step by the adaptive FMM G (created on this forest's leaves,
 * distributed like it): solves_per_step 1 = once on the step's initial state, held over the three
 * RK stages; 3 = before every RK stage on that stage's input state (the paper's hydro coupling,
 * PAPER.md:240); 6 = the paper's count: per stage a second solve on the stage's
 * provisional density moves the source to the trapezoid of the two fields (grav_source.cu; not
 * with TMGPU_EXACT_GHOSTS). grav_flags: TMGPU_GRAV_AM. phi [n*512], g and g2 [3][comp_stride]
 * (g2 and rho_tilde [n*512] only for 6) are device buffers by local slot the caller keeps alive;
 * g holds the last stage-input field. Solves run on the gravity stream when one is set (each
 * overlapping that stage's ghost exchange). G NULL turns it off. */
int tmgpu_forest_set_gravity_solver(tmgpu_forest* f, tmgpu_gravity_amr* G, int solves_per_step,
                                    int grav_flags, double* phi, double* g, double* g2,
                                    double* rho_tilde, long long comp_stride, tmgpu_error* err);
/* the stream the next steps' gravity is computed on (NULL: the step's stream): the step runs its
 * CFL reduction and first ghost exchange concurrently and waits for that stream's work (enqueued
 * before the step call) only before the first stage kernel */
int tmgpu_forest_set_gravity_stream(tmgpu_forest* f, void* stream, tmgpu_error* err);
/* multi-GPU ghost exchange over peer memory instead of NCCL send/recv (collective over the
 * forest's communicator; 2..8 ranks on one node with CUDA IPC): each rank packs its cross-GPU
 * slabs straight into the receivers' buffers and synchronises by flag words (a wait that does
 * not complete within 20 s traps). Re-call after tmgpu_forest_alloc; on = 0 returns to NCCL.
 * No reference counterpart (the reference moves ghosts through HPX channels). */
int tmgpu_forest_set_peer(tmgpu_forest* f, int on, tmgpu_error* err);
/* `waiter` waits for the work enqueued so far on `signaller` (CUDA streams; NULL = default) */
int tmgpu_stream_wait(void* waiter, void* signaller);
int tmgpu_forest_step(tmgpu_forest* f, double dt, double cfl, double gamma, int flags,
                      void* stream, double* dt_used, tmgpu_error* err);
/* the step with its input and output as compact interiors [slot][vars][E^3] in device memory
 * (either may be NULL): the input is scattered into the arena by the step's first pass (fused
 * with the CFL wave speeds when cfl > 0; stage 1's gravity masses read it directly) and the
 * output written by the last stage's epilogue (a separate gather with reflux or the 6-solve
 * cadence, whose corrections follow that stage) — the end-to-end path's copies without
 * separate scatter/gather passes. Equal to set_interior + step + get_interior, bit for bit. */
int tmgpu_forest_step_io(tmgpu_forest* f, const double* in_compact, double* out_compact, double dt,
                         double cfl, double gamma, int flags, void* stream, double* dt_used,
                         tmgpu_error* err);
int tmgpu_forest_check(tmgpu_forest* f, void* stream, tmgpu_error* err);
/* per-phase device timing (CUDA events) of subsequent steps: accumulated ms */
int tmgpu_forest_set_timing(tmgpu_forest* f, int on, tmgpu_error* err);
int tmgpu_forest_timing(tmgpu_forest* f, double* ms_cfl, double* ms_exchange, double* ms_stage,
                        long long* steps);
int tmgpu_forest_floor_hits(tmgpu_forest* f, double* per_leaf_host, tmgpu_error* err);

/* ---------------------------------------------------------------- aggregation executor
 * agg::ExecutorPool / agg::AggregationRegion (include/taskmesh/aggregator.hpp:57-172,
 * src/aggregator.cpp) with CUDA streams as executors. Pool bookkeeping is host-only
 * (no CUDA until the first launch). */
typedef struct tmgpu_execpool tmgpu_execpool;
typedef struct tmgpu_region tmgpu_region;
tmgpu_execpool* tmgpu_execpool_create(size_t count, tmgpu_error* err);   /* ExecutorPool(count) */
void tmgpu_execpool_destroy(tmgpu_execpool* p);
size_t tmgpu_execpool_size(tmgpu_execpool* p);
size_t tmgpu_execpool_acquire(tmgpu_execpool* p);                        /* acquire() -> lease index */
size_t tmgpu_execpool_pick_index(tmgpu_execpool* p);                     /* pick_index() */
int tmgpu_execpool_acquire_at(tmgpu_execpool* p, size_t index, tmgpu_error* err); /* acquire_at */
void tmgpu_execpool_release(tmgpu_execpool* p, size_t index);            /* ExecutorLease::reset */
uint64_t tmgpu_execpool_in_flight(tmgpu_execpool* p, size_t index);
/* kind 1: the hydro stage (make_stage_kernel, stage.cpp:229-246; slice sizes from the
 * geometry); other kinds are rejected (use tmgpu_region_create_kernel).
 * counters: optional uint64[3] {launches, fused_slices, solo_launches}. */
tmgpu_region* tmgpu_region_create(tmgpu_execpool* pool, int kind, size_t in_slice,
                                  size_t out_slice, int edge, int ghost, int vars, int flags,
                                  size_t max_slices, size_t capacity, uint64_t* counters,
                                  tmgpu_error* err);
/* A device kernel registered like a reference KernelSpec (aggregator.hpp:94-106): launch one
 * aggregated kernel over `count` packed DEVICE slices at in + s*in_slice on `stream`; return 0
 * or non-zero (the whole batch fails, aggregator.cpp:164-167). */
typedef int (*tmgpu_device_kernel)(const double* in, double* out, size_t in_slice, size_t out_slice,
                                   size_t count, void* stream, void* user);
tmgpu_region* tmgpu_region_create_kernel(tmgpu_execpool* pool, tmgpu_device_kernel fn, void* user,
                                         size_t in_slice, size_t out_slice, size_t max_slices,
                                         size_t capacity, uint64_t* counters, tmgpu_error* err);
long long tmgpu_region_submit(tmgpu_region* r, const double* input, size_t len,
                              tmgpu_error* err);                          /* submit_slice */
int tmgpu_region_flush(tmgpu_region* r, tmgpu_error* err);              /* flush */
int tmgpu_region_wait(tmgpu_region* r, long long ticket, tmgpu_error* err); /* Future::get */
const double* tmgpu_region_output(tmgpu_region* r, long long ticket);   /* SliceOutput::values */
size_t tmgpu_region_submitted(tmgpu_region* r);                           /* submitted() */
void tmgpu_region_destroy(tmgpu_region* r);

/* ---------------------------------------------------------------- gravity (FMM)
 * No reference implementation exists: our cell-level FMM,
 * restated bitwise in oracle/gravity_oracle.c. Uniform cell level D (N = 2^D per
 * axis, unit box, isolated boundaries, G = 1); outputs phi[N^3], g[3][N^3] in
 * (k,j,i) order. */
typedef struct tmgpu_gravity tmgpu_gravity;
tmgpu_gravity* tmgpu_gravity_create(int D, tmgpu_error* err);
void tmgpu_gravity_destroy(tmgpu_gravity* g);
int tmgpu_gravity_solve(tmgpu_gravity* G, const double* mass, double* phi, double* g, int flags,
                        void* stream, tmgpu_error* err);
int tmgpu_gravity_mass_from_arena(tmgpu_gravity* G, const double* arena, const int* leaf_ijk_dev,
                                  long long nleaves, int vars, double dV, void* stream,
                                  tmgpu_error* err);

/* AMR forest (oracle/gravity_amr_oracle.c): adaptive FMM over the cell tree of
 * the leaves (U, V, W, X lists). leaves: host [n][4] = (level, I, J, K) in
 * canonical slot order, one root = the unit cube. mass: [n][512] ((k,j,i) per
 * leaf) or NULL for the workspace masses (tmgpu_gravity_amr_mass_from_arena);
 * outputs phi[n*512], g[3][n*512] by slot. flags: TMGPU_HOST_PTRS, TMGPU_ASYNC,
 * TMGPU_GRAV_AM. info: [0] levels, [1] nodes, [2] W/X pairs, [3] U-cross pairs. */
tmgpu_gravity_amr* tmgpu_gravity_amr_create(const int* leaves, long long nleaves, tmgpu_error* err);
void tmgpu_gravity_amr_destroy(tmgpu_gravity_amr* G);
int tmgpu_gravity_amr_info(const tmgpu_gravity_amr* G, long long* out);
int tmgpu_gravity_amr_plan_info(const int* leaves, long long nleaves, long long* out,
                                tmgpu_error* err); /* host only: plan validation + info */
int tmgpu_gravity_amr_mass_from_arena(tmgpu_gravity_amr* G, const double* arena, int vars,
                                      void* stream, tmgpu_error* err);
/* masses from a device density [n][512] by local slot (m = rho * h^3, as mass_from_arena) */
int tmgpu_gravity_amr_mass_from_density(tmgpu_gravity_amr* G, const double* rho, void* stream,
                                        tmgpu_error* err);
/* the same from a density at slot stride `slot_stride` doubles (>= 512), e.g. var 0 of compact
 * interiors [n][vars][512] (slot_stride = vars * 512) */
int tmgpu_gravity_amr_mass_from_compact(tmgpu_gravity_amr* G, const double* rho, long long slot_stride,
                                        void* stream, tmgpu_error* err);
int tmgpu_gravity_amr_solve(tmgpu_gravity_amr* G, const double* mass, double* phi, double* g,
                            int flags, void* stream, tmgpu_error* err);
int tmgpu_gravity_amr_am_stats(tmgpu_gravity_amr* G, double* out);
/* algorithmic work of one solve (bench roofline), out[15]: [V pairs, W/X entries,
 * same-depth P2P pairs, cross-depth U entries, V pairs evaluated, V pairs into
 * leaf patches, W/X entries into leaf patches] (leaf targets need only L0, L_i), then
 * V pairs and W/X entries by (target, source) kind: [7..10] V (leaf<-leaf,
 * leaf<-internal, internal<-leaf, internal<-internal), [11..14] W/X likewise (a leaf
 * source's D and Q are zero: its term is the monopole one), [15] V pairs of the patches the
 * monopole-source kernel takes (leaf patches whose neighbours are all leaves; out holds 16) */
int tmgpu_gravity_amr_work(const tmgpu_gravity_amr* G, long long* out);
/* multi-GPU (locally essential tree, multipole-moment exchange over NCCL): this rank (comm)
 * owns canonical slots [slot_bounds[r], slot_bounds[r+1]); masses and outputs become by local
 * slot; results equal the one-GPU solve bitwise */
int tmgpu_gravity_amr_distribute(tmgpu_gravity_amr* G, tmgpu_comm* comm, const long long* slot_bounds,
                                 tmgpu_error* err);
/* multi-GPU moment exchange over peer memory (collective; 2..8 ranks of one node, CUDA IPC):
 * subtree roots and halo patches are stored straight into the peers' moment arrays with
 * flag-word synchronisation (a wait that does not complete within 20 s traps) instead of the
 * NCCL all-gather + send/recv. Re-call after tmgpu_gravity_amr_distribute; on = 0 returns to NCCL. */
int tmgpu_gravity_amr_set_peer(tmgpu_gravity_amr* G, int on, tmgpu_error* err);
/* host-only: per-level counts of the patches a rank owning slots [lo, hi) evaluates
 * M2L/L2L for; returns the level count (negative error code on failure) */
int tmgpu_gravity_amr_plan_need(const int* leaves, long long nleaves, long long lo, long long hi,
                                long long* counts, int max_levels, tmgpu_error* err);
/* host-only: the multipole-moment exchange (LET) plan of rank `me`: out[4] = owned internal
 * patches, shared top patches, own subtree roots, halo leaf patches; per peer q the send /
 * receive patch counts and list hashes (rank r's send list to q == q's receive list from r) */
int tmgpu_gravity_amr_let_plan(const int* leaves, long long nleaves, const long long* bounds, int world,
                               int me, long long* out, long long* send, long long* recv,
                               long long* send_hash, long long* recv_hash, tmgpu_error* err);
/* per-phase device timing: totals in ms of [up (P2M + owned-subtree M2M), let (subtree-root
 * all-gather, shared-top M2M, halo-moment exchange; the top on one GPU), m2l, l2l, l2p, am,
 * then the M2L kernels alone: mono, fused, W/X] (ms holds 9). A timed solve runs those three
 * kernels one after another on the solve's stream (untimed solves overlap them). */
int tmgpu_gravity_amr_set_timing(tmgpu_gravity_amr* G, int on);
int tmgpu_gravity_amr_timing(tmgpu_gravity_amr* G, double* ms, long long* solves);
const double* tmgpu_gravity_amr_mass_ptr(const tmgpu_gravity_amr* G);

/* ---------------------------------------------------------------- build info */
const char* tmgpu_version(void);
/* number of kernels launched by this library since load (bench/gpu_launches) */
uint64_t tmgpu_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* TMGPU_H */
