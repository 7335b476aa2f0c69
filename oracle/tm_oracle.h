/* TEST INFRASTRUCTURE ONLY — the checker, never the product.
 *
 * Plain-C restatement of the reference mini-app's per-subgrid hot path
 * (/root/reference/proj). Every function cites the reference file:line it
 * restates. Parity of this restatement is PINNED: tests/test_oracle_*.py
 * compare it bitwise against the unmodified reference compiled in place
 * (oracle/_ref/libtmref.so) and against the reference's own test vectors.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.
 */
#ifndef TM_ORACLE_H
#define TM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* hydro: stage.cpp:93-246, euler.hpp, limiter.hpp */
double tmo_minmod_scalar(double a, double b);
double tmo_minmod_lane(double a, double b);
void tmo_reconstruct_face(double um1, double u0, double up1, double up2, double* lr);
void tmo_rusanov_euler(const double* ql, const double* qr, double gamma, int axis, double* f5);
double tmo_rusanov_scalar(double a, double l, double r);
/* returns 0 ok, 1 non-finite (cell written to bad_cell[3] = i,j,k) */
int tmo_stage_subgrid(const double* header8, int edge, int ghost, int vars,
                      const double* in, double* out, int* bad_cell);
/* returns 0 ok, else 1 + index of the first failing slice in *bad_slice */
int tmo_stage_subgrid_grav(const double* h, int E, int G, int V, const double* in,
                           const double* grav, double* out, int* bad_cell);
int tmo_stage_fused(const double* in, double* out, size_t in_slice, size_t out_slice,
                    size_t count, int edge, int ghost, int vars, size_t* bad_slice,
                    int* bad_cell);
double tmo_max_wavespeed(const double* header8, int edge, int ghost, int vars,
                         const double* ghosted);
double tmo_rk3_combine(int stage, double u0, double v);

/* indexing: morton.hpp:32-66, octree.hpp:29-41, octree.cpp:374-399 */
int tmo_morton_encode(int level, uint64_t i, uint64_t j, uint64_t k, uint64_t* index);
int tmo_morton_decode(int level, uint64_t index, uint64_t* ijk);
uint64_t tmo_morton_dfs_rank(int level, uint64_t index);
int tmo_partition_leaves(const uint64_t* weights, size_t n, int localities, int* owner);

/* tree restated over a leaf list: octree.cpp:52-132, ghost.cpp:168-296.
 * leaves: packed NodeIds (any order); the forest derives internal nodes. */
typedef struct tmo_tree tmo_tree;
tmo_tree* tmo_tree_create(int edge, int ghost, int vars, const int* root_dims,
                          const int* bc, const uint64_t* leaves, size_t n);
void tmo_tree_destroy(tmo_tree* t);
/* canonical leaf order (octree.cpp:52-77) */
size_t tmo_tree_leaves(const tmo_tree* t, uint64_t* out, size_t cap);
int tmo_tree_face_neighbor(const tmo_tree* t, uint64_t leaf, int axis, int dir,
                           uint64_t* ids4, int* count);
/* rows of 7 int64: dst, src(-1 boundary), kind, axis, dir, qt1, qt2 */
size_t tmo_tree_plan(const tmo_tree* t, int axis, int64_t* rows, size_t cap);
/* grids[l] = ghosted grid of canonical leaf l (vars*S^3 doubles) */
int tmo_fill_ghosts_sync(const tmo_tree* t, double** grids);
int tmo_reflux_apply(const tmo_tree* t, double** grids, double* const* faces, int E, int G, int V,
                     const double* dx, double dt, double coef);
int tmo_flag_refinement(const tmo_tree* t, const double* grid, double theta, double rho_floor);

/* gravity (our FMM specification, parity unpinned: no reference code) — gravity_oracle.c */
void tmo_grav_geom(const double* R, double* e);
void tmo_grav_m2l_geom(const double* mom, const double* e, double* out);
void tmo_grav_m2l(const double* mom, const double* R, double* out);
void tmo_grav_p2p_geom(double Rx, double Ry, double Rz, double* w);
void tmo_grav_m2m(const double* ch, const double* s, double* out);
void tmo_grav_l2l(const double* L, const double* s, double* out);
int tmo_grav_solve(int D, const double* mass, double* phi, double* g);
int tmo_grav_direct(int D, const double* mass, double* phi, double* g);
/* AMR forest (gravity_amr_oracle.c): leaves [n][4] = (level, I, J, K), mass [n][512] */
int tmo_grav_amr_solve(long nleaves, const int* leaves, const double* mass, int flags, double* phi,
                       double* g);
int tmo_grav_amr_solve_ex(long nleaves, const int* leaves, const double* mass, int flags,
                          double* phi, double* g, long* counts);
/* patch-sparse restatement (gravity_amr_sparse.c): bitwise equal to tmo_grav_amr_solve_ex,
 * any depth, OpenMP; the CPU baseline of the gravity half */
int tmo_grav_amr_sparse(long nleaves, const int* leaves, const double* mass, int flags, double* phi,
                        double* g, long* counts);
/* the same split like the GPU solver: plan (topology, lists) once, solve per mass field */
typedef struct tmo_grav_plan tmo_grav_plan;
tmo_grav_plan* tmo_grav_plan_create(long nleaves, const int* leaves, int* rc);
int tmo_grav_plan_solve(tmo_grav_plan* P, const double* mass, int flags, double* phi, double* g,
                        long* counts);
void tmo_grav_plan_destroy(tmo_grav_plan* P);
int tmo_grav_amr_direct(long nleaves, const int* leaves, const double* mass, double* phi, double* g);
void tmo_grav_am_solve(const double* S, double* R, double* w);
int tmo_grav_am_correct(long nleaves, const double* mass, const double* pos, double* g,
                        double* S_out, double* w_out);

#ifdef __cplusplus
}
#endif
#endif
