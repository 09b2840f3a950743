/*
 * oracle.h -- C ABI of the CPU ORACLE.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load liboracle.so.  The
 * product path (paper_2202_12309_b200/) never includes, links or calls this.
 * The oracle shares no source, header, table or helper with the CUDA path.
 *
 * What it computes: the per-cycle update of Parthenon-hydro (§4.1,
 * "a two-stage Runge-Kutta integrator, piecewise linear
 * reconstruction and HLLE Riemann solver") over a block-structured mesh
 * (§2.1), with ghost exchange incl. restriction/prolongation
 * (§3.7), flux correction, CFL dt reduction
 * (P:640-650), Z-order distribution and remeshing.
 * Where the paper is silent the readings of SURVEY.md §8(c) (A1-A30) are used;
 * DESIGN.md lists them.  Plain scalar loops, fp64, built -O2 -ffp-contract=off.
 */
#ifndef ORACLE_H
#define ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_ERR_INVALID_ARG = 1, ORC_ERR_CONFIG = 2, ORC_ERR_PHYSICS = 6, ORC_ERR_STATE = 7 };
enum { ORC_BC_PERIODIC = 0, ORC_BC_OUTFLOW = 1, ORC_BC_REFLECT = 2 };
enum { ORC_RECON_MINMOD = 0, ORC_RECON_VANLEER = 1, ORC_RECON_MC = 2, ORC_RECON_PPM = 3, ORC_RECON_WENOZ = 4 };
enum { ORC_INT_RK2 = 0, ORC_INT_VL2 = 1 };
enum { ORC_PROB_LINEAR_WAVE = 0, ORC_PROB_SOD = 1, ORC_PROB_BLAST = 2, ORC_PROB_KH = 3 };
enum { ORC_REF_NONE = 0, ORC_REF_STATIC = 1, ORC_REF_ADAPTIVE = 2 };
/* HLLE wave-speed estimates (A4): Davis min/max of the face states' u -+ c (default), or Einfeldt
 * (1988): the Roe-averaged speeds u~ -+ c~ also enter the min/max (S_L = min(u_L - c_L, u~ - c~),
 * S_R = max(u_R + c_R, u~ + c~)). */
enum { ORC_WS_DAVIS = 0, ORC_WS_EINFELDT = 1 };

typedef struct {
  int64_t mesh_nx[3];      /* root-grid cells per dim */
  int64_t block_nx[3];     /* cells per block per dim (must divide mesh_nx) */
  int32_t nghost;          /* 2 (PLM) or 3 (PPM, WENO-Z; uniform meshes) */
  int32_t max_level;       /* levels above root */
  double xmin[3], xmax[3];
  int32_t bc_inner[3], bc_outer[3];
  double gamma, cfl;
  int32_t recon, integrator;
  int32_t refinement;      /* ORC_REF_* */
  double refine_tol, derefine_tol;
  int32_t derefine_interval;
  int32_t nregions;        /* static regions: regions[7*r] = level, x1min,x1max,x2min,x2max,x3min,x3max */
  const double* regions;
  int32_t nranks;          /* simulated ranks: only the partition depends on it */
  int32_t nthreads;        /* OpenMP threads over blocks (0 = default) */
  int32_t wavespeed;       /* ORC_WS_* (PLM meshes; PPM / WENO-Z use Davis) */
} orc_config;

typedef struct { int64_t gid; int32_t level, rank; int64_t lx[3]; double xmin[3], xmax[3]; } orc_block;
typedef struct { int64_t gid; int32_t rank; int8_t off[3]; int8_t dlevel; int8_t fine[2]; } orc_neighbor;

typedef struct orc_mesh orc_mesh;

int orc_mesh_create(const orc_config* cfg, orc_mesh** out);
int orc_mesh_destroy(orc_mesh* m);
/* Problem generators.  LINEAR_WAVE p = {A, k1, k2, k3}; SOD p = {x_split};
 * BLAST p = {p_in, p_out, radius, cx, cy, cz}; KH p = {A, sigma} (reading A36).
 * Applies AMR pre-refinement when adaptive. */
int orc_set_problem(orc_mesh* m, int32_t problem, const double* p, int32_t np);
int orc_set_state(orc_mesh* m, int64_t gid, const double* cons, int64_t nelem); /* [5][n3][n2][n1] */
int orc_get_state(const orc_mesh* m, int64_t gid, double* cons, int64_t nelem);
/* Full array incl. ghosts, [5][n3+2g][n2+2g][n1+2g]; for exchange tests. */
int orc_get_state_full(const orc_mesh* m, int64_t gid, double* out, int64_t nelem);
int orc_set_state_full(orc_mesh* m, int64_t gid, const double* in, int64_t nelem);
int orc_exchange(orc_mesh* m);             /* ghost exchange O7 on U0 */
int orc_compute_dt(orc_mesh* m, double* dt); /* O6 on U0 (sets the mesh dt) */
int orc_step(orc_mesh* m, int32_t ncycles, double tlim);
int orc_get_time(const orc_mesh* m, double* t, double* dt, int64_t* cycle);
int orc_num_blocks(const orc_mesh* m, int64_t* n);
int orc_get_blocks(const orc_mesh* m, orc_block* out, int64_t cap, int64_t* n);
int orc_get_neighbors(const orc_mesh* m, int64_t gid, orc_neighbor* out, int32_t cap, int32_t* n);
int orc_get_refine_flags(const orc_mesh* m, int8_t* out, int64_t cap, int64_t* n);
int orc_get_indicators(const orc_mesh* m, double* out, int64_t cap, int64_t* n);
int orc_get_history(const orc_mesh* m, double* out, int64_t cap_rows, int64_t* nrows);
int orc_totals(const orc_mesh* m, double out[5]);
int orc_level_counts(const orc_mesh* m, int64_t* out, int32_t cap);
/* AMR: tag on current U0 and remesh (O9); used by orc_step automatically when adaptive. */
int orc_tag_and_remesh(orc_mesh* m);
const char* orc_last_error(void);

/* ---- point functions for pins ---- */
int orc_cons_to_prim(const double U[5], double gamma, double W[5]);
void orc_prim_to_cons(const double W[5], double gamma, double U[5]);
/* PLM on one component: returns the two face states of cell i: qR_{i-1/2}, qL_{i+1/2} */
void orc_plm(double qm, double q0, double qp, int32_t recon, double* q_left_face, double* q_right_face);
/* PPM (A37) / WENO-Z (A38) face values of cell q[2], q[0..4] = q_{i-2} .. q_{i+2} */
void orc_recon5(const double q[5], int32_t recon, double* q_left_face, double* q_right_face);
/* HLLE in the face-normal frame: W = (rho, u_normal, v_t1, v_t2, p) */
void orc_hlle(const double WL[5], const double WR[5], double gamma, double F[5]);
void orc_hlle_ws(const double WL[5], const double WR[5], double gamma, int32_t wavespeed, double F[5]);
void orc_flux_phys(const double W[5], double gamma, double F[5]);
double orc_restrict8(const double v[8]); /* v in (k,j,i) child order */
/* prolongation of one coarse value with neighbours cm[d] = C_{-d}, cp[d] = C_{+d}; out[8] in (k,j,i) child order */
void orc_prolong(double c, const double cm[3], const double cp[3], double out[8]);
uint64_t orc_morton_key(int32_t level, const int64_t lx[3], int32_t max_level);
void orc_partition(int64_t nblocks, int32_t nranks, int32_t rank, int64_t* lo, int64_t* hi);
double orc_pairwise_sum(const double* a, int64_t n);

#ifdef __cplusplus
}
#endif
#endif
