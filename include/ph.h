/*
 * ph.h -- C ABI of the B200-native Parthenon-hydro hot path (ABI version 3).
 *
 * What it computes (PAPER.md = arXiv 2202.12309, cited P:line):
 *   the per-cycle update of the Parthenon-hydro miniapp (§4.1: "a two-stage
 *   Runge-Kutta integrator, piecewise linear reconstruction and HLLE Riemann solver") over
 *   packed MeshBlocks (§3.6) on a block-structured oct-tree mesh (§2.1),
 *   with the fill-in-one ghost exchange incl. restriction / prolongation at coarse-fine
 *   boundaries (§3.7), flux correction, the CFL dt min-reduction as a
 *   global reduction (§3.10), Z-order (Morton) distribution of blocks over GPUs
 *    and remeshing with load balancing (§3.8).
 *   Readings where the paper is silent are SURVEY.md §8(c) A1-A30 plus DESIGN.md A5'-A41.
 *
 * Conventions
 *   - Every function returns ph_status; PH_OK == 0.  No C++ exception crosses this boundary: every
 *     entry point catches (std::bad_alloc -> PH_ERR_OOM, std::logic_error -> PH_ERR_INVALID_ARG,
 *     anything else -> PH_ERR_STATE) and reports the exception text through ph_last_error().
 *     On error, ph_last_error() returns a thread-local message valid until the next call.
 *   - Ownership: the caller owns every host buffer it passes and states its capacity; the
 *     library never retains host pointers.  The library owns all device memory (obtained
 *     through cfg->dev_alloc when given, else cudaMalloc).  The CUDA stream is borrowed.
 *   - Synchronisation: ph_step only enqueues work on cfg->stream (except AMR tag passes, which
 *     read refinement flags back, and when info != NULL).  Getters synchronise the stream.
 *     Device-side physics errors (rho <= 0 or p <= 0) are latched in a device word and reported
 *     as PH_ERR_PHYSICS by the next synchronising call, with gid and cell in the message.
 *   - Multi-GPU (cfg->nranks > 1): one process per GPU; every rank calls every function
 *     collectively with identical arguments (except gid / buffers).  NCCL is bootstrapped from
 *     a 128-byte ncclUniqueId that rank 0 obtains with ph_nccl_unique_id and the caller
 *     broadcasts (the Python binding uses torch.distributed).  On uniform meshes the per-cycle
 *     halo travels by peer-memory puts over NVLink (CUDA IPC; cfg->halo_transport) or NCCL;
 *     blocks with remote faces are updated first, interior blocks meanwhile on a second stream.
 *     The dt / totals reduction is an allgather in rank order, so N GPUs reproduce 1 GPU bitwise.
 *   - ph_get_state_full after ph_step returns valid ghosts on one rank (a full exchange is run when
 *     the direct halo left local face ghosts stale); on several ranks call ph_exchange first.
 *   - Host state layout: [5][n3][n2][n1], interior cells only, i fastest, variables
 *     (rho, m1, m2, m3, E) -- conserved variables of the Euler equations.
 *   - Calls on one handle must be serialised by the caller.
 */
#ifndef PH_H
#define PH_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define PH_ABI_VERSION 3

typedef struct ph_mesh ph_mesh; /* opaque; owned by the caller until ph_mesh_destroy */

typedef enum {
  PH_OK = 0,
  PH_ERR_INVALID_ARG = 1,
  PH_ERR_CONFIG = 2,  /* e.g. block size does not tile the root grid */
  PH_ERR_CUDA = 3,
  PH_ERR_COMM = 4,
  PH_ERR_OOM = 5,
  PH_ERR_PHYSICS = 6, /* rho <= 0 or p <= 0 (A24) */
  PH_ERR_STATE = 7,   /* call out of order, or host-only handle asked for device work */
  PH_ERR_UNSUPPORTED = 8
} ph_status;

typedef enum { PH_BC_PERIODIC = 0, PH_BC_OUTFLOW = 1, PH_BC_REFLECT = 2 } ph_bc;       /* A9 */
typedef enum {
  PH_RECON_PLM_MINMOD = 0, PH_RECON_PLM_VANLEER = 1, PH_RECON_PLM_MC = 2, /* A3; nghost 2 */
  PH_RECON_PPM = 3, PH_RECON_WENOZ = 4                                   /* NEXT 3 (A37, A38); nghost 3 */
} ph_recon;
typedef enum { PH_INT_RK2 = 0, PH_INT_VL2 = 1 } ph_integrator;                      /* A1 */
/* HLLE wave-speed estimates (A4): Davis S_L = min(u_L - c_L, u_R - c_R), S_R = max(u_L + c_L, u_R + c_R)
 * (default), or Einfeldt (1988) S_L = min(u_L - c_L, u~ - c~), S_R = max(u_R + c_R, u~ + c~) with Roe
 * averages (sqrt(rho) weights) of velocity and total enthalpy.  Einfeldt: PLM reconstructions only. */
typedef enum { PH_WS_DAVIS = 0, PH_WS_EINFELDT = 1 } ph_wavespeed;
typedef enum { PH_PROB_LINEAR_WAVE = 0, PH_PROB_SOD = 1, PH_PROB_BLAST = 2, PH_PROB_KH = 3 } ph_problem;
typedef enum { PH_REF_NONE = 0, PH_REF_STATIC = 1, PH_REF_ADAPTIVE = 2 } ph_refinement;
/* How the per-cycle halo of a (non-adaptive) multi-GPU mesh travels between GPUs.  On uniform meshes
 * blocks with remote faces are updated first and their faces sent while the interior blocks compute. */
typedef enum {
  PH_HALO_AUTO = 0,  /* peer memory when every rank can map its peers' receive buffers, else NCCL */
  PH_HALO_NCCL = 1,  /* pack -> grouped ncclSend/ncclRecv -> unpack into ghost cells */
  PH_HALO_PEER = 2   /* peer memory, or PH_ERR_UNSUPPORTED: the pack kernel stores boundary faces
                        straight into the receiving GPU's buffer over NVLink (CUDA IPC) and raises
                        a flag there; the receiver waits on the flag and unpacks.  No NCCL. */
} ph_halo_transport;

typedef struct {
  int32_t abi_version;     /* must equal PH_ABI_VERSION, else PH_ERR_INVALID_ARG */
  int32_t nghost;          /* ghost width: 2 (PLM) or 3 (PPM / WENO-Z, uniform meshes only; A8, A39) */
  int64_t mesh_nx[3];      /* root-grid cells per dim */
  int64_t block_nx[3];     /* cells per MeshBlock per dim; must divide mesh_nx;
                              even and >= 2*nghost when max_level > 0 */
  int32_t max_level;       /* refinement levels above the root (0 = uniform) */
  int32_t refinement;      /* ph_refinement */
  double xmin[3], xmax[3]; /* physical domain (Cartesian only) */
  int32_t bc_inner[3], bc_outer[3]; /* ph_bc per face; periodic must be paired */
  double gamma, cfl;       /* ideal-gas gamma (A6); CFL number (A7, default 0.3) */
  int32_t recon, integrator;
  double refine_tol, derefine_tol;  /* AMR thresholds on the pressure-gradient indicator (A14) */
  int32_t derefine_interval;        /* derefinement gate, cycles (A16) */
  int32_t nregions;                 /* static refinement regions */
  const double* regions;            /* [nregions][7]: level, x1min,x1max, x2min,x2max, x3min,x3max */
  int32_t pack_size;                /* blocks per stage-kernel launch; <= 0 means all (A25) */
  int32_t rank, nranks;             /* this process' rank and the number of GPUs */
  int32_t device;                   /* CUDA device ordinal */
  int32_t host_only;                /* 1: build the mesh/partition/exchange plan only (no GPU) */
  int32_t no_direct_halo;           /* 1: materialise every ghost each exchange (the paper's scheme);
                                       0 (default): the stage kernel of every block without coarse
                                       staging reads its local same-level face neighbours' interiors
                                       directly (all blocks of a uniform mesh) */
  void* stream;                     /* cudaStream_t to enqueue on (borrowed); NULL = legacy default */
  const void* nccl_id;              /* 128-byte ncclUniqueId (nranks > 1), else NULL */
  void* (*dev_alloc)(size_t bytes, void* ctx); /* optional device allocator (torch caching allocator) */
  void (*dev_free)(void* ptr, void* ctx);
  void* alloc_ctx;
  int32_t halo_transport;           /* ph_halo_transport (ABI 2).  Peer memory applies to nghost-2
                                       meshes (uniform, static multilevel or adaptive: a remesh
                                       rebuilds the receive regions and mappings, collectively) with
                                       nranks > 1; its receive buffers come from cudaMalloc (CUDA IPC),
                                       not dev_alloc.  The full exchange (ph_refresh, ph_exchange) and
                                       the remesh's block migration stay on NCCL. */
  int32_t wavespeed;                /* ph_wavespeed (ABI 3); 0 = Davis */
} ph_config;

/* One leaf block.  gid = position in Z-order (A19); rank from the contiguous Morton partition. */
typedef struct {
  int64_t gid;
  int32_t level, rank;
  int64_t lx[3];
  double xmin[3], xmax[3];
} ph_block;

/* One neighbour entry in the canonical order of SURVEY §8(c) O3:
 * offsets o3 outer, o2, o1 inner (skipping 0,0,0); dlevel = neighbour level - own level;
 * fine[] = child indices along the free dims (o_d == 0) for finer neighbours. */
typedef struct {
  int64_t gid;
  int32_t rank;
  int8_t off[3];
  int8_t dlevel;
  int8_t fine[2];
} ph_neighbor;

typedef struct {
  int64_t cycle;
  double t, dt;          /* time after the last cycle; dt for the next cycle */
  int64_t zone_cycles;   /* interior cells x cycles run by this call (all ranks) */
} ph_step_info;

/* Exchange-plan summary of this rank (for tests of the multi-GPU plumbing). */
typedef struct {
  int64_t n_local_tasks;        /* buffers filled rank-locally per exchange */
  int64_t n_send_tasks, n_recv_tasks;
  int64_t send_doubles_to[64];  /* per peer rank: doubles packed per exchange */
  int64_t recv_doubles_from[64];
  uint64_t send_hash_to[64];    /* order-sensitive hash of the (dst gid, entry) sequence */
  uint64_t recv_hash_from[64];
  /* the per-cycle exchange (direct halo: blocks without coarse staging drop local same-level face
     copies and edge / corner entries; on uniform meshes only remote faces and physical BCs remain) */
  int64_t cyc_send_doubles_to[64];
  int64_t cyc_recv_doubles_from[64];
  uint64_t cyc_send_hash_to[64];
  uint64_t cyc_recv_hash_from[64];
  int32_t direct_halo;          /* 1 if stage kernels of blocks without coarse staging read local
                                   same-level face neighbours directly (uniform and multilevel meshes) */
  int64_t n_cyc_local_tasks;
  int32_t peer_halo;            /* 1 if the per-cycle halo travels by peer-memory puts (ABI 2) */
} ph_plan_info;

/* ---- lifecycle ---------------------------------------------------------------------------- */
/* Get a fresh ncclUniqueId (128 bytes) on rank 0; out must hold 128 bytes. */
ph_status ph_nccl_unique_id(void* out, int32_t cap);
/* Build tree (O1), Morton order and partition (O2), neighbour lists (O3), exchange plan, and
 * (unless host_only) allocate the device block pool U0/U1 [slot][5][n3+2g][n2+2g][n1+2g] fp64. */
ph_status ph_mesh_create(const ph_config* cfg, ph_mesh** out);
ph_status ph_mesh_destroy(ph_mesh* m);

/* ---- state -------------------------------------------------------------------------------- */
/* Problem generator on the device (O4): LINEAR_WAVE p = {A, k1, k2, k3};
 * SOD p = {x_split}; BLAST p = {p_in, p_out, radius[, cx, cy, cz]}; KH p = {A, sigma}
 * (Kelvin-Helmholtz shear layers, the paper's AMR demo P:702, A36).  Runs AMR pre-refinement
 * when refinement is adaptive, fills ghosts and computes the initial dt.  Collective. */
ph_status ph_set_problem(ph_mesh* m, int32_t problem, const double* p, int32_t np);
/* Upload one block's interior [5][n3][n2][n1] (only the rank owning gid copies; others no-op).
 * Call ph_refresh after the last upload to fill ghosts and recompute dt. */
ph_status ph_set_state(ph_mesh* m, int64_t gid, const double* cons, int64_t nelem);
ph_status ph_refresh(ph_mesh* m); /* exchange + dt on the current state; collective */
/* Read one block's interior; only the owning rank copies (others return PH_OK, n untouched). */
ph_status ph_get_state(const ph_mesh* m, int64_t gid, double* cons_out, int64_t nelem);
/* Read the block with ghosts [5][n3+2g][n2+2g][n1+2g] (tests of the exchange). */
ph_status ph_get_state_full(const ph_mesh* m, int64_t gid, double* out, int64_t nelem);
ph_status ph_set_state_full(ph_mesh* m, int64_t gid, const double* in, int64_t nelem);
ph_status ph_exchange(ph_mesh* m); /* ghost exchange of U0 only (O7); collective */

/* ---- evolution ---------------------------------------------------------------------------- */
/* Run ncycles cycles of O5 (stage 1, exchange, stage 2, exchange, [AMR remesh], dt, history).
 * tlim > 0 caps the last dt so that t <= tlim; cycles after t reaches tlim are no-ops. */
ph_status ph_step(ph_mesh* m, int32_t ncycles, double tlim, ph_step_info* info /*nullable*/);
/* Host-buffer end-to-end call: upload the interiors of all local blocks from `host_in`
 * ([nlocal][5][n3][n2][n1], local gid order), run ncycles, download them into `host_out`.
 * Times the full path incl. host<->device copies (bench e2e leg).  Both buffers hold exactly
 * nelem doubles (checked against the local block count; PH_ERR_INVALID_ARG otherwise).
 * Adaptive meshes return PH_ERR_UNSUPPORTED: a remesh inside the call would change the local
 * block set, and with it the layout of host_out. */
ph_status ph_step_host(ph_mesh* m, const double* host_in, double* host_out, int64_t nelem,
                       int32_t ncycles, double tlim);
/* The same, enqueued on cfg->stream without waiting (host buffers must be pinned and stay valid until
 * ph_sync; adaptive meshes: PH_ERR_UNSUPPORTED as above).  Two meshes on two streams can
 * overlap one problem's device->host copy with the next one's host->device copy. */
ph_status ph_step_host_async(ph_mesh* m, const double* host_in, double* host_out, int64_t nelem,
                             int32_t ncycles, double tlim);
/* Wait for everything enqueued on the mesh's stream; reports latched device errors (PH_ERR_PHYSICS). */
ph_status ph_sync(ph_mesh* m);

/* ---- queries ------------------------------------------------------------------------------ */
ph_status ph_num_blocks(const ph_mesh* m, int64_t* nglobal, int64_t* nlocal);
ph_status ph_get_blocks(const ph_mesh* m, ph_block* out, int64_t cap, int64_t* n); /* gid order */
ph_status ph_get_neighbors(const ph_mesh* m, int64_t gid, ph_neighbor* out, int32_t cap, int32_t* n);
ph_status ph_get_refine_flags(const ph_mesh* m, int8_t* out, int64_t cap, int64_t* n); /* last tag pass */
/* history rows [t, dt, M, M1, M2, M3, E] (conserved totals, O10), one per cycle */
ph_status ph_get_history(const ph_mesh* m, double* out, int64_t cap_rows, int64_t* nrows);
ph_status ph_get_time(const ph_mesh* m, double* t, double* dt, int64_t* cycle);
ph_status ph_totals(ph_mesh* m, double out[5]); /* current conserved totals; collective */
ph_status ph_get_plan_info(const ph_mesh* m, ph_plan_info* out);
/* Number of kernels the library enqueued since creation (gpu_launches evidence for bench.py). */
ph_status ph_launch_count(const ph_mesh* m, int64_t* n);
/* Record CUDA events around the stage kernels of the next ph_step (bench roofline): returns the
 * summed device ms of all stage-kernel launches and their count since the last reset. */
ph_status ph_kernel_timing(ph_mesh* m, int32_t enable, double* stage_ms, int64_t* stage_launches,
                           double* exch_ms, int64_t* exch_launches);
const char* ph_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
