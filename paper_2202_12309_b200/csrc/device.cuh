// device.cuh -- plain structs shared by the host orchestration (api.cu) and the sm_100a
// kernels (kernels.cu).  Product code only; nothing here is shared with oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ph {

constexpr int NVAR = 5;  // rho, m1, m2, m3, E

// Per-launch geometry of the block pool.  Pool layout (a1): U[slot][v][k][j][i], fp64,
// i fastest, extents (n+2g) -- the paper's slowest-first index order.
struct Geom {
  int n[3];        // interior cells per dim
  int g;           // ghost width (2)
  int N[3];        // n + 2g
  int64_t vstride; // N1*N2*N3
  int64_t bstride; // 5*vstride
  int nc[3];       // coarse staging interior (n/2)
  int cg;          // coarse staging ghosts
  int NC[3];       // nc + 2cg
  int64_t cvstride, cbstride;
  int64_t fstride; // doubles per face-flux slot (5 * max face cells)
  double gamma, gm1, inv_gm1;
  double cfl;
  int exact;       // 1: high-order path computes in the oracle's exact operation order (NEXT 3)
  int wavespeed;   // HLLE wave speeds: 0 Davis, 1 Einfeldt (A4)
  int no_stage2;   // 1: the mesh is too small to fill the GPU with stage2's 16x16 tiles (round-1 kernel)
};

// Per local block slot.
struct BlockMeta {
  double idx[3];     // 1/dx
  double dV;
  double xmin[3];
  double dx[3];
  int64_t gid;
  int level;
  int cslot;         // coarse staging slot, -1 if none
  int fslot[6];      // face-flux slot for faces -x,+x,-y,+y,-z,+z (coarse-fine faces), else -1
  int nb[6];         // direct halo: slot of the local same-level face neighbour, else -1 (use ghosts)
  int prank[6];      // fused peer put: rank receiving this face's g boundary layers, else -1
  long long poff[6]; // ... and the offset (doubles) of its [v][box] task in that rank's receive half
  int rfx;           // bit f: face f receives flux correction (this block is the coarse side)
};

// Ghost-exchange task (fill-in-one).  One task fills one destination box.
enum TaskKind : int {
  T_COPY = 0,       // same level: U_dst[d] = U_src[d + so]
  T_RESTRICT = 1,   // finer source: U_dst[d] = mean8(U_src[2d - so ...])
  T_CCOPY = 2,      // coarser source into my staging: C_dst[d] = U_src[d + so]
  T_CRESTRICT = 3,  // own fine cells into own staging: C[d] = mean8(U[2d ...])
  T_PROLONG = 4,    // staging first layer -> 8 fine ghosts
  T_BC_FINE = 5,    // physical BC on fine ghosts (direct composition of x1,x2,x3 passes)
  T_BC_COARSE = 6,  // physical BC on staging ghosts
  T_UNPACK_U = 7,   // recv buffer -> U box
  T_UNPACK_C = 8    // recv buffer -> C box
};

struct XTask {
  int kind;
  int dst_slot;      // pool slot (U or C by kind); -1 = send buffer (pack)
  int src_slot;      // pool slot; -1 = recv buffer (unpack)
  int lo[3];         // first destination cell
  int ext[3];        // box extents
  int so[3];         // source shift (see kinds)
  int bc;            // BC kinds: per dim d, bits [4d,4d+2) low face, [4d+2,4d+4) high face: 0 none, 1 outflow, 2 reflect;
                     // pack tasks: -1 = my send buffer, else the peer rank whose receive buffer is written (put)
  int ncell;
  int64_t buf;       // offset (doubles) into the send / recv buffer; payload [v][cell]
};

struct Chunk {
  int task;
  int begin;
};

// Reflux (flux correction, O8 / a8): one coarse face with 4 finer face neighbours.
struct RefluxTask {
  int cslot;         // coarse block slot
  int dir, side;     // face dim, -1 low / +1 high
  int cfs;           // coarse face-flux slot
  int ffs;           // fine face-flux slot
  int t0lo, t1lo;    // coarse tangential start of this fine block's quarter
  int64_t roff;      // >= 0: the fine block lives on another rank; its restricted fluxes are at
                     // recv-buffer offset roff ([v][B0][A0] over the quarter)
};

// Fine side of a cross-rank flux correction: restrict (mean of 4) this fine block's face fluxes
// and pack them for the coarse block's rank (flux correction is communicated).
struct FluxPackTask {
  int ffs;           // fine face-flux slot
  int dir;
  int64_t off;       // send-buffer offset
};

struct ErrWord {
  int flag;
  int stage;
  long long gid;
  int k, j, i;
};

// Device-resident cycle state (dt, t, history).  Updated only by kernels.
struct CycleState {
  double t, dt, dt_used, tlim;
  long long cycle;
  int active;
  int pad;
  long long hist_count;
};

constexpr int TILE_X = 32, TILE_Y = 8;  // default stage-kernel tile (i, j); 16x16 for 16-wide blocks

struct StageArgs {
  const double* Uin;   // pool with valid ghosts (stage input)
  const double* U0;    // base state U^n (interior reads), may alias Uout
  double* Uout;        // output pool (interior writes)
  const BlockMeta* meta;
  const int* slots;    // pack: list of block slots
  const CycleState* st;
  double* fbuf;        // face-flux slots (multilevel)
  double* partials;    // [ncta][6] (max speed/dx, 5 totals) when REDUCE
  ErrWord* err;
  double a0, b1, cdt;  // out = a0*U0 + b1*Uin + cdt*dt*L
  int ntx, nty, nkc, KC;
  int cta_base;        // offset of this launch's CTAs in partials
  int stage;
  // uniform full-tile path: stage 1 also writes the cell-local base of stage 2,
  // H = ha0 U^n + hb1 U^1, and stage 2 reads H instead of U^n and U^1 at the cell (null = off)
  double* H;
  double ha0, hb1;
  // fused peer put (boundary blocks, peer transport): finished cells within g layers of a remote face
  // are also stored into that peer's receive half (M.prank / M.poff); null = off
  double* const* peer_rbuf;
  int pool_slots;       // slots allocated in the U0 / U1 / H pools (tensor-map extent, stage2.cu)
};

struct XArgs {
  const XTask* tasks;
  const Chunk* chunks;
  double* U;           // fine pool (read and write)
  double* C;           // coarse staging pool
  double* sbuf;        // send buffer (pack tasks)
  const double* rbuf;  // recv buffer (unpack tasks)
  double* const* peer_rbuf;  // peer transport: [nranks] IPC-mapped receive buffers (put tasks)
};

struct PgenArgs {
  int problem;
  double p[8];
  double xmin[3], L[3];
};

// Remesh data movement (O9): new pool <- old pool, possibly through the migration
// send / recv buffers.  MOVE: interior copy; REFINE: prolongate a parent (full block incl. ghosts)
// into child ch; OCT: restrict a child into octant ch of its parent; OCTCOPY: packed octant ->
// octant ch.  dst < 0: packed into the send buffer at dst_off; src < 0: from the recv buffer at
// src_off (packed interior / packed octant / a full block laid out like a pool slot for REFINE).
enum RemeshKind : int { R_MOVE = 0, R_REFINE = 1, R_OCT = 2, R_OCTCOPY = 3 };
struct RemeshTask {
  int kind;
  int dst, src;
  int64_t dst_off, src_off;
  int ch[3];
};

constexpr int XCHUNK = 256;  // cells per exchange chunk (one CTA, one cell per thread; 2 per thread in pair mode)

// Pair mode of a copy / unpack / pack task: every thread moves two cells adjacent in i with 16-byte
// accesses.  Needs an even row extent and even (16-B aligned) first indices on both sides; the host
// (chunking) and the kernel evaluate the same rule.
__host__ __device__ inline bool xtask_pairs(const XTask& t, int g, int cg) {
  if ((t.ext[0] & 1) || (g & 1) || (cg & 1) || (t.lo[0] & 1)) return false;
  switch (t.kind) {
    case T_COPY:
    case T_CCOPY:
      return ((t.so[0] & 1) == 0) && (t.dst_slot >= 0 || (t.buf & 1) == 0);
    case T_UNPACK_U:
    case T_UNPACK_C:
      return (t.buf & 1) == 0;
    default:
      return false;
  }
}

// launchers (kernels.cu)
cudaError_t launch_stage(int recon, bool reduce, bool use_u0, int nblk_cta, const StageArgs& a, const Geom& G,
                         cudaStream_t s);
// Peer halo transport: signal / wait on IPC-mapped epoch flags (see kernels.cu).
cudaError_t launch_peer_signal(unsigned long long* const* peer_flags, unsigned long long* ctr, int me,
                               unsigned long long mask, cudaStream_t s);
cudaError_t launch_peer_wait(const unsigned long long* my_flags, unsigned long long* ctr, unsigned long long mask,
                             ErrWord* err, cudaStream_t s);
cudaError_t launch_xfill(int nchunks, const XArgs& a, const Geom& G, cudaStream_t s);
cudaError_t launch_reflux(int ntasks, const RefluxTask* t, double* U, const BlockMeta* meta, const double* fbuf,
                          const double* rbuf, const CycleState* st, double w, const Geom& G, cudaStream_t s,
                          double* H = nullptr, double hb1 = 0.0);
cudaError_t launch_flux_pack(int ntasks, const FluxPackTask* t, const double* fbuf, double* sbuf, const Geom& G,
                             cudaStream_t s);
cudaError_t launch_pgen(double* U, const BlockMeta* meta, int nslots, const PgenArgs& P, const Geom& G,
                        cudaStream_t s);
cudaError_t launch_reduce(const double* U, const BlockMeta* meta, int nslots, double* partials, ErrWord* err,
                          const Geom& G, cudaStream_t s);
cudaError_t launch_rank_reduce(const double* partials, int n, double* out, cudaStream_t s);
cudaError_t launch_finalize(const double* all, int nranks, CycleState* st, double* hist, int hist_cap, double cfl,
                            int mode, double* tot_out, int exact, cudaStream_t s);
cudaError_t launch_cycle_begin(CycleState* st, double tlim, int set_tlim, cudaStream_t s);
cudaError_t launch_interior_copy(double* U, double* buf, int slot0, int nslots, int to_pool, const Geom& G,
                                 cudaStream_t s);
// AMR indicator per block; with partials != null also the dt / totals partials of U (one row of 6
// per CTA, tag_ctas_per_block(G) CTAs per block, same layout as reduce_kernel)
// dt / totals partials of the cells in the corrected face layers (after the reflux), one row per
// (block slot, face) pair; edge / corner cells counted once (by their lowest corrected face)
cudaError_t launch_rfx_reduce(const int2* faces, int nfaces, const double* U, const BlockMeta* meta, double* partials,
                              ErrWord* err, const Geom& G, cudaStream_t s);
cudaError_t launch_tag(const double* U, const BlockMeta* meta, int nslots, unsigned long long* eps_bits,
                       double* partials, ErrWord* err, const Geom& G, cudaStream_t s);
int tag_ctas_per_block(const Geom& G);
// stage2.cu: the TMA-fed tag pass (16 x 16 tiles) for blocks whose x / y extents are multiples of 16
bool tag2_applies(const Geom& G);
int tag2_ctas_per_block(const Geom& G);
cudaError_t launch_tag2(const double* U, const BlockMeta* meta, int nslots, unsigned long long* eps_bits,
                        double* partials, ErrWord* err, const Geom& G, cudaStream_t s);
cudaError_t launch_remesh(const RemeshTask* t, int ntasks, const double* Uold, double* Unew, const double* rbuf,
                          double* sbuf, const Geom& G, cudaStream_t s);
cudaError_t launch_highorder_stage(int recon, bool reduce, bool use_u0, int nslots, const StageArgs& a, double* W,
                                   double* Fx, double* Fy, double* Fz, bool w_ready, bool w_out, const Geom& G,
                                   cudaStream_t s);
size_t stage_smem_bytes();
// stage2.cu: the round-2 uniform-mesh stage kernel (16 x 16 tiles, bulk-copy plane ring); applies to
// minmod + Davis on uniform levels with n1, n2 multiples of 16 and nghost 2 (PH_STAGE_V1=1 disables it)
bool stage2_applies(const Geom& G, int recon, bool ml);
cudaError_t launch_stage2(bool reduce, bool use_u0, int nctas, const StageArgs& a, const Geom& G, cudaStream_t s);
// stage-kernel tile (tx x ty columns) for this block extent; true = full-tile (minmod, uniform) path
bool stage_tile(const Geom& G, int recon, bool ml, int* tx, int* ty);

}  // namespace ph
