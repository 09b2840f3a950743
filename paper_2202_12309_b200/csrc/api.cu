// api.cu -- C ABI (include/ph.h): mesh/plan construction, device block pool, the per-cycle
// schedule (O5: one CUDA graph per cycle; boundary-first two-stream cycle on several GPUs), the halo
// transports (peer-memory puts over CUDA IPC, or NCCL), AMR remesh and migration.  Hot work runs in
// kernels.cu.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <array>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/ph.h"
#include "device.cuh"
#include "mesh.hpp"

namespace ph {
constexpr int TX = TILE_X, TY = TILE_Y;
}

using namespace ph;

// NVTX ranges (header-only NVTX3) around each stage, exchange, tag / remesh and cycle: named spans in any
// CUPTI / Nsight timeline of a run (tools/timeline.py records the kernels themselves).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

static thread_local std::string g_err;
static ph_status fail(ph_status s, const std::string& m) {
  g_err = m;
  return s;
}
#define CU(x)                                                                                         \
  do {                                                                                                \
    cudaError_t e_ = (x);                                                                             \
    if (e_ != cudaSuccess) return fail(PH_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)
#define NC(x)                                                                                          \
  do {                                                                                                 \
    ncclResult_t r_ = (x);                                                                             \
    if (r_ != ncclSuccess) return fail(PH_ERR_COMM, std::string(#x) + ": " + ncclGetErrorString(r_)); \
  } while (0)
#define TRY(x)                    \
  do {                            \
    ph_status s_ = (x);           \
    if (s_ != PH_OK) return s_;   \
  } while (0)

struct Phase {
  std::vector<XTask> tasks;
  std::vector<Chunk> chunks;
  XTask* d_tasks = nullptr;
  Chunk* d_chunks = nullptr;
  int nchunks() const { return (int)chunks.size(); }
};

// One exchange plan: the fill-in-one phases of SURVEY O7 (A: pack / local / unpack, B1, B2, C, D)
// plus the per-peer buffer layout.  plan[0] = full exchange (all 26 directions), plan[1] = the
// per-cycle exchange (== full unless the direct-halo path makes some of it unnecessary).
struct Plan {
  Phase pack, local, unpack, b1, b2, pro, bcf;
  std::vector<int64_t> send_off, send_cnt, recv_off, recv_cnt;  // per peer, doubles
  std::vector<uint64_t> send_hash, recv_hash;
  int64_t sbuf_n = 0, rbuf_n = 0;
  std::vector<Phase*> phases() { return {&pack, &local, &unpack, &b1, &b2, &pro, &bcf}; }
};

struct ph_mesh {
  ph_config cfg;
  std::vector<double> regions;
  MeshCfg mc;
  Tree* tree = nullptr;
  std::vector<BlockInfo> blocks;
  std::unordered_map<LocKey, int64_t> gid_of;
  std::vector<int64_t> local_gids;  // slot -> gid
  Geom G;
  int rank = 0, nranks = 1;
  bool host_only = false;
  bool multilevel = false;
  bool cross_rank_reflux = false;
  cudaStream_t stream = nullptr, comm_stream = nullptr;
  cudaEvent_t ev_pack = nullptr, ev_comm = nullptr;
  ncclComm_t comm = nullptr;
  // device memory
  std::vector<void*> allocs;   // mesh-dependent (replaced on every remesh)
  std::vector<void*> pallocs;  // persistent (cycle state, history, reductions)
  unsigned long long* d_eps = nullptr;      // AMR indicator per local slot (double bits), padded
  unsigned long long* d_eps_all = nullptr;  // all ranks' indicators (allgather)
  double *U0 = nullptr, *U1 = nullptr, *C = nullptr, *fbuf = nullptr;
  double *partials = nullptr, *my6 = nullptr, *all6 = nullptr, *tot5 = nullptr, *hist = nullptr, *stage_buf = nullptr;
  BlockMeta* d_meta = nullptr;
  int* d_slots = nullptr;
  CycleState* d_st = nullptr;
  ErrWord* d_err = nullptr;
  double *sbuf = nullptr, *rbuf = nullptr;
  int64_t sbuf_n = 0, rbuf_n = 0;
  int hist_cap = 1 << 16;
  int n_cslots = 0, n_fslots = 0;
  std::vector<BlockMeta> meta;
  // plans: [0] full exchange, [1] per-cycle exchange
  Plan plan[2];
  bool no_direct_halo = false;  // config: force materialised ghosts every exchange
  bool ghosts_stale = false;
  bool w_ready = false;     // nghost-3 path: Wpool holds the primitives of U0 incl. ghosts (A49)
  bool ho_fold = true;      // nghost-3 path: the update writes W, the per-cycle exchange moves W (PH_HO_NOFOLD=1: off)
  bool ho = false;                      // nghost 3: generic high-order path (NEXT 3)
  double *Wpool = nullptr, *Fxb = nullptr, *Fyb = nullptr, *Fzb = nullptr;
  double* Hpool = nullptr;  // stage-2 base H = a0 U^n + b1 U^1 (uniform full-tile minmod path)
  bool overlap = false;                 // multi-GPU direct halo: interior blocks overlap the exchange
  int n_int = 0;                        // slots [0, n_int) of slot_order have no remote / physical face
  std::vector<int> slot_order;
  ncclComm_t comm2 = nullptr;           // split communicator for the dt / totals allgather
  bool use_graph = true;                 // PH_NO_GRAPH=1 disables
  cudaGraphExec_t graph_exec = nullptr;  // one captured cycle
  cudaStream_t gstream = nullptr;        // private capture / replay stream
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int64_t graph_launches = 0;  // a direct-halo cycle ran since the last full exchange
  bool direct_halo = false;  // uniform mesh: stage kernels read local same-level face neighbours directly
  std::vector<RefluxTask> reflux[3];
  std::vector<int2> rfx_faces;  // (slot, face) pairs receiving flux correction (static multilevel dt)
  int2* d_rfx_faces = nullptr;
  RefluxTask* d_reflux[3] = {nullptr, nullptr, nullptr};
  // cross-rank flux correction: fine-side packs and per-peer layout
  std::vector<FluxPackTask> fpack;
  FluxPackTask* d_fpack = nullptr;
  std::vector<int64_t> fsend_off, fsend_cnt, frecv_off, frecv_cnt;
  int64_t fsbuf_n = 0, frbuf_n = 0;
  double *fsbuf = nullptr, *frbuf = nullptr;
  // stage launch geometry
  int ntx = 1, nty = 1, nkc = 1, KC = 1;
  int stage_ctas = 0;
  int pack_size = 0;
  int64_t partials_n = 0;
  // bookkeeping
  int64_t launches = 0;
  bool have_state = false;
  std::vector<int8_t> last_flags;
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> t_stage, t_exch;
  std::vector<cudaEvent_t> ev_pool;
  // peer transport of the per-cycle halo (uniform multi-GPU meshes): [64 flags | recv half 0 |
  // recv half 1] in one IPC-exported cudaMalloc region per rank.  The pack kernel stores boundary
  // faces straight into the peers' receive halves (U1 exchange: half 0, U0 exchange: half 1),
  // then signals; the receiver waits on its flags and unpacks locally.
  bool peer = false;
  void* peer_region = nullptr;
  std::vector<void*> peer_open;                     // per rank: mapped peer region (nullptr for me)
  double** d_prbuf[2] = {nullptr, nullptr};         // device [R]: every rank's receive half 0 / 1
  double* my_rbuf[2] = {nullptr, nullptr};
  unsigned long long** d_pflags = nullptr;          // device [R]: every rank's flag array
  unsigned long long* my_flags = nullptr;           // [64] in my region, written by peers
  unsigned long long* d_ctr = nullptr;              // [2] signal / wait epoch counters (device)
  void* d_peer_rec = nullptr;                       // device [R + 1] set-up records (allgather)
  unsigned long long send_mask = 0, recv_mask = 0;  // peers I put to / receive from per exchange
  bool fused_put = false;  // the boundary blocks' stage kernel stores the faces itself (no put kernel)
  // boundary-first schedule of the multi-GPU cycle: B (high priority) runs boundary blocks and the
  // halo, I runs interior blocks concurrently
  cudaStream_t bstream = nullptr, istream = nullptr;
  // concurrent packs (NEXT 4; the paper's best GPU setting is 2 packs per rank): when a
  // stage is split into several pack launches they rotate over the caller's stream and pstream[]
  static constexpr int kMaxPackStreams = 8;
  int pack_streams = 8;
  cudaStream_t pstream[kMaxPackStreams] = {};
  cudaEvent_t ev_pfork = nullptr, ev_pjoin[kMaxPackStreams] = {};
  cudaEvent_t ev_a = nullptr, ev_b1 = nullptr, ev_i1 = nullptr, ev_b2 = nullptr, ev_i2 = nullptr;
};

/* ------------------------------------------------------------------------------- helpers */
static ph_status dalloc(ph_mesh* m, void** p, size_t bytes, bool persistent = false) {
  *p = nullptr;
  if (bytes == 0) return PH_OK;
  if (m->cfg.dev_alloc) {
    *p = m->cfg.dev_alloc(bytes, m->cfg.alloc_ctx);
    if (!*p) return fail(PH_ERR_OOM, "dev_alloc returned NULL for " + std::to_string(bytes) + " bytes");
  } else {
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess) return fail(PH_ERR_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  }
  (persistent ? m->pallocs : m->allocs).push_back(*p);
  return PH_OK;
}

template <class T>
static ph_status upload(ph_mesh* m, T** d, const std::vector<T>& h) {
  *d = nullptr;
  if (h.empty()) return PH_OK;
  TRY(dalloc(m, (void**)d, h.size() * sizeof(T)));
  CU(cudaMemcpy(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return PH_OK;
}

static void free_list(ph_mesh* m, std::vector<void*>& l) {
  for (void* p : l) {
    if (m->cfg.dev_free) m->cfg.dev_free(p, m->cfg.alloc_ctx);
    else cudaFree(p);
  }
  l.clear();
}

static void free_all(ph_mesh* m) {
  if (m->host_only) return;
  cudaStreamSynchronize(m->stream);
  free_list(m, m->allocs);
  free_list(m, m->pallocs);
}

static uint64_t mix(uint64_t h, uint64_t x) {
  h ^= x + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  return h;
}

static void add_chunks(Phase& P, const XTask& t, const Geom& G) {
  int id = (int)P.tasks.size();
  P.tasks.push_back(t);
  const int step = xtask_pairs(t, G.g, G.cg) ? 2 * XCHUNK : XCHUNK;  // pair mode: 2 cells per thread
  for (int b = 0; b < t.ncell; b += step) P.chunks.push_back(Chunk{id, b});
}

static int bc_bits(const ph_mesh* m, const BlockInfo& b) {
  int bits = 0;
  for (int d = 0; d < 3; ++d) {
    int lo = b.phys_lo[d] ? (m->cfg.bc_inner[d] == PH_BC_REFLECT ? 2 : 1) : 0;
    int hi = b.phys_hi[d] ? (m->cfg.bc_outer[d] == PH_BC_REFLECT ? 2 : 1) : 0;
    bits |= (lo | (hi << 2)) << (4 * d);
  }
  return bits;
}

/* geometry of one neighbour entry as seen by destination block b (O7 phase A) */
static XTask entry_task(const ph_mesh* m, const BlockInfo& b, const Neighbor& e) {
  XTask t{};
  const int* n = m->G.n;
  const int g = m->G.g, cg = m->G.cg;
  if (e.dlevel == 0) {
    t.kind = T_COPY;
    for (int d = 0; d < 3; ++d) {
      if (e.off[d] < 0) { t.lo[d] = -g; t.ext[d] = g; t.so[d] = n[d]; }
      else if (e.off[d] > 0) { t.lo[d] = n[d]; t.ext[d] = g; t.so[d] = -n[d]; }
      else { t.lo[d] = 0; t.ext[d] = n[d]; t.so[d] = 0; }
    }
  } else if (e.dlevel == 1) {
    t.kind = T_RESTRICT;
    int f = 0;
    for (int d = 0; d < 3; ++d) {
      int ch = e.off[d] ? (e.off[d] == 1 ? 0 : 1) : e.fine[f++];
      if (e.off[d] < 0) { t.lo[d] = -g; t.ext[d] = g; }
      else if (e.off[d] > 0) { t.lo[d] = n[d]; t.ext[d] = g; }
      else { t.lo[d] = ch * n[d] / 2; t.ext[d] = n[d] / 2; }
      t.so[d] = (2 * e.off[d] + ch) * n[d];
    }
  } else {
    t.kind = T_CCOPY;
    for (int d = 0; d < 3; ++d) {
      int nc = m->G.nc[d];
      if (e.off[d] < 0) { t.lo[d] = -cg; t.ext[d] = cg; }
      else if (e.off[d] > 0) { t.lo[d] = nc; t.ext[d] = cg; }
      else { t.lo[d] = 0; t.ext[d] = nc; }
      int64_t lx = b.loc.x[d];
      int64_t a = lx + e.off[d];
      int64_t P = (a >= 0) ? a / 2 : -((-a + 1) / 2);
      t.so[d] = (int)(lx * nc - P * n[d]);
    }
  }
  t.ncell = t.ext[0] * t.ext[1] * t.ext[2];
  return t;
}

static bool region_physical(const BlockInfo& b, const int o[3]) {
  for (int d = 0; d < 3; ++d) {
    if (o[d] < 0 && b.phys_lo[d]) return true;
    if (o[d] > 0 && b.phys_hi[d]) return true;
  }
  return false;
}

/* One exchange plan of this rank (fill-in-one phases A-D, remote first).  cyc: per-cycle plan of
 * the direct-halo path -- drops the face copies between local same-level blocks (the stage kernel
 * reads those neighbours' interiors directly) and, on uniform meshes, all edge / corner regions
 * (the stage stencil is a plus shape: it never reads them). */
// Per-cycle plan of a block with coarse staging and no physical face: the staging cells of the first
// ghost layer at a non-coarser offset op that a prolongation actually reads.  The prolongation of the
// first ghost layer R_o at each coarser-neighbour offset o takes one minmod slope per dimension over
// +-1 coarse cell, so it reads R_o +- e_d; the part of that in op's ghost layer, as a bounding box in
// coarse coordinates [lo, hi).  false: nothing there is read.
static bool staging_need(const ph_mesh* m, const int kind[27], const int op[3], int lo[3], int hi[3]) {
  const int* nc = m->G.nc;
  int glo[3], ghi[3];
  for (int d = 0; d < 3; ++d) {
    glo[d] = op[d] < 0 ? -1 : (op[d] > 0 ? nc[d] : 0);
    ghi[d] = op[d] < 0 ? 0 : (op[d] > 0 ? nc[d] + 1 : nc[d]);
    lo[d] = 1 << 30;
    hi[d] = -(1 << 30);
  }
  bool any = false;
  for (int q = 0; q < 27; ++q) {
    if (q == 13 || kind[q] != -1) continue;
    const int o[3] = {q % 3 - 1, (q / 3) % 3 - 1, q / 9 - 1};
    int rlo[3], rhi[3];
    for (int d = 0; d < 3; ++d) {
      rlo[d] = o[d] < 0 ? -1 : (o[d] > 0 ? nc[d] : 0);
      rhi[d] = o[d] < 0 ? 0 : (o[d] > 0 ? nc[d] + 1 : nc[d]);
    }
    for (int d = 0; d < 3; ++d)
      for (int sgn = -1; sgn <= 1; sgn += 2) {
        int a[3], b[3];
        bool ok = true;
        for (int e = 0; e < 3; ++e) {
          a[e] = std::max(rlo[e] + (e == d ? sgn : 0), glo[e]);
          b[e] = std::min(rhi[e] + (e == d ? sgn : 0), ghi[e]);
          ok = ok && a[e] < b[e];
        }
        if (!ok) continue;
        any = true;
        for (int e = 0; e < 3; ++e) {
          lo[e] = std::min(lo[e], a[e]);
          hi[e] = std::max(hi[e], b[e]);
        }
      }
  }
  return any;
}

static bool any_physical(const BlockInfo& b) {
  for (int d = 0; d < 3; ++d)
    if (b.phys_lo[d] || b.phys_hi[d]) return true;
  return false;
}

// clip task t's destination box (fine cells) to the fine cells covering coarse box [clo, chi)
static void clip_to_coarse(XTask& t, const int clo[3], const int chi[3]) {
  for (int d = 0; d < 3; ++d) {
    const int a = std::max(t.lo[d], 2 * clo[d]), b = std::min(t.lo[d] + t.ext[d], 2 * chi[d]);
    t.lo[d] = a;
    t.ext[d] = std::max(b - a, 0);
  }
  t.ncell = t.ext[0] * t.ext[1] * t.ext[2];
}

static void build_exchange(ph_mesh* m, Plan& P, bool cyc, const std::vector<int>& cslot) {
  const int R = m->nranks, me = m->rank;
  for (Phase* ph : P.phases()) {
    ph->tasks.clear();
    ph->chunks.clear();
  }
  P.send_off.assign(R, 0);
  P.send_cnt.assign(R, 0);
  P.recv_off.assign(R, 0);
  P.recv_cnt.assign(R, 0);
  P.send_hash.assign(R, 0);
  P.recv_hash.assign(R, 0);
  // ---- phase A: per destination block (gid order), entries in canonical order
  std::vector<int64_t> soff(R, 0), roff(R, 0);
  std::vector<int> pack_peer, unpack_peer;
  for (auto& b : m->blocks) {
    for (auto& e : b.nbrs) {
      const BlockInfo& s = m->blocks[e.gid];
      bool dst_here = (b.rank == me), src_here = (s.rank == me);
      if (!dst_here && !src_here) continue;
      bool clip = false;
      int clo[3], chi[3];
      if (cyc && !b.has_coarser) {  // destination without coarse staging (all blocks of a uniform mesh)
        int nz = (e.off[0] != 0) + (e.off[1] != 0) + (e.off[2] != 0);
        if (nz > 1) continue;                               // edges / corners: never read
        if (dst_here && src_here && e.dlevel == 0) continue;  // read directly by the stage kernel
      } else if (cyc && b.has_coarser && e.dlevel >= 0 && !any_physical(b) && !getenv("PH_FULL_STAGING")) {
        // staged block: the stage kernel reads local same-level faces directly (direct halo); other
        // faces it reads whole; beyond that, only the ghosts a prolongation slope reads (through
        // their restriction into the staging's first ghost layer) are needed
        int nz = (e.off[0] != 0) + (e.off[1] != 0) + (e.off[2] != 0);
        const bool stage_reads = nz == 1 && !(dst_here && src_here && e.dlevel == 0);
        if (!stage_reads) {
          int kind[27];
          for (int q = 0; q < 27; ++q) kind[q] = -2;
          for (auto& f : b.nbrs) kind[(f.off[2] + 1) * 9 + (f.off[1] + 1) * 3 + (f.off[0] + 1)] = f.dlevel;
          const int op[3] = {e.off[0], e.off[1], e.off[2]};
          if (!staging_need(m, kind, op, clo, chi)) continue;
          clip = true;
        }
      }
      XTask t = entry_task(m, b, e);
      if (clip) {
        clip_to_coarse(t, clo, chi);
        if (t.ncell == 0) continue;
      }
      int cs = (t.kind == T_CCOPY) ? cslot[b.gid] : (int)b.local;
      if (dst_here && src_here) {
        t.dst_slot = cs;
        t.src_slot = (int)s.local;
        add_chunks(P.local, t, m->G);
      } else if (src_here) {  // pack for b.rank
        int peer = b.rank;
        t.dst_slot = -1;
        t.bc = -1;
        t.src_slot = (int)s.local;
        t.buf = soff[peer];
        soff[peer] += (int64_t)NVAR * t.ncell;
        P.send_hash[peer] = mix(P.send_hash[peer], (uint64_t)b.gid * 64 + (uint64_t)(&e - &b.nbrs[0]));
        pack_peer.push_back(peer);
        add_chunks(P.pack, t, m->G);
      } else {  // unpack from s.rank
        int peer = s.rank;
        t.kind = (t.kind == T_CCOPY) ? T_UNPACK_C : T_UNPACK_U;
        t.dst_slot = cs;
        t.src_slot = -1;
        t.buf = roff[peer];
        roff[peer] += (int64_t)NVAR * t.ncell;
        P.recv_hash[peer] = mix(P.recv_hash[peer], (uint64_t)b.gid * 64 + (uint64_t)(&e - &b.nbrs[0]));
        unpack_peer.push_back(peer);
        add_chunks(P.unpack, t, m->G);
      }
    }
  }
  // per-peer buffer offsets (peer-major)
  int64_t so = 0, ro = 0;
  for (int p = 0; p < R; ++p) {
    P.send_off[p] = so;
    P.send_cnt[p] = soff[p];
    so += soff[p];
    P.recv_off[p] = ro;
    P.recv_cnt[p] = roff[p];
    ro += roff[p];
  }
  for (size_t i = 0; i < P.pack.tasks.size(); ++i) P.pack.tasks[i].buf += P.send_off[pack_peer[i]];
  for (size_t i = 0; i < P.unpack.tasks.size(); ++i) P.unpack.tasks[i].buf += P.recv_off[unpack_peer[i]];
  P.sbuf_n = so;
  P.rbuf_n = ro;
  // ---- phases B, C, D per local block
  const int* n = m->G.n;
  const int g = m->G.g, cg = m->G.cg;
  for (int64_t gid : m->local_gids) {
    const BlockInfo& b = m->blocks[gid];
    int kind[27];
    for (int q = 0; q < 27; ++q) kind[q] = -2;
    for (auto& e : b.nbrs) kind[(e.off[2] + 1) * 9 + (e.off[1] + 1) * 3 + (e.off[0] + 1)] = e.dlevel;
    bool anyphys = false;
    for (int d = 0; d < 3; ++d) anyphys = anyphys || b.phys_lo[d] || b.phys_hi[d];
    int bits = bc_bits(m, b);
    if (b.has_coarser) {
      int cs = cslot[gid];
      // own interior into the staging -- only the coarse cells something reads: the prolongation of the
      // first ghost layer at each coarser-neighbour offset o takes minmod slopes over +-1 coarse cell, so
      // it reads the interior layer next to o (I_d = 0 for o_d < 0, nc_d - 1 for o_d > 0, all I_d for
      // o_d = 0); physical BCs on the staging mirror the cg interior layers next to each physical face.
      // A mask over the nc^3 staging interior, cut into disjoint boxes (x-runs merged over j, then k).
      // This phase is HBM-bound (it reads fine interior cells): round 1 restricted the whole 2-layer shell.
      const int* nc = m->G.nc;
      const int T = m->G.cg;
      auto restrict_box = [&](int lo0, int e0, int lo1, int e1, int lo2, int e2) {
        XTask t{};
        t.kind = T_CRESTRICT;
        t.dst_slot = cs;
        t.src_slot = (int)b.local;
        t.lo[0] = lo0; t.ext[0] = e0;
        t.lo[1] = lo1; t.ext[1] = e1;
        t.lo[2] = lo2; t.ext[2] = e2;
        t.ncell = e0 * e1 * e2;
        if (t.ncell > 0) add_chunks(P.b1, t, m->G);
      };
      if (getenv("PH_FULL_STAGING")) {
        restrict_box(0, nc[0], 0, nc[1], 0, nc[2]);
      } else {
        const int64_t NCV = (int64_t)nc[0] * nc[1] * nc[2];
        std::vector<uint8_t> need((size_t)NCV, 0);
        auto mark = [&](const int lo[3], const int hi[3]) {
          for (int k = std::max(lo[2], 0); k < std::min(hi[2], nc[2]); ++k)
            for (int j = std::max(lo[1], 0); j < std::min(hi[1], nc[1]); ++j)
              for (int i = std::max(lo[0], 0); i < std::min(hi[0], nc[0]); ++i)
                need[((size_t)k * nc[1] + j) * nc[0] + i] = 1;
        };
        for (int q = 0; q < 27; ++q) {
          if (q == 13 || kind[q] != -1) continue;
          const int o[3] = {q % 3 - 1, (q / 3) % 3 - 1, q / 9 - 1};
          int lo[3], hi[3];
          for (int d = 0; d < 3; ++d) {
            lo[d] = o[d] > 0 ? nc[d] - 1 : 0;
            hi[d] = o[d] < 0 ? 1 : nc[d];
          }
          mark(lo, hi);
        }
        for (int d = 0; d < 3; ++d) {
          for (int side = 0; side < 2; ++side) {
            if (!(side ? b.phys_hi[d] : b.phys_lo[d])) continue;
            int lo[3] = {0, 0, 0}, hi[3] = {nc[0], nc[1], nc[2]};
            if (side) lo[d] = nc[d] - T; else hi[d] = T;
            mark(lo, hi);
          }
        }
        // disjoint boxes: x-runs per (j, k) row, merged over consecutive j with the same run, then over
        // consecutive k with the same (run, j-range)
        struct Box { int i0, ie, j0, je, k0, ke; };
        std::vector<Box> prev, cur, done;
        for (int k = 0; k < nc[2]; ++k) {
          std::vector<Box> plane;
          for (int j = 0; j < nc[1]; ++j) {
            for (int i = 0; i < nc[0];) {
              if (!need[((size_t)k * nc[1] + j) * nc[0] + i]) { ++i; continue; }
              int e = i;
              while (e < nc[0] && need[((size_t)k * nc[1] + j) * nc[0] + e]) ++e;
              bool merged = false;
              for (Box& bx : plane)
                if (bx.i0 == i && bx.ie == e && bx.je == j) { bx.je = j + 1; merged = true; break; }
              if (!merged) plane.push_back(Box{i, e, j, j + 1, k, k + 1});
              i = e;
            }
          }
          cur.clear();
          for (Box bx : plane) {
            bool merged = false;
            for (Box& pb : prev)
              if (pb.i0 == bx.i0 && pb.ie == bx.ie && pb.j0 == bx.j0 && pb.je == bx.je && pb.ke == k) {
                pb.ke = k + 1;
                cur.push_back(pb);
                pb.ke = -1;  // moved to cur
                merged = true;
                break;
              }
            if (!merged) cur.push_back(bx);
          }
          for (Box& pb : prev)
            if (pb.ke >= 0) done.push_back(pb);
          prev.swap(cur);
        }
        for (Box& pb : prev) done.push_back(pb);
        for (const Box& bx : done)
          restrict_box(bx.i0, bx.ie - bx.i0, bx.j0, bx.je - bx.j0, bx.k0, bx.ke - bx.k0);
      }
      const bool clip1 = cyc && !anyphys && !getenv("PH_FULL_STAGING");
      for (int q = 0; q < 27; ++q) {
        if (q == 13 || kind[q] == -2 || kind[q] == -1) continue;
        int o[3] = {q % 3 - 1, (q / 3) % 3 - 1, q / 9 - 1};
        XTask r{};
        r.kind = T_CRESTRICT;
        r.dst_slot = cs;
        r.src_slot = (int)b.local;
        for (int d = 0; d < 3; ++d) {
          if (o[d] < 0) { r.lo[d] = -1; r.ext[d] = 1; }
          else if (o[d] > 0) { r.lo[d] = m->G.nc[d]; r.ext[d] = 1; }
          else { r.lo[d] = 0; r.ext[d] = m->G.nc[d]; }
          r.so[d] = 0;
        }
        if (clip1) {  // per-cycle plan: only the staging cells a prolongation slope reads (staging_need)
          int clo[3], chi[3];
          if (!staging_need(m, kind, o, clo, chi)) continue;
          for (int d = 0; d < 3; ++d) {
            const int a = std::max(r.lo[d], clo[d]), e2 = std::min(r.lo[d] + r.ext[d], chi[d]);
            r.lo[d] = a;
            r.ext[d] = std::max(e2 - a, 0);
          }
        }
        r.ncell = r.ext[0] * r.ext[1] * r.ext[2];
        if (r.ncell > 0) add_chunks(P.b1, r, m->G);
      }
      for (int q = 0; q < 27 && anyphys; ++q) {
        if (q == 13) continue;
        int o[3] = {q % 3 - 1, (q / 3) % 3 - 1, q / 9 - 1};
        if (!region_physical(b, o)) continue;
        XTask r{};
        r.kind = T_BC_COARSE;
        r.dst_slot = cs;
        r.src_slot = cs;
        r.bc = bits;
        for (int d = 0; d < 3; ++d) {
          if (o[d] < 0) { r.lo[d] = -cg; r.ext[d] = cg; }
          else if (o[d] > 0) { r.lo[d] = m->G.nc[d]; r.ext[d] = cg; }
          else { r.lo[d] = 0; r.ext[d] = m->G.nc[d]; }
        }
        r.ncell = r.ext[0] * r.ext[1] * r.ext[2];
        add_chunks(P.b2, r, m->G);
      }
      for (int q = 0; q < 27; ++q) {
        if (q == 13 || kind[q] != -1) continue;
        int o[3] = {q % 3 - 1, (q / 3) % 3 - 1, q / 9 - 1};
        XTask r{};
        r.kind = T_PROLONG;
        r.dst_slot = (int)b.local;
        r.src_slot = cs;
        for (int d = 0; d < 3; ++d) {
          if (o[d] < 0) { r.lo[d] = -1; r.ext[d] = 1; }
          else if (o[d] > 0) { r.lo[d] = m->G.nc[d]; r.ext[d] = 1; }
          else { r.lo[d] = 0; r.ext[d] = m->G.nc[d]; }
        }
        r.ncell = r.ext[0] * r.ext[1] * r.ext[2];
        add_chunks(P.pro, r, m->G);
      }
    }
    if (anyphys) {
      for (int q = 0; q < 27; ++q) {
        if (q == 13) continue;
        int o[3] = {q % 3 - 1, (q / 3) % 3 - 1, q / 9 - 1};
        if (!region_physical(b, o)) continue;
        if (cyc && !b.has_coarser && ((o[0] != 0) + (o[1] != 0) + (o[2] != 0)) > 1) continue;
        XTask r{};
        r.kind = T_BC_FINE;
        r.dst_slot = (int)b.local;
        r.src_slot = (int)b.local;
        r.bc = bits;
        for (int d = 0; d < 3; ++d) {
          if (o[d] < 0) { r.lo[d] = -g; r.ext[d] = g; }
          else if (o[d] > 0) { r.lo[d] = n[d]; r.ext[d] = g; }
          else { r.lo[d] = 0; r.ext[d] = n[d]; }
        }
        r.ncell = r.ext[0] * r.ext[1] * r.ext[2];
        add_chunks(P.bcf, r, m->G);
      }
    }
  }
}

/* Slots, staging / face-flux slots, block metadata, reflux tasks and both exchange plans. */
static ph_status build_plan(ph_mesh* m) {
  const int me = m->rank;
  for (int d = 0; d < 3; ++d) m->reflux[d].clear();
  m->cross_rank_reflux = false;
  // slots
  m->local_gids.clear();
  for (auto& b : m->blocks)
    if (b.rank == me) m->local_gids.push_back(b.gid);
  const int64_t nloc = (int64_t)m->local_gids.size();
  // coarse staging and face-flux slots
  std::vector<int> cslot(m->blocks.size(), -1);
  std::vector<std::array<int, 6>> fslot(m->blocks.size());
  m->n_cslots = 0;
  m->n_fslots = 0;
  m->multilevel = false;
  for (auto& b : m->blocks) {
    fslot[b.gid].fill(-1);
    for (auto& e : b.nbrs)
      if (e.dlevel != 0) m->multilevel = true;
  }
  for (auto& b : m->blocks) {
    if (b.rank != me) continue;
    if (b.has_coarser) cslot[b.gid] = m->n_cslots++;
    for (auto& e : b.nbrs) {
      int nz = (e.off[0] != 0) + (e.off[1] != 0) + (e.off[2] != 0);
      if (nz != 1 || e.dlevel == 0) continue;
      int d = e.off[0] ? 0 : (e.off[1] ? 1 : 2);
      int face = 2 * d + (e.off[d] > 0 ? 1 : 0);
      if (fslot[b.gid][face] < 0) fslot[b.gid][face] = m->n_fslots++;
    }
  }
  m->ho = m->G.g == 3;
  m->G.exact = m->ho ? 1 : 0;
  // direct halo: stage kernels (and the AMR tag kernel) of blocks without a coarser neighbour read
  // their local same-level face neighbours' interiors; blocks with coarse staging keep every ghost
  // (their staging restricts first-layer ghosts incl. edges and corners, O7 B)
  m->direct_halo = !m->no_direct_halo && !m->ho;
  build_exchange(m, m->plan[0], false, cslot);
  build_exchange(m, m->plan[1], m->direct_halo, cslot);
  if (const char* dump = getenv("PH_PLAN_DUMP")) {  // diagnostics: tasks / cells per phase and task kind
    if (FILE* f = fopen(dump, "a")) {
      const char* names[] = {"pack", "local", "unpack", "b1", "b2", "pro", "bcf"};
      for (int pi = 0; pi < 2; ++pi) {
        auto ph = m->plan[pi].phases();
        for (size_t q = 0; q < ph.size(); ++q) {
          int64_t nt[16] = {0}, nc[16] = {0};
          for (const XTask& t : ph[q]->tasks) {
            nt[t.kind & 15]++;
            nc[t.kind & 15] += t.ncell;
          }
          for (int k = 0; k < 16; ++k)
            if (nt[k])
              fprintf(f, "{\"plan\": %d, \"phase\": \"%s\", \"kind\": %d, \"tasks\": %lld, \"cells\": %lld, "
                         "\"chunks\": %d}\n", pi, names[q], k, (long long)nt[k], (long long)nc[k], ph[q]->nchunks());
        }
      }
      fclose(f);
    }
  }
  // reflux tasks (coarse side) and, across ranks, the fine-side flux packs (O8).
  // Per (sender, receiver) pair both ranks enumerate coarse blocks in gid order and their finer
  // face entries in canonical order, so buffer offsets agree without any handshake.
  const int* n = m->G.n;
  const int R = m->nranks;
  m->fpack.clear();
  std::vector<int64_t> fso(R, 0), fro(R, 0);
  std::vector<int> fpack_peer;
  std::vector<std::pair<int, size_t>> rflux_peer;  // (peer, index into reflux[d]) for rebasing
  for (auto& b : m->blocks) {
    for (auto& e : b.nbrs) {
      int nz = (e.off[0] != 0) + (e.off[1] != 0) + (e.off[2] != 0);
      if (nz != 1 || e.dlevel != 1) continue;
      int d = e.off[0] ? 0 : (e.off[1] ? 1 : 2);
      const BlockInfo& f = m->blocks[e.gid];
      int ta = (d == 0) ? 1 : 0, tb = (d == 2) ? 1 : 2;
      int64_t qsize = (int64_t)NVAR * (n[ta] / 2) * (n[tb] / 2);
      int ffs_face = 2 * d + (e.off[d] > 0 ? 0 : 1);
      if (b.rank == me) {
        RefluxTask rt{};
        rt.cslot = (int)b.local;
        rt.dir = d;
        rt.side = e.off[d];
        rt.cfs = fslot[b.gid][2 * d + (e.off[d] > 0 ? 1 : 0)];
        rt.t0lo = e.fine[0] * n[ta] / 2;
        rt.t1lo = e.fine[1] * n[tb] / 2;
        if (f.rank == me) {
          rt.ffs = fslot[e.gid][ffs_face];
          rt.roff = -1;
        } else {
          rt.ffs = -1;
          rt.roff = fro[f.rank];
          fro[f.rank] += qsize;
          rflux_peer.push_back({f.rank, 0});
          rflux_peer.back().second = ((size_t)d << 32) | m->reflux[d].size();
        }
        m->reflux[d].push_back(rt);
      } else if (f.rank == me) {
        FluxPackTask ft{};
        ft.ffs = fslot[e.gid][ffs_face];
        ft.dir = d;
        ft.off = fso[b.rank];
        fso[b.rank] += qsize;
        fpack_peer.push_back(b.rank);
        m->fpack.push_back(ft);
      }
    }
  }
  m->fsend_off.assign(R, 0);
  m->fsend_cnt.assign(R, 0);
  m->frecv_off.assign(R, 0);
  m->frecv_cnt.assign(R, 0);
  int64_t fs_acc = 0, fr_acc = 0;
  for (int p = 0; p < R; ++p) {
    m->fsend_off[p] = fs_acc;
    m->fsend_cnt[p] = fso[p];
    fs_acc += fso[p];
    m->frecv_off[p] = fr_acc;
    m->frecv_cnt[p] = fro[p];
    fr_acc += fro[p];
  }
  for (size_t i = 0; i < m->fpack.size(); ++i) m->fpack[i].off += m->fsend_off[fpack_peer[i]];
  for (auto& pr : rflux_peer) {
    int d = (int)(pr.second >> 32);
    size_t idx = pr.second & 0xffffffffu;
    m->reflux[d][idx].roff += m->frecv_off[pr.first];
  }
  m->fsbuf_n = fs_acc;
  m->frbuf_n = fr_acc;
  // block metadata
  m->meta.assign(nloc, BlockMeta{});
  for (int64_t s = 0; s < nloc; ++s) {
    const BlockInfo& b = m->blocks[m->local_gids[s]];
    BlockMeta& M = m->meta[s];
    for (int d = 0; d < 3; ++d) {
      M.idx[d] = 1.0 / b.dx[d];
      M.dx[d] = b.dx[d];
      M.xmin[d] = b.xmin[d];
    }
    M.dV = (b.dx[0] * b.dx[1]) * b.dx[2];
    M.gid = b.gid;
    M.level = b.loc.level;
    M.cslot = cslot[b.gid];
    for (int f = 0; f < 6; ++f) {
      M.fslot[f] = fslot[b.gid][f];
      M.nb[f] = -1;
      M.prank[f] = -1;
      M.poff[f] = 0;
    }
    M.rfx = 0;
    // direct halo: every block (with coarse staging too, since round 2) reads its local same-level face
    // neighbours' interiors; the per-cycle plan copies those faces only where the staging needs them
    if (m->direct_halo && (!b.has_coarser || (!any_physical(b) && !getenv("PH_FULL_STAGING")))) {
      for (auto& e : b.nbrs) {
        int nz = (e.off[0] != 0) + (e.off[1] != 0) + (e.off[2] != 0);
        if (nz != 1 || e.dlevel != 0 || m->blocks[e.gid].rank != me) continue;
        int d = e.off[0] ? 0 : (e.off[1] ? 1 : 2);
        M.nb[2 * d + (e.off[d] > 0 ? 1 : 0)] = (int)m->blocks[e.gid].local;
      }
    }
  }
  // faces receiving flux correction (coarse side): their first cell layer is reduced after the reflux
  m->rfx_faces.clear();
  for (int d = 0; d < 3; ++d)
    for (const RefluxTask& rt : m->reflux[d]) m->meta[rt.cslot].rfx |= 1 << (2 * rt.dir + (rt.side > 0 ? 1 : 0));
  for (int64_t s = 0; s < nloc; ++s)
    for (int f = 0; f < 6; ++f)
      if ((m->meta[s].rfx >> f) & 1) m->rfx_faces.push_back(make_int2((int)s, f));
  // stage launch order: with the multi-GPU direct halo, blocks that have no remote or physical
  // face come first so their stage can run while the halo exchange is in flight
  m->overlap = m->direct_halo && m->nranks > 1 && !m->multilevel && m->cfg.refinement != PH_REF_ADAPTIVE;
  m->slot_order.clear();
  std::vector<int> bnd;
  for (int64_t s = 0; s < nloc; ++s) {
    const BlockInfo& b = m->blocks[m->local_gids[s]];
    bool boundary = false;
    for (int d = 0; d < 3; ++d) boundary = boundary || b.phys_lo[d] || b.phys_hi[d];
    for (auto& e : b.nbrs) {
      int nz = (e.off[0] != 0) + (e.off[1] != 0) + (e.off[2] != 0);
      if (nz == 1 && m->blocks[e.gid].rank != me) boundary = true;
    }
    if (m->overlap && boundary) bnd.push_back((int)s);
    else m->slot_order.push_back((int)s);
  }
  m->n_int = m->overlap ? (int)m->slot_order.size() : (int)nloc;
  for (int s : bnd) m->slot_order.push_back(s);
  return PH_OK;
}

static ph_status upload_phase(ph_mesh* m, Phase& P) {
  TRY(upload(m, &P.d_tasks, P.tasks));
  TRY(upload(m, &P.d_chunks, P.chunks));
  return PH_OK;
}

/* (Re)allocate every device structure that depends on the mesh (creation and remesh). */
static ph_status setup_device(ph_mesh* m) {
  const int64_t nloc = (int64_t)m->local_gids.size();
  const Geom& G = m->G;
  TRY(dalloc(m, (void**)&m->U0, (size_t)std::max<int64_t>(nloc, 1) * G.bstride * sizeof(double)));
  TRY(dalloc(m, (void**)&m->U1, (size_t)std::max<int64_t>(nloc, 1) * G.bstride * sizeof(double)));
  CU(cudaMemsetAsync(m->U0, 0, (size_t)std::max<int64_t>(nloc, 1) * G.bstride * sizeof(double), m->stream));
  CU(cudaMemsetAsync(m->U1, 0, (size_t)std::max<int64_t>(nloc, 1) * G.bstride * sizeof(double), m->stream));
  if (m->n_cslots) TRY(dalloc(m, (void**)&m->C, (size_t)m->n_cslots * G.cbstride * sizeof(double)));
  if (m->n_fslots) TRY(dalloc(m, (void**)&m->fbuf, (size_t)m->n_fslots * G.fstride * sizeof(double)));
  TRY(upload(m, &m->d_meta, m->meta));
  TRY(upload(m, &m->d_slots, m->slot_order));
  for (Plan& pl : m->plan)
    for (Phase* P : pl.phases()) TRY(upload_phase(m, *P));
  m->sbuf_n = std::max(m->plan[0].sbuf_n, m->plan[1].sbuf_n);
  m->rbuf_n = std::max(m->plan[0].rbuf_n, m->plan[1].rbuf_n);
  for (int d = 0; d < 3; ++d) TRY(upload(m, &m->d_reflux[d], m->reflux[d]));
  TRY(upload(m, &m->d_fpack, m->fpack));
  if (m->fsbuf_n) TRY(dalloc(m, (void**)&m->fsbuf, m->fsbuf_n * sizeof(double)));
  if (m->frbuf_n) TRY(dalloc(m, (void**)&m->frbuf, m->frbuf_n * sizeof(double)));
  if (m->sbuf_n) TRY(dalloc(m, (void**)&m->sbuf, m->sbuf_n * sizeof(double)));
  if (m->rbuf_n) TRY(dalloc(m, (void**)&m->rbuf, m->rbuf_n * sizeof(double)));
  // stage launch geometry.  A mesh of fewer than 8 stage2 tiles (16 x 16 columns) in total -- config 1,
  // one 32^3 block, has 4 -- runs the round-1 kernel, whose lighter prologue suits the k-split CTAs of
  // a few planes such a mesh needs (config 1: 24.9 vs 28.1 us per cycle).  Decided on the global block
  // count, so every rank and every rank count pick the same kernel (N GPUs stay bitwise equal to one).
  m->G.no_stage2 = ((int64_t)m->blocks.size() * (G.n[0] / 16) * (G.n[1] / 16) < 8) ? 1 : 0;
  int tile_x = TX, tile_y = TY;
  const bool full_tile = stage_tile(G, m->cfg.recon, m->fbuf != nullptr, &tile_x, &tile_y);
  m->ntx = (G.n[0] + tile_x - 1) / tile_x;
  m->nty = (G.n[1] + tile_y - 1) / tile_y;
  int64_t base = std::max<int64_t>(nloc, 1) * m->ntx * m->nty;
  // split the k-march of small meshes until ~8 CTAs per SM exist, down to min_kc planes per CTA
  const int min_kc = getenv("PH_MIN_KC") ? std::max(1, atoi(getenv("PH_MIN_KC"))) : 1;
  int nkc = 1;
  while (base * nkc < 1184 && G.n[2] / (nkc * 2) >= min_kc) nkc *= 2;
  m->KC = (G.n[2] + nkc - 1) / nkc;
  m->nkc = (G.n[2] + m->KC - 1) / m->KC;
  m->pack_size = (m->cfg.pack_size > 0) ? (int)std::min<int64_t>(m->cfg.pack_size, nloc) : (int)nloc;
  m->stage_ctas = (int)(nloc * m->ntx * m->nty * m->nkc);
  if (m->ho) {
    // generic high-order path: primitives of the whole pool + face fluxes per direction
    const int64_t nf[3] = {(int64_t)(G.n[0] + 1) * G.n[1] * G.n[2], (int64_t)G.n[0] * (G.n[1] + 1) * G.n[2],
                           (int64_t)G.n[0] * G.n[1] * (G.n[2] + 1)};
    const int64_t ns = std::max<int64_t>(nloc, 1);
    TRY(dalloc(m, (void**)&m->Wpool, (size_t)ns * G.bstride * sizeof(double)));
    TRY(dalloc(m, (void**)&m->Fxb, (size_t)ns * NVAR * nf[0] * sizeof(double)));
    TRY(dalloc(m, (void**)&m->Fyb, (size_t)ns * NVAR * nf[1] * sizeof(double)));
    TRY(dalloc(m, (void**)&m->Fzb, (size_t)ns * NVAR * nf[2] * sizeof(double)));
    m->stage_ctas = (int)(nloc * G.n[2]);
  }
  // stage-2 base pool: on the uniform full-tile minmod path (the kernels' H template), not under
  // flux correction (it would also have to correct H) nor AMR
  m->Hpool = nullptr;
  // stage2.cu needs H (also on multilevel / AMR meshes, where the reflux corrects H with U^1); the round-1
  // kernel (PH_STAGE_V1=1) has no H on multilevel meshes
  const bool s2 = stage2_applies(G, m->cfg.recon, m->fbuf != nullptr);
  if (!m->ho && full_tile && !getenv("PH_NO_HBASE") &&
      (s2 || (!m->multilevel && m->cfg.refinement != PH_REF_ADAPTIVE)))
    TRY(dalloc(m, (void**)&m->Hpool, (size_t)std::max<int64_t>(nloc, 1) * G.bstride * sizeof(double)));
  m->partials_n = std::max<int64_t>({(int64_t)m->stage_ctas + (int64_t)m->rfx_faces.size(), nloc * G.n[2],
                                      nloc * tag_ctas_per_block(G), 1});
  TRY(upload(m, &m->d_rfx_faces, m->rfx_faces));
  TRY(dalloc(m, (void**)&m->partials, m->partials_n * 6 * sizeof(double)));
  CU(cudaMemsetAsync(m->partials, 0, m->partials_n * 6 * sizeof(double), m->stream));
  {
    const int64_t nglob = (int64_t)m->blocks.size();
    const int64_t maxloc = std::max<int64_t>((nglob + m->nranks - 1) / m->nranks, 1);
    TRY(dalloc(m, (void**)&m->d_eps, (size_t)maxloc * sizeof(unsigned long long)));
    CU(cudaMemsetAsync(m->d_eps, 0, (size_t)maxloc * sizeof(unsigned long long), m->stream));
    if (m->nranks > 1)
      TRY(dalloc(m, (void**)&m->d_eps_all, (size_t)maxloc * m->nranks * sizeof(unsigned long long)));
  }
  TRY(dalloc(m, (void**)&m->stage_buf, (size_t)std::max<int64_t>(nloc, 1) * NVAR * G.n[0] * G.n[1] * G.n[2] * sizeof(double)));
  return PH_OK;
}

/* Peer transport set-up (collective; after build_plan).  Each rank cudaMallocs [64 flags | recv
 * half 0 | recv half 1] (each half sized for the per-cycle plan), exports it with CUDA IPC and
 * allgathers handle, half size and its per-source receive offsets over NCCL; then maps the regions
 * of the peers it sends to.  The ranks agree (NCCL min) on whether every mapping succeeded; if not,
 * *ok = false and the halo stays on NCCL.  On success the per-cycle pack tasks become puts: each
 * writes at the offset the receiving rank's unpack task reads.  Flags are zeroed before the
 * agreement, so no peer can signal into them earlier. */
static void host_barrier(ph_mesh* m);

/* Undo setup_peer (collective): nobody may still write into my region or read through a mapping when
 * it goes -- every rank drains its stream and meets the others before and after unmapping. */
static void teardown_peer(ph_mesh* m) {
  if (!m->peer_region) return;
  cudaStreamSynchronize(m->stream);
  host_barrier(m);
  for (void* p : m->peer_open)
    if (p) cudaIpcCloseMemHandle(p);
  m->peer_open.clear();
  host_barrier(m);
  cudaFree(m->peer_region);
  m->peer_region = nullptr;
  m->my_flags = nullptr;
  m->peer = false;
}

static ph_status setup_peer(ph_mesh* m, bool* ok_out) {
  *ok_out = false;
  const int R = m->nranks, me = m->rank;
  Plan& PL = m->plan[1];
  const int64_t rb = std::max<int64_t>(PL.rbuf_n, 1);
  struct Rec {
    cudaIpcMemHandle_t h;
    int64_t rb;
    int32_t ok, pad;
    int64_t recv_off[64];
  };
  Rec mine{};
  mine.rb = rb;
  mine.ok = 1;
  for (int p = 0; p < R; ++p) mine.recv_off[p] = PL.recv_off[p];
  const size_t flag_bytes = 64 * sizeof(unsigned long long);
  if (cudaMalloc(&m->peer_region, flag_bytes + 2 * (size_t)rb * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    m->peer_region = nullptr;
    mine.ok = 0;
  } else if (cudaIpcGetMemHandle(&mine.h, m->peer_region) != cudaSuccess) {
    cudaGetLastError();
    mine.ok = 0;
  }
  if (m->peer_region) {
    m->my_flags = (unsigned long long*)m->peer_region;
    CU(cudaMemsetAsync(m->my_flags, 0, flag_bytes, m->stream));
  }
  m->send_mask = m->recv_mask = 0;
  for (int p = 0; p < R; ++p) {
    if (p == me) continue;
    if (PL.send_cnt[p] > 0) m->send_mask |= 1ull << p;
    if (PL.recv_cnt[p] > 0) m->recv_mask |= 1ull << p;
  }
  if (!m->d_peer_rec) TRY(dalloc(m, &m->d_peer_rec, (size_t)(R + 1) * sizeof(Rec), true));  // once (remesh re-runs this)
  void* dbuf = m->d_peer_rec;
  CU(cudaMemcpyAsync((char*)dbuf + (size_t)R * sizeof(Rec), &mine, sizeof(Rec), cudaMemcpyHostToDevice, m->stream));
  NC(ncclAllGather((char*)dbuf + (size_t)R * sizeof(Rec), dbuf, sizeof(Rec), ncclUint8, m->comm, m->stream));
  std::vector<Rec> all(R);
  CU(cudaMemcpyAsync(all.data(), dbuf, (size_t)R * sizeof(Rec), cudaMemcpyDeviceToHost, m->stream));
  CU(cudaStreamSynchronize(m->stream));
  int32_t ok = 1;
  m->peer_open.assign(R, nullptr);
  for (int p = 0; p < R; ++p) {
    if (!all[p].ok) ok = 0;
    if (p == me || !all[p].ok || !m->peer_region || !((m->send_mask >> p) & 1ull)) continue;
    void* ptr = nullptr;
    if (cudaIpcOpenMemHandle(&ptr, all[p].h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess) m->peer_open[p] = ptr;
    else {
      cudaGetLastError();
      ok = 0;
    }
  }
  int32_t* dok = (int32_t*)dbuf;
  CU(cudaMemcpyAsync(dok, &ok, sizeof ok, cudaMemcpyHostToDevice, m->stream));
  NC(ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, m->comm, m->stream));
  CU(cudaMemcpyAsync(&ok, dok, sizeof ok, cudaMemcpyDeviceToHost, m->stream));
  CU(cudaStreamSynchronize(m->stream));
  if (!ok) {
    for (void* p : m->peer_open)
      if (p) cudaIpcCloseMemHandle(p);
    m->peer_open.clear();
    if (m->peer_region) cudaFree(m->peer_region);
    m->peer_region = nullptr;
    m->my_flags = nullptr;
    return PH_OK;
  }
  std::vector<double*> h0(R, nullptr), h1(R, nullptr);
  std::vector<unsigned long long*> fl(R, nullptr);
  for (int p = 0; p < R; ++p) {
    char* base = (char*)(p == me ? m->peer_region : m->peer_open[p]);
    if (!base) continue;
    fl[p] = (unsigned long long*)base;
    h0[p] = (double*)(base + flag_bytes);
    h1[p] = (double*)(base + flag_bytes + (size_t)all[p].rb * sizeof(double));
  }
  m->my_rbuf[0] = h0[me];
  m->my_rbuf[1] = h1[me];
  if (!m->d_prbuf[0]) {
    TRY(dalloc(m, (void**)&m->d_prbuf[0], R * sizeof(double*), true));
    TRY(dalloc(m, (void**)&m->d_prbuf[1], R * sizeof(double*), true));
    TRY(dalloc(m, (void**)&m->d_pflags, R * sizeof(void*), true));
    TRY(dalloc(m, (void**)&m->d_ctr, 2 * sizeof(unsigned long long), true));
  }
  CU(cudaMemcpyAsync(m->d_prbuf[0], h0.data(), R * sizeof(double*), cudaMemcpyHostToDevice, m->stream));
  CU(cudaMemcpyAsync(m->d_prbuf[1], h1.data(), R * sizeof(double*), cudaMemcpyHostToDevice, m->stream));
  CU(cudaMemcpyAsync(m->d_pflags, fl.data(), R * sizeof(void*), cudaMemcpyHostToDevice, m->stream));
  CU(cudaMemsetAsync(m->d_ctr, 0, 2 * sizeof(unsigned long long), m->stream));
  CU(cudaStreamSynchronize(m->stream));
  // per-cycle pack tasks -> puts at the receiver's offsets (both sides enumerate in the same order)
  for (XTask& t : PL.pack.tasks) {
    int p = 0;
    while (p + 1 < R && t.buf >= PL.send_off[p] + PL.send_cnt[p]) ++p;
    t.bc = p;
    t.buf = t.buf - PL.send_off[p] + all[p].recv_off[me];
  }
  // fused put (PH_FUSED_PUT=1): on the full-tile path the boundary blocks' stage kernel stores its g
  // boundary layers itself, as cells are finished, instead of a separate put kernel.  Correct (bitwise
  // vs 1 GPU) but slower at N = 4 (2b -3.5 %, config 4 -7 %, profiles/r01_multi_gpu_halo.md): the
  // x-face layers are 16 B per row, so those remote stores are fine-grained and add to the stage
  // kernel's store pressure, while the put kernel writes the packed faces as 256-B warp stores.
  // Each per-cycle pack task is one face of one block (uniform mesh: faces only), whose source shift
  // so names the face -- so[d] = +n: the sender's +d layers, -n: its -d layers.
  int tx = 0, ty = 0;
  m->fused_put = getenv("PH_FUSED_PUT") && atoi(getenv("PH_FUSED_PUT")) != 0 && !m->multilevel &&
                 stage_tile(m->G, m->cfg.recon, false, &tx, &ty);
  for (const XTask& t : PL.pack.tasks) {
    int d = 0;
    while (d < 2 && t.so[d] == 0) ++d;
    if (t.kind != T_COPY || t.so[d] == 0 || t.ext[d] != m->G.g) m->fused_put = false;  // not a plain face
    if (!m->fused_put) break;
    BlockMeta& M = m->meta[t.src_slot];
    const int f = 2 * d + (t.so[d] > 0 ? 1 : 0);
    M.prank[f] = t.bc;
    M.poff[f] = t.buf;
  }
  if (!m->fused_put)
    for (BlockMeta& M : m->meta)
      for (int f = 0; f < 6; ++f) M.prank[f] = -1;
  *ok_out = true;
  return PH_OK;
}

/* Host-side rendezvous of all ranks (teardown of the peer mappings). */
static void host_barrier(ph_mesh* m) {
  if (m->nranks < 2 || !m->comm || !m->my6) return;
  ncclAllReduce(m->my6, m->my6 + 1, 1, ncclDouble, ncclSum, m->comm, m->stream);
  cudaStreamSynchronize(m->stream);
}

static ph_status setup_persistent(ph_mesh* m) {
  TRY(dalloc(m, (void**)&m->my6, 8 * sizeof(double), true));
  TRY(dalloc(m, (void**)&m->all6, (size_t)6 * m->nranks * sizeof(double), true));
  TRY(dalloc(m, (void**)&m->tot5, 8 * sizeof(double), true));
  TRY(dalloc(m, (void**)&m->hist, (size_t)m->hist_cap * 7 * sizeof(double), true));
  TRY(dalloc(m, (void**)&m->d_st, sizeof(CycleState), true));
  TRY(dalloc(m, (void**)&m->d_err, sizeof(ErrWord), true));
  CU(cudaMemsetAsync(m->d_st, 0, sizeof(CycleState), m->stream));
  CU(cudaMemsetAsync(m->d_err, 0, sizeof(ErrWord), m->stream));
  return PH_OK;
}

static ph_status check_err(const ph_mesh* m) {
  if (m->host_only) return PH_OK;
  CU(cudaStreamSynchronize(m->stream));
  ErrWord e;
  CU(cudaMemcpy(&e, m->d_err, sizeof(e), cudaMemcpyDeviceToHost));
  if (e.flag) {
    char buf[256];
    if (e.stage == -2) {
      snprintf(buf, sizeof buf, "peer-halo barrier timed out waiting for rank %lld", (long long)e.gid);
      return fail(PH_ERR_COMM, buf);
    }
    snprintf(buf, sizeof buf, "non-positive density or pressure at gid %lld cell (k,j,i)=(%d,%d,%d) stage %d",
             (long long)e.gid, e.k, e.j, e.i, e.stage);
    return fail(PH_ERR_PHYSICS, buf);
  }
  return PH_OK;
}

/* ------------------------------------------------------------------------------- exchange */
static cudaEvent_t pool_event(ph_mesh* m) {
  cudaEvent_t e;
  cudaEventCreate(&e);
  m->ev_pool.push_back(e);
  return e;
}

/* Exchange, split in two so that compute can run between them (O7; remote buffers first,
 * P:1279-1285).  begin: pack remote buffers and start the grouped NCCL send/recv on the comm
 * stream.  end: rank-local fills, unpack, staging completion, prolongation, physical BCs. */
static ph_status exchange_begin(ph_mesh* m, double* U, int which) {
  Plan& PL = m->plan[which];
  const bool remote = (m->nranks > 1) && (PL.sbuf_n > 0 || PL.rbuf_n > 0);
  if (!remote) return PH_OK;
  XArgs a{};
  a.U = U;
  a.C = m->C;
  a.sbuf = m->sbuf;
  a.rbuf = m->rbuf;
  const bool put = m->peer && which == 1;  // peer transport: pack straight into the peers' receive halves
  if (put) a.peer_rbuf = m->d_prbuf[U == m->U1 ? 0 : 1];
  if (PL.pack.nchunks() && !(put && m->fused_put)) {  // fused: the boundary stage kernel stored them
    a.tasks = PL.pack.d_tasks;
    a.chunks = PL.pack.d_chunks;
    CU(launch_xfill(PL.pack.nchunks(), a, m->G, m->stream));
    m->launches++;
  }
  if (put) {
    CU(launch_peer_signal(m->d_pflags, m->d_ctr, m->rank, m->send_mask, m->stream));
    m->launches++;
    return PH_OK;
  }
  CU(cudaEventRecord(m->ev_pack, m->stream));
  CU(cudaStreamWaitEvent(m->comm_stream, m->ev_pack, 0));
  NC(ncclGroupStart());
  for (int p = 0; p < m->nranks; ++p) {
    if (p == m->rank) continue;
    if (PL.send_cnt[p]) NC(ncclSend(m->sbuf + PL.send_off[p], PL.send_cnt[p], ncclDouble, p, m->comm, m->comm_stream));
    if (PL.recv_cnt[p]) NC(ncclRecv(m->rbuf + PL.recv_off[p], PL.recv_cnt[p], ncclDouble, p, m->comm, m->comm_stream));
  }
  NC(ncclGroupEnd());
  CU(cudaEventRecord(m->ev_comm, m->comm_stream));
  return PH_OK;
}

static ph_status exchange_end(ph_mesh* m, double* U, int which) {
  Plan& PL = m->plan[which];
  const bool remote = (m->nranks > 1) && (PL.sbuf_n > 0 || PL.rbuf_n > 0);
  XArgs a{};
  a.U = U;
  a.C = m->C;
  a.sbuf = m->sbuf;
  a.rbuf = m->rbuf;
  auto run = [&](Phase& P) -> ph_status {
    if (P.nchunks() == 0) return PH_OK;
    a.tasks = P.d_tasks;
    a.chunks = P.d_chunks;
    CU(launch_xfill(P.nchunks(), a, m->G, m->stream));
    m->launches++;
    return PH_OK;
  };
  TRY(run(PL.local));
  if (remote) {
    if (m->peer && which == 1) {
      CU(launch_peer_wait(m->my_flags, m->d_ctr + 1, m->recv_mask, m->d_err, m->stream));
      m->launches++;
      a.rbuf = m->my_rbuf[U == m->U1 ? 0 : 1];
    } else {
      CU(cudaStreamWaitEvent(m->stream, m->ev_comm, 0));
    }
    TRY(run(PL.unpack));
  }
  TRY(run(PL.b1));
  TRY(run(PL.b2));
  TRY(run(PL.pro));
  TRY(run(PL.bcf));
  return PH_OK;
}

static ph_status exchange(ph_mesh* m, double* U, int which) {
  NvtxRange nvtx_("ph:exchange");
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  if (m->timing) {
    t0 = pool_event(m);
    t1 = pool_event(m);
    CU(cudaEventRecord(t0, m->stream));
  }
  TRY(exchange_begin(m, U, which));
  TRY(exchange_end(m, U, which));
  if (m->timing) {
    CU(cudaEventRecord(t1, m->stream));
    m->t_exch.push_back({t0, t1});
  }
  return PH_OK;
}

/* rank reduce -> allgather -> finalize (dt min and totals) */
static ph_status reduce_finalize(ph_mesh* m, int ncta, int mode) {
  CU(launch_rank_reduce(m->partials, ncta, m->nranks > 1 ? m->my6 : m->all6, m->stream));
  m->launches++;
  if (m->nranks > 1)
    NC(ncclAllGather(m->my6, m->all6, 6, ncclDouble, m->comm2 ? m->comm2 : m->comm, m->stream));
  CU(launch_finalize(m->all6, m->nranks, m->d_st, m->hist, m->hist_cap, m->G.cfl, mode, m->tot5, m->G.exact, m->stream));
  m->launches++;
  return PH_OK;
}

static ph_status standalone_reduce(ph_mesh* m, double* U, int mode) {
  int nloc = (int)m->local_gids.size();
  if (nloc > 0) {
    CU(launch_reduce(U, m->d_meta, nloc, m->partials, m->d_err, m->G, m->stream));
    m->launches++;
  }
  return reduce_finalize(m, nloc * m->G.n[2], mode);
}

/* one stage over all local blocks, pack by pack (a2-a5) */
static ph_status run_stage(ph_mesh* m, const double* Uin, double* Uout, double a0, double b1, double cdt,
                           bool reduce, int stage, int s0 = 0, int s1 = -1, bool post = true, bool put = false) {
  NvtxRange nvtx_(stage == 1 ? "ph:stage1" : "ph:stage2");
  const int nloc = (int)m->local_gids.size();
  if (s1 < 0) s1 = nloc;
  if (m->ho) {
    StageArgs A{};
    A.Uin = Uin;
    A.U0 = m->U0;
    A.Uout = Uout;
    A.meta = m->d_meta;
    A.st = m->d_st;
    A.partials = m->partials;
    A.err = m->d_err;
    A.a0 = a0;
    A.b1 = b1;
    A.cdt = cdt;
    A.stage = stage;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (m->timing) {
      t0 = pool_event(m);
      t1 = pool_event(m);
      CU(cudaEventRecord(t0, m->stream));
    }
    const bool w_ready = m->ho_fold && m->w_ready;
    CU(launch_highorder_stage(m->cfg.recon, reduce, a0 != 0.0, nloc, A, m->Wpool, m->Fxb, m->Fyb, m->Fzb, w_ready,
                              m->ho_fold, m->G, m->stream));
    m->launches += w_ready ? 4 : 5;
    m->w_ready = false;  // W now holds the new interior; its ghosts arrive with the W exchange
    if (m->timing) {
      CU(cudaEventRecord(t1, m->stream));
      m->t_stage.push_back({t0, t1});
    }
    return PH_OK;
  }
  const int per_blk = m->ntx * m->nty * m->nkc;
  const cudaStream_t S = m->stream;
  const int npacks = (s1 - s0 + m->pack_size - 1) / std::max(m->pack_size, 1);
  const int nps = std::min(std::min(m->pack_streams, (int)ph_mesh::kMaxPackStreams), npacks);
  const bool multi = nps > 1 && !m->timing;
  if (multi) {
    if (!m->ev_pfork) CU(cudaEventCreateWithFlags(&m->ev_pfork, cudaEventDisableTiming));
    CU(cudaEventRecord(m->ev_pfork, S));
    for (int i = 1; i < nps; ++i) {
      if (!m->pstream[i]) {
        CU(cudaStreamCreateWithFlags(&m->pstream[i], cudaStreamNonBlocking));
        CU(cudaEventCreateWithFlags(&m->ev_pjoin[i], cudaEventDisableTiming));
      }
      CU(cudaStreamWaitEvent(m->pstream[i], m->ev_pfork, 0));
    }
  }
  int ipack = 0;
  for (int p0 = s0; p0 < s1; p0 += m->pack_size, ++ipack) {
    int np = std::min(m->pack_size, s1 - p0);
    // packs rotate over the streams: packs of one stage write disjoint blocks and partials
    const cudaStream_t ps = (multi && (ipack % nps)) ? m->pstream[ipack % nps] : S;
    StageArgs A{};
    A.Uin = Uin;
    A.U0 = m->U0;
    A.Uout = Uout;
    A.meta = m->d_meta;
    A.slots = m->d_slots + p0;
    A.st = m->d_st;
    A.fbuf = m->fbuf;
    A.partials = m->partials;
    A.err = m->d_err;
    A.a0 = a0;
    A.b1 = b1;
    A.cdt = cdt;
    A.ntx = m->ntx;
    A.nty = m->nty;
    A.nkc = m->nkc;
    A.KC = m->KC;
    A.cta_base = p0 * per_blk;
    A.pool_slots = (int)std::max<int64_t>((int64_t)m->local_gids.size(), 1);
    A.stage = stage;
    if (put && m->fused_put) A.peer_rbuf = m->d_prbuf[Uout == m->U1 ? 0 : 1];
    if (m->Hpool) {
      const bool vl2 = m->cfg.integrator == PH_INT_VL2;
      A.H = m->Hpool;
      A.ha0 = vl2 ? 1.0 : 0.5;  // the stage-2 coefficients of U^n and U^1 (O5)
      A.hb1 = vl2 ? 0.0 : 0.5;
    }
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (m->timing) {
      t0 = pool_event(m);
      t1 = pool_event(m);
      CU(cudaEventRecord(t0, m->stream));
    }
    CU(launch_stage(m->cfg.recon, reduce, a0 != 0.0, np * per_blk, A, m->G, ps));
    m->launches++;
    if (m->timing) {
      CU(cudaEventRecord(t1, m->stream));
      m->t_stage.push_back({t0, t1});
    }
  }
  if (multi) {
    for (int i = 1; i < nps; ++i) {
      CU(cudaEventRecord(m->ev_pjoin[i], m->pstream[i]));
      CU(cudaStreamWaitEvent(S, m->ev_pjoin[i], 0));
    }
  }
  if (m->multilevel && post) {
    if (m->nranks > 1 && (m->fsbuf_n > 0 || m->frbuf_n > 0)) {
      // fine ranks restrict and send their coarse-fine face fluxes to the coarse blocks' ranks
      if (!m->fpack.empty()) {
        CU(launch_flux_pack((int)m->fpack.size(), m->d_fpack, m->fbuf, m->fsbuf, m->G, m->stream));
        m->launches++;
      }
      NC(ncclGroupStart());
      for (int p = 0; p < m->nranks; ++p) {
        if (p == m->rank) continue;
        if (m->fsend_cnt[p]) NC(ncclSend(m->fsbuf + m->fsend_off[p], m->fsend_cnt[p], ncclDouble, p, m->comm, m->stream));
        if (m->frecv_cnt[p]) NC(ncclRecv(m->frbuf + m->frecv_off[p], m->frecv_cnt[p], ncclDouble, p, m->comm, m->stream));
      }
      NC(ncclGroupEnd());
    }
    for (int d = 0; d < 3; ++d) {
      if (m->reflux[d].empty()) continue;
      // stage 1 on the H path: H = ha0 U^n + hb1 U^1 must see the corrected U^1
      const bool fixH = m->Hpool && Uout == m->U1;
      const double hb1 = m->cfg.integrator == PH_INT_VL2 ? 0.0 : 0.5;
      CU(launch_reflux((int)m->reflux[d].size(), m->d_reflux[d], Uout, m->d_meta, m->fbuf, m->frbuf, m->d_st, cdt,
                       m->G, m->stream, fixH ? m->Hpool : nullptr, hb1));
      m->launches++;
    }
  }
  return PH_OK;
}

static ph_status tag_and_remesh(ph_mesh* m, bool refine_only, bool allow_deref, bool move, bool* changed,
                                int deref_interval = 0);

static ph_status one_cycle(ph_mesh* m) {
  NvtxRange nvtx_("ph:cycle");
  CU(launch_cycle_begin(m->d_st, 0.0, 0, m->stream));
  m->launches++;
  const bool adaptive = m->cfg.refinement == PH_REF_ADAPTIVE;
  const bool fuse_reduce = !m->multilevel && !adaptive;
  const int nloc = (int)m->local_gids.size();
  if (m->overlap && fuse_reduce) {
    // multi-GPU, uniform mesh, boundary first: stream B (high priority) runs the blocks
    // with remote or physical faces and then their halo (NCCL, or puts into peer memory); stream I
    // runs the interior blocks at the same time, so each exchange hides behind interior work.
    //   B: S1(bnd) -> send U1 -> [I: S1(int) done] -> recv U1 -> S2(bnd) -> send U0 -> recv U0
    //   I: S1(int) -> [B: S1(bnd) done] -> S2(int)
    // then the caller's stream joins both and reduces dt / totals (split communicator).
    const bool vl2 = m->cfg.integrator == PH_INT_VL2;
    const double c1 = vl2 ? 0.5 : 1.0, a2 = vl2 ? 1.0 : 0.5, b2 = vl2 ? 0.0 : 0.5, c2 = vl2 ? 1.0 : 0.5;
    cudaStream_t S = m->stream;
    struct Restore {
      ph_mesh* m;
      cudaStream_t s;
      ~Restore() { m->stream = s; }
    } restore{m, S};
    CU(cudaEventRecord(m->ev_a, S));
    CU(cudaStreamWaitEvent(m->bstream, m->ev_a, 0));
    CU(cudaStreamWaitEvent(m->istream, m->ev_a, 0));
    m->stream = m->bstream;
    TRY(run_stage(m, m->U0, m->U1, 0.0, 1.0, c1, false, 1, m->n_int, nloc, true, true));
    CU(cudaEventRecord(m->ev_b1, m->bstream));
    TRY(exchange_begin(m, m->U1, 1));
    m->stream = m->istream;
    TRY(run_stage(m, m->U0, m->U1, 0.0, 1.0, c1, false, 1, 0, m->n_int));
    CU(cudaEventRecord(m->ev_i1, m->istream));
    m->stream = m->bstream;
    TRY(exchange_end(m, m->U1, 1));
    CU(cudaStreamWaitEvent(m->bstream, m->ev_i1, 0));
    TRY(run_stage(m, m->U1, m->U0, a2, b2, c2, true, 2, m->n_int, nloc, true, true));
    TRY(exchange_begin(m, m->U0, 1));
    TRY(exchange_end(m, m->U0, 1));
    CU(cudaEventRecord(m->ev_b2, m->bstream));
    m->stream = m->istream;
    CU(cudaStreamWaitEvent(m->istream, m->ev_b1, 0));
    TRY(run_stage(m, m->U1, m->U0, a2, b2, c2, true, 2, 0, m->n_int));
    CU(cudaEventRecord(m->ev_i2, m->istream));
    m->stream = S;
    CU(cudaStreamWaitEvent(S, m->ev_b2, 0));
    CU(cudaStreamWaitEvent(S, m->ev_i2, 0));
    TRY(reduce_finalize(m, nloc > 0 ? m->stage_ctas : 0, 1));
    return PH_OK;
  }
  // static multilevel: stage 2 reduces dt / totals of all cells but the flux-corrected layers, which
  // are reduced after the reflux (no standalone pass over the whole pool)
  const bool ml_fuse = m->multilevel && !adaptive && !m->ho && !getenv("PH_NO_ML_FUSE");
  const bool red2 = fuse_reduce || ml_fuse;
  // nghost-3 path: the update kernels write the primitives of their output and the per-cycle exchange
  // moves W instead of U (reading A49: W of exchanged U == exchanged W, bit for bit); U's ghosts are
  // then refreshed only on demand (ghosts_stale)
  const bool wx = m->ho && m->ho_fold;
  auto xchg = [&](double* U) -> ph_status {
    TRY(exchange(m, wx ? m->Wpool : U, 1));
    if (wx) m->w_ready = true;
    return PH_OK;
  };
  if (m->cfg.integrator == PH_INT_VL2) {
    TRY(run_stage(m, m->U0, m->U1, 0.0, 1.0, 0.5, false, 1));
    TRY(xchg(m->U1));
    TRY(run_stage(m, m->U1, m->U0, 1.0, 0.0, 1.0, red2, 2));
  } else {
    TRY(run_stage(m, m->U0, m->U1, 0.0, 1.0, 1.0, false, 1));
    TRY(xchg(m->U1));
    TRY(run_stage(m, m->U1, m->U0, 0.5, 0.5, 0.5, red2, 2));
  }
  if (ml_fuse && !m->rfx_faces.empty()) {
    CU(launch_rfx_reduce(m->d_rfx_faces, (int)m->rfx_faces.size(), m->U0, m->d_meta,
                         m->partials + (int64_t)m->stage_ctas * 6, m->d_err, m->G, m->stream));
    m->launches++;
  }
  TRY(xchg(m->U0));
  bool tag_partials = false;  // the tag pass also reduced dt / totals of the unchanged mesh
  if (adaptive) {
    // O5 step 6: tag after the cycle, remesh, exchange; dt and totals on the new mesh.  The cycle
    // state (active, cycle count for the derefinement gate) is read back in the tag pass's sync.
    const int iv = m->cfg.derefine_interval > 0 ? m->cfg.derefine_interval : 1;
    bool changed = false;
    TRY(tag_and_remesh(m, false, false, true, &changed, iv));
    if (changed) TRY(exchange(m, m->U0, 0));
    tag_partials = !changed;
  }
  if (fuse_reduce) TRY(reduce_finalize(m, nloc > 0 ? m->stage_ctas : 0, 1));
  else if (ml_fuse) TRY(reduce_finalize(m, (nloc > 0 ? m->stage_ctas : 0) + (int)m->rfx_faces.size(), 1));
  else if (tag_partials) TRY(reduce_finalize(m, nloc * tag_ctas_per_block(m->G), 1));
  else TRY(standalone_reduce(m, m->U0, 1));
  return PH_OK;
}

/* ------------------------------------------------------------------------------- AMR (O9) */
/* Install a new leaf set: rebuild blocks / partition / plan / device pools (P:214, P:583-592:
 * the tree is rebuilt first and the new distribution computed from it, then populated) and, when
 * move, fill the new pool: same-level blocks are moved (sent if their owner changes), refined
 * parents are sent whole and prolongated on the receiving rank, derefined siblings are restricted
 * on their sending rank and sent as octants.  Per (sender, receiver) pair both ranks enumerate
 * the new blocks in gid order, so buffer offsets agree without a handshake. */
static ph_status remesh(ph_mesh* m, const std::unordered_set<LocKey>& leaves, bool move) {
  m->w_ready = false;
  const int R = m->nranks, me = m->rank;
  // peer halo (AMR): the plan changes, so the receive regions, offsets and mappings are rebuilt after it
  const bool had_peer = m->peer && !m->host_only;  // (host-only meshes: plan only, nothing mapped)
  if (had_peer) teardown_peer(m);
  if (m->graph_exec) {
    cudaGraphExecDestroy(m->graph_exec);
    m->graph_exec = nullptr;
  }
  struct Old { int rank; int slot; };
  std::unordered_map<LocKey, Old> old;
  for (auto& b : m->blocks) old[pack(b.loc)] = Old{b.rank, (int)b.local};
  double* oldU0 = m->U0;
  std::vector<void*> old_allocs;
  old_allocs.swap(m->allocs);
  m->tree->set_leaves(leaves);
  try {
    build_blocks(*m->tree, m->nranks, m->rank, m->blocks, m->gid_of);
  } catch (const std::exception& ex) {
    return fail(PH_ERR_STATE, ex.what());
  }
  TRY(build_plan(m));
  if (had_peer) {
    bool ok = false;
    TRY(setup_peer(m, &ok));
    m->peer = ok;
    if (!ok && m->cfg.halo_transport == PH_HALO_PEER)
      return fail(PH_ERR_UNSUPPORTED, "peer halo: a rank cannot map its peers' memory after the remesh");
  }
  TRY(setup_device(m));
  if (move) {
    const Geom& G = m->G;
    const int64_t nint = (int64_t)NVAR * G.n[0] * G.n[1] * G.n[2];
    const int64_t noct = (int64_t)NVAR * G.nc[0] * G.nc[1] * G.nc[2];
    std::vector<RemeshTask> send_t, work_t;      // send: pack kernels; work: local + from recv buffer
    std::vector<std::pair<int, int64_t>> send_full;  // (old slot, offset) whole-block sends
    std::vector<int> send_peer, work_peer, full_peer;
    std::vector<int64_t> so(R, 0), ro(R, 0);
    std::map<std::pair<LocKey, int>, bool> parent_sent;
    std::map<LocKey, int64_t> parent_recv;  // parent -> recv offset (relative, peer in parent_recv_peer)
    std::map<LocKey, int> parent_recv_peer;
    for (auto& b : m->blocks) {
      const int Rn = b.rank;
      const LocKey key = pack(b.loc);
      auto it = old.find(key);
      if (it != old.end()) {  // same-level move
        const int Ro = it->second.rank;
        RemeshTask t{};
        t.kind = R_MOVE;
        if (Ro == me && Rn == me) {
          t.src = it->second.slot;
          t.dst = (int)b.local;
          work_t.push_back(t);
          work_peer.push_back(-1);
        } else if (Ro == me) {
          t.src = it->second.slot;
          t.dst = -1;
          t.dst_off = so[Rn];
          so[Rn] += nint;
          send_t.push_back(t);
          send_peer.push_back(Rn);
        } else if (Rn == me) {
          t.src = -1;
          t.src_off = ro[Ro];
          ro[Ro] += nint;
          t.dst = (int)b.local;
          work_t.push_back(t);
          work_peer.push_back(Ro);
        }
        continue;
      }
      const LocKey pk = b.loc.level > 0 ? pack(parent(b.loc)) : 0;
      auto ip = b.loc.level > 0 ? old.find(pk) : old.end();
      if (ip != old.end()) {  // refined: prolongate the parent on the child's new rank
        const int Ro = ip->second.rank;
        if (Ro == me && Rn != me && !parent_sent[{pk, Rn}]) {
          parent_sent[{pk, Rn}] = true;
          send_full.push_back({ip->second.slot, so[Rn]});
          full_peer.push_back(Rn);
          so[Rn] += G.bstride;
        }
        if (Rn == me) {
          RemeshTask t{};
          t.kind = R_REFINE;
          t.dst = (int)b.local;
          for (int d = 0; d < 3; ++d) t.ch[d] = (int)(b.loc.x[d] & 1);
          if (Ro == me) {
            t.src = ip->second.slot;
            work_peer.push_back(-1);
          } else {
            if (!parent_recv.count(pk)) {
              parent_recv[pk] = ro[Ro];
              parent_recv_peer[pk] = Ro;
              ro[Ro] += G.bstride;
            }
            t.src = -1;
            t.src_off = parent_recv[pk];
            work_peer.push_back(Ro);
          }
          work_t.push_back(t);
        }
        continue;
      }
      // derefined: 8 old children -> octants of this block
      for (int c = 0; c < 8; ++c) {
        auto ic = old.find(pack(child(b.loc, c)));
        if (ic == old.end()) return fail(PH_ERR_STATE, "remesh: block has no source");
        const int Ro = ic->second.rank;
        RemeshTask t{};
        t.ch[0] = c & 1;
        t.ch[1] = (c >> 1) & 1;
        t.ch[2] = (c >> 2) & 1;
        if (Ro == me && Rn == me) {
          t.kind = R_OCT;
          t.src = ic->second.slot;
          t.dst = (int)b.local;
          work_t.push_back(t);
          work_peer.push_back(-1);
        } else if (Ro == me) {
          t.kind = R_OCT;
          t.src = ic->second.slot;
          t.dst = -1;
          t.dst_off = so[Rn];
          so[Rn] += noct;
          send_t.push_back(t);
          send_peer.push_back(Rn);
        } else if (Rn == me) {
          t.kind = R_OCTCOPY;
          t.src = -1;
          t.src_off = ro[Ro];
          ro[Ro] += noct;
          t.dst = (int)b.local;
          work_t.push_back(t);
          work_peer.push_back(Ro);
        }
      }
    }
    // concatenate per-peer regions
    std::vector<int64_t> soff(R, 0), roff(R, 0);
    int64_t stot = 0, rtot = 0;
    for (int q = 0; q < R; ++q) {
      soff[q] = stot;
      stot += so[q];
      roff[q] = rtot;
      rtot += ro[q];
    }
    for (size_t i = 0; i < send_t.size(); ++i) send_t[i].dst_off += soff[send_peer[i]];
    for (size_t i = 0; i < send_full.size(); ++i) send_full[i].second += soff[full_peer[i]];
    for (size_t i = 0; i < work_t.size(); ++i)
      if (work_peer[i] >= 0) work_t[i].src_off += roff[work_peer[i]];
    double *msb = nullptr, *mrb = nullptr;
    std::vector<void*> keep;
    keep.swap(m->allocs);  // migration buffers and task arrays go to a temporary list
    if (stot) TRY(dalloc(m, (void**)&msb, stot * sizeof(double)));
    if (rtot) TRY(dalloc(m, (void**)&mrb, rtot * sizeof(double)));
    RemeshTask *d_send = nullptr, *d_work = nullptr;
    TRY(upload(m, &d_send, send_t));
    TRY(upload(m, &d_work, work_t));
    std::vector<void*> tmp;
    tmp.swap(m->allocs);
    m->allocs.swap(keep);
    for (void* q : tmp) old_allocs.push_back(q);
    // 1. sender side: pack moved interiors / restricted octants, copy whole parents
    CU(launch_remesh(d_send, (int)send_t.size(), oldU0, m->U0, mrb, msb, G, m->stream));
    m->launches++;
    for (auto& sf : send_full)
      CU(cudaMemcpyAsync(msb + sf.second, oldU0 + (int64_t)sf.first * G.bstride, G.bstride * sizeof(double),
                         cudaMemcpyDeviceToDevice, m->stream));
    // 2. exchange the migration buffers
    if (R > 1 && (stot || rtot)) {
      NC(ncclGroupStart());
      for (int q = 0; q < R; ++q) {
        if (q == me) continue;
        if (so[q]) NC(ncclSend(msb + soff[q], so[q], ncclDouble, q, m->comm, m->stream));
        if (ro[q]) NC(ncclRecv(mrb + roff[q], ro[q], ncclDouble, q, m->comm, m->stream));
      }
      NC(ncclGroupEnd());
    }
    // 3. local moves / prolongations / restrictions and the received data
    CU(launch_remesh(d_work, (int)work_t.size(), oldU0, m->U0, mrb, msb, G, m->stream));
    m->launches++;
  }
  CU(cudaStreamSynchronize(m->stream));
  free_list(m, old_allocs);
  return PH_OK;
}

/* Tag every local block (eps_B, A14), gather the indicators of all ranks, normalise the flags
 * (O9) identically on every rank and install the new mesh if it changed. */
/* deref_interval > 0: per-cycle call; the cycle state is read in the same sync as the indicators,
 * inactive cycles (t >= tlim) change nothing, and derefinement is allowed when the cycle count after
 * this cycle's increment is a multiple of the interval (A16). */
static ph_status tag_and_remesh(ph_mesh* m, bool refine_only, bool allow_deref, bool move, bool* changed,
                                int deref_interval) {
  NvtxRange nvtx_("ph:tag_remesh");
  *changed = false;
  const int nloc = (int)m->local_gids.size();
  const int R = m->nranks;
  const int64_t nglob = (int64_t)m->blocks.size();
  const int64_t maxloc = (nglob + R - 1) / R;
  CU(launch_tag(m->U0, m->d_meta, nloc, m->d_eps, m->partials, m->d_err, m->G, m->stream));
  m->launches++;
  std::vector<unsigned long long> bits((size_t)maxloc * R, 0ull);
  if (R > 1) {
    NC(ncclAllGather(m->d_eps, m->d_eps_all, maxloc, ncclUint64, m->comm, m->stream));
    CU(cudaMemcpyAsync(bits.data(), m->d_eps_all, bits.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       m->stream));
  } else if (nloc) {
    CU(cudaMemcpyAsync(bits.data(), m->d_eps, nloc * sizeof(unsigned long long), cudaMemcpyDeviceToHost, m->stream));
  }
  CycleState st{};
  if (deref_interval > 0) CU(cudaMemcpyAsync(&st, m->d_st, sizeof st, cudaMemcpyDeviceToHost, m->stream));
  CU(cudaStreamSynchronize(m->stream));
  if (deref_interval > 0) {
    if (!st.active) return PH_OK;
    allow_deref = ((st.cycle + 1) % deref_interval) == 0;
  }
  std::vector<Loc> locs;
  std::vector<int8_t> flags;
  for (int r = 0; r < R; ++r) {
    int64_t lo, hi;
    partition_range(nglob, R, r, &lo, &hi);
    for (int64_t g = lo; g < hi; ++g) {
      const BlockInfo& b = m->blocks[g];
      double eps;
      memcpy(&eps, &bits[(size_t)r * maxloc + (g - lo)], sizeof eps);
      int8_t f = 0;
      if (eps > m->cfg.refine_tol && b.loc.level < m->cfg.max_level) f = 1;
      else if (eps < m->cfg.derefine_tol && b.loc.level > 0) f = -1;
      if (refine_only && f < 0) f = 0;
      locs.push_back(b.loc);
      flags.push_back(f);
    }
  }
  if (!refine_only) m->last_flags = flags;
  // nothing can change without a refinement request, or a derefinement request on a gate cycle
  bool any = false;
  const bool deref_ok = allow_deref && !refine_only;
  for (int8_t f : flags) any = any || f > 0 || (f < 0 && deref_ok);
  if (!any) return PH_OK;
  std::unordered_set<LocKey> nl = normalize_flags(*m->tree, locs, flags, allow_deref && !refine_only);
  if (nl == m->tree->leaves()) return PH_OK;
  // the prolongation of refined parents reads their ghosts (A11): materialise every ghost first
  if (move && m->direct_halo) TRY(exchange(m, m->U0, 0));
  TRY(remesh(m, nl, move));
  *changed = true;
  return PH_OK;
}

/* ------------------------------------------------------------------------------- C ABI */
// Every extern "C" entry point runs inside PH_API_BEGIN / PH_API_END: no C++ exception crosses the
// ABI (ph.h); a throw becomes a status code with the message in ph_last_error().
#define PH_API_BEGIN try {
#define PH_API_END                                                                          \
  }                                                                                         \
  catch (const std::bad_alloc&) { return fail(PH_ERR_OOM, "out of host memory"); }         \
  catch (const std::logic_error& e) { return fail(PH_ERR_INVALID_ARG, e.what()); }         \
  catch (const std::exception& e) { return fail(PH_ERR_STATE, e.what()); }                 \
  catch (...) { return fail(PH_ERR_STATE, "unknown C++ exception"); }

extern "C" {

const char* ph_last_error(void) { return g_err.c_str(); }

ph_status ph_nccl_unique_id(void* out, int32_t cap) {
  PH_API_BEGIN
  if (!out || cap < (int32_t)sizeof(ncclUniqueId)) return fail(PH_ERR_INVALID_ARG, "need 128 bytes");
  ncclUniqueId id;
  NC(ncclGetUniqueId(&id));
  memcpy(out, &id, sizeof id);
  return PH_OK;
  PH_API_END
}

ph_status ph_mesh_create(const ph_config* cfg, ph_mesh** out) {
  PH_API_BEGIN
  if (!cfg || !out) return fail(PH_ERR_INVALID_ARG, "null argument");
  *out = nullptr;
  if (cfg->abi_version != PH_ABI_VERSION) return fail(PH_ERR_INVALID_ARG, "abi_version mismatch");
  if (cfg->nghost != 2 && cfg->nghost != 3) return fail(PH_ERR_CONFIG, "nghost must be 2 (PLM) or 3 (PPM, WENO-Z; A8)");
  if (cfg->recon >= PH_RECON_PPM && cfg->nghost != 3) return fail(PH_ERR_CONFIG, "PPM / WENO-Z need nghost = 3 (A8)");
  if (cfg->nghost == 3 && cfg->max_level > 0 && cfg->refinement != PH_REF_NONE)
    return fail(PH_ERR_CONFIG, "nghost = 3 is supported on uniform meshes only (reading A39)");
  if (!(cfg->gamma > 1.0) || !(cfg->gamma < 0x1p50) || !(cfg->cfl > 0.0))  // (gamma < 2^50: ddiv_k's range)
    return fail(PH_ERR_CONFIG, "gamma must lie in (1, 2^50) and cfl be positive");
  if (cfg->nranks < 1 || cfg->nranks > 64 || cfg->rank < 0 || cfg->rank >= cfg->nranks)
    return fail(PH_ERR_INVALID_ARG, "bad rank / nranks");
  if (cfg->recon < 0 || cfg->recon > 4 || cfg->integrator < 0 || cfg->integrator > 1)
    return fail(PH_ERR_CONFIG, "unknown recon / integrator");
  if (cfg->wavespeed != PH_WS_DAVIS && cfg->wavespeed != PH_WS_EINFELDT)
    return fail(PH_ERR_CONFIG, "unknown wave-speed estimate");
  if (cfg->wavespeed == PH_WS_EINFELDT && cfg->recon >= PH_RECON_PPM)
    return fail(PH_ERR_CONFIG, "Einfeldt wave speeds are implemented for PLM (PPM / WENO-Z use Davis)");
  if (cfg->max_level < 0 || cfg->max_level > 10) return fail(PH_ERR_CONFIG, "max_level out of range");
  MeshCfg mc{};
  for (int d = 0; d < 3; ++d) {
    if (cfg->block_nx[d] < cfg->nghost || cfg->mesh_nx[d] <= 0 || cfg->mesh_nx[d] % cfg->block_nx[d] != 0)
      return fail(PH_ERR_CONFIG, "block size does not tile the root grid (S:144)");
    if ((cfg->bc_inner[d] == PH_BC_PERIODIC) != (cfg->bc_outer[d] == PH_BC_PERIODIC))
      return fail(PH_ERR_CONFIG, "periodic boundaries must be paired");
    for (int bc : {cfg->bc_inner[d], cfg->bc_outer[d]})
      if (bc < 0 || bc > 2) return fail(PH_ERR_CONFIG, "unknown boundary tag (S:414)");
    if (cfg->max_level > 0 && (cfg->block_nx[d] % 2 || cfg->block_nx[d] < 2 * cfg->nghost))
      return fail(PH_ERR_CONFIG, "refinement needs even block sizes >= 2*nghost");
    mc.n[d] = cfg->block_nx[d];
    mc.nrb[d] = cfg->mesh_nx[d] / cfg->block_nx[d];
    mc.periodic[d] = cfg->bc_inner[d] == PH_BC_PERIODIC;
    mc.bc_in[d] = cfg->bc_inner[d];
    mc.bc_out[d] = cfg->bc_outer[d];
    mc.xmin[d] = cfg->xmin[d];
    mc.xmax[d] = cfg->xmax[d];
    if (!(cfg->xmax[d] > cfg->xmin[d])) return fail(PH_ERR_CONFIG, "empty domain");
    if ((mc.nrb[d] << cfg->max_level) >= (1 << 19)) return fail(PH_ERR_CONFIG, "too many blocks per dim");
  }
  mc.max_level = cfg->max_level;
  ph_mesh* m = new ph_mesh();
  m->cfg = *cfg;
  if (cfg->nregions > 0 && cfg->regions) m->regions.assign(cfg->regions, cfg->regions + 7 * cfg->nregions);
  m->cfg.regions = nullptr;
  m->mc = mc;
  m->rank = cfg->rank;
  m->nranks = cfg->nranks;
  m->host_only = cfg->host_only != 0;
  m->no_direct_halo = cfg->no_direct_halo != 0;
  m->use_graph = !(getenv("PH_NO_GRAPH") && atoi(getenv("PH_NO_GRAPH")) != 0);
  m->ho_fold = !(getenv("PH_HO_NOFOLD") && atoi(getenv("PH_HO_NOFOLD")) != 0);
  if (getenv("PH_PACK_STREAMS")) m->pack_streams = atoi(getenv("PH_PACK_STREAMS"));
  Geom& G = m->G;
  G.g = cfg->nghost;
  G.cg = (G.g + 1) / 2 + 1;
  int64_t maxface = 0;
  for (int d = 0; d < 3; ++d) {
    G.n[d] = (int)cfg->block_nx[d];
    G.N[d] = G.n[d] + 2 * G.g;
    G.nc[d] = G.n[d] / 2;
    G.NC[d] = G.nc[d] + 2 * G.cg;
  }
  maxface = std::max<int64_t>({(int64_t)G.n[1] * G.n[2], (int64_t)G.n[0] * G.n[2], (int64_t)G.n[0] * G.n[1]});
  G.vstride = (int64_t)G.N[0] * G.N[1] * G.N[2];
  G.bstride = NVAR * G.vstride;
  G.cvstride = (int64_t)G.NC[0] * G.NC[1] * G.NC[2];
  G.cbstride = NVAR * G.cvstride;
  G.fstride = NVAR * maxface;
  G.gamma = cfg->gamma;
  G.gm1 = cfg->gamma - 1.0;
  G.inv_gm1 = 1.0 / (cfg->gamma - 1.0);
  G.cfl = cfg->cfl;
  G.wavespeed = cfg->wavespeed;
  try {
    m->tree = new Tree(mc);
    if (cfg->refinement != PH_REF_NONE && cfg->max_level > 0) m->tree->refine_regions(m->regions);
    build_blocks(*m->tree, m->nranks, m->rank, m->blocks, m->gid_of);
  } catch (const std::exception& e) {
    delete m->tree;
    delete m;
    return fail(PH_ERR_CONFIG, e.what());
  }
  if (cfg->halo_transport < PH_HALO_AUTO || cfg->halo_transport > PH_HALO_PEER) {
    delete m->tree;
    delete m;
    return fail(PH_ERR_CONFIG, "unknown halo_transport");
  }
  bool uniform = true;
  for (auto& b : m->blocks) uniform = uniform && b.loc.level == 0;
  // peer transport: uniform, static multilevel and adaptive meshes (AMR re-runs the set-up at each remesh)
  (void)uniform;
  const bool peer_cfg = m->nranks > 1 && !m->no_direct_halo &&
                        G.g == 2 && cfg->halo_transport != PH_HALO_NCCL;
  if (cfg->halo_transport == PH_HALO_PEER && !peer_cfg) {
    delete m->tree;
    delete m;
    return fail(PH_ERR_UNSUPPORTED, "peer halo needs nranks > 1 and an nghost-2 mesh with the direct halo");
  }
  ph_status st = build_plan(m);
  if (st != PH_OK) {
    delete m->tree;
    delete m;
    return st;
  }
  if (m->host_only) m->peer = peer_cfg;  // plan only (the per-cycle plan is the same for both transports)
  if (!m->host_only) {
    cudaError_t e = cudaSetDevice(cfg->device);
    if (e != cudaSuccess) {
      delete m->tree;
      delete m;
      return fail(PH_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    }
    m->stream = (cudaStream_t)cfg->stream;
    cudaStreamCreateWithFlags(&m->comm_stream, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&m->ev_pack, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&m->ev_comm, cudaEventDisableTiming);
    if (m->nranks > 1) {
      if (!cfg->nccl_id) {
        delete m->tree;
        delete m;
        return fail(PH_ERR_INVALID_ARG, "nranks > 1 needs nccl_id");
      }
      ncclUniqueId id;
      memcpy(&id, cfg->nccl_id, sizeof id);
      ncclResult_t r = ncclCommInitRank(&m->comm, m->nranks, id, m->rank);
      if (r != ncclSuccess) {
        delete m->tree;
        delete m;
        return fail(PH_ERR_COMM, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
      }
      // a second communicator for the scalar reductions, so they never queue behind the halo
      r = ncclCommSplit(m->comm, 0, m->rank, &m->comm2, nullptr);
      if (r != ncclSuccess) m->comm2 = nullptr;
    }
    if (m->nranks > 1) {
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      cudaStreamCreateWithPriority(&m->bstream, cudaStreamNonBlocking, hi);
      cudaStreamCreateWithFlags(&m->istream, cudaStreamNonBlocking);
      for (cudaEvent_t* e : {&m->ev_a, &m->ev_b1, &m->ev_i1, &m->ev_b2, &m->ev_i2})
        cudaEventCreateWithFlags(e, cudaEventDisableTiming);
    }
    st = setup_persistent(m);
    if (st == PH_OK && peer_cfg) {
      bool ok = false;
      st = setup_peer(m, &ok);
      m->peer = ok;
      if (st == PH_OK && !ok && cfg->halo_transport == PH_HALO_PEER)
        st = fail(PH_ERR_UNSUPPORTED, "peer halo requested but some rank cannot map its peers' memory (CUDA IPC)");
    }
    if (st == PH_OK) st = setup_device(m);
    if (st == PH_OK) {
      cudaError_t e2 = cudaStreamSynchronize(m->stream);
      if (e2 != cudaSuccess) st = fail(PH_ERR_CUDA, cudaGetErrorString(e2));
    }
    if (st != PH_OK) {
      std::string msg = g_err;
      ph_mesh_destroy(m);
      g_err = msg;
      return st;
    }
  }
  *out = m;
  return PH_OK;
  PH_API_END
}

ph_status ph_mesh_destroy(ph_mesh* m) {
  PH_API_BEGIN
  if (!m) return PH_OK;
  if (m->graph_exec) cudaGraphExecDestroy(m->graph_exec);
  if (m->ev_fork) cudaEventDestroy(m->ev_fork);
  if (m->ev_join) cudaEventDestroy(m->ev_join);
  teardown_peer(m);  // nobody may still read my pools when I unmap / free
  free_all(m);
  for (auto& p : m->t_stage) (void)p;
  for (cudaEvent_t e : m->ev_pool) cudaEventDestroy(e);
  if (m->ev_pack) cudaEventDestroy(m->ev_pack);
  if (m->ev_comm) cudaEventDestroy(m->ev_comm);
  if (m->comm_stream) cudaStreamDestroy(m->comm_stream);
  if (m->bstream) cudaStreamDestroy(m->bstream);
  for (int i = 0; i < ph_mesh::kMaxPackStreams; ++i) {
    if (m->pstream[i]) cudaStreamDestroy(m->pstream[i]);
    if (m->ev_pjoin[i]) cudaEventDestroy(m->ev_pjoin[i]);
  }
  if (m->ev_pfork) cudaEventDestroy(m->ev_pfork);
  if (m->istream) cudaStreamDestroy(m->istream);
  for (cudaEvent_t e : {m->ev_a, m->ev_b1, m->ev_i1, m->ev_b2, m->ev_i2})
    if (e) cudaEventDestroy(e);
  if (m->gstream) cudaStreamDestroy(m->gstream);
  if (m->comm2) ncclCommDestroy(m->comm2);
  if (m->comm) ncclCommDestroy(m->comm);
  delete m->tree;
  delete m;
  return PH_OK;
  PH_API_END
}

static ph_status need_device(const ph_mesh* m) {
  if (!m) return fail(PH_ERR_INVALID_ARG, "null mesh");
  if (m->host_only) return fail(PH_ERR_STATE, "host-only mesh has no device state");
  return PH_OK;
}

ph_status ph_exchange(ph_mesh* m) {
  PH_API_BEGIN
  if (m) m->w_ready = false;  // U0 changes (or is re-exchanged): W is rebuilt at the next step
  TRY(need_device(m));
  TRY(exchange(m, m->U0, 0));
  return check_err(m);
  PH_API_END
}

ph_status ph_refresh(ph_mesh* m) {
  PH_API_BEGIN
  if (m) m->w_ready = false;  // U0 changes (or is re-exchanged): W is rebuilt at the next step
  TRY(need_device(m));
  TRY(exchange(m, m->U0, 0));
  TRY(standalone_reduce(m, m->U0, 0));
  m->have_state = true;
  return check_err(m);
  PH_API_END
}

ph_status ph_set_problem(ph_mesh* m, int32_t problem, const double* p, int32_t np) {
  PH_API_BEGIN
  if (m) m->w_ready = false;  // U0 changes (or is re-exchanged): W is rebuilt at the next step
  TRY(need_device(m));
  PgenArgs P{};
  P.problem = problem;
  for (int d = 0; d < 3; ++d) {
    P.xmin[d] = m->cfg.xmin[d];
    P.L[d] = m->cfg.xmax[d] - m->cfg.xmin[d];
  }
  if (np > 8) return fail(PH_ERR_INVALID_ARG, "too many problem parameters");
  for (int i = 0; i < np; ++i) P.p[i] = p[i];
  if (problem == PH_PROB_LINEAR_WAVE) {
    if (np < 4) return fail(PH_ERR_INVALID_ARG, "linear wave needs {A,k1,k2,k3}");
  } else if (problem == PH_PROB_SOD) {
    if (np < 1) P.p[0] = 0.5 * (m->cfg.xmin[0] + m->cfg.xmax[0]);
  } else if (problem == PH_PROB_BLAST) {
    if (np < 3) return fail(PH_ERR_INVALID_ARG, "blast needs {p_in,p_out,r[,cx,cy,cz]}");
    if (np < 6)
      for (int d = 0; d < 3; ++d) P.p[3 + d] = 0.5 * (m->cfg.xmin[d] + m->cfg.xmax[d]);
    if (!(P.p[0] > 0 && P.p[1] > 0 && P.p[2] > 0)) return fail(PH_ERR_INVALID_ARG, "blast parameters out of range");
  } else if (problem == PH_PROB_KH) {
    if (np < 1) P.p[0] = 0.01;
    if (np < 2) P.p[1] = 0.05;
    if (!(P.p[1] > 0)) return fail(PH_ERR_INVALID_ARG, "KH sigma must be positive");
  } else {
    return fail(PH_ERR_INVALID_ARG, "unknown problem");
  }
  if (m->cfg.refinement == PH_REF_ADAPTIVE) {
    // O9: AMR pre-refinement at t = 0 (generate, exchange, tag refine-only, refine + 2:1)
    for (int it = 0; it < m->cfg.max_level; ++it) {
      CU(launch_pgen(m->U0, m->d_meta, (int)m->local_gids.size(), P, m->G, m->stream));
      m->launches++;
      TRY(exchange(m, m->U0, 0));
      bool changed = false;
      TRY(tag_and_remesh(m, true, false, false, &changed));
      if (!changed) break;
    }
  }
  CU(launch_pgen(m->U0, m->d_meta, (int)m->local_gids.size(), P, m->G, m->stream));
  m->launches++;
  CU(cudaMemsetAsync(m->d_st, 0, sizeof(CycleState), m->stream));
  TRY(exchange(m, m->U0, 0));
  TRY(standalone_reduce(m, m->U0, 0));
  m->have_state = true;
  return check_err(m);
  PH_API_END
}

static int64_t slot_of(const ph_mesh* m, int64_t gid) {
  if (gid < 0 || gid >= (int64_t)m->blocks.size()) return -2;
  const BlockInfo& b = m->blocks[gid];
  return b.rank == m->rank ? b.local : -1;
}

ph_status ph_set_state(ph_mesh* m, int64_t gid, const double* cons, int64_t nelem) {
  PH_API_BEGIN
  if (m) m->w_ready = false;  // U0 changes (or is re-exchanged): W is rebuilt at the next step
  TRY(need_device(m));
  int64_t s = slot_of(m, gid);
  if (s == -2) return fail(PH_ERR_INVALID_ARG, "bad gid");
  const Geom& G = m->G;
  int64_t ni = (int64_t)NVAR * G.n[0] * G.n[1] * G.n[2];
  if (nelem != ni) return fail(PH_ERR_INVALID_ARG, "bad nelem");
  if (s < 0) return PH_OK;
  CU(cudaMemcpyAsync(m->stage_buf, cons, ni * sizeof(double), cudaMemcpyHostToDevice, m->stream));
  CU(launch_interior_copy(m->U0, m->stage_buf, (int)s, 1, 1, G, m->stream));
  m->launches++;
  CU(cudaStreamSynchronize(m->stream));
  m->have_state = true;
  return PH_OK;
  PH_API_END
}

ph_status ph_get_state(const ph_mesh* mc, int64_t gid, double* cons, int64_t nelem) {
  PH_API_BEGIN
  ph_mesh* m = const_cast<ph_mesh*>(mc);
  TRY(need_device(m));
  int64_t s = slot_of(m, gid);
  if (s == -2) return fail(PH_ERR_INVALID_ARG, "bad gid");
  const Geom& G = m->G;
  int64_t ni = (int64_t)NVAR * G.n[0] * G.n[1] * G.n[2];
  if (nelem != ni) return fail(PH_ERR_INVALID_ARG, "bad nelem");
  TRY(check_err(m));
  if (s < 0) return PH_OK;
  CU(launch_interior_copy(m->U0, m->stage_buf, (int)s, 1, 0, G, m->stream));
  m->launches++;
  CU(cudaMemcpyAsync(cons, m->stage_buf, ni * sizeof(double), cudaMemcpyDeviceToHost, m->stream));
  CU(cudaStreamSynchronize(m->stream));
  return PH_OK;
  PH_API_END
}

ph_status ph_get_state_full(const ph_mesh* mc, int64_t gid, double* out, int64_t nelem) {
  PH_API_BEGIN
  ph_mesh* m = const_cast<ph_mesh*>(mc);
  TRY(need_device(m));
  int64_t s = slot_of(m, gid);
  if (s == -2) return fail(PH_ERR_INVALID_ARG, "bad gid");
  if (nelem != m->G.bstride) return fail(PH_ERR_INVALID_ARG, "bad nelem");
  TRY(check_err(m));
  if (s < 0) return PH_OK;
  if (m->ghosts_stale && m->nranks == 1) {  // direct-halo cycles leave local face ghosts stale
    TRY(exchange(m, m->U0, 0));
    m->ghosts_stale = false;
  }
  CU(cudaMemcpyAsync(out, m->U0 + s * m->G.bstride, nelem * sizeof(double), cudaMemcpyDeviceToHost, m->stream));
  CU(cudaStreamSynchronize(m->stream));
  return PH_OK;
  PH_API_END
}

ph_status ph_set_state_full(ph_mesh* m, int64_t gid, const double* in, int64_t nelem) {
  PH_API_BEGIN
  if (m) m->w_ready = false;  // U0 changes (or is re-exchanged): W is rebuilt at the next step
  TRY(need_device(m));
  int64_t s = slot_of(m, gid);
  if (s == -2) return fail(PH_ERR_INVALID_ARG, "bad gid");
  if (nelem != m->G.bstride) return fail(PH_ERR_INVALID_ARG, "bad nelem");
  if (s < 0) return PH_OK;
  CU(cudaMemcpyAsync(m->U0 + s * m->G.bstride, in, nelem * sizeof(double), cudaMemcpyHostToDevice, m->stream));
  CU(cudaStreamSynchronize(m->stream));
  m->have_state = true;
  return PH_OK;
  PH_API_END
}

ph_status ph_step(ph_mesh* m, int32_t ncycles, double tlim, ph_step_info* info) {
  PH_API_BEGIN
  TRY(need_device(m));
  if (!m->have_state) return fail(PH_ERR_STATE, "no state: call ph_set_problem or ph_set_state + ph_refresh");
  CU(launch_cycle_begin(m->d_st, tlim, 1, m->stream));
  m->launches++;
  // Steady state: one CUDA graph per cycle (captured once, replayed; pointers are stable until a
  // remesh), on a private stream forked from / joined to the caller's stream (the legacy default
  // stream cannot be captured).  Adaptive meshes (host-side remesh decisions) and kernel-timing
  // runs stay eager on the caller's stream.
  const int32_t ncycles_req = ncycles;
  if (m->ho && m->ho_fold && !m->w_ready && ncycles > 0) {  // W from U0 first (prim_kernel): one eager cycle,
    TRY(one_cycle(m));                                     // so the captured graph can assume W is ready
    --ncycles;
    m->ghosts_stale = true;
  }
  const bool graph_ok = m->use_graph && !m->timing && m->cfg.refinement != PH_REF_ADAPTIVE && ncycles > 0;
  if (graph_ok) {
    if (!m->gstream) {
      CU(cudaStreamCreateWithFlags(&m->gstream, cudaStreamNonBlocking));
      CU(cudaEventCreateWithFlags(&m->ev_fork, cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&m->ev_join, cudaEventDisableTiming));
    }
    CU(cudaEventRecord(m->ev_fork, m->stream));
    CU(cudaStreamWaitEvent(m->gstream, m->ev_fork, 0));
    cudaStream_t caller = m->stream;
    m->stream = m->gstream;
    ph_status st = PH_OK;
    if (!m->graph_exec) {
      const int64_t l0 = m->launches;
      cudaGraph_t gr = nullptr;
      cudaError_t eb = cudaStreamBeginCapture(m->stream, cudaStreamCaptureModeThreadLocal);
      if (eb == cudaSuccess) {
        st = one_cycle(m);
        cudaError_t ec = cudaStreamEndCapture(m->stream, &gr);
        if (st == PH_OK && ec != cudaSuccess) st = fail(PH_ERR_CUDA, std::string("capture: ") + cudaGetErrorString(ec));
        if (st == PH_OK) {
          // keep the captured stream priorities (the boundary-first schedule's high-priority stream B):
          // without this flag a graph runs every node at the launching stream's priority, and the
          // interior blocks' stage kernel can take the GPU before the boundary blocks' one
          cudaError_t ei = cudaGraphInstantiate(&m->graph_exec, gr, cudaGraphInstantiateFlagUseNodePriority);
          if (ei != cudaSuccess) st = fail(PH_ERR_CUDA, std::string("instantiate: ") + cudaGetErrorString(ei));
        }
        if (gr) cudaGraphDestroy(gr);
      } else {
        st = fail(PH_ERR_CUDA, std::string("begin capture: ") + cudaGetErrorString(eb));
      }
      m->graph_launches = m->launches - l0;
      m->launches = l0;
    }
    for (int c = 0; c < ncycles && st == PH_OK; ++c) {
      cudaError_t e = cudaGraphLaunch(m->graph_exec, m->stream);
      if (e != cudaSuccess) st = fail(PH_ERR_CUDA, std::string("graph launch: ") + cudaGetErrorString(e));
      m->launches += m->graph_launches;
    }
    m->stream = caller;
    CU(cudaEventRecord(m->ev_join, m->gstream));
    CU(cudaStreamWaitEvent(m->stream, m->ev_join, 0));
    TRY(st);
  } else {
    for (int c = 0; c < ncycles; ++c) TRY(one_cycle(m));
  }
  if (ncycles > 0 && (m->direct_halo || (m->ho && m->ho_fold))) m->ghosts_stale = true;
  if (info) {
    TRY(check_err(m));
    CycleState st;
    CU(cudaMemcpy(&st, m->d_st, sizeof st, cudaMemcpyDeviceToHost));
    info->cycle = st.cycle;
    info->t = st.t;
    info->dt = st.dt;
    int64_t cells = (int64_t)m->blocks.size() * m->G.n[0] * m->G.n[1] * m->G.n[2];
    info->zone_cycles = cells * ncycles_req;
  }
  return PH_OK;
  PH_API_END
}

ph_status ph_step_host(ph_mesh* m, const double* host_in, double* host_out, int64_t nelem, int32_t ncycles,
                       double tlim) {
  PH_API_BEGIN
  TRY(ph_step_host_async(m, host_in, host_out, nelem, ncycles, tlim));
  return check_err(m);
  PH_API_END
}

ph_status ph_sync(ph_mesh* m) {
  PH_API_BEGIN
  TRY(need_device(m));
  return check_err(m);
  PH_API_END
}

ph_status ph_step_host_async(ph_mesh* m, const double* host_in, double* host_out, int64_t nelem, int32_t ncycles,
                             double tlim) {
  PH_API_BEGIN
  if (m) m->w_ready = false;
  TRY(need_device(m));
  // an adaptive mesh may remesh inside ph_step: the local block set (and so the layout of host_out)
  // would change under the copy-back
  if (m->cfg.refinement == PH_REF_ADAPTIVE)
    return fail(PH_ERR_UNSUPPORTED, "ph_step_host on an adaptive mesh: use ph_set_state / ph_step / ph_get_state");
  const Geom& G = m->G;
  int64_t nloc = (int64_t)m->local_gids.size();
  int64_t ni = nloc * NVAR * G.n[0] * G.n[1] * G.n[2];
  if (nelem != ni) return fail(PH_ERR_INVALID_ARG, "bad nelem (expect nlocal*5*n3*n2*n1)");
  if (ni) CU(cudaMemcpyAsync(m->stage_buf, host_in, ni * sizeof(double), cudaMemcpyHostToDevice, m->stream));
  if (nloc) {
    CU(launch_interior_copy(m->U0, m->stage_buf, 0, (int)nloc, 1, G, m->stream));
    m->launches++;
  }
  m->have_state = true;
  TRY(exchange(m, m->U0, 0));
  TRY(standalone_reduce(m, m->U0, 0));
  TRY(ph_step(m, ncycles, tlim, nullptr));
  if (nloc) {
    CU(launch_interior_copy(m->U0, m->stage_buf, 0, (int)nloc, 0, G, m->stream));
    m->launches++;
  }
  if (ni) CU(cudaMemcpyAsync(host_out, m->stage_buf, ni * sizeof(double), cudaMemcpyDeviceToHost, m->stream));
  return PH_OK;
  PH_API_END
}

ph_status ph_num_blocks(const ph_mesh* m, int64_t* nglobal, int64_t* nlocal) {
  PH_API_BEGIN
  if (!m) return fail(PH_ERR_INVALID_ARG, "null mesh");
  if (nglobal) *nglobal = (int64_t)m->blocks.size();
  if (nlocal) *nlocal = (int64_t)m->local_gids.size();
  return PH_OK;
  PH_API_END
}

ph_status ph_get_blocks(const ph_mesh* m, ph_block* out, int64_t cap, int64_t* n) {
  PH_API_BEGIN
  if (!m || !n) return fail(PH_ERR_INVALID_ARG, "null argument");
  *n = (int64_t)m->blocks.size();
  for (int64_t g = 0; g < *n && g < cap; ++g) {
    const BlockInfo& b = m->blocks[g];
    out[g].gid = b.gid;
    out[g].level = b.loc.level;
    out[g].rank = b.rank;
    for (int d = 0; d < 3; ++d) {
      out[g].lx[d] = b.loc.x[d];
      out[g].xmin[d] = b.xmin[d];
      out[g].xmax[d] = b.xmax[d];
    }
  }
  return PH_OK;
  PH_API_END
}

ph_status ph_get_neighbors(const ph_mesh* m, int64_t gid, ph_neighbor* out, int32_t cap, int32_t* n) {
  PH_API_BEGIN
  if (!m || !n) return fail(PH_ERR_INVALID_ARG, "null argument");
  if (gid < 0 || gid >= (int64_t)m->blocks.size()) return fail(PH_ERR_INVALID_ARG, "bad gid");
  const BlockInfo& b = m->blocks[gid];
  *n = (int32_t)b.nbrs.size();
  for (int32_t q = 0; q < *n && q < cap; ++q) {
    const Neighbor& e = b.nbrs[q];
    out[q].gid = e.gid;
    out[q].rank = e.rank;
    for (int d = 0; d < 3; ++d) out[q].off[d] = e.off[d];
    out[q].dlevel = e.dlevel;
    out[q].fine[0] = e.fine[0];
    out[q].fine[1] = e.fine[1];
  }
  return PH_OK;
  PH_API_END
}

ph_status ph_get_refine_flags(const ph_mesh* m, int8_t* out, int64_t cap, int64_t* n) {
  PH_API_BEGIN
  if (!m || !n) return fail(PH_ERR_INVALID_ARG, "null argument");
  *n = (int64_t)m->last_flags.size();
  for (int64_t i = 0; i < *n && i < cap; ++i) out[i] = m->last_flags[i];
  return PH_OK;
  PH_API_END
}

ph_status ph_get_history(const ph_mesh* mc, double* out, int64_t cap_rows, int64_t* nrows) {
  PH_API_BEGIN
  ph_mesh* m = const_cast<ph_mesh*>(mc);
  TRY(need_device(m));
  TRY(check_err(m));
  CycleState st;
  CU(cudaMemcpy(&st, m->d_st, sizeof st, cudaMemcpyDeviceToHost));
  int64_t n = std::min<int64_t>(st.hist_count, m->hist_cap);
  *nrows = n;
  std::vector<double> h((size_t)m->hist_cap * 7);
  CU(cudaMemcpy(h.data(), m->hist, h.size() * sizeof(double), cudaMemcpyDeviceToHost));
  int64_t first = st.hist_count - n;
  for (int64_t r = 0; r < n && r < cap_rows; ++r) {
    int64_t q = (first + r) % m->hist_cap;
    for (int c = 0; c < 7; ++c) out[r * 7 + c] = h[q * 7 + c];
  }
  return PH_OK;
  PH_API_END
}

ph_status ph_get_time(const ph_mesh* mc, double* t, double* dt, int64_t* cycle) {
  PH_API_BEGIN
  ph_mesh* m = const_cast<ph_mesh*>(mc);
  TRY(need_device(m));
  TRY(check_err(m));
  CycleState st;
  CU(cudaMemcpy(&st, m->d_st, sizeof st, cudaMemcpyDeviceToHost));
  if (t) *t = st.t;
  if (dt) *dt = st.dt;
  if (cycle) *cycle = st.cycle;
  return PH_OK;
  PH_API_END
}

ph_status ph_totals(ph_mesh* m, double out[5]) {
  PH_API_BEGIN
  TRY(need_device(m));
  int nloc = (int)m->local_gids.size();
  if (nloc > 0) {
    CU(launch_reduce(m->U0, m->d_meta, nloc, m->partials, m->d_err, m->G, m->stream));
    m->launches++;
  }
  CU(launch_rank_reduce(m->partials, nloc * m->G.n[2], m->nranks > 1 ? m->my6 : m->all6, m->stream));
  m->launches++;
  if (m->nranks > 1) NC(ncclAllGather(m->my6, m->all6, 6, ncclDouble, m->comm, m->stream));
  CU(launch_finalize(m->all6, m->nranks, m->d_st, m->hist, m->hist_cap, m->G.cfl, 2, m->tot5, m->G.exact, m->stream));
  m->launches++;
  TRY(check_err(m));
  CU(cudaMemcpy(out, m->tot5, 5 * sizeof(double), cudaMemcpyDeviceToHost));
  return PH_OK;
  PH_API_END
}

ph_status ph_get_plan_info(const ph_mesh* m, ph_plan_info* out) {
  PH_API_BEGIN
  if (!m || !out) return fail(PH_ERR_INVALID_ARG, "null argument");
  memset(out, 0, sizeof *out);
  const Plan& PL = m->plan[0];
  out->n_local_tasks = (int64_t)PL.local.tasks.size();
  out->n_send_tasks = (int64_t)PL.pack.tasks.size();
  out->n_recv_tasks = (int64_t)PL.unpack.tasks.size();
  for (int p = 0; p < m->nranks && p < 64; ++p) {
    out->send_doubles_to[p] = PL.send_cnt[p];
    out->recv_doubles_from[p] = PL.recv_cnt[p];
    out->send_hash_to[p] = PL.send_hash[p];
    out->recv_hash_from[p] = PL.recv_hash[p];
    out->cyc_send_doubles_to[p] = m->plan[1].send_cnt[p];
    out->cyc_recv_doubles_from[p] = m->plan[1].recv_cnt[p];
    out->cyc_send_hash_to[p] = m->plan[1].send_hash[p];
    out->cyc_recv_hash_from[p] = m->plan[1].recv_hash[p];
  }
  out->direct_halo = m->direct_halo ? 1 : 0;
  out->peer_halo = m->peer ? 1 : 0;
  out->n_cyc_local_tasks = (int64_t)m->plan[1].local.tasks.size();
  return PH_OK;
  PH_API_END
}

ph_status ph_launch_count(const ph_mesh* m, int64_t* n) {
  PH_API_BEGIN
  if (!m || !n) return fail(PH_ERR_INVALID_ARG, "null argument");
  *n = m->launches;
  return PH_OK;
  PH_API_END
}

ph_status ph_kernel_timing(ph_mesh* m, int32_t enable, double* stage_ms, int64_t* stage_launches, double* exch_ms,
                           int64_t* exch_launches) {
  PH_API_BEGIN
  TRY(need_device(m));
  CU(cudaStreamSynchronize(m->stream));
  double s = 0, x = 0;
  for (auto& p : m->t_stage) {
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, p.first, p.second));
    s += ms;
  }
  for (auto& p : m->t_exch) {
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, p.first, p.second));
    x += ms;
  }
  if (stage_ms) *stage_ms = s;
  if (stage_launches) *stage_launches = (int64_t)m->t_stage.size();
  if (exch_ms) *exch_ms = x;
  if (exch_launches) *exch_launches = (int64_t)m->t_exch.size();
  m->t_stage.clear();
  m->t_exch.clear();
  for (cudaEvent_t e : m->ev_pool) cudaEventDestroy(e);
  m->ev_pool.clear();
  m->timing = enable != 0;
  return PH_OK;
  PH_API_END
}

}  // extern "C"
