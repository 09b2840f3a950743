// stage2.cu -- the uniform-mesh stage kernel, second design (round 2).
//
// Same method as stage_kernel in kernels.cu (cons->prim a2, PLM-minmod a3, HLLE a4 on every x/y/z
// face, flux divergence + RK stage combine a5, CFL / totals partials a6 / a10; SURVEY §8(c) O5,
// P:696-698), re-mapped onto the resources that bound it on B200 (profiles/r02_ubench_fp64.jsonl:
// fp64 DFMA/DADD 60 lanes/clk/SM, MUFU.RCP64H/RSQ64H 16, shared memory 128 B/clk/SM, issue
// ~3 warp-instr/clk/SM when fp64 is mixed in):
//
//  * CTA = a 16 x 16 (i, j) tile of one block marching up a k-range, 128 threads, 3 CTAs per SM.
//    Thread (row r, pair p) owns the x-pair of cells (2p, 2p+1) of row r; warp w owns rows 4w..4w+3.
//  * Planes arrive by TMA (cp.async.bulk.tensor over a 5-D tensor map of the pool [slot][v][k][j][i],
//    SASS UTMALDG) on an mbarrier per ring slot: one elected thread issues <= 5 boxes per plane
//    (16 x 16 centre, 2 x 16 x-halo columns on each side, 16 x 2 y-halo rows on each side, all 5
//    variables per box) one full step ahead into a 4-slot ring; the plane is converted to
//    primitives in place.  Halo boxes outside the block come straight from the local same-level
//    face neighbour's interior (direct halo: just another slot coordinate), else from the block's
//    own ghost zone.  No per-thread global loads, no prefetch registers.
//  * One __syncthreads per plane (after the conversion); every face a warp needs is computed by
//    that warp: x faces 2p-1/2 and 2p+1/2 per lane (lane 0 of a row builds the left halo cell's
//    state itself), each cell's x slope once, the left neighbour's top state and the right
//    neighbour's face flux by warp shuffles; y faces j-1/2 per lane with the 4-row stencil read by
//    128-bit shared loads, face j+1/2 shuffled down from the row above, or -- for the warp's top row
//    -- taken from the warp above through shared memory behind a pairwise named barrier (bar.arrive /
//    bar.sync, 64 threads), so no face is computed twice.  The tile's 16 top y faces and 16 right x
//    faces are computed one step ahead by one warp (rotating) into a double-buffered area.  z: each
//    column's top state and last face flux are carried in registers (one slope per cell).  The 128
//    halo cells of a plane are converted one per thread.  (PH_S2_V3=1: the earlier variant in which
//    every warp computes its own top faces in an extra round, 2.5x the extra faces.)
//  * HLLE in the alpha/beta form: with a = b+/(b+ - b-), b = -b-/(b+ - b-), e = a b-,
//      beta_L = a u_L - e, beta_R = b u_R + e, alpha = rho beta,
//      F = (alpha_L + alpha_R, u_L alpha_L + u_R alpha_R + a p_L + b p_R, v alpha.., w alpha..,
//           H_L beta_L + H_R beta_R + e (p_L - p_R)),   H = E + p,
//    which is algebraically ((b+ F_L - b- F_R) + b+ b- (U_R - U_L)) / (b+ - b-) (O5 / A5) in 60
//    fp64 operations instead of ~78; results agree with the oracle's form to round-off.
//  * The finish operand of plane c (U^n for stage 1, H = a0 U^n + b1 U^1 for stage 2) is a TMA box
//    issued at the start of the same step; finished cells leave with 128-bit stores.
//
// Shared memory per CTA: ring 4 x 15,360 B + finish 10,240 + reduction 192 + tile-boundary faces 2,560
// + warp-boundary faces 1,920 + 5 mbarriers = 76,392 B (3 CTAs per SM: 3 x (76,392 + 1,024 reserved)
// <= 228 KB).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "device.cuh"
#include "point.cuh"

namespace ph {
namespace s2 {

constexpr int TX = 16, TY = 16, NTH = 128, NW = NTH / 32;
// one ring slot (doubles): centre [5][TY][TX], x-halo [5][TY][2] left and right, y-halo [5][2][TX]
// below and above -- each region is exactly what one TMA box lands (offsets are 128-B aligned)
constexpr int VM = TY * TX, VX = TY * 2, VY = 2 * TX;  // variable strides of the regions
constexpr int R_M = 0, R_XL = NVAR * VM, R_XR = R_XL + NVAR * VX, R_YL = R_XR + NVAR * VX, R_YH = R_YL + NVAR * VY;
constexpr int PLANE = R_YH + NVAR * VY;                // 1920 doubles = 15,360 B
constexpr int NSLOT = 4;
constexpr int OFF_FIN = NSLOT * PLANE;                 // [5][TY][TX]
constexpr int OFF_RED = OFF_FIN + NVAR * VM;           // [NW][6]
#ifndef PH_S2_V3
constexpr int OFF_XB = OFF_RED + NW * 6;               // [2][5][32]: tile-top y faces (16) + right x faces (16), one step ahead
constexpr int OFF_FB = OFF_XB + 2 * NVAR * 32;         // [NW-1][5][TX]: bottom-row y faces of warps 1..3 for the warp below
constexpr int OFF_BAR = OFF_FB + (NW - 1) * NVAR * TX; // full[NSLOT], fin
#else
constexpr int OFF_FE = OFF_RED + NW * 6;               // [NW][5][20]: the extra round's faces
constexpr int OFF_BAR = OFF_FE + NW * NVAR * 20;       // full[NSLOT], fin
#endif
constexpr int SMEM_DOUBLES = OFF_BAR + NSLOT + 1;
constexpr size_t SMEM_BYTES = SMEM_DOUBLES * sizeof(double);
constexpr uint32_t MAIN_BYTES = PLANE * 8;             // centre + 4 halo boxes
constexpr uint32_t OWN_BYTES = NVAR * VM * 8;          // halo planes (centre only) and the finish operand
static_assert((R_XL * 8) % 128 == 0 && (R_XR * 8) % 128 == 0 && (R_YL * 8) % 128 == 0 && (R_YH * 8) % 128 == 0 &&
                  (PLANE * 8) % 128 == 0 && (OFF_FIN * 8) % 128 == 0,
              "TMA destinations are 128-B aligned");

// tensor maps of one stage launch (5-D over a pool: i, j, k, v, slot; box extents differ)
struct Maps {
  CUtensorMap c;   // input pool, box {TX, TY, 1, 5, 1}
  CUtensorMap xh;  // input pool, box {2, TY, 1, 5, 1}
  CUtensorMap yh;  // input pool, box {TX, 2, 1, 5, 1}
  CUtensorMap f;   // finish-operand pool, box {TX, TY, 1, 5, 1}
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra.uni WAIT_%=;\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
// TMA box load: global (tensor map, 5 coordinates) -> shared, completion counted on `bar`
__device__ __forceinline__ void tma5(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, int c4,
                                     uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
      "%6}], [%7];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(su32(bar))
      : "memory");
}
// TMA box prefetch into L2 (no shared memory, no completion): the next step's loads then hit L2
__device__ __forceinline__ void tma5_l2(const CUtensorMap* map, int c0, int c1, int c2, int c3, int c4) {
  asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void sts2(double* p, double a, double b) { *reinterpret_cast<double2*>(p) = make_double2(a, b); }
__device__ __forceinline__ void stg2(double* p, double a, double b) {
  __stcg(reinterpret_cast<double2*>(p), make_double2(a, b));
}

// q + h m with h = 0.5 (same strict sign) or 0, m the smaller-magnitude difference: q + 0.5 minmod
__device__ __forceinline__ void mm_states(double dl, double dr, double q, double& bot, double& top) {
  const double h = minmod_half(dl, dr), m = minmod_pick(dl, dr);
  bot = fma(-h, m, q);
  top = fma(h, m, q);
}

// max(x, 0) and min(x, 0) on the integer pipe (sign-bit mask; no fp64 compare)
__device__ __forceinline__ double pos_part(double x) {
  const int hi = __double2hiint(x), m = ~(hi >> 31);
  return __hiloint2double(hi & m, __double2loint(x) & m);
}
__device__ __forceinline__ double neg_part(double x) {
  const int hi = __double2hiint(x), m = hi >> 31;
  return __hiloint2double(hi & m, __double2loint(x) & m);
}

// HLLE (Davis speeds, clamped, branch-free) in the alpha/beta form; normal velocity component N.
template <int N>
__device__ __forceinline__ void hlle_ab(const double* wl, const double* wr, double gamma, double ggm1, double* F) {
  constexpr int T1 = N == 1 ? 2 : (N == 2 ? 3 : 1), T2 = N == 1 ? 3 : (N == 2 ? 1 : 2);
  const double rl = wl[0], ul = wl[N], pl = wl[4], rr = wr[0], ur = wr[N], pr = wr[4];
  const double cl = sound_speed(rl, pl, gamma), cr = sound_speed(rr, pr, gamma);
  const double sl = dmin(ul - cl, ur - cr), sr = dmax(ul + cl, ur + cr);
  const double bp = pos_part(sr), bm = neg_part(sl);
  const double inv = rcp_nr(bp - bm);
  const double a = bp * inv, b = -bm * inv, e = a * bm;
  const double btl = fma(a, ul, -e), btr = fma(b, ur, e);
  const double al = rl * btl, ar = rr * btr;
  F[0] = al + ar;
  F[N] = fma(ul, al, fma(ur, ar, fma(a, pl, b * pr)));
  F[T1] = fma(wl[T1], al, wr[T1] * ar);
  F[T2] = fma(wl[T2], al, wr[T2] * ar);
  const double kl = fma(ul, ul, fma(wl[T1], wl[T1], wl[T2] * wl[T2]));
  const double kr = fma(ur, ur, fma(wr[T1], wr[T1], wr[T2] * wr[T2]));
  const double hl = fma(pl, ggm1, (0.5 * rl) * kl), hr = fma(pr, ggm1, (0.5 * rr) * kr);
  F[4] = fma(hl, btl, fma(hr, btr, e * (pl - pr)));
}

// two faces at once (the pair's two columns / faces): the same arithmetic as hlle_ab, written so
// the two dependency chains interleave (PH_S2_X2 A/B knob; default: two hlle_ab calls)
template <int N>
__device__ __forceinline__ void hlle_ab2(const double (&wl)[2][NVAR], const double (&wr)[2][NVAR], double gamma,
                                         double ggm1, double (&F)[2][NVAR]) {
#ifdef PH_S2_X2
  constexpr int T1 = N == 1 ? 2 : (N == 2 ? 3 : 1), T2 = N == 1 ? 3 : (N == 2 ? 1 : 2);
  double cl[2], cr[2], bp[2], bm[2], inv[2], a[2], b[2], e[2], btl[2], btr[2], al[2], ar[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    cl[k] = sound_speed(wl[k][0], wl[k][4], gamma);
    cr[k] = sound_speed(wr[k][0], wr[k][4], gamma);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double ul = wl[k][N], ur = wr[k][N];
    bp[k] = pos_part(dmax(ul + cl[k], ur + cr[k]));
    bm[k] = neg_part(dmin(ul - cl[k], ur - cr[k]));
    inv[k] = rcp_nr(bp[k] - bm[k]);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    a[k] = bp[k] * inv[k];
    b[k] = -bm[k] * inv[k];
    e[k] = a[k] * bm[k];
    btl[k] = fma(a[k], wl[k][N], -e[k]);
    btr[k] = fma(b[k], wr[k][N], e[k]);
    al[k] = wl[k][0] * btl[k];
    ar[k] = wr[k][0] * btr[k];
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double ul = wl[k][N], ur = wr[k][N], pl = wl[k][4], pr = wr[k][4];
    F[k][0] = al[k] + ar[k];
    F[k][N] = fma(ul, al[k], fma(ur, ar[k], fma(a[k], pl, b[k] * pr)));
    F[k][T1] = fma(wl[k][T1], al[k], wr[k][T1] * ar[k]);
    F[k][T2] = fma(wl[k][T2], al[k], wr[k][T2] * ar[k]);
    const double kl = fma(ul, ul, fma(wl[k][T1], wl[k][T1], wl[k][T2] * wl[k][T2]));
    const double kr = fma(ur, ur, fma(wr[k][T1], wr[k][T1], wr[k][T2] * wr[k][T2]));
    const double hl = fma(pl, ggm1, (0.5 * wl[k][0]) * kl), hr = fma(pr, ggm1, (0.5 * wr[k][0]) * kr);
    F[k][4] = fma(hl, btl[k], fma(hr, btr[k], e[k] * (pl - pr)));
  }
#else
  hlle_ab<N>(wl[0], wr[0], gamma, ggm1, F[0]);
  hlle_ab<N>(wl[1], wr[1], gamma, ggm1, F[1]);
#endif
}

// cons -> prim of the cell pair at p (in place, variable stride vs), a2; returns the primitives
__device__ __forceinline__ void convert_pair(double* p, int vs, double gm1, double (&w)[2][NVAR], ErrWord* err,
                                             int stage, long long gid, int k, int j, int i) {
  double u[2][NVAR];
#pragma unroll
  for (int v = 0; v < NVAR; ++v) {
    const double2 t = lds2(p + v * vs);
    u[0][v] = t.x;
    u[1][v] = t.y;
  }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const double rho = u[e][0], ir = rcp_nr(rho);
    const double v1 = u[e][1] * ir, v2 = u[e][2] * ir, v3 = u[e][3] * ir;
    const double ke = 0.5 * ((u[e][1] * v1 + u[e][2] * v2) + u[e][3] * v3);
    const double pr = gm1 * (u[e][4] - ke);
    if (!(rho > 0.0) || !(pr > 0.0)) set_error(err, stage, gid, k, j, i + e);
    w[e][0] = rho;
    w[e][1] = v1;
    w[e][2] = v2;
    w[e][3] = v3;
    w[e][4] = pr;
  }
#pragma unroll
  for (int v = 0; v < NVAR; ++v) sts2(p + v * vs, w[0][v], w[1][v]);
}

// one face from its 4-cell stencil: cells c-2, c-1 at pa, pa + st (variable stride sa) and c, c+1 at
// pb, pb + st (variable stride sb) of a primitive plane; normal component n (runtime: the boundary
// round mixes x and y faces); flux in natural order
__device__ __forceinline__ void face4(const double* pa, int sa, const double* pb, int sb, int st, int n, double gamma,
                                      double ggm1, double* F) {
  const int t1 = n == 1 ? 2 : 3, t2 = n == 1 ? 3 : 1;
  const int cv[NVAR] = {0, n, t1, t2, 4};
  double wl[NVAR], wr[NVAR], Fc[NVAR];
#pragma unroll
  for (int s = 0; s < NVAR; ++s) {
    const double a = pa[cv[s] * sa], b = pa[cv[s] * sa + st], c = pb[cv[s] * sb], d = pb[cv[s] * sb + st];
    double t;
    mm_states(b - a, c - b, b, t, wl[s]);
    mm_states(c - b, d - c, c, wr[s], t);
  }
  hlle_ab<1>(wl, wr, gamma, ggm1, Fc);
  F[0] = Fc[0];
  F[n] = Fc[1];
  F[t1] = Fc[2];
  F[t2] = Fc[3];
  F[4] = Fc[4];
}

// row rr (-2 .. TY+1) of column pair i0 in a ring slot: offset and variable stride
__device__ __forceinline__ void row_at(int rr, int i0, int& off, int& vs) {
  if (rr < 0) { off = R_YL + (rr + 2) * TX + i0; vs = VY; }
  else if (rr >= TY) { off = R_YH + (rr - TY) * TX + i0; vs = VY; }
  else { off = R_M + rr * TX + i0; vs = VM; }
}

// S2 = false: stage 1 (finish operand U_in = U^n; writes U1 and H = ha0 U^n + hb1 U1);
// S2 = true: stage 2 (finish operand H; writes H + cdt dt L).  REDUCE: CFL / totals partials.
#ifndef PH_S2_MINB
#define PH_S2_MINB 3  // CTAs per SM the register allocation is sized for (A/B knob)
#endif
// PUT: fused peer put (boundary blocks, peer-memory halo, PH_FUSED_PUT=1): finished cells within g
// layers of a face whose neighbour lives on another GPU are also stored into that GPU's receive
// buffer, at the place its unpack reads ([v][box], box (k, j, i)-major).
// ML: multilevel meshes (a8): fluxes of faces on a coarse-fine block face also go to the face-flux
// slots (M.fslot) for the reflux, and with REDUCE the cells of flux-corrected layers are left to
// rfx_reduce_kernel (they change after this kernel).
template <bool REDUCE, bool S2, bool PUT, bool ML>
__global__ void __launch_bounds__(NTH, PH_S2_MINB) stage2_kernel(StageArgs A, Geom G, const __grid_constant__ Maps maps) {
  extern __shared__ __align__(128) double sm[];
  double* fin = sm + OFF_FIN;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + OFF_BAR);  // full[0..NSLOT), fin = bar[NSLOT]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kr = lane >> 3, r = (warp << 2) + kr, p = lane & 7, i0 = 2 * p;
  int bid = blockIdx.x;
  const int kc = bid % A.nkc;
  bid /= A.nkc;
  const int tyi = bid % A.nty;
  bid /= A.nty;
  const int txi = bid % A.ntx;
  const int slot = A.slots[bid / A.ntx];
  const BlockMeta& M = A.meta[slot];
  const int x0 = txi * TX, y0 = tyi * TY;
  const int k0 = kc * A.KC, k1 = min(k0 + A.KC, G.n[2]);
  const int g = G.g, n3 = G.n[2];
  const int64_t plane = (int64_t)G.N[0] * G.N[1];
  const long long gid = M.gid;
  const double idx1 = M.idx[0], idx2 = M.idx[1], idx3 = M.idx[2];
  const double gamma = G.gamma, gm1 = G.gm1, ggm1 = G.gamma * G.inv_gm1;
  const double cdt = A.cdt * A.st->dt_used;
  const int own = R_M + r * TX + i0;  // own pair in a ring slot (centre region)
  // multilevel: flux F of the face at index (a, b) of block face f into its slot ([v][b][a] over the
  // face's two tangential extents, the slower one b)
  auto ml_put = [&](int f, int a, int b, const double* F) {
    const int fs = M.fslot[f];
    if (fs < 0) return;
    const int d = f >> 1, ta = d == 0 ? 1 : 0, tb = d == 2 ? 1 : 2;
    const int64_t fstr = (int64_t)G.n[ta] * G.n[tb];
    double* o = A.fbuf + (int64_t)fs * G.fstride + (int64_t)b * G.n[ta] + a;
#pragma unroll
    for (int v = 0; v < NVAR; ++v) o[v * fstr] = F[v];
  };

  auto issue_plane = [&](int q, int s) {  // tid 0 only
    uint64_t* fb = bar + s;
    double* base = sm + s * PLANE;
    fence_proxy_async();
    if (q >= k0 && q < k1) {
      // halo boxes: direct halo from the local same-level face neighbour when there is one, else the
      // own block's ghost zone (coordinates are pool indices incl. the ghost offset)
      const int n1 = G.n[0], n2 = G.n[1];
      const int nb0 = M.nb[0], nb1 = M.nb[1], nb2 = M.nb[2], nb3 = M.nb[3];
      const bool dl = x0 == 0 && nb0 >= 0, dr = x0 + TX == n1 && nb1 >= 0;
      const bool db = y0 == 0 && nb2 >= 0, dt = y0 + TY == n2 && nb3 >= 0;
      const int xl_b = dl ? nb0 : slot, xl_x = dl ? n1 - 2 + g : x0 - 2 + g;
      const int xr_b = dr ? nb1 : slot, xr_x = dr ? g : x0 + TX + g;
      const int yl_b = db ? nb2 : slot, yl_y = db ? n2 - 2 + g : y0 - 2 + g;
      const int yh_b = dt ? nb3 : slot, yh_y = dt ? g : y0 + TY + g;
      mbar_expect_tx(fb, MAIN_BYTES);
      const int z = q + g;
      tma5(base + R_M, &maps.c, x0 + g, y0 + g, z, 0, slot, fb);
      tma5(base + R_XL, &maps.xh, xl_x, y0 + g, z, 0, xl_b, fb);
      tma5(base + R_XR, &maps.xh, xr_x, y0 + g, z, 0, xr_b, fb);
      tma5(base + R_YL, &maps.yh, x0 + g, yl_y, z, 0, yl_b, fb);
      tma5(base + R_YH, &maps.yh, x0 + g, yh_y, z, 0, yh_b, fb);
    } else {
      int b = slot, qq = q;
      const int zl_b = M.nb[4], zh_b = M.nb[5];
      if (q < 0 && zl_b >= 0) { b = zl_b; qq += n3; }
      else if (q >= n3 && zh_b >= 0) { b = zh_b; qq -= n3; }
      mbar_expect_tx(fb, OWN_BYTES);
      tma5(base + R_M, &maps.c, x0 + g, y0 + g, qq + g, 0, b, fb);
    }
  };

  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.c)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.xh)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.yh)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.f)) : "memory");
#pragma unroll
    for (int b = 0; b <= NSLOT; ++b) mbar_init(bar + b, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  double topz[2][NVAR], fzp[2][NVAR];
#pragma unroll
  for (int e = 0; e < 2; ++e)
#pragma unroll
    for (int v = 0; v < NVAR; ++v) topz[e][v] = fzp[e][v] = 0.0;
  double tmax = 0.0, tsum[NVAR] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const int qbeg = k0 - 2, qend = k1 + 2;
  if (tid == 0) issue_plane(qbeg, 0);
  int s = 0;
#ifdef PH_S2_UNROLL2
#pragma unroll 2
#else
#pragma unroll 1
#endif
  for (int q = qbeg; q < qend; ++q) {
    const int idx = q - qbeg;
    const int s1 = (s + NSLOT - 1) & (NSLOT - 1);  // slot of plane q-1
    const int s2 = (s + NSLOT - 2) & (NSLOT - 1);  // slot of plane q-2
    const int c = q - 2;
    const bool mainp = q >= k0 && q < k1, cact = c >= k0 && c < k1;
    double* Wq = sm + s * PLANE;
    ph_jitter(4 * q + 0);
    mbar_wait(bar + s, (uint32_t)(idx / NSLOT) & 1u);
    // ---- a2: cons -> prim of plane q, in place
    double wq[2][NVAR];
    convert_pair(Wq + own, VM, gm1, wq, A.err, A.stage, gid, q, y0 + r, x0 + i0);
    if (mainp) {
      // 128 halo cells, one per thread (no idle half-warps): x-halo left / right (2 per row), y-halo
      // below / above (16 per row)
      const int h = tid;
      int off, vs, jj, ii;
      if (h < 64) {
        const int rr = (h >> 1) & 15, e = h & 1;
        off = (h < 32 ? R_XL : R_XR) + rr * 2 + e;
        vs = VX;
        jj = rr;
        ii = (h < 32 ? -2 : TX) + e;
      } else {
        const int hh = h - 64, hr = (hh >> 4) & 1, col = hh & 15;
        off = (hh < 32 ? R_YL : R_YH) + hr * TX + col;
        vs = VY;
        jj = hh < 32 ? hr - 2 : TY + hr;
        ii = col;
      }
      double u[NVAR];
#pragma unroll
      for (int v = 0; v < NVAR; ++v) u[v] = Wq[off + v * vs];
      const double rho = u[0], ir = rcp_nr(rho);
      const double v1 = u[1] * ir, v2 = u[2] * ir, v3 = u[3] * ir;
      const double ke = 0.5 * ((u[1] * v1 + u[2] * v2) + u[3] * v3);
      const double pr = gm1 * (u[4] - ke);
      if (!(rho > 0.0) || !(pr > 0.0)) set_error(A.err, A.stage, gid, q, y0 + jj, x0 + ii);
      Wq[off] = rho;
      Wq[off + vs] = v1;
      Wq[off + 2 * vs] = v2;
      Wq[off + 3 * vs] = v3;
      Wq[off + 4 * vs] = pr;
    }
    ph_jitter(4 * q + 1);
    __syncthreads();  // plane q primitives visible; step q-1 done everywhere (its slot and fin free)
    ph_jitter(4 * q + 2);
    if (tid == 0) {
      if (q + 1 < qend) issue_plane(q + 1, (s + 1) & (NSLOT - 1));
      if (cact) {
        fence_proxy_async();
        mbar_expect_tx(bar + NSLOT, OWN_BYTES);
        tma5(fin, &maps.f, x0 + g, y0 + g, c + g, 0, slot, bar + NSLOT);
      }
#ifdef PH_S2_PF
      // (A/B knob, off: 2b 1.03e10 with both prefetches vs 1.06e10 without) one step further ahead, into L2
      // only: the finish operand of plane c+1 (and with PH_S2_PF=2 the centre box of plane q+2)
#if PH_S2_PF > 1
      if (q + 2 >= k0 && q + 2 < k1) tma5_l2(&maps.c, x0 + g, y0 + g, q + 2 + g, 0, slot);
#endif
      if (c + 1 >= k0 && c + 1 < k1) tma5_l2(&maps.f, x0 + g, y0 + g, c + 1 + g, 0, slot);
#endif
    }

    double dz[2][NVAR];
#if !defined(PH_S2_V3) && defined(PH_S2_XSTART)
    // one step ahead, one warp (rotating): plane q-1's tile-top y faces (lanes 0..15, rows 14..17) and
    // right x faces (lanes 16..31, cells 14..17 of row lane-16), for every warp's use next step
    if (q - 1 >= k0 && q - 1 < k1 && warp == (q & (NW - 1))) {
      const double* W1 = sm + s1 * PLANE;
      double Fe[NVAR];
      if (lane < TX)
        face4(W1 + R_M + (TY - 2) * TX + lane, VM, W1 + R_YH + lane, VY, TX, 2, gamma, ggm1, Fe);
      else
        face4(W1 + R_M + (lane - TX) * TX + TX - 2, VM, W1 + R_XR + (lane - TX) * 2, VX, 1, 1, gamma, ggm1, Fe);
      double* xo = sm + OFF_XB + ((q - 1) & 1) * NVAR * 32 + lane;
#pragma unroll
      for (int v = 0; v < NVAR; ++v) xo[v * 32] = Fe[v];
      if (ML) {
        if (lane < TX && y0 + TY == G.n[1]) ml_put(3, x0 + lane, q - 1, Fe);             // y face n2: [v][k][i]
        if (lane >= TX && x0 + TX == G.n[0]) ml_put(1, y0 + lane - TX, q - 1, Fe);       // x face n1: [v][k][j]
      }
    }
#endif
    // ---- z: slope of plane q-1 (own pair), face q-1 between planes q-2 and q-1
    if (idx >= 2) {
      const double* pm = sm + s2 * PLANE + own;
      const double* p0 = sm + s1 * PLANE + own;
      double bot[2][NVAR], top[2][NVAR];
#pragma unroll
      for (int v = 0; v < NVAR; ++v) {
        const double2 a = lds2(pm + v * VM), b = lds2(p0 + v * VM);
        mm_states(b.x - a.x, wq[0][v] - b.x, b.x, bot[0][v], top[0][v]);
        mm_states(b.y - a.y, wq[1][v] - b.y, b.y, bot[1][v], top[1][v]);
      }
      if (q - 1 >= k0 && q - 1 <= k1) {
        double F[2][NVAR];
        hlle_ab2<3>(topz, bot, gamma, ggm1, F);
        if (ML && (q - 1 == 0 || q - 1 == n3)) {  // z face on the block's low / high face: [v][j][i]
          ml_put(q - 1 == 0 ? 4 : 5, x0 + i0, y0 + r, F[0]);
          ml_put(q - 1 == 0 ? 4 : 5, x0 + i0 + 1, y0 + r, F[1]);
        }
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int v = 0; v < NVAR; ++v) {
            dz[e][v] = (F[e][v] - fzp[e][v]) * idx3;
            fzp[e][v] = F[e][v];
          }
      }
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int v = 0; v < NVAR; ++v) topz[e][v] = top[e][v];  // plane q-1's top state
    }


    double sxy[2][NVAR];  // dx + (dy + dz) of the own pair of plane c
    if (cact) {
      const double* Wc = sm + s2 * PLANE;
#ifdef PH_S2_V3
      // ---- extra round: the warp's top y faces and its rows' right x faces, then distributed
      // extra round: lanes 0..15 the y face 4w+4-1/2 of column `lane` (rows 4w+2 .. 4w+5), lanes
      // 16..18 and 31 the x face 16-1/2 of row 4w + 0..3 (cells 14, 15 | 16, 17)
      double Fe[NVAR];
      if (lane < TX) {
        int ao, av, bo, bv;
        row_at(4 * warp + 2, lane, ao, av);
        row_at(4 * warp + 4, lane, bo, bv);
        face4(Wc + ao, av, Wc + bo, bv, bv == VM ? TX : TX, 2, gamma, ggm1, Fe);
      } else if (lane < TX + 3 || lane == 31) {  // row 4w+3's face on lane 31, its consumer
        const int rr = 4 * warp + (lane == 31 ? 3 : lane - TX);
        face4(Wc + R_M + rr * TX + TX - 2, VM, Wc + R_XR + rr * 2, VX, 1, 1, gamma, ggm1, Fe);
      }
      double* fe = sm + OFF_FE + warp * NVAR * 20;
      {
        const int es = lane < TX ? lane : (lane == 31 ? TX + 3 : lane - TX + TX);
        if (lane < TX + 3 || lane == 31) {
#pragma unroll
          for (int v = 0; v < NVAR; ++v) fe[v * 20 + es] = Fe[v];
        }
      }
      __syncwarp();
      if (ML) {
        if (lane < TX && warp == NW - 1 && y0 + TY == G.n[1]) ml_put(3, x0 + lane, c, Fe);  // y face n2: [v][k][i]
        if ((lane >= TX && lane < TX + 3) || lane == 31) {
          if (x0 + TX == G.n[0]) ml_put(1, y0 + 4 * warp + (lane == 31 ? 3 : lane - TX), c, Fe);  // x face n1: [v][k][j]
        }
      }
#else
      const double* xb = sm + OFF_XB + (c & 1) * NVAR * 32;  // plane c's tile-top / right faces
#endif
      // ---- y faces j-1/2 of the own pair (rows r-2 .. r+1); j+1/2 from the row above
      double dy[2][NVAR];
      {
        double wl[2][NVAR], wr[2][NVAR];
#if defined(PH_S2_YS) && !defined(PH_S2_V3)
        // each row's y slope once: my row's bottom state (face r-1/2) and top state (face r+1/2, for
        // the row above); the top state of row r-1 comes from the lane 8 below (same warp), from the
        // warp below through shared memory (kr == 0; the buffer the warp above later reuses for its
        // bottom-face hand-over, FB), or for warp 0 from the y-halo rows -2, -1.  Same operations on
        // the same operands as the 4-row stencil: bit for bit.
        {
          double tp[2][NVAR];
          int yo[3], yv[3];
#pragma unroll
          for (int t = 0; t < 3; ++t) row_at(r - 1 + t, i0, yo[t], yv[t]);
          double2 bm[NVAR];
#pragma unroll
          for (int v = 0; v < NVAR; ++v) {
            const double2 b = lds2(Wc + yo[0] + v * yv[0]), cc = lds2(Wc + yo[1] + v * yv[1]),
                          d = lds2(Wc + yo[2] + v * yv[2]);
            bm[v] = b;
            mm_states(cc.x - b.x, d.x - cc.x, cc.x, wr[0][v], tp[0][v]);
            mm_states(cc.y - b.y, d.y - cc.y, cc.y, wr[1][v], tp[1][v]);
          }
          if (warp < NW - 1) {  // my row 3's top state for the warp above
            if (kr == 3) {
              double* ts = sm + OFF_FB + warp * NVAR * TX + i0;
#pragma unroll
              for (int v = 0; v < NVAR; ++v) sts2(ts + v * TX, tp[0][v], tp[1][v]);
            }
            asm volatile("bar.arrive %0, %1;" ::"r"(NW + 1 + warp), "r"(64) : "memory");
          }
#pragma unroll
          for (int v = 0; v < NVAR; ++v) {
            wl[0][v] = __shfl_up_sync(0xffffffffu, tp[0][v], 8);
            wl[1][v] = __shfl_up_sync(0xffffffffu, tp[1][v], 8);
          }
          if (warp == 0) {
            if (kr == 0) {  // row -1 from the y-halo rows -2, -1 and row 0
#pragma unroll
              for (int v = 0; v < NVAR; ++v) {
                const double2 a = lds2(Wc + R_YL + i0 + v * VY), b = bm[v],
                              cc = lds2(Wc + R_M + i0 + v * VM);
                double t;
                mm_states(b.x - a.x, cc.x - b.x, b.x, t, wl[0][v]);
                mm_states(b.y - a.y, cc.y - b.y, b.y, t, wl[1][v]);
              }
            }
          } else {
            asm volatile("bar.sync %0, %1;" ::"r"(NW + warp), "r"(64) : "memory");
            if (kr == 0) {
              const double* ts = sm + OFF_FB + (warp - 1) * NVAR * TX + i0;
#pragma unroll
              for (int v = 0; v < NVAR; ++v) {
                const double2 h = lds2(ts + v * TX);
                wl[0][v] = h.x;
                wl[1][v] = h.y;
              }
            }
          }
        }
#else
        int yo[4], yv[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) row_at(r - 2 + t, i0, yo[t], yv[t]);
#pragma unroll
        for (int v = 0; v < NVAR; ++v) {
          const double2 a = lds2(Wc + yo[0] + v * yv[0]), b = lds2(Wc + yo[1] + v * yv[1]),
                        cc = lds2(Wc + yo[2] + v * yv[2]), d = lds2(Wc + yo[3] + v * yv[3]);
          double t;
          mm_states(b.x - a.x, cc.x - b.x, b.x, t, wl[0][v]);
          mm_states(cc.x - b.x, d.x - cc.x, cc.x, wr[0][v], t);
          mm_states(b.y - a.y, cc.y - b.y, b.y, t, wl[1][v]);
          mm_states(cc.y - b.y, d.y - cc.y, cc.y, wr[1][v], t);
        }
#endif
        double FF[2][NVAR];
        hlle_ab2<2>(wl, wr, gamma, ggm1, FF);
        const double(&F0)[NVAR] = FF[0];
        const double(&F1)[NVAR] = FF[1];
        if (ML && r == 0 && y0 == 0) {  // y face 0 of the block: [v][k][i]
          ml_put(2, x0 + i0, c, F0);
          ml_put(2, x0 + i0 + 1, c, F1);
        }
#ifndef PH_S2_V3
        if (warp > 0) {  // the bottom row's faces are the top faces of the warp below: hand them over
          if (kr == 0) {
            double* fb = sm + OFF_FB + (warp - 1) * NVAR * TX + i0;
#pragma unroll
            for (int v = 0; v < NVAR; ++v) sts2(fb + v * TX, F0[v], F1[v]);
          }
          asm volatile("bar.arrive %0, %1;" ::"r"(warp), "r"(64) : "memory");
        }
#endif
#pragma unroll
        for (int v = 0; v < NVAR; ++v) {
          double h0 = __shfl_down_sync(0xffffffffu, F0[v], 8), h1 = __shfl_down_sync(0xffffffffu, F1[v], 8);
#ifndef PH_S2_V3
          if (kr == 3) {  // warp 3: the tile top (computed a step ahead); warps 0..2: added after the x round
            const double2 ee = warp == NW - 1 ? lds2(xb + v * 32 + i0) : make_double2(0.0, 0.0);
            h0 = ee.x;
            h1 = ee.y;
          }
          if (kr == 3 && warp < NW - 1) {
            dy[0][v] = -F0[v] * idx2;
            dy[1][v] = -F1[v] * idx2;
          } else {
            dy[0][v] = (h0 - F0[v]) * idx2;
            dy[1][v] = (h1 - F1[v]) * idx2;
          }
#else
          if (kr == 3) {
            const double2 ee = lds2(fe + v * 20 + i0);
            h0 = ee.x;
            h1 = ee.y;
          }
          dy[0][v] = (h0 - F0[v]) * idx2;
          dy[1][v] = (h1 - F1[v]) * idx2;
#endif
          // fold dz in now: L = -(dx + (dy + dz)) (the oracle sums (dx + dy) + dz; round-off only, reading
          // A43) keeps 20 fewer registers live through the x round (+0.3 % on 2b)
          dy[0][v] += dz[0][v];
          dy[1][v] += dz[1][v];
        }
      }
      // ---- x faces 2p-1/2 and 2p+1/2 of the own pair; 2p+3/2 from the right neighbour lane
      double dx[2][NVAR];
      {
        double lo[NVAR], bt0[NVAR], tp0[NVAR], bt1[NVAR], tp1[NVAR];
        // x stencil cells 2p-1 and 2p+2: centre region, or the x-halo columns for the outer lanes
        // cells 2p-2, 2p-1 as one 128-bit load (lane 0: the x-halo cells -2, -1)
        const int xlo = p > 0 ? own - 2 : R_XL + r * 2, xlv = p > 0 ? VM : VX;
        const int xro = p < 7 ? own + 2 : R_XR + r * 2, xrv = p < 7 ? VM : VX;
#pragma unroll
        for (int v = 0; v < NVAR; ++v) {
          const double2 lf = lds2(Wc + xlo + v * xlv);
          const double a = lf.y, d = Wc[xro + v * xrv];
          const double2 b = lds2(Wc + own + v * VM);
          const double d0 = b.y - b.x;
          mm_states(b.x - a, d0, b.x, bt0[v], tp0[v]);
          mm_states(d0, d - b.y, b.y, bt1[v], tp1[v]);
          lo[v] = __shfl_up_sync(0xffffffffu, tp1[v], 1, 8);
          if (p == 0) {  // top state of the halo cell -1 (cells -2, -1 in the x-halo, 0 own)
            double t;
            mm_states(a - lf.x, b.x - a, a, t, lo[v]);
          }
        }
        double xl[2][NVAR], xr[2][NVAR], FX[2][NVAR];
#pragma unroll
        for (int v = 0; v < NVAR; ++v) {
          xl[0][v] = lo[v];
          xr[0][v] = bt0[v];
          xl[1][v] = tp0[v];
          xr[1][v] = bt1[v];
        }
        hlle_ab2<1>(xl, xr, gamma, ggm1, FX);
        double(&FL)[NVAR] = FX[0];
        const double(&FM)[NVAR] = FX[1];
        if (ML && p == 0 && x0 == 0) ml_put(0, y0 + r, c, FL);  // x face 0 of the block: [v][k][j]
#pragma unroll
        for (int v = 0; v < NVAR; ++v) {
          double FR = __shfl_down_sync(0xffffffffu, FL[v], 1, 8);
#ifndef PH_S2_V3
          if (p == 7) FR = xb[v * 32 + TX + r];
#else
          if (p == 7) FR = fe[v * 20 + TX + kr];
#endif
          dx[0][v] = (FM[v] - FL[v]) * idx1;
          dx[1][v] = (FR - FM[v]) * idx1;
        }
      }
#ifndef PH_S2_V3
      if (warp < NW - 1) {  // the top faces of my row 3 = the bottom faces of the warp above
        asm volatile("bar.sync %0, %1;" ::"r"(warp + 1), "r"(64) : "memory");
        if (kr == 3) {
          const double* fb = sm + OFF_FB + warp * NVAR * TX + i0;
#pragma unroll
          for (int v = 0; v < NVAR; ++v) {
            const double2 h = lds2(fb + v * TX);
            dy[0][v] = fma(h.x, idx2, dy[0][v]);
            dy[1][v] = fma(h.y, idx2, dy[1][v]);
          }
        }
      }
#endif
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int v = 0; v < NVAR; ++v) sxy[e][v] = dx[e][v] + dy[e][v];  // dx + (dy + dz)
      // ---- a5: divergence + RK combine of the own pair of plane c
      ph_jitter(4 * q + 3);
      mbar_wait(bar + NSLOT, (uint32_t)(c - k0) & 1u);
      const int64_t cell = (int64_t)slot * G.bstride + (int64_t)(c + g) * plane + (int64_t)(y0 + r + g) * G.N[0] +
                           (x0 + i0 + g);
      double un[2][NVAR];
#pragma unroll
      for (int v = 0; v < NVAR; ++v) {
        const double2 f = lds2(fin + v * VM + r * TX + i0);
        const double L0 = -sxy[0][v];
        const double L1 = -sxy[1][v];
        if (S2) {
          un[0][v] = fma(cdt, L0, f.x);
          un[1][v] = fma(cdt, L1, f.y);
        } else {
          un[0][v] = fma(A.b1, f.x, cdt * L0);
          un[1][v] = fma(A.b1, f.y, cdt * L1);
          stg2(A.H + cell + v * G.vstride, fma(A.hb1, un[0][v], A.ha0 * f.x), fma(A.hb1, un[1][v], A.ha0 * f.y));
        }
        stg2(A.Uout + cell + v * G.vstride, un[0][v], un[1][v]);
      }
      if (PUT) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cc[3] = {x0 + i0 + e, y0 + r, c};
#pragma unroll
          for (int f = 0; f < 6; ++f) {
            const int pr = M.prank[f];
            if (pr < 0) continue;
            const int d = f >> 1;
            const int l = (f & 1) ? cc[d] - (G.n[d] - g) : cc[d];  // layer within the face box
            if (l < 0 || l >= g) continue;
            const int b0 = d == 0 ? g : G.n[0], b1 = d == 1 ? g : G.n[1], b2 = d == 2 ? g : G.n[2];
            const int i2 = d == 0 ? l : cc[0], j2 = d == 1 ? l : cc[1], k2 = d == 2 ? l : cc[2];
            const int64_t nbox = (int64_t)b0 * b1 * b2;
            double* dst = A.peer_rbuf[pr] + M.poff[f] + ((int64_t)k2 * b1 + j2) * b0 + i2;
#pragma unroll
            for (int v = 0; v < NVAR; ++v) dst[v * nbox] = un[e][v];
          }
        }
      }
      if (REDUCE) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (ML && M.rfx) {  // first cell layer of a flux-corrected face: reduced after the reflux
            const int cc[3] = {x0 + i0 + e, y0 + r, c};
            bool corrected = false;
#pragma unroll
            for (int f = 0; f < 6; ++f)
              if (((M.rfx >> f) & 1) && cc[f >> 1] == ((f & 1) ? G.n[f >> 1] - 1 : 0)) corrected = true;
            if (corrected) continue;
          }
          const double ir = rcp_nr(un[e][0]);
          const double v1 = un[e][1] * ir, v2 = un[e][2] * ir, v3 = un[e][3] * ir;
          const double ke = 0.5 * ((un[e][1] * v1 + un[e][2] * v2) + un[e][3] * v3);
          const double pr = gm1 * (un[e][4] - ke);
          const double cs = sound_speed(un[e][0], pr, gamma);
          const double sx = (fabs(v1) + cs) * idx1, sy = (fabs(v2) + cs) * idx2, sz = (fabs(v3) + cs) * idx3;
          tmax = dmax(tmax, dmax(sx, dmax(sy, sz)));
#pragma unroll
          for (int v = 0; v < NVAR; ++v) tsum[v] += un[e][v];
        }
      }
    }
#if !defined(PH_S2_V3) && !defined(PH_S2_XSTART)
    // one step ahead, one warp (rotating): plane q-1's tile-top y faces (lanes 0..15, rows 14..17) and
    // right x faces (lanes 16..31, cells 14..17 of row lane-16), for every warp's use next step
    if (q - 1 >= k0 && q - 1 < k1 && warp == (q & (NW - 1))) {
      const double* W1 = sm + s1 * PLANE;
      double Fe[NVAR];
      if (lane < TX)
        face4(W1 + R_M + (TY - 2) * TX + lane, VM, W1 + R_YH + lane, VY, TX, 2, gamma, ggm1, Fe);
      else
        face4(W1 + R_M + (lane - TX) * TX + TX - 2, VM, W1 + R_XR + (lane - TX) * 2, VX, 1, 1, gamma, ggm1, Fe);
      double* xo = sm + OFF_XB + ((q - 1) & 1) * NVAR * 32 + lane;
#pragma unroll
      for (int v = 0; v < NVAR; ++v) xo[v * 32] = Fe[v];
      if (ML) {
        if (lane < TX && y0 + TY == G.n[1]) ml_put(3, x0 + lane, q - 1, Fe);             // y face n2: [v][k][i]
        if (lane >= TX && x0 + TX == G.n[0]) ml_put(1, y0 + lane - TX, q - 1, Fe);       // x face n1: [v][k][j]
      }
    }
#endif
    s = (s + 1) & (NSLOT - 1);
  }
  if (REDUCE) {
    // deterministic CTA reduction: warp shuffles, then thread 0 over the warps in order
    __syncthreads();
    double* red = sm + OFF_RED;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      tmax = fmax(tmax, __shfl_xor_sync(0xffffffffu, tmax, off));
#pragma unroll
      for (int v = 0; v < NVAR; ++v) tsum[v] += __shfl_xor_sync(0xffffffffu, tsum[v], off);
    }
    if (lane == 0) {
      red[warp * 6] = tmax;
#pragma unroll
      for (int v = 0; v < NVAR; ++v) red[warp * 6 + 1 + v] = tsum[v];
    }
    __syncthreads();
    if (tid == 0) {
      double mx = 0.0, su[NVAR] = {0, 0, 0, 0, 0};
      for (int w = 0; w < NW; ++w) {
        mx = fmax(mx, red[w * 6]);
        for (int v = 0; v < NVAR; ++v) su[v] += red[w * 6 + 1 + v];
      }
      double* o = A.partials + (int64_t)(A.cta_base + blockIdx.x) * 6;
      o[0] = mx;
      for (int v = 0; v < NVAR; ++v) o[1 + v] = su[v] * M.dV;
    }
  }
}

// 5-D tensor map over a pool [slot][v][k][j][i] with box {bx, by, 1, 5, 1}
static cudaError_t make_map(CUtensorMap* m, const double* base, const Geom& G, int nslots, int bx, int by) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[5] = {(cuuint64_t)G.N[0], (cuuint64_t)G.N[1], (cuuint64_t)G.N[2], (cuuint64_t)NVAR,
                              (cuuint64_t)nslots};
  const cuuint64_t str[4] = {(cuuint64_t)G.N[0] * 8, (cuuint64_t)G.N[0] * G.N[1] * 8, (cuuint64_t)G.vstride * 8,
                             (cuuint64_t)G.bstride * 8};
  const cuuint32_t box[5] = {(cuuint32_t)bx, (cuuint32_t)by, 1, (cuuint32_t)NVAR, 1};
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double*>(base), dims, str, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <bool RD, bool S2, bool PUT, bool ML = false>
static cudaError_t launch_t(int nctas, const StageArgs& a, const Maps& mp, const Geom& G, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(stage2_kernel<RD, S2, PUT, ML>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)SMEM_BYTES);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(stage2_kernel<RD, S2, PUT, ML>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    if (getenv("PH_DEBUG_ATTR")) {
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, stage2_kernel<RD, S2, PUT, ML>);
      fprintf(stderr, "stage2_kernel<%d,%d,%d>: regs %d local %zu dyn smem %zu\n", (int)RD, (int)S2, (int)PUT, fa.numRegs,
              fa.localSizeBytes, SMEM_BYTES);
    }
    attr = true;
  }
  stage2_kernel<RD, S2, PUT, ML><<<nctas, NTH, SMEM_BYTES, s>>>(a, G, mp);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------ AMR tag pass
// tag2_kernel: the AMR indicator eps_B (O9, A14, arithmetic A46) of every block, fused with the dt /
// totals partials of the unchanged mesh (a6, a10) -- the same per-cell formulas as tag_kernel
// (kernels.cu), re-mapped like stage2: 16 x 16 tiles of x-pairs, planes by TMA (the same boxes and
// direct halo) into a 2-slot cons ring, pressures into a 3-plane ring with a 1-cell halo, one
// __syncthreads per plane.  Pressures and eps are bit-identical to tag_kernel's.
constexpr int PW = TX + 2, PH = TY + 2, PPL = PW * PH;  // pressure plane with its 1-cell halo
constexpr int T_OFF_P = 2 * PLANE;                      // [3][PH][PW]
constexpr int T_OFF_RED = T_OFF_P + 3 * PPL;            // [NW][7]
constexpr int T_OFF_BAR = T_OFF_RED + NW * 7;           // full[2]
constexpr size_t TAG_SMEM = (T_OFF_BAR + 2) * sizeof(double);

__global__ void __launch_bounds__(NTH, 4) tag2_kernel(const double* U, const BlockMeta* meta,
                                                      unsigned long long* eps_bits, double* partials, ErrWord* err,
                                                      Geom G, const __grid_constant__ Maps maps) {
  extern __shared__ __align__(128) double sm[];
  double* Pr = sm + T_OFF_P;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + T_OFF_BAR);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kr = lane >> 3, r = (warp << 2) + kr, p = lane & 7, i0 = 2 * p;
  const int ntx = G.n[0] / TX, nty = G.n[1] / TY;
  int b = blockIdx.x;
  const int txi = b % ntx;
  b /= ntx;
  const int tyi = b % nty;
  const int slot = b / nty;
  const BlockMeta& M = meta[slot];
  const int x0 = txi * TX, y0 = tyi * TY, g = G.g, n3 = G.n[2];
  const double gm1 = G.gm1, gamma = G.gamma;
  const double idx1 = M.idx[0], idx2 = M.idx[1], idx3 = M.idx[2];
  const int own = R_M + r * TX + i0;

  auto issue_plane = [&](int q, int sl) {  // tid 0 only: main boxes for q in [0, n3), own rows for z halos
    uint64_t* fb = bar + sl;
    double* base = sm + sl * PLANE;
    fence_proxy_async();
    if (q >= 0 && q < n3) {
      const int n1 = G.n[0], n2 = G.n[1];
      const int nb0 = M.nb[0], nb1 = M.nb[1], nb2 = M.nb[2], nb3 = M.nb[3];
      const bool dl = x0 == 0 && nb0 >= 0, dr = x0 + TX == n1 && nb1 >= 0;
      const bool db = y0 == 0 && nb2 >= 0, dt = y0 + TY == n2 && nb3 >= 0;
      mbar_expect_tx(fb, MAIN_BYTES);
      const int z = q + g;
      tma5(base + R_M, &maps.c, x0 + g, y0 + g, z, 0, slot, fb);
      tma5(base + R_XL, &maps.xh, dl ? n1 - 2 + g : x0 - 2 + g, y0 + g, z, 0, dl ? nb0 : slot, fb);
      tma5(base + R_XR, &maps.xh, dr ? g : x0 + TX + g, y0 + g, z, 0, dr ? nb1 : slot, fb);
      tma5(base + R_YL, &maps.yh, x0 + g, db ? n2 - 2 + g : y0 - 2 + g, z, 0, db ? nb2 : slot, fb);
      tma5(base + R_YH, &maps.yh, x0 + g, dt ? g : y0 + TY + g, z, 0, dt ? nb3 : slot, fb);
    } else {
      int bb = slot, qq = q;
      const int zl = M.nb[4], zh = M.nb[5];
      if (q < 0 && zl >= 0) { bb = zl; qq += n3; }
      else if (q >= n3 && zh >= 0) { bb = zh; qq -= n3; }
      mbar_expect_tx(fb, OWN_BYTES);
      tma5(base + R_M, &maps.c, x0 + g, y0 + g, qq + g, 0, bb, fb);
    }
  };
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.c)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.xh)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.yh)) : "memory");
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // pressure with the stage kernels' (and tag_kernel's) arithmetic; the dt / totals terms of own cells
  double mx = 0.0, tmax = 0.0, ts[NVAR] = {0.0, 0.0, 0.0, 0.0, 0.0};
  auto pressure = [&](const double* u, int vs, int q, int j, int i, bool own_cell) -> double {
    const double rho = u[0], m1 = u[vs], m2 = u[2 * vs], m3 = u[3 * vs], E = u[4 * vs];
    const double fr = rcp_nr(rho);
    const double w1 = m1 * fr, w2 = m2 * fr, w3 = m3 * fr;
    const double fke = 0.5 * ((m1 * w1 + m2 * w2) + m3 * w3);
    const double pr = gm1 * (E - fke);
    if (own_cell) {
      if (!(rho > 0.0) || !(pr > 0.0)) set_error(err, 0, M.gid, q, y0 + j, x0 + i);
      const double cs = sound_speed(rho, pr, gamma);
      const double s1 = (fabs(w1) + cs) * idx1, s2 = (fabs(w2) + cs) * idx2, s3 = (fabs(w3) + cs) * idx3;
      tmax = dmax(tmax, dmax(s1, dmax(s2, s3)));
      ts[0] += rho;
      ts[1] += m1;
      ts[2] += m2;
      ts[3] += m3;
      ts[4] += E;
    }
    return pr;
  };
  if (tid == 0) issue_plane(-1, 0);
#pragma unroll 1
  for (int q = -1; q <= n3; ++q) {
    const int idx = q + 1, sl = idx & 1;
    const double* Wq = sm + sl * PLANE;
    double* Pq = Pr + (idx % 3) * PPL;
    mbar_wait(bar + sl, (uint32_t)(idx >> 1) & 1u);
    const bool mainp = q >= 0 && q < n3;
    {  // own pair
      const double pa = pressure(Wq + own, VM, q, r, i0, mainp), pb = pressure(Wq + own + 1, VM, q, r, i0 + 1, mainp);
      Pq[(r + 1) * PW + i0 + 1] = pa;
      Pq[(r + 1) * PW + i0 + 2] = pb;
    }
    if (mainp && tid < 64) {  // the 1-cell halo ring of the tile: x columns -1 / 16, y rows -1 / 16
      int off, vs, pj, pi;
      if (tid < 32) {
        const int rr = tid & 15;
        off = tid < 16 ? R_XL + rr * 2 + 1 : R_XR + rr * 2;
        vs = VX;
        pj = rr + 1;
        pi = tid < 16 ? 0 : TX + 1;
      } else {
        const int t = tid - 32, col = t & 15;
        off = t < 16 ? R_YL + TX + col : R_YH + col;
        vs = VY;
        pj = t < 16 ? 0 : TY + 1;
        pi = col + 1;
      }
      Pq[pj * PW + pi] = pressure(Wq + off, vs, q, pj - 1, pi - 1, false);
    }
    ph_jitter(q + 7);
    __syncthreads();  // plane q's pressures visible; slot sl free for plane q + 2
    if (tid == 0 && q + 1 <= n3) issue_plane(q + 1, sl ^ 1);
    const int c = q - 1;  // plane whose indicator is complete now
    if (c >= 0) {
      const double* Pm = Pr + ((idx + 1) % 3) * PPL;  // plane q-2
      const double* P0 = Pr + ((idx + 2) % 3) * PPL;  // plane q-1
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int o = (r + 1) * PW + i0 + 1 + e;
        const double g1 = 0.5 * (P0[o + 1] - P0[o - 1]);
        const double g2 = 0.5 * (P0[o + PW] - P0[o - PW]);
        const double g3 = 0.5 * (Pq[o] - Pm[o]);
        const double ss = (g1 * g1 + g2 * g2) + g3 * g3;
        const double ev = ss > 0.0 ? (ss * rsqrt_nr(ss)) * rcp_nr(P0[o]) : 0.0;
        mx = fmax(mx, ev);
      }
    }
    __syncthreads();  // the pressure ring slot of plane q-2 is rewritten next step (plane q+1)
  }
  for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if (lane == 0) atomicMax(eps_bits + slot, (unsigned long long)__double_as_longlong(mx));
  if (partials) {  // deterministic: warp shuffles, then thread 0 in warp order
    for (int off = 16; off > 0; off >>= 1) {
      tmax = fmax(tmax, __shfl_xor_sync(0xffffffffu, tmax, off));
#pragma unroll
      for (int v = 0; v < NVAR; ++v) ts[v] += __shfl_xor_sync(0xffffffffu, ts[v], off);
    }
    double* red = sm + T_OFF_RED;
    if (lane == 0) {
      red[warp * 7] = tmax;
      for (int v = 0; v < NVAR; ++v) red[warp * 7 + 1 + v] = ts[v];
    }
    __syncthreads();
    if (tid == 0) {
      double m = 0.0, su[NVAR] = {0, 0, 0, 0, 0};
      for (int w = 0; w < NW; ++w) {
        m = fmax(m, red[w * 7]);
        for (int v = 0; v < NVAR; ++v) su[v] += red[w * 7 + 1 + v];
      }
      double* o = partials + (int64_t)blockIdx.x * 6;
      o[0] = m;
      for (int v = 0; v < NVAR; ++v) o[1 + v] = su[v] * M.dV;
    }
  }
}

}  // namespace s2

bool stage2_applies(const Geom& G, int recon, bool ml) {
  (void)ml;  // multilevel meshes too (flux slots, template ML)
  if (getenv("PH_STAGE_V1") || getenv("PH_NO_HBASE")) return false;  // it needs the stage-2 base pool H
  if (G.no_stage2) return false;
  return recon == 0 && G.wavespeed == 0 && G.g == 2 && G.n[0] % s2::TX == 0 && G.n[1] % s2::TY == 0 &&
         G.n[0] >= s2::TX && G.n[1] >= s2::TY;
}

bool tag2_applies(const Geom& G) {
  if (getenv("PH_STAGE_V1") || getenv("PH_TAG_V1")) return false;
  return G.g == 2 && G.n[0] % s2::TX == 0 && G.n[1] % s2::TY == 0 && G.n[0] >= s2::TX && G.n[1] >= s2::TY;
}

int tag2_ctas_per_block(const Geom& G) { return (G.n[0] / s2::TX) * (G.n[1] / s2::TY); }

cudaError_t launch_tag2(const double* U, const BlockMeta* meta, int nslots, unsigned long long* eps_bits,
                        double* partials, ErrWord* err, const Geom& G, cudaStream_t s) {
  s2::Maps mp;
  cudaError_t e;
  if ((e = s2::make_map(&mp.c, U, G, nslots, s2::TX, s2::TY)) != cudaSuccess) return e;
  if ((e = s2::make_map(&mp.xh, U, G, nslots, 2, s2::TY)) != cudaSuccess) return e;
  if ((e = s2::make_map(&mp.yh, U, G, nslots, s2::TX, 2)) != cudaSuccess) return e;
  mp.f = mp.c;
  static bool attr = false;
  if (!attr) {
    e = cudaFuncSetAttribute(s2::tag2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2::TAG_SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  s2::tag2_kernel<<<nslots * tag2_ctas_per_block(G), s2::NTH, s2::TAG_SMEM, s>>>(U, meta, eps_bits, partials, err, G, mp);
  return cudaGetLastError();
}

cudaError_t launch_stage2(bool reduce, bool use_u0, int nctas, const StageArgs& a, const Geom& G, cudaStream_t s) {
  if (!a.H || a.pool_slots <= 0 || (a.fbuf && a.peer_rbuf)) return cudaErrorNotSupported;
  s2::Maps mp;
  cudaError_t e;
  if ((e = s2::make_map(&mp.c, a.Uin, G, a.pool_slots, s2::TX, s2::TY)) != cudaSuccess) return e;
  if ((e = s2::make_map(&mp.xh, a.Uin, G, a.pool_slots, 2, s2::TY)) != cudaSuccess) return e;
  if ((e = s2::make_map(&mp.yh, a.Uin, G, a.pool_slots, s2::TX, 2)) != cudaSuccess) return e;
  if ((e = s2::make_map(&mp.f, use_u0 ? a.H : a.Uin, G, a.pool_slots, s2::TX, s2::TY)) != cudaSuccess) return e;
  using namespace s2;
  if (a.fbuf) {  // multilevel (flux slots)
    if (use_u0)
      return reduce ? launch_t<true, true, false, true>(nctas, a, mp, G, s) : launch_t<false, true, false, true>(nctas, a, mp, G, s);
    return reduce ? launch_t<true, false, false, true>(nctas, a, mp, G, s) : launch_t<false, false, false, true>(nctas, a, mp, G, s);
  }
  if (a.peer_rbuf) {
    if (use_u0)
      return reduce ? launch_t<true, true, true>(nctas, a, mp, G, s) : launch_t<false, true, true>(nctas, a, mp, G, s);
    return reduce ? launch_t<true, false, true>(nctas, a, mp, G, s) : launch_t<false, false, true>(nctas, a, mp, G, s);
  }
  if (use_u0)
    return reduce ? launch_t<true, true, false>(nctas, a, mp, G, s) : launch_t<false, true, false>(nctas, a, mp, G, s);
  return reduce ? launch_t<true, false, false>(nctas, a, mp, G, s) : launch_t<false, false, false>(nctas, a, mp, G, s);
}

}  // namespace ph
