// kernels.cu -- sm_100a kernels of the Parthenon-hydro hot path.
//
// Paper: Parthenon-hydro update = RK2 + PLM + HLLE over packs of
// MeshBlocks in one launch; fill-in-one boundary kernels incl. restriction and
// prolongation; flux correction; CFL dt as a global reduction
// (P:640-650).  Formulas and their operation order follow SURVEY.md §8(c) O5-O8.
//
// No tensor cores: every kernel here is an fp64 stencil or copy (bandwidth / fp64-issue bound).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "device.cuh"
#include "point.cuh"

namespace ph {

// ------------------------------------------------------------------------------ point math
// full-tile path: the tile-boundary faces (x face 0 of every row, y face row 0) of planes c+1 and
// c+2 are computed during plane c's 4th face round by warps that would otherwise wait at the
// barrier, into a small side buffer; those planes then need 3 face rounds (4/3/3 instead of 4/4/4).
constexpr int EXTRA_AHEAD = 2;
// plane loads bypass L1 (ld.global.cg): there is no reuse in L1 (+0.6 % over ld.global.nc)
__device__ __forceinline__ double ld_plane(const double* p) { return __ldcg(p); }
// finished cells are stored L2-only (st.global.cg; +0.1 % over plain / .cs stores, which are equal)
__device__ __forceinline__ void st_cell(double* p, double v) { __stcg(p, v); }
template <int RECON>
__device__ __forceinline__ double slope(double dl, double dr) {
  if (RECON == 0) return minmod_i(dl, dr);
  bool same = (dl > 0.0 && dr > 0.0) || (dl < 0.0 && dr < 0.0);
  if (!same) return 0.0;
  if (RECON == 1) return 2.0 * dl * dr / (dl + dr);  // van Leer (A3)
  double s = dl > 0.0 ? 1.0 : -1.0;                  // MC
  double m = fmin(fmin(2.0 * fabs(dl), 2.0 * fabs(dr)), 0.5 * fabs(dl + dr));
  return s * m;
}

// PLM face states of the face between cells c-1 and c from q0=W(c-2) .. q3=W(c+1) (a3, O5)
template <int RECON>
__device__ __forceinline__ void plm_face(double q0, double q1, double q2, double q3, double& wl, double& wr) {
  double d0 = q1 - q0, d1 = q2 - q1, d2 = q3 - q2;
  if (RECON == 0) {
    // minmod with the sign test folded into the coefficient: h = same sign ? 0.5 : 0 (one select
    // on the high word), state = q + h * (smaller-magnitude difference); equals q + 0.5*minmod
    wl = fma(minmod_half(d0, d1), minmod_pick(d0, d1), q1);
    wr = fma(-minmod_half(d1, d2), minmod_pick(d1, d2), q2);
    return;
  }
  double s1 = slope<RECON>(d0, d1);
  double s2 = slope<RECON>(d1, d2);
  wl = fma(0.5, s1, q1);   // == q1 + 0.5*s1 exactly (0.5*s1 is exact)
  wr = fma(-0.5, s2, q2);
}

// HLLE in the clamped branch-free form (a4; A4, A5).  w = (rho, u_n, v_t1, v_t2, p).  Wave speeds:
// Davis (EIN = false), or Einfeldt (EIN = true): the Roe averages (sqrt(rho) weights) of velocity
// and total enthalpy H = (E + p) / rho give c~^2 = (gamma - 1)(H~ - |v~|^2 / 2), and
// S_L = min(u_L - c_L, u~ - c~), S_R = max(u_R + c_R, u~ + c~).
template <bool EIN = false>
__device__ __forceinline__ void hlle(const double* wl, const double* wr, const Geom& G, double* F) {
  double cl = sound_speed(wl[0], wl[4], G.gamma);
  double cr = sound_speed(wr[0], wr[4], G.gamma);
  double mul = wl[0] * wl[1];
  double mur = wr[0] * wr[1];
#ifdef PH_STRICT  // strict diagnostic build: p / (gamma - 1) as the oracle writes it
  double El = wl[4] / G.gm1 + (0.5 * wl[0]) * (wl[1] * wl[1] + (wl[2] * wl[2] + wl[3] * wl[3]));
  double Er = wr[4] / G.gm1 + (0.5 * wr[0]) * (wr[1] * wr[1] + (wr[2] * wr[2] + wr[3] * wr[3]));
#else
  double El = wl[4] * G.inv_gm1 + (0.5 * wl[0]) * (wl[1] * wl[1] + (wl[2] * wl[2] + wl[3] * wl[3]));
  double Er = wr[4] * G.inv_gm1 + (0.5 * wr[0]) * (wr[1] * wr[1] + (wr[2] * wr[2] + wr[3] * wr[3]));
#endif
  double sl, sr;
  if (EIN) {
    const double rl = wl[0] * rsqrt_nr(wl[0]), rr = wr[0] * rsqrt_nr(wr[0]);  // sqrt(rho)
    const double is = rcp_nr(rl + rr);
    const double u = (rl * wl[1] + rr * wr[1]) * is, v = (rl * wl[2] + rr * wr[2]) * is,
                 w = (rl * wl[3] + rr * wr[3]) * is;
    const double h = (rl * ((El + wl[4]) * rcp_nr(wl[0])) + rr * ((Er + wr[4]) * rcp_nr(wr[0]))) * is;
    const double c2 = G.gm1 * (h - 0.5 * (u * u + (v * v + w * w)));
    const double c = c2 * rsqrt_nr(c2);
    sl = dmin(wl[1] - cl, u - c);
    sr = dmax(wr[1] + cr, u + c);
  } else {
    sl = dmin(wl[1] - cl, wr[1] - cr);
    sr = dmax(wl[1] + cl, wr[1] + cr);
  }
  double bp = dmax(sr, 0.0);
  double bm = dmin(sl, 0.0);
  double inv = rcp_nr(bp - bm);
  double bb = bp * bm;
  // F = ((bp FL - bm FR) + bb (UR - UL)) * inv
  F[0] = ((bp * mul - bm * mur) + bb * (wr[0] - wl[0])) * inv;
  F[1] = ((bp * (mul * wl[1] + wl[4]) - bm * (mur * wr[1] + wr[4])) + bb * (mur - mul)) * inv;
  F[2] = ((bp * (mul * wl[2]) - bm * (mur * wr[2])) + bb * (wr[0] * wr[2] - wl[0] * wl[2])) * inv;
  F[3] = ((bp * (mul * wl[3]) - bm * (mur * wr[3])) + bb * (wr[0] * wr[3] - wl[0] * wl[3])) * inv;
  F[4] = ((bp * ((El + wl[4]) * wl[1]) - bm * ((Er + wr[4]) * wr[1])) + bb * (Er - El)) * inv;
}


// ---- exact-arithmetic variants (explicitly rounded, the oracle's operation order).  WENO-Z's
// nonlinear weights and PPM's extremum switch amplify round-off (a smoothness indicator that is 0
// on one side and 1e-33 on the other changes a weight by 40 orders of magnitude), so the
// high-order path computes bit for bit what the oracle computes: parity is then exact.

__device__ __forceinline__ double slope_rn(double qm, double q0, double qp, int recon) {
  const double dl = __dsub_rn(q0, qm), dr = __dsub_rn(qp, q0);
  const bool same = (dl > 0.0 && dr > 0.0) || (dl < 0.0 && dr < 0.0);
  if (!same) return 0.0;
  if (recon == 1) return __ddiv_rn(__dmul_rn(__dmul_rn(2.0, dl), dr), __dadd_rn(dl, dr));
  if (recon == 2) {
    const double s = dl > 0.0 ? 1.0 : -1.0;
    double m = __dmul_rn(2.0, fabs(dl)), b = __dmul_rn(2.0, fabs(dr)), c = __dmul_rn(0.5, fabs(__dadd_rn(dl, dr)));
    m = m < b ? m : b;
    m = m < c ? m : c;
    return __dmul_rn(s, m);
  }
  if (dl > 0.0) return dl < dr ? dl : dr;
  return dl > dr ? dl : dr;
}

// PPM's limited slope and interface values with selects in place of branches: every candidate is
// computed (all are exact single operations on finite inputs) and the oracle's conditions pick one, so
// the results are the oracle's bit for bit while the warp issues no data-dependent branches (the line
// kernels' top stall was branch resolution)
__device__ __forceinline__ double ppm_dm_rn(double a, double b, double c) {
  const double dl = __dsub_rn(b, a), dr = __dsub_rn(c, b);
  const bool same = (dl > 0.0 && dr > 0.0) || (dl < 0.0 && dr < 0.0);
  const double dq = __dmul_rn(0.5, __dsub_rn(c, a));
  double m = fabs(dq);
  const double tl = __dmul_rn(2.0, fabs(dl)), tr = __dmul_rn(2.0, fabs(dr));
  m = tl < m ? tl : m;
  m = tr < m ? tr : m;
  const double r = dq > 0.0 ? m : -m;
  return same ? r : 0.0;
}

// PPM interface values of one cell from its neighbours qm, c, qp and the three limited slopes
// dm_m, dm_0, dm_p (cells c-1, c, c+1); split out so a line march can reuse each slope three times.
// Oracle: if (R-c)(c-L) <= 0 then L = R = c; else if d m6 > d^2 then L = 3c - 2R; else if -d^2 > d m6
// then R = 3c - 2L.
__device__ __forceinline__ void ppm_lr_rn(double qm, double c, double qp, double dm_m, double dm_0, double dm_p,
                                          double& ql, double& qr) {
  const double L = __dsub_rn(__dadd_rn(qm, __dmul_rn(0.5, __dsub_rn(c, qm))), ddiv_k(__dsub_rn(dm_0, dm_m), K6, RK6));
  const double R = __dsub_rn(__dadd_rn(c, __dmul_rn(0.5, __dsub_rn(qp, c))), ddiv_k(__dsub_rn(dm_p, dm_0), K6, RK6));
  const bool flat = __dmul_rn(__dsub_rn(R, c), __dsub_rn(c, L)) <= 0.0;
  const double d = __dsub_rn(R, L), m6 = __dmul_rn(6.0, __dsub_rn(c, __dmul_rn(0.5, __dadd_rn(L, R))));
  const double dd = __dmul_rn(d, d), dm6 = __dmul_rn(d, m6);
  const bool fixl = dm6 > dd, fixr = !fixl && (-dd > dm6);
  const double Lx = __dsub_rn(__dmul_rn(3.0, c), __dmul_rn(2.0, R)), Rx = __dsub_rn(__dmul_rn(3.0, c), __dmul_rn(2.0, L));
  ql = flat ? c : (fixl ? Lx : L);
  qr = flat ? c : (fixr ? Rx : R);
}

__device__ __forceinline__ void ppm_cell_rn(const double* q, double& ql, double& qr) {
  const double dm_m = ppm_dm_rn(q[0], q[1], q[2]), dm_0 = ppm_dm_rn(q[1], q[2], q[3]), dm_p = ppm_dm_rn(q[2], q[3], q[4]);
  ppm_lr_rn(q[1], q[2], q[3], dm_m, dm_0, dm_p, ql, qr);
}

// WENO-Z's general divisions: inlined (default) or one out-of-line copy (PH_WENO_DIV_CALL, A/B knob: the
// per-face kernel inlines 43 IEEE division sequences and stalls on instruction fetch)
#ifdef PH_WENO_DIV_CALL
__device__ __noinline__ double wdiv(double a, double b) { return __ddiv_rn(a, b); }
#else
__device__ __forceinline__ double wdiv(double a, double b) { return __ddiv_rn(a, b); }
#endif

__device__ __forceinline__ double wenoz_rn(double a, double b, double c, double d, double e) {
  const double t0 = __dadd_rn(__dsub_rn(a, __dmul_rn(2.0, b)), c), u0 = __dadd_rn(__dsub_rn(a, __dmul_rn(4.0, b)), __dmul_rn(3.0, c));
  const double t1 = __dadd_rn(__dsub_rn(b, __dmul_rn(2.0, c)), d), u1 = __dsub_rn(b, d);
  const double t2 = __dadd_rn(__dsub_rn(c, __dmul_rn(2.0, d)), e), u2 = __dadd_rn(__dsub_rn(__dmul_rn(3.0, c), __dmul_rn(4.0, d)), e);
  const double k13 = 13.0 / 12.0;
  const double b0 = __dadd_rn(__dmul_rn(k13, __dmul_rn(t0, t0)), __dmul_rn(0.25, __dmul_rn(u0, u0)));
  const double b1 = __dadd_rn(__dmul_rn(k13, __dmul_rn(t1, t1)), __dmul_rn(0.25, __dmul_rn(u1, u1)));
  const double b2 = __dadd_rn(__dmul_rn(k13, __dmul_rn(t2, t2)), __dmul_rn(0.25, __dmul_rn(u2, u2)));
  const double tau = fabs(__dsub_rn(b0, b2));
  const double r0 = wdiv(tau, __dadd_rn(b0, 1e-40)), r1 = wdiv(tau, __dadd_rn(b1, 1e-40)),
               r2 = wdiv(tau, __dadd_rn(b2, 1e-40));
  const double a0 = __dmul_rn(0.1, __dadd_rn(1.0, __dmul_rn(r0, r0)));
  const double a1 = __dmul_rn(0.6, __dadd_rn(1.0, __dmul_rn(r1, r1)));
  const double a2 = __dmul_rn(0.3, __dadd_rn(1.0, __dmul_rn(r2, r2)));
  const double q0 = ddiv_k(__dadd_rn(__dsub_rn(__dmul_rn(2.0, a), __dmul_rn(7.0, b)), __dmul_rn(11.0, c)), K6, RK6);
  const double q1 = ddiv_k(__dadd_rn(__dadd_rn(-b, __dmul_rn(5.0, c)), __dmul_rn(2.0, d)), K6, RK6);
  const double q2 = ddiv_k(__dsub_rn(__dadd_rn(__dmul_rn(2.0, c), __dmul_rn(5.0, d)), e), K6, RK6);
  return wdiv(__dadd_rn(__dadd_rn(__dmul_rn(a0, q0), __dmul_rn(a1, q1)), __dmul_rn(a2, q2)),
                   __dadd_rn(__dadd_rn(a0, a1), a2));
}

template <int RECON>
__device__ __forceinline__ void recon_face6_rn(const double* q, double& wl, double& wr) {
  if (RECON == 3) {
    double a, b;
    ppm_cell_rn(q, a, wl);
    ppm_cell_rn(q + 1, wr, b);
  } else if (RECON == 4) {
    wl = wenoz_rn(q[0], q[1], q[2], q[3], q[4]);
    wr = wenoz_rn(q[5], q[4], q[3], q[2], q[1]);
  } else {
    wl = __dadd_rn(q[2], __dmul_rn(0.5, slope_rn(q[1], q[2], q[3], RECON)));
    wr = __dsub_rn(q[3], __dmul_rn(0.5, slope_rn(q[2], q[3], q[4], RECON)));
  }
}

__device__ __forceinline__ void phys_rn(const double* W, double gm1, double igm1, double* U, double* F) {
  const double rho = W[0], u = W[1], v = W[2], w = W[3], p = W[4];
  const double mu = __dmul_rn(rho, u);
  const double E = __dadd_rn(ddiv_k(p, gm1, igm1), __dmul_rn(__dmul_rn(0.5, rho),
                                                         __dadd_rn(__dmul_rn(u, u), __dadd_rn(__dmul_rn(v, v), __dmul_rn(w, w)))));
  U[0] = rho; U[1] = mu; U[2] = __dmul_rn(rho, v); U[3] = __dmul_rn(rho, w); U[4] = E;
  F[0] = mu; F[1] = __dadd_rn(__dmul_rn(mu, u), p); F[2] = __dmul_rn(mu, v); F[3] = __dmul_rn(mu, w);
  F[4] = __dmul_rn(__dadd_rn(E, p), u);
}

__device__ __forceinline__ void hlle_rn(const double* WL, const double* WR, const Geom& G, double* F) {
  const double cl = __dsqrt_rn(__ddiv_rn(__dmul_rn(G.gamma, WL[4]), WL[0]));
  const double cr = __dsqrt_rn(__ddiv_rn(__dmul_rn(G.gamma, WR[4]), WR[0]));
  double a = __dsub_rn(WL[1], cl), b = __dsub_rn(WR[1], cr);
  const double sl = a < b ? a : b;
  a = __dadd_rn(WL[1], cl);
  b = __dadd_rn(WR[1], cr);
  const double sr = a > b ? a : b;
  const double bp = sr > 0.0 ? sr : 0.0, bm = sl < 0.0 ? sl : 0.0;
  double UL[NVAR], FL[NVAR], UR[NVAR], FR[NVAR];
  phys_rn(WL, G.gm1, G.inv_gm1, UL, FL);
  phys_rn(WR, G.gm1, G.inv_gm1, UR, FR);
  const double inv = __ddiv_rn(1.0, __dsub_rn(bp, bm));
  const double bb = __dmul_rn(bp, bm);
#pragma unroll
  for (int n = 0; n < NVAR; ++n)
    F[n] = __dmul_rn(__dadd_rn(__dsub_rn(__dmul_rn(bp, FL[n]), __dmul_rn(bm, FR[n])), __dmul_rn(bb, __dsub_rn(UR[n], UL[n]))), inv);
}

// exact cons -> prim (oracle order); returns false if rho <= 0 or p <= 0
__device__ __forceinline__ bool cons2prim_rn(double rho, double m1, double m2, double m3, double E, double gm1,
                                             double* W) {
  const double ir = __ddiv_rn(1.0, rho);
  const double v1 = __dmul_rn(m1, ir), v2 = __dmul_rn(m2, ir), v3 = __dmul_rn(m3, ir);
  const double ke = __dmul_rn(0.5, __dadd_rn(__dadd_rn(__dmul_rn(m1, v1), __dmul_rn(m2, v2)), __dmul_rn(m3, v3)));
  const double p = __dmul_rn(gm1, __dsub_rn(E, ke));
  W[0] = rho; W[1] = v1; W[2] = v2; W[3] = v3; W[4] = p;
  return (rho > 0.0) && (p > 0.0);
}

// exact per-cell CFL term (O6): min_d dx_d / (|v_d| + sqrt(gamma p / rho))
__device__ __forceinline__ double cfl_term_rn(const double* W, const BlockMeta& M, double gamma) {
  const double c = __dsqrt_rn(__ddiv_rn(__dmul_rn(gamma, W[4]), W[0]));
  double r = __ddiv_rn(M.dx[0], __dadd_rn(fabs(W[1]), c));
  const double r2 = __ddiv_rn(M.dx[1], __dadd_rn(fabs(W[2]), c));
  const double r3 = __ddiv_rn(M.dx[2], __dadd_rn(fabs(W[3]), c));
  r = r2 < r ? r2 : r;
  return r3 < r ? r3 : r;
}


// ------------------------------------------------------------------------------ stage kernel
// One CTA = a TX x TY tile of (i,j) columns of one block, marching up a k-range of KC planes, one
// thread per column, 2 CTAs per SM.  Plane q is converted to primitives (a2) into slot q%3 of a
// 3-plane smem ring (plus-shaped x/y halo, read from the face neighbours directly when they are
// local and same-level).  Iteration q then computes the x and y faces of plane c = q-2 as flat work
// lists over all threads and the z face between planes c and c+1 of each column (its z states
// carried in registers) -- a3 PLM + a4 HLLE, one code path per face -- and finishes the cells of
// plane c: flux divergence and the RK stage combine (a5).  The final stage also reduces the CFL
// term and the totals (a6, a10).
constexpr int TX = TILE_X, TY = TILE_Y, NCELL = TX * TY, NT = NCELL;

// One face: PLM states from the 4 stencil points p0..p3 (cells c-2 .. c+1 along the normal) of
// the smem primitives, permuted so that w = (rho, u_normal, v_t1, v_t2, p), then HLLE.  F is
// returned in natural component order.  CN/C1/C2: variable index of normal, t1, t2.
template <int RECON, int CN, int C1, int C2, int VSv, bool EIN = false>
__device__ __forceinline__ void face_flux(const double* p0, const double* p1, const double* p2, const double* p3,
                                          const Geom& G, double* F) {
  constexpr int cv[NVAR] = {0, CN, C1, C2, 4};
  double wl[NVAR], wr[NVAR], Fn[NVAR];
#pragma unroll
  for (int s = 0; s < NVAR; ++s) {
    const int o = cv[s] * VSv;
    plm_face<RECON>(p0[o], p1[o], p2[o], p3[o], wl[s], wr[s]);
  }
  hlle<EIN>(wl, wr, G, Fn);
  F[0] = Fn[0];
  F[CN] = Fn[1];
  F[C1] = Fn[2];
  F[C2] = Fn[3];
  F[4] = Fn[4];
}

template <int RECON, bool REDUCE, bool USE_U0, bool ML, bool FULL, bool HB, int TXv = TILE_X, int TYv = TILE_Y,
          bool EIN = false, bool PUT = false>
__global__ void __launch_bounds__(TXv * TYv, 2) stage_kernel(StageArgs A, Geom G) {
  // tile geometry (32x8, or 16x16 for 16-wide blocks), shadowing the 32x8 constants
  constexpr int TX = TXv, TY = TYv, NCELL = TX * TY, NT = NCELL;
  constexpr int SWX = TX + 4, SWY = TY + 4, VS = SWY * SWX, SLOT = NVAR * VS;
  constexpr int FXS = TY * (TX + 1), FYS = (TY + 1) * TX, FZS = NCELL;
  extern __shared__ double smem[];
  double* sW = smem;                       // [3][5][SWY][SWX]: planes q-2, q-1, q
  double* sFx = sW + 3 * SLOT;             // [5][TY][TX+1]
  double* sFy = sFx + NVAR * FXS;          // [5][TY+1][TX]
  double* sFz = sFy + NVAR * FYS;          // [2][5][TY][TX]
  double* exF = sFz + 2 * NVAR * FZS;      // [EXTRA_AHEAD][5][TY + TX]: later planes' x faces fi = 0, y faces jf = 0
  constexpr int EXS = NVAR * (TX + TY);
  constexpr bool PRE = FULL;               // boundary-face precompute on the regular full-tile path

  const int tid = threadIdx.x;
  const int tx = tid % TX, ty = tid / TX;
  const int warp_id = tid >> 5, lane = tid & 31;
  int bid = blockIdx.x;
  const int kc = bid % A.nkc;
  bid /= A.nkc;
  const int tyi = bid % A.nty;
  bid /= A.nty;
  const int txi = bid % A.ntx;
  const int pb = bid / A.ntx;
  const int slot = A.slots[pb];
  const BlockMeta& M = A.meta[slot];
  const int x0 = txi * TX, y0 = tyi * TY;
  const int nxt = FULL ? TX : min(TX, G.n[0] - x0), nyt = FULL ? TY : min(TY, G.n[1] - y0);
  const int k0 = kc * A.KC;
  const int k1 = min(k0 + A.KC, G.n[2]);
  const int g = G.g;
  const int64_t plane = (int64_t)G.N[0] * G.N[1];
  const double* Ub = A.Uin + (int64_t)slot * G.bstride;
  const double dt = A.st->dt_used;
  const double idx1 = M.idx[0], idx2 = M.idx[1], idx3 = M.idx[2];
  const bool own = FULL || ((tx < nxt) && (ty < nyt));

  // ---- load-slot geometry: the plus-shaped halo plane is 2 cells per thread ----
  int sl_i[2], sl_j[2];
  bool sl_ok[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    int c = tid + s * NT;
    int i, j;
    bool ok;
    if (c < SWX * TY) {
      j = c / SWX;
      i = c % SWX - 2;
      ok = (j < nyt) && (i < nxt + 2);
      if (j >= nyt && j < nyt + 2 && i >= 0 && i < nxt) ok = true;  // ragged tile: rows nyt, nyt+1
    } else {
      int c2 = c - SWX * TY;
      int r = c2 / TX;
      i = c2 % TX;
      j = (r < 2) ? r - 2 : TY + r - 2;
      ok = (c2 < 4 * TX) && (i < nxt) && ((r < 2) || (nyt == TY));
    }
    sl_i[s] = i;
    sl_j[s] = j;
    sl_ok[s] = ok;
  }

  // ---- per-slot source pointers (without the plane offset).  Direct halo: a halo cell outside
  // the block in x or y is read from the local same-level face neighbour's interior (M.nb).
  const double* sbase[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    int gi = x0 + sl_i[s], gj = y0 + sl_j[s], bs = slot;
    if (gi < 0 && M.nb[0] >= 0) { bs = M.nb[0]; gi += G.n[0]; }
    else if (gi >= G.n[0] && M.nb[1] >= 0) { bs = M.nb[1]; gi -= G.n[0]; }
    if (gj < 0 && M.nb[2] >= 0) { bs = M.nb[2]; gj += G.n[1]; }
    else if (gj >= G.n[1] && M.nb[3] >= 0) { bs = M.nb[3]; gj -= G.n[1]; }
    sbase[s] = A.Uin + (int64_t)bs * G.bstride + (int64_t)(gj + g) * G.N[0] + (gi + g);
  }
  const int64_t colo = (int64_t)(y0 + ty + g) * G.N[0] + (x0 + tx + g);
  const double* obase = Ub + colo;
  const double* zlo = M.nb[4] >= 0 ? A.Uin + (int64_t)M.nb[4] * G.bstride + colo + (int64_t)G.n[2] * plane : obase;
  const double* zhi = M.nb[5] >= 0 ? A.Uin + (int64_t)M.nb[5] * G.bstride + colo - (int64_t)G.n[2] * plane : obase;

  double pf[2][NVAR];
  auto slot_ptr = [&](int q, int s) -> const double* {
    const bool halo = (q < k0) || (q >= k1);
    const int64_t qo = (int64_t)(q + g) * plane;
    return halo ? ((q < 0 ? zlo : (q >= G.n[2] ? zhi : obase)) + qo) : (sbase[s] + qo);
  };
  auto slot_ok = [&](int q, int s) -> bool {
    const bool halo = (q < k0) || (q >= k1);
    return halo ? (s == 0 && own) : sl_ok[s];
  };
  auto issue_load = [&](int q) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      if (slot_ok(q, s)) {
        const double* p = slot_ptr(q, s);
#pragma unroll
        for (int v = 0; v < NVAR; ++v) pf[s][v] = ld_plane(p + v * G.vstride);
      }
    }
  };
  auto store_prims = [&](int q) {
    const bool halo = (q < k0) || (q >= k1);
    double* W = sW + ((q + 3) % 3) * SLOT;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      int i = halo ? tx : sl_i[s], j = halo ? ty : sl_j[s];
      bool ok = halo ? (s == 0 && own) : sl_ok[s];
      if (ok) {
        double rho = pf[s][0];
        double ir = rcp_nr(rho);
        double v1 = pf[s][1] * ir, v2 = pf[s][2] * ir, v3 = pf[s][3] * ir;
        double ke = 0.5 * ((pf[s][1] * v1 + pf[s][2] * v2) + pf[s][3] * v3);
        double p = G.gm1 * (pf[s][4] - ke);
        if (!(rho > 0.0) || !(p > 0.0)) set_error(A.err, A.stage, M.gid, q, y0 + j, x0 + i);
        int o = (j + 2) * SWX + (i + 2);
        W[o] = rho;
        W[VS + o] = v1;
        W[2 * VS + o] = v2;
        W[3 * VS + o] = v3;
        W[4 * VS + o] = p;
      }
    }
  };

  double tmax = 0.0, tsum[NVAR] = {0.0, 0.0, 0.0, 0.0, 0.0};
  double topz[NVAR] = {0.0, 0.0, 0.0, 0.0, 0.0};  // z top state of plane q-2 (my column)
  const int qbeg = k0 - 2, qend = k1 + 2;
  issue_load(qbeg);
  for (int q = qbeg; q < qend; ++q) {
    store_prims(q);
    if (q + 1 < qend) issue_load(q + 1);  // the next plane's loads fly during this plane's faces
    ph_jitter(2 * q);
    __syncthreads();
    const int c = q - 2;                 // plane whose x/y faces and cells are done now
    const int fz = q - 1;                // z face between planes q-2 and q-1
    const bool xy = (c >= k0) && (c < k1);
    const bool zf = (fz >= k0) && (fz <= k1);
    const double* Wc = sW + ((c + 3) % 3) * SLOT;
    // prefetch the finish-phase operands of my cell so their latency hides behind the faces
    // (without it the kernel is 7 % slower): U_in and U^n, or on the H path only H
    double uin[NVAR], u0v[NVAR];
    const int64_t cell = (int64_t)slot * G.bstride + (int64_t)(c + g) * plane +
                         (int64_t)(y0 + ty + g) * G.N[0] + (x0 + tx + g);
    if (xy && own) {
#pragma unroll
      for (int v = 0; v < NVAR; ++v) {
        if (HB && USE_U0) {
          uin[v] = ld_plane(A.H + cell + v * G.vstride);
        } else {
          uin[v] = ld_plane(A.Uin + cell + v * G.vstride);
          if (USE_U0) u0v[v] = A.U0[cell + v * G.vstride];
        }
      }
    }
    // x faces of plane c: 33 per row, item t -> (row t/33, face t%33); rounds 0,1 (warp 0 only)
    const int phase = (c - k0) % (EXTRA_AHEAD + 1);  // 0: full plane; else boundary faces precomputed
    const bool reduced = PRE && phase != 0;
    // multilevel: x / y face fluxes on a coarse-fine block face also go to the face-flux slots (a8)
    auto ml_x = [&](int pl, int fi, int j, const double* F) {
      const int gi = x0 + fi;
      const int fs = (gi == 0) ? M.fslot[0] : ((gi == G.n[0]) ? M.fslot[1] : -1);
      if (fs >= 0) {
        const int64_t fstr = (int64_t)G.n[1] * G.n[2];
        double* o = A.fbuf + (int64_t)fs * G.fstride + (int64_t)pl * G.n[1] + (y0 + j);
#pragma unroll
        for (int v = 0; v < NVAR; ++v) o[v * fstr] = F[v];
      }
    };
    auto ml_y = [&](int pl, int jf, int i, const double* F) {
      const int gj = y0 + jf;
      const int fs = (gj == 0) ? M.fslot[2] : ((gj == G.n[1]) ? M.fslot[3] : -1);
      if (fs >= 0) {
        const int64_t fstr = (int64_t)G.n[0] * G.n[2];
        double* o = A.fbuf + (int64_t)fs * G.fstride + (int64_t)pl * G.n[0] + (x0 + i);
#pragma unroll
        for (int v = 0; v < NVAR; ++v) o[v * fstr] = F[v];
      }
    };
    if (xy && reduced) {
      // interior faces only: x faces 1..TX of every row, y face rows 1..TY, one round each
#pragma unroll 1
      for (int t = tid; t < TX * TY; t += NT) {
        const int j = t / TX, fi = t - j * TX + 1;
        const double* p = Wc + (j + 2) * SWX + fi;
        double F[NVAR];
        face_flux<RECON, 1, 2, 3, VS, EIN>(p, p + 1, p + 2, p + 3, G, F);
        double* d = sFx + j * (TX + 1) + fi;
        d[0] = F[0]; d[FXS] = F[1]; d[2 * FXS] = F[2]; d[3 * FXS] = F[3]; d[4 * FXS] = F[4];
        if (ML) ml_x(c, fi, j, F);
      }
#pragma unroll 1
      for (int t = tid; t < TX * TY; t += NT) {
        const int jf = t / TX + 1, i = t - (jf - 1) * TX;
        const double* p = Wc + jf * SWX + (i + 2);
        double F[NVAR];
        face_flux<RECON, 2, 3, 1, VS, EIN>(p, p + SWX, p + 2 * SWX, p + 3 * SWX, G, F);
        double* d = sFy + jf * TX + i;
        d[0] = F[0]; d[FYS] = F[1]; d[2 * FYS] = F[2]; d[3 * FYS] = F[3]; d[4 * FYS] = F[4];
        if (ML) ml_y(c, jf, i, F);
      }
      const double* ex = exF + (phase - 1) * EXS;
      for (int t = tid; t < NVAR * (TX + TY); t += NT) {  // the precomputed boundary faces
        const int v = t / (TX + TY), e = t - v * (TX + TY);
        if (e < TY) sFx[v * FXS + e * (TX + 1)] = ex[t];
        else sFy[v * FYS + (e - TY)] = ex[t];
      }
    } else if (xy) {
      if (PRE) {
        // boundary faces of planes c+1 .. c+AHEAD (their primitives are in the ring already) on
        // warps 1-2 and 3,5, which otherwise idle through this plane's 4th round
        const int a = (warp_id == 1 || warp_id == 2) ? 1 : ((warp_id == 3 || warp_id == 5) ? 2 : 0);
        if (a != 0 && a <= EXTRA_AHEAD && c + a < k1) {
          const double* Wn = sW + ((c + a + 3) % 3) * SLOT;
          double* ex = exF + (a - 1) * EXS;
          if ((warp_id == 1 || warp_id == 3) && lane < TY) {
            const double* p = Wn + (lane + 2) * SWX;
            double F[NVAR];
            face_flux<RECON, 1, 2, 3, VS, EIN>(p, p + 1, p + 2, p + 3, G, F);
#pragma unroll
            for (int v = 0; v < NVAR; ++v) ex[v * (TX + TY) + lane] = F[v];
            if (ML) ml_x(c + a, 0, lane, F);
          } else if ((warp_id == 2 || warp_id == 5) && lane < TX) {
            const double* p = Wn + (lane + 2);
            double F[NVAR];
            face_flux<RECON, 2, 3, 1, VS, EIN>(p, p + SWX, p + 2 * SWX, p + 3 * SWX, G, F);
#pragma unroll
            for (int v = 0; v < NVAR; ++v) ex[v * (TX + TY) + TY + lane] = F[v];
            if (ML) ml_y(c + a, 0, lane, F);
          }
        }
      }
#pragma unroll 1
      for (int t = tid; t < (TX + 1) * TY; t += NT) {
        const int j = t / (TX + 1), fi = t - j * (TX + 1);
        if (FULL || (j < nyt && fi <= nxt)) {
          const double* p = Wc + (j + 2) * SWX + fi;
          double F[NVAR];
          face_flux<RECON, 1, 2, 3, VS, EIN>(p, p + 1, p + 2, p + 3, G, F);
          double* d = sFx + j * (TX + 1) + fi;
          d[0] = F[0]; d[FXS] = F[1]; d[2 * FXS] = F[2]; d[3 * FXS] = F[3]; d[4 * FXS] = F[4];
          if (ML) {
            const int gi = x0 + fi;
            const int fs = (gi == 0) ? M.fslot[0] : ((gi == G.n[0]) ? M.fslot[1] : -1);
            if (fs >= 0) {
              const int64_t fstr = (int64_t)G.n[1] * G.n[2];
              double* o = A.fbuf + (int64_t)fs * G.fstride + (int64_t)c * G.n[1] + (y0 + j);
#pragma unroll
              for (int v = 0; v < NVAR; ++v) o[v * fstr] = F[v];
            }
          }
        }
      }
      // y faces: 9 rows of 32; items rotated by 128 so the 9th row lands on warps 4-7
#pragma unroll 1
      for (int r = 0; r < 2; ++r) {
        const int t = (tid + NT / 2) % NT + r * NT;
        if (t >= TX * (TY + 1)) break;
        const int jf = t / TX, i = t - jf * TX;
        if (FULL || (jf <= nyt && i < nxt)) {
          const double* p = Wc + jf * SWX + (i + 2);
          double F[NVAR];
          face_flux<RECON, 2, 3, 1, VS, EIN>(p, p + SWX, p + 2 * SWX, p + 3 * SWX, G, F);
          double* d = sFy + jf * TX + i;
          d[0] = F[0]; d[FYS] = F[1]; d[2 * FYS] = F[2]; d[3 * FYS] = F[3]; d[4 * FYS] = F[4];
          if (ML) {
            const int gj = y0 + jf;
            const int fs = (gj == 0) ? M.fslot[2] : ((gj == G.n[1]) ? M.fslot[3] : -1);
            if (fs >= 0) {
              const int64_t fstr = (int64_t)G.n[0] * G.n[2];
              double* o = A.fbuf + (int64_t)fs * G.fstride + (int64_t)c * G.n[0] + (x0 + i);
#pragma unroll
              for (int v = 0; v < NVAR; ++v) o[v * fstr] = F[v];
            }
          }
        }
      }
    }
    // z direction of my column: the slope of plane q-1 gives its bottom state (right state of the
    // face between q-2 and q-1) and its top state, carried in registers to the next face.
    if (own && q >= qbeg + 2) {
      const int o = (ty + 2) * SWX + (tx + 2);
      const double* pm = sW + ((q + 1) % 3) * SLOT + o;
      const double* p0 = sW + ((q + 2) % 3) * SLOT + o;
      const double* pp = sW + ((q + 3) % 3) * SLOT + o;
      double bot[NVAR], top[NVAR];
#pragma unroll
      for (int v = 0; v < NVAR; ++v) {
        const double a = p0[v * VS];
        if (RECON == 0) {
          const double dl = a - pm[v * VS], dr = pp[v * VS] - a;
          const double h = minmod_half(dl, dr), mp = minmod_pick(dl, dr);
          bot[v] = fma(-h, mp, a);
          top[v] = fma(h, mp, a);
          continue;
        }
        const double s = slope<RECON>(a - pm[v * VS], pp[v * VS] - a);
        bot[v] = fma(-0.5, s, a);
        top[v] = fma(0.5, s, a);
      }
      if (zf) {
        const double wl[NVAR] = {topz[0], topz[3], topz[1], topz[2], topz[4]};  // normal = x3
        const double wr[NVAR] = {bot[0], bot[3], bot[1], bot[2], bot[4]};
        double Fn[NVAR];
        hlle<EIN>(wl, wr, G, Fn);
        const double F[NVAR] = {Fn[0], Fn[2], Fn[3], Fn[1], Fn[4]};
        double* d = sFz + (fz & 1) * NVAR * FZS + tid;
        d[0] = F[0]; d[FZS] = F[1]; d[2 * FZS] = F[2]; d[3 * FZS] = F[3]; d[4 * FZS] = F[4];
        if (ML) {
          const int fs = (fz == 0) ? M.fslot[4] : ((fz == G.n[2]) ? M.fslot[5] : -1);
          if (fs >= 0) {
            const int64_t fstr = (int64_t)G.n[0] * G.n[1];
            double* ob = A.fbuf + (int64_t)fs * G.fstride + (int64_t)(y0 + ty) * G.n[0] + (x0 + tx);
#pragma unroll
            for (int v = 0; v < NVAR; ++v) ob[v * fstr] = F[v];
          }
        }
      }
#pragma unroll
      for (int v = 0; v < NVAR; ++v) topz[v] = top[v];
    }
    ph_jitter(2 * q + 1);
    __syncthreads();
    // ---- finish the cells of plane c: L = -(((dF1 + dF2) + dF3)) and the RK combine ----
    if (xy && own) {
      const double* fzl = sFz + (c & 1) * NVAR * FZS + tid;        // face c   (lower)
      const double* fzu = sFz + ((c + 1) & 1) * NVAR * FZS + tid;  // face c+1 (upper)
      double un[NVAR];
#pragma unroll
      for (int v = 0; v < NVAR; ++v) {
#ifdef PH_STRICT  // strict diagnostic build: the oracle's division by dx
        double d1 = (sFx[v * FXS + ty * (TX + 1) + tx + 1] - sFx[v * FXS + ty * (TX + 1) + tx]) / M.dx[0];
        double d2 = (sFy[v * FYS + (ty + 1) * TX + tx] - sFy[v * FYS + ty * TX + tx]) / M.dx[1];
        double d3 = (fzu[v * FZS] - fzl[v * FZS]) / M.dx[2];
#else
        double d1 = (sFx[v * FXS + ty * (TX + 1) + tx + 1] - sFx[v * FXS + ty * (TX + 1) + tx]) * idx1;
        double d2 = (sFy[v * FYS + (ty + 1) * TX + tx] - sFy[v * FYS + ty * TX + tx]) * idx2;
        double d3 = (fzu[v * FZS] - fzl[v * FZS]) * idx3;
#endif
        double L = -((d1 + d2) + d3);
        double out;
        if (HB && USE_U0) {
          out = fma(A.cdt * dt, L, uin[v]);  // H + cdt dt L
        } else {
          out = fma(A.b1, uin[v], (A.cdt * dt) * L);
          if (USE_U0) out = fma(A.a0, u0v[v], out);
          if (HB && !USE_U0) st_cell(A.H + cell + v * G.vstride, fma(A.hb1, out, A.ha0 * uin[v]));  // stage 1: write H
        }
        un[v] = out;
        st_cell(A.Uout + cell + v * G.vstride, out);
      }
      if (PUT) {
        // fused halo put: a cell within g layers of a face whose neighbour lives on another GPU is
        // stored, as it is finished, straight into that GPU's receive buffer over NVLink -- at the
        // place its unpack reads: the face box (g layers x n x n), [v][cell], cell (k, j, i)-major
        const int cc[3] = {x0 + tx, y0 + ty, c};
#pragma unroll
        for (int f = 0; f < 6; ++f) {
          const int pr = M.prank[f];
          if (pr < 0) continue;
          const int d = f >> 1;
          const int l = (f & 1) ? cc[d] - (G.n[d] - g) : cc[d];  // layer within the face box
          if (l < 0 || l >= g) continue;
          const int e0 = d == 0 ? g : G.n[0], e1 = d == 1 ? g : G.n[1], e2 = d == 2 ? g : G.n[2];
          const int i2 = d == 0 ? l : cc[0], j2 = d == 1 ? l : cc[1], k2 = d == 2 ? l : cc[2];
          const int64_t nbox = (int64_t)e0 * e1 * e2;
          double* dst = A.peer_rbuf[pr] + M.poff[f] + ((int64_t)k2 * e1 + j2) * e0 + i2;
#pragma unroll
          for (int v = 0; v < NVAR; ++v) dst[v * nbox] = un[v];
        }
      }
      // multilevel: the cells of a flux-corrected face layer change after this kernel (reflux); they
      // are reduced after it (rfx_reduce_kernel)
      bool corrected = false;
      if (ML && REDUCE && M.rfx) {
        const int cc[3] = {x0 + tx, y0 + ty, c};
#pragma unroll
        for (int f = 0; f < 6; ++f)
          if (((M.rfx >> f) & 1) && cc[f >> 1] == ((f & 1) ? G.n[f >> 1] - 1 : 0)) corrected = true;
      }
      if (REDUCE && !corrected) {
        double ir = rcp_nr(un[0]);
        double v1 = un[1] * ir, v2 = un[2] * ir, v3 = un[3] * ir;
        double ke = 0.5 * ((un[1] * v1 + un[2] * v2) + un[3] * v3);
        double p = G.gm1 * (un[4] - ke);
        double cs = sound_speed(un[0], p, G.gamma);
        double s1 = (fabs(v1) + cs) * idx1, s2 = (fabs(v2) + cs) * idx2, s3 = (fabs(v3) + cs) * idx3;
        tmax = dmax(tmax, dmax(s1, dmax(s2, s3)));
#pragma unroll
        for (int v = 0; v < NVAR; ++v) tsum[v] += un[v];
      }
    }
  }
  if (REDUCE) {
    // deterministic CTA reduction: warp shuffles then thread 0 in fixed warp order
    __syncthreads();
    double* red = smem;
    for (int off = 16; off > 0; off >>= 1) {
      tmax = fmax(tmax, __shfl_xor_sync(0xffffffffu, tmax, off));
#pragma unroll
      for (int v = 0; v < NVAR; ++v) tsum[v] += __shfl_xor_sync(0xffffffffu, tsum[v], off);
    }
    int warp = tid / 32, lane = tid % 32;
    if (lane == 0) {
      red[warp * 6] = tmax;
#pragma unroll
      for (int v = 0; v < NVAR; ++v) red[warp * 6 + 1 + v] = tsum[v];
    }
    __syncthreads();
    if (tid == 0) {
      double m = 0.0, s[NVAR] = {0, 0, 0, 0, 0};
      for (int w = 0; w < NT / 32; ++w) {
        m = fmax(m, red[w * 6]);
        for (int v = 0; v < NVAR; ++v) s[v] += red[w * 6 + 1 + v];
      }
      double* o = A.partials + (int64_t)(A.cta_base + blockIdx.x) * 6;
      o[0] = m;
      for (int v = 0; v < NVAR; ++v) o[1 + v] = s[v] * M.dV;
    }
  }
}

template <int TXv, int TYv>
size_t stage_smem_bytes_t() {
  constexpr int TX = TXv, TY = TYv, NCELL = TX * TY;
  constexpr int SLOT = NVAR * (TX + 4) * (TY + 4), FXS = TY * (TX + 1), FYS = (TY + 1) * TX, FZS = NCELL;
  return sizeof(double) * (3 * SLOT + NVAR * FXS + NVAR * FYS + 2 * NVAR * FZS + EXTRA_AHEAD * NVAR * (TX + TY));
}
size_t stage_smem_bytes() { return stage_smem_bytes_t<TILE_X, TILE_Y>(); }

// Tile of the stage kernel for blocks of extent n: the full-tile (no bounds checks) minmod path on
// uniform levels uses 32x8 when n1 is a multiple of 32, else 16x16 when n1 and n2 are multiples of 16
// (e.g. 16^3 blocks, which would leave half of a 32-wide tile idle); everything else runs 32x8 tiles
// with bounds checks.  Returns whether the full-tile path applies.
bool stage_tile(const Geom& G, int recon, bool ml, int* tx, int* ty) {
  const bool mm = recon == 0 && !ml && G.wavespeed == 0;  // the Einfeldt variant runs bounds-checked tiles
  if (stage2_applies(G, recon, ml)) {  // stage2.cu: 16 x 16 tiles
    *tx = 16;
    *ty = 16;
    return true;
  }
  if (mm && G.n[0] % TILE_X == 0 && G.n[1] % TILE_Y == 0) {
    *tx = TILE_X;
    *ty = TILE_Y;
    return true;
  }
  if (mm && G.n[0] % 16 == 0 && G.n[1] % 16 == 0) {
    *tx = 16;
    *ty = 16;
    return true;
  }
  *tx = TILE_X;
  *ty = TILE_Y;
  return false;
}

// ------------------------------------------------------------------------------ exchange kernel
// One CTA per chunk of <= XCHUNK cells of one task; all tasks of one phase in one launch
// ("fill-in-one").
constexpr int XT = 256;



__device__ __forceinline__ double mean8(const double* p, int64_t sj, int64_t sk) {
  double a = p[0], b = p[1], c = p[sj], d = p[sj + 1];
  double e = p[sk], f = p[sk + 1], gg = p[sk + sj], h = p[sk + sj + 1];
  return (((a + b) + (c + d)) + ((e + f) + (gg + h))) * 0.125;  // pairwise, (k,j,i) order (A10)
}

// mean8 with the i-pairs as 16-byte loads (p 16-B aligned); same sums in the same order (A10)
__device__ __forceinline__ double mean8v(const double* p, int64_t sj, int64_t sk) {
  const double2 ab = *reinterpret_cast<const double2*>(p), cd = *reinterpret_cast<const double2*>(p + sj);
  const double2 ef = *reinterpret_cast<const double2*>(p + sk), gh = *reinterpret_cast<const double2*>(p + sk + sj);
  return (((ab.x + ab.y) + (cd.x + cd.y)) + ((ef.x + ef.y) + (gh.x + gh.y))) * 0.125;
}

__device__ __forceinline__ int bc_map(int idx, int n, int lo_kind, int hi_kind, bool& flip) {
  if (idx < 0 && lo_kind) {
    if (lo_kind == 2) { flip = !flip; return -1 - idx; }
    return 0;
  }
  if (idx >= n && hi_kind) {
    if (hi_kind == 2) { flip = !flip; return 2 * n - 1 - idx; }
    return n - 1;
  }
  return idx;
}

// pair mode (xtask_pairs): copies, packs and unpacks move two i-adjacent cells per thread with 16-byte
// loads / stores (the x-face boxes are rows of 2 cells, the y / z ones rows of n)
__device__ __forceinline__ void xfill_pair(const XArgs& A, const XTask& t, const Geom& G, int c, int i, int j, int k) {
  double2 v[NVAR];
  if (t.kind == T_UNPACK_U || t.kind == T_UNPACK_C) {
    const double* s = A.rbuf + t.buf + c;
#pragma unroll
    for (int q = 0; q < NVAR; ++q) v[q] = *reinterpret_cast<const double2*>(s + (int64_t)q * t.ncell);
  } else {
    const double* s = A.U + (int64_t)t.src_slot * G.bstride +
                      ((int64_t)(k + t.so[2] + G.g) * G.N[1] + (j + t.so[1] + G.g)) * G.N[0] + (i + t.so[0] + G.g);
#pragma unroll
    for (int q = 0; q < NVAR; ++q) v[q] = __ldcg(reinterpret_cast<const double2*>(s + q * G.vstride));
  }
  double* d;
  int64_t vs;
  if (t.dst_slot < 0) {  // pack into my send buffer or put into peer bc's receive buffer ([v][cell])
    d = (t.bc >= 0 ? A.peer_rbuf[t.bc] : A.sbuf) + t.buf + c;
    vs = t.ncell;
  } else if (t.kind == T_COPY || t.kind == T_UNPACK_U) {
    d = A.U + (int64_t)t.dst_slot * G.bstride + ((int64_t)(k + G.g) * G.N[1] + (j + G.g)) * G.N[0] + (i + G.g);
    vs = G.vstride;
  } else {
    d = A.C + (int64_t)t.dst_slot * G.cbstride + ((int64_t)(k + G.cg) * G.NC[1] + (j + G.cg)) * G.NC[0] + (i + G.cg);
    vs = G.cvstride;
  }
#pragma unroll
  for (int q = 0; q < NVAR; ++q) *reinterpret_cast<double2*>(d + q * vs) = v[q];
}

__global__ void __launch_bounds__(XT) xfill_kernel(XArgs A, Geom G) {
  ph_jitter(threadIdx.x & 31);
  const Chunk ch = A.chunks[blockIdx.x];
  const XTask t = A.tasks[ch.task];
  const int e0 = t.ext[0], e01 = t.ext[0] * t.ext[1];
  if (xtask_pairs(t, G.g, G.cg)) {
    const int end = min(ch.begin + 2 * XCHUNK, t.ncell);
    for (int c = ch.begin + 2 * threadIdx.x; c < end; c += 2 * XT) {
      const int ck = c / e01, rem = c - ck * e01;
      const int cj = rem / e0, ci = rem - cj * e0;
      xfill_pair(A, t, G, c, t.lo[0] + ci, t.lo[1] + cj, t.lo[2] + ck);
    }
    return;
  }
  const int end = min(ch.begin + XCHUNK, t.ncell);
  for (int c = ch.begin + threadIdx.x; c < end; c += XT) {
    const int ck = c / e01, rem = c - ck * e01;
    const int cj = rem / e0, ci = rem - cj * e0;
    const int i = t.lo[0] + ci, j = t.lo[1] + cj, k = t.lo[2] + ck;
    switch (t.kind) {
      case T_COPY:
      case T_CCOPY: {
        const double* s = A.U + (int64_t)t.src_slot * G.bstride +
                          ((int64_t)(k + t.so[2] + G.g) * G.N[1] + (j + t.so[1] + G.g)) * G.N[0] + (i + t.so[0] + G.g);
        if (t.dst_slot < 0) {
          // pack: into my send buffer, or (T_PUT kind stored in bc >= 0) straight into the receive
          // buffer of peer bc over NVLink -- [v][cell] layout, so a warp stores 256 contiguous bytes
          double* d = (t.bc >= 0 ? A.peer_rbuf[t.bc] : A.sbuf) + t.buf + c;
#pragma unroll
          for (int v = 0; v < NVAR; ++v) d[(int64_t)v * t.ncell] = s[v * G.vstride];
        } else if (t.kind == T_COPY) {
          double* d = A.U + (int64_t)t.dst_slot * G.bstride + ((int64_t)(k + G.g) * G.N[1] + (j + G.g)) * G.N[0] + (i + G.g);
#pragma unroll
          for (int v = 0; v < NVAR; ++v) d[v * G.vstride] = s[v * G.vstride];
        } else {
          double* d = A.C + (int64_t)t.dst_slot * G.cbstride + ((int64_t)(k + G.cg) * G.NC[1] + (j + G.cg)) * G.NC[0] + (i + G.cg);
#pragma unroll
          for (int v = 0; v < NVAR; ++v) d[v * G.cvstride] = s[v * G.vstride];
        }
        break;
      }
      case T_RESTRICT:
      case T_CRESTRICT: {
        const int fi = 2 * i - t.so[0], fj = 2 * j - t.so[1], fk = 2 * k - t.so[2];
        const double* s = A.U + (int64_t)t.src_slot * G.bstride + ((int64_t)(fk + G.g) * G.N[1] + (fj + G.g)) * G.N[0] + (fi + G.g);
        const int64_t sj = G.N[0], sk = (int64_t)G.N[0] * G.N[1];
        const bool vec = ((t.so[0] | G.g) & 1) == 0;  // fine i-pairs 16-B aligned (uniform per task)
        double m8[NVAR];
#pragma unroll
        for (int v = 0; v < NVAR; ++v) m8[v] = vec ? mean8v(s + v * G.vstride, sj, sk) : mean8(s + v * G.vstride, sj, sk);
        if (t.dst_slot < 0) {  // pack (or put into peer bc's receive buffer, as for copies)
          double* d = (t.bc >= 0 ? A.peer_rbuf[t.bc] : A.sbuf) + t.buf + c;
#pragma unroll
          for (int v = 0; v < NVAR; ++v) d[(int64_t)v * t.ncell] = m8[v];
        } else if (t.kind == T_RESTRICT) {
          double* d = A.U + (int64_t)t.dst_slot * G.bstride + ((int64_t)(k + G.g) * G.N[1] + (j + G.g)) * G.N[0] + (i + G.g);
#pragma unroll
          for (int v = 0; v < NVAR; ++v) d[v * G.vstride] = m8[v];
        } else {
          double* d = A.C + (int64_t)t.dst_slot * G.cbstride + ((int64_t)(k + G.cg) * G.NC[1] + (j + G.cg)) * G.NC[0] + (i + G.cg);
#pragma unroll
          for (int v = 0; v < NVAR; ++v) d[v * G.cvstride] = m8[v];
        }
        break;
      }
      case T_UNPACK_U: {
        const double* s = A.rbuf + t.buf + c;
        double* d = A.U + (int64_t)t.dst_slot * G.bstride + ((int64_t)(k + G.g) * G.N[1] + (j + G.g)) * G.N[0] + (i + G.g);
#pragma unroll
        for (int v = 0; v < NVAR; ++v) d[v * G.vstride] = s[(int64_t)v * t.ncell];
        break;
      }
      case T_UNPACK_C: {
        const double* s = A.rbuf + t.buf + c;
        double* d = A.C + (int64_t)t.dst_slot * G.cbstride + ((int64_t)(k + G.cg) * G.NC[1] + (j + G.cg)) * G.NC[0] + (i + G.cg);
#pragma unroll
        for (int v = 0; v < NVAR; ++v) d[v * G.cvstride] = s[(int64_t)v * t.ncell];
        break;
      }
      case T_PROLONG: {
        // staging cell (i,j,k) -> fine cells 2i..2i+1 (A11): C + (s1/4)d1 + (s2/4)d2 + (s3/4)d3
        const double* cc = A.C + (int64_t)t.src_slot * G.cbstride + ((int64_t)(k + G.cg) * G.NC[1] + (j + G.cg)) * G.NC[0] + (i + G.cg);
        double* d = A.U + (int64_t)t.dst_slot * G.bstride + ((int64_t)(2 * k + G.g) * G.N[1] + (2 * j + G.g)) * G.N[0] + (2 * i + G.g);
        const int64_t cj = G.NC[0], ckk = (int64_t)G.NC[0] * G.NC[1];
        const int64_t fj = G.N[0], fk = (int64_t)G.N[0] * G.N[1];
#pragma unroll
        for (int v = 0; v < NVAR; ++v) {
          const double* p = cc + v * G.cvstride;
          double c0 = p[0];
          double s1 = minmod_i(c0 - p[-1], p[1] - c0);
          double s2 = minmod_i(c0 - p[-cj], p[cj] - c0);
          double s3 = minmod_i(c0 - p[-ckk], p[ckk] - c0);
          double* q = d + v * G.vstride;
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              double val[2];
#pragma unroll
              for (int e = 0; e < 2; ++e)
                val[e] = __dadd_rn(__dadd_rn(__dadd_rn(c0, __dmul_rn(e ? 0.25 : -0.25, s1)),
                                             __dmul_rn(b ? 0.25 : -0.25, s2)),
                                   __dmul_rn(a ? 0.25 : -0.25, s3));
              // fine cells 2i, 2i+1 are 16-B aligned when g is even: one 128-bit store
              if ((G.g & 1) == 0) {
                *reinterpret_cast<double2*>(q + a * fk + b * fj) = make_double2(val[0], val[1]);
              } else {
                q[a * fk + b * fj] = val[0];
                q[a * fk + b * fj + 1] = val[1];
              }
            }
        }
        break;
      }
      case T_BC_FINE:
      case T_BC_COARSE: {
        const bool coarse = (t.kind == T_BC_COARSE);
        const int n0 = coarse ? G.nc[0] : G.n[0], n1 = coarse ? G.nc[1] : G.n[1], n2 = coarse ? G.nc[2] : G.n[2];
        bool f0 = false, f1 = false, f2 = false;
        int si = bc_map(i, n0, t.bc & 3, (t.bc >> 2) & 3, f0);
        int sj = bc_map(j, n1, (t.bc >> 4) & 3, (t.bc >> 6) & 3, f1);
        int sk = bc_map(k, n2, (t.bc >> 8) & 3, (t.bc >> 10) & 3, f2);
        if (coarse) {
          double* base = A.C + (int64_t)t.dst_slot * G.cbstride;
          int64_t dq = ((int64_t)(k + G.cg) * G.NC[1] + (j + G.cg)) * G.NC[0] + (i + G.cg);
          int64_t sq = ((int64_t)(sk + G.cg) * G.NC[1] + (sj + G.cg)) * G.NC[0] + (si + G.cg);
#pragma unroll
          for (int v = 0; v < NVAR; ++v) {
            double val = base[v * G.cvstride + sq];
            bool fl = (v == 1 && f0) || (v == 2 && f1) || (v == 3 && f2);
            base[v * G.cvstride + dq] = fl ? -val : val;
          }
        } else {
          double* base = A.U + (int64_t)t.dst_slot * G.bstride;
          int64_t dq = ((int64_t)(k + G.g) * G.N[1] + (j + G.g)) * G.N[0] + (i + G.g);
          int64_t sq = ((int64_t)(sk + G.g) * G.N[1] + (sj + G.g)) * G.N[0] + (si + G.g);
#pragma unroll
          for (int v = 0; v < NVAR; ++v) {
            double val = base[v * G.vstride + sq];
            bool fl = (v == 1 && f0) || (v == 2 && f1) || (v == 3 && f2);
            base[v * G.vstride + dq] = fl ? -val : val;
          }
        }
        break;
      }
    }
  }
}

// ------------------------------------------------------------------------------ reflux (O8 / a8)
// U_c(adjacent cell) += w dt s (F_own - F_corr) / dx, F_corr = pairwise mean of 4 fine fluxes.
__global__ void reflux_kernel(const RefluxTask* tasks, double* U, const BlockMeta* meta, const double* fbuf,
                              const double* rbuf, const CycleState* st, double w, Geom G, double* H, double hb1) {
  const RefluxTask t = tasks[blockIdx.x];  // tasks on x: up to 2^31 - 1
  const int d = t.dir;
  const int ta = (d == 0) ? 1 : 0, tb = (d == 2) ? 1 : 2;  // tangential dims, increasing
  const int na = G.n[ta], nb = G.n[tb];
  const int qa = na / 2, qb = nb / 2;
  const int idxc = blockIdx.y * blockDim.x + threadIdx.x;
  if (idxc >= qa * qb) return;
  const int A0 = idxc % qa, B0 = idxc / qa;
  const int Ac = t.t0lo + A0, Bc = t.t1lo + B0;
  const double dt = st->dt_used;
  const double fac = w * dt * meta[t.cslot].idx[d] * (double)t.side;
  const int64_t fst = (int64_t)na * nb;
  const double* ff = fbuf + (int64_t)t.ffs * G.fstride;
  const double* cf = fbuf + (int64_t)t.cfs * G.fstride;
  int c[3];
  c[d] = (t.side < 0) ? 0 : G.n[d] - 1;
  c[ta] = Ac;
  c[tb] = Bc;
  double* u = U + (int64_t)t.cslot * G.bstride + ((int64_t)(c[2] + G.g) * G.N[1] + (c[1] + G.g)) * G.N[0] + (c[0] + G.g);
  const int a0 = 2 * A0, b0 = 2 * B0;
#pragma unroll
  for (int v = 0; v < NVAR; ++v) {
    double corr;
    if (t.roff >= 0) {
      corr = rbuf[t.roff + (int64_t)v * qa * qb + (int64_t)B0 * qa + A0];
    } else {
      const double* f = ff + v * fst;
      double f00 = f[(int64_t)b0 * na + a0], f10 = f[(int64_t)b0 * na + a0 + 1];
      double f01 = f[(int64_t)(b0 + 1) * na + a0], f11 = f[(int64_t)(b0 + 1) * na + a0 + 1];
      corr = ((f00 + f10) + (f01 + f11)) * 0.25;
    }
    double own = cf[v * fst + (int64_t)Bc * na + Ac];
    const double du = fac * (own - corr);
    u[v * G.vstride] += du;
    // stage 1 on the H path: the stage-2 base H = ha0 U^n + hb1 U^1 follows the corrected U^1
    if (H) H[(u - U) + v * G.vstride] += hb1 * du;
  }
}

__global__ void flux_pack_kernel(const FluxPackTask* tasks, const double* fbuf, double* sbuf, Geom G) {
  const FluxPackTask t = tasks[blockIdx.x];
  const int d = t.dir;
  const int ta = (d == 0) ? 1 : 0, tb = (d == 2) ? 1 : 2;
  const int na = G.n[ta], nb = G.n[tb];
  const int qa = na / 2, qb = nb / 2;
  const int idxc = blockIdx.y * blockDim.x + threadIdx.x;
  if (idxc >= qa * qb) return;
  const int A0 = idxc % qa, B0 = idxc / qa;
  const int a0 = 2 * A0, b0 = 2 * B0;
  const int64_t fst = (int64_t)na * nb;
  const double* ff = fbuf + (int64_t)t.ffs * G.fstride;
#pragma unroll
  for (int v = 0; v < NVAR; ++v) {
    const double* f = ff + v * fst;
    double f00 = f[(int64_t)b0 * na + a0], f10 = f[(int64_t)b0 * na + a0 + 1];
    double f01 = f[(int64_t)(b0 + 1) * na + a0], f11 = f[(int64_t)(b0 + 1) * na + a0 + 1];
    sbuf[t.off + (int64_t)v * qa * qb + (int64_t)B0 * qa + A0] = ((f00 + f10) + (f01 + f11)) * 0.25;
  }
}

// ------------------------------------------------------------------------------ problem generators (O4)


__global__ void pgen_kernel(double* U, const BlockMeta* meta, int nslots, PgenArgs P, Geom G) {
  const int row = blockIdx.x;  // (slot, k, j)
  const int j = row % G.n[1];
  const int k = (row / G.n[1]) % G.n[2];
  const int slot = row / (G.n[1] * G.n[2]);
  if (slot >= nslots) return;
  const BlockMeta& M = meta[slot];
  const double gamma = G.gamma;
  for (int i = threadIdx.x; i < G.n[0]; i += blockDim.x) {
    double x = __dadd_rn(M.xmin[0], __dmul_rn((double)i + 0.5, M.dx[0]));
    double y = __dadd_rn(M.xmin[1], __dmul_rn((double)j + 0.5, M.dx[1]));
    double z = __dadd_rn(M.xmin[2], __dmul_rn((double)k + 0.5, M.dx[2]));
    double W[5];
    if (P.problem == 0) {  // linear wave, right-going acoustic eigenvector (A20)
      double A = P.p[0];
      double K1 = P.p[1] / P.L[0], K2 = P.p[2] / P.L[1], K3 = P.p[3] / P.L[2];
      double kn = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(K1, K1), __dmul_rn(K2, K2)), __dmul_rn(K3, K3)));
      double ph = __dadd_rn(__dadd_rn(__dmul_rn(K1, __dsub_rn(x, P.xmin[0])), __dmul_rn(K2, __dsub_rn(y, P.xmin[1]))),
                            __dmul_rn(K3, __dsub_rn(z, P.xmin[2])));
      double s = sin(__dmul_rn(2.0 * 3.14159265358979323846, ph));
      W[0] = __dadd_rn(1.0, __dmul_rn(A, s));
      double va = __dmul_rn(A, s);  // c0 = 1
      W[1] = __dmul_rn(va, K1 / kn);
      W[2] = __dmul_rn(va, K2 / kn);
      W[3] = __dmul_rn(va, K3 / kn);
      W[4] = __dadd_rn(1.0 / gamma, __dmul_rn(A, s));
    } else if (P.problem == 1) {  // Sod (A22)
      bool left = x < P.p[0];
      W[0] = left ? 1.0 : 0.125;
      W[4] = left ? 1.0 : 0.1;
      W[1] = W[2] = W[3] = 0.0;
    } else if (P.problem == 3) {  // Kelvin-Helmholtz (A36)
      double xx = __ddiv_rn(__dsub_rn(x, P.xmin[0]), P.L[0]);
      double yy = __ddiv_rn(__dsub_rn(y, P.xmin[1]), P.L[1]);
      bool in = fabs(__dsub_rn(yy, 0.5)) < 0.25;
      double e1 = __ddiv_rn(__dsub_rn(yy, 0.25), P.p[1]), e2 = __ddiv_rn(__dsub_rn(yy, 0.75), P.p[1]);
      W[0] = in ? 2.0 : 1.0;
      W[1] = in ? 0.5 : -0.5;
      W[2] = __dmul_rn(__dmul_rn(P.p[0], sin(__dmul_rn(4.0 * 3.14159265358979323846, xx))),
                       __dadd_rn(exp(-__dmul_rn(e1, e1)), exp(-__dmul_rn(e2, e2))));
      W[3] = 0.0;
      W[4] = 2.5;
    } else {  // blast (A21)
      double dx = __dsub_rn(x, P.p[3]), dy = __dsub_rn(y, P.p[4]), dz = __dsub_rn(z, P.p[5]);
      double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
      W[0] = 1.0;
      W[1] = W[2] = W[3] = 0.0;
      W[4] = (r2 < __dmul_rn(P.p[2], P.p[2])) ? P.p[0] : P.p[1];
    }
    double* u = U + (int64_t)slot * G.bstride + ((int64_t)(k + G.g) * G.N[1] + (j + G.g)) * G.N[0] + (i + G.g);
    double rho = W[0];
    u[0] = rho;
    u[G.vstride] = __dmul_rn(rho, W[1]);
    u[2 * G.vstride] = __dmul_rn(rho, W[2]);
    u[3 * G.vstride] = __dmul_rn(rho, W[3]);
    double ke = __dadd_rn(__dadd_rn(__dmul_rn(W[1], W[1]), __dmul_rn(W[2], W[2])), __dmul_rn(W[3], W[3]));
    u[4 * G.vstride] = __dadd_rn(W[4] / G.gm1, __dmul_rn(__dmul_rn(0.5, rho), ke));
  }
}

// ------------------------------------------------------------------------------ reductions (a6, a10)
// Standalone dt / totals pass over interiors (initial dt, multilevel after reflux, ph_totals).
__global__ void reduce_kernel(const double* U, const BlockMeta* meta, int nslots, double* partials, int cta_base,
                              ErrWord* err, Geom G) {
  const int row = blockIdx.x;  // (slot, k)
  const int k = row % G.n[2];
  const int slot = row / G.n[2];
  double tmax = -INFINITY, ts[NVAR] = {0, 0, 0, 0, 0};
  if (slot < nslots) {
    const BlockMeta& M = meta[slot];
    const int nij = G.n[0] * G.n[1];
    for (int c = threadIdx.x; c < nij; c += blockDim.x) {
      int j = c / G.n[0], i = c % G.n[0];
      const double* u = U + (int64_t)slot * G.bstride + ((int64_t)(k + G.g) * G.N[1] + (j + G.g)) * G.N[0] + (i + G.g);
      double un[NVAR];
#pragma unroll
      for (int v = 0; v < NVAR; ++v) un[v] = u[v * G.vstride];
      if (G.exact) {
        double Wn[NVAR];
        if (!cons2prim_rn(un[0], un[1], un[2], un[3], un[4], G.gm1, Wn)) set_error(err, 0, M.gid, k, j, i);
        tmax = fmax(tmax, -cfl_term_rn(Wn, M, G.gamma));
      } else {
        double ir = rcp_nr(un[0]);
        double v1 = un[1] * ir, v2 = un[2] * ir, v3 = un[3] * ir;
        double ke = 0.5 * ((un[1] * v1 + un[2] * v2) + un[3] * v3);
        double p = G.gm1 * (un[4] - ke);
        if (!(un[0] > 0.0) || !(p > 0.0)) set_error(err, 0, M.gid, k, j, i);
        double cs = sound_speed(un[0], p, G.gamma);
        double s1 = (fabs(v1) + cs) * M.idx[0], s2 = (fabs(v2) + cs) * M.idx[1], s3 = (fabs(v3) + cs) * M.idx[2];
        tmax = dmax(tmax, dmax(s1, dmax(s2, s3)));
      }
#pragma unroll
      for (int v = 0; v < NVAR; ++v) ts[v] += un[v];
    }
  }
  __shared__ double red[32][6];
  for (int off = 16; off > 0; off >>= 1) {
    tmax = fmax(tmax, __shfl_xor_sync(0xffffffffu, tmax, off));
#pragma unroll
    for (int v = 0; v < NVAR; ++v) ts[v] += __shfl_xor_sync(0xffffffffu, ts[v], off);
  }
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane == 0) {
    red[warp][0] = tmax;
    for (int v = 0; v < NVAR; ++v) red[warp][1 + v] = ts[v];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = -INFINITY, s[NVAR] = {0, 0, 0, 0, 0};
    for (int w = 0; w < (int)blockDim.x / 32; ++w) {
      m = fmax(m, red[w][0]);
      for (int v = 0; v < NVAR; ++v) s[v] += red[w][1 + v];
    }
    double dV = slot < nslots ? meta[slot].dV : 0.0;
    double* o = partials + (int64_t)(cta_base + blockIdx.x) * 6;
    o[0] = m;
    for (int v = 0; v < NVAR; ++v) o[1 + v] = s[v] * dV;
  }
}

// partials [n][6] -> out[6] (max, 5 sums), deterministic for fixed n
__global__ void rank_reduce_kernel(const double* partials, int n, double* out) {
  __shared__ double sm[256][6];
  double m = -INFINITY, s[NVAR] = {0, 0, 0, 0, 0};
  for (int c = threadIdx.x; c < n; c += 256) {
    const double* p = partials + (int64_t)c * 6;
    m = fmax(m, p[0]);
    for (int v = 0; v < NVAR; ++v) s[v] += p[1 + v];
  }
  sm[threadIdx.x][0] = m;
  for (int v = 0; v < NVAR; ++v) sm[threadIdx.x][1 + v] = s[v];
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      sm[threadIdx.x][0] = fmax(sm[threadIdx.x][0], sm[threadIdx.x + w][0]);
      for (int v = 0; v < NVAR; ++v) sm[threadIdx.x][1 + v] += sm[threadIdx.x + w][1 + v];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int v = 0; v < 6; ++v) out[v] = sm[0][v];
}

// mode 0: initial dt (no history); mode 1: end of cycle; mode 2: totals only (out6 -> tot)
__global__ void finalize_kernel(const double* all, int nranks, CycleState* st, double* hist, int hist_cap,
                                double cfl, int mode, double* tot_out, int exact) {
  double m = -INFINITY, s[NVAR] = {0, 0, 0, 0, 0};
  for (int r = 0; r < nranks; ++r) {
    m = fmax(m, all[r * 6]);
    for (int v = 0; v < NVAR; ++v) s[v] += all[r * 6 + 1 + v];
  }
  if (tot_out)
    for (int v = 0; v < NVAR; ++v) tot_out[v] = s[v];
  if (mode == 2) return;
  // cfl * min(dx/(|v|+c)) (O6); exact mode carries -min(dx/(|v|+c)) itself
  double dt_new = exact ? __dmul_rn(cfl, -m) : cfl / m;
  if (mode == 0) {
    st->dt = dt_new;
    return;
  }
  if (!st->active) return;
  st->t += st->dt_used;
  st->cycle += 1;
  st->dt = dt_new;
  long long r = st->hist_count % hist_cap;
  double* h = hist + r * 7;
  h[0] = st->t;
  h[1] = st->dt_used;
  for (int v = 0; v < NVAR; ++v) h[2 + v] = s[v];
  st->hist_count += 1;
}

__global__ void cycle_begin_kernel(CycleState* st, double tlim, int set_tlim) {
  if (set_tlim) st->tlim = tlim;
  double t = st->t, dt = st->dt, tl = st->tlim;
  int active = !(tl > 0.0 && t >= tl);
  double du = dt;
  if (tl > 0.0 && t + dt > tl) du = tl - t;
  st->active = active;
  st->dt_used = active ? du : 0.0;
}

// ------------------------------------------------------------------------------ interior copies
// buf [slot][5][n3][n2][n1] <-> pool interiors (host-state upload / download, e2e path)
__global__ void interior_copy_kernel(double* U, double* buf, int slot0, int to_pool, Geom G) {
  const int row = blockIdx.x;  // (slot, v, k, j)
  const int j = row % G.n[1];
  const int k = (row / G.n[1]) % G.n[2];
  const int v = (row / (G.n[1] * G.n[2])) % NVAR;
  const int s = row / (G.n[1] * G.n[2] * NVAR);
  double* u = U + (int64_t)(slot0 + s) * G.bstride + v * G.vstride + ((int64_t)(k + G.g) * G.N[1] + (j + G.g)) * G.N[0] + G.g;
  double* b = buf + (int64_t)row * G.n[0];
  for (int i = threadIdx.x; i < G.n[0]; i += blockDim.x) {
    if (to_pool) u[i] = b[i];
    else b[i] = u[i];
  }
}

// ------------------------------------------------------------------------------ NEXT 3: PPM / WENO-Z
// Generic high-order path (nghost = 3, uniform meshes): primitives of every pool cell, one face-flux
// kernel per direction (6-point stencils), then divergence + RK update.  Formulas as the oracle's
// readings A37 (PPM, Colella & Woodward 1984 eqs. 1.6-1.10) and A38 (WENO-Z, Borges et al. 2008).
__device__ __forceinline__ double ppm_dm(double a, double b, double c) {
  const double dl = b - a, dr = c - b;
  const bool same = (dl > 0.0 && dr > 0.0) || (dl < 0.0 && dr < 0.0);
  if (!same) return 0.0;
  const double dq = 0.5 * (c - a);
  const double m = fmin(fabs(dq), fmin(2.0 * fabs(dl), 2.0 * fabs(dr)));
  return dq > 0.0 ? m : -m;
}

__device__ __forceinline__ void ppm_cell(const double* q, double& ql, double& qr) {
  const double dm_m = ppm_dm(q[0], q[1], q[2]), dm_0 = ppm_dm(q[1], q[2], q[3]), dm_p = ppm_dm(q[2], q[3], q[4]);
  double L = q[1] + 0.5 * (q[2] - q[1]) - (dm_0 - dm_m) / 6.0;
  double R = q[2] + 0.5 * (q[3] - q[2]) - (dm_p - dm_0) / 6.0;
  const double c = q[2];
  if ((R - c) * (c - L) <= 0.0) {
    L = c;
    R = c;
  } else {
    const double d = R - L, m6 = 6.0 * (c - 0.5 * (L + R));
    if (d * m6 > d * d) L = 3.0 * c - 2.0 * R;
    else if (-(d * d) > d * m6) R = 3.0 * c - 2.0 * L;
  }
  ql = L;
  qr = R;
}

__device__ __forceinline__ double wenoz_face(double a, double b, double c, double d, double e) {
  const double t0 = a - 2.0 * b + c, u0 = a - 4.0 * b + 3.0 * c;
  const double t1 = b - 2.0 * c + d, u1 = b - d;
  const double t2 = c - 2.0 * d + e, u2 = 3.0 * c - 4.0 * d + e;
  const double b0 = (13.0 / 12.0) * (t0 * t0) + 0.25 * (u0 * u0);
  const double b1 = (13.0 / 12.0) * (t1 * t1) + 0.25 * (u1 * u1);
  const double b2 = (13.0 / 12.0) * (t2 * t2) + 0.25 * (u2 * u2);
  const double tau = fabs(b0 - b2);
  const double r0 = tau / (b0 + 1e-40), r1 = tau / (b1 + 1e-40), r2 = tau / (b2 + 1e-40);
  const double a0 = 0.1 * (1.0 + r0 * r0), a1 = 0.6 * (1.0 + r1 * r1), a2 = 0.3 * (1.0 + r2 * r2);
  const double q0 = (2.0 * a - 7.0 * b + 11.0 * c) / 6.0;
  const double q1 = (-b + 5.0 * c + 2.0 * d) / 6.0;
  const double q2 = (2.0 * c + 5.0 * d - e) / 6.0;
  return ((a0 * q0 + a1 * q1) + a2 * q2) / ((a0 + a1) + a2);
}

template <int RECON>
__device__ __forceinline__ void recon_face6(const double* q, double& wl, double& wr) {
  // q[0..5] = cells c-3 .. c+2 of the face between c-1 and c
  if (RECON == 3) {
    double a, b;
    ppm_cell(q, a, wl);
    ppm_cell(q + 1, wr, b);
  } else if (RECON == 4) {
    wl = wenoz_face(q[0], q[1], q[2], q[3], q[4]);
    wr = wenoz_face(q[5], q[4], q[3], q[2], q[1]);
  } else {
    plm_face<RECON>(q[1], q[2], q[3], q[4], wl, wr);
  }
}

__global__ void prim_kernel(const double* U, double* W, const BlockMeta* meta, ErrWord* err, int stage, Geom G) {
  const int kk = blockIdx.x % G.N[2];
  const int slot = blockIdx.x / G.N[2];
  const double* u = U + (int64_t)slot * G.bstride + (int64_t)kk * G.N[0] * G.N[1];
  double* w = W + (int64_t)slot * G.bstride + (int64_t)kk * G.N[0] * G.N[1];
  const int k = kk - G.g;
  for (int c = threadIdx.x; c < G.N[0] * G.N[1]; c += blockDim.x) {
    const int j = c / G.N[0] - G.g, i = c % G.N[0] - G.g;
    const int out = (k < 0 || k >= G.n[2]) + (j < 0 || j >= G.n[1]) + (i < 0 || i >= G.n[0]);
    if (out > 1) continue;  // only the cross-shaped halo is ever read
    double Wc[NVAR];
    if (!cons2prim_rn(u[c], u[c + G.vstride], u[c + 2 * G.vstride], u[c + 3 * G.vstride], u[c + 4 * G.vstride], G.gm1, Wc))
      set_error(err, stage, meta[slot].gid, k, j, i);
#pragma unroll
    for (int v = 0; v < NVAR; ++v) w[c + v * G.vstride] = Wc[v];
  }
}

template <int DIR, int RECON>
__device__ __forceinline__ void hoflux_body(const double* W, double* F, const Geom& G) {
  const int e0 = G.n[0] + (DIR == 0), e1 = G.n[1] + (DIR == 1), e2 = G.n[2] + (DIR == 2);
  const int k = blockIdx.x % e2;
  const int slot = blockIdx.x / e2;
  const int64_t st = (DIR == 0) ? 1 : ((DIR == 1) ? G.N[0] : (int64_t)G.N[0] * G.N[1]);
  constexpr int CN = 1 + DIR, C1 = 1 + (DIR + 1) % 3, C2 = 1 + (DIR + 2) % 3;
  const int64_t fvs = (int64_t)e0 * e1 * e2;
  double* fb = F + (int64_t)slot * NVAR * fvs + (int64_t)k * e0 * e1;
  const double* wb = W + (int64_t)slot * G.bstride;
  for (int c = threadIdx.x; c < e0 * e1; c += blockDim.x) {
    const int j = c / e0, i = c % e0;
    const double* p = wb + ((int64_t)(k + G.g) * G.N[1] + (j + G.g)) * G.N[0] + (i + G.g);
    double wl[NVAR], wr[NVAR];
    const int cv[NVAR] = {0, CN, C1, C2, 4};
#pragma unroll
    for (int s = 0; s < NVAR; ++s) {
      const double* q0 = p + cv[s] * G.vstride;
      double q[6];
#pragma unroll
      for (int t = 0; t < 6; ++t) q[t] = q0[(t - 3) * st];
      recon_face6_rn<RECON>(q, wl[s], wr[s]);
    }
    double Fn[NVAR];
    hlle_rn(wl, wr, G, Fn);
    double Fo[NVAR];
    Fo[0] = Fn[0];
    Fo[CN] = Fn[1];
    Fo[C1] = Fn[2];
    Fo[C2] = Fn[3];
    Fo[4] = Fn[4];
#pragma unroll
    for (int v = 0; v < NVAR; ++v) fb[v * fvs + c] = Fo[v];
  }
}

// Line-march variant of hoflux_kernel (same arithmetic, bit for bit): one thread owns a line of
// faces along DIR (or a segment of it, when there are too few lines to fill the GPU) and slides a
// 6-cell register window up the line, so each cell is loaded once per line instead of six times,
// and the per-cell pieces of the reconstruction are computed once and carried: PLM's limited slope
// (used by the two faces of a cell) and PPM's limited slopes dm and right interface value (each
// dm feeds three cells, each cell two faces).  WENO-Z's two face values share no exact
// sub-expression (the mirrored smoothness indicators round differently), so only the loads are
// saved.  Lines are numbered with the fastest non-DIR axis fastest (coalesced for DIR = y, z).
template <int DIR, int RECON>
__device__ __forceinline__ void holine_body(const double* W, double* F, int nslots, int nseg, const Geom& G) {
  constexpr int AX = (DIR == 0) ? 1 : 0, BX = (DIR == 2) ? 1 : 2;
  constexpr int CN = 1 + DIR, C1 = 1 + (DIR + 1) % 3, C2 = 1 + (DIR + 2) % 3;
  const int na = G.n[AX], nb = G.n[BX], nm = G.n[DIR];
  const int64_t lines = (int64_t)na * nb;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= lines * nseg * nslots) return;
  const int64_t line = t % lines;
  const int seg = (int)((t / lines) % nseg);
  const int slot = (int)(t / (lines * nseg));
  const int a = (int)(line % na), b = (int)(line / na);
  const int m0 = (int)((int64_t)seg * (nm + 1) / nseg), m1 = (int)((int64_t)(seg + 1) * (nm + 1) / nseg);
  int c3[3];
  c3[DIR] = 0;
  c3[AX] = a;
  c3[BX] = b;
  const int64_t st = (DIR == 0) ? 1 : ((DIR == 1) ? G.N[0] : (int64_t)G.N[0] * G.N[1]);
  const double* p = W + (int64_t)slot * G.bstride + ((int64_t)(c3[2] + G.g) * G.N[1] + (c3[1] + G.g)) * G.N[0] + (c3[0] + G.g);
  const int e0 = G.n[0] + (DIR == 0), e1 = G.n[1] + (DIR == 1), e2 = G.n[2] + (DIR == 2);
  const int64_t fvs = (int64_t)e0 * e1 * e2;
  const int64_t fst = (DIR == 0) ? 1 : ((DIR == 1) ? e0 : (int64_t)e0 * e1);
  double* fb = F + (int64_t)slot * NVAR * fvs + ((int64_t)c3[2] * e1 + c3[1]) * e0 + c3[0];
  const int cv[NVAR] = {0, CN, C1, C2, 4};
  double q[NVAR][6], c1v[NVAR], c2v[NVAR], c3v[NVAR];  // window; carried per-cell terms
#pragma unroll
  for (int s = 0; s < NVAR; ++s) {
    const double* qs = p + cv[s] * G.vstride;
#pragma unroll
    for (int u = 0; u < 6; ++u) q[s][u] = qs[(int64_t)(m0 - 3 + u) * st];
    if (RECON <= 2) {
      c1v[s] = slope_rn(q[s][1], q[s][2], q[s][3], RECON);  // slope of cell m0-1
    } else if (RECON == 3) {
      double Ldummy;
      ppm_cell_rn(&q[s][0], Ldummy, c1v[s]);               // R of cell m0-1
      c2v[s] = ppm_dm_rn(q[s][1], q[s][2], q[s][3]);       // dm of cell m0-1
      c3v[s] = ppm_dm_rn(q[s][2], q[s][3], q[s][4]);       // dm of cell m0
    }
  }
  for (int m = m0; m < m1; ++m) {
    double nx[NVAR];
    const bool more = m + 1 < m1;
#pragma unroll
    for (int s = 0; s < NVAR; ++s) nx[s] = more ? p[cv[s] * G.vstride + (int64_t)(m + 3) * st] : 0.0;
    double wl[NVAR], wr[NVAR];
#pragma unroll
    for (int s = 0; s < NVAR; ++s) {
      const double* qq = q[s];
      if (RECON <= 2) {
        const double sm = slope_rn(qq[2], qq[3], qq[4], RECON);
        wl[s] = __dadd_rn(qq[2], __dmul_rn(0.5, c1v[s]));
        wr[s] = __dsub_rn(qq[3], __dmul_rn(0.5, sm));
        c1v[s] = sm;
      } else if (RECON == 3) {
        const double dp = ppm_dm_rn(qq[3], qq[4], qq[5]);
        double L, R;
        ppm_lr_rn(qq[2], qq[3], qq[4], c2v[s], c3v[s], dp, L, R);
        wl[s] = c1v[s];
        wr[s] = L;
        c1v[s] = R;
        c2v[s] = c3v[s];
        c3v[s] = dp;
      } else {
        wl[s] = wenoz_rn(qq[0], qq[1], qq[2], qq[3], qq[4]);
        wr[s] = wenoz_rn(qq[5], qq[4], qq[3], qq[2], qq[1]);
      }
    }
    double Fn[NVAR];
    hlle_rn(wl, wr, G, Fn);
    double* fo = fb + (int64_t)m * fst;
    fo[0] = Fn[0];
    fo[CN * fvs] = Fn[1];
    fo[C1 * fvs] = Fn[2];
    fo[C2 * fvs] = Fn[3];
    fo[4 * fvs] = Fn[4];
#pragma unroll
    for (int s = 0; s < NVAR; ++s) {
#pragma unroll
      for (int u = 0; u < 5; ++u) q[s][u] = q[s][u + 1];
      q[s][5] = nx[s];
    }
  }
}

template <int DIR, int RECON>
__global__ void hoflux_kernel(const double* W, double* F, Geom G) {
  hoflux_body<DIR, RECON>(W, F, G);
}

// x fluxes with one cell per lane (PLM / PPM): each lane reconstructs its own cell's two interface values
// once -- PPM's three limited slopes and L / R, PLM's one slope -- and face f (cells f-1 | f) takes R of
// cell f-1 from the lane below by a shuffle, halving hoflux_kernel<0>'s reconstruction work (it builds
// both cells of every face).  A warp holds 32 consecutive cells of the flattened sequence (row j, cell
// -1..n0) and emits the faces whose left cell it also holds; consecutive warps overlap by one cell.
// Same operations on the same operands as hoflux_kernel<0, RECON>: bit for bit (A40).
template <int RECON>
__global__ void __launch_bounds__(128) hofx_kernel(const double* W, double* F, Geom G) {
  const int n0 = G.n[0], n1 = G.n[1], e0 = n0 + 1, RC = n0 + 2, total = n1 * RC;
  const int k = blockIdx.x % G.n[2], slot = blockIdx.x / G.n[2];
  const int nch = (total - 1 + 30) / 31;
  const int64_t fvs = (int64_t)e0 * n1 * G.n[2];
  double* fb = F + (int64_t)slot * NVAR * fvs + (int64_t)k * e0 * n1;
  const double* wb = W + (int64_t)slot * G.bstride + (int64_t)(k + G.g) * G.N[1] * G.N[0];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int ch = warp; ch < nch; ch += nw) {
    const int t = ch * 31 + lane;
    const bool valid = t < total;
    const int j = valid ? t / RC : 0, ci = valid ? t % RC - 1 : 0;
    const double* p = wb + (int64_t)(j + G.g) * G.N[0] + (ci + G.g);
    double L[NVAR], R[NVAR];
#pragma unroll
    for (int v = 0; v < NVAR; ++v) {
      double q[5];
#pragma unroll
      for (int u = 0; u < 5; ++u) q[u] = (valid && (RECON == 3 || (u >= 1 && u <= 3))) ? p[v * G.vstride + (u - 2)] : 1.0;
      if (RECON == 3) {
        ppm_cell_rn(q, L[v], R[v]);
      } else {
        const double sl = slope_rn(q[1], q[2], q[3], RECON);
        R[v] = __dadd_rn(q[2], __dmul_rn(0.5, sl));
        L[v] = __dsub_rn(q[2], __dmul_rn(0.5, sl));
      }
    }
    double wl[NVAR];
#pragma unroll
    for (int v = 0; v < NVAR; ++v) wl[v] = __shfl_up_sync(0xffffffffu, R[v], 1);
    if (valid && lane > 0 && ci >= 0) {
      double Fn[NVAR];
      hlle_rn(wl, L, G, Fn);
      double* fo = fb + (int64_t)j * e0 + ci;
#pragma unroll
      for (int v = 0; v < NVAR; ++v) fo[v * fvs] = Fn[v];
    }
  }
}
// PPM's march is capped at 128 registers (4 CTAs of 128 per SM; some spills): +2 % over 158-174
// registers, 3 % over a 168-register cap.  A cap on the per-face WENO-Z kernel (80/72/64 registers)
// loses 7/14/23 % (profiles/r01_ho_line_march.md).
#ifndef PH_HOLINE_MINB
#define PH_HOLINE_MINB 3  // CTAs per SM the PPM line march is compiled for (round 2, after the
                          // branchless PPM: 3 -> 6.86, 4 -> 7.65, 2 -> 7.33 ms per cycle)
#endif
template <int DIR, int RECON>
__global__ void __launch_bounds__(128, RECON == 3 ? PH_HOLINE_MINB : 1) holine_kernel(const double* W, double* F, int nslots,
                                                                         int nseg, Geom G) {
  holine_body<DIR, RECON>(W, F, nslots, nseg, G);
}

template <bool REDUCE, bool USE_U0>
__global__ void houpdate_kernel(StageArgs A, const double* Fx, const double* Fy, const double* Fz, double* Wout,
                                Geom G) {
  const int k = blockIdx.x % G.n[2];
  const int slot = blockIdx.x / G.n[2];
  const BlockMeta& M = A.meta[slot];
  const double dt = A.st->dt_used;
  const int64_t fx = (int64_t)(G.n[0] + 1) * G.n[1] * G.n[2], fy = (int64_t)G.n[0] * (G.n[1] + 1) * G.n[2],
                fz = (int64_t)G.n[0] * G.n[1] * (G.n[2] + 1);
  double tmax = -INFINITY, ts[NVAR] = {0, 0, 0, 0, 0};
  double smax[3] = {-INFINITY, -INFINITY, -INFINITY};  // max over this thread's cells of |v_d| + c
  // x / dx == x * (1/dx) bit for bit when dx is a power of two (both are exact scalings): the IEEE
  // division (a ~20-instruction sequence) becomes one multiply, the result unchanged (A40 holds)
  bool p2[3];
#pragma unroll
  for (int d = 0; d < 3; ++d)
    p2[d] = (__double_as_longlong(M.dx[d]) & 0xFFFFFFFFFFFFFll) == 0 && M.idx[d] * M.dx[d] == 1.0;
  for (int c = threadIdx.x; c < G.n[0] * G.n[1]; c += blockDim.x) {
    const int j = c / G.n[0], i = c % G.n[0];
    const int64_t cell = (int64_t)slot * G.bstride + ((int64_t)(k + G.g) * G.N[1] + (j + G.g)) * G.N[0] + (i + G.g);
    const int64_t ix = ((int64_t)k * G.n[1] + j) * (G.n[0] + 1) + i;
    const int64_t iy = ((int64_t)k * (G.n[1] + 1) + j) * G.n[0] + i;
    const int64_t iz = ((int64_t)k * G.n[1] + j) * G.n[0] + i;
    double un[NVAR];
    // every operand of the cell first (40 independent loads in flight per thread: the kernel is bound
    // by memory latency, not by its arithmetic), then the update in the oracle's order
    double xl[NVAR], xr[NVAR], yl[NVAR], yr[NVAR], zl[NVAR], zr[NVAR], ui[NVAR], u0[NVAR];
#pragma unroll
    for (int v = 0; v < NVAR; ++v) {
      const double* px = Fx + (int64_t)slot * NVAR * fx + v * fx + ix;
      const double* py = Fy + (int64_t)slot * NVAR * fy + v * fy + iy;
      const double* pz = Fz + (int64_t)slot * NVAR * fz + v * fz + iz;
      xl[v] = __ldg(px);
      xr[v] = __ldg(px + 1);
      yl[v] = __ldg(py);
      yr[v] = __ldg(py + G.n[0]);
      zl[v] = __ldg(pz);
      zr[v] = __ldg(pz + (int64_t)G.n[0] * G.n[1]);
      ui[v] = A.Uin[cell + v * G.vstride];
      u0[v] = USE_U0 ? A.U0[cell + v * G.vstride] : 0.0;
    }
#pragma unroll
    for (int v = 0; v < NVAR; ++v) {
      const double f1 = __dsub_rn(xr[v], xl[v]), f2 = __dsub_rn(yr[v], yl[v]), f3 = __dsub_rn(zr[v], zl[v]);
      const double d1 = p2[0] ? __dmul_rn(f1, M.idx[0]) : __ddiv_rn(f1, M.dx[0]);
      const double d2 = p2[1] ? __dmul_rn(f2, M.idx[1]) : __ddiv_rn(f2, M.dx[1]);
      const double d3 = p2[2] ? __dmul_rn(f3, M.idx[2]) : __ddiv_rn(f3, M.dx[2]);
      const double L = -__dadd_rn(__dadd_rn(d1, d2), d3);
      const double dtw = __dmul_rn(A.cdt, dt);
      const double uin = ui[v];
      double out;
      if (USE_U0 && A.b1 != 0.0)  // RK2 stage 2: 0.5 U0 + 0.5 (U1 + dt L)
        out = __dadd_rn(__dmul_rn(0.5, u0[v]), __dmul_rn(0.5, __dadd_rn(uin, __dmul_rn(dt, L))));
      else if (USE_U0)            // VL2 stage 2: U0 + dt L
        out = __dadd_rn(u0[v], __dmul_rn(dtw, L));
      else                        // stage 1: U0 + w dt L
        out = __dadd_rn(uin, __dmul_rn(dtw, L));
      un[v] = out;
      A.Uout[cell + v * G.vstride] = out;
    }
    double Wn[NVAR];
    if (REDUCE || Wout) {
      // the primitives of the new state (prim_kernel's exact arithmetic): the next stage's W interior
      // (its ghosts come from exchanging W: bit-identical to converting exchanged U, reading A49);
      // an invalid cell is reported for the stage that converts it next, as prim_kernel would
      if (!cons2prim_rn(un[0], un[1], un[2], un[3], un[4], G.gm1, Wn) && Wout)
        set_error(A.err, A.stage == 1 ? 2 : 1, M.gid, k, j, i);
      if (Wout) {
#pragma unroll
        for (int v = 0; v < NVAR; ++v) Wout[cell + v * G.vstride] = Wn[v];
      }
    }
    if (REDUCE) {
      // exact CFL term, kept as -min(...) in the 'max' slot (finalize: dt = cfl * (-m), G.exact)
      const double cs = __dsqrt_rn(__ddiv_rn(__dmul_rn(G.gamma, Wn[4]), Wn[0]));
#pragma unroll
      for (int d = 0; d < 3; ++d) smax[d] = fmax(smax[d], __dadd_rn(fabs(Wn[1 + d]), cs));
#pragma unroll
      for (int v = 0; v < NVAR; ++v) ts[v] += un[v];
    }
  }
  if (REDUCE) {
    // the oracle's min over cells of min_d RN(dx_d / s_d) (cfl_term_rn) == min_d RN(dx_d / max s_d): s ->
    // RN(dx / s) is non-increasing, so the divisions move out of the cell loop (3 per thread instead of
    // 3 per cell), the result bit-identical (A40); NaN speeds (a failed cell, flagged) are skipped by fmax
    if (smax[0] > -INFINITY || smax[1] > -INFINITY || smax[2] > -INFINITY) {
      double r = INFINITY;
#pragma unroll
      for (int d = 0; d < 3; ++d)
        if (smax[d] > -INFINITY) {
          const double rd = __ddiv_rn(M.dx[d], smax[d]);
          r = rd < r ? rd : r;
        }
      tmax = -r;
    }
    __shared__ double red[32][6];
    for (int off = 16; off > 0; off >>= 1) {
      tmax = fmax(tmax, __shfl_xor_sync(0xffffffffu, tmax, off));
#pragma unroll
      for (int v = 0; v < NVAR; ++v) ts[v] += __shfl_xor_sync(0xffffffffu, ts[v], off);
    }
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (lane == 0) {
      red[warp][0] = tmax;
      for (int v = 0; v < NVAR; ++v) red[warp][1 + v] = ts[v];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double m = -INFINITY, s[NVAR] = {0, 0, 0, 0, 0};
      for (int w = 0; w < (int)blockDim.x / 32; ++w) {
        m = fmax(m, red[w][0]);
        for (int v = 0; v < NVAR; ++v) s[v] += red[w][1 + v];
      }
      double* o = A.partials + (int64_t)(A.cta_base + blockIdx.x) * 6;
      o[0] = m;
      for (int v = 0; v < NVAR; ++v) o[1 + v] = s[v] * M.dV;
    }
  }
}


// ------------------------------------------------------------------------------ AMR (O9)
// Refinement indicator eps_B = max over interior cells of |grad p| / p with central differences
// (A14).  Written with explicitly rounded ops in the oracle's order so that the flags match it.
__device__ __forceinline__ double pressure_rn(const double* u, int64_t vs, double gm1) {
  double rho = u[0];
  double ir = __ddiv_rn(1.0, rho);
  double m1 = u[vs], m2 = u[2 * vs], m3 = u[3 * vs];
  double v1 = __dmul_rn(m1, ir), v2 = __dmul_rn(m2, ir), v3 = __dmul_rn(m3, ir);
  double ke = __dmul_rn(0.5, __dadd_rn(__dadd_rn(__dmul_rn(m1, v1), __dmul_rn(m2, v2)), __dmul_rn(m3, v3)));
  return __dmul_rn(gm1, __dsub_rn(u[4 * vs], ke));
}

// dt / totals of the flux-corrected face layers of coarse blocks (static multilevel meshes), run after
// the reflux: one CTA per (slot, face) pair; a cell on several corrected layers is counted by its
// lowest corrected face only.  Fast-path arithmetic of the stage kernel's reduction.
__global__ void __launch_bounds__(256) rfx_reduce_kernel(const int2* faces, const double* U, const BlockMeta* meta,
                                                         double* partials, ErrWord* err, Geom G) {
  const int2 sf = faces[blockIdx.x];
  const int slot = sf.x, f = sf.y, d = f >> 1;
  const BlockMeta& M = meta[slot];
  const int ta = (d == 0) ? 1 : 0, tb = (d == 2) ? 1 : 2;
  const int na = G.n[ta], nb = G.n[tb];
  double tmax = 0.0, ts[NVAR] = {0, 0, 0, 0, 0};
  for (int t = threadIdx.x; t < na * nb; t += blockDim.x) {
    int cc[3];
    cc[d] = (f & 1) ? G.n[d] - 1 : 0;
    cc[ta] = t % na;
    cc[tb] = t / na;
    bool dup = false;
    for (int e = 0; e < f; ++e)
      if (((M.rfx >> e) & 1) && cc[e >> 1] == ((e & 1) ? G.n[e >> 1] - 1 : 0)) dup = true;
    if (dup) continue;
    const double* u = U + (int64_t)slot * G.bstride + ((int64_t)(cc[2] + G.g) * G.N[1] + (cc[1] + G.g)) * G.N[0] +
                      (cc[0] + G.g);
    double un[NVAR];
#pragma unroll
    for (int v = 0; v < NVAR; ++v) un[v] = u[v * G.vstride];
    const double ir = rcp_nr(un[0]);
    const double v1 = un[1] * ir, v2 = un[2] * ir, v3 = un[3] * ir;
    const double ke = 0.5 * ((un[1] * v1 + un[2] * v2) + un[3] * v3);
    const double p = G.gm1 * (un[4] - ke);
    if (!(un[0] > 0.0) || !(p > 0.0)) set_error(err, 0, M.gid, cc[2], cc[1], cc[0]);
    const double cs = sound_speed(un[0], p, G.gamma);
    const double s1 = (fabs(v1) + cs) * M.idx[0], s2 = (fabs(v2) + cs) * M.idx[1], s3 = (fabs(v3) + cs) * M.idx[2];
    tmax = dmax(tmax, dmax(s1, dmax(s2, s3)));
#pragma unroll
    for (int v = 0; v < NVAR; ++v) ts[v] += un[v];
  }
  __shared__ double red[8][6];
  for (int off = 16; off > 0; off >>= 1) {
    tmax = fmax(tmax, __shfl_xor_sync(0xffffffffu, tmax, off));
#pragma unroll
    for (int v = 0; v < NVAR; ++v) ts[v] += __shfl_xor_sync(0xffffffffu, ts[v], off);
  }
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane == 0) {
    red[warp][0] = tmax;
    for (int v = 0; v < NVAR; ++v) red[warp][1 + v] = ts[v];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0, s[NVAR] = {0, 0, 0, 0, 0};
    for (int w = 0; w < 8; ++w) {
      m = fmax(m, red[w][0]);
      for (int v = 0; v < NVAR; ++v) s[v] += red[w][1 + v];
    }
    double* o = partials + (int64_t)blockIdx.x * 6;
    o[0] = m;
    for (int v = 0; v < NVAR; ++v) o[1 + v] = s[v] * M.dV;
  }
}

cudaError_t launch_rfx_reduce(const int2* faces, int nfaces, const double* U, const BlockMeta* meta, double* partials,
                              ErrWord* err, const Geom& G, cudaStream_t s) {
  if (nfaces <= 0) return cudaSuccess;
  rfx_reduce_kernel<<<nfaces, 256, 0, s>>>(faces, U, meta, partials, err, G);
  return cudaGetLastError();
}

// AMR indicator (O9, A14): eps_B = max over the block of |grad p| / p with central differences, in
// the oracle's exact operation order (flags must be bit-exact).  One CTA = a 32x8 tile of (i,j)
// columns marching up the block; the pressure of every cell is computed once into a 3-plane smem
// ring with a plus-shaped halo of 1 (x/y neighbours) -- the z neighbours come from the ring.
constexpr int TGX = 32, TGY = 8, TGT = TGX * TGY, TGW = TGX + 2, TGP = (TGY + 2) * TGW;
__global__ void __launch_bounds__(TGT, 4) tag_kernel(const double* U, const BlockMeta* meta, unsigned long long* eps_bits,
                                                  double* partials, ErrWord* err, Geom G) {
  __shared__ double sp[3][TGP];
  __shared__ double red[TGT / 32][6];
  double tmax = 0.0, ts[NVAR] = {0, 0, 0, 0, 0};  // dt / totals partials of this tile (a6, a10)
  const int ntx = (G.n[0] + TGX - 1) / TGX, nty = (G.n[1] + TGY - 1) / TGY;
  int b = blockIdx.x;
  const int txi = b % ntx;
  b /= ntx;
  const int tyi = b % nty;
  const int slot = b / nty;
  const int x0 = txi * TGX, y0 = tyi * TGY;
  const int nxt = min(TGX, G.n[0] - x0), nyt = min(TGY, G.n[1] - y0);
  const BlockMeta& M = meta[slot];
  const int64_t vs = G.vstride;
  const int tid = threadIdx.x, tx = tid % TGX, ty = tid / TGX;
  // cell (i,j,q) of this block, or -- direct halo -- of the same-level face neighbour it lies in
  // (the plus-shaped stencil has at most one coordinate outside the block)
  auto at = [&](int i, int j, int q) -> const double* {
    int b = slot;
    if (i < 0 && M.nb[0] >= 0) { b = M.nb[0]; i += G.n[0]; }
    else if (i >= G.n[0] && M.nb[1] >= 0) { b = M.nb[1]; i -= G.n[0]; }
    else if (j < 0 && M.nb[2] >= 0) { b = M.nb[2]; j += G.n[1]; }
    else if (j >= G.n[1] && M.nb[3] >= 0) { b = M.nb[3]; j -= G.n[1]; }
    else if (q < 0 && M.nb[4] >= 0) { b = M.nb[4]; q += G.n[2]; }
    else if (q >= G.n[2] && M.nb[5] >= 0) { b = M.nb[5]; q -= G.n[2]; }
    return U + (int64_t)b * G.bstride + ((int64_t)(q + G.g) * G.N[1] + (j + G.g)) * G.N[0] + (i + G.g);
  };
  const bool own = tx < nxt && ty < nyt;
  double mx = 0.0;
  // plane loads are prefetched one plane ahead (2 cells per thread of the plus-shaped tile plane)
  constexpr int NS = (TGP + TGT - 1) / TGT;
  double uq[NS][NVAR];
  auto need_cell = [&](int c, int q, int& i, int& j) -> bool {
    j = c / TGW - 1;
    i = c % TGW - 1;
    if (c >= TGP) return false;
    const bool xin = i >= 0 && i < nxt, yin = j >= 0 && j < nyt;
    // the z ghost planes (q = -1, n3) only at the tile's own columns
    return (q < 0 || q >= G.n[2]) ? (xin && yin) : ((xin && j >= -1 && j <= nyt) || (yin && i >= -1 && i <= nxt));
  };
  auto load_plane = [&](int q) {
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      int i, j;
      if (need_cell(tid + s * TGT, q, i, j)) {
        const double* u = at(x0 + i, y0 + j, q);
#pragma unroll
        for (int v = 0; v < NVAR; ++v) uq[s][v] = u[v * vs];
      }
    }
  };
  load_plane(-1);
  for (int q = -1; q <= G.n[2]; ++q) {
    double* P = sp[(q + 3) % 3];
    // pressures of plane q over the tile and its plus-shaped halo, in the oracle's exact order
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      int i, j;
      const int c = tid + s * TGT;
      if (!need_cell(c, q, i, j)) continue;
      const double* un = uq[s];
      // one cons -> prim per cell (the stage kernels' MUFU-seeded arithmetic, A31): the pressure feeds
      // the indicator (reading A46) and, for the tile's own cells, the dt / totals partials
      const double fr = rcp_nr(un[0]);
      const double w1 = un[1] * fr, w2 = un[2] * fr, w3 = un[3] * fr;
      const double fke = 0.5 * ((un[1] * w1 + un[2] * w2) + un[3] * w3);
      const double p = G.gm1 * (un[4] - fke);
      P[c] = p;
      if (partials && q >= 0 && q < G.n[2] && i >= 0 && i < nxt && j >= 0 && j < nyt) {
        if (!(un[0] > 0.0) || !(p > 0.0)) set_error(err, 0, M.gid, q, y0 + j, x0 + i);
        const double cs = sound_speed(un[0], p, G.gamma);
        const double s1 = (fabs(w1) + cs) * M.idx[0], s2 = (fabs(w2) + cs) * M.idx[1], s3 = (fabs(w3) + cs) * M.idx[2];
        tmax = dmax(tmax, dmax(s1, dmax(s2, s3)));
#pragma unroll
        for (int v = 0; v < NVAR; ++v) ts[v] += un[v];
      }
    }
    if (q < G.n[2]) load_plane(q + 1);
    ph_jitter(q + 7);
    __syncthreads();
    const int c = q - 1;  // plane whose indicator is complete now
    if (c >= 0 && own) {
      const double* Pm = sp[(c + 2) % 3];
      const double* P0 = sp[(c + 3) % 3];
      const double* Pp = sp[(c + 4) % 3];
      const int o = (ty + 1) * TGW + (tx + 1);
      const double g1 = 0.5 * (P0[o + 1] - P0[o - 1]);
      const double g2 = 0.5 * (P0[o + TGW] - P0[o - TGW]);
      const double g3 = 0.5 * (Pp[o] - Pm[o]);
      const double s = (g1 * g1 + g2 * g2) + g3 * g3;
      // sqrt(s) / p with MUFU-seeded rsqrt / rcp (a uniform region gives s = 0 exactly, eps = 0)
      const double e = s > 0.0 ? (s * rsqrt_nr(s)) * rcp_nr(P0[o]) : 0.0;
      mx = fmax(mx, e);
    }
    __syncthreads();
  }
  for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if ((threadIdx.x & 31) == 0) atomicMax(eps_bits + slot, (unsigned long long)__double_as_longlong(mx));
  if (partials) {  // deterministic: warp shuffles, then thread 0 in warp order
    for (int off = 16; off > 0; off >>= 1) {
      tmax = fmax(tmax, __shfl_xor_sync(0xffffffffu, tmax, off));
#pragma unroll
      for (int v = 0; v < NVAR; ++v) ts[v] += __shfl_xor_sync(0xffffffffu, ts[v], off);
    }
    const int warp = tid / 32, lane = tid % 32;
    if (lane == 0) {
      red[warp][0] = tmax;
      for (int v = 0; v < NVAR; ++v) red[warp][1 + v] = ts[v];
    }
    __syncthreads();
    if (tid == 0) {
      double m = 0.0, s[NVAR] = {0, 0, 0, 0, 0};
      for (int w = 0; w < TGT / 32; ++w) {
        m = fmax(m, red[w][0]);
        for (int v = 0; v < NVAR; ++v) s[v] += red[w][1 + v];
      }
      double* o = partials + (int64_t)blockIdx.x * 6;
      o[0] = m;
      for (int v = 0; v < NVAR; ++v) o[1 + v] = s[v] * M.dV;
    }
  }
}

int tag_ctas_per_block(const Geom& G) {
  if (tag2_applies(G)) return tag2_ctas_per_block(G);
  return ((G.n[0] + TGX - 1) / TGX) * ((G.n[1] + TGY - 1) / TGY);
}

// new pool <- old pool (see RemeshTask): same-level move, 8-child prolongation of a refined parent
// using the parent's valid ghosts for the slopes (A11), pairwise restriction of derefined
// siblings (A10) -- optionally through the migration buffers
__global__ void remesh_kernel(const RemeshTask* tasks, const double* Uold, double* Unew, const double* rbuf,
                              double* sbuf, Geom G) {
  const RemeshTask t = tasks[blockIdx.x];  // tasks on x: up to 2^31 - 1
  const int k = blockIdx.y;
  const bool oct = (t.kind == R_OCT || t.kind == R_OCTCOPY);
  const int e0 = oct ? G.nc[0] : G.n[0], e1 = oct ? G.nc[1] : G.n[1], e2 = oct ? G.nc[2] : G.n[2];
  if (k >= e2) return;
  const int64_t sj = G.N[0], sk = (int64_t)G.N[0] * G.N[1];
  const int64_t pstride = (int64_t)e0 * e1 * e2;  // packed var stride
  for (int c = threadIdx.x; c < e0 * e1; c += blockDim.x) {
    const int j = c / e0, i = c % e0;
    const int64_t pk = ((int64_t)k * e1 + j) * e0 + i;  // packed index
    // destination pointer (per var stride dvs)
    double* d;
    int64_t dvs;
    if (t.dst < 0) {
      d = sbuf + t.dst_off + pk;
      dvs = pstride;
    } else {
      const int oi = oct ? t.ch[0] * G.nc[0] : 0, oj = oct ? t.ch[1] * G.nc[1] : 0, ok = oct ? t.ch[2] * G.nc[2] : 0;
      d = Unew + (int64_t)t.dst * G.bstride + ((int64_t)(k + ok + G.g) * G.N[1] + (j + oj + G.g)) * G.N[0] + (i + oi + G.g);
      dvs = G.vstride;
    }
    if (t.kind == R_MOVE || t.kind == R_OCTCOPY) {
      const double* s;
      int64_t svs;
      if (t.src < 0) {
        s = rbuf + t.src_off + pk;
        svs = pstride;
      } else {
        s = Uold + (int64_t)t.src * G.bstride + ((int64_t)(k + G.g) * G.N[1] + (j + G.g)) * G.N[0] + (i + G.g);
        svs = G.vstride;
      }
#pragma unroll
      for (int v = 0; v < NVAR; ++v) d[v * dvs] = s[v * svs];
    } else if (t.kind == R_REFINE) {
      const double* base = (t.src < 0) ? rbuf + t.src_off : Uold + (int64_t)t.src * G.bstride;
      const int I = t.ch[0] * G.nc[0] + i / 2, J = t.ch[1] * G.nc[1] + j / 2, K = t.ch[2] * G.nc[2] + k / 2;
      const double* p = base + ((int64_t)(K + G.g) * G.N[1] + (J + G.g)) * G.N[0] + (I + G.g);
      const double s1 = (i & 1) ? 0.25 : -0.25, s2 = (j & 1) ? 0.25 : -0.25, s3 = (k & 1) ? 0.25 : -0.25;
#pragma unroll
      for (int v = 0; v < NVAR; ++v) {
        const double* q = p + v * G.vstride;
        const double c0 = q[0];
        const double a1 = minmod_i(c0 - q[-1], q[1] - c0);
        const double a2 = minmod_i(c0 - q[-sj], q[sj] - c0);
        const double a3 = minmod_i(c0 - q[-sk], q[sk] - c0);
        d[v * dvs] = __dadd_rn(__dadd_rn(__dadd_rn(c0, __dmul_rn(s1, a1)), __dmul_rn(s2, a2)), __dmul_rn(s3, a3));
      }
    } else {  // R_OCT: restrict the child's fine cells 2i..2i+1
      const double* p = Uold + (int64_t)t.src * G.bstride + ((int64_t)(2 * k + G.g) * G.N[1] + (2 * j + G.g)) * G.N[0] + (2 * i + G.g);
#pragma unroll
      for (int v = 0; v < NVAR; ++v) d[v * dvs] = mean8(p + v * G.vstride, sj, sk);
    }
  }
}

// ------------------------------------------------------------------------------ launchers
#define PH_CHECK_LAUNCH() cudaGetLastError()

template <int R, bool RD, bool U0, bool ML, bool FULL, bool HB = false, int TXv = TILE_X, int TYv = TILE_Y,
          bool EIN = false, bool PUT = false>
static cudaError_t launch_stage_t(int nblk_cta, const StageArgs& a, const Geom& G, cudaStream_t s) {
  const size_t sm = stage_smem_bytes_t<TXv, TYv>();
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(stage_kernel<R, RD, U0, ML, FULL, HB, TXv, TYv, EIN, PUT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    if (getenv("PH_DEBUG_ATTR")) {
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, stage_kernel<R, RD, U0, ML, FULL, HB, TXv, TYv, EIN, PUT>);
      fprintf(stderr, "stage_kernel<%d,%d,%d,%d,%d>: regs %d maxThreads %d static smem %zu local %zu dyn %zu (max dyn %d) NT %d\n",
              R, (int)RD, (int)U0, (int)ML, (int)FULL, fa.numRegs, fa.maxThreadsPerBlock, fa.sharedSizeBytes,
              fa.localSizeBytes, sm, fa.maxDynamicSharedSizeBytes, NT);
    }
    // shared-memory carveout hint (percent of the maximum); the rest of the 256 KB is L1
    if (const char* cv = getenv("PH_CARVEOUT")) {
      e = cudaFuncSetAttribute(stage_kernel<R, RD, U0, ML, FULL, HB, TXv, TYv, EIN, PUT>, cudaFuncAttributePreferredSharedMemoryCarveout,
                               atoi(cv));
      if (e != cudaSuccess) return e;
    }
    attr = true;
  }
  stage_kernel<R, RD, U0, ML, FULL, HB, TXv, TYv, EIN, PUT><<<nblk_cta, TXv * TYv, sm, s>>>(a, G);
  return cudaGetLastError();
}

template <int R, bool RD, bool U0>
static cudaError_t launch_stage_ml(bool ml, int n, const StageArgs& a, const Geom& G, cudaStream_t s) {
  // full-tile fast path (block extents multiples of the tile): minmod, uniform-level meshes
  int tx, ty;
  const bool full = stage_tile(G, R, ml, &tx, &ty);
  if (a.H && !full) return cudaErrorInvalidValue;  // the host enables H only where the full-tile path runs
  if (a.peer_rbuf && !full) return cudaErrorInvalidValue;  // the host fuses the put only on full tiles
  if (full && tx == 16 && a.H && stage2_applies(G, R, ml)) return launch_stage2(RD, U0, n, a, G, s);
  if (ml && full && tx == 16) return cudaErrorInvalidValue;  // 16 x 16 multilevel tiles exist only in stage2
  if (full && tx == 16) {
    if (a.peer_rbuf)
      return a.H ? launch_stage_t<0, RD, U0, false, true, true, 16, 16, false, true>(n, a, G, s)
                 : launch_stage_t<0, RD, U0, false, true, false, 16, 16, false, true>(n, a, G, s);
    if (a.H) return launch_stage_t<0, RD, U0, false, true, true, 16, 16>(n, a, G, s);
    return launch_stage_t<0, RD, U0, false, true, false, 16, 16>(n, a, G, s);
  }
  if (full && a.peer_rbuf)
    return a.H ? launch_stage_t<0, RD, U0, false, true, true, TILE_X, TILE_Y, false, true>(n, a, G, s)
               : launch_stage_t<0, RD, U0, false, true, false, TILE_X, TILE_Y, false, true>(n, a, G, s);
  if (full && a.H) return launch_stage_t<0, RD, U0, false, true, true>(n, a, G, s);
  if (full) return launch_stage_t<0, RD, U0, false, true>(n, a, G, s);
  // multilevel meshes whose blocks tile exactly: the bounds-check-free variant (no boundary-face
  // precompute and no H there: coarse-fine faces store fluxes for the reflux)
  if (ml && R == 0 && !G.wavespeed && G.n[0] % TILE_X == 0 && G.n[1] % TILE_Y == 0 && !getenv("PH_NO_ML_FULL"))
    return launch_stage_t<0, RD, U0, true, true>(n, a, G, s);
  if (G.wavespeed)  // Einfeldt wave speeds (A4 variant)
    return ml ? launch_stage_t<R, RD, U0, true, false, false, TILE_X, TILE_Y, true>(n, a, G, s)
              : launch_stage_t<R, RD, U0, false, false, false, TILE_X, TILE_Y, true>(n, a, G, s);
  return ml ? launch_stage_t<R, RD, U0, true, false>(n, a, G, s) : launch_stage_t<R, RD, U0, false, false>(n, a, G, s);
}

template <int R>
static cudaError_t launch_stage_r(bool reduce, bool use_u0, bool ml, int n, const StageArgs& a, const Geom& G,
                                  cudaStream_t s) {
  if (reduce) return use_u0 ? launch_stage_ml<R, true, true>(ml, n, a, G, s) : launch_stage_ml<R, true, false>(ml, n, a, G, s);
  return use_u0 ? launch_stage_ml<R, false, true>(ml, n, a, G, s) : launch_stage_ml<R, false, false>(ml, n, a, G, s);
}

cudaError_t launch_stage(int recon, bool reduce, bool use_u0, int nblk_cta, const StageArgs& a, const Geom& G,
                         cudaStream_t s) {
  const bool ml = a.fbuf != nullptr;
  if (recon == 0) return launch_stage_r<0>(reduce, use_u0, ml, nblk_cta, a, G, s);
  if (recon == 1) return launch_stage_r<1>(reduce, use_u0, ml, nblk_cta, a, G, s);
  if (recon == 2) return launch_stage_r<2>(reduce, use_u0, ml, nblk_cta, a, G, s);
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------------------ peer signal / wait
// Peer transport of the halo (one-sided over NVLink).  After the put kernel has stored this rank's
// boundary faces into its peers' receive buffers, signal publishes a new epoch into the flag slot
// for me of every peer in `mask` (system fence, then a system-scope release store).  wait spins
// (system-scope acquire) until every peer in `mask` has published that epoch into my flags.  Each
// rank runs the same sequence of exchanges, so the signal and wait counters advance in lockstep.
// A peer that never arrives ends the spin after ~35 s with the error word set (stage -2).
__global__ void peer_signal_kernel(unsigned long long* const* peer_flags, unsigned long long* ctr, int me,
                                   unsigned long long mask) {
  __shared__ unsigned long long e;
  if (threadIdx.x == 0) e = *ctr + 1;
  __syncthreads();
  const int p = threadIdx.x;
  if (p < 64 && ((mask >> p) & 1ull)) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peer_flags[p] + me), "l"(e) : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) *ctr = e;
}

__global__ void peer_wait_kernel(const unsigned long long* my_flags, unsigned long long* ctr, unsigned long long mask,
                                 ErrWord* err) {
  __shared__ unsigned long long e;
  if (threadIdx.x == 0) e = *ctr + 1;
  __syncthreads();
  const int p = threadIdx.x;
  if (p < 64 && ((mask >> p) & 1ull)) {
    const long long t0 = clock64();
    unsigned long long v = 0;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(my_flags + p) : "memory");
      if (v >= e) break;
      if (clock64() - t0 > (1ll << 36)) {
        if (atomicCAS(&err->flag, 0, 1) == 0) {
          err->stage = -2;
          err->gid = p;
          __threadfence();
        }
        break;
      }
      __nanosleep(32);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *ctr = e;
}

cudaError_t launch_peer_signal(unsigned long long* const* peer_flags, unsigned long long* ctr, int me,
                               unsigned long long mask, cudaStream_t s) {
  peer_signal_kernel<<<1, 64, 0, s>>>(peer_flags, ctr, me, mask);
  return cudaGetLastError();
}

cudaError_t launch_peer_wait(const unsigned long long* my_flags, unsigned long long* ctr, unsigned long long mask,
                             ErrWord* err, cudaStream_t s) {
  peer_wait_kernel<<<1, 64, 0, s>>>(my_flags, ctr, mask, err);
  return cudaGetLastError();
}

cudaError_t launch_xfill(int nchunks, const XArgs& a, const Geom& G, cudaStream_t s) {
  if (nchunks <= 0) return cudaSuccess;
  xfill_kernel<<<nchunks, XT, 0, s>>>(a, G);
  return PH_CHECK_LAUNCH();
}

static int max_quarter(const Geom& G) {
  int qa = G.n[1] / 2 * G.n[2] / 2;  // upper bound of face quarter cells over dirs
  int q2 = G.n[0] / 2 * G.n[2] / 2, q3 = G.n[0] / 2 * G.n[1] / 2;
  int q = qa > q2 ? qa : q2;
  return q > q3 ? q : q3;
}

cudaError_t launch_reflux(int ntasks, const RefluxTask* t, double* U, const BlockMeta* meta, const double* fbuf,
                          const double* rbuf, const CycleState* st, double w, const Geom& G, cudaStream_t s,
                          double* H, double hb1) {
  if (ntasks <= 0) return cudaSuccess;
  dim3 grid(ntasks, (max_quarter(G) + 127) / 128);
  reflux_kernel<<<grid, 128, 0, s>>>(t, U, meta, fbuf, rbuf, st, w, G, H, hb1);
  return PH_CHECK_LAUNCH();
}

cudaError_t launch_flux_pack(int ntasks, const FluxPackTask* t, const double* fbuf, double* sbuf, const Geom& G,
                             cudaStream_t s) {
  if (ntasks <= 0) return cudaSuccess;
  dim3 grid(ntasks, (max_quarter(G) + 127) / 128);
  flux_pack_kernel<<<grid, 128, 0, s>>>(t, fbuf, sbuf, G);
  return PH_CHECK_LAUNCH();
}

cudaError_t launch_pgen(double* U, const BlockMeta* meta, int nslots, const PgenArgs& P, const Geom& G,
                        cudaStream_t s) {
  if (nslots <= 0) return cudaSuccess;
  pgen_kernel<<<nslots * G.n[1] * G.n[2], 128, 0, s>>>(U, meta, nslots, P, G);
  return PH_CHECK_LAUNCH();
}

cudaError_t launch_reduce(const double* U, const BlockMeta* meta, int nslots, double* partials, ErrWord* err,
                          const Geom& G, cudaStream_t s) {
  if (nslots <= 0) return cudaSuccess;
  reduce_kernel<<<nslots * G.n[2], 256, 0, s>>>(U, meta, nslots, partials, 0, err, G);
  return PH_CHECK_LAUNCH();
}

cudaError_t launch_rank_reduce(const double* partials, int n, double* out, cudaStream_t s) {
  rank_reduce_kernel<<<1, 256, 0, s>>>(partials, n, out);
  return PH_CHECK_LAUNCH();
}

cudaError_t launch_finalize(const double* all, int nranks, CycleState* st, double* hist, int hist_cap, double cfl,
                            int mode, double* tot_out, int exact, cudaStream_t s) {
  finalize_kernel<<<1, 1, 0, s>>>(all, nranks, st, hist, hist_cap, cfl, mode, tot_out, exact);
  return PH_CHECK_LAUNCH();
}

cudaError_t launch_cycle_begin(CycleState* st, double tlim, int set_tlim, cudaStream_t s) {
  cycle_begin_kernel<<<1, 1, 0, s>>>(st, tlim, set_tlim);
  return PH_CHECK_LAUNCH();
}

cudaError_t launch_interior_copy(double* U, double* buf, int slot0, int nslots, int to_pool, const Geom& G,
                                 cudaStream_t s) {
  if (nslots <= 0) return cudaSuccess;
  interior_copy_kernel<<<nslots * NVAR * G.n[2] * G.n[1], 128, 0, s>>>(U, buf, slot0, to_pool, G);
  return PH_CHECK_LAUNCH();
}

template <int DIR, int R>
static void launch_holine(const double* W, double* F, int nslots, const Geom& G, cudaStream_t s) {
  const int64_t lines = (int64_t)G.n[DIR == 0 ? 1 : 0] * G.n[DIR == 2 ? 1 : 2] * nslots;
  // enough threads for ~4 resident CTAs of 128 per SM; split lines into segments only when short of that
  const int64_t want = 148LL * 4 * 128;
  int nseg = (int)std::min<int64_t>(G.n[DIR] + 1, std::max<int64_t>(1, (want + lines - 1) / lines));
  if (const char* e = getenv("PH_HO_NSEG")) nseg = std::max(1, std::min(G.n[DIR] + 1, atoi(e)));  // tests
  const int64_t threads = lines * nseg;
  const unsigned grid = (unsigned)((threads + 127) / 128);
  holine_kernel<DIR, R><<<grid, 128, 0, s>>>(W, F, nslots, nseg, G);
}

template <int DIR, int R>
static void launch_hoface(const double* W, double* F, int nslots, const Geom& G, cudaStream_t s) {
  const int grid = nslots * (G.n[2] + (DIR == 2));
  hoflux_kernel<DIR, R><<<grid, 128, 0, s>>>(W, F, G);
}

// Flux kernel per direction (ncu, 256^3 in 64^3 blocks, us per launch, per-face / line march):
//   PLM   x 530 / 1352   y 523 / 335   z 546 / 332
//   PPM   x 2561 / 2388  y 2572 / 1803 z 2577 / 1785
//   WENO  x 3795 / 4963  y 4036 / 4485 z 3975 / 4427
// The x march is slow for PLM (its lines run across rows: 32 rows per warp load and store), and
// WENO-Z shares nothing across faces while the march's window costs it occupancy, so those take the
// per-face kernel.  PH_HO_FACE=1 / PH_HO_LINE=1 force one kernel for every direction (A/B, tests).
template <int R>
static cudaError_t launch_hoflux_r(const double* W, double* Fx, double* Fy, double* Fz, int nslots, const Geom& G,
                                   cudaStream_t s) {
  const char* pf = getenv("PH_HO_FACE");
  const char* pl = getenv("PH_HO_LINE");
  const bool all_face = pf && pf[0] == '1', all_line = pl && pl[0] == '1';
  // x: PPM one cell per lane with the left state by shuffle (hofx_kernel: 0.80 ms vs 0.99 per face), the
  // per-face kernel for PLM (its slope is cheap) and WENO-Z (nothing to share between a cell's two faces);
  // the x march's lanes walk 32 rows (PPM 1.39 ms, r02_launches_ho_ppm.md)
  const bool line_x = all_line;
  const bool line_yz = all_line || (!all_face && R != 4);
  if (line_x) launch_holine<0, R>(W, Fx, nslots, G, s);
  else if (R == 3 && !all_face) hofx_kernel<3><<<nslots * G.n[2], 128, 0, s>>>(W, Fx, G);
  else launch_hoface<0, R>(W, Fx, nslots, G, s);
  if (line_yz) {
    launch_holine<1, R>(W, Fy, nslots, G, s);
    launch_holine<2, R>(W, Fz, nslots, G, s);
  } else {
    launch_hoface<1, R>(W, Fy, nslots, G, s);
    launch_hoface<2, R>(W, Fz, nslots, G, s);
  }
  return cudaGetLastError();
}

constexpr int HOU_T = 128;  // update kernel CTA (up to ~150 registers with the loads hoisted: 3 CTAs per SM)

cudaError_t launch_highorder_stage(int recon, bool reduce, bool use_u0, int nslots, const StageArgs& a, double* W,
                                   double* Fx, double* Fy, double* Fz, bool w_ready, bool w_out, const Geom& G,
                                   cudaStream_t s) {
  if (nslots <= 0) return cudaSuccess;
  if (!w_ready) prim_kernel<<<nslots * G.N[2], 256, 0, s>>>(a.Uin, W, a.meta, a.err, a.stage, G);
  cudaError_t e;
  switch (recon) {
    case 0: e = launch_hoflux_r<0>(W, Fx, Fy, Fz, nslots, G, s); break;
    case 1: e = launch_hoflux_r<1>(W, Fx, Fy, Fz, nslots, G, s); break;
    case 2: e = launch_hoflux_r<2>(W, Fx, Fy, Fz, nslots, G, s); break;
    case 3: e = launch_hoflux_r<3>(W, Fx, Fy, Fz, nslots, G, s); break;
    default: e = launch_hoflux_r<4>(W, Fx, Fy, Fz, nslots, G, s); break;
  }
  if (e != cudaSuccess) return e;
  const int grid = nslots * G.n[2];
  if (reduce) {
    if (use_u0) houpdate_kernel<true, true><<<grid, HOU_T, 0, s>>>(a, Fx, Fy, Fz, w_out ? W : nullptr, G);
    else houpdate_kernel<true, false><<<grid, HOU_T, 0, s>>>(a, Fx, Fy, Fz, w_out ? W : nullptr, G);
  } else {
    if (use_u0) houpdate_kernel<false, true><<<grid, HOU_T, 0, s>>>(a, Fx, Fy, Fz, w_out ? W : nullptr, G);
    else houpdate_kernel<false, false><<<grid, HOU_T, 0, s>>>(a, Fx, Fy, Fz, w_out ? W : nullptr, G);
  }
  return cudaGetLastError();
}

cudaError_t launch_tag(const double* U, const BlockMeta* meta, int nslots, unsigned long long* eps_bits,
                       double* partials, ErrWord* err, const Geom& G, cudaStream_t s) {
  if (nslots <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(eps_bits, 0, sizeof(unsigned long long) * nslots, s);
  if (e != cudaSuccess) return e;
  if (tag2_applies(G)) return launch_tag2(U, meta, nslots, eps_bits, partials, err, G, s);  // stage2.cu
  const int tiles = ((G.n[0] + TGX - 1) / TGX) * ((G.n[1] + TGY - 1) / TGY);
  tag_kernel<<<nslots * tiles, TGT, 0, s>>>(U, meta, eps_bits, partials, err, G);
  return cudaGetLastError();
}

cudaError_t launch_remesh(const RemeshTask* t, int ntasks, const double* Uold, double* Unew, const double* rbuf,
                          double* sbuf, const Geom& G, cudaStream_t s) {
  if (ntasks <= 0) return cudaSuccess;
  dim3 grid(ntasks, G.n[2]);
  remesh_kernel<<<grid, 128, 0, s>>>(t, Uold, Unew, rbuf, sbuf, G);
  return cudaGetLastError();
}

}  // namespace ph
