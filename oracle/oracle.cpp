/*
 * oracle.cpp -- plain, slow, obviously-correct CPU oracle of the Parthenon-hydro
 * per-cycle update.  TEST INFRASTRUCTURE ONLY (see oracle.h): only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  Shares no code with the CUDA path.
 *
 * Citation key: P:n = line n of PAPER.md (arXiv 2202.12309 LaTeX source);
 * S:n = line n of SPEC.md (used for interfaces only); O1..O10 and A1..A30 are
 * the algorithm steps and readings of SURVEY.md §8(c), restated in DESIGN.md.
 *
 * Build: g++ -O2 -ffp-contract=off -fopenmp -shared -fPIC (no -ffast-math).
 * Every formula below is written in the canonical operation order of §8(c) so
 * that rounding differences versus the GPU stay at the ulp level.
 */
#include "oracle.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

thread_local std::string g_err;
int fail(int code, const std::string& msg) { g_err = msg; return code; }

/* ---------------- logical locations ---------------- */
struct LL {
  int level;
  int64_t x[3];
};
bool operator<(const LL& a, const LL& b) {
  if (a.level != b.level) return a.level < b.level;
  for (int d = 2; d >= 0; --d)
    if (a.x[d] != b.x[d]) return a.x[d] < b.x[d];
  return false;
}
bool operator==(const LL& a, const LL& b) {
  return a.level == b.level && a.x[0] == b.x[0] && a.x[1] == b.x[1] && a.x[2] == b.x[2];
}
int64_t floordiv2(int64_t a) { return (a >= 0) ? a / 2 : -((-a + 1) / 2); }

struct Nbr {
  int64_t gid;
  int rank;
  int off[3];
  int dlevel;  /* neighbour level minus own level */
  int fine[2]; /* free-dim child indices (finer neighbours) */
};

struct Block {
  LL loc;
  int64_t gid = 0;
  int rank = 0;
  double bxmin[3], bxmax[3], dx[3];
  std::vector<double> U0, U1; /* [5][N3][N2][N1] with ghosts */
  std::vector<double> C;      /* coarse staging [5][nc3+2cg][nc2+2cg][nc1+2cg] */
  std::vector<double> F[3];   /* stored face fluxes (multilevel only) */
  std::vector<Nbr> nbrs;
  bool has_coarser = false;
};

/* ---------------- point physics ---------------- */

/* a2: conserved -> primitive.  ir = 1/rho; v = m*ir; ke = 0.5*((m1v1+m2v2)+m3v3); p = (g-1)(E-ke). */
int cons_to_prim(const double* U, double gamma, double* W) {
  double rho = U[0];
  if (!(rho > 0.0)) return 1;
  double ir = 1.0 / rho;
  double v1 = U[1] * ir, v2 = U[2] * ir, v3 = U[3] * ir;
  double ke = 0.5 * ((U[1] * v1 + U[2] * v2) + U[3] * v3);
  double p = (gamma - 1.0) * (U[4] - ke);
  W[0] = rho; W[1] = v1; W[2] = v2; W[3] = v3; W[4] = p;
  if (!(p > 0.0)) return 2;
  return 0;
}

void prim_to_cons(const double* W, double gamma, double* U) {
  double rho = W[0];
  U[0] = rho;
  U[1] = rho * W[1];
  U[2] = rho * W[2];
  U[3] = rho * W[3];
  U[4] = W[4] / (gamma - 1.0) + (0.5 * rho) * ((W[1] * W[1] + W[2] * W[2]) + W[3] * W[3]);
}

/* textbook minmod: sgn(a) min(|a|,|b|) if a, b have the same strict sign, else 0 */
double minmod(double a, double b) {
  if (a > 0.0 && b > 0.0) return (a < b) ? a : b;
  if (a < 0.0 && b < 0.0) return (a > b) ? a : b;
  return 0.0;
}

/* a3: limited slope of PLM (reading A3: minmod default, van Leer / MC selectable) */
double plm_slope(double qm, double q0, double qp, int recon) {
  double dl = q0 - qm, dr = qp - q0;
  bool same = (dl > 0.0 && dr > 0.0) || (dl < 0.0 && dr < 0.0);
  if (!same) return 0.0;
  if (recon == ORC_RECON_VANLEER) return 2.0 * dl * dr / (dl + dr);
  if (recon == ORC_RECON_MC) {
    double s = (dl > 0.0) ? 1.0 : -1.0;
    double a = 2.0 * std::fabs(dl), b = 2.0 * std::fabs(dr), c = 0.5 * std::fabs(dl + dr);
    double m = a < b ? a : b;
    m = m < c ? m : c;
    return s * m;
  }
  return minmod(dl, dr);
}

/* NEXT 3, reading A37: PPM of Colella & Woodward (1984) eqs. 1.6-1.10 on primitives.
 * q[0..4] = q_{i-2} .. q_{i+2}; returns the left-face (i-1/2) and right-face (i+1/2) values. */
double ppm_dm(double a, double b, double c) {
  /* limited centred slope: sgn(dq) min(|dq|, 2|b-a|, 2|c-b|) if b is not an extremum, else 0 */
  double dl = b - a, dr = c - b;
  bool same = (dl > 0.0 && dr > 0.0) || (dl < 0.0 && dr < 0.0);
  if (!same) return 0.0;
  double dq = 0.5 * (c - a);
  double m = std::fabs(dq);
  if (2.0 * std::fabs(dl) < m) m = 2.0 * std::fabs(dl);
  if (2.0 * std::fabs(dr) < m) m = 2.0 * std::fabs(dr);
  return dq > 0.0 ? m : -m;
}

void ppm_cell(const double* q, double* ql, double* qr) {
  double dm_m = ppm_dm(q[0], q[1], q[2]), dm_0 = ppm_dm(q[1], q[2], q[3]), dm_p = ppm_dm(q[2], q[3], q[4]);
  double L = q[1] + 0.5 * (q[2] - q[1]) - (dm_0 - dm_m) / 6.0; /* eq. 1.6 at i-1/2 */
  double R = q[2] + 0.5 * (q[3] - q[2]) - (dm_p - dm_0) / 6.0; /* eq. 1.6 at i+1/2 */
  double c = q[2];
  if ((R - c) * (c - L) <= 0.0) {
    L = c;
    R = c;                                                       /* eq. 1.10, local extremum */
  } else {
    double d = R - L, m6 = 6.0 * (c - 0.5 * (L + R));
    if (d * m6 > d * d) L = 3.0 * c - 2.0 * R;                   /* overshoot at the left */
    else if (-(d * d) > d * m6) R = 3.0 * c - 2.0 * L;           /* overshoot at the right */
  }
  *ql = L;
  *qr = R;
}

/* NEXT 3, reading A38: WENO-Z of Borges et al. (2008), 5th order, p = 2, eps = 1e-40, on
 * primitives.  Value at the right face of c from the stencil a, b, c, d, e. */
double wenoz_face(double a, double b, double c, double d, double e) {
  double t0 = a - 2.0 * b + c, u0 = a - 4.0 * b + 3.0 * c;
  double t1 = b - 2.0 * c + d, u1 = b - d;
  double t2 = c - 2.0 * d + e, u2 = 3.0 * c - 4.0 * d + e;
  double b0 = (13.0 / 12.0) * (t0 * t0) + 0.25 * (u0 * u0);
  double b1 = (13.0 / 12.0) * (t1 * t1) + 0.25 * (u1 * u1);
  double b2 = (13.0 / 12.0) * (t2 * t2) + 0.25 * (u2 * u2);
  double tau = std::fabs(b0 - b2);
  const double eps = 1e-40;
  double r0 = tau / (b0 + eps), r1 = tau / (b1 + eps), r2 = tau / (b2 + eps);
  double a0 = 0.1 * (1.0 + r0 * r0), a1 = 0.6 * (1.0 + r1 * r1), a2 = 0.3 * (1.0 + r2 * r2);
  double q0 = (2.0 * a - 7.0 * b + 11.0 * c) / 6.0;
  double q1 = (-b + 5.0 * c + 2.0 * d) / 6.0;
  double q2 = (2.0 * c + 5.0 * d - e) / 6.0;
  return ((a0 * q0 + a1 * q1) + a2 * q2) / ((a0 + a1) + a2);
}

/* face values of cell q[2] for the high-order reconstructions (q[0..4] = q_{i-2} .. q_{i+2}) */
void recon5(const double* q, int recon, double* ql, double* qr) {
  if (recon == ORC_RECON_PPM) {
    ppm_cell(q, ql, qr);
  } else {
    *qr = wenoz_face(q[0], q[1], q[2], q[3], q[4]);
    *ql = wenoz_face(q[4], q[3], q[2], q[1], q[0]);
  }
}

/* physical flux and conserved state of a face state in the normal frame (O5 a4) */
void phys(const double* W, double gamma, double* U, double* F) {
  double rho = W[0], u = W[1], v = W[2], w = W[3], p = W[4];
  double mu = rho * u;
  /* u^2 + (v^2 + w^2): the normal term first keeps axis-transposition symmetry bitwise
   * (x<->y: v1^2 + (v2^2 + v3^2) vs v2^2 + (v3^2 + v1^2) differ only by commutation) */
  double E = p / (gamma - 1.0) + (0.5 * rho) * (u * u + (v * v + w * w));
  U[0] = rho; U[1] = mu; U[2] = rho * v; U[3] = rho * w; U[4] = E;
  F[0] = mu; F[1] = mu * u + p; F[2] = mu * v; F[3] = mu * w; F[4] = (E + p) * u;
}

/* a4: HLLE in the clamped branch-free form (A4, A5) with Davis wave speeds, or Einfeldt's:
 * the Roe averages (weights sqrt(rho)) of velocity and total enthalpy H = (E + p) / rho give
 * c~^2 = (gamma - 1)(H~ - |v~|^2 / 2), and u~ -+ c~ join the min / max. */
void hlle(const double* WL, const double* WR, double gamma, double* F, int ws = ORC_WS_DAVIS) {
  double cl = std::sqrt(gamma * WL[4] / WL[0]);
  double cr = std::sqrt(gamma * WR[4] / WR[0]);
  double UL[5], FL[5], UR[5], FR[5];
  phys(WL, gamma, UL, FL);
  phys(WR, gamma, UR, FR);
  // Davis: S_L = min(u_L - c_L, u_R - c_R), S_R = max(u_L + c_L, u_R + c_R)
  double a = WL[1] - cl, b = WR[1] - cr;
  double sl = a < b ? a : b;
  a = WL[1] + cl;
  b = WR[1] + cr;
  double sr = a > b ? a : b;
  if (ws == ORC_WS_EINFELDT) {
    // Einfeldt: S_L = min(u_L - c_L, u~ - c~), S_R = max(u_R + c_R, u~ + c~)
    const double rl = std::sqrt(WL[0]), rr = std::sqrt(WR[0]);
    const double u = (rl * WL[1] + rr * WR[1]) / (rl + rr);
    const double v = (rl * WL[2] + rr * WR[2]) / (rl + rr);
    const double w = (rl * WL[3] + rr * WR[3]) / (rl + rr);
    const double hl = (UL[4] + WL[4]) / WL[0], hr = (UR[4] + WR[4]) / WR[0];
    const double h = (rl * hl + rr * hr) / (rl + rr);
    const double c = std::sqrt((gamma - 1.0) * (h - 0.5 * (u * u + (v * v + w * w))));
    a = WL[1] - cl;
    sl = a < u - c ? a : u - c;
    b = WR[1] + cr;
    sr = b > u + c ? b : u + c;
  }
  double bp = sr > 0.0 ? sr : 0.0;
  double bm = sl < 0.0 ? sl : 0.0;
  double inv = 1.0 / (bp - bm);
  double bb = bp * bm;
  for (int n = 0; n < 5; ++n) F[n] = ((bp * FL[n] - bm * FR[n]) + bb * (UR[n] - UL[n])) * inv;
}

/* A10: pairwise mean of the 8 children, (k,j,i) order */
double restrict8(const double* v) {
  return (((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]))) * 0.125;
}

/* A11: minmod-limited linear prolongation; out in (k,j,i) child order */
void prolong(double c, const double* cm, const double* cp, double* out) {
  double s[3];
  for (int d = 0; d < 3; ++d) s[d] = minmod(c - cm[d], cp[d] - c);
  for (int ck = 0; ck < 2; ++ck)
    for (int cj = 0; cj < 2; ++cj)
      for (int ci = 0; ci < 2; ++ci) {
        double s1 = ci ? 1.0 : -1.0, s2 = cj ? 1.0 : -1.0, s3 = ck ? 1.0 : -1.0;
        out[ck * 4 + cj * 2 + ci] = ((c + (s1 * 0.25) * s[0]) + (s2 * 0.25) * s[1]) + (s3 * 0.25) * s[2];
      }
}

double pairwise_sum(const double* a, int64_t n) {
  if (n <= 0) return 0.0;
  if (n == 1) return a[0];
  int64_t h = n / 2;
  return pairwise_sum(a, h) + pairwise_sum(a + h, n - h);
}

uint64_t morton(int level, const int64_t* x, int max_level) {
  uint64_t X[3];
  for (int d = 0; d < 3; ++d) X[d] = (uint64_t)x[d] << (max_level - level);
  uint64_t key = 0;
  for (int b = 0; b < 21; ++b)
    for (int d = 0; d < 3; ++d) key |= ((X[d] >> b) & 1ull) << (3 * b + d);
  return key;
}

}  // namespace

/* ================================= mesh ================================= */
struct orc_mesh {
  orc_config cfg;
  std::vector<double> regions;
  int64_t n[3];
  int g = 2, cg = 2;
  int64_t nc[3];
  int64_t N[3];   /* n + 2g */
  int64_t NC[3];  /* nc + 2cg */
  int64_t nrb[3];
  std::set<LL> leaves;
  std::vector<Block> blocks;
  std::map<LL, int64_t> gid_of;
  bool multilevel = false;
  double t = 0.0, dt = 0.0;
  int64_t cycle = 0;
  bool have_state = false;
  std::vector<std::array<double, 7>> hist;
  std::vector<int8_t> last_flags;
  std::vector<double> last_eps;
  int problem = -1;
  std::vector<double> pparams;

  bool periodic(int d) const { return cfg.bc_inner[d] == ORC_BC_PERIODIC; }
  int64_t nblk(int d, int level) const { return nrb[d] << level; }
  int64_t idx(int v, int64_t k, int64_t j, int64_t i) const {
    return ((v * N[2] + (k + g)) * N[1] + (j + g)) * N[0] + (i + g);
  }
  int64_t cidx(int v, int64_t k, int64_t j, int64_t i) const {
    return ((v * NC[2] + (k + cg)) * NC[1] + (j + cg)) * NC[0] + (i + cg);
  }
  int64_t fidx(int d, int v, int64_t k, int64_t j, int64_t i) const {
    int64_t e0 = n[0] + (d == 0), e1 = n[1] + (d == 1), e2 = n[2] + (d == 2);
    return ((v * e2 + k) * e1 + j) * e0 + i;
  }
  int64_t fsize(int d) const { return 5 * (n[0] + (d == 0)) * (n[1] + (d == 1)) * (n[2] + (d == 2)); }

  /* wrap a same-level location into the domain; false if it leaves a non-periodic edge */
  bool wrap(LL& l) const {
    for (int d = 0; d < 3; ++d) {
      int64_t nb = nblk(d, l.level);
      if (l.x[d] < 0 || l.x[d] >= nb) {
        if (!periodic(d)) return false;
        l.x[d] = ((l.x[d] % nb) + nb) % nb;
      }
    }
    return true;
  }
  /* 0: a leaf sits at l; -k: covered by a leaf k levels coarser (out); +1: refined (finer leaves) */
  int lookup(const std::set<LL>& lv, const LL& l, LL* out) const {
    if (lv.count(l)) { if (out) *out = l; return 0; }
    for (int m = l.level - 1; m >= 0; --m) {
      int s = l.level - m;
      LL p{m, {l.x[0] >> s, l.x[1] >> s, l.x[2] >> s}};
      if (lv.count(p)) { if (out) *out = p; return m - l.level; }
    }
    return 1;
  }
  static void refine(std::set<LL>& lv, const LL& p) {
    lv.erase(p);
    for (int c = 0; c < 8; ++c)
      lv.insert(LL{p.level + 1, {2 * p.x[0] + (c & 1), 2 * p.x[1] + ((c >> 1) & 1), 2 * p.x[2] + ((c >> 2) & 1)}});
  }
  /* O1: refine-only 2:1 closure over faces, edges and corners (A15) */
  void balance(std::set<LL>& lv) const {
    for (;;) {
      std::set<LL> todo;
      for (const LL& l : lv) {
        if (l.level < 2) continue;
        for (int o3 = -1; o3 <= 1; ++o3)
          for (int o2 = -1; o2 <= 1; ++o2)
            for (int o1 = -1; o1 <= 1; ++o1) {
              if (!o1 && !o2 && !o3) continue;
              LL q{l.level, {l.x[0] + o1, l.x[1] + o2, l.x[2] + o3}};
              if (!wrap(q)) continue;
              LL c;
              if (lookup(lv, q, &c) < -1) todo.insert(c);
            }
      }
      if (todo.empty()) return;
      for (const LL& c : todo) refine(lv, c);
    }
  }
  void box(const LL& l, double* bmin, double* bmax) const {
    for (int d = 0; d < 3; ++d) {
      double w = (cfg.xmax[d] - cfg.xmin[d]) / (double)nblk(d, l.level);
      bmin[d] = cfg.xmin[d] + (double)l.x[d] * w;
      bmax[d] = cfg.xmin[d] + (double)(l.x[d] + 1) * w;
    }
  }
  /* O2 + O3: rebuild block list (Morton order = gid), partition and neighbour lists */
  void rebuild_blocks(std::vector<Block>& out) {
    std::vector<std::pair<uint64_t, LL>> keyed;
    for (const LL& l : leaves) keyed.push_back({morton(l.level, l.x, cfg.max_level), l});
    std::sort(keyed.begin(), keyed.end(), [](const std::pair<uint64_t, LL>& a, const std::pair<uint64_t, LL>& b) {
      return a.first < b.first;
    });
    int64_t nb = (int64_t)keyed.size();
    out.clear();
    out.resize(nb);
    gid_of.clear();
    multilevel = false;
    for (int64_t gid = 0; gid < nb; ++gid) {
      Block& b = out[gid];
      b.loc = keyed[gid].second;
      b.gid = gid;
      gid_of[b.loc] = gid;
      if (b.loc.level != keyed[0].second.level) multilevel = true;
    }
    int R = cfg.nranks > 0 ? cfg.nranks : 1;
    for (int r = 0; r < R; ++r) {
      int64_t lo, hi;
      orc_partition(nb, R, r, &lo, &hi);
      for (int64_t gid = lo; gid < hi; ++gid) out[gid].rank = r;
    }
    for (Block& b : out) {
      box(b.loc, b.bxmin, b.bxmax);
      for (int d = 0; d < 3; ++d) {
        double w = (cfg.xmax[d] - cfg.xmin[d]) / (double)nblk(d, b.loc.level);
        b.dx[d] = w / (double)n[d];
      }
      b.nbrs.clear();
      b.has_coarser = false;
      for (int o3 = -1; o3 <= 1; ++o3)
        for (int o2 = -1; o2 <= 1; ++o2)
          for (int o1 = -1; o1 <= 1; ++o1) {
            if (!o1 && !o2 && !o3) continue;
            int o[3] = {o1, o2, o3};
            LL q{b.loc.level, {b.loc.x[0] + o1, b.loc.x[1] + o2, b.loc.x[2] + o3}};
            if (!wrap(q)) continue;
            LL c;
            int r = lookup(leaves, q, &c);
            if (r == 0 || r == -1) {
              Nbr e;
              e.gid = gid_of.at(c);
              e.rank = 0;
              for (int d = 0; d < 3; ++d) e.off[d] = o[d];
              e.dlevel = r;
              e.fine[0] = e.fine[1] = 0;
              b.nbrs.push_back(e);
              if (r == -1) b.has_coarser = true;
            } else if (r > 0) {
              int fixed[3], nfree = 0, freed[3];
              for (int d = 0; d < 3; ++d) {
                fixed[d] = (o[d] == 1) ? 0 : 1;
                if (o[d] == 0) freed[nfree++] = d;
              }
              int cnt = 1 << nfree;
              /* free dims: highest dim outermost, lowest innermost */
              for (int cc = 0; cc < cnt; ++cc) {
                int ch[3] = {fixed[0], fixed[1], fixed[2]};
                int fi[2] = {0, 0};
                for (int f = 0; f < nfree; ++f) {
                  int bit = (cc >> f) & 1;
                  ch[freed[f]] = bit;
                  fi[f] = bit;
                }
                LL fl{q.level + 1, {2 * q.x[0] + ch[0], 2 * q.x[1] + ch[1], 2 * q.x[2] + ch[2]}};
                Nbr e;
                auto it = gid_of.find(fl);
                e.gid = (it == gid_of.end()) ? -1 : it->second; /* -1 would mean a 2:1 violation */
                e.rank = 0;
                for (int d = 0; d < 3; ++d) e.off[d] = o[d];
                e.dlevel = 1;
                e.fine[0] = fi[0];
                e.fine[1] = fi[1];
                b.nbrs.push_back(e);
              }
            } else {
              /* two or more levels coarser: a 2:1 violation; record nothing (caught by tests) */
            }
          }
    }
    for (Block& b : out)
      for (Nbr& e : b.nbrs) e.rank = (e.gid >= 0) ? out[e.gid].rank : -1;
  }
  bool allocated = false;
  void ensure_alloc() {
    if (allocated) return;
    for (Block& b : blocks) alloc_block(b);
    allocated = true;
  }
  void alloc_block(Block& b) {
    int64_t sz = 5 * N[0] * N[1] * N[2];
    b.U0.assign(sz, 0.0);
    b.U1.assign(sz, 0.0);
    if (b.has_coarser) b.C.assign(5 * NC[0] * NC[1] * NC[2], 0.0);
    else b.C.clear();
    for (int d = 0; d < 3; ++d) {
      if (multilevel) b.F[d].assign(fsize(d), 0.0);
      else b.F[d].clear();
    }
  }
};

namespace {

int nthreads_of(const orc_mesh* m) {
#ifdef _OPENMP
  return m->cfg.nthreads > 0 ? m->cfg.nthreads : omp_get_max_threads();
#else
  (void)m;
  return 1;
#endif
}

/* ---------------- O4 problem generators (A20-A22) ---------------- */
void pgen_block(const orc_mesh* m, Block& b) {
  const double gamma = m->cfg.gamma;
  const double* pp = m->pparams.data();
  for (int64_t k = 0; k < m->n[2]; ++k)
    for (int64_t j = 0; j < m->n[1]; ++j)
      for (int64_t i = 0; i < m->n[0]; ++i) {
        double x = b.bxmin[0] + ((double)i + 0.5) * b.dx[0];
        double y = b.bxmin[1] + ((double)j + 0.5) * b.dx[1];
        double z = b.bxmin[2] + ((double)k + 0.5) * b.dx[2];
        double W[5], U[5];
        if (m->problem == ORC_PROB_LINEAR_WAVE) {
          double A = pp[0], k1 = pp[1], k2 = pp[2], k3 = pp[3];
          double L1 = m->cfg.xmax[0] - m->cfg.xmin[0], L2 = m->cfg.xmax[1] - m->cfg.xmin[1],
                 L3 = m->cfg.xmax[2] - m->cfg.xmin[2];
          double K1 = k1 / L1, K2 = k2 / L2, K3 = k3 / L3;
          double kn = std::sqrt((K1 * K1 + K2 * K2) + K3 * K3);
          double phi = 2.0 * M_PI * ((K1 * (x - m->cfg.xmin[0]) + K2 * (y - m->cfg.xmin[1])) + K3 * (z - m->cfg.xmin[2]));
          double s = std::sin(phi);
          double rho0 = 1.0, p0 = 1.0 / gamma, c0 = 1.0;
          W[0] = rho0 + A * s;
          double va = A * c0 * s;
          W[1] = va * (K1 / kn);
          W[2] = va * (K2 / kn);
          W[3] = va * (K3 / kn);
          W[4] = p0 + A * (c0 * c0) * s;
        } else if (m->problem == ORC_PROB_SOD) {
          double xs = pp[0];
          if (x < xs) { W[0] = 1.0; W[4] = 1.0; }
          else { W[0] = 0.125; W[4] = 0.1; }
          W[1] = W[2] = W[3] = 0.0;
        } else if (m->problem == ORC_PROB_KH) {
          /* Kelvin-Helmholtz (reading A36): dense (rho 2) slab |y' - 1/2| < 1/4 moving at
           * +1/2 in x through rho 1 at -1/2, p = 2.5, vy = A sin(4 pi x') (exp(-((y'-1/4)/s)^2) +
           * exp(-((y'-3/4)/s)^2)), x', y' the coordinates scaled to [0,1) */
          double A = pp[0], sig = pp[1];
          double xx = (x - m->cfg.xmin[0]) / (m->cfg.xmax[0] - m->cfg.xmin[0]);
          double yy = (y - m->cfg.xmin[1]) / (m->cfg.xmax[1] - m->cfg.xmin[1]);
          bool in = std::fabs(yy - 0.5) < 0.25;
          double e1 = (yy - 0.25) / sig, e2 = (yy - 0.75) / sig;
          W[0] = in ? 2.0 : 1.0;
          W[1] = in ? 0.5 : -0.5;
          W[2] = A * std::sin(4.0 * M_PI * xx) * (std::exp(-(e1 * e1)) + std::exp(-(e2 * e2)));
          W[3] = 0.0;
          W[4] = 2.5;
        } else {
          double pin = pp[0], pout = pp[1], r = pp[2];
          double dx = x - pp[3], dy = y - pp[4], dz = z - pp[5];
          W[0] = 1.0; W[1] = W[2] = W[3] = 0.0;
          W[4] = ((dx * dx + dy * dy) + dz * dz < r * r) ? pin : pout;
        }
        prim_to_cons(W, gamma, U);
        for (int v = 0; v < 5; ++v) b.U0[m->idx(v, k, j, i)] = U[v];
      }
}

/* ---------------- O7 ghost exchange, phases A-D (A9-A12) ---------------- */
typedef std::vector<double> Block::*Arr;

void bc_fine(const orc_mesh* m, Block& b, Arr arr) {
  std::vector<double>& U = b.*arr;
  const int64_t g = m->g;
  for (int d = 0; d < 3; ++d) {
    if (m->periodic(d)) continue;
    for (int side = 0; side < 2; ++side) {
      bool at = side == 0 ? (b.loc.x[d] == 0) : (b.loc.x[d] == m->nblk(d, b.loc.level) - 1);
      if (!at) continue;
      int bc = side == 0 ? m->cfg.bc_inner[d] : m->cfg.bc_outer[d];
      int e1 = (d + 1) % 3, e2 = (d + 2) % 3;
      for (int64_t a2 = -g; a2 < m->n[e2] + g; ++a2)
        for (int64_t a1 = -g; a1 < m->n[e1] + g; ++a1)
          for (int64_t mm = 0; mm < g; ++mm) {
            int64_t gi = side == 0 ? -1 - mm : m->n[d] + mm;
            int64_t si;
            if (bc == ORC_BC_REFLECT) si = side == 0 ? mm : m->n[d] - 1 - mm;
            else si = side == 0 ? 0 : m->n[d] - 1;
            int64_t cg_[3], cs[3];
            cg_[d] = gi; cs[d] = si;
            cg_[e1] = cs[e1] = a1;
            cg_[e2] = cs[e2] = a2;
            for (int v = 0; v < 5; ++v) {
              double val = U[m->idx(v, cs[2], cs[1], cs[0])];
              if (bc == ORC_BC_REFLECT && v == 1 + d) val = -val;
              U[m->idx(v, cg_[2], cg_[1], cg_[0])] = val;
            }
          }
    }
  }
}

void bc_coarse(const orc_mesh* m, Block& b) {
  const int64_t cg = m->cg;
  for (int d = 0; d < 3; ++d) {
    if (m->periodic(d)) continue;
    for (int side = 0; side < 2; ++side) {
      bool at = side == 0 ? (b.loc.x[d] == 0) : (b.loc.x[d] == m->nblk(d, b.loc.level) - 1);
      if (!at) continue;
      int bc = side == 0 ? m->cfg.bc_inner[d] : m->cfg.bc_outer[d];
      int e1 = (d + 1) % 3, e2 = (d + 2) % 3;
      for (int64_t a2 = -cg; a2 < m->nc[e2] + cg; ++a2)
        for (int64_t a1 = -cg; a1 < m->nc[e1] + cg; ++a1)
          for (int64_t mm = 0; mm < cg; ++mm) {
            int64_t gi = side == 0 ? -1 - mm : m->nc[d] + mm;
            int64_t si;
            if (bc == ORC_BC_REFLECT) si = side == 0 ? mm : m->nc[d] - 1 - mm;
            else si = side == 0 ? 0 : m->nc[d] - 1;
            int64_t cg_[3], cs[3];
            cg_[d] = gi; cs[d] = si;
            cg_[e1] = cs[e1] = a1;
            cg_[e2] = cs[e2] = a2;
            for (int v = 0; v < 5; ++v) {
              double val = b.C[m->cidx(v, cs[2], cs[1], cs[0])];
              if (bc == ORC_BC_REFLECT && v == 1 + d) val = -val;
              b.C[m->cidx(v, cg_[2], cg_[1], cg_[0])] = val;
            }
          }
    }
  }
}

/* restrict 2x2x2 fine cells of array U (block fine coords) starting at (fk,fj,fi) */
double restrict_at(const orc_mesh* m, const std::vector<double>& U, int v, int64_t fk, int64_t fj, int64_t fi) {
  double c[8];
  for (int a = 0; a < 2; ++a)
    for (int bb = 0; bb < 2; ++bb)
      for (int cc = 0; cc < 2; ++cc) c[a * 4 + bb * 2 + cc] = U[m->idx(v, fk + a, fj + bb, fi + cc)];
  return restrict8(c);
}

void phase_A(orc_mesh* m, Block& b, Arr arr) {
  std::vector<double>& U = b.*arr;
  const int64_t g = m->g;
  for (const Nbr& e : b.nbrs) {
    const Block& s = m->blocks[e.gid];
    const std::vector<double>& S = s.*arr;
    int64_t lo[3], hi[3];
    if (e.dlevel == 0) {
      int64_t so[3]; /* source index = dest index + so */
      for (int d = 0; d < 3; ++d) {
        if (e.off[d] < 0) { lo[d] = -g; hi[d] = 0; so[d] = m->n[d]; }
        else if (e.off[d] > 0) { lo[d] = m->n[d]; hi[d] = m->n[d] + g; so[d] = -m->n[d]; }
        else { lo[d] = 0; hi[d] = m->n[d]; so[d] = 0; }
      }
      for (int v = 0; v < 5; ++v)
        for (int64_t k = lo[2]; k < hi[2]; ++k)
          for (int64_t j = lo[1]; j < hi[1]; ++j)
            for (int64_t i = lo[0]; i < hi[0]; ++i)
              U[m->idx(v, k, j, i)] = S[m->idx(v, k + so[2], j + so[1], i + so[0])];
    } else if (e.dlevel == 1) {
      /* finer neighbour: restrict its cells covering my ghost box */
      int ch[3];
      int f = 0;
      for (int d = 0; d < 3; ++d) {
        if (e.off[d] != 0) ch[d] = (e.off[d] == 1) ? 0 : 1;
        else ch[d] = e.fine[f++];
      }
      int64_t sh[3];
      for (int d = 0; d < 3; ++d) {
        if (e.off[d] < 0) { lo[d] = -g; hi[d] = 0; }
        else if (e.off[d] > 0) { lo[d] = m->n[d]; hi[d] = m->n[d] + g; }
        else { lo[d] = ch[d] * m->n[d] / 2; hi[d] = (ch[d] + 1) * m->n[d] / 2; }
        sh[d] = (2 * e.off[d] + ch[d]) * m->n[d];
      }
      for (int v = 0; v < 5; ++v)
        for (int64_t k = lo[2]; k < hi[2]; ++k)
          for (int64_t j = lo[1]; j < hi[1]; ++j)
            for (int64_t i = lo[0]; i < hi[0]; ++i)
              U[m->idx(v, k, j, i)] = restrict_at(m, S, v, 2 * k - sh[2], 2 * j - sh[1], 2 * i - sh[0]);
    } else {
      /* coarser neighbour: copy its cells into my coarse staging */
      const int64_t cg = m->cg;
      int64_t so[3];
      for (int d = 0; d < 3; ++d) {
        if (e.off[d] < 0) { lo[d] = -cg; hi[d] = 0; }
        else if (e.off[d] > 0) { lo[d] = m->nc[d]; hi[d] = m->nc[d] + cg; }
        else { lo[d] = 0; hi[d] = m->nc[d]; }
        int64_t P = floordiv2(b.loc.x[d] + e.off[d]);
        so[d] = b.loc.x[d] * m->nc[d] - P * m->n[d];
      }
      for (int v = 0; v < 5; ++v)
        for (int64_t k = lo[2]; k < hi[2]; ++k)
          for (int64_t j = lo[1]; j < hi[1]; ++j)
            for (int64_t i = lo[0]; i < hi[0]; ++i)
              b.C[m->cidx(v, k, j, i)] = S[m->idx(v, k + so[2], j + so[1], i + so[0])];
    }
  }
}

/* classify each of the 27 offsets: -2 none (physical edge), -1 coarser, 0 same, 1 finer */
void offset_kinds(const Block& b, int kind[27]) {
  for (int q = 0; q < 27; ++q) kind[q] = -2;
  for (const Nbr& e : b.nbrs) {
    int q = (e.off[2] + 1) * 9 + (e.off[1] + 1) * 3 + (e.off[0] + 1);
    kind[q] = e.dlevel;
  }
}

void phase_B(orc_mesh* m, Block& b, Arr arr) {
  if (!b.has_coarser) return;
  const std::vector<double>& U = b.*arr;
  int kind[27];
  offset_kinds(b, kind);
  for (int v = 0; v < 5; ++v)
    for (int64_t k = 0; k < m->nc[2]; ++k)
      for (int64_t j = 0; j < m->nc[1]; ++j)
        for (int64_t i = 0; i < m->nc[0]; ++i) b.C[m->cidx(v, k, j, i)] = restrict_at(m, U, v, 2 * k, 2 * j, 2 * i);
  for (int o3 = -1; o3 <= 1; ++o3)
    for (int o2 = -1; o2 <= 1; ++o2)
      for (int o1 = -1; o1 <= 1; ++o1) {
        if (!o1 && !o2 && !o3) continue;
        int q = (o3 + 1) * 9 + (o2 + 1) * 3 + (o1 + 1);
        if (kind[q] == -2 || kind[q] == -1) continue;
        int o[3] = {o1, o2, o3};
        int64_t lo[3], hi[3];
        for (int d = 0; d < 3; ++d) {
          if (o[d] < 0) { lo[d] = -1; hi[d] = 0; }
          else if (o[d] > 0) { lo[d] = m->nc[d]; hi[d] = m->nc[d] + 1; }
          else { lo[d] = 0; hi[d] = m->nc[d]; }
        }
        for (int v = 0; v < 5; ++v)
          for (int64_t k = lo[2]; k < hi[2]; ++k)
            for (int64_t j = lo[1]; j < hi[1]; ++j)
              for (int64_t i = lo[0]; i < hi[0]; ++i)
                b.C[m->cidx(v, k, j, i)] = restrict_at(m, U, v, 2 * k, 2 * j, 2 * i);
      }
  bc_coarse(m, b);
}

void phase_C(orc_mesh* m, Block& b, Arr arr) {
  if (!b.has_coarser) return;
  std::vector<double>& U = b.*arr;
  int kind[27];
  offset_kinds(b, kind);
  for (int o3 = -1; o3 <= 1; ++o3)
    for (int o2 = -1; o2 <= 1; ++o2)
      for (int o1 = -1; o1 <= 1; ++o1) {
        if (!o1 && !o2 && !o3) continue;
        int q = (o3 + 1) * 9 + (o2 + 1) * 3 + (o1 + 1);
        if (kind[q] != -1) continue;
        int o[3] = {o1, o2, o3};
        int64_t lo[3], hi[3];
        for (int d = 0; d < 3; ++d) {
          if (o[d] < 0) { lo[d] = -1; hi[d] = 0; }
          else if (o[d] > 0) { lo[d] = m->nc[d]; hi[d] = m->nc[d] + 1; }
          else { lo[d] = 0; hi[d] = m->nc[d]; }
        }
        for (int v = 0; v < 5; ++v)
          for (int64_t k = lo[2]; k < hi[2]; ++k)
            for (int64_t j = lo[1]; j < hi[1]; ++j)
              for (int64_t i = lo[0]; i < hi[0]; ++i) {
                double c = b.C[m->cidx(v, k, j, i)];
                double cm[3] = {b.C[m->cidx(v, k, j, i - 1)], b.C[m->cidx(v, k, j - 1, i)], b.C[m->cidx(v, k - 1, j, i)]};
                double cp[3] = {b.C[m->cidx(v, k, j, i + 1)], b.C[m->cidx(v, k, j + 1, i)], b.C[m->cidx(v, k + 1, j, i)]};
                double out[8];
                prolong(c, cm, cp, out);
                for (int a = 0; a < 2; ++a)
                  for (int bb = 0; bb < 2; ++bb)
                    for (int cc = 0; cc < 2; ++cc)
                      U[m->idx(v, 2 * k + a, 2 * j + bb, 2 * i + cc)] = out[a * 4 + bb * 2 + cc];
              }
      }
}

void exchange(orc_mesh* m, Arr arr) {
  int64_t nb = (int64_t)m->blocks.size();
  int nt = nthreads_of(m);
#pragma omp parallel for num_threads(nt) schedule(dynamic)
  for (int64_t b = 0; b < nb; ++b) phase_A(m, m->blocks[b], arr);
#pragma omp parallel for num_threads(nt) schedule(dynamic)
  for (int64_t b = 0; b < nb; ++b) phase_B(m, m->blocks[b], arr);
#pragma omp parallel for num_threads(nt) schedule(dynamic)
  for (int64_t b = 0; b < nb; ++b) phase_C(m, m->blocks[b], arr);
#pragma omp parallel for num_threads(nt) schedule(dynamic)
  for (int64_t b = 0; b < nb; ++b) bc_fine(m, m->blocks[b], arr);
}

/* ---------------- O5 stage: prim, PLM, HLLE, divergence ---------------- */
struct Err {
  int code = 0;
  std::string msg;
};

/* fluxes of all faces of block b from array src, into F[3] (each sized fsize(d)) */
int compute_fluxes(const orc_mesh* m, const Block& b, const std::vector<double>& src, std::vector<double>& W,
                   std::vector<double>* F, std::string* msg) {
  const int64_t g = m->g;
  const double gamma = m->cfg.gamma;
  std::fill(W.begin(), W.end(), NAN);
  /* a2 on the interior plus the g-wide cross-shaped halo */
  for (int64_t k = -g; k < m->n[2] + g; ++k)
    for (int64_t j = -g; j < m->n[1] + g; ++j)
      for (int64_t i = -g; i < m->n[0] + g; ++i) {
        int out = (k < 0 || k >= m->n[2]) + (j < 0 || j >= m->n[1]) + (i < 0 || i >= m->n[0]);
        if (out > 1) continue;
        double U[5], w[5];
        for (int v = 0; v < 5; ++v) U[v] = src[m->idx(v, k, j, i)];
        int rc = cons_to_prim(U, gamma, w);
        if (rc) {
          char buf[256];
          snprintf(buf, sizeof buf, "non-positive %s at gid %lld cell (k,j,i)=(%lld,%lld,%lld)",
                   rc == 1 ? "density" : "pressure", (long long)b.gid, (long long)k, (long long)j, (long long)i);
          *msg = buf;
          return ORC_ERR_PHYSICS;
        }
        for (int v = 0; v < 5; ++v) W[m->idx(v, k, j, i)] = w[v];
      }
  for (int d = 0; d < 3; ++d) {
    int t1 = (d + 1) % 3, t2 = (d + 2) % 3;
    int64_t e[3] = {m->n[0], m->n[1], m->n[2]};
    e[d] += 1;
    for (int64_t k = 0; k < e[2]; ++k)
      for (int64_t j = 0; j < e[1]; ++j)
        for (int64_t i = 0; i < e[0]; ++i) {
          /* face between cell c-1 and c along d, c = (i,j,k) */
          int64_t c[3] = {i, j, k};
          double WL[5], WR[5];
          for (int v = 0; v < 5; ++v) {
            if (m->cfg.recon >= ORC_RECON_PPM) {
              /* 6 points c-3 .. c+2: cell c-1 uses q[0..4], cell c uses q[1..5] */
              double q[6], a, bb;
              for (int s = 0; s < 6; ++s) {
                int64_t cc[3] = {c[0], c[1], c[2]};
                cc[d] += s - 3;
                q[s] = W[m->idx(v, cc[2], cc[1], cc[0])];
              }
              recon5(q, m->cfg.recon, &a, &WL[v]);      /* right face of cell c-1 */
              recon5(q + 1, m->cfg.recon, &WR[v], &bb); /* left face of cell c */
              (void)a;
              (void)bb;
              continue;
            }
            double q[4];
            for (int s = 0; s < 4; ++s) {
              int64_t cc[3] = {c[0], c[1], c[2]};
              cc[d] += s - 2;
              q[s] = W[m->idx(v, cc[2], cc[1], cc[0])];
            }
            double DL = plm_slope(q[0], q[1], q[2], m->cfg.recon);
            double DR = plm_slope(q[1], q[2], q[3], m->cfg.recon);
            WL[v] = q[1] + 0.5 * DL; /* q^L_{i-1/2} from cell i-1 */
            WR[v] = q[2] - 0.5 * DR; /* q^R_{i-1/2} from cell i   */
          }
          if (!(WL[0] > 0.0) || !(WL[4] > 0.0) || !(WR[0] > 0.0) || !(WR[4] > 0.0)) {
            char buf[256];
            snprintf(buf, sizeof buf, "non-positive face state at gid %lld face dir %d (k,j,i)=(%lld,%lld,%lld)",
                     (long long)b.gid, d, (long long)k, (long long)j, (long long)i);
            *msg = buf;
            return ORC_ERR_PHYSICS;
          }
          double wl[5] = {WL[0], WL[1 + d], WL[1 + t1], WL[1 + t2], WL[4]};
          double wr[5] = {WR[0], WR[1 + d], WR[1 + t1], WR[1 + t2], WR[4]};
          double fn[5];
          hlle(wl, wr, gamma, fn, m->cfg.wavespeed);
          double fo[5];
          fo[0] = fn[0];
          fo[1 + d] = fn[1];
          fo[1 + t1] = fn[2];
          fo[1 + t2] = fn[3];
          fo[4] = fn[4];
          for (int v = 0; v < 5; ++v) F[d][m->fidx(d, v, k, j, i)] = fo[v];
        }
  }
  return 0;
}

/* O8: coarse face flux <- pairwise mean of the 4 fine face fluxes (A13) */
void flux_correct(orc_mesh* m, Block& b) {
  for (const Nbr& e : b.nbrs) {
    if (e.dlevel != 1) continue;
    int nz = (e.off[0] != 0) + (e.off[1] != 0) + (e.off[2] != 0);
    if (nz != 1) continue;
    int d = e.off[0] ? 0 : (e.off[1] ? 1 : 2);
    int side = e.off[d];
    const Block& f = m->blocks[e.gid];
    int t[2], nt = 0;
    for (int a = 0; a < 3; ++a)
      if (a != d) t[nt++] = a;
    int64_t cface = side < 0 ? 0 : m->n[d];
    int64_t fface = side < 0 ? m->n[d] : 0;
    int64_t lo0 = e.fine[0] * m->n[t[0]] / 2, lo1 = e.fine[1] * m->n[t[1]] / 2;
    for (int v = 0; v < 5; ++v)
      for (int64_t B = lo1; B < lo1 + m->n[t[1]] / 2; ++B)
        for (int64_t A = lo0; A < lo0 + m->n[t[0]] / 2; ++A) {
          double fv[2][2];
          for (int bb = 0; bb < 2; ++bb)
            for (int aa = 0; aa < 2; ++aa) {
              int64_t c[3];
              c[d] = fface;
              c[t[0]] = 2 * (A - lo0) + aa;
              c[t[1]] = 2 * (B - lo1) + bb;
              fv[aa][bb] = f.F[d][m->fidx(d, v, c[2], c[1], c[0])];
            }
          int64_t cc[3];
          cc[d] = cface;
          cc[t[0]] = A;
          cc[t[1]] = B;
          b.F[d][m->fidx(d, v, cc[2], cc[1], cc[0])] = ((fv[0][0] + fv[1][0]) + (fv[0][1] + fv[1][1])) * 0.25;
        }
  }
}

/* a5: L(U) and the RK stage combine.  mode 0: dst = base + w*dt*L (stage 1 RK2 w=1, VL2 w=0.5; VL2 stage 2 w=1)
 * mode 1 (RK2 stage 2): dst = 0.5*base + 0.5*(src + dt*L) */
void update(const orc_mesh* m, Block& b, const std::vector<double>* F, const std::vector<double>& base,
            const std::vector<double>& src, std::vector<double>& dst, double dtw, int mode) {
  for (int v = 0; v < 5; ++v)
    for (int64_t k = 0; k < m->n[2]; ++k)
      for (int64_t j = 0; j < m->n[1]; ++j)
        for (int64_t i = 0; i < m->n[0]; ++i) {
          double d1 = (F[0][m->fidx(0, v, k, j, i + 1)] - F[0][m->fidx(0, v, k, j, i)]) / b.dx[0];
          double d2 = (F[1][m->fidx(1, v, k, j + 1, i)] - F[1][m->fidx(1, v, k, j, i)]) / b.dx[1];
          double d3 = (F[2][m->fidx(2, v, k + 1, j, i)] - F[2][m->fidx(2, v, k, j, i)]) / b.dx[2];
          double L = -((d1 + d2) + d3);
          int64_t q = m->idx(v, k, j, i);
          if (mode == 0) dst[q] = base[q] + dtw * L;
          else dst[q] = 0.5 * base[q] + 0.5 * (src[q] + dtw * L);
        }
}

/* one stage over all blocks.  src holds valid ghosts. */
int stage(orc_mesh* m, Arr src, Arr dst, double dtw, int mode) {
  int64_t nb = (int64_t)m->blocks.size();
  int nt = nthreads_of(m);
  Err err;
  int64_t wsz = 5 * m->N[0] * m->N[1] * m->N[2];
  if (m->multilevel) {
#pragma omp parallel num_threads(nt)
    {
      std::vector<double> W(wsz);
#pragma omp for schedule(dynamic)
      for (int64_t b = 0; b < nb; ++b) {
        std::string msg;
        int rc = compute_fluxes(m, m->blocks[b], m->blocks[b].*src, W, m->blocks[b].F, &msg);
        if (rc) {
#pragma omp critical
          if (!err.code) { err.code = rc; err.msg = msg; }
        }
      }
    }
    if (err.code) return fail(err.code, err.msg);
    for (int64_t b = 0; b < nb; ++b) flux_correct(m, m->blocks[b]);
#pragma omp parallel for num_threads(nt) schedule(dynamic)
    for (int64_t b = 0; b < nb; ++b) {
      Block& B = m->blocks[b];
      update(m, B, B.F, B.U0, B.*src, B.*dst, dtw, mode);
    }
  } else {
#pragma omp parallel num_threads(nt)
    {
      std::vector<double> W(wsz);
      std::vector<double> F[3];
      for (int d = 0; d < 3; ++d) F[d].resize(m->fsize(d));
#pragma omp for schedule(dynamic)
      for (int64_t b = 0; b < nb; ++b) {
        Block& B = m->blocks[b];
        std::string msg;
        int rc = compute_fluxes(m, B, B.*src, W, F, &msg);
        if (rc) {
#pragma omp critical
          if (!err.code) { err.code = rc; err.msg = msg; }
          continue;
        }
        update(m, B, F, B.U0, B.*src, B.*dst, dtw, mode);
      }
    }
    if (err.code) return fail(err.code, err.msg);
  }
  return 0;
}

/* O6: dt = cfl * min over interior cells and dims of dx_d/(|v_d| + c) (A7) */
int compute_dt(orc_mesh* m, double* out) {
  int64_t nb = (int64_t)m->blocks.size();
  std::vector<double> bmin(nb, INFINITY);
  int nt = nthreads_of(m);
  Err err;
#pragma omp parallel for num_threads(nt) schedule(dynamic)
  for (int64_t b = 0; b < nb; ++b) {
    Block& B = m->blocks[b];
    double mn = INFINITY;
    for (int64_t k = 0; k < m->n[2]; ++k)
      for (int64_t j = 0; j < m->n[1]; ++j)
        for (int64_t i = 0; i < m->n[0]; ++i) {
          double U[5], W[5];
          for (int v = 0; v < 5; ++v) U[v] = B.U0[m->idx(v, k, j, i)];
          if (cons_to_prim(U, m->cfg.gamma, W)) {
#pragma omp critical
            if (!err.code) { err.code = ORC_ERR_PHYSICS; err.msg = "non-positive state in dt estimate"; }
            continue;
          }
          double c = std::sqrt(m->cfg.gamma * W[4] / W[0]);
          for (int d = 0; d < 3; ++d) {
            double r = B.dx[d] / (std::fabs(W[1 + d]) + c);
            if (r < mn) mn = r;
          }
        }
    bmin[b] = mn;
  }
  if (err.code) return fail(err.code, err.msg);
  double mn = INFINITY;
  for (double v : bmin) mn = v < mn ? v : mn;
  *out = m->cfg.cfl * mn;
  return 0;
}

/* O10: totals; per block pairwise over interior (k,j,i) order times dV, then pairwise over gids */
void totals(const orc_mesh* m, double out[5]) {
  int64_t nb = (int64_t)m->blocks.size();
  std::vector<double> part(5 * nb);
  int64_t ncell = m->n[0] * m->n[1] * m->n[2];
  for (int64_t b = 0; b < nb; ++b) {
    const Block& B = m->blocks[b];
    std::vector<double> tmp(ncell);
    double dV = (B.dx[0] * B.dx[1]) * B.dx[2];
    for (int v = 0; v < 5; ++v) {
      int64_t q = 0;
      for (int64_t k = 0; k < m->n[2]; ++k)
        for (int64_t j = 0; j < m->n[1]; ++j)
          for (int64_t i = 0; i < m->n[0]; ++i) tmp[q++] = B.U0[m->idx(v, k, j, i)];
      part[v * nb + b] = pairwise_sum(tmp.data(), ncell) * dV;
    }
  }
  for (int v = 0; v < 5; ++v) out[v] = pairwise_sum(&part[v * nb], nb);
}

/* ---------------- O9 tagging and remesh (A14, A16, A26) ---------------- */
int indicators(orc_mesh* m, std::vector<double>& eps) {
  int64_t nb = (int64_t)m->blocks.size();
  eps.assign(nb, 0.0);
  const int64_t g = m->g;
  for (int64_t b = 0; b < nb; ++b) {
    Block& B = m->blocks[b];
    std::vector<double> P(m->N[0] * m->N[1] * m->N[2], NAN);
    auto pidx = [&](int64_t k, int64_t j, int64_t i) { return ((k + g) * m->N[1] + (j + g)) * m->N[0] + (i + g); };
    for (int64_t k = -1; k < m->n[2] + 1; ++k)
      for (int64_t j = -1; j < m->n[1] + 1; ++j)
        for (int64_t i = -1; i < m->n[0] + 1; ++i) {
          int out = (k < 0 || k >= m->n[2]) + (j < 0 || j >= m->n[1]) + (i < 0 || i >= m->n[0]);
          if (out > 1) continue;
          double U[5], W[5];
          for (int v = 0; v < 5; ++v) U[v] = B.U0[m->idx(v, k, j, i)];
          if (cons_to_prim(U, m->cfg.gamma, W)) return fail(ORC_ERR_PHYSICS, "non-positive state in tagging");
          P[pidx(k, j, i)] = W[4];
        }
    double mx = 0.0;
    for (int64_t k = 0; k < m->n[2]; ++k)
      for (int64_t j = 0; j < m->n[1]; ++j)
        for (int64_t i = 0; i < m->n[0]; ++i) {
          double g1 = 0.5 * (P[pidx(k, j, i + 1)] - P[pidx(k, j, i - 1)]);
          double g2 = 0.5 * (P[pidx(k, j + 1, i)] - P[pidx(k, j - 1, i)]);
          double g3 = 0.5 * (P[pidx(k + 1, j, i)] - P[pidx(k - 1, j, i)]);
          double e = std::sqrt((g1 * g1 + g2 * g2) + g3 * g3) / P[pidx(k, j, i)];
          if (e > mx) mx = e;
        }
    eps[b] = mx;
  }
  return 0;
}

void flags_from(const orc_mesh* m, const std::vector<double>& eps, std::vector<int8_t>& fl) {
  int64_t nb = (int64_t)m->blocks.size();
  fl.assign(nb, 0);
  for (int64_t b = 0; b < nb; ++b) {
    int lev = m->blocks[b].loc.level;
    if (eps[b] > m->cfg.refine_tol && lev < m->cfg.max_level) fl[b] = 1;
    else if (eps[b] < m->cfg.derefine_tol && lev > 0) fl[b] = -1;
  }
}

/* install a new leaf set; old blocks' data moved / prolongated / restricted into the new ones */
void install(orc_mesh* m, const std::set<LL>& newleaves, bool move_data) {
  std::vector<Block> old;
  old.swap(m->blocks);
  std::map<LL, int64_t> oldgid = m->gid_of;
  m->leaves = newleaves;
  std::vector<Block> nb;
  m->rebuild_blocks(nb);
  for (Block& b : nb) m->alloc_block(b);
  if (move_data) {
    for (Block& b : nb) {
      auto it = oldgid.find(b.loc);
      if (it != oldgid.end()) {
        b.U0 = old[it->second].U0;
        continue;
      }
      if (b.loc.level > 0) {
        LL p{b.loc.level - 1, {b.loc.x[0] >> 1, b.loc.x[1] >> 1, b.loc.x[2] >> 1}};
        auto ip = oldgid.find(p);
        if (ip != oldgid.end()) {
          const std::vector<double>& PU = old[ip->second].U0;
          int64_t ch[3] = {b.loc.x[0] & 1, b.loc.x[1] & 1, b.loc.x[2] & 1};
          for (int v = 0; v < 5; ++v)
            for (int64_t k = 0; k < m->n[2]; ++k)
              for (int64_t j = 0; j < m->n[1]; ++j)
                for (int64_t i = 0; i < m->n[0]; ++i) {
                  int64_t I = ch[0] * m->nc[0] + i / 2, J = ch[1] * m->nc[1] + j / 2, K = ch[2] * m->nc[2] + k / 2;
                  double c = PU[m->idx(v, K, J, I)];
                  double cm[3] = {PU[m->idx(v, K, J, I - 1)], PU[m->idx(v, K, J - 1, I)], PU[m->idx(v, K - 1, J, I)]};
                  double cp[3] = {PU[m->idx(v, K, J, I + 1)], PU[m->idx(v, K, J + 1, I)], PU[m->idx(v, K + 1, J, I)]};
                  double out[8];
                  prolong(c, cm, cp, out);
                  b.U0[m->idx(v, k, j, i)] = out[(k & 1) * 4 + (j & 1) * 2 + (i & 1)];
                }
          continue;
        }
      }
      /* derefined: restrict the 8 old children */
      for (int c = 0; c < 8; ++c) {
        int64_t ch[3] = {c & 1, (c >> 1) & 1, (c >> 2) & 1};
        LL cl{b.loc.level + 1, {2 * b.loc.x[0] + ch[0], 2 * b.loc.x[1] + ch[1], 2 * b.loc.x[2] + ch[2]}};
        const std::vector<double>& CU = old[oldgid.at(cl)].U0;
        for (int v = 0; v < 5; ++v)
          for (int64_t k = 0; k < m->nc[2]; ++k)
            for (int64_t j = 0; j < m->nc[1]; ++j)
              for (int64_t i = 0; i < m->nc[0]; ++i)
                b.U0[m->idx(v, ch[2] * m->nc[2] + k, ch[1] * m->nc[1] + j, ch[0] * m->nc[0] + i)] =
                    restrict_at(m, CU, v, 2 * k, 2 * j, 2 * i);
      }
    }
  }
  m->blocks.swap(nb);
}

/* normalise flags (O9) and return the new leaf set; derefine only when allowed */
std::set<LL> normalise(orc_mesh* m, const std::vector<int8_t>& fl, bool allow_deref) {
  std::set<LL> nl = m->leaves;
  for (size_t b = 0; b < m->blocks.size(); ++b)
    if (fl[b] == 1) orc_mesh::refine(nl, m->blocks[b].loc);
  m->balance(nl);
  if (!allow_deref) return nl;
  std::map<LL, int> cnt;
  for (size_t b = 0; b < m->blocks.size(); ++b) {
    const LL& l = m->blocks[b].loc;
    if (fl[b] != -1 || l.level == 0) continue;
    if (!nl.count(l)) continue; /* got refined */
    LL p{l.level - 1, {l.x[0] >> 1, l.x[1] >> 1, l.x[2] >> 1}};
    cnt[p]++;
  }
  std::vector<LL> accept;
  for (auto& kv : cnt) {
    if (kv.second != 8) continue;
    const LL& P = kv.first;
    bool ok = true;
    for (int c = 0; c < 8 && ok; ++c) {
      LL ch{P.level + 1, {2 * P.x[0] + (c & 1), 2 * P.x[1] + ((c >> 1) & 1), 2 * P.x[2] + ((c >> 2) & 1)}};
      for (int o3 = -1; o3 <= 1 && ok; ++o3)
        for (int o2 = -1; o2 <= 1 && ok; ++o2)
          for (int o1 = -1; o1 <= 1 && ok; ++o1) {
            if (!o1 && !o2 && !o3) continue;
            LL q{ch.level, {ch.x[0] + o1, ch.x[1] + o2, ch.x[2] + o3}};
            if (!m->wrap(q)) continue;
            LL qp{q.level - 1, {q.x[0] >> 1, q.x[1] >> 1, q.x[2] >> 1}};
            if (qp == P) continue;
            if (m->lookup(nl, q, nullptr) == 1) ok = false;
          }
    }
    if (ok) accept.push_back(P);
  }
  for (const LL& P : accept) {
    for (int c = 0; c < 8; ++c)
      nl.erase(LL{P.level + 1, {2 * P.x[0] + (c & 1), 2 * P.x[1] + ((c >> 1) & 1), 2 * P.x[2] + ((c >> 2) & 1)}});
    nl.insert(P);
  }
  return nl;
}

}  // namespace

/* ================================= C ABI ================================= */
extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

int orc_cons_to_prim(const double U[5], double gamma, double W[5]) { return cons_to_prim(U, gamma, W) ? ORC_ERR_PHYSICS : 0; }
void orc_prim_to_cons(const double W[5], double gamma, double U[5]) { prim_to_cons(W, gamma, U); }
void orc_plm(double qm, double q0, double qp, int32_t recon, double* ql, double* qr) {
  double D = plm_slope(qm, q0, qp, recon);
  *ql = q0 - 0.5 * D;
  *qr = q0 + 0.5 * D;
}
void orc_recon5(const double q[5], int32_t recon, double* ql, double* qr) { recon5(q, recon, ql, qr); }
void orc_hlle(const double WL[5], const double WR[5], double gamma, double F[5]) { hlle(WL, WR, gamma, F); }
void orc_hlle_ws(const double WL[5], const double WR[5], double gamma, int32_t wavespeed, double F[5]) {
  hlle(WL, WR, gamma, F, wavespeed);
}
void orc_flux_phys(const double W[5], double gamma, double F[5]) {
  double U[5];
  phys(W, gamma, U, F);
}
double orc_restrict8(const double v[8]) { return restrict8(v); }
void orc_prolong(double c, const double cm[3], const double cp[3], double out[8]) { prolong(c, cm, cp, out); }
uint64_t orc_morton_key(int32_t level, const int64_t lx[3], int32_t max_level) { return morton(level, lx, max_level); }
void orc_partition(int64_t nb, int32_t R, int32_t r, int64_t* lo, int64_t* hi) {
  int64_t q = nb / R, e = nb % R;
  *lo = r * q + std::min<int64_t>(r, e);
  *hi = (r + 1) * q + std::min<int64_t>(r + 1, e);
}
double orc_pairwise_sum(const double* a, int64_t n) { return pairwise_sum(a, n); }

int orc_mesh_create(const orc_config* cfg, orc_mesh** out) {
  if (!cfg || !out) return fail(ORC_ERR_INVALID_ARG, "null argument");
  *out = nullptr;
  if (cfg->nghost != 2 && cfg->nghost != 3) return fail(ORC_ERR_CONFIG, "nghost must be 2 (PLM) or 3 (PPM, WENO-Z)");
  if (cfg->recon >= ORC_RECON_PPM && cfg->nghost != 3) return fail(ORC_ERR_CONFIG, "PPM / WENO-Z need nghost = 3 (A8)");
  if (cfg->nghost == 3 && cfg->max_level > 0)
    return fail(ORC_ERR_CONFIG, "nghost = 3 is supported on uniform meshes only (reading A39)");
  if (cfg->wavespeed != ORC_WS_DAVIS && cfg->wavespeed != ORC_WS_EINFELDT)
    return fail(ORC_ERR_CONFIG, "unknown wave-speed estimate");
  if (cfg->wavespeed == ORC_WS_EINFELDT && cfg->recon >= ORC_RECON_PPM)
    return fail(ORC_ERR_CONFIG, "Einfeldt wave speeds are implemented for PLM (PPM / WENO-Z use Davis)");
  if (!(cfg->gamma > 1.0)) return fail(ORC_ERR_CONFIG, "gamma must exceed 1");
  if (!(cfg->cfl > 0.0)) return fail(ORC_ERR_CONFIG, "cfl must be positive");
  if (cfg->max_level < 0 || cfg->max_level > 10) return fail(ORC_ERR_CONFIG, "max_level out of range");
  orc_mesh* m = new orc_mesh();
  m->cfg = *cfg;
  if (cfg->nregions > 0 && cfg->regions) m->regions.assign(cfg->regions, cfg->regions + 7 * cfg->nregions);
  m->cfg.regions = nullptr;
  m->g = cfg->nghost;
  m->cg = (m->g + 1) / 2 + 1;
  for (int d = 0; d < 3; ++d) {
    m->n[d] = cfg->block_nx[d];
    if (m->n[d] < m->g || cfg->mesh_nx[d] <= 0 || cfg->mesh_nx[d] % m->n[d] != 0) {
      delete m;
      return fail(ORC_ERR_CONFIG, "block size does not tile the root grid (S:144)");
    }
    if ((cfg->bc_inner[d] == ORC_BC_PERIODIC) != (cfg->bc_outer[d] == ORC_BC_PERIODIC)) {
      delete m;
      return fail(ORC_ERR_CONFIG, "periodic boundaries must be paired");
    }
    for (int s = 0; s < 2; ++s) {
      int bc = s ? cfg->bc_outer[d] : cfg->bc_inner[d];
      if (bc < 0 || bc > 2) { delete m; return fail(ORC_ERR_CONFIG, "unknown boundary tag (S:414)"); }
    }
    if (cfg->max_level > 0 && (m->n[d] % 2 != 0 || m->n[d] < 2 * m->g)) {
      delete m;
      return fail(ORC_ERR_CONFIG, "refinement needs even block sizes >= 2*nghost");
    }
    m->nc[d] = m->n[d] / 2;
    m->N[d] = m->n[d] + 2 * m->g;
    m->NC[d] = m->nc[d] + 2 * m->cg;
    m->nrb[d] = cfg->mesh_nx[d] / m->n[d];
  }
  for (int64_t z = 0; z < m->nrb[2]; ++z)
    for (int64_t y = 0; y < m->nrb[1]; ++y)
      for (int64_t x = 0; x < m->nrb[0]; ++x) m->leaves.insert(LL{0, {x, y, z}});
  /* static regions / initial refinement, level by level, then 2:1 (O1) */
  if (cfg->refinement != ORC_REF_NONE) {
    for (int lev = 0; lev < cfg->max_level; ++lev) {
      std::vector<LL> todo;
      for (const LL& l : m->leaves) {
        if (l.level != lev) continue;
        double bmin[3], bmax[3];
        m->box(l, bmin, bmax);
        for (int r = 0; r < cfg->nregions; ++r) {
          const double* R = &m->regions[7 * r];
          if ((int)R[0] <= lev) continue;
          bool ov = true;
          for (int d = 0; d < 3; ++d) ov = ov && (bmin[d] < R[2 + 2 * d]) && (bmax[d] > R[1 + 2 * d]);
          if (ov) { todo.push_back(l); break; }
        }
      }
      for (const LL& l : todo) orc_mesh::refine(m->leaves, l);
      m->balance(m->leaves);
    }
  }
  m->rebuild_blocks(m->blocks);
  /* field arrays are allocated lazily (ensure_alloc) so that pure mesh queries stay cheap */
  *out = m;
  return 0;
}

int orc_mesh_destroy(orc_mesh* m) {
  delete m;
  return 0;
}

int orc_exchange(orc_mesh* m) {
  if (!m->allocated) return fail(ORC_ERR_STATE, "no state set");
  exchange(m, &Block::U0);
  return 0;
}

int orc_compute_dt(orc_mesh* m, double* dt) {
  if (!m->allocated) return fail(ORC_ERR_STATE, "no state set");
  int rc = compute_dt(m, &m->dt);
  if (rc) return rc;
  if (dt) *dt = m->dt;
  return 0;
}

int orc_set_problem(orc_mesh* m, int32_t problem, const double* p, int32_t np) {
  if (!m) return fail(ORC_ERR_INVALID_ARG, "null mesh");
  std::vector<double> pp(p, p + np);
  if (problem == ORC_PROB_LINEAR_WAVE) {
    if (np < 4) return fail(ORC_ERR_INVALID_ARG, "linear wave needs {A,k1,k2,k3}");
  } else if (problem == ORC_PROB_SOD) {
    if (np < 1) pp = {0.5 * (m->cfg.xmin[0] + m->cfg.xmax[0])};
  } else if (problem == ORC_PROB_BLAST) {
    if (np < 3) return fail(ORC_ERR_INVALID_ARG, "blast needs {p_in,p_out,r[,cx,cy,cz]}");
    if (np < 6) {
      pp.resize(6);
      for (int d = 0; d < 3; ++d) pp[3 + d] = 0.5 * (m->cfg.xmin[d] + m->cfg.xmax[d]);
    }
    if (!(pp[0] > 0 && pp[1] > 0 && pp[2] > 0)) return fail(ORC_ERR_INVALID_ARG, "blast parameters out of range");
  } else if (problem == ORC_PROB_KH) {
    if (np < 1) pp.push_back(0.01);
    if (pp.size() < 2) pp.push_back(0.05);
    if (!(pp[1] > 0)) return fail(ORC_ERR_INVALID_ARG, "KH sigma must be positive");
  } else {
    return fail(ORC_ERR_INVALID_ARG, "unknown problem");
  }
  m->problem = problem;
  m->pparams = pp;
  m->ensure_alloc();
  if (m->cfg.refinement == ORC_REF_ADAPTIVE) {
    /* O9: AMR pre-refinement at t=0 */
    for (int it = 0; it < m->cfg.max_level; ++it) {
      for (Block& b : m->blocks) pgen_block(m, b);
      exchange(m, &Block::U0);
      std::vector<double> eps;
      int rc = indicators(m, eps);
      if (rc) return rc;
      std::vector<int8_t> fl;
      flags_from(m, eps, fl);
      bool any = false;
      for (auto& f : fl) {
        if (f == -1) f = 0;
        if (f == 1) any = true;
      }
      if (!any) break;
      std::set<LL> nl = normalise(m, fl, false);
      install(m, nl, false);
    }
  }
  for (Block& b : m->blocks) pgen_block(m, b);
  exchange(m, &Block::U0);
  m->t = 0.0;
  m->cycle = 0;
  m->hist.clear();
  m->have_state = true;
  return compute_dt(m, &m->dt);
}

int orc_set_state(orc_mesh* m, int64_t gid, const double* cons, int64_t nelem) {
  if (!m || gid < 0 || gid >= (int64_t)m->blocks.size()) return fail(ORC_ERR_INVALID_ARG, "bad gid");
  m->ensure_alloc();
  if (nelem != 5 * m->n[0] * m->n[1] * m->n[2]) return fail(ORC_ERR_INVALID_ARG, "bad nelem");
  Block& b = m->blocks[gid];
  int64_t q = 0;
  for (int v = 0; v < 5; ++v)
    for (int64_t k = 0; k < m->n[2]; ++k)
      for (int64_t j = 0; j < m->n[1]; ++j)
        for (int64_t i = 0; i < m->n[0]; ++i) b.U0[m->idx(v, k, j, i)] = cons[q++];
  m->have_state = true;
  return 0;
}

int orc_get_state(const orc_mesh* m, int64_t gid, double* cons, int64_t nelem) {
  if (!m || gid < 0 || gid >= (int64_t)m->blocks.size()) return fail(ORC_ERR_INVALID_ARG, "bad gid");
  if (!m->allocated) return fail(ORC_ERR_STATE, "no state set");
  if (nelem != 5 * m->n[0] * m->n[1] * m->n[2]) return fail(ORC_ERR_INVALID_ARG, "bad nelem");
  const Block& b = m->blocks[gid];
  int64_t q = 0;
  for (int v = 0; v < 5; ++v)
    for (int64_t k = 0; k < m->n[2]; ++k)
      for (int64_t j = 0; j < m->n[1]; ++j)
        for (int64_t i = 0; i < m->n[0]; ++i) cons[q++] = b.U0[m->idx(v, k, j, i)];
  return 0;
}

int orc_get_state_full(const orc_mesh* m, int64_t gid, double* out, int64_t nelem) {
  if (!m || gid < 0 || gid >= (int64_t)m->blocks.size()) return fail(ORC_ERR_INVALID_ARG, "bad gid");
  if (!m->allocated) return fail(ORC_ERR_STATE, "no state set");
  if (nelem != (int64_t)m->blocks[gid].U0.size()) return fail(ORC_ERR_INVALID_ARG, "bad nelem");
  std::memcpy(out, m->blocks[gid].U0.data(), nelem * sizeof(double));
  return 0;
}

int orc_set_state_full(orc_mesh* m, int64_t gid, const double* in, int64_t nelem) {
  if (!m || gid < 0 || gid >= (int64_t)m->blocks.size()) return fail(ORC_ERR_INVALID_ARG, "bad gid");
  m->ensure_alloc();
  if (nelem != (int64_t)m->blocks[gid].U0.size()) return fail(ORC_ERR_INVALID_ARG, "bad nelem");
  std::memcpy(m->blocks[gid].U0.data(), in, nelem * sizeof(double));
  m->have_state = true;
  return 0;
}

int orc_tag_and_remesh(orc_mesh* m) {
  if (!m->allocated) return fail(ORC_ERR_STATE, "no state set");
  std::vector<double> eps;
  int rc = indicators(m, eps);
  if (rc) return rc;
  std::vector<int8_t> fl;
  flags_from(m, eps, fl);
  m->last_flags = fl;
  m->last_eps = eps;
  int iv = m->cfg.derefine_interval > 0 ? m->cfg.derefine_interval : 1;
  bool allow = (m->cycle % iv) == 0;
  std::set<LL> nl = normalise(m, fl, allow);
  if (nl != m->leaves) {
    install(m, nl, true);
    exchange(m, &Block::U0);
  }
  return 0;
}

/* O5: the per-cycle schedule, RK2 (A1) or VL2 */
int orc_step(orc_mesh* m, int32_t ncycles, double tlim) {
  if (!m || !m->have_state) return fail(ORC_ERR_STATE, "no state set");
  for (int32_t c = 0; c < ncycles; ++c) {
    if (tlim > 0.0 && m->t >= tlim) break;
    double dt = m->dt;
    if (tlim > 0.0 && m->t + dt > tlim) dt = tlim - m->t;
    int rc;
    if (m->cfg.integrator == ORC_INT_VL2) {
      rc = stage(m, &Block::U0, &Block::U1, 0.5 * dt, 0);
      if (rc) return rc;
      exchange(m, &Block::U1);
      rc = stage(m, &Block::U1, &Block::U0, dt, 0);
      if (rc) return rc;
    } else {
      rc = stage(m, &Block::U0, &Block::U1, dt, 0);
      if (rc) return rc;
      exchange(m, &Block::U1);
      rc = stage(m, &Block::U1, &Block::U0, dt, 1);
      if (rc) return rc;
    }
    exchange(m, &Block::U0);
    m->t += dt;
    m->cycle += 1;
    if (m->cfg.refinement == ORC_REF_ADAPTIVE) {
      rc = orc_tag_and_remesh(m);
      if (rc) return rc;
    }
    rc = compute_dt(m, &m->dt);
    if (rc) return rc;
    double tot[5];
    totals(m, tot);
    m->hist.push_back({m->t, dt, tot[0], tot[1], tot[2], tot[3], tot[4]});
  }
  return 0;
}

int orc_get_time(const orc_mesh* m, double* t, double* dt, int64_t* cycle) {
  if (t) *t = m->t;
  if (dt) *dt = m->dt;
  if (cycle) *cycle = m->cycle;
  return 0;
}

int orc_num_blocks(const orc_mesh* m, int64_t* n) {
  *n = (int64_t)m->blocks.size();
  return 0;
}

int orc_get_blocks(const orc_mesh* m, orc_block* out, int64_t cap, int64_t* n) {
  *n = (int64_t)m->blocks.size();
  for (int64_t b = 0; b < *n && b < cap; ++b) {
    const Block& B = m->blocks[b];
    out[b].gid = B.gid;
    out[b].level = B.loc.level;
    out[b].rank = B.rank;
    for (int d = 0; d < 3; ++d) {
      out[b].lx[d] = B.loc.x[d];
      out[b].xmin[d] = B.bxmin[d];
      out[b].xmax[d] = B.bxmax[d];
    }
  }
  return 0;
}

int orc_get_neighbors(const orc_mesh* m, int64_t gid, orc_neighbor* out, int32_t cap, int32_t* n) {
  if (gid < 0 || gid >= (int64_t)m->blocks.size()) return fail(ORC_ERR_INVALID_ARG, "bad gid");
  const Block& B = m->blocks[gid];
  *n = (int32_t)B.nbrs.size();
  for (int32_t q = 0; q < *n && q < cap; ++q) {
    const Nbr& e = B.nbrs[q];
    out[q].gid = e.gid;
    out[q].rank = e.rank;
    for (int d = 0; d < 3; ++d) out[q].off[d] = (int8_t)e.off[d];
    out[q].dlevel = (int8_t)e.dlevel;
    out[q].fine[0] = (int8_t)e.fine[0];
    out[q].fine[1] = (int8_t)e.fine[1];
  }
  return 0;
}

int orc_get_refine_flags(const orc_mesh* m, int8_t* out, int64_t cap, int64_t* n) {
  *n = (int64_t)m->last_flags.size();
  for (int64_t b = 0; b < *n && b < cap; ++b) out[b] = m->last_flags[b];
  return 0;
}

int orc_get_indicators(const orc_mesh* m, double* out, int64_t cap, int64_t* n) {
  *n = (int64_t)m->last_eps.size();
  for (int64_t b = 0; b < *n && b < cap; ++b) out[b] = m->last_eps[b];
  return 0;
}

int orc_get_history(const orc_mesh* m, double* out, int64_t cap, int64_t* nrows) {
  *nrows = (int64_t)m->hist.size();
  for (int64_t r = 0; r < *nrows && r < cap; ++r)
    for (int c = 0; c < 7; ++c) out[7 * r + c] = m->hist[r][c];
  return 0;
}

int orc_totals(const orc_mesh* m, double out[5]) {
  if (!m->allocated) return fail(ORC_ERR_STATE, "no state set");
  totals(m, out);
  return 0;
}

int orc_level_counts(const orc_mesh* m, int64_t* out, int32_t cap) {
  for (int32_t l = 0; l < cap; ++l) out[l] = 0;
  for (const Block& b : m->blocks)
    if (b.loc.level < cap) out[b.loc.level]++;
  return 0;
}

}  // extern "C"
