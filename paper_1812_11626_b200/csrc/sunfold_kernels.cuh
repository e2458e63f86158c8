// sunfold_kernels.cuh — sm_100a fp64 kernels of the SU(N) unfold (arXiv:1812.11626).
//
// Row s of Q is the generator expansion of the Hermitian matrix G_s = L^+(F_s), where
//   L^+(X) = i[H, X] + sum_p gamma_p (L_p^+ X L_p - 1/2 {L_p^+ L_p, X})
// is the Hilbert-Schmidt adjoint of the GKSL generator (Eq. 1):
//   Q_sm = Tr(F_s L(F_m)) = Tr(L^+(F_s) F_m),   K_s = Tr(F_s L(I/N)) = Tr(L^+(F_s))/N.
// This is the paper's contraction of Eq. 6 (q_sn = sum_m f_mns h_m) and Eqs. 10-11
// (R = -1/2 gamma Re(Y^H X), K; P:200-211 with readings R1/R2) evaluated per output row: the
// structure constants f_mns = -i Tr(F_s[F_m,F_n]) and d_mns = Tr(F_s{F_m,F_n}) (Eq. 4,
// P:152-158) are products of matrix units E_ab E_cd = delta_bc E_ad, so their nonzero
// index patterns (the "triangle" class for generators sharing one index, the
// "pair" class for coincident pairs, and the D^l chains) are enumerated here as the
// support of G_s inside small index windows; no f/d tensor is stored.
// DESIGN.md gives the derivation and the algebra below.
//
// Band storage (the GPU form of the paper's coefficient "index map"):
//   K  = H0 + (i/2) sum_p gamma_p L_p^+ L_p     n x (2 wK + 1) complex, row-major by row
//   H  = H0                                     n x (2 wK + 1)   (D rows only)
//   Lt_p = sqrt(gamma_p) L_p                    n x (2 wL + 1), p = 0..P-1
// For S_ab / J_ab rows (a < b) with U = L^+(E_ab) (so G = (U + U^+)/sqrt2 or (-iU + iU^+)/sqrt2):
//   U_cd = i K_ca [d = b] - i conj(K_db) [c = a] + sum_p conj(Lt_p,ac) Lt_p,bd
//   row S_ab:  S_cd -> Re(U_cd + U_dc),  J_cd -> Im(U_dc - U_cd),  D^l <- g_c = sqrt2 Re U_cc
//   row J_ab:  S_cd -> Im(U_cd + U_dc),  J_cd -> Re(U_cd - U_dc),  D^l <- g_c = sqrt2 Im U_cc
//   D^l coefficient = (sum_{c<l} g_c - l g_l)/sqrt(l(l+1)),   K_s = sum_c g_c / N.
// U lives in rows [a-W, a+W] x cols [b-W, b+W] (W = max(wK, wL)); for a "far" pair
// (b - a > 2W) U_dc = 0 for every c < d and there is no diagonal, so each row has at most
// npos_far entries per block and no D chain.  For D^lam rows, with f = diag(D^lam):
//   G_cd = i H_cd (f_d - f_c) + sum_p sum_x (f_x - (f_c + f_d)/2) conj(Lt_p,xc) Lt_p,xd
// which vanishes unless {c, d, x} straddle lam, so G lives in [lam - wK, lam + wK]^2.
//
// Pattern rule (R6): an entry is stored iff |q| > tau.  Every value is computed by
// one lane in a fixed order, identically in the count and fill passes (same code), so the
// two passes agree and the output is bitwise deterministic.  Duplicate (row, col)
// contributions are merged by construction (position-major generation), not by atomics.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sunk {

constexpr int WMAX = 15;            // max(wK, wL) supported by the banded kernels
constexpr int WIN_MAX = 4 * WMAX + 2;  // near-pair window bound (4W+1), padded
constexpr unsigned FULL = 0xffffffffu;

struct Band {
  const double2* v;  // v[r * (2w+1) + (c - r + w)]
  int w;
};

struct Prob {
  int n, P, wK, wL, W;
  long long np;  // n(n-1)/2
  long long m;   // n^2 - 1
  Band K, H;
  const double2* L;  // P bands of half-width wL (sqrt(gamma)-scaled)
  double tau;
  int has_k;  // write K
  int mode;   // 0 thread-per-pair (staged), 1 warp-per-pair (direct)
  int tp;     // pairs per tile
  long long npt, ndt;  // pair tiles, D tiles
};

__device__ __forceinline__ double2 bget(const Band B, int r, int c) {
  int o = c - r;
  if (o < -B.w || o > B.w) return make_double2(0.0, 0.0);
  return __ldg(&B.v[(long long)r * (2 * B.w + 1) + (o + B.w)]);
}

__device__ __forceinline__ double2 lget(const Prob& pr, int p, int r, int c) {
  int o = c - r;
  if (o < -pr.wL || o > pr.wL) return make_double2(0.0, 0.0);
  return __ldg(&pr.L[((long long)p * pr.n + r) * (2 * pr.wL + 1) + (o + pr.wL)]);
}

__device__ __forceinline__ long long pidx(long long n, long long a, long long b) {
  return a * (2 * n - a - 1) / 2 + (b - a - 1);
}

// pair index p -> (a, b), a < b < n, lexicographic (R5)
__device__ __forceinline__ void pair_decode(long long n, long long p, int& a_out, int& b_out) {
  double t = (double)(2 * n - 1);
  double disc = t * t - 8.0 * (double)p;
  long long a = (long long)floor((t - sqrt(disc > 0.0 ? disc : 0.0)) * 0.5);
  if (a < 0) a = 0;
  if (a > n - 2) a = n - 2;
  while (a > 0 && a * (2 * n - a - 1) / 2 > p) --a;
  while (a + 1 <= n - 2 && (a + 1) * (2 * n - a - 2) / 2 <= p) ++a;
  a_out = (int)a;
  b_out = (int)(a + 1 + (p - a * (2 * n - a - 1) / 2));
}

// local upper-triangle index k in an nw x nw window -> (i, j), i < j
__device__ __forceinline__ void win_decode(int nw, int k, int& i, int& j) {
  int r = 0;
  while (k >= nw - 1 - r) {
    k -= nw - 1 - r;
    ++r;
  }
  i = r;
  j = r + 1 + k;
}

__device__ __forceinline__ double inv_sqrt_ll1(int l) { return 1.0 / sqrt((double)l * (double)(l + 1)); }

// U = L^+(E_ab) element (c, d)
__device__ __forceinline__ double2 U_elem(const Prob& pr, int a, int b, int c, int d) {
  double ux = 0.0, uy = 0.0;
  if (d == b) {  // + i K_ca
    double2 k = bget(pr.K, c, a);
    ux -= k.y;
    uy += k.x;
  }
  if (c == a) {  // - i conj(K_db)
    double2 k = bget(pr.K, d, b);
    ux -= k.y;
    uy -= k.x;
  }
  int dc = c - a, dd = d - b;
  if (dc >= -pr.wL && dc <= pr.wL && dd >= -pr.wL && dd <= pr.wL) {
    for (int p = 0; p < pr.P; ++p) {
      double2 la = lget(pr, p, a, c);
      double2 lb = lget(pr, p, b, d);
      ux += la.x * lb.x + la.y * lb.y;  // conj(la) * lb
      uy += la.x * lb.y - la.y * lb.x;
    }
  }
  return make_double2(ux, uy);
}

// G = L^+(D^lam) element (c, d)
__device__ __forceinline__ double fdiag(int x, int lam, double alpha) {
  return x < lam ? alpha : (x == lam ? -(double)lam * alpha : 0.0);
}

__device__ __forceinline__ double2 G_elem(const Prob& pr, int lam, double alpha, int c, int d) {
  double fc = fdiag(c, lam, alpha), fd = fdiag(d, lam, alpha);
  double2 h = bget(pr.H, c, d);
  double df = fd - fc;
  double gx = -h.y * df, gy = h.x * df;  // i H_cd (f_d - f_c)
  int lo = max(c, d) - pr.wL, hi = min(c, d) + pr.wL;
  if (lo <= hi && pr.P > 0) {
    double fm = 0.5 * (fc + fd);
    if (lo < 0) lo = 0;
    if (hi > pr.n - 1) hi = pr.n - 1;
    for (int x = lo; x <= hi; ++x) {
      double coef = fdiag(x, lam, alpha) - fm;
      if (coef == 0.0) continue;
      for (int p = 0; p < pr.P; ++p) {
        double2 l1 = lget(pr, p, x, c);
        double2 l2 = lget(pr, p, x, d);
        gx += coef * (l1.x * l2.x + l1.y * l2.y);
        gy += coef * (l1.x * l2.y - l1.y * l2.x);
      }
    }
  }
  return make_double2(gx, gy);
}

// Enumerate the far-pair positions (c, d) of U in lexicographic order.
template <class F>
__device__ __forceinline__ void far_positions(const Prob& pr, int a, int b, F&& f) {
  const int n = pr.n, W = pr.W, wL = pr.wL, wK = pr.wK;
  for (int dc = -W; dc <= W; ++dc) {
    int c = a + dc;
    if (c < 0 || c >= n) continue;
    int adc = dc < 0 ? -dc : dc;
    if (dc == 0) {
      for (int dd = -W; dd <= W; ++dd) {
        int d = b + dd;
        if (d < n) f(c, d);
      }
    } else if (adc <= wL) {
      for (int dd = -wL; dd <= wL; ++dd) {
        int d = b + dd;
        if (d < n) f(c, d);
      }
    } else if (adc <= wK) {
      f(c, b);
    }
  }
}

// ---------------------------------------------------------------------------------------
// Output sinks
// ---------------------------------------------------------------------------------------
struct Seg {  // one contiguous CSR segment (a row or a tile segment)
  int* scol;        // shared staging (nullptr: write global)
  double* sval;
  int32_t* gcol;    // global col/val base pointers already offset to the segment start
  double* gval;
  __device__ __forceinline__ void emit(long long off, long long col, double v) const {
    if (scol) {
      scol[off] = (int)col;
      sval[off] = v;
    } else {
      gcol[off] = (int32_t)col;
      gval[off] = v;
    }
  }
};

// ---------------------------------------------------------------------------------------
// Far pair, one thread.  Counts (nre, nim); with EMIT writes both rows.
//   row S_ab: [Re U_cd > tau at p(c,d)] then [-Im U_cd at NP + p(c,d)]
//   row J_ab: [Im U_cd at p(c,d)]       then [Re U_cd at NP + p(c,d)]
// ---------------------------------------------------------------------------------------
template <bool EMIT>
__device__ __forceinline__ void far_pair_thread(const Prob& pr, int a, int b, int& nre, int& nim,
                                                const Seg& sS, long long offS, const Seg& sJ,
                                                long long offJ) {
  const double tau = pr.tau;
  if (!EMIT) {
    int cr = 0, ci = 0;
    far_positions(pr, a, b, [&](int c, int d) {
      double2 u = U_elem(pr, a, b, c, d);
      cr += fabs(u.x) > tau;
      ci += fabs(u.y) > tau;
    });
    nre = cr;
    nim = ci;
    return;
  }
  const long long n = pr.n, np = pr.np;
  long long ire = 0, iim = 0;
  const long long nR = nre, nI = nim;
  far_positions(pr, a, b, [&](int c, int d) {
    double2 u = U_elem(pr, a, b, c, d);
    long long q = pidx(n, c, d);
    if (fabs(u.x) > tau) {
      sS.emit(offS + ire, q, u.x);
      sJ.emit(offJ + nI + ire, np + q, u.x);
      ++ire;
    }
    if (fabs(u.y) > tau) {
      sS.emit(offS + nR + iim, np + q, -u.y);
      sJ.emit(offJ + iim, q, u.y);
      ++iim;
    }
  });
}

// ---------------------------------------------------------------------------------------
// D^l chain of one row from the diagonal g over window [lo, hi] (warp-cooperative).
// pre[j] = sum_{i<j} g[i] (j = 0..nw), computed by lane 0 in ascending order.
// Returns the number of kept entries; with EMIT writes them at seg/off.
// ---------------------------------------------------------------------------------------
template <bool EMIT>
__device__ int warp_dchain(const Prob& pr, int lo, int hi, const double* g, const double* pre,
                           const Seg& seg, long long off) {
  const int lane = threadIdx.x & 31;
  const int n = pr.n;
  const double tau = pr.tau;
  const int nw = hi - lo + 1;
  const double tr = pre[nw];
  const long long dbase = 2 * pr.np - 1;  // column of D^l is 2NP + l - 1
  int kept = 0;
  int lstart = lo < 1 ? 1 : lo;
  for (int l0 = lstart; l0 < n; l0 += 32) {
    int l = l0 + lane;
    bool valid = l < n;
    double coef = 0.0;
    if (valid) {
      double il = inv_sqrt_ll1(l);
      if (l <= hi)
        coef = (pre[l - lo] - (double)l * g[l - lo]) * il;
      else
        coef = tr * il;
    }
    bool keep = valid && fabs(coef) > tau;
    unsigned km = __ballot_sync(FULL, keep);
    if (EMIT && keep) seg.emit(off + kept + __popc(km & ((1u << lane) - 1u)), dbase + l, coef);
    kept += __popc(km);
    // beyond hi |tr * inv(l)| is non-increasing in l: stop after the first drop there
    unsigned dropped_beyond = __ballot_sync(FULL, valid && l > hi && !keep);
    if (dropped_beyond) break;
  }
  return kept;
}

// ---------------------------------------------------------------------------------------
// Near pair (b - a <= 2W), warp-cooperative.  scratch: per-warp shared arrays of WIN_MAX+1.
// Outputs counts (cS, cJ) and K values; with EMIT writes rows S_ab (seg sS at offS) and
// J_ab (seg sJ at offJ).
// ---------------------------------------------------------------------------------------
template <bool EMIT>
__device__ void warp_near_pair(const Prob& pr, int a, int b, double* gS, double* gJ, double* pS,
                               double* pJ, int& cS, int& cJ, double& kS, double& kJ, const Seg& sS,
                               long long offS, const Seg& sJ, long long offJ) {
  const int lane = threadIdx.x & 31;
  const int n = pr.n, W = pr.W;
  const long long np = pr.np;
  const double tau = pr.tau;
  const int lo = a - W < 0 ? 0 : a - W;
  const int hi = b + W > n - 1 ? n - 1 : b + W;
  const int nw = hi - lo + 1;
  const int npos = nw * (nw - 1) / 2;
  const unsigned lt = (1u << lane) - 1u;
  // pass 1: counts of the four parts
  int nSS = 0, nSJ = 0, nJS = 0, nJJ = 0;
  for (int k0 = 0; k0 < npos; k0 += 32) {
    int k = k0 + lane;
    double vSS = 0, vSJ = 0, vJS = 0, vJJ = 0;
    if (k < npos) {
      int i, j;
      win_decode(nw, k, i, j);
      int c = lo + i, d = lo + j;
      double2 ucd = U_elem(pr, a, b, c, d), udc = U_elem(pr, a, b, d, c);
      vSS = ucd.x + udc.x;
      vSJ = udc.y - ucd.y;
      vJS = ucd.y + udc.y;
      vJJ = ucd.x - udc.x;
    }
    nSS += __popc(__ballot_sync(FULL, fabs(vSS) > tau));
    nSJ += __popc(__ballot_sync(FULL, fabs(vSJ) > tau));
    nJS += __popc(__ballot_sync(FULL, fabs(vJS) > tau));
    nJJ += __popc(__ballot_sync(FULL, fabs(vJJ) > tau));
  }
  // pass 2 (EMIT only): write the S and J blocks
  if (EMIT) {
    int iSS = 0, iSJ = 0, iJS = 0, iJJ = 0;
    for (int k0 = 0; k0 < npos; k0 += 32) {
      int k = k0 + lane;
      double vSS = 0, vSJ = 0, vJS = 0, vJJ = 0;
      long long q = 0;
      if (k < npos) {
        int i, j;
        win_decode(nw, k, i, j);
        int c = lo + i, d = lo + j;
        double2 ucd = U_elem(pr, a, b, c, d), udc = U_elem(pr, a, b, d, c);
        vSS = ucd.x + udc.x;
        vSJ = udc.y - ucd.y;
        vJS = ucd.y + udc.y;
        vJJ = ucd.x - udc.x;
        q = pidx(n, c, d);
      }
      unsigned m;
      bool kp;
      kp = fabs(vSS) > tau; m = __ballot_sync(FULL, kp);
      if (kp) sS.emit(offS + iSS + __popc(m & lt), q, vSS);
      iSS += __popc(m);
      kp = fabs(vSJ) > tau; m = __ballot_sync(FULL, kp);
      if (kp) sS.emit(offS + nSS + iSJ + __popc(m & lt), np + q, vSJ);
      iSJ += __popc(m);
      kp = fabs(vJS) > tau; m = __ballot_sync(FULL, kp);
      if (kp) sJ.emit(offJ + iJS + __popc(m & lt), q, vJS);
      iJS += __popc(m);
      kp = fabs(vJJ) > tau; m = __ballot_sync(FULL, kp);
      if (kp) sJ.emit(offJ + nJS + iJJ + __popc(m & lt), np + q, vJJ);
      iJJ += __popc(m);
    }
  }
  // diagonal -> g, prefix sums (lane 0, ascending), D chains
  const double s2 = 1.4142135623730951;
  for (int i = lane; i < nw; i += 32) {
    double2 u = U_elem(pr, a, b, lo + i, lo + i);
    gS[i] = s2 * u.x;
    gJ[i] = s2 * u.y;
  }
  __syncwarp();
  if (lane == 0) {
    double aS = 0.0, aJ = 0.0;
    for (int i = 0; i < nw; ++i) {
      pS[i] = aS;
      pJ[i] = aJ;
      aS += gS[i];
      aJ += gJ[i];
    }
    pS[nw] = aS;
    pJ[nw] = aJ;
  }
  __syncwarp();
  int chS = warp_dchain<EMIT>(pr, lo, hi, gS, pS, sS, offS + nSS + nSJ);
  int chJ = warp_dchain<EMIT>(pr, lo, hi, gJ, pJ, sJ, offJ + nJS + nJJ);
  cS = nSS + nSJ + chS;
  cJ = nJS + nJJ + chJ;
  kS = pS[nw] / (double)n;
  kJ = pJ[nw] / (double)n;
  __syncwarp();
}

// ---------------------------------------------------------------------------------------
// Far pair, warp-cooperative (warp mode): lane k of each 32-chunk owns far position k
// (pos_dc/pos_dd: the far_positions() order, relative to (a, b)).  Pass 1 counts the Re and
// Im parts; with EMIT pass 2 recomputes and writes both rows (same layout as the thread path).
// ---------------------------------------------------------------------------------------
template <bool EMIT>
__device__ void warp_far_pair(const Prob& pr, int a, int b, const int* pos_dc, const int* pos_dd,
                              int npos, int& cnt, const Seg& sS, long long offS, const Seg& sJ,
                              long long offJ) {
  const int lane = threadIdx.x & 31;
  const int n = pr.n;
  const long long np = pr.np;
  const double tau = pr.tau;
  const unsigned lt = (1u << lane) - 1u;
  int nR = 0, nI = 0;
  for (int k0 = 0; k0 < npos; k0 += 32) {
    int k = k0 + lane;
    bool okr = false, oki = false;
    if (k < npos) {
      int c = a + pos_dc[k], d = b + pos_dd[k];
      if (c >= 0 && c < n && d < n) {
        double2 u = U_elem(pr, a, b, c, d);
        okr = fabs(u.x) > tau;
        oki = fabs(u.y) > tau;
      }
    }
    nR += __popc(__ballot_sync(FULL, okr));
    nI += __popc(__ballot_sync(FULL, oki));
  }
  cnt = nR + nI;
  if (!EMIT) return;
  int iR = 0, iI = 0;
  for (int k0 = 0; k0 < npos; k0 += 32) {
    int k = k0 + lane;
    bool okr = false, oki = false;
    double2 u = make_double2(0.0, 0.0);
    long long q = 0;
    if (k < npos) {
      int c = a + pos_dc[k], d = b + pos_dd[k];
      if (c >= 0 && c < n && d < n) {
        u = U_elem(pr, a, b, c, d);
        okr = fabs(u.x) > tau;
        oki = fabs(u.y) > tau;
        q = pidx(n, c, d);
      }
    }
    unsigned mr = __ballot_sync(FULL, okr), mi = __ballot_sync(FULL, oki);
    if (okr) {
      int r = iR + __popc(mr & lt);
      sS.emit(offS + r, q, u.x);
      sJ.emit(offJ + nI + r, np + q, u.x);
    }
    if (oki) {
      int r = iI + __popc(mi & lt);
      sS.emit(offS + nR + r, np + q, -u.y);
      sJ.emit(offJ + r, q, u.y);
    }
    iR += __popc(mr);
    iI += __popc(mi);
  }
}

// ---------------------------------------------------------------------------------------
// D^lam row, warp-cooperative.
// ---------------------------------------------------------------------------------------
template <bool EMIT>
__device__ void warp_d_row(const Prob& pr, int lam, double* g, double* pre, int& cnt, double& kval,
                           const Seg& seg, long long off) {
  const int lane = threadIdx.x & 31;
  const int n = pr.n;
  const long long np = pr.np;
  const double tau = pr.tau;
  const double alpha = inv_sqrt_ll1(lam);
  const int lo = lam - pr.wK < 0 ? 0 : lam - pr.wK;
  const int hi = lam + pr.wK > n - 1 ? n - 1 : lam + pr.wK;
  const int nw = hi - lo + 1;
  const int npos = nw * (nw - 1) / 2;
  const unsigned lt = (1u << lane) - 1u;
  const double s2 = 1.4142135623730951;
  int nS = 0, nJ = 0;
  for (int k0 = 0; k0 < npos; k0 += 32) {
    int k = k0 + lane;
    double vS = 0, vJ = 0;
    if (k < npos) {
      int i, j;
      win_decode(nw, k, i, j);
      double2 gv = G_elem(pr, lam, alpha, lo + i, lo + j);
      vS = s2 * gv.x;
      vJ = -s2 * gv.y;
    }
    nS += __popc(__ballot_sync(FULL, fabs(vS) > tau));
    nJ += __popc(__ballot_sync(FULL, fabs(vJ) > tau));
  }
  if (EMIT) {
    int iS = 0, iJ = 0;
    for (int k0 = 0; k0 < npos; k0 += 32) {
      int k = k0 + lane;
      double vS = 0, vJ = 0;
      long long q = 0;
      if (k < npos) {
        int i, j;
        win_decode(nw, k, i, j);
        double2 gv = G_elem(pr, lam, alpha, lo + i, lo + j);
        vS = s2 * gv.x;
        vJ = -s2 * gv.y;
        q = pidx(n, lo + i, lo + j);
      }
      bool kp = fabs(vS) > tau;
      unsigned m = __ballot_sync(FULL, kp);
      if (kp) seg.emit(off + iS + __popc(m & lt), q, vS);
      iS += __popc(m);
      kp = fabs(vJ) > tau;
      m = __ballot_sync(FULL, kp);
      if (kp) seg.emit(off + nS + iJ + __popc(m & lt), np + q, vJ);
      iJ += __popc(m);
    }
  }
  for (int i = lane; i < nw; i += 32) g[i] = G_elem(pr, lam, alpha, lo + i, lo + i).x;
  __syncwarp();
  if (lane == 0) {
    double acc = 0.0;
    for (int i = 0; i < nw; ++i) {
      pre[i] = acc;
      acc += g[i];
    }
    pre[nw] = acc;
  }
  __syncwarp();
  int ch = warp_dchain<EMIT>(pr, lo, hi, g, pre, seg, off + nS + nJ);
  cnt = nS + nJ + ch;
  kval = pre[nw] / (double)n;
  __syncwarp();
}

// ---------------------------------------------------------------------------------------
// Block-wide exclusive scan of one int per thread (blockDim.x <= 1024, multiple of 32).
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ int block_exclusive_scan(int v, int* warp_tot, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int t = lane < nwarps ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(FULL, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nwarps) warp_tot[lane] = t;  // inclusive
  }
  __syncthreads();
  int before = wid > 0 ? warp_tot[wid - 1] : 0;
  total = warp_tot[nwarps - 1];
  __syncthreads();
  return before + x - v;
}

}  // namespace sunk
