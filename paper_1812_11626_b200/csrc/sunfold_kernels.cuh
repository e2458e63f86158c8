// sunfold_kernels.cuh — sm_100a fp64 device code of the SU(N) unfold (arXiv:1812.11626).
//
// Row s of Q is the generator expansion of the Hermitian matrix G_s = L^+(F_s), where
//   L^+(X) = i[H, X] + sum_p gamma_p (L_p^+ X L_p - 1/2 {L_p^+ L_p, X})
// is the Hilbert-Schmidt adjoint of the GKSL generator (Eq. 1):
//   Q_sm = Tr(F_s L(F_m)) = Tr(L^+(F_s) F_m),   K_s = Tr(F_s L(I/N)) = Tr(L^+(F_s))/N.
// This is the paper's contraction of Eq. 6 (q_sn = sum_m f_mns h_m) and Eqs. 10-11
// (R = -1/2 gamma Re(Y^H X), K; P:200-211 with readings R1/R2) evaluated per output row: the
// structure constants f_mns = -i Tr(F_s[F_m,F_n]) and d_mns = Tr(F_s{F_m,F_n}) (Eq. 4,
// P:152-158) are traces of products of matrix units E_ab E_cd = delta_bc E_ad, so their
// nonzero index patterns (the "triangle" class for generators sharing one index,
// the "pair" class for coincident pairs, and the D^l chains) are enumerated here as the
// support of G_s inside small index windows; no f/d tensor is stored.
// DESIGN.md gives the derivation.
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

#include <type_traits>

namespace sunk {

constexpr int WMAX = 15;               // max(wK, wL) supported by the banded kernels
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
  const double2* L;    // P bands of half-width wL (sqrt(gamma)-scaled)
  const double* inv;   // inv[l] = 1/sqrt(l(l+1)), l = 1..n-1
  const double* tau_ptr;  // drop threshold in device memory (computed by the expand step)
  double tau;             // loaded from tau_ptr at kernel entry
  int mode;            // 0 group-per-pair far kernels (compile-time widths), 1 warp-per-pair (runtime widths)
  int tp;              // pairs per tile (one scan slot per tile for the S rows, one for the J rows)
  long long npt, ndt;  // pair tiles, D slots
  long long nb_near;   // mode 0: units of 8 near-pair / D-row items (one warp each)
};

// Programmatic dependent launch (sm_90+): a kernel launched with the PDL attribute may start
// while its predecessor in the stream still runs; griddepcontrol.wait blocks until the
// predecessor grid has completed and its writes are visible (a no-op without the attribute).
// Every kernel of the unfold sequence waits before touching global memory, then lets its own
// dependents launch, so the next kernel's CTAs are resident when this one ends.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_trigger();
}

// (x, y) += conj(la) lb with every rounding explicit: the compiler has no contraction choice
// left, so each evaluation of a value (count pass, fill pass, matrix-free stages; whatever
// kernel it is inlined into) performs the identical operations and the passes take identical
// tau decisions.
__device__ __forceinline__ void conj_mul_acc(double& x, double& y, const double2 la, const double2 lb) {
  x = __fma_rn(la.x, lb.x, __fma_rn(la.y, lb.y, x));   // two fused operations per component
  y = __fma_rn(la.x, lb.y, __fma_rn(-la.y, lb.x, y));
}

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

// p(c,d) = c(2n-c-1)/2 + (d-c-1) < 2^31 for n <= 46340 (unsigned intermediate < 2^32)
__device__ __forceinline__ int pidx32(int n, int c, int d) {
  const unsigned uc = (unsigned)c;
  return (int)((uc * (2u * (unsigned)n - uc - 1u)) / 2u + (unsigned)(d - c - 1));
}

// pair index p -> (a, b), a < b < n, lexicographic (R5)
// (fp32 square-root estimate, |error| <= a few rows for n <= 46340, fixed by the exact integer
// corrections below)
// Unsigned 32-bit arithmetic throughout (p < NP <= 1.07e9 and a (2n - a - 1) <= n^2 < 2^32 for
// n <= 46340): the 64-bit multiplies of the corrections cost ~10 % of the count pass.
__device__ __forceinline__ void pair_decode(long long n_, long long p_, int& a_out, int& b_out) {
  const unsigned n = (unsigned)n_, p = (unsigned)p_;
  const unsigned t2 = 2u * n - 1u;
  const long long d = (long long)((unsigned long long)t2 * t2) - 8ll * p;  // exact, then one rounding
  const float disc = (float)d;
  int ai = (int)(((float)t2 - sqrtf(disc > 0.0f ? disc : 0.0f)) * 0.5f);
  if (ai < 0) ai = 0;
  if (ai > (int)n - 2) ai = (int)n - 2;
  unsigned a = (unsigned)ai;
  auto first = [n](unsigned x) { return (x * (2u * n - x - 1u)) >> 1; };  // index of pair (x, x + 1)
  while (a > 0u && first(a) > p) --a;
  while (a + 2u <= n - 1u && first(a + 1u) <= p) ++a;
  a_out = (int)a;
  b_out = (int)(a + 1u + (p - first(a)));
}

// Pairs p_first + lane of a warp: decode once (lane 0), then walk.
__device__ __forceinline__ void warp_pairs(int n, long long p_first, int& a, int& b) {
  const int lane = threadIdx.x & 31;
  int a0 = 0, b0 = 1;
  if (lane == 0) pair_decode(n, p_first, a0, b0);
  a0 = __shfl_sync(FULL, a0, 0);
  b0 = __shfl_sync(FULL, b0, 0);
  int k = lane;
  a = a0;
  b = b0;
  while (b + k >= n) {
    if (a >= n - 2) {  // past the last pair (caller masks p >= NP)
      a = n - 2;
      b = n - 1;
      k = 0;
      break;
    }
    k -= n - b;
    a += 1;
    b = a + 1;
  }
  b += k;
}

// Pairs of a warp whose first pair (a0, b0) is known (every lane holds it): the walk of
// warp_pairs without the decode.
__device__ __forceinline__ void warp_pairs_from(int n, int a0, int b0, int& a, int& b) {
  int k = threadIdx.x & 31;
  a = a0;
  b = b0;
  while (b + k >= n) {
    if (a >= n - 2) {  // past the last pair (caller masks p >= NP)
      a = n - 2;
      b = n - 1;
      k = 0;
      break;
    }
    k -= n - b;
    a += 1;
    b = a + 1;
  }
  b += k;
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

// U = L^+(E_ab) element (c, d), general (runtime band widths)
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
      conj_mul_acc(ux, uy, la, lb);  // conj(la) * lb
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

// ---------------------------------------------------------------------------------------
// Output sink: a contiguous CSR segment in global memory (writes beyond the capacity dropped).
// ---------------------------------------------------------------------------------------
struct Seg {
  int32_t* gcol;  // global col/val pointers already offset to the segment start
  double* gval;
  long long lim;  // entries writable from the segment start (output capacity - start)
  __device__ __forceinline__ void emit(long long off, int col, double v) const {
    if (off < lim) {
      gcol[off] = col;
      gval[off] = v;
    }
  }
};

// ---------------------------------------------------------------------------------------
// Warp / block helpers
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ int warp_excl_scan(int v, int& total) {
  const int lane = threadIdx.x & 31;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  total = __shfl_sync(FULL, x, 31);
  return x - v;
}

// Block-wide exclusive scan of one int per thread (blockDim.x <= 1024, multiple of 32).
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

// ---------------------------------------------------------------------------------------
// Last l in (hi, n-1] with |tr * inv[l]| > tau (hi if none).  The predicate is monotone
// (non-increasing) in l, so the answer is unique; it is located from the estimate
// l ~ |tr|/tau - 1/2 (inv[l] ~ 1/(l + 1/2)) checked by the 32 lanes in parallel, with a
// binary search as fallback.  Warp-uniform result, identical in the count and fill passes.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ int chain_tail_end(const double* inv, int n, int hi, double tr, double tau) {
  const int lane = threadIdx.x & 31;
  if (hi + 1 > n - 1) return hi;
  const double atr = fabs(tr);
  if (!(atr * __ldg(&inv[hi + 1]) > tau)) return hi;       // nothing kept beyond the window
  if (atr * __ldg(&inv[n - 1]) > tau) return n - 1;          // everything kept
  double est = atr / tau - 0.5;
  long long e = est > (double)(n - 1) ? (long long)(n - 1) : (long long)est;
  int base = (int)e - 15;
  if (base < hi + 1) base = hi + 1;
  if (base > n - 32) base = n - 32 > hi + 1 ? n - 32 : hi + 1;
  const int l = base + lane;
  const bool in = l <= n - 1;
  const bool kept = in && fabs(tr * __ldg(&inv[l])) > tau;
  const unsigned km = __ballot_sync(FULL, kept), im = __ballot_sync(FULL, in);
  // kept lanes must form a prefix of the in-range lanes, boundary strictly inside the window
  if (km != 0u && km != im && (km & (km + 1u)) == 0u) return base + __popc(km) - 1;
  if (km == 0u && base == hi + 1) return hi;  // (cannot happen: inv[hi+1] kept)
  int lo_b = hi + 1, hi_b = n - 1;            // fallback: binary search (lo_b kept)
  while (lo_b < hi_b) {
    const int mid = (lo_b + hi_b + 1) >> 1;
    if (fabs(tr * __ldg(&inv[mid])) > tau)
      lo_b = mid;
    else
      hi_b = mid - 1;
  }
  return lo_b;
}

// Exclusive prefix sums pre[0..nw] of g[0..nw-1] (shared, per warp) by warp shuffles in
// 32-element chunks (fixed tree order: deterministic, same in both passes).
__device__ __forceinline__ void warp_prefix(const double* g, double* pre, int nw) {
  const int lane = threadIdx.x & 31;
  double carry = 0.0;
  for (int i0 = 0; i0 < nw; i0 += 32) {
    const int i = i0 + lane;
    const double v = i < nw ? g[i] : 0.0;
    double x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    if (i < nw) pre[i] = carry + (x - v);
    carry += __shfl_sync(FULL, x, 31);
  }
  if (lane == 0) pre[nw] = carry;
  __syncwarp();
}

// ---------------------------------------------------------------------------------------
// D^l chain of one row from its diagonal g over the window [lo, hi] (warp-cooperative).
// pre[j] = sum_{i<j} g[i] (j = 0..nw) in ascending order.  For l > hi the coefficient is
// tr * inv[l] with |tr * inv[l]| non-increasing in l (correctly rounded sqrt, division and
// product are monotone), so the kept tail is (hi, lend], found by binary search -- identical
// in the count and fill passes.  Returns the kept count; with EMIT writes them at seg/off.
// ---------------------------------------------------------------------------------------
// Tail of a row's D-chain: entries tr * inv[l] for l in (hi, lend], after `nwin` entries
// (the row's S/J window entries and its D entries inside the window).
struct TailInfo {
  double tr;
  int nwin, hi, lend;
  int n1, n2;  // split side rows (SEG > 0): entries of segments 1 and 2 (segment 3 = nwin - n1 - n2)
};

// Side buffer of the near rows (row 2i = S row / D row of near item i, 2i+1 = J row).
// Side row slot of nc = NW^2 entries (NW = 4W + 1), three segments written in one pass:
// [0, seg) the row's S_cd entries, [seg, 2 seg) its J_cd entries, [2 seg, ..) its D^l entries
// inside the window; seg = NW (NW - 1) / 2.  The output row is seg 1, seg 2, seg 3, tail.
struct NearMeta {
  double tr, k;     // D-chain trace (tail value tr * inv[l]) and the row's K value
  int n1, n2, nd;   // entries of the three segments
  int hi, lend;     // chain tail: l in (hi, lend]
  int pad;
};
struct NearSide {
  int32_t* col;  // [2 * items * nc]
  double* val;   // [2 * items * nc]
  NearMeta* meta;
  int nc;        // entries per row slot: (4W + 1)^2
  int seg;       // segment stride: (4W + 1) 4W / 2
};


template <bool EMIT, bool TAIL = true>
__device__ __forceinline__ int warp_dchain(const Prob& pr, int lo, int hi, const double* g, const double* pre,
                                           const Seg& seg, long long off, int nbefore = 0, TailInfo* ti = nullptr) {
  const int lane = threadIdx.x & 31;
  const int n = pr.n;
  const double tau = pr.tau;
  const int nw = hi - lo + 1;
  const double tr = pre[nw];
  const int dbase = (int)(2 * pr.np - 1);  // column of D^l is 2NP + l - 1
  const double* inv = pr.inv;
  int kept = 0;
  const int lstart = lo < 1 ? 1 : lo;
  for (int l0 = lstart; l0 <= hi; l0 += 32) {  // inside the window
    const int l = l0 + lane;
    double coef = 0.0;
    const bool valid = l <= hi;
    if (valid) coef = (pre[l - lo] - (double)l * g[l - lo]) * __ldg(&inv[l]);
    const bool keep = valid && fabs(coef) > tau;
    const unsigned km = __ballot_sync(FULL, keep);
    if (EMIT && keep) seg.emit(off + kept + __popc(km & ((1u << lane) - 1u)), dbase + l, coef);
    kept += __popc(km);
  }
  const int lend = chain_tail_end(inv, n, hi, tr, tau);  // tail beyond the window: l in (hi, lend]
  if (EMIT && TAIL) {
    for (int l = hi + 1 + lane; l <= lend; l += 32)
      seg.emit(off + kept + (l - hi - 1), dbase + l, tr * __ldg(&inv[l]));
  }
  if (ti) *ti = TailInfo{tr, nbefore + kept, hi, lend};
  return kept + (lend - hi);
}

// ---------------------------------------------------------------------------------------
// Both rows (S_ab, J_ab) of a near pair (b - a <= 2W), warp-cooperative.
// TW > 0: U = L^+(E_ab) is first evaluated once on its support tile [a-W, a+W] x [b-W, b+W]
//         (TW = 2W + 1 entries per side, one lane per entry) into shared memory; the window
//         positions then read the tile.  TW == 0: every value through U_elem (wide bands).
// scr: per-warp shared scratch: tile (TW*TW double2) | gS | gJ | pS | pJ (each SW doubles).
// Returns the row lengths (cS, cJ) and K values (kS, kJ); with EMIT writes the rows.
// ---------------------------------------------------------------------------------------
// SEG > 0 (with EMIT): split side rows, one pass (segments at offS, offS + SEG, offS + 2 SEG).
template <bool EMIT, int TW, int SW, bool TAIL = true, int SEG = 0>
__device__ __forceinline__ void warp_near_pair(const Prob& pr, int a, int b, double* scr, int& cS, int& cJ, double& kS,
                                            double& kJ, Seg sS, long long offS, Seg sJ, long long offJ,
                                            TailInfo* tS = nullptr, TailInfo* tJ = nullptr) {
  const int lane = threadIdx.x & 31;
  const int n = pr.n, W = pr.W;
  const int np = (int)pr.np;
  const double tau = pr.tau;
  double2* tile = reinterpret_cast<double2*>(scr);
  double* gS = scr + 2 * TW * TW;
  double* gJ = gS + SW;
  double* pS = gJ + SW;
  double* pJ = pS + SW;
  const int lo = a - W < 0 ? 0 : a - W;
  const int hi = b + W > n - 1 ? n - 1 : b + W;
  const int nw = hi - lo + 1;
  const int npos = nw * (nw - 1) / 2;
  const unsigned lt = (1u << lane) - 1u;
  if constexpr (TW > 0) {
    for (int k = lane; k < TW * TW; k += 32) {
      const int c = a - W + k / TW, d = b - W + k % TW;
      tile[k] = (c >= 0 && d < n) ? U_elem(pr, a, b, c, d) : make_double2(0.0, 0.0);
    }
    __syncwarp();
  }
  auto U = [&](int c, int d) -> double2 {
    if constexpr (TW > 0) {
      const int i = c - (a - W), j = d - (b - W);
      return (i >= 0 && i < TW && j >= 0 && j < TW) ? tile[i * TW + j] : make_double2(0.0, 0.0);
    } else {
      return U_elem(pr, a, b, c, d);
    }
  };
  int n1S = 0, n2S = 0, n1J = 0, n2J = 0;
  constexpr bool SPLIT = EMIT && SEG > 0;
  if (!SPLIT)
  for (int k0 = 0; k0 < npos; k0 += 32) {
    const int k = k0 + lane;
    double v1S = 0, v2S = 0, v1J = 0, v2J = 0;
    if (k < npos) {
      int i, j;
      win_decode(nw, k, i, j);
      const double2 ucd = U(lo + i, lo + j), udc = U(lo + j, lo + i);
      v1S = ucd.x + udc.x;
      v2S = udc.y - ucd.y;
      v1J = ucd.y + udc.y;
      v2J = ucd.x - udc.x;
    }
    n1S += __popc(__ballot_sync(FULL, fabs(v1S) > tau));
    n2S += __popc(__ballot_sync(FULL, fabs(v2S) > tau));
    n1J += __popc(__ballot_sync(FULL, fabs(v1J) > tau));
    n2J += __popc(__ballot_sync(FULL, fabs(v2J) > tau));
  }
  if (EMIT) {
    // second halves: after the first (counted above) or at the fixed segment SEG (one pass)
    const long long o2S = SPLIT ? offS + SEG : offS + n1S, o2J = SPLIT ? offJ + SEG : offJ + n1J;
    int i1S = 0, i2S = 0, i1J = 0, i2J = 0;
    for (int k0 = 0; k0 < npos; k0 += 32) {
      const int k = k0 + lane;
      double v1S = 0, v2S = 0, v1J = 0, v2J = 0;
      int q = 0;
      if (k < npos) {
        int i, j;
        win_decode(nw, k, i, j);
        const double2 ucd = U(lo + i, lo + j), udc = U(lo + j, lo + i);
        v1S = ucd.x + udc.x;
        v2S = udc.y - ucd.y;
        v1J = ucd.y + udc.y;
        v2J = ucd.x - udc.x;
        q = pidx32(n, lo + i, lo + j);
      }
      bool kp;
      unsigned m;
      kp = fabs(v1S) > tau; m = __ballot_sync(FULL, kp);
      if (kp) sS.emit(offS + i1S + __popc(m & lt), q, v1S);
      i1S += __popc(m);
      kp = fabs(v2S) > tau; m = __ballot_sync(FULL, kp);
      if (kp) sS.emit(o2S + i2S + __popc(m & lt), np + q, v2S);
      i2S += __popc(m);
      kp = fabs(v1J) > tau; m = __ballot_sync(FULL, kp);
      if (kp) sJ.emit(offJ + i1J + __popc(m & lt), q, v1J);
      i1J += __popc(m);
      kp = fabs(v2J) > tau; m = __ballot_sync(FULL, kp);
      if (kp) sJ.emit(o2J + i2J + __popc(m & lt), np + q, v2J);
      i2J += __popc(m);
    }
    if (SPLIT) {
      n1S = i1S;
      n2S = i2S;
      n1J = i1J;
      n2J = i2J;
    }
  }
  const double s2 = 1.4142135623730951;
  for (int i = lane; i < nw; i += 32) {
    const double2 u = U(lo + i, lo + i);
    gS[i] = s2 * u.x;
    gJ[i] = s2 * u.y;
  }
  __syncwarp();
  warp_prefix(gS, pS, nw);
  warp_prefix(gJ, pJ, nw);
  const int chS = warp_dchain<EMIT, TAIL>(pr, lo, hi, gS, pS, sS, SPLIT ? offS + 2 * SEG : offS + n1S + n2S,
                                          n1S + n2S, tS);
  const int chJ = warp_dchain<EMIT, TAIL>(pr, lo, hi, gJ, pJ, sJ, SPLIT ? offJ + 2 * SEG : offJ + n1J + n2J,
                                          n1J + n2J, tJ);
  if (tS) {
    tS->n1 = n1S;
    tS->n2 = n2S;
  }
  if (tJ) {
    tJ->n1 = n1J;
    tJ->n2 = n2J;
  }
  cS = n1S + n2S + chS;
  cJ = n1J + n2J + chJ;
  kS = pS[nw] / (double)n;
  kJ = pJ[nw] / (double)n;
  __syncwarp();
}

// ---------------------------------------------------------------------------------------
// D^lam row, warp-cooperative.
// ---------------------------------------------------------------------------------------
template <bool EMIT, bool TAIL = true, int SEG = 0>
__device__ __forceinline__ int warp_d_row(const Prob& pr, int lam, double* g, double* pre, double& kval, Seg seg,
                                       long long off, TailInfo* ti = nullptr) {
  const int lane = threadIdx.x & 31;
  const int n = pr.n;
  const int np = (int)pr.np;
  const double tau = pr.tau;
  const double alpha = __ldg(&pr.inv[lam]);
  const int lo = lam - pr.wK < 0 ? 0 : lam - pr.wK;
  const int hi = lam + pr.wK > n - 1 ? n - 1 : lam + pr.wK;
  const int nw = hi - lo + 1;
  const int npos = nw * (nw - 1) / 2;
  const unsigned lt = (1u << lane) - 1u;
  const double s2 = 1.4142135623730951;
  int nS = 0, nJ = 0;
  constexpr bool SPLIT = EMIT && SEG > 0;
  if (!SPLIT)
  for (int k0 = 0; k0 < npos; k0 += 32) {
    const int k = k0 + lane;
    double vS = 0, vJ = 0;
    if (k < npos) {
      int i, j;
      win_decode(nw, k, i, j);
      const double2 gv = G_elem(pr, lam, alpha, lo + i, lo + j);
      vS = s2 * gv.x;
      vJ = -s2 * gv.y;
    }
    nS += __popc(__ballot_sync(FULL, fabs(vS) > tau));
    nJ += __popc(__ballot_sync(FULL, fabs(vJ) > tau));
  }
  if (EMIT) {
    const long long o2 = SPLIT ? off + SEG : off + nS;
    int iS = 0, iJ = 0;
    for (int k0 = 0; k0 < npos; k0 += 32) {
      const int k = k0 + lane;
      double vS = 0, vJ = 0;
      int q = 0;
      if (k < npos) {
        int i, j;
        win_decode(nw, k, i, j);
        const double2 gv = G_elem(pr, lam, alpha, lo + i, lo + j);
        vS = s2 * gv.x;
        vJ = -s2 * gv.y;
        q = pidx32(n, lo + i, lo + j);
      }
      bool kp = fabs(vS) > tau;
      unsigned m = __ballot_sync(FULL, kp);
      if (kp) seg.emit(off + iS + __popc(m & lt), q, vS);
      iS += __popc(m);
      kp = fabs(vJ) > tau;
      m = __ballot_sync(FULL, kp);
      if (kp) seg.emit(o2 + iJ + __popc(m & lt), np + q, vJ);
      iJ += __popc(m);
    }
    if (SPLIT) {
      nS = iS;
      nJ = iJ;
    }
  }
  for (int i = lane; i < nw; i += 32) g[i] = G_elem(pr, lam, alpha, lo + i, lo + i).x;
  __syncwarp();
  warp_prefix(g, pre, nw);
  const int ch = warp_dchain<EMIT, TAIL>(pr, lo, hi, g, pre, seg, SPLIT ? off + 2 * SEG : off + nS + nJ, nS + nJ, ti);
  if (ti) {
    ti->n1 = nS;
    ti->n2 = nJ;
  }
  kval = pre[nw] / (double)n;
  __syncwarp();
  return nS + nJ + ch;
}

// ---------------------------------------------------------------------------------------
#ifndef SUN_PB_WIDE
#define SUN_PB_WIDE 1  // far_values, runtime P, wL >= 1: dissipators whose band rows are loaded together (2: spills, c3 fill 96 -> 102 us)
#endif
// Far pair (b - a > 2W) with compile-time half-bandwidths (WK >= WL), thread per pair: the
// band values the pair needs are loaded up front (independent loads) and the NPOS values of
// U = L^+(E_ab) stay in registers.  Far positions, in lexicographic (dc, dd) order, which is
// ascending column order q(a + dc, b + dd):
//   dc = 0: dd in [-WK, WK];  0 < |dc| <= WL: dd in [-WL, WL];  WL < |dc| <= WK: dd = 0
// ---------------------------------------------------------------------------------------
template <int WK, int WL>
struct FarT {
  static_assert(WK >= WL, "far-pair kernels need wK >= wL");
  static constexpr int NPOS = (2 * WK + 1) + 2 * WL * (2 * WL + 1) + 2 * (WK - WL);
  static_assert(NPOS <= 64, "mask width");
  // kept-position bit masks: 32 bits, or 64 for wide bands (e.g. (wK, wL) = (4, 2): 33 positions)
  using Mask = typename std::conditional<(NPOS > 32), unsigned long long, unsigned>::type;
};
__device__ __forceinline__ int mpopc(unsigned m) { return __popc(m); }
__device__ __forceinline__ int mpopc(unsigned long long m) { return __popcll(m); }

template <int WK, int WL, class F>
__device__ __forceinline__ void far_foreach(F&& f) {
  int k = 0;
#pragma unroll
  for (int dc = -WK; dc <= WK; ++dc) {
    const int adc = dc < 0 ? -dc : dc;
    const int w = dc == 0 ? WK : (adc <= WL ? WL : 0);
#pragma unroll
    for (int dd = -w; dd <= w; ++dd) {
      f(k, dc, dd);
      ++k;
    }
  }
}

// The far-pair kernels' view of the problem (kept in registers).
struct FarCtx {
  const double2* K;  // band K, half-width WK
  const double2* L;  // P bands Lt_p, half-width WL
  double tau;
  long long np;
  int n, P;
};

// U_cd = i K_ca [d = b] - i conj(K_db) [c = a] + sum_p conj(Lt_p,ac) Lt_p,bd at all far positions.
// PT: dissipators known at compile time (0 or 1), -1 = runtime P.
template <int WK, int WL, int PT>
__device__ __forceinline__ void far_values(const FarCtx& pr, int a, int b, double (&ux)[FarT<WK, WL>::NPOS],
                                           double (&uy)[FarT<WK, WL>::NPOS]) {
  constexpr int W = WK;
  constexpr int SK = 2 * WK + 1, SL = 2 * WL + 1;
  const int n = pr.n;
  double2 kc[2 * W + 1], kr[2 * W + 1];
  // band rows through base pointers: compile-time offsets (i SK + 2W - i) from K(a - W, .)
  const double2* Ka = pr.K + (long long)(a - W) * SK;
  const double2* Kb = pr.K + (long long)(b - W) * SK;
#pragma unroll
  for (int i = 0; i <= 2 * W; ++i) {
    const int c = a + i - W;  // K(c, a): row c, offset a - c = W - i
    kc[i] = c >= 0 ? __ldg(Ka + (i * SK + 2 * W - i)) : make_double2(0.0, 0.0);
    const int d = b + i - W;  // K(d, b): row d, offset b - d = W - i
    kr[i] = d < n ? __ldg(Kb + (i * SK + 2 * W - i)) : make_double2(0.0, 0.0);
  }
  // outer block O_ij = sum_p conj(Lt_p(a, a-WL+i)) Lt_p(b, b-WL+j)
  double ox[SL][SL], oy[SL][SL];
#pragma unroll
  for (int i = 0; i < SL; ++i)
#pragma unroll
    for (int j = 0; j < SL; ++j) ox[i][j] = oy[i][j] = 0.0;
  if constexpr (PT > 0) {
    for (int p = 0; p < PT; ++p) {
      const double2* La = pr.L + ((long long)p * n + a) * SL;
      const double2* Lb = pr.L + ((long long)p * n + b) * SL;
      double2 la[SL], lb[SL];
#pragma unroll
      for (int i = 0; i < SL; ++i) {
        la[i] = __ldg(&La[i]);
        lb[i] = __ldg(&Lb[i]);
      }
#pragma unroll
      for (int i = 0; i < SL; ++i)
#pragma unroll
        for (int j = 0; j < SL; ++j) {
          conj_mul_acc(ox[i][j], oy[i][j], la[i], lb[j]);
        }
    }
  } else if constexpr (PT < 0) {
    // runtime P: the band rows of PB dissipators are loaded together before their first use
    // (one L2 round trip per PB dissipators instead of one per dissipator); the accumulation
    // order p = 0, 1, ... is unchanged, so every value is bitwise the same
    constexpr int PB = SL == 1 ? 8 : SUN_PB_WIDE;
    const long long ps = (long long)n * SL;
    const double2* La = pr.L + (long long)a * SL;
    const double2* Lb = pr.L + (long long)b * SL;
    for (int p0 = 0; p0 < pr.P; p0 += PB) {
      double2 la[PB][SL], lb[PB][SL];
#pragma unroll
      for (int u = 0; u < PB; ++u)
#pragma unroll
        for (int i = 0; i < SL; ++i) {
          const bool in = p0 + u < pr.P;
          la[u][i] = in ? __ldg(La + (p0 + u) * ps + i) : make_double2(0.0, 0.0);
          lb[u][i] = in ? __ldg(Lb + (p0 + u) * ps + i) : make_double2(0.0, 0.0);
        }
#pragma unroll
      for (int u = 0; u < PB; ++u) {
        if (p0 + u < pr.P) {
#pragma unroll
          for (int i = 0; i < SL; ++i)
#pragma unroll
            for (int j = 0; j < SL; ++j) conj_mul_acc(ox[i][j], oy[i][j], la[u][i], lb[u][j]);
        }
      }
    }
  }
  far_foreach<WK, WL>([&](int k, int dc, int dd) {
    const int adc = dc < 0 ? -dc : dc, add = dd < 0 ? -dd : dd;
    double x = 0.0, y = 0.0;
    if (PT != 0 && adc <= WL && add <= WL) {
      x = ox[dc + WL][dd + WL];
      y = oy[dc + WL][dd + WL];
    }
    if (dd == 0) {  // + i K_ca
      x -= kc[dc + W].y;
      y += kc[dc + W].x;
    }
    if (dc == 0) {  // - i conj(K_db)
      x -= kr[dd + W].y;
      y -= kr[dd + W].x;
    }
    ux[k] = x;
    uy[k] = y;
  });
}

// kept bits of the far positions: bit k of mr (Re U) / mi (Im U), |.| > tau and in range
template <int WK, int WL>
__device__ __forceinline__ void far_masks(int n, double tau, int a, int b, const double (&ux)[FarT<WK, WL>::NPOS],
                                          const double (&uy)[FarT<WK, WL>::NPOS], typename FarT<WK, WL>::Mask& mr,
                                          typename FarT<WK, WL>::Mask& mi) {
  using M = typename FarT<WK, WL>::Mask;
  M r = 0u, i = 0u;
  far_foreach<WK, WL>([&](int k, int dc, int dd) {
    const bool ok = (dc >= 0 || a + dc >= 0) && (dd <= 0 || b + dd < n);
    r |= (M)(ok && fabs(ux[k]) > tau) << k;
    i |= (M)(ok && fabs(uy[k]) > tau) << k;
  });
  mr = r;
  mi = i;
}

// column indices q(a + dc, b + dd) of the far positions (S_cd; J_cd is NP + q)
template <int WK, int WL>
__device__ __forceinline__ void far_cols(int n, int a, int b, int (&q)[FarT<WK, WL>::NPOS]) {
  const int q0 = pidx32(n, a, b);
  far_foreach<WK, WL>([&](int k, int dc, int dd) {
    // rows c = a + dc < 0 are masked out; clamp keeps the arithmetic in range
    const int c = a + dc < 0 ? 0 : a + dc;
    q[k] = dc == 0 ? q0 + dd : pidx32(n, c, b + dd);
  });
}

// column bases of the far positions: q(a + dc, b + dd) = qb[dc + WK] + dd (p(c, d) is linear in d;
// 2 WK + 1 registers instead of NPOS)
template <int WK>
__device__ __forceinline__ void far_colbase(int n, int a, int b, int (&qb)[2 * WK + 1]) {
#pragma unroll
  for (int dc = -WK; dc <= WK; ++dc) {
    const int c = a + dc < 0 ? 0 : a + dc;  // rows c < 0 are masked out
    qb[dc + WK] = pidx32(n, c, b);
  }
}

// Predicated shared stores of one staged entry (col, val) at 32-bit shared addresses; the
// addresses advance by the kept bit (branch-free: no divergence, no reconvergence code).
__device__ __forceinline__ void sts_entry(unsigned keep, unsigned& pc, unsigned& pv, int col, double val) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t@p st.shared.u32 [%1], %2;\n\t@p st.shared.f64 [%3], %4;\n\t}" ::"r"(keep),
      "r"(pc), "r"(col), "r"(pv), "d"(val)
      : "memory");
  pc += keep << 2;
  pv += keep << 3;
}

// Stage one row of a far pair (ROW 0 = S_ab, ROW 1 = J_ab) at scol/sval[off ..]:
//   row S_ab: [Re U at q] [-Im U at NP + q];   row J_ab: [Im U at q] [Re U at NP + q]
// Two running pointers (first and second half of the row), one predicated store pair per
// position and half; the masks are consumed bit by bit.
template <int WK, int WL, int ROW>
__device__ __forceinline__ void far_stage_row(int np, const int (&qb)[2 * WK + 1],
                                              const double (&ux)[FarT<WK, WL>::NPOS],
                                              const double (&uy)[FarT<WK, WL>::NPOS], typename FarT<WK, WL>::Mask mr,
                                              typename FarT<WK, WL>::Mask mi, int* scol, double* sval, int off) {
  typename FarT<WK, WL>::Mask m1 = ROW ? mi : mr, m2 = ROW ? mr : mi;
  const int off2 = off + mpopc(m1);
  unsigned pc1 = (unsigned)__cvta_generic_to_shared(scol + off), pv1 = (unsigned)__cvta_generic_to_shared(sval + off);
  unsigned pc2 = (unsigned)__cvta_generic_to_shared(scol + off2), pv2 = (unsigned)__cvta_generic_to_shared(sval + off2);
  far_foreach<WK, WL>([&](int k, int dc, int dd) {
    const int q = qb[dc + WK] + dd;
    const double v1 = ROW ? uy[k] : ux[k];
    const double v2 = ROW ? ux[k] : -uy[k];
    sts_entry((unsigned)(m1 & 1u), pc1, pv1, q, v1);
    sts_entry((unsigned)(m2 & 1u), pc2, pv2, np + q, v2);
    m1 >>= 1;
    m2 >>= 1;
  });
}

// ---------------------------------------------------------------------------------------
// TMA 1D bulk store (cp.async.bulk, sm_90+): shared -> global, 16-byte aligned, bulk_group
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, unsigned bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(ssrc);
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---------------------------------------------------------------------------------------
// Far pair, warp-cooperative (mode 1): lane k of each 32-chunk owns far position k
// (pos_dc/pos_dd: offsets in lexicographic order).  Pass 1 counts; EMIT pass 2 writes.
// ---------------------------------------------------------------------------------------
// Count word of a mode-1 far pair's S row: bits 0-19 the row length, 20-31 nR (the kept Re
// parts), so the fill pass emits in one pass.
constexpr int CNT_BITS = 20;
constexpr int CNT_MASK = (1 << CNT_BITS) - 1;

// nR_known >= 0 (EMIT only): the kept counts are known (nR, total - nR): pass 1 is skipped.
template <bool EMIT>
__device__ __forceinline__ int warp_far_pair(const Prob& pr, int a, int b, const int* pos_dc, const int* pos_dd,
                                             int npos, const Seg& sS, long long offS, const Seg& sJ,
                                             long long offJ, int* nR_out = nullptr, int nR_known = -1,
                                             int total_known = 0) {
  const int lane = threadIdx.x & 31;
  const int n = pr.n;
  const int np = (int)pr.np;
  const double tau = pr.tau;
  const unsigned lt = (1u << lane) - 1u;
  int nR = 0, nI = 0;
  if (EMIT && nR_known >= 0) {
    nR = nR_known;
    nI = total_known - nR_known;
  } else
  for (int k0 = 0; k0 < npos; k0 += 32) {
    const int k = k0 + lane;
    bool okr = false, oki = false;
    if (k < npos) {
      const int c = a + pos_dc[k], d = b + pos_dd[k];
      if (c >= 0 && c < n && d < n) {
        const double2 u = U_elem(pr, a, b, c, d);
        okr = fabs(u.x) > tau;
        oki = fabs(u.y) > tau;
      }
    }
    nR += __popc(__ballot_sync(FULL, okr));
    nI += __popc(__ballot_sync(FULL, oki));
  }
  if (EMIT) {
    int iR = 0, iI = 0;
    for (int k0 = 0; k0 < npos; k0 += 32) {
      const int k = k0 + lane;
      bool okr = false, oki = false;
      double2 u = make_double2(0.0, 0.0);
      int q = 0;
      if (k < npos) {
        const int c = a + pos_dc[k], d = b + pos_dd[k];
        if (c >= 0 && c < n && d < n) {
          u = U_elem(pr, a, b, c, d);
          okr = fabs(u.x) > tau;
          oki = fabs(u.y) > tau;
          q = pidx32(n, c, d);
        }
      }
      const unsigned mr = __ballot_sync(FULL, okr), mi = __ballot_sync(FULL, oki);
      if (okr) {
        const int r = iR + __popc(mr & lt);
        sS.emit(offS + r, q, u.x);
        sJ.emit(offJ + nI + r, np + q, u.x);
      }
      if (oki) {
        const int r = iI + __popc(mi & lt);
        sS.emit(offS + nR + r, np + q, -u.y);
        sJ.emit(offJ + r, q, u.y);
      }
      iR += __popc(mr);
      iI += __popc(mi);
    }
  }
  if (nR_out) *nR_out = nR;
  return nR + nI;
}

// ---------------------------------------------------------------------------------------
// Far pair, warp-cooperative with compile-time widths (mode 1 fast path for wide bands):
// lane j owns far positions k = h 32 + j (h < NCH) of the fixed lexicographic list
// (far_foreach order).  The values of both rounds stay in registers between the count and
// the emit, so the fill emits in one pass.  PT: dissipators at compile time (0, 1), -1 runtime.
// ---------------------------------------------------------------------------------------
template <int WK, int WL>
__device__ __forceinline__ void far_pos(int k, int& dc, int& dd) {
  int idx = 0;
  dc = 0;
  dd = 0;
#pragma unroll
  for (int c = -WK; c <= WK; ++c) {
    const int ac = c < 0 ? -c : c;
    const int w = (c == 0) ? WK : (ac <= WL ? WL : 0);
    if (k >= idx && k < idx + 2 * w + 1) {
      dc = c;
      dd = k - idx - w;
    }
    idx += 2 * w + 1;
  }
}

// U at far position k of pair (a, b) (the same expression wherever it is evaluated: the count
// and fill passes must take identical tau decisions); returns whether the position is in range
template <int WK, int WL, int PT>
__device__ __forceinline__ bool far_value_at(const Prob& pr, int a, int b, int k, double& x, double& y, int& c,
                                             int& d) {
  constexpr int NPOS = FarT<WK, WL>::NPOS;
  constexpr int SK = 2 * WK + 1, SL = 2 * WL + 1;
  const int n = pr.n;
  const int P = PT < 0 ? pr.P : PT;
  int dc, dd;
  far_pos<WK, WL>(k < NPOS ? k : 0, dc, dd);
  c = a + dc;
  d = b + dd;
  const bool ok = k < NPOS && c >= 0 && d < n;
  x = 0.0;
  y = 0.0;
  if (ok) {
    const int adc = dc < 0 ? -dc : dc, add = dd < 0 ? -dd : dd;
    // every load is issued before the first use: the K terms, then the dissipators four at a
    // time (the accumulation order, p = 0, 1, ..., is the same whatever the batching)
    const double2 kca = dd == 0 ? __ldg(&pr.K.v[(long long)c * SK + (WK - dc)]) : make_double2(0.0, 0.0);
    const double2 kdb = dc == 0 ? __ldg(&pr.K.v[(long long)d * SK + (WK - dd)]) : make_double2(0.0, 0.0);
    if (PT != 0 && adc <= WL && add <= WL) {
      const double2* La = pr.L + (long long)a * SL + (dc + WL);
      const double2* Lb = pr.L + (long long)b * SL + (dd + WL);
      const long long ps = (long long)n * SL;
      for (int p0 = 0; p0 < P; p0 += 4) {
        double2 la[4], lb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          la[i] = p0 + i < P ? __ldg(La + (p0 + i) * ps) : make_double2(0.0, 0.0);
          lb[i] = p0 + i < P ? __ldg(Lb + (p0 + i) * ps) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (p0 + i < P) conj_mul_acc(x, y, la[i], lb[i]);  // conj(Lt_p,ac) Lt_p,bd
      }
    }
    if (dd == 0) {  // + i K_ca
      x -= kca.y;
      y += kca.x;
    }
    if (dc == 0) {  // - i conj(K_db)
      x -= kdb.y;
      y -= kdb.x;
    }
  }
  return ok;
}

template <int WK, int WL, int PT, bool EMIT>
__device__ __forceinline__ int far_warp_pair(const Prob& pr, int a, int b, const Seg& sS, long long offS,
                                             const Seg& sJ, long long offJ, int* nR_out = nullptr) {
  constexpr int NPOS = FarT<WK, WL>::NPOS, NCH = (NPOS + 31) / 32;
  const int lane = threadIdx.x & 31;
  const int n = pr.n, np = (int)pr.np;
  const double tau = pr.tau;
  const unsigned lt = (1u << lane) - 1u;
  double ux[NCH], uy[NCH];
  unsigned mr[NCH], mi[NCH];
  int qq[NCH];
  int nR = 0, nI = 0;
#pragma unroll
  for (int h = 0; h < NCH; ++h) {
    const int k = h * 32 + lane;
    double x, y;
    int c, d;
    const bool ok = far_value_at<WK, WL, PT>(pr, a, b, k, x, y, c, d);
    ux[h] = x;
    uy[h] = y;
    qq[h] = ok ? pidx32(n, c, d) : 0;
    mr[h] = __ballot_sync(FULL, ok && fabs(x) > tau);
    mi[h] = __ballot_sync(FULL, ok && fabs(y) > tau);
    nR += __popc(mr[h]);
    nI += __popc(mi[h]);
  }
  if (EMIT) {
    int bR = 0, bI = 0;
#pragma unroll
    for (int h = 0; h < NCH; ++h) {
      const int rR = bR + __popc(mr[h] & lt), rI = bI + __popc(mi[h] & lt);
      if ((mr[h] >> lane) & 1u) {
        sS.emit(offS + rR, qq[h], ux[h]);
        sJ.emit(offJ + nI + rR, np + qq[h], ux[h]);
      }
      if ((mi[h] >> lane) & 1u) {
        sS.emit(offS + nR + rI, np + qq[h], -uy[h]);
        sJ.emit(offJ + rI, qq[h], uy[h]);
      }
      bR += __popc(mr[h]);
      bI += __popc(mi[h]);
    }
  }
  if (nR_out) *nR_out = nR;
  return nR + nI;
}

}  // namespace sunk
