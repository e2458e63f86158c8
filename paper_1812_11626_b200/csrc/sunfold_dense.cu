// sunfold_dense.cu — dense unfold of a GKSL generator given by a rate matrix A (include/sunfold.h,
// sun_unfold_dense).  SURVEY §8(f) F3 ("a 'dense', randomly generated, rate matrix A
// ... N = 100 ... more than 10^3 realizations") and the general-A half of F4 (Eq. 7).
//
//   L(X) = -i[H, X] + sum_jk a_jk (F_j X F_k - 1/2 {F_k F_j, X})      (Eq. 7 with F_k^+ = F_k)
//   Q_sm = Tr(F_s L(F_m)),  K_s = Tr(F_s L(I/N))
//
// No structure constants and no contraction: in the matrix-unit basis the superoperator is
//   S[(ab),(cd)] = [L(E_cd)]_ab = Y[(a,c),(d,b)] + (-i Kh)_ac d_db + d_ac (i Kh^+)_db,
//   Y = Fm A Fm^T  (Fm[(a,c), j] = (F_j)_ac),  G = sum_jk a_jk F_k F_j,  Kh = H - (i/2) G,
// and Q = (basis change of S on both sides).  Every basis change is a 2 x 2 combination
// (S_ab, J_ab have two entries) or a prefix / suffix sum over the diagonal (D^l), so the whole
// unfold is O(M^2) = O(N^4) and HBM-bound.  Two streaming passes carry the bulk:
//   k_dense_expand   A rows S(p), J(p) -> Z[b][a][c][d] = Y[(a,c),(d,b)] for (a,c) = p, (c,a)
//                    (Z is Y realigned so that each pass reads and writes contiguous runs)
//   k_dense_project  Z rows (x,y), (y,x) (+ the Kh terms) -> Q rows S(p), J(p) and K
// plus O(N^3) kernels for the D^l rows/columns (k_dense_dexp, k_dense_zdiag, k_dense_kh,
// k_dense_vdiag, k_dense_drows).  Shares no code with the oracle (oracle/gks.py).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "sunfold.h"

int sunfold_cuda_fail(cudaError_t e);  // sunfold.cu: records the message for sun_status_string

namespace {

constexpr int DT = 256;  // threads per CTA
constexpr unsigned FULLM = 0xffffffffu;
constexpr double RS2 = 0.70710678118654752440;  // 1/sqrt(2)

struct DenseArgs {
  int n, batch;
  long long m, np;          // M = N^2 - 1, N(N-1)/2
  const double2* H;         // [batch][N][N]
  const double2* A;         // [batch][M][M] or null
  double* Q;                // [batch][M][M]
  double* K;                // [batch][M] or null
  double2* Z;               // [chunk][N^4]
  double2* UD;              // [chunk][N-1][N^2]  (U = A Fm^T on the D rows of A; reused for VD)
  double2* Kh;              // [chunk][N^2]
  int r0;                   // first realisation of this chunk
};

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cmuli(double2 a) { return make_double2(-a.y, a.x); }   // i a
__device__ __forceinline__ double2 cmulmi(double2 a) { return make_double2(a.y, -a.x); }  // -i a
__device__ __forceinline__ double inv_ll1(int l) { return 1.0 / sqrt((double)l * (double)(l + 1)); }

__device__ __forceinline__ long long pair_idx(long long n, long long u, long long w) {  // u < w
  return u * (2 * n - u - 1) / 2 + (w - u - 1);
}
// pair q -> (u, w), u < w (lexicographic)
__device__ __forceinline__ void pair_of(long long n, long long q, int& u, int& w) {
  const double t = 2.0 * (double)n - 1.0;
  const double disc = t * t - 8.0 * (double)q;
  long long a = (long long)floor((t - sqrt(disc > 0.0 ? disc : 0.0)) * 0.5);
  if (a < 0) a = 0;
  while (a > 0 && a * (2 * n - a - 1) / 2 > q) --a;
  while (a + 1 <= n - 2 && (a + 1) * (2 * n - a - 2) / 2 <= q) ++a;
  u = (int)a;
  w = (int)(a + 1 + (q - a * (2 * n - a - 1) / 2));
}

// Warp 0: diag[d] = sum_l delta_l(d) c_l for d in [0, n) from the D coefficients c_l = dv[l-1]
// (delta_l(d) = 1/sqrt(l(l+1)) for d < l, -l/sqrt(l(l+1)) for d = l, else 0; A.1).
// Suffix sums S(l) = sum_{l' >= l} w_l', w_l = c_l inv(l):  diag[l] = S(l) - (l+1) w_l,
// diag[0] = S(1).
__device__ void warp_diag_from_d(const double2* __restrict__ dv, double2* diag, int n) {
  const int lane = threadIdx.x & 31;
  double2 carry = make_double2(0.0, 0.0);
  for (int top = n - 1; top >= 1; top -= 32) {
    const int l = top - lane;
    const double2 w = l >= 1 ? cscale(dv[l - 1], inv_ll1(l)) : make_double2(0.0, 0.0);
    double2 s = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double x = __shfl_up_sync(FULLM, s.x, o), y = __shfl_up_sync(FULLM, s.y, o);
      if (lane >= o) {
        s.x += x;
        s.y += y;
      }
    }
    const double2 S = cadd(carry, s);
    if (l >= 1) diag[l] = csub(S, cscale(w, (double)(l + 1)));
    carry = make_double2(__shfl_sync(FULLM, S.x, 31), __shfl_sync(FULLM, S.y, 31));
  }
  if (lane == 0) diag[0] = carry;
}

// Warp 0: out[l-1] = (sum_{c<l} v_c - l v_l) / sqrt(l(l+1)) for l in [1, n) (Tr(D^l X) from the
// diagonal v of X; A.1), and *tot = sum_c v_c.  Only real parts are needed.
__device__ void warp_d_from_diag(const double* v, double* out, double* tot, int n) {
  const int lane = threadIdx.x & 31;
  double carry = 0.0;
  for (int base = 0; base < n; base += 32) {
    const int c = base + lane;
    const double x = c < n ? v[c] : 0.0;
    double s = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(FULLM, s, o);
      if (lane >= o) s += y;
    }
    const double excl = carry + s - x;  // sum_{c' < c}
    if (c >= 1 && c < n) out[c - 1] = (excl - (double)c * x) * inv_ll1(c);
    carry += __shfl_sync(FULLM, s, 31);
  }
  if (lane == 0) *tot = carry;
}

// U = A Fm^T on one row of A (length M): U[(d,b)] = sum_k a_k (F_k)_db, for d != b the 2-term
// combination over S(min,max), J(min,max); for d == b the suffix table `diag`.
__device__ __forceinline__ double2 expand_entry(const double2* __restrict__ arow, const double2* diag, long long n,
                                                long long np, int d, int b) {
  if (d == b) return diag[d];
  const bool lo = d < b;
  const long long q = lo ? pair_idx(n, d, b) : pair_idx(n, b, d);
  const double2 s = __ldg(arow + q), j = __ldg(arow + np + q);
  // (S_q)_db = 1/sqrt2;  (J_q)_db = -i/sqrt2 if d < b, +i/sqrt2 if d > b
  return cscale(cadd(s, lo ? cmulmi(j) : cmuli(j)), RS2);
}

// (1) U rows of the D^l rows of A: UD[l-1][b][d] = sum_k A[D^l][k] (F_k)_db.  grid (N-1, chunk)
__global__ void __launch_bounds__(DT) k_dense_dexp(const DenseArgs g) {
  extern __shared__ double2 sdiag[];  // [N]
  const int n = g.n, r = blockIdx.y, l = blockIdx.x + 1;
  const long long m = g.m, np = g.np, n2 = (long long)n * n;
  const double2* arow = g.A + (long long)(g.r0 + r) * m * m + (2 * np + l - 1) * m;
  if (threadIdx.x < 32) warp_diag_from_d(arow + 2 * np, sdiag, n);
  __syncthreads();
  double2* out = g.UD + ((long long)r * (n - 1) + (l - 1)) * n2;
  for (long long t = threadIdx.x; t < n2; t += DT) {
    const int b = (int)(t / n), d = (int)(t % n);
    out[t] = expand_entry(arow, sdiag, n, np, d, b);
  }
}

// (2) the pair rows: CTA per pair p = (x, y), x < y.  U rows S(p), J(p) on the fly, then
//   Y[(x,y),(d,b)] = (U_S - i U_J)/sqrt2,  Y[(y,x),(d,b)] = (U_S + i U_J)/sqrt2
// written to Z[b][x][y][d] and Z[b][y][x][d] (contiguous in d).  The (b, d) plane is walked in
// 16 x 16 tiles on and above the diagonal (d >= b), one tile per warp at a time (warp-private
// staging, no CTA barrier): each A entry pair(b, d) is read once (contiguous in d) and gives
// both (d, b) -- written directly, d fastest -- and the mirrored (b, d) position, staged in
// shared memory and written out transposed.  grid (np, chunk)
constexpr int TW = 16;           // warp tile edge
constexpr int WPC = DT / 32;     // warps per CTA
struct WarpTile {
  double2 a[TW][TW + 1], b[TW][TW + 1];
};
__device__ __forceinline__ double2 jcomb(double2 s, double2 j, bool minus) {  // (s -+ i j)/sqrt2
  return cscale(cadd(s, minus ? cmulmi(j) : cmuli(j)), RS2);
}
// WP (small N, a single tile per row): warp per pair instead of CTA per pair, WPC pairs per CTA.
template <bool WP>
__global__ void __launch_bounds__(DT, 2) k_dense_expand(const DenseArgs g) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpTile& T = reinterpret_cast<WarpTile*>(dsm)[wid];
  const int n = g.n, r = blockIdx.y;
  const long long m = g.m, np = g.np, n2 = (long long)n * n;
  const long long p = WP ? (long long)blockIdx.x * WPC + wid : blockIdx.x;
  if (WP && p >= np) return;  // warp-uniform; no CTA barrier in WP mode
  double2* sdiag = reinterpret_cast<double2*>(dsm + WPC * sizeof(WarpTile)) + (WP ? wid * 2 * n : 0);  // [2][N]
  int x, y;
  pair_of(n, p, x, y);
  const double2* A = g.A + (long long)(g.r0 + r) * m * m;
  const double2 *aS = A + p * m, *aJ = A + (np + p) * m;
  if constexpr (WP) {
    warp_diag_from_d(aS + 2 * np, sdiag, n);
    warp_diag_from_d(aJ + 2 * np, sdiag + n, n);
    __syncwarp();
  } else {
    if (wid == 0)
      warp_diag_from_d(aS + 2 * np, sdiag, n);
    else if (wid == 1)
      warp_diag_from_d(aJ + 2 * np, sdiag + n, n);
    __syncthreads();
  }
  double2* Z = g.Z + (long long)r * n2 * n2;
  double2* zxy = Z + ((long long)x * n + y) * n;  // + b N^3 + d
  double2* zyx = Z + ((long long)y * n + x) * n;
  const long long n3 = n2 * n;
  const int nt = (n + TW - 1) / TW;
  const int hi = lane >> 4, lo = lane & 15;
  int cnt = 0;
  // Only the half b <= a of Z is stored (Z[b][a][c][d] = conj(Z[a][b][d][c]) for Hermitian A,
  // see k_dense_project; the plane b = a feeds G and the D rows): Z[b][x][.][.] for b <= x,
  // Z[b][y][.][.] for b <= y.  A tile with b0 > y (so every b, d > y) has no output and is not
  // read: its A entries reach Q through the conjugate entries of the rows (b, d) (A Hermitian).
  const int tmax = y / TW + 1;  // tiles with b0 <= y
  for (int tb = 0; tb < tmax; ++tb) {
    for (int td = tb; td < nt; ++td) {
      if (!WP && cnt++ % WPC != wid) continue;  // warp-uniform
      const int b0 = tb * TW, d0 = td * TW;
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // two batches of 4 rows: all loads first, then the math
        double2 sS[4], sJ[4], jS[4], jJ[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int b = b0 + 8 * h + 2 * k + hi, d = d0 + lo;
          const bool ok = b < n && d < n && d > b;
          const long long q = ok ? pair_idx(n, b, d) : 0;  // a valid address either way
          sS[k] = __ldg(aS + q);
          sJ[k] = __ldg(aS + np + q);
          jS[k] = __ldg(aJ + q);
          jJ[k] = __ldg(aJ + np + q);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int i = 8 * h + 2 * k + hi, j = lo;
          const int b = b0 + i, d = d0 + j;
          if (b < n && d < n && d >= b) {
            double2 uS, uJ;  // U at (d, b)
            if (d == b) {
              uS = sdiag[d];
              uJ = sdiag[n + d];
            } else {
              // (S_q)_db = (S_q)_bd = 1/sqrt2; (J_q)_db = +i/sqrt2 (d > b), (J_q)_bd = -i/sqrt2
              uS = jcomb(sS[k], sJ[k], false);
              uJ = jcomb(jS[k], jJ[k], false);
              const double2 vS = jcomb(sS[k], sJ[k], true), vJ = jcomb(jS[k], jJ[k], true);  // U at (b, d)
              T.a[i][j] = jcomb(vS, vJ, true);   // Y[(x,y),(b,d)] -> Z[d][x][y][b]
              T.b[i][j] = jcomb(vS, vJ, false);  // Y[(y,x),(b,d)] -> Z[d][y][x][b]
            }
            if (b <= x) zxy[b * n3 + d] = jcomb(uS, uJ, true);
            if (b <= y) zyx[b * n3 + d] = jcomb(uS, uJ, false);
          }
        }
      }
      __syncwarp();
#pragma unroll 4
      for (int k = 0; k < TW / 2; ++k) {
        const int i = 2 * k + hi, j = lo;  // row d = d0 + i, column b = b0 + j
        const int d = d0 + i, b = b0 + j;
        if (b < n && d < n && d > b) {
          if (d <= x) zxy[(long long)d * n3 + b] = T.a[j][i];
          if (d <= y) zyx[(long long)d * n3 + b] = T.b[j][i];
        }
      }
      __syncwarp();
    }
  }
}

// (3) the diagonal rows a = c = x:  Z[b][x][x][d] = sum_l delta_l(x) UD[l-1][b][d] (suffix sums
// over l).  grid (ceil(N^2 / DT), chunk), thread per (b, d)
__global__ void __launch_bounds__(DT) k_dense_zdiag(const DenseArgs g) {
  const int n = g.n, r = blockIdx.y;
  const long long n2 = (long long)n * n;
  const long long t = (long long)blockIdx.x * DT + threadIdx.x;
  if (t >= n2) return;
  const int b = (int)(t / n), d = (int)(t % n);
  const double2* ud = g.UD + (long long)r * (n - 1) * n2 + t;
  double2* Z = g.Z + (long long)r * n2 * n2 + (long long)b * n2 * n + d;  // + (x N + x) N
  double2 S = make_double2(0.0, 0.0);
#pragma unroll 8
  for (int l = n - 1; l >= 1; --l) {
    const double2 w = cscale(ud[(long long)(l - 1) * n2], inv_ll1(l));
    Z[((long long)l * n + l) * n] = csub(S, cscale(w, (double)l));
    S = cadd(S, w);
  }
  Z[0] = S;
}

// (4) G_ce = sum_x Z[x][x][e][c] (= sum_jk a_jk (F_k F_j)_ce) and Kh = H - (i/2) G.
// grid (ceil(N^2 / DT), chunk), thread per (e, c)
__global__ void __launch_bounds__(DT) k_dense_kh(const DenseArgs g) {
  const int n = g.n, r = blockIdx.y;
  const long long n2 = (long long)n * n;
  const long long t = (long long)blockIdx.x * DT + threadIdx.x;
  if (t >= n2) return;
  const int e = (int)(t / n), c = (int)(t % n);
  double2 G = make_double2(0.0, 0.0);
  if (g.A) {
    const double2* Z = g.Z + (long long)r * n2 * n2 + t;
#pragma unroll 8
    for (int x = 0; x < n; ++x) G = cadd(G, Z[((long long)x * n + x) * n2]);
  }
  const double2 h = g.H[(long long)(g.r0 + r) * n2 + (long long)c * n + e];
  g.Kh[(long long)r * n2 + (long long)c * n + e] = make_double2(h.x + 0.5 * G.y, h.y - 0.5 * G.x);
}

// the Kh terms of S in Z coordinates (added to a raw Z value)
__device__ __forceinline__ double2 zdelta(double2 z, const double2* __restrict__ kh, int n, int b, int a, int c, int d) {
  if (d == b) z = cadd(z, cmulmi(__ldg(kh + (long long)a * n + c)));
  if (a == c) {
    const double2 k = __ldg(kh + (long long)b * n + d);
    z = cadd(z, cmuli(make_double2(k.x, -k.y)));
  }
  return z;
}
// S in Z coordinates: Z'[b][a][c][d] = Z[b][a][c][d] + (-i Kh_ac) [d == b] + (i conj(Kh_bd)) [a == c]
__device__ __forceinline__ double2 zprime(const double2* __restrict__ zrow, const double2* __restrict__ kh, int n,
                                          bool has_a, int b, int a, int c, int d) {
  double2 z = has_a ? __ldg(zrow + (long long)c * n + d) : make_double2(0.0, 0.0);
  if (d == b) z = cadd(z, cmulmi(__ldg(kh + (long long)a * n + c)));
  if (a == c) {
    const double2 k = __ldg(kh + (long long)b * n + d);
    z = cadd(z, cmuli(make_double2(k.x, -k.y)));
  }
  return z;
}

// (5) the pair rows of Q: CTA per pair p = (x, y).  Rows (b,a) = (x,y), (y,x) of Z':
//   V_S = (Z'_xy + Z'_yx)/sqrt2,  V_J = (-i Z'_xy + i Z'_yx)/sqrt2     [(F_s)_ba weights]
//   Q[s][S(u,w)] = Re(V_s[u,w] + V_s[w,u])/sqrt2,  Q[s][J(u,w)] = Re(-i V_s[u,w] + i V_s[w,u])/sqrt2
//   Q[s][D^l] from the diagonal V_s[c,c] (prefix sums), K_s = sum_c Re V_s[c,c] / N.
// The (u, w) plane (u < w) is walked in 16 x 16 tiles, one per warp at a time: the transposed
// blocks Z'[w][u] of both rows are staged in warp-private shared memory (contiguous loads),
// the direct blocks Z'[u][w] are read in the compute phase (contiguous); outputs pair(u, w)
// go out in runs of consecutive pairs.  grid (np, chunk)
template <bool WP>
__global__ void __launch_bounds__(DT, 2) k_dense_project(const DenseArgs g) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpTile& T = reinterpret_cast<WarpTile*>(dsm)[wid];
  const int n = g.n, r = blockIdx.y;
  const long long m = g.m, np = g.np, n2 = (long long)n * n;
  const long long p = WP ? (long long)blockIdx.x * WPC + wid : blockIdx.x;
  if (WP && p >= np) return;  // warp-uniform; no CTA barrier in WP mode
  // [2][N] diagonal of V_S, V_J
  double* sv = reinterpret_cast<double*>(dsm + WPC * sizeof(WarpTile)) + (WP ? wid * 2 * n : 0);
  int x, y;
  pair_of(n, p, x, y);
  const bool has_a = g.A != nullptr;
  const double2* Z = g.Z + (long long)r * n2 * n2;
  // Row (b,a) = (x,y) of Z' only: L preserves Hermiticity (H and A Hermitian), so
  // S[(ab),(cd)] = conj(S[(ba),(dc)]), i.e. Z'[y][x][c][d] = conj(Z'[x][y][d][c]); the row (y,x)
  // is the conjugate transpose of the row (x,y) (and the expand stores only Z[b][a], b <= a).
  const double2* zxy = Z + ((long long)x * n + y) * n2;  // row (b,a) = (x,y)
  const double2* kh = g.Kh + (long long)r * n2;
  double* qS = g.Q + (long long)(g.r0 + r) * m * m + p * m;
  double* qJ = qS + np * m;
  const int nt = (n + TW - 1) / TW;
  const int hi = lane >> 4, lo = lane & 15;
  int cnt = 0;
  for (int tu = 0; tu < nt; ++tu) {
    for (int tw = tu; tw < nt; ++tw) {
      if (!WP && cnt++ % WPC != wid) continue;  // warp-uniform
      const int u0 = tu * TW, w0 = tw * TW;
      {  // stage the transposed block Z'_xy[w][u]: all loads first
        double2 za[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int i = 2 * k + hi, j = lo;  // row w = w0 + i, column u = u0 + j
          const bool ok = has_a && w0 + i < n && u0 + j < n;
          const long long o = ok ? (long long)(w0 + i) * n + (u0 + j) : 0;
          za[k] = ok ? __ldg(zxy + o) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int i = 2 * k + hi, j = lo;
          if (w0 + i < n && u0 + j < n) T.a[i][j] = zdelta(za[k], kh, n, x, y, w0 + i, u0 + j);
        }
      }
      __syncwarp();
      double2 za[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {  // direct block Z'_xy[u][w]: all loads first
        const int u = u0 + 2 * k + hi, w = w0 + lo;
        const bool ok = has_a && u < w && w < n;
        const long long o = ok ? (long long)u * n + w : 0;
        za[k] = ok ? __ldg(zxy + o) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int k = 0; k < TW / 2; ++k) {
        const int i = 2 * k + hi, j = lo;  // u = u0 + i, w = w0 + j
        const int u = u0 + i, w = w0 + j;
        if (u < w && w < n) {
          // a = Z'_xy, b = Z'_yx: b1 = Z'_yx[u][w] = conj(Z'_xy[w][u]), b2 = Z'_yx[w][u] = conj(Z'_xy[u][w])
          const double2 a1 = zdelta(za[k], kh, n, x, y, u, w), a2 = T.a[j][i];
          const double2 b1 = make_double2(a2.x, -a2.y), b2 = make_double2(a1.x, -a1.y);
          // V_S at (u,w), (w,u) and V_J at (u,w), (w,u)
          const double2 s1 = cscale(cadd(a1, b1), RS2), s2 = cscale(cadd(a2, b2), RS2);
          const double2 j1 = cscale(cadd(cmulmi(a1), cmuli(b1)), RS2), j2 = cscale(cadd(cmulmi(a2), cmuli(b2)), RS2);
          const long long q = pair_idx(n, u, w);
          // Re(V1 + V2)/sqrt2 and Re(-i V1 + i V2)/sqrt2 = (Im V1 - Im V2)/sqrt2
          qS[q] = (s1.x + s2.x) * RS2;
          qS[np + q] = (s1.y - s2.y) * RS2;
          qJ[q] = (j1.x + j2.x) * RS2;
          qJ[np + q] = (j1.y - j2.y) * RS2;
        }
      }
      __syncwarp();
    }
  }
  for (int c = WP ? lane : (int)threadIdx.x; c < n; c += WP ? 32 : DT) {
    const double2 a = zprime(zxy, kh, n, has_a, x, y, c, c);  // Z'_yx[c][c] = conj(a)
    sv[c] = (a.x + a.x) * RS2;            // Re V_S[c,c] = Re(a + conj a)/sqrt2
    sv[n + c] = (a.y + a.y) * RS2;        // Re V_J[c,c] = Re((-i a + i conj a)/sqrt2)
  }
  __shared__ double tot_all[WPC][2];
  double* tot = tot_all[WP ? wid : 0];
  if constexpr (WP) {
    __syncwarp();
    warp_d_from_diag(sv, qS + 2 * np, &tot[0], n);
    warp_d_from_diag(sv + n, qJ + 2 * np, &tot[1], n);
    __syncwarp();
  } else {
    __syncthreads();
    if (wid == 0)
      warp_d_from_diag(sv, qS + 2 * np, &tot[0], n);
    else if (wid == 1)
      warp_d_from_diag(sv + n, qJ + 2 * np, &tot[1], n);
    __syncthreads();
  }
  if (g.K && (WP ? lane == 0 : threadIdx.x == 0)) {
    double* K = g.K + (long long)(g.r0 + r) * m;
    K[p] = tot[0] / n;
    K[np + p] = tot[1] / n;
  }
}

// (6) V rows of the D^l rows of Q: VD[l-1][(c,d)] = sum_x delta_l(x) Z'[x][x][c][d] (prefix sums
// over x).  grid (ceil(N^2 / DT), chunk), thread per (c, d).  VD reuses the UD buffer.
__global__ void __launch_bounds__(DT) k_dense_vdiag(const DenseArgs g) {
  const int n = g.n, r = blockIdx.y;
  const long long n2 = (long long)n * n;
  const long long t = (long long)blockIdx.x * DT + threadIdx.x;
  if (t >= n2) return;
  const int c = (int)(t / n), d = (int)(t % n);
  const bool has_a = g.A != nullptr;
  const double2* Z = g.Z + (long long)r * n2 * n2;
  const double2* kh = g.Kh + (long long)r * n2;
  double2* vd = g.UD + (long long)r * (n - 1) * n2 + t;
  double2 P = make_double2(0.0, 0.0);
#pragma unroll 8
  for (int xx = 0; xx < n; ++xx) {
    const double2 z = zprime(Z + ((long long)xx * n + xx) * n2, kh, n, has_a, xx, xx, c, d);
    if (xx >= 1) vd[(long long)(xx - 1) * n2] = cscale(csub(P, cscale(z, (double)xx)), inv_ll1(xx));
    P = cadd(P, z);
  }
}

// (7) Q rows D^l from VD: CTA per l.  grid (N-1, chunk)
__global__ void __launch_bounds__(DT) k_dense_drows(const DenseArgs g) {
  extern __shared__ double sv[];  // [N]
  const int n = g.n, r = blockIdx.y, l = blockIdx.x + 1;
  const long long m = g.m, np = g.np, n2 = (long long)n * n;
  const double2* V = g.UD + ((long long)r * (n - 1) + (l - 1)) * n2;
  const long long s = 2 * np + l - 1;
  double* qrow = g.Q + (long long)(g.r0 + r) * m * m + s * m;
  for (long long q = threadIdx.x; q < np; q += DT) {
    int u, w;
    pair_of(n, q, u, w);
    const double2 v1 = __ldg(V + (long long)u * n + w), v2 = __ldg(V + (long long)w * n + u);
    qrow[q] = (v1.x + v2.x) * RS2;
    qrow[np + q] = (v1.y - v2.y) * RS2;
  }
  for (int c = threadIdx.x; c < n; c += DT) sv[c] = V[(long long)c * n + c].x;
  __syncthreads();
  __shared__ double tot;
  if (threadIdx.x < 32) warp_d_from_diag(sv, qrow + 2 * np, &tot, n);
  __syncthreads();
  if (g.K && threadIdx.x == 0) g.K[(long long)(g.r0 + r) * m + s] = tot / n;
}

constexpr int DENSE_NMAX = 1024;  // shared-memory tables of 2N complex per CTA (<= 32 KB)

size_t per_realisation_bytes(long long n) {
  const long long n2 = n * n;
  auto al = [](long long b) { return (size_t)((b + 255) & ~255LL); };
  return al(16 * n2 * n2) + al(16 * (n - 1) * n2) + al(16 * n2);
}

}  // namespace

extern "C" {

size_t sun_dense_work_bytes(int32_t n, int32_t chunk) {
  if (n < 2 || n > DENSE_NMAX || chunk < 1) return 0;
  return per_realisation_bytes(n) * (size_t)chunk;
}

int sun_unfold_dense(int32_t n, int32_t batch, const double* H, const double* A, double* Q, double* K, void* work,
                     size_t work_bytes, void* stream) {
  if (n < 2 || n > DENSE_NMAX) return SUN_ERR_DIM;
  if (batch < 0) return SUN_ERR_ARG;
  if (batch == 0) return SUN_OK;
  if (!H || !Q || !work) return SUN_ERR_ARG;
  const size_t per = per_realisation_bytes(n);
  if (work_bytes < per) return SUN_ERR_CAPACITY;
  long long chunk = (long long)(work_bytes / per);
  if (chunk > batch) chunk = batch;
  if (chunk > 65535) chunk = 65535;
  cudaStream_t st = (cudaStream_t)stream;
  const long long nn = n, n2 = nn * nn;
  DenseArgs g;
  g.n = n;
  g.batch = batch;
  g.m = n2 - 1;
  g.np = nn * (nn - 1) / 2;
  g.H = reinterpret_cast<const double2*>(H);
  g.A = reinterpret_cast<const double2*>(A);
  g.Q = Q;
  g.K = K;
  char* ws = (char*)work;
  auto al = [](long long b) { return (size_t)((b + 255) & ~255LL); };
  g.Z = reinterpret_cast<double2*>(ws);
  g.UD = reinterpret_cast<double2*>(ws + chunk * al(16 * n2 * n2));
  g.Kh = reinterpret_cast<double2*>(ws + chunk * (al(16 * n2 * n2) + al(16 * (nn - 1) * n2)));
  const unsigned gsq = (unsigned)((n2 + DT - 1) / DT);
  // N <= 2 TW: at most 3 tiles of 16 x 16 per pair row, so one warp per pair (WPC pairs per CTA)
#ifndef SUN_DENSE_WP_MAXN
#define SUN_DENSE_WP_MAXN 32
#endif
  const bool wp = n <= SUN_DENSE_WP_MAXN;
  const size_t sm_exp = WPC * sizeof(WarpTile) + (wp ? WPC : 1) * 2 * n * sizeof(double2);
  const size_t sm_prj = WPC * sizeof(WarpTile) + (wp ? WPC : 1) * 2 * n * sizeof(double);
  const unsigned gpair = (unsigned)(wp ? (g.np + WPC - 1) / WPC : g.np);
  {
    cudaError_t e = cudaFuncSetAttribute(wp ? k_dense_expand<true> : k_dense_expand<false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_exp);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(wp ? k_dense_project<true> : k_dense_project<false>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_prj);
    if (e != cudaSuccess) return sunfold_cuda_fail(e);
  }
  for (long long r0 = 0; r0 < batch; r0 += chunk) {
    const unsigned cb = (unsigned)(batch - r0 < chunk ? batch - r0 : chunk);
    g.r0 = (int)r0;
    if (A) {
      k_dense_dexp<<<dim3((unsigned)(n - 1), cb), DT, n * sizeof(double2), st>>>(g);
      if (wp)
        k_dense_expand<true><<<dim3(gpair, cb), DT, sm_exp, st>>>(g);
      else
        k_dense_expand<false><<<dim3(gpair, cb), DT, sm_exp, st>>>(g);
      k_dense_zdiag<<<dim3(gsq, cb), DT, 0, st>>>(g);
    }
    k_dense_kh<<<dim3(gsq, cb), DT, 0, st>>>(g);
    if (wp)
      k_dense_project<true><<<dim3(gpair, cb), DT, sm_prj, st>>>(g);
    else
      k_dense_project<false><<<dim3(gpair, cb), DT, sm_prj, st>>>(g);
    k_dense_vdiag<<<dim3(gsq, cb), DT, 0, st>>>(g);
    k_dense_drows<<<dim3((unsigned)(n - 1), cb), DT, n * sizeof(double), st>>>(g);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return sunfold_cuda_fail(e);
  }
  return SUN_OK;
}

int sun_dense_launches(int32_t n, int32_t batch, int32_t has_a, size_t work_bytes) {
  if (n < 2 || n > DENSE_NMAX || batch <= 0) return 0;
  const size_t per = per_realisation_bytes(n);
  if (work_bytes < per) return 0;
  long long chunk = (long long)(work_bytes / per);
  if (chunk > batch) chunk = batch;
  if (chunk > 65535) chunk = 65535;
  const long long chunks = (batch + chunk - 1) / chunk;
  return (int)(chunks * (has_a ? 7 : 4));
}

}  // extern "C"
