// sunfold_general.cu — mode 3 of the unfold: operators of any pattern (sunfold_general.cuh).
//
// Launches per sun_count: k_g_expand (a1: validation, norms, Hermiticity, inv[l], tau, column
// counts of the dissipators), k_g_colscan, k_g_scatter, k_g_colsort (column access of every
// L_p, sorted by row: deterministic), k_g_light<count> (a3: warp per generator pair, rows with
// at most GW_CAP candidate terms), k_g_heavy<count> (a3: CTA per D row and per heavier pair,
// key-range chunks).  Per sun_unfold: k_g_light<fill>, k_g_heavy<fill> (a5).  The scan (a4) is
// sunfold.cu's chained scan over the same slot layout as modes 0/2.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "sunfold_general.cuh"
#include "sunfold_kernels.cuh"

namespace sung {
namespace {

constexpr unsigned FULLM = 0xffffffffu;
constexpr int GF_MALFORMED = 1, GF_TOOBIG = 16;  // header flags (sunfold.cu F_*)
constexpr int GE_THREADS = 256;                  // expand: rows per CTA
#ifndef SUN_GW_CAP
#define SUN_GW_CAP 256
#endif
#ifndef SUN_GW_WARPS
#define SUN_GW_WARPS 8
#endif
constexpr int GW_CAP = SUN_GW_CAP, GW_WARPS = SUN_GW_WARPS;  // light engine: candidates per warp, warps per CTA
constexpr int GH_CAP = 2048, GH_NT = 256;        // heavy engine: candidates per CTA, threads
constexpr int GH_NB = 256, GH_LEV = 4;           // heavy engine: histogram bins, levels
constexpr double SQ2 = 1.4142135623730951;

struct GBlk {
  double nrm2;
  unsigned long long herm;
  int flags;
  int pad;
};

__device__ __forceinline__ double2 cjmul(double2 a, double2 b) {  // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ long long lbound(const int32_t* __restrict__ ci, long long lo, long long hi, int c) {
  while (lo < hi) {  // first k in [lo, hi) with ci[k] >= c
    const long long mid = (lo + hi) >> 1;
    if (__ldg(ci + mid) < c) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ long long ubound(const int32_t* __restrict__ ci, long long lo, long long hi, int c) {
  while (lo < hi) {  // first k in [lo, hi) with ci[k] > c
    const long long mid = (lo + hi) >> 1;
    if (__ldg(ci + mid) <= c) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// =========================================================================================
// (a1) expand for mode 3
// =========================================================================================
struct GExpandArgs {
  GExpandIn in;
  GBlk* blk;
  int* colcnt;  // P x (n + 1), zeroed before the launch
  double* inv;
  int* zero32;
  unsigned long long* zero64;
  long long nz32, nz64;
  GHeaderRef hdr;
  int nrb, nA, nB;
};

__global__ void __launch_bounds__(GE_THREADS) k_g_expand(const GExpandArgs A) {
  const GExpandIn& in = A.in;
  const int n = in.n;
  const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gstride = (long long)gridDim.x * blockDim.x;
  for (long long i = gtid; i < A.nz32; i += gstride) A.zero32[i] = 0;
  for (long long i = gtid; i < A.nz64; i += gstride) A.zero64[i] = 0ull;
  if (gtid == 0) A.hdr.ticket[0] = A.hdr.ticket[1] = 0u;
  __shared__ double red[GE_THREADS];
  __shared__ int sfl[GE_THREADS / 32];
  __shared__ unsigned long long sh[GE_THREADS / 32];
  __shared__ int last;
  if ((int)blockIdx.x < A.nA) {
    const int op = blockIdx.x / A.nrb, rb = blockIdx.x % A.nrb;
    const int r = rb * blockDim.x + threadIdx.x;
    double acc = 0.0;
    int flags = 0;
    unsigned long long hd = 0ull;
    if (!(op == 1 && !in.has_h1) && r < n) {
      const int64_t* rp = in.rp[op];
      const int32_t* ci = in.ci[op];
      const double2* v = in.v[op];
      const int64_t lo = rp[r], hi = rp[r + 1];
      if (hi < lo) flags |= GF_MALFORMED;
      int prev = -1;
      for (int64_t k = lo; k < hi; ++k) {
        const int c = ci[k];
        if (c < 0 || c >= n || c <= prev) { flags |= GF_MALFORMED; break; }
        prev = c;
        const double2 x = v[k];
        acc += x.x * x.x + x.y * x.y;
        if (op < 2) {  // Hermiticity: compare with the transposed entry (0 if absent)
          const int64_t b0 = rp[c], b1 = rp[c + 1];
          const long long q = b1 > b0 ? lbound(ci, b0, b1, r) : b1;
          double2 t = make_double2(0.0, 0.0);
          if (q < b1 && ci[q] == r) t = v[q];
          const double d = fmax(fabs(x.x - t.x), fabs(x.y + t.y));
          const unsigned long long db = (unsigned long long)__double_as_longlong(d);
          hd = db > hd ? db : hd;
        } else {
          atomicAdd(&A.colcnt[(long long)(op - 2) * (n + 1) + c], 1);
        }
      }
    }
    red[threadIdx.x] = acc;
    int wf = flags;
    unsigned long long wh = hd;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      wf |= __shfl_xor_sync(FULLM, wf, o);
      const unsigned long long t = __shfl_xor_sync(FULLM, wh, o);
      wh = t > wh ? t : wh;
    }
    if ((threadIdx.x & 31) == 0) {
      sfl[threadIdx.x >> 5] = wf;
      sh[threadIdx.x >> 5] = wh;
    }
    __syncthreads();
    for (int st = GE_THREADS / 2; st > 0; st >>= 1) {  // fixed-order tree: deterministic
      if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      int f = 0;
      unsigned long long h = 0ull;
      for (int i = 0; i < GE_THREADS / 32; ++i) {
        f |= sfl[i];
        h = sh[i] > h ? sh[i] : h;
      }
      A.blk[blockIdx.x] = GBlk{red[0], h, f, 0};
    }
  } else {
    const long long t = (long long)(blockIdx.x - A.nA) * blockDim.x + threadIdx.x;
    if (t < n) A.inv[t] = t > 0 ? 1.0 / sqrt((double)t * (double)(t + 1)) : 0.0;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(A.hdr.done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last || threadIdx.x >= 32) return;
  __threadfence();
  const int lane = threadIdx.x;
  int flags = 0;
  double s0 = 0.0;
  unsigned long long hm[2] = {0ull, 0ull};
  for (int op = 0; op < in.nops; ++op) {
    if (op == 1 && !in.has_h1) continue;
    double acc = 0.0;
    unsigned long long h = 0ull;
    for (int i = lane; i < A.nrb; i += 32) {  // fixed order per lane, then a fixed tree
      const GBlk bi = A.blk[op * A.nrb + i];
      acc += bi.nrm2;
      h = bi.herm > h ? bi.herm : h;
      flags |= bi.flags;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      acc += __shfl_xor_sync(FULLM, acc, o);
      const unsigned long long t = __shfl_xor_sync(FULLM, h, o);
      h = t > h ? t : h;
    }
    if (op < 2) hm[op] = h;
    if (lane == 0) {
      A.hdr.nrm2[op] = acc;
      if (op == 0) s0 += sqrt(acc);
      if (op >= 2) s0 += in.gamma[op] * acc;
      if (op < 2) A.hdr.nrm2_h[op] = acc;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) flags |= __shfl_xor_sync(FULLM, flags, o);
  if (lane == 0) {
    *A.hdr.flags = flags;
    A.hdr.herm[0] = hm[0];
    A.hdr.herm[1] = in.has_h1 ? hm[1] : 0ull;
    A.hdr.tau[0] = 1e-14 * s0;
    A.hdr.tau[1] = in.has_h1 ? 1e-14 * sqrt(A.hdr.nrm2_h[1]) : 0.0;
    if (!in.has_h1) A.hdr.nrm2_h[1] = 0.0;
    *A.hdr.done = 0u;
  }
}

// column counts -> column pointers (exclusive scan, one CTA per dissipator); the counters
// become the scatter cursors
__global__ void __launch_bounds__(1024) k_g_colscan(int n, int* colcnt, int* cp) {
  const int p = blockIdx.x;
  int* cc = colcnt + (long long)p * (n + 1);
  int* out = cp + (long long)p * (n + 1);
  __shared__ int ws[32];
  __shared__ int carry_s;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int v = i < n ? cc[i] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULLM, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int w = lane < (int)(blockDim.x >> 5) ? ws[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULLM, w, o);
        if (lane >= o) w += y;
      }
      ws[lane] = w;
    }
    __syncthreads();
    const int ex = carry_s + (wid > 0 ? ws[wid - 1] : 0) + x - v;
    if (i < n) {
      out[i] = ex;
      cc[i] = ex;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry_s = ex + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = carry_s;
}

struct GColArgs {
  const int64_t* rp[GMAXP];
  const int32_t* ci[GMAXP];
  int2* xr[GMAXP];
  int n, P;
};

// (x, k) of every entry into its column's segment (order within a column fixed by k_g_colsort)
__global__ void k_g_scatter(const GColArgs A, int* cur) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)A.P * A.n) return;
  const int p = (int)(t / A.n), x = (int)(t % A.n);
  const int64_t* rp = A.rp[p];
  const int32_t* ci = A.ci[p];
  int* cc = cur + (long long)p * (A.n + 1);
  for (int64_t k = rp[x]; k < rp[x + 1]; ++k) {
    const int slot = atomicAdd(&cc[ci[k]], 1);
    A.xr[p][slot] = make_int2(x, (int)k);
  }
}

// sort each column segment by row (warp per column): bitonic in shared memory up to 256
// entries; longer columns are rebuilt in row order by scanning the rows for the column
__global__ void __launch_bounds__(256) k_g_colsort(const GColArgs A, const int* cp) {
  __shared__ int2 buf[8][256];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long t = (long long)blockIdx.x * 8 + wid;
  if (t >= (long long)A.P * A.n) return;
  const int p = (int)(t / A.n), c = (int)(t % A.n);
  const int* cpp = cp + (long long)p * (A.n + 1);
  const int b = cpp[c], e = cpp[c + 1], len = e - b;
  if (len <= 1) return;
  int2* xr = A.xr[p];
  if (len <= 256) {
    int n2 = 32;
    while (n2 < len) n2 <<= 1;
    for (int i = lane; i < n2; i += 32) buf[wid][i] = i < len ? xr[b + i] : make_int2(0x7fffffff, 0);
    __syncwarp();
    for (int k = 2; k <= n2; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = lane; i < n2; i += 32) {
          const int ij = i ^ j;
          if (ij > i) {
            const int2 u = buf[wid][i], w = buf[wid][ij];
            const bool asc = (i & k) == 0;
            if ((u.x > w.x) == asc) {
              buf[wid][i] = w;
              buf[wid][ij] = u;
            }
          }
        }
        __syncwarp();
      }
    for (int i = lane; i < len; i += 32) xr[b + i] = buf[wid][i];
    return;
  }
  const int64_t* rp = A.rp[p];
  const int32_t* ci = A.ci[p];
  int o = b;
  for (int x0 = 0; x0 < A.n; x0 += 32) {
    const int x = x0 + lane;
    int pos = -1;
    if (x < A.n) {
      const long long q = lbound(ci, rp[x], rp[x + 1], c);
      if (q < rp[x + 1] && ci[q] == c) pos = (int)q;
    }
    const unsigned m = __ballot_sync(FULLM, pos >= 0);
    if (pos >= 0) xr[o + __popc(m & ((1u << lane) - 1u))] = make_int2(x, pos);
    o += __popc(m);
  }
}

// =========================================================================================
// Candidate enumeration (identical in every pass)
// =========================================================================================
struct Item {
  int kind;  // 0: generator pair (a, b) -> rows S_ab and J_ab;  1: row D^lam
  int a, b, lam;
  double alpha;  // inv[lam]
};

__device__ __forceinline__ unsigned key_of(const GProb& G, int r, int s, int& tr) {
  if (r == s) {
    tr = 0;
    return (unsigned)(G.np + r);
  }
  if (r < s) {
    tr = 0;
    return (unsigned)sunk::pidx32(G.n, r, s);
  }
  tr = 1;
  return (unsigned)sunk::pidx32(G.n, s, r);
}

__device__ __forceinline__ long long num_sources(const GProb& G, const Item& it) {
  if (it.kind == 1) return (long long)it.lam + 1 + (long long)G.P * G.n;
  long long s = 2;
  for (int p = 0; p < G.P; ++p) {
    const int* cp = G.C[p].cp;
    s += (long long)(__ldg(cp + it.a + 1) - __ldg(cp + it.a)) + (__ldg(cp + it.b + 1) - __ldg(cp + it.b)) +
         (G.L[p].rp[it.a + 1] - G.L[p].rp[it.a]);
  }
  return s;
}

__device__ __forceinline__ double fD(const Item& it, int c) {
  return c < it.lam ? it.alpha : (c == it.lam ? -(double)it.lam * it.alpha : 0.0);
}

// Source `src` of item `it`: number of candidates (COUNT_ONLY) or emit them as
// vis(key, seq, value, transposed) with seq = seq0 + local index.  part / nparts: emit only the
// part-th of nparts interleaved slices (frame mode splits one source over a group; every source
// emits pairwise distinct keys); seq is meaningful only for nparts == 1.
template <bool COUNT_ONLY, bool NEEDVAL, class V>
__device__ __forceinline__ unsigned long long source(const GProb& G, const Item& it, long long src, unsigned seq0,
                                                     V& vis, int part = 0, int nparts = 1) {
  const int n = G.n;
  if (it.kind == 1) {  // ---- row D^lam
    const int lam = it.lam;
    if (src <= lam) {  // TH: row c = src of H, d >= max(lam, c + 1)
      const int c = (int)src;
      const long long r0 = G.H.rp[c], r1 = G.H.rp[c + 1];
      const long long k0 = lbound(G.H.ci, r0, r1, lam > c + 1 ? lam : c + 1);
      if (COUNT_ONLY) return (unsigned long long)(r1 - k0);
      const double fc = fD(it, c);
      for (long long k = k0 + part; k < r1; k += nparts) {
        const int d = __ldg(G.H.ci + k);
        double2 w = make_double2(0.0, 0.0);
        if (NEEDVAL) {
          const double2 h = __ldg(G.H.v + k);
          const double df = fD(it, d) - fc;
          w = make_double2(-h.y * df, h.x * df);
        }
        vis((unsigned)sunk::pidx32(n, c, d), seq0 + (unsigned)(k - k0), w, 0);
      }
      return 0;
    }
    const long long t = src - (lam + 1);
    const int p = (int)(t / n), x = (int)(t % n);
    const GOp& L = G.L[p];
    const long long r0 = L.rp[x], r1 = L.rp[x + 1];
    const long long r = r1 - r0;
    if (r == 0) return 0;
    long long j0 = 0, i1 = 0;
    int cnt_case;
    if (x < lam) {
      j0 = lbound(L.ci, r0, r1, lam) - r0;
      cnt_case = 0;
    } else if (x > lam) {
      i1 = ubound(L.ci, r0, r1, lam) - r0;
      cnt_case = 1;
    } else {
      cnt_case = 2;
    }
    if (COUNT_ONLY) {
      if (cnt_case == 0) return (unsigned long long)(r * (r + 1) / 2 - j0 * (j0 + 1) / 2);
      if (cnt_case == 1) return (unsigned long long)(i1 * r - i1 * (i1 - 1) / 2);
      const long long q = lbound(L.ci, r0, r1, lam);
      return (unsigned long long)(r * (r + 1) / 2 - ((q < r1 && __ldg(L.ci + q) == lam) ? 1 : 0));
    }
    const double fx = fD(it, x), gam = G.g[p];
    unsigned s = seq0;
    auto pairv = [&](long long ii, long long jj) {
      const int c = __ldg(L.ci + r0 + ii), d = __ldg(L.ci + r0 + jj);
      double2 w = make_double2(0.0, 0.0);
      if (NEEDVAL) {
        const double coef = fx - 0.5 * (fD(it, c) + fD(it, d));
        const double2 tt = cjmul(__ldg(L.v + r0 + ii), __ldg(L.v + r0 + jj));
        const double sc = gam * coef;
        w = make_double2(sc * tt.x, sc * tt.y);
      }
      vis(c == d ? (unsigned)(G.np + c) : (unsigned)sunk::pidx32(n, c, d), s++, w, 0);
    };
    if (cnt_case == 0) {
      for (long long jj = j0 + part; jj < r; jj += nparts)
        for (long long ii = 0; ii <= jj; ++ii) pairv(ii, jj);
    } else if (cnt_case == 1) {
      for (long long ii = part; ii < i1; ii += nparts)
        for (long long jj = ii; jj < r; ++jj) pairv(ii, jj);
    } else {
      for (long long ii = part; ii < r; ii += nparts)
        for (long long jj = ii; jj < r; ++jj)
          if (!(jj == ii && __ldg(L.ci + r0 + ii) == lam)) pairv(ii, jj);
    }
    return 0;
  }
  // ---- rows S_ab / J_ab: candidates of U = L^+(E_ab)
  const int a = it.a, b = it.b;
  if (src < 2) {  // T1 / T2: the Hamiltonian part of K
    const int row = src == 0 ? a : b;
    const long long r0 = G.H.rp[row], r1 = G.H.rp[row + 1];
    if (COUNT_ONLY) return (unsigned long long)(r1 - r0);
    for (long long k = r0 + part; k < r1; k += nparts) {
      const int c = __ldg(G.H.ci + k);
      double2 U = make_double2(0.0, 0.0);
      if (NEEDVAL) {
        const double2 h = __ldg(G.H.v + k);
        U = src == 0 ? make_double2(h.y, h.x) : make_double2(h.y, -h.x);  // i conj(H_ac) | -i H_bd
      }
      int tr;
      const unsigned key = src == 0 ? key_of(G, c, b, tr) : key_of(G, a, c, tr);
      vis(key, seq0 + (unsigned)(k - r0), U, tr);
    }
    return 0;
  }
  long long i = src - 2;
  for (int p = 0; p < G.P; ++p) {
    const GOp& L = G.L[p];
    const int* cp = G.C[p].cp;
    const int ca0 = __ldg(cp + a), ncA = __ldg(cp + a + 1) - ca0;
    const int cb0 = __ldg(cp + b), ncB = __ldg(cp + b + 1) - cb0;
    const long long ra0 = L.rp[a], rA = L.rp[a + 1] - ra0;
    const double gam = G.g[p];
    if (i < ncA + ncB) {  // T3 / T4: the dissipator part of K, via column access
      const bool t3 = i < ncA;
      const int2 e = __ldg(G.C[p].xr + (t3 ? ca0 + i : cb0 + (i - ncA)));
      const int x = e.x;
      const long long r0 = L.rp[x], r1 = L.rp[x + 1];
      if (COUNT_ONLY) return (unsigned long long)(r1 - r0);
      const double2 lx = NEEDVAL ? __ldg(L.v + e.y) : make_double2(0.0, 0.0);  // L_xa (T3) | L_xb (T4)
      for (long long k = r0 + part; k < r1; k += nparts) {
        const int c = __ldg(L.ci + k);
        double2 U = make_double2(0.0, 0.0);
        if (NEEDVAL) {
          const double2 tt = t3 ? cjmul(__ldg(L.v + k), lx) : cjmul(lx, __ldg(L.v + k));
          const double sc = -0.5 * gam;
          U = make_double2(sc * tt.x, sc * tt.y);
        }
        int tr;
        const unsigned key = t3 ? key_of(G, c, b, tr) : key_of(G, a, c, tr);
        vis(key, seq0 + (unsigned)(k - r0), U, tr);
      }
      return 0;
    }
    i -= ncA + ncB;
    if (i < rA) {  // T5: gamma conj(L_ac) L_bd
      const long long rb0 = L.rp[b], rb1 = L.rp[b + 1];
      if (COUNT_ONLY) return (unsigned long long)(rb1 - rb0);
      const int c = __ldg(L.ci + ra0 + i);
      const double2 lac = NEEDVAL ? __ldg(L.v + ra0 + i) : make_double2(0.0, 0.0);
      for (long long k = rb0 + part; k < rb1; k += nparts) {
        const int d = __ldg(L.ci + k);
        double2 U = make_double2(0.0, 0.0);
        if (NEEDVAL) {
          const double2 tt = cjmul(lac, __ldg(L.v + k));
          U = make_double2(gam * tt.x, gam * tt.y);
        }
        int tr;
        const unsigned key = key_of(G, c, d, tr);
        vis(key, seq0 + (unsigned)(k - rb0), U, tr);
      }
      return 0;
    }
    i -= rA;
  }
  return 0;
}

// =========================================================================================
// Group primitives: NT = 32 (one warp) or NT = blockDim.x (one CTA)
// =========================================================================================
template <int NT>
__device__ __forceinline__ int grank() {
  return NT == 32 ? (int)(threadIdx.x & 31) : (int)threadIdx.x;
}
template <int NT>
__device__ __forceinline__ void gsync() {
  if (NT == 32) __syncwarp(); else __syncthreads();
}
// exclusive scan of a 64-bit value over the group; *total = group sum.  `sc`: >= 33 shared
// 64-bit words (CTA groups only)
template <int NT>
__device__ __forceinline__ unsigned long long gscan(unsigned long long v, unsigned long long* total,
                                                    unsigned long long* sc) {
  const int lane = threadIdx.x & 31;
  unsigned long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(FULLM, x, o);
    if (lane >= o) x += y;
  }
  if (NT == 32) {
    *total = __shfl_sync(FULLM, x, 31);
    return x - v;
  }
  const int wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 31) sc[wid] = x;
  __syncthreads();
  if (wid == 0) {
    unsigned long long w = lane < NT / 32 ? sc[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(FULLM, w, o);
      if (lane >= o) w += y;
    }
    sc[lane] = w;
  }
  __syncthreads();
  *total = sc[NT / 32 - 1];
  return (wid > 0 ? sc[wid - 1] : 0ull) + x - v;
}

// Enumerate every candidate of the item: sources in rounds of NT (thread r of the group takes
// source s0 + r), sequence bases from a group scan of the sources' sizes.
template <int NT, bool NEEDVAL, class V>
__device__ __forceinline__ unsigned enumerate(const GProb& G, const Item& it, long long nsrc, unsigned long long* sc,
                                              V& vis) {
  unsigned carry = 0;
  for (long long s0 = 0; s0 < nsrc; s0 += NT) {
    const long long src = s0 + grank<NT>();
    const unsigned long long c = src < nsrc ? source<true, false>(G, it, src, 0u, vis) : 0ull;
    unsigned long long tot;
    const unsigned long long ex = gscan<NT>(c, &tot, sc);
    if (src < nsrc && c > 0) source<false, NEEDVAL>(G, it, src, carry + (unsigned)ex, vis);
    carry += (unsigned)tot;
  }
  return carry;  // number of candidates
}

template <int NT>
__device__ __forceinline__ unsigned long long total_candidates(const GProb& G, const Item& it, long long nsrc,
                                                               unsigned long long* sc) {
  auto none = [](unsigned, unsigned, double2, int) {};
  unsigned long long c = 0;
  for (long long s = grank<NT>(); s < nsrc; s += NT) c += source<true, false>(G, it, s, 0u, none);
  unsigned long long tot;
  (void)gscan<NT>(c, &tot, sc);
  return tot;
}

// =========================================================================================
// Row assembly: sorted candidates -> entries (count or write), D chain
// =========================================================================================
template <int CAP>
struct GBuf {
  unsigned long long key[CAP];  // (key << 32) | seq
  double2 val[CAP];
  unsigned short slot[CAP];     // index into val | transposed << 15
  int dc[CAP];                  // diagonal keys of the chunk (c) ...
  double2 dg[CAP];              // ... and their g values (row 0, row 1)
  unsigned long long sc[33];
  int cnt, nd;
};
struct GHeavyExtra {
  int hist[GH_LEV][GH_NB];
};

enum { PASS_COUNT = 0, PASS_SJ = 1, PASS_WRITE = 2 };

struct RowState {
  long long nS[2], nJ[2], nD[2];  // running counts of the S, J and D parts of rows 0 / 1
  long long TS[2], TJ[2];         // totals of the S and J parts (PASS_WRITE)
  long long O[2];                 // row offsets (PASS_WRITE)
  double P[2];                    // D-chain prefix sums (warp 0)
  int prev;                       // next l of the D chain (warp 0)
};

// number of l in [s0, e), from s0, with |P inv[l]| > tau (monotone: |P inv[l]| non-increasing)
__device__ __forceinline__ int seg_kept(double P, int s0, int e, const double* __restrict__ inv, double tau) {
  if (s0 >= e || !(fabs(P) > 0.0)) return 0;
  int lo = s0, hi = e;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (fabs(P * __ldg(inv + mid)) > tau) lo = mid + 1; else hi = mid;
  }
  return lo - s0;
}

__device__ __forceinline__ void put(const GOut& O, long long pos, int col, double v) {
  if (pos < O.cap) {
    O.col[pos] = col;
    O.val[pos] = v;
  }
}

template <int NT>
__device__ __forceinline__ void bitonic(unsigned long long* key, unsigned short* slot, int cnt) {
  int n2 = 2;
  while (n2 < cnt) n2 <<= 1;
  for (int i = cnt + grank<NT>(); i < n2; i += NT) {
    key[i] = ~0ull;
    slot[i] = 0;
  }
  gsync<NT>();
  for (int k = 2; k <= n2; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = grank<NT>(); i < n2; i += NT) {
        const int ij = i ^ j;
        if (ij > i) {
          const unsigned long long u = key[i], w = key[ij];
          if ((u > w) == ((i & k) == 0)) {
            key[i] = w;
            key[ij] = u;
            const unsigned short t = slot[i];
            slot[i] = slot[ij];
            slot[ij] = t;
          }
        }
      }
      gsync<NT>();
    }
}

// Off-diagonal runs -> S / J entries (counted, or written at their positions); diagonal runs
// -> (c, g) list for the D chain.  B.key / B.slot sorted, B.cnt entries.
template <int NT, int CAP>
__device__ void assemble_runs(const GProb& G, const Item& it, GBuf<CAP>& B, RowState& rs, int pass, double tau,
                              const GOut& O) {
  const int cnt = B.cnt;
  const unsigned npk = (unsigned)G.np;
  const int nrow = it.kind == 0 ? 2 : 1;
  int nd = 0;
  for (int base = 0; base < cnt; base += NT) {
    const int i = base + grank<NT>();
    const bool valid = i < cnt;
    const unsigned k32 = valid ? (unsigned)(B.key[i] >> 32) : 0xffffffffu;
    const bool head = valid && (i == 0 || (unsigned)(B.key[i - 1] >> 32) != k32);
    double2 A = make_double2(0.0, 0.0), Bs = make_double2(0.0, 0.0);
    if (head) {
      for (int j = i; j < cnt && (unsigned)(B.key[j] >> 32) == k32; ++j) {
        // light warps (register sort): value index and transposition in the key's low word;
        // CTA groups: the slot array moved with the keys
        const unsigned lw = (unsigned)B.key[j];
        const unsigned short s = NT == 32 ? (unsigned short)((lw & 0x7fffu) | ((lw >> 16) & 0x8000u)) : B.slot[j];
        const double2 U = B.val[s & 0x7fff];
        if (s & 0x8000) {  // transposed candidate U_dc: conj for G_S, -conj for G_J
          A.x += U.x; A.y -= U.y;
          Bs.x -= U.x; Bs.y += U.y;
        } else {
          A.x += U.x; A.y += U.y;
          Bs.x += U.x; Bs.y += U.y;
        }
      }
    }
    const bool diag = head && k32 >= npk;
    const bool off = head && !diag;
    double v0S, v0J, v1S = 0.0, v1J = 0.0;
    if (it.kind == 0) {  // row S_ab: S <- Re A, J <- -Im A;  row J_ab: S <- Im B, J <- Re B
      v0S = A.x; v0J = -A.y; v1S = Bs.y; v1J = Bs.x;
    } else {             // row D^lam: S <- sqrt2 Re G, J <- -sqrt2 Im G
      v0S = SQ2 * A.x; v0J = -SQ2 * A.y;
    }
    const bool f0S = off && fabs(v0S) > tau, f0J = off && fabs(v0J) > tau;
    const bool f1S = off && nrow == 2 && fabs(v1S) > tau, f1J = off && nrow == 2 && fabs(v1J) > tau;
    // five 12-bit fields (each at most NT <= 1024 per round)
    const unsigned long long fl = (unsigned long long)f0S | ((unsigned long long)f0J << 12) |
                                  ((unsigned long long)f1S << 24) | ((unsigned long long)f1J << 36) |
                                  ((unsigned long long)diag << 48);
    unsigned long long tot;
    const unsigned long long ex = gscan<NT>(fl, &tot, B.sc);
    auto fld = [](unsigned long long x, int k) { return (long long)((x >> (12 * k)) & 0xfff); };
    if (pass == PASS_WRITE) {
      if (f0S) put(O, rs.O[0] + rs.nS[0] + fld(ex, 0), (int)k32, v0S);
      if (f0J) put(O, rs.O[0] + rs.TS[0] + rs.nJ[0] + fld(ex, 1), (int)(npk + k32), v0J);
      if (f1S) put(O, rs.O[1] + rs.nS[1] + fld(ex, 2), (int)k32, v1S);
      if (f1J) put(O, rs.O[1] + rs.TS[1] + rs.nJ[1] + fld(ex, 3), (int)(npk + k32), v1J);
    }
    if (diag) {
      const int q = nd + (int)fld(ex, 4);
      B.dc[q] = (int)(k32 - npk);
      B.dg[q] = it.kind == 0 ? make_double2(SQ2 * A.x, SQ2 * A.y) : make_double2(A.x, 0.0);
    }
    rs.nS[0] += fld(tot, 0);
    rs.nJ[0] += fld(tot, 1);
    rs.nS[1] += fld(tot, 2);
    rs.nJ[1] += fld(tot, 3);
    nd += (int)fld(tot, 4);
  }
  B.nd = nd;  // every thread writes the same value
  gsync<NT>();
}

// D chain over the chunk's diagonal list (warp 0 of the group): for each diagonal key c (in
// order), the segment l in [prev, c) with coefficient P inv[l] (kept prefix by a binary
// search), then l = c with (P - c g_c) inv[c]; P += g_c.  Both rows of a pair item.
template <int NT, class DG>
__device__ void d_chain_f(const GProb& G, const Item& it, int nd, DG diag, RowState& rs, int pass, double tau,
                          const GOut& O) {
  if (NT != 32 && threadIdx.x >= 32) return;  // CTA groups: warp 0 only
  const int lane = threadIdx.x & 31;
  const int nrow = it.kind == 0 ? 2 : 1;
  const int dbase = (int)(2 * G.np - 1);
  for (int base = 0; base < nd; base += 32) {
    const int k = base + lane;
    const bool valid = k < nd;
    int c = 0x7fffffff;
    double2 g = make_double2(0.0, 0.0);
    if (valid) diag(k, c, g);
    const int nv = nd - base < 32 ? nd - base : 32;
    const int cprev = __shfl_up_sync(FULLM, c, 1);
    int s0 = lane == 0 ? rs.prev : cprev + 1;
    if (s0 < 1) s0 = 1;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (r >= nrow) break;
      const double gr = r == 0 ? g.x : g.y;
      double x = gr;  // inclusive scan (fixed tree)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(FULLM, x, o);
        if (lane >= o) x += y;
      }
      const double Pb = rs.P[r] + (x - gr);  // prefix before c
      const int k1 = valid ? seg_kept(Pb, s0, c, G.inv, tau) : 0;
      double vc = 0.0;
      bool atc = false;
      if (valid && c >= 1) {
        vc = (Pb - (double)c * gr) * __ldg(G.inv + c);
        atc = fabs(vc) > tau;
      }
      const int cd = k1 + (atc ? 1 : 0);
      int xo = cd;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULLM, xo, o);
        if (lane >= o) xo += y;
      }
      const int totd = __shfl_sync(FULLM, xo, 31);
      const int offd = xo - cd;
      if (pass == PASS_WRITE) {
        const long long b0 = rs.O[r] + rs.TS[r] + rs.TJ[r] + rs.nD[r];
        for (int j = 0; j < nv; ++j) {
          const int s0j = __shfl_sync(FULLM, s0, j), k1j = __shfl_sync(FULLM, k1, j);
          const int offj = __shfl_sync(FULLM, offd, j), cj = __shfl_sync(FULLM, c, j);
          const double Pj = __shfl_sync(FULLM, Pb, j), vj = __shfl_sync(FULLM, vc, j);
          const bool aj = __shfl_sync(FULLM, atc ? 1 : 0, j) != 0;
          const long long lim = O.dlim > 0 ? O.dlim - rs.nD[r] - offj : 0x7fffffffffffffffLL;
          for (int t = lane; t < k1j && t < lim; t += 32) put(O, b0 + offj + t, dbase + s0j + t, Pj * __ldg(G.inv + s0j + t));
          if (aj && lane == 0 && k1j < lim) put(O, b0 + offj + k1j, dbase + cj, vj);
        }
      }
      rs.nD[r] += totd;
      rs.P[r] = __shfl_sync(FULLM, Pb + gr, nv - 1);
    }
    rs.prev = __shfl_sync(FULLM, c, nv - 1) + 1;
  }
}

template <int NT, int CAP>
__device__ __forceinline__ void d_chain(const GProb& G, const Item& it, GBuf<CAP>& B, RowState& rs, int pass,
                                        double tau, const GOut& O) {
  auto dg = [&](int k, int& c, double2& g) {
    c = B.dc[k];
    g = B.dg[k];
  };
  d_chain_f<NT>(G, it, B.nd, dg, rs, pass, tau, O);
}

// tail of the D chain after the last diagonal key: l in [prev, n) with P inv[l]
__device__ __forceinline__ void d_tail(const GProb& G, const Item& it, RowState& rs, int pass, double tau,
                                       const GOut& O) {
  const int lane = threadIdx.x & 31;
  const int nrow = it.kind == 0 ? 2 : 1;
  const int dbase = (int)(2 * G.np - 1);
  const int s0 = rs.prev < 1 ? 1 : rs.prev;
  for (int r = 0; r < nrow; ++r) {
    const int k1 = seg_kept(rs.P[r], s0, G.n, G.inv, tau);
    if (pass == PASS_WRITE) {
      const long long b0 = rs.O[r] + rs.TS[r] + rs.TJ[r] + rs.nD[r];
      const long long lim = O.dlim > 0 ? O.dlim - rs.nD[r] : 0x7fffffffffffffffLL;
      for (int t = lane; t < k1 && t < lim; t += 32) put(O, b0 + t, dbase + s0 + t, rs.P[r] * __ldg(G.inv + s0 + t));
    }
    rs.nD[r] += k1;
  }
}

// gather the candidates with key in [lo, hi) into B (unsorted)
template <int NT, int CAP>
__device__ __forceinline__ void gather(const GProb& G, const Item& it, long long nsrc, GBuf<CAP>& B, unsigned lo,
                                       unsigned hi) {
  if (grank<NT>() == 0) B.cnt = 0;
  gsync<NT>();
  if (NT == 32) {  // light warps: one chunk holding every candidate; index = sequence number
    auto vis = [&](unsigned key, unsigned seq, double2 U, int tr) {
      B.key[seq] = ((unsigned long long)key << 32) | ((unsigned)tr << 31) | seq;
      B.val[seq] = U;
    };
    const unsigned c = enumerate<NT, true>(G, it, nsrc, B.sc, vis);
    if ((threadIdx.x & 31) == 0) B.cnt = (int)c;
    __syncwarp();
    return;
  }
  auto vis = [&](unsigned key, unsigned seq, double2 U, int tr) {
    if (key >= lo && key < hi) {
      const int i = atomicAdd(&B.cnt, 1);
      B.key[i] = ((unsigned long long)key << 32) | seq;
      B.val[i] = U;
      B.slot[i] = (unsigned short)(i | (tr << 15));
    }
  };
  enumerate<NT, true>(G, it, nsrc, B.sc, vis);
  gsync<NT>();
}

// bitonic sort of cnt <= 32 R 64-bit keys in registers (R per lane, element e = lane + 32 q)
template <int R>
__device__ __forceinline__ void warp_sort_regs(unsigned long long* key, int cnt) {
  const int lane = threadIdx.x & 31;
  unsigned long long v[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int e = lane + 32 * q;
    v[q] = e < cnt ? key[e] : ~0ull;
  }
  int n2 = 2;
  while (n2 < cnt) n2 <<= 1;
  for (int k = 2; k <= n2; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {  // partner in another register of this lane
        const int jq = j >> 5;
        // register distance as a compile-time constant (a runtime q ^ jq index would put v[]
        // in local memory)
#pragma unroll
        for (int t = 1; t < R; t <<= 1) {
          if (jq == t) {
#pragma unroll
            for (int q = 0; q < R; ++q) {
              const int q2 = q ^ t;
              if (q2 > q && q2 < R) {
                const int e = lane + 32 * q;
                const bool asc = (e & k) == 0;
                const unsigned long long a = v[q], b = v[q2];
                if ((a > b) == asc) {
                  v[q] = b;
                  v[q2] = a;
                }
              }
            }
          }
        }
      } else {
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int e = lane + 32 * q;
          const unsigned long long o = __shfl_xor_sync(FULLM, v[q], j);
          const bool lower = (lane & j) == 0, asc = (e & k) == 0;
          v[q] = (lower == asc) ? (o < v[q] ? o : v[q]) : (o > v[q] ? o : v[q]);
        }
      }
    }
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int e = lane + 32 * q;
    if (e < cnt) key[e] = v[q];
  }
  __syncwarp();
}

template <int NT, int CAP>
__device__ __forceinline__ void sort_gathered(GBuf<CAP>& B) {
  if constexpr (NT == 32) {
    static_assert(CAP <= 256, "register sort holds <= 8 keys per lane");
    const int c = B.cnt;
    if (c <= 32) warp_sort_regs<1>(B.key, c);
    else if (c <= 64) warp_sort_regs<2>(B.key, c);
    else if (c <= 128 || CAP <= 128) warp_sort_regs<(CAP < 128 ? CAP : 128) / 32>(B.key, c);
    else warp_sort_regs<CAP / 32>(B.key, c);
  } else {
    bitonic<NT>(B.key, B.slot, B.cnt);
  }
}

// one chunk: gather, sort, runs (+ D chain)
template <int NT, int CAP>
__device__ __forceinline__ void chunk(const GProb& G, const Item& it, long long nsrc, GBuf<CAP>& B, RowState& rs,
                                      int pass, double tau, const GOut& O, unsigned lo, unsigned hi) {
  gather<NT, CAP>(G, it, nsrc, B, lo, hi);
  sort_gathered<NT, CAP>(B);
  assemble_runs<NT, CAP>(G, it, B, rs, pass, tau, O);
  if (pass != PASS_SJ) d_chain<NT, CAP>(G, it, B, rs, pass, tau, O);
  gsync<NT>();
}

// a single key with more than CAP candidates: per-thread partial sums in enumeration order,
// then a fixed-order tree over the group -> two pseudo-candidates (direct, transposed)
template <int NT, int CAP>
__device__ void overflow_key(const GProb& G, const Item& it, long long nsrc, GBuf<CAP>& B, RowState& rs, int pass,
                             double tau, const GOut& O, unsigned key) {
  double2 sN = make_double2(0.0, 0.0), sT = make_double2(0.0, 0.0);
  auto vis = [&](unsigned k, unsigned, double2 U, int tr) {
    if (k == key) {
      if (tr) { sT.x += U.x; sT.y += U.y; }
      else { sN.x += U.x; sN.y += U.y; }
    }
  };
  enumerate<NT, true>(G, it, nsrc, B.sc, vis);
  const int r = grank<NT>();
  B.val[r] = sN;  // CAP >= 2 NT
  B.val[NT + r] = sT;
  gsync<NT>();
  for (int s = NT / 2; s > 0; s >>= 1) {
    if (r < s) {
      B.val[r].x += B.val[r + s].x; B.val[r].y += B.val[r + s].y;
      B.val[NT + r].x += B.val[NT + r + s].x; B.val[NT + r].y += B.val[NT + r + s].y;
    }
    gsync<NT>();
  }
  if (r == 0) {
    B.val[1] = B.val[NT];
    B.key[0] = (unsigned long long)key << 32;
    B.key[1] = ((unsigned long long)key << 32) | 1ull;
    B.slot[0] = 0;
    B.slot[1] = (unsigned short)(1 | 0x8000);
    B.cnt = 2;
  }
  gsync<NT>();
  assemble_runs<NT, CAP>(G, it, B, rs, pass, tau, O);
  if (pass != PASS_SJ) d_chain<NT, CAP>(G, it, B, rs, pass, tau, O);
  gsync<NT>();
}

// ---- frame mode: items whose keys span a window of the shared buffer (dense operators) ----
// The group accumulates every candidate straight into a key-indexed frame (direct and
// transposed sums apart), one source after another with a barrier in between: a source emits
// pairwise distinct keys, so no two threads touch one key at a time and every key's sum is
// formed in source order (deterministic).  The D chain reads the diagonal keys of the window.
template <int CAP>
__device__ __forceinline__ int frame_keys(const Item& it) {
  constexpr int W2 = (46 * CAP) / 16;  // double2 slots in key[] .. dg[]
  return it.kind == 0 ? W2 / 2 : W2;
}

template <int NT>
__device__ __forceinline__ void key_span(const GProb& G, const Item& it, long long nsrc, unsigned long long* sc,
                                         unsigned& kmin, unsigned& kmax) {
  unsigned mn = 0xffffffffu, mx = 0u;
  auto vis = [&](unsigned key, unsigned, double2, int) {
    mn = key < mn ? key : mn;
    mx = key > mx ? key : mx;
  };
  for (long long s = grank<NT>(); s < nsrc; s += NT) source<false, false>(G, it, s, 0u, vis);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned a = __shfl_xor_sync(FULLM, mn, o), b = __shfl_xor_sync(FULLM, mx, o);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  if (NT != 32) {
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
      sc[threadIdx.x >> 5] = mn;
      sc[16 + (threadIdx.x >> 5)] = mx;
    }
    __syncthreads();
    for (int w = 0; w < NT / 32; ++w) {
      mn = (unsigned)sc[w] < mn ? (unsigned)sc[w] : mn;
      mx = (unsigned)sc[16 + w] > mx ? (unsigned)sc[16 + w] : mx;
    }
    __syncthreads();
  }
  kmin = mn;
  kmax = mx;
}

template <int NT, int CAP>
__device__ void frame_accum(const GProb& G, const Item& it, long long nsrc, GBuf<CAP>& B, unsigned lo, unsigned hi) {
  double2* F = reinterpret_cast<double2*>(&B.key[0]);
  const int W = frame_keys<CAP>(it);
  const int span = (int)(hi - lo);
  for (int i = grank<NT>(); i < span; i += NT) {
    F[i] = make_double2(0.0, 0.0);
    if (it.kind == 0) F[W + i] = make_double2(0.0, 0.0);
  }
  gsync<NT>();
  auto vis = [&](unsigned key, unsigned, double2 U, int tr) {
    if (key >= lo && key < hi) {
      double2& a = F[(tr ? W : 0) + (int)(key - lo)];
      a.x += U.x;
      a.y += U.y;
    }
  };
  for (long long src = 0; src < nsrc; ++src) {
    source<false, true>(G, it, src, 0u, vis, grank<NT>(), NT);
    gsync<NT>();
  }
}

// off-diagonal keys of the window -> S / J entries (counted or written)
template <int NT, int CAP>
__device__ void assemble_frame(const GProb& G, const Item& it, GBuf<CAP>& B, unsigned lo, unsigned hi, RowState& rs,
                               int pass, double tau, const GOut& O) {
  const double2* F = reinterpret_cast<const double2*>(&B.key[0]);
  const int W = frame_keys<CAP>(it);
  const unsigned npk = (unsigned)G.np;
  const int nrow = it.kind == 0 ? 2 : 1;
  const unsigned ohi = hi < npk ? hi : npk;
  for (unsigned base = lo; base < ohi; base += NT) {
    const unsigned k = base + (unsigned)grank<NT>();
    const bool valid = k < ohi;
    double2 N = make_double2(0.0, 0.0), T = make_double2(0.0, 0.0);
    if (valid) {
      N = F[k - lo];
      if (it.kind == 0) T = F[W + (k - lo)];
    }
    const double2 A = make_double2(N.x + T.x, N.y - T.y);   // direct + conj(transposed)
    const double2 Bs = make_double2(N.x - T.x, N.y + T.y);  // direct - conj(transposed)
    double v0S, v0J, v1S = 0.0, v1J = 0.0;
    if (it.kind == 0) {
      v0S = A.x; v0J = -A.y; v1S = Bs.y; v1J = Bs.x;
    } else {
      v0S = SQ2 * A.x; v0J = -SQ2 * A.y;
    }
    const bool f0S = valid && fabs(v0S) > tau, f0J = valid && fabs(v0J) > tau;
    const bool f1S = valid && nrow == 2 && fabs(v1S) > tau, f1J = valid && nrow == 2 && fabs(v1J) > tau;
    const unsigned long long fl = (unsigned long long)f0S | ((unsigned long long)f0J << 12) |
                                  ((unsigned long long)f1S << 24) | ((unsigned long long)f1J << 36);
    unsigned long long tot;
    const unsigned long long ex = gscan<NT>(fl, &tot, B.sc);
    auto fld = [](unsigned long long x, int q) { return (long long)((x >> (12 * q)) & 0xfff); };
    if (pass == PASS_WRITE) {
      if (f0S) put(O, rs.O[0] + rs.nS[0] + fld(ex, 0), (int)k, v0S);
      if (f0J) put(O, rs.O[0] + rs.TS[0] + rs.nJ[0] + fld(ex, 1), (int)(npk + k), v0J);
      if (f1S) put(O, rs.O[1] + rs.nS[1] + fld(ex, 2), (int)k, v1S);
      if (f1J) put(O, rs.O[1] + rs.TS[1] + rs.nJ[1] + fld(ex, 3), (int)(npk + k), v1J);
    }
    rs.nS[0] += fld(tot, 0);
    rs.nJ[0] += fld(tot, 1);
    rs.nS[1] += fld(tot, 2);
    rs.nJ[1] += fld(tot, 3);
  }
  gsync<NT>();
}

// D chain over the diagonal keys of the window (every key np + c in it, g = 0 where untouched)
template <int NT, int CAP>
__device__ __forceinline__ void frame_chain(const GProb& G, const Item& it, GBuf<CAP>& B, unsigned lo, unsigned hi,
                                            RowState& rs, int pass, double tau, const GOut& O) {
  const unsigned npk = (unsigned)G.np;
  const unsigned dlo = lo > npk ? lo : npk;
  const int nd = hi > dlo ? (int)(hi - dlo) : 0;
  const double2* F = reinterpret_cast<const double2*>(&B.key[0]);
  const bool pair = it.kind == 0;
  auto dg = [&](int k, int& c, double2& g) {
    c = (int)(dlo - npk) + k;
    const double2 N = F[(dlo - lo) + k];
    g = pair ? make_double2(SQ2 * N.x, SQ2 * N.y) : make_double2(N.x, 0.0);
  };
  d_chain_f<NT>(G, it, nd, dg, rs, pass, tau, O);
  gsync<NT>();
}

// every window of [kmin, kmax] in key order: accumulate, emit, chain
template <int NT, int CAP>
__device__ void frame_sweep(const GProb& G, const Item& it, long long nsrc, GBuf<CAP>& B, unsigned kmin,
                            unsigned kmax, RowState& rs, int pass, double tau, const GOut& O) {
  const unsigned W = (unsigned)frame_keys<CAP>(it);
  for (unsigned lo = kmin; lo <= kmax; lo += W) {
    const unsigned hi = kmax - lo + 1 < W ? kmax + 1 : lo + W;
    frame_accum<NT, CAP>(G, it, nsrc, B, lo, hi);
    assemble_frame<NT, CAP>(G, it, B, lo, hi, rs, pass, tau, O);
    if (pass != PASS_SJ) frame_chain<NT, CAP>(G, it, B, lo, hi, rs, pass, tau, O);
    if (hi == kmax + 1) break;
  }
}

// every chunk of the item in key order.  Items with at most CAP candidates: one chunk.
// Otherwise (CTA groups) key-range chunks from histograms of GH_NB bins, refined (up to
// GH_LEV levels) where a bin holds more than CAP candidates.
template <int NT, int CAP>
__device__ void sweep(const GProb& G, const Item& it, long long nsrc, unsigned long long C, GBuf<CAP>& B,
                      GHeavyExtra* X, RowState& rs, int pass, double tau, const GOut& O) {
  const unsigned kend = (unsigned)(G.np + G.n);
  const int cap = G.cap < CAP ? G.cap : CAP;
  if (C <= (unsigned long long)cap || X == nullptr) {
    chunk<NT, CAP>(G, it, nsrc, B, rs, pass, tau, O, 0u, kend);
    return;
  }
  unsigned lo[GH_LEV], w[GH_LEV];
  int nb[GH_LEV], pos[GH_LEV];
  auto hist = [&](int d, unsigned blo, unsigned bhi) {
    lo[d] = blo;
    const unsigned span = bhi - blo;
    w[d] = (span + GH_NB - 1) / GH_NB;
    nb[d] = (int)((span + w[d] - 1) / w[d]);
    pos[d] = 0;
    for (int i = grank<NT>(); i < GH_NB; i += NT) X->hist[d][i] = 0;
    gsync<NT>();
    const unsigned ww = w[d];
    int* h = X->hist[d];
    auto vis = [&](unsigned key, unsigned, double2, int) {
      if (key >= blo && key < bhi) atomicAdd(&h[(key - blo) / ww], 1);
    };
    enumerate<NT, false>(G, it, nsrc, B.sc, vis);
    gsync<NT>();
  };
  hist(0, 0u, kend);
  int d = 0;
  while (true) {
    if (pos[d] == nb[d]) {
      if (d == 0) break;
      --d;
      continue;
    }
    const int b = pos[d];
    const int hb = X->hist[d][b];
    const unsigned blo = lo[d] + (unsigned)b * w[d];
    const unsigned bhi = blo + w[d] < kend ? blo + w[d] : kend;
    if (hb > cap) {
      pos[d] = b + 1;
      if (w[d] == 1 || d == GH_LEV - 1) {
        overflow_key<NT, CAP>(G, it, nsrc, B, rs, pass, tau, O, blo);  // w == 1 here (GH_NB^4 > 2^32)
      } else {
        ++d;
        hist(d, blo, bhi);
      }
      continue;
    }
    int e = b, sum = 0;
    while (e < nb[d] && X->hist[d][e] <= cap && sum + X->hist[d][e] <= cap) sum += X->hist[d][e++];
    const unsigned chi = lo[d] + (unsigned)e * w[d];
    if (sum > 0) chunk<NT, CAP>(G, it, nsrc, B, rs, pass, tau, O, blo, chi < kend ? chi : kend);
    pos[d] = e;
  }
}

__device__ __forceinline__ Item make_item(const GProb& G, long long idx, bool is_d, int lam) {
  Item it;
  if (is_d) {
    it.kind = 1;
    it.lam = lam;
    it.a = it.b = 0;
    it.alpha = __ldg(G.inv + lam);
  } else {
    it.kind = 0;
    sunk::pair_decode(G.n, idx, it.a, it.b);
    it.lam = 0;
    it.alpha = 0.0;
  }
  return it;
}

// Process one item (all group threads).  COUNT: write cnt and the slot sums.  FILL: offsets
// from the scan, then an S/J counting sweep (when the row needs more than one round or chunk)
// and the writing sweep; row_ptr and K.
template <int NT, int CAP, bool FILL>
__device__ void run_item(const GProb& G, const Item& it, long long idx, unsigned long long C, GBuf<CAP>& B,
                         GHeavyExtra* X, double tau, int* cnt, int* ts, const GOut& O) {
  const long long nsrc = num_sources(G, it);
  RowState rs;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    rs.nS[r] = rs.nJ[r] = rs.nD[r] = rs.TS[r] = rs.TJ[r] = rs.O[r] = 0;
    rs.P[r] = 0.0;
  }
  rs.prev = 1;
  const long long np = G.np;
  const int lane = threadIdx.x & 31;
  const unsigned kend = (unsigned)(G.np + G.n);
  // path: 0 one sorted chunk; 1 key-range chunks (sorted); 2 key-indexed frame (<= 2 windows)
  const int cap = G.cap < CAP ? G.cap : CAP;
  int path = 0;
  unsigned kmin = 0, kmax = 0;
  if (C > (unsigned long long)cap) {
    path = 1;
    if (X != nullptr && G.cap >= CAP) {
      key_span<NT>(G, it, nsrc, B.sc, kmin, kmax);
      const unsigned W = (unsigned)frame_keys<CAP>(it);
      if ((unsigned long long)(kmax - kmin) + 1 <= 2ull * W) path = 2;
    }
  }
  if (!FILL) {
    // D row with a stash: the writing pass into the row's three stash segments (S, J, D parts at
    // fixed offsets), which counts exactly as the counting pass does
    const bool dst = it.kind == 1 && G.dseg > 0;
    // light pair with a stash (one sorted chunk): the same writing pass into its two stash rows
    // (S part <= GW_CAP distinct keys, J part likewise; the D part bounded by dlim)
    const bool pst = NT == 32 && it.kind == 0 && G.scap > 0 && path == 0;
    GOut CO = O;
    int pc = PASS_COUNT;
    if (dst) {
      rs.O[0] = (long long)(it.lam - 1) * G.drow;
      rs.TS[0] = rs.TJ[0] = G.dseg;
      CO = GOut{nullptr, G.dcol, G.dval, (long long)it.lam * G.drow, nullptr, nullptr, nullptr, 0};
      pc = PASS_WRITE;
    } else if (pst) {
      rs.O[0] = idx * G.scap;
      rs.O[1] = (np + idx) * G.scap;
      rs.TS[0] = rs.TJ[0] = rs.TS[1] = rs.TJ[1] = GW_CAP;
      CO = GOut{nullptr, G.scol, G.sval, 0x7fffffffffffffffLL, nullptr, nullptr, nullptr, (long long)G.scap - 2 * GW_CAP};
      pc = PASS_WRITE;
    }
    if (path == 2) frame_sweep<NT, CAP>(G, it, nsrc, B, kmin, kmax, rs, pc, tau, CO);
    else sweep<NT, CAP>(G, it, nsrc, C, B, X, rs, pc, tau, CO);
    d_tail(G, it, rs, (threadIdx.x < 32 || NT == 32) ? pc : PASS_COUNT, tau, CO);  // warp 0 owns the chain
    if (dst && threadIdx.x == 0) {
      const bool ok = rs.nS[0] <= G.dseg && rs.nJ[0] <= G.dseg;
      G.dflag[it.lam - 1] = ok ? 1 : 0;
      if (ok) G.dK[it.lam - 1] = rs.P[0] / (double)G.n;  // K_s = Tr(G_s)/N, as the fill writes it
    }
    if (pst && lane == 0) {
      const bool ok = rs.nD[0] <= G.scap - 2 * GW_CAP && rs.nD[1] <= G.scap - 2 * GW_CAP;
      G.sflag[idx] = ok ? 1 : 0;
      if (ok) {  // K_s = Tr(G_s)/N, as the fill writes it
        G.sK[idx] = rs.P[0] / (double)G.n;
        G.sK[np + idx] = rs.P[1] / (double)G.n;
        G.snj[idx] = make_int2((int)rs.nS[0], (int)rs.nJ[0]);
        G.snj[np + idx] = make_int2((int)rs.nS[1], (int)rs.nJ[1]);
      }
    }
    if (NT == 32 && it.kind == 0 && G.scap > 0 && !pst && lane == 0) G.sflag[idx] = 0;
    if (grank<NT>() == 0) {
      if (it.kind == 0) {
        const int t0 = (int)(rs.nS[0] + rs.nJ[0] + rs.nD[0]), t1 = (int)(rs.nS[1] + rs.nJ[1] + rs.nD[1]);
        cnt[idx] = t0;
        cnt[np + idx] = t1;
        atomicAdd(&ts[idx / GSLOT], t0);
        atomicAdd(&ts[G.npt + idx / GSLOT], t1);
      } else {
        const int t0 = (int)(rs.nS[0] + rs.nJ[0] + rs.nD[0]);
        cnt[2 * np + it.lam - 1] = t0;
        ts[2 * G.npt + it.lam - 1] = t0;
        G.dtot[2 * (it.lam - 1)] = (int)rs.nS[0];  // S / J part lengths: the fill skips its counting sweep
        G.dtot[2 * (it.lam - 1) + 1] = (int)rs.nJ[0];
      }
    }
    gsync<NT>();
    return;
  }
  // row offsets (warp 0; broadcast through B.sc for CTA groups)
  if (threadIdx.x < 32 || NT == 32) {
    long long o0, o1 = 0;
    if (it.kind == 0) {
      const long long s = idx / GSLOT, q0 = s * GSLOT;
      int a0 = 0, a1 = 0;
      if (q0 + lane < idx) {
        a0 = __ldg(cnt + q0 + lane);
        a1 = __ldg(cnt + np + q0 + lane);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a0 += __shfl_xor_sync(FULLM, a0, o);
        a1 += __shfl_xor_sync(FULLM, a1, o);
      }
      o0 = __ldg(O.toff + s) + a0;
      o1 = __ldg(O.toff + G.npt + s) + a1;
    } else {
      o0 = __ldg(O.toff + 2 * G.npt + it.lam - 1);
    }
    rs.O[0] = o0;
    rs.O[1] = o1;
    if (NT != 32 && lane == 0) {
      B.sc[0] = (unsigned long long)o0;
      B.sc[1] = (unsigned long long)o1;
    }
  }
  if (NT != 32) {
    __syncthreads();
    rs.O[0] = (long long)B.sc[0];
    rs.O[1] = (long long)B.sc[1];
    __syncthreads();
  }
  if (grank<NT>() == 0) {
    if (it.kind == 0) {
      O.row_ptr[idx] = rs.O[0];
      O.row_ptr[np + idx] = rs.O[1];
    } else {
      O.row_ptr[2 * np + it.lam - 1] = rs.O[0];
    }
  }
  // S / J totals first (the J part follows the whole S part, the D part follows both); a
  // single chunk / window keeps its data for the writing pass
  const bool frame1 = path == 2 && (unsigned long long)(kmax - kmin) + 1 <= (unsigned long long)frame_keys<CAP>(it);
  const bool known = it.kind == 1 && path != 0;  // D row: S / J lengths from the count pass
  if (known) {
    rs.nS[0] = __ldg(G.dtot + 2 * (it.lam - 1));
    rs.nJ[0] = __ldg(G.dtot + 2 * (it.lam - 1) + 1);
    if (frame1) frame_accum<NT, CAP>(G, it, nsrc, B, kmin, kmax + 1);
  } else if (path == 0) {
    gather<NT, CAP>(G, it, nsrc, B, 0u, kend);
    sort_gathered<NT, CAP>(B);
    assemble_runs<NT, CAP>(G, it, B, rs, PASS_SJ, tau, O);
  } else if (frame1) {
    frame_accum<NT, CAP>(G, it, nsrc, B, kmin, kmax + 1);
    assemble_frame<NT, CAP>(G, it, B, kmin, kmax + 1, rs, PASS_SJ, tau, O);
  } else if (path == 2) {
    frame_sweep<NT, CAP>(G, it, nsrc, B, kmin, kmax, rs, PASS_SJ, tau, O);
  } else {
    sweep<NT, CAP>(G, it, nsrc, C, B, X, rs, PASS_SJ, tau, O);
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    rs.TS[r] = rs.nS[r];
    rs.TJ[r] = rs.nJ[r];
    rs.nS[r] = rs.nJ[r] = 0;
  }
  if (path == 0) {
    assemble_runs<NT, CAP>(G, it, B, rs, PASS_WRITE, tau, O);
    d_chain<NT, CAP>(G, it, B, rs, PASS_WRITE, tau, O);
    gsync<NT>();
  } else if (frame1) {  // (frame accumulated above)
    assemble_frame<NT, CAP>(G, it, B, kmin, kmax + 1, rs, PASS_WRITE, tau, O);
    frame_chain<NT, CAP>(G, it, B, kmin, kmax + 1, rs, PASS_WRITE, tau, O);
  } else if (path == 2) {
    frame_sweep<NT, CAP>(G, it, nsrc, B, kmin, kmax, rs, PASS_WRITE, tau, O);
  } else {
    sweep<NT, CAP>(G, it, nsrc, C, B, X, rs, PASS_WRITE, tau, O);
  }
  if (threadIdx.x < 32 || NT == 32) {
    d_tail(G, it, rs, PASS_WRITE, tau, O);
    if (lane == 0 && O.K) {  // K_s = Tr(G_s)/N = (sum_c g_c)/N
      if (it.kind == 0) {
        O.K[idx] = rs.P[0] / (double)G.n;
        O.K[np + idx] = rs.P[1] / (double)G.n;
      } else {
        O.K[2 * np + it.lam - 1] = rs.P[0] / (double)G.n;
      }
    }
  }
  gsync<NT>();
}

// fill of a stashed light pair (warp): row offsets as run_item's fill, row_ptr, K, and the two
// rows copied from the stash (lanes stride the concatenation of both rows)
__device__ __forceinline__ void copy_stashed(const GProb& G, long long p, const int* __restrict__ cnt,
                                             const GOut& O) {
  const int lane = threadIdx.x & 31;
  const long long np = G.np;
  const long long s = p / GSLOT, q0 = s * GSLOT;
  int a0 = 0, a1 = 0;
  if (q0 + lane < p) {
    a0 = __ldg(cnt + q0 + lane);
    a1 = __ldg(cnt + np + q0 + lane);
  }
  const int t0 = __ldg(cnt + p), t1 = __ldg(cnt + np + p);
  const long long b0 = __ldg(O.toff + s), b1 = __ldg(O.toff + G.npt + s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a0 += __shfl_xor_sync(FULLM, a0, o);
    a1 += __shfl_xor_sync(FULLM, a1, o);
  }
  const long long o0 = b0 + a0, o1 = b1 + a1;
  if (lane == 0) {
    O.row_ptr[p] = o0;
    O.row_ptr[np + p] = o1;
    if (O.K) {
      O.K[p] = __ldg(G.sK + p);
      O.K[np + p] = __ldg(G.sK + np + p);
    }
  }
  const int2 nj0 = __ldg(G.snj + p), nj1 = __ldg(G.snj + np + p);
  const long long s0 = p * G.scap, s1 = (np + p) * G.scap;
  const int tt = t0 + t1;
#pragma unroll 4
  for (int k = lane; k < tt; k += 32) {
    const bool r1 = k >= t0;
    const int e = r1 ? k - t0 : k;  // entry of the row: S part, J part, D part
    const int2 nj = r1 ? nj1 : nj0;
    const int seg = e < nj.x ? e : (e < nj.x + nj.y ? GW_CAP + (e - nj.x) : 2 * GW_CAP + (e - nj.x - nj.y));
    const long long src = (r1 ? s1 : s0) + seg;
    const long long dst = (r1 ? o1 : o0) + e;
    put(O, dst, __ldg(G.scol + src), __ldg(G.sval + src));
  }
}

// fill of the stashed light pairs: a warp per pair, no shared memory (full occupancy)
__global__ void __launch_bounds__(256) k_g_copy(const GProb G, const int* __restrict__ cnt, const GOut O) {
  const long long nw = (long long)gridDim.x * 8;
  for (long long p = (long long)blockIdx.x * 8 + (threadIdx.x >> 5); p < G.np; p += nw)
    if (__ldg(G.sflag + p)) copy_stashed(G, p, cnt, O);
}

// light engine: a warp per generator pair (rows S_ab, J_ab) with at most GW_CAP candidates;
// heavier pairs are listed (count pass) for the heavy engine
template <bool FILL>
__global__ void __launch_bounds__(32 * GW_WARPS) k_g_light(const GProb G, int* cnt, int* ts, const GOut O) {
  extern __shared__ __align__(16) unsigned char gsm[];
  GBuf<GW_CAP>& B = reinterpret_cast<GBuf<GW_CAP>*>(gsm)[threadIdx.x >> 5];
  const double tau = *G.tau_ptr;
  const long long nw = (long long)gridDim.x * GW_WARPS;
  for (long long p = (long long)blockIdx.x * GW_WARPS + (threadIdx.x >> 5); p < G.np; p += nw) {
    if (FILL && G.scap > 0 && __ldg(G.sflag + p)) continue;  // written by k_g_copy
    const Item it = make_item(G, p, false, 0);
    const long long nsrc = num_sources(G, it);
    const unsigned long long C = total_candidates<32>(G, it, nsrc, B.sc);
    if (C > (unsigned long long)(G.cap < GW_CAP ? G.cap : GW_CAP)) {
      if (!FILL && (threadIdx.x & 31) == 0) {
        G.heavy[atomicAdd(G.nheavy, 1)] = (int)p;
        if (G.scap > 0) G.sflag[p] = 0;
      }
      continue;
    }
    run_item<32, GW_CAP, FILL>(G, it, p, C, B, nullptr, tau, cnt, ts, O);
  }
}

// heavy engine: a CTA per D row and per listed pair; key-range chunks or a key-indexed frame.
// part: 0 = the D rows only, 1 = the listed pairs only, 2 = both
template <bool FILL>
__global__ void __launch_bounds__(GH_NT) k_g_heavy(const GProb G, int* cnt, int* ts, const GOut O, int part) {
  extern __shared__ __align__(16) unsigned char gsm[];
  GBuf<GH_CAP>& B = *reinterpret_cast<GBuf<GH_CAP>*>(gsm);
  GHeavyExtra* X = reinterpret_cast<GHeavyExtra*>(gsm + sizeof(GBuf<GH_CAP>));
  const double tau = *G.tau_ptr;
  const long long nd = part == 1 ? 0 : G.n - 1;
  const long long items = nd + (part == 0 ? 0 : *G.nheavy);
  if (FILL && part != 1 && blockIdx.x == 0 && threadIdx.x == 0) O.row_ptr[G.m] = *O.nnz;
  for (long long t = blockIdx.x; t < items; t += gridDim.x) {
    const bool isd = t < nd;
    if (FILL && isd && G.dseg > 0 && __ldg(G.dflag + t)) {  // stashed D row lam = t + 1: copy its parts
      const int lam = (int)t + 1;
      const long long o = __ldg(O.toff + 2 * G.npt + lam - 1);
      const int nS = __ldg(G.dtot + 2 * t), nJ = __ldg(G.dtot + 2 * t + 1);
      const int tot = __ldg(cnt + 2 * G.np + t);
      if (threadIdx.x == 0) {
        O.row_ptr[2 * G.np + t] = o;
        if (O.K) O.K[2 * G.np + t] = __ldg(G.dK + t);
      }
      const long long base = t * G.drow;
      for (int k = threadIdx.x; k < tot; k += GH_NT) {
        const long long src = base + (k < nS ? k : (k < nS + nJ ? G.dseg + (k - nS) : 2LL * G.dseg + (k - nS - nJ)));
        put(O, o + k, __ldg(G.dcol + src), __ldg(G.dval + src));
      }
      continue;
    }
    const long long p = isd ? 0 : (long long)__ldg(G.heavy + (t - nd));
    const Item it = make_item(G, p, isd, isd ? (int)t + 1 : 0);
    const long long nsrc = num_sources(G, it);
    const unsigned long long C = total_candidates<GH_NT>(G, it, nsrc, B.sc);
    if (C >= (1ull << 32)) {  // sequence numbers are 32-bit
      if (threadIdx.x == 0) atomicOr(G.flags, GF_TOOBIG);
      continue;
    }
    run_item<GH_NT, GH_CAP, FILL>(G, it, isd ? 0 : p, C, B, X, tau, cnt, ts, O);
  }
}

constexpr size_t LIGHT_SMEM = sizeof(GBuf<GW_CAP>) * GW_WARPS;
constexpr size_t HEAVY_SMEM = sizeof(GBuf<GH_CAP>) + sizeof(GHeavyExtra);

int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) !=
                                                  cudaSuccess)
      sms = 148;
  }
  return sms;
}

int light_occ = 1;  // resident light CTAs per SM (set_attrs)
cudaError_t set_attrs() {
  static bool done = false;
  if (done) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k_g_light<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LIGHT_SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_g_light<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LIGHT_SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_g_heavy<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)HEAVY_SMEM);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_g_heavy<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)HEAVY_SMEM);
  if (e == cudaSuccess) {  // the light engines' persistent grids: one wave of resident CTAs
    int a = 0, b = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_g_light<false>, 32 * GW_WARPS, LIGHT_SMEM);
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_g_light<true>, 32 * GW_WARPS, LIGHT_SMEM);
    light_occ = a < b ? a : b;
    if (light_occ < 1) light_occ = 1;
  }
  done = e == cudaSuccess;
  return e;
}

size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

#ifndef SUN_G_SCAP_MAX
#define SUN_G_SCAP_MAX 1024
#endif
// a light pair has <= GW_CAP candidates: S and J parts of <= GW_CAP entries each per row, plus
// <= n - 1 D-part entries (segment of at most SUN_G_SCAP_MAX - 2 GW_CAP: rows with a longer D
// part are assembled again by the fill)
int g_stash_scap(int n) {
  const long long w = 2LL * GW_CAP + n - 1;
  return (int)(((w < SUN_G_SCAP_MAX ? w : SUN_G_SCAP_MAX) + 3) & ~3LL);
}
#ifndef SUN_G_DSEG_MAX
#define SUN_G_DSEG_MAX 16384
#endif
// D rows: S and J parts of at most dseg entries each (<= np distinct keys), D part <= n - 1
static int g_dseg(int n) {
  const long long np = (long long)n * (n - 1) / 2;
  return (int)(((np < SUN_G_DSEG_MAX ? np : SUN_G_DSEG_MAX) + 3) & ~3LL);
}
static int g_drow(int n) { return (int)((2LL * g_dseg(n) + n - 1 + 3) & ~3LL); }
size_t g_stash_bytes(int n) {
  const long long np = (long long)n * (n - 1) / 2;
  if (np <= 0) return 0;
  const size_t sc = (size_t)g_stash_scap(n), nd = (size_t)(n - 1), dr = (size_t)g_drow(n);
  return al256((size_t)np) + al256((size_t)2 * np * sizeof(double)) + al256((size_t)2 * np * sizeof(int2)) +
         al256((size_t)2 * np * sc * sizeof(int32_t)) + al256((size_t)2 * np * sc * sizeof(double)) + al256(nd) + al256(nd * sizeof(double)) +
         al256(nd * dr * sizeof(int32_t)) + al256(nd * dr * sizeof(double));
}
void g_stash_set(GProb& G, char* base) {
  if (!base || G.np <= 0) {
    G.scap = 0;
    G.sflag = nullptr;
    G.scol = nullptr;
    G.sval = nullptr;
    G.sK = nullptr;
    G.snj = nullptr;
    G.dseg = G.drow = 0;
    G.dflag = nullptr;
    G.dcol = nullptr;
    G.dval = nullptr;
    G.dK = nullptr;
    return;
  }
  const long long np = G.np;
  const size_t sc = (size_t)g_stash_scap(G.n);
  size_t off = 0;
  G.sflag = reinterpret_cast<unsigned char*>(base + off); off += al256((size_t)np);
  G.sK = reinterpret_cast<double*>(base + off);           off += al256((size_t)2 * np * sizeof(double));
  G.snj = reinterpret_cast<int2*>(base + off);            off += al256((size_t)2 * np * sizeof(int2));
  G.scol = reinterpret_cast<int32_t*>(base + off);        off += al256((size_t)2 * np * sc * sizeof(int32_t));
  G.sval = reinterpret_cast<double*>(base + off);          off += al256((size_t)2 * np * sc * sizeof(double));
  G.scap = (int)sc;
  const size_t nd = (size_t)(G.n - 1), dr = (size_t)g_drow(G.n);
  G.dflag = reinterpret_cast<unsigned char*>(base + off); off += al256(nd);
  G.dK = reinterpret_cast<double*>(base + off);           off += al256(nd * sizeof(double));
  G.dcol = reinterpret_cast<int32_t*>(base + off);        off += al256(nd * dr * sizeof(int32_t));
  G.dval = reinterpret_cast<double*>(base + off);
  G.dseg = g_dseg(G.n);
  G.drow = (int)dr;
}

GLayout g_layout(int n, int P, const long long* nnzL, size_t base) {
  GLayout g;
  size_t off = al256(base);
  const long long np = (long long)n * (n - 1) / 2;
  g.colcnt = off; off = al256(off + (size_t)(P > 0 ? P : 1) * (n + 1) * sizeof(int));
  g.cp = off;     off = al256(off + (size_t)(P > 0 ? P : 1) * (n + 1) * sizeof(int));
  g.xr = off;
  long long tot = 0;
  for (int p = 0; p < P; ++p) {
    g.xr_off[p] = tot;
    tot += nnzL[p];
  }
  off = al256(off + (size_t)(tot > 0 ? tot : 1) * sizeof(int2));
  g.heavy0 = off; off = al256(off + (size_t)(np > 0 ? np : 1) * sizeof(int));
  g.heavy1 = off; off = al256(off + (size_t)(np > 0 ? np : 1) * sizeof(int));
  g.nheavy = off; off = al256(off + 2 * sizeof(int));
  g.nrb = (n + GE_THREADS - 1) / GE_THREADS;
  g.blk = off;    off = al256(off + (size_t)(2 + P) * g.nrb * sizeof(GBlk));
  g.dtot0 = off;  off = al256(off + (size_t)2 * n * sizeof(int));
  g.dtot1 = off;  off = al256(off + (size_t)2 * n * sizeof(int));
  g.total = off;
  return g;
}

cudaError_t g_expand(const GExpandIn& in, char* ws, const GLayout& gl, double* inv, int* zero32, long long nz32,
                     unsigned long long* zero64, long long nz64, GHeaderRef hdr, cudaStream_t st) {
  const int n = in.n, P = in.nops - 2;
  int* colcnt = (int*)(ws + gl.colcnt);
  int* cp = (int*)(ws + gl.cp);
  cudaError_t e = cudaMemsetAsync(colcnt, 0, (size_t)(P > 0 ? P : 1) * (n + 1) * sizeof(int), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(ws + gl.nheavy, 0, 2 * sizeof(int), st);
  if (e != cudaSuccess) return e;
  GExpandArgs A;
  A.in = in;
  A.blk = (GBlk*)(ws + gl.blk);
  A.colcnt = colcnt;
  A.inv = inv;
  A.zero32 = zero32;
  A.zero64 = zero64;
  A.nz32 = nz32;
  A.nz64 = nz64;
  A.hdr = hdr;
  A.nrb = (int)gl.nrb;
  A.nA = (int)gl.nrb * in.nops;
  A.nB = (n + GE_THREADS - 1) / GE_THREADS;
  k_g_expand<<<(unsigned)(A.nA + A.nB), GE_THREADS, 0, st>>>(A);
  if ((e = cudaGetLastError()) != cudaSuccess || P == 0) return e;
  GColArgs C;
  C.n = n;
  C.P = P;
  for (int p = 0; p < P; ++p) {
    C.rp[p] = in.rp[2 + p];
    C.ci[p] = in.ci[2 + p];
    C.xr[p] = (int2*)(ws + gl.xr) + gl.xr_off[p];
  }
  k_g_colscan<<<(unsigned)P, 1024, 0, st>>>(n, colcnt, cp);
  const long long rows = (long long)P * n;
  k_g_scatter<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(C, colcnt);
  k_g_colsort<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(C, cp);
  return cudaGetLastError();
}

cudaError_t g_prepare() {
  (void)sm_count();
  return set_attrs();
}

// The D rows (heavy engine, part 0) run on `aux` concurrently with the light pairs on `st`; the
// listed heavy pairs (part 1) follow the light count on `st` (the list is its output).  The
// caller orders `aux` after `st` before and joins it afterwards.
cudaError_t g_count(const GProb& pr, int* cnt, int* ts, cudaStream_t st, cudaStream_t aux) {
  cudaError_t e = set_attrs();
  if (e != cudaSuccess) return e;
  GOut none{};
  const int sms = sm_count();
  const long long lw = (pr.np + GW_WARPS - 1) / GW_WARPS;
  const long long lcap = (long long)light_occ * sms;
  const unsigned lg = (unsigned)(lw < lcap ? (lw > 0 ? lw : 1) : lcap);
  const unsigned hd = (unsigned)(pr.n - 1 < 2LL * sms ? pr.n - 1 : 2LL * sms);
  k_g_heavy<false><<<hd > 0 ? hd : 1, GH_NT, HEAVY_SMEM, aux>>>(pr, cnt, ts, none, 0);
  k_g_light<false><<<lg, 32 * GW_WARPS, LIGHT_SMEM, st>>>(pr, cnt, ts, none);
  k_g_heavy<false><<<(unsigned)(2 * sms), GH_NT, HEAVY_SMEM, st>>>(pr, cnt, ts, none, 1);
  return cudaGetLastError();
}

cudaError_t g_fill(const GProb& pr, const int* cnt, const GOut& out, cudaStream_t st, cudaStream_t aux) {
  cudaError_t e = set_attrs();
  if (e != cudaSuccess) return e;
  const int sms = sm_count();
  const long long lw = (pr.np + GW_WARPS - 1) / GW_WARPS;
  const long long lcap = (long long)light_occ * sms;
  const unsigned lg = (unsigned)(lw < lcap ? (lw > 0 ? lw : 1) : lcap);
  k_g_heavy<true><<<(unsigned)(2 * sms), GH_NT, HEAVY_SMEM, aux>>>(pr, const_cast<int*>(cnt), nullptr, out, 2);
  if (pr.scap > 0) {
    const long long cw = (pr.np + 7) / 8, cc = 8LL * sms;
    k_g_copy<<<(unsigned)(cw < cc ? (cw > 0 ? cw : 1) : cc), 256, 0, st>>>(pr, cnt, out);
  }
  k_g_light<true><<<lg, 32 * GW_WARPS, LIGHT_SMEM, st>>>(pr, const_cast<int*>(cnt), nullptr, out);
  return cudaGetLastError();
}

}  // namespace sung
