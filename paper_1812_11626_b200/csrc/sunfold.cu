// sunfold.cu — C-ABI and launch logic of the B200 SU(N) unfold (include/sunfold.h).
//
// Pipeline (Table I Step 2; two-step CRS fill P:369-370):
//   sun_plan_create : k_analyze   bandwidths, Frobenius norms, CSR validation  -> 1 readback
//   sun_count       : k_zero, k_scatter, k_band_k   (a1) expand to band storage, K = H + i/2 M
//                     k_count<mode>                  (a3) per-row counts (values thresholded)
//                     k_scan                         (a4) tile offsets, nnz
//   sun_plan_nnz    : 16-byte readback (nnz Q0, Q1) + validation flags
//   sun_unfold      : k_fill<mode>                   (a5) row_ptr, col, val, K; (a6) Q1
//   sun_apply       : k_apply                        (a7) dv/dt = Q0 v + eps Q1 v + K
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "../../include/sunfold.h"
#include "sunfold_kernels.cuh"

using namespace sunk;

namespace {

constexpr int MAXOPS = 66;     // H0, H1 and up to 64 dissipators
constexpr int WLMAX = WMAX / 2;  // wK >= 2 wL
constexpr int F_MALFORMED = 1, F_H0_NOT_HERM = 2, F_H1_NOT_HERM = 4;
constexpr int THREAD_TP = 128;   // thread mode: pairs per tile == threads per CTA
constexpr int WARP_TP = 64;      // warp mode: pairs per tile
constexpr int WARP_THREADS = 256;
constexpr int STAGE_BYTES = 72 * 1024;  // thread-mode shared staging per CTA
constexpr int FAR_MAXPOS = 1024;

struct DevHeader {
  int flags;
  int pad;
  long long nnz[2];
  int bw[MAXOPS];
  double nrm2[MAXOPS];
};

struct OpDesc {
  const int64_t* rp;
  const int32_t* ci;
  const double2* v;
};
struct OpList {
  OpDesc op[MAXOPS];
  int nops;
  int n;
};

thread_local char g_errbuf[512];

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct FarPos {
  int dc[1024];
  int dd[1024];
};

struct Layout {
  size_t hdr, fp0, fp1, sqrtg, kb0, hb0, hb1, lb, cnt0, cnt1, ts0, ts1, total;
  long long maxslots;
};

Layout make_layout(int n, int P) {
  Layout L;
  long long m = (long long)n * n - 1;
  long long np = (long long)n * (n - 1) / 2;
  long long maxslots = 2 * (np / 32 + 2) + n + 2;
  size_t off = 0;
  L.hdr = off; off = align256(off + sizeof(DevHeader));
  L.fp0 = off; off = align256(off + sizeof(FarPos));
  L.fp1 = off; off = align256(off + sizeof(FarPos));
  L.sqrtg = off; off = align256(off + MAXOPS * sizeof(double));
  L.kb0 = off; off = align256(off + (size_t)n * (2 * WMAX + 1) * sizeof(double2));
  L.hb0 = off; off = align256(off + (size_t)n * (2 * WMAX + 1) * sizeof(double2));
  L.hb1 = off; off = align256(off + (size_t)n * (2 * WMAX + 1) * sizeof(double2));
  L.lb = off;  off = align256(off + (size_t)(P > 0 ? P : 1) * n * (2 * WLMAX + 1) * sizeof(double2));
  L.cnt0 = off; off = align256(off + (size_t)m * sizeof(int));
  L.cnt1 = off; off = align256(off + (size_t)m * sizeof(int));
  L.ts0 = off; off = align256(off + (size_t)maxslots * sizeof(long long));
  L.ts1 = off; off = align256(off + (size_t)maxslots * sizeof(long long));
  L.total = off;
  L.maxslots = maxslots;
  return L;
}

}  // namespace

struct sun_plan_s {
  int n, P, has_h1;
  FarPos hfp[2];   // far-position tables (host copies; uploaded in sun_plan_create)
  double hsqrtg[MAXOPS];
  sun_zcsr H0, H1;
  std::vector<sun_zcsr> L;
  std::vector<double> gamma;
  char* ws;
  size_t ws_bytes;
  Layout lay;
  int wH0, wH1, wL, wK;
  double tau0, tau1, herm_tol0, herm_tol1;
  Prob pr[2];
  int counted;
  cudaStream_t count_stream;
  long long nnz[2];
  int npos_far[2];
  std::vector<int> pos_dc[2], pos_dd[2];
};

// =========================================================================================
// Kernels
// =========================================================================================

// (validation + pattern analysis) one CTA per operator: half-bandwidth, ||.||_F^2, CSR checks.
__global__ void k_analyze(OpList ops, DevHeader* hdr) {
  const int op = blockIdx.x;
  const OpDesc d = ops.op[op];
  const int n = ops.n;
  __shared__ double red[256];
  __shared__ int bwmax;
  if (threadIdx.x == 0) bwmax = 0;
  __syncthreads();
  double acc = 0.0;
  int bw = 0, bad = 0;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    int64_t lo = d.rp[r], hi = d.rp[r + 1];
    if (hi < lo) { bad = 1; continue; }
    int prev = -1;
    for (int64_t k = lo; k < hi; ++k) {
      int c = d.ci[k];
      if (c < 0 || c >= n || c <= prev) bad = 1;
      prev = c;
      int o = c > r ? c - r : r - c;
      double2 v = d.v[k];
      if (v.x != 0.0 || v.y != 0.0) bw = o > bw ? o : bw;
      acc += v.x * v.x + v.y * v.y;
    }
  }
  if (bad) atomicOr(&hdr->flags, F_MALFORMED);
  atomicMax(&bwmax, bw);
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {  // fixed-order tree: deterministic
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    hdr->bw[op] = bwmax;
    hdr->nrm2[op] = red[0];
  }
}

__global__ void k_zero(double* p, long long count) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
    p[i] = 0.0;
}

// (a1) CSR -> band storage.  ops: 0 = H0 (into Hb0, width wK), 1 = H1 (Hb1, width wH1),
// 2+p = L_p (Lb[p], width wL, scaled by sqrt(gamma_p)).  One thread per (operator, row).
__global__ void k_scatter(OpList ops, int has_h1, double2* hb0, int wK, double2* hb1, int wH1, double2* lb,
                          int wL, const double* __restrict__ sqrtg) {
  const int n = ops.n;
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)ops.nops * n) return;
  int op = (int)(t / n), r = (int)(t % n);
  if (op == 1 && !has_h1) return;
  const OpDesc d = ops.op[op];
  double2* dst;
  int w;
  double s = 1.0;
  if (op == 0) { dst = hb0; w = wK; }
  else if (op == 1) { dst = hb1; w = wH1; }
  else { dst = lb + (long long)(op - 2) * n * (2 * wL + 1); w = wL; s = sqrtg[op - 2]; }
  for (int64_t k = d.rp[r]; k < d.rp[r + 1]; ++k) {
    int o = d.ci[k] - r;
    if (o < -w || o > w) continue;  // only exact zeros can lie outside (bandwidth from k_analyze)
    double2 v = d.v[k];
    dst[(long long)r * (2 * w + 1) + (o + w)] = make_double2(s * v.x, s * v.y);
  }
}

// (a1) K = H0 + (i/2) M, M = sum_p Lt_p^+ Lt_p (Lt = sqrt(gamma) L); Hermiticity checks of H0, H1.
__global__ void k_band_k(int n, int P, const double2* __restrict__ hb0, double2* kb0, int wK,
                         const double2* __restrict__ lb, int wL, const double2* __restrict__ hb1, int wH1,
                         int has_h1, double tol0, double tol1, DevHeader* hdr) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int sw = 2 * wK + 1;
  if (t >= (long long)n * sw) return;
  int r = (int)(t / sw), o = (int)(t % sw) - wK;
  int c = r + o;
  if (c < 0 || c >= n) {
    kb0[t] = make_double2(0.0, 0.0);
    return;
  }
  double mx = 0.0, my = 0.0;
  int lo = max(r, c) - wL, hi = min(r, c) + wL;
  if (lo < 0) lo = 0;
  if (hi > n - 1) hi = n - 1;
  for (int p = 0; p < P; ++p) {
    const double2* Lp = lb + (long long)p * n * (2 * wL + 1);
    for (int x = lo; x <= hi; ++x) {
      double2 a = Lp[(long long)x * (2 * wL + 1) + (r - x + wL)];  // L_xr
      double2 b = Lp[(long long)x * (2 * wL + 1) + (c - x + wL)];  // L_xc
      mx += a.x * b.x + a.y * b.y;  // conj(L_xr) L_xc
      my += a.x * b.y - a.y * b.x;
    }
  }
  double2 h = hb0[t];
  kb0[t] = make_double2(h.x - 0.5 * my, h.y + 0.5 * mx);
  double2 ht = hb0[(long long)c * sw + (r - c + wK)];
  if (fabs(h.x - ht.x) > tol0 || fabs(h.y + ht.y) > tol0) atomicOr(&hdr->flags, F_H0_NOT_HERM);
  if (has_h1 && o >= -wH1 && o <= wH1) {
    double2 g = hb1[(long long)r * (2 * wH1 + 1) + (o + wH1)];
    double2 gt = hb1[(long long)c * (2 * wH1 + 1) + (r - c + wH1)];
    if (fabs(g.x - gt.x) > tol1 || fabs(g.y + gt.y) > tol1) atomicOr(&hdr->flags, F_H1_NOT_HERM);
  }
}

// ---------------------------------------------------------------------------------------
// (a3) count pass.  Grid: npt pair tiles, then ndt D tiles.
// ---------------------------------------------------------------------------------------

template <int MODE>
__global__ void __launch_bounds__(MODE == 0 ? THREAD_TP : WARP_THREADS)
    k_count(Prob pr, const FarPos* __restrict__ fp, int npos_far, int* __restrict__ cnt,
            long long* __restrict__ tsum) {
  __shared__ double scratch[(MODE == 0 ? THREAD_TP : WARP_THREADS) / 32][4][WIN_MAX + 2];
  __shared__ int wtot[32];
  __shared__ int spos_dc[MODE == 1 ? FAR_MAXPOS : 1], spos_dd[MODE == 1 ? FAR_MAXPOS : 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  double* gS = scratch[wid][0];
  double* gJ = scratch[wid][1];
  double* pS = scratch[wid][2];
  double* pJ = scratch[wid][3];
  const Seg none = {nullptr, nullptr, nullptr, nullptr};
  const long long t = blockIdx.x;
  if (t < pr.npt) {
    int cS = 0, cJ = 0;
    if (MODE == 0) {
      long long p = t * pr.tp + threadIdx.x;
      bool valid = p < pr.np;
      int a = 0, b = 1;
      if (valid) pair_decode(pr.n, p, a, b);
      bool far = valid && (b - a > 2 * pr.W);
      if (far) {
        int nre, nim;
        far_pair_thread<false>(pr, a, b, nre, nim, none, 0, none, 0);
        cS = cJ = nre + nim;
      }
      unsigned nm = __ballot_sync(FULL, valid && !far);
      while (nm) {
        int src = __ffs(nm) - 1;
        nm &= nm - 1;
        int aa = __shfl_sync(FULL, a, src), bb = __shfl_sync(FULL, b, src);
        int c1, c2;
        double k1, k2;
        warp_near_pair<false>(pr, aa, bb, gS, gJ, pS, pJ, c1, c2, k1, k2, none, 0, none, 0);
        if (lane == src) { cS = c1; cJ = c2; }
      }
      if (valid) {
        cnt[p] = cS;
        cnt[pr.np + p] = cJ;
      }
    } else {
      for (int i = threadIdx.x; i < npos_far; i += blockDim.x) {
        spos_dc[i] = fp->dc[i];
        spos_dd[i] = fp->dd[i];
      }
      __syncthreads();
      for (int i = wid; i < pr.tp; i += nwarps) {
        long long p = t * pr.tp + i;
        if (p >= pr.np) break;
        int a, b;
        pair_decode(pr.n, p, a, b);
        int c1, c2;
        if (b - a > 2 * pr.W) {
          warp_far_pair<false>(pr, a, b, spos_dc, spos_dd, npos_far, c1, none, 0, none, 0);
          c2 = c1;
        } else {
          double k1, k2;
          warp_near_pair<false>(pr, a, b, gS, gJ, pS, pJ, c1, c2, k1, k2, none, 0, none, 0);
        }
        if (lane == 0) {
          cnt[p] = c1;
          cnt[pr.np + p] = c2;
          cS += c1;
          cJ += c2;
        }
      }
    }
    int totS, totJ;
    block_exclusive_scan(cS, wtot, totS);
    block_exclusive_scan(cJ, wtot, totJ);
    if (threadIdx.x == 0) {
      tsum[t] = totS;
      tsum[pr.npt + t] = totJ;
    }
  } else {
    const long long u = t - pr.npt;
    int c = 0;
    int lam = (int)(u * nwarps + wid + 1);
    if (lam <= pr.n - 1) {
      double kv;
      warp_d_row<false>(pr, lam, gS, pS, c, kv, none, 0);
      if (lane == 0) cnt[2 * pr.np + lam - 1] = c;
    }
    int tot;
    block_exclusive_scan(lane == 0 ? c : 0, wtot, tot);
    if (threadIdx.x == 0) tsum[2 * pr.npt + u] = tot;
  }
}

// (a4) exclusive scan of the tile sums (one CTA, fixed order: deterministic); nnz -> hdr.
__global__ void __launch_bounds__(1024) k_scan(long long* ts, long long nslots, long long* nnz_out) {
  __shared__ long long wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  long long per = (nslots + blockDim.x - 1) / blockDim.x;
  long long lo = tid * per, hi = lo + per < nslots ? lo + per : nslots;
  long long local = 0;
  for (long long i = lo; i < hi; ++i) local += ts[i];
  long long x = local;
  for (int o = 1; o < 32; o <<= 1) {
    long long y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    long long s = wsum[lane];
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(FULL, s, o);
      if (lane >= o) s += y;
    }
    wsum[lane] = s;
  }
  __syncthreads();
  long long run = (wid > 0 ? wsum[wid - 1] : 0) + x - local;
  for (long long i = lo; i < hi; ++i) {
    long long v = ts[i];
    ts[i] = run;
    run += v;
  }
  if (tid == blockDim.x - 1) *nnz_out = wsum[31];
}

// ---------------------------------------------------------------------------------------
// (a5) fill pass (+ K).  Same tiling as k_count.
// ---------------------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(MODE == 0 ? THREAD_TP : WARP_THREADS)
    k_fill(Prob pr, const FarPos* __restrict__ fp, int npos_far, const int* __restrict__ cnt,
           const long long* __restrict__ toff, const long long* __restrict__ nnz_total,
           int64_t* __restrict__ row_ptr, int32_t* __restrict__ col, double* __restrict__ val,
           double* __restrict__ K, int cap) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ double scratch[(MODE == 0 ? THREAD_TP : WARP_THREADS) / 32][4][WIN_MAX + 2];
  __shared__ int wtot[32];
  __shared__ int spos_dc[MODE == 1 ? FAR_MAXPOS : 1], spos_dd[MODE == 1 ? FAR_MAXPOS : 1];
  __shared__ long long soffS[MODE == 1 ? WARP_TP : 1], soffJ[MODE == 1 ? WARP_TP : 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  double* gS = scratch[wid][0];
  double* gJ = scratch[wid][1];
  double* pS = scratch[wid][2];
  double* pJ = scratch[wid][3];
  const long long t = blockIdx.x;
  const long long np = pr.np;
  if (t == 0 && threadIdx.x == 0) row_ptr[pr.m] = *nnz_total;
  if (t < pr.npt) {
    const long long baseS = toff[t], baseJ = toff[pr.npt + t];
    if (MODE == 0) {
      long long p = t * pr.tp + threadIdx.x;
      bool valid = p < np;
      int cS = valid ? cnt[p] : 0, cJ = valid ? cnt[np + p] : 0;
      int totS, totJ;
      int exS = block_exclusive_scan(cS, wtot, totS);
      int exJ = block_exclusive_scan(cJ, wtot, totJ);
      if (valid) {
        row_ptr[p] = baseS + exS;
        row_ptr[np + p] = baseJ + exJ;
      }
      const bool staged = (totS + totJ) <= cap;
      double* sval = reinterpret_cast<double*>(dyn);
      int* scol = reinterpret_cast<int*>(dyn + (size_t)cap * sizeof(double));
      Seg sS, sJ;
      if (staged) {
        sS = {scol, sval, nullptr, nullptr};
        sJ = {scol + totS, sval + totS, nullptr, nullptr};
      } else {
        sS = {nullptr, nullptr, col + baseS, val + baseS};
        sJ = {nullptr, nullptr, col + baseJ, val + baseJ};
      }
      int a = 0, b = 1;
      if (valid) pair_decode(pr.n, p, a, b);
      bool far = valid && (b - a > 2 * pr.W);
      double kS = 0.0, kJ = 0.0;
      if (far) {
        int nre, nim;
        far_pair_thread<false>(pr, a, b, nre, nim, sS, 0, sJ, 0);
        far_pair_thread<true>(pr, a, b, nre, nim, sS, exS, sJ, exJ);
      }
      unsigned nm = __ballot_sync(FULL, valid && !far);
      while (nm) {
        int src = __ffs(nm) - 1;
        nm &= nm - 1;
        int aa = __shfl_sync(FULL, a, src), bb = __shfl_sync(FULL, b, src);
        long long oS = __shfl_sync(FULL, exS, src), oJ = __shfl_sync(FULL, exJ, src);
        int c1, c2;
        double k1, k2;
        warp_near_pair<true>(pr, aa, bb, gS, gJ, pS, pJ, c1, c2, k1, k2, sS, oS, sJ, oJ);
        if (lane == src) { kS = k1; kJ = k2; }
      }
      if (valid && pr.has_k) {
        K[p] = kS;
        K[np + p] = kJ;
      }
      __syncthreads();
      if (staged) {
        for (int i = threadIdx.x; i < totS; i += blockDim.x) {
          col[baseS + i] = scol[i];
          val[baseS + i] = sval[i];
        }
        for (int i = threadIdx.x; i < totJ; i += blockDim.x) {
          col[baseJ + i] = scol[totS + i];
          val[baseJ + i] = sval[totS + i];
        }
      }
    } else {
      for (int i = threadIdx.x; i < npos_far; i += blockDim.x) {
        spos_dc[i] = fp->dc[i];
        spos_dd[i] = fp->dd[i];
      }
      int i0 = threadIdx.x;
      long long p0 = t * pr.tp + i0;
      bool valid = i0 < pr.tp && p0 < np;
      int cS = valid ? cnt[p0] : 0, cJ = valid ? cnt[np + p0] : 0;
      int totS, totJ;
      int exS = block_exclusive_scan(cS, wtot, totS);
      int exJ = block_exclusive_scan(cJ, wtot, totJ);
      if (i0 < WARP_TP) {
        soffS[i0] = exS;
        soffJ[i0] = exJ;
      }
      if (valid) {
        row_ptr[p0] = baseS + exS;
        row_ptr[np + p0] = baseJ + exJ;
      }
      __syncthreads();
      const Seg sS = {nullptr, nullptr, col + baseS, val + baseS};
      const Seg sJ = {nullptr, nullptr, col + baseJ, val + baseJ};
      for (int i = wid; i < pr.tp; i += nwarps) {
        long long p = t * pr.tp + i;
        if (p >= np) break;
        int a, b;
        pair_decode(pr.n, p, a, b);
        double k1 = 0.0, k2 = 0.0;
        int c1, c2;
        if (b - a > 2 * pr.W) {
          warp_far_pair<true>(pr, a, b, spos_dc, spos_dd, npos_far, c1, sS, soffS[i], sJ, soffJ[i]);
        } else {
          warp_near_pair<true>(pr, a, b, gS, gJ, pS, pJ, c1, c2, k1, k2, sS, soffS[i], sJ, soffJ[i]);
        }
        if (lane == 0 && pr.has_k) {
          K[p] = k1;
          K[np + p] = k2;
        }
      }
    }
  } else {
    const long long u = t - pr.npt;
    const long long baseD = toff[2 * pr.npt + u];
    int lam = (int)(u * nwarps + wid + 1);
    bool valid = lam <= pr.n - 1;
    int c = valid ? cnt[2 * np + lam - 1] : 0;
    int tot;
    int ex = block_exclusive_scan(lane == 0 ? c : 0, wtot, tot);
    ex = __shfl_sync(FULL, ex, 0);
    if (valid) {
      if (lane == 0) row_ptr[2 * np + lam - 1] = baseD + ex;
      const Seg sD = {nullptr, nullptr, col + baseD, val + baseD};
      int cc;
      double kv;
      warp_d_row<true>(pr, lam, gS, pS, cc, kv, sD, ex);
      if (lane == 0 && pr.has_k) K[2 * np + lam - 1] = kv;
    }
  }
}

// (a7) dv/dt = Q0 v + eps Q1 v + K ; 8 lanes per row, fixed-order reduction.
__global__ void k_apply(long long m, const int64_t* __restrict__ rp0, const int32_t* __restrict__ c0,
                        const double* __restrict__ v0, const int64_t* __restrict__ rp1,
                        const int32_t* __restrict__ c1, const double* __restrict__ v1, double eps,
                        const double* __restrict__ Kv, const double* __restrict__ x, double* __restrict__ y) {
  long long gt = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long row = gt >> 3;
  int sub = threadIdx.x & 7;
  bool ok = row < m;
  double s0 = 0.0, s1 = 0.0;
  if (ok) {
    for (int64_t k = rp0[row] + sub; k < rp0[row + 1]; k += 8) s0 += v0[k] * __ldg(&x[c0[k]]);
    if (rp1)
      for (int64_t k = rp1[row] + sub; k < rp1[row + 1]; k += 8) s1 += v1[k] * __ldg(&x[c1[k]]);
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(FULL, s0, o);
    s1 += __shfl_xor_sync(FULL, s1, o);
  }
  if (ok && sub == 0) y[row] = s0 + eps * s1 + (Kv ? Kv[row] : 0.0);
}

// =========================================================================================
// Host side
// =========================================================================================
namespace {

int cuda_fail(cudaError_t e) {
  snprintf(g_errbuf, sizeof(g_errbuf), "CUDA error: %s", cudaGetErrorString(e));
  return SUN_ERR_CUDA;
}
#define CK(x)                                    \
  do {                                           \
    cudaError_t e_ = (x);                        \
    if (e_ != cudaSuccess) return cuda_fail(e_); \
  } while (0)

bool zcsr_ok(const sun_zcsr* A, int n) {
  return A && A->n == n && A->nnz >= 0 && A->row_ptr && (A->nnz == 0 || (A->col && A->val));
}

// far-pair position list in far_positions() order (relative offsets to (a, b))
void build_far_positions(int W, int wL, int wK, std::vector<int>& dc, std::vector<int>& dd) {
  dc.clear();
  dd.clear();
  for (int a = -W; a <= W; ++a) {
    int aa = a < 0 ? -a : a;
    if (a == 0) {
      for (int b = -W; b <= W; ++b) { dc.push_back(a); dd.push_back(b); }
    } else if (aa <= wL) {
      for (int b = -wL; b <= wL; ++b) { dc.push_back(a); dd.push_back(b); }
    } else if (aa <= wK) {
      dc.push_back(a);
      dd.push_back(0);
    }
  }
}

void setup_prob(sun_plan_s* pl, int which) {
  Prob& pr = pl->pr[which];
  const Layout& L = pl->lay;
  pr.n = pl->n;
  pr.np = (long long)pl->n * (pl->n - 1) / 2;
  pr.m = (long long)pl->n * pl->n - 1;
  if (which == 0) {
    pr.P = pl->P;
    pr.wK = pl->wK;
    pr.wL = pl->wL;
    pr.K = {reinterpret_cast<const double2*>(pl->ws + L.kb0), pl->wK};
    pr.H = {reinterpret_cast<const double2*>(pl->ws + L.hb0), pl->wK};
    pr.L = reinterpret_cast<const double2*>(pl->ws + L.lb);
    pr.tau = pl->tau0;
    pr.has_k = 1;
  } else {
    pr.P = 0;
    pr.wK = pl->wH1;
    pr.wL = 0;
    pr.K = {reinterpret_cast<const double2*>(pl->ws + L.hb1), pl->wH1};
    pr.H = pr.K;
    pr.L = nullptr;
    pr.tau = pl->tau1;
    pr.has_k = 0;
  }
  pr.W = pr.wK > pr.wL ? pr.wK : pr.wL;
  build_far_positions(pr.W, pr.wL, pr.wK, pl->pos_dc[which], pl->pos_dd[which]);
  int npos = (int)pl->pos_dc[which].size();
  pl->npos_far[which] = npos;
  for (int i = 0; i < npos && i < FAR_MAXPOS; ++i) {
    pl->hfp[which].dc[i] = pl->pos_dc[which][i];
    pl->hfp[which].dd[i] = pl->pos_dd[which][i];
  }
  // thread-per-pair with shared staging while a pair emits few entries (<= 4 npos); else
  // warp-per-pair with direct coalesced row stores
  pr.mode = (npos <= 16) ? 0 : 1;
  pr.tp = pr.mode == 0 ? THREAD_TP : WARP_TP;
  pr.npt = (pr.np + pr.tp - 1) / pr.tp;
  int dpt = (pr.mode == 0 ? THREAD_TP : WARP_THREADS) / 32;
  pr.ndt = (pl->n - 1 + dpt - 1) / dpt;
}

int stage_cap_entries() { return STAGE_BYTES / (int)(sizeof(double) + sizeof(int)); }

}  // namespace

extern "C" {

const char* sun_version(void) { return "sunfold 0.1 (sm_100a, fp64)"; }

const char* sun_status_string(int status) {
  switch (status) {
    case SUN_OK: return "ok";
    case SUN_ERR_ARG: return "invalid argument (null/inconsistent pointers or malformed CSR)";
    case SUN_ERR_DIM: return "invalid dimension (need 2 <= N <= 46340 and equal N for all operators)";
    case SUN_ERR_NOT_HERMITIAN: return "H0 or H1 is not Hermitian (max|H - H^+| > 1e-12 ||H||_F)";
    case SUN_ERR_RATE: return "invalid rate (gamma_p must be finite and >= 0)";
    case SUN_ERR_CAPACITY: return "output CSR capacity below the required nnz";
    case SUN_ERR_CUDA: return g_errbuf[0] ? g_errbuf : "CUDA error";
    case SUN_ERR_BANDWIDTH:
      return "operator half-bandwidth exceeds the banded kernels' limit (max(w_H, 2 w_L) <= 15, w_L <= 7)";
    case SUN_ERR_STATE: return "call out of sequence";
    default: return "unknown status";
  }
}

int64_t sun_gen_index(int32_t n, int32_t kind, int32_t a, int32_t b) {
  if (n < 2) return -1;
  long long np = (long long)n * (n - 1) / 2;
  if (kind == 0 || kind == 1) {
    if (a < 0 || b <= a || b >= n) return -1;
    long long p = (long long)a * (2LL * n - a - 1) / 2 + (b - a - 1);
    return kind == 0 ? p : np + p;
  }
  if (kind == 2) {
    if (a < 1 || a > n - 1) return -1;
    return 2 * np + a - 1;
  }
  return -1;
}

size_t sun_workspace_bytes(int32_t n, int32_t P) {
  if (n < 2 || n > 46340 || P < 0 || P > MAXOPS - 2) return 0;
  return make_layout(n, P).total;
}

int sun_plan_create(sun_plan* out, const sun_zcsr* H0, const sun_zcsr* H1, const sun_zcsr* const* L,
                    const double* gamma, int32_t P, void* workspace, size_t workspace_bytes, void* stream) {
  if (!out) return SUN_ERR_ARG;
  *out = nullptr;
  g_errbuf[0] = 0;
  if (!H0) return SUN_ERR_ARG;
  const int n = H0->n;
  if (n < 2 || n > 46340) return SUN_ERR_DIM;
  if (P < 0 || P > MAXOPS - 2 || (P > 0 && (!L || !gamma))) return SUN_ERR_ARG;
  if (!zcsr_ok(H0, n)) return SUN_ERR_ARG;
  if (H1) {
    if (H1->n != n) return SUN_ERR_DIM;
    if (!zcsr_ok(H1, n)) return SUN_ERR_ARG;
  }
  for (int p = 0; p < P; ++p) {
    if (!L[p]) return SUN_ERR_ARG;
    if (L[p]->n != n) return SUN_ERR_DIM;
    if (!zcsr_ok(L[p], n)) return SUN_ERR_ARG;
    if (!(gamma[p] >= 0.0) || !isfinite(gamma[p])) return SUN_ERR_RATE;
  }
  Layout lay = make_layout(n, P);
  if (!workspace || workspace_bytes < lay.total || ((uintptr_t)workspace & 255)) return SUN_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = (char*)workspace;
  DevHeader* hdr = (DevHeader*)(ws + lay.hdr);
  OpList ops;
  memset(&ops, 0, sizeof(ops));
  ops.n = n;
  ops.nops = 2 + P;
  ops.op[0] = {H0->row_ptr, H0->col, (const double2*)H0->val};
  ops.op[1] = H1 ? OpDesc{H1->row_ptr, H1->col, (const double2*)H1->val} : ops.op[0];
  for (int p = 0; p < P; ++p) ops.op[2 + p] = {L[p]->row_ptr, L[p]->col, (const double2*)L[p]->val};
  CK(cudaMemsetAsync(hdr, 0, sizeof(DevHeader), st));
  k_analyze<<<ops.nops, 256, 0, st>>>(ops, hdr);
  CK(cudaGetLastError());
  DevHeader h;
  CK(cudaMemcpyAsync(&h, hdr, sizeof(DevHeader), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (h.flags & F_MALFORMED) return SUN_ERR_ARG;
  sun_plan_s* pl = new sun_plan_s();
  pl->n = n;
  pl->P = P;
  pl->has_h1 = H1 != nullptr;
  pl->H0 = *H0;
  if (H1) pl->H1 = *H1;
  for (int p = 0; p < P; ++p) {
    pl->L.push_back(*L[p]);
    pl->gamma.push_back(gamma[p]);
    pl->hsqrtg[p] = sqrt(gamma[p]);
  }
  pl->ws = ws;
  pl->ws_bytes = workspace_bytes;
  pl->lay = lay;
  pl->wH0 = h.bw[0];
  pl->wH1 = H1 ? h.bw[1] : 0;
  int wL = 0;
  for (int p = 0; p < P; ++p) wL = h.bw[2 + p] > wL ? h.bw[2 + p] : wL;
  pl->wL = wL;
  pl->wK = pl->wH0 > 2 * wL ? pl->wH0 : 2 * wL;
  if (pl->wK > n - 1) pl->wK = n - 1;  // M = L^+L has half-bandwidth <= n-1
  if (pl->wK < pl->wH0) pl->wK = pl->wH0;
  if (pl->wK > WMAX || pl->wL > WLMAX || pl->wH1 > WMAX) {
    delete pl;
    return SUN_ERR_BANDWIDTH;
  }
  double s0 = sqrt(h.nrm2[0]);
  for (int p = 0; p < P; ++p) s0 += gamma[p] * h.nrm2[2 + p];
  pl->tau0 = 1e-14 * s0;
  pl->tau1 = H1 ? 1e-14 * sqrt(h.nrm2[1]) : 0.0;
  pl->herm_tol0 = 1e-12 * sqrt(h.nrm2[0]);
  pl->herm_tol1 = H1 ? 1e-12 * sqrt(h.nrm2[1]) : 0.0;
  setup_prob(pl, 0);
  if (pl->has_h1) setup_prob(pl, 1);
  if (pl->npos_far[0] > FAR_MAXPOS || (pl->has_h1 && pl->npos_far[1] > FAR_MAXPOS)) {
    delete pl;
    return SUN_ERR_BANDWIDTH;
  }
  // constant per-plan tables
  cudaError_t e = cudaMemcpyAsync(ws + lay.fp0, &pl->hfp[0], sizeof(FarPos), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && pl->has_h1)
    e = cudaMemcpyAsync(ws + lay.fp1, &pl->hfp[1], sizeof(FarPos), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && P > 0)
    e = cudaMemcpyAsync(ws + lay.sqrtg, pl->hsqrtg, P * sizeof(double), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) {
    delete pl;
    return cuda_fail(e);
  }
  pl->counted = 0;
  pl->nnz[0] = pl->nnz[1] = -1;
  *out = pl;
  return SUN_OK;
}

int sun_count(sun_plan pl, void* stream) {
  if (!pl) return SUN_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const Layout& L = pl->lay;
  const int n = pl->n;
  char* ws = pl->ws;
  DevHeader* hdr = (DevHeader*)(ws + L.hdr);
  // (a1) expand into band storage
  long long band_doubles = (long long)((L.cnt0 - L.kb0) / sizeof(double));
  k_zero<<<296, 256, 0, st>>>((double*)(ws + L.kb0), band_doubles);
  CK(cudaGetLastError());
  OpList ops;
  memset(&ops, 0, sizeof(ops));
  ops.n = n;
  ops.nops = 2 + pl->P;
  ops.op[0] = {pl->H0.row_ptr, pl->H0.col, (const double2*)pl->H0.val};
  ops.op[1] = pl->has_h1 ? OpDesc{pl->H1.row_ptr, pl->H1.col, (const double2*)pl->H1.val} : ops.op[0];
  for (int p = 0; p < pl->P; ++p) ops.op[2 + p] = {pl->L[p].row_ptr, pl->L[p].col, (const double2*)pl->L[p].val};
  long long nthreads = (long long)ops.nops * n;
  k_scatter<<<(unsigned)((nthreads + 255) / 256), 256, 0, st>>>(
      ops, pl->has_h1, (double2*)(ws + L.hb0), pl->wK, (double2*)(ws + L.hb1), pl->wH1, (double2*)(ws + L.lb),
      pl->wL, (const double*)(ws + L.sqrtg));
  CK(cudaGetLastError());
  long long nk = (long long)n * (2 * pl->wK + 1);
  k_band_k<<<(unsigned)((nk + 255) / 256), 256, 0, st>>>(
      n, pl->P, (const double2*)(ws + L.hb0), (double2*)(ws + L.kb0), pl->wK, (const double2*)(ws + L.lb), pl->wL,
      (const double2*)(ws + L.hb1), pl->wH1, pl->has_h1, pl->herm_tol0, pl->herm_tol1, hdr);
  CK(cudaGetLastError());
  // (a3) count pass + (a4) prefix scan, per output matrix
  for (int which = 0; which < 1 + pl->has_h1; ++which) {
    const Prob& pr = pl->pr[which];
    int* cnt = (int*)(ws + (which ? L.cnt1 : L.cnt0));
    long long* ts = (long long*)(ws + (which ? L.ts1 : L.ts0));
    const FarPos* fp = (const FarPos*)(ws + (which ? L.fp1 : L.fp0));
    unsigned grid = (unsigned)(pr.npt + pr.ndt);
    if (pr.mode == 0)
      k_count<0><<<grid, THREAD_TP, 0, st>>>(pr, fp, pl->npos_far[which], cnt, ts);
    else
      k_count<1><<<grid, WARP_THREADS, 0, st>>>(pr, fp, pl->npos_far[which], cnt, ts);
    CK(cudaGetLastError());
    k_scan<<<1, 1024, 0, st>>>(ts, 2 * pr.npt + pr.ndt, &hdr->nnz[which]);
    CK(cudaGetLastError());
  }
  pl->counted = 1;
  pl->count_stream = st;
  pl->nnz[0] = pl->nnz[1] = -1;
  return SUN_OK;
}

int sun_plan_nnz(sun_plan pl, int64_t* nnz_q0, int64_t* nnz_q1) {
  if (!pl) return SUN_ERR_ARG;
  if (!pl->counted) return SUN_ERR_STATE;
  DevHeader* hdr = (DevHeader*)(pl->ws + pl->lay.hdr);
  struct {
    int flags;
    int pad;
    long long nnz[2];
  } h;
  CK(cudaMemcpyAsync(&h, hdr, sizeof(h), cudaMemcpyDeviceToHost, pl->count_stream));
  CK(cudaStreamSynchronize(pl->count_stream));
  if (h.flags & (F_H0_NOT_HERM | F_H1_NOT_HERM)) return SUN_ERR_NOT_HERMITIAN;
  if (h.flags & F_MALFORMED) return SUN_ERR_ARG;
  pl->nnz[0] = h.nnz[0];
  pl->nnz[1] = pl->has_h1 ? h.nnz[1] : 0;
  if (nnz_q0) *nnz_q0 = pl->nnz[0];
  if (nnz_q1) *nnz_q1 = pl->nnz[1];
  return SUN_OK;
}

int sun_unfold(sun_plan pl, sun_dcsr* Q0, sun_dcsr* Q1, double* K, void* stream) {
  if (!pl || !Q0 || !K) return SUN_ERR_ARG;
  if (!pl->counted || pl->nnz[0] < 0) return SUN_ERR_STATE;
  if (pl->has_h1 && !Q1) return SUN_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const Layout& L = pl->lay;
  char* ws = pl->ws;
  DevHeader* hdr = (DevHeader*)(ws + L.hdr);
  const long long m = (long long)pl->n * pl->n - 1;
  for (int which = 0; which < 1 + pl->has_h1; ++which) {
    sun_dcsr* Q = which ? Q1 : Q0;
    if (Q->m != m || !Q->row_ptr || (pl->nnz[which] > 0 && (!Q->col || !Q->val))) return SUN_ERR_ARG;
    if (Q->nnz < pl->nnz[which]) return SUN_ERR_CAPACITY;
  }
  for (int which = 0; which < 1 + pl->has_h1; ++which) {
    sun_dcsr* Q = which ? Q1 : Q0;
    const Prob& pr = pl->pr[which];
    const int* cnt = (const int*)(ws + (which ? L.cnt1 : L.cnt0));
    const long long* ts = (const long long*)(ws + (which ? L.ts1 : L.ts0));
    const FarPos* fp = (const FarPos*)(ws + (which ? L.fp1 : L.fp0));
    unsigned grid = (unsigned)(pr.npt + pr.ndt);
    if (pr.mode == 0) {
      int cap = stage_cap_entries();
      size_t smem = (size_t)cap * (sizeof(double) + sizeof(int));
      CK(cudaFuncSetAttribute(k_fill<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_fill<0><<<grid, THREAD_TP, smem, st>>>(pr, fp, pl->npos_far[which], cnt, ts, &hdr->nnz[which], Q->row_ptr,
                                                Q->col, Q->val, which ? nullptr : K, cap);
    } else {
      k_fill<1><<<grid, WARP_THREADS, 0, st>>>(pr, fp, pl->npos_far[which], cnt, ts, &hdr->nnz[which], Q->row_ptr,
                                                Q->col, Q->val, which ? nullptr : K, 0);
    }
    CK(cudaGetLastError());
  }
  return SUN_OK;
}

int sun_apply(const sun_dcsr* Q0, const sun_dcsr* Q1, double eps, const double* K, const double* v, double* dvdt,
              void* stream) {
  if (!Q0 || !Q0->row_ptr || !v || !dvdt || v == dvdt) return SUN_ERR_ARG;
  if (Q1 && (Q1->m != Q0->m || !Q1->row_ptr)) return SUN_ERR_ARG;
  long long m = Q0->m;
  if (m <= 0) return SUN_ERR_DIM;
  long long threads = m * 8;
  k_apply<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      m, Q0->row_ptr, Q0->col, Q0->val, Q1 ? Q1->row_ptr : nullptr, Q1 ? Q1->col : nullptr,
      Q1 ? Q1->val : nullptr, eps, K, v, dvdt);
  CK(cudaGetLastError());
  return SUN_OK;
}

int sun_plan_info(sun_plan pl, sun_plan_info_t* info) {
  if (!pl || !info) return SUN_ERR_ARG;
  memset(info, 0, sizeof(*info));
  info->n = pl->n;
  info->P = pl->P;
  info->w_h0 = pl->wH0;
  info->w_h1 = pl->wH1;
  info->w_l = pl->wL;
  info->w_k = pl->wK;
  info->tau_q0 = pl->tau0;
  info->tau_q1 = pl->tau1;
  info->mode_q0 = pl->pr[0].mode;
  info->mode_q1 = pl->has_h1 ? pl->pr[1].mode : -1;
  info->pairs_per_tile_q0 = pl->pr[0].tp;
  info->pairs_per_tile_q1 = pl->has_h1 ? pl->pr[1].tp : 0;
  info->tiles_q0 = pl->pr[0].npt + pl->pr[0].ndt;
  info->tiles_q1 = pl->has_h1 ? pl->pr[1].npt + pl->pr[1].ndt : 0;
  info->has_h1 = pl->has_h1;
  info->npos_far_q0 = pl->npos_far[0];
  info->npos_far_q1 = pl->has_h1 ? pl->npos_far[1] : 0;
  return SUN_OK;
}

void sun_plan_destroy(sun_plan pl) { delete pl; }

}  // extern "C"
