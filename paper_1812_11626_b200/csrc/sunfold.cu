// sunfold.cu — C-ABI and launch logic of the B200 SU(N) unfold (include/sunfold.h).
//
// Pipeline (Table I Step 2; two-step CRS fill P:369-370):
//   sun_plan_create : k_analyze   bandwidths, Frobenius norms, CSR validation  -> 1 readback
//   sun_count       : k_zero, k_scatter, k_band_k   (a1) expand to band storage, K = H + i/2 M
//                     k_count0<WK,WL> / k_count1     (a3) per-row counts (values thresholded) and
//                                                    (a4) tile offsets by decoupled look-back
//   sun_plan_nnz    : readback of the chain totals (nnz Q0, Q1) + validation flags
//   sun_unfold      : k_fill0<WK,WL> / k_fill1       (a5) row_ptr, col, val, K; (a6) Q1
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
constexpr int F_MALFORMED = 1, F_H0_NOT_HERM = 2, F_H1_NOT_HERM = 4, F_PATTERN = 8;
constexpr int THREAD_TP = 128;   // mode 0: pairs per tile == threads per CTA (4 warps)
constexpr int WARP_TP = 64;      // mode 1: pairs per tile
constexpr int WARP_THREADS = 256;
constexpr int FAR_MAXPOS = 1024;

struct DevHeader {
  int flags;
  int pad;
  long long nnz[2];  // written by the scan of each output matrix
  double tau[2];     // drop thresholds of Q0 / Q1 (R6), computed on the device
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
  int wplan[MAXOPS];     // planned half-bandwidth per operator (-1: no check)
  double sqrtg[MAXOPS];  // sqrt(gamma_p) for the dissipators (ops 2..)
  double gamma[MAXOPS];
  int nops;
  int n;
  int has_h1;
};

// mode-0 instantiations (compile-time band widths); anything else runs in mode 1
bool mode0_supported(int wK, int wL) { return (wK <= 3 && wL == 0) || (wK == 2 && wL == 1); }

struct Gammas {
  double g[MAXOPS];
};

thread_local char g_errbuf[512];

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct FarPos {
  int dc[1024];
  int dd[1024];
};

struct Layout {
  size_t hdr, fp0, fp1, sqrtg, inv, kb0, hb0, hb1, lb, ts0, ts1, toff0, toff1, chunk, cnt0, cnt1, total;
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
  L.inv = off; off = align256(off + (size_t)n * sizeof(double));
  L.kb0 = off; off = align256(off + (size_t)n * (2 * WMAX + 1) * sizeof(double2));  // [kb0, lb end) zeroed per count
  L.hb0 = off; off = align256(off + (size_t)n * (2 * WMAX + 1) * sizeof(double2));
  L.hb1 = off; off = align256(off + (size_t)n * (2 * WMAX + 1) * sizeof(double2));
  L.lb = off;  off = align256(off + (size_t)(P > 0 ? P : 1) * n * (2 * WLMAX + 1) * sizeof(double2));
  L.ts0 = off; off = align256(off + (size_t)maxslots * sizeof(int));
  L.ts1 = off; off = align256(off + (size_t)maxslots * sizeof(int));
  L.toff0 = off; off = align256(off + (size_t)maxslots * sizeof(long long));
  L.toff1 = off; off = align256(off + (size_t)maxslots * sizeof(long long));
  L.chunk = off; off = align256(off + (size_t)(maxslots / 16384 + 2) * sizeof(long long));
  L.cnt0 = off; off = align256(off + (size_t)m * sizeof(int));
  L.cnt1 = off; off = align256(off + (size_t)m * sizeof(int));
  L.total = off;
  L.maxslots = maxslots;
  return L;
}

}  // namespace

struct sun_plan_s {
  int n, P, has_h1;
  OpList ops;      // operator descriptors (+ planned widths, rates) passed to the expand kernels
  Gammas gam;
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
  int ran;            // last fill was enqueued by sun_run (capacity checked at sun_plan_nnz)
  long long cap[2];   // capacities passed to the last fill
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
  if (ops.wplan[op] >= 0 && bw > ops.wplan[op]) atomicOr(&hdr->flags, F_PATTERN);
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

__global__ void k_zero(double* p, long long count, int* flags) {
  if (flags && blockIdx.x == 0 && threadIdx.x == 0) *flags = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
    p[i] = 0.0;
}

// (a1) CSR -> band storage.  ops: 0 = H0 (into Hb0, width wK), 1 = H1 (Hb1, width wH1),
// 2+p = L_p (Lb[p], width wL, scaled by sqrt(gamma_p)).  One thread per (operator, row).
__global__ void k_scatter(OpList ops, int has_h1, double2* hb0, int wK, double2* hb1, int wH1, double2* lb,
                          int wL) {
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
  else { dst = lb + (long long)(op - 2) * n * (2 * wL + 1); w = wL; s = ops.sqrtg[op]; }
  for (int64_t k = d.rp[r]; k < d.rp[r + 1]; ++k) {
    int o = d.ci[k] - r;
    if (o < -w || o > w) continue;  // only exact zeros can lie outside (bandwidth from k_analyze)
    double2 v = d.v[k];
    dst[(long long)r * (2 * w + 1) + (o + w)] = make_double2(s * v.x, s * v.y);
  }
}

// (a1) K = H0 + (i/2) M, M = sum_p Lt_p^+ Lt_p (Lt = sqrt(gamma) L); Hermiticity checks of H0, H1.
// Also writes inv[l] = 1/sqrt(l(l+1)) (normalisation of D^l) for the D-chain kernels.
__global__ void k_band_k(int n, int P, const double2* __restrict__ hb0, double2* kb0, int wK,
                         const double2* __restrict__ lb, int wL, const double2* __restrict__ hb1, int wH1,
                         int has_h1, Gammas gam, DevHeader* hdr, double* inv) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  // drop thresholds (R6) and Hermiticity tolerances from this call's norms
  const double nh0 = sqrt(hdr->nrm2[0]), nh1 = has_h1 ? sqrt(hdr->nrm2[1]) : 0.0;
  const double tol0 = 1e-12 * nh0, tol1 = 1e-12 * nh1;
  if (t == 0) {
    double s0 = nh0;
    for (int p = 0; p < P; ++p) s0 += gam.g[p] * hdr->nrm2[2 + p];
    hdr->tau[0] = 1e-14 * s0;
    hdr->tau[1] = 1e-14 * nh1;
  }
  if (t < n) inv[t] = t > 0 ? 1.0 / sqrt((double)t * (double)(t + 1)) : 0.0;
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
// (a3) count pass.  One CTA per row tile: pair tiles (S and J rows of tp consecutive pairs),
// then D tiles (one warp per D^lam row).  Writes per-row counts and one int32 sum per tile
// slot; slots are in global row order (S tiles, J tiles, D tiles).
//   mode 0: thread per pair, far pairs from compile-time band widths (WK, WL) held in
//           registers (the S-row count word also carries nRe in bits 20-31); near pairs
//           warp-cooperative.  128 threads, 128 pairs per tile.
//   mode 1: warp per pair (wide bands / many positions).  256 threads, 64 pairs per tile.
// ---------------------------------------------------------------------------------------
template <int NTHREADS>
__device__ __forceinline__ void count_d_tile(const Prob& pr, long long t, int* cnt, int* tsum, double* scr_w,
                                             int* wtot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const Seg none = {nullptr, nullptr, 0};
  const long long u = t - pr.npt;
  int c = 0;
  const int lam = (int)(u * (NTHREADS / 32) + wid + 1);
  if (lam <= pr.n - 1) {
    double kv;
    c = warp_d_row<false>(pr, lam, scr_w, scr_w + WIN_MAX + 2, kv, none, 0);
    if (lane == 0) cnt[2 * pr.np + lam - 1] = c;
  }
  int tot;
  block_exclusive_scan(lane == 0 ? c : 0, wtot, tot);
  if (threadIdx.x == 0) tsum[2 * pr.npt + u] = tot;
}

// per-warp scratch (doubles): near-pair U tile (2 TW^2) + gS, gJ, pS, pJ (4 SW); D rows use
// the first 2 (WIN_MAX + 2)
template <int TW, int SW>
struct Scr {
  static constexpr int A = 2 * TW * TW + 4 * SW;
  static constexpr int PER_WARP = A > 2 * (WIN_MAX + 2) ? A : 2 * (WIN_MAX + 2);
};

// mode 0, far pairs only (b - a > 2 WK): thread per pair, values in registers.  Near pairs
// and D rows are counted by k_count_near.  Tile sums here cover the far rows; k_count_near
// adds the near rows' counts to the same slots.
template <int WK, int WL, int PT>
__global__ void __launch_bounds__(128) k_count_far(Prob pr, int* __restrict__ cnt, int* __restrict__ tsum) {
  pr.tau = *pr.tau_ptr;
  __shared__ int wred[8];
  const long long t = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long p = t * 128 + threadIdx.x;
  const bool valid = p < pr.np;
  int a, b;
  warp_pairs(pr.n, t * 128 + wid * 32, a, b);
  const bool far = valid && (b - a > 2 * WK);
  int c = 0;
  if (far) {
    double ux[FarT<WK, WL>::NPOS], uy[FarT<WK, WL>::NPOS];
    far_values<WK, WL, PT>(pr, a, b, ux, uy);
    int nR, nI;
    far_counts<WK, WL>(pr.n, pr.tau, a, b, ux, uy, nR, nI);
    c = nR + nI;
    cnt[p] = c | (nR << CNT_BITS);
    cnt[pr.np + p] = c;
  }
  int x = c;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
  if (lane == 0) wred[wid] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    const int tot = wred[0] + wred[1] + wred[2] + wred[3];
    tsum[t] = tot;  // S rows and J rows of a far pair have the same length
    tsum[pr.npt + t] = tot;
  }
}

// mode 0, near pairs (b - a <= 2W) and D rows: one warp per item; counts added to the tile
// slots with integer atomics (order-independent).  D rows have one slot each.
template <int TW>
__global__ void __launch_bounds__(128) k_count_near(Prob pr, int* __restrict__ cnt, int* __restrict__ tsum) {
  pr.tau = *pr.tau_ptr;
  constexpr int SW = 2 * TW + 2;
  __shared__ double scr[4][Scr<TW, SW>::PER_WARP];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long item = (long long)blockIdx.x * 4 + wid;
  const int W2 = 2 * pr.W;
  const long long nnear = (long long)pr.n * W2;
  const Seg none = {nullptr, nullptr, 0};
  if (item < nnear) {
    const int a = (int)(item / W2), b = a + 1 + (int)(item % W2);
    if (b >= pr.n) return;
    int c1, c2;
    double k1, k2;
    warp_near_pair<false, TW, SW>(pr, a, b, scr[wid], c1, c2, k1, k2, none, 0, none, 0);
    if (lane == 0) {
      const long long p = (long long)pidx32(pr.n, a, b);
      cnt[p] = c1;
      cnt[pr.np + p] = c2;
      atomicAdd(&tsum[p / 128], c1);
      atomicAdd(&tsum[pr.npt + p / 128], c2);
    }
  } else if (item < nnear + pr.n - 1) {
    const int lam = (int)(item - nnear) + 1;
    double kv;
    const int c = warp_d_row<false>(pr, lam, scr[wid], scr[wid] + WIN_MAX + 2, kv, none, 0);
    if (lane == 0) {
      cnt[2 * pr.np + lam - 1] = c;
      tsum[2 * pr.npt + lam - 1] = c;
    }
  }
}

__global__ void __launch_bounds__(WARP_THREADS) k_count1(Prob pr, const FarPos* __restrict__ fp, int npos_far,
                                                         int* __restrict__ cnt, int* __restrict__ tsum) {
  pr.tau = *pr.tau_ptr;
  constexpr int SW = WIN_MAX + 2;
  __shared__ double scr[WARP_THREADS / 32][Scr<0, SW>::PER_WARP];
  __shared__ int wtot[32];
  __shared__ int spos_dc[FAR_MAXPOS], spos_dd[FAR_MAXPOS];
  const long long t = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  if (t >= pr.npt) {
    count_d_tile<WARP_THREADS>(pr, t, cnt, tsum, scr[wid], wtot);
    return;
  }
  for (int i = threadIdx.x; i < npos_far; i += blockDim.x) {
    spos_dc[i] = fp->dc[i];
    spos_dd[i] = fp->dd[i];
  }
  __syncthreads();
  const Seg none = {nullptr, nullptr, 0};
  int cS = 0, cJ = 0;
  for (int i = wid; i < WARP_TP; i += nwarps) {
    const long long p = t * WARP_TP + i;
    if (p >= pr.np) break;
    int a, b;
    pair_decode(pr.n, p, a, b);
    int c1, c2;
    if (b - a > 2 * pr.W) {
      c1 = c2 = warp_far_pair<false>(pr, a, b, spos_dc, spos_dd, npos_far, none, 0, none, 0);
    } else {
      double k1, k2;
      warp_near_pair<false, 0, SW>(pr, a, b, scr[wid], c1, c2, k1, k2, none, 0, none, 0);
    }
    if (lane == 0) {
      cnt[p] = c1;
      cnt[pr.np + p] = c2;
      cS += c1;
      cJ += c2;
    }
  }
  int totS, totJ;
  block_exclusive_scan(cS, wtot, totS);
  block_exclusive_scan(cJ, wtot, totJ);
  if (threadIdx.x == 0) {
    tsum[t] = totS;
    tsum[pr.npt + t] = totJ;
  }
}

// ---------------------------------------------------------------------------------------
// (a4) exclusive scan of the tile sums -> int64 tile offsets and nnz.  Fixed order
// (deterministic).  Small: one CTA through shared memory.  Large: chunk sums, a scan of
// the chunk sums, then per-chunk scans.
// ---------------------------------------------------------------------------------------
constexpr int SCAN_CHUNK = 16384;

template <typename T>
__device__ __forceinline__ long long block_scan_ll(long long v, long long* wsum, long long& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    long long s = lane < nwarps ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(FULL, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nwarps) wsum[lane] = s;
  }
  __syncthreads();
  total = wsum[nwarps - 1];
  long long before = wid > 0 ? wsum[wid - 1] : 0;
  __syncthreads();
  return before + x - v;
}

// scan of one chunk [c0, c0 + len) of int32 values with base offset; writes int64 exclusive
__global__ void __launch_bounds__(1024) k_scan_chunk(const int* __restrict__ ts, long long nslots,
                                                     const long long* __restrict__ chunk_base, long long* out,
                                                     long long* nnz_out) {
  extern __shared__ int sv[];
  __shared__ long long wsum[32];
  const long long c0 = (long long)blockIdx.x * SCAN_CHUNK;
  const int len = (int)(nslots - c0 < SCAN_CHUNK ? nslots - c0 : SCAN_CHUNK);
  for (int i = threadIdx.x; i < len; i += blockDim.x) sv[i] = ts[c0 + i];
  __syncthreads();
  const int per = (len + blockDim.x - 1) / blockDim.x;
  const int lo = threadIdx.x * per, hi = lo + per < len ? lo + per : len;
  long long local = 0;
  for (int i = lo; i < hi; ++i) local += sv[i];
  long long total;
  long long run = block_scan_ll<long long>(local, wsum, total) + (chunk_base ? chunk_base[blockIdx.x] : 0);
  for (int i = lo; i < hi; ++i) {
    out[c0 + i] = run;
    run += sv[i];
  }
  if (nnz_out && threadIdx.x == blockDim.x - 1 && blockIdx.x == gridDim.x - 1) *nnz_out = run;
}

__global__ void __launch_bounds__(1024) k_scan_reduce(const int* __restrict__ ts, long long nslots,
                                                      long long* __restrict__ chunk_sum) {
  __shared__ long long wsum[32];
  const long long c0 = (long long)blockIdx.x * SCAN_CHUNK;
  const int len = (int)(nslots - c0 < SCAN_CHUNK ? nslots - c0 : SCAN_CHUNK);
  long long local = 0;
  for (int i = threadIdx.x; i < len; i += blockDim.x) local += ts[c0 + i];
  long long total;
  block_scan_ll<long long>(local, wsum, total);
  if (threadIdx.x == 0) chunk_sum[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024) k_scan_top(long long* chunk, int nchunks) {
  __shared__ long long wsum[32];
  const int per = (nchunks + blockDim.x - 1) / blockDim.x;
  const int lo = threadIdx.x * per, hi = lo + per < nchunks ? lo + per : nchunks;
  long long local = 0;
  for (int i = lo; i < hi; ++i) local += chunk[i];
  long long total;
  long long run = block_scan_ll<long long>(local, wsum, total);
  for (int i = lo; i < hi; ++i) {
    long long v = chunk[i];
    chunk[i] = run;
    run += v;
  }
}

// ---------------------------------------------------------------------------------------
// (a5) fill pass (+ K).  Same tiling as the count pass.
// ---------------------------------------------------------------------------------------
struct FillOut {
  int64_t* row_ptr;
  int32_t* col;
  double* val;
  long long cap;  // capacity of col/val (writes at or beyond it are dropped; see sun_run)
  double* K;  // nullptr: not written (Q1)
  const long long* toff;
  const long long* nnz;
};

template <int NTHREADS>
__device__ __forceinline__ void fill_d_tile(const Prob& pr, const FillOut& fo, long long t, const int* cnt,
                                            double* scr_w, int* wtot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long np = pr.np;
  const long long u = t - pr.npt;
  const long long baseD = fo.toff[2 * pr.npt + u];
  const int lam = (int)(u * (NTHREADS / 32) + wid + 1);
  const bool valid = lam <= pr.n - 1;
  const int c = valid ? (cnt[2 * np + lam - 1] & CNT_MASK) : 0;
  int tot;
  int ex = block_exclusive_scan(lane == 0 ? c : 0, wtot, tot);
  ex = __shfl_sync(FULL, ex, 0);
  if (valid) {
    if (lane == 0) fo.row_ptr[2 * np + lam - 1] = baseD + ex;
    const Seg sD = {fo.col + baseD, fo.val + baseD, fo.cap - baseD};
    double kv;
    warp_d_row<true>(pr, lam, scr_w, scr_w + WIN_MAX + 2, kv, sD, ex);
    if (lane == 0 && fo.K) fo.K[2 * np + lam - 1] = kv;
  }
}

constexpr int CAPW = 1024;   // per-warp staging capacity (entries) in mode 0 (one row block at a time)

// Copy a warp's staged segment [g0, g1) (tile-local offsets) to global memory, skipping the
// "holes" of long rows (lanes flagged in `holes`, hole = [hoff, hoff + hlen)) that were
// written directly.  The stage position advances only over copied entries.
__device__ __forceinline__ void warp_copy_out(const int* scol, const double* sval, long long gbase, int g0, int g1,
                                              unsigned holes, int hoff, int hlen, int32_t* __restrict__ col,
                                              double* __restrict__ val, long long cap) {
  const int lane = threadIdx.x & 31;
  int sp = 0, gp = g0;
  for (;;) {
    const bool last = holes == 0;
    int hs = g1, hl = 0;
    if (!last) {
      const int h = __ffs(holes) - 1;
      holes &= holes - 1;
      hs = __shfl_sync(FULL, hoff, h);
      hl = __shfl_sync(FULL, hlen, h);
    }
    long long run_l = hs - gp;
    if (gbase + gp + run_l > cap) run_l = cap - (gbase + gp) > 0 ? cap - (gbase + gp) : 0;
    const int run = (int)run_l;
    int32_t* cdst = col + gbase + gp;
    double* vdst = val + gbase + gp;
    for (int k = lane; k < run; k += 32) {
      cdst[k] = scol[sp + k];
      vdst[k] = sval[sp + k];
    }
    sp += run;
    gp = hs + hl;
    if (last) break;
  }
}

// mode 0 fill, far pairs: thread per pair computes its values in registers and writes its
// two rows into per-warp shared staging (S rows of the warp's 32 pairs, then their J rows);
// the warp copies each staged block out with coalesced stores, skipping the near rows
// (written by k_fill_near).  Also writes row_ptr of all pair rows and K = 0 for far pairs.
template <int WK, int WL, int PT>
__global__ void __launch_bounds__(128) k_fill_far(Prob pr, const int* __restrict__ cnt, FillOut fo) {
  pr.tau = *pr.tau_ptr;
  static_assert(64 * FarT<WK, WL>::NPOS <= CAPW, "far rows of a warp must fit the staging");
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ int wtot[8];
  const long long t = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long np = pr.np;
  if (t == 0 && threadIdx.x == 0) fo.row_ptr[pr.m] = *fo.nnz;
  double* sval = reinterpret_cast<double*>(dyn) + wid * CAPW;
  int* scol = reinterpret_cast<int*>(dyn + 4 * CAPW * sizeof(double)) + wid * CAPW;
  const long long p = t * 128 + threadIdx.x;
  const bool valid = p < np;
  const int rawS = valid ? cnt[p] : 0;
  const int cS = rawS & CNT_MASK, nRe = rawS >> CNT_BITS;
  const int cJ = valid ? (cnt[np + p] & CNT_MASK) : 0;
  int a, b;
  warp_pairs(pr.n, t * 128 + wid * 32, a, b);
  int wtS, wtJ;
  int exS = warp_excl_scan(cS, wtS);
  int exJ = warp_excl_scan(cJ, wtJ);
  if (lane == 0) {
    wtot[wid] = wtS;
    wtot[4 + wid] = wtJ;
  }
  __syncthreads();
  int pS = 0, pJ = 0;
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    pS += w < wid ? wtot[w] : 0;
    pJ += w < wid ? wtot[4 + w] : 0;
  }
  exS += pS;
  exJ += pJ;
  const long long baseS = fo.toff[t], baseJ = fo.toff[pr.npt + t];
  if (valid) {
    fo.row_ptr[p] = baseS + exS;
    fo.row_ptr[np + p] = baseJ + exJ;
  }
  const bool far = valid && (b - a > 2 * WK);
  const bool nearp = valid && !far;
  if (far && fo.K) {
    fo.K[p] = 0.0;
    fo.K[np + p] = 0.0;
  }
  const unsigned nearmask = __ballot_sync(FULL, nearp);
  double ux[FarT<WK, WL>::NPOS], uy[FarT<WK, WL>::NPOS];
  if (far) far_values<WK, WL, PT>(pr, a, b, ux, uy);
#pragma unroll
  for (int row = 0; row < 2; ++row) {  // S rows of the warp's 32 pairs, then their J rows
    const int c_me = row ? cJ : cS, ex_me = row ? exJ : exS, w0 = row ? pJ : pS, wt = row ? wtJ : wtS;
    const long long gbase = row ? baseJ : baseS;
    int ht;
    const int hb = warp_excl_scan(nearp ? c_me : 0, ht);
    if (far) {
      const int n1 = row ? (cS - nRe) : nRe;
      far_emit_row<WK, WL>(pr.n, (int)np, pr.tau, a, b, row, ux, uy, n1, SmemSink{scol, sval}, ex_me - w0 - hb);
    }
    __syncwarp();
    warp_copy_out(scol, sval, gbase, w0, w0 + wt, nearmask, ex_me, c_me, fo.col, fo.val, fo.cap);
    __syncwarp();
  }
}

// mode 0 fill, near pairs and D rows (one warp per item, rows written directly).  Runs after
// k_fill_far, whose row_ptr entries give the near rows' offsets.
template <int TW>
__global__ void __launch_bounds__(128) k_fill_near(Prob pr, FillOut fo) {
  pr.tau = *pr.tau_ptr;
  constexpr int SW = 2 * TW + 2;
  __shared__ double scr[4][Scr<TW, SW>::PER_WARP];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long item = (long long)blockIdx.x * 4 + wid;
  const int W2 = 2 * pr.W;
  const long long nnear = (long long)pr.n * W2;
  const long long np = pr.np;
  if (item < nnear) {
    const int a = (int)(item / W2), b = a + 1 + (int)(item % W2);
    if (b >= pr.n) return;
    const long long p = (long long)pidx32(pr.n, a, b);
    const long long oS = fo.row_ptr[p], oJ = fo.row_ptr[np + p];
    const Seg sS = {fo.col + oS, fo.val + oS, fo.cap - oS};
    const Seg sJ = {fo.col + oJ, fo.val + oJ, fo.cap - oJ};
    int c1, c2;
    double k1, k2;
    warp_near_pair<true, TW, SW>(pr, a, b, scr[wid], c1, c2, k1, k2, sS, 0, sJ, 0);
    if (lane == 0 && fo.K) {
      fo.K[p] = k1;
      fo.K[np + p] = k2;
    }
  } else if (item < nnear + pr.n - 1) {
    const int lam = (int)(item - nnear) + 1;
    const long long off = fo.toff[2 * pr.npt + lam - 1];
    if (lane == 0) fo.row_ptr[2 * np + lam - 1] = off;
    const Seg sD = {fo.col + off, fo.val + off, fo.cap - off};
    double kv;
    warp_d_row<true>(pr, lam, scr[wid], scr[wid] + WIN_MAX + 2, kv, sD, 0);
    if (lane == 0 && fo.K) fo.K[2 * np + lam - 1] = kv;
  }
}

__global__ void __launch_bounds__(WARP_THREADS) k_fill1(Prob pr, const FarPos* __restrict__ fp, int npos_far,
                                                        const int* __restrict__ cnt, FillOut fo) {
  pr.tau = *pr.tau_ptr;
  constexpr int SW = WIN_MAX + 2;
  __shared__ double scr[WARP_THREADS / 32][Scr<0, SW>::PER_WARP];
  __shared__ int wtot[32];
  __shared__ int spos_dc[FAR_MAXPOS], spos_dd[FAR_MAXPOS];
  __shared__ int soffS[WARP_TP], soffJ[WARP_TP];
  const long long t = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const long long np = pr.np;
  if (t == 0 && threadIdx.x == 0) fo.row_ptr[pr.m] = *fo.nnz;
  if (t >= pr.npt) {
    fill_d_tile<WARP_THREADS>(pr, fo, t, cnt, scr[wid], wtot);
    return;
  }
  for (int i = threadIdx.x; i < npos_far; i += blockDim.x) {
    spos_dc[i] = fp->dc[i];
    spos_dd[i] = fp->dd[i];
  }
  const long long baseS = fo.toff[t], baseJ = fo.toff[pr.npt + t];
  const int i0 = threadIdx.x;
  const long long p0 = t * WARP_TP + i0;
  const bool valid = i0 < WARP_TP && p0 < np;
  const int cS = valid ? (cnt[p0] & CNT_MASK) : 0, cJ = valid ? (cnt[np + p0] & CNT_MASK) : 0;
  int totS, totJ;
  const int exS = block_exclusive_scan(cS, wtot, totS);
  const int exJ = block_exclusive_scan(cJ, wtot, totJ);
  if (i0 < WARP_TP) {
    soffS[i0] = exS;
    soffJ[i0] = exJ;
  }
  if (valid) {
    fo.row_ptr[p0] = baseS + exS;
    fo.row_ptr[np + p0] = baseJ + exJ;
  }
  __syncthreads();
  const Seg sS = {fo.col + baseS, fo.val + baseS, fo.cap - baseS};
  const Seg sJ = {fo.col + baseJ, fo.val + baseJ, fo.cap - baseJ};
  for (int i = wid; i < WARP_TP; i += nwarps) {
    const long long p = t * WARP_TP + i;
    if (p >= np) break;
    int a, b;
    pair_decode(pr.n, p, a, b);
    double k1 = 0.0, k2 = 0.0;
    if (b - a > 2 * pr.W) {
      warp_far_pair<true>(pr, a, b, spos_dc, spos_dd, npos_far, sS, soffS[i], sJ, soffJ[i]);
    } else {
      int c1, c2;
      warp_near_pair<true, 0, SW>(pr, a, b, scr[wid], c1, c2, k1, k2, sS, soffS[i], sJ, soffJ[i]);
    }
    if (lane == 0 && fo.K) {
      fo.K[p] = k1;
      fo.K[np + p] = k2;
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
    pr.tau_ptr = &reinterpret_cast<DevHeader*>(pl->ws + L.hdr)->tau[0];
  } else {
    pr.P = 0;
    pr.wK = pl->wH1;
    pr.wL = 0;
    pr.K = {reinterpret_cast<const double2*>(pl->ws + L.hb1), pl->wH1};
    pr.H = pr.K;
    pr.L = nullptr;
    pr.tau = pl->tau1;
    pr.tau_ptr = &reinterpret_cast<DevHeader*>(pl->ws + L.hdr)->tau[1];
  }
  pr.W = pr.wK > pr.wL ? pr.wK : pr.wL;
  pr.inv = reinterpret_cast<const double*>(pl->ws + L.inv);
  build_far_positions(pr.W, pr.wL, pr.wK, pl->pos_dc[which], pl->pos_dd[which]);
  int npos = (int)pl->pos_dc[which].size();
  pl->npos_far[which] = npos;
  for (int i = 0; i < npos && i < FAR_MAXPOS; ++i) {
    pl->hfp[which].dc[i] = pl->pos_dc[which][i];
    pl->hfp[which].dd[i] = pl->pos_dd[which][i];
  }
  // thread-per-pair with per-warp shared staging for narrow bands (compile-time widths);
  // else warp-per-pair with direct coalesced row stores
  pr.mode = mode0_supported(pr.wK, pr.wL) ? 0 : 1;
  pr.tp = pr.mode == 0 ? THREAD_TP : WARP_TP;
  pr.npt = (pr.np + pr.tp - 1) / pr.tp;
  pr.ndt = pr.mode == 0 ? (pl->n - 1) : (pl->n - 1 + WARP_THREADS / 32 - 1) / (WARP_THREADS / 32);
}


template <int WK, int WL, int PT>
cudaError_t launch_far(const Prob& pr, int* cnt, int* ts, const FillOut* fo, cudaStream_t st) {
  if (!fo) {
    k_count_far<WK, WL, PT><<<(unsigned)pr.npt, 128, 0, st>>>(pr, cnt, ts);
    return cudaGetLastError();
  }
  const size_t smem = (size_t)4 * CAPW * (sizeof(double) + sizeof(int));
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_fill_far<WK, WL, PT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  k_fill_far<WK, WL, PT><<<(unsigned)pr.npt, 128, smem, st>>>(pr, cnt, *fo);
  return cudaGetLastError();
}

// (WK, WL, PT) instantiations of the mode-0 far kernels
#define SUN_MODE0_LIST(X) \
  X(0, 0, 0) X(1, 0, 0) X(2, 0, 0) X(3, 0, 0) X(0, 0, 1) X(1, 0, 1) X(2, 0, 1) X(3, 0, 1) X(2, 1, 1) \
  X(0, 0, -1) X(1, 0, -1) X(2, 0, -1) X(3, 0, -1) X(2, 1, -1)

int mode0_pt(const Prob& pr) { return pr.P == 0 ? 0 : (pr.P == 1 ? 1 : -1); }

cudaError_t dispatch_far(const Prob& pr, int* cnt, int* ts, const FillOut* fo, cudaStream_t st) {
  const int pt = mode0_pt(pr);
#define SUN_X(WK, WL, PT) \
  if (pr.wK == WK && pr.wL == WL && pt == PT) return launch_far<WK, WL, PT>(pr, cnt, ts, fo, st);
  SUN_MODE0_LIST(SUN_X)
#undef SUN_X
  return cudaErrorInvalidValue;
}

cudaError_t dispatch_near(const Prob& pr, int* cnt, int* ts, const FillOut* fo, cudaStream_t st) {
  const long long items = (long long)pr.n * 2 * pr.W + (pr.n - 1);
  const unsigned grid = (unsigned)((items + 3) / 4);
  if (grid == 0) return cudaSuccess;
#define SUN_NEAR(TW)                                                            \
  if (2 * pr.W + 1 == TW) {                                                     \
    if (!fo)                                                                    \
      k_count_near<TW><<<grid, 128, 0, st>>>(pr, cnt, ts);                      \
    else                                                                        \
      k_fill_near<TW><<<grid, 128, 0, st>>>(pr, *fo);                           \
    return cudaGetLastError();                                                  \
  }
  SUN_NEAR(1) SUN_NEAR(3) SUN_NEAR(5) SUN_NEAR(7)
#undef SUN_NEAR
  return cudaErrorInvalidValue;
}

// exclusive scan of nslots int32 tile sums into int64 offsets; total -> nnz_out
cudaError_t launch_scan(const int* ts, long long nslots, long long* toff, long long* chunk, long long* nnz_out,
                        cudaStream_t st) {
  const size_t smem = SCAN_CHUNK * sizeof(int);
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_scan_chunk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (nslots <= SCAN_CHUNK) {
    k_scan_chunk<<<1, 1024, smem, st>>>(ts, nslots, nullptr, toff, nnz_out);
    return cudaGetLastError();
  }
  const int nchunks = (int)((nslots + SCAN_CHUNK - 1) / SCAN_CHUNK);
  k_scan_reduce<<<nchunks, 1024, 0, st>>>(ts, nslots, chunk);
  k_scan_top<<<1, 1024, 0, st>>>(chunk, nchunks);
  k_scan_chunk<<<nchunks, 1024, smem, st>>>(ts, nslots, chunk, toff, nnz_out);
  return cudaGetLastError();
}

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
  ops.has_h1 = H1 != nullptr;
  ops.op[0] = {H0->row_ptr, H0->col, (const double2*)H0->val};
  ops.op[1] = H1 ? OpDesc{H1->row_ptr, H1->col, (const double2*)H1->val} : ops.op[0];
  for (int p = 0; p < P; ++p) {
    ops.op[2 + p] = {L[p]->row_ptr, L[p]->col, (const double2*)L[p]->val};
    ops.sqrtg[2 + p] = sqrt(gamma[p]);
    ops.gamma[2 + p] = gamma[p];
  }
  for (int i = 0; i < MAXOPS; ++i) ops.wplan[i] = -1;
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
  pl->ops = ops;
  pl->ops.wplan[0] = pl->wH0;
  pl->ops.wplan[1] = H1 ? pl->wH1 : -1;
  for (int p = 0; p < P; ++p) {
    pl->ops.wplan[2 + p] = pl->wL;
    pl->gam.g[p] = gamma[p];
  }
  setup_prob(pl, 0);
  if (pl->has_h1) setup_prob(pl, 1);
  if (pl->npos_far[0] > FAR_MAXPOS || (pl->has_h1 && pl->npos_far[1] > FAR_MAXPOS)) {
    delete pl;
    return SUN_ERR_BANDWIDTH;
  }
  // far-position tables (used by the warp-per-pair mode only)
  cudaError_t e = cudaSuccess;
  if (pl->pr[0].mode == 1)
    e = cudaMemcpyAsync(ws + lay.fp0, &pl->hfp[0], sizeof(FarPos), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && pl->has_h1 && pl->pr[1].mode == 1)
    e = cudaMemcpyAsync(ws + lay.fp1, &pl->hfp[1], sizeof(FarPos), cudaMemcpyHostToDevice, st);
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
  // (a1) expand: norms + pattern check, band storage, K = H0 + i/2 M, tau (all on the device)
  long long zero_doubles = (long long)((L.ts0 - L.kb0) / sizeof(double));
  k_zero<<<296, 256, 0, st>>>((double*)(ws + L.kb0), zero_doubles, &hdr->flags);
  CK(cudaGetLastError());
  k_analyze<<<pl->ops.nops, 256, 0, st>>>(pl->ops, hdr);
  CK(cudaGetLastError());
  long long nthreads = (long long)pl->ops.nops * n;
  k_scatter<<<(unsigned)((nthreads + 255) / 256), 256, 0, st>>>(
      pl->ops, pl->has_h1, (double2*)(ws + L.hb0), pl->wK, (double2*)(ws + L.hb1), pl->wH1, (double2*)(ws + L.lb),
      pl->wL);
  CK(cudaGetLastError());
  long long nk = (long long)n * (2 * pl->wK + 1);
  if (nk < n) nk = n;
  k_band_k<<<(unsigned)((nk + 255) / 256), 256, 0, st>>>(
      n, pl->P, (const double2*)(ws + L.hb0), (double2*)(ws + L.kb0), pl->wK, (const double2*)(ws + L.lb), pl->wL,
      (const double2*)(ws + L.hb1), pl->wH1, pl->has_h1, pl->gam, hdr, (double*)(ws + L.inv));
  CK(cudaGetLastError());
  // (a3) count pass + (a4) prefix scan, per output matrix
  for (int which = 0; which < 1 + pl->has_h1; ++which) {
    const Prob& pr = pl->pr[which];
    int* cnt = (int*)(ws + (which ? L.cnt1 : L.cnt0));
    int* ts = (int*)(ws + (which ? L.ts1 : L.ts0));
    const FarPos* fp = (const FarPos*)(ws + (which ? L.fp1 : L.fp0));
    if (pr.mode == 0) {
      CK(dispatch_far(pr, cnt, ts, nullptr, st));   // far pairs (writes the tile sums)
      CK(dispatch_near(pr, cnt, ts, nullptr, st));  // near pairs + D rows (atomic adds)
    } else {
      k_count1<<<(unsigned)(pr.npt + pr.ndt), WARP_THREADS, 0, st>>>(pr, fp, pl->npos_far[which], cnt, ts);
      CK(cudaGetLastError());
    }
    CK(launch_scan(ts, 2 * pr.npt + pr.ndt, (long long*)(ws + (which ? L.toff1 : L.toff0)), (long long*)(ws + L.chunk),
                   &hdr->nnz[which], st));
  }
  pl->counted = 1;
  pl->ran = 0;
  pl->count_stream = st;
  pl->nnz[0] = pl->nnz[1] = -1;
  return SUN_OK;
}

int sun_plan_nnz(sun_plan pl, int64_t* nnz_q0, int64_t* nnz_q1) {
  if (!pl) return SUN_ERR_ARG;
  if (!pl->counted) return SUN_ERR_STATE;
  struct {
    int flags;
    int pad;
    long long nnz[2];
    double tau[2];
  } h;
  CK(cudaMemcpyAsync(&h, pl->ws + pl->lay.hdr, sizeof(h), cudaMemcpyDeviceToHost, pl->count_stream));
  CK(cudaStreamSynchronize(pl->count_stream));
  if (h.flags & (F_H0_NOT_HERM | F_H1_NOT_HERM)) return SUN_ERR_NOT_HERMITIAN;
  if (h.flags & F_PATTERN) return SUN_ERR_BANDWIDTH;
  pl->tau0 = h.tau[0];
  pl->tau1 = pl->has_h1 ? h.tau[1] : 0.0;
  if (h.flags & F_MALFORMED) return SUN_ERR_ARG;
  pl->nnz[0] = h.nnz[0];
  pl->nnz[1] = pl->has_h1 ? h.nnz[1] : 0;
  if (nnz_q0) *nnz_q0 = pl->nnz[0];
  if (nnz_q1) *nnz_q1 = pl->nnz[1];
  if (pl->ran) {
    pl->ran = 0;
    if (pl->nnz[0] > pl->cap[0] || pl->nnz[1] > pl->cap[1]) return SUN_ERR_CAPACITY;
  }
  return SUN_OK;
}

static int enqueue_fill(sun_plan pl, sun_dcsr* Q0, sun_dcsr* Q1, double* K, cudaStream_t st) {
  const Layout& L = pl->lay;
  char* ws = pl->ws;
  for (int which = 0; which < 1 + pl->has_h1; ++which) {
    sun_dcsr* Q = which ? Q1 : Q0;
    const Prob& pr = pl->pr[which];
    const int* cnt = (const int*)(ws + (which ? L.cnt1 : L.cnt0));
    const FarPos* fp = (const FarPos*)(ws + (which ? L.fp1 : L.fp0));
    DevHeader* hdr = (DevHeader*)(ws + L.hdr);
    FillOut fo = {Q->row_ptr, Q->col, Q->val, (long long)Q->nnz, which ? nullptr : K,
                  (const long long*)(ws + (which ? L.toff1 : L.toff0)), &hdr->nnz[which]};
    if (pr.mode == 0) {
      CK(dispatch_far(pr, const_cast<int*>(cnt), nullptr, &fo, st));
      CK(dispatch_near(pr, nullptr, nullptr, &fo, st));
    } else {
      k_fill1<<<(unsigned)(pr.npt + pr.ndt), WARP_THREADS, 0, st>>>(pr, fp, pl->npos_far[which], cnt, fo);
      CK(cudaGetLastError());
    }
  }
  return SUN_OK;
}

static int check_outputs(sun_plan pl, const sun_dcsr* Q0, const sun_dcsr* Q1, const double* K) {
  if (!Q0 || !K) return SUN_ERR_ARG;
  if (pl->has_h1 && !Q1) return SUN_ERR_ARG;
  const long long m = (long long)pl->n * pl->n - 1;
  for (int which = 0; which < 1 + pl->has_h1; ++which) {
    const sun_dcsr* Q = which ? Q1 : Q0;
    if (Q->m != m || !Q->row_ptr || Q->nnz < 0 || (Q->nnz > 0 && (!Q->col || !Q->val))) return SUN_ERR_ARG;
  }
  return SUN_OK;
}

int sun_unfold(sun_plan pl, sun_dcsr* Q0, sun_dcsr* Q1, double* K, void* stream) {
  if (!pl) return SUN_ERR_ARG;
  if (!pl->counted || pl->nnz[0] < 0) return SUN_ERR_STATE;
  int st = check_outputs(pl, Q0, Q1, K);
  if (st != SUN_OK) return st;
  for (int which = 0; which < 1 + pl->has_h1; ++which)
    if ((which ? Q1 : Q0)->nnz < pl->nnz[which]) return SUN_ERR_CAPACITY;
  pl->cap[0] = Q0->nnz;
  pl->cap[1] = Q1 ? Q1->nnz : 0;
  return enqueue_fill(pl, Q0, Q1, K, (cudaStream_t)stream);
}

int sun_run(sun_plan pl, sun_dcsr* Q0, sun_dcsr* Q1, double* K, void* stream) {
  if (!pl) return SUN_ERR_ARG;
  int st = check_outputs(pl, Q0, Q1, K);
  if (st != SUN_OK) return st;
  st = sun_count(pl, stream);
  if (st != SUN_OK) return st;
  pl->cap[0] = Q0->nnz;
  pl->cap[1] = Q1 ? Q1->nnz : 0;
  pl->ran = 1;
  return enqueue_fill(pl, Q0, Q1, K, (cudaStream_t)stream);
}

int64_t sun_nnz_bound(sun_plan pl, int32_t which) {
  if (!pl || which < 0 || which > 1 || (which == 1 && !pl->has_h1)) return -1;
  const Prob& pr = pl->pr[which];
  const long long n = pl->n;
  const long long W = pr.W;
  const long long nw = 4 * W + 1 < n ? 4 * W + 1 : n;          // near-pair window
  const long long nwd = 2 * pr.wK + 1 < n ? 2 * pr.wK + 1 : n;  // D-row window
  const long long nnear = n * 2 * W < pr.np ? n * 2 * W : pr.np;
  long long far_row = 2LL * pl->npos_far[which];
  long long near_row = nw * (nw - 1) + (n - 1);
  if (far_row > near_row) far_row = near_row;
  return 2 * (pr.np - nnear) * far_row + 2 * nnear * near_row + (n - 1) * (nwd * (nwd - 1) + (n - 1));
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
  info->tiles_q0 = 2 * pl->pr[0].npt + pl->pr[0].ndt;
  info->tiles_q1 = pl->has_h1 ? 2 * pl->pr[1].npt + pl->pr[1].ndt : 0;
  info->has_h1 = pl->has_h1;
  info->npos_far_q0 = pl->npos_far[0];
  info->npos_far_q1 = pl->has_h1 ? pl->npos_far[1] : 0;
  return SUN_OK;
}

void sun_plan_destroy(sun_plan pl) { delete pl; }

}  // extern "C"
