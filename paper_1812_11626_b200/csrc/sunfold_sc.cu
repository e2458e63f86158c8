// sunfold_sc.cu — the nonzero SU(N) structure constants f_mns, d_mns from index arithmetic
// (include/sunfold.h, sun_structure_constants).  SURVEY §8 row (a2); PAPER.md Step 2.2
// ("the nonzero elements of f and d are computed analytically ... O(N^3)") and
// Eqs. 2-4.  The unfold kernels never store these tensors (they apply the adjoint
// generator to F_s directly); this entry point makes the structure constants
// themselves available and testable.
//
// Closed-form classes (0-based, a < b < c, l, l' in [1, N-1]; delta_l(x) = (D^l)_xx):
//   triangle (pairs (a,b), (b,c), (a,c)):
//     f(S_ab,S_bc,J_ac) = +1/sqrt2, f(S_ab,J_bc,S_ac) = f(J_ab,S_bc,S_ac) = f(J_ab,J_bc,J_ac) = -1/sqrt2
//     d(S_ab,S_bc,S_ac) = d(S_ab,J_bc,J_ac) = d(J_ab,S_bc,J_ac) = +1/sqrt2, d(J_ab,J_bc,S_ac) = -1/sqrt2
//   pair:  f(S_ab,J_ab,D^l) = delta_l(a) - delta_l(b)   (nonzero iff max(a,1) <= l <= b)
//          d(S_ab,S_ab,D^l) = d(J_ab,J_ab,D^l) = delta_l(a) + delta_l(b)   (l >= max(a,1), not (0,1,1))
//   DDD:   d(D^l,D^l,D^l') = 2/sqrt(l'(l'+1)) (l < l'),  d(D^l,D^l,D^l) = 2(1-l)/sqrt(l(l+1)) (l >= 2)
// f is totally antisymmetric, d totally symmetric: every ordered triple is emitted.
// Work items: one per index pair (a, b) (the triangles with (a, b) as first pair, then the
// pair class) and one per l (the DDD class); item sizes are closed forms, offsets come from a
// one-CTA scan, so the order is fixed.  Shares no code with the oracle (oracle/basis.py).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "sunfold.h"

int sunfold_cuda_fail(cudaError_t e);  // sunfold.cu

namespace {

constexpr double RS2 = 0.70710678118654752440;  // 1/sqrt(2)

struct ScArgs {
  int n, which;  // which: 0 = f, 1 = d
  long long np, items;
  long long* sizes;  // [items + 1] -> exclusive offsets, [items] = total
  int32_t* idx;      // [cap][3] or null
  double* val;       // [cap] or null
  long long cap;
};

__device__ __forceinline__ long long pidx(long long n, long long a, long long b) {  // a < b
  return a * (2 * n - a - 1) / 2 + (b - a - 1);
}
__device__ __forceinline__ void pdecode(long long n, long long p, int& a, int& b) {
  const double t = 2.0 * (double)n - 1.0;
  long long x = (long long)floor((t - sqrt(fmax(t * t - 8.0 * (double)p, 0.0))) * 0.5);
  if (x < 0) x = 0;
  while (x > 0 && x * (2 * n - x - 1) / 2 > p) --x;
  while (x + 1 <= n - 2 && (x + 1) * (2 * n - x - 2) / 2 <= p) ++x;
  a = (int)x;
  b = (int)(x + 1 + (p - x * (2 * n - x - 1) / 2));
}
__device__ __forceinline__ double delta(int l, int x) {  // (D^l)_xx
  const double r = 1.0 / sqrt((double)l * (double)(l + 1));
  return x < l ? r : (x == l ? -(double)l * r : 0.0);
}

__device__ long long item_size(const ScArgs& A, long long i) {
  const long long n = A.n;
  if (i < A.np) {
    int a, b;
    pdecode(n, i, a, b);
    const long long tri = 24 * (n - 1 - b);
    const long long lo = a > 1 ? a : 1;
    if (A.which == 0) return tri + 6 * (b >= lo ? b - lo + 1 : 0);
    return tri + 6 * ((n - 1 - lo + 1) - (a == 0 && b == 1 ? 1 : 0));
  }
  if (A.which == 0) return 0;
  const long long l = i - A.np + 1;
  return 3 * (n - 1 - l) + (l >= 2 ? 1 : 0);
}

__global__ void k_sc_sizes(const ScArgs A) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < A.items) A.sizes[i] = item_size(A, i);
}

// one CTA: exclusive scan of sizes[0, items) in place, total into sizes[items] (fixed order)
__global__ void __launch_bounds__(1024) k_sc_scan(const ScArgs A) {
  __shared__ long long wsum[32];
  __shared__ long long carry_s;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (long long base = 0; base < A.items; base += blockDim.x) {
    const long long i = base + threadIdx.x;
    const long long v = i < A.items ? A.sizes[i] : 0;
    long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      long long t = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      wsum[lane] = t;
    }
    __syncthreads();
    const long long carry = carry_s;
    const long long incl = carry + (wid > 0 ? wsum[wid - 1] : 0) + x;
    if (i < A.items) A.sizes[i] = incl - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry_s = incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) A.sizes[A.items] = carry_s;
}

struct Out {
  const ScArgs* A;
  long long o;
  __device__ void put(int m, int n, int s, double v) {
    if (o < A->cap) {
      A->idx[3 * o] = m;
      A->idx[3 * o + 1] = n;
      A->idx[3 * o + 2] = s;
      A->val[o] = v;
    }
    ++o;
  }
  // all orderings of a representative (i, j, k): f antisymmetric, d symmetric
  __device__ void f6(int i, int j, int k, double v) {
    put(i, j, k, v);
    put(j, k, i, v);
    put(k, i, j, v);
    put(j, i, k, -v);
    put(i, k, j, -v);
    put(k, j, i, -v);
  }
  __device__ void d6(int i, int j, int k, double v) {
    put(i, j, k, v);
    put(j, k, i, v);
    put(k, i, j, v);
    put(j, i, k, v);
    put(i, k, j, v);
    put(k, j, i, v);
  }
  __device__ void d3(int i, int k, double v) {  // d(i, i, k), i != k
    put(i, i, k, v);
    put(i, k, i, v);
    put(k, i, i, v);
  }
};

__global__ void k_sc_emit(const ScArgs A) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= A.items) return;
  Out out{&A, A.sizes[i]};
  const long long n = A.n, np = A.np;
  auto S = [&](int x, int y) { return (int)pidx(n, x, y); };
  auto J = [&](int x, int y) { return (int)(np + pidx(n, x, y)); };
  auto D = [&](int l) { return (int)(2 * np + l - 1); };
  if (i < np) {
    int a, b;
    pdecode(n, i, a, b);
    for (int c = b + 1; c < n; ++c) {  // triangles (a, b, c)
      if (A.which == 0) {
        out.f6(S(a, b), S(b, c), J(a, c), RS2);
        out.f6(S(a, b), J(b, c), S(a, c), -RS2);
        out.f6(J(a, b), S(b, c), S(a, c), -RS2);
        out.f6(J(a, b), J(b, c), J(a, c), -RS2);
      } else {
        out.d6(S(a, b), S(b, c), S(a, c), RS2);
        out.d6(S(a, b), J(b, c), J(a, c), RS2);
        out.d6(J(a, b), S(b, c), J(a, c), RS2);
        out.d6(J(a, b), J(b, c), S(a, c), -RS2);
      }
    }
    const int lo = a > 1 ? a : 1;
    if (A.which == 0) {
      for (int l = lo; l <= b; ++l) out.f6(S(a, b), J(a, b), D(l), delta(l, a) - delta(l, b));
    } else {
      for (int l = lo; l < n; ++l) {
        if (a == 0 && b == 1 && l == 1) continue;  // delta_1(0) + delta_1(1) = 0
        const double v = delta(l, a) + delta(l, b);
        out.d3(S(a, b), D(l), v);
        out.d3(J(a, b), D(l), v);
      }
    }
  } else if (A.which == 1) {
    const int l = (int)(i - np + 1);
    for (int lp = l + 1; lp < n; ++lp) out.d3(D(l), D(lp), 2.0 / sqrt((double)lp * (double)(lp + 1)));
    if (l >= 2) out.put(D(l), D(l), D(l), 2.0 * (1.0 - l) / sqrt((double)l * (double)(l + 1)));
  }
}

}  // namespace

extern "C" {

size_t sun_sc_work_bytes(int32_t n) {
  if (n < 2 || n > 1024) return 0;
  const long long np = (long long)n * (n - 1) / 2;
  return (size_t)(np + n + 1) * sizeof(long long);
}

int sun_structure_constants(int32_t n, int32_t which, int32_t* idx, double* val, int64_t cap, int64_t* nnz,
                            void* work, size_t work_bytes, void* stream) {
  if (n < 2 || n > 1024) return SUN_ERR_DIM;
  if ((which != 0 && which != 1) || !nnz || !work || cap < 0 || (cap > 0 && (!idx || !val))) return SUN_ERR_ARG;
  if (work_bytes < sun_sc_work_bytes(n)) return SUN_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  ScArgs A;
  A.n = n;
  A.which = which;
  A.np = (long long)n * (n - 1) / 2;
  A.items = A.np + (n - 1);
  A.sizes = (long long*)work;
  A.idx = idx;
  A.val = val;
  A.cap = idx && val ? cap : 0;
  const unsigned g = (unsigned)((A.items + 255) / 256);
  k_sc_sizes<<<g, 256, 0, st>>>(A);
  k_sc_scan<<<1, 1024, 0, st>>>(A);
  if (A.cap > 0) k_sc_emit<<<g, 256, 0, st>>>(A);
  cudaError_t e = cudaGetLastError();
  long long total = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&total, A.sizes + A.items, sizeof(total), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return sunfold_cuda_fail(e);
  *nnz = total;
  return A.cap > 0 && total > A.cap ? SUN_ERR_CAPACITY : SUN_OK;
}

}  // extern "C"
