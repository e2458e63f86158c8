// sunfold.cu — C-ABI and launch logic of the B200 SU(N) unfold (include/sunfold.h).
//
// Pipeline (Table I Step 2; two-step CRS fill P:369-370), launches per sun_run:
//   sun_plan_create : k_analyze         bandwidths, Frobenius norms, CSR validation -> 1 readback
//   sun_count       : k_expand          (a1) CSR -> band storage, K = H0 + i/2 sum gamma L^+L, inv[l],
//                                        norms / flags / Hermiticity -> tau (last block), zeroing
//                     k_count0 / k_count1 (a3) per-row counts (values thresholded), tile sums;
//                                        one launch per output matrix (near items + far tiles),
//                                        Q1's on an auxiliary stream
//                     k_scan_chain      (a4) chained (decoupled look-back) scan of the tile sums of
//                                        both matrices -> int64 tile offsets and nnz
//   sun_plan_nnz    : readback of nnz + validation flags (16 B + header)
//   sun_unfold      : k_fill_far0 + k_fill_near0 / k_fill1  (a5) row_ptr, col, val, K; (a6) Q1
//                                        Q0 far tiles on the caller's stream, Q0 near items and Q1
//                                        on two auxiliary streams (fork/join with events)
//   sun_apply       : k_apply           (a7) dv/dt = Q0 v + eps Q1 v + K
#include <cuda_runtime.h>
#include <math.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <type_traits>
#include <vector>

#include "../../include/sunfold.h"
#include "sunfold_general.cuh"
#include "sunfold_kernels.cuh"

using namespace sunk;

namespace {

constexpr int MAXOPS = 66;       // H0, H1 and up to 64 dissipators
constexpr int WLMAX = WMAX / 2;  // wK >= 2 wL
constexpr int F_MALFORMED = 1, F_PATTERN = 8, F_TOOBIG = 16;  // F_TOOBIG: sunfold_general.cu
constexpr int TP0 = 256;          // modes 0/2: pairs per fill tile == threads per fill CTA
constexpr int SLOTS_PER_TILE = 8;
#ifndef SUN_TILE_SYNC_MIN_N
#define SUN_TILE_SYNC_MIN_N 1200  // N from which the fill's output (> ~0.4 GB) streams to DRAM
#endif  // modes 0/2: scan slots (one per count warp and per fill warp) per fill tile
constexpr int WARP_TP = 64;       // mode 1: pairs per tile
constexpr int WARP_THREADS = 256;
constexpr int FAR_MAXPOS = 1024;
constexpr int EXP_THREADS = 256;  // k_expand rows (or K-band entries) per CTA
constexpr int EXP_LSTAGE = 2048;  // k_expand: staged dissipator band values per K block (32 KB)
#ifndef SUN_SCAN_IPT
#define SUN_SCAN_IPT 4
#endif
#ifndef SUN_SCAN_THREADS
#define SUN_SCAN_THREADS 256
#endif
constexpr int SCAN_THREADS = SUN_SCAN_THREADS, SCAN_IPT = SUN_SCAN_IPT, SCAN_TILE = SCAN_THREADS * SCAN_IPT;  // 1k slots per chunk (c4: 6.3 us; 4k: 8.2, 16k: 12, 512: 6.3-6.7)
static_assert(SCAN_IPT % 4 == 0, "int4 loads");
constexpr unsigned long long SCAN_A = 1ull << 62, SCAN_P = 2ull << 62, SCAN_V = (1ull << 62) - 1;

// Device header.  The prefix up to `ticket` is read back by sun_plan_nnz.
struct DevHeader {
  int flags;
  int pad;
  long long nnz[2];                  // written by the scan of each output matrix
  double tau[2];                     // drop thresholds of Q0 / Q1 (R6), on the device
  unsigned long long herm_dev[2];    // max |H - H^+| (component-wise) of H0, H1 (bits of a double >= 0)
  double nrm2_h[2];                  // ||H0||_F^2, ||H1||_F^2 (this call's values)
  unsigned int seq, pad2;            // banded count sequences run on this plan (k_expand counts)
  unsigned int ticket[2];            // chained-scan chunk tickets
  unsigned int done;                 // count-pass CTA completion counter (scan by the last CTA)
  unsigned long long wctr[2];        // fill: dynamic warp-unit counter, finished warps (reset by the last)
  int bw[MAXOPS];
  double nrm2[MAXOPS];
};
struct HeaderPrefix {
  int flags;
  int pad;
  long long nnz[2];
  double tau[2];
  unsigned long long herm_dev[2];
  double nrm2_h[2];
  unsigned int seq, pad2;  // written last by the fill (sun_run): the prefix of this sequence is complete
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

struct BlkInfo {  // k_expand: one per (operator, row block), reduced by the last block
  double nrm2;
  int bw;
  int flags;
};

struct Gammas {
  double g[MAXOPS];
};

// NVTX ranges: host-side ranges around the enqueue of each pass, named after the
// paper's steps; with graphs they mark the capture (first call) or the replay launch.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

thread_local char g_errbuf[512];

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct FarPos {
  int dc[FAR_MAXPOS];
  int dd[FAR_MAXPOS];
};

struct Layout {
  size_t hdr, fp0, fp1, inv, kb0, hb0, hb1, lb, blk, herm, ts0, ts1, st0, st1, toff0, toff1, cnt0, cnt1, sab;
  size_t side_col[2], side_val[2], side_meta[2], total;
  long long side_rows;
  long long maxslots, maxchunks, nrb;
};

Layout make_layout(int n, int P) {
  Layout L;
  long long m = (long long)n * n - 1;
  long long np = (long long)n * (n - 1) / 2;
  // slots: S tiles + J tiles + D slots
  long long maxslots = 2 * (np / 32 + 2) + n + 2;  // smallest slot: 32 pairs (modes 0 and 2)
  long long maxchunks = (maxslots + SCAN_TILE - 1) / SCAN_TILE + 1;
  long long nrb = (n + EXP_THREADS - 1) / EXP_THREADS;
  size_t off = 0;
  L.hdr = off; off = align256(off + sizeof(DevHeader));
  L.fp0 = off; off = align256(off + sizeof(FarPos));
  L.fp1 = off; off = align256(off + sizeof(FarPos));
  L.inv = off; off = align256(off + (size_t)n * sizeof(double));
  L.kb0 = off; off = align256(off + (size_t)n * (2 * WMAX + 1) * sizeof(double2));
  L.hb0 = off; off = align256(off + (size_t)n * (2 * WMAX + 1) * sizeof(double2));
  L.hb1 = off; off = align256(off + (size_t)n * (2 * WMAX + 1) * sizeof(double2));
  L.lb = off;  off = align256(off + (size_t)(P > 0 ? P : 1) * n * (2 * WLMAX + 1) * sizeof(double2));
  L.blk = off; off = align256(off + (size_t)(2 + P) * nrb * sizeof(BlkInfo));
  L.herm = off; off = align256(off + (size_t)2 * ((long long)n * (2 * WMAX + 1) / EXP_THREADS + 2) * sizeof(unsigned long long));
  L.ts0 = off; off = align256(off + (size_t)maxslots * sizeof(int));   // [ts0, toff0) zeroed per count
  L.ts1 = off; off = align256(off + (size_t)maxslots * sizeof(int));
  // status words of the chained scan, then one "offsets written" flag per chunk (k_scan_near0)
  L.st0 = off; off = align256(off + (size_t)2 * maxchunks * sizeof(unsigned long long));
  L.st1 = off; off = align256(off + (size_t)2 * maxchunks * sizeof(unsigned long long));
  L.toff0 = off; off = align256(off + (size_t)maxslots * sizeof(long long));
  L.toff1 = off; off = align256(off + (size_t)maxslots * sizeof(long long));
  L.cnt0 = off; off = align256(off + (size_t)m * sizeof(int));
  L.cnt1 = off; off = align256(off + (size_t)m * sizeof(int));
  L.sab = off;  off = align256(off + (size_t)maxslots * sizeof(int2));  // first pair of each Q0 scan slot
  // near-row side buffers of mode 0 (W <= 3): 2 rows per near item, (4W + 1)^2 entries per row
  // near-row side buffers of modes 0 and 2 (W <= 4): 2 rows per near item, (4W + 1)^2 entries
  const long long side_rows = 2 * ((long long)n * 2 * 4 + n);
  const long long ncmax = 17 * 17;
  for (int k = 0; k < 2; ++k) {
    L.side_col[k] = off; off = align256(off + (size_t)(side_rows * ncmax) * sizeof(int32_t));
    L.side_val[k] = off; off = align256(off + (size_t)(side_rows * ncmax) * sizeof(double));
    L.side_meta[k] = off; off = align256(off + (size_t)side_rows * sizeof(NearMeta));
  }
  L.side_rows = side_rows;
  L.total = off;
  L.maxslots = maxslots;
  L.maxchunks = maxchunks;
  L.nrb = nrb;
  return L;
}

// Streams, events and the pinned readback slot of a plan, recycled across plans (creating and
// destroying them, and cudaFreeHost in particular, dominated the cost of a one-shot unfold).
struct PlanRes {
  int device = -1;
  cudaStream_t aux[2] = {nullptr, nullptr}, cap = nullptr;
  cudaEvent_t fork = nullptr, join[2] = {nullptr, nullptr};
  cudaEvent_t done = nullptr;  // recorded after each readback into hpin (released plans wait on it)
  HeaderPrefix* hpin = nullptr;
  HeaderPrefix* dpin = nullptr;  // device alias of hpin (mapped): the scan writes the header there
};
std::mutex g_res_mu;
std::vector<PlanRes> g_res_free;

cudaError_t res_acquire(PlanRes& r) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  {
    std::lock_guard<std::mutex> lk(g_res_mu);
    for (size_t i = 0; i < g_res_free.size(); ++i)
      if (g_res_free[i].device == dev) {
        r = g_res_free[i];
        g_res_free.erase(g_res_free.begin() + i);
        return cudaSuccess;
      }
  }
  r = PlanRes();
  r.device = dev;
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
    e = cudaStreamCreateWithFlags(&r.aux[i], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r.join[i], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r.fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&r.done, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&r.cap, cudaStreamNonBlocking);
  if (e == cudaSuccess) {  // mapped pinned slot: the scan kernel stores the header prefix into it
    if (cudaHostAlloc(&r.hpin, sizeof(HeaderPrefix), cudaHostAllocMapped) == cudaSuccess) {
      if (cudaHostGetDevicePointer(&r.dpin, r.hpin, 0) != cudaSuccess) r.dpin = nullptr;
    } else if (cudaMallocHost(&r.hpin, sizeof(HeaderPrefix)) != cudaSuccess) {
      r.hpin = nullptr;  // pageable fallback in sun_plan_nnz
    }
    (void)cudaGetLastError();
  }
  return e;
}

void res_release(const PlanRes& r) {
  if (r.device < 0 || !r.aux[0] || !r.aux[1] || !r.cap || !r.fork || !r.join[0] || !r.join[1] || !r.done) return;
  std::lock_guard<std::mutex> lk(g_res_mu);
  g_res_free.push_back(r);
}

}  // namespace

struct sun_plan_s {
  int n, P, has_h1;
  OpList ops;      // operator descriptors (+ planned widths, rates) passed to the expand kernels
  Gammas gam;
  FarPos hfp[2];   // far-position tables (host copies; uploaded in sun_plan_create)
  sun_zcsr H0, H1;
  std::vector<sun_zcsr> L;
  std::vector<double> gamma;
  char* ws;
  size_t ws_bytes;
  Layout lay;
  int wH0, wH1, wL, wK;
  double tau0, tau1;
  Prob pr[2];
  int counted;
  int ran;            // last fill was enqueued by sun_run (capacity checked at sun_plan_nnz)
  long long cap[2];   // capacities passed to the last fill
  cudaStream_t count_stream;
  long long nnz[2];
  int npos_far[2];
  int launches_count, launches_fill;
  std::vector<int> pos_dc[2], pos_dd[2];
  NearSide side[2];
  int combined;         // mode 0 with Q1 absent or Q1 = Q_H[diagonal H1]: one launch per pass
  int near_sep = 0;     // combined: near rows by k_near0 before the fill (SUNFOLD_NEAR_SEP=1)
  int near_conc = 0;    // near_sep: k_near0 on aux[0] concurrently with the fill (SUNFOLD_NEAR_CONC)
  int scan_near = 0;    // combined, sun_run: near rows written by the scan's launch (k_scan_near0)
  int scan_direct = 1;  // chain-free scan while the chunks are few (SUNFOLD_SCAN_DIRECT=0 for A/B)
  int pdl = 0;          // combined: programmatic dependent launch between the sequence's kernels
  int pdl_run = 0;      // PDL also inside sun_run's sequence (SUNFOLD_PDL_RUN=1; A/B only)
  // phase timing (sun_plan_set_timing): events before the count, between count and fill, after
  int timing = 0;
  cudaEvent_t tev[3] = {nullptr, nullptr, nullptr};
  int timed_kind = -1;  // kind of the last timed sequence (-1: none)
  long long fill_grid[2];
  // auxiliary streams: the Q1 passes and the near-item fill run concurrently with Q0's far
  // tiles (fork/join with events on the caller's stream; also valid under graph capture)
  cudaStream_t aux[2] = {nullptr, nullptr};
  cudaEvent_t ev_fork = nullptr, ev_join[2] = {nullptr, nullptr};
  // CUDA graphs of the enqueue sequences (captured on cap_stream, launched on the caller's
  // stream), keyed by kind and output buffers; small LRU cache
  struct GraphEntry {
    uintptr_t key[12];
    cudaGraphExec_t exec;
    unsigned long long used;
  };
  cudaStream_t cap_stream = nullptr;
  std::vector<GraphEntry> graphs;
  // mode 3 (general-pattern operators, sunfold_general.cu)
  int general = 0;
  int small_cap = 0;  // SUN_PLAN_SMALLCAP (tests)
  char* stash = nullptr;  // mode 3: light-row stash (sun_plan_set_stash; caller-owned)
  sung::GLayout glay;
  sung::GProb gp[2];
  unsigned long long graph_clock = 0;
  bool use_graphs = true;
  HeaderPrefix* hpin = nullptr;  // pinned host copy of the header prefix (nnz readback)
  int hdr_enqueued = 0;          // the last count/run sequence already copies the header to hpin
  int hdr_poll = 0;              // ... and its fill stores it with a sequence number (sun_run, modes 0/2)
  unsigned seq_expect = 0;       // banded count sequences launched on this plan (DevHeader::seq)
  PlanRes res;                   // pooled streams / events / pinned slot (res_acquire)
  std::vector<std::vector<uintptr_t>> seen;  // enqueue keys run once directly (captured on reuse)
  ~sun_plan_s() {
    for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
    for (auto& e : tev)
      if (e) cudaEventDestroy(e);
    if (aux[0]) {  // nothing of this plan may still run on the pooled streams or write hpin
      cudaStreamSynchronize(aux[0]);
      cudaStreamSynchronize(aux[1]);
      cudaEventSynchronize(res.done);
      (void)cudaGetLastError();  // a destructor reports nothing: leave no error for the next call
    }
    res_release(res);
  }
};

namespace {
// fork `n` auxiliary streams off `st`
cudaError_t fork_aux(sun_plan_s* pl, cudaStream_t st, int n) {
  cudaError_t e = cudaEventRecord(pl->ev_fork, st);
  for (int i = 0; i < n && e == cudaSuccess; ++i) e = cudaStreamWaitEvent(pl->aux[i], pl->ev_fork, 0);
  return e;
}
// join `n` auxiliary streams back into `st`
cudaError_t join_aux(sun_plan_s* pl, cudaStream_t st, int n) {
  cudaError_t e = cudaSuccess;
  for (int i = 0; i < n && e == cudaSuccess; ++i) {
    e = cudaEventRecord(pl->ev_join[i], pl->aux[i]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, pl->ev_join[i], 0);
  }
  return e;
}
}  // namespace

// =========================================================================================
// Kernels
// =========================================================================================

// (validation + pattern analysis, sun_plan_create) one CTA per operator: half-bandwidth,
// ||.||_F^2, CSR checks.
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

// (a1) expand, one launch.  Blocks [0, nA): CSR -> band storage, one thread per (operator,
// row) (op 0 = H0 -> Hb0 at width wK, op 1 = H1 -> Hb1 at width wH1, op 2+p = L_p -> Lb[p] at
// width wL scaled by sqrt(gamma_p)), CSR validation, values beyond the planned bandwidth,
// ||.||_F^2 per row block (fixed-order tree).  Blocks [nA, ..): one thread per entry (r, o) of
// the K = H0 + (i/2) sum_p gamma_p L_p^+ L_p band, read straight from the CSR inputs (so no
// block waits for another), the Hermiticity deviations of H0 / H1, inv[l] = 1/sqrt(l(l+1))
// (D^l normalisation).  The last block to finish reduces the per-block records in
// fixed order into the header: norms, bandwidths, flags, Hermiticity deviations and the drop
// thresholds tau (R6).
struct ExpandArgs {
  OpList ops;
  Gammas gam;
  double2 *hb0, *hb1, *lb, *kb0;
  double* inv;
  BlkInfo* blk;             // nA records
  unsigned long long* herm; // 2 per K block
  int* zero32;
  unsigned long long* zero64;
  long long nz32, nz64;
  DevHeader* hdr;
  unsigned int* done;       // completion counter (0 between launches)
  int wK, wH1, wL, wX;      // wX = max(wK, wH1): width of the K-block grid
  int nrb, nA, nB, P;
};

// entry (r, c) of a banded CSR operator of planned half-width w: a complete band row stores
// column c at rp[r] + c - max(r - w, 0), so the column index and the value are fetched in
// parallel right after rp (two dependent loads); a search only if the guess misses
__device__ __forceinline__ double2 csr_get(const OpDesc& d, int r, int c);
__device__ __forceinline__ double2 csr_get_band(const OpDesc& d, int r, int c, int w) {
  const int64_t b = __ldg(d.rp + r), e = __ldg(d.rp + r + 1);
  const int lo = r - w > 0 ? r - w : 0;
  const int64_t g = b + (int64_t)(c - lo);
  if (c >= lo && g < e) {
    const int cc = __ldg(d.ci + g);
    const double2 vv = __ldg(d.v + g);
    if (cc == c) return vv;
  }
  return csr_get(d, r, c);
}
__device__ __forceinline__ double2 csr_get(const OpDesc& d, int r, int c) {
  for (int64_t k = d.rp[r], e = d.rp[r + 1]; k < e; ++k) {
    const int cc = d.ci[k];
    if (cc == c) return d.v[k];
    if (cc > c) break;
  }
  return make_double2(0.0, 0.0);
}

__global__ void __launch_bounds__(EXP_THREADS) k_expand(const ExpandArgs A) {
  pdl_enter();
  const OpList& ops = A.ops;
  const int n = ops.n;
  const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gstride = (long long)gridDim.x * blockDim.x;
  for (long long i = gtid; i < A.nz32; i += gstride) A.zero32[i] = 0;
  for (long long i = gtid; i < A.nz64; i += gstride) A.zero64[i] = 0ull;
  if (gtid == 0) A.hdr->ticket[0] = A.hdr->ticket[1] = 0u;
  __shared__ double red[EXP_THREADS];
  __shared__ int sbw[EXP_THREADS / 32], sfl[EXP_THREADS / 32];
  __shared__ unsigned long long sh0[EXP_THREADS / 32], sh1[EXP_THREADS / 32];
  __shared__ int last;
  __shared__ double2 A_ls[EXP_LSTAGE];
  if ((int)blockIdx.x < A.nA) {
    const int op = blockIdx.x / A.nrb, rb = blockIdx.x % A.nrb;
    double acc = 0.0;
    int bw = 0, flags = 0;
    const int r = rb * blockDim.x + threadIdx.x;
    if (!(op == 1 && !ops.has_h1) && r < n) {
      const OpDesc d = ops.op[op];
      double2* dst;
      int w;
      double sc = 1.0;
      if (op == 0) { dst = A.hb0; w = A.wK; }
      else if (op == 1) { dst = A.hb1; w = A.wH1; }
      else { dst = A.lb + (long long)(op - 2) * n * (2 * A.wL + 1); w = A.wL; sc = ops.sqrtg[op]; }
      double2* row = dst + (long long)r * (2 * w + 1);
      for (int o = 0; o <= 2 * w; ++o) row[o] = make_double2(0.0, 0.0);
      const int64_t lo = d.rp[r], hi = d.rp[r + 1];
      if (hi < lo) flags |= F_MALFORMED;
      int prev = -1;
#pragma unroll 4
      for (int64_t k = lo; k < hi; ++k) {
        const int c = __ldg(d.ci + k);
        if (c < 0 || c >= n || c <= prev) { flags |= F_MALFORMED; break; }
        prev = c;
        const double2 v = __ldg(d.v + k);
        const int o = c - r;
        const int ao = o < 0 ? -o : o;
        if (v.x != 0.0 || v.y != 0.0) bw = ao > bw ? ao : bw;
        acc += v.x * v.x + v.y * v.y;
        if (ao <= w) row[o + w] = make_double2(sc * v.x, sc * v.y);
      }
      if (ops.wplan[op] >= 0 && bw > ops.wplan[op]) flags |= F_PATTERN;
    }
    red[threadIdx.x] = acc;
    int wb = bw, wf = flags;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      wb = max(wb, __shfl_xor_sync(FULL, wb, o));
      wf |= __shfl_xor_sync(FULL, wf, o);
    }
    if ((threadIdx.x & 31) == 0) {
      sbw[threadIdx.x >> 5] = wb;
      sfl[threadIdx.x >> 5] = wf;
    }
    __syncthreads();
    for (int st = EXP_THREADS / 2; st > 0; st >>= 1) {  // fixed-order tree: deterministic
      if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      int bb = 0, f = 0;
      for (int i = 0; i < EXP_THREADS / 32; ++i) {
        bb = max(bb, sbw[i]);
        f |= sfl[i];
      }
      A.blk[blockIdx.x] = BlkInfo{red[0], bb, f};
    }
  } else {
    const long long t = (long long)(blockIdx.x - A.nA) * blockDim.x + threadIdx.x;
    if (t < n) A.inv[t] = t > 0 ? 1.0 / sqrt((double)t * (double)(t + 1)) : 0.0;
    unsigned long long d0 = 0ull, d1 = 0ull;
    const int sw = 2 * A.wX + 1;
    // the block's dissipator rows x in [x0, x0 + nx) as dense band rows in shared memory
    // (Ls[(p nx + x - x0) SL + o] = L_p(x, x + o - wL)): every CSR lookup issued at once,
    // instead of two dependent lookups per (p, x) in each K entry's loop
    const int SLd = 2 * A.wL + 1;
    const long long tb = (long long)(blockIdx.x - A.nA) * blockDim.x;
    const int rf = (int)(tb / sw), rl = (int)min((long long)n - 1, (tb + blockDim.x - 1) / sw);
    const int x0 = max(0, rf - A.wL), nx = min(n - 1, rl + A.wL) - x0 + 1;
    const bool staged = A.P > 0 && (long long)A.P * nx * SLd <= EXP_LSTAGE;
    // this thread's K entry (r, r + o) and its H0 / H1 lookups (independent of the staged rows:
    // issued before the staging barrier, so both sets of loads are in flight together); offsets
    // beyond an operator's planned width are zero (a value there raises F_PATTERN in the
    // row blocks), so no CSR search runs for them
    const bool kent = t < (long long)n * sw;
    const int r = kent ? (int)(t / sw) : 0, o = kent ? (int)(t % sw) - A.wX : 0;
    const int c = r + o;
    const bool in = kent && c >= 0 && c < n;
    const int wh = ops.wplan[0] >= 0 ? ops.wplan[0] : A.wK;
    double2 h = make_double2(0.0, 0.0), ht = h, g = h, gt = h;
    if (in && o >= -A.wK && o <= A.wK && o >= -wh && o <= wh) {
      h = csr_get_band(ops.op[0], r, c, wh);
      ht = csr_get_band(ops.op[0], c, r, wh);
    }
    if (in && ops.has_h1 && o >= -A.wH1 && o <= A.wH1) {
      g = csr_get_band(ops.op[1], r, c, A.wH1);
      gt = csr_get_band(ops.op[1], c, r, A.wH1);
    }
    if (staged) {
      for (int e = threadIdx.x; e < A.P * nx * SLd; e += blockDim.x) {
        const int p = e / (nx * SLd), f = e % (nx * SLd), x = x0 + f / SLd, cc = x + f % SLd - A.wL;
        A_ls[e] = (cc >= 0 && cc < n) ? csr_get_band(ops.op[2 + p], x, cc, A.wL) : make_double2(0.0, 0.0);
      }
    }
    __syncthreads();
    if (kent) {
      if (o >= -A.wK && o <= A.wK) {
        double2 kv = make_double2(0.0, 0.0);
        if (in) {
          double mx = 0.0, my = 0.0;
          int lo = max(r, c) - A.wL, hi = min(r, c) + A.wL;
          if (lo < 0) lo = 0;
          if (hi > n - 1) hi = n - 1;
          for (int p = 0; p < A.P; ++p) {
            const OpDesc L = ops.op[2 + p];
            double px = 0.0, py = 0.0;
            for (int x = lo; x <= hi; ++x) {
              double2 a, b;  // conj(L_xr) L_xc
              if (staged) {
                const double2* row = A_ls + ((long long)p * nx + (x - x0)) * SLd - x + A.wL;
                a = row[r];
                b = row[c];
              } else {
                a = csr_get_band(L, x, r, A.wL);
                b = csr_get_band(L, x, c, A.wL);
              }
              px += a.x * b.x + a.y * b.y;
              py += a.x * b.y - a.y * b.x;
            }
            mx += ops.gamma[2 + p] * px;
            my += ops.gamma[2 + p] * py;
          }
          kv = make_double2(h.x - 0.5 * my, h.y + 0.5 * mx);
          d0 = (unsigned long long)__double_as_longlong(fmax(fabs(h.x - ht.x), fabs(h.y + ht.y)));
        }
        A.kb0[(long long)r * (2 * A.wK + 1) + (o + A.wK)] = kv;
      }
      if (in && ops.has_h1 && o >= -A.wH1 && o <= A.wH1)
        d1 = (unsigned long long)__double_as_longlong(fmax(fabs(g.x - gt.x), fabs(g.y + gt.y)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      d0 = max(d0, __shfl_xor_sync(FULL, d0, o));
      d1 = max(d1, __shfl_xor_sync(FULL, d1, o));
    }
    if ((threadIdx.x & 31) == 0) {
      sh0[threadIdx.x >> 5] = d0;
      sh1[threadIdx.x >> 5] = d1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long m0 = 0ull, m1 = 0ull;
      for (int i = 0; i < EXP_THREADS / 32; ++i) {
        m0 = max(m0, sh0[i]);
        m1 = max(m1, sh1[i]);
      }
      A.herm[2 * (blockIdx.x - A.nA)] = m0;
      A.herm[2 * (blockIdx.x - A.nA) + 1] = m1;
    }
  }
  // the last block reduces the records (fixed order)
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(A.done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last || threadIdx.x >= 32) return;
  __threadfence();
  const int lane = threadIdx.x;
  DevHeader* hdr = A.hdr;
  int flags = 0;
  double s0 = 0.0;
  for (int op = 0; op < ops.nops; ++op) {
    if (op == 1 && !ops.has_h1) continue;
    double acc = 0.0;
    int bb = 0;
    for (int i = lane; i < A.nrb; i += 32) {  // fixed order per lane, then a fixed tree
      const BlkInfo bi = A.blk[op * A.nrb + i];
      acc += bi.nrm2;
      bb = max(bb, bi.bw);
      flags |= bi.flags;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      acc += __shfl_xor_sync(FULL, acc, o);
      bb = max(bb, __shfl_xor_sync(FULL, bb, o));
    }
    if (lane == 0) {
      hdr->nrm2[op] = acc;
      hdr->bw[op] = bb;
      if (op == 0) s0 += sqrt(acc);
      if (op >= 2) s0 += A.gam.g[op - 2] * acc;
      if (op < 2) hdr->nrm2_h[op] = acc;
    }
  }
  unsigned long long m0 = 0ull, m1 = 0ull;
  for (int i = lane; i < A.nB; i += 32) {
    m0 = max(m0, A.herm[2 * i]);
    m1 = max(m1, A.herm[2 * i + 1]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    flags |= __shfl_xor_sync(FULL, flags, o);
    m0 = max(m0, __shfl_xor_sync(FULL, m0, o));
    m1 = max(m1, __shfl_xor_sync(FULL, m1, o));
  }
  if (lane == 0) {
    hdr->flags = flags;
    hdr->herm_dev[0] = m0;
    hdr->herm_dev[1] = ops.has_h1 ? m1 : 0ull;
    hdr->tau[0] = 1e-14 * s0;
    hdr->tau[1] = ops.has_h1 ? 1e-14 * sqrt(hdr->nrm2_h[1]) : 0.0;
    if (!ops.has_h1) hdr->nrm2_h[1] = 0.0;
    hdr->seq = hdr->seq + 1u;  // one per banded count sequence (sun_plan_nnz waits for it, see store_header)
    *A.done = 0u;  // ready for the next launch
  }
}

// per-warp scratch (doubles): near-pair U tile (2 TW^2) + gS, gJ, pS, pJ (4 SW); D rows use
// the first 2 (WIN_MAX + 2)
template <int TW, int SW>
struct Scr {
  static constexpr int A = 2 * TW * TW + 4 * SW;
  static constexpr int PER_WARP = A > 2 * (WIN_MAX + 2) ? A : 2 * (WIN_MAX + 2);
};

// ---------------------------------------------------------------------------------------
// Mode 0 (compile-time widths).  One launch per output matrix and pass.
//   count: units = far tiles (TP0 = 256 consecutive pairs, thread per pair, values in
//          registers) and near units (8 near-pair / D-row items, one warp each), interleaved
//          evenly in blockIdx order so latency-bound near work overlaps the far work.  A near
//          unit also stores its rows' window entries (all S/J entries and the D entries
//          inside the window) and the D-chain tail data in a side buffer (NearSide).
//   fill:  far tiles write their far rows (staging + TMA bulk stores) and copy their near
//          rows from the side buffer, generating the chain tails; D units do the D rows.
// Tile sums (S tile t, J tile t, D slot l) are accumulated with integer atomics into zeroed
// slots (order-independent, deterministic).
// ---------------------------------------------------------------------------------------
template <int WK, int WL>
struct Mode0 {
  static constexpr int W = WK;
  static constexpr int TW = 2 * W + 1;
  static constexpr int SW = 2 * TW + 2;
  static constexpr int PER_WARP = Scr<TW, SW>::PER_WARP;
  static constexpr int NW = 4 * W + 1;             // near window bound
  static constexpr int SEG = NW * (NW - 1) / 2;    // side row segment stride (nc = NW^2)
};

// Pairs per tile: staging-free configurations (W = 0, rows of <= 2 entries) take 8 pairs per
// thread (tile = 2048 pairs) to amortise the per-tile prologue; others one pair per thread.
template <int WK, int WL>
struct Tiling {
  static constexpr bool DIRECT = FarT<WK, WL>::NPOS <= 2;
  static constexpr int PPT = DIRECT ? 8 : 1;
  static constexpr int TP = 256 * PPT;
};

// (a, b) -> the pair k positions later in lexicographic order (k >= 0; past the end: a > n-2)
__device__ __forceinline__ void pair_advance(int n, int& a, int& b, int k) {
  b += k;
  while (b >= n && a < n - 2) {
    b -= n;
    ++a;
    b += a + 1;
  }
}

// near item -> (a, b) of a near pair (b - a <= 2W) or a D row lam; returns 0 none, 1 pair, 2 D
__device__ __forceinline__ int near_item(const Prob& pr, long long item, int& a, int& b, int& lam) {
  const int W2 = 2 * pr.W;
  const long long nnear = (long long)pr.n * W2;
  if (item < nnear) {  // item < n 2W < 2^31: 32-bit division
    const unsigned it = (unsigned)item, w2 = (unsigned)W2;
    a = (int)(it / w2);
    b = a + 1 + (int)(it - (unsigned)a * w2);
    return b < pr.n ? 1 : 0;
  }
  if (item < nnear + pr.n - 1) {
    lam = (int)(item - nnear) + 1;
    return 2;
  }
  return 0;
}



// ---- count pass ------------------------------------------------------------------------
// Every count CTA is a single warp, so no unit waits on a slow sibling warp:
//   near item i: a near pair (both rows) or a D row, warp-cooperative; its window entries and
//               chain-tail data go to the side buffer (the fill pass copies them)
//   far slot s:  the far pairs of pairs [s tp, (s + 1) tp), thread per pair (PPT rounds)
// Scan slots: S slot s, J slot s (tp pairs each), one slot per D row.  Slot sums are
// accumulated with integer atomics into zeroed slots (order-independent, deterministic).
template <int WK, int WL>
__device__ __forceinline__ void count_near_item(const Prob& pr, long long item, double* scr, int* __restrict__ cnt,
                                                int* __restrict__ tsum, const NearSide& side) {
  using MC = Mode0<WK, WL>;
  const int lane = threadIdx.x & 31;
  const long long np = pr.np;
  int a, b, lam;
  const int kind = near_item(pr, item, a, b, lam);
  const long long r0 = 2 * item * side.nc, r1 = r0 + side.nc;
  if (kind == 1) {
    int c1, c2;
    double k1, k2;
    TailInfo tS, tJ;
    const Seg sS = {side.col + r0, side.val + r0, side.nc}, sJ = {side.col + r1, side.val + r1, side.nc};
    warp_near_pair<true, MC::TW, MC::SW, false, MC::SEG>(pr, a, b, scr, c1, c2, k1, k2, sS, 0, sJ, 0, &tS, &tJ);
    if (lane == 0) {
      side.meta[2 * item] = NearMeta{tS.tr, k1, tS.n1, tS.n2, tS.nwin - tS.n1 - tS.n2, tS.hi, tS.lend, 0};
      side.meta[2 * item + 1] = NearMeta{tJ.tr, k2, tJ.n1, tJ.n2, tJ.nwin - tJ.n1 - tJ.n2, tJ.hi, tJ.lend, 0};
      const long long p = (long long)pidx32(pr.n, a, b);
      cnt[p] = c1;
      cnt[np + p] = c2;
      atomicAdd(&tsum[p / pr.tp], c1);
      atomicAdd(&tsum[pr.npt + p / pr.tp], c2);
    }
  } else if (kind == 2) {
    double kv;
    TailInfo t;
    const Seg sD = {side.col + r0, side.val + r0, side.nc};
    const int c = warp_d_row<true, false, MC::SEG>(pr, lam, scr, scr + WIN_MAX + 2, kv, sD, 0, &t);
    if (lane == 0) {
      side.meta[2 * item] = NearMeta{t.tr, kv, t.n1, t.n2, t.nwin - t.n1 - t.n2, t.hi, t.lend, 0};
      cnt[2 * np + lam - 1] = c;
      tsum[2 * pr.npt + lam - 1] = c;
    }
  }
}

template <int WK, int WL, int PT>
__device__ __forceinline__ void count_far_slot(const FarCtx& pr, long long npt, long long s, int* __restrict__ cnt,
                                               int* __restrict__ tsum, int2* __restrict__ sab) {
  using MC = Mode0<WK, WL>;
  using TL = Tiling<WK, WL>;
  const int lane = threadIdx.x & 31;
  const long long np = pr.np;
  const long long pw = s * (32 * TL::PPT);  // the slot's first pair
  int a, b;
  warp_pairs(pr.n, pw, a, b);
  if (sab && lane == 0) sab[s] = make_int2(a, b);  // the fill warps of this slot start from it
  int c = 0;
#pragma unroll 1
  for (int j = 0; j < TL::PPT; ++j) {
    const long long p = pw + j * 32 + lane;
    if (j) pair_advance(pr.n, a, b, 32);
    const bool far = p < np && (b - a > 2 * MC::W);
    if (far) {
      int cp = 0;
      if constexpr (FarT<WK, WL>::NPOS > 32) {
        // wide bands: the positions one by one with the per-position expression (far_value_at:
        // the same operations as far_values, so the fill's decisions agree bit for bit) -- the
        // 33 complex values of far_values would hold ~240 registers (8 count warps per SM)
        Prob pp{};
        pp.n = pr.n;
        pp.P = pr.P;
        pp.K.v = pr.K;
        pp.L = pr.L;
#pragma unroll
        for (int k = 0; k < FarT<WK, WL>::NPOS; ++k) {
          double x, y;
          int cc, dd;
          if (far_value_at<WK, WL, PT>(pp, a, b, k, x, y, cc, dd)) cp += (fabs(x) > pr.tau) + (fabs(y) > pr.tau);
        }
      } else {
        double ux[FarT<WK, WL>::NPOS], uy[FarT<WK, WL>::NPOS];
        far_values<WK, WL, PT>(pr, a, b, ux, uy);
        typename FarT<WK, WL>::Mask mr, mi;
        far_masks<WK, WL>(pr.n, pr.tau, a, b, ux, uy, mr, mi);
        cp = mpopc(mr) + mpopc(mi);
      }
      cnt[p] = cp;
      cnt[np + p] = cp;
      c += cp;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
  if (lane == 0 && c) {  // into this count warp's scan slot (near items of the slot add theirs)
    atomicAdd(&tsum[s], c);  // S rows and J rows of a far pair have the same length
    atomicAdd(&tsum[npt + s], c);
  }
}

// One output matrix's arguments of the count pass.
struct MatCount {
  Prob pr;
  int* cnt;
  int* tsum;
  NearSide side;
  int2* sab;  // mode 0: first pair (a, b) of each scan slot, for the fill (nullptr: not stored)
};

#ifndef SUN_FILL_DYN
#define SUN_FILL_DYN 1  // k_fill0: warp-level units claimed from a global counter (combined plans)
#endif
#ifndef SUN_PDL_DEFAULT
#define SUN_PDL_DEFAULT 3  // launches with the PDL attribute (bits: 1 count, 2 scan, 4 near, 8 fill);
// measured at c4 (B200, bench step, same box): sun_count's sequence 42.7 -> 39.6 us with count +
// scan; inside the full sun_run sequence every PDL edge made the step slower (108.6 us without,
// +0.8 scan, +1.6 fill, +3 count, +4 all), so sun_run launches without it
#endif
#ifndef SUN_PDL_COUNT
#define SUN_PDL_COUNT 1  // 0: no PDL code in the count kernel, 1: wait only, 2: wait + early trigger
#endif

// One unit of the count pass of Q0 (compile-time widths WK, WL, PT) and, with Q1W >= 0, of Q1
// (widths Q1W, 0, no dissipators), warp-cooperative; units in the order
//   [Q0 near items][Q1 near items][Q0 far slots][Q1 far slots]   (long near items first)
// scr: the warp's shared scratch (Mode0 PER_WARP doubles).
template <int WK, int WL, int PT, int Q1W>
struct Count0 {
  static constexpr int Q1K = Q1W > 0 ? Q1W : 0;
  static constexpr int PW0 = Mode0<WK, WL>::PER_WARP, PW1 = Mode0<Q1K, 0>::PER_WARP;
  static constexpr int PW = PW0 > PW1 ? PW0 : PW1;
  static constexpr bool HAS1 = Q1W >= 0;
  static __host__ __device__ long long near_units(const MatCount& m0, const MatCount& m1) {
    return m0.pr.nb_near + (HAS1 ? m1.pr.nb_near : 0);
  }
  static __host__ __device__ long long units(const MatCount& m0, const MatCount& m1) {
    return near_units(m0, m1) + m0.pr.npt + (HAS1 ? m1.pr.npt : 0);
  }
};

template <int WK, int WL, int PT, int Q1W>
__device__ __forceinline__ void count0_unit(const MatCount& m0, const MatCount& m1, long long u, double* scr) {
  using C = Count0<WK, WL, PT, Q1W>;
  constexpr int Q1K = C::Q1K;
  constexpr bool HAS1 = C::HAS1;
  const long long nn0 = m0.pr.nb_near, nn1 = HAS1 ? m1.pr.nb_near : 0;
  if (u < nn0) {
    Prob prn = m0.pr;
    prn.tau = *m0.pr.tau_ptr;
    count_near_item<WK, WL>(prn, u, scr, m0.cnt, m0.tsum, m0.side);
    return;
  }
  u -= nn0;
  if (u < nn1) {
    if constexpr (HAS1 && Q1W == 0) {
      // Q1 = Q_H[H1] with H1 diagonal (this instantiation): its near items are the D rows, and
      // L^+(D^l) = i[H1, D^l] is exactly zero (diagonal matrices: h_a d_a - d_a h_a = 0 in
      // floating point too), so every D row is empty; record that without evaluating it
      if ((threadIdx.x & 31) == 0) {
        const long long lam = u + 1;  // Q1 has W = 0: near item u is the D row l = u + 1
        m1.cnt[2 * m1.pr.np + lam - 1] = 0;
        m1.tsum[2 * m1.pr.npt + lam - 1] = 0;
        m1.side.meta[2 * u] = NearMeta{0.0, 0.0, 0, 0, 0, 0, 0, 0};
      }
    } else if constexpr (HAS1) {
      Prob prn = m1.pr;
      prn.tau = *m1.pr.tau_ptr;
      count_near_item<Q1K, 0>(prn, u, scr, m1.cnt, m1.tsum, m1.side);
    }
    return;
  }
  u -= nn1;
  const long long nw0 = m0.pr.npt;  // one count warp per scan slot
  if (u < nw0) {
    const FarCtx prf{m0.pr.K.v, m0.pr.L, *m0.pr.tau_ptr, m0.pr.np, m0.pr.n, m0.pr.P};
    count_far_slot<WK, WL, PT>(prf, m0.pr.npt, u, m0.cnt, m0.tsum, m0.sab);
    return;
  }
  u -= nw0;
  if constexpr (HAS1) {
    const FarCtx prf{m1.pr.K.v, m1.pr.L, *m1.pr.tau_ptr, m1.pr.np, m1.pr.n, m1.pr.P};
    count_far_slot<Q1K, 0, 0>(prf, m1.pr.npt, u, m1.cnt, m1.tsum, nullptr);
  }
}

// one single-warp CTA per unit (2 or 4 independent warps per CTA measured slower at c3 and c4: the
// step 127 -> 134 us and 97 -> 99 / 103 us)
template <int WK, int WL, int PT, int Q1W>
__global__ void __launch_bounds__(32) k_count0(const MatCount m0, const MatCount m1) {
#if SUN_PDL_COUNT == 1
  pdl_wait();
#elif SUN_PDL_COUNT == 2
  pdl_enter();
#endif
  __shared__ double scr[Count0<WK, WL, PT, Q1W>::PW];
  count0_unit<WK, WL, PT, Q1W>(m0, m1, blockIdx.x, scr);
}

// ---------------------------------------------------------------------------------------
// (a5) fill pass outputs
// ---------------------------------------------------------------------------------------
struct FillOut {
  int64_t* row_ptr;
  int32_t* col;
  double* val;
  long long cap;  // capacity of col/val (writes at or beyond it are dropped; see sun_run)
  double* K;      // nullptr: not written (Q1)
  const long long* toff;
  const long long* nnz;
};

// Near rows (the S and J rows of near pairs, and the D rows) are written by near units, one
// warp per row, from the count pass's side buffer: window entries copied, chain-tail entries
// tr * inv[l], l in (hi, lend], generated with the count pass's expression (bitwise
// identical).  Row offset = tile offset + the tile's earlier counts (warp reduction); D rows
// have a scan slot of their own.  Loops are unrolled so the loads of several iterations are in
// flight together.
__device__ __forceinline__ void warp_near_row_write(const NearSide& side, long long srow, const NearMeta& m,
                                                   const double* __restrict__ inv, int dbase, const FillOut& fo,
                                                   long long o) {
  const int lane = threadIdx.x & 31;
  const long long lim = fo.cap - o;
  const int32_t* sc = side.col + srow * side.nc;
  const double* sv = side.val + srow * side.nc;
  // window: segments [0, n1), [seg, seg + n2), [2 seg, 2 seg + nd) -> output [0, nwin)
  const int nwin = m.n1 + m.n2 + m.nd, b2 = m.n1 + m.n2;
#pragma unroll 3
  for (int k = lane; k < nwin; k += 32) {
    const int sidx = k < m.n1 ? k : (k < b2 ? side.seg + (k - m.n1) : 2 * side.seg + (k - b2));
    const int c = __ldg(&sc[sidx]);
    const double v = __ldg(&sv[sidx]);
    if (k < lim) {
      fo.col[o + k] = c;
      fo.val[o + k] = v;
    }
  }
  const long long ot = o + nwin;
  const long long limt = lim - nwin;
#pragma unroll 4
  for (int l = m.hi + 1 + lane; l <= m.lend; l += 32) {
    const int k = l - m.hi - 1;
    const double v = m.tr * __ldg(&inv[l]);
    if (k < limt) {
      fo.col[ot + k] = dbase + l;
      fo.val[ot + k] = v;
    }
  }
}

// near unit j (modes 0, 1-row-per-warp): side rows 8j .. 8j + 7 (row 2i = S row / D row of near
// item i, 2i + 1 = J row)
__device__ __forceinline__ void fill_near_unit(const Prob& pr, long long j, const int* __restrict__ cnt,
                                               const FillOut& fo, const NearSide& side) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long np = pr.np;
  const long long srow = j * 8 + wid;
  const long long item = srow >> 1;
  const int half = (int)(srow & 1);
  int a, b, lam;
  const int kind = near_item(pr, item, a, b, lam);
  long long o;
  if (kind == 1) {
    const long long p = (long long)pidx32(pr.n, a, b);
    const long long tb = p / pr.tp, ts = tb * pr.tp;
    const int* c = cnt + (half ? np : 0);
    int s1 = 0;
    for (long long q = ts + lane; q < p; q += 32) s1 += __ldg(&c[q]) & CNT_MASK;  // mode 2 packs nR above
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) s1 += __shfl_xor_sync(FULL, s1, sh);
    o = fo.toff[(half ? pr.npt : 0) + tb] + s1;
    const NearMeta m = side.meta[srow];
    if (lane == 0 && fo.K) fo.K[(half ? np : 0) + p] = m.k;
    warp_near_row_write(side, srow, m, pr.inv, (int)(2 * np - 1), fo, o);
  } else if (kind == 2 && half == 0) {
    o = fo.toff[2 * pr.npt + lam - 1];
    const NearMeta m = side.meta[srow];
    if (lane == 0) {
      fo.row_ptr[2 * np + lam - 1] = o;
      if (fo.K) fo.K[2 * np + lam - 1] = m.k;
    }
    warp_near_row_write(side, srow, m, pr.inv, (int)(2 * np - 1), fo, o);
  }
}

// Mode-0 near unit j with two rows per warp (16-lane halves): side rows 16 j .. 16 j + 15.  The
// two rows' dependent lookups (slot prefix, offsets, metadata) overlap in one instruction
// stream; every shuffle is on convergent code, the copies are half-warp strided loops.
#ifndef SUN_NEAR_RPW
#define SUN_NEAR_RPW 2
#endif
constexpr int NEAR_RPW = SUN_NEAR_RPW;        // near rows per warp (lane groups of 32 / NEAR_RPW)
constexpr int NEAR_GL = 32 / NEAR_RPW;        // lanes per row
constexpr int NEAR_UROWS = 8 * NEAR_RPW;      // side rows per near unit
// inv: the inv[l] table (SMEM_INV: a shared-memory copy, else global through the read-only path).
// srow0: the warp's first side row (its NEAR_RPW rows are srow0, srow0 + 1, ...)
// done: when not null, the scan of this launch is still running (k_scan_near0): the row's slot
// offset is read once done[slot's chunk] is set, after every lookup that does not depend on it.
template <bool SMEM_INV>
__device__ __forceinline__ void fill_near_rows_w(const Prob& pr, long long srow0, const int* __restrict__ cnt,
                                                 const FillOut& fo, const NearSide& side, const double* inv,
                                                 const unsigned long long* done = nullptr) {
  const int lane = threadIdx.x & 31;
  const int hl = lane & (NEAR_GL - 1);
  const long long np = pr.np;
  const long long nside = 2 * ((long long)pr.n * 2 * pr.W + pr.n - 1);
  const long long srow = srow0 + lane / NEAR_GL;
  int kind = 0, half = 0, a = 0, b = 0, lam = 0;
  long long p = 0;
  if (srow < nside) {
    half = (int)(srow & 1);
    kind = near_item(pr, srow >> 1, a, b, lam);
    if (kind == 2 && half) kind = 0;
    if (kind == 1) p = (long long)pidx32(pr.n, a, b);
  }
  // every lookup of the row issued together (metadata, slot offset, the slot's earlier counts:
  // independent loads), reduced after: one round trip before the copy instead of three
  NearMeta m{};
  long long o = 0;
  int s1 = 0;
  const long long slot = kind == 1 ? (half ? pr.npt : 0) + p / pr.tp : 2 * pr.npt + lam - 1;
  if (kind != 0) {
    m = side.meta[srow];
    if (!done) o = __ldg(&fo.toff[slot]);
  }
  if (kind == 1) {
    const long long ts = (p / pr.tp) * pr.tp;
    const int* c = cnt + (half ? np : 0);
    static_assert(SLOTS_PER_TILE * 32 == TP0, "slot = 32 pairs");
#pragma unroll
    for (int i = 0; i < 32 / NEAR_GL; ++i) {  // the slot's <= 31 earlier pairs (tp = 32)
      const long long q = ts + hl + i * NEAR_GL;
      s1 += q < p ? (__ldg(&c[q]) & CNT_MASK) : 0;  // mode 2 packs nR above
    }
    for (long long q = ts + hl + 32; q < p; q += NEAR_GL) s1 += __ldg(&c[q]) & CNT_MASK;  // (tp > 32)
  }
#pragma unroll
  for (int sh = NEAR_GL / 2; sh > 0; sh >>= 1) s1 += __shfl_xor_sync(FULL, s1, sh);  // within each group
  if (done) {  // warp-uniform wait for the scan chunks of the warp's rows, then the offsets from L2
    const volatile unsigned long long* vd = done + (kind != 0 ? slot / SCAN_TILE : 0);
    bool ready = kind == 0 || *vd != 0ull;
    while (!__all_sync(FULL, ready)) {
      __nanosleep(64);
      if (!ready) ready = *vd != 0ull;
    }
    __threadfence();
    if (kind != 0) o = __ldcg(&fo.toff[slot]);
  }
  if (kind == 0) return;  // no shuffles below
  if (kind == 1) {
    o += s1;
    if (hl == 0 && fo.K) fo.K[(half ? np : 0) + p] = m.k;
  } else if (hl == 0) {
    fo.row_ptr[2 * np + lam - 1] = o;
    if (fo.K) fo.K[2 * np + lam - 1] = m.k;
  }
  const long long lim = fo.cap - o;
  const int32_t* sc = side.col + srow * side.nc;
  const double* sv = side.val + srow * side.nc;
  const int nwin = m.n1 + m.n2 + m.nd, b2 = m.n1 + m.n2;
#pragma unroll 2
  for (int k = hl; k < nwin; k += NEAR_GL) {
    const int sidx = k < m.n1 ? k : (k < b2 ? side.seg + (k - m.n1) : 2 * side.seg + (k - b2));
    const int c = __ldg(&sc[sidx]);
    const double v = __ldg(&sv[sidx]);
    if (k < lim) {
      fo.col[o + k] = c;
      fo.val[o + k] = v;
    }
  }
  const long long ot = o + nwin, limt = lim - nwin;
  const int dbase = (int)(2 * np - 1);
#pragma unroll 4
  for (int l = m.hi + 1 + hl; l <= m.lend; l += NEAR_GL) {
    const int k = l - m.hi - 1;
    const double v = m.tr * (SMEM_INV ? inv[l] : __ldg(&inv[l]));
    if (k < limt) {
      fo.col[ot + k] = dbase + l;
      fo.val[ot + k] = v;
    }
  }
}

// near unit j: side rows j NEAR_UROWS .. + NEAR_UROWS - 1 over the CTA's 8 warps
template <bool SMEM_INV>
__device__ __forceinline__ void fill_near_unit_h(const Prob& pr, long long j, const int* __restrict__ cnt,
                                                 const FillOut& fo, const NearSide& side, const double* inv) {
  fill_near_rows_w<SMEM_INV>(pr, j * NEAR_UROWS + (threadIdx.x >> 5) * NEAR_RPW, cnt, fo, side, inv);
}

__host__ __device__ inline long long near_units1(long long n, long long W) {  // units of 8 side rows
  return (2 * (n * 2 * W + n - 1) + 7) / 8;
}

// Mode 2 (long window rows, N^2 tails): near units of NEAR_UNIT_ROWS side rows (batched).
// Near rows written by near units of
// NEAR_UNIT_ROWS side rows (8 per warp) from the count pass's side buffer: window entries
// copied, chain-tail entries tr * inv[l], l in (hi, lend], generated with the count pass's
// expression (bitwise identical).  Row offset = slot offset + the slot's earlier counts; D
// rows have a scan slot of their own.  Each warp first resolves its 8 rows' offsets and
// metadata together (lane r: row r; the slot prefix sums by warp-wide loads, all issued
// before any is consumed), then writes the 8 rows as one flattened, lane-strided stream, so
// no row waits on another's lookups.
#ifndef SUN_NEAR_WARP_ROWS
#define SUN_NEAR_WARP_ROWS 8
#endif
constexpr int NEAR_WARP_ROWS = SUN_NEAR_WARP_ROWS;
constexpr int NEAR_UNIT_ROWS = 8 * NEAR_WARP_ROWS;
__host__ __device__ inline long long near_units(long long n, long long W) {
  return (2 * (n * 2 * W + n - 1) + NEAR_UNIT_ROWS - 1) / NEAR_UNIT_ROWS;
}
struct NearRowP {
  long long o, sbase;  // output offset of the row, side-buffer offset of its slot
  double tr;           // chain-tail trace
  int pref, len;       // exclusive prefix of len over the warp's rows; entries to write
  int n1, b2, nwin, hi;
};

__device__ __forceinline__ void fill_near_unit_b(const Prob& pr, long long j, const int* __restrict__ cnt,
                                                 const FillOut& fo, const NearSide& side, NearRowP* rows) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long np = pr.np;
  const long long nside = 2 * ((long long)pr.n * 2 * pr.W + pr.n - 1);
  const long long srow = j * NEAR_UNIT_ROWS + wid * NEAR_WARP_ROWS + lane;  // lanes 0..7: the warp's rows
  int kind = 0, half = 0, lam = 0;
  long long p = 0;
  if (lane < NEAR_WARP_ROWS && srow < nside) {
    int a, b;
    half = (int)(srow & 1);
    kind = near_item(pr, srow >> 1, a, b, lam);
    if (kind == 2 && half) kind = 0;  // D items use one side row
    if (kind == 1) p = (long long)pidx32(pr.n, a, b);
  }
  // slot prefix sums of the near-pair rows (mode 2 packs nR above CNT_BITS)
  int s1 = 0;
#pragma unroll
  for (int r = 0; r < NEAR_WARP_ROWS; ++r) {
    const int kr = __shfl_sync(FULL, kind, r);
    const long long pr_ = __shfl_sync(FULL, p, r);
    const int hr = __shfl_sync(FULL, half, r);
    int sum = 0;
    if (kr == 1) {  // warp-uniform
      const long long ts = (pr_ / pr.tp) * pr.tp;
      const int* c = cnt + (hr ? np : 0);
      for (long long q = ts + lane; q < pr_; q += 32) sum += __ldg(&c[q]) & CNT_MASK;
    }
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) sum += __shfl_xor_sync(FULL, sum, sh);
    if (lane == r) s1 = sum;
  }
  int len = 0;
  NearRowP rp{};
  if (kind != 0) {
    const NearMeta m = side.meta[srow];
    long long o;
    if (kind == 1) {
      o = fo.toff[(half ? pr.npt : 0) + p / pr.tp] + s1;
      if (fo.K) fo.K[(half ? np : 0) + p] = m.k;
    } else {
      o = fo.toff[2 * pr.npt + lam - 1];
      fo.row_ptr[2 * np + lam - 1] = o;
      if (fo.K) fo.K[2 * np + lam - 1] = m.k;
    }
    const int nwin = m.n1 + m.n2 + m.nd;
    const long long want = nwin + (m.lend > m.hi ? m.lend - m.hi : 0);
    const long long room = fo.cap - o;  // writes at or beyond the capacity are dropped
    len = (int)(want < room ? want : (room > 0 ? room : 0));
    rp = NearRowP{o, srow * side.nc, m.tr, 0, len, m.n1, m.n1 + m.n2, nwin, m.hi};
  }
  int ex = len;  // exclusive prefix over lanes 0..7
#pragma unroll
  for (int o = 1; o < NEAR_WARP_ROWS; o <<= 1) {
    const int y = __shfl_up_sync(FULL, ex, o);
    if (lane >= o) ex += y;
  }
  const int total = __shfl_sync(FULL, ex, NEAR_WARP_ROWS - 1);
  ex -= len;
  if (lane < NEAR_WARP_ROWS) {
    rp.pref = ex;
    rp.len = len;
    rows[lane] = rp;
  }
  __syncwarp();
  const int dbase = (int)(2 * np - 1);
  int pf[NEAR_WARP_ROWS], pe[NEAR_WARP_ROWS];  // row t owns [pf[t], pe[t])
#pragma unroll
  for (int t = 0; t < NEAR_WARP_ROWS; ++t) {
    pf[t] = __shfl_sync(FULL, ex, t);
    pe[t] = pf[t] + __shfl_sync(FULL, len, t);
  }
#pragma unroll 4
  for (int k = lane; k < total; k += 32) {
    int r = 0;
#pragma unroll
    for (int t = 1; t < NEAR_WARP_ROWS; ++t)
      if (pf[t] <= k && k < pe[t]) r = t;
    const NearRowP& R = rows[r];
    const int idx = k - R.pref;
    int c;
    double v;
    if (idx < R.nwin) {
      const int sidx = idx < R.n1 ? idx : (idx < R.b2 ? side.seg + (idx - R.n1) : 2 * side.seg + (idx - R.b2));
      c = __ldg(&side.col[R.sbase + sidx]);
      v = __ldg(&side.val[R.sbase + sidx]);
    } else {
      const int l = R.hi + 1 + (idx - R.nwin);
      c = dbase + l;
      v = R.tr * __ldg(&pr.inv[l]);
    }
    fo.col[R.o + idx] = c;
    fo.val[R.o + idx] = v;
  }
  __syncwarp();  // rows[] reused by the warp's next unit
}

// Copy a warp's staged segment [g0, g1) (tile-local offsets) to global memory, skipping the
// "holes" of near rows (lanes flagged in `holes`, hole = [hoff, hoff + hlen)).  The stage
// position advances only over copied entries.
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

template <int WK, int WL>
struct FillFar {
  static constexpr int NPOS = FarT<WK, WL>::NPOS;
  static constexpr bool DIRECT = NPOS <= 2;             // rows of <= 4 entries: no staging
  static constexpr int CAPW = DIRECT ? 0 : 64 * NPOS;   // entries of one 32-row block, worst case
  static constexpr int COLW = DIRECT ? 0 : (CAPW + 4 + 3) & ~3;  // int32 slots (+ pad), 16-B multiple
  static constexpr int VALW = DIRECT ? 0 : (CAPW + 2 + 1) & ~1;  // fp64 slots (+ pad)
  static constexpr int BYTES_PER_WARP = COLW * 4 + VALW * 8;
  static constexpr int SMEM = 8 * BYTES_PER_WARP;
  // resident fill CTAs per SM: 2 (16 warps) while the staging fits twice; wide bands (e.g. 33
  // positions: 203 KB of staging) run one CTA per SM with the whole register file per thread
  static constexpr int MINB = SMEM <= 112 * 1024 ? 2 : 1;
};

// Far tile t (256 pairs, thread per pair): row_ptr of all the tile's rows, K of its pairs;
// each warp stages its 32 far S rows (then J rows) in shared memory and writes the block out
// with TMA bulk stores (cp.async.bulk) when the block has no near-row holes (16-byte phase
// matched in the staging, head/tail entries by lanes), else with coalesced warp stores; the
// warp then writes its near rows from the side buffer.
// per-tile inputs, loaded one unit ahead (software pipelining of the persistent loop)
struct TileIn {
  int cS, cJ;
  long long baseS, baseJ;
  int2 ab;  // first pair of the warp's slot (count pass table), x < 0: decode it
};
// w: the warp's slot within the tile (its 32 pairs)
__device__ __forceinline__ TileIn load_tile_in(long long np, long long npt, long long t, const int* __restrict__ cnt,
                                               const long long* __restrict__ toff, const int2* __restrict__ sab,
                                               int w) {
  const long long p = t * TP0 + w * 32 + (threadIdx.x & 31);
  const long long slot = t * SLOTS_PER_TILE + w;
  TileIn ti;
  ti.cS = p < np ? cnt[p] : 0;
  ti.cJ = p < np ? cnt[np + p] : 0;
  ti.baseS = slot < npt ? toff[slot] : 0;
  ti.baseJ = slot < npt ? toff[npt + slot] : 0;
  ti.ab = sab && slot < npt ? __ldg(&sab[slot]) : make_int2(-1, -1);
  return ti;
}
// the pairs of this warp's 32 lanes in far tile t: from the slot table, else decoded
__device__ __forceinline__ void tile_pairs(int n, long long t, int w, int2 ab, int& a, int& b) {
  if (ab.x >= 0)
    warp_pairs_from(n, ab.x, ab.y, a, b);
  else
    warp_pairs(n, t * TP0 + w * 32, a, b);
}

template <int WK, int WL, int PT>
__device__ __forceinline__ void fill_far_tile(const FarCtx& pr, long long npt, long long t, int w, const TileIn& ti,
                                              const FillOut& fo, int* scol, double* sval) {
  using MC = Mode0<WK, WL>;
  using FF = FillFar<WK, WL>;
  const int lane = threadIdx.x & 31;
  const long long np = pr.np;
  const long long p = t * TP0 + w * 32 + lane;
  const bool valid = p < np;
  const int cS = ti.cS, cJ = ti.cJ;
  int a, b;
  tile_pairs(pr.n, t, w, ti.ab, a, b);
  const bool far = valid && (b - a > 2 * MC::W);
  const bool nearp = valid && !far;
  // U values first, for every lane (any 0 <= a < b < n is a safe address set; non-far lanes
  // are masked below): the band loads are in flight during the offset scans and row_ptr stores
  double ux[FarT<WK, WL>::NPOS], uy[FarT<WK, WL>::NPOS];
#ifdef SUN_EXP_NO_COMPUTE
#pragma unroll
  for (int k = 0; k < FarT<WK, WL>::NPOS; ++k) {
    ux[k] = 1.0 + k;
    uy[k] = k < 9 ? 1.0 : 0.0;
  }
#else
  far_values<WK, WL, PT>(pr, a, b, ux, uy);
#endif
  int totS, totJ;  // warp-local offsets: every warp has a scan slot of its own (no CTA barrier)
  const int exS = warp_excl_scan(cS, totS), exJ = warp_excl_scan(cJ, totJ);
  const long long baseS = ti.baseS, baseJ = ti.baseJ;
  if (valid) {
    fo.row_ptr[p] = baseS + exS;
    fo.row_ptr[np + p] = baseJ + exJ;
    if (fo.K && far) {
      fo.K[p] = 0.0;
      fo.K[np + p] = 0.0;
    }
  }
#ifdef SUN_EXP_PROLOGUE_ONLY
  return;
#endif
  int qb[2 * WK + 1];
  typename FarT<WK, WL>::Mask mr = 0u, mi = 0u;
  if (far) {
    far_masks<WK, WL>(pr.n, pr.tau, a, b, ux, uy, mr, mi);
    far_colbase<WK>(pr.n, a, b, qb);
  }
  const unsigned nearmask = __ballot_sync(FULL, nearp);
  if constexpr (FF::DIRECT) {
    // rows of <= 4 entries: each thread writes its rows directly (adjacent lanes write
    // adjacent rows, so the stores are already coalesced)
    if (far) {
      const Seg seg = {fo.col, fo.val, fo.cap};
#pragma unroll
      for (int row = 0; row < 2; ++row) {
        const long long o = (row ? baseJ + exJ : baseS + exS);
        const auto m1 = row ? mi : mr, m2 = row ? mr : mi;
        int o1 = 0, o2 = mpopc(m1);
        far_foreach<WK, WL>([&](int k, int dc, int dd) {
          const int qk = qb[dc + WK] + dd;
          if ((m1 >> k) & 1u) seg.emit(o + o1++, qk, row ? uy[k] : ux[k]);
          if ((m2 >> k) & 1u) seg.emit(o + o2++, (int)np + qk, row ? ux[k] : -uy[k]);
        });
      }
    }
  } else {
    // the warp's 32 S rows, then its 32 J rows
    auto do_row = [&](auto row_c) {
      constexpr int row = decltype(row_c)::value;
      const int c_me = row ? cJ : cS, ex_me = row ? exJ : exS;
      const long long gbase = row ? baseJ : baseS;
      const int w0 = __shfl_sync(FULL, ex_me, 0);
      const int wt = __shfl_sync(FULL, ex_me + c_me, 31) - w0;  // rows of invalid lanes have c = 0
      const long long g = gbase + w0;                              // global index of the block's first entry
      const bool bulk = nearmask == 0u && g + wt <= fo.cap;
      if (lane == 0) bulk_wait_read0();  // earlier bulk reads of this warp's staging are done
      __syncwarp();
      int pc = 0, pv = 0, hb = 0;
      if (bulk) {  // stage with the global 16-byte phase of the block's first entry
        pc = (int)(((uintptr_t)(fo.col + g) >> 2) & 3);
        pv = (int)(((uintptr_t)(fo.val + g) >> 3) & 1);
      } else {
        int ht;
        hb = warp_excl_scan(nearp ? c_me : 0, ht);
      }
#ifndef SUN_EXP_NO_STAGE
      if (far) far_stage_row<WK, WL, row>((int)np, qb, ux, uy, mr, mi, scol + pc, sval + pv, ex_me - w0 - hb);
#endif
#ifndef SUN_EXP_NO_FENCE
      if (bulk) fence_async_smem();  // make the staged entries visible to the async (TMA) proxy
#endif
      __syncwarp();
      if (bulk) {
        // col: int32, 16 B = 4 entries; val: fp64, 16 B = 2 entries
        const long long end = g + wt;
        const long long ca = g + ((4 - pc) & 3), ce = ca <= end ? ca + ((end - ca) & ~3ll) : ca;
        const long long va = g + pv, ve = va <= end ? va + ((end - va) & ~1ll) : va;
#ifndef SUN_EXP_NO_STORE
        if (lane == 0) {
          if (ce > ca) bulk_s2g(fo.col + ca, scol + pc + (ca - g), (unsigned)((ce - ca) * 4));
          if (ve > va) bulk_s2g(fo.val + va, sval + pv + (va - g), (unsigned)((ve - va) * 8));
          bulk_commit();
        }
#endif
        // head / tail entries outside the aligned middles (at most 3 + 3 col, 1 + 1 val)
        if (ce > ca) {
          const long long k = lane < 4 ? g + lane : ce + (lane - 4);
          if ((lane < 4 && k < ca) || (lane >= 4 && lane < 8 && k < end)) fo.col[k] = scol[pc + (k - g)];
        } else if (lane < wt) {
          fo.col[g + lane] = scol[pc + lane];
        }
        if (ve > va) {
          const long long k = lane < 2 ? g + lane : ve + (lane - 2);
          if ((lane < 2 && k < va) || (lane >= 2 && lane < 4 && k < end)) fo.val[k] = sval[pv + (k - g)];
        } else if (lane < wt) {
          fo.val[g + lane] = sval[pv + lane];
        }
      } else {
        warp_copy_out(scol, sval, gbase, w0, w0 + wt, nearmask, ex_me, c_me, fo.col, fo.val, fo.cap);
      }
      __syncwarp();
    };
    do_row(std::integral_constant<int, 0>{});
    do_row(std::integral_constant<int, 1>{});
  }
}

// Staging-free far tile (W = 0: every pair is far, rows of <= 2 entries), TP = 2048 pairs:
// warp w owns pairs [t TP + 256 w, + 256), 8 coalesced iterations of 32 pairs; row offsets
// from warp scans with a running carry and a block scan of the warp totals.
template <int WK, int WL, int PT>
__device__ __forceinline__ void fill_direct_tile(const FarCtx& pr, long long npt, long long t,
                                                 const int* __restrict__ cnt, const FillOut& fo) {
  using TL = Tiling<WK, WL>;
  static_assert(TL::DIRECT && WK == 0, "direct tile: W = 0");
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long np = pr.np;
  const long long pw = t * TL::TP + (long long)wid * 32 * TL::PPT;
  int cS[TL::PPT], cJ[TL::PPT];
  int sS = 0, sJ = 0;
#pragma unroll
  for (int j = 0; j < TL::PPT; ++j) {
    const long long p = pw + j * 32 + lane;
    cS[j] = p < np ? cnt[p] : 0;
    cJ[j] = p < np ? cnt[np + p] : 0;
    sS += cS[j];
    sJ += cJ[j];
  }
  (void)sS;
  (void)sJ;
  // warp w's 32 PPT pairs are scan slot t SLOTS_PER_TILE + w (no CTA barrier)
  const long long slot = t * SLOTS_PER_TILE + wid;
  if (slot >= npt) return;  // warp-uniform
  const long long baseS = fo.toff[slot];
  const long long baseJ = fo.toff[npt + slot];
  long long carryS = 0, carryJ = 0;
  int a, b;
  warp_pairs(pr.n, pw, a, b);
  const Seg seg = {fo.col, fo.val, fo.cap};
#pragma unroll 1
  for (int j = 0; j < TL::PPT; ++j) {
    const long long p = pw + j * 32 + lane;
    if (j) pair_advance(pr.n, a, b, 32);
    int tS, tJ;
    const int eS = warp_excl_scan(cS[j], tS), eJ = warp_excl_scan(cJ[j], tJ);
    const long long rS = baseS + carryS + eS, rJ = baseJ + carryJ + eJ;
    carryS += tS;
    carryJ += tJ;
    if (p >= np) continue;
    fo.row_ptr[p] = rS;
    fo.row_ptr[np + p] = rJ;
    if (fo.K) {
      fo.K[p] = 0.0;
      fo.K[np + p] = 0.0;
    }
    double ux[1], uy[1];
    far_values<WK, WL, PT>(pr, a, b, ux, uy);
    unsigned mr, mi;
    far_masks<WK, WL>(pr.n, pr.tau, a, b, ux, uy, mr, mi);
    const int q = pidx32(pr.n, a, b);
    // S row: [Re U at q] [-Im U at NP + q];  J row: [Im U at q] [Re U at NP + q]
    int o = 0;
    if (mr & 1u) seg.emit(rS + o++, q, ux[0]);
    if (mi & 1u) seg.emit(rS + o, (int)np + q, -uy[0]);
    o = 0;
    if (mi & 1u) seg.emit(rJ + o++, q, uy[0]);
    if (mr & 1u) seg.emit(rJ + o, (int)np + q, ux[0]);
  }
}

// Q1 rows of the warp's 32 pairs of Q0 far tile t (combined fill, Q1 = Q_H[diagonal H1], all
// pairs "far" at width 0, rows of <= 2 entries): Q1's scan slot t covers the same 256 pairs,
// so the warp's offset is the slot offset plus the counts of the tile's earlier warps.
__device__ __forceinline__ void fill_q1_chunk(const FarCtx& f1, long long npt1, long long t, const int* __restrict__ cnt1,
                                              const FillOut& fo, int2 ab, int w) {
  const int lane = threadIdx.x & 31;
  const long long np = f1.np;
  const long long p = t * TP0 + w * 32 + lane;
  const bool valid = p < np;
  // every load of the chunk issued before the first use (counts, slot offsets, the drive's
  // diagonal values), one round trip
  int a, b;  // walked again (cheaper than keeping the far tile's pair live across its staging)
  tile_pairs(f1.n, t, w, ab, a, b);
  const int c = valid ? __ldg(&cnt1[p]) : 0;  // S and J rows of a pair have the same length
  int bq[TP0 / 32 - 1];
#pragma unroll
  for (int i = 0; i < TP0 / 32 - 1; ++i) {  // the tile's earlier warps
    const long long q = t * TP0 + i * 32 + lane;
    bq[i] = (i < w && q < np) ? __ldg(&cnt1[q]) : 0;
  }
  const long long b0S = __ldg(&fo.toff[t]), b0J = __ldg(&fo.toff[npt1 + t]);
  double ux[1], uy[1];
  far_values<0, 0, 0>(f1, a, b, ux, uy);
  int before = 0;
#pragma unroll
  for (int i = 0; i < TP0 / 32 - 1; ++i) before += bq[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) before += __shfl_xor_sync(FULL, before, o);
  int tot;
  const int ex = warp_excl_scan(c, tot);
  if (!valid) return;
  const long long rS = b0S + before + ex, rJ = b0J + before + ex;
  fo.row_ptr[p] = rS;
  fo.row_ptr[np + p] = rJ;
  unsigned mr, mi;
  far_masks<0, 0>(f1.n, f1.tau, a, b, ux, uy, mr, mi);
  const Seg seg = {fo.col, fo.val, fo.cap};
  // S row: [Re U at p] [-Im U at NP + p];  J row: [Im U at p] [Re U at NP + p]
  int o = 0;
  if (mr & 1u) seg.emit(rS + o++, (int)p, ux[0]);
  if (mi & 1u) seg.emit(rS + o, (int)(np + p), -uy[0]);
  o = 0;
  if (mi & 1u) seg.emit(rJ + o++, (int)p, uy[0]);
  if (mr & 1u) seg.emit(rJ + o, (int)(np + p), ux[0]);
}

// One output matrix's arguments of the fill pass.
struct MatFill {
  Prob pr;
  const int* cnt;
  FillOut fo;
  NearSide side;
  int tile_sync;  // keep a CTA's warps on the same far tile (large outputs; see k_fill0)
  int near_sep;   // the near rows are written by k_near0 (launched before the fill), not by its units
  const DevHeader* hdr;  // with hout (sun_run of modes 0 / 2): CTA 0 stores the header prefix into
  HeaderPrefix* hout;    // mapped host memory at the start of the fill (final since the scan)
  const int2* sab;       // mode 0, Q0: first pair of each scan slot (count pass), or nullptr
  unsigned long long* wctr;  // dynamic warp-level units (SUN_FILL_DYN; DevHeader::wctr), or nullptr
};

// header prefix -> mapped pinned host memory (sun_plan_nnz reads it after the stream)
__device__ __forceinline__ void store_header(const DevHeader* h, HeaderPrefix* o, int has1) {
  o->flags = h->flags;
  o->pad = 0;
  o->nnz[0] = h->nnz[0];
  o->nnz[1] = has1 ? h->nnz[1] : 0;
  o->tau[0] = h->tau[0];
  o->tau[1] = h->tau[1];
  o->herm_dev[0] = h->herm_dev[0];
  o->herm_dev[1] = h->herm_dev[1];
  o->nrm2_h[0] = h->nrm2_h[0];
  o->nrm2_h[1] = h->nrm2_h[1];
  o->pad2 = 0u;
  // the sequence number last, after the fields are visible to the host: sun_plan_nnz returns as
  // soon as it sees it (the fill keeps running; its outputs are ordered on the stream)
  __threadfence_system();
  *reinterpret_cast<volatile unsigned*>(&o->seq) = h->seq;
}

// Fill pass of Q0 and, with Q1W >= 0, of Q1 (widths Q1W, 0, no dissipators; staging-free
// rows only, i.e. Q1W = 0) in one persistent launch: units u = blockIdx.x + k gridDim.x over
//   [Q0 near units][Q0 far tiles, last first][Q1 near][Q1 tiles]
// The next far tile's counts and offsets are loaded before the current unit runs.
template <int WK, int WL, int PT, int Q1W>
__global__ void __launch_bounds__(256, FillFar<WK, WL>::MINB) k_fill0(const MatFill m0, const MatFill m1) {
  pdl_enter();
  using FF = FillFar<WK, WL>;
  static_assert(Q1W <= 0, "combined fill: Q1 rows must be staging-free");
  extern __shared__ __align__(128) unsigned char dyn[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr bool HAS1 = Q1W >= 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    m0.fo.row_ptr[m0.pr.m] = *m0.fo.nnz;
    if (HAS1) m1.fo.row_ptr[m1.pr.m] = *m1.fo.nnz;
    if (m0.hout) store_header(m0.hdr, m0.hout, HAS1);
  }
  // near units: NEAR_UNIT_ROWS side rows each (2 per near item)
  const long long nn0 = m0.near_sep ? 0 : (2 * (m0.pr.n * 2LL * m0.pr.W + m0.pr.n - 1) + NEAR_UROWS - 1) / NEAR_UROWS;
  // Q1 tiles: none when the Q0 far tiles write Q1's rows (staged Q0 tiles of 256 pairs)
  constexpr bool Q1MERGED = HAS1 && !FF::DIRECT;
  // Q1's near items are its D rows; with the diagonal drive they are empty (count pass), so
  // their row pointers all equal nnz(Q1): CTA 0 writes them instead of near units
  const long long nn1 = HAS1 && !Q1MERGED ? near_units1(m1.pr.n, m1.pr.W) : 0;
  if (Q1MERGED && blockIdx.x == 0)
    for (long long l = threadIdx.x; l < m1.pr.n - 1; l += blockDim.x) m1.fo.row_ptr[2 * m1.pr.np + l] = *m1.fo.nnz;
  // fill tiles: SLOTS_PER_TILE scan slots (one per warp) each
  const long long nt0 = (m0.pr.npt + SLOTS_PER_TILE - 1) / SLOTS_PER_TILE;
  const long long nt1 = HAS1 && !Q1MERGED ? (m1.pr.npt + SLOTS_PER_TILE - 1) / SLOTS_PER_TILE : 0;
  const long long U0 = nt0 + nn0, U = U0 + nn1 + nt1;
  int* scol = reinterpret_cast<int*>(dyn + wid * FF::BYTES_PER_WARP);
  double* sval = reinterpret_cast<double*>(dyn + wid * FF::BYTES_PER_WARP + FF::COLW * 4);
  const FarCtx prf0{m0.pr.K.v, m0.pr.L, *m0.pr.tau_ptr, m0.pr.np, m0.pr.n, m0.pr.P};
  FarCtx prf1{};
  if (HAS1) prf1 = FarCtx{m1.pr.K.v, m1.pr.L, *m1.pr.tau_ptr, m1.pr.np, m1.pr.n, m1.pr.P};
  // unit -> kind: 0 Q0 far tile, 1 Q0 near unit, 2 Q1 near unit, 3 Q1 tile; idx
  auto decode = [&](long long v, long long& idx) -> int {
    if (v < nn0) {  // the latency-bound near units first (measured: equal at c4, faster at c2)
      idx = v;
      return 1;
    }
    if (v < U0) {
      idx = nt0 - 1 - (v - nn0);  // far tiles, last first
      return 0;
    }
    v -= U0;
    if (v < nn1) {
      idx = v;
      return 2;
    }
    idx = v - nn1;
    return 3;
  };
  TileIn nxt{0, 0, 0, 0, make_int2(-1, -1)};
  auto prefetch = [&](long long v) {
    long long idx;
    if (v < U && decode(v, idx) == 0 && !FF::DIRECT)
      nxt = load_tile_in(m0.pr.np, m0.pr.npt, idx, m0.cnt, m0.fo.toff, m0.sab, wid);
  };
#if SUN_FILL_DYN
  if constexpr (!FF::DIRECT && (Q1MERGED || !HAS1)) {
    if (m0.wctr && !m0.tile_sync) {
      // Warp-level units claimed dynamically (the SMs finished up to 9 % apart with CTA units
      // assigned round robin): near units of NEAR_RPW side rows, then the far slots (32 pairs,
      // last first); each warp's first unit is static, the next one is claimed from a global
      // counter one unit ahead (its tile inputs prefetched).  The last warp to finish resets it.
      const long long nside = 2 * (m0.pr.n * 2LL * m0.pr.W + m0.pr.n - 1);
      const long long nw0 = m0.near_sep ? 0 : (nside + NEAR_RPW - 1) / NEAR_RPW;
      const long long ns0 = nt0 * SLOTS_PER_TILE;
      const long long UW = nw0 + ns0;
      const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
      auto claim = [&]() -> long long {
        unsigned long long v = 0;
        if (lane == 0) v = atomicAdd(m0.wctr, 1ull);
        return (long long)__shfl_sync(FULL, v, 0) + nwarps;
      };
      auto slot_of = [&](long long v, long long& t, int& w) {  // v >= nw0: far slot, last first
        const long long sl = ns0 - 1 - (v - nw0);
        t = sl / SLOTS_PER_TILE;
        w = (int)(sl % SLOTS_PER_TILE);
      };
      TileIn nw{0, 0, 0, 0, make_int2(-1, -1)};
      auto wprefetch = [&](long long v) {
        if (v >= nw0 && v < UW) {
          long long t;
          int w;
          slot_of(v, t, w);
          nw = load_tile_in(m0.pr.np, m0.pr.npt, t, m0.cnt, m0.fo.toff, m0.sab, w);
        }
      };
      long long u = (long long)blockIdx.x * (blockDim.x >> 5) + wid;
      wprefetch(u);
      while (u < UW) {  // warp-uniform
        const TileIn cur = nw;
        const long long un = claim();
        wprefetch(un);
        if (u < nw0) {
#ifndef SUN_EXP_NO_NEAR
          fill_near_rows_w<false>(m0.pr, u * NEAR_RPW, m0.cnt, m0.fo, m0.side, m0.pr.inv);
#endif
        } else {
          long long t;
          int w;
          slot_of(u, t, w);
          fill_far_tile<WK, WL, PT>(prf0, m0.pr.npt, t, w, cur, m0.fo, scol, sval);
          if constexpr (Q1MERGED) fill_q1_chunk(prf1, m1.pr.npt, t, m1.cnt, m1.fo, cur.ab, w);
        }
        u = un;
      }
      if (lane == 0) {
        bulk_wait0();  // staging must outlive the bulk reads
        __threadfence();
        if (atomicAdd(m0.wctr + 1, 1ull) == (unsigned long long)nwarps - 1) {  // every claim is done
          m0.wctr[0] = 0ull;
          m0.wctr[1] = 0ull;
        }
      }
      return;
    }
  }
#endif
  prefetch(blockIdx.x);
  for (long long u = blockIdx.x; u < U; u += gridDim.x) {  // block-uniform
    const TileIn cur = nxt;
    prefetch(u + gridDim.x);
    long long idx;
    const int kind = decode(u, idx);
    if (kind == 0) {
      // Large outputs stream past L2 to DRAM: a barrier per far tile keeps the CTA's 8 warps
      // writing one contiguous ~110 KB region together (DRAM write locality; measured at
      // N = 4000-8000: +14-24 %).  Outputs that stay in L2 are faster without it (N = 1000: -3 %).
      if (m0.tile_sync) __syncthreads();
      if constexpr (FF::DIRECT)
        fill_direct_tile<WK, WL, PT>(prf0, m0.pr.npt, idx, m0.cnt, m0.fo);
      else
        fill_far_tile<WK, WL, PT>(prf0, m0.pr.npt, idx, wid, cur, m0.fo, scol, sval);
      if constexpr (Q1MERGED) fill_q1_chunk(prf1, m1.pr.npt, idx, m1.cnt, m1.fo, cur.ab, wid);
    } else if (kind == 1) {
#ifndef SUN_EXP_NO_NEAR
      fill_near_unit_h<false>(m0.pr, idx, m0.cnt, m0.fo, m0.side, m0.pr.inv);
#endif
    } else if (kind == 2) {
      if constexpr (HAS1) fill_near_unit(m1.pr, idx, m1.cnt, m1.fo, m1.side);
    } else {
      if constexpr (HAS1) fill_direct_tile<0, 0, 0>(prf1, m1.pr.npt, idx, m1.cnt, m1.fo);
    }
  }
  if (!FF::DIRECT && lane == 0) bulk_wait0();  // staging must outlive the bulk reads
}

// Near rows of a combined mode-0 plan (the near pairs' S and J rows, the D rows; K of those
// rows) in a launch of their own between the scan and the fill: latency-bound copies from the
// side buffer plus the chain tails, one wave of 8-warp CTAs at up to 64 warps per SM (inside
// the fill they ran as its first units at 16 warps per SM).
// The chain tails (up to n entries per row, tr * inv[l]) read inv[] from a shared-memory copy
// when it fits (NEAR_SMEM_INV doubles), not one dependent L2 load per entry.
constexpr int NEAR_SMEM_INV = 8192;
#ifndef SUN_SCAN_NEAR_DEFAULT
#define SUN_SCAN_NEAR_DEFAULT 0  // measured slower (c4 step 97 -> 106 us, c3 127 -> 131 us): A/B switch only
#endif
#ifndef SUN_NEAR_CONC_DEFAULT
#define SUN_NEAR_CONC_DEFAULT 0
#endif
__global__ void __launch_bounds__(256) k_near0(const MatFill m0) {
  pdl_enter();
  extern __shared__ double sinv[];
  const int n = m0.pr.n;
  if (n <= NEAR_SMEM_INV) {
    for (int l = threadIdx.x; l < n; l += blockDim.x) sinv[l] = __ldg(&m0.pr.inv[l]);
    __syncthreads();
    fill_near_unit_h<true>(m0.pr, blockIdx.x, m0.cnt, m0.fo, m0.side, sinv);
  } else {
    fill_near_unit_h<false>(m0.pr, blockIdx.x, m0.cnt, m0.fo, m0.side, m0.pr.inv);
  }
}

// ---------------------------------------------------------------------------------------
// Mode 2 (compile-time widths, many far positions: e.g. (wK, wL) = (4, 2), NPOS = 33): mode
// 0's structure (single-warp count CTAs with the near side buffer; a persistent fill with near
// units) with the warp-per-pair far path far_warp_pair (rows of ~70 entries are stored
// coalesced by the warp; no staging).  Scan slot = fill tile of TP0 pairs = 8 count warps.
// ---------------------------------------------------------------------------------------
template <int WK, int WL, int PT>
__global__ void __launch_bounds__(32) k_count2(const MatCount mc) {
  using MC = Mode0<WK, WL>;
  __shared__ double scr[MC::PER_WARP];
  const Prob& p0 = mc.pr;
  long long u = blockIdx.x;
  Prob pr = p0;
  pr.tau = *p0.tau_ptr;
  if (u < p0.nb_near) {
    count_near_item<WK, WL>(pr, u, scr, mc.cnt, mc.tsum, mc.side);
    return;
  }
  u -= p0.nb_near;  // far warp u: pairs [32 u, 32 u + 32), thread per pair
  const int lane = threadIdx.x & 31;
  const long long np = pr.np;
  const long long pw = u * 32;
  int a, b;
  warp_pairs(pr.n, pw, a, b);
  const long long p = pw + lane;
  int tot = 0;
  if (p < np && b - a > 2 * MC::W) {
    // the positions one by one with the fill's per-position expression (far_value_at)
    int nR = 0, nI = 0;
#pragma unroll
    for (int k = 0; k < FarT<WK, WL>::NPOS; ++k) {  // compile-time positions (decode folded away)
      double x, y;
      int c, d;
      if (far_value_at<WK, WL, PT>(pr, a, b, k, x, y, c, d)) {
        nR += fabs(x) > pr.tau;
        nI += fabs(y) > pr.tau;
      }
    }
    tot = nR + nI;
    mc.cnt[p] = tot | (nR << CNT_BITS);
    mc.cnt[np + p] = tot;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(FULL, tot, o);
  if (lane == 0 && tot) {  // scan slot u = this warp's 32 pairs
    atomicAdd(&mc.tsum[u], tot);
    atomicAdd(&mc.tsum[pr.npt + u], tot);
  }
}

template <int WK, int WL, int PT>
__device__ __forceinline__ void fill2_far_tile(const Prob& pr, long long t, const int* __restrict__ cnt,
                                               const FillOut& fo) {
  using MC = Mode0<WK, WL>;
  const int wid = threadIdx.x >> 5;
  const long long np = pr.np;
  const long long p = t * TP0 + threadIdx.x;
  const long long slot = t * SLOTS_PER_TILE + wid;  // the warp's 32 pairs (no CTA barrier)
  if (slot >= pr.npt) return;                       // warp-uniform
  const bool valid = p < np;
  const int w = valid ? cnt[p] : 0;
  const int cS = w & CNT_MASK, cJ = valid ? cnt[np + p] : 0;
  int2 ex2, tot2;
  ex2.x = warp_excl_scan(cS, tot2.x);
  ex2.y = warp_excl_scan(cJ, tot2.y);
  const long long baseS = fo.toff[slot], baseJ = fo.toff[pr.npt + slot];
  int a, b;
  warp_pairs(pr.n, t * TP0 + wid * 32, a, b);
  const bool far = valid && (b - a > 2 * MC::W);
  if (valid) {
    fo.row_ptr[p] = baseS + ex2.x;
    fo.row_ptr[np + p] = baseJ + ex2.y;
    if (fo.K && far) {
      fo.K[p] = 0.0;
      fo.K[np + p] = 0.0;
    }
  }
  const Seg seg = {fo.col, fo.val, fo.cap};
  // the warp's 32 pairs, one after the other (lane-parallel positions)
  const unsigned farmask = __ballot_sync(FULL, far);
  for (int j = 0; j < 32; ++j) {
    if (!((farmask >> j) & 1u)) continue;  // warp-uniform
    const int aj = __shfl_sync(FULL, a, j), bj = __shfl_sync(FULL, b, j);
    const int oS = __shfl_sync(FULL, ex2.x, j), oJ = __shfl_sync(FULL, ex2.y, j);
    far_warp_pair<WK, WL, PT, true>(pr, aj, bj, seg, baseS + oS, seg, baseJ + oJ);
  }
}

template <int WK, int WL, int PT>
__global__ void __launch_bounds__(256) k_fill2(const MatFill mf) {
  __shared__ NearRowP nrows[8][NEAR_WARP_ROWS];
  const Prob& p0 = mf.pr;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    mf.fo.row_ptr[p0.m] = *mf.fo.nnz;
    if (mf.hout) store_header(mf.hdr, mf.hout, 0);
  }
  Prob pr = p0;
  pr.tau = *p0.tau_ptr;
  const long long nn = near_units(p0.n, p0.W);
  const long long nt = (p0.npt + SLOTS_PER_TILE - 1) / SLOTS_PER_TILE, U = nt + nn;
  for (long long u = blockIdx.x; u < U; u += gridDim.x) {  // block-uniform: near units first
    const bool nearu = u < nn;
    const long long idx = nearu ? u : u - nn;
    if (nearu) {
      fill_near_unit_b(pr, idx, mf.cnt, mf.fo, mf.side, nrows[threadIdx.x >> 5]);
    } else {
      fill2_far_tile<WK, WL, PT>(pr, nt - 1 - idx, mf.cnt, mf.fo);
    }
  }
}

// ---------------------------------------------------------------------------------------
// Mode 1 (runtime widths): warp per pair, far positions from a table in shared memory.
// Tiles of WARP_TP pairs (S and J), then D tiles of 8 rows.  Sole owner of each slot.
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

// FK >= 0: compile-time far path far_warp_pair<FK, FL, PT> (else the runtime position table)
template <int FK, int FL, int PT>
__device__ __forceinline__ int mode1_far(const Prob& pr, int a, int b, const int* pos_dc, const int* pos_dd, int npos,
                                         const Seg& sS, long long offS, const Seg& sJ, long long offJ, int* nR_out,
                                         int nR_known, int total_known, bool emit) {
  if constexpr (FK >= 0) {
    if (emit) return far_warp_pair<FK, FL, PT, true>(pr, a, b, sS, offS, sJ, offJ, nR_out);
    return far_warp_pair<FK, FL, PT, false>(pr, a, b, sS, offS, sJ, offJ, nR_out);
  } else {
    if (emit)
      return warp_far_pair<true>(pr, a, b, pos_dc, pos_dd, npos, sS, offS, sJ, offJ, nR_out, nR_known, total_known);
    return warp_far_pair<false>(pr, a, b, pos_dc, pos_dd, npos, sS, offS, sJ, offJ, nR_out);
  }
}

template <int FK, int FL, int PT>
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
    int c1, c2, nR = 0;
    if (b - a > 2 * pr.W) {
      c1 = c2 = mode1_far<FK, FL, PT>(pr, a, b, spos_dc, spos_dd, npos_far, none, 0, none, 0, &nR, -1, 0, false);
    } else {
      double k1, k2;
      warp_near_pair<false, 0, SW>(pr, a, b, scr[wid], c1, c2, k1, k2, none, 0, none, 0);
    }
    if (lane == 0) {
      cnt[p] = c1 | (nR << CNT_BITS);
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

template <int NTHREADS>
__device__ __forceinline__ void fill_d_tile(const Prob& pr, const FillOut& fo, long long t, const int* cnt,
                                            double* scr_w, int* wtot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const long long np = pr.np;
  const long long u = t - pr.npt;
  const long long baseD = fo.toff[2 * pr.npt + u];
  const int lam = (int)(u * (NTHREADS / 32) + wid + 1);
  const bool valid = lam <= pr.n - 1;
  const int c = valid ? cnt[2 * np + lam - 1] : 0;
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

template <int FK, int FL, int PT>
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
  const int cS = valid ? (cnt[p0] & CNT_MASK) : 0, cJ = valid ? cnt[np + p0] : 0;
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
      const int w = cnt[p];  // row length and nR from the count pass: emit in one pass
      mode1_far<FK, FL, PT>(pr, a, b, spos_dc, spos_dd, npos_far, sS, soffS[i], sJ, soffJ[i], nullptr, w >> CNT_BITS,
                            w & CNT_MASK, true);
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

// ---------------------------------------------------------------------------------------
// (a4) exclusive scan of the int32 tile sums of both matrices (blockIdx.y) into int64 tile
// offsets and nnz, in one launch: chained scan with decoupled look-back.  Chunks are taken
// in ticket order, so every predecessor of a running chunk is resident or done.  Integer
// sums: the result does not depend on the order (deterministic).
// ---------------------------------------------------------------------------------------
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

struct ScanArgs {
  const int* ts[2];
  long long* toff[2];
  unsigned long long* status[2];
  long long* nnz[2];
  long long nslots[2];
  unsigned int* ticket;
  const DevHeader* hdr;  // with hout: the header prefix is also stored in mapped host memory
  HeaderPrefix* hout;    // (sun_plan_nnz then reads it after the stream; no copy node)
  int direct;            // few chunks: every CTA sums the slots before its chunk itself (no chain)
};
// Up to this many chunks per matrix a chunk's CTA computes its own prefix: it re-reads the slot sums
// before its chunk (at most SCAN_DIRECT_MAX x 4 KB, from L2, all loads independent) instead of
// waiting on its predecessors' status words (one dependent L2 round trip per link of the chain).
// Integer sums: bit-identical.
#ifndef SUN_SCAN_DIRECT_MAX
#define SUN_SCAN_DIRECT_MAX 16  // measured: 3 chunks (c2) step 41.9 -> 40.2 us, 9 chunks (c3) equal, 32 chunks (c4) scan 6.7 -> 8.0 us
#endif

// One chunk (SCAN_TILE slots) of matrix y's chained scan by the whole CTA.  done: when not null,
// done[chunk] is set once the chunk's offsets are in toff (k_scan_near0's near units wait on it).
__device__ __forceinline__ void scan_chunk(const ScanArgs& A, int y, long long chunk, int ny, long long* wsum,
                                           long long& prefix_s, unsigned long long* done) {
  const long long nslots = A.nslots[y];
  const long long nchunks = (nslots + SCAN_TILE - 1) / SCAN_TILE;
  if (chunk >= (nchunks > 0 ? nchunks : 1)) return;  // block-uniform
  const long long c0 = chunk * SCAN_TILE + (long long)threadIdx.x * SCAN_IPT;
  const int* ts = A.ts[y];
  int v[SCAN_IPT];
  if (c0 + SCAN_IPT <= nslots) {
#pragma unroll
    for (int i = 0; i < SCAN_IPT; i += 4) {
      const int4 q = *reinterpret_cast<const int4*>(ts + c0 + i);  // 16-byte aligned (c0 % 4 == 0)
      v[i] = q.x; v[i + 1] = q.y; v[i + 2] = q.z; v[i + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < SCAN_IPT; ++i) v[i] = c0 + i < nslots ? ts[c0 + i] : 0;
  }
  long long pre = 0;
  if (A.direct) {  // the slots before this chunk (chunk * SCAN_TILE of them: whole int4s)
    const int4* p4 = reinterpret_cast<const int4*>(ts);
    const long long n4 = chunk * (SCAN_TILE / 4);
#pragma unroll 4
    for (long long i = threadIdx.x; i < n4; i += SCAN_THREADS) {
      const int4 q = __ldcg(p4 + i);
      pre += (long long)q.x + q.y + q.z + q.w;
    }
  }
  long long local = 0;
#pragma unroll
  for (int i = 0; i < SCAN_IPT; ++i) local += v[i];
  long long total;
  const long long ex = block_scan_ll(local, wsum, total);
  long long pre_total = 0;
  if (A.direct) block_scan_ll(pre, wsum, pre_total);
  unsigned long long* st = A.status[y];
  if (threadIdx.x < 32) {  // warp 0: publish the aggregate, then a warp-parallel look-back
    const int lane = threadIdx.x;
    long long prefix = 0;
    if (A.direct) {
      prefix = pre_total;
    } else if (chunk == 0) {
      if (lane == 0) {
        __threadfence();
        atomicExch(&st[0], SCAN_P | (unsigned long long)total);
      }
    } else {
      if (lane == 0) {
        __threadfence();
        atomicExch(&st[chunk], SCAN_A | (unsigned long long)total);
      }
      // lanes read 32 predecessors at once (lane 0 = the closest); the window ends at the
      // closest inclusive prefix (P), aggregates (A) before it are summed
      for (long long khi = chunk - 1;; khi -= 32) {
        const long long k = khi - lane;
        const volatile unsigned long long* vst = st;
        unsigned long long s = k >= 0 ? vst[k] : SCAN_P;  // beyond chunk 0: an empty P
        while (__any_sync(FULL, (s & ~SCAN_V) == 0ull))
          if ((s & ~SCAN_V) == 0ull) s = vst[k];
        const unsigned pmask = __ballot_sync(FULL, (s & ~SCAN_V) == SCAN_P);
        const int lim = pmask ? __ffs(pmask) - 1 : 31;
        long long part = lane <= lim ? (long long)(s & SCAN_V) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(FULL, part, o);
        prefix += part;
        if (pmask) break;
      }
      if (lane == 0) {
        __threadfence();
        atomicExch(&st[chunk], SCAN_P | (unsigned long long)(prefix + total));
      }
    }
    if (lane == 0) {
      prefix_s = prefix;
      if (chunk == nchunks - 1 || nchunks == 0) {
        *A.nnz[y] = prefix + total;
        if (A.hout) A.hout->nnz[y] = prefix + total;
      }
      if (A.hout && y == 0 && chunk == 0) {  // the rest of the prefix is final (expand / count kernels)
        const DevHeader* h = A.hdr;
        A.hout->flags = h->flags;
        A.hout->pad = 0;
        A.hout->tau[0] = h->tau[0];
        A.hout->tau[1] = h->tau[1];
        A.hout->herm_dev[0] = h->herm_dev[0];
        A.hout->herm_dev[1] = h->herm_dev[1];
        A.hout->nrm2_h[0] = h->nrm2_h[0];
        A.hout->nrm2_h[1] = h->nrm2_h[1];
        if (ny == 1) A.hout->nnz[1] = 0;
      }
    }
  }
  __syncthreads();
  long long run = prefix_s + ex;
  long long o[SCAN_IPT];
#pragma unroll
  for (int i = 0; i < SCAN_IPT; ++i) {
    o[i] = run;
    run += v[i];
  }
  long long* out = A.toff[y];
  if (c0 + SCAN_IPT <= nslots) {
#pragma unroll
    for (int i = 0; i < SCAN_IPT; i += 2) reinterpret_cast<longlong2*>(out + c0)[i / 2] = make_longlong2(o[i], o[i + 1]);
  } else {
#pragma unroll
    for (int i = 0; i < SCAN_IPT; ++i)
      if (c0 + i < nslots) out[c0 + i] = o[i];
  }
  if (done) {  // publish: every thread's offsets before the flag
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) atomicExch(&done[chunk], 1ull);
  }
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_chain(ScanArgs A) {
  pdl_enter();
  const int y = blockIdx.y;
  __shared__ unsigned int chunk_s;
  __shared__ long long wsum[32];
  __shared__ long long prefix_s;
  if (threadIdx.x == 0) chunk_s = A.direct ? blockIdx.x : atomicAdd(&A.ticket[y], 1u);
  __syncthreads();
  scan_chunk(A, y, chunk_s, (int)gridDim.y, wsum, prefix_s, nullptr);
}

// (a4) + the near rows of (a5) in one launch (sun_run on a combined mode-0 plan: the outputs are
// known when the scan is enqueued).  CTAs take roles in ticket order: the first nch0 + nch1
// tickets are the scan chunks of Q0 and Q1 (every scan CTA is resident before any near CTA takes
// a ticket, and never waits on one), the rest are near units of NEAR_UROWS side rows.  A near
// warp issues everything that does not depend on the scan (inv[] copy, metadata, the slot's
// earlier counts) and then waits for its slot's chunk to be published, so the near rows' lookup
// chains run under the scan's look-back chain instead of after it.
struct ScanNearArgs {
  ScanArgs sa;
  long long nch[2];                  // scan chunks of Q0, Q1 (0: no Q1)
  const unsigned long long* done0;   // Q0's per-chunk "offsets written" flags
  unsigned long long* done[2];
};
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_near0(const ScanNearArgs A, const MatFill m0) {
  static_assert(SCAN_THREADS == 256, "near units: 8 warps");
  extern __shared__ double sinv[];
  __shared__ unsigned int ticket_s;
  __shared__ long long wsum[32];
  __shared__ long long prefix_s;
  if (threadIdx.x == 0) ticket_s = atomicAdd(&A.sa.ticket[0], 1u);
  __syncthreads();
  const long long t = ticket_s;
  const int ny = A.nch[1] > 0 ? 2 : 1;
  if (t < A.nch[0]) {
    scan_chunk(A.sa, 0, t, ny, wsum, prefix_s, A.done[0]);
    return;
  }
  if (t < A.nch[0] + A.nch[1]) {
    scan_chunk(A.sa, 1, t - A.nch[0], ny, wsum, prefix_s, nullptr);
    return;
  }
  const long long j = t - A.nch[0] - A.nch[1];
  const int n = m0.pr.n;
  if (n <= NEAR_SMEM_INV) {
    for (int l = threadIdx.x; l < n; l += blockDim.x) sinv[l] = __ldg(&m0.pr.inv[l]);
    __syncthreads();
    fill_near_rows_w<true>(m0.pr, j * NEAR_UROWS + (threadIdx.x >> 5) * NEAR_RPW, m0.cnt, m0.fo, m0.side, sinv, A.done0);
  } else {
    fill_near_rows_w<false>(m0.pr, j * NEAR_UROWS + (threadIdx.x >> 5) * NEAR_RPW, m0.cnt, m0.fo, m0.side, m0.pr.inv,
                            A.done0);
  }
}

// (a7) dv/dt = Q0 v + eps Q1 v + K as a streamed CSR product.  A CTA owns R consecutive rows (R
// chosen by the host from the mean row length so that a block holds about two tiles of entries;
// the last row blocks, the long D rows, are scheduled first), reads their entries (col, val) as
// one contiguous, fully coalesced stream in tiles of APPLY_TILE entries (the next tile's loads in
// flight during the current tile's sums), gathers x (8 MB at N = 1000: L2 resident) and leaves
// the products in shared memory.  The rows that intersect the tile (binary search in the staged
// row pointers) are then summed by G = 256 / rows lanes each (a power of two <= 32), lane-strided
// with a fixed shuffle tree; a row with more than APPLY_LONG G entries in the tile (a near row's
// D-chain tail among short rows) is summed by its whole warp.  Blocks whose rows average <= 32
// entries skip the search: thread t sums row t in entry order (long segments by the warp).  Every
// order is fixed: the result is deterministic.  The 8-lanes-per-row kernel this replaces read col/val in 32- and 64-byte
// pieces per row (120 us at c4, 0.33 of HBM).
#ifndef SUN_APPLY_TILE
#define SUN_APPLY_TILE 2048
#endif
constexpr int APPLY_THREADS = 256, APPLY_TILE = SUN_APPLY_TILE, APPLY_LONG = 64;
// number of i in [0, n) with a[i] < key (strict = true) or a[i] <= key; a ascending (shared memory)
__device__ __forceinline__ int apply_count_below(const long long* a, int n, long long key, bool strict) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const long long x = a[mid];
    if (strict ? x < key : x <= key)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}
// The sums of one tile: prod holds the products of entries [e0, e0 + APPLY_TILE) (0 outside the
// block).  simple: thread t adds row t's part to acc1; else the intersecting rows' parts go to racc.
__device__ __forceinline__ void apply_tile_sums(const long long* rp_s, int nrows, long long e0, const double* prod,
                                                bool simple, long long rs, long long re, double& acc1, double* racc) {
  const int tid = threadIdx.x, lane = tid & 31;
  const long long t1 = e0 + APPLY_TILE;
  if (simple) {  // short rows: thread t sums row t in entry order, long segments by the warp
    const int lo = (int)((rs > e0 ? rs : e0) - e0), hi = (int)((re < t1 ? re : t1) - e0);  // hi <= lo: none here
    const bool lng = hi - lo > APPLY_LONG;
    unsigned lm = __ballot_sync(FULL, lng);
    double part = 0.0;
    if (!lng)
      for (int k = lo; k < hi; ++k) part += prod[k];
    while (lm) {  // warp-uniform
      const int src = __ffs(lm) - 1;
      lm &= lm - 1;
      const int l = __shfl_sync(FULL, lo, src), h = __shfl_sync(FULL, hi, src);
      double t = 0.0;
      for (int k = l + lane; k < h; k += 32) t += prod[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(FULL, t, o);
      if (lane == src) part = t;
    }
    acc1 += part;
    return;
  }
  // rows [rcur, rend) intersect the tile (empty rows among them are harmless)
  int rcur = apply_count_below(rp_s, nrows + 1, e0, false) - 1;
  if (rcur < 0) rcur = 0;
  const int rend = apply_count_below(rp_s, nrows, t1, true);
  const int nint = rend - rcur;
  int G = 1;
  while (G < 32 && 2 * G * nint <= APPLY_THREADS) G <<= 1;  // 256 / G >= nint: one row per group
  const int g = tid / G, gl = tid & (G - 1), r = rcur + g;
  const bool valid = g < nint;
  int lo = 0, hi = 0;
  if (valid) {
    const long long a = rp_s[r], b = rp_s[r + 1];
    lo = (int)((a > e0 ? a : e0) - e0);
    hi = (int)((b < t1 ? b : t1) - e0);
  }
  const bool lng = hi - lo > APPLY_LONG * G;
  double part = 0.0;
  if (!lng) {
#pragma unroll 4
    for (int k = lo + gl; k < hi; k += G) part += prod[k];
  }
  unsigned lm = __ballot_sync(FULL, lng && gl == 0);
  while (lm) {  // warp-uniform: the long rows of this warp's groups, one after the other
    const int src = __ffs(lm) - 1;
    lm &= lm - 1;
    const int l = __shfl_sync(FULL, lo, src), h = __shfl_sync(FULL, hi, src);
    double t = 0.0;
#pragma unroll 4
    for (int k = l + lane; k < h; k += 32) t += prod[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(FULL, t, o);
    if (lane == src) part = t;  // the group's other lanes hold 0
  }
  for (int o = G >> 1; o > 0; o >>= 1) part += __shfl_xor_sync(FULL, part, o);
  if (valid && gl == 0) racc[r] += part;  // one group per row and tile; tiles in ascending order
}

__device__ __forceinline__ double apply_stream_rows(const long long* rp_s, int nrows, const int32_t* __restrict__ col,
                                                    const double* __restrict__ val, const double* __restrict__ x,
                                                    double* prod, double* racc) {
  const int tid = threadIdx.x;
  const long long eb = rp_s[0], ee = rp_s[nrows];
  // a block whose rows average <= 32 entries: thread t owns row t (no search, no row accumulators)
  const bool simple = ee - eb <= 32LL * nrows;
  const long long rs = tid < nrows ? rp_s[tid] : ee, re = tid < nrows ? rp_s[tid + 1] : ee;
  double acc1 = 0.0;
  racc[tid] = 0.0;  // ordered before its first use by the tile loop's barrier
  constexpr int IPT = APPLY_TILE / APPLY_THREADS;
  int c[IPT];
  double v[IPT];
  auto load_tile = [&](long long e0) {  // the tile's entries, lane-contiguous (coalesced), streaming
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
      const long long k = e0 + i * APPLY_THREADS + tid;
      const bool in = k >= eb && k < ee;
      c[i] = in ? __ldcs(col + k) : 0;
      v[i] = in ? __ldcs(val + k) : 0.0;
    }
  };
  const long long e00 = eb - (eb & 31);
  if (e00 < ee) load_tile(e00);
  for (long long e0 = e00; e0 < ee; e0 += APPLY_TILE) {  // block-uniform
#pragma unroll
    for (int i = 0; i < IPT; ++i) prod[i * APPLY_THREADS + tid] = v[i] * __ldg(&x[c[i]]);
    __syncthreads();
    const long long t1 = e0 + APPLY_TILE;
    if (t1 < ee) load_tile(t1);  // in flight during this tile's sums
    apply_tile_sums(rp_s, nrows, e0, prod, simple, rs, re, acc1, racc);
    __syncthreads();
  }
  __syncthreads();
  const double acc = simple ? acc1 : racc[tid];
  __syncthreads();
  return acc;
}

// Tried and removed (measured on B200, same box): the entry tiles brought in by TMA 1D bulk loads
// (cp.async.bulk.shared.global on an mbarrier, a two-stage shared-memory ring, products in place):
// c4 82.0 us with either kernel, c3 121 us against 86 us.  ncu shows why the loads are not the
// limiter: the L1 data pipe (shared-memory product stores and reads plus the gathers' wavefronts)
// is the busiest unit at 65 % of peak, L2 at 30 %, DRAM below that.
#ifndef SUN_APPLY_MINB
#define SUN_APPLY_MINB 4
#endif
__global__ void __launch_bounds__(APPLY_THREADS, SUN_APPLY_MINB) k_apply(long long m, int R, const int64_t* __restrict__ rp0,
                                                         const int32_t* __restrict__ c0, const double* __restrict__ v0,
                                                         const int64_t* __restrict__ rp1, const int32_t* __restrict__ c1,
                                                         const double* __restrict__ v1, double eps,
                                                         const double* __restrict__ Kv, const double* __restrict__ x,
                                                         double* __restrict__ y) {
  __shared__ double prod[APPLY_TILE];
  __shared__ double racc[APPLY_THREADS];
  __shared__ long long rp_s[2][APPLY_THREADS + 1];
  const long long r0 = (long long)(gridDim.x - 1 - blockIdx.x) * R;  // last rows (the D rows: the longest) first
  const int nrows = (int)(m - r0 < R ? m - r0 : R);
  const int tid = threadIdx.x;
  for (int i = tid; i <= nrows; i += APPLY_THREADS) {
    rp_s[0][i] = rp0[r0 + i];
    if (rp1) rp_s[1][i] = rp1[r0 + i];
  }
  const double kv = Kv && tid < nrows ? Kv[r0 + tid] : 0.0;
  __syncthreads();
  const double s0 = apply_stream_rows(rp_s[0], nrows, c0, v0, x, prod, racc);
  double s1 = 0.0;
  if (rp1) s1 = apply_stream_rows(rp_s[1], nrows, c1, v1, x, prod, racc);
  if (tid < nrows) y[r0 + tid] = s0 + eps * s1 + kv;
}

// ---------------------------------------------------------------------------------------
// Propagation (F1) and states (F2)
// ---------------------------------------------------------------------------------------
// One RK4 stage: y = Q0 x + eps Q1 x + K with x = v + c kp (formed in the gather; kp = NULL:
// x = v).  Rows of Q0 with at most RK4_LONG entries: one thread per row, entries in order,
// four independent entries in flight per round; longer rows (the D-chain rows): one warp per
// row from a list, fixed-order tree reduction.  Epilogue by `mode`:
//   0: kout = y, acc = y        1: kout = y, acc += 2 y        2: vout = v + h6 (acc + y)
constexpr int RK4_LONG = 64;
struct Rk4Stage {
  const int64_t* rp0;
  const int32_t* c0;
  const double* v0;
  const int64_t* rp1;
  const int32_t* c1;
  const double* v1;
  const double* K;
  const double* v;
  const double* kp;
  double* kout;
  double* acc;
  double* vout;
  const int* longrows;
  double eps, c, h6;
  long long m;
  int nlong, nshort_blocks, mode;
};

__device__ __forceinline__ double rk4_x(const Rk4Stage& S, int j) {
  return S.kp ? __ldg(&S.v[j]) + S.c * __ldg(&S.kp[j]) : __ldg(&S.v[j]);
}

__device__ __forceinline__ void rk4_epilogue(const Rk4Stage& S, long long row, double y) {
  if (S.mode == 0) {
    S.kout[row] = y;
    S.acc[row] = y;
  } else if (S.mode == 1) {
    S.kout[row] = y;
    S.acc[row] += 2.0 * y;
  } else {
    S.vout[row] = S.v[row] + S.h6 * (S.acc[row] + y);
  }
}

__global__ void __launch_bounds__(256) k_rk4_stage(const Rk4Stage S) {
  if ((int)blockIdx.x < S.nshort_blocks) {
    const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= S.m) return;
    const int64_t b0 = S.rp0[row], e0 = S.rp0[row + 1];
    if (e0 - b0 > RK4_LONG) return;  // a warp of the long-row part does this row
    double s0 = 0.0;
    int64_t k = b0;
    for (; k + 4 <= e0; k += 4) {
      const int j0 = __ldg(&S.c0[k]), j1 = __ldg(&S.c0[k + 1]), j2 = __ldg(&S.c0[k + 2]), j3 = __ldg(&S.c0[k + 3]);
      const double a0 = __ldg(&S.v0[k]), a1 = __ldg(&S.v0[k + 1]), a2 = __ldg(&S.v0[k + 2]), a3 = __ldg(&S.v0[k + 3]);
      const double x0 = rk4_x(S, j0), x1 = rk4_x(S, j1), x2 = rk4_x(S, j2), x3 = rk4_x(S, j3);
      s0 += a0 * x0;
      s0 += a1 * x1;
      s0 += a2 * x2;
      s0 += a3 * x3;
    }
    for (; k < e0; ++k) s0 += __ldg(&S.v0[k]) * rk4_x(S, __ldg(&S.c0[k]));
    double s1 = 0.0;
    if (S.rp1)
      for (int64_t q = S.rp1[row]; q < S.rp1[row + 1]; ++q) s1 += __ldg(&S.v1[q]) * rk4_x(S, __ldg(&S.c1[q]));
    rk4_epilogue(S, row, s0 + S.eps * s1 + (S.K ? S.K[row] : 0.0));
    return;
  }
  const int lane = threadIdx.x & 31;
  const long long w = (long long)(blockIdx.x - S.nshort_blocks) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= S.nlong) return;  // warp-uniform
  const long long row = S.longrows[w];
  double s0 = 0.0, s1 = 0.0;
  const int64_t e0 = S.rp0[row + 1];
#pragma unroll 4
  for (int64_t k = S.rp0[row] + lane; k < e0; k += 32) s0 += __ldg(&S.v0[k]) * rk4_x(S, __ldg(&S.c0[k]));
  if (S.rp1)
    for (int64_t q = S.rp1[row] + lane; q < S.rp1[row + 1]; q += 32) s1 += __ldg(&S.v1[q]) * rk4_x(S, __ldg(&S.c1[q]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(FULL, s0, o);
    s1 += __shfl_xor_sync(FULL, s1, o);
  }
  if (lane == 0) rk4_epilogue(S, row, s0 + S.eps * s1 + (S.K ? S.K[row] : 0.0));
}

// ---------------------------------------------------------------------------------------
// F1, matrix-free (sun_rk4_plan): one RK4 stage y = (Q0 + eps Q1) x + K with x = v + c k_prev,
// Q0 and Q1 never read from memory.  Far pairs: thread per pair, the U values regenerated from
// the band storage exactly as the count / fill passes do (same expressions, same tau masks), so
// each stored entry of Q0 is reproduced bit for bit.  Near-pair and D rows: warp per side row,
// window entries from the count pass's side buffer, the chain tail sum_l tr inv[l] x_{D^l} in
// O(1) from the prefix P[l] = sum_{l' <= l} inv[l'] x_{D^l'} (k_mf_prefix, one CTA per stage).
// Q1: a diagonal drive only (Q1 = Q_H[H1] couples S_ab and J_ab), from the H1 band.  Mode 0.
// ---------------------------------------------------------------------------------------
struct MfStage {
  Prob p0, p1;        // Q0 and (has1) Q1 problems of the plan
  NearSide side;      // Q0 side buffer (count pass)
  int has1;
  const double* pref; // [n]
  double* pref_out;
  const double* x;    // this stage's input (v, v + h/2 k1, v + h/2 k2, v + h k3)
  double* xn;         // the next stage's input, written by the epilogue (stages 1-3)
  const double* v;
  double* acc;
  double* vout;
  double eps, cn, h6; // cn: the next stage's step (h/2, h/2, h)
  long long m;
  int mode, nfar_blocks;
};

__device__ __forceinline__ double mf_x(const MfStage& S, long long j) { return __ldg(&S.x[j]); }
// stage k_i = y: acc = k1 / acc += 2 k_i, and the next input v + cn k_i; or the RK4 update
__device__ __forceinline__ void mf_epilogue(const MfStage& S, long long row, double y) {
  if (S.mode == 0) {
    S.acc[row] = y;
    S.xn[row] = S.v[row] + S.cn * y;
  } else if (S.mode == 1) {
    S.acc[row] += 2.0 * y;
    S.xn[row] = S.v[row] + S.cn * y;
  } else if (S.mode == 2) {
    S.vout[row] = S.v[row] + S.h6 * (S.acc[row] + y);
  } else {  // 3: plain apply, vout = y
    S.vout[row] = y;
  }
}

__global__ void __launch_bounds__(1024) k_mf_prefix(const MfStage S) {
  __shared__ double wsum[32];
  __shared__ double carry_s;
  const int n = S.p0.n;
  const long long dcol = 2 * S.p0.np - 1;  // column of D^l = dcol + l
  if (threadIdx.x == 0) carry_s = 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base < n; base += blockDim.x) {
    const int l = base + threadIdx.x;
    const double w = (l >= 1 && l < n) ? S.p0.inv[l] * mf_x(S, dcol + l) : 0.0;
    double x = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      double t = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0.0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(FULL, t, o);
        if (lane >= o) t += y;
      }
      wsum[lane] = t;
    }
    __syncthreads();
    const double incl = carry_s + (wid > 0 ? wsum[wid - 1] : 0.0) + x;
    if (l < n) S.pref_out[l] = incl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry_s = incl;
    __syncthreads();
  }
}

// Q1 = Q_H[diagonal H1] on the rows S_ab (half 0) / J_ab (half 1): U1 at (a, b) only
__device__ __forceinline__ double mf_q1(const MfStage& S, const FarCtx& f1, int a, int b, long long p, int half) {
  double ux[1], uy[1];
  far_values<0, 0, 0>(f1, a, b, ux, uy);
  unsigned mr, mi;
  far_masks<0, 0>(f1.n, f1.tau, a, b, ux, uy, mr, mi);
  const long long np = f1.np;
  const double xs = mf_x(S, p), xj = mf_x(S, np + p);
  // S row: [Re U at p] [-Im U at NP + p];  J row: [Im U at p] [Re U at NP + p]
  if (half == 0) return ((mr & 1u) ? ux[0] * xs : 0.0) + ((mi & 1u) ? -uy[0] * xj : 0.0);
  return ((mi & 1u) ? uy[0] * xs : 0.0) + ((mr & 1u) ? ux[0] * xj : 0.0);
}

template <int WK, int WL, int PT>
__global__ void __launch_bounds__(256) k_mf_stage(const MfStage S) {
  using MC = Mode0<WK, WL>;
  constexpr int NPOS = FarT<WK, WL>::NPOS;
  const int lane = threadIdx.x & 31;
  const long long np = S.p0.np;
  const FarCtx f0{S.p0.K.v, S.p0.L, *S.p0.tau_ptr, np, S.p0.n, S.p0.P};
  FarCtx f1{};
  if (S.has1) f1 = FarCtx{S.p1.K.v, S.p1.L, *S.p1.tau_ptr, np, S.p1.n, 0};
  if ((int)blockIdx.x < S.nfar_blocks) {  // far pairs, thread per pair
    const long long p0w = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
    if (p0w >= np) return;  // warp-uniform
    int a, b;
    warp_pairs(S.p0.n, p0w, a, b);
    const long long p = p0w + lane;
    if (p >= np || b - a <= 2 * MC::W) return;  // near pairs: the side-row part
    double ux[NPOS], uy[NPOS];
    far_values<WK, WL, PT>(f0, a, b, ux, uy);
    int q[NPOS];
    far_cols<WK, WL>(f0.n, a, b, q);
    double yS = 0.0, yJ = 0.0;
    // kept entries as in far_masks (in range and |.| > tau), inline: NPOS may exceed 32
    far_foreach<WK, WL>([&](int k, int dc, int dd) {
      const bool ok = (dc >= 0 || a + dc >= 0) && (dd <= 0 || b + dd < f0.n);
      const bool kr = ok && fabs(ux[k]) > f0.tau, ki = ok && fabs(uy[k]) > f0.tau;
      const double xs = (kr || ki) ? mf_x(S, q[k]) : 0.0;
      const double xj = (kr || ki) ? mf_x(S, np + q[k]) : 0.0;
      if (kr) {
        yS += ux[k] * xs;
        yJ += ux[k] * xj;
      }
      if (ki) {
        yS -= uy[k] * xj;
        yJ += uy[k] * xs;
      }
    });
    if (S.has1) {
      yS += S.eps * mf_q1(S, f1, a, b, p, 0);
      yJ += S.eps * mf_q1(S, f1, a, b, p, 1);
    }
    mf_epilogue(S, p, yS);  // K = 0 on far rows
    mf_epilogue(S, np + p, yJ);
    return;
  }
  // side rows (near pairs' S / J rows, D rows), warp per row
  const long long srow = (long long)(blockIdx.x - S.nfar_blocks) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long nside = 2 * ((long long)S.p0.n * 2 * S.p0.W + S.p0.n - 1);
  if (srow >= nside) return;  // warp-uniform
  int a, b, lam;
  const int half = (int)(srow & 1);
  const int kind = near_item(S.p0, srow >> 1, a, b, lam);
  if (kind == 0 || (kind == 2 && half)) return;
  const NearMeta mt = S.side.meta[srow];
  const int32_t* sc = S.side.col + srow * S.side.nc;
  const double* sv = S.side.val + srow * S.side.nc;
  const int nwin = mt.n1 + mt.n2 + mt.nd, b2 = mt.n1 + mt.n2;
  double y = 0.0;
  for (int k = lane; k < nwin; k += 32) {
    const int sidx = k < mt.n1 ? k : (k < b2 ? S.side.seg + (k - mt.n1) : 2 * S.side.seg + (k - b2));
    y += __ldg(&sv[sidx]) * mf_x(S, __ldg(&sc[sidx]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(FULL, y, o);
  if (lane == 0) {
    if (mt.lend > mt.hi) y += mt.tr * (S.pref[mt.lend] - S.pref[mt.hi]);  // chain tail l in (hi, lend]
    y += mt.k;
    long long row;
    if (kind == 1) {
      const long long p = (long long)pidx32(S.p0.n, a, b);
      row = (half ? np : 0) + p;
      if (S.has1) y += S.eps * mf_q1(S, f1, a, b, p, half);
    } else {
      row = 2 * np + lam - 1;  // Q1 D rows are empty for a diagonal drive
    }
    mf_epilogue(S, row, y);
  }
}

// rows of Q0 longer than RK4_LONG, listed in ascending order (ballot compaction per warp and
// an atomic per warp: the list order is fixed by the row order within each warp, the warps'
// slots may vary, which does not change any row's result)
__global__ void k_rk4_longrows(long long m, const int64_t* __restrict__ rp, int* list, int* count) {
  const long long row = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool lg = row < m && rp[row + 1] - rp[row] > RK4_LONG;
  const unsigned bal = __ballot_sync(FULL, lg);
  if (!bal) return;
  const int lane = threadIdx.x & 31;
  int base = 0;
  if (lane == 0) base = atomicAdd(count, __popc(bal));
  base = __shfl_sync(FULL, base, 0);
  if (lg) list[base + __popc(bal & ((1u << lane) - 1u))] = (int)row;
}

// v = Re Tr(F_s rho): S_ab / J_ab from the off-diagonal entries (two addends per coefficient,
// added to zero: the result does not depend on their order), then the D^l chain from the
// diagonal (one CTA, fixed-order scan).
__global__ void k_state_zero(double* v, long long m) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
    v[i] = 0.0;
}

__global__ void k_state_offdiag(int n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                const double2* __restrict__ val, double* v) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const long long np = (long long)n * (n - 1) / 2;
  const double is2 = 0.70710678118654752440;
  for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
    const int c = ci[k];
    if (c == r) continue;
    const double2 x = val[k];
    const int a = r < c ? r : c, b = r < c ? c : r;
    const long long p = (long long)a * (2LL * n - a - 1) / 2 + (b - a - 1);
    // Tr(S_ab rho) = (rho_ab + rho_ba)/sqrt2;  Tr(J_ab rho) = i (rho_ab - rho_ba)/sqrt2
    atomicAdd(&v[p], is2 * x.x);
    atomicAdd(&v[np + p], r < c ? -is2 * x.y : is2 * x.y);
  }
}

__global__ void __launch_bounds__(1024) k_state_diag(int n, const int64_t* __restrict__ rp,
                                                     const int32_t* __restrict__ ci,
                                                     const double2* __restrict__ val, double* v) {
  __shared__ double carry_s;
  __shared__ double wsum[32];
  const long long dbase = (long long)n * (n - 1) - 1;  // v index of D^l is N(N-1) + l - 1
  if (threadIdx.x == 0) carry_s = 0.0;
  __syncthreads();
  for (int base = 0; base < n; base += blockDim.x) {
    const int c = base + threadIdx.x;
    double d = 0.0;
    if (c < n)
      for (int64_t k = rp[c]; k < rp[c + 1]; ++k)
        if (ci[k] == c) d = val[k].x;
    // block inclusive scan of d (fixed order)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double x = d;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      double t = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0.0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(FULL, t, o);
        if (lane >= o) t += y;
      }
      wsum[lane] = t;
    }
    __syncthreads();
    const double carry = carry_s;
    const double incl = carry + (wid > 0 ? wsum[wid - 1] : 0.0) + x;
    const double pre = incl - d;  // sum_{c' < c} rho_c'c'
    if (c >= 1 && c < n) v[dbase + c] = (pre - (double)c * d) / sqrt((double)c * (double)(c + 1));
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry_s = incl;
    __syncthreads();
  }
}

// rho(T) (Step 3.2; Eq. 5): rho = I/N + sum_j v_j F_j as a dense complex N x N array.
// Off-diagonal entries from the S/J pair (thread per pair): rho_ab = (v_S - i v_J)/sqrt2,
// rho_ba = (v_S + i v_J)/sqrt2; the diagonal comes from k_state_pop writing with a stride.
__global__ void k_state_rho_offdiag(int n, const double* __restrict__ v, double2* __restrict__ rho) {
  const long long np = (long long)n * (n - 1) / 2;
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= np) return;
  const double t = 2.0 * n - 1.0;
  long long a = (long long)floor((t - sqrt(fmax(t * t - 8.0 * (double)p, 0.0))) * 0.5);
  if (a < 0) a = 0;
  while (a > 0 && a * (2LL * n - a - 1) / 2 > p) --a;
  while (a + 1 <= n - 2 && (a + 1) * (2LL * n - a - 2) / 2 <= p) ++a;
  const long long b = a + 1 + (p - a * (2LL * n - a - 1) / 2);
  const double s = v[p], j = v[np + p];
  const double r = 0.70710678118654752440;
  rho[a * n + b] = make_double2(s * r, -j * r);
  rho[b * n + a] = make_double2(s * r, j * r);
}

// diag[a] = 1/N + sum_{l >= max(a,1)} v_{D^l} delta_l(a): delta_l(a) = 1/sqrt(l(l+1)) for
// l > a, -a/sqrt(a(a+1)) for l = a.  Suffix sums by one CTA (fixed order).
// dstride: element stride of the output (1: diag[a]; 2(N+1): the real parts of the diagonal of
// an interleaved complex N x N array, whose imaginary parts are then set to 0)
__global__ void __launch_bounds__(1024) k_state_pop(int n, const double* __restrict__ v, double* diag,
                                                    long long dstride = 1) {
  __shared__ double carry_s;
  __shared__ double wsum[32];
  const long long dbase = (long long)n * (n - 1) - 1;
  if (threadIdx.x == 0) carry_s = 0.0;
  __syncthreads();
  // process l from n-1 down in blocks: suffix[a] = sum_{l > a} v_l / sqrt(l(l+1))
  for (int top = n - 1; top >= 0; top -= blockDim.x) {
    const int a = top - (int)threadIdx.x;  // descending
    double w = 0.0;                          // term of l = a + 1 (for the suffix over l > a)
    if (a >= 0 && a + 1 <= n - 1) w = v[dbase + a + 1] / sqrt((double)(a + 1) * (double)(a + 2));
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double x = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      double t = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0.0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(FULL, t, o);
        if (lane >= o) t += y;
      }
      wsum[lane] = t;
    }
    __syncthreads();
    const double suf = carry_s + (wid > 0 ? wsum[wid - 1] : 0.0) + x;  // sum_{l > a}
    if (a >= 0) {
      const double self = a >= 1 ? -(double)a * v[dbase + a] / sqrt((double)a * (double)(a + 1)) : 0.0;
      diag[(long long)a * dstride] = 1.0 / (double)n + suf + self;
      if (dstride > 1) diag[(long long)a * dstride + 1] = 0.0;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry_s = suf;
    __syncthreads();
  }
}

// =========================================================================================
// Host side
// =========================================================================================
namespace {

int cuda_fail(cudaError_t e) {
  snprintf(g_errbuf, sizeof(g_errbuf), "CUDA error: %s", cudaGetErrorString(e));
  return SUN_ERR_CUDA;
}
}  // namespace
// shared with sunfold_dense.cu (same library)
int sunfold_cuda_fail(cudaError_t e) { return cuda_fail(e); }
namespace {
#define CK(x)                                    \
  do {                                           \
    cudaError_t e_ = (x);                        \
    if (e_ != cudaSuccess) return cuda_fail(e_); \
  } while (0)

// kernel launch, with the programmatic-dependent-launch attribute when `pdl` (the kernel
// starts while its predecessor in the stream finishes; it waits in pdl_enter)
template <typename... KArgs, typename... Args>
cudaError_t launch_k(bool pdl, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

bool zcsr_ok(const sun_zcsr* A, int n) {
  return A && A->n == n && A->nnz >= 0 && A->row_ptr && (A->nnz == 0 || (A->col && A->val));
}

// far-pair position list (relative offsets to (a, b)), lexicographic; same as far_pos()
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

// ---- mode-0 instantiations: (WK, WL, PT) ----
#define SUN_MODE0_LIST(X)                                        \
  X(0, 0, 0) X(1, 0, 0) X(2, 0, 0) X(3, 0, 0)                    \
  X(0, 0, 1) X(1, 0, 1) X(2, 0, 1) X(3, 0, 1) X(2, 1, 1)         \
  X(0, 0, -1) X(1, 0, -1) X(2, 0, -1) X(3, 0, -1) X(2, 1, -1)    \
  X(4, 2, 1) X(4, 2, -1)

int mode0_pt(int P) { return P == 0 ? 0 : (P == 1 ? 1 : -1); }

bool mode0_supported(int wK, int wL, int P) {
  const int pt = mode0_pt(P);
  if (wK == 4 && wL == 2) {  // A/B against the warp-per-pair mode 2 (SUNFOLD_MODE2=1)
    const char* m2 = getenv("SUNFOLD_MODE2");
    if (m2 && m2[0] && m2[0] != '0') return false;
  }
#define SUN_X(WK, WL, PT) \
  if (wK == WK && wL == WL && pt == PT) return true;
  SUN_MODE0_LIST(SUN_X)
#undef SUN_X
  return false;
}

// ---- mode-2 instantiations (compile-time warp-per-pair far path) ----
bool mode2_supported(int wK, int wL, int P) { return wK == 4 && wL == 2 && P >= 1; }

template <int WK, int WL, int PT>
cudaError_t launch2_t(const Prob& pr, const MatCount* mc, const MatFill* mf, long long* grid_out, long long grid,
                      cudaStream_t st) {
  if (grid_out) {  // plan creation: persistent fill grid
    int dev = 0, sms = 0, nb = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_fill2<WK, WL, PT>, 256, 0);
    if (e != cudaSuccess) return e;
    const long long U = (pr.npt + SLOTS_PER_TILE - 1) / SLOTS_PER_TILE + near_units(pr.n, pr.W);
    *grid_out = (long long)(nb > 0 ? nb : 1) * sms;
    if (*grid_out > U) *grid_out = U;
    return cudaSuccess;
  }
  if (mc) {
    const long long U = pr.nb_near + (pr.np + 31) / 32;
    k_count2<WK, WL, PT><<<(unsigned)U, 32, 0, st>>>(*mc);
  } else {
    k_fill2<WK, WL, PT><<<(unsigned)grid, 256, 0, st>>>(*mf);
  }
  return cudaGetLastError();
}

cudaError_t launch2(const Prob& pr, const MatCount* mc, const MatFill* mf, long long* grid_out, long long grid,
                    cudaStream_t st) {
  if (pr.wK == 4 && pr.wL == 2) {
    if (pr.P == 1) return launch2_t<4, 2, 1>(pr, mc, mf, grid_out, grid, st);
    return launch2_t<4, 2, -1>(pr, mc, mf, grid_out, grid, st);
  }
  return cudaErrorInvalidValue;
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
    pr.tau_ptr = &reinterpret_cast<DevHeader*>(pl->ws + L.hdr)->tau[0];
  } else {
    pr.P = 0;
    pr.wK = pl->wH1;
    pr.wL = 0;
    pr.K = {reinterpret_cast<const double2*>(pl->ws + L.hb1), pl->wH1};
    pr.H = pr.K;
    pr.L = nullptr;
    pr.tau_ptr = &reinterpret_cast<DevHeader*>(pl->ws + L.hdr)->tau[1];
  }
  pr.tau = 0.0;
  pr.W = pr.wK > pr.wL ? pr.wK : pr.wL;
  pr.inv = reinterpret_cast<const double*>(pl->ws + L.inv);
  build_far_positions(pr.W, pr.wL, pr.wK, pl->pos_dc[which], pl->pos_dd[which]);
  int npos = (int)pl->pos_dc[which].size();
  pl->npos_far[which] = npos;
  for (int i = 0; i < npos && i < FAR_MAXPOS; ++i) {
    pl->hfp[which].dc[i] = pl->pos_dc[which][i];
    pl->hfp[which].dd[i] = pl->pos_dd[which][i];
  }
  pr.mode = mode0_supported(pr.wK, pr.wL, pr.P) ? 0 : (mode2_supported(pr.wK, pr.wL, pr.P) ? 2 : 1);
  pl->side[which] = NearSide{reinterpret_cast<int32_t*>(pl->ws + L.side_col[which]),
                             reinterpret_cast<double*>(pl->ws + L.side_val[which]),
                             reinterpret_cast<NearMeta*>(pl->ws + L.side_meta[which]), (4 * pr.W + 1) * (4 * pr.W + 1),
                             (4 * pr.W + 1) * (4 * pr.W) / 2};
  if (pr.mode == 2) {
    pr.tp = TP0 / SLOTS_PER_TILE;  // scan slot = one count warp's 32 pairs
    pr.npt = (pr.np + pr.tp - 1) / pr.tp;
    pr.ndt = pl->n - 1;
    pr.nb_near = (long long)pl->n * 2 * pr.W + (pl->n - 1);
  } else if (pr.mode == 0) {
    // scan slot = one count warp's pairs = one fill warp's pairs (Tiling<WK, WL>::TP / 8:
    // 32, or 256 for the staging-free W = 0 tiles of 8 pairs per thread)
    pr.tp = (pr.wK == 0 ? 2048 : TP0) / SLOTS_PER_TILE;
    pr.npt = (pr.np + pr.tp - 1) / pr.tp;
    pr.ndt = pl->n - 1;
    const long long items = (long long)pl->n * 2 * pr.W + (pl->n - 1);
    pr.nb_near = items;  // count-pass near items: one warp-CTA each
  } else {
    pr.tp = WARP_TP;
    pr.npt = (pr.np + WARP_TP - 1) / WARP_TP;
    pr.ndt = (pl->n - 1 + WARP_THREADS / 32 - 1) / (WARP_THREADS / 32);
    pr.nb_near = 0;
  }
}

// ---- mode-0 launchers.  Q1W = -1: one matrix per launch; Q1W = 0: Q0 + Q1 (Q1 = (0, 0, 0)).
template <int WK, int WL, int PT, int Q1W>
cudaError_t launch_count0(const MatCount& m0, const MatCount& m1, cudaStream_t st, bool pdl) {
  auto warps = [](const Prob& p) { return p.npt; };  // one count warp per scan slot
  const long long U = warps(m0.pr) + m0.pr.nb_near + (Q1W >= 0 ? warps(m1.pr) + m1.pr.nb_near : 0);
  if (U <= 0) return cudaGetLastError();
  return launch_k(pdl, k_count0<WK, WL, PT, Q1W>, dim3((unsigned)U), dim3(32), 0, st, m0, m1);
}

// called at plan creation (outside any graph capture): dynamic shared memory limit and the
// persistent fill grid (resident CTAs x SMs, capped by the number of units)
template <int WK, int WL, int PT, int Q1W>
cudaError_t attr_fill0(const Prob& p0, const Prob* p1, long long& grid) {
  const int smem = FillFar<WK, WL>::SMEM;
  static int c_sms = 0, c_nb = 0;  // per instantiation: set once (attribute, occupancy)
  int sms = c_sms, nb = c_nb;
  if (!c_sms) {
    cudaError_t e = cudaFuncSetAttribute(k_fill0<WK, WL, PT, Q1W>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int dev = 0;
    if (e == cudaSuccess) e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_fill0<WK, WL, PT, Q1W>, 256, smem);
    if (e != cudaSuccess) return e;
    c_nb = nb;
    c_sms = sms;
  }
  auto tiles = [](const Prob& p) { return (p.npt + SLOTS_PER_TILE - 1) / SLOTS_PER_TILE; };
  long long U = tiles(p0) + (2 * (p0.n * 2LL * p0.W + p0.n - 1) + NEAR_UROWS - 1) / NEAR_UROWS;
  if (Q1W >= 0 && p1) U += tiles(*p1) + near_units1(p1->n, p1->W);
  grid = (long long)(nb > 0 ? nb : 1) * sms;
  if (grid > U) grid = U;
  return cudaSuccess;
}

template <int WK, int WL, int PT, int Q1W>
cudaError_t launch_fill0(const MatFill& m0, const MatFill& m1, long long grid, cudaStream_t st, bool pdl) {
  return launch_k(pdl, k_fill0<WK, WL, PT, Q1W>, dim3((unsigned)grid), dim3(256), FillFar<WK, WL>::SMEM, st, m0, m1);
}

#define SUN_DISPATCH0(pr, q1w, CALL)                              \
  do {                                                            \
    const int pt_ = mode0_pt((pr).P);                             \
    if ((q1w) == 0) {                                             \
      SUN_MODE0_LIST(SUN_X0)                                      \
    } else {                                                      \
      SUN_MODE0_LIST(SUN_X1)                                      \
    }                                                             \
    return cudaErrorInvalidValue;                                 \
  } while (0)

cudaError_t dispatch_attr0(const Prob& p0, const Prob* p1, int q1w, long long& grid) {
#define SUN_X0(WK, WL, PT) \
  if (p0.wK == WK && p0.wL == WL && pt_ == PT) return attr_fill0<WK, WL, PT, 0>(p0, p1, grid);
#define SUN_X1(WK, WL, PT) \
  if (p0.wK == WK && p0.wL == WL && pt_ == PT) return attr_fill0<WK, WL, PT, -1>(p0, p1, grid);
  SUN_DISPATCH0(p0, q1w, 0);
#undef SUN_X0
#undef SUN_X1
}

cudaError_t dispatch_count0(const MatCount& m0, const MatCount& m1, int q1w, cudaStream_t st, bool pdl) {
#define SUN_X0(WK, WL, PT) \
  if (m0.pr.wK == WK && m0.pr.wL == WL && pt_ == PT) return launch_count0<WK, WL, PT, 0>(m0, m1, st, pdl);
#define SUN_X1(WK, WL, PT) \
  if (m0.pr.wK == WK && m0.pr.wL == WL && pt_ == PT) return launch_count0<WK, WL, PT, -1>(m0, m1, st, pdl);
  SUN_DISPATCH0(m0.pr, q1w, 0);
#undef SUN_X0
#undef SUN_X1
}

cudaError_t dispatch_fill0(const MatFill& m0, const MatFill& m1, int q1w, long long grid, cudaStream_t st,
                           bool pdl) {
#define SUN_X0(WK, WL, PT) \
  if (m0.pr.wK == WK && m0.pr.wL == WL && pt_ == PT) return launch_fill0<WK, WL, PT, 0>(m0, m1, grid, st, pdl);
#define SUN_X1(WK, WL, PT) \
  if (m0.pr.wK == WK && m0.pr.wL == WL && pt_ == PT) return launch_fill0<WK, WL, PT, -1>(m0, m1, grid, st, pdl);
  SUN_DISPATCH0(m0.pr, q1w, 0);
#undef SUN_X0
#undef SUN_X1
}

template <int WK, int WL, int PT>
cudaError_t launch_mf_t(const MfStage& S, unsigned grid, cudaStream_t st) {
  k_mf_stage<WK, WL, PT><<<grid, 256, 0, st>>>(S);
  return cudaGetLastError();
}
cudaError_t dispatch_mf(const MfStage& S, unsigned grid, cudaStream_t st) {
  if (S.p0.mode == 2 && S.p0.wK == 4 && S.p0.wL == 2)  // mode-2 widths (c3)
    return S.p0.P == 1 ? launch_mf_t<4, 2, 1>(S, grid, st) : launch_mf_t<4, 2, -1>(S, grid, st);
  const int pt_ = mode0_pt(S.p0.P);
#define SUN_XM(WK, WL, PT) \
  if (S.p0.wK == WK && S.p0.wL == WL && pt_ == PT) return launch_mf_t<WK, WL, PT>(S, grid, st);
  SUN_MODE0_LIST(SUN_XM)
#undef SUN_XM
  return cudaErrorInvalidValue;
}

long long nslots_of(const Prob& pr) { return 2 * pr.npt + pr.ndt; }

// mode 1 (warp per pair): compile-time far path for the widths listed, else the runtime table
template <int FK, int FL, int PT>
cudaError_t launch_mode1_t(const Prob& pr, const FarPos* fp, int npos, int* cnt, int* ts, const FillOut* fo,
                           cudaStream_t st) {
  const unsigned grid = (unsigned)(pr.npt + pr.ndt);
  if (!fo)
    k_count1<FK, FL, PT><<<grid, WARP_THREADS, 0, st>>>(pr, fp, npos, cnt, ts);
  else
    k_fill1<FK, FL, PT><<<grid, WARP_THREADS, 0, st>>>(pr, fp, npos, cnt, *fo);
  return cudaGetLastError();
}

cudaError_t launch_mode1(const Prob& pr, const FarPos* fp, int npos, int* cnt, int* ts, const FillOut* fo,
                         cudaStream_t st) {
  const int pt = mode0_pt(pr.P);
  if (pr.wK == 4 && pr.wL == 2) {
    if (pt == 1) return launch_mode1_t<4, 2, 1>(pr, fp, npos, cnt, ts, fo, st);
    if (pt == -1) return launch_mode1_t<4, 2, -1>(pr, fp, npos, cnt, ts, fo, st);
  }
  return launch_mode1_t<-1, 0, 0>(pr, fp, npos, cnt, ts, fo, st);
}

// mode 3: general-pattern operators (sunfold_general.cu).  Slot layout as modes 0/2: S slots and
// J slots of 32 pairs, one slot per D row.
void setup_general(sun_plan_s* pl) {
  const Layout& L = pl->lay;
  const sung::GLayout& g = pl->glay;
  char* ws = pl->ws;
  DevHeader* hdr = (DevHeader*)(ws + L.hdr);
  for (int which = 0; which < 1 + pl->has_h1; ++which) {
    Prob& pr = pl->pr[which];
    memset(&pr, 0, sizeof(pr));
    pr.n = pl->n;
    pr.np = (long long)pl->n * (pl->n - 1) / 2;
    pr.m = (long long)pl->n * pl->n - 1;
    pr.P = which ? 0 : pl->P;
    pr.mode = 3;
    pr.tp = sung::GSLOT;
    pr.npt = (pr.np + sung::GSLOT - 1) / sung::GSLOT;
    pr.ndt = pl->n - 1;
    pr.inv = reinterpret_cast<const double*>(ws + L.inv);
    pr.tau_ptr = &hdr->tau[which];
    pl->npos_far[which] = 0;
    sung::GProb& G = pl->gp[which];
    memset(&G, 0, sizeof(G));
    G.n = pl->n;
    G.P = pr.P;
    G.np = pr.np;
    G.m = pr.m;
    const OpDesc& h = pl->ops.op[which];
    G.H = {h.rp, h.ci, h.v};
    for (int p = 0; p < G.P; ++p) {
      const OpDesc& d = pl->ops.op[2 + p];
      G.L[p] = {d.rp, d.ci, d.v};
      G.C[p] = {reinterpret_cast<const int*>(ws + g.cp) + (long long)p * (pl->n + 1),
                reinterpret_cast<const int2*>(ws + g.xr) + g.xr_off[p]};
      G.g[p] = pl->gamma[p];
    }
    G.inv = pr.inv;
    G.tau_ptr = pr.tau_ptr;
    G.npt = pr.npt;
    G.heavy = reinterpret_cast<int*>(ws + (which ? g.heavy1 : g.heavy0));
    G.nheavy = reinterpret_cast<int*>(ws + g.nheavy) + which;
    G.dtot = reinterpret_cast<int*>(ws + (which ? g.dtot1 : g.dtot0));
    G.flags = &hdr->flags;
    G.cap = pl->small_cap ? 16 : (1 << 30);
  }
}

long long general_nnz(const sun_zcsr* const* L, int P, long long* nnzL) {
  long long tot = 0;
  for (int p = 0; p < P; ++p) {
    nnzL[p] = L[p]->nnz;
    tot += nnzL[p];
  }
  return tot;
}

}  // namespace

extern "C" {

const char* sun_version(void) { return "sunfold 0.2 (sm_100a, fp64)"; }

const char* sun_status_string(int status) {
  switch (status) {
    case SUN_OK: return "ok";
    case SUN_ERR_ARG: return "invalid argument (null/inconsistent pointers or malformed CSR)";
    case SUN_ERR_DIM: return "invalid dimension (need 2 <= N <= 46340 and equal N for all operators)";
    case SUN_ERR_NOT_HERMITIAN: return "H0 or H1 is not Hermitian (max|H - H^+| > 1e-12 ||H||_F)";
    case SUN_ERR_RATE: return "invalid rate (gamma_p must be finite and >= 0)";
    case SUN_ERR_CAPACITY: return "output CSR capacity below the required nnz";
    case SUN_ERR_CUDA: return g_errbuf[0] ? g_errbuf : "CUDA error";
    case SUN_ERR_UNSUPPORTED:
      return "unsupported for this plan (matrix-free propagation needs a banded plan; or a row with >= 2^32 "
             "candidate terms)";
    case SUN_ERR_STATE: return "call out of sequence (or operator values outside the plan's pattern: new plan)";
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

size_t sun_workspace_bytes_ops(const sun_zcsr* H0, const sun_zcsr* H1, const sun_zcsr* const* L, int32_t P) {
  (void)H1;
  if (!H0 || P < 0 || P > MAXOPS - 2 || (P > 0 && !L)) return 0;
  const int n = H0->n;
  if (n < 2 || n > 46340) return 0;
  long long nnzL[MAXOPS];
  for (int p = 0; p < P; ++p) {
    if (!L[p] || L[p]->nnz < 0) return 0;
    nnzL[p] = L[p]->nnz;
  }
  const size_t base = make_layout(n, P).total;
  return sung::g_layout(n, P, nnzL, base).total;
}

int sun_plan_create(sun_plan* out, const sun_zcsr* H0, const sun_zcsr* H1, const sun_zcsr* const* L,
                    const double* gamma, int32_t P, void* workspace, size_t workspace_bytes, void* stream) {
  return sun_plan_create_ex(out, H0, H1, L, gamma, P, 0, workspace, workspace_bytes, stream);
}

int sun_plan_create_ex(sun_plan* out, const sun_zcsr* H0, const sun_zcsr* H1, const sun_zcsr* const* L,
                       const double* gamma, int32_t P, int32_t flags, void* workspace, size_t workspace_bytes,
                       void* stream) {
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
  NvtxRange r_("sun_plan_create (analyse)");
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
  // operators beyond the banded kernels' widths (or SUN_PLAN_GENERAL): mode 3
  pl->general = (flags & (SUN_PLAN_GENERAL | SUN_PLAN_SMALLCAP)) || pl->wK > WMAX || pl->wL > WLMAX || pl->wH1 > WMAX;
  pl->small_cap = (flags & SUN_PLAN_SMALLCAP) != 0;
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
  if (!pl->general) {
    setup_prob(pl, 0);
    if (pl->has_h1) setup_prob(pl, 1);
    pl->general = pl->npos_far[0] > FAR_MAXPOS || (pl->has_h1 && pl->npos_far[1] > FAR_MAXPOS);
  }
  if (pl->general) {
    long long nnzL[MAXOPS];
    general_nnz(L, P, nnzL);
    pl->glay = sung::g_layout(n, P, nnzL, lay.total);
    if (workspace_bytes < pl->glay.total) {
      delete pl;
      return SUN_ERR_CAPACITY;  // general-pattern operators: size from sun_workspace_bytes_ops
    }
    for (int i = 0; i < MAXOPS; ++i) pl->ops.wplan[i] = -1;
    setup_general(pl);
    cudaError_t e1 = sung::g_prepare();
    if (e1 != cudaSuccess) {
      delete pl;
      return cuda_fail(e1);
    }
  }
  const int nmat = 1 + pl->has_h1;
  {
    const Prob& p0 = pl->pr[0];
    const Prob& p1 = pl->pr[1];
    pl->combined = p0.mode == 0 && (!pl->has_h1 || (p1.mode == 0 && p1.wK == 0 && p1.wL == 0 && p1.P == 0));
  }
  pl->launches_count = 1 + (pl->combined ? 1 : nmat) + 1;  // expand, count, scan
  {  // measured equal at c4 (k_near0 10.2 us + fill 53.2 us vs fill 61 us): off by default there;
     // on for wide bands, whose fill runs one CTA (8 warps) per SM (c3: near units inside the
     // fill 98 us, k_near0 12 us + fill 78 us)
    const char* nf = getenv("SUNFOLD_NEAR_SEP");
    const bool dflt = pl->pr[0].W >= 4;
    pl->near_sep = pl->combined && (nf && nf[0] ? nf[0] != '0' : dflt);
    const char* nc = getenv("SUNFOLD_NEAR_CONC");
    pl->near_conc = pl->near_sep ? (nc && nc[0] ? atoi(nc) : SUN_NEAR_CONC_DEFAULT) : 0;
  }
  pl->launches_fill = pl->combined ? 1 + pl->near_sep : nmat;
  {
    const char* sd = getenv("SUNFOLD_SCAN_DIRECT");
    pl->scan_direct = !(sd && sd[0] == '0');
  }
  {  // sun_run: near rows inside the scan's launch (k_scan_near0); SUNFOLD_SCAN_NEAR=1 for A/B (off: slower)
    const char* sn = getenv("SUNFOLD_SCAN_NEAR");
    pl->scan_near = pl->combined && (sn && sn[0] ? sn[0] != '0' : SUN_SCAN_NEAR_DEFAULT);
  }
  {
    const char* np_ = getenv("SUNFOLD_NO_PDL");
    const char* pm = getenv("SUNFOLD_PDL_MASK");  // bits: 1 count, 2 scan, 4 near, 8 fill
    const char* pr_ = getenv("SUNFOLD_PDL_RUN");
    pl->pdl_run = pr_ && pr_[0] && pr_[0] != '0';
    pl->pdl = pl->combined && !(np_ && np_[0] && np_[0] != '0') ? (pm && pm[0] ? atoi(pm) : SUN_PDL_DEFAULT) : 0;
  }
  if (pl->general) {
    pl->launches_count = (P > 0 ? sung::G_LAUNCHES_EXPAND : 1) + sung::G_LAUNCHES_COUNT * nmat + 1;
    pl->launches_fill = sung::G_LAUNCHES_FILL * nmat;
  }
  {
    cudaError_t e1 = res_acquire(pl->res);
    if (e1 != cudaSuccess) {
      delete pl;
      return cuda_fail(e1);
    }
    for (int i = 0; i < 2; ++i) {
      pl->aux[i] = pl->res.aux[i];
      pl->ev_join[i] = pl->res.join[i];
    }
    pl->ev_fork = pl->res.fork;
    pl->cap_stream = pl->res.cap;
    pl->hpin = pl->res.hpin;
    // the pooled slot may hold another plan's sequence number: none of this plan's (1, 2, ...)
    if (pl->hpin) *reinterpret_cast<volatile unsigned*>(&pl->hpin->seq) = 0xFFFFFFFFu;
    const char* ng = getenv("SUNFOLD_NO_GRAPHS");
    pl->use_graphs = !(ng && ng[0] && ng[0] != '0');
    if (pl->general) {
      // no band kernels
    } else if (pl->combined) {
      e1 = dispatch_attr0(pl->pr[0], pl->has_h1 ? &pl->pr[1] : nullptr, pl->has_h1 ? 0 : -1, pl->fill_grid[0]);
      static bool near_attr = false;  // k_near0's shared inv[] table: up to 64 KB
      if (e1 == cudaSuccess && !near_attr) {
        e1 = cudaFuncSetAttribute(k_near0, cudaFuncAttributeMaxDynamicSharedMemorySize, NEAR_SMEM_INV * (int)sizeof(double));
        if (e1 == cudaSuccess)
          e1 = cudaFuncSetAttribute(k_scan_near0, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    NEAR_SMEM_INV * (int)sizeof(double));
        near_attr = e1 == cudaSuccess;
      }
    } else {
      for (int which = 0; which < nmat && e1 == cudaSuccess; ++which) {
        if (pl->pr[which].mode == 0) e1 = dispatch_attr0(pl->pr[which], nullptr, -1, pl->fill_grid[which]);
        if (pl->pr[which].mode == 2) e1 = launch2(pl->pr[which], nullptr, nullptr, &pl->fill_grid[which], 0, nullptr);
      }
    }
    if (e1 != cudaSuccess) {
      delete pl;
      return cuda_fail(e1);
    }
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

static int enqueue_count_general(sun_plan pl, cudaStream_t st, bool scan_hdr) {
  const Layout& L = pl->lay;
  char* ws = pl->ws;
  DevHeader* hdr = (DevHeader*)(ws + L.hdr);
  sung::GExpandIn in;
  memset(&in, 0, sizeof(in));
  in.n = pl->n;
  in.nops = pl->ops.nops;
  in.has_h1 = pl->has_h1;
  for (int op = 0; op < in.nops; ++op) {
    in.rp[op] = pl->ops.op[op].rp;
    in.ci[op] = pl->ops.op[op].ci;
    in.v[op] = pl->ops.op[op].v;
    in.gamma[op] = pl->ops.gamma[op];
  }
  sung::GHeaderRef hr{&hdr->flags, hdr->tau, hdr->herm_dev, hdr->nrm2_h, hdr->nrm2, &hdr->done, hdr->ticket};
  const long long nz32 = (long long)((L.st0 - L.ts0) / sizeof(int));
  const long long nz64 = (long long)((L.toff0 - L.st0) / sizeof(unsigned long long));
  CK(sung::g_expand(in, ws, pl->glay, (double*)(ws + L.inv), (int*)(ws + L.ts0), nz32,
                    (unsigned long long*)(ws + L.st0), nz64, hr, st));
  const int nmat = 1 + pl->has_h1;
  ScanArgs sa;
  memset(&sa, 0, sizeof(sa));
  long long maxchunks = 1;
  CK(fork_aux(pl, st, nmat));  // D rows of matrix `which` on aux[which], concurrent with the pairs
  for (int which = 0; which < nmat; ++which) {
    int* cnt = (int*)(ws + (which ? L.cnt1 : L.cnt0));
    int* ts = (int*)(ws + (which ? L.ts1 : L.ts0));
    CK(sung::g_count(pl->gp[which], cnt, ts, st, pl->aux[which]));
    sa.ts[which] = ts;
    sa.toff[which] = (long long*)(ws + (which ? L.toff1 : L.toff0));
    sa.status[which] = (unsigned long long*)(ws + (which ? L.st1 : L.st0));
    sa.nnz[which] = &hdr->nnz[which];
    sa.nslots[which] = nslots_of(pl->pr[which]);
    const long long nc = (sa.nslots[which] + SCAN_TILE - 1) / SCAN_TILE;
    if (nc > maxchunks) maxchunks = nc;
  }
  CK(join_aux(pl, st, nmat));
  sa.ticket = hdr->ticket;
  sa.hdr = hdr;
  sa.hout = scan_hdr ? pl->res.dpin : nullptr;
  k_scan_chain<<<dim3((unsigned)maxchunks, nmat), SCAN_THREADS, 0, st>>>(sa);
  CK(cudaGetLastError());
  return SUN_OK;
}

// scan_hdr: the scan stores the header prefix into the mapped slot (else the fill does: see
// header_in_fill)
// pdl_ok: programmatic dependent launch allowed (the count-only sequence; see SUN_PDL_DEFAULT)
// near_mf: sun_run on a combined plan (scan_near_fused): the fill arguments of Q0; the scan's
// launch then also writes the near rows (k_scan_near0)
static int enqueue_count(sun_plan pl, cudaStream_t st, bool scan_hdr, bool pdl_ok, const MatFill* near_mf = nullptr) {
  NvtxRange r_("sunfold: expand (a1) + count (a3) + scan (a4)");
  if (pl->general) return enqueue_count_general(pl, st, scan_hdr);
  const Layout& L = pl->lay;
  const int n = pl->n;
  char* ws = pl->ws;
  DevHeader* hdr = (DevHeader*)(ws + L.hdr);
  // (a1) expand: band storage + norms/flags per row block; zero the scan state
  const long long nz32 = (long long)((L.st0 - L.ts0) / sizeof(int));
  const long long nz64 = (long long)((L.toff0 - L.st0) / sizeof(unsigned long long));
  ExpandArgs ea;
  ea.ops = pl->ops;
  ea.gam = pl->gam;
  ea.hb0 = (double2*)(ws + L.hb0);
  ea.hb1 = (double2*)(ws + L.hb1);
  ea.lb = (double2*)(ws + L.lb);
  ea.kb0 = (double2*)(ws + L.kb0);
  ea.inv = (double*)(ws + L.inv);
  ea.blk = (BlkInfo*)(ws + L.blk);
  ea.herm = (unsigned long long*)(ws + L.herm);
  ea.zero32 = (int*)(ws + L.ts0);
  ea.zero64 = (unsigned long long*)(ws + L.st0);
  ea.nz32 = nz32;
  ea.nz64 = nz64;
  ea.hdr = hdr;
  ea.done = &hdr->done;
  ea.wK = pl->wK;
  ea.wH1 = pl->wH1;
  ea.wL = pl->wL;
  ea.wX = pl->wK > pl->wH1 ? pl->wK : pl->wH1;
  ea.nrb = (int)L.nrb;
  ea.nA = (int)L.nrb * pl->ops.nops;
  {
    long long nk = (long long)n * (2 * ea.wX + 1);
    if (nk < n) nk = n;
    ea.nB = (int)((nk + EXP_THREADS - 1) / EXP_THREADS);
  }
  ea.P = pl->P;
  k_expand<<<(unsigned)(ea.nA + ea.nB), EXP_THREADS, 0, st>>>(ea);
  CK(cudaGetLastError());
  // (a3) count pass (+ (a4) prefix scan in the last CTA when small)
  const int nmat = 1 + pl->has_h1;
  MatCount mc[2];
  ScanArgs sa;
  memset(&sa, 0, sizeof(sa));
  long long maxchunks = 1;
  for (int which = 0; which < nmat; ++which) {
    const Prob& pr = pl->pr[which];
    int* cnt = (int*)(ws + (which ? L.cnt1 : L.cnt0));
    int* ts = (int*)(ws + (which ? L.ts1 : L.ts0));
    mc[which] = MatCount{pr, cnt, ts, pl->side[which], which == 0 && pr.mode == 0 ? (int2*)(ws + L.sab) : nullptr};
    sa.ts[which] = ts;
    sa.toff[which] = (long long*)(ws + (which ? L.toff1 : L.toff0));
    sa.status[which] = (unsigned long long*)(ws + (which ? L.st1 : L.st0));
    sa.nnz[which] = &hdr->nnz[which];
    sa.nslots[which] = nslots_of(pr);
    const long long nc = (sa.nslots[which] + SCAN_TILE - 1) / SCAN_TILE;
    if (nc > maxchunks) maxchunks = nc;
  }
  if (nmat == 1) mc[1] = mc[0];
  sa.ticket = hdr->ticket;
  sa.hdr = hdr;
  sa.hout = scan_hdr ? pl->res.dpin : nullptr;
  if (pl->combined) {
    CK(dispatch_count0(mc[0], mc[1], pl->has_h1 ? 0 : -1, st, pdl_ok && (pl->pdl & 1) && SUN_PDL_COUNT > 0));
  } else {
    if (pl->has_h1) CK(fork_aux(pl, st, 1));  // Q1's count pass runs concurrently on aux[0]
    for (int which = 0; which < nmat; ++which) {
      const Prob& pr = pl->pr[which];
      cudaStream_t s = which ? pl->aux[0] : st;
      if (pr.mode == 0) {
        CK(dispatch_count0(mc[which], mc[which], -1, s, false));
      } else if (pr.mode == 2) {
        CK(launch2(pr, &mc[which], nullptr, nullptr, 0, s));
      } else {
        const FarPos* fp = (const FarPos*)(ws + (which ? L.fp1 : L.fp0));
        CK(launch_mode1(pr, fp, pl->npos_far[which], mc[which].cnt, mc[which].tsum, nullptr, s));
      }
    }
    if (pl->has_h1) CK(join_aux(pl, st, 1));
  }
  // (a4) chained scan of both matrices' slot sums
  sa.direct = pl->scan_direct && maxchunks <= SUN_SCAN_DIRECT_MAX ? 1 : 0;
  if (near_mf) {
    const Prob& p0 = pl->pr[0];
    ScanNearArgs na;
    na.sa = sa;
    for (int which = 0; which < 2; ++which) {
      na.nch[which] = which < nmat ? (sa.nslots[which] + SCAN_TILE - 1) / SCAN_TILE : 0;
      if (which < nmat && na.nch[which] < 1) na.nch[which] = 1;  // the empty matrix's chunk writes nnz = 0
      na.done[which] = which < nmat ? sa.status[which] + L.maxchunks : nullptr;
    }
    na.done0 = na.done[0];
    MatFill m0 = *near_mf;
    m0.near_sep = 1;
    const long long nn0 = (2 * (p0.n * 2LL * p0.W + p0.n - 1) + NEAR_UROWS - 1) / NEAR_UROWS;
    const size_t sm = p0.n <= NEAR_SMEM_INV ? (size_t)p0.n * sizeof(double) : 0;
    CK(launch_k(false, k_scan_near0, dim3((unsigned)(na.nch[0] + na.nch[1] + nn0)), dim3(SCAN_THREADS), sm, st, na, m0));
    return SUN_OK;
  }
  CK(launch_k(pdl_ok && pl->combined && (pl->pdl & 2), k_scan_chain, dim3((unsigned)maxchunks, nmat), dim3(SCAN_THREADS), 0, st, sa));
  return SUN_OK;
}

int sun_plan_nnz(sun_plan pl, int64_t* nnz_q0, int64_t* nnz_q1) {
  if (!pl) return SUN_ERR_ARG;
  NvtxRange r_("sun_plan_nnz (readback)");
  if (!pl->counted) return SUN_ERR_STATE;
  HeaderPrefix hloc;
  HeaderPrefix* hp = pl->hpin ? pl->hpin : &hloc;
  if (pl->hdr_poll && pl->hdr_enqueued && pl->hpin) {
    // sun_run: the fill stores the header (final since the scan) into the mapped slot at its
    // start, sequence number last; return as soon as this sequence's number is there instead of
    // waiting for the whole stream (the fill's outputs stay ordered on the stream)
    const volatile unsigned* vs = &pl->hpin->seq;
    for (unsigned it = 0;; ++it) {
      if (*vs == pl->seq_expect) break;
      if ((it & 255u) == 255u) {
        const cudaError_t q = cudaStreamQuery(pl->count_stream);
        if (q == cudaSuccess) break;  // the sequence has completed: the slot is final
        if (q != cudaErrorNotReady) return cuda_fail(q);
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
  } else {
    if (!pl->hdr_enqueued)
      CK(cudaMemcpyAsync(hp, pl->ws + pl->lay.hdr, sizeof(HeaderPrefix), cudaMemcpyDeviceToHost, pl->count_stream));
    CK(cudaStreamSynchronize(pl->count_stream));
  }
  HeaderPrefix h;
  memcpy(&h, (const void*)hp, sizeof(h));
  if (h.flags & F_MALFORMED) return SUN_ERR_ARG;
  for (int k = 0; k < 1 + pl->has_h1; ++k) {
    double dev;
    memcpy(&dev, &h.herm_dev[k], sizeof(dev));
    if (dev > 1e-12 * sqrt(h.nrm2_h[k])) return SUN_ERR_NOT_HERMITIAN;
  }
  if (h.flags & F_PATTERN) return SUN_ERR_STATE;        // values outside the plan's bands: new plan
  if (h.flags & F_TOOBIG) return SUN_ERR_UNSUPPORTED;   // a row with >= 2^32 candidate terms
  pl->tau0 = h.tau[0];
  pl->tau1 = pl->has_h1 ? h.tau[1] : 0.0;
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

// sun_run on a mode-0 / mode-2 plan with a mapped header slot: the fill kernel stores the header
static bool header_in_fill(sun_plan pl) {
  return pl->res.dpin && !pl->general && (pl->combined || (!pl->has_h1 && pl->pr[0].mode == 2));
}

// the fill pass's per-matrix arguments for these outputs
static void build_matfill(sun_plan pl, sun_dcsr* Q0, sun_dcsr* Q1, double* K, bool fill_hdr, MatFill mf[2]) {
  const Layout& L = pl->lay;
  char* ws = pl->ws;
  DevHeader* hdr = (DevHeader*)(ws + L.hdr);
  const int nmat = 1 + pl->has_h1;
  for (int which = 0; which < nmat; ++which) {
    sun_dcsr* Q = which ? Q1 : Q0;
    FillOut fo = {Q->row_ptr, Q->col, Q->val, (long long)Q->nnz, which ? nullptr : K,
                  (const long long*)(ws + (which ? L.toff1 : L.toff0)), &hdr->nnz[which]};
    mf[which] = MatFill{pl->pr[which], (const int*)(ws + (which ? L.cnt1 : L.cnt0)), fo, pl->side[which],
                        pl->n >= SUN_TILE_SYNC_MIN_N ? 1 : 0, 0};
  }
  if (fill_hdr) {
    mf[0].hdr = hdr;
    mf[0].hout = pl->res.dpin;
  }
  if (pl->pr[0].mode == 0) mf[0].sab = (const int2*)(ws + L.sab);  // written by this plan's count pass
  if (pl->combined) mf[0].wctr = hdr->wctr;  // k_fill0's dynamic warp units (SUN_FILL_DYN)
  if (nmat == 1) mf[1] = mf[0];
}

// sun_run on a combined plan: the near rows are written by the scan's launch (k_scan_near0)
static bool scan_near_fused(sun_plan pl, int kind) { return kind == 2 && pl->combined && pl->scan_near; }

// pdl_first: the fill directly follows this plan's scan in the stream (sun_run)
// near_done: the near rows have been written by k_scan_near0 (the count sequence of this sun_run)
static int enqueue_fill(sun_plan pl, sun_dcsr* Q0, sun_dcsr* Q1, double* K, cudaStream_t st, bool fill_hdr,
                        bool pdl_first, bool near_done) {
  NvtxRange r_("sunfold: fill (a5) + K + Q1 (a6)");
  const Layout& L = pl->lay;
  char* ws = pl->ws;
  const int nmat = 1 + pl->has_h1;
  MatFill mf[2];
  build_matfill(pl, Q0, Q1, K, fill_hdr, mf);
  if (pl->general) {
    CK(fork_aux(pl, st, nmat));  // heavy rows of matrix `which` on aux[which]
    for (int which = 0; which < nmat; ++which) {
      const FillOut& fo = mf[which].fo;
      const sung::GOut go{fo.row_ptr, fo.col, fo.val, fo.cap, fo.K, fo.toff, fo.nnz};
      CK(sung::g_fill(pl->gp[which], mf[which].cnt, go, st, pl->aux[which]));
    }
    CK(join_aux(pl, st, nmat));
    return SUN_OK;
  }
  if (pl->combined) {
    if (near_done) {
      mf[0].near_sep = 1;
    } else if (pl->near_sep) {
      mf[0].near_sep = 1;
      const Prob& p0 = pl->pr[0];
      const long long nn0 = (2 * (p0.n * 2LL * p0.W + p0.n - 1) + NEAR_UROWS - 1) / NEAR_UROWS;
      const size_t sm = p0.n <= NEAR_SMEM_INV ? (size_t)p0.n * sizeof(double) : 0;
      if (nn0 > 0 && pl->near_conc) {
        // the near rows and the far tiles write disjoint outputs: k_near0 on aux[0] beside the
        // fill (its CTAs hold SMs until the fill's persistent CTAs, which claim units
        // dynamically, take them over)
        CK(fork_aux(pl, st, 1));
        const bool swap = pl->near_conc == 2;  // A/B: the fill on the aux stream instead
        CK(launch_k(false, k_near0, dim3((unsigned)nn0), dim3(256), sm, swap ? st : pl->aux[0], mf[0]));
        CK(dispatch_fill0(mf[0], mf[1], pl->has_h1 ? 0 : -1, pl->fill_grid[0], swap ? pl->aux[0] : st, false));
        CK(join_aux(pl, st, 1));
        return SUN_OK;
      }
      if (nn0 > 0) CK(launch_k((pl->pdl & 4) && pdl_first, k_near0, dim3((unsigned)nn0), dim3(256), sm, st, mf[0]));
    }
    CK(dispatch_fill0(mf[0], mf[1], pl->has_h1 ? 0 : -1, pl->fill_grid[0], st, (pl->pdl & 8) && pdl_first));
    return SUN_OK;
  }
  // Q0 on st; Q1 concurrently on aux[0]
  if (pl->has_h1) CK(fork_aux(pl, st, 1));
  for (int which = pl->has_h1; which >= 0; --which) {  // Q1 (small) first
    const Prob& pr = pl->pr[which];
    cudaStream_t s = which ? pl->aux[0] : st;
    if (pr.mode == 0) {
      CK(dispatch_fill0(mf[which], mf[which], -1, pl->fill_grid[which], s, false));
    } else if (pr.mode == 2) {
      CK(launch2(pr, nullptr, &mf[which], nullptr, pl->fill_grid[which], s));
    } else {
      const FarPos* fp = (const FarPos*)(ws + (which ? L.fp1 : L.fp0));
      CK(launch_mode1(pr, fp, pl->npos_far[which], const_cast<int*>(mf[which].cnt), nullptr, &mf[which].fo, s));
    }
  }
  if (pl->has_h1) CK(join_aux(pl, st, 1));
  return SUN_OK;
}

// Enqueue kind 0 (count), 1 (fill) or 2 (count + fill) on `st`: replay a cached CUDA graph of
// the sequence (captured on the plan's capture stream; kernel arguments, including the output
// pointers and capacities, are part of the key), or enqueue directly if graphs are disabled.
static int enqueue_kind(sun_plan pl, int kind, sun_dcsr* Q0, sun_dcsr* Q1, double* K, cudaStream_t st) {
  NvtxRange r_(kind == 0 ? "sun_count" : (kind == 1 ? "sun_unfold" : "sun_run"));
  // the nnz / flags readback of sun_plan_nnz rides in the same sequence (a memcpy node of the
  // graph into pinned host memory), so sun_plan_nnz only waits for the stream
  const bool readback = kind != 1 && pl->hpin;
  const bool mapped = pl->res.dpin != nullptr;  // the scan stores the header into hpin itself
  // event records (external: event-record nodes under capture) around the phases when timing
  auto tmark = [&](cudaStream_t s, int i) -> int {
    if (!pl->timing) return SUN_OK;
    const cudaError_t e = s == pl->cap_stream ? cudaEventRecordWithFlags(pl->tev[i], s, cudaEventRecordExternal)
                                              : cudaEventRecord(pl->tev[i], s);
    return e == cudaSuccess ? SUN_OK : cuda_fail(e);
  };
  auto direct = [&](cudaStream_t s) -> int {
    int rc = SUN_OK;
    const bool fill_hdr = kind == 2 && header_in_fill(pl);
    const bool fused = scan_near_fused(pl, kind);
    MatFill nmf[2];
    if (fused) build_matfill(pl, Q0, Q1, K, false, nmf);
    if (kind != 1) rc = tmark(s, 0);
    if (rc == SUN_OK && kind != 1) rc = enqueue_count(pl, s, !fill_hdr, kind == 0 || pl->pdl_run, fused ? &nmf[0] : nullptr);
    if (rc == SUN_OK && kind != 0) rc = tmark(s, 1);
    if (rc == SUN_OK && kind != 0) rc = enqueue_fill(pl, Q0, Q1, K, s, fill_hdr, kind == 2, fused);
    if (rc == SUN_OK && kind == 0) rc = tmark(s, 1);
    if (rc == SUN_OK && kind != 0) rc = tmark(s, 2);
    if (rc == SUN_OK && readback && !mapped) {
      const cudaError_t e =
          cudaMemcpyAsync(pl->hpin, pl->ws + pl->lay.hdr, sizeof(HeaderPrefix), cudaMemcpyDeviceToHost, s);
      if (e != cudaSuccess) rc = cuda_fail(e);
    }
    return rc;
  };
  pl->hdr_enqueued = 0;
  pl->hdr_poll = 0;
  auto mark = [&](int rc) {  // the pooled pinned slot is written by this sequence: track its end
    if (rc == SUN_OK && readback) {
      const cudaError_t e = cudaEventRecord(pl->res.done, st);
      if (e != cudaSuccess) return cuda_fail(e);
    }
    if (rc == SUN_OK && kind != 1 && !pl->general) ++pl->seq_expect;  // k_expand ran once more
    if (rc == SUN_OK && pl->timing) pl->timed_kind = kind;
    if (rc == SUN_OK && kind == 2 && mapped && header_in_fill(pl)) pl->hdr_poll = 1;
    return rc;
  };
  if (!pl->use_graphs) {
    const int rc = mark(direct(st));
    pl->hdr_enqueued = rc == SUN_OK && readback ? 1 : 0;
    return rc;
  }
  uintptr_t key[12] = {(uintptr_t)kind, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  if (kind != 0) {
    key[1] = (uintptr_t)Q0->row_ptr; key[2] = (uintptr_t)Q0->col; key[3] = (uintptr_t)Q0->val;
    key[4] = (uintptr_t)Q0->nnz;     key[5] = (uintptr_t)K;
    if (Q1) {
      key[6] = (uintptr_t)Q1->row_ptr; key[7] = (uintptr_t)Q1->col; key[8] = (uintptr_t)Q1->val;
      key[9] = (uintptr_t)Q1->nnz;
    }
  }
  cudaGraphExec_t exec = nullptr;
  for (auto& g : pl->graphs)
    if (memcmp(g.key, key, sizeof(key)) == 0) {
      exec = g.exec;
      g.used = ++pl->graph_clock;
      break;
    }
  if (!exec) {  // first use of this sequence: launch directly; capture a graph when it recurs
    std::vector<uintptr_t> kv(key, key + 12);
    bool again = false;
    for (const auto& k : pl->seen) again |= k == kv;
    if (!again) {
      if (pl->seen.size() >= 16) pl->seen.erase(pl->seen.begin());
      pl->seen.push_back(kv);
      const int rc = mark(direct(st));
      pl->hdr_enqueued = rc == SUN_OK && readback ? 1 : 0;
      return rc;
    }
  }
  if (!exec) {
    CK(cudaStreamBeginCapture(pl->cap_stream, cudaStreamCaptureModeThreadLocal));
    int rc = direct(pl->cap_stream);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(pl->cap_stream, &graph);
    if (rc != SUN_OK) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (e != cudaSuccess) return cuda_fail(e);
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(e);
    constexpr size_t MAXG = 8;
    if (pl->graphs.size() >= MAXG) {  // evict the least recently used
      size_t v = 0;
      for (size_t i = 1; i < pl->graphs.size(); ++i)
        if (pl->graphs[i].used < pl->graphs[v].used) v = i;
      cudaGraphExecDestroy(pl->graphs[v].exec);
      pl->graphs.erase(pl->graphs.begin() + v);
    }
    sun_plan_s::GraphEntry ge;
    memcpy(ge.key, key, sizeof(key));
    ge.exec = exec;
    ge.used = ++pl->graph_clock;
    pl->graphs.push_back(ge);
  }
  CK(cudaGraphLaunch(exec, st));
  const int rc = mark(SUN_OK);
  pl->hdr_enqueued = rc == SUN_OK && readback ? 1 : 0;
  return rc;
}

int sun_count(sun_plan pl, void* stream) {
  if (!pl) return SUN_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int rc = enqueue_kind(pl, 0, nullptr, nullptr, nullptr, st);
  if (rc != SUN_OK) return rc;
  pl->counted = 1;
  pl->ran = 0;
  pl->count_stream = st;
  pl->nnz[0] = pl->nnz[1] = -1;
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
  return enqueue_kind(pl, 1, Q0, pl->has_h1 ? Q1 : nullptr, K, (cudaStream_t)stream);
}

int sun_run(sun_plan pl, sun_dcsr* Q0, sun_dcsr* Q1, double* K, void* stream) {
  if (!pl) return SUN_ERR_ARG;
  int st = check_outputs(pl, Q0, Q1, K);
  if (st != SUN_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  st = enqueue_kind(pl, 2, Q0, pl->has_h1 ? Q1 : nullptr, K, s);
  if (st != SUN_OK) return st;
  pl->counted = 1;
  pl->count_stream = s;
  pl->nnz[0] = pl->nnz[1] = -1;
  pl->cap[0] = Q0->nnz;
  pl->cap[1] = pl->has_h1 ? Q1->nnz : 0;
  pl->ran = 1;
  return SUN_OK;
}

int64_t sun_nnz_bound(sun_plan pl, int32_t which) {
  if (!pl || which < 0 || which > 1 || (which == 1 && !pl->has_h1)) return -1;
  const Prob& pr = pl->pr[which];
  const long long n = pl->n;
  if (pl->general) return pr.m * pr.m;  // no structural bound short of dense
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
  // rows per CTA: at least 4096 entries per block on average (8 .. 256 rows, a power of two)
  const long long nz = Q0->nnz + (Q1 ? Q1->nnz : 0);
  int R = APPLY_THREADS;
  while (R > 8 && nz > 0 && (long long)(R / 2) * nz >= 4096LL * m) R >>= 1;
  k_apply<<<(unsigned)((m + R - 1) / R), APPLY_THREADS, 0, (cudaStream_t)stream>>>(
      m, R, Q0->row_ptr, Q0->col, Q0->val, Q1 ? Q1->row_ptr : nullptr, Q1 ? Q1->col : nullptr,
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
  info->tiles_q0 = nslots_of(pl->pr[0]);
  info->tiles_q1 = pl->has_h1 ? nslots_of(pl->pr[1]) : 0;
  info->has_h1 = pl->has_h1;
  info->npos_far_q0 = pl->npos_far[0];
  info->npos_far_q1 = pl->has_h1 ? pl->npos_far[1] : 0;
  info->launches_count = pl->launches_count;
  info->launches_fill = pl->launches_fill;
  return SUN_OK;
}

int sun_expand_state(const sun_zcsr* rho, double* v, void* stream) {
  if (!rho || !v || !rho->row_ptr || (rho->nnz > 0 && (!rho->col || !rho->val))) return SUN_ERR_ARG;
  const int n = rho->n;
  if (n < 2 || n > 46340) return SUN_ERR_DIM;
  cudaStream_t st = (cudaStream_t)stream;
  const long long m = (long long)n * n - 1;
  k_state_zero<<<296, 256, 0, st>>>(v, m);
  CK(cudaGetLastError());
  k_state_offdiag<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(n, rho->row_ptr, rho->col,
                                                                (const double2*)rho->val, v);
  CK(cudaGetLastError());
  k_state_diag<<<1, 1024, 0, st>>>(n, rho->row_ptr, rho->col, (const double2*)rho->val, v);
  CK(cudaGetLastError());
  return SUN_OK;
}

int sun_state_diag(const double* v, int32_t n, double* diag, void* stream) {
  if (!v || !diag) return SUN_ERR_ARG;
  if (n < 2 || n > 46340) return SUN_ERR_DIM;
  k_state_pop<<<1, 1024, 0, (cudaStream_t)stream>>>(n, v, diag);
  CK(cudaGetLastError());
  return SUN_OK;
}

int sun_state_reconstruct(const double* v, int32_t n, double* rho, void* stream) {
  if (!v || !rho) return SUN_ERR_ARG;
  if (n < 2 || n > 46340) return SUN_ERR_DIM;
  cudaStream_t st = (cudaStream_t)stream;
  const long long np = (long long)n * (n - 1) / 2;
  double2* r = reinterpret_cast<double2*>(rho);
  k_state_rho_offdiag<<<(unsigned)((np + 255) / 256), 256, 0, st>>>(n, v, r);
  k_state_pop<<<1, 1024, 0, st>>>(n, v, rho, 2LL * (n + 1));
  CK(cudaGetLastError());
  return SUN_OK;
}

size_t sun_rk4_work_bytes(int64_t m) {
  if (m <= 0) return 0;
  return (size_t)(4 * m) * sizeof(double) + (size_t)(m + 2) * sizeof(int);
}

int sun_rk4(const sun_dcsr* Q0, const sun_dcsr* Q1, const double* K, double eps0, double eps1, double omega,
            double t0, double h, int64_t nsteps, double* v, void* work, void* stream) {
  if (!Q0 || !Q0->row_ptr || !v || !work || nsteps < 0) return SUN_ERR_ARG;
  if (Q0->nnz > 0 && (!Q0->col || !Q0->val)) return SUN_ERR_ARG;
  if (Q1 && (Q1->m != Q0->m || !Q1->row_ptr || (Q1->nnz > 0 && (!Q1->col || !Q1->val)))) return SUN_ERR_ARG;
  const long long m = Q0->m;
  if (m <= 0 || m > 0x7fffffffLL) return SUN_ERR_DIM;
  if (nsteps == 0) return SUN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  // stage vectors are double-buffered: a stage gathers k_{i-1} (other rows) while it writes k_i
  double* kA = (double*)work;
  double* kB = kA + m;
  double* acc = kA + 2 * m;
  double* vb = kA + 3 * m;
  int* cntp = (int*)(vb + m);
  int* list = cntp + 2;
  // the long-row list of this Q0 (one small readback per call)
  CK(cudaMemsetAsync(cntp, 0, sizeof(int), st));
  k_rk4_longrows<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(m, Q0->row_ptr, list, cntp);
  CK(cudaGetLastError());
  int nlong = 0;
  CK(cudaMemcpyAsync(&nlong, cntp, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  double* cur = v;
  double* nxt = vb;
  Rk4Stage S;
  S.rp0 = Q0->row_ptr; S.c0 = Q0->col; S.v0 = Q0->val;
  S.rp1 = Q1 ? Q1->row_ptr : nullptr; S.c1 = Q1 ? Q1->col : nullptr; S.v1 = Q1 ? Q1->val : nullptr;
  S.K = K; S.m = m; S.acc = acc; S.h6 = h / 6.0;
  S.longrows = list;
  S.nlong = nlong;
  S.nshort_blocks = (int)((m + 255) / 256);
  const unsigned grid = (unsigned)(S.nshort_blocks + (nlong + 7) / 8);
  auto eps = [&](double t) { return eps0 + eps1 * sin(omega * t); };
  for (int64_t i = 0; i < nsteps; ++i) {
    const double t = t0 + (double)i * h;
    S.v = cur;
    S.vout = nxt;
    S.kp = nullptr; S.kout = kA; S.c = 0.0; S.eps = eps(t); S.mode = 0;        // k1 = f(t, v)
    k_rk4_stage<<<grid, 256, 0, st>>>(S);
    S.kp = kA; S.kout = kB; S.c = 0.5 * h; S.eps = eps(t + 0.5 * h); S.mode = 1;  // k2 = f(t + h/2, v + h/2 k1)
    k_rk4_stage<<<grid, 256, 0, st>>>(S);
    S.kp = kB; S.kout = kA; S.mode = 1;                                       // k3 = f(t + h/2, v + h/2 k2)
    k_rk4_stage<<<grid, 256, 0, st>>>(S);
    S.kp = kA; S.kout = nullptr; S.c = h; S.eps = eps(t + h); S.mode = 2;     // k4 = f(t + h, v + h k3); v'
    k_rk4_stage<<<grid, 256, 0, st>>>(S);
    CK(cudaGetLastError());
    double* tmp = cur;
    cur = nxt;
    nxt = tmp;
  }
  if (cur != v) CK(cudaMemcpyAsync(v, cur, (size_t)m * sizeof(double), cudaMemcpyDeviceToDevice, st));
  return SUN_OK;
}

size_t sun_rk4_plan_work_bytes(sun_plan pl) {
  if (!pl) return 0;
  const long long m = (long long)pl->n * pl->n - 1;
  return (size_t)(4 * m + pl->n) * sizeof(double);
}

int sun_apply_plan(sun_plan pl, double eps, const double* v, double* dvdt, void* work, size_t work_bytes,
                   void* stream) {
  if (!pl || !v || !dvdt || !work || v == dvdt) return SUN_ERR_ARG;
  if (!pl->counted) return SUN_ERR_STATE;
  if (!(pl->pr[0].mode == 0 || (pl->pr[0].mode == 2 && pl->wK == 4 && pl->wL == 2)) || (pl->has_h1 && pl->wH1 != 0))
    return SUN_ERR_UNSUPPORTED;
  if (work_bytes < (size_t)pl->n * sizeof(double)) return SUN_ERR_CAPACITY;
  cudaStream_t st = (cudaStream_t)stream;
  MfStage S{};
  S.p0 = pl->pr[0];
  S.p1 = pl->has_h1 ? pl->pr[1] : pl->pr[0];
  S.has1 = pl->has_h1;
  S.side = pl->side[0];
  S.pref = (double*)work;
  S.pref_out = (double*)work;
  S.x = v;
  S.v = v;
  S.vout = dvdt;
  S.eps = eps;
  S.mode = 3;
  S.m = pl->pr[0].m;
  S.nfar_blocks = (int)((pl->pr[0].np + 255) / 256);
  const long long nside = 2 * ((long long)pl->n * 2 * S.p0.W + pl->n - 1);
  const unsigned grid = (unsigned)(S.nfar_blocks + (nside + 7) / 8);
  k_mf_prefix<<<1, 1024, 0, st>>>(S);
  CK(cudaGetLastError());
  CK(dispatch_mf(S, grid, st));
  return SUN_OK;
}

int sun_rk4_plan(sun_plan pl, double eps0, double eps1, double omega, double t0, double h, int64_t nsteps,
                 double* v, void* work, size_t work_bytes, void* stream) {
  if (!pl || !v || !work || nsteps < 0) return SUN_ERR_ARG;
  if (!pl->counted) return SUN_ERR_STATE;
  if (!(pl->pr[0].mode == 0 || (pl->pr[0].mode == 2 && pl->wK == 4 && pl->wL == 2)) || (pl->has_h1 && pl->wH1 != 0))
    return SUN_ERR_UNSUPPORTED;
  if (work_bytes < sun_rk4_plan_work_bytes(pl)) return SUN_ERR_CAPACITY;
  if (nsteps == 0) return SUN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const long long m = pl->pr[0].m, np = pl->pr[0].np;
  double* kA = (double*)work;
  double* kB = kA + m;
  double* acc = kA + 2 * m;
  double* vb = kA + 3 * m;
  double* pref = kA + 4 * m;
  MfStage S{};
  S.p0 = pl->pr[0];
  S.p1 = pl->has_h1 ? pl->pr[1] : pl->pr[0];
  S.has1 = pl->has_h1;
  S.side = pl->side[0];
  S.pref = pref;
  S.pref_out = pref;
  S.acc = acc;
  S.h6 = h / 6.0;
  S.m = m;
  S.nfar_blocks = (int)((np + 255) / 256);
  const long long nside = 2 * ((long long)pl->n * 2 * S.p0.W + pl->n - 1);
  const unsigned grid = (unsigned)(S.nfar_blocks + (nside + 7) / 8);
  auto eps = [&](double t) { return eps0 + eps1 * sin(omega * t); };
  double* cur = v;
  double* nxt = vb;
  auto stage = [&]() -> cudaError_t {
    k_mf_prefix<<<1, 1024, 0, st>>>(S);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = dispatch_mf(S, grid, st);
    return e;
  };
  // stage inputs x are double-buffered in kA / kB (each stage writes the next one's input)
  for (int64_t i = 0; i < nsteps; ++i) {
    const double t = t0 + (double)i * h;
    S.v = cur;
    S.vout = nxt;
    S.x = cur; S.xn = kA; S.cn = 0.5 * h; S.eps = eps(t); S.mode = 0;               // k1 = f(t, v)
    CK(stage());
    S.x = kA; S.xn = kB; S.cn = 0.5 * h; S.eps = eps(t + 0.5 * h); S.mode = 1;      // k2 at v + h/2 k1
    CK(stage());
    S.x = kB; S.xn = kA; S.cn = h; S.mode = 1;                                      // k3 at v + h/2 k2
    CK(stage());
    S.x = kA; S.xn = nullptr; S.eps = eps(t + h); S.mode = 2;                       // k4 at v + h k3; v'
    CK(stage());
    double* tmp = cur;
    cur = nxt;
    nxt = tmp;
  }
  if (cur != v) CK(cudaMemcpyAsync(v, cur, (size_t)m * sizeof(double), cudaMemcpyDeviceToDevice, st));
  return SUN_OK;
}

int sun_plan_set_graphs(sun_plan pl, int32_t enable) {
  if (!pl) return SUN_ERR_ARG;
  pl->use_graphs = enable != 0;
  return SUN_OK;
}

size_t sun_plan_stash_bytes(sun_plan pl) {
  if (!pl || !pl->general) return 0;
  return sung::g_stash_bytes(pl->n) * (size_t)(1 + pl->has_h1);
}

int sun_plan_set_stash(sun_plan pl, void* buf, size_t bytes) {
  if (!pl) return SUN_ERR_ARG;
  if (buf && (!pl->general || bytes < sun_plan_stash_bytes(pl) || ((uintptr_t)buf & 255))) return SUN_ERR_ARG;
  const size_t per = sung::g_stash_bytes(pl->n);
  for (int which = 0; which < 1 + pl->has_h1 && pl->general; ++which)
    sung::g_stash_set(pl->gp[which], buf ? (char*)buf + which * per : nullptr);
  pl->stash = (char*)buf;
  if (pl->general) pl->launches_fill = (sung::G_LAUNCHES_FILL + (buf ? 1 : 0)) * (1 + pl->has_h1);  // + k_g_copy
  for (auto& g : pl->graphs) cudaGraphExecDestroy(g.exec);  // the kernels' arguments changed
  pl->graphs.clear();
  pl->seen.clear();
  pl->counted = 0;  // the next fill needs a count pass that wrote the stash
  return SUN_OK;
}

int sun_plan_set_timing(sun_plan pl, int32_t enable) {
  if (!pl) return SUN_ERR_ARG;
  const int on = enable != 0;
  if (on == pl->timing) return SUN_OK;
  for (int i = 0; i < 3 && on; ++i)
    if (!pl->tev[i]) CK(cudaEventCreate(&pl->tev[i]));
  for (auto& g : pl->graphs) cudaGraphExecDestroy(g.exec);  // captured with / without the records
  pl->graphs.clear();
  pl->seen.clear();
  pl->timing = on;
  pl->timed_kind = -1;
  return SUN_OK;
}

int sun_plan_phase_ms(sun_plan pl, float* count_ms, float* fill_ms) {
  if (!pl) return SUN_ERR_ARG;
  if (!pl->timing || pl->timed_kind < 0) return SUN_ERR_STATE;
  const int k = pl->timed_kind;
  float c = -1.0f, f = -1.0f;
  if (k != 1) {
    CK(cudaEventSynchronize(pl->tev[1]));
    CK(cudaEventElapsedTime(&c, pl->tev[0], pl->tev[1]));
  }
  if (k != 0) {
    CK(cudaEventSynchronize(pl->tev[2]));
    CK(cudaEventElapsedTime(&f, pl->tev[1], pl->tev[2]));
  }
  if (count_ms) *count_ms = c;
  if (fill_ms) *fill_ms = f;
  return SUN_OK;
}

void sun_plan_destroy(sun_plan pl) { delete pl; }

}  // extern "C"
