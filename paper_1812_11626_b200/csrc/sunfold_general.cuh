// sunfold_general.cuh — general-pattern unfold (mode 3): any sparse or dense H0, H1 and L_p.
//
// The banded modes (0-2) index operators through band storage of bounded half-width.  Mode 3
// takes the operators as they are, in CSR ("any complex N x N matrix could be chosen as an
// operator L_p", Eq. 1), and assembles each output row from candidate
// terms that are merged on the device:
//
//   row S_ab / J_ab (a < b), U = L^+(E_ab):
//     U_cd = i K_ca [d = b] - i conj(K_db) [c = a] + sum_p gamma_p conj(L_p,ac) L_p,bd,
//     K = H + (i/2) sum_p gamma_p L_p^+ L_p, expanded term by term (no K is stored):
//       T1  c in row_H(a)          (c, b)   i conj(H_ac)                 (H Hermitian)
//       T2  d in row_H(b)          (a, d)  -i H_bd
//       T3  x in col_p(a), c in row_p(x)   (c, b)  -1/2 gamma_p conj(L_xc) L_xa
//       T4  x in col_p(b), d in row_p(x)   (a, d)  -1/2 gamma_p conj(L_xb) L_xd
//       T5  c in row_p(a), d in row_p(b)   (c, d)   gamma_p conj(L_ac) L_bd
//   row D^lam, f = diag(D^lam) (f_c = alpha for c < lam, -lam alpha at lam, 0 beyond):
//       TH  c <= lam, d in row_H(c), d >= lam, d > c:  G_cd += i H_cd (f_d - f_c)
//       TL  x, (c <= d) in row_p(x)^2:  G_cd += gamma_p (f_x - (f_c + f_d)/2) conj(L_xc) L_xd
//           (terms whose coefficient is exactly zero -- x, c, d all below or all above lam,
//           or x = c = d = lam -- are not generated)
//
// Every candidate (r, s, value) gets the key of its unordered generator pair {r, s}
// (p(min, max) of DESIGN.md R5) or, on the diagonal, np + r, and a sequence number fixed by
// the enumeration order.  A group of threads (a warp for light rows, a CTA for heavy rows and
// the D rows) gathers the candidates of a key range into shared memory, sorts them by
// (key, sequence) -- a bitonic sort -- and reduces each run of equal keys in sequence order
// (a segmented reduction): the GPU form of the paper's red-black-tree accumulation
// (P:444-448).  Rows with more candidates than the buffer are processed in key-range chunks
// planned from histograms.  The count and fill passes run the same code, so they agree bit
// for bit, and the result does not depend on scheduling (no floating-point atomics).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sung {

constexpr int GMAXP = 64;  // dissipators

struct GOp {  // CSR operator (device)
  const int64_t* rp;
  const int32_t* ci;
  const double2* v;
};
struct GCol {      // column access to a dissipator: entries of column c are xr[cp[c] .. cp[c+1])
  const int* cp;   // [n + 1]
  const int2* xr;  // (row x, CSR position of (x, c)), ascending in x
};

struct GProb {
  int n, P;
  long long np, m;
  GOp H;  // H0 (Q0) or H1 (Q1)
  GOp L[GMAXP];
  GCol C[GMAXP];
  double g[GMAXP];
  const double* inv;      // inv[l] = 1/sqrt(l(l+1))
  const double* tau_ptr;  // drop threshold (device, written by the expand step)
  long long npt;          // S (or J) scan slots: 32 pairs each
  int* heavy;             // heavy pair list (count pass appends, fill pass reads)
  int* nheavy;            // its length
  int* flags;             // header flags (F_* of sunfold.cu)
  int* dtot;              // [2 (n-1)]: S / J part lengths of the D rows (count pass -> fill pass)
  int cap;                // candidate buffer limit (testing: a small value forces the chunked
                          // and single-key paths); the engines use min(their buffer, cap)
  // light-row stash (sun_plan_set_stash; scap = 0: off): the count pass keeps the assembled
  // entries of each light pair's two rows (when both have <= scap entries), the fill pass
  // copies them to their offsets instead of assembling the rows again
  // (stash row r: S part at r scap, J part at + GW_CAP, D part at + 2 GW_CAP, as the D rows)
  int scap;               // entries per stashed row
  unsigned char* sflag;   // [np]: 1 = pair p's rows S_p (stash row p) and J_p (row np + p) are stashed
  int32_t* scol;          // [2 np][scap]
  double* sval;           // [2 np][scap]
  double* sK;             // [2 np]: K of the two rows
  int2* snj;              // [2 np]: S and J part lengths of the two rows
  // D-row stash (same buffer): row lam's S part at dcol/dval[(lam - 1) drow], its J part at
  // + dseg, its D part at + 2 dseg (the count pass writes the three parts while counting them;
  // rows whose S or J part exceeds dseg entries are assembled again by the fill); dseg = 0: off
  int dseg, drow;
  unsigned char* dflag;   // [n - 1]
  int32_t* dcol;          // [n - 1][drow]
  double* dval;           // [n - 1][drow]
  double* dK;             // [n - 1]
};

struct GOut {  // fill outputs (capacity-checked)
  int64_t* row_ptr;
  int32_t* col;
  double* val;
  long long cap;
  double* K;  // nullptr: not written (Q1)
  const long long* toff;
  const long long* nnz;
  long long dlim;  // > 0: D-part entries of a row beyond dlim are not written (stash rows)
};

constexpr int GSLOT = 32;  // pairs per scan slot (as modes 0/2: S slots, J slots, one slot per D row)

// Host side (sunfold_general.cu).  Layout of the general region of the workspace.
struct GLayout {
  size_t colcnt, cp, xr, heavy0, heavy1, nheavy, blk, dtot0, dtot1, total;
  long long xr_off[GMAXP];
  long long nrb;  // row blocks of the expand kernel
};
GLayout g_layout(int n, int P, const long long* nnzL, size_t base);

struct GExpandIn {
  const int64_t* rp[GMAXP + 2];
  const int32_t* ci[GMAXP + 2];
  const double2* v[GMAXP + 2];
  double gamma[GMAXP + 2];
  int nops, n, has_h1;
};
// expand (a1) for mode 3: CSR validation, ||.||_F^2, Hermiticity of H0/H1, inv[l], the drop
// thresholds (into the header at hdr_tau / hdr_flags ...), zeroing of the scan state, and the
// column access (CSC) of every dissipator.  `hdr` points to sunfold.cu's DevHeader.
struct GHeaderRef {
  int* flags;
  double* tau;               // [2]
  unsigned long long* herm;  // [2]
  double* nrm2_h;            // [2]
  double* nrm2;              // [nops]
  unsigned int* done;
  unsigned int* ticket;      // [2]
};
cudaError_t g_expand(const GExpandIn& in, char* ws, const GLayout& gl, double* inv, int* zero32, long long nz32,
                     unsigned long long* zero64, long long nz64, GHeaderRef hdr, cudaStream_t st);
// kernel attributes (dynamic shared memory); call outside any stream capture
cudaError_t g_prepare();
// count pass (a3) of one matrix: per-row counts and slot sums (modes 0/2 slot layout); the D
// rows on `aux` (ordered after `st` by the caller, joined afterwards)
cudaError_t g_count(const GProb& pr, int* cnt, int* ts, cudaStream_t st, cudaStream_t aux);
// fill pass (a5): row_ptr, col, val (and K); heavy rows on `aux`
cudaError_t g_fill(const GProb& pr, const int* cnt, const GOut& out, cudaStream_t st, cudaStream_t aux);
// light-row stash of one matrix: entries per row and bytes (0 when np = 0)
int g_stash_scap(int n);
size_t g_stash_bytes(int n);
// points G's stash at `base` (g_stash_bytes(n) bytes), or switches it off (base = nullptr)
void g_stash_set(GProb& G, char* base);
// kernels per count / fill call
constexpr int G_LAUNCHES_EXPAND = 4, G_LAUNCHES_COUNT = 3, G_LAUNCHES_FILL = 2;

}  // namespace sung
