// tq_trunc.cu — truncated tensor-train engine for sm_100a.
//
// One CTA per theta-set runs the whole TEBD program of the reference's simulate_tt
// (tt.py:186-244) on a train held in HBM, then evaluates every Pauli term's window.
// - One-site gates act in place on their core.  A single-site unitary preserves every
//   isometry, so the reference's centre move before it (tt.py:205-208) only changes the
//   gauge and is skipped.
// - Before a two-site gate the orthogonality centre moves onto the gate's left site
//   through isometric splits, which replace the reference's QR steps (tt.py:118-161).
// - The merged two-site block is split by a one-sided (Hestenes) Jacobi SVD in shared
//   memory.  Sigma goes to the thin side, and the spectrum is cut by the reference rule
//   (tt.py:85-115): sigma_i / sigma_max > eps, at most chi_max, renormalised by the kept
//   weight.  Rotations accumulate in V, so the isometric factor is exactly unitary even
//   when singular values vanish (the reference's eps = 0 keeps exact zeros).
// - Term values use full left/right norm environments plus one window per term
//   (hamiltonians.py:129-164).
// tests/mirror_trunc.py is the numpy mirror of exactly this algorithm.

#include <cuda_runtime.h>
#include "tq_debug.cuh"
#include <math.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/tq_trunc.h"

namespace tq {
extern thread_local char g_err[512];
}

namespace tqt {

template <typename R> struct CT;
template <> struct CT<float> { using T = float2; };
template <> struct CT<double> { using T = double2; };

template <typename C> __device__ __forceinline__ C cmk(decltype(C::x) x, decltype(C::x) y) { C r; r.x = x; r.y = y; return r; }
template <typename C> __device__ __forceinline__ C cconj(C a) { return cmk<C>(a.x, -a.y); }
template <typename C> __device__ __forceinline__ C cmul(C a, C b) { return cmk<C>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
template <typename C> __device__ __forceinline__ void cfma(C& acc, C a, C b) {   // acc += a b
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
}
template <typename C> __device__ __forceinline__ void cfmac(C& acc, C a, C b) {  // acc += conj(a) b
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(-a.y, b.x, acc.y);
}

constexpr int NT = 128;   // threads per CTA: six resident CTAs (theta-sets) per SM hide each other's Jacobi barriers
constexpr int NW = NT / 32;

template <typename R>
__device__ __forceinline__ R warp_sum(R v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// deterministic block-wide sum (fixed order: lanes, then warps)
__device__ double block_sum(double v, double* red) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < NW; ++w) t += red[w];
  __syncthreads();
  return t;
}

struct Params {
  int n, n_gates, batch, chi_cap, chi_max, n_terms;
  const tq_tgate* gates;
  const void* theta;
  int64_t theta_stride;
  double eps;
  const int32_t *term_lo, *term_hi, *code_off;
  const int8_t* codes;
  double2* values;
  double* discarded;
  double* norm2;
  int32_t* bonds;
  int32_t* flags;
  int32_t* centers;  // [B] orthogonality centre of each train (optional)
  void* cores;     // [B][n][2 cap^2] complex
  void* envl;      // [B][n+1][cap^2]
  void* envr;      // [B][n+1][cap^2]
  // straight-through tape (PH_TAPE writes it, PH_REPLAY reads it): per recorded theta-set and
  // two-site gate, the split's constant isometric factor (U_k, m x k, or Vh_k, k x n) in a slot
  // of 2 cap^2 complex, and its (k, side, rescale)
  void* tape;
  struct TapeMeta* meta;
  const int32_t* parent;   // PH_REPLAY: the recorded theta-set whose tape row b replays
  int32_t n2;              // two-site gates in the program (tape slots per theta-set)
  // optional input train (one train shared by every row, slot layout [n][2 cap^2], bonds [n+1]):
  // PH_RUN starts from it instead of |0...0>
  const void* init_cores;
  const int32_t* init_bonds;
  int32_t inplace;         // PH_RUN continues from the trains already in cores / bonds / centers
};

struct TapeMeta { int32_t k; int32_t left_iso; double scale; };

// Shared scratch of one CTA: X and V are (2cap) x (2cap) complex, column-major with leading
// dimension 2cap (Jacobi columns are contiguous, rows are spread over lanes).
template <typename R, int CAP>
struct Scratch {
  using C = typename CT<R>::T;
  static constexpr int LD = 2 * CAP;
  C X[LD * LD];
  C V[LD * LD];
  C G[16];
  R nrm[LD];
  int perm[LD];
  C hdiag[LD];   // Householder QR: diagonal of R
  R htau[LD];    //                 reflector scales
  double dred[NT / 32];
  int k;         // kept rank of the last split
  R scale;       // renormalisation of the kept weight
  double disc;   // discarded weight of the last split
};

// Orthogonalise the ncols columns (length nrows) of X; V (ncols x ncols) accumulates the
// rotations (X_out = X_in V).  Parallel round-robin ordering: one warp per column pair.
template <typename R, int CAP>
__device__ void jacobi(Scratch<R, CAP>& s, int nrows, int ncols) {
  using C = typename CT<R>::T;
  constexpr int LD = Scratch<R, CAP>::LD;
  const int tid = threadIdx.x;
  const R tol = sizeof(R) == 8 ? R(1e-14) : R(1e-6);
  const R tiny = sizeof(R) == 8 ? R(1e-280) : R(1e-35);
  const int max_sweeps = sizeof(R) == 8 ? 40 : 20;
  for (int e = tid; e < ncols * ncols; e += NT) {
    const int col = e / ncols, row = e - col * ncols;
    s.V[col * LD + row] = cmk<C>(row == col ? R(1) : R(0), R(0));
  }
  // squared Frobenius norm: a column below eps_mach * ||X|| is numerically zero, and rotating
  // pairs of such columns never converges in low precision (eps = 0 keeps exact zeros)
  double fro = 0.0;
  for (int e = tid; e < ncols * nrows; e += NT) {
    const int col = e / nrows, row = e - col * nrows;
    const C u = s.X[col * LD + row];
    fro += double(u.x) * u.x + double(u.y) * u.y;
  }
  fro = block_sum(fro, s.dred);
  const R floor2 = R(fro * (sizeof(R) == 8 ? 1e-30 : 1e-13));
  if (ncols < 2) return;
  const int np = ncols + (ncols & 1);
  // sub-warp groups: every pair of a round gets its own group when there are more pairs than
  // warps (64 columns -> 32 pairs on 32 half-warps), so a round is one pass
  const int sw = (np / 2 > NW) ? 16 : 32;
  const int grp = tid / sw, gl = tid % sw, ngrp = NT / sw;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    int any = 0;
    for (int round = 0; round < np - 1; ++round) {
      for (int pi0 = 0; pi0 < np / 2; pi0 += ngrp) {   // uniform trip count: shuffles stay converged
        const int pi = pi0 + grp;
        int p = 0, q = 0;
        bool live = pi < np / 2;
        if (live) {
          if (pi == 0) { p = round; q = np - 1; }
          else {                                        // (round +- pi) mod (np - 1), no integer division
            p = round + pi; if (p >= np - 1) p -= np - 1;
            q = round - pi; if (q < 0) q += np - 1;
          }
          if (p > q) { const int t = p; p = q; q = t; }
          live = q < ncols;   // bye for an odd column count
        }
        C* xp = s.X + p * LD;
        C* xq = s.X + q * LD;
        R a = R(0), b = R(0);
        C g = cmk<C>(R(0), R(0));
        if (live) {
          for (int r = gl; r < nrows; r += sw) {
            const C u = xp[r], v = xq[r];
            a = fma(u.x, u.x, fma(u.y, u.y, a));
            b = fma(v.x, v.x, fma(v.y, v.y, b));
            cfmac(g, u, v);
          }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          if (off < sw) {
            a += __shfl_xor_sync(0xffffffffu, a, off);
            b += __shfl_xor_sync(0xffffffffu, b, off);
            g.x += __shfl_xor_sync(0xffffffffu, g.x, off);
            g.y += __shfl_xor_sync(0xffffffffu, g.y, off);
          }
        }
        const R ag2 = g.x * g.x + g.y * g.y;
        // |g| <= tol sqrt(a b)  <=>  |g|^2 <= tol^2 a b  (no square roots on the convergence test)
        if (!live || !(ag2 > tol * tol * a * b) || ag2 < tiny * tiny || (a < floor2 && b < floor2)) continue;
        any = 1;
        const R inv = rsqrt(ag2), ag = ag2 * inv;
        const C e = cmk<C>(g.x * inv, g.y * inv);
        const R zeta = (b - a) * (R(0.5) * inv);
        R t;
        if (fabs(zeta) > R(1e30)) t = R(0.5) / zeta;
        else t = copysign(R(1), zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, R(1))));
        const R c = rsqrt(fma(t, t, R(1))), sn = c * t;
        (void)ag;
        const C se = cmk<C>(sn * e.x, sn * e.y);          // s e
        const C sec = cmk<C>(sn * e.x, -sn * e.y);        // s conj(e)
        for (int r = gl; r < nrows; r += sw) {
          const C u = xp[r], v = xq[r];
          C nu = cmk<C>(c * u.x, c * u.y), nv = cmk<C>(c * v.x, c * v.y);
          const C m1 = cmul(sec, v), m2 = cmul(se, u);
          nu.x -= m1.x; nu.y -= m1.y;
          nv.x += m2.x; nv.y += m2.y;
          xp[r] = nu; xq[r] = nv;
        }
        C* vp = s.V + p * LD;
        C* vq = s.V + q * LD;
        for (int r = gl; r < ncols; r += sw) {
          const C u = vp[r], v = vq[r];
          C nu = cmk<C>(c * u.x, c * u.y), nv = cmk<C>(c * v.x, c * v.y);
          const C m1 = cmul(sec, v), m2 = cmul(se, u);
          nu.x -= m1.x; nu.y -= m1.y;
          nv.x += m2.x; nv.y += m2.y;
          vp[r] = nu; vq[r] = nv;
        }
      }
      __syncthreads();
    }
    if (!__syncthreads_or(any)) break;
  }
}

// Column norms of X, descending stable ranking into perm, and the kept rank by the reference
// rule over the first r = min(m, n) values (truncate = false keeps all r, no rescale).
template <typename R, int CAP>
__device__ void rank_and_cut(Scratch<R, CAP>& s, int nrows, int ncols, int r, bool truncate,
                             double eps, int chi_max, int cap, int32_t* flag) {
  constexpr int LD = Scratch<R, CAP>::LD;
  const int tid = threadIdx.x;
  if (tid < ncols) {
    R acc = R(0);
    for (int i = 0; i < nrows; ++i) {
      const auto u = s.X[tid * LD + i];
      acc = fma(u.x, u.x, fma(u.y, u.y, acc));
    }
    const R v = sqrt(acc);
    if (!(v == v)) atomicMax(flag, 2);           // NaN (NotFinite) outranks a cap overflow (BondTooLarge)
    s.nrm[tid] = v == v ? v : R(0);              // keep the ranking a permutation
  }
  __syncthreads();
  if (tid < ncols) {
    const R mine = s.nrm[tid];
    int rank = 0;
    for (int i = 0; i < ncols; ++i) {
      const R o = s.nrm[i];
      rank += (o > mine) || (o == mine && i < tid);
    }
    s.perm[rank] = tid;
  }
  __syncthreads();
  if (tid == 0) {
    double total = 0.0;
    for (int i = 0; i < r; ++i) { const double v = s.nrm[s.perm[i]]; total += v * v; }
    int k = r;
    if (truncate) {
      const double s0 = s.nrm[s.perm[0]];
      if (eps > 0.0 && s0 > 0.0) {
        int cnt = 0;
        for (int i = 0; i < r; ++i) cnt += double(s.nrm[s.perm[i]]) > eps * s0;
        k = cnt > 1 ? cnt : 1;
      }
      if (chi_max > 0 && k > chi_max) k = chi_max;
    }
    if (k > cap) { atomicMax(flag, 1); k = cap; }
    double kept = 0.0;
    for (int i = 0; i < k; ++i) { const double v = s.nrm[s.perm[i]]; kept += v * v; }
    double disc = 0.0, scale = 1.0;
    if (truncate && total > 0.0) {
      disc = 1.0 - kept / total;
      if (disc < 0.0) disc = 0.0;
      scale = kept > 0.0 ? sqrt(total / kept) : 1.0;
    }
    if (!truncate) { disc = 0.0; scale = 1.0; }
    if (k < 1) k = 1;
    s.k = k; s.scale = R(scale); s.disc = disc;
  }
  __syncthreads();
}

// Householder QR of X (rows x cols, column-major): reflectors overwrite X below the diagonal,
// R's strict upper triangle stays in X and its diagonal goes to hdiag; Q (rows x k,
// k = min(rows, cols)) is accumulated into V.  Robust for rank-deficient X (a zero column
// gets tau = 0, so Q stays exactly isometric), which the reference's eps = 0 zeros need.
template <typename R, int CAP>
__device__ int house_qr(Scratch<R, CAP>& s, int rows, int cols) {
  using C = typename CT<R>::T;
  constexpr int LD = Scratch<R, CAP>::LD;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int k = rows < cols ? rows : cols;
  for (int j = 0; j < k; ++j) {
    if (warp == 0) {
      C* x = s.X + j * LD;
      R sig2 = R(0);
      for (int r = j + 1 + lane; r < rows; r += 32) sig2 = fma(x[r].x, x[r].x, fma(x[r].y, x[r].y, sig2));
      sig2 = warp_sum(sig2);
      const C x0 = x[j];
      const R a0 = sqrt(x0.x * x0.x + x0.y * x0.y);
      const R sig = sqrt(sig2 + a0 * a0);
      if (!(sig >= (sizeof(R) == 8 ? R(1e-150) : R(1e-18)))) {   // numerically zero column (or NaN): H = I
        if (lane == 0) { s.htau[j] = R(0); s.hdiag[j] = cmk<C>(R(0), R(0)); }
      } else {
        const C ph = a0 > R(0) ? cmk<C>(x0.x / a0, x0.y / a0) : cmk<C>(R(1), R(0));
        const C alpha = cmk<C>(-ph.x * sig, -ph.y * sig);          // H x = alpha e_j
        const C v0 = cmk<C>(x0.x - alpha.x, x0.y - alpha.y);
        const R vn2 = sig2 + v0.x * v0.x + v0.y * v0.y;
        if (lane == 0) { s.htau[j] = R(2) / vn2; s.hdiag[j] = alpha; x[j] = v0; }
      }
    }
    __syncthreads();
    const R tau = s.htau[j];
    if (tau != R(0)) {
      const C* v = s.X + j * LD;
      for (int c = j + 1 + warp; c < cols; c += NW) {          // X[j:, c] -= tau v (v^H X[j:, c])
        C* xc = s.X + c * LD;
        C w = cmk<C>(R(0), R(0));
        for (int r = j + lane; r < rows; r += 32) cfmac(w, v[r], xc[r]);
        w.x = warp_sum(w.x); w.y = warp_sum(w.y);
        w.x *= tau; w.y *= tau;
        for (int r = j + lane; r < rows; r += 32) { const C t = cmul(v[r], w); xc[r].x -= t.x; xc[r].y -= t.y; }
      }
    }
    __syncthreads();
  }
  // Q = H_0 ... H_{k-1} [I_k; 0], backward accumulation, one warp per column
  for (int e = tid; e < rows * k; e += NT) {
    const int c = e / rows, r = e - c * rows;
    s.V[c * LD + r] = cmk<C>(r == c ? R(1) : R(0), R(0));
  }
  __syncthreads();
  for (int j = k - 1; j >= 0; --j) {
    const R tau = s.htau[j];
    if (tau != R(0)) {
      const C* v = s.X + j * LD;
      for (int c = j + warp; c < k; c += NW) {                  // columns < j are untouched
        C* qc = s.V + c * LD;
        C w = cmk<C>(R(0), R(0));
        for (int r = j + lane; r < rows; r += 32) cfmac(w, v[r], qc[r]);
        w.x = warp_sum(w.x); w.y = warp_sum(w.y);
        w.x *= tau; w.y *= tau;
        for (int r = j + lane; r < rows; r += 32) { const C t = cmul(v[r], w); qc[r].x -= t.x; qc[r].y -= t.y; }
      }
    }
    __syncthreads();
  }
  return k;
}

// element (r, c) of R after house_qr
template <typename R, int CAP>
__device__ __forceinline__ typename CT<R>::T house_r(const Scratch<R, CAP>& s, int r, int c) {
  using C = typename CT<R>::T;
  constexpr int LD = Scratch<R, CAP>::LD;
  if (r == c) return s.hdiag[r];
  return r < c ? s.X[c * LD + r] : cmk<C>(R(0), R(0));
}

// centre c -> c + 1 (reference _shift_center_right, tt.py:118-122): core_c (2 chi_l x chi_r)
// = Q R, Q stays, R folds into core_{c+1}
template <typename R, int CAP>
__device__ void shift_right(Scratch<R, CAP>& s, typename CT<R>::T* cores, int32_t* dims, int c, int32_t*) {
  using C = typename CT<R>::T;
  constexpr int LD = Scratch<R, CAP>::LD;
  constexpr int SLOT = 2 * CAP * CAP;
  const int tid = threadIdx.x;
  const int cl = dims[c], cr = dims[c + 1], cr2 = dims[c + 2];
  C* A = cores + (size_t)c * SLOT;
  C* B = cores + (size_t)(c + 1) * SLOT;
  const int m = 2 * cl;
  for (int e = tid; e < m * cr; e += NT) {
    const int row = e / cr, col = e - row * cr;
    s.X[col * LD + row] = A[e];
  }
  __syncthreads();
  const int k = house_qr<R, CAP>(s, m, cr);
  for (int e = tid; e < m * k; e += NT) {
    const int row = e / k, rr = e - row * k;
    A[e] = s.V[rr * LD + row];
  }
  C* Rm = s.V + (size_t)LD * LD - k * cr;        // R (k x cr) in the tail of V (Q is consumed)
  __syncthreads();
  for (int e = tid; e < k * cr; e += NT) {
    const int rr = e / cr, col = e - rr * cr;
    Rm[e] = house_r<R, CAP>(s, rr, col);
  }
  const int nb = 2 * cr2;
  __syncthreads();
  for (int e = tid; e < cr * nb; e += NT) s.X[e] = B[e];   // stage core_{c+1} (cr x 2 cr2)
  __syncthreads();
  for (int e = tid; e < k * nb; e += NT) {
    const int rr = e / nb, col = e - rr * nb;
    C acc = cmk<C>(R(0), R(0));
    for (int i = rr; i < cr; ++i) cfma(acc, Rm[rr * cr + i], s.X[i * nb + col]);   // R upper triangular
    B[e] = acc;
  }
  __syncthreads();
  if (tid == 0) dims[c + 1] = k;
  __syncthreads();
}

// centre c -> c - 1 (reference _shift_center_left, tt.py:125-129): core_c^H (2 chi_r x chi_l)
// = Q R, so core_c = R^H Q^H; Q^H stays, R^H folds into core_{c-1}
template <typename R, int CAP>
__device__ void shift_left(Scratch<R, CAP>& s, typename CT<R>::T* cores, int32_t* dims, int c, int32_t*) {
  using C = typename CT<R>::T;
  constexpr int LD = Scratch<R, CAP>::LD;
  constexpr int SLOT = 2 * CAP * CAP;
  const int tid = threadIdx.x;
  const int cl0 = dims[c - 1], cl = dims[c], cr = dims[c + 1];
  C* A = cores + (size_t)c * SLOT;
  C* P = cores + (size_t)(c - 1) * SLOT;
  const int n = 2 * cr;                          // X = M^H : n rows x cl columns
  for (int e = tid; e < cl * n; e += NT) {
    const int i = e / n, j = e - i * n;        // M[i][j] = A flat [i * n + j]
    s.X[i * LD + j] = cconj(A[e]);
  }
  __syncthreads();
  const int k = house_qr<R, CAP>(s, n, cl);
  for (int e = tid; e < k * n; e += NT) {        // core_c[rr][col] = conj(Q[col][rr])
    const int rr = e / n, col = e - rr * n;
    A[e] = cconj(s.V[rr * LD + col]);
  }
  C* Lm = s.V + (size_t)LD * LD - cl * k;        // L = R^H (cl x k)
  __syncthreads();
  for (int e = tid; e < cl * k; e += NT) {
    const int i = e / k, rr = e - i * k;
    Lm[e] = cconj(house_r<R, CAP>(s, rr, i));
  }
  const int mp = 2 * cl0;
  __syncthreads();
  for (int e = tid; e < mp * cl; e += NT) s.X[e] = P[e];   // stage core_{c-1} (2 cl0 x cl)
  __syncthreads();
  for (int e = tid; e < mp * k; e += NT) {
    const int row = e / k, rr = e - row * k;
    C acc = cmk<C>(R(0), R(0));
    for (int i = rr; i < cl; ++i) cfma(acc, s.X[row * cl + i], Lm[i * k + rr]);      // L lower triangular
    P[e] = acc;
  }
  __syncthreads();
  if (tid == 0) dims[c] = k;
  __syncthreads();
}

// compress step at site c (reference compress, tt.py:311-318): core_c (chi_l x 2 chi_r) = (U S) Vh
// by one-sided Jacobi on its columns, truncated by (eps, chi_max) and renormalised; Vh stays,
// U S folds into core_{c-1}
template <typename R, int CAP>
__device__ void truncate_left(Scratch<R, CAP>& s, const Params& p, typename CT<R>::T* cores, int32_t* dims, int c,
                              double& disc_total, int32_t* flag) {
  using C = typename CT<R>::T;
  constexpr int LD = Scratch<R, CAP>::LD;
  constexpr int SLOT = 2 * CAP * CAP;
  const int tid = threadIdx.x;
  const int cl0 = dims[c - 1], cl = dims[c], cr = dims[c + 1];
  C* A = cores + (size_t)c * SLOT;
  C* P = cores + (size_t)(c - 1) * SLOT;
  const int n = 2 * cr;
  for (int e = tid; e < cl * n; e += NT) {
    const int i = e / n, j = e - i * n;
    s.X[j * LD + i] = A[e];
  }
  __syncthreads();
  jacobi<R, CAP>(s, cl, n);
  rank_and_cut<R, CAP>(s, cl, n, cl < n ? cl : n, true, p.eps, p.chi_max, p.chi_cap, flag);
  const int k = s.k;
  const R sc = s.scale;
  for (int e = tid; e < k * n; e += NT) {        // core_c[rr][col] = conj(V[perm[rr]][col])
    const int rr = e / n, col = e - rr * n;
    A[e] = cconj(s.V[s.perm[rr] * LD + col]);
  }
  C* Lm = s.V + (size_t)LD * LD - cl * k;        // (U S)[i][rr] = X[perm[rr]][i] * scale
  __syncthreads();
  for (int e = tid; e < cl * k; e += NT) {
    const int i = e / k, rr = e - i * k;
    const C x = s.X[s.perm[rr] * LD + i];
    Lm[e] = cmk<C>(x.x * sc, x.y * sc);
  }
  const int mp = 2 * cl0;
  __syncthreads();
  for (int e = tid; e < mp * cl; e += NT) s.X[e] = P[e];
  __syncthreads();
  for (int e = tid; e < mp * k; e += NT) {
    const int row = e / k, rr = e - row * k;
    C acc = cmk<C>(R(0), R(0));
    for (int i = 0; i < cl; ++i) cfma(acc, s.X[row * cl + i], Lm[i * k + rr]);
    P[e] = acc;
  }
  __syncthreads();
  if (tid == 0) dims[c] = k;
  disc_total += s.disc;
  __syncthreads();
}

template <typename R>
__device__ void gate_matrix(const tq_tgate& g, const R* theta_b, typename CT<R>::T* G) {
  using C = typename CT<R>::T;
  const int d = g.kind == 1 ? 2 : 4;
  for (int i = 0; i < d * d; ++i) G[i] = cmk<C>(R(g.m[2 * i]), R(g.m[2 * i + 1]));
  if (g.rot == 0) return;
  const double t = double(theta_b[g.slot]);
  double sn, cs;
  sincos(0.5 * t, &sn, &cs);
  const R c = R(cs), s = R(sn), z = R(0);
  if (g.rot == 1) { G[0] = cmk<C>(c, z); G[1] = cmk<C>(z, -s); G[2] = cmk<C>(z, -s); G[3] = cmk<C>(c, z); }
  else if (g.rot == 2) { G[0] = cmk<C>(c, z); G[1] = cmk<C>(-s, z); G[2] = cmk<C>(s, z); G[3] = cmk<C>(c, z); }
  else if (g.rot == 3) { G[0] = cmk<C>(c, -s); G[1] = cmk<C>(z, z); G[2] = cmk<C>(z, z); G[3] = cmk<C>(c, s); }
  else {   // crz, control on the first wire; flip swaps the legs
    for (int i = 0; i < 16; ++i) G[i] = cmk<C>(z, z);
    G[0] = cmk<C>(R(1), z); G[5] = cmk<C>(R(1), z);
    G[10] = cmk<C>(c, -s); G[15] = cmk<C>(c, s);
    if (g.flip) { G[5] = cmk<C>(c, -s); G[10] = cmk<C>(R(1), z); }
  }
}

template <typename R, int CAP>
__device__ void two_site(Scratch<R, CAP>& s, const Params& p, typename CT<R>::T* cores, int32_t* dims, int i,
                         double& disc_total, int32_t* flag) {
  using C = typename CT<R>::T;
  constexpr int LD = Scratch<R, CAP>::LD;
  constexpr int SLOT = 2 * CAP * CAP;
  const int tid = threadIdx.x;
  const int cl = dims[i], cm = dims[i + 1], cr = dims[i + 2];
  C* A = cores + (size_t)i * SLOT;
  C* B = cores + (size_t)(i + 1) * SLOT;
  const int m = 2 * cl, n = 2 * cr;
  const bool left_iso = m <= n;                   // sigma to the right (tt.py:112-115)
  C* As = s.V;
  C* Bs = s.V + SLOT;
  for (int e = tid; e < cl * 2 * cm; e += NT) As[e] = A[e];
  for (int e = tid; e < cm * 2 * cr; e += NT) Bs[e] = B[e];
  __syncthreads();
  for (int e = tid; e < cl * cr; e += NT) {
    const int a = e / cr, b = e - a * cr;
    C t[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) t[q] = cmk<C>(R(0), R(0));
    for (int mid = 0; mid < cm; ++mid) {
      const C a0 = As[(a * 2 + 0) * cm + mid], a1 = As[(a * 2 + 1) * cm + mid];
      const C b0 = Bs[(mid * 2 + 0) * cr + b], b1 = Bs[(mid * 2 + 1) * cr + b];
      cfma(t[0], a0, b0); cfma(t[1], a0, b1); cfma(t[2], a1, b0); cfma(t[3], a1, b1);
    }
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      C acc = cmk<C>(R(0), R(0));
#pragma unroll
      for (int q = 0; q < 4; ++q) cfma(acc, s.G[o * 4 + q], t[q]);
      const int row = a * 2 + (o >> 1), col = (o & 1) * cr + b;
      if (left_iso) s.X[row * LD + col] = cconj(acc);   // X = M^H
      else s.X[col * LD + row] = acc;                   // X = M
    }
  }
  __syncthreads();
  const int nrows = left_iso ? n : m, ncols = left_iso ? m : n;
  jacobi<R, CAP>(s, nrows, ncols);
  rank_and_cut<R, CAP>(s, nrows, ncols, m < n ? m : n, true, p.eps, p.chi_max, p.chi_cap, flag);
  const int k = s.k;
  const R sc = s.scale;
  if (left_iso) {
    for (int e = tid; e < m * k; e += NT) {       // core_i[(a,s0)][rr] = V[perm[rr]][(a,s0)]
      const int row = e / k, rr = e - row * k;
      A[e] = s.V[s.perm[rr] * LD + row];
    }
    for (int e = tid; e < k * n; e += NT) {       // core_{i+1}[rr][col] = conj(X[perm[rr]][col]) * scale
      const int rr = e / n, col = e - rr * n;
      const C x = s.X[s.perm[rr] * LD + col];
      B[e] = cmk<C>(x.x * sc, -x.y * sc);
    }
  } else {
    for (int e = tid; e < m * k; e += NT) {       // core_i[(a,s0)][rr] = X[perm[rr]][(a,s0)] * scale
      const int row = e / k, rr = e - row * k;
      const C x = s.X[s.perm[rr] * LD + row];
      A[e] = cmk<C>(x.x * sc, x.y * sc);
    }
    for (int e = tid; e < k * n; e += NT) {       // core_{i+1}[rr][col] = conj(V[perm[rr]][col])
      const int rr = e / n, col = e - rr * n;
      B[e] = cconj(s.V[s.perm[rr] * LD + col]);
    }
  }
  __syncthreads();
  if (tid == 0) dims[i + 1] = k;
  disc_total += s.disc;
  __syncthreads();
}

// Straight-through split replay (reference _tt_taped_split, autodiff.py:315-336): the merged,
// gated block M (m x n) is split with the RECORDED constant factor of the unshifted run instead
// of a fresh SVD -- left = U_k, right = rescale U_k^H M when m <= n; right = Vh_k,
// left = rescale M Vh_k^H otherwise.  The tape's value as a function of one angle (constants
// frozen) is a trigonometric polynomial, so shifted replays give its exact derivative.
template <typename R, int CAP>
__device__ void replay_two_site(Scratch<R, CAP>& s, typename CT<R>::T* cores, int32_t* dims, int i,
                                const typename CT<R>::T* iso, TapeMeta mt) {
  using C = typename CT<R>::T;
  constexpr int SLOT = 2 * CAP * CAP;
  const int tid = threadIdx.x;
  const int cl = dims[i], cm = dims[i + 1], cr = dims[i + 2];
  C* A = cores + (size_t)i * SLOT;
  C* B = cores + (size_t)(i + 1) * SLOT;
  const int m = 2 * cl, n = 2 * cr, k = mt.k;
  const R sc = R(mt.scale);
  C* As = s.V;
  C* Bs = s.V + SLOT;
  C* M = s.X;                                     // row-major m x n
  for (int e = tid; e < cl * 2 * cm; e += NT) As[e] = A[e];
  for (int e = tid; e < cm * 2 * cr; e += NT) Bs[e] = B[e];
  __syncthreads();
  for (int e = tid; e < cl * cr; e += NT) {
    const int a = e / cr, b = e - a * cr;
    C t[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) t[q] = cmk<C>(R(0), R(0));
    for (int mid = 0; mid < cm; ++mid) {
      const C a0 = As[(a * 2 + 0) * cm + mid], a1 = As[(a * 2 + 1) * cm + mid];
      const C b0 = Bs[(mid * 2 + 0) * cr + b], b1 = Bs[(mid * 2 + 1) * cr + b];
      cfma(t[0], a0, b0); cfma(t[1], a0, b1); cfma(t[2], a1, b0); cfma(t[3], a1, b1);
    }
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      C acc = cmk<C>(R(0), R(0));
#pragma unroll
      for (int q = 0; q < 4; ++q) cfma(acc, s.G[o * 4 + q], t[q]);
      M[(a * 2 + (o >> 1)) * n + (o & 1) * cr + b] = acc;
    }
  }
  __syncthreads();
  if (mt.left_iso) {
    for (int e = tid; e < m * k; e += NT) A[e] = iso[e];
    for (int e = tid; e < k * n; e += NT) {
      const int rr = e / n, col = e - rr * n;
      C acc = cmk<C>(R(0), R(0));
      for (int row = 0; row < m; ++row) cfmac(acc, iso[row * k + rr], M[row * n + col]);
      B[e] = cmk<C>(acc.x * sc, acc.y * sc);
    }
  } else {
    for (int e = tid; e < k * n; e += NT) B[e] = iso[e];
    for (int e = tid; e < m * k; e += NT) {
      const int row = e / k, rr = e - row * k;
      C acc = cmk<C>(R(0), R(0));
      for (int col = 0; col < n; ++col) {   // acc += M[row][col] conj(Vh[rr][col])
        const C x = M[row * n + col], v = iso[rr * n + col];
        acc.x = fma(x.x, v.x, fma(x.y, v.y, acc.x));
        acc.y = fma(x.y, v.x, fma(-x.x, v.y, acc.y));
      }
      A[e] = cmk<C>(acc.x * sc, acc.y * sc);
    }
  }
  __syncthreads();
  if (tid == 0) dims[i + 1] = k;
  __syncthreads();
}

// ---- environments and term windows ---------------------------------------------------------
// x' [c][d] = sum_{a,s,s'} conj(A[a][s][c]) P[s][s'] x[a][b] A[b][s'][d]   (P = I for code 0)
template <typename R, int CAP>
__device__ void left_step(Scratch<R, CAP>& s, const typename CT<R>::T* A, int ca, int cb, int code,
                          const typename CT<R>::T* x, typename CT<R>::T* out) {
  using C = typename CT<R>::T;
  const int tid = threadIdx.x;
  C* T = s.X;                                     // T[a][(s', d)] = sum_b x[a][b] A[b][s'][d]
  const int w = 2 * cb;
  for (int e = tid; e < ca * w; e += NT) {
    const int a = e / w, col = e - a * w;
    C acc = cmk<C>(R(0), R(0));
    for (int b = 0; b < ca; ++b) cfma(acc, x[a * ca + b], A[b * w + col]);
    T[e] = acc;
  }
  __syncthreads();
  for (int e = tid; e < cb * cb; e += NT) {
    const int c = e / cb, d = e - c * cb;
    C acc = cmk<C>(R(0), R(0));
    for (int a = 0; a < ca; ++a) {
#pragma unroll
      for (int sp = 0; sp < 2; ++sp) {
        // (P T)[a][(sp, d)] with one nonzero per Pauli row
        C u;
        const C t0 = T[a * w + 0 * cb + d], t1 = T[a * w + 1 * cb + d];
        if (code == 0) u = sp == 0 ? t0 : t1;
        else if (code == 1) u = sp == 0 ? t1 : t0;
        else if (code == 2) u = sp == 0 ? cmk<C>(t1.y, -t1.x) : cmk<C>(-t0.y, t0.x);
        else u = sp == 0 ? t0 : cmk<C>(-t1.x, -t1.y);
        cfmac(acc, A[a * w + sp * cb + c], u);
      }
    }
    out[e] = acc;
  }
  __syncthreads();
}

// R_k[a][b] = sum_{s,c,d} conj(A[a][s][c]) R[c][d] A[b][s][d]
template <typename R, int CAP>
__device__ void right_step(Scratch<R, CAP>& s, const typename CT<R>::T* A, int ca, int cb,
                           const typename CT<R>::T* rin, typename CT<R>::T* out) {
  using C = typename CT<R>::T;
  const int tid = threadIdx.x;
  C* T = s.X;                                     // T[(b, s)][c] = sum_d R[c][d] A[b][s][d]
  for (int e = tid; e < 2 * ca * cb; e += NT) {
    const int bs = e / cb, c = e - bs * cb;
    C acc = cmk<C>(R(0), R(0));
    for (int d = 0; d < cb; ++d) cfma(acc, rin[c * cb + d], A[bs * cb + d]);
    T[e] = acc;
  }
  __syncthreads();
  for (int e = tid; e < ca * ca; e += NT) {
    const int a = e / ca, b = e - a * ca;
    C acc = cmk<C>(R(0), R(0));
    for (int sp = 0; sp < 2; ++sp)
      for (int c = 0; c < cb; ++c) cfmac(acc, A[(a * 2 + sp) * cb + c], T[(b * 2 + sp) * cb + c]);
    out[e] = acc;
  }
  __syncthreads();
}

constexpr int PH_RUN = 1, PH_COMPRESS = 2, PH_VALUES = 4;
// straight-through gradient: PH_TAPE runs the reference's TAPED state construction
// (_tt_taped_state, autodiff.py:339-363: no centre moves, every two-site gate split as in
// _tt_taped_split) and records each split's constant factor; PH_REPLAY re-runs it at shifted
// angles with those factors frozen
constexpr int PH_TAPE = 8, PH_REPLAY = 16;

template <typename R, int CAP, int PHASE>
// Six resident 128-thread CTAs per SM (80 registers, no spills; 34 KB shared memory each):
// f3 7893 sims/s at 4 x SMs theta-sets with 4 per SM -> 9339 at 6 x SMs with 6 per SM
// (same-box A/B; 5 per SM: 8813 at 5 x SMs).
#ifndef TQT_MINB
#define TQT_MINB 6
#endif
__global__ void __launch_bounds__(NT, TQT_MINB) tt_kernel(Params p) {
  using C = typename CT<R>::T;
  constexpr int SLOT = 2 * CAP * CAP;
  constexpr int ESLOT = CAP * CAP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TQ_SMEM_POISON(smem_raw);
  Scratch<R, CAP>& s = *reinterpret_cast<Scratch<R, CAP>*>(smem_raw);
  const int b = blockIdx.x;
  const int tid = threadIdx.x;
  const int n = p.n;
  C* cores = reinterpret_cast<C*>(p.cores) + (size_t)b * n * SLOT;
  C* envl = reinterpret_cast<C*>(p.envl) + (size_t)b * (n + 1) * ESLOT;
  C* envr = reinterpret_cast<C*>(p.envr) + (size_t)b * (n + 1) * ESLOT;
  int32_t* dims = p.bonds + (size_t)b * (n + 1);
  int32_t* flag = p.flags + b;
  if constexpr ((PHASE & PH_RUN) != 0) {
  const R* theta_b = reinterpret_cast<const R*>(p.theta) + (int64_t)b * p.theta_stride;
  if (p.inplace) {
    // the row's own train (cores, dims and centre as the caller left them) is the input state
  } else if (p.init_cores) {   // a caller's train (reference TTState) as the input state
    const C* src = reinterpret_cast<const C*>(p.init_cores);
    for (int k = 0; k < n; ++k) {
      const int cnt = p.init_bonds[k] * 2 * p.init_bonds[k + 1];
      for (int e = tid; e < cnt; e += NT) cores[(size_t)k * SLOT + e] = src[(size_t)k * SLOT + e];
    }
    for (int k = tid; k <= n; k += NT) dims[k] = p.init_bonds[k];
  } else {   // |0...0>: bond 1 everywhere
    for (int k = tid; k < n; k += NT) {
      cores[(size_t)k * SLOT + 0] = cmk<C>(R(1), R(0));
      cores[(size_t)k * SLOT + 1] = cmk<C>(R(0), R(0));
    }
    for (int k = tid; k <= n; k += NT) dims[k] = 1;
  }
  __syncthreads();
  int center = (p.inplace && p.centers) ? p.centers[b] : 0;
  double disc = 0.0;
  constexpr bool TAPED = (PHASE & (PH_TAPE | PH_REPLAY)) != 0;
  constexpr int TSLOT = 2 * CAP * CAP;
  int j2 = 0;   // two-site gates so far (tape slot)
  for (int gi = 0; gi < p.n_gates; ++gi) {
    const tq_tgate& g = p.gates[gi];
    if (tid == 0) gate_matrix<R>(g, theta_b, s.G);
    __syncthreads();
    const int site = g.site;
    if (g.kind == 1) {
      const int cl = dims[site], cr = dims[site + 1];
      C* A = cores + (size_t)site * SLOT;
      for (int e = tid; e < cl * cr; e += NT) {
        const int a = e / cr, bb = e - a * cr;
        const C x0 = A[(a * 2 + 0) * cr + bb], x1 = A[(a * 2 + 1) * cr + bb];
        C y0 = cmk<C>(R(0), R(0)), y1 = y0;
        cfma(y0, s.G[0], x0); cfma(y0, s.G[1], x1);
        cfma(y1, s.G[2], x0); cfma(y1, s.G[3], x1);
        A[(a * 2 + 0) * cr + bb] = y0; A[(a * 2 + 1) * cr + bb] = y1;
      }
      __syncthreads();
      continue;
    }
    if constexpr (TAPED) {
      if constexpr ((PHASE & PH_REPLAY) != 0) {
        const size_t slot = (size_t)p.parent[b] * p.n2 + j2;
        replay_two_site<R, CAP>(s, cores, dims, site, reinterpret_cast<const C*>(p.tape) + slot * TSLOT, p.meta[slot]);
      } else {
        const int m = 2 * dims[site], nn = 2 * dims[site + 2];
        two_site<R, CAP>(s, p, cores, dims, site, disc, flag);
        const size_t slot = (size_t)b * p.n2 + j2;
        const int k = dims[site + 1];
        C* dst = reinterpret_cast<C*>(p.tape) + slot * TSLOT;
        const C* src = cores + (size_t)(m <= nn ? site : site + 1) * SLOT;   // the constant factor
        const int cnt = m <= nn ? m * k : k * nn;
        for (int e = tid; e < cnt; e += NT) dst[e] = src[e];
        if (tid == 0) { p.meta[slot].k = k; p.meta[slot].left_iso = m <= nn; p.meta[slot].scale = double(s.scale); }
        __syncthreads();
      }
      ++j2;
      continue;
    }
    while (center < site) { shift_right<R, CAP>(s, cores, dims, center, flag); ++center; }
    while (center > site) { shift_left<R, CAP>(s, cores, dims, center, flag); --center; }
    const int m = 2 * dims[site], nn = 2 * dims[site + 2];
    two_site<R, CAP>(s, p, cores, dims, site, disc, flag);
    center = m <= nn ? site + 1 : site;
  }
  if (tid == 0) {
    if (p.discarded) p.discarded[b] = (p.inplace ? p.discarded[b] : 0.0) + disc;   // in place: accumulates
    if (p.centers) p.centers[b] = center;
  }
  __syncthreads();
  }
  if constexpr ((PHASE & PH_COMPRESS) != 0) {
    // reference compress (tt.py:299-320): QR sweep to the right end, then truncating SVD
    // steps back to site 0; the centre ends at 0
    for (int c = 0; c < n - 1; ++c) shift_right<R, CAP>(s, cores, dims, c, flag);
    double disc = 0.0;
    for (int c = n - 1; c >= 1; --c) truncate_left<R, CAP>(s, p, cores, dims, c, disc, flag);
    if (tid == 0) { p.discarded[b] += disc; if (p.centers) p.centers[b] = 0; }
    __syncthreads();
  }
  if constexpr ((PHASE & PH_VALUES) == 0) return;
  // norm environments
  if (tid == 0) { envl[0] = cmk<C>(R(1), R(0)); envr[(size_t)n * ESLOT] = cmk<C>(R(1), R(0)); }
  __syncthreads();
  for (int k = 0; k < n; ++k)
    left_step<R, CAP>(s, cores + (size_t)k * SLOT, dims[k], dims[k + 1], 0, envl + (size_t)k * ESLOT,
                      envl + (size_t)(k + 1) * ESLOT);
  if (tid == 0 && p.norm2) p.norm2[b] = double(envl[(size_t)n * ESLOT].x);   // <psi|psi>
  for (int k = n - 1; k >= 0; --k)
    right_step<R, CAP>(s, cores + (size_t)k * SLOT, dims[k], dims[k + 1], envr + (size_t)(k + 1) * ESLOT,
                       envr + (size_t)k * ESLOT);
  // term windows: x = L_lo, one left step per site (Pauli or identity), closed with R_{hi+1}
  C* xa = s.V;
  C* xb = s.V + ESLOT;
  for (int t = 0; t < p.n_terms; ++t) {
    const int lo = p.term_lo[t], hi = p.term_hi[t];
    if (hi < lo) {   // an empty term: 1 (untaped expval), <psi|psi> on the tape (_tt_term_nodes)
      if (tid == 0) {
        const C nrm = envl[(size_t)n * ESLOT];
        p.values[(size_t)b * p.n_terms + t] =
            (PHASE & (PH_TAPE | PH_REPLAY)) ? make_double2(double(nrm.x), double(nrm.y)) : make_double2(1.0, 0.0);
      }
      continue;
    }
    const int c0 = dims[lo];
    for (int e = tid; e < c0 * c0; e += NT) xa[e] = envl[(size_t)lo * ESLOT + e];
    __syncthreads();
    C* cur = xa;
    C* nxt = xb;
    for (int k = lo; k <= hi; ++k) {
      left_step<R, CAP>(s, cores + (size_t)k * SLOT, dims[k], dims[k + 1], p.codes[p.code_off[t] + (k - lo)], cur, nxt);
      C* tmp = cur; cur = nxt; nxt = tmp;
    }
    const int ce = dims[hi + 1];
    const C* rr = envr + (size_t)(hi + 1) * ESLOT;
    double re = 0.0, im = 0.0;
    for (int e = tid; e < ce * ce; e += NT) {   // sum_ab x[a][b] R[a][b]
      const C x = cur[e], r = rr[e];
      re += double(x.x) * r.x - double(x.y) * r.y;
      im += double(x.x) * r.y + double(x.y) * r.x;
    }
    __shared__ double red_re[NT], red_im[NT];
    red_re[tid] = re; red_im[tid] = im;
    __syncthreads();
    for (int h = NT / 2; h > 0; h >>= 1) {
      if (tid < h) { red_re[tid] += red_re[tid + h]; red_im[tid] += red_im[tid + h]; }
      __syncthreads();
    }
    if (tid == 0) p.values[(size_t)b * p.n_terms + t] = make_double2(red_re[0], red_im[0]);
    __syncthreads();
  }
}

// <a_b|b_b> of two trains per batch row (reference tt_inner, tt.py:247-255): left-to-right
// transfer env' = sum_s A_s^H env B_s, A conjugated.  One CTA per row.
template <typename R, int CAP>
__global__ void __launch_bounds__(NT, 1) tt_inner_kernel(int n, const void* cores_a, const int32_t* bonds_a,
                                                         const void* cores_b, const int32_t* bonds_b, double2* out) {
  using C = typename CT<R>::T;
  constexpr int SLOT = 2 * CAP * CAP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TQ_SMEM_POISON(smem_raw);
  Scratch<R, CAP>& s = *reinterpret_cast<Scratch<R, CAP>*>(smem_raw);
  const int row = blockIdx.x, tid = threadIdx.x;
  const C* A = reinterpret_cast<const C*>(cores_a) + (size_t)row * n * SLOT;
  const C* B = reinterpret_cast<const C*>(cores_b) + (size_t)row * n * SLOT;
  const int32_t* da = bonds_a + (size_t)row * (n + 1);
  const int32_t* db = bonds_b + (size_t)row * (n + 1);
  C* env = s.V;                 // [ca][cb]
  C* T = s.X;                   // [ca][(s, d)]
  if (tid == 0) env[0] = cmk<C>(R(1), R(0));
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    const int ca = da[k], cb = db[k], ca2 = da[k + 1], cb2 = db[k + 1];
    const C* Ak = A + (size_t)k * SLOT;
    const C* Bk = B + (size_t)k * SLOT;
    const int w = 2 * cb2;
    for (int e = tid; e < ca * w; e += NT) {      // T[a][(s, d)] = sum_b env[a][b] B[b][s][d]
      const int a = e / w, col = e - a * w;
      C acc = cmk<C>(R(0), R(0));
      for (int bb = 0; bb < cb; ++bb) cfma(acc, env[a * cb + bb], Bk[bb * w + col]);
      T[e] = acc;
    }
    __syncthreads();
    for (int e = tid; e < ca2 * cb2; e += NT) {   // env'[c][d] = sum_{a,s} conj(A[a][s][c]) T[a][(s, d)]
      const int c = e / cb2, d = e - c * cb2;
      C acc = cmk<C>(R(0), R(0));
      for (int a = 0; a < ca; ++a)
#pragma unroll
        for (int sp = 0; sp < 2; ++sp) cfmac(acc, Ak[(a * 2 + sp) * ca2 + c], T[a * w + sp * cb2 + d]);
      env[e] = acc;
    }
    __syncthreads();
  }
  if (tid == 0) out[row] = make_double2(double(env[0].x), double(env[0].y));
}

template <typename R, int CAP, int PHASE>
static tq_status launch(const Params& p, cudaStream_t st) {
  const size_t smem = sizeof(Scratch<R, CAP>);
  if (smem > 227 * 1024) {
    snprintf(tq::g_err, sizeof(tq::g_err), "truncated engine: bond capacity %d needs %zu bytes of shared memory", CAP, smem);
    return TQ_ERR_UNSUPPORTED;
  }
  cudaFuncSetAttribute(tt_kernel<R, CAP, PHASE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tt_kernel<R, CAP, PHASE><<<p.batch, NT, smem, st>>>(p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(tq::g_err, sizeof(tq::g_err), "%s", cudaGetErrorString(e));
    return TQ_ERR_CUDA;
  }
  return TQ_OK;
}

static int cap_bucket(int chi) { int c = 4; while (c < chi) c <<= 1; return c; }

static size_t align256(size_t x) { return (x + 255) / 256 * 256; }

template <int PHASE>
static tq_status dispatch(const Params& p, int dtype, cudaStream_t st) {
  const int c = cap_bucket(p.chi_cap);
  if (dtype == TQ_C128) {
    if (c <= 4) return launch<double, 4, PHASE>(p, st);
    if (c <= 8) return launch<double, 8, PHASE>(p, st);
    if (c <= 16) return launch<double, 16, PHASE>(p, st);
    return launch<double, 32, PHASE>(p, st);
  }
  if (c <= 4) return launch<float, 4, PHASE>(p, st);
  if (c <= 8) return launch<float, 8, PHASE>(p, st);
  if (c <= 16) return launch<float, 16, PHASE>(p, st);
  return launch<float, 32, PHASE>(p, st);
}

static size_t state_bytes(int n, int batch, int cap, int dtype) {
  const size_t csz = dtype == TQ_C128 ? 16 : 8;
  const int c = cap_bucket(cap);
  return (size_t)batch * n * 2 * c * c * csz;
}

static size_t env_bytes(int n, int batch, int cap, int dtype) {
  const size_t csz = dtype == TQ_C128 ? 16 : 8;
  const int c = cap_bucket(cap);
  return 2 * align256((size_t)batch * (n + 1) * c * c * csz);
}

static bool bad_sizes(const char* who, int n, int batch, int cap, int dtype) {
  if (n < 1 || batch < 1 || cap < 1 || cap > 32 || (dtype != TQ_C64 && dtype != TQ_C128)) {
    snprintf(tq::g_err, sizeof(tq::g_err), "%s: invalid sizes (n=%d batch=%d cap=%d)", who, n, batch, cap);
    return true;
  }
  return false;
}

struct WsParts { size_t cores, envl, envr, total; };

static WsParts ws_parts(int n, int batch, int cap, int dtype) {
  const size_t csz = dtype == TQ_C128 ? 16 : 8;
  const int c = cap_bucket(cap);
  WsParts w{};
  w.cores = 0;
  w.envl = align256((size_t)batch * n * 2 * c * c * csz);
  w.envr = w.envl + align256((size_t)batch * (n + 1) * c * c * csz);
  w.total = w.envr + align256((size_t)batch * (n + 1) * c * c * csz);
  return w;
}

__global__ void dfma_probe(double* out, int iters, double seed) {
  double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  const double r = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (r == 12345.678) out[blockIdx.x] = r;
}

}  // namespace tqt

extern "C" {

tq_status tq_tt_dfma_peak(int32_t iters, void* stream, double* tflops_out) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double) * sms * 8) != cudaSuccess) {
    snprintf(tq::g_err, sizeof(tq::g_err), "cudaMalloc failed");
    return TQ_ERR_CUDA;
  }
  const int blocks = sms * 8, threads = 256;
  tqt::dfma_probe<<<blocks, threads, 0, st>>>(out, 4, 1.0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  tqt::dfma_probe<<<blocks, threads, 0, st>>>(out, iters, 1.0);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0); cudaEventDestroy(e1);
  cudaFree(out);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(tq::g_err, sizeof(tq::g_err), "%s", cudaGetErrorString(e));
    return TQ_ERR_CUDA;
  }
  *tflops_out = 2.0 * 8 * 16 * (double)iters * blocks * threads / (ms * 1e-3) / 1e12;
  return TQ_OK;
}


size_t tq_tt_workspace_bytes(int n_qubits, int batch, int chi_cap, int dtype) {
  if (n_qubits < 1 || batch < 1 || chi_cap < 1) return 0;
  return tqt::ws_parts(n_qubits, batch, chi_cap, dtype).total;
}

tq_status tq_tt_simulate(int n_qubits, const void* gates, int n_gates, int dtype, int batch,
                         const void* theta, int64_t theta_stride, double eps, int chi_cap, int chi_max,
                         const int32_t* term_lo, const int32_t* term_hi, const int32_t* code_off,
                         const int8_t* codes, int n_terms, void* values, double* discarded,
                         double* norm2, int32_t* bonds, int32_t* flags, void* workspace,
                         size_t workspace_bytes, void* stream) {
  using namespace tqt;
  if (n_qubits < 1 || batch < 1 || n_gates < 0 || n_terms < 0 || chi_cap < 1 || chi_cap > 32 ||
      (dtype != TQ_C64 && dtype != TQ_C128)) {
    snprintf(tq::g_err, sizeof(tq::g_err), "tq_tt_simulate: invalid sizes (n=%d batch=%d cap=%d)", n_qubits, batch, chi_cap);
    return TQ_ERR_INPUT;
  }
  const WsParts w = ws_parts(n_qubits, batch, chi_cap, dtype);
  if (workspace_bytes < w.total) {
    snprintf(tq::g_err, sizeof(tq::g_err), "tq_tt_simulate: workspace %zu < %zu bytes", workspace_bytes, w.total);
    return TQ_ERR_WORKSPACE;
  }
  Params p{};
  p.n = n_qubits; p.n_gates = n_gates; p.batch = batch; p.chi_cap = chi_cap; p.chi_max = chi_max;
  p.n_terms = n_terms; p.gates = reinterpret_cast<const tq_tgate*>(gates); p.theta = theta;
  p.theta_stride = theta_stride; p.eps = eps; p.term_lo = term_lo; p.term_hi = term_hi;
  p.code_off = code_off; p.codes = codes; p.values = reinterpret_cast<double2*>(values);
  p.discarded = discarded; p.norm2 = norm2; p.bonds = bonds; p.flags = flags;
  unsigned char* base = reinterpret_cast<unsigned char*>(workspace);
  p.cores = base + w.cores; p.envl = base + w.envl; p.envr = base + w.envr;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaMemsetAsync(flags, 0, sizeof(int32_t) * batch, st);
  return dispatch<PH_RUN | PH_VALUES>(p, dtype, st);
}

size_t tq_tt_state_bytes(int n_qubits, int batch, int chi_cap, int dtype) {
  if (n_qubits < 1 || batch < 1 || chi_cap < 1) return 0;
  return tqt::state_bytes(n_qubits, batch, chi_cap, dtype);
}

tq_status tq_tt_run(int n_qubits, const void* gates, int n_gates, int dtype, int batch, const void* theta,
                    int64_t theta_stride, double eps, int chi_cap, int chi_max, void* cores, int32_t* bonds,
                    int32_t* centers, double* discarded, int32_t* flags, void* stream) {
  using namespace tqt;
  if (bad_sizes("tq_tt_run", n_qubits, batch, chi_cap, dtype) || n_gates < 0) return TQ_ERR_INPUT;
  Params p{};
  p.n = n_qubits; p.n_gates = n_gates; p.batch = batch; p.chi_cap = chi_cap; p.chi_max = chi_max;
  p.gates = reinterpret_cast<const tq_tgate*>(gates); p.theta = theta; p.theta_stride = theta_stride;
  p.eps = eps; p.discarded = discarded; p.bonds = bonds; p.flags = flags; p.centers = centers; p.cores = cores;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaMemsetAsync(flags, 0, sizeof(int32_t) * batch, st);
  return dispatch<PH_RUN>(p, dtype, st);
}

tq_status tq_tt_apply(int n_qubits, const void* gates, int n_gates, int dtype, int batch, const void* theta,
                      int64_t theta_stride, double eps, int chi_cap, int chi_max, void* cores, int32_t* bonds,
                      int32_t* centers, double* discarded, int32_t* flags, void* stream) {
  using namespace tqt;
  if (bad_sizes("tq_tt_apply", n_qubits, batch, chi_cap, dtype) || n_gates < 0) return TQ_ERR_INPUT;
  Params p{};
  p.n = n_qubits; p.n_gates = n_gates; p.batch = batch; p.chi_cap = chi_cap; p.chi_max = chi_max;
  p.gates = reinterpret_cast<const tq_tgate*>(gates); p.theta = theta; p.theta_stride = theta_stride;
  p.eps = eps; p.bonds = bonds; p.flags = flags; p.centers = centers; p.cores = cores; p.inplace = 1;
  p.discarded = discarded;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaMemsetAsync(flags, 0, sizeof(int32_t) * batch, st);
  return dispatch<PH_RUN>(p, dtype, st);
}

tq_status tq_tt_compress(int n_qubits, int dtype, int batch, double eps, int chi_cap, int chi_max, void* cores,
                         int32_t* bonds, int32_t* centers, double* discarded, int32_t* flags, void* stream) {
  using namespace tqt;
  if (bad_sizes("tq_tt_compress", n_qubits, batch, chi_cap, dtype)) return TQ_ERR_INPUT;
  if (eps < 0.0 || chi_max == 0) {
    snprintf(tq::g_err, sizeof(tq::g_err), "tq_tt_compress: eps must be >= 0 and chi_max >= 1 (or -1)");
    return TQ_ERR_INPUT;
  }
  Params p{};
  p.n = n_qubits; p.batch = batch; p.chi_cap = chi_cap; p.chi_max = chi_max; p.eps = eps;
  p.discarded = discarded; p.bonds = bonds; p.flags = flags; p.centers = centers; p.cores = cores;
  return dispatch<PH_COMPRESS>(p, dtype, reinterpret_cast<cudaStream_t>(stream));
}

size_t tq_tt_tape_bytes(int n_two_site, int batch, int chi_cap, int dtype) {
  if (n_two_site < 0 || batch < 1 || chi_cap < 1) return 0;
  const size_t csz = dtype == TQ_C128 ? 16 : 8;
  const int c = tqt::cap_bucket(chi_cap);
  const size_t slots = (size_t)batch * (n_two_site > 0 ? n_two_site : 1);
  return tqt::align256(slots * 2 * c * c * csz) + slots * sizeof(tqt::TapeMeta);
}

static tq_status tt_taped_common(int phase, int n_qubits, const void* gates, int n_gates, int n_two_site, int dtype,
                                 int batch, const void* theta, int64_t theta_stride, double eps, int chi_cap,
                                 int chi_max, const int32_t* parent, const int32_t* term_lo, const int32_t* term_hi,
                                 const int32_t* code_off, const int8_t* codes, int n_terms, void* values,
                                 double* norm2, int32_t* bonds, int32_t* flags, void* tape, int tape_batch,
                                 const void* init_cores, const int32_t* init_bonds,
                                 void* workspace, size_t workspace_bytes, void* stream) {
  using namespace tqt;
  if (bad_sizes("tq_tt_taped", n_qubits, batch, chi_cap, dtype) || n_gates < 0 || n_terms < 0 || n_two_site < 0)
    return TQ_ERR_INPUT;
  const WsParts w = ws_parts(n_qubits, batch, chi_cap, dtype);
  if (workspace_bytes < w.total) {
    snprintf(tq::g_err, sizeof(tq::g_err), "tq_tt_taped: workspace %zu < %zu bytes", workspace_bytes, w.total);
    return TQ_ERR_WORKSPACE;
  }
  Params p{};
  p.n = n_qubits; p.n_gates = n_gates; p.batch = batch; p.chi_cap = chi_cap; p.chi_max = chi_max;
  p.n_terms = n_terms; p.gates = reinterpret_cast<const tq_tgate*>(gates); p.theta = theta;
  p.theta_stride = theta_stride; p.eps = eps; p.term_lo = term_lo; p.term_hi = term_hi;
  p.code_off = code_off; p.codes = codes; p.values = reinterpret_cast<double2*>(values);
  p.discarded = nullptr; p.norm2 = norm2; p.bonds = bonds; p.flags = flags;
  unsigned char* base = reinterpret_cast<unsigned char*>(workspace);
  p.cores = base + w.cores; p.envl = base + w.envl; p.envr = base + w.envr;
  const size_t csz = dtype == TQ_C128 ? 16 : 8;
  const int c = cap_bucket(chi_cap);
  const size_t slots = (size_t)tape_batch * (n_two_site > 0 ? n_two_site : 1);
  p.tape = tape;
  p.meta = reinterpret_cast<TapeMeta*>(reinterpret_cast<unsigned char*>(tape) + align256(slots * 2 * c * c * csz));
  p.parent = parent; p.n2 = n_two_site;
  p.init_cores = init_cores; p.init_bonds = init_bonds;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaMemsetAsync(flags, 0, sizeof(int32_t) * batch, st);
  return phase == PH_TAPE ? dispatch<PH_RUN | PH_TAPE | PH_VALUES>(p, dtype, st)
                          : dispatch<PH_RUN | PH_REPLAY | PH_VALUES>(p, dtype, st);
}

tq_status tq_tt_taped(int n_qubits, const void* gates, int n_gates, int n_two_site, int dtype, int batch,
                      const void* theta, int64_t theta_stride, double eps, int chi_cap, int chi_max,
                      const int32_t* term_lo, const int32_t* term_hi, const int32_t* code_off, const int8_t* codes,
                      int n_terms, void* values, double* norm2, int32_t* bonds, int32_t* flags, void* tape,
                      const void* init_cores, const int32_t* init_bonds,
                      void* workspace, size_t workspace_bytes, void* stream) {
  return tt_taped_common(tqt::PH_TAPE, n_qubits, gates, n_gates, n_two_site, dtype, batch, theta, theta_stride, eps,
                         chi_cap, chi_max, nullptr, term_lo, term_hi, code_off, codes, n_terms, values, norm2, bonds,
                         flags, tape, batch, init_cores, init_bonds, workspace, workspace_bytes, stream);
}

tq_status tq_tt_replay(int n_qubits, const void* gates, int n_gates, int n_two_site, int dtype, int rows,
                       const void* theta, int64_t theta_stride, int chi_cap, const int32_t* parent, int tape_batch,
                       const void* tape, const int32_t* term_lo, const int32_t* term_hi, const int32_t* code_off,
                       const int8_t* codes, int n_terms, void* values, double* norm2, int32_t* bonds, int32_t* flags,
                       const void* init_cores, const int32_t* init_bonds,
                       void* workspace, size_t workspace_bytes, void* stream) {
  return tt_taped_common(tqt::PH_REPLAY, n_qubits, gates, n_gates, n_two_site, dtype, rows, theta, theta_stride, 0.0,
                         chi_cap, -1, parent, term_lo, term_hi, code_off, codes, n_terms, values, norm2, bonds, flags,
                         const_cast<void*>(tape), tape_batch, init_cores, init_bonds, workspace, workspace_bytes,
                         stream);
}

tq_status tq_tt_inner(int n_qubits, int dtype, int batch, int chi_cap, const void* cores_a, const int32_t* bonds_a,
                      const void* cores_b, const int32_t* bonds_b, void* out, void* stream) {
  using namespace tqt;
  if (bad_sizes("tq_tt_inner", n_qubits, batch, chi_cap, dtype)) return TQ_ERR_INPUT;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int c = cap_bucket(chi_cap);
  double2* o = reinterpret_cast<double2*>(out);
#define TQ_INNER(R, CAPV)                                                                                         \
  {                                                                                                               \
    const size_t smem = sizeof(Scratch<R, CAPV>);                                                                 \
    cudaFuncSetAttribute(tt_inner_kernel<R, CAPV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);      \
    tt_inner_kernel<R, CAPV><<<batch, NT, smem, st>>>(n_qubits, cores_a, bonds_a, cores_b, bonds_b, o);          \
  }
  if (dtype == TQ_C128) {
    if (c <= 4) TQ_INNER(double, 4) else if (c <= 8) TQ_INNER(double, 8) else if (c <= 16) TQ_INNER(double, 16)
    else TQ_INNER(double, 32)
  } else {
    if (c <= 4) TQ_INNER(float, 4) else if (c <= 8) TQ_INNER(float, 8) else if (c <= 16) TQ_INNER(float, 16)
    else TQ_INNER(float, 32)
  }
#undef TQ_INNER
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(tq::g_err, sizeof(tq::g_err), "%s", cudaGetErrorString(e));
    return TQ_ERR_CUDA;
  }
  return TQ_OK;
}

size_t tq_tt_values_workspace_bytes(int n_qubits, int batch, int chi_cap, int dtype) {
  if (n_qubits < 1 || batch < 1 || chi_cap < 1) return 0;
  return tqt::env_bytes(n_qubits, batch, chi_cap, dtype);
}

tq_status tq_tt_values(int n_qubits, int dtype, int batch, int chi_cap, const void* cores, const int32_t* bonds,
                       const int32_t* term_lo, const int32_t* term_hi, const int32_t* code_off, const int8_t* codes,
                       int n_terms, void* values, double* norm2, void* workspace, size_t workspace_bytes,
                       void* stream) {
  using namespace tqt;
  if (bad_sizes("tq_tt_values", n_qubits, batch, chi_cap, dtype) || n_terms < 0) return TQ_ERR_INPUT;
  const size_t need = env_bytes(n_qubits, batch, chi_cap, dtype);
  if (workspace_bytes < need) {
    snprintf(tq::g_err, sizeof(tq::g_err), "tq_tt_values: workspace %zu < %zu bytes", workspace_bytes, need);
    return TQ_ERR_WORKSPACE;
  }
  Params p{};
  p.n = n_qubits; p.batch = batch; p.chi_cap = chi_cap; p.n_terms = n_terms;
  p.term_lo = term_lo; p.term_hi = term_hi; p.code_off = code_off; p.codes = codes;
  p.values = reinterpret_cast<double2*>(values); p.norm2 = norm2;
  p.bonds = const_cast<int32_t*>(bonds); p.cores = const_cast<void*>(cores);
  unsigned char* base = reinterpret_cast<unsigned char*>(workspace);
  p.envl = base; p.envr = base + env_bytes(n_qubits, batch, chi_cap, dtype) / 2;
  return dispatch<PH_VALUES>(p, dtype, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
