// tq_engine.cu — sm_100a kernels for TT-circuit expectation values and gradients.
//
// Work decomposition.  One "team" (a warp for chi <= 8, a whole CTA for chi = 16/32)
// owns one work item = (theta-set b, light-cone segment g) and sweeps the sites of
// that segment's sub-chain sequentially.  Per site everything lives in shared memory:
// the folded core A_k[s] (and its conjugate transpose), the MPO transfer environments
// and the GEMM intermediates; only the right environments cross HBM (written by the
// right-to-left sweep, re-read once by the left-to-right gradient sweep).
//
// Per site k (chi_l x chi_r core, D MPO channels):
//   fold   A[s]_{ab} = <s| O_L(a,b) ... O_1(a,b) |init>            (column of 2x2 ops)
//   RL     N[b][s] = A[s] P[b];  BR[a][s'] = sum_edges c O_{s's} N[b][s];
//          P'[a]  = sum_s' BR[a][s'] A[s']^H                        (energy = P'[START] at the left end)
//   LR     M[a][s] = Lam[a] A[s]; BR[b][s'] = sum_edges c O_{s's} M[a][s];
//          Lam'[b] = sum_s' A[s']^H BR[b][s'];  G[s'] = sum_b BR[b][s'] P[b]
//          dE/dtheta_l = sum_{a,b} Im<u_l, sigma_l v_l>  (per-pair column adjoint, u = Post^H G)
//
// The reference computes the same quantities with SVD-split cores and a generic tape
// (tt.py:186-244, autodiff.py:315-402, 190-247); see DESIGN.md for the derivation.

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/tq_engine.h"

namespace tq {

// ------------------------------------------------------------------ complex helpers
template <typename R> struct CT;
template <> struct CT<float> { using T = float2; };
template <> struct CT<double> { using T = double2; };

template <typename C> __device__ __forceinline__ C cmk(decltype(C::x) x, decltype(C::x) y) { C r; r.x = x; r.y = y; return r; }
template <typename C> __device__ __forceinline__ C cadd(C a, C b) { return cmk<C>(a.x + b.x, a.y + b.y); }
template <typename C> __device__ __forceinline__ C cmul(C a, C b) { return cmk<C>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
template <typename C> __device__ __forceinline__ C cconj(C a) { return cmk<C>(a.x, -a.y); }
// acc += a * b
template <typename C> __device__ __forceinline__ void cfma(C& acc, C a, C b) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a) * b
template <typename C> __device__ __forceinline__ void cfmac(C& acc, C a, C b) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(-a.y, b.x, acc.y);
}

// ------------------------------------------------------------------ kernel parameters
struct Layout {          // byte offsets inside one team's shared-memory slab (host computed)
  int32_t a, ah, env, m, br, pin, mr, contrib, mres, minfo, mps;
  int32_t team_bytes;
  int32_t nslot_env, nslot_m, nslot_br, nslot_pin, nslot_mr;
};

struct Params {
  tq_chain c;
  Layout L;
  int32_t batch;
  const void* theta; int64_t theta_stride;
  const void* coef; int64_t coef_stride;
  void* env;        // [B][env_total] complex (stored right environments)
  void* epart;      // [B][n_segments] complex
  void* gpart;      // [B][n_gslots] real
  double* values;   // [B][n_terms][2]
  int32_t store_env;
  int32_t mode;     // 0 energy-grad, 1 values
};

// Team barrier: a warp team syncs with __syncwarp, a CTA team with __syncthreads.
template <int TEAM> __device__ __forceinline__ void team_sync() {
  if (TEAM == 32) __syncwarp(); else __syncthreads();
}

template <typename R> __device__ __forceinline__ R theta_at(const Params& p, int b, int slot) {
  return reinterpret_cast<const R*>(p.theta)[(int64_t)b * p.theta_stride + slot];
}
template <typename R> __device__ __forceinline__ R coef_at(const Params& p, int b, int idx) {
  if (idx < 0) return R(1);
  return reinterpret_cast<const R*>(p.coef)[(int64_t)b * p.coef_stride + idx];
}

// Pauli op element <s'|O|s>: for op in {I,X,Y,Z} the only nonzero s for a given s' and its factor.
template <typename C> __device__ __forceinline__ int pauli_src(int op, int sp) { return (op == 1 || op == 2) ? 1 - sp : sp; }
template <typename C> __device__ __forceinline__ C pauli_fac(int op, int sp) {
  using R = decltype(C::x);
  if (op == 2) return sp == 0 ? cmk<C>(R(0), R(-1)) : cmk<C>(R(0), R(1));
  if (op == 3 && sp == 1) return cmk<C>(R(-1), R(0));
  return cmk<C>(R(1), R(0));
}

// ------------------------------------------------------------------ stage helpers
// Resolve the site's 2x2 factor table for this theta-set into shared memory.
template <typename R, int TEAM>
__device__ void resolve_mats(const Params& p, const tq_site& st, int b, int tid,
                             typename CT<R>::T* mres, int* minfo, R* mps) {
  using C = typename CT<R>::T;
  for (int oi = 0; oi < st.op_count; ++oi) {
    const tq_op op = p.c.ops[st.op_begin + oi];
    const int nd = 1 << op.bits;
    for (int d = 0; d < nd; ++d) {
      const int e = op.lmat + d;
      if ((e % TEAM) != tid) continue;
      const tq_mat mt = p.c.mats[op.mat + d];
      C m00, m01, m10, m11;
      if (mt.kind == 0) {
        m00 = cmk<C>(R(mt.m[0]), R(mt.m[1])); m01 = cmk<C>(R(mt.m[2]), R(mt.m[3]));
        m10 = cmk<C>(R(mt.m[4]), R(mt.m[5])); m11 = cmk<C>(R(mt.m[6]), R(mt.m[7]));
      } else {
        const R t = mt.slot >= 0 ? theta_at<R>(p, b, mt.slot) : R(mt.angle);
        R s, c;
        if (sizeof(R) == 4) { float sf, cf; sincosf(float(t) * 0.5f, &sf, &cf); s = R(sf); c = R(cf); }
        else { double sd, cd; sincos(double(t) * 0.5, &sd, &cd); s = R(sd); c = R(cd); }
        const R z = R(0);
        if (mt.kind == 1) { m00 = cmk<C>(c, z); m01 = cmk<C>(z, -s); m10 = cmk<C>(z, -s); m11 = cmk<C>(c, z); }
        else if (mt.kind == 2) { m00 = cmk<C>(c, z); m01 = cmk<C>(-s, z); m10 = cmk<C>(s, z); m11 = cmk<C>(c, z); }
        else { m00 = cmk<C>(c, -s); m01 = cmk<C>(z, z); m10 = cmk<C>(z, z); m11 = cmk<C>(c, s); }
      }
      mres[4 * e + 0] = m00; mres[4 * e + 1] = m01; mres[4 * e + 2] = m10; mres[4 * e + 3] = m11;
      minfo[e] = (mt.kind & 0xff) | ((mt.cls & 0xff) << 8);
      mps[e] = R(mt.pscale);
    }
  }
}

__device__ __forceinline__ int op_digit(const tq_op& op, int al, int be) {
  const int mask = (1 << op.bits) - 1;
  return op.src == 1 ? ((al >> op.shift) & mask) : (op.src == 2 ? ((be >> op.shift) & mask) : 0);
}

__device__ __forceinline__ bool pass_ok(const Params& p, const tq_site& st, int al, int be) {
  for (int i = 0; i < st.pass_count; ++i) {
    const tq_pass ps = p.c.passes[st.pass_begin + i];
    const int m = (1 << ps.bits) - 1;
    if (((al >> ps.sa) & m) != ((be >> ps.sb) & m)) return false;
  }
  return true;
}

// Fold the column of site st into A[s] (chi_l x chi_r, row stride LD) and AH[s] = A[s]^H.
template <typename R, int LD, int TEAM>
__device__ void fold_site(const Params& p, const tq_site& st, int tid, const typename CT<R>::T* mres,
                          typename CT<R>::T* A, typename CT<R>::T* AH, int lcr) {
  using C = typename CT<R>::T;
  const int npair = st.chi_l * st.chi_r;
  for (int pi = tid; pi < npair; pi += TEAM) {
    const int al = pi >> lcr, be = pi & (st.chi_r - 1);
    C v0 = cmk<C>(R(st.init[0]), R(st.init[1]));
    C v1 = cmk<C>(R(st.init[2]), R(st.init[3]));
    if (!pass_ok(p, st, al, be)) { v0 = cmk<C>(R(0), R(0)); v1 = v0; }
    else {
      for (int oi = 0; oi < st.op_count; ++oi) {
        const tq_op op = p.c.ops[st.op_begin + oi];
        const C* M = mres + 4 * (op.lmat + op_digit(op, al, be));
        C n0 = cmul(M[0], v0); cfma(n0, M[1], v1);
        C n1 = cmul(M[2], v0); cfma(n1, M[3], v1);
        v0 = n0; v1 = n1;
      }
    }
    A[al * LD + be] = v0; A[LD * LD + al * LD + be] = v1;   // A slots are LD*LD apart
    AH[be * LD + al] = cconj(v0); AH[LD * LD + be * LD + al] = cconj(v1);
  }
}

// Register-tiled complex GEMM over a group of equally shaped tasks:
//   C_t[m x n] = sum_{q < nq} A_{t,q}[m x kk] * B_{t,q}[kk x n]   (all row stride LD)
// Each item computes rt consecutive rows of one column; a warp's lanes walk columns so the
// A operand is a broadcast and the B operand a contiguous row.
template <typename C, int LD, int TEAM, typename FA, typename FB, typename FS>
__device__ __forceinline__ void gemm_group(int tid, int ntasks, int m, int n, int kk, int nq, FA fa, FB fb, FS store) {
  const int rt = m >= 4 ? 4 : m;
  const int lrt = rt == 4 ? 2 : (rt == 2 ? 1 : 0);
  const int ln = 31 - __clz(n);
  const int lmb = (31 - __clz(m)) - lrt;
  const int lper = lmb + ln;
  const int total = ntasks << lper;
  for (int it = tid; it < total; it += TEAM) {
    const int task = it >> lper;
    const int r = it & ((1 << lper) - 1);
    const int j = r & (n - 1);
    const int i0 = (r >> ln) << lrt;
    C acc0 = {0, 0}, acc1 = {0, 0}, acc2 = {0, 0}, acc3 = {0, 0};
    for (int q = 0; q < nq; ++q) {
      const C* Ab = fa(task, q) + i0 * LD;
      const C* Bb = fb(task, q) + j;
      if (rt == 4) {
#pragma unroll 4
        for (int k = 0; k < kk; ++k) {
          const C bv = Bb[k * LD];
          cfma(acc0, Ab[k], bv); cfma(acc1, Ab[LD + k], bv);
          cfma(acc2, Ab[2 * LD + k], bv); cfma(acc3, Ab[3 * LD + k], bv);
        }
      } else {
        for (int k = 0; k < kk; ++k) {
          const C bv = Bb[k * LD];
          cfma(acc0, Ab[k], bv);
          if (rt == 2) cfma(acc1, Ab[LD + k], bv);
        }
      }
    }
    store(task, i0, j, rt, acc0, acc1, acc2, acc3);
  }
}

// ------------------------------------------------------------------ right-to-left sweep
// Computes the MPO right environments P^{(a)}_k for every cut of the segment's sub-chain,
// optionally storing them, and the segment's partial energy P^{START}_{lo}.
template <typename R, int CHI, int TEAM>
__global__ void __launch_bounds__(TEAM == 32 ? 128 : TEAM)
rl_sweep(Params p) {
  using C = typename CT<R>::T;
  constexpr int LD = CHI + 1;
  constexpr int MS = LD * LD;   // complex elements per matrix slot
  constexpr int TEAMS = TEAM == 32 ? 4 : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int team = threadIdx.x / TEAM;
  const int tid = threadIdx.x % TEAM;
  const int item = blockIdx.x * TEAMS + team;
  const int S = p.c.n_segments;
  if (item >= p.batch * S) return;
  const int b = item / S, g = item % S;
  unsigned char* base = smem_raw + (size_t)team * p.L.team_bytes;
  C* A = reinterpret_cast<C*>(base + p.L.a);
  C* AH = reinterpret_cast<C*>(base + p.L.ah);
  C* PIN = reinterpret_cast<C*>(base + p.L.env);
  C* N = reinterpret_cast<C*>(base + p.L.m);
  C* BR = reinterpret_cast<C*>(base + p.L.br);
  C* mres = reinterpret_cast<C*>(base + p.L.mres);
  int* minfo = reinterpret_cast<int*>(base + p.L.minfo);
  R* mps = reinterpret_cast<R*>(base + p.L.mps);

  const tq_segment seg = p.c.segs[g];
  C* env_g = reinterpret_cast<C*>(p.env) + (size_t)b * p.c.env_total + seg.env_base;
  // boundary: DONE channel = [[1]] at the right end of the sub-chain
  if (tid == 0) PIN[0] = cmk<C>(R(1), R(0));
  team_sync<TEAM>();
  {
    const tq_site last = p.c.sites[seg.site_begin + seg.site_count - 1];
    if (p.store_env && tid == 0 && last.env_in >= 0) env_g[last.env_in] = PIN[0];
  }
  for (int q = seg.site_count - 1; q >= 0; --q) {
    const tq_site st = p.c.sites[seg.site_begin + q];
    const int cl = st.chi_l, cr = st.chi_r;
    const int lcr = 31 - __clz(cr);
    resolve_mats<R, TEAM>(p, st, b, tid, mres, minfo, mps);
    team_sync<TEAM>();
    fold_site<R, LD, TEAM>(p, st, tid, mres, A, AH, lcr);
    team_sync<TEAM>();
    // N[b][s] = A[s] * P[b]
    const int db = st.rl_db, da = st.rl_da;
    gemm_group<C, LD, TEAM>(tid, db * 2, cl, cr, cr, 1,
        [&](int t, int) { return A + (t & 1) * MS; },
        [&](int t, int) { return PIN + (t >> 1) * MS; },
        [&](int t, int i0, int j, int rt, C a0, C a1, C a2, C a3) {
          C* o = N + t * MS + i0 * LD + j;
          o[0] = a0; if (rt > 1) o[LD] = a1; if (rt > 2) { o[2 * LD] = a2; o[3 * LD] = a3; }
        });
    team_sync<TEAM>();
    // BR[a][s'] = sum over edges (a <- bb) of coef * O_{s's} N[bb][s]
    {
      const int nel = da * 2 * cl * cr;
      for (int e = tid; e < nel; e += TEAM) {
        const int ij = e % (cl * cr);
        const int as = e / (cl * cr);
        const int a = as >> 1, sp = as & 1;
        const int i = ij >> lcr, j = ij & (cr - 1);
        C acc = cmk<C>(R(0), R(0));
        for (int ei = 0; ei < st.rl_edge_count; ++ei) {
          const tq_edge ed = p.c.edges[st.rl_edge_begin + ei];
          if (ed.a != a) continue;
          const R cf = coef_at<R>(p, b, ed.coef);
          const int s = pauli_src<C>(ed.op, sp);
          const C f = pauli_fac<C>(ed.op, sp);
          const C nv = N[(ed.b * 2 + s) * MS + i * LD + j];
          const C t = cmul(f, nv);
          acc.x += cf * t.x; acc.y += cf * t.y;
        }
        BR[(a * 2 + sp) * MS + i * LD + j] = acc;
      }
    }
    team_sync<TEAM>();
    // P'[a] = sum_s' BR[a][s'] AH[s']  -> PIN slots (P[b] is dead) + HBM
    const bool store = p.store_env && st.env_out >= 0;
    C* envo = env_g + (store ? st.env_out : 0);
    gemm_group<C, LD, TEAM>(tid, da, cl, cl, cr, 2,
        [&](int t, int qq) { return BR + (t * 2 + qq) * MS; },
        [&](int, int qq) { return AH + qq * MS; },
        [&](int t, int i0, int j, int rt, C a0, C a1, C a2, C a3) {
          C* o = PIN + t * MS + i0 * LD + j;
          o[0] = a0; if (rt > 1) o[LD] = a1; if (rt > 2) { o[2 * LD] = a2; o[3 * LD] = a3; }
          if (store) {
            C* h = envo + (size_t)t * cl * cl + i0 * cl + j;
            h[0] = a0; if (rt > 1) h[cl] = a1; if (rt > 2) { h[2 * cl] = a2; h[3 * cl] = a3; }
          }
        });
    team_sync<TEAM>();
  }
  if (tid == 0) reinterpret_cast<C*>(p.epart)[(size_t)b * S + g] = PIN[0];
}

// ------------------------------------------------------------------ left-to-right sweep
// mode 0: gradient (G + per-pair column adjoint); mode 1: per-term values.
template <typename R, int CHI, int TEAM>
__global__ void __launch_bounds__(TEAM == 32 ? 128 : TEAM)
lr_sweep(Params p) {
  using C = typename CT<R>::T;
  constexpr int LD = CHI + 1;
  constexpr int MS = LD * LD;
  constexpr int TEAMS = TEAM == 32 ? 4 : 1;
  constexpr int MAXSAVE = 48;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int team = threadIdx.x / TEAM;
  const int tid = threadIdx.x % TEAM;
  const int item = blockIdx.x * TEAMS + team;
  const int S = p.c.n_segments;
  if (item >= p.batch * S) return;
  const int b = item / S, g = item % S;
  unsigned char* base = smem_raw + (size_t)team * p.L.team_bytes;
  C* A = reinterpret_cast<C*>(base + p.L.a);
  C* AH = reinterpret_cast<C*>(base + p.L.ah);
  C* LAM = reinterpret_cast<C*>(base + p.L.env);
  C* M = reinterpret_cast<C*>(base + p.L.m);
  C* BR = reinterpret_cast<C*>(base + p.L.br);
  C* PIN = reinterpret_cast<C*>(base + p.L.pin);
  C* MR = reinterpret_cast<C*>(base + p.L.mr);
  R* contrib = reinterpret_cast<R*>(base + p.L.contrib);
  C* mres = reinterpret_cast<C*>(base + p.L.mres);
  int* minfo = reinterpret_cast<int*>(base + p.L.minfo);
  R* mps = reinterpret_cast<R*>(base + p.L.mps);
  C* G = M;  // gradient cores alias the M slots (dead after the bracket stage)

  const tq_segment seg = p.c.segs[g];
  const C* env_g = reinterpret_cast<const C*>(p.env) + (size_t)b * p.c.env_total + seg.env_base;
  R* gpart = reinterpret_cast<R*>(p.gpart) + (size_t)b * p.c.n_gslots + seg.gslot_begin;
  if (tid == 0) LAM[0] = cmk<C>(R(1), R(0));
  team_sync<TEAM>();
  for (int q = 0; q < seg.site_count; ++q) {
    const tq_site st = p.c.sites[seg.site_begin + q];
    const int cl = st.chi_l, cr = st.chi_r;
    const int lcr = 31 - __clz(cr);
    const int da = st.lr_da, db = st.lr_db;
    const int npin = p.mode == 0 ? st.rl_db : 1;
    resolve_mats<R, TEAM>(p, st, b, tid, mres, minfo, mps);
    // stored right environments at cut k+1 -> PIN (dense cr x cr in HBM)
    {
      const C* src = env_g + st.env_in;
      const int per = cr * cr;
      for (int e = tid; e < npin * per; e += TEAM) {
        const int ch = e / per, r = e % per;
        PIN[ch * MS + (r >> lcr) * LD + (r & (cr - 1))] = src[e];
      }
    }
    team_sync<TEAM>();
    fold_site<R, LD, TEAM>(p, st, tid, mres, A, AH, lcr);
    team_sync<TEAM>();
    // M[a][s] = Lam[a] * A[s]
    gemm_group<C, LD, TEAM>(tid, da * 2, cl, cr, cl, 1,
        [&](int t, int) { return LAM + (t >> 1) * MS; },
        [&](int t, int) { return A + (t & 1) * MS; },
        [&](int t, int i0, int j, int rt, C a0, C a1, C a2, C a3) {
          C* o = M + t * MS + i0 * LD + j;
          o[0] = a0; if (rt > 1) o[LD] = a1; if (rt > 2) { o[2 * LD] = a2; o[3 * LD] = a3; }
        });
    team_sync<TEAM>();
    // BR[bb][s'] = sum over edges (a -> bb) of coef * O_{s's} M[a][s]
    {
      const int nel = db * 2 * cl * cr;
      for (int e = tid; e < nel; e += TEAM) {
        const int ij = e % (cl * cr);
        const int bs = e / (cl * cr);
        const int bb = bs >> 1, sp = bs & 1;
        const int i = ij >> lcr, j = ij & (cr - 1);
        C acc = cmk<C>(R(0), R(0));
        for (int ei = 0; ei < st.lr_edge_count; ++ei) {
          const tq_edge ed = p.c.edges[st.lr_edge_begin + ei];
          if (ed.b != bb) continue;
          const R cf = coef_at<R>(p, b, ed.coef);
          const int s = pauli_src<C>(ed.op, sp);
          const C f = pauli_fac<C>(ed.op, sp);
          const C t = cmul(f, M[(ed.a * 2 + s) * MS + i * LD + j]);
          acc.x += cf * t.x; acc.y += cf * t.y;
        }
        BR[(bb * 2 + sp) * MS + i * LD + j] = acc;
      }
    }
    team_sync<TEAM>();
    // Lam'[bb] = sum_s' AH[s'] BR[bb][s']
    gemm_group<C, LD, TEAM>(tid, db, cr, cr, cl, 2,
        [&](int, int qq) { return AH + qq * MS; },
        [&](int t, int qq) { return BR + (t * 2 + qq) * MS; },
        [&](int t, int i0, int j, int rt, C a0, C a1, C a2, C a3) {
          C* o = LAM + t * MS + i0 * LD + j;
          o[0] = a0; if (rt > 1) o[LD] = a1; if (rt > 2) { o[2 * LD] = a2; o[3 * LD] = a3; }
        });
    if (p.mode == 0) {
      // G[s'] = sum_bb BR[bb][s'] PIN[bb]   (writes over M, read only by the BR stage)
      gemm_group<C, LD, TEAM>(tid, 2, cl, cr, cr, db,
          [&](int t, int qq) { return BR + (qq * 2 + t) * MS; },
          [&](int, int qq) { return PIN + qq * MS; },
          [&](int t, int i0, int j, int rt, C a0, C a1, C a2, C a3) {
            C* o = G + t * MS + i0 * LD + j;
            o[0] = a0; if (rt > 1) o[LD] = a1; if (rt > 2) { o[2 * LD] = a2; o[3 * LD] = a3; }
          });
      team_sync<TEAM>();
      // ---- column adjoint: per (alpha, beta) pair forward fold with checkpoints of the
      // components projectors discard, then the backward walk accumulating Im<u, sigma v>.
      const int ntr = st.n_train;
      for (int t = 0; t < ntr; ++t) contrib[t * TEAM + tid] = R(0);
      const int npair = cl * cr;
      for (int pi = tid; pi < npair; pi += TEAM) {
        const int al = pi >> lcr, be = pi & (cr - 1);
        if (!pass_ok(p, st, al, be)) continue;
        C sv[MAXSAVE];
        int ns = 0;
        C v0 = cmk<C>(R(st.init[0]), R(st.init[1]));
        C v1 = cmk<C>(R(st.init[2]), R(st.init[3]));
        for (int oi = 0; oi < st.op_count; ++oi) {
          const tq_op op = p.c.ops[st.op_begin + oi];
          const int e = op.lmat + op_digit(op, al, be);
          const int cls = (minfo[e] >> 8) & 0xff;
          if (cls == 1) sv[ns++] = v1;
          else if (cls == 2) sv[ns++] = v0;
          else if (cls == 3) { sv[ns++] = v0; sv[ns++] = v1; }
          const C* Mm = mres + 4 * e;
          C n0 = cmul(Mm[0], v0); cfma(n0, Mm[1], v1);
          C n1 = cmul(Mm[2], v0); cfma(n1, Mm[3], v1);
          v0 = n0; v1 = n1;
        }
        C u0 = G[al * LD + be], u1 = G[MS + al * LD + be];
        for (int oi = st.op_count - 1; oi >= 0; --oi) {
          const tq_op op = p.c.ops[st.op_begin + oi];
          const int e = op.lmat + op_digit(op, al, be);
          const int info = minfo[e];
          const int kind = info & 0xff, cls = (info >> 8) & 0xff;
          if (op.tidx >= 0 && kind != 0) {
            // Im<u, sigma v>, sigma = X (kind 1), Y (2), Z (3)
            C s0, s1;
            if (kind == 1) { s0 = v1; s1 = v0; }
            else if (kind == 2) { s0 = cmk<C>(v1.y, -v1.x); s1 = cmk<C>(-v0.y, v0.x); }
            else { s0 = v0; s1 = cmk<C>(-v1.x, -v1.y); }
            C d = cmk<C>(R(0), R(0));
            cfmac(d, u0, s0); cfmac(d, u1, s1);
            contrib[op.tidx * TEAM + tid] += d.y;
          }
          const C* Mm = mres + 4 * e;
          // u <- M^H u
          C w0 = cmk<C>(R(0), R(0)), w1 = w0;
          cfmac(w0, Mm[0], u0); cfmac(w0, Mm[2], u1);
          cfmac(w1, Mm[1], u0); cfmac(w1, Mm[3], u1);
          u0 = w0; u1 = w1;
          // v <- state before this op
          if (cls == 0) {
            C x0 = cmk<C>(R(0), R(0)), x1 = x0;
            cfmac(x0, Mm[0], v0); cfmac(x0, Mm[2], v1);
            cfmac(x1, Mm[1], v0); cfmac(x1, Mm[3], v1);
            v0 = x0; v1 = x1;
          } else if (cls == 1) {
            const R sc = R(1) / mps[e];
            v0 = cmk<C>(v0.x * sc, v0.y * sc); v1 = sv[--ns];
          } else if (cls == 2) {
            const R sc = R(1) / mps[e];
            v1 = cmk<C>(v1.x * sc, v1.y * sc); v0 = sv[--ns];
          } else {
            v1 = sv[--ns]; v0 = sv[--ns];
          }
        }
      }
      team_sync<TEAM>();
      // deterministic per-op reduction: warp w handles ops w, w + nwarps, ...
      {
        const int warp = tid >> 5, lane = tid & 31;
        constexpr int NW = TEAM / 32;
        for (int oi = warp; oi < st.op_count; oi += NW) {
          const tq_op op = p.c.ops[st.op_begin + oi];
          if (op.tidx < 0) continue;
          R s = R(0);
          for (int k = lane; k < TEAM; k += 32) s += contrib[op.tidx * TEAM + k];
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
          if (lane == 0) gpart[op.gidx] = s;
        }
      }
      team_sync<TEAM>();
    } else {
      // ---- values: rho_a[s'][s] = <A[s'], M[a][s] R> for every source channel a
      gemm_group<C, LD, TEAM>(tid, da * 2, cl, cr, cr, 1,
          [&](int t, int) { return M + t * MS; },
          [&](int, int) { return PIN; },
          [&](int t, int i0, int j, int rt, C a0, C a1, C a2, C a3) {
            C* o = MR + t * MS + i0 * LD + j;
            o[0] = a0; if (rt > 1) o[LD] = a1; if (rt > 2) { o[2 * LD] = a2; o[3 * LD] = a3; }
          });
      team_sync<TEAM>();
      if (st.fin_count > 0) {
        const int ncombo = da * 4;  // (a, s', s)
        R* part = contrib;          // [2 * ncombo][TEAM] partial sums (re, im)
        for (int cmb = 0; cmb < ncombo; ++cmb) {
          const int a = cmb >> 2, sp = (cmb >> 1) & 1, s = cmb & 1;
          C acc = cmk<C>(R(0), R(0));
          for (int e = tid; e < cl * cr; e += TEAM) {
            const int i = e >> lcr, j = e & (cr - 1);
            cfmac(acc, A[sp * MS + i * LD + j], MR[(a * 2 + s) * MS + i * LD + j]);
          }
          part[(2 * cmb) * TEAM + tid] = acc.x;
          part[(2 * cmb + 1) * TEAM + tid] = acc.y;
        }
        team_sync<TEAM>();
        // reduce and finalise (one warp, fixed order)
        if (tid < 32) {
          for (int fi = 0; fi < st.fin_count; ++fi) {
            const tq_edge fe = p.c.fins[st.fin_begin + fi];
            double vre = 0.0, vim = 0.0;
            for (int sp = 0; sp < 2; ++sp) {
              const int s = pauli_src<C>(fe.op, sp);
              const C f = pauli_fac<C>(fe.op, sp);
              const int cmb = fe.a * 4 + sp * 2 + s;
              R re = R(0), im = R(0);
              for (int k = tid; k < TEAM; k += 32) { re += part[(2 * cmb) * TEAM + k]; im += part[(2 * cmb + 1) * TEAM + k]; }
#pragma unroll
              for (int off = 16; off > 0; off >>= 1) {
                re += __shfl_xor_sync(0xffffffffu, re, off);
                im += __shfl_xor_sync(0xffffffffu, im, off);
              }
              vre += double(f.x) * re - double(f.y) * im;
              vim += double(f.x) * im + double(f.y) * re;
            }
            if (tid == 0) {
              double* o = p.values + ((size_t)b * p.c.n_terms + fe.b) * 2;
              o[0] = vre; o[1] = vim;
            }
          }
        }
      }
      team_sync<TEAM>();
    }
  }
}

// ------------------------------------------------------------------ reductions
template <typename R>
__global__ void reduce_energy(const tq_chain c, int batch, const void* epart, double* energy) {
  using C = typename CT<R>::T;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const C* e = reinterpret_cast<const C*>(epart) + (size_t)b * c.n_segments;
  double re = c.e_const_re, im = c.e_const_im;
  for (int g = 0; g < c.n_segments; ++g) { re += double(e[g].x); im += double(e[g].y); }
  energy[2 * b] = re; energy[2 * b + 1] = im;
}

template <typename R>
__global__ void reduce_grad(const tq_chain c, int batch, const R* gpart, R* grad) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)batch * c.n_params) return;
  const int b = int(idx / c.n_params), pp = int(idx % c.n_params);
  const R* src = gpart + (size_t)b * c.n_gslots;
  R s = R(0);
  for (int i = c.gred_ptr[pp]; i < c.gred_ptr[pp + 1]; ++i) s += src[c.gred_idx[i]];
  grad[idx] = s;
}

__global__ void fill_identity_values(const tq_chain c, int batch, double* values) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)batch * c.n_terms) return;
  const int t = int(idx % c.n_terms);
  if (c.term_active[t] == 0) { values[2 * idx] = 1.0; values[2 * idx + 1] = 0.0; }
}

// FP32 SIMT peak probe: 8 independent FFMA chains per thread (the roofline denominator
// for the SIMT-bound sweeps; MEASURED_PEAKS.json holds only HBM and bf16 tensor figures).
__global__ void ffma_probe(float* out, int iters, float seed) {
  float a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const float m = 0.999999f, c = 1e-7f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fmaf(a0, m, c); a1 = fmaf(a1, m, c); a2 = fmaf(a2, m, c); a3 = fmaf(a3, m, c);
      a4 = fmaf(a4, m, c); a5 = fmaf(a5, m, c); a6 = fmaf(a6, m, c); a7 = fmaf(a7, m, c);
    }
  }
  const float r = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (r == 12345.678f) out[blockIdx.x] = r;  // keep the chains alive
}

// ------------------------------------------------------------------ host side
static thread_local char g_err[512];

static tq_status fail(tq_status s, const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return s;
}

static int team_for_chi(int chi) { return chi <= 8 ? 32 : (chi == 16 ? 128 : 256); }
static int chi_bucket(int chi) { int c = 2; while (c < chi) c <<= 1; return c; }

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Shared-memory layout of one team for the given pass; mirrors the pointer carving above.
static Layout make_layout(const tq_chain* c, int chi, int team, size_t rsz, bool lr, int mode) {
  Layout L{};
  const size_t csz = 2 * rsz;
  const int LD = chi + 1;
  const size_t ms = (size_t)LD * LD * csz;
  const int D = c->d_max < 1 ? 1 : c->d_max;
  size_t off = 0;
  L.a = (int32_t)off; off += 2 * ms;
  L.ah = (int32_t)off; off += 2 * ms;
  L.env = (int32_t)off; off += (size_t)D * ms;       // RL: P in/out; LR: Lambda
  L.m = (int32_t)off; off += (size_t)2 * D * ms;     // RL: N; LR: M (G aliases)
  L.br = (int32_t)off; off += (size_t)2 * D * ms;
  L.pin = (int32_t)off;
  if (lr) off += (size_t)D * ms;
  L.mr = (int32_t)off;
  if (lr && mode == 1) off += (size_t)2 * D * ms;
  // contrib / value partials: alias the bracket region when it fits
  const int ntr = c->max_train > 0 ? c->max_train : 1;
  size_t need = lr ? (size_t)(mode == 0 ? ntr : 8 * D) * team * rsz : 0;
  if (need <= (size_t)2 * D * ms) L.contrib = L.br;
  else { L.contrib = (int32_t)off; off += align_up(need, 16); }
  L.mres = (int32_t)off; off += (size_t)c->max_lmat * 4 * csz;
  off = align_up(off, 16);
  L.minfo = (int32_t)off; off += align_up((size_t)c->max_lmat * 4, 16);
  L.mps = (int32_t)off; off += align_up((size_t)c->max_lmat * rsz, 16);
  L.team_bytes = (int32_t)align_up(off, 128);
  return L;
}

struct WsLayout { size_t env, epart, gpart, total; };

static WsLayout ws_layout(const tq_chain* c, int batch, int flags, int dtype) {
  const size_t rsz = dtype == TQ_C128 ? 8 : 4;
  WsLayout w{};
  size_t off = 0;
  w.env = off;
  if (flags & (TQ_FLAG_GRAD | TQ_FLAG_VALUES)) off += align_up((size_t)batch * c->env_total * 2 * rsz, 256);
  w.epart = off; off += align_up((size_t)batch * c->n_segments * 2 * rsz, 256);
  w.gpart = off;
  if (flags & TQ_FLAG_GRAD) off += align_up((size_t)batch * (c->n_gslots > 0 ? c->n_gslots : 1) * rsz, 256);
  w.total = off + 256;
  return w;
}

struct Timing { cudaEvent_t ev[4]; bool on; };
static thread_local Timing g_timing = {{nullptr, nullptr, nullptr, nullptr}, false};

template <typename R, int CHI>
static tq_status launch_pair(Params& prm, bool run_lr, cudaStream_t s) {
  constexpr int TEAM = CHI <= 8 ? 32 : (CHI == 16 ? 128 : 256);
  constexpr int TEAMS = TEAM == 32 ? 4 : 1;
  const int items = prm.batch * prm.c.n_segments;
  const int grid = (items + TEAMS - 1) / TEAMS;
  {
    Params q = prm;
    q.L = make_layout(&prm.c, CHI, TEAM, sizeof(R), false, prm.mode);
    const size_t smem = (size_t)q.L.team_bytes * TEAMS;
    if (smem > 227 * 1024) return fail(TQ_ERR_UNSUPPORTED, "shared-memory layout exceeds 227 KB (too many MPO channels for this bond dimension)");
    cudaFuncSetAttribute(rl_sweep<R, CHI, TEAM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (g_timing.on) cudaEventRecord(g_timing.ev[0], s);
    rl_sweep<R, CHI, TEAM><<<grid, TEAM * TEAMS, smem, s>>>(q);
    if (g_timing.on) cudaEventRecord(g_timing.ev[1], s);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(TQ_ERR_CUDA, cudaGetErrorString(e));
  }
  if (run_lr) {
    Params q = prm;
    q.L = make_layout(&prm.c, CHI, TEAM, sizeof(R), true, prm.mode);
    const size_t smem = (size_t)q.L.team_bytes * TEAMS;
    if (smem > 227 * 1024) return fail(TQ_ERR_UNSUPPORTED, "shared-memory layout exceeds 227 KB (too many MPO channels for this bond dimension)");
    cudaFuncSetAttribute(lr_sweep<R, CHI, TEAM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (g_timing.on) cudaEventRecord(g_timing.ev[2], s);
    lr_sweep<R, CHI, TEAM><<<grid, TEAM * TEAMS, smem, s>>>(q);
    if (g_timing.on) cudaEventRecord(g_timing.ev[3], s);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(TQ_ERR_CUDA, cudaGetErrorString(e));
  }
  return TQ_OK;
}

template <typename R>
static tq_status dispatch(Params& prm, bool run_lr, cudaStream_t s) {
  const int chi = chi_bucket(prm.c.chi_max);
  switch (chi) {
    case 2: return launch_pair<R, 2>(prm, run_lr, s);
    case 4: return launch_pair<R, 4>(prm, run_lr, s);
    case 8: return launch_pair<R, 8>(prm, run_lr, s);
    case 16: return launch_pair<R, 16>(prm, run_lr, s);
    case 32:
      if (sizeof(R) == 8) return fail(TQ_ERR_UNSUPPORTED, "complex128 mode supports bond dimension <= 16");
      return launch_pair<R, 32>(prm, run_lr, s);
    default: return fail(TQ_ERR_UNSUPPORTED, "bond dimension exceeds 32");
  }
}

static tq_status check_chain(const tq_chain* c, int batch) {
  if (!c) return fail(TQ_ERR_INPUT, "null chain");
  if (batch < 0) return fail(TQ_ERR_INPUT, "negative batch");
  if (c->chi_max > 32) return fail(TQ_ERR_UNSUPPORTED, "bond dimension exceeds 32");
  return TQ_OK;
}

template <typename R>
static tq_status energy_grad_impl(const tq_chain* c, int batch, const void* theta, int64_t ts, const void* coef,
                                  int64_t cs, double* energy, void* grad, void* ws, size_t wsb, cudaStream_t s) {
  const int flags = grad ? TQ_FLAG_GRAD : 0;
  const int dtype = sizeof(R) == 8 ? TQ_C128 : TQ_C64;
  WsLayout w = ws_layout(c, batch, flags, dtype);
  if (wsb < w.total) return fail(TQ_ERR_WORKSPACE, "workspace too small");
  unsigned char* wb = reinterpret_cast<unsigned char*>(align_up(reinterpret_cast<size_t>(ws), 256));
  Params prm{};
  prm.c = *c; prm.batch = batch; prm.theta = theta; prm.theta_stride = ts; prm.coef = coef; prm.coef_stride = cs;
  prm.env = wb + w.env; prm.epart = wb + w.epart; prm.gpart = wb + w.gpart; prm.values = nullptr;
  prm.store_env = grad ? 1 : 0; prm.mode = 0;
  if (batch == 0) return TQ_OK;
  if (c->n_segments > 0) {
    tq_status st = dispatch<R>(prm, grad != nullptr, s);
    if (st != TQ_OK) return st;
  }
  reduce_energy<R><<<(batch + 127) / 128, 128, 0, s>>>(*c, batch, prm.epart, energy);
  if (grad) {
    const int64_t n = (int64_t)batch * c->n_params;
    if (n > 0) reduce_grad<R><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(*c, batch, reinterpret_cast<const R*>(prm.gpart), reinterpret_cast<R*>(grad));
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(TQ_ERR_CUDA, cudaGetErrorString(e));
  return TQ_OK;
}

template <typename R>
static tq_status values_impl(const tq_chain* c, int batch, const void* theta, int64_t ts, double* values,
                             void* ws, size_t wsb, cudaStream_t s) {
  const int dtype = sizeof(R) == 8 ? TQ_C128 : TQ_C64;
  WsLayout w = ws_layout(c, batch, TQ_FLAG_VALUES, dtype);
  if (wsb < w.total) return fail(TQ_ERR_WORKSPACE, "workspace too small");
  unsigned char* wb = reinterpret_cast<unsigned char*>(align_up(reinterpret_cast<size_t>(ws), 256));
  Params prm{};
  prm.c = *c; prm.batch = batch; prm.theta = theta; prm.theta_stride = ts; prm.coef = nullptr; prm.coef_stride = 0;
  prm.env = wb + w.env; prm.epart = wb + w.epart; prm.gpart = nullptr; prm.values = values;
  prm.store_env = 1; prm.mode = 1;
  if (batch == 0) return TQ_OK;
  const int64_t n = (int64_t)batch * c->n_terms;
  if (n > 0) fill_identity_values<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(*c, batch, values);
  if (c->n_segments > 0) {
    tq_status st = dispatch<R>(prm, true, s);
    if (st != TQ_OK) return st;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(TQ_ERR_CUDA, cudaGetErrorString(e));
  return TQ_OK;
}

}  // namespace tq

using namespace tq;

extern "C" {

size_t tq_workspace_bytes(const tq_chain* chain, int32_t batch, int32_t flags, int32_t dtype) {
  if (!chain) return 0;
  return ws_layout(chain, batch, flags, dtype).total;
}

tq_status tq_energy_grad(const tq_chain* chain, int32_t dtype, int32_t batch, const void* theta, int64_t theta_stride,
                         const void* coef, int64_t coef_stride, double* energy, void* grad, void* workspace,
                         size_t workspace_bytes, void* stream) {
  tq_status st = check_chain(chain, batch);
  if (st != TQ_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == TQ_C64) return energy_grad_impl<float>(chain, batch, theta, theta_stride, coef, coef_stride, energy, grad, workspace, workspace_bytes, s);
  if (dtype == TQ_C128) return energy_grad_impl<double>(chain, batch, theta, theta_stride, coef, coef_stride, energy, grad, workspace, workspace_bytes, s);
  return fail(TQ_ERR_INPUT, "unknown dtype");
}

tq_status tq_term_values(const tq_chain* chain, int32_t dtype, int32_t batch, const void* theta, int64_t theta_stride,
                         double* values, void* workspace, size_t workspace_bytes, void* stream) {
  tq_status st = check_chain(chain, batch);
  if (st != TQ_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == TQ_C64) return values_impl<float>(chain, batch, theta, theta_stride, values, workspace, workspace_bytes, s);
  if (dtype == TQ_C128) return values_impl<double>(chain, batch, theta, theta_stride, values, workspace, workspace_bytes, s);
  return fail(TQ_ERR_INPUT, "unknown dtype");
}

tq_status tq_energy_grad_timed(const tq_chain* chain, int32_t dtype, int32_t batch, const void* theta,
                               int64_t theta_stride, const void* coef, int64_t coef_stride, double* energy, void* grad,
                               void* workspace, size_t workspace_bytes, void* stream, float* ms_out) {
  for (int i = 0; i < 4; ++i) cudaEventCreate(&g_timing.ev[i]);
  g_timing.on = true;
  tq_status st = tq_energy_grad(chain, dtype, batch, theta, theta_stride, coef, coef_stride, energy, grad, workspace,
                                workspace_bytes, stream);
  g_timing.on = false;
  if (st == TQ_OK) {
    cudaEventSynchronize(g_timing.ev[grad ? 3 : 1]);
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, g_timing.ev[0], g_timing.ev[1]);
    if (grad) cudaEventElapsedTime(&b, g_timing.ev[2], g_timing.ev[3]);
    ms_out[0] = a; ms_out[1] = b;
  }
  for (int i = 0; i < 4; ++i) cudaEventDestroy(g_timing.ev[i]);
  return st;
}

tq_status tq_ffma_peak(int32_t iters, void* stream, double* tflops_out) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* out = nullptr;
  if (cudaMalloc(&out, sizeof(float) * sms * 8) != cudaSuccess) return fail(TQ_ERR_CUDA, "cudaMalloc failed");
  const int blocks = sms * 8, threads = 256;
  ffma_probe<<<blocks, threads, 0, s>>>(out, 8, 1.0f);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  ffma_probe<<<blocks, threads, 0, s>>>(out, iters, 1.0f);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0); cudaEventDestroy(e1);
  cudaFree(out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(TQ_ERR_CUDA, cudaGetErrorString(e));
  const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  *tflops_out = flops / (ms * 1e-3) / 1e12;
  return TQ_OK;
}

tq_status tq_inner(const tq_chain*, const void*, int64_t, const tq_chain*, const void*, int64_t, int32_t, int32_t,
                   double*, void*) {
  return fail(TQ_ERR_UNSUPPORTED, "tq_inner is not built in this version");
}

const char* tq_status_string(tq_status s) {
  switch (s) {
    case TQ_OK: return "ok";
    case TQ_ERR_INPUT: return "invalid input";
    case TQ_ERR_UNSUPPORTED: return "unsupported configuration";
    case TQ_ERR_CUDA: return "CUDA error";
    case TQ_ERR_WORKSPACE: return "workspace too small";
    default: return "unknown status";
  }
}

const char* tq_last_error(void) { return g_err; }

int32_t tq_abi_layout(int32_t* sizes, int32_t n) {
  const int32_t v[7] = {(int32_t)sizeof(tq_site), (int32_t)sizeof(tq_op), (int32_t)sizeof(tq_mat), (int32_t)sizeof(tq_edge),
                        (int32_t)sizeof(tq_pass), (int32_t)sizeof(tq_segment), (int32_t)sizeof(tq_chain)};
  for (int i = 0; i < n && i < 7; ++i) sizes[i] = v[i];
  return 7;
}

const char* tq_build_info(void) {
  return "tq_engine sm_100a: rl_sweep/lr_sweep<float|double, chi 2..32>, reduce_energy, reduce_grad, ffma_probe";
}

}  // extern "C"
