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
#include "tq_debug.cuh"
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>

#include <algorithm>
#include <mutex>

#include "../../include/tq_engine.h"

#ifndef TQ_RE_TILE44
#define TQ_RE_TILE44 1   // real-path 4x4 register tiles (0: the complex path's 4x2 tiling)
#endif
#ifndef TQ_RE_HERM44
#define TQ_RE_HERM44 1   // real-path 4x4 tiles for the Hermitian X^H-operand GEMM (LR Lambda)
#endif
#ifndef TQ_TEAM32
#define TQ_TEAM32 512   // threads per chi = 32 team (one CTA); same-box A/B cfg4: 512 3387, 384 3278, 256 3335 evals/s
#endif

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

// acc += a * conj(b)
template <typename C> __device__ __forceinline__ void cfmacb(C& acc, C a, C b) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.y, b.x, acc.y); acc.y = fma(-a.x, b.y, acc.y);
}

// ------------------------------------------------------------------ kernel parameters
// Complex multiply-accumulate of the GEMMs (K: 0 a*b, 1 conj(a)*b, 2 a*conj(b)), or with RE the
// real part alone: the real-path sweeps (tq_chain.real_path) hold complex operands whose
// imaginary parts are exact zeros, so the real FMA chain is the complex one's real part, bit for bit.
template <bool RE, int K, typename C>
__device__ __forceinline__ void gmac(C& acc, C a, C b) {
  if constexpr (RE) acc.x = fma(a.x, b.x, acc.x);
  else if constexpr (K == 0) cfma(acc, a, b);
  else if constexpr (K == 1) cfmac(acc, a, b);
  else cfmacb(acc, a, b);
}

struct Layout {          // byte offsets inside one team's shared-memory slab (host computed)
  int32_t a, ah, env, m, br, pin, mr, contrib, mres, minfo, mps, ocode, ogidx, obase, sedge;
  int32_t tree;          // 0: per-pair column walks; 1: digit tree, dedicated levels; 2: digit tree in M/BR scratch
  int32_t lev, ubuf;     // digit-tree level storage and the adjoint's ping-pong buffers
  int32_t raw0, raw1;    // descriptor-blob double buffer
  int32_t dstride;       // bytes between the two resolved-descriptor buffers (mres .. sbuf)
  int32_t sbuf;          // blob header + tq_site copy inside a resolved-descriptor buffer
  int32_t direct;        // warp teams, one (alpha,beta) pair per lane: G computed in-lane, no G slots;
                         // folded cores (A, A2 ping-pong) and P (dense) are cp.async-prefetched
  int32_t a2;            // second folded-core buffer (direct path)
  int32_t wc;            // fused path: per-site channel-pair 2x2 bracket matrices + nonzero mask
  int32_t lrpf;          // chi >= 16 gradient LR sweep: A (ping-pong A / A2) and P cp.async-prefetched
  int32_t rlpre;         // chi >= 16 energy RL sweep: the next site is folded into A2 (ping-pong) during P
  int32_t team_bytes;
};

// Site edge staged in shared memory with its coefficient already resolved for this theta-set.
template <typename R> struct SEdge { int a, b, op; R coef; };

// Packed column op: lmat[0:9] src[9:11] kshift[11:16] bits[16:18] tidx+1[18:24] toff[24:29].
// kshift is the digit's bit position in the pair key al | be << 8 (shift, plus 8 when the digit
// comes from beta), so the decode is one shift and mask; bits = 0 (no digit) gives digit 0.
__device__ __forceinline__ int oc_lmat(int c) { return c & 511; }
__device__ __forceinline__ int oc_tidx(int c) { return ((c >> 18) & 63) - 1; }
__device__ __forceinline__ int oc_toff(int c) { return (c >> 24) & 31; }
__device__ __forceinline__ int oc_bits(int c) { return (c >> 16) & 3; }
__device__ __forceinline__ int oc_shift(int c) { return (c >> 11) & 7; }   // within al or be
__device__ __forceinline__ int oc_digit(int c, int al, int be) {
  return ((al | (be << 8)) >> ((c >> 11) & 31)) & ((1 << ((c >> 16) & 3)) - 1);
}

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
  const unsigned char* wct;   // per-(site, direction) bracket matrices built once per launch (or null)
  int32_t wct_row;            // bytes per table row
};

// Optional per-stage cycle accounting (diagnostic build with -DTQ_STAGE_TIMING only).
#ifdef TQ_STAGE_TIMING
__device__ unsigned long long g_stage_cycles[2][16];
#define STAGE_BEGIN() long long _t_prev = clock64(); long long _acc[16]; for (int _i = 0; _i < 16; ++_i) _acc[_i] = 0;
#define STAGE(k) do { const long long _t = clock64(); _acc[k] += _t - _t_prev; _t_prev = _t; } while (0)
#define STAGE_END(kern) do { if (tid == 0) for (int _i = 0; _i < 16; ++_i) atomicAdd(&g_stage_cycles[kern][_i], (unsigned long long)_acc[_i]); } while (0)
#else
#define STAGE_BEGIN()
#define STAGE(k)
#define STAGE_END(kern)
#endif

// Team barrier: a warp team syncs with __syncwarp, a CTA team with __syncthreads.
template <int TEAM> __device__ __forceinline__ void team_sync() {
  if (TEAM == 32) __syncwarp(); else __syncthreads();
}

// Barrier 1 over the upper N threads of a CTA (the half the split stages hand independent work)
template <int N> __device__ __forceinline__ void upper_sync() {
#ifdef TQ_DEBUG_RACE
  tq_dbg_delay();
#endif
  asm volatile("bar.sync 1, %0;" :: "r"(N) : "memory");
}
// The same barrier, also returning the AND of every participating thread's predicate
template <int N> __device__ __forceinline__ bool upper_sync_and(bool pred) {
#ifdef TQ_DEBUG_RACE
  tq_dbg_delay();
#endif
  unsigned out;
  asm volatile("{\n .reg .pred p, q;\n setp.ne.u32 p, %1, 0;\n bar.red.and.pred q, 1, %2, p;\n selp.u32 %0, 1, 0, q;\n}"
               : "=r"(out) : "r"((unsigned)pred), "r"(N) : "memory");
  return out != 0;
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
// cos(t/2), sin(t/2) of a rotation angle.  complex64 takes the fp64 sincos rounded to fp32:
// CUDA's fp32 sincosf is biased outward (mean c^2 + s^2 - 1 = +1.79e-8 over uniform angles,
// tools/micro/sincos_bias.cu), which grows the state norm by ~1.8e-7 per 10-rotation column and
// scales a 1000-site chain's energy by 1 + 1.8e-4 (tools/prec_diag.py); the rounded fp64 values
// are unbiased (mean -4.6e-12).
template <typename R>
__device__ __forceinline__ void half_angle_sincos(R t, R& sn, R& cs) {
  double sd, cd;
  sincos(double(t) * 0.5, &sd, &cd);
  sn = R(sd); cs = R(cd);
}

// Stage one site's descriptors for this theta-set into shared memory: the resolved
// 2x2 factors (entry e of the site lives at mats[ent_begin + e]), packed op codes and
// the MPO edges of the current sweep with their coefficients looked up once.
template <typename R, int TEAM>
__device__ void stage_site(const tq_chain& ch, const R* theta_row, const R* coef_row, const tq_site& st, int tid, bool rl,
                           typename CT<R>::T* mres, int* minfo, R* mps, int* ocode, int* ogidx, int* obase,
                           SEdge<R>* sedge) {
  using C = typename CT<R>::T;
  for (int e = tid; e < st.lmat_count; e += TEAM) {
    const tq_mat& mt = ch.mats[st.ent_begin + e];
    const int kind = mt.kind;
    C m00, m01, m10, m11;
    if (kind == 0) {
      m00 = cmk<C>(R(mt.m[0]), R(mt.m[1])); m01 = cmk<C>(R(mt.m[2]), R(mt.m[3]));
      m10 = cmk<C>(R(mt.m[4]), R(mt.m[5])); m11 = cmk<C>(R(mt.m[6]), R(mt.m[7]));
    } else {
      const R t = mt.slot >= 0 ? theta_row[mt.slot] : R(mt.angle);
      R sn, cs;
      half_angle_sincos<R>(t, sn, cs);
      const R z = R(0);
      if (kind == 1) { m00 = cmk<C>(cs, z); m01 = cmk<C>(z, -sn); m10 = cmk<C>(z, -sn); m11 = cmk<C>(cs, z); }
      else if (kind == 2) { m00 = cmk<C>(cs, z); m01 = cmk<C>(-sn, z); m10 = cmk<C>(sn, z); m11 = cmk<C>(cs, z); }
      else { m00 = cmk<C>(cs, -sn); m01 = cmk<C>(z, z); m10 = cmk<C>(z, z); m11 = cmk<C>(cs, sn); }
    }
    mres[4 * e + 0] = m00; mres[4 * e + 1] = m01; mres[4 * e + 2] = m10; mres[4 * e + 3] = m11;
    minfo[e] = (kind & 0xff) | ((mt.cls & 0xff) << 8);
    mps[e] = R(1) / R(mt.pscale);   // reciprocal: the adjoint rebuilds v[a] = v'[a] / pscale
  }
  for (int o = tid; o < st.op_count; o += TEAM) {
    const tq_op& op = ch.ops[st.op_begin + o];
    const int ksh = op.shift + (op.src == 2 ? 8 : 0);
    ocode[o] = op.lmat | (op.src << 9) | (ksh << 11) | ((op.src ? op.bits : 0) << 16) | ((op.tidx + 1) << 18) | (op.toff << 24);
    if (op.tidx >= 0) ogidx[op.tidx] = op.gidx;   // trainable index -> partial-gradient slot
    obase[o] = op.tbase;
  }
  const int eb = rl ? st.rl_edge_begin : st.lr_edge_begin;
  const int ec = rl ? st.rl_edge_count : st.lr_edge_count;
  for (int ei = tid; ei < ec; ei += TEAM) {
    const tq_edge ed = ch.edges[eb + ei];
    SEdge<R> se; se.a = ed.a; se.b = ed.b; se.op = ed.op; se.coef = ed.coef < 0 ? R(1) : coef_row[ed.coef];
    sedge[ei] = se;
  }
}


// ------------------------------------------------------------------ descriptor blobs
constexpr int SITE_UNITS = sizeof(tq_site) / 16;
static_assert(sizeof(tq_site) % 16 == 0, "tq_site must be a multiple of 16 bytes");
// One site's descriptors live in a contiguous 16-byte-aligned blob (include/tq_engine.h);
// the sweeps copy the NEXT site's blob into a shared-memory double buffer with cp.async
// while the current site computes, so descriptor staging never waits on global memory.
__device__ __forceinline__ void async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void blob_prefetch(int4* dst, const int4* src, int units, int tid, int team,
                                              bool commit = true) {
  for (int c = tid; c < units; c += team) {
    const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(dst + c));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(saddr), "l"(src + c) : "memory");
  }
  if (commit) async_commit();
}
// one complex element global -> shared, asynchronously (8 or 16 bytes)
template <typename C>
__device__ __forceinline__ void async_elem(C* dst, const C* src) {
  const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  if constexpr (sizeof(C) == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" :: "r"(saddr), "l"(src) : "memory");
  else
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(saddr), "l"(src) : "memory");
}
// folded core [2][cl][cr] (dense, HBM) -> padded LD layout in shared memory
template <typename C, int LD, int TEAM>
__device__ __forceinline__ void async_core(C* dst, const C* src, int cl, int cr, int lcr, int tid) {
  constexpr int MS = LD * LD;
  const int np = cl * cr;
  for (int e = tid; e < 2 * np; e += TEAM) {
    const int sidx = e >= np, r = e - sidx * np;
    async_elem(dst + sidx * MS + (r >> lcr) * LD + (r & (cr - 1)), src + e);
  }
}
// nch stored environments [nch][cr][cr] (dense, HBM) -> padded LD layout in shared memory
template <typename C, int LD, int TEAM>
__device__ __forceinline__ void async_env(C* dst, const C* src, int nch, int cr, int lcr, int tid) {
  constexpr int MS = LD * LD;
  const int lper = 2 * lcr;
  for (int e = tid; e < (nch << lper); e += TEAM) {
    const int ch = e >> lper, r = e & ((1 << lper) - 1);
    async_elem(dst + ch * MS + (r >> lcr) * LD + (r & (cr - 1)), src + e);
  }
}
// n contiguous complex elements (element granularity: offsets are only element-aligned)
template <typename C, int TEAM>
__device__ __forceinline__ void async_dense(C* dst, const C* src, int n, int tid) {
  for (int e = tid; e < n; e += TEAM) async_elem(dst + e, src + e);
}
__device__ __forceinline__ void blob_wait() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

template <typename R, int TEAM, int DMW = 0>
__device__ void stage_blob(const int4* raw, const tq_site& st, const R* theta_row, const R* coef_row, bool rl, int tid,
                           typename CT<R>::T* mres, int* minfo, R* mps, int* ocode, int* ogidx, int* obase,
                           SEdge<R>* sedge, int4* sbuf, typename CT<R>::T* wc = nullptr,
                           const typename CT<R>::T* wct_row = nullptr, bool wct_async = false,
                           bool th_pre_ok = false, R th_pre = R(0)) {
  using C = typename CT<R>::T;
  constexpr int EU = sizeof(R) == 4 ? 3 : 6;    // 16-byte units per factor entry
  constexpr int FO = sizeof(R) == 4 ? 2 : 1;    // first real-valued field (1/pscale) within an entry
  if (tid < 1 + SITE_UNITS) sbuf[tid] = raw[tid];   // header + site struct for the sweep loop
  const int4* ops = raw + 1 + SITE_UNITS;
  const int4* ents = ops + st.op_count;
  const int4* edg = ents + EU * st.lmat_count + (rl ? 0 : st.rl_edge_count);
  for (int o = tid; o < st.op_count; o += TEAM) {
    const int4 r = ops[o];
    ocode[o] = r.x;
    obase[o] = r.z;
    if (r.w >= 0) ogidx[r.w] = r.y;
  }
  for (int e = tid; e < st.lmat_count; e += TEAM) {
    const int* ip = reinterpret_cast<const int*>(ents + EU * e);
    const R* rp = reinterpret_cast<const R*>(ents + EU * e);
    const int kind = ip[0] & 0xff, slot = ip[1];
    C m00, m01, m10, m11;
    if (kind == 0) {
      const R* m = rp + FO + 2;
      m00 = cmk<C>(m[0], m[1]); m01 = cmk<C>(m[2], m[3]); m10 = cmk<C>(m[4], m[5]); m11 = cmk<C>(m[6], m[7]);
    } else {
      // the caller may have loaded this lane's first angle ahead of time (latency off the path)
      const R t = slot >= 0 ? ((th_pre_ok && e == tid) ? th_pre : theta_row[slot]) : rp[FO + 1];
      R sn, cs;
      half_angle_sincos<R>(t, sn, cs);
      const R z = R(0);
      if (kind == 1) { m00 = cmk<C>(cs, z); m01 = cmk<C>(z, -sn); m10 = cmk<C>(z, -sn); m11 = cmk<C>(cs, z); }
      else if (kind == 2) { m00 = cmk<C>(cs, z); m01 = cmk<C>(-sn, z); m10 = cmk<C>(sn, z); m11 = cmk<C>(cs, z); }
      else { m00 = cmk<C>(cs, -sn); m01 = cmk<C>(z, z); m10 = cmk<C>(z, z); m11 = cmk<C>(cs, sn); }
    }
    mres[4 * e + 0] = m00; mres[4 * e + 1] = m01; mres[4 * e + 2] = m10; mres[4 * e + 3] = m11;
    minfo[e] = ip[0];
    mps[e] = rp[FO];
  }
  if constexpr (DMW > 0) {
    if (wct_row) {   // shared coefficients: the launch's table row replaces the edges entirely
      if (!wct_async)  // (else the caller cp.async-copied it already)
        for (int e = tid; e < 4 * DMW * DMW + 1; e += TEAM) wc[e] = wct_row[e];
      return;
    }
  }
  const int ec = sedge ? (rl ? st.rl_edge_count : st.lr_edge_count) : 0;
  for (int ei = tid; ei < ec; ei += TEAM) {
    const int4 r = edg[ei];
    SEdge<R> se; se.a = r.x; se.b = r.y; se.op = r.z; se.coef = r.w < 0 ? R(1) : coef_row[r.w];
    sedge[ei] = se;
  }
  if constexpr (DMW > 0) {
    // Channel-pair bracket matrices for the fused stages: W_c[s'][s] = sum coef <s'|O|s> over
    // the edges of channel pair c = src * DMW + tgt.  Bit c of the trailing mask word says W_c
    // is nonzero (the stage skips empty pairs).
    static_assert(2 * DMW * DMW <= 32, "fused bracket matrices are built by one warp");
    // staged edges (coefficients resolved) must be visible to the building warp: when warp 0
    // staged all of them a warp barrier suffices, otherwise the whole team synchronises
    if (TEAM == 32 || ec > 32) team_sync<TEAM>();
    else if (tid < 32) __syncwarp();
    // lane = (c, s'): each lane folds the edges of its channel pair into one row W_c[s'][.]
    C wa = cmk<C>(R(0), R(0)), wb = wa;
    bool any = false;
    if (tid < 2 * DMW * DMW) {
      const int cmb = tid >> 1, sp = tid & 1;
      const int csrc = cmb / DMW, ctgt = cmb % DMW;
      for (int ei = 0; ei < ec; ++ei) {
        const SEdge<R> ed = sedge[ei];
        const int src = rl ? ed.b : ed.a, tgt = rl ? ed.a : ed.b;
        if (src != csrc || tgt != ctgt) continue;
        any = true;
        const int sidx = pauli_src<C>(ed.op, sp);
        C f = pauli_fac<C>(ed.op, sp);
        f.x *= ed.coef; f.y *= ed.coef;
        const R m0 = sidx == 0 ? R(1) : R(0), m1 = R(1) - m0;
        wa.x = fma(m0, f.x, wa.x); wa.y = fma(m0, f.y, wa.y);
        wb.x = fma(m1, f.x, wb.x); wb.y = fma(m1, f.y, wb.y);
      }
      wc[2 * tid + 0] = wa; wc[2 * tid + 1] = wb;   // = wc[4 * cmb + 2 * sp + {0, 1}]
    }
    if (tid < 32) {
      const unsigned pm = __ballot_sync(0xffffffffu, any);
      unsigned m = 0;
#pragma unroll
      for (int c2 = 0; c2 < DMW * DMW; ++c2) m |= ((pm >> (2 * c2)) & 1u) << c2;
      if (tid == 0) reinterpret_cast<int*>(wc + 4 * DMW * DMW)[0] = (int)m;
    }
  }
}

// Per-(site, direction) channel-pair bracket matrices for a launch whose coefficient row is shared
// by every theta-set (the energy sweeps of a Hamiltonian): built once here instead of once per
// (theta-set, site) inside the sweeps.  Warp 0: right-to-left edges, warp 1: left-to-right.
template <typename R, int DMW>
__global__ void __launch_bounds__(64) build_wct(Params p) {
  using C = typename CT<R>::T;
  constexpr int EU = sizeof(R) == 4 ? 3 : 6;
  const int si = blockIdx.x, dir = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int4* raw = reinterpret_cast<const int4*>(p.c.blob) + p.c.blob_off[si];
  const tq_site st = *reinterpret_cast<const tq_site*>(raw + 1);
  const bool rl = dir == 0;
  const int4* edg = raw + 1 + SITE_UNITS + st.op_count + EU * st.lmat_count + (rl ? 0 : st.rl_edge_count);
  const int ec = rl ? st.rl_edge_count : st.lr_edge_count;
  const R* coef_row = reinterpret_cast<const R*>(p.coef);
  C* out = reinterpret_cast<C*>(const_cast<unsigned char*>(p.wct) + ((size_t)si * 2 + dir) * p.wct_row);
  C wa = cmk<C>(R(0), R(0)), wb = wa;
  bool any = false;
  if (lane < 2 * DMW * DMW) {
    const int cmb = lane >> 1, sp = lane & 1;
    const int csrc = cmb / DMW, ctgt = cmb % DMW;
    for (int ei = 0; ei < ec; ++ei) {
      const int4 r = edg[ei];
      const int src = rl ? r.y : r.x, tgt = rl ? r.x : r.y;
      if (src != csrc || tgt != ctgt) continue;
      any = true;
      const R cf = r.w < 0 ? R(1) : coef_row[r.w];
      const int sidx = pauli_src<C>(r.z, sp);
      C f = pauli_fac<C>(r.z, sp);
      f.x *= cf; f.y *= cf;
      const R m0 = sidx == 0 ? R(1) : R(0), m1 = R(1) - m0;
      wa.x = fma(m0, f.x, wa.x); wa.y = fma(m0, f.y, wa.y);
      wb.x = fma(m1, f.x, wb.x); wb.y = fma(m1, f.y, wb.y);
    }
    out[2 * lane + 0] = wa; out[2 * lane + 1] = wb;
  }
  const unsigned pm = __ballot_sync(0xffffffffu, any);
  unsigned m = 0;
#pragma unroll
  for (int c2 = 0; c2 < DMW * DMW; ++c2) m |= ((pm >> (2 * c2)) & 1u) << c2;
  if (lane == 0) {
    C mk = cmk<C>(R(0), R(0));
    reinterpret_cast<int*>(&mk)[0] = (int)m;
    out[4 * DMW * DMW] = mk;
  }
}

// Angle of entry `tid` of a site's descriptor blob, loaded early by the sweeps so its global
// latency overlaps the current site's GEMM (stage_blob then consumes it: th_pre).
template <typename R>
__device__ __forceinline__ R blob_theta(const int4* raw, const tq_site& st, const R* theta_row, int tid) {
  constexpr int EU = sizeof(R) == 4 ? 3 : 6;
  if (tid >= st.lmat_count) return R(0);
  const int4* ents = raw + 1 + SITE_UNITS + st.op_count;
  const int* ip = reinterpret_cast<const int*>(ents + EU * tid);
  const int slot = ip[1];
  return ((ip[0] & 0xff) != 0 && slot >= 0) ? theta_row[slot] : R(0);
}

__device__ __forceinline__ bool pass_ok(const tq_chain& ch, const tq_site& st, int al, int be) {
  for (int i = 0; i < st.pass_count; ++i) {
    const tq_pass ps = ch.passes[st.pass_begin + i];
    const int m = (1 << ps.bits) - 1;
    if (((al >> ps.sa) & m) != ((be >> ps.sb) & m)) return false;
  }
  return true;
}

// Fold the column of site st into A[s] (chi_l x chi_r, row stride LD) and AH[s] = A[s]^H.
template <typename R, int LD, int TEAM>
__device__ void fold_site(const tq_chain& ch, const tq_site& st, int tid, const typename CT<R>::T* mres,
                          const int* ocode, typename CT<R>::T* A, typename CT<R>::T* AH, int lcr) {
  using C = typename CT<R>::T;
  const int npair = st.chi_l * st.chi_r;
  for (int pi = tid; pi < npair; pi += TEAM) {
    const int al = pi >> lcr, be = pi & (st.chi_r - 1);
    C v0 = cmk<C>(R(st.init[0]), R(st.init[1]));
    C v1 = cmk<C>(R(st.init[2]), R(st.init[3]));
    if (st.pass_count && !pass_ok(ch, st, al, be)) { v0 = cmk<C>(R(0), R(0)); v1 = v0; }
    else {
#pragma unroll 4
      for (int oi = 0; oi < st.op_count; ++oi) {
        const int c = ocode[oi];
        const C* M = mres + 4 * (oc_lmat(c) + oc_digit(c, al, be));
        C n0 = cmul(M[0], v0); cfma(n0, M[1], v1);
        C n1 = cmul(M[2], v0); cfma(n1, M[3], v1);
        v0 = n0; v1 = n1;
      }
    }
    A[al * LD + be] = v0; A[LD * LD + al * LD + be] = v1;   // A slots are LD*LD apart
    if (AH) { AH[be * LD + al] = cconj(v0); AH[LD * LD + be * LD + al] = cconj(v1); }
  }
}

// Real parts of a resolved 2x2 factor (4 complex entries, 16-byte aligned in shared memory).
// complex64: two 16-byte loads instead of four 4-byte ones (the fold is shared-memory bound).
template <typename R>
__device__ __forceinline__ void real_factor(const typename CT<R>::T* M, R& m0, R& m1, R& m2, R& m3) {
  if constexpr (sizeof(R) == 4) {
    const float4 a = *reinterpret_cast<const float4*>(M), b = *reinterpret_cast<const float4*>(M + 2);
    m0 = a.x; m1 = a.z; m2 = b.x; m3 = b.z;
  } else {
    m0 = M[0].x; m1 = M[1].x; m2 = M[2].x; m3 = M[3].x;
  }
}

// fold_site (no AH) for a real column, as fold_site4r: real 2-vectors, 4 FMA per op, bit-identical.
template <typename R, int LD, int TEAM>
__device__ void fold_site_real(const tq_chain& ch, const tq_site& st, int tid, const typename CT<R>::T* mres,
                               const int* ocode, typename CT<R>::T* A, int lcr) {
  using C = typename CT<R>::T;
  const int npair = st.chi_l * st.chi_r;
  for (int pi = tid; pi < npair; pi += TEAM) {
    const int al = pi >> lcr, be = pi & (st.chi_r - 1);
    R v0 = R(st.init[0]), v1 = R(st.init[2]);
    if (st.pass_count && !pass_ok(ch, st, al, be)) { v0 = R(0); v1 = R(0); }
    else {
#pragma unroll 4
      for (int oi = 0; oi < st.op_count; ++oi) {
        const int c = ocode[oi];
        const C* M = mres + 4 * (oc_lmat(c) + oc_digit(c, al, be));
        R m0, m1, m2, m3;
        real_factor<R>(M, m0, m1, m2, m3);
        const R n0 = fma(m1, v1, m0 * v0);
        const R n1 = fma(m3, v1, m2 * v0);
        v0 = n0; v1 = n1;
      }
    }
    A[al * LD + be] = cmk<C>(v0, R(0)); A[LD * LD + al * LD + be] = cmk<C>(v1, R(0));
  }
}

// Is the column real?  Checks the resolved factors with indices tid, tid + STRIDE, ... (ry and
// real constants are real; rx / rz and complex constants are not) and the input vector; the
// caller ANDs the result over the threads that cover every factor.
template <typename R, int STRIDE>
__device__ __forceinline__ bool column_real(const tq_site& st, int tid, const typename CT<R>::T* mres, const int* minfo) {
  using C = typename CT<R>::T;
  bool real = st.init[1] == 0.0 && st.init[3] == 0.0;
  for (int e = tid; e < st.lmat_count; e += STRIDE) {
    const int kind = minfo[e] & 0xff;
    const C* m = mres + 4 * e;
    if (kind == 1 || kind == 3 || (kind == 0 && (m[0].y != R(0) || m[1].y != R(0) || m[2].y != R(0) || m[3].y != R(0))))
      real = false;
  }
  return real;
}

// The same fold with two pairs per thread walked in lockstep (CTA teams, chi >= 16: 1024 pairs
// on 512 threads).  The column is a chain of dependent 2x2 matvecs; interleaving two
// independent chains hides the shared-memory load and FMA latencies of each op.
template <typename R, int LD, int TEAM>
__device__ void fold_site2(const tq_chain& ch, const tq_site& st, int tid, const typename CT<R>::T* mres,
                           const int* ocode, typename CT<R>::T* A, int lcr) {
  using C = typename CT<R>::T;
  const int npair = st.chi_l * st.chi_r;
  const C i0 = cmk<C>(R(st.init[0]), R(st.init[1])), i1 = cmk<C>(R(st.init[2]), R(st.init[3]));
  const C z = cmk<C>(R(0), R(0));
  for (int pa = tid; pa < npair; pa += 2 * TEAM) {
    const int pb = pa + TEAM;
    const bool hb = pb < npair;
    const int ala = pa >> lcr, bea = pa & (st.chi_r - 1);
    const int alb = hb ? pb >> lcr : ala, beb = hb ? pb & (st.chi_r - 1) : bea;
    C a0 = i0, a1 = i1, b0 = i0, b1 = i1;
#pragma unroll 2
    for (int oi = 0; oi < st.op_count; ++oi) {
      const int c = ocode[oi];
      const C* Ma = mres + 4 * (oc_lmat(c) + oc_digit(c, ala, bea));
      const C* Mb = mres + 4 * (oc_lmat(c) + oc_digit(c, alb, beb));
      const C ma0 = Ma[0], ma1 = Ma[1], ma2 = Ma[2], ma3 = Ma[3];
      const C mb0 = Mb[0], mb1 = Mb[1], mb2 = Mb[2], mb3 = Mb[3];
      C na0 = cmul(ma0, a0), nb0 = cmul(mb0, b0);
      C na1 = cmul(ma2, a0), nb1 = cmul(mb2, b0);
      cfma(na0, ma1, a1); cfma(nb0, mb1, b1);
      cfma(na1, ma3, a1); cfma(nb1, mb3, b1);
      a0 = na0; a1 = na1; b0 = nb0; b1 = nb1;
    }
    if (st.pass_count && !pass_ok(ch, st, ala, bea)) { a0 = z; a1 = z; }
    A[ala * LD + bea] = a0; A[LD * LD + ala * LD + bea] = a1;
    if (hb) {
      if (st.pass_count && !pass_ok(ch, st, alb, beb)) { b0 = z; b1 = z; }
      A[alb * LD + beb] = b0; A[LD * LD + alb * LD + beb] = b1;
    }
  }
}

// Four pairs per thread in lockstep: the RL sweep's next-site fold on half a CTA (1024 pairs on
// 256 threads) while the other half runs the Hermitian P GEMM.
template <typename R, int LD, int TEAM>
__device__ void fold_site4(const tq_chain& ch, const tq_site& st, int tid, const typename CT<R>::T* mres,
                           const int* ocode, typename CT<R>::T* A, int lcr) {
  using C = typename CT<R>::T;
  const int npair = st.chi_l * st.chi_r;
  const C i0 = cmk<C>(R(st.init[0]), R(st.init[1])), i1 = cmk<C>(R(st.init[2]), R(st.init[3]));
  const C z = cmk<C>(R(0), R(0));
  for (int p0 = tid; p0 < npair; p0 += 4 * TEAM) {
    int al[4], be[4];
    C v0[4], v1[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int pp = p0 + k * TEAM < npair ? p0 + k * TEAM : p0;
      al[k] = pp >> lcr; be[k] = pp & (st.chi_r - 1);
      v0[k] = i0; v1[k] = i1;
    }
    for (int oi = 0; oi < st.op_count; ++oi) {
      const int c = ocode[oi];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const C* M = mres + 4 * (oc_lmat(c) + oc_digit(c, al[k], be[k]));
        const C m0 = M[0], m1 = M[1], m2 = M[2], m3 = M[3];
        C n0 = cmul(m0, v0[k]), n1 = cmul(m2, v0[k]);
        cfma(n0, m1, v1[k]); cfma(n1, m3, v1[k]);
        v0[k] = n0; v1[k] = n1;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (p0 + k * TEAM >= npair) break;
      if (st.pass_count && !pass_ok(ch, st, al[k], be[k])) { v0[k] = z; v1[k] = z; }
      A[al[k] * LD + be[k]] = v0[k]; A[LD * LD + al[k] * LD + be[k]] = v1[k];
    }
  }
}

// fold_site4 for a real column (real initial vector, every factor real: ry rotations and real
// constant factors such as the CZ / CNOT projector splits): the walk runs on real 2-vectors,
// 4 FMA per op and pair instead of 16, and A gets zero imaginary parts.  Bit-identical to the
// complex walk (every imaginary term it would add is an exact zero).
template <typename R, int LD, int TEAM>
__device__ void fold_site4r(const tq_chain& ch, const tq_site& st, int tid, const typename CT<R>::T* mres,
                            const int* ocode, typename CT<R>::T* A, int lcr) {
  using C = typename CT<R>::T;
  const int npair = st.chi_l * st.chi_r;
  const R i0 = R(st.init[0]), i1 = R(st.init[2]);
  for (int p0 = tid; p0 < npair; p0 += 4 * TEAM) {
    int al[4], be[4];
    R v0[4], v1[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int pp = p0 + k * TEAM < npair ? p0 + k * TEAM : p0;
      al[k] = pp >> lcr; be[k] = pp & (st.chi_r - 1);
      v0[k] = i0; v1[k] = i1;
    }
    for (int oi = 0; oi < st.op_count; ++oi) {
      const int c = ocode[oi];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const C* M = mres + 4 * (oc_lmat(c) + oc_digit(c, al[k], be[k]));
        R m0, m1, m2, m3;
        real_factor<R>(M, m0, m1, m2, m3);
        const R n0 = fma(m1, v1[k], m0 * v0[k]);
        const R n1 = fma(m3, v1[k], m2 * v0[k]);
        v0[k] = n0; v1[k] = n1;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (p0 + k * TEAM >= npair) break;
      R a0 = v0[k], a1 = v1[k];
      if (st.pass_count && !pass_ok(ch, st, al[k], be[k])) { a0 = R(0); a1 = R(0); }
      A[al[k] * LD + be[k]] = cmk<C>(a0, R(0)); A[LD * LD + al[k] * LD + be[k]] = cmk<C>(a1, R(0));
    }
  }
}

// ------------------------------------------------------------------ digit-tree column adjoint
// The column's ops introduce bond digits one at a time, so after op l the distinct column
// vectors are indexed by the digits introduced so far (toff_l + bits_l bits, the newest digit
// on top): level l holds 2^(toff_l+bits_l) 2-vectors, and the last level is A[.][alpha][beta]
// at index idx(alpha, beta).  Cost per column: sum_l 2^(bits so far) matvecs instead of
// chi_l*chi_r*L for per-pair walks.
//
// Compact storage (adj_sweep, chi >= 16): the adjoint reads a forward level V_l only at a
// trainable op, so only those levels are kept (levt, at per-op offsets tbase[oi]); the others
// ping-pong through two scratch buffers of 2^(bits) vectors, which the backward walk then reuses
// for U.  cfg4: 16 KB of kept levels instead of 49 KB for all of them, so four 128-thread units
// fit on an SM.
template <typename R, int TEAM, bool RE = false>
__device__ void ctree_forward(const tq_site& st, int tid, const typename CT<R>::T* mres, const int* ocode,
                              typename CT<R>::T* levt, typename CT<R>::T* scratch, int* tbase) {
  using C = typename CT<R>::T;
  const C i0 = cmk<C>(R(st.init[0]), R(st.init[1])), i1 = cmk<C>(R(st.init[2]), R(st.init[3]));
  const C* src = nullptr;   // null: the initial vector
  int tb = 0;
  for (int oi = 0; oi < st.op_count; ++oi) {
    const int c = ocode[oi];
    const int toff = oc_toff(c), nd = 1 << oc_bits(c), npv = 1 << toff;
    C* dst;
    if (oc_tidx(c) >= 0) {
      dst = levt + 2 * tb;
      if (tid == 0) tbase[oi] = tb;
      tb += npv * nd;
    } else {
      dst = scratch;   // possibly the level being read: one thread owns idx and all its children
    }
    const C* Mb = mres + 4 * oc_lmat(c);
    for (int idx = tid; idx < npv; idx += TEAM) {
      const C v0 = src ? src[2 * idx] : i0;
      const C v1 = src ? src[2 * idx + 1] : i1;
      for (int d = 0; d < nd; ++d) {
        const C* M = Mb + 4 * d;
        C n0, n1;
        if constexpr (RE) {   // real path: the complex product's real part, bit for bit
          R m0, m1, m2, m3;
          real_factor<R>(M, m0, m1, m2, m3);
          n0 = cmk<C>(fma(m1, v1.x, m0 * v0.x), R(0));
          n1 = cmk<C>(fma(m3, v1.x, m2 * v0.x), R(0));
        } else {
          n0 = cmul(M[0], v0); cfma(n0, M[1], v1);
          n1 = cmul(M[2], v0); cfma(n1, M[3], v1);
        }
        const int e = idx + (d << toff);
        dst[2 * e] = n0; dst[2 * e + 1] = n1;
      }
    }
    team_sync<TEAM>();
    src = dst;
  }
}

__device__ __forceinline__ int tree_index(const int* ocode, int nops, int al, int be) {
  int idx = 0;
  for (int oi = 0; oi < nops; ++oi) {
    const int c = ocode[oi];
    if (oc_bits(c)) idx |= oc_digit(c, al, be) << oc_toff(c);
  }
  return idx;
}

// Column adjoint on the compact tree: U_last[idx] = sum over passthrough-matched (alpha, beta)
// of the core cotangent (G[0], G[1])[alpha][beta] (read straight from HBM, dense [2][cl][cr]);
// walking down, every trainable rotation accumulates Im<U_l, sigma V_l> (per-warp partials in
// contrib) and U_{l-1}[idx] = sum_d M_l(d)^H U_l[idx | d << toff_l].
template <typename R, int TEAM, bool RE = false>
__device__ void ctree_adjoint(const tq_chain& ch, const tq_site& st, int tid, const typename CT<R>::T* mres,
                              const int* minfo, const int* ocode, const typename CT<R>::T* levt, const int* tbase,
                              typename CT<R>::T* ua, int* tal, const typename CT<R>::T* gg, int lcr, R* contrib) {
  using C = typename CT<R>::T;
  const int nops = st.op_count;
  if (nops == 0) return;
  const int np = st.chi_l * st.chi_r;
  const int clast = ocode[nops - 1];
  const int nlast = 1 << (oc_toff(clast) + oc_bits(clast));
  int npb = 0;
  for (int i = 0; i < st.pass_count; ++i) npb += ch.passes[st.pass_begin + i].bits;
  if (st.pass_count == 0) {
    // every bond bit is introduced by an op here: (alpha, beta) -> tree index is a bijection
    // onto the last level, so G is read coalesced in its natural order and scattered in smem.
    // The index separates, idx(al, be) = idx(al, 0) | idx(0, be) (alpha and beta digits land on
    // disjoint bits): one table per side instead of an op walk per pair.
    int* tbe = tal + st.chi_l;
    for (int x = tid; x < st.chi_l + st.chi_r; x += TEAM)
      (x < st.chi_l ? tal[x] : tbe[x - st.chi_l]) =
          x < st.chi_l ? tree_index(ocode, nops, x, 0) : tree_index(ocode, nops, 0, x - st.chi_l);
    team_sync<TEAM>();
    for (int pi = tid; pi < np; pi += TEAM) {
      const int e = tal[pi >> lcr] | tbe[pi & ((1 << lcr) - 1)];
      ua[2 * e] = gg[pi]; ua[2 * e + 1] = gg[np + pi];
    }
  }
  for (int e = tid; st.pass_count && e < nlast; e += TEAM) {
    int al = 0, be = 0;
    for (int oi = 0; oi < nops; ++oi) {
      const int c = ocode[oi];
      const int bits = oc_bits(c);
      if (!bits) continue;
      const int d = (e >> oc_toff(c)) & ((1 << bits) - 1);
      const int src = (c >> 9) & 3, shift = oc_shift(c);
      if (src == 1) al |= d << shift; else be |= d << shift;
    }
    C g0 = cmk<C>(R(0), R(0)), g1 = g0;
    for (int cmb = 0; cmb < (1 << npb); ++cmb) {
      int a2 = al, b2 = be, used = 0;
      for (int i = 0; i < st.pass_count; ++i) {
        const tq_pass ps = ch.passes[st.pass_begin + i];
        const int v = (cmb >> used) & ((1 << ps.bits) - 1);
        a2 |= v << ps.sa; b2 |= v << ps.sb; used += ps.bits;
      }
      const C x0 = gg[(a2 << lcr) + b2], x1 = gg[np + (a2 << lcr) + b2];
      g0.x += x0.x; g0.y += x0.y; g1.x += x1.x; g1.y += x1.y;
    }
    ua[2 * e] = g0; ua[2 * e + 1] = g1;
  }
  for (int oi = nops - 1; oi >= 0; --oi) {
    team_sync<TEAM>();
    const int c = ocode[oi];
    const int toff = oc_toff(c), bits = oc_bits(c);
    const int nn = 1 << (toff + bits);
    const int tix = oc_tidx(c);
    const int lm = oc_lmat(c);
    if (tix >= 0) {
      const C* V = levt + 2 * tbase[oi];
      R acc = R(0);
      for (int e = tid; e < nn; e += TEAM) {
        const int kind = minfo[lm + (e >> toff)] & 0xff;
        if (kind == 0) continue;
        const C u0 = ua[2 * e], u1 = ua[2 * e + 1];
        const C v0 = V[2 * e], v1 = V[2 * e + 1];
        if constexpr (RE) {   // real path: only ry (sigma = Y) is trainable; Im<u, Y v> in real terms
          acc += fma(u1.x, v0.x, -u0.x * v1.x);
          continue;
        }
        C s0, s1;
        if (kind == 1) { s0 = v1; s1 = v0; }
        else if (kind == 2) { s0 = cmk<C>(v1.y, -v1.x); s1 = cmk<C>(-v0.y, v0.x); }
        else { s0 = v0; s1 = cmk<C>(-v1.x, -v1.y); }
        C d = cmk<C>(R(0), R(0));
        cfmac(d, u0, s0); cfmac(d, u1, s1);
        acc += d.y;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if ((tid & 31) == 0) contrib[tix * (TEAM / 32) + (tid >> 5)] += acc;   // per-warp partials
    }
    if (oi > 0) {
      // in place: entry idx is read (with its children idx | d << toff) and written by one thread
      const int npv = 1 << toff;
      for (int idx = tid; idx < npv; idx += TEAM) {
        C w0 = cmk<C>(R(0), R(0)), w1 = w0;
        for (int d = 0; d < (1 << bits); ++d) {
          const C* M = mres + 4 * (lm + d);
          const C u0 = ua[2 * (idx | (d << toff))], u1 = ua[2 * (idx | (d << toff)) + 1];
          gmac<RE, 1>(w0, M[0], u0); gmac<RE, 1>(w0, M[2], u1);
          gmac<RE, 1>(w1, M[1], u0); gmac<RE, 1>(w1, M[3], u1);
        }
        ua[2 * idx] = w0; ua[2 * idx + 1] = w1;
      }
    }
  }
  team_sync<TEAM>();
}


// Warp-direct variant for one pair per lane (warp teams): every lane walks its pair (zero
// cotangent when it has none), each trainable op's contributions are summed with an xor tree
// inside the backward walk and lane 0 writes the partial gradient -- no shared-memory
// contribution array and no separate reduction stage.
template <typename R, int NR>
__device__ __forceinline__ void pair_adjoint_warp(int nops, int al, int be, const int* ocode, const int* ogidx,
                                                  const typename CT<R>::T* mres, const int* minfo,
                                                  typename CT<R>::T i0, typename CT<R>::T i1,
                                                  typename CT<R>::T u0, typename CT<R>::T u1,
                                                  R* gpart, int lane) {
  using C = typename CT<R>::T;
  C v0[NR + 1], v1[NR + 1];
  int ent[NR], code[NR];
  v0[0] = i0; v1[0] = i1;
#pragma unroll
  for (int l = 0; l < NR; ++l) {
    if (l < nops) {
      const int c = ocode[l];
      code[l] = c;
      ent[l] = oc_lmat(c) + oc_digit(c, al, be);
      const C* M = mres + 4 * ent[l];
      C n0 = cmul(M[0], v0[l]); cfma(n0, M[1], v1[l]);
      C n1 = cmul(M[2], v0[l]); cfma(n1, M[3], v1[l]);
      v0[l + 1] = n0; v1[l + 1] = n1;
    } else {
      code[l] = 0; ent[l] = 0; v0[l + 1] = v0[l]; v1[l + 1] = v1[l];
    }
  }
#pragma unroll
  for (int l = NR - 1; l >= 0; --l) {
    if (l < nops) {
      const int tix = oc_tidx(code[l]);
      if (tix >= 0) {   // uniform across the warp
        const int kind = minfo[ent[l]] & 0xff;
        R val = R(0);
        if (kind != 0) {
          const C a0 = v0[l + 1], a1 = v1[l + 1];
          C s0, s1;
          if (kind == 1) { s0 = a1; s1 = a0; }
          else if (kind == 2) { s0 = cmk<C>(a1.y, -a1.x); s1 = cmk<C>(-a0.y, a0.x); }
          else { s0 = a0; s1 = cmk<C>(-a1.x, -a1.y); }
          C d = cmk<C>(R(0), R(0));
          cfmac(d, u0, s0); cfmac(d, u1, s1);
          val = d.y;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) val += __shfl_xor_sync(0xffffffffu, val, off);
        if (lane == 0) gpart[ogidx[tix]] = val;
      }
      const C* M = mres + 4 * ent[l];
      C w0 = cmk<C>(R(0), R(0)), w1 = w0;
      cfmac(w0, M[0], u0); cfmac(w0, M[2], u1);
      cfmac(w1, M[1], u0); cfmac(w1, M[3], u1);
      u0 = w0; u1 = w1;
    }
  }
}

// Register-tiled complex GEMM over a group of equally shaped tasks:
//   C_t[m x n] = sum_{q < nq} A_{t,q}[m x kk] * B_{t,q}[kk x n]   (all row stride LD)
// Each item computes rt consecutive rows of one column; a warp's lanes walk columns so the
// A operand is a broadcast and the B operand a contiguous row.
template <typename C, int LD, int TEAM, bool CTA = false, bool CTB = false, bool HERM = false, bool RE = false,
          typename FA, typename FB, typename FS>
__device__ __forceinline__ void gemm_group(int tid, int ntasks, int m, int n, int kk, int nq, FA fa, FB fb, FS store) {
  // CTA: the A operand is stored as X (kk x m) and used as X^H; CTB likewise for B (n x kk).
  // HERM: every output C_t is Hermitian (m == n): only the tiles touching the upper triangle are
  // computed and each strictly-upper element is stored twice, (i, j) and conj at (j, i).
  // (chi = 32 on the tensor pipe with 3xTF32 mma.sync was measured and reverted: its biased fp32
  // accumulation drifts the norm over long chains, profiles/r02_mma3_tf32_trial.txt)
#if TQ_RE_HERM44
  // (CTA only, i.e. LR's Lambda: on RL's P GEMM, CTB, the 4 x 4 tiles measured 0.4% slower)
  if constexpr (HERM && RE && CTA) {
    if (LD >= 17 && m == n && n >= 16) {
      // real path: 4 x 4 tiles (row quad b, column quad c >= b), 36 of 64 at 32 x 32; same
      // per-element (q, k) order as the 4 x 2 tiles below, so results are identical
      // (cfg4 LR 4.72 -> 4.57 ms, same-box A/B)
      const int nb = m >> 2;
      const int per = nb * (nb + 1) / 2;
      const int total = ntasks * per;
      for (int it = tid; it < total; it += TEAM) {
        const int task = it / per;
        int r = it - task * per, b = 0;
        while (r >= nb - b) { r -= nb - b; ++b; }
        const int i0 = b << 2, j0 = (b + r) << 2;
        C acc[4][4];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int u = 0; u < 4; ++u) acc[x][u] = C{0, 0};
        for (int q = 0; q < nq; ++q) {
          const C* Ab = fa(task, q) + (CTA ? i0 : i0 * LD);
          const C* Bb = fb(task, q) + (CTB ? j0 * LD : j0);
#pragma unroll 4
          for (int k = 0; k < kk; ++k) {
            C a[4], bv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) bv[u] = CTB ? Bb[u * LD + k] : Bb[k * LD + u];
#pragma unroll
            for (int x = 0; x < 4; ++x) a[x] = CTA ? Ab[k * LD + x] : Ab[x * LD + k];
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
              for (int u = 0; u < 4; ++u) gmac<RE, 0>(acc[x][u], a[x], bv[u]);
          }
        }
        const C z = {0, 0};
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = i0 + x, j = j0 + u;
            if (j >= i) store(task, i, j, 1, acc[x][u], z, z, z);
            if (j > i) store(task, j, i, 1, cconj(acc[x][u]), z, z, z);
          }
      }
      return;
    }
  }
#endif
  if constexpr (HERM) {
    if (LD >= 17 && m == n && n >= 16) {
      // 4 rows x 2 adjacent columns per item, tiles (row block b, column pair c) with 2c + 1 >= 4b:
      // 72 of 128 tiles at 32 x 32 (the environment transfers of the MPO sweeps are Hermitian:
      // real coefficients, Hermitian Paulis)
      const int nb = m >> 2, nc = n >> 1;
      const int per = nb * nc - nb * (nb - 1);
      const int total = ntasks * per;
      for (int it = tid; it < total; it += TEAM) {
        const int task = it / per;
        int r = it - task * per, b = 0;
        while (r >= nc - 2 * b) { r -= nc - 2 * b; ++b; }
        const int i0 = b << 2, j0 = (2 * b + r) << 1;
        C c00 = {0, 0}, c10 = {0, 0}, c20 = {0, 0}, c30 = {0, 0};
        C c01 = {0, 0}, c11 = {0, 0}, c21 = {0, 0}, c31 = {0, 0};
        for (int q = 0; q < nq; ++q) {
          const C* Ab = fa(task, q) + (CTA ? i0 : i0 * LD);
          const C* B0 = fb(task, q) + (CTB ? j0 * LD : j0);
          const C* B1 = B0 + (CTB ? LD : 1);
          const int sa = CTA ? LD : 1, ra = CTA ? 1 : LD, sb = CTB ? 1 : LD;
#pragma unroll 4
          for (int k = 0; k < kk; ++k) {
            C b0 = B0[k * sb], b1 = B1[k * sb];
            if (CTB) { b0 = cconj(b0); b1 = cconj(b1); }
            const C a0 = Ab[k * sa], a1 = Ab[ra + k * sa], a2 = Ab[2 * ra + k * sa], a3 = Ab[3 * ra + k * sa];
            if (CTA) {
              gmac<RE, 1>(c00, a0, b0); gmac<RE, 1>(c10, a1, b0); gmac<RE, 1>(c20, a2, b0); gmac<RE, 1>(c30, a3, b0);
              gmac<RE, 1>(c01, a0, b1); gmac<RE, 1>(c11, a1, b1); gmac<RE, 1>(c21, a2, b1); gmac<RE, 1>(c31, a3, b1);
            } else {
              gmac<RE, 0>(c00, a0, b0); gmac<RE, 0>(c10, a1, b0); gmac<RE, 0>(c20, a2, b0); gmac<RE, 0>(c30, a3, b0);
              gmac<RE, 0>(c01, a0, b1); gmac<RE, 0>(c11, a1, b1); gmac<RE, 0>(c21, a2, b1); gmac<RE, 0>(c31, a3, b1);
            }
          }
        }
        const C v[4][2] = {{c00, c01}, {c10, c11}, {c20, c21}, {c30, c31}};
        const C z = {0, 0};
#pragma unroll
        for (int rr = 0; rr < 4; ++rr)
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const int i = i0 + rr, j = j0 + cc;
            if (j >= i) store(task, i, j, 1, v[rr][cc], z, z, z);
            if (j > i) store(task, j, i, 1, cconj(v[rr][cc]), z, z, z);
          }
      }
      return;
    }
  }
#if TQ_RE_TILE44
  if constexpr (RE && !CTA && !CTB) {
    if (LD >= 17 && n >= 16 && m >= 4) {
      // real path: 4 rows x 4 columns (j + u n/4) per item.  The real FMA chain is smem-bound
      // (the dead imaginary halves share every wavefront): 8 loads per 16 FMA instead of 6 per 8.
      // Per output element the (q, k) accumulation order is unchanged, so results are identical.
      const int qn = n >> 2;
      const int lqn = 31 - __clz(qn);
      const int lmb = (31 - __clz(m)) - 2;
      const int lper = lmb + lqn;
      const int total = ntasks << lper;
      for (int it = tid; it < total; it += TEAM) {
        const int task = it >> lper;
        const int r = it & ((1 << lper) - 1);
        const int j = r & (qn - 1);
        const int i0 = (r >> lqn) << 2;
        C acc[4][4];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int u = 0; u < 4; ++u) acc[x][u] = C{0, 0};
        for (int q = 0; q < nq; ++q) {
          const C* Ab = fa(task, q) + i0 * LD;
          const C* Bb = fb(task, q) + j;
#pragma unroll 4
          for (int k = 0; k < kk; ++k) {
            C a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) b[u] = Bb[k * LD + u * qn];
#pragma unroll
            for (int x = 0; x < 4; ++x) a[x] = Ab[x * LD + k];
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
              for (int u = 0; u < 4; ++u) gmac<RE, 0>(acc[x][u], a[x], b[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) store(task, i0, j + u * qn, 4, acc[0][u], acc[1][u], acc[2][u], acc[3][u]);
      }
      return;
    }
  }
#endif
  if (LD >= 17 && n >= 16 && m >= 4) {
    // 4 rows x 2 columns (j, j + n/2) per item: 4 broadcast A loads + 2 B loads per 8 cMAC
    const int hn = n >> 1;
    const int lhn = 31 - __clz(hn);
    const int lmb = (31 - __clz(m)) - 2;
    const int lper = lmb + lhn;
    const int total = ntasks << lper;
    for (int it = tid; it < total; it += TEAM) {
      const int task = it >> lper;
      const int r = it & ((1 << lper) - 1);
      const int j = r & (hn - 1);
      const int i0 = (r >> lhn) << 2;
      C c00 = {0, 0}, c10 = {0, 0}, c20 = {0, 0}, c30 = {0, 0};
      C c01 = {0, 0}, c11 = {0, 0}, c21 = {0, 0}, c31 = {0, 0};
      for (int q = 0; q < nq; ++q) {
        const C* Ab = fa(task, q) + (CTA ? i0 : i0 * LD);
        const C* B0 = fb(task, q) + (CTB ? j * LD : j);
        const C* B1 = B0 + (CTB ? hn * LD : hn);
        const int sa = CTA ? LD : 1, ra = CTA ? 1 : LD, sb = CTB ? 1 : LD;
#pragma unroll 4
        for (int k = 0; k < kk; ++k) {
          C b0 = B0[k * sb], b1 = B1[k * sb];
          if (CTB) { b0 = cconj(b0); b1 = cconj(b1); }
          const C a0 = Ab[k * sa], a1 = Ab[ra + k * sa], a2 = Ab[2 * ra + k * sa], a3 = Ab[3 * ra + k * sa];
          if (CTA) {
            gmac<RE, 1>(c00, a0, b0); gmac<RE, 1>(c10, a1, b0); gmac<RE, 1>(c20, a2, b0); gmac<RE, 1>(c30, a3, b0);
            gmac<RE, 1>(c01, a0, b1); gmac<RE, 1>(c11, a1, b1); gmac<RE, 1>(c21, a2, b1); gmac<RE, 1>(c31, a3, b1);
          } else {
            gmac<RE, 0>(c00, a0, b0); gmac<RE, 0>(c10, a1, b0); gmac<RE, 0>(c20, a2, b0); gmac<RE, 0>(c30, a3, b0);
            gmac<RE, 0>(c01, a0, b1); gmac<RE, 0>(c11, a1, b1); gmac<RE, 0>(c21, a2, b1); gmac<RE, 0>(c31, a3, b1);
          }
        }
      }
      store(task, i0, j, 4, c00, c10, c20, c30);
      store(task, i0, j + hn, 4, c01, c11, c21, c31);
    }
    return;
  }
  // rows per item: minimise the critical path (rounds x rows) over the team; ties keep the
  // taller tile (fewer operand loads).  At chi <= 8 the shapes are tiny (e.g. 3 tasks of 4x4
  // leave 20 of 32 lanes idle with 4-row items), so the choice matters.
  int rt = 1;
  {
    const int cells = ntasks * m * n;
    int best = 1 << 30;
    for (int r = 4; r >= 1; r >>= 1) {
      if (r > m) continue;
      const int cost = (((cells >> (r >> 1)) + TEAM - 1) / TEAM) * r;
      if (cost < best) { best = cost; rt = r; }
    }
  }
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
      const C* Ab = fa(task, q) + (CTA ? i0 : i0 * LD);
      const C* Bb = fb(task, q) + (CTB ? j * LD : j);
      const int sa = CTA ? LD : 1;      // stride of A along k
      const int ra = CTA ? 1 : LD;      // stride of A along rows
      const int sb = CTB ? 1 : LD;      // stride of B along k
      if (rt == 4) {
#pragma unroll 4
        for (int k = 0; k < kk; ++k) {
          const C bv = Bb[k * sb];
          const C a0 = Ab[k * sa], a1 = Ab[ra + k * sa], a2 = Ab[2 * ra + k * sa], a3 = Ab[3 * ra + k * sa];
          if (CTA) {
            if (CTB) { C cb = cconj(bv); gmac<RE, 1>(acc0, a0, cb); gmac<RE, 1>(acc1, a1, cb); gmac<RE, 1>(acc2, a2, cb); gmac<RE, 1>(acc3, a3, cb); }
            else { gmac<RE, 1>(acc0, a0, bv); gmac<RE, 1>(acc1, a1, bv); gmac<RE, 1>(acc2, a2, bv); gmac<RE, 1>(acc3, a3, bv); }
          } else if (CTB) {
            gmac<RE, 2>(acc0, a0, bv); gmac<RE, 2>(acc1, a1, bv); gmac<RE, 2>(acc2, a2, bv); gmac<RE, 2>(acc3, a3, bv);
          } else {
            gmac<RE, 0>(acc0, a0, bv); gmac<RE, 0>(acc1, a1, bv); gmac<RE, 0>(acc2, a2, bv); gmac<RE, 0>(acc3, a3, bv);
          }
        }
      } else {
        for (int k = 0; k < kk; ++k) {
          const C bv = Bb[k * sb];
          const C a0 = Ab[k * sa];
          const C b2 = CTB ? cconj(bv) : bv;
          if (CTA) gmac<RE, 1>(acc0, a0, b2); else gmac<RE, 0>(acc0, a0, b2);
          if (rt == 2) {
            const C a1 = Ab[ra + k * sa];
            if (CTA) gmac<RE, 1>(acc1, a1, b2); else gmac<RE, 0>(acc1, a1, b2);
          }
        }
      }
    }
    store(task, i0, j, rt, acc0, acc1, acc2, acc3);
  }
}

// ------------------------------------------------------------------ shared-memory carving
template <typename R>
struct TeamSmem {
  using C = typename CT<R>::T;
  C *A, *AH, *ENV, *M, *BR, *PIN, *MR, *mres;
  R *contrib, *mps;
  int *minfo, *ocode, *ogidx, *obase;
  C *lev, *ubuf;
  SEdge<R>* sedge;
  int4* sbuf;
  __device__ TeamSmem(unsigned char* base, const Layout& L) {
    A = reinterpret_cast<C*>(base + L.a); AH = reinterpret_cast<C*>(base + L.ah);
    ENV = reinterpret_cast<C*>(base + L.env); M = reinterpret_cast<C*>(base + L.m);
    BR = reinterpret_cast<C*>(base + L.br); PIN = reinterpret_cast<C*>(base + L.pin);
    MR = reinterpret_cast<C*>(base + L.mr); mres = reinterpret_cast<C*>(base + L.mres);
    contrib = reinterpret_cast<R*>(base + L.contrib); mps = reinterpret_cast<R*>(base + L.mps);
    minfo = reinterpret_cast<int*>(base + L.minfo); ocode = reinterpret_cast<int*>(base + L.ocode);
    ogidx = reinterpret_cast<int*>(base + L.ogidx); sedge = reinterpret_cast<SEdge<R>*>(base + L.sedge);
    obase = reinterpret_cast<int*>(base + L.obase);
    lev = reinterpret_cast<C*>(base + L.lev); ubuf = reinterpret_cast<C*>(base + L.ubuf);
    base_ = base; L_ = &L;
  }
  unsigned char* base_;
  const Layout* L_;
  // point the descriptor fields at resolved buffer `buf` (0/1)
  __device__ void sel(int buf) {
    unsigned char* b = base_ + (size_t)buf * L_->dstride;
    mres = reinterpret_cast<C*>(b + L_->mres); mps = reinterpret_cast<R*>(b + L_->mps);
    minfo = reinterpret_cast<int*>(b + L_->minfo); ocode = reinterpret_cast<int*>(b + L_->ocode);
    ogidx = reinterpret_cast<int*>(b + L_->ogidx); obase = reinterpret_cast<int*>(b + L_->obase);
    sedge = reinterpret_cast<SEdge<R>*>(b + L_->sedge);
    sbuf = reinterpret_cast<int4*>(b + L_->sbuf);
  }
  __device__ const int4* sel_sbuf(int buf) const {
    return reinterpret_cast<const int4*>(base_ + (size_t)buf * L_->dstride + L_->sbuf);
  }
};

// BR[t][s'] = sum over staged edges with target t of coef * <s'|O|s> * SRC[src][s]
// (elementwise over chi_l x chi_r; `rl` selects which edge end is the target).
template <typename R, int LD, int TEAM>
__device__ __forceinline__ void bracket_stage(int tid, int ntarget, int ec, const SEdge<R>* sedge, bool rl,
                                              const typename CT<R>::T* SRC, typename CT<R>::T* BR,
                                              int lcl, int lcr) {
  using C = typename CT<R>::T;
  constexpr int MS = LD * LD;
  constexpr int U = 4;   // independent elements per thread iteration (ILP)
  const int lpair = lcl + lcr;
  const int nel = (ntarget * 2) << lpair;
  for (int e0 = tid; e0 < nel; e0 += TEAM * U) {
    int off[U], t[U], sp[U];
    bool on[U];
    R ax[U], ay[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * TEAM;
      on[u] = e < nel;
      const int ij = e & ((1 << lpair) - 1);
      const int ts = e >> lpair;
      t[u] = ts >> 1; sp[u] = ts & 1;
      off[u] = (ij >> lcr) * LD + (ij & ((1 << lcr) - 1));
      ax[u] = R(0); ay[u] = R(0);
    }
    for (int ei = 0; ei < ec; ++ei) {
      const SEdge<R> ed = sedge[ei];
      const int tgt = rl ? ed.a : ed.b, src = rl ? ed.b : ed.a;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!on[u] || tgt != t[u]) continue;
        const int s = pauli_src<C>(ed.op, sp[u]);
        const C f = pauli_fac<C>(ed.op, sp[u]);
        const C tt = cmul(f, SRC[(src * 2 + s) * MS + off[u]]);
        ax[u] = fma(ed.coef, tt.x, ax[u]);
        ay[u] = fma(ed.coef, tt.y, ay[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (on[u]) BR[(t[u] * 2 + sp[u]) * MS + off[u]] = cmk<C>(ax[u], ay[u]);
  }
}

// The same bracket from the site's channel-pair 2x2 matrices W_(src,tgt)[s'][s] (built once per
// launch by build_wct, or per site by stage_blob): every thread owns two (i, j) elements and
// forms all (target, s') outputs from all (source, s) inputs in registers, skipping channel pairs
// the mask marks empty.  chi >= 16 (the per-edge loop of bracket_stage is latency bound there).
template <typename R, int LD, int TEAM, int DM, bool RE = false>
__device__ __forceinline__ void wbracket_stage(int tid, int nsrc, int ntgt, const typename CT<R>::T* SRC,
                                               const typename CT<R>::T* wc, typename CT<R>::T* BR, int lcl, int lcr) {
  using C = typename CT<R>::T;
  constexpr int MS = LD * LD;
  constexpr int U = 2;
  const int wmask = reinterpret_cast<const int*>(wc + 4 * DM * DM)[0];
  const int nel = 1 << (lcl + lcr);
  for (int e0 = tid; e0 < nel; e0 += TEAM * U) {
    int off[U];
    bool on[U];
    C v[U][DM][2];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * TEAM;
      on[u] = e < nel;
      off[u] = on[u] ? (e >> lcr) * LD + (e & ((1 << lcr) - 1)) : 0;
#pragma unroll
      for (int x = 0; x < DM; ++x)
#pragma unroll
        for (int s = 0; s < 2; ++s)
          v[u][x][s] = (x < nsrc && on[u]) ? SRC[(x * 2 + s) * MS + off[u]] : cmk<C>(R(0), R(0));
    }
#pragma unroll
    for (int xt = 0; xt < DM; ++xt) {
      if (xt >= ntgt) continue;
      C o[U][2];
#pragma unroll
      for (int u = 0; u < U; ++u) { o[u][0] = cmk<C>(R(0), R(0)); o[u][1] = o[u][0]; }
#pragma unroll
      for (int xs = 0; xs < DM; ++xs) {
        if (!((wmask >> (xs * DM + xt)) & 1)) continue;
        const C* w = wc + 4 * (xs * DM + xt);
        const C w00 = w[0], w01 = w[1], w10 = w[2], w11 = w[3];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          gmac<RE, 0>(o[u][0], w00, v[u][xs][0]); gmac<RE, 0>(o[u][0], w01, v[u][xs][1]);
          gmac<RE, 0>(o[u][1], w10, v[u][xs][0]); gmac<RE, 0>(o[u][1], w11, v[u][xs][1]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (on[u]) { BR[(xt * 2 + 0) * MS + off[u]] = o[u][0]; BR[(xt * 2 + 1) * MS + off[u]] = o[u][1]; }
    }
  }
}

// Rows per item for the fused product+bracket stages: enough items for every thread.
__device__ __forceinline__ int fused_rows(int m, int nel, int team, int rtmax) {
  int rt = nel / team;
  rt = rt >= 4 ? 4 : (rt >= 2 ? 2 : 1);
  if (rt > rtmax) rt = rtmax;
  if (rt > m) rt = m;
  return rt;
}

// Select acc[idx][s][r] with runtime idx/s from a register array (unrolled, no local memory).
template <typename C, int DM, int RT>
__device__ __forceinline__ C pick(const C (&acc)[DM][2][RT], int idx, int s, int r) {
  C v = acc[0][0][0];
#pragma unroll
  for (int x = 0; x < DM; ++x)
#pragma unroll
    for (int y = 0; y < 2; ++y)
#pragma unroll
      for (int z = 0; z < RT; ++z)
        if (x == idx && y == s && z == r) v = acc[x][y][z];
  return v;
}

// Fused MPO product + bracket.  Right-to-left form (rl = true):
//   N[b][s] = A[s] (m x n) * P[b] (n x n);  BR[a][s'] = sum_edges(a<-b) coef <s'|O|s> N[b][s]
// Left-to-right form (rl = false):
//   M[a][s] = Lam[a] (m x m) * A[s] (m x n);  BR[b][s'] = sum_edges(a->b) coef <s'|O|s> M[a][s]
// Every item owns rows i0..i0+rt-1 of one column j for ALL (channel, s) products, so the
// products stay in registers and the bracket combination never touches shared memory.
template <typename R, int LD, int TEAM, int DM, int RT>
__device__ void product_bracket(int tid, bool rl, int nsrc, int ntgt, int m, int n, int lm, int ln,
                                const typename CT<R>::T* A, const typename CT<R>::T* ENV,
                                const typename CT<R>::T* wc, typename CT<R>::T* BR) {
  using C = typename CT<R>::T;
  constexpr int MS = LD * LD;
  const int wmask = reinterpret_cast<const int*>(wc + 4 * DM * DM)[0];
  const int rt = fused_rows(m, m * n, TEAM, RT);
  const int lrt = rt == 4 ? 2 : (rt == 2 ? 1 : 0);
  const int items = (m >> lrt) << ln;
  const int kk = rl ? n : m;
  for (int it = tid; it < items; it += TEAM) {
    const int j = it & (n - 1);
    const int i0 = (it >> ln) << lrt;
    C acc[DM][2][RT];
#pragma unroll
    for (int x = 0; x < DM; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y)
#pragma unroll
        for (int z = 0; z < RT; ++z) acc[x][y][z] = cmk<C>(R(0), R(0));
    if (rl) {
      for (int k = 0; k < kk; ++k) {
        C pb[DM];
#pragma unroll
        for (int x = 0; x < DM; ++x) pb[x] = x < nsrc ? ENV[x * MS + k * LD + j] : cmk<C>(R(0), R(0));
#pragma unroll
        for (int y = 0; y < 2; ++y)
#pragma unroll
          for (int z = 0; z < RT; ++z) {
            if (z < rt) {
              const C a = A[y * MS + (i0 + z) * LD + k];
#pragma unroll
              for (int x = 0; x < DM; ++x) if (x < nsrc) cfma(acc[x][y][z], a, pb[x]);
            }
          }
      }
    } else {
      for (int k = 0; k < kk; ++k) {
        const C b0 = A[k * LD + j], b1 = A[MS + k * LD + j];
#pragma unroll
        for (int x = 0; x < DM; ++x) {
          if (x < nsrc) {
#pragma unroll
            for (int z = 0; z < RT; ++z) {
              if (z < rt) {
                const C l = ENV[x * MS + (i0 + z) * LD + k];
                cfma(acc[x][0][z], l, b0);
                cfma(acc[x][1][z], l, b1);
              }
            }
          }
        }
      }
    }
    C br[DM][2][RT];
#pragma unroll
    for (int x = 0; x < DM; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y)
#pragma unroll
        for (int z = 0; z < RT; ++z) br[x][y][z] = cmk<C>(R(0), R(0));
    // BR[t][s'] += W_(src,t)[s'][s] acc[src][s] over the nonzero channel pairs (uniform mask;
    // every register index is a compile-time constant)
#pragma unroll
    for (int xs = 0; xs < DM; ++xs)
#pragma unroll
      for (int xt = 0; xt < DM; ++xt) {
        if (!((wmask >> (xs * DM + xt)) & 1)) continue;
        const C* w = wc + 4 * (xs * DM + xt);
        const C w00 = w[0], w01 = w[1], w10 = w[2], w11 = w[3];
#pragma unroll
        for (int z = 0; z < RT; ++z) {
          cfma(br[xt][0][z], w00, acc[xs][0][z]); cfma(br[xt][0][z], w01, acc[xs][1][z]);
          cfma(br[xt][1][z], w10, acc[xs][0][z]); cfma(br[xt][1][z], w11, acc[xs][1][z]);
        }
      }
#pragma unroll
    for (int x = 0; x < DM; ++x)
      if (x < ntgt)
#pragma unroll
        for (int y = 0; y < 2; ++y)
#pragma unroll
          for (int z = 0; z < RT; ++z)
            if (z < rt) BR[(x * 2 + y) * MS + (i0 + z) * LD + j] = br[x][y][z];
  }
}

template <typename C, int LD>
__device__ __forceinline__ void store_rows(C* o, int rt, C a0, C a1, C a2, C a3) {
  o[0] = a0;
  if (rt > 1) o[LD] = a1;
  if (rt > 2) { o[2 * LD] = a2; o[3 * LD] = a3; }
}

// Row of the launch's bracket-matrix table for (site, direction), or null (built in the sweep).
template <typename C>
__device__ __forceinline__ const C* wct_row_of(const Params& p, int site, int dir) {
  return p.wct ? reinterpret_cast<const C*>(p.wct + ((size_t)site * 2 + dir) * p.wct_row) : nullptr;
}
#define wct_row(p, site, dir) wct_row_of<C>(p, site, dir)

// ------------------------------------------------------------------ right-to-left sweep
// Computes the MPO right environments P^{(a)}_k for every cut of the segment's sub-chain,
// optionally storing them, and the segment's partial energy P^{START}_{lo}.
#ifndef TQ_RL_MINB
#define TQ_RL_MINB 4
#endif
#ifndef TQ_LR_MINB
#define TQ_LR_MINB 4
#endif
template <typename R, int CHI, int TEAM, int FD, bool RE = false>
__global__ void __launch_bounds__(TEAM == 32 ? 128 : TEAM, TEAM == 32 ? (sizeof(R) == 4 ? TQ_RL_MINB : 4) : 1)
rl_sweep(Params p) {
  using C = typename CT<R>::T;
  constexpr int LD = CHI + 1;
  constexpr int MS = LD * LD;
  constexpr int TEAMS = TEAM == 32 ? 4 : 1;
  constexpr bool FUSE = FD > 0 && CHI <= 8;       // register-fused product+bracket (host: chi <= 8 && D <= FD)
  constexpr bool WBR = FD > 0 && CHI >= 16;       // unfused GEMMs, matrix bracket (host: chi >= 16 && D <= FD)
  constexpr int FDM = FD > 0 ? FD : 4;            // channels handled by the fused / matrix-bracket stages
  constexpr int DMW = (FUSE || WBR) ? FDM : 0;    // channel-pair bracket matrices staged with the descriptors
  constexpr int FRT = CHI >= 16 ? 2 : 1;          // rows per fused item
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TQ_SMEM_POISON(smem_raw);
  const int team = threadIdx.x / TEAM;
  const int tid = threadIdx.x % TEAM;
  const int item = blockIdx.x * TEAMS + team;
  const int S = p.c.n_segments;
  if (item >= p.batch * S) return;
  const int b = item / S, g = item % S;
  TeamSmem<R> sm(smem_raw + (size_t)team * p.L.team_bytes, p.L);
  C* const WC = reinterpret_cast<C*>(smem_raw + (size_t)team * p.L.team_bytes + p.L.wc);
  const R* theta_b = reinterpret_cast<const R*>(p.theta) + (int64_t)b * p.theta_stride;
  const R* coef_b = p.coef ? reinterpret_cast<const R*>(p.coef) + (int64_t)b * p.coef_stride : nullptr;
  C* PIN = sm.ENV;   // P at the right cut (in) / left cut (out)
  C* N = sm.M;
  STAGE_BEGIN();

  const tq_segment seg = p.c.segs[g];
  C* env_g = reinterpret_cast<C*>(p.env) + (size_t)b * p.c.env_total + seg.env_base;
  const int4* blob = reinterpret_cast<const int4*>(p.c.blob);
  int4* const raw0 = reinterpret_cast<int4*>(smem_raw + (size_t)team * p.L.team_bytes + p.L.raw0);
  int4* const raw1 = reinterpret_cast<int4*>(smem_raw + (size_t)team * p.L.team_bytes + p.L.raw1);
  blob_prefetch(raw0, blob + p.c.blob_off[seg.site_begin + seg.site_count - 1], p.c.blob_max, tid, TEAM);
  if (tid == 0) {
    PIN[0] = cmk<C>(R(1), R(0));   // DONE channel = [[1]] at the right end
    const tq_site last = p.c.sites[seg.site_begin + seg.site_count - 1];
    if (p.store_env && last.env_in >= 0) env_g[last.env_in] = PIN[0];
  }
  // prologue: resolve the first site into descriptor buffer 0, then prefetch the second blob
  blob_wait();
  team_sync<TEAM>();
  {
    const tq_site s0 = *reinterpret_cast<const tq_site*>(raw0 + 1);
    sm.sel(0);
    stage_blob<R, TEAM, DMW>(raw0, s0, theta_b, coef_b, true, tid, sm.mres, sm.minfo, sm.mps, sm.ocode, sm.ogidx, sm.obase, sm.sedge, sm.sbuf, WC,
                             wct_row(p, seg.site_begin + seg.site_count - 1, 0));
    const int nx = raw0[0].y;
    team_sync<TEAM>();
    if (nx >= 0) blob_prefetch(raw0, blob + nx, p.c.blob_max, tid, TEAM);
  }
  int cur = 0;
  // CTA teams in energy mode: the folded core ping-pongs between A and A2, and the next site is
  // folded (and stored) by the half of the CTA the Hermitian P GEMM leaves idle
  C* Acur = sm.A;
  C* Anext = reinterpret_cast<C*>(smem_raw + (size_t)team * p.L.team_bytes + p.L.a2);
  bool folded = false;
  for (int q = seg.site_count - 1; q >= 0; --q, cur ^= 1) {
    team_sync<TEAM>();
    sm.sel(cur);
    const tq_site st = *reinterpret_cast<const tq_site*>(sm.sbuf + 1);
    const bool has_next = sm.sbuf[0].y >= 0;
    const int cl = st.chi_l, cr = st.chi_r;
    const int lcl = 31 - __clz(cl), lcr = 31 - __clz(cr);
    const int db = st.rl_db, da = st.rl_da;
    STAGE(0);
    if (!folded) {
      // per-pair column walks: the digit-tree fold (levels in the dead N/BR slots) was measured
      // slower at chi = 32 (11.7k vs 7.7k cycles per site: 20 team barriers over small levels)
      if constexpr (TEAM >= 128) fold_site2<R, LD, TEAM>(p.c, st, tid, sm.mres, sm.ocode, Acur, lcr);
      else if (__all_sync(0xffffffffu, column_real<R, TEAM>(st, tid, sm.mres, sm.minfo)))
        fold_site_real<R, LD, TEAM>(p.c, st, tid, sm.mres, sm.ocode, Acur, lcr);
      else fold_site<R, LD, TEAM>(p.c, st, tid, sm.mres, sm.ocode, Acur, nullptr, lcr);
      team_sync<TEAM>();
      if (p.store_env) {   // the left-to-right sweep reloads the folded core instead of refolding
        C* ag = env_g + st.a_off;
        const int np = cl * cr;
        for (int e = tid; e < 2 * np; e += TEAM) {
          const int sidx = e >= np, r = e - sidx * np;
          ag[e] = Acur[sidx * MS + (r >> lcr) * LD + (r & (cr - 1))];
        }
      }
    }
    STAGE(1);
    if constexpr (FUSE) {
      // fused: N[b][s] = A[s] P[b] kept in registers, brackets written directly
      product_bracket<R, LD, TEAM, FDM, FRT>(tid, true, db, da, cl, cr, lcl, lcr, Acur, PIN, WC, sm.BR);
      blob_wait();
      team_sync<TEAM>();
      STAGE(2);
    } else {
      // N[b][s] = A[s] * P[b]
      gemm_group<C, LD, TEAM, false, false, false, RE>(tid, db * 2, cl, cr, cr, 1,
            [&](int t, int) { return Acur + (t & 1) * MS; },
            [&](int t, int) { return PIN + (t >> 1) * MS; },
            [&](int t, int i0, int j, int rt, C a0, C a1, C a2, C a3) { store_rows<C, LD>(N + t * MS + i0 * LD + j, rt, a0, a1, a2, a3); });
      team_sync<TEAM>();
      STAGE(2);
      if constexpr (WBR) wbracket_stage<R, LD, TEAM, FDM, RE>(tid, db, da, N, WC, sm.BR, lcl, lcr);
      else bracket_stage<R, LD, TEAM>(tid, da, st.rl_edge_count, sm.sedge, true, N, sm.BR, lcl, lcr);
      blob_wait();
      team_sync<TEAM>();
      STAGE(3);
    }
    // CTA teams: the next site's descriptors are resolved by the half of the team the Hermitian
    // GEMM below leaves idle (rotated thread index), with no barrier in between (disjoint data).
    // With the A2 buffer (energy mode, descriptors staged without a team barrier) that half also
    // folds the next site and stores its core while the other half runs the GEMM.
    int nx2 = -1;
    const bool pre = TEAM >= 128 && p.L.rlpre && has_next && p.mode == 0 &&
                     (DMW == 0 || wct_row(p, seg.site_begin + q - 1, 0) != nullptr);
    const bool store = p.store_env && st.env_out >= 0;
    C* envo = env_g + (store ? st.env_out : 0);
    auto pa = [&](int t, int qq) { return sm.BR + (t * 2 + qq) * MS; };
    auto pb = [&](int, int qq) { return Acur + qq * MS; };
    auto ps = [&](int t, int i0, int j, int rt, C a0, C a1, C a2, C a3) {
      store_rows<C, LD>(PIN + t * MS + i0 * LD + j, rt, a0, a1, a2, a3);
      if (store) {
        C* h = envo + ((size_t)t << (2 * lcl)) + (i0 << lcl) + j;
        h[0] = a0; if (rt > 1) h[cl] = a1; if (rt > 2) { h[2 * cl] = a2; h[3 * cl] = a3; }
      }
    };
    if constexpr (TEAM >= 128) if (pre) {
      nx2 = raw0[0].y;
      if (tid >= TEAM / 2) {
        const int ut = tid - TEAM / 2;
        const tq_site sn = *reinterpret_cast<const tq_site*>(raw0 + 1);
        sm.sel(cur ^ 1);
        stage_blob<R, TEAM / 2, DMW>(raw0, sn, theta_b, coef_b, true, ut, sm.mres, sm.minfo, sm.mps, sm.ocode,
                                     sm.ogidx, sm.obase, sm.sedge, sm.sbuf, WC, wct_row(p, seg.site_begin + q - 1, 0));
        // is the column real?  each thread checks the factors it just resolved (ry and real
        // constants are real; rx / rz or a complex constant are not); the barrier ANDs them
        const bool real = upper_sync_and<TEAM / 2>(column_real<R, TEAM / 2>(sn, ut, sm.mres, sm.minfo));
        const int ncr = sn.chi_r, nlcr = 31 - __clz(ncr);
        if (real) fold_site4r<R, LD, TEAM / 2>(p.c, sn, ut, sm.mres, sm.ocode, Anext, nlcr);
        else fold_site4<R, LD, TEAM / 2>(p.c, sn, ut, sm.mres, sm.ocode, Anext, nlcr);
        if (p.store_env) {
          upper_sync<TEAM / 2>();
          C* ag = env_g + sn.a_off;
          const int np = sn.chi_l * ncr;
          for (int e = ut; e < 2 * np; e += TEAM / 2) {
            const int sidx = e >= np, r = e - sidx * np;
            ag[e] = Anext[sidx * MS + (r >> nlcr) * LD + (r & (ncr - 1))];
          }
        }
      } else {
        gemm_group<C, LD, TEAM / 2, false, true, true, RE>(tid, da, cl, cl, cr, 2, pa, pb, ps);
      }
      team_sync<TEAM>();
      STAGE(4);
      if (nx2 >= 0) blob_prefetch(raw0, blob + nx2, p.c.blob_max, tid, TEAM);
      C* t = Acur; Acur = Anext; Anext = t;
      folded = true;
      continue;
    }
    folded = false;
    if (TEAM >= 128 && has_next) {
      const tq_site sn = *reinterpret_cast<const tq_site*>(raw0 + 1);
      nx2 = raw0[0].y;
      sm.sel(cur ^ 1);
      stage_blob<R, TEAM, DMW>(raw0, sn, theta_b, coef_b, true, (tid + TEAM / 2) % TEAM, sm.mres, sm.minfo, sm.mps,
                               sm.ocode, sm.ogidx, sm.obase, sm.sedge, sm.sbuf, WC, wct_row(p, seg.site_begin + q - 1, 0));
    }
    // P'[a] = sum_s' BR[a][s'] AH[s']  -> PIN slots (P[b] is dead) + HBM
    {
      // the environments of the energy / gradient MPO are Hermitian (real coefficients): half the work
      if (CHI >= 16 && p.mode == 0) gemm_group<C, LD, TEAM, false, true, true, RE>(tid, da, cl, cl, cr, 2, pa, pb, ps);
      else gemm_group<C, LD, TEAM, false, true, false, RE>(tid, da, cl, cl, cr, 2, pa, pb, ps);
    }
    STAGE(5);
    // warp teams: resolve the next site's descriptors after the GEMM (independent work)
    if (TEAM < 128 && has_next) {
      const tq_site sn = *reinterpret_cast<const tq_site*>(raw0 + 1);
      nx2 = raw0[0].y;
      sm.sel(cur ^ 1);
      stage_blob<R, TEAM, DMW>(raw0, sn, theta_b, coef_b, true, tid, sm.mres, sm.minfo, sm.mps, sm.ocode, sm.ogidx, sm.obase, sm.sedge, sm.sbuf, WC,
                               wct_row(p, seg.site_begin + q - 1, 0));
    }
    team_sync<TEAM>();
    STAGE(4);
    if (nx2 >= 0) blob_prefetch(raw0, blob + nx2, p.c.blob_max, tid, TEAM);
  }
  if (tid == 0) reinterpret_cast<C*>(p.epart)[(size_t)b * S + g] = PIN[0];
  STAGE_END(0);
}

// ------------------------------------------------------------------ left-to-right sweep
// MODE 0: gradient (G + column adjoint); MODE 1: per-term values.  Separate instantiations
// keep each kernel's code small enough for the instruction cache.
template <typename R, int CHI, int TEAM, int MODE, int FD, bool RE = false>
__global__ void __launch_bounds__(TEAM == 32 ? 128 : TEAM, TEAM == 32 ? (sizeof(R) == 4 ? TQ_LR_MINB : 4) : 1)
lr_sweep(Params p) {
  using C = typename CT<R>::T;
  constexpr int LD = CHI + 1;
  constexpr int MS = LD * LD;
  constexpr int TEAMS = TEAM == 32 ? 4 : 1;
  constexpr int MAXSAVE = 48;
  constexpr bool FUSE = FD > 0 && CHI <= 8;       // register-fused product+bracket (host: chi <= 8 && D <= FD)
  constexpr bool WBR = FD > 0 && CHI >= 16;       // unfused GEMMs, matrix bracket (host: chi >= 16 && D <= FD)
  constexpr int FDM = FD > 0 ? FD : 4;            // channels handled by the fused / matrix-bracket stages
  constexpr int DMW = (FUSE || WBR) ? FDM : 0;    // channel-pair bracket matrices staged with the descriptors
  constexpr int FRT = CHI >= 16 ? 2 : 1;          // rows per fused item
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TQ_SMEM_POISON(smem_raw);
  const int team = threadIdx.x / TEAM;
  const int tid = threadIdx.x % TEAM;
  const int item = blockIdx.x * TEAMS + team;
  const int S = p.c.n_segments;
  if (item >= p.batch * S) return;
  const int b = item / S, g = item % S;
  TeamSmem<R> sm(smem_raw + (size_t)team * p.L.team_bytes, p.L);
  C* const WC = reinterpret_cast<C*>(smem_raw + (size_t)team * p.L.team_bytes + p.L.wc);
  const R* theta_b = reinterpret_cast<const R*>(p.theta) + (int64_t)b * p.theta_stride;
  const R* coef_b = p.coef ? reinterpret_cast<const R*>(p.coef) + (int64_t)b * p.coef_stride : nullptr;
  C* LAM = sm.ENV;
  C* M = sm.M;
  C* G = sm.M;  // gradient cores alias the M slots (dead after the bracket stage)
  C* PIN = sm.PIN;
  STAGE_BEGIN();

  const tq_segment seg = p.c.segs[g];
  C* env_g_w = reinterpret_cast<C*>(p.env) + (size_t)b * p.c.env_total + seg.env_base;
  const C* env_g = env_g_w;
  if (tid == 0) LAM[0] = cmk<C>(R(1), R(0));
  const int4* blob = reinterpret_cast<const int4*>(p.c.blob);
  int4* const raw0 = reinterpret_cast<int4*>(smem_raw + (size_t)team * p.L.team_bytes + p.L.raw0);
  int4* const raw1 = reinterpret_cast<int4*>(smem_raw + (size_t)team * p.L.team_bytes + p.L.raw1);
  // direct path: folded cores ping-pong between A / A2 and P lives dense in PIN; both are
  // cp.async-prefetched one stage ahead (A(q+1) during site q's Lambda GEMM, P(q+1) after
  // site q's G), so the sweep never waits on HBM/L2 at a site boundary.
  const bool pf = MODE == 0 && FUSE && p.L.direct;
  // chi >= 16 gradient sweep: the same one-stage-ahead prefetch in the padded layout.  Group order
  // per site: A(q+1) at the site's start, then blob(q+2) and P(q+1) at its end, so "all but the
  // newest group" at a site's start is A(q) + its blob, and P(q) is waited only before the G GEMM.
  const bool pf2 = MODE == 0 && !FUSE && CHI >= 16 && p.L.lrpf;
  C* const abuf1 = reinterpret_cast<C*>(smem_raw + (size_t)team * p.L.team_bytes + p.L.a2);
  blob_prefetch(raw0, blob + p.c.blob_off[seg.site_begin], p.c.blob_max, tid, TEAM);
  blob_wait();
  team_sync<TEAM>();
  {
    const tq_site s0 = *reinterpret_cast<const tq_site*>(raw0 + 1);
    sm.sel(0);
    stage_blob<R, TEAM, DMW>(raw0, s0, theta_b, coef_b, false, tid, sm.mres, sm.minfo, sm.mps, sm.ocode, sm.ogidx, sm.obase, sm.sedge, sm.sbuf, WC,
                             wct_row(p, seg.site_begin, 1));
    const int nx = raw0[0].z;
    team_sync<TEAM>();
    if (pf) {
      async_core<C, LD, TEAM>(sm.A, env_g + s0.a_off, s0.chi_l, s0.chi_r, 31 - __clz(s0.chi_r), tid);
      async_commit();
    }
    if (pf2) {
      async_core<C, LD, TEAM>(sm.A, env_g + s0.a_off, s0.chi_l, s0.chi_r, 31 - __clz(s0.chi_r), tid);
      async_commit();
    }
    if (nx >= 0) blob_prefetch(raw0, blob + nx, p.c.blob_max, tid, TEAM, !pf);
    if (pf) {
      async_dense<C, TEAM>(PIN, env_g + s0.env_in, s0.rl_db * s0.chi_r * s0.chi_r, tid);
      async_commit();
    }
    if (pf2) {
      async_env<C, LD, TEAM>(PIN, env_g + s0.env_in, s0.rl_db, s0.chi_r, 31 - __clz(s0.chi_r), tid);
      async_commit();
    }
  }
  int cur = 0;
  for (int q = 0; q < seg.site_count; ++q, cur ^= 1) {
    team_sync<TEAM>();
    sm.sel(cur);
    const tq_site st = *reinterpret_cast<const tq_site*>(sm.sbuf + 1);
    const bool has_next = sm.sbuf[0].z >= 0;
    const int cl = st.chi_l, cr = st.chi_r;
    const int lcl = 31 - __clz(cl), lcr = 31 - __clz(cr);
    const int da = st.lr_da, db = st.lr_db;
    const int npin = MODE == 0 ? st.rl_db : 1;
    R th_pre = R(0);      // next site's first angle, requested ahead of the Lambda GEMM
    bool wct_as = false;  // next site's bracket-matrix row already on its way (cp.async)
    C* const Acur = ((pf || pf2) && (q & 1)) ? abuf1 : sm.A;
    if (pf || pf2) {
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");   // A(q) landed (P(q) may still be in flight)
    } else {
      // stored right environments at cut k+1 -> PIN (dense cr x cr in HBM), folded core -> A
      const C* src = env_g + st.env_in;
      const int lper = 2 * lcr;
      for (int e = tid; e < (npin << lper); e += TEAM) {
        const int ch = e >> lper, r = e & ((1 << lper) - 1);
        PIN[ch * MS + (r >> lcr) * LD + (r & (cr - 1))] = src[e];
      }
      const C* ag = env_g + st.a_off;
      const int np = cl * cr;
      for (int e = tid; e < 2 * np; e += TEAM) {
        const int sidx = e >= np, r = e - sidx * np;
        sm.A[sidx * MS + (r >> lcr) * LD + (r & (cr - 1))] = ag[e];
      }
    }
    team_sync<TEAM>();
    if (pf2 && has_next) {   // A(q+1) into the other buffer; lands during this site's GEMMs
      const tq_site sn = *reinterpret_cast<const tq_site*>(raw0 + 1);
      async_core<C, LD, TEAM>((q & 1) ? sm.A : abuf1, env_g + sn.a_off, sn.chi_l, sn.chi_r, 31 - __clz(sn.chi_r), tid);
      async_commit();
    }
    STAGE(0);
    STAGE(1);
    if constexpr (FUSE && MODE == 0) {
      // fused: M[a][s] = Lam[a] A[s] kept in registers, brackets written directly
      product_bracket<R, LD, TEAM, FDM, FRT>(tid, false, da, db, cl, cr, lcl, lcr, Acur, LAM, WC, sm.BR);
      blob_wait();
      team_sync<TEAM>();
      if (pf && has_next) {   // A(q+1) into the other buffer (A(q) stays live for the Lambda GEMM)
        const tq_site sn = *reinterpret_cast<const tq_site*>(raw0 + 1);
        async_core<C, LD, TEAM>((q & 1) ? sm.A : abuf1, env_g + sn.a_off, sn.chi_l, sn.chi_r,
                                31 - __clz(sn.chi_r), tid);
        if constexpr (DMW > 0) {   // and its bracket-matrix row (WC is dead after this site's bracket)
          const C* wr = wct_row(p, seg.site_begin + q + 1, 1);
          if (wr) {
            for (int e = tid; e < 4 * DMW * DMW + 1; e += TEAM) async_elem(WC + e, wr + e);
            wct_as = true;
          }
        }
        async_commit();
      }
      if (has_next) th_pre = blob_theta<R>(raw0, *reinterpret_cast<const tq_site*>(raw0 + 1), theta_b, tid);
      STAGE(2);
    } else {
      // M[a][s] = Lam[a] * A[s]
      gemm_group<C, LD, TEAM, false, false, false, RE>(tid, da * 2, cl, cr, cl, 1,
          [&](int t, int) { return LAM + (t >> 1) * MS; },
          [&](int t, int) { return Acur + (t & 1) * MS; },
          [&](int t, int i0, int j, int rt, C a0, C a1, C a2, C a3) { store_rows<C, LD>(M + t * MS + i0 * LD + j, rt, a0, a1, a2, a3); });
      team_sync<TEAM>();
      STAGE(2);
      if constexpr (WBR) wbracket_stage<R, LD, TEAM, FDM, RE>(tid, da, db, M, WC, sm.BR, lcl, lcr);
      else bracket_stage<R, LD, TEAM>(tid, db, st.lr_edge_count, sm.sedge, false, M, sm.BR, lcl, lcr);
      if (!pf2) blob_wait();   // pf2: the blob landed with A(q) at the site's start
      team_sync<TEAM>();
      STAGE(3);
    }
    int nx2 = -1;
    // CTA teams, gradient mode: the Lambda GEMM (Hermitian, half the tiles) and the core-cotangent
    // GEMM G are independent (LAM vs the dead M slots), so they run side by side on the two halves
    // of the team, and the next site's descriptors are resolved by the Lambda half's last warp
    constexpr bool SPLIT = CHI >= 16 && MODE == 0 && TEAM >= 128 && !FUSE;
    if (pf2 && SPLIT) {   // G reads P(q): landed (with A(q+1))
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      team_sync<TEAM>();
    }
    if (TEAM >= 128 && has_next) {
      const tq_site sn = *reinterpret_cast<const tq_site*>(raw0 + 1);
      nx2 = raw0[0].z;
      sm.sel(cur ^ 1);
      const int rtid = SPLIT ? (tid + TEAM / 2 + 32) % TEAM : (tid + TEAM / 2) % TEAM;
      stage_blob<R, TEAM, DMW>(raw0, sn, theta_b, coef_b, false, rtid, sm.mres, sm.minfo, sm.mps,
                               sm.ocode, sm.ogidx, sm.obase, sm.sedge, sm.sbuf, WC, wct_row(p, seg.site_begin + q + 1, 1),
                               wct_as, false, th_pre);
      sm.sel(cur);
    }
    // Lam'[bb] = sum_s' AH[s'] BR[bb][s']
    {
      auto la = [&](int, int qq) { return Acur + qq * MS; };
      auto lb = [&](int t, int qq) { return sm.BR + (t * 2 + qq) * MS; };
      auto ls = [&](int t, int i0, int j, int rt, C a0, C a1, C a2, C a3) { store_rows<C, LD>(LAM + t * MS + i0 * LD + j, rt, a0, a1, a2, a3); };
      if constexpr (SPLIT) {
        if (tid < TEAM / 2) {
          gemm_group<C, LD, TEAM / 2, true, false, true, RE>(tid, db, cr, cr, cl, 2, la, lb, ls);
        } else {   // G[s'] = sum_bb BR[bb][s'] PIN[bb], straight from the epilogue to HBM (dense [2][cl][cr])
          C* const gg = env_g_w + st.g_off;
          const int np = cl * cr;
          gemm_group<C, LD, TEAM / 2, false, false, false, RE>(tid - TEAM / 2, 2, cl, cr, cr, db,
              [&](int t, int qq) { return sm.BR + (qq * 2 + t) * MS; },
              [&](int, int qq) { return PIN + qq * MS; },
              [&](int t, int i0, int j, int rt, C a0, C a1, C a2, C a3) {
                C* h = gg + (size_t)t * np + i0 * cr + j;
                h[0] = a0; if (rt > 1) h[cr] = a1; if (rt > 2) { h[2 * cr] = a2; h[3 * cr] = a3; }
              });
        }
      } else if (CHI >= 16 && MODE == 0) {
        gemm_group<C, LD, TEAM, true, false, true, RE>(tid, db, cr, cr, cl, 2, la, lb, ls);
      } else {
        gemm_group<C, LD, TEAM, true, false, false, RE>(tid, db, cr, cr, cl, 2, la, lb, ls);
      }
    }
    if (TEAM < 128 && has_next) {   // warp teams: next site's descriptors, overlapped with this site's GEMMs
      const tq_site sn = *reinterpret_cast<const tq_site*>(raw0 + 1);
      nx2 = raw0[0].z;
      sm.sel(cur ^ 1);
      stage_blob<R, TEAM, DMW>(raw0, sn, theta_b, coef_b, false, tid, sm.mres, sm.minfo, sm.mps, sm.ocode, sm.ogidx, sm.obase, sm.sedge, sm.sbuf, WC,
                               wct_row(p, seg.site_begin + q + 1, 1), wct_as, has_next && FUSE && MODE == 0, th_pre);
      sm.sel(cur);
    }
    if constexpr (MODE == 0) {
      if (pf2 && !SPLIT) {   // P(q) (and A(q+1)) landed
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        team_sync<TEAM>();
      }
      // G[s'] = sum_bb BR[bb][s'] PIN[bb]   (writes over M, read only by the bracket stage)
      if (!SPLIT && !(FUSE && p.L.direct)) gemm_group<C, LD, TEAM, false, false, false, RE>(tid, 2, cl, cr, cr, db,
          [&](int t, int qq) { return sm.BR + (qq * 2 + t) * MS; },
          [&](int, int qq) { return PIN + qq * MS; },
          [&](int t, int i0, int j, int rt, C a0, C a1, C a2, C a3) { store_rows<C, LD>(G + t * MS + i0 * LD + j, rt, a0, a1, a2, a3); });
      team_sync<TEAM>();
      STAGE(4);
      // ---- core cotangent G_k -> HBM; the column adjoint runs in adj_sweep (off the critical path)
      C* gg = env_g_w + st.g_off;
      const int np = cl * cr;
      if (FUSE && p.L.direct) {
        // G[s'][al][be] = sum_b sum_k BR[b][s'][al][k] P[b][k][be], one pair per lane, P through L1
        if (tid < np) {
          const int al = tid >> lcr, be = tid & (cr - 1);
          C g0 = cmk<C>(R(0), R(0)), g1 = g0;
          const C* pg = PIN;   // dense [bb][k][be], prefetched
          for (int bb = 0; bb < db; ++bb) {
            const C* br0 = sm.BR + (bb * 2) * MS + al * LD;
            const C* br1 = br0 + MS;
            const C* pb = pg + (size_t)bb * cr * cr + be;
            for (int k = 0; k < cr; ++k) {
              const C pv = pb[k * cr];
              cfma(g0, br0[k], pv);
              cfma(g1, br1[k], pv);
            }
          }
          gg[tid] = g0; gg[np + tid] = g1;
        }
      } else if (!SPLIT) {
        for (int e = tid; e < 2 * np; e += TEAM) {
          const int sidx = e >= np, r = e - sidx * np;
          gg[e] = G[sidx * MS + (r >> lcr) * LD + (r & (cr - 1))];
        }
      }
      STAGE(5);
    } else {
      // ---- values: rho_a[s'][s] = <A[s'], M[a][s] R> for every source channel a
      gemm_group<C, LD, TEAM, false, false, false, RE>(tid, da * 2, cl, cr, cr, 1,
          [&](int t, int) { return M + t * MS; },
          [&](int, int) { return PIN; },
          [&](int t, int i0, int j, int rt, C a0, C a1, C a2, C a3) { store_rows<C, LD>(sm.MR + t * MS + i0 * LD + j, rt, a0, a1, a2, a3); });
      team_sync<TEAM>();
      STAGE(7);
      if (st.fin_count > 0) {
        const int ncombo = da * 4;  // (a, s', s)
        R* part = sm.contrib;       // [2 * ncombo][TEAM] partial sums (re, im)
        for (int cmb = 0; cmb < ncombo; ++cmb) {
          const int a = cmb >> 2, sp = (cmb >> 1) & 1, s = cmb & 1;
          C acc = cmk<C>(R(0), R(0));
          for (int e = tid; e < cl * cr; e += TEAM) {
            const int off = (e >> lcr) * LD + (e & (cr - 1));
            cfmac(acc, sm.A[sp * MS + off], sm.MR[(a * 2 + s) * MS + off]);
          }
          part[(2 * cmb) * TEAM + tid] = acc.x;
          part[(2 * cmb + 1) * TEAM + tid] = acc.y;
        }
        team_sync<TEAM>();
        STAGE(8);
        if (tid < 32) {  // reduce and finalise (one warp, fixed order)
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
      STAGE(9);
    }
    if (pf && has_next) team_sync<TEAM>();   // every lane is done reading P(q)
    if (nx2 >= 0) blob_prefetch(raw0, blob + nx2, p.c.blob_max, tid, TEAM, !pf);
    if (pf && has_next) {
      const tq_site sn = *reinterpret_cast<const tq_site*>(sm.sel_sbuf(cur ^ 1) + 1);
      async_dense<C, TEAM>(PIN, env_g + sn.env_in, sn.rl_db * sn.chi_r * sn.chi_r, tid);
      async_commit();
    }
    if (pf2 && has_next) {   // P(q+1): PIN is no longer read (the barrier after the G GEMM)
      const tq_site sn = *reinterpret_cast<const tq_site*>(sm.sel_sbuf(cur ^ 1) + 1);
      async_env<C, LD, TEAM>(PIN, env_g + sn.env_in, sn.rl_db, sn.chi_r, 31 - __clz(sn.chi_r), tid);
      async_commit();
    }
  }
  STAGE_END(1);
}



// ------------------------------------------------------------------ column adjoint kernel
// One team per (theta-set, site): resolves the site's descriptors, reads the core cotangent
// G_k written by lr_sweep and pushes it through the column to the site's trainable angles.
// Every (theta-set, site) is independent, so this runs at full occupancy instead of on
// the left-to-right sweep's sequential critical path.
struct AdjLayout {
  int32_t g, mres, minfo, mps, ocode, ogidx, obase, sbuf, raw, lev, ubuf, contrib, team_bytes, tree;
  int32_t ubuf_vec;   // 2-vectors in the compact digit tree's scratch / U buffer
  int32_t utab;       // the leaf-index tables (alpha and beta sides) of the adjoint's gather
};

// Min resident 128-thread adjoint CTAs per SM (team-of-32 path).  6 measured best
// on cfg2 (adj 0.0830 -> 0.0787 ms vs 4; 8 gives 0.0814), tools/exp_variant.sh.
// fp32 only: at 6 the fp64 CHI=8 instance spills ~500 B, so fp64 keeps 4.
#ifndef TQ_ADJ_MINB
#define TQ_ADJ_MINB 6
#endif
#ifndef TQ_ADJ128_MINB
#define TQ_ADJ128_MINB 4
#endif
template <typename R, int CHI, int TEAM, bool RE = false>
__global__ void __launch_bounds__(TEAM == 32 ? 128 : TEAM, TEAM == 32 ? (sizeof(R) == 4 ? TQ_ADJ_MINB : 4) : (TEAM == 128 ? (sizeof(R) == 4 ? TQ_ADJ128_MINB : 4) : 1))
adj_sweep(Params p, AdjLayout A) {
  using C = typename CT<R>::T;
  constexpr int LD = CHI + 1;
  constexpr int MS = LD * LD;
  constexpr int TEAMS = TEAM == 32 ? 4 : 1;
  constexpr int MAXSAVE = 48;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TQ_SMEM_POISON(smem_raw);
  const int team = threadIdx.x / TEAM;
  const int tid = threadIdx.x % TEAM;
  const int nsites = p.c.n_sites;
  const int unit = blockIdx.x * TEAMS + team;
  if (unit >= p.batch * nsites) return;
  const int b = unit / nsites, si = unit % nsites;
  unsigned char* base = smem_raw + (size_t)team * A.team_bytes;
  C* Gs = reinterpret_cast<C*>(base + A.g);
  C* mres = reinterpret_cast<C*>(base + A.mres);
  int* minfo = reinterpret_cast<int*>(base + A.minfo);
  R* mps = reinterpret_cast<R*>(base + A.mps);
  int* ocode = reinterpret_cast<int*>(base + A.ocode);
  int* ogidx = reinterpret_cast<int*>(base + A.ogidx);
  int* obase = reinterpret_cast<int*>(base + A.obase);
  int4* sbuf = reinterpret_cast<int4*>(base + A.sbuf);
  int4* raw = reinterpret_cast<int4*>(base + A.raw);
  const int4* blob = reinterpret_cast<const int4*>(p.c.blob) + p.c.blob_off[si];
  blob_prefetch(raw, blob, p.c.blob_max, tid, TEAM);   // every 16-byte unit in flight at once
  if (CHI >= 16 && A.tree) {
    // the core cotangent (written by lr_sweep, long evicted from L2) is read after the forward
    // tree: pull its lines into L2 now so that read costs an L2 hit, not an HBM round trip
    const tq_site* sg = p.c.sites + si;
    const int64_t goff = sg->g_off;
    const tq_segment* sgs = p.c.segs + reinterpret_cast<const int*>(blob)[3];
    const char* gl = reinterpret_cast<const char*>(reinterpret_cast<const C*>(p.env) + (size_t)b * p.c.env_total +
                                                    sgs->env_base + goff);
    const int nbytes = 2 * sg->chi_l * sg->chi_r * (int)sizeof(C);
    for (int o = tid * 128; o < nbytes; o += TEAM * 128) asm volatile("prefetch.global.L2 [%0];" :: "l"(gl + o));
  }
  blob_wait();
  team_sync<TEAM>();
  const tq_site st = *reinterpret_cast<const tq_site*>(raw + 1);
  if (st.n_train == 0) return;   // uniform across the team
  const int g = raw[0].w;
  const tq_segment seg = p.c.segs[g];
  const R* theta_b = reinterpret_cast<const R*>(p.theta) + (int64_t)b * p.theta_stride;
  const C* gg = reinterpret_cast<const C*>(p.env) + (size_t)b * p.c.env_total + seg.env_base + st.g_off;
  R* gpart = reinterpret_cast<R*>(p.gpart) + (size_t)b * p.c.n_gslots + seg.gslot_begin;
  const int cl = st.chi_l, cr = st.chi_r;
  const int lcr = 31 - __clz(cr);
  const int np = cl * cr;
  const int nops = st.op_count;
  if (TEAM == 32 && CHI <= 8 && np <= 32 && nops <= 12) {
    // the core cotangent is loaded into registers before the descriptors are resolved, so
    // its HBM/L2 latency overlaps the resolve
    const int al = tid >> lcr, be = tid & (cr - 1);
    const bool have = tid < np && !(st.pass_count && !pass_ok(p.c, st, al, be));
    const C z = cmk<C>(R(0), R(0));
    const C g0 = have ? gg[tid] : z, g1 = have ? gg[np + tid] : z;
    stage_blob<R, TEAM>(raw, st, theta_b, nullptr, true, tid, mres, minfo, mps, ocode, ogidx, obase, nullptr, sbuf);
    team_sync<TEAM>();
    pair_adjoint_warp<R, 12>(nops, have ? al : 0, have ? be : 0, ocode, ogidx, mres, minfo,
                             cmk<C>(R(st.init[0]), R(st.init[1])), cmk<C>(R(st.init[2]), R(st.init[3])),
                             g0, g1, gpart, tid);
    return;
  }
  stage_blob<R, TEAM>(raw, st, theta_b, nullptr, true, tid, mres, minfo, mps, ocode, ogidx, obase, nullptr, sbuf);
  if (!A.tree)   // per-pair walks read G from shared memory; the digit tree reads it from HBM once
    for (int e = tid; e < 2 * np; e += TEAM) {
      const int sidx = e >= np, r = e - sidx * np;
      Gs[sidx * MS + (r >> lcr) * LD + (r & (cr - 1))] = gg[e];
    }
  const int ntr = st.n_train;
  R* contrib = reinterpret_cast<R*>(base + A.contrib);
  const int cw = A.tree ? TEAM / 32 : TEAM;
  if (tid < cw) for (int t = 0; t < ntr; ++t) contrib[t * cw + tid] = R(0);
  team_sync<TEAM>();
  if constexpr (CHI >= 16) {
    if (A.tree) {
      C* lev = reinterpret_cast<C*>(base + A.lev);
      C* u0 = reinterpret_cast<C*>(base + A.ubuf);       // forward scratch, then U (in place)
      int* tal = reinterpret_cast<int*>(base + A.utab);
      int* tbase = obase;   // host tbase offsets are for the full tree; the compact ones go here
      ctree_forward<R, TEAM, RE>(st, tid, mres, ocode, lev, u0, tbase);
      ctree_adjoint<R, TEAM, RE>(p.c, st, tid, mres, minfo, ocode, lev, tbase, u0, tal, gg, lcr, contrib);
    }
  }
  const bool one_pair = np <= TEAM;
  for (int pi = tid; !A.tree && pi < np; pi += TEAM) {
    const int al = pi >> lcr, be = pi & (cr - 1);
    if (st.pass_count && !pass_ok(p.c, st, al, be)) continue;
    C sv[MAXSAVE];
    int ns = 0;
    C v0 = cmk<C>(R(st.init[0]), R(st.init[1]));
    C v1 = cmk<C>(R(st.init[2]), R(st.init[3]));
    for (int oi = 0; oi < nops; ++oi) {
      const int c = ocode[oi];
      const int e = oc_lmat(c) + oc_digit(c, al, be);
      const int cls = (minfo[e] >> 8) & 0xff;
      if (cls == 1) sv[ns++] = v1;
      else if (cls == 2) sv[ns++] = v0;
      else if (cls == 3) { sv[ns++] = v0; sv[ns++] = v1; }
      const C* Mm = mres + 4 * e;
      C n0 = cmul(Mm[0], v0); cfma(n0, Mm[1], v1);
      C n1 = cmul(Mm[2], v0); cfma(n1, Mm[3], v1);
      v0 = n0; v1 = n1;
    }
    C u0 = Gs[al * LD + be], u1 = Gs[MS + al * LD + be];
    for (int oi = nops - 1; oi >= 0; --oi) {
      const int c = ocode[oi];
      const int e = oc_lmat(c) + oc_digit(c, al, be);
      const int info = minfo[e];
      const int kind = info & 0xff, cls = (info >> 8) & 0xff;
      const int tix = oc_tidx(c);
      if (tix >= 0 && kind != 0) {
        C s0, s1;
        if (kind == 1) { s0 = v1; s1 = v0; }
        else if (kind == 2) { s0 = cmk<C>(v1.y, -v1.x); s1 = cmk<C>(-v0.y, v0.x); }
        else { s0 = v0; s1 = cmk<C>(-v1.x, -v1.y); }
        C d = cmk<C>(R(0), R(0));
        cfmac(d, u0, s0); cfmac(d, u1, s1);
        if (one_pair) contrib[tix * TEAM + tid] = d.y;
        else contrib[tix * TEAM + tid] += d.y;
      }
      const C* Mm = mres + 4 * e;
      C w0 = cmk<C>(R(0), R(0)), w1 = w0;
      cfmac(w0, Mm[0], u0); cfmac(w0, Mm[2], u1);
      cfmac(w1, Mm[1], u0); cfmac(w1, Mm[3], u1);
      u0 = w0; u1 = w1;
      if (cls == 0) {
        C x0 = cmk<C>(R(0), R(0)), x1 = x0;
        cfmac(x0, Mm[0], v0); cfmac(x0, Mm[2], v1);
        cfmac(x1, Mm[1], v0); cfmac(x1, Mm[3], v1);
        v0 = x0; v1 = x1;
      } else if (cls == 1) {
        const R sc = mps[e];
        v0 = cmk<C>(v0.x * sc, v0.y * sc); v1 = sv[--ns];
      } else if (cls == 2) {
        const R sc = mps[e];
        v1 = cmk<C>(v1.x * sc, v1.y * sc); v0 = sv[--ns];
      } else {
        v1 = sv[--ns]; v0 = sv[--ns];
      }
    }
  }
  team_sync<TEAM>();
  {
    const int warp = tid >> 5, lane = tid & 31;
    constexpr int NW = TEAM / 32;
    for (int t0 = warp * 4; t0 < ntr; t0 += NW * 4) {
      R sacc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        sacc[u] = R(0);
        if (t0 + u < ntr)
          for (int k = lane; k < cw; k += 32) sacc[u] += contrib[(t0 + u) * cw + k];
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int u = 0; u < 4; ++u) sacc[u] += __shfl_xor_sync(0xffffffffu, sacc[u], off);
      if (lane == 0)
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (t0 + u < ntr) gpart[ogidx[t0 + u]] = sacc[u];
    }
  }
}

// ------------------------------------------------------------------ inner product sweep
// out[b] = <bra(theta_bra_b) | ket(theta_ket_b)>: one left-to-right transfer with distinct
// bra and ket columns, env L (chi_bra x chi_ket):  L' = sum_s Ab[s]^H (L Ak[s])  (tt_inner, tt.py:247-255).
struct InnerParams {
  tq_chain ket, bra;
  int32_t batch;
  const void* theta_ket; int64_t ket_stride;
  const void* theta_bra; int64_t bra_stride;
  double* out;
  int32_t team_bytes;
  int32_t off_ak, off_ahk, off_ab, off_ahb, off_t, off_l, off_mk, off_ik, off_pk, off_ok, off_gk, off_qk, off_mb, off_ib, off_pb, off_ob, off_gb, off_qb;
};

template <typename R, int CHI, int TEAM>
__global__ void __launch_bounds__(TEAM == 32 ? 128 : TEAM, TEAM == 32 ? 4 : 1)
inner_sweep(InnerParams p) {
  using C = typename CT<R>::T;
  constexpr int LD = CHI + 1;
  constexpr int MS = LD * LD;
  constexpr int TEAMS = TEAM == 32 ? 4 : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TQ_SMEM_POISON(smem_raw);
  const int team = threadIdx.x / TEAM;
  const int tid = threadIdx.x % TEAM;
  const int b = blockIdx.x * TEAMS + team;
  if (b >= p.batch) return;
  unsigned char* base = smem_raw + (size_t)team * p.team_bytes;
  C* Ak = reinterpret_cast<C*>(base + p.off_ak); C* AHk = reinterpret_cast<C*>(base + p.off_ahk);
  C* Ab = reinterpret_cast<C*>(base + p.off_ab); C* AHb = reinterpret_cast<C*>(base + p.off_ahb);
  C* T = reinterpret_cast<C*>(base + p.off_t); C* L = reinterpret_cast<C*>(base + p.off_l);
  const R* thk = reinterpret_cast<const R*>(p.theta_ket) + (int64_t)b * p.ket_stride;
  const R* thb = reinterpret_cast<const R*>(p.theta_bra) + (int64_t)b * p.bra_stride;
  if (tid == 0) L[0] = cmk<C>(R(1), R(0));
  const int n = p.ket.segs[0].site_count;
  for (int q = 0; q < n; ++q) {
    const tq_site sk = p.ket.sites[p.ket.segs[0].site_begin + q];
    const tq_site sb = p.bra.sites[p.bra.segs[0].site_begin + q];
    stage_site<R, TEAM>(p.ket, thk, nullptr, sk, tid, true, reinterpret_cast<C*>(base + p.off_mk),
                        reinterpret_cast<int*>(base + p.off_ik), reinterpret_cast<R*>(base + p.off_pk),
                        reinterpret_cast<int*>(base + p.off_ok), reinterpret_cast<int*>(base + p.off_gk),
                        reinterpret_cast<int*>(base + p.off_qk), nullptr);
    stage_site<R, TEAM>(p.bra, thb, nullptr, sb, tid, true, reinterpret_cast<C*>(base + p.off_mb),
                        reinterpret_cast<int*>(base + p.off_ib), reinterpret_cast<R*>(base + p.off_pb),
                        reinterpret_cast<int*>(base + p.off_ob), reinterpret_cast<int*>(base + p.off_gb),
                        reinterpret_cast<int*>(base + p.off_qb), nullptr);
    team_sync<TEAM>();
    fold_site<R, LD, TEAM>(p.ket, sk, tid, reinterpret_cast<C*>(base + p.off_mk), reinterpret_cast<int*>(base + p.off_ok),
                           Ak, nullptr, 31 - __clz(sk.chi_r));
    fold_site<R, LD, TEAM>(p.bra, sb, tid, reinterpret_cast<C*>(base + p.off_mb), reinterpret_cast<int*>(base + p.off_ob),
                           Ab, nullptr, 31 - __clz(sb.chi_r));
    team_sync<TEAM>();
    // T[s] = L * Ak[s]
    gemm_group<C, LD, TEAM>(tid, 2, sb.chi_l, sk.chi_r, sk.chi_l, 1,
        [&](int, int) { return L; },
        [&](int t, int) { return Ak + t * MS; },
        [&](int t, int i0, int j, int rt, C a0, C a1, C a2, C a3) { store_rows<C, LD>(T + t * MS + i0 * LD + j, rt, a0, a1, a2, a3); });
    team_sync<TEAM>();
    // L' = sum_s AHb[s] T[s]
    gemm_group<C, LD, TEAM, true, false>(tid, 1, sb.chi_r, sk.chi_r, sb.chi_l, 2,
        [&](int, int qq) { return Ab + qq * MS; },
        [&](int, int qq) { return T + qq * MS; },
        [&](int, int i0, int j, int rt, C a0, C a1, C a2, C a3) { store_rows<C, LD>(L + i0 * LD + j, rt, a0, a1, a2, a3); });
    team_sync<TEAM>();
  }
  if (tid == 0) { p.out[2 * b] = double(L[0].x); p.out[2 * b + 1] = double(L[0].y); }
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
thread_local char g_err[512];   // shared with tq_trunc.cu

static tq_status fail(tq_status s, const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return s;
}

// cudaFuncSetAttribute only when a launch needs more dynamic shared memory than the kernel
// was last opened to on this device.  The eager entry points run in loops, and re-setting the
// attribute on every launch dominated their host cost.  The limit only ever grows (process-wide,
// under a mutex), so concurrent callers with different plans never shrink each other's.
static void set_smem_attr(const void* fn, size_t smem) {
  static std::mutex mu;
  static const void* keys[256];
  static size_t vals[256];
  static int devs[256];
  static int used = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  for (int i = 0; i < used; ++i)
    if (keys[i] == fn && devs[i] == dev) {
      if (vals[i] >= smem) return;
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      vals[i] = smem;
      return;
    }
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (used < 256) { keys[used] = fn; devs[used] = dev; vals[used] = smem; ++used; }
}

static int team_for_chi(int chi) { return chi <= 8 ? 32 : (chi == 16 ? 128 : TQ_TEAM32); }
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
  const bool fused = chi <= 8 && D <= 4 && (!lr || mode == 0);   // kernels: FUSE && D <= FDM
  const bool wbr = chi >= 16 && D <= 4 && (!lr || mode == 0);     // kernels: WBR (matrix bracket, chi >= 16)
  L.direct = (lr && mode == 0 && fused && team == 32 && c->max_pairs <= 32 && c->max_ops <= 12) ? 1 : 0;
  L.a = (int32_t)off; off += 2 * ms;
  L.ah = L.a;                                        // conjugate transposes are read in place
  L.env = (int32_t)off; off += (size_t)D * ms;       // RL: P in/out; LR: Lambda
  L.m = (int32_t)off; off += (size_t)(fused ? (lr && !L.direct ? 2 : 0) : 2 * D) * ms;   // RL: N; LR: M (G aliases)
  L.br = (int32_t)off; off += (size_t)2 * D * ms;
  L.pin = (int32_t)off;
  if (lr) off += (size_t)D * ms;                      // direct path: P dense, prefetched
  L.lrpf = (lr && mode == 0 && chi >= 16) ? 1 : 0;
  L.rlpre = (!lr && mode == 0 && chi >= 16 && team >= 128) ? 1 : 0;
  L.a2 = (int32_t)off;
  if (L.direct || L.lrpf || L.rlpre) off += 2 * ms;
  off = align_up(off, 16);
  L.wc = (int32_t)off;
  if (fused || wbr) { const int dm = D <= 3 ? 3 : 4; off += align_up((size_t)dm * dm * 4 * csz + 16, 16); }
  L.mr = (int32_t)off;
  if (lr && mode == 1) off += (size_t)2 * D * ms;
  // digit tree (gradient sweep, chi >= 16): per-warp contribution partials; adjoint
  // ping-pong buffers in the M slots after G (free during the adjoint); levels dedicated
  // when they fit (then the fold builds them and the adjoint reuses them), else in scratch.
  const int ntr = c->max_train > 0 ? c->max_train : 1;
  const bool want_tree = false;   // the column adjoint lives in adj_sweep
  size_t need = (lr && mode == 1) ? (size_t)8 * D * team * rsz : 0;
  if (need <= (size_t)2 * D * ms && !want_tree) L.contrib = L.br;
  else { L.contrib = (int32_t)off; off += align_up(need, 16); }
  off = align_up(off, 16);
  L.mres = (int32_t)off; off += (size_t)c->max_lmat * 4 * csz;
  off = align_up(off, 16);
  L.minfo = (int32_t)off; off += align_up((size_t)c->max_lmat * 4, 16);
  L.mps = (int32_t)off; off += align_up((size_t)c->max_lmat * rsz, 16);
  L.ocode = (int32_t)off; off += align_up((size_t)(c->max_ops > 0 ? c->max_ops : 1) * 4, 16);
  L.ogidx = (int32_t)off; off += align_up((size_t)(c->max_ops > 0 ? c->max_ops : 1) * 4, 16);
  L.obase = (int32_t)off; off += align_up((size_t)(c->max_ops > 0 ? c->max_ops : 1) * 4, 16);
  L.sedge = (int32_t)off; off += align_up((size_t)(c->max_edges > 0 ? c->max_edges : 1) * (rsz == 8 ? 24 : 16), 16);
  off = align_up(off, 16);
  L.sbuf = (int32_t)off; off += 16 + sizeof(tq_site);
  L.dstride = (int32_t)(off - (size_t)L.mres);
  off += (size_t)L.dstride;                          // second resolved-descriptor buffer
  L.raw0 = (int32_t)off; off += (size_t)c->blob_max * 16;   // single blob landing buffer
  L.raw1 = L.raw0;
  const size_t lev_bytes = align_up((size_t)(c->max_tree > 0 ? c->max_tree : 1) * 2 * csz, 16);
  const size_t u_bytes = (size_t)2 * chi * chi * 2 * csz;
  const size_t m_free = (size_t)(L.br - L.m) > 2 * ms ? (size_t)(L.br - L.m) - 2 * ms : 0;  // M slots after G
  const size_t budget = (size_t)227 * 1024 / (team == 32 ? 4 : 1);
  L.tree = 0; L.lev = 0; L.ubuf = 0;
  if (want_tree) {
    (void)m_free; (void)budget;
    {
      const size_t avail = (size_t)(L.br - L.m) + (size_t)2 * D * ms - 2 * ms;
      if (lev_bytes + u_bytes <= avail) { L.tree = 2; L.lev = (int32_t)(L.m + 2 * ms); L.ubuf = (int32_t)(L.lev + lev_bytes); }
    }
  }
  L.team_bytes = (int32_t)align_up(off, 128);
  return L;
}

struct WsLayout { size_t env, epart, gpart, wct, wct_row, total; };

static WsLayout ws_layout(const tq_chain* c, int batch, int flags, int dtype) {
  const size_t rsz = dtype == TQ_C128 ? 8 : 4;
  WsLayout w{};
  size_t off = 0;
  w.env = off;
  if (flags & (TQ_FLAG_GRAD | TQ_FLAG_VALUES)) off += align_up((size_t)batch * c->env_total * 2 * rsz, 256);
  w.epart = off; off += align_up((size_t)batch * c->n_segments * 2 * rsz, 256);
  w.gpart = off;
  if (flags & TQ_FLAG_GRAD) off += align_up((size_t)batch * (c->n_gslots > 0 ? c->n_gslots : 1) * rsz, 256);
  w.wct_row = align_up((size_t)(4 * 16 + 1) * 2 * rsz, 16);   // up to 4 channels
  w.wct = off;
  if (!(flags & TQ_FLAG_VALUES)) off += align_up((size_t)(c->n_sites > 0 ? c->n_sites : 1) * 2 * w.wct_row, 256);
  w.total = off + 256;
  return w;
}

struct Timing { cudaEvent_t ev[6]; bool on; };
static thread_local Timing g_timing = {{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr}, false};

// Adjoint teams (launch_pair_f): a warp per (theta-set, site) up to chi = 8, 128 threads from
// chi = 16 (four units per SM at cfg4 with the compact digit tree).
static AdjLayout make_adj_layout(const tq_chain* c, int chi, int team, size_t rsz) {
  AdjLayout A{};
  const size_t csz = 2 * rsz;
  const size_t ms = (size_t)(chi + 1) * (chi + 1) * csz;
  size_t off = 0;
  auto take = [&](size_t bytes) { const int32_t o = (int32_t)off; off = align_up(off + bytes, 16); return o; };
  A.mres = take((size_t)c->max_lmat * 4 * csz);
  A.minfo = take((size_t)c->max_lmat * 4);
  A.mps = take((size_t)c->max_lmat * rsz);
  const size_t nops = (size_t)(c->max_ops > 0 ? c->max_ops : 1);
  A.ocode = take(nops * 4); A.ogidx = take(nops * 4); A.obase = take(nops * 4);
  A.sbuf = take(16 + sizeof(tq_site));
  A.raw = take((size_t)c->blob_max * 16);
  const int ntr = c->max_train > 0 ? c->max_train : 1;
  const size_t budget = (size_t)227 * 1024 / (team == 32 ? 4 : 1);
  A.tree = 0;
  A.ubuf_vec = chi * chi;
  if (chi >= 16) {
    // compact digit tree: kept (trainable) levels + one buffer of chi^2 2-vectors (forward
    // scratch, then U; both walks run in place) + the gather's leaf tables; G is read from HBM,
    // so no G slab
    const int kept = c->max_ttree > 0 ? c->max_ttree : (c->max_tree > 0 ? c->max_tree : 1);
    const size_t lev = (size_t)kept * 2 * csz;
    const size_t ub = (size_t)A.ubuf_vec * 2 * csz;
    const size_t tab = (size_t)2 * chi * 4;
    const size_t ctb = (size_t)ntr * (team / 32) * rsz;
    if (align_up(off + lev + ub + tab + ctb + 96, 128) <= budget) {
      A.tree = 1; A.lev = take(lev); A.ubuf = take(ub); A.utab = take(tab); A.contrib = take(ctb);
    }
  }
  if (!A.tree) { A.g = take(2 * ms); A.contrib = take((size_t)ntr * team * rsz); }
  A.team_bytes = (int32_t)align_up(off, 128);
  return A;
}

template <typename R, int CHI, int FUSED>
static tq_status launch_pair_f(Params& prm, bool run_lr, cudaStream_t s) {
  constexpr int TEAM = CHI <= 8 ? 32 : (CHI == 16 ? 128 : TQ_TEAM32);
  constexpr int TEAMS = TEAM == 32 ? 4 : 1;
  const int items = prm.batch * prm.c.n_segments;
  const int grid = (items + TEAMS - 1) / TEAMS;
  {
    Params q = prm;
    q.L = make_layout(&prm.c, CHI, TEAM, sizeof(R), false, prm.mode);
    const size_t smem = (size_t)q.L.team_bytes * TEAMS;
    if (smem > 227 * 1024) return fail(TQ_ERR_UNSUPPORTED, "shared-memory layout exceeds 227 KB (too many MPO channels for this bond dimension)");
    if (g_timing.on) cudaEventRecord(g_timing.ev[0], s);
    if (sizeof(R) == 4 && prm.c.real_path && prm.mode == 0) {
      set_smem_attr(reinterpret_cast<const void*>(rl_sweep<R, CHI, TEAM, FUSED, sizeof(R) == 4>), smem);
      rl_sweep<R, CHI, TEAM, FUSED, sizeof(R) == 4><<<grid, TEAM * TEAMS, smem, s>>>(q);
    } else {
      set_smem_attr(reinterpret_cast<const void*>(rl_sweep<R, CHI, TEAM, FUSED>), smem);
      rl_sweep<R, CHI, TEAM, FUSED><<<grid, TEAM * TEAMS, smem, s>>>(q);
    }
    if (g_timing.on) cudaEventRecord(g_timing.ev[1], s);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(TQ_ERR_CUDA, cudaGetErrorString(e));
  }
  if (run_lr) {
    Params q = prm;
    q.L = make_layout(&prm.c, CHI, TEAM, sizeof(R), true, prm.mode);
    const size_t smem = (size_t)q.L.team_bytes * TEAMS;
    if (smem > 227 * 1024) return fail(TQ_ERR_UNSUPPORTED, "shared-memory layout exceeds 227 KB (too many MPO channels for this bond dimension)");
    if (g_timing.on) cudaEventRecord(g_timing.ev[2], s);
    if (prm.mode == 0 && sizeof(R) == 4 && prm.c.real_path) {
      set_smem_attr(reinterpret_cast<const void*>(lr_sweep<R, CHI, TEAM, 0, FUSED, sizeof(R) == 4>), smem);
      lr_sweep<R, CHI, TEAM, 0, FUSED, sizeof(R) == 4><<<grid, TEAM * TEAMS, smem, s>>>(q);
    } else if (prm.mode == 0) {
      set_smem_attr(reinterpret_cast<const void*>(lr_sweep<R, CHI, TEAM, 0, FUSED>), smem);
      lr_sweep<R, CHI, TEAM, 0, FUSED><<<grid, TEAM * TEAMS, smem, s>>>(q);
    } else {
      set_smem_attr(reinterpret_cast<const void*>(lr_sweep<R, CHI, TEAM, 1, 0>), smem);
      lr_sweep<R, CHI, TEAM, 1, 0><<<grid, TEAM * TEAMS, smem, s>>>(q);
    }
    if (g_timing.on) cudaEventRecord(g_timing.ev[3], s);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(TQ_ERR_CUDA, cudaGetErrorString(e));
    if (prm.mode == 0) {
      constexpr int ATEAM = CHI <= 8 ? 32 : 128;   // adj_team_for_chi
      constexpr int ATEAMS = ATEAM == 32 ? 4 : 1;
      AdjLayout A = make_adj_layout(&prm.c, CHI, ATEAM, sizeof(R));
      const size_t asmem = (size_t)A.team_bytes * ATEAMS;
      if (asmem > 227 * 1024) return fail(TQ_ERR_UNSUPPORTED, "adjoint shared-memory layout exceeds 227 KB");
      const int64_t units = (int64_t)prm.batch * prm.c.n_sites;
      const unsigned agrid = (unsigned)((units + ATEAMS - 1) / ATEAMS);
      if (g_timing.on) cudaEventRecord(g_timing.ev[4], s);
      if (sizeof(R) == 4 && prm.c.real_path && A.tree) {
        set_smem_attr(reinterpret_cast<const void*>(adj_sweep<R, CHI, ATEAM, sizeof(R) == 4>), asmem);
        adj_sweep<R, CHI, ATEAM, sizeof(R) == 4><<<agrid, ATEAM * ATEAMS, asmem, s>>>(prm, A);
      } else {
        set_smem_attr(reinterpret_cast<const void*>(adj_sweep<R, CHI, ATEAM>), asmem);
        adj_sweep<R, CHI, ATEAM><<<agrid, ATEAM * ATEAMS, asmem, s>>>(prm, A);
      }
      if (g_timing.on) cudaEventRecord(g_timing.ev[5], s);
      e = cudaGetLastError();
      if (e != cudaSuccess) return fail(TQ_ERR_CUDA, cudaGetErrorString(e));
    }
  }
  return TQ_OK;
}

// The register-fused product+bracket path needs chi <= 8 and at most 4 MPO channels (the
// shared-memory layout in make_layout makes the same decision).
template <typename R, int CHI>
static tq_status launch_pair(Params& prm, bool run_lr, cudaStream_t s) {
  // chi <= 8: register-fused product + bracket.  chi >= 16: the fused stages were measured
  // slower than GEMM + bracket (profiles/r01_stages_cfg4.txt); the GEMMs stay unfused and the
  // bracket uses the same channel-pair matrices (wbracket_stage)
  if (prm.c.d_max <= 3) return launch_pair_f<R, CHI, 3>(prm, run_lr, s);
  if (prm.c.d_max <= 4) return launch_pair_f<R, CHI, 4>(prm, run_lr, s);
  return launch_pair_f<R, CHI, 0>(prm, run_lr, s);
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
      if constexpr (sizeof(R) == 8) return fail(TQ_ERR_UNSUPPORTED, "complex128 mode supports bond dimension <= 16");
      else return launch_pair<R, 32>(prm, run_lr, s);
    default: return fail(TQ_ERR_UNSUPPORTED, "bond dimension exceeds 32");
  }
}

static tq_status check_chain(const tq_chain* c, int batch) {
  if (!c) return fail(TQ_ERR_INPUT, "null chain");
  if (!c->blob || !c->blob_off) return fail(TQ_ERR_INPUT, "chain has no descriptor blobs");
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
  prm.wct = nullptr; prm.wct_row = (int32_t)w.wct_row;
  if (batch == 0) return TQ_OK;
  // one coefficient row for the whole batch + fused small-chi sweeps: build the bracket
  // matrices once per launch instead of once per (theta-set, site)
  if (cs == 0 && coef != nullptr && c->n_sites > 0 && c->d_max <= 4) {
    prm.wct = wb + w.wct;
    if (c->d_max <= 3) build_wct<R, 3><<<c->n_sites, 64, 0, s>>>(prm);
    else build_wct<R, 4><<<c->n_sites, 64, 0, s>>>(prm);
  }
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
  prm.wct = nullptr; prm.wct_row = 0;
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


template <typename R, int CHI>
static tq_status launch_inner(InnerParams& ip, cudaStream_t s) {
  constexpr int TEAM = CHI <= 8 ? 32 : (CHI == 16 ? 128 : TQ_TEAM32);
  constexpr int TEAMS = TEAM == 32 ? 4 : 1;
  const size_t csz = 2 * sizeof(R), ms = (size_t)(CHI + 1) * (CHI + 1) * csz;
  size_t off = 0;
  auto take = [&](size_t bytes) { const int32_t o = (int32_t)off; off = align_up(off + bytes, 16); return o; };
  ip.off_ak = take(2 * ms); ip.off_ab = take(2 * ms); ip.off_ahk = ip.off_ak; ip.off_ahb = ip.off_ab;
  ip.off_t = take(2 * ms); ip.off_l = take(ms);
  ip.off_mk = take((size_t)ip.ket.max_lmat * 4 * csz); ip.off_ik = take((size_t)ip.ket.max_lmat * 4);
  ip.off_pk = take((size_t)ip.ket.max_lmat * sizeof(R)); ip.off_ok = take((size_t)(ip.ket.max_ops + 1) * 4);
  ip.off_gk = take((size_t)(ip.ket.max_ops + 1) * 4);
  ip.off_qk = take((size_t)(ip.ket.max_ops + 1) * 4);
  ip.off_mb = take((size_t)ip.bra.max_lmat * 4 * csz); ip.off_ib = take((size_t)ip.bra.max_lmat * 4);
  ip.off_pb = take((size_t)ip.bra.max_lmat * sizeof(R)); ip.off_ob = take((size_t)(ip.bra.max_ops + 1) * 4);
  ip.off_gb = take((size_t)(ip.bra.max_ops + 1) * 4);
  ip.off_qb = take((size_t)(ip.bra.max_ops + 1) * 4);
  ip.team_bytes = (int32_t)align_up(off, 128);
  const size_t smem = (size_t)ip.team_bytes * TEAMS;
  if (smem > 227 * 1024) return fail(TQ_ERR_UNSUPPORTED, "inner product layout exceeds shared memory");
  set_smem_attr(reinterpret_cast<const void*>(inner_sweep<R, CHI, TEAM>), smem);
  inner_sweep<R, CHI, TEAM><<<(ip.batch + TEAMS - 1) / TEAMS, TEAM * TEAMS, smem, s>>>(ip);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(TQ_ERR_CUDA, cudaGetErrorString(e));
  return TQ_OK;
}

template <typename R>
static tq_status inner_impl(InnerParams& ip, cudaStream_t s) {
  const int chi = chi_bucket(ip.ket.chi_max > ip.bra.chi_max ? ip.ket.chi_max : ip.bra.chi_max);
  switch (chi) {
    case 2: return launch_inner<R, 2>(ip, s);
    case 4: return launch_inner<R, 4>(ip, s);
    case 8: return launch_inner<R, 8>(ip, s);
    case 16: return launch_inner<R, 16>(ip, s);
    case 32:
      if constexpr (sizeof(R) == 8) return fail(TQ_ERR_UNSUPPORTED, "complex128 mode supports bond dimension <= 16");
      else return launch_inner<R, 32>(ip, s);
    default: return fail(TQ_ERR_UNSUPPORTED, "bond dimension exceeds 32");
  }
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
  if (chain->blob_dtype != dtype) return fail(TQ_ERR_INPUT, "chain blobs were packed for a different dtype");
  if (dtype == TQ_C64) return energy_grad_impl<float>(chain, batch, theta, theta_stride, coef, coef_stride, energy, grad, workspace, workspace_bytes, s);
  if (dtype == TQ_C128) return energy_grad_impl<double>(chain, batch, theta, theta_stride, coef, coef_stride, energy, grad, workspace, workspace_bytes, s);
  return fail(TQ_ERR_INPUT, "unknown dtype");
}

tq_status tq_term_values(const tq_chain* chain, int32_t dtype, int32_t batch, const void* theta, int64_t theta_stride,
                         double* values, void* workspace, size_t workspace_bytes, void* stream) {
  tq_status st = check_chain(chain, batch);
  if (st != TQ_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (chain->blob_dtype != dtype) return fail(TQ_ERR_INPUT, "chain blobs were packed for a different dtype");
  if (dtype == TQ_C64) return values_impl<float>(chain, batch, theta, theta_stride, values, workspace, workspace_bytes, s);
  if (dtype == TQ_C128) return values_impl<double>(chain, batch, theta, theta_stride, values, workspace, workspace_bytes, s);
  return fail(TQ_ERR_INPUT, "unknown dtype");
}

tq_status tq_energy_grad_timed(const tq_chain* chain, int32_t dtype, int32_t batch, const void* theta,
                               int64_t theta_stride, const void* coef, int64_t coef_stride, double* energy, void* grad,
                               void* workspace, size_t workspace_bytes, void* stream, float* ms_out) {
  for (int i = 0; i < 6; ++i) cudaEventCreate(&g_timing.ev[i]);
  g_timing.on = true;
  tq_status st = tq_energy_grad(chain, dtype, batch, theta, theta_stride, coef, coef_stride, energy, grad, workspace,
                                workspace_bytes, stream);
  g_timing.on = false;
  if (st == TQ_OK) {
    cudaEventSynchronize(g_timing.ev[grad ? 5 : 1]);
    float a = 0.f, b = 0.f, c2 = 0.f;
    cudaEventElapsedTime(&a, g_timing.ev[0], g_timing.ev[1]);
    if (grad) { cudaEventElapsedTime(&b, g_timing.ev[2], g_timing.ev[3]); cudaEventElapsedTime(&c2, g_timing.ev[4], g_timing.ev[5]); }
    ms_out[0] = a; ms_out[1] = b; ms_out[2] = c2;
  }
  for (int i = 0; i < 6; ++i) cudaEventDestroy(g_timing.ev[i]);
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

tq_status tq_inner(const tq_chain* bra, const void* theta_bra, int64_t bra_stride, const tq_chain* ket,
                   const void* theta_ket, int64_t ket_stride, int32_t dtype, int32_t batch, double* out, void* stream) {
  if (!bra || !ket) return fail(TQ_ERR_INPUT, "null chain");
  if (bra->n_segments != 1 || ket->n_segments != 1) return fail(TQ_ERR_INPUT, "inner product chains must have one segment");
  if (batch <= 0) return TQ_OK;
  InnerParams ip{};
  ip.ket = *ket; ip.bra = *bra; ip.batch = batch;
  ip.theta_ket = theta_ket; ip.ket_stride = ket_stride; ip.theta_bra = theta_bra; ip.bra_stride = bra_stride; ip.out = out;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (dtype == TQ_C64) return inner_impl<float>(ip, s);
  if (dtype == TQ_C128) return inner_impl<double>(ip, s);
  return fail(TQ_ERR_INPUT, "unknown dtype");
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

#ifdef TQ_STAGE_TIMING
int32_t tq_stage_cycles(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, tq::g_stage_cycles, sizeof(unsigned long long) * 32);
  unsigned long long z[32] = {0};
  cudaMemcpyToSymbol(tq::g_stage_cycles, z, sizeof(z));
  return 32;
}
#endif

const char* tq_build_info(void) {
  return "tq_engine sm_100a: rl_sweep/lr_sweep<float|double, chi 2..32>, adj_sweep, reduce_energy, reduce_grad, inner_sweep, ffma_probe";
}

}  // extern "C"
