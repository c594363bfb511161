/*
 * tq_engine.h — C ABI of the B200 TT-circuit expectation/gradient engine.
 *
 * This is the drop-in boundary for the reference's contraction engine.  The
 * reference (tnsim, pure Python) has no FFI; its only engine seam is the string
 * engine in {"dense","tt"} (autodiff.py:456-459) dispatched at
 * taped_expectations (autodiff.py:421-425), _taped_expval_output
 * (autodiff.py:430-435), evaluate_expval (autodiff.py:500-503) and expval
 * (hamiltonians.py:173-182).  Everything below that seam is replaced:
 *
 *   tq_energy_grad  replaces  grad_expval(engine="tt", eps=0)      autodiff.py:471-487
 *                             (tape build _tt_taped_state autodiff.py:339-363,
 *                              _tt_term_nodes autodiff.py:366-402,
 *                              GradTape.backward autodiff.py:190-247)
 *                   and, with grad == NULL,
 *                             evaluate_expval(engine="tt")         autodiff.py:490-503
 *                             (simulate_tt tt.py:237-244, _expval_tt hamiltonians.py:129-164)
 *   tq_term_values  replaces  taped_expectations(engine="tt")      autodiff.py:405-425
 *                             (the per-readout values vertex_expectations maxcut.py:206-216 uses)
 *   tq_inner        replaces  tt_inner                             tt.py:247-255
 *
 * All arrays are caller-owned device memory (the library never allocates);
 * the chain tables are built by the host compiler (paper_2112_10239_b200/chain.py)
 * and uploaded by the caller.  Calls are reentrant, run on the caller's stream and
 * are deterministic (no float atomics, fixed-order reductions).  The only process-wide
 * state is a mutex-protected cache of each kernel's opened dynamic-shared-memory
 * limit (it only grows, so it never changes a result; it saves a
 * cudaFuncSetAttribute per launch) and the last error message (thread_local).
 *
 * dtype: TQ_C64 -> theta/coef/grad are float32, TQ_C128 -> float64.
 * energy / values outputs are always float64 (re, im) pairs.
 */
#ifndef TQ_ENGINE_H
#define TQ_ENGINE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t tq_status;
#define TQ_OK 0
#define TQ_ERR_INPUT 1        /* maps to InputError (CLI exit 2) */
#define TQ_ERR_UNSUPPORTED 2  /* maps to BondTooLarge / InputError */
#define TQ_ERR_CUDA 3         /* maps to EngineError (NumericalError, exit 1) */
#define TQ_ERR_WORKSPACE 4    /* workspace too small: InputError */

#define TQ_C64 0
#define TQ_C128 1

#define TQ_FLAG_GRAD 1        /* workspace for the gradient sweeps */
#define TQ_FLAG_VALUES 2      /* workspace for per-term values */

/* One site of a sub-chain (chain.py SITE_DTYPE). */
typedef struct {
  int32_t op_begin, op_count, lmat_count, chi_l, chi_r;
  int32_t pass_begin, pass_count;
  int32_t rl_edge_begin, rl_edge_count, lr_edge_begin, lr_edge_count;
  int32_t fin_begin, fin_count;
  int32_t rl_da, rl_db, lr_da, lr_db;
  int32_t n_train, ent_begin; /* ent_begin: first of this site's contiguous tq_mat entries */
  int64_t env_in, env_out;  /* complex offsets of the stored right envs at cut k+1 / cut k (-1: none) */
  double init[4];           /* input product-state vector of this qubit (re,im,re,im) */
  int64_t a_off;            /* complex offset of the folded core A[2][chi_l][chi_r] (RL stores, LR reloads) */
  int64_t g_off;            /* complex offset of the core cotangent G[2][chi_l][chi_r] (LR stores, adjoint reads) */
} tq_site;

/* One operator of a column: selects table entry mat + digit (chain.py OP_DTYPE).
 * toff: digit bits introduced by earlier ops of the column (digit-tree level width),
 * tbase: entries held by the earlier levels of the column's digit tree. */
typedef struct {
  int32_t mat, lmat, src, shift, bits, tidx, gidx, toff, tbase, pad;
} tq_op;

/* 2x2 factor table entry (chain.py MAT_DTYPE): kind 0 const, 1 rx, 2 ry, 3 rz. */
typedef struct {
  int32_t kind, slot, cls, pad;
  double angle, pscale;
  double m[8];
} tq_mat;

/* MPO transfer edge a -> b with Pauli op (0 I,1 X,2 Y,3 Z); coef < 0 means 1.
 * Finalisation edges reuse the struct with b = term index. */
typedef struct {
  int32_t a, b, op, coef;
} tq_edge;

typedef struct {
  int32_t sa, sb, bits, pad;
} tq_pass;

typedef struct {
  int32_t site_begin, site_count, gslot_begin, gslot_count, lo, hi;
  int64_t env_base, env_elems;
} tq_segment;

/* Compiled chain: sizes + device pointers to the tables above. */
typedef struct {
  int32_t n_segments, n_sites, n_params, n_terms;
  int32_t chi_max, d_max, max_ops, max_lmat, max_train, n_gslots;
  int32_t max_edges, max_tree; /* max_tree: largest digit tree (entries) of any column */
  int64_t env_total; /* complex elements of stored envs per theta-set */
  double e_const_re, e_const_im; /* identity-term coefficients */
  const tq_site* sites;
  const tq_op* ops;
  const tq_mat* mats;
  const tq_edge* edges;
  const tq_edge* fins;
  const tq_pass* passes;
  const tq_segment* segs;
  const int32_t* gred_ptr;
  const int32_t* gred_idx;
  const int32_t* term_active; /* [n_terms] 0 for identity terms (value 1) */
  /* Per-site descriptor blobs (16-byte units), prefetched with cp.async one site ahead:
   * [header {len, next_rl, next_lr, segment}] [tq_site: 9 units] [ops: {opcode, gidx, tbase, tidx}]
   * [factor entries: complex64 3 units / complex128 6 units] [rl edges] [lr edges]. */
  const void* blob;
  const int32_t* blob_off;    /* [n_sites] offset of each site's blob (16-byte units) */
  int32_t blob_max, blob_dtype; /* largest blob (units); dtype the entries were packed for */
  int32_t max_pairs;            /* largest chi_l*chi_r of any site */
  int32_t max_ttree;            /* largest sum of trainable-op digit-tree levels (entries) of any column;
                                   0 = unknown (the adjoint then sizes its kept levels by max_tree) */
  int32_t real_path;            /* 1: every factor matrix, input vector and MPO edge is real (ry
                                   rotations, real constant factors, Paulis I/X/Z): the complex64
                                   chi >= 16 energy sweeps then accumulate real parts only (their
                                   imaginary parts are exact zeros; results bit-identical) */
  int32_t reserved;
} tq_chain;

/* Bytes of device workspace one call needs. */
size_t tq_workspace_bytes(const tq_chain* chain, int32_t batch, int32_t flags, int32_t dtype);

/* E_b = sum_t coef[b,t] <psi(theta_b)|P_t|psi(theta_b)> (+ e_const) and, if grad != NULL,
 * grad[b,:] = dRe(E_b)/dtheta_b.  theta: [B, n_params] (row stride theta_stride elements);
 * coef: [B or 1, n_terms] real (row stride coef_stride, 0 = shared); energy: [B,2] float64.
 * energy and grad are written once, coalesced, by the final reduction kernels: they may be
 * device memory or pinned host memory (cudaHostAlloc; the same pointer under UVA), which
 * returns the results to the host without a separate copy. */
tq_status tq_energy_grad(const tq_chain* chain, int32_t dtype, int32_t batch,
                         const void* theta, int64_t theta_stride,
                         const void* coef, int64_t coef_stride,
                         double* energy, void* grad,
                         void* workspace, size_t workspace_bytes, void* stream);

/* values[b,t] = <psi(theta_b)|P_t|psi(theta_b)> for every term (chain compiled in values mode). */
tq_status tq_term_values(const tq_chain* chain, int32_t dtype, int32_t batch,
                         const void* theta, int64_t theta_stride, double* values,
                         void* workspace, size_t workspace_bytes, void* stream);

/* out[b] = <bra(theta_bra_b)|ket(theta_ket_b)>, first argument conjugated (tt_inner).
 * Both chains must be compiled with segments=1 over the same qubits (values mode, no terms). */
tq_status tq_inner(const tq_chain* bra, const void* theta_bra, int64_t bra_stride,
                   const tq_chain* ket, const void* theta_ket, int64_t ket_stride,
                   int32_t dtype, int32_t batch, double* out, void* stream);

/* tq_energy_grad with CUDA events around the kernels on `stream` (synchronises);
 * ms_out[0] = right-to-left sweep, ms_out[1] = left-to-right sweep, ms_out[2] = column
 * adjoint (adj_sweep).  Bench/diagnostic. */
tq_status tq_energy_grad_timed(const tq_chain* chain, int32_t dtype, int32_t batch,
                               const void* theta, int64_t theta_stride,
                               const void* coef, int64_t coef_stride,
                               double* energy, void* grad,
                               void* workspace, size_t workspace_bytes, void* stream, float* ms_out);

/* FP32 FFMA throughput probe (TFLOP/s): the SIMT roofline denominator. */
tq_status tq_ffma_peak(int32_t iters, void* stream, double* tflops_out);

const char* tq_status_string(tq_status status);
/* Message of the last failing call on this host thread. */
const char* tq_last_error(void);
/* Writes sizeof of the 7 structs (site, op, mat, edge, pass, segment, chain) into sizes[0..6]. */
int32_t tq_abi_layout(int32_t* sizes, int32_t n);
/* Kernel variants compiled into this library (for the driver's evidence). */
const char* tq_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* TQ_ENGINE_H */
